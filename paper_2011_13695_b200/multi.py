"""Multi-GPU plumbing (host side): independent channels sharded over ranks, one packed
all-reduce of the BER/EVM counters per round (BASELINE.json config 5:
"64 independent mixed PAM/KK-QAM channels sharded over 8xB200, NCCL allreduce of BER/EVM
counters").

The receive chain itself never crosses GPUs: each channel is one librx handle on one device,
so there is no data-path collective. torch.distributed (NCCL on GPUs, gloo in the CPU tests)
carries only the tiny counter vector.
"""
from __future__ import annotations

import math

from .rx import COUNTERS, NCOUNTERS  # noqa: F401

# counter slots (rx_export_counters order)
IDX = {name: i for i, name in enumerate(COUNTERS)}


def channel_shard(n_channels: int, world: int, rank: int) -> list[int]:
    """Contiguous block of channels owned by `rank` (every channel exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = n_channels * rank // world
    hi = n_channels * (rank + 1) // world
    return list(range(lo, hi))


def allreduce_counters(t, group=None):
    """Sum a packed counter tensor [..., NCOUNTERS] (float64) over all ranks in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def q_db_from_ber(ber: float) -> float:
    """Q = 20 log10(sqrt(2) erfcinv(2 BER)) (Q estimated from the BER)."""
    import torch
    if not (0.0 < ber < 0.5):
        return float("inf") if ber == 0.0 else float("nan")
    x = torch.special.erfinv(torch.tensor(1.0 - 2.0 * ber, dtype=torch.float64))
    return 20.0 * math.log10(math.sqrt(2.0) * float(x))


def summarize(counters) -> dict:
    """Host summary of a (reduced) counter vector: BER, Q, EVM."""
    c = [float(v) for v in counters]
    bits = c[IDX["bits"]]
    ber = c[IDX["bit_errors"]] / bits if bits > 0 else float("nan")
    evm = 10.0 * math.log10(c[IDX["evm_num"]] / c[IDX["evm_den"]]) if c[IDX["evm_den"]] > 0 else float("nan")
    return {"bit_errors": int(c[IDX["bit_errors"]]), "bits": int(bits), "ber": ber,
            "q_db": q_db_from_ber(ber) if bits > 0 else float("nan"), "evm_db": evm,
            "symbols": int(c[IDX["symbols_counted"]]), "clipped": int(c[IDX["clipped"]]),
            "domain_errors": int(c[IDX["domain_errors"]])}


# ---------------------------------------------------------------------------- time sharding
def gather_carry(rec, group=None):
    """All-gather the shards' carry records (uint8 CUDA tensor of rx_carry_size bytes each) in
    rank order into one device buffer (NCCL all-gather; gloo on a shared GPU in the tests)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(world * rec.numel(), dtype=rec.dtype, device=rec.device)
    try:
        dist.all_gather_into_tensor(out, rec, group=group)
    except (RuntimeError, NotImplementedError, AttributeError):
        parts = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(parts, rec, group=group)
        out = torch.cat(parts)
    return out


def shard_inputs(n_samples: int, buffer_samples: int, beta: int, pre: int, post: int):
    """Input range [p0, p1) of paper buffer beta for its shard (include/rx.h rx_shard_process)
    and whether it holds the stream end."""
    p0 = max(0, beta * buffer_samples - pre)
    p1 = min(n_samples, (beta + 1) * buffer_samples + post)
    return p0, p1, p1 >= n_samples


def run_time_sharded(R, codes, buffer_samples: int, labels, rank: int, world: int, gather=None,
                     stream=None):
    """SURVEY §8(e) mode 2 on one rank: this rank's handle R (shard_count = world, shard_index =
    rank) processes paper buffers rank, rank + world, ... of the stream `codes` (a device tensor
    of u16 codes holding the whole stream here; a deployment would receive only its buffers with
    their halos, R.shard_halo()), exchanging one carry record per round, then one more exchange
    that finishes the pending buffers. gather(rec) -> all records (rank order); default:
    gather_carry over the default process group."""
    import torch
    gather = gather or gather_carry
    pre, post = R.shard_halo()
    n = codes.numel()
    nbuf = -(-n // buffer_samples)
    rec = torch.zeros(R.carry_size(), dtype=torch.uint8, device=codes.device)
    for r in range(-(-nbuf // world) + 1):
        b = r * world + rank
        if b < nbuf:
            p0, p1, last = shard_inputs(n, buffer_samples, b, pre, post)
            R.shard_process(b, codes[p0:p1], last=last, labels=labels, stream=stream)
        R.export_carry(rec, stream=stream)
        R.import_carry(gather(rec), world, rank, stream=stream)
