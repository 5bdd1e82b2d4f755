"""Helpers shared by the -m gpu parity tests: run a generated record through librx (the
CUDA path, via the C ABI) and through the oracle, and compare them."""
from __future__ import annotations

import math

import numpy as np

from oracle import rx_oracle as O

RX_FIELDS = ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu", "train_symbols",
             "sync_start", "sync_window", "warmup_symbols", "cpr_test_phases", "tap_lag_epochs",
             "sync_min_corr", "buffer_blocks", "clock_avg_half", "cfo_enable", "lms_batch_segments",
             "input_format", "widely_linear", "q_window_symbols", "cpr_anchor", "lms_mode",
             "fused_front_end")


def oracle_params(rec, rx) -> O.RxParams:
    kw = {k: v for k, v in rx.items() if k in O.RxParams.__dataclass_fields__}
    return O.RxParams(fmt=rec.fmt, M=rec.M, static_taps=rec.static_taps,
                      dc_offset=rec.dc_offset, **kw)


def run_oracle(rec, rx):
    p = oracle_params(rec, rx)
    return O.receive_pam(rec.codes, p) if rec.fmt == "pam" else O.receive_kk(rec.codes, p)


def run_gpu(rec, rx, chunk=1 << 22, history_buffers=None, device=0, keep=True, pre=None):
    """Stream the record through librx in `chunk`-sample calls, flush, return (Receiver,
    labels numpy, stats). rx["input_format"] = 1 streams x = (code - 2047.5)/2047.5 as float32;
    ``pre(R)`` runs before the first call (e.g. rx_set_taps)."""
    import torch
    from paper_2011_13695_b200 import RX_PAM, RX_QAM_KK, Receiver
    fam = RX_PAM if rec.fmt == "pam" else RX_QAM_KK
    fields = {k: v for k, v in rx.items() if k in RX_FIELDS}
    bb = fields.get("buffer_blocks", 8192)
    if history_buffers is None:
        history_buffers = max(3, -(-rec.n // (bb * 512)) + 2)
    fields["history_buffers"] = history_buffers
    if fam == RX_QAM_KK:
        fields["dc_offset"] = rec.dc_offset
    R = Receiver(fam, rec.M, rec.static_taps, device=device, **fields)
    packed = fields.get("input_format", 0) == 2
    if fields.get("input_format", 0) == 1:
        x = ((rec.codes.astype(np.float64) - 2047.5) / 2047.5).astype(np.float32)
        codes = torch.from_numpy(x).to(f"cuda:{device}")
    elif packed:                          # RX_IN_U12_PACKED: 3 bytes per 2 codes
        from rxsynth.gen import pack_u12
        codes = torch.from_numpy(pack_u12(rec.codes)).to(f"cuda:{device}")
    else:
        codes = torch.from_numpy(rec.codes.view(np.int16)).to(f"cuda:{device}")
    if pre is not None:
        pre(R)
    nsym_ub = rec.n // (2 if fam == RX_PAM else 4) + 4096
    labels = torch.full((nsym_ub,), 0xFF, dtype=torch.uint8, device=f"cuda:{device}")
    for off in range(0, rec.n, chunk):
        if packed:
            R.process(codes[off * 3 // 2:(off + chunk) * 3 // 2], labels)
        else:
            R.process(codes[off:off + chunk], labels)
    R.flush(labels)
    st = R.stats()
    return R, labels.cpu().numpy(), st


def rel_l2(a, b) -> float:
    a = np.asarray(a); b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def near_threshold(soft, fmt, M, delta):
    """Distance of each oracle soft value (segment frame z') to the nearest decision boundary
    is < delta (per axis for QAM)."""
    if fmt == "pam":
        t = O.midpoints(O.pam_levels(M))
        return np.min(np.abs(np.real(soft)[:, None] - t[None, :]), axis=1) < delta
    ax = O.qam_axis(M)
    t = O.midpoints(ax)
    dI = np.min(np.abs(soft.real[:, None] - t[None, :]), axis=1)
    dQ = np.min(np.abs(soft.imag[:, None] - t[None, :]), axis=1)
    return np.minimum(dI, dQ) < delta


def evm_db(num, den):
    return 10 * math.log10(num / den)
