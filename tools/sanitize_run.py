"""Small configs through librx for compute-sanitizer (SURVEY §4 layer 5): a PAM record (C1) and a
KK record (C3 structure, 2^18 samples, 128-block buffers), streamed in several calls so the
history ring, the equaliser side stream and the flush all run.

  compute-sanitizer --tool memcheck  python tools/sanitize_run.py
  compute-sanitizer --tool racecheck python tools/sanitize_run.py
  compute-sanitizer --tool synccheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from rxsynth import make_config  # noqa: E402
from tests.gpu_util import run_gpu  # noqa: E402

rec, rx = make_config("C1")
rx.update(buffer_blocks=32)
_, _, st = run_gpu(rec, rx, chunk=512 * 32)
print("PAM", st["bit_errors"], st["bits"], st["status_flags"])
rec, rx = make_config("C3", n_samples=1 << 18)
rx.update(buffer_blocks=128, train_symbols=4096, warmup_symbols=8192)
_, _, st = run_gpu(rec, rx, chunk=512 * 128)
print("KK", st["bit_errors"], st["bits"], st["status_flags"])
# the other code paths: c-9 stitch chain, widely-linear taps, packed input, Q windows, calibrations
rec, rx = make_config("C3", n_samples=1 << 18)
rx.update(buffer_blocks=128, train_symbols=4096, warmup_symbols=8192, cpr_anchor=0, widely_linear=1)
_, _, st = run_gpu(rec, rx, chunk=512 * 128)
print("KK chain + WL", st["bit_errors"], st["bits"], st["status_flags"])
rec, rx = make_config("C1")
rx.update(buffer_blocks=32, input_format=2, q_window_symbols=4096)
R, _, st = run_gpu(rec, rx, chunk=512 * 32)
print("PAM packed", st["bit_errors"], st["bits"], R.q_trace(0, 4)[0].tolist())
print("thresholds", R.calibrate_thresholds(rx["train_symbols"] + 4096, 8192)[0].tolist())
# round-2 paths: BPS equaliser (C4 structure), data-aided and per-symbol DDLMS modes, time sharding
rec, rx = make_config("C4", n_samples=1 << 18)
rx.update(buffer_blocks=128, train_symbols=4096, warmup_symbols=8192)
_, _, st = run_gpu(rec, rx, chunk=512 * 128)
print("KK BPS", st["bit_errors"], st["bits"], st["status_flags"])
# round-2b: the fused KK front-end (k_kk_fe, E in shared memory) over ragged calls
rx.update(fused_front_end=1)
_, _, st = run_gpu(rec, rx, chunk=512 * 37)
print("KK fused front-end", st["bit_errors"], st["bits"], st["status_flags"])
for mode, extra in ((1, {}), (2, dict(lms_block=1, lms_taps=4, widely_linear=1))):
    rec, rx = make_config("C3", n_samples=1 << 18, linewidth_hz=1e3)
    rx.update(buffer_blocks=128, train_symbols=4096, warmup_symbols=8192, lms_mode=mode, **extra)
    _, _, st = run_gpu(rec, rx, chunk=512 * 128)
    print("KK lms_mode", mode, st["bit_errors"], st["bits"], st["status_flags"])
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2011_13695_b200 import RX_QAM_KK, Receiver, multi  # noqa: E402
rec, rx = make_config("C4", n_samples=6 * 128 * 512)
fields = {k: v for k, v in rx.items() if k in ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu",
                                               "cpr_test_phases", "sync_start", "sync_window")}
hs = [Receiver(RX_QAM_KK, rec.M, rec.static_taps, dc_offset=rec.dc_offset, history_buffers=4, buffer_blocks=128,
               train_symbols=4096, warmup_symbols=8192, shard_count=2, shard_index=g, **fields) for g in range(2)]
codes = torch.from_numpy(rec.codes.view(np.int16)).cuda()
labs = [torch.zeros(rec.n // 4 + 4096, dtype=torch.uint8, device="cuda") for _ in range(2)]
recs = [torch.zeros(hs[0].carry_size(), dtype=torch.uint8, device="cuda") for _ in range(2)]
nbuf = rec.n // (128 * 512)
for r in range(nbuf // 2 + 1):
    for g in range(2):
        b = 2 * r + g
        if b < nbuf:
            p0, p1, last = multi.shard_inputs(rec.n, 128 * 512, b, 4096, 4096)
            hs[g].shard_process(b, codes[p0:p1], last=last, labels=labs[g])
        hs[g].export_carry(recs[g])
    for g in range(2):
        hs[g].import_carry(torch.cat(recs), 2, g)
print("KK 2 shards", [h.stats()["bits"] for h in hs])
# PAM time shards (C2 structure, 2 shards, 8 buffers of 128 blocks, PB look-back + clock halos)
from paper_2011_13695_b200 import RX_PAM  # noqa: E402
rec, rx = make_config("C2", n_samples=8 * 128 * 512)
fields = {k: v for k, v in rx.items() if k in ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu",
                                               "sync_start", "sync_window")}
hs = [Receiver(RX_PAM, rec.M, rec.static_taps, history_buffers=4, buffer_blocks=128, train_symbols=8192,
               warmup_symbols=8192, shard_count=2, shard_index=g, **fields) for g in range(2)]
pre, post = hs[0].shard_halo()
codes = torch.from_numpy(rec.codes.view(np.int16)).cuda()
labs = [torch.zeros(rec.n // 2 + 4096, dtype=torch.uint8, device="cuda") for _ in range(2)]
recs = [torch.zeros(hs[0].carry_size(), dtype=torch.uint8, device="cuda") for _ in range(2)]
nbuf = rec.n // (128 * 512)
for r in range(nbuf // 2 + 1):
    for g in range(2):
        b = 2 * r + g
        if b < nbuf:
            p0, p1, last = multi.shard_inputs(rec.n, 128 * 512, b, pre, post)
            hs[g].shard_process(b, codes[p0:p1], last=last, labels=labs[g])
        hs[g].export_carry(recs[g])
    for g in range(2):
        hs[g].import_carry(torch.cat(recs), 2, g)
print("PAM 2 shards", [h.stats()["bits"] for h in hs])
