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
