"""Run one config through librx (debug helper): python tools/run_one.py C1 [n] [buffer_blocks]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rxsynth import make_config  # noqa: E402
from tests.gpu_util import run_gpu  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
rec, rx = make_config(name, n_samples=n)
if len(sys.argv) > 3:
    rx["buffer_blocks"] = int(sys.argv[3])
R, labels, st = run_gpu(rec, rx, chunk=rx.get("buffer_blocks", 8192) * 512)
print({k: st[k] for k in ("bit_errors", "bits", "symbols_out", "sync_offset", "status_flags", "launches")})
