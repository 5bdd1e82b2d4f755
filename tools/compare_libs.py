"""Bit-level comparison of two librx builds on one small record (GPU box): the KK field E and z
probes and the labels of C3 (2^20 samples) through each library (RX_SO selects it; one child
process per library).  python tools/compare_libs.py a.so b.so"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    from rxsynth import make_config
    from tests.gpu_util import run_gpu
    rec, rx = make_config(os.environ.get("CMP_CFG", "C3"), n_samples=1 << 20)
    rx["buffer_blocks"] = 256
    if rec.fmt == "pam":
        R, lab, st = run_gpu(rec, rx, chunk=256 * 512)
        nu = st["symbols_out"]
        arrs = (("U", R.probe("U", 0, nu)), ("UHAT", R.probe("UHAT", 0, nu)), ("labels", lab))
    else:
        rx["fused_front_end"] = 0
        R, lab, st = run_gpu(rec, rx, chunk=256 * 512)
        nE = (rec.n // 512 - 1) * 512 - 256
        arrs = (("E", R.probe("E", 0, nE)), ("z", R.probe("Z", 0, (rec.n // 512 - 2) * 256 - 128)), ("labels", lab))
    out = {k: hashlib.sha1(v.tobytes()).hexdigest()[:16] for k, v in arrs}
    out["bit_errors"] = st["bit_errors"]
    print("RESULT " + json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child()
    else:
        for so in sys.argv[1:]:
            env = dict(os.environ, RX_SO=os.path.abspath(so))
            r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
            print(os.path.basename(so), line[-1][7:] if line else r.stderr[-800:])
