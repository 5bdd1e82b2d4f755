"""Diagnose GPU-vs-oracle label mismatches on the full C4 record (bench launch configuration):
for each mismatch outside the excluded set, print the oracle soft value's distance to the nearest
decision boundary, the GPU / oracle equaliser outputs around it, the block's rotation difference
and the epoch. GPU box only."""
import numpy as np
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rxsynth import make_config
from tests.gpu_util import run_gpu, run_oracle, near_threshold
from oracle import rx_oracle as O

rec, rx = make_config("C4")
out = run_oracle(rec, rx)
R, labels, st = run_gpu(rec, rx, chunk=4 << 22, history_buffers=18)
m_end = out["m_end"]
lab_o = out["labels"][:m_end]; lab_g = labels[:m_end]
mism = np.nonzero(lab_o != lab_g)[0]
zo = out["lms"]["z"][:m_end]
zg = R.probe("Y", 0, m_end)
ax = O.qam_axis(rec.M); t = O.midpoints(ax)
S = rx["lms_segment"]; E = 8192 * 128
print("mismatches", mism.size)
for m in mism:
    s = m // S
    dI = np.min(np.abs(zo[m].real - t)); dQ = np.min(np.abs(zo[m].imag - t))
    b0 = (m // 32) * 32
    dphi = np.angle(zg[b0:b0 + 32] * np.conj(zo[b0:b0 + 32]))
    seg0 = s * S
    err = np.abs(zg[seg0:m] - zo[seg0:m]) / np.maximum(np.abs(zo[seg0:m]), 1e-9)
    print(f"m {m} seg {s} epoch {m // E} dist I {dI:.2e} Q {dQ:.2e} zo {zo[m]:.5f} zg {zg[m]:.5f} "
          f"block dphi med {np.median(dphi):.2e} max {np.max(np.abs(dphi)):.2e} "
          f"seg rel err before: max {err.max() if err.size else 0:.2e} mean {err.mean() if err.size else 0:.2e}")

# per segment: relative error of the GPU equaliser output over its first 256 and last 256 symbols
nseg = m_end // S
first_err = np.zeros(nseg); last_err = np.zeros(nseg); onset = np.full(nseg, -1)
for s in range(nseg):
    a, b = s * S, (s + 1) * S
    r = np.abs(zg[a:b] - zo[a:b]) / np.maximum(np.abs(zo[a:b]), 1e-9)
    first_err[s] = np.median(r[:256]); last_err[s] = np.median(r[-256:])
    big = np.nonzero(r > 1e-3)[0]
    onset[s] = big[0] if big.size else -1
E_seg = E // S
for e in range(nseg // E_seg):
    sl = slice(e * E_seg, (e + 1) * E_seg)
    diverged = np.nonzero(onset[sl] >= 0)[0]
    print(f"epoch {e}: median first-256 err {np.median(first_err[sl]):.2e}, max {first_err[sl].max():.2e}; "
          f"segments with |dz| > 1e-3 somewhere: {diverged.size} (onsets {list(onset[sl][diverged][:8])}, "
          f"segs {list(diverged[:8] + e * E_seg)})")
