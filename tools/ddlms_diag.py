import numpy as np, sys
sys.path.insert(0, '.')
from rxsynth import make_config
from tests.gpu_util import run_gpu, run_oracle, rel_l2
rec, rx = make_config("C3", n_samples=1 << 21, linewidth_hz=1e3)
rx.update(buffer_blocks=256, lms_taps=4, lms_block=1, lms_mode=2, widely_linear=1)
out = run_oracle(rec, rx)
R, labels, st = run_gpu(rec, rx, chunk=256 * 512)
m_end = out["m_end"]
Y = R.probe("Y", 0, m_end); z = out["lms"]["z"][:m_end]
S = 4096
errs = [rel_l2(Y[s:s+S], z[s:s+S]) for s in range(0, m_end - S + 1, S)]
print("per-seg rel", np.round(np.array(errs) * 1e4, 2))
s0 = int(np.argmax(errs)) * S
d = np.abs(Y[s0:s0+S] - z[s0:s0+S]) / np.abs(z[s0:s0+S]).mean()
print("worst seg", s0 // S, "err along the segment (x1e4):", np.round([d[i:i+256].mean()*1e4 for i in range(0, S, 256)], 2))
seg = R.probe("SEG", 0, m_end // S)
print("R gpu", seg[:20, 0].astype(int), "oracle", out["lms"]["R"][:20])
w, v = R.train_taps()
print("w_train rel", rel_l2(w, out["lms"]["w_train"]), "v_train rel", rel_l2(v, out["lms"]["v_train"]))
for s in (0, 1, 2, 9, 20):
    d = np.abs(Y[s*S:(s+1)*S] - z[s*S:(s+1)*S]) / np.abs(z[s*S:(s+1)*S]).mean()
    print("seg", s, np.round([d[i:i+256].mean()*1e6 for i in range(0, S, 256)], 1))
mism = out["labels"][:m_end] != labels[:m_end]
print("label flips at", np.nonzero(mism)[0][:10])
