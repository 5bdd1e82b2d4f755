"""Print GPU-vs-oracle parity metrics for a config (diagnostic; used for DESIGN.md evidence).

python tools/parity_report.py C2 2097152 256   (config, n_samples, buffer_blocks)
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from rxsynth import make_config  # noqa: E402
from tests.gpu_util import near_threshold, rel_l2, run_gpu, run_oracle  # noqa: E402


def report(name, n, bb, chunk=None):
    rec, rx = make_config(name, n_samples=n)
    rx["buffer_blocks"] = bb
    t = time.time(); out = run_oracle(rec, rx); t_or = time.time() - t
    t = time.time(); R, labels, st = run_gpu(rec, rx, chunk=chunk or bb * 512); t_gpu = time.time() - t
    r = dict(config=name, n=n, buffer_blocks=bb, t_oracle=t_or, t_gpu_wall=t_gpu)
    if rec.fmt == "pam":
        nb = rec.n // 512
        r["C_rel"] = rel_l2(R.probe("C", 0, nb), out["C"])
        r["tau_maxabs"] = float(np.max(np.abs(R.probe("TAU", 0, nb) - out["clock"]["tau"])))
        Mb = R.probe("MB", 0, nb)
        r["Mb_mismatch"] = int(np.sum(Mb != out["clock"]["M"]))
        m_end = out["u"].shape[0]
        r["u_rel"] = rel_l2(R.probe("U", 0, m_end), out["u"])
        r["uhat_rel"] = rel_l2(R.probe("UHAT", 0, m_end), out["u_hat"])
    else:
        r["E_rel"] = rel_l2(R.probe("E", 0, out["E"].shape[0]), out["E"])
        r["z_rel"] = rel_l2(R.probe("Z", 0, out["z"].shape[0]), out["z"])
        nbuf = out["cfo"]["P"].shape[0]
        cfo = R.probe("CFO", 0, nbuf)
        r["P_rel_max"] = float(np.max(np.abs(cfo[:, 0] / out["cfo"]["P"] - 1)))
        r["df_gpu"] = cfo[:, 1].tolist()
        r["df_oracle"] = out["cfo"]["df"].tolist()
        r["df_absdiff_max"] = float(np.max(np.abs(cfo[:, 1] - out["cfo"]["df"])))
        r["domain"] = (st["domain_errors"], out["domain"])
    r["sync"] = (st["sync_offset"], out["sync"]["offset"], st["sync_phase"], out["sync"]["phase"])
    r["gamma"] = (st["sync_gamma"], out["sync"]["gamma"])
    r["wtrain_rel"] = rel_l2(R.train_taps(), out["lms"]["w_train"])
    m_end = out["m_end"]
    mism = labels[:m_end].astype(int) != out["labels"][:m_end].astype(int)
    soft = out["lms"]["z"][:m_end]
    r["m_end"] = (int(st["symbols_out"]), int(m_end))
    r["label_mismatch"] = int(mism.sum())
    for dlt in (1e-3, 1e-2, 5e-2):
        nt = near_threshold(soft, rec.fmt, rec.M, dlt)
        r[f"mism_not_within_{dlt}"] = int(np.sum(mism & ~nt))
        r[f"frac_within_{dlt}"] = float(nt.mean())
    y = R.probe("Y", 0, m_end)
    r["y_rel_all"] = rel_l2(y if rec.fmt == "qam" else y.real, soft)
    r["bit_errors"] = (st["bit_errors"], out["bit_errors"])
    r["bits"] = (st["bits"], out["bits"])
    r["evm_db"] = (10 * math.log10(st["evm_num"] / st["evm_den"]), out["evm_db"])
    r["flags"] = st["status_flags"]
    r["launches"] = st["launches"]
    if rec.fmt == "qam":
        nseg = -(-m_end // rx["lms_segment"])
        seg = R.probe("SEG", 0, nseg)
        r["R_gpu_head"] = seg[:12, 0].astype(int).tolist()
        r["R_or_head"] = out["lms"]["R"][:12].tolist()
        r["R_mismatch"] = int(np.sum(seg[:, 0].astype(int) != out["lms"]["R"]))
        S = rx["lms_segment"]
        rots = []
        for s_ in range(min(12, nseg)):
            a, b = y[s_ * S:(s_ + 1) * S], soft[s_ * S:(s_ + 1) * S]
            res = [rel_l2(a, b * (1j) ** k) for k in range(4)]
            rots.append((int(np.argmin(res)), float(min(res))))
        r["seg_rot_vs_oracle"] = rots
        r["r_gpu_head"] = seg[:12, 1].astype(int).tolist()
        r["r_or_head"] = out["lms"]["r_rel"][:12].tolist()
    return r


if __name__ == "__main__":
    args = sys.argv[1:] or ["C1", str(1 << 16), "8192"]
    out = report(args[0], int(args[1]), int(args[2]), int(args[3]) if len(args) > 3 else None)
    print(json.dumps(out, default=lambda o: o if not isinstance(o, np.generic) else o.item()))
