"""Labels/counters of a long C2 stream (continuous +20 ppm ring) must not depend on the
equaliser batch size or call size (debug/evidence tool; GPU)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_13695_b200 import RX_PAM, Receiver  # noqa: E402
from rxsynth import make_config  # noqa: E402
from rxsynth.configs import N_C2  # noqa: E402
from rxsynth.ring import pam_ring  # noqa: E402

nrec = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rec, rx = make_config("C2", keep_tx=True)
dev = torch.device("cuda", 0)
ring = pam_ring(rec, nrec * N_C2, dev)
keys = ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu", "train_symbols", "sync_start",
        "sync_window", "warmup_symbols")
res = {}
for batch, callb in ((0, 1), (2048, 4), (4096, 4), (60000, 4)):
    R = Receiver(RX_PAM, rec.M, rec.static_taps, history_buffers=max(callb + 2, 3) if batch != 60000 else 4 * nrec + 4,
                 lms_batch_segments=batch, **{k: rx[k] for k in keys})
    lab = torch.full((nrec * N_C2 // 2 + 8192,), 255, dtype=torch.uint8, device=dev)
    call = callb << 22
    for off in range(0, ring.numel(), call):
        R.process(ring[off:off + call], lab)
    R.flush(lab)
    st = R.stats()
    res[(batch, callb)] = (lab.cpu().numpy(), st)
    print(batch, callb, {k: st[k] for k in ("bit_errors", "bits", "symbols_out", "status_flags")},
          10 * np.log10(st["evm_num"] / st["evm_den"]), flush=True)
    R.close()
ref = res[(0, 1)][0]
for k, (lab, st) in res.items():
    print(k, "label mismatches vs batch-0:", int(np.sum(lab != ref)))
