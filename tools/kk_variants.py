"""Time kernel variants of librx on the C4 workload (bench.py's headline configuration), one child
process per variant (RX_SO selects the library): value (GSa/s, live, overlapped), per-class
breakdown (live) and the isolated class times. The C4 record is generated once and cached.

  python tools/kk_variants.py lib1.so lib2.so ...        (GPU box)"""
import json
import os
import pickle
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CACHE = "/tmp/rx_c4_record.pkl"


def child(so, steps=10, chunk=None, lms_batch=0):
    import torch
    import bench
    from paper_2011_13695_b200 import RX_QAM_KK, Receiver
    from rxsynth.ring import tiled_ring
    rec, rx = pickle.load(open(CACHE, "rb"))
    dev = torch.device("cuda", 0)
    ring = tiled_ring(rec, 12 * rec.n, dev)

    def make_kk(**kw):
        f = dict(bench.rx_fields(rx), history_buffers=bench.CALL_BUFFERS + 2,
                 equaliser_lag=int(os.environ.get("LMS_LAG", "0")))
        if lms_batch:
            f["lms_batch_segments"] = lms_batch
        if os.environ.get("RX_FUSED"):
            f["fused_front_end"] = int(os.environ["RX_FUSED"])
        if os.environ.get("LMS_D"):
            f["tap_lag_epochs"] = int(os.environ["LMS_D"])
        f.update(kw)
        return Receiver(RX_QAM_KK, rec.M, rec.static_taps, device=0, dc_offset=rec.dc_offset, **f)
    R = make_kk()
    chunk = int(os.environ.get("KV_CHUNK", "0")) or bench.CHUNK     # samples per rx_process call
    res = bench.run_mode(torch, None, R, ring, rec.n, steps, 3, 1, dev, chunk=chunk)
    st = res["stats"]
    R.close()
    iso = bench.isolated_classes(torch, make_kk, ring, rec.n, rx, True, dev, 72.2, 2, chunk) if not os.environ.get("KV_NOISO") else {}
    out = {"so": os.path.basename(so), "fused": os.environ.get("RX_FUSED", "1"),
           "fe_per_cta": os.environ.get("RX_FE_PER_CTA", "auto"), "chunk": chunk, "lag": os.environ.get("LMS_LAG", "0"), "D": os.environ.get("LMS_D", "8"),
           "batch": lms_batch, "value": round(rec.n * steps / (res["ms"] / 1e3) / 1e9, 3),
           "ms": round(res["ms"] / steps, 4), "live": res["breakdown"],
           "iso": {k: v["ms_per_step"] for k, v in iso.items()},
           "ber": st["bit_errors"] / max(st["bits"], 1), "bits": st["bits"], "clocks": res["clocks"]}
    print("RESULT " + json.dumps(out), flush=True)


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2], lms_batch=int(os.environ.get("LMS_BATCH", "0")))
        return
    if not os.path.exists(CACHE):
        from rxsynth import make_config
        t = time.time()
        pickle.dump(make_config("C4"), open(CACHE, "wb"), protocol=4)
        print(f"generated C4 in {time.time() - t:.1f} s", flush=True)
    for so in sys.argv[1:]:
        env = dict(os.environ, RX_SO=os.path.abspath(so))
        r = subprocess.run([sys.executable, __file__, "--child", so], env=env, capture_output=True, text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        print(line[-1][7:] if line else f"{so}: FAILED {r.stderr[-1500:]}", flush=True)


if __name__ == "__main__":
    main()
