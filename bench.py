#!/usr/bin/env python
"""bench.py — received Gsample/s through the full receiver DSP chain (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpu|reference] [--backend nccl|gloo]

Headline workload (BASELINE.json's metric names no config, so the N = 1 line is quoted on the
largest single-GPU config, configs[3] = SURVEY C4): 1 GBaud Kramers-Kronig 64-QAM, 4 sps,
67,106,816 samples per step per GPU, CSPR 11 dB, ROADM-filtered, 10 kHz phase noise, 5 MHz CFO,
203-tap static EQ, 8-tap T/2 block-LMS with BPS-32 CPR, PRBS-15 BER. One step = one C4 record
streamed through rx_process in calls of four 2^22-sample paper buffers, i.e. one pass
of every KK row of SURVEY §8(a). Inputs come from a >= 1 GiB device ring (larger than the
126 MB L2) that tiles the periodic record, so every step reads fresh samples from HBM.

Also reported (extra keys): "pam" = configs[1] (C2 PAM-16, 2^24) measured the same way,
"per_buffer_call" = the paper's hand-off granularity (one 2^22 buffer per rx_process call),
"c3_sweep" = configs[2], "c5" = configs[4] (8 mixed channels per GPU), the CPU oracle on one
thread and on all cores.

Multi-GPU: `--gpus N` (N > 1) launches N ranks itself (torch.distributed.run, 127.0.0.1) unless
it already runs under torchrun. One process per GPU; every rank runs its own independent channel
(weak scaling, SURVEY §8(e) mode 1); once per step the packed BER/EVM counters are all-reduced
(NCCL; `--backend gloo` for CPU-only / shared-GPU smoke runs). Timing: W warm-up steps, then K
steps bracketed by barrier + synchronize, CUDA events on the processing stream, max over ranks.

--impl reference times the fp64 CPU oracle (oracle/) on the host on a bounded sample of the same
workload (one 2^22-sample buffer of the C4 record per step); under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import pickle
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "received Gsample/s through full Rx DSP chain at 1/2/4/8 B200; % HBM roofline"
PAPER_REALTIME_GSA = 4.0          # 12-bit 4 GSa/s real-time (unnamed GPU)
BUFFER = 1 << 22                  # one paper buffer
CALL_BUFFERS = 4                  # paper buffers per rx_process call (history_buffers = this + 2)
CHUNK = CALL_BUFFERS * BUFFER
SM_COUNT, FP32_LANES = 148, 128   # B200 (B200_PROFILING.md); FP32 FMA = 2 flop
HBM_GBS = 6548.8                  # MEASURED_PEAKS.json fallback (read at run time when present)

# Algorithmic flops per unit (SURVEY §8(d) 'Which roofline bounds the path': complex N-point FFT =
# 5 N log2 N, half for real-input / real-output; bin products 6 flop; C_b 8 flop/bin; KK
# reconstruction 12 flop per kept sample; block-LMS 4K flop per real T-spaced symbol, 16K per
# complex T/2 symbol + BPS 17 flop per test phase; CFO periodogram 136 flop per symbol).
FFT_R1024 = 2.5 * 1024 * 10
FLOPS_PER_BLOCK = {
    "PAM_FE": FFT_R1024 + 513 * 6 + 512 * 8,          # R2C + static EQ + C_b         = 32,774
    "PAM_BE": FFT_R1024 + 513 * 6,                    # clock ramp (H5) + C2R         = 28,678
    "KK_S1": 2 * FFT_R1024 + 512 * 12,                # R2C + C2R + reconstruction   = 57,344
    "KK_S2": 5 * 1024 * 10 + 512 * 6 + 5 * 512 * 9,   # C2C + EQ + IFFT-512           = 77,312
}
FLOPS_PER_BLOCK["KK_FE"] = FLOPS_PER_BLOCK["KK_S1"] + FLOPS_PER_BLOCK["KK_S2"]   # fused stages = 134,656


def class_flops(name, n_step, rx, kk):
    """Algorithmic flops of one kernel class per step (None: no flop model, HBM/latency class)."""
    if name in FLOPS_PER_BLOCK:
        return FLOPS_PER_BLOCK[name] * (n_step // 512)
    nsym = n_step // (4 if kk else 2)
    if name == "LMS":
        if kk:
            return (16 * rx["lms_taps"] + 17 * rx.get("cpr_test_phases", 0)) * nsym
        return 4 * rx["lms_taps"] * nsym
    if name == "CFO" and kk:
        return 136 * nsym
    return None


def chain_flops(n_step, rx, kk):
    names = ("KK_S1", "KK_S2", "CFO", "LMS") if kk else ("PAM_FE", "PAM_BE", "LMS")
    return sum(class_flops(n, n_step, rx, kk) for n in names)


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return HBM_GBS, "fallback"


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].lower() == "active"})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def fp32_peak(dev_index: int):
    """Measured FP32 FFMA throughput of this GPU (paper_2011_13695_b200/csrc/fp32_peak.cu)."""
    import ctypes
    from paper_2011_13695_b200 import build
    lib = ctypes.CDLL(build.build_peak())
    lib.fp32_peak_tflops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]
    t, ms = ctypes.c_double(), ctypes.c_double()
    if lib.fp32_peak_tflops(dev_index, 5, ctypes.byref(t), ctypes.byref(ms)) != 0:
        return None
    return t.value


# ------------------------------------------------------------------------ inputs
def _gen(name, kw):
    from rxsynth import make_config
    return make_config(name, **kw)


class Records:
    """Seeded synthetic records (rxsynth), generated concurrently in worker processes while the
    GPU measures. Under N > 1 ranks rank 0 generates and the others load its pickles (every rank
    runs an independent channel of the same content: weak scaling)."""

    def __init__(self, jobs: dict, rank: int, world: int, dist):
        self.rank, self.world, self.dist = rank, world, dist
        self.run_id = os.environ.get("TORCHELASTIC_RUN_ID", str(os.getpid()))
        self.jobs = jobs
        self.fut = {}
        self.t0 = time.time()
        if rank == 0 and jobs:
            import concurrent.futures as cf
            import multiprocessing as mp
            self.pool = cf.ProcessPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1, 6)),
                                               mp_context=mp.get_context("spawn"))
            for k, (name, kw) in jobs.items():
                self.fut[k] = self.pool.submit(_gen, name, kw)

    def _path(self, key):
        return f"/tmp/rxbench_{self.run_id}_{key.replace(':', '_')}.pkl"

    def get(self, key):
        if self.world == 1:
            return self.fut[key].result()
        if self.rank == 0:
            rec = self.fut[key].result()
            with open(self._path(key) + ".tmp", "wb") as f:
                pickle.dump(rec, f, protocol=4)
            os.replace(self._path(key) + ".tmp", self._path(key))
        self.dist.barrier()
        if self.rank != 0:
            with open(self._path(key), "rb") as f:
                rec = pickle.load(f)
        self.dist.barrier()
        if self.rank == 0:
            try:
                os.remove(self._path(key))
            except OSError:
                pass
        return rec

    def close(self):
        if getattr(self, "pool", None):
            self.pool.shutdown(wait=False, cancel_futures=True)


def rx_fields(rx: dict) -> dict:
    keys = ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu", "train_symbols",
            "sync_start", "sync_window", "warmup_symbols", "cpr_test_phases", "cpr_anchor")
    return {k: v for k, v in rx.items() if k in keys}


def multi_summary(counters):
    from paper_2011_13695_b200 import multi
    out = multi.summarize(counters)
    return {k: (round(v, 6) if isinstance(v, float) else v) for k, v in out.items()}


# ------------------------------------------------------------------------ timed runs
class Stream1:
    """One channel: a Receiver fed from a device ring in `chunk`-sample calls."""

    def __init__(self, R, ring, n_step, labels, stream, chunk=CHUNK):
        import ctypes
        self.R, self.ring, self.n_step, self.labels, self.stream = R, ring, n_step, labels, stream
        self.nsteps_ring = ring.numel() // n_step
        self.k = 0
        self.chunk = chunk
        self.sp = ctypes.c_void_p(stream.cuda_stream)

    def step(self):
        base = (self.k % self.nsteps_ring) * self.n_step
        ptr = self.ring.data_ptr() + 2 * base
        for off in range(0, self.n_step, self.chunk):
            n = min(self.chunk, self.n_step - off)
            self.R.process_ptr(ptr + 2 * off, n, self.labels.data_ptr(), self.labels.numel(), self.sp)
        self.k += 1


def run_mode(torch, dist, R, ring, n_step, steps, warmup, world, dev, chunk=CHUNK, with_profile=True,
             monitor=False):
    """Warm up, profile the kernel classes (untimed), then time `steps` steps."""
    from paper_2011_13695_b200 import multi
    stream = torch.cuda.Stream(device=dev)
    labels = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(8, dtype=torch.float64, device=dev)
    ch = Stream1(R, ring, n_step, labels, stream, chunk)

    def one_step():
        ch.step()
        R.export_counters(cnt, stream=stream)
        if world > 1:                      # one packed all-reduce of the counters per round
            with torch.cuda.stream(stream):
                multi.allreduce_counters(cnt)

    for _ in range(warmup):
        one_step()
    torch.cuda.synchronize(dev)
    breakdown, dominant = {}, None
    if with_profile:
        R.profile_enable()
        for _ in range(2):
            one_step()
        prof = R.profile_read()
        R.profile_enable(())
        breakdown = {k: round(v[0] / 2, 4) for k, v in prof.items()}
        dominant = max(breakdown, key=breakdown.get)
        R.profile_enable((dominant,))
    st0 = R.stats(stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    clocks.start()
    if monitor:
        R.rt_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    th0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    host_ms = (time.perf_counter() - th0) * 1e3 / steps
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    rt = None
    if monitor:
        rt = R.rt_stats()
        R.rt_enable(False)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    st1 = R.stats(stream)
    dom = None
    if with_profile and dominant:
        prof = R.profile_read()
        R.profile_enable(())
        if dominant in prof:
            dom = dict(name=dominant, ms=prof[dominant][0], launches=prof[dominant][1])
    return dict(ms=ms_max, clocks=clk, breakdown=breakdown, dominant=dom, host_ms=host_ms,
                launches=st1["launches"] - st0["launches"], stats=st1, counters=cnt.cpu().tolist(), rt=rt)


def e2e_run(torch, R, n_step, host_codes, steps, dev, packed=False, world=1, dist=None):
    """Same metric end to end through the public API: every step copies its input from pinned
    host memory to the device, runs the rx_process calls and reads its labels and counters back
    into pinned host memory, all inside the timed region. Double-buffered on three streams (H2D,
    processing, D2H) so the copy engines overlap the kernels of the neighbouring steps, as a
    streaming receiver would run. Returns the max-over-ranks time."""
    import ctypes
    proc = torch.cuda.Stream(device=dev)
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    sp = ctypes.c_void_p(proc.cuda_stream)
    if packed:        # RX_IN_U12_PACKED: the digitiser's 12-bit stream, 1.5 B per sample
        from rxsynth.gen import pack_u12
        pinned_in = torch.from_numpy(pack_u12(host_codes[:n_step])).pin_memory()
    else:
        pinned_in = torch.from_numpy(host_codes[:n_step].view("int16")).pin_memory()
    bps = 3 if packed else 4          # input bytes per 2 samples
    dbuf = [torch.empty_like(pinned_in, device=dev) for _ in range(2)]
    nlab = n_step // R.sps
    labels = torch.zeros(1 << 25, dtype=torch.uint8, device=dev)
    pinned_out = [torch.empty(nlab, dtype=torch.uint8).pin_memory() for _ in range(2)]
    cnt = [torch.zeros(8, dtype=torch.float64, device=dev) for _ in range(2)]
    cnt_host = [torch.empty(8, dtype=torch.float64).pin_memory() for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def one(k):
        i = k % 2
        with torch.cuda.stream(h2d):
            h2d.wait_event(ev_done[i])                  # dbuf[i] free again
            dbuf[i].copy_(pinned_in, non_blocking=True)
            ev_in[i].record(h2d)
        proc.wait_event(ev_in[i])
        for off in range(0, n_step, CHUNK):
            n = min(CHUNK, n_step - off)
            R.process_ptr(dbuf[i].data_ptr() + bps * off // 2, n, labels.data_ptr(), labels.numel(), sp)
        R.export_counters(cnt[i], stream=proc)
        ev_done[i].record(proc)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_done[i])
            d2h.wait_event(ev_out[i])                   # host buffer i read back two steps ago
            pinned_out[i].copy_(labels[i * nlab:(i + 1) * nlab], non_blocking=True)
            cnt_host[i].copy_(cnt[i], non_blocking=True)
            ev_out[i].record(d2h)

    for k in range(2):
        one(k)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(proc)
    h2d.wait_event(e0)
    for k in range(steps):
        one(k)
    proc.wait_stream(d2h)
    proc.wait_stream(h2d)
    e1.record(proc)
    torch.cuda.synchronize(dev)
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return dict(ms=float(t.item()), h2d=pinned_in.numel() * pinned_in.element_size(), d2h=nlab + 8 * 8)


def isolated_classes(torch, make_rx, ring, n_step, rx, kk, dev, peak, steps=2, chunk=CHUNK):
    """Per-class kernel time with the equaliser stage serialised on the caller's stream
    (rx_config.serial_equaliser = 1: no overlap between kernel classes), CUDA events per launch:
    the kernel-quality view of the roofline next to the live (overlapped) one."""
    R = make_rx(serial_equaliser=1)
    st = torch.cuda.Stream(device=dev)
    lab = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    ch = Stream1(R, ring, n_step, lab, st, chunk)
    for _ in range(3):
        ch.step()
    torch.cuda.synchronize(dev)
    R.profile_enable()
    for _ in range(steps):
        ch.step()
    prof = R.profile_read()
    R.close()
    out = {}
    for name, (ms, n) in prof.items():
        f = class_flops(name, n_step, rx, kk)
        e = {"ms_per_step": round(ms / steps, 4)}
        if f and ms > 0:
            a = f * steps / (ms / 1e3) / 1e12
            e.update(achieved_tflops=round(a, 3), frac=round(a / peak, 4))
        out[name] = e
    return out


def record_quality(torch, make_rx, rec, dev):
    """BER / EVM of one whole record streamed through a fresh handle and flushed (every symbol
    final, start-up included)."""
    codes = torch.from_numpy(rec.codes.view("int16")).to(dev)
    R = make_rx(history_buffers=CALL_BUFFERS + 2)
    lab = torch.zeros(1 << 25, dtype=torch.uint8, device=dev)
    for off in range(0, rec.n, CHUNK):
        R.process(codes[off:off + CHUNK], lab)
    R.flush(lab)
    s = R.stats()
    R.close()
    return {"ber": s["bit_errors"] / max(s["bits"], 1), "bit_errors": s["bit_errors"], "bits": s["bits"],
            "evm_db": round(10 * math.log10(s["evm_num"] / s["evm_den"]), 3) if s["evm_den"] > 0 else None}


def roofline_block(res, n_step, steps, rx, kk, peak, peak_nom, iso, traffic_key, value_gsa, bytes_per_sample):
    """The bench line's roofline object: the dominant kernel class of the timed region."""
    dom = res["dominant"]
    if not dom:
        return None
    name = dom["name"]
    f = class_flops(name, n_step, rx, kk)
    achieved = f * steps / (dom["ms"] / 1e3) / 1e12 if f else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        t = json.load(open(tp)).get(traffic_key + name)
        traffic = t.get("dram_bytes_per_launch") if isinstance(t, dict) else t
    hbm, hbm_src = hbm_peak()
    fc = chain_flops(n_step, rx, kk)
    chain_tf = fc * steps / (res["ms"] / 1e3) / 1e12
    return {"kernel_class": name, "bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/ncu_traffic.json)",
            "kernel_ms_per_step": dom["ms"] / steps, "launches_per_step": dom["launches"] / steps,
            "share_of_step": dom["ms"] / res["ms"],
            "peak_kind": "measured FP32 FFMA throughput of this GPU (csrc/fp32_peak.cu, best of 5)",
            "peak_nominal": peak_nom, "frac_of_nominal": (achieved / peak_nom) if achieved else None,
            "chain": {"flop_per_sample": round(fc / n_step, 1), "achieved_tflops": round(chain_tf, 3),
                      "frac": round(chain_tf / peak, 4)},
            "hbm_literal": {"bytes_per_sample": bytes_per_sample, "achieved_gbs": round(value_gsa * bytes_per_sample, 1),
                            "peak_gbs": hbm, "peak_source": hbm_src,
                            "frac": round(value_gsa * bytes_per_sample / hbm, 5)},
            "isolated": iso,
            "note": "algorithmic flops (SURVEY §8(d)) of the class / its CUDA-event time in the timed region "
                    "(live: the equaliser side stream overlaps the front-end); isolated = serial_equaliser=1 "
                    "(untimed pass); the path is FP32/smem bound, HBM literal fraction shown beside it"}


def _gen_c3(cspr):
    from rxsynth import make_config
    return make_config("C3", cspr_db=cspr)


def c3_sweep(torch, dev, local, recs):
    """BASELINE.json configs[2]: 1 GBaud KK QAM-4 with a 20 MHz frequency offset at
    OSNR 10 dB, swept over the carrier-to-signal power ratio (P:246 reports the optimum near
    6 dB); one 16,776,704-sample record per point through a fresh handle, device-resident input,
    CUDA events around each record's rx_process calls + flush."""
    import ctypes
    from paper_2011_13695_b200 import RX_QAM_KK, Receiver
    from rxsynth.configs import C3_CSPR_DB
    st = torch.cuda.Stream(device=dev)
    sp = ctypes.c_void_p(st.cuda_stream)
    lab = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    pts, ms_tot, n_tot = [], 0.0, 0
    for cspr in C3_CSPR_DB:
        rec, rx = recs.get(f"C3:{cspr}")
        codes = torch.from_numpy(rec.codes.view("int16")).to(dev)
        R = Receiver(RX_QAM_KK, rec.M, rec.static_taps, device=local, dc_offset=rec.dc_offset,
                     history_buffers=CALL_BUFFERS + 2, **rx_fields(rx))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for off in range(0, rec.n, CHUNK):
            n = min(CHUNK, rec.n - off)
            R.process_ptr(codes.data_ptr() + 2 * off, n, lab.data_ptr(), lab.numel(), sp)
        R.flush(lab, stream=st)
        e1.record(st)
        s1 = R.stats(st)
        ms = e0.elapsed_time(e1)
        ms_tot += ms
        n_tot += rec.n
        ber = s1["bit_errors"] / max(s1["bits"], 1)
        pts.append({"cspr_db": cspr, "ber": round(ber, 6), "evm_db": round(10 * math.log10(s1["evm_num"] / s1["evm_den"]), 2)
                    if s1["evm_den"] > 0 else None, "domain_errors": s1["domain_errors"], "ms": round(ms, 3)})
        R.close()
    best = min(pts, key=lambda p: p["ber"])
    return {"workload": "C3: KK QAM-4, +20 MHz CFO, 100 kHz linewidth, OSNR 10 dB, CSPR sweep, 16,776,704 "
                        "samples per point (one record, streamed + flushed)",
            "points": pts, "best_cspr_db": best["cspr_db"], "paper_optimum_cspr_db": 6,
            "value": round(n_tot / (ms_tot / 1e3) / 1e9, 3), "unit": "GSa/s",
            "note": "includes handle start-up (sync, training) and the flush of each record"}


def c5_run(torch, dist, rank, world, dev, steps, warmup, ring_gib, recs):
    """BASELINE.json configs[4]: 8 independent channels per GPU, mixed PAM-2/4/8/16
    and KK QAM-4/16/64/16 (C2/C4-style impairments), each one librx handle on its own CUDA
    stream so the channels' kernels overlap; the 8N channels' packed counters are all-reduced
    once per step (SURVEY §8(e) mode 1). One step = one 16,776,704-sample record per channel.
    Returns the bench sub-object (value = all ranks' samples / max-over-ranks time)."""
    from paper_2011_13695_b200 import RX_PAM, RX_QAM_KK, Receiver, multi
    from rxsynth.ring import pam_ring, tiled_ring
    chans = multi.channel_shard(8 * world, world, rank)      # 8 channels per rank
    chs, fmts = [], []
    for ch in chans:
        rec, rx = recs.get(f"C5:{ch % 8}")
        n_c = rec.n
        per_ring = max(warmup + steps + 1, int(ring_gib * (1 << 30) / 8 / 2 // n_c)) * n_c
        if rec.fmt == "pam":
            ring = pam_ring(rec, per_ring, dev, seed=7000 + ch)
            R = Receiver(RX_PAM, rec.M, rec.static_taps, device=dev.index or 0,
                         history_buffers=CALL_BUFFERS + 2, **rx_fields(rx))
        else:
            ring = tiled_ring(rec, per_ring, dev)
            R = Receiver(RX_QAM_KK, rec.M, rec.static_taps, device=dev.index or 0,
                         dc_offset=rec.dc_offset, history_buffers=CALL_BUFFERS + 2, **rx_fields(rx))
        fmts.append(f"{'PAM' if rec.fmt == 'pam' else 'QAM'}-{rec.M}")
        labels = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
        chs.append(Stream1(R, ring, n_c, labels, torch.cuda.Stream(device=dev)))
    main = torch.cuda.Stream(device=dev)
    cnt = torch.zeros(len(chs), 8, dtype=torch.float64, device=dev)
    fork, joins = torch.cuda.Event(), [torch.cuda.Event() for _ in chs]

    def one_step():
        fork.record(main)
        for i, c in enumerate(chs):
            c.stream.wait_event(fork)
            c.step()
            c.R.export_counters(cnt[i], stream=c.stream)
            joins[i].record(c.stream)
        for j in joins:
            main.wait_event(j)
        if world > 1:
            with torch.cuda.stream(main):
                multi.allreduce_counters(cnt)

    for _ in range(warmup):
        one_step()
    torch.cuda.synchronize(dev)
    l0 = sum(c.R.stats(c.stream)["launches"] for c in chs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(steps):
        one_step()
    e1.record(main)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    launches = sum(c.R.stats(c.stream)["launches"] for c in chs) - l0
    per_fmt = {}
    for f, c in zip(fmts, cnt.cpu().tolist()):
        acc = per_fmt.setdefault(f, [0.0] * 8)
        for k in range(8):
            acc[k] += c[k]
    for c in chs:
        c.R.close()
    del chs
    torch.cuda.empty_cache()
    return {"workload": "C5: 8 independent channels per GPU (PAM-2/4/8/16 C2-style, KK QAM-4/16/64/16 "
                        "C4-style), one 16,776,704-sample record per channel per step, one CUDA stream "
                        "per channel, all-reduce of the packed counters per step",
            "value": round(8 * world * n_c * steps / (ms / 1e3) / 1e9, 3), "unit": "GSa/s",
            "channels": 8 * world, "steps": steps, "ms_per_step": round(ms / steps, 4),
            "gpu_launches": launches, "clocks": clk,
            "input": f"per-channel device rings {per_ring * 2 / 2**20:.0f} MiB (8 per GPU > L2)",
            "quality_all_ranks_by_format" if world > 1 else "quality_by_format":
                {k: {kk: v for kk, v in multi_summary(c).items() if kk in ("ber", "evm_db", "bits")}
                 for k, c in sorted(per_fmt.items())}}


# ------------------------------------------------------------------------ CPU oracle baseline
def _oracle_window(args):
    """One bounded oracle run (a worker of the all-core baseline): samples [off, off + n) of the
    record as a stream of its own (sync, training, equaliser)."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import rx_oracle as O
    from tests.gpu_util import oracle_params
    rec, rx, off, n = args
    codes = np.ascontiguousarray(rec.codes[off:off + n]) if off is not None else rec.codes
    p = oracle_params(rec, rx)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        O.receive_pam(codes, p) if rec.fmt == "pam" else O.receive_kk(codes, p)
        return time.perf_counter() - t0


def cpu_oracle_baseline(rec, rx, n: int, max_procs: int = 16):
    """The fp64 oracle as it stands, on the host: one thread on one bounded window, then one
    window per core on min(nproc, max_procs) cores concurrently (independent windows of the same
    record). Returns the bench's cpu_baseline object."""
    import concurrent.futures as cf
    import dataclasses
    import multiprocessing as mp

    def window(off):                      # a light copy holding only the window's codes
        return dataclasses.replace(rec, codes=rec.codes[off:off + n].copy(), meta={}, tx_index=None)
    dt1 = _oracle_window((window(0), rx, None, n))
    ncpu = os.cpu_count() or 1
    procs = max(1, min(ncpu, max_procs, rec.n // n))
    offs = [(i * n) % (rec.n - n + 1) for i in range(procs)]
    wins = [(window(o), rx, None, n) for o in offs]
    t0 = time.perf_counter()
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("fork")) as ex:
        list(ex.map(_oracle_window, wins))
    wall = time.perf_counter() - t0
    v_all = procs * n / wall / 1e9
    return {"value": round(v_all, 6), "unit": "GSa/s", "cores": procs, "kind": "oracle",
            "sample": f"{procs} windows of {n} samples (one 2^22 paper buffer each, independent streams) of the "
                      f"bench record, fp64 numpy oracle, one process per core, {wall:.1f} s wall; nproc = {ncpu}",
            "value_1core": round(n / dt1 / 1e9, 6), "sample_1core": f"one window of {n} samples, 1 thread, {dt1:.1f} s"}


# ------------------------------------------------------------------------ GPU arm
def gpu_main(args):
    import numpy as np
    import torch
    rank, world, local = env_rank()
    dist = None
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % max(ndev, 1))
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    from paper_2011_13695_b200 import RX_PAM, RX_QAM_KK, Receiver, build
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    from rxsynth.configs import C3_CSPR_DB, N_C2, N_C4
    from rxsynth.ring import pam_ring, tiled_ring
    peak_meas = fp32_peak(dev.index)
    n1 = world == 1
    sc = args.record_scale                 # 1 = the configs' sizes (smoke tests shrink them)

    def nrec(n):
        return None if sc == 1 else max(1 << 19, n // sc // 512 * 512)
    jobs = {"C4": ("C4", {"n_samples": nrec(N_C4)})}
    if n1 and not args.no_pam:
        jobs["C2"] = ("C2", {"keep_tx": True, "n_samples": nrec(N_C2)})
    if not args.no_c5:
        for ch in range(8):
            jobs[f"C5:{ch}"] = (f"C5:{ch}", dict({"keep_tx": True} if ch < 4 else {}, n_samples=nrec(N_C2)))
    if n1 and not args.no_c3:
        for c in C3_CSPR_DB:
            jobs[f"C3:{c}"] = ("C3", {"cspr_db": c, "n_samples": nrec(N_C2)})
    recs = Records(jobs, rank, world, dist)
    extra, extra_launches = {}, 0
    # (configs[1], [2], [4] first: their records are ready while C4's is still being generated)
    e_steps = max(5, args.steps)
    peak_nom0 = SM_COUNT * FP32_LANES * 2 * 1965.0 * 1e6 / 1e12
    peak = peak_meas if peak_meas else peak_nom0

    # ---- C2 PAM-16 (configs[1]) at N = 1
    if n1 and not args.no_pam:
        rec2, rx2 = recs.get("C2")
        n2 = rec2.n
        ring2 = pam_ring(rec2, max(int(args.ring_gib * (1 << 30) / 2 // n2), args.warmup + args.steps + 6) * n2,
                         dev, seed=2001)

        def make_pam(**kw):
            f = dict(rx_fields(rx2), history_buffers=CALL_BUFFERS + 2, equaliser_lag=1)
            f.update(kw)
            return Receiver(RX_PAM, rec2.M, rec2.static_taps, device=dev.index, **f)
        W21 = round(0.021 * 2e9 / 4096) * 4096     # 21 ms of 2 GBaud symbols, whole segments
        R2 = make_pam(q_window_symbols=W21)
        r2 = run_mode(torch, None, R2, ring2, n2, args.steps, args.warmup, 1, dev)
        v2 = n2 * args.steps / (r2["ms"] / 1e3) / 1e9
        iso2 = None if args.timed_only else isolated_classes(torch, make_pam, ring2, n2, rx2, False, dev, peak, 2)
        s2 = r2["stats"]
        pam = {"workload": "C2: PAM-16 2 GBaud 2 sps, 16,776,704 samples/step, 91 km-like ISI, +20 ppm, SNR 32 dB, "
                           "503-tap static EQ, 105-block clock recovery, 31-tap block-LMS",
               "value": round(v2, 3), "unit": "GSa/s", "ms_per_step": round(r2["ms"] / args.steps, 4),
               "roofline": roofline_block(r2, n2, args.steps, rx2, False, peak, peak_nom0, iso2, "PAM_", v2, 2.5),
               "breakdown_ms_per_step": r2["breakdown"], "gpu_launches": r2["launches"], "clocks": r2["clocks"],
               "quality": {"ber": s2["bit_errors"] / max(s2["bits"], 1),
                           "evm_db": 10 * math.log10(s2["evm_num"] / s2["evm_den"]) if s2["evm_den"] > 0 else None}}
        from paper_2011_13695_b200 import multi as _multi
        nwin = s2["symbols_out"] // W21
        if nwin > 0:
            qe, qb = R2.q_trace(0, int(nwin))
            pam["q_trace_21ms_db"] = [round(_multi.q_db_from_ber(int(e) / int(b)), 2) if b else None
                                      for e, b in zip(qe, qb)]
        R2.close()
        if not args.timed_only:
            Rp2 = make_pam(input_format=2)
            Rp2.sps = 2
            r = e2e_run(torch, Rp2, n2, rec2.codes, e_steps, dev, packed=True)
            Rp2.close()
            pam["e2e"] = {"value": round(n2 * e_steps / (r["ms"] / 1e3) / 1e9, 3), "unit": "GSa/s",
                          "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]}
        extra["pam"] = pam
        extra_launches += r2["launches"]
        del ring2
        torch.cuda.empty_cache()
    # ---- C3: CSPR sweep (N = 1)
    if n1 and not args.no_c3:
        extra["c3_sweep"] = c3_sweep(torch, dev, dev.index, recs)
    # ---- C5: 8 mixed channels per GPU, concurrent streams (every N)
    if not args.no_c5:
        extra["c5"] = c5_run(torch, dist, rank, world, dev, args.c5_steps, 2, args.ring_gib, recs)
        extra_launches += extra["c5"]["gpu_launches"]
    # ---- headline: C4 KK 64-QAM (the largest single-GPU config)
    rec4, rx4 = recs.get("C4")
    n4 = rec4.n
    t_gen4 = time.time() - recs.t0
    ring4 = tiled_ring(rec4, max(args.warmup + args.steps + 6, int(args.ring_gib * (1 << 30) / 2 // n4)) * n4, dev)

    def make_kk(**kw):
        # equaliser_lag = 1: a call's equaliser rounds (side stream) overlap the next call's
        # front-end - the paper overlaps consecutive buffers across its streams; labels
        # and counters are identical to lag 0 (rx.h)
        f = dict(rx_fields(rx4), history_buffers=CALL_BUFFERS + 2, equaliser_lag=1)
        if args.lms_batch:
            f["lms_batch_segments"] = args.lms_batch
        if args.fused_fe:
            f["fused_front_end"] = 1
        f.update(kw)
        return Receiver(RX_QAM_KK, rec4.M, rec4.static_taps, device=dev.index, dc_offset=rec4.dc_offset, **f)

    R4 = make_kk()
    res = run_mode(torch, dist, R4, ring4, n4, args.steps, args.warmup, world, dev)
    value = world * n4 * args.steps / (res["ms"] / 1e3) / 1e9
    sm_max = res["clocks"].get("sm_max_mhz") or 1965.0
    peak_nom = SM_COUNT * FP32_LANES * 2 * sm_max * 1e6 / 1e12
    peak = peak_meas if peak_meas else peak_nom
    iso = isolated_classes(torch, make_kk, ring4, n4, rx4, True, dev, peak, 2) if n1 and not args.timed_only else None
    roof = roofline_block(res, n4, args.steps, rx4, True, peak, peak_nom, iso, "KK_", value / world, 2.25)
    st = res["stats"]
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GSa/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms"] / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (rxsynth, seeded C4: KK 64-QAM 1 GBaud 4 sps, CSPR 11 dB, OSNR 30 dB, ROADM 1.5 GHz, "
                "10 kHz linewidth, 5 MHz CFO)",
        "config": {"workload": "C4: KK 64-QAM, 67,106,816 samples/step per GPU, 203-tap static EQ, 4th-power CFO, "
                               "8-tap T/2 block-LMS + BPS-32 CPR, PRBS-15 BER",
                   "samples_per_step_per_gpu": n4, "record_scale": sc, "call_size": CHUNK,
                   "input": f"device ring {ring4.numel() * 2 / 2**30:.2f} GiB > L2 (fresh samples every step)",
                   "parallelism": f"{world} independent channel(s), 1 per GPU; all-reduce ({args.backend if world > 1 else 'none'}) "
                                  f"of the packed counters per step",
                   "equaliser_lag": 1},
        "roofline": roof,
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "breakdown_ms_per_step": res["breakdown"],
        "host_enqueue_ms_per_step": round(res["host_ms"], 4),
        "x_paper_realtime": round(value / world / PAPER_REALTIME_GSA, 2),
        "quality": {"ber": st["bit_errors"] / max(st["bits"], 1),
                    "evm_db": 10 * math.log10(st["evm_num"] / st["evm_den"]) if st["evm_den"] > 0 else None,
                    "quadrants": "anchored per segment (cpr_anchor = 1, DESIGN R-ANCHOR2)"},
        "quality_all_ranks": multi_summary(res["counters"]),
    }
    R4.close()
    if n1 and not args.timed_only:
        # the paper's hand-off granularity: one 2^22 buffer per rx_process call
        # (equaliser_lag = L: a call's equaliser stage overlaps the next L calls' front-ends, the
        # paper's cross-buffer stream overlap; a round runs every lms_batch_segments / 256 =
        # 8 one-buffer calls, so L = 8 hides it; lag 0 = every call joins its own stage)
        pb = {}
        for lag in (8, 1, 0):
            R1 = make_kk(history_buffers=3, equaliser_lag=lag)
            ks = max(3, args.steps // 2)
            r1 = run_mode(torch, None, R1, ring4, n4, ks, 3, 1, dev, chunk=BUFFER, with_profile=False, monitor=True)
            R1.close()
            v1 = n4 * ks / (r1["ms"] / 1e3) / 1e9
            rt = r1["rt"] or {}
            pb[lag] = {"value": round(v1, 3), "ms_per_buffer": round(r1["ms"] / ks / (n4 // BUFFER), 4),
                       "host_enqueue_ms_per_buffer": round(r1["host_ms"] / (n4 // BUFFER), 4),
                       "rt_monitor": {"calls": rt.get("calls"), "realtime_ratio": round(rt.get("realtime_ratio", 0), 3),
                                      "max_call_ms": round(rt.get("max_call_ms", 0), 4),
                                      "max_load": round(rt.get("max_load", 0), 4), "overruns": rt.get("overruns")}}
        line["per_buffer_call"] = dict(pb[8], unit="GSa/s", call_samples=BUFFER, equaliser_lag=8,
                                       realtime_ratio=round(pb[8]["value"] / PAPER_REALTIME_GSA, 2),
                                       equaliser_lag_1=pb[1], equaliser_lag_0=pb[0])
        # quadrant modes on one flushed record: anchored (default) and the c-9 stitch chain
        qa = record_quality(torch, make_kk, rec4, dev)
        qc = record_quality(torch, lambda **kw: make_kk(cpr_anchor=0, **kw), rec4, dev)
        line["quality"]["record_anchored"] = qa
        line["quality"]["record_chain_mode"] = qc
    # ---- e2e through the public API with host buffers (packed 12-bit input, the ADC's format)
    if not args.timed_only:
        Rp = make_kk(input_format=2)
        Rp.sps = 4
        r = e2e_run(torch, Rp, n4, rec4.codes, e_steps, dev, packed=True, world=world, dist=dist)
        Rp.close()
        line["e2e"] = {"value": round(world * n4 * e_steps / (r["ms"] / 1e3) / 1e9, 3), "unit": "GSa/s",
                       "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                       "input": "pinned host, RX_IN_U12_PACKED (2 codes per 3 bytes); labels + counters read back"}
    del ring4
    torch.cuda.empty_cache()

    line.update(extra)
    # ---- CPU oracle baseline (rank 0, N = 1)
    if n1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_baseline(rec4, rx4, BUFFER)
    else:
        line["cpu_baseline"] = None
    recs.close()
    line["gen_seconds_c4"] = round(t_gen4, 1)
    # compact summary last, so the end of the line (what a truncated log tail shows) carries it
    line["summary"] = {"kk_c4_gsa": line["value"], "pam_c2_gsa": line.get("pam", {}).get("value"),
                       "c5_gsa": line.get("c5", {}).get("value"), "e2e_c4_gsa": line.get("e2e", {}).get("value"),
                       "per_buffer_call_gsa": line.get("per_buffer_call", {}).get("value"),
                       "dominant_class": (roof or {}).get("kernel_class"), "dominant_frac": (roof or {}).get("frac"), "chain_frac": (roof or {}).get("chain", {}).get("frac"),
                       "fp32_peak_tflops": round(peak, 2), "n_gpus": world}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------ reference arm
def reference_main(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from rxsynth import make_config
    rec, rx = make_config("C4", n_samples=BUFFER)       # the bounded sample: one paper buffer of C4
    for _ in range(args.warmup):
        _oracle_window((rec, rx, 0, BUFFER))
    t = 0.0
    for _ in range(args.steps):
        t += _oracle_window((rec, rx, 0, BUFFER))
    v = args.steps * BUFFER / t / 1e9
    sample = (f"one 2^22-sample paper buffer (P:116) of the C4 workload per step (generated with C4's "
              f"parameters at that length), fp64 numpy oracle, 1 thread")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GSa/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (rxsynth, seeded C4)",
            "config": {"workload": "C4: KK 64-QAM (bounded sample)", "samples_per_step": BUFFER},
            "cpu_baseline": {"value": round(v, 6), "unit": "GSa/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "GSa/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def launch_ranks(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks (one per GPU) ourselves."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # communicator init (rank count) in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("gpu", "reference"), default="gpu")
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl")
    ap.add_argument("--no-pam", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--c5-steps", type=int, default=4)
    ap.add_argument("--ring-gib", type=float, default=1.0)
    ap.add_argument("--record-scale", type=int, default=1,
                    help="divide every record length by this (smoke tests only; 1 = the configs' sizes)")
    ap.add_argument("--timed-only", action="store_true",
                    help="profiling runs (ncu): only the timed C2 / C4 regions, no isolated passes, "
                         "per-buffer calls, record quality or e2e; implies --no-c3 --no-c5 --no-cpu")
    ap.add_argument("--lms-batch", type=int, default=0,
                    help="segments per equaliser launch (rx_config.lms_batch_segments; 0 = library "
                         "default: D epochs, i.e. 4096 PAM / 2048 KK)")
    ap.add_argument("--fused-fe", action="store_true",
                    help="KK: rx_config.fused_front_end = 1 (k_kk_fe, E in shared memory; profiling / comparison)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.timed_only:
        args.no_c3 = args.no_c5 = args.no_cpu = True
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.impl == "reference":
        reference_main(args)
    else:
        gpu_main(args)


if __name__ == "__main__":
    main()
