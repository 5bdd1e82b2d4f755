#!/usr/bin/env python
"""bench.py — received Gsample/s through the full receiver DSP chain (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gpu|reference] [--no-kk]

Workload (BASELINE.json configs[1] = SURVEY C2): 2 GBaud PAM-16, 2 sps, 91 km-like ISI,
+20 ppm clock offset, SNR 32 dB, 503-tap static EQ, 31-tap block-LMS, PRBS-15 BER tester.
One step = one C2 record (16,776,704 samples = "2^24") streamed through rx_process in calls
of up to four 2^22-sample paper buffers, i.e. one pass of every PAM row of SURVEY §8(a).
Inputs come from a >= 1 GiB device ring (larger than the 126 MB L2) that continues the
seeded record seamlessly, so every step reads fresh samples from HBM.

Multi-GPU (torchrun, one rank per GPU): every rank runs its own independent channel (weak
scaling); once per step the packed BER/EVM counters are all-reduced over NCCL.
Timing: W warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on the
processing stream, max over ranks. The KK-QAM mode (C4, 64-QAM, 2^26 samples) is measured the
same way at N = 1 and reported under "kk".

--impl reference times the fp64 CPU oracle (oracle/) on the host on a bounded sample of the
same workload (one 2^22-sample buffer per step); under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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

# Algorithmic flops per unit (complex N-point FFT = 5 N log2 N, half for
# real-input / real-output; bin products 6 flop; C_b 8 flop/bin; block-LMS 4K flop per real
# T-spaced symbol, 16K per complex T/2 symbol + BPS 17 flop per test phase).
FFT_R1024 = 2.5 * 1024 * 10
FLOPS_PER_UNIT = {
    "PAM_FE": FFT_R1024 + 513 * 6 + 512 * 8,               # per block
    "PAM_BE": FFT_R1024 + 2 * 513 * 6,                     # per block (C2R; R2C counted in PAM_FE)
    "KK_S1": 2 * FFT_R1024 + 512 * 20,                     # per block
    "KK_S2": 5 * 1024 * 10 + 512 * 6 + 5 * 512 * 9,        # per block
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


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


# ------------------------------------------------------------------------ helpers
def multi_summary(counters):
    from paper_2011_13695_b200 import multi
    out = multi.summarize(counters)
    return {k: (round(v, 6) if isinstance(v, float) else v) for k, v in out.items()}


def rx_fields(rx: dict) -> dict:
    keys = ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu", "train_symbols",
            "sync_start", "sync_window", "warmup_symbols", "cpr_test_phases")
    return {k: v for k, v in rx.items() if k in keys}


def cpu_oracle_rate(rec, rx, n_samples: int):
    """Time the fp64 oracle, as it stands, on the first n_samples of the record (1 thread)."""
    from threadpoolctl import threadpool_limits
    from oracle import rx_oracle as O
    from tests.gpu_util import oracle_params
    codes = rec.codes[:n_samples]
    p = oracle_params(rec, rx)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        out = O.receive_pam(codes, p) if rec.fmt == "pam" else O.receive_kk(codes, p)
        dt = time.perf_counter() - t0
    return n_samples / dt / 1e9, dt, out


class Stream1:
    """One channel: a Receiver fed from a device ring in buffer-sized calls."""

    def __init__(self, R, ring, n_step, labels, stream):
        self.R, self.ring, self.n_step, self.labels, self.stream = R, ring, n_step, labels, stream
        self.nsteps_ring = ring.numel() // n_step
        self.k = 0
        import ctypes
        self.sp = ctypes.c_void_p(stream.cuda_stream)

    def step(self):
        base = (self.k % self.nsteps_ring) * self.n_step
        ptr = self.ring.data_ptr() + 2 * base
        for off in range(0, self.n_step, CHUNK):
            n = min(CHUNK, self.n_step - off)
            self.R.process_ptr(ptr + 2 * off, n, self.labels.data_ptr(), self.labels.numel(), self.sp)
        self.k += 1


def run_mode(torch, dist, R, ring, n_step, steps, warmup, world, dev, units, label_cap=1 << 24,
             with_profile=True):
    """Warm up, profile the kernel classes (untimed), then time `steps` steps."""
    stream = torch.cuda.Stream(device=dev)
    labels = torch.zeros(label_cap, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(8, dtype=torch.float64, device=dev)
    ch = Stream1(R, ring, n_step, labels, stream)

    from paper_2011_13695_b200 import multi

    def one_step():
        ch.step()
        R.export_counters(cnt, stream=stream)
        if world > 1:                      # one packed NCCL all-reduce of the counters per round
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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    th0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    host_ms = (time.perf_counter() - th0) * 1e3 / steps
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
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
                launches=st1["launches"] - st0["launches"], stats=st1, counters=cnt.cpu().tolist())


def e2e_run(torch, R, n_step, host_codes, steps, dev, packed=False):
    """Same metric end to end through the public API: every step copies its input from pinned
    host memory to the device, runs the rx_process calls and reads its labels and counters back
    into pinned host memory, all inside the timed region. Double-buffered on three streams (H2D,
    processing, D2H) so the copy engines overlap the kernels of the neighbouring steps, as a
    streaming receiver would run."""
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
    labels = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    nlab = n_step // 2
    pinned_out = [torch.empty(nlab, dtype=torch.uint8).pin_memory() for _ in range(2)]
    cnt = [torch.zeros(8, dtype=torch.float64, device=dev) for _ in range(2)]
    cnt_host = [torch.empty(8, dtype=torch.float64).pin_memory() for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]      # input of buffer i on the device
    ev_done = [torch.cuda.Event() for _ in range(2)]    # processing of buffer i finished
    ev_out = [torch.cuda.Event() for _ in range(2)]     # labels of buffer i on the host

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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(proc)
    h2d.wait_event(e0)
    for k in range(steps):
        one(k)
    proc.wait_stream(d2h)
    proc.wait_stream(h2d)
    e1.record(proc)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    return dict(ms=ms, h2d=pinned_in.numel() * pinned_in.element_size(), d2h=nlab + 8 * 8)


def class_flops(name, n_step, rx, kk):
    """Algorithmic flops of one kernel class per step, None if the
    class has no flop model (HBM / latency classes)."""
    if name in FLOPS_PER_UNIT:
        return FLOPS_PER_UNIT[name] * (n_step // 512)
    if name == "LMS":
        if kk:   # 16K flop per complex T/2 symbol + BPS 17 flop per test phase
            return (16 * rx["lms_taps"] + 17 * rx["cpr_test_phases"]) * (n_step // 4)
        return 4 * rx["lms_taps"] * (n_step // 2)
    return None


def isolated_classes(torch, make_rx, ring, n_step, rx, kk, dev, peak, steps=2):
    """Per-class kernel time with the equaliser stage serialised on the caller's stream
    (rx_config.serial_equaliser = 1: no overlap between kernel classes), CUDA events per launch:
    the kernel-quality view of the roofline next to the live (overlapped) one."""
    R = make_rx(serial_equaliser=1)
    st = torch.cuda.Stream(device=dev)
    lab = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    ch = Stream1(R, ring, n_step, lab, st)
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


def _gen_c3(cspr):
    from rxsynth import make_config
    return make_config("C3", cspr_db=cspr)


def c3_sweep(torch, dev, local):
    """BASELINE.json configs[2]: 1 GBaud KK QAM-4 with a 20 MHz frequency offset at
    OSNR 10 dB, swept over the carrier-to-signal power ratio (P:246 reports the optimum near
    6 dB); one 16,776,704-sample record per point through a fresh handle, device-resident input,
    CUDA events around each record's rx_process calls + flush."""
    import concurrent.futures as cf
    import ctypes
    import multiprocessing as mp
    from paper_2011_13695_b200 import RX_QAM_KK, Receiver
    from rxsynth.configs import C3_CSPR_DB
    t0 = time.time()
    with cf.ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1),
                                mp_context=mp.get_context("spawn")) as ex:
        recs = list(ex.map(_gen_c3, C3_CSPR_DB))
    t_gen = time.time() - t0
    st = torch.cuda.Stream(device=dev)
    sp = ctypes.c_void_p(st.cuda_stream)
    lab = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    pts, ms_tot, n_tot = [], 0.0, 0
    for cspr, (rec, rx) in zip(C3_CSPR_DB, recs):
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
        pts.append({"cspr_db": cspr, "ber": ber, "evm_db": round(10 * math.log10(s1["evm_num"] / s1["evm_den"]), 3)
                    if s1["evm_den"] > 0 else None, "domain_errors": s1["domain_errors"],
                    "sync_gamma": round(s1["sync_gamma"], 4), "ms": round(ms, 3)})
        R.close()
    best = min(pts, key=lambda p: p["ber"])
    return {"workload": "C3: KK QAM-4 1 GBaud 4 sps, +20 MHz CFO, 100 kHz linewidth, OSNR 10 dB, "
                        "CSPR sweep, 16,776,704 samples per point (one record, streamed + flushed)",
            "points": pts, "best_cspr_db": best["cspr_db"], "paper_optimum_cspr_db": 6,
            "value": round(n_tot / (ms_tot / 1e3) / 1e9, 3), "unit": "GSa/s",
            "note": "value includes handle start-up (sync, training) and the flush of each record; "
                    "at fixed OSNR a high CSPR leaves too little signal power, a low one breaks the "
                    "minimum-phase condition (domain errors)",
            "gen_seconds": round(t_gen, 1)}


def _gen_c5(ch):
    from rxsynth import make_config
    return make_config(f"C5:{ch}", keep_tx=True) if ch % 8 < 4 else make_config(f"C5:{ch}")


def c5_run(torch, dist, rank, world, dev, steps, warmup, ring_gib):
    """BASELINE.json configs[4]: 8 independent channels per GPU, mixed PAM-2/4/8/16
    and KK QAM-4/16/64/16 (C2/C4-style impairments), each one librx handle on its own CUDA
    stream so the channels' kernels overlap; the 8N channels' packed counters are all-reduced
    over NCCL once per step (SURVEY §8(e) mode 1). One step = one 16,776,704-sample record per
    channel. Returns the bench sub-object (value = all ranks' samples / max-over-ranks time)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    from paper_2011_13695_b200 import RX_PAM, RX_QAM_KK, Receiver, multi
    from rxsynth.configs import N_C2
    from rxsynth.ring import pam_ring, tiled_ring
    chans = multi.channel_shard(8 * world, world, rank)      # 8 channels per rank
    t0 = time.time()
    with cf.ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1),
                                mp_context=mp.get_context("spawn")) as ex:
        recs = list(ex.map(_gen_c5, chans))
    t_gen = time.time() - t0
    # PAM rings continue the record with its clock offset and must not wrap inside the run
    # (a wrap restarts the PRBS); KK records are exactly periodic and tile seamlessly
    per_ring = max(warmup + steps + 1, int(ring_gib * (1 << 30) / 8 / 2 // N_C2)) * N_C2
    chs = []
    for ch, (rec, rx) in zip(chans, recs):
        if rec.fmt == "pam":
            ring = pam_ring(rec, per_ring, dev, seed=7000 + ch)
            R = Receiver(RX_PAM, rec.M, rec.static_taps, device=dev.index or 0,
                         history_buffers=CALL_BUFFERS + 2, **rx_fields(rx))
        else:
            ring = tiled_ring(rec, per_ring, dev)
            R = Receiver(RX_QAM_KK, rec.M, rec.static_taps, device=dev.index or 0,
                         dc_offset=rec.dc_offset, history_buffers=CALL_BUFFERS + 2, **rx_fields(rx))
        rec.meta.pop("x_tx", None)
        labels = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
        chs.append(Stream1(R, ring, N_C2, labels, torch.cuda.Stream(device=dev)))
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
    c_all = cnt.cpu().tolist()
    for (rec, _), c in zip(recs, c_all):
        key = f"{'PAM' if rec.fmt == 'pam' else 'QAM'}-{rec.M}"
        acc = per_fmt.setdefault(key, [0.0] * 8)
        for k in range(8):
            acc[k] += c[k]
    for c in chs:
        c.R.close()
    del chs
    torch.cuda.empty_cache()
    return {"workload": "C5: 8 independent channels per GPU (PAM-2/4/8/16 C2-style, KK QAM-4/16/64/16 "
                        "C4-style), one 16,776,704-sample record per channel per step, one CUDA stream "
                        "per channel, NCCL all-reduce of the packed counters per step",
            "value": round(8 * world * N_C2 * steps / (ms / 1e3) / 1e9, 3), "unit": "GSa/s",
            "channels": 8 * world, "steps": steps, "ms_per_step": round(ms / steps, 4),
            "gpu_launches": launches, "clocks": clk, "gen_seconds": round(t_gen, 1),
            "input": f"per-channel device rings {per_ring * 2 / 2**20:.0f} MiB (8 per GPU, "
                     f"{8 * per_ring * 2 / 2**30:.2f} GiB > L2)",
            "quality_rank0_by_format": {k: multi_summary(v) for k, v in sorted(per_fmt.items())}}


# ------------------------------------------------------------------------ GPU arm
def gpu_main(args):
    import numpy as np
    import torch
    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2011_13695_b200 import RX_PAM, RX_QAM_KK, Receiver, build
    build.build()
    from rxsynth import make_config
    from rxsynth.configs import N_C2, N_C4
    from rxsynth.ring import pam_ring, tiled_ring

    # ---- C2 (headline)
    seed = 2001 + 17 * rank
    t0 = time.time()
    rec, rx = make_config("C2", seed=seed, keep_tx=True)
    t_gen = time.time() - t0
    n_step = N_C2
    # >= 1 GiB (> L2) and long enough that the timed steps never wrap (a wrap restarts the
    # clock-offset waveform and the PRBS): warm-up + 2 profiled + K timed + 3 isolated steps
    ring_samples = max(int(args.ring_gib * (1 << 30) / 2 // n_step), args.warmup + args.steps + 6) * n_step
    ring = pam_ring(rec, ring_samples, dev, seed=seed)
    def make_pam(**kw):
        return Receiver(RX_PAM, rec.M, rec.static_taps, device=local, history_buffers=CALL_BUFFERS + 2,
                        **({"lms_batch_segments": args.lms_batch} if args.lms_batch else {}),
                        **rx_fields(rx), **kw)
    W21 = round(0.021 * 2e9 / 4096) * 4096     # 21 ms of 2 GBaud symbols, whole segments
    R = make_pam(q_window_symbols=W21)
    res = run_mode(torch, dist, R, ring, n_step, args.steps, args.warmup, world, dev, None)
    value = world * n_step * args.steps / (res["ms"] / 1e3) / 1e9
    ms_step = res["ms"] / args.steps
    st = res["stats"]
    # roofline of the dominant kernel class, measured live in the timed region
    roof = None
    sm_max = res["clocks"].get("sm_max_mhz") or 1965.0
    peak_fp32 = SM_COUNT * FP32_LANES * 2 * sm_max * 1e6 / 1e12
    dom = res["dominant"]
    if dom:
        name = dom["name"]
        blocks_per_step = n_step // 512
        if name in FLOPS_PER_UNIT:
            flops = FLOPS_PER_UNIT[name] * blocks_per_step * args.steps
        elif name == "LMS":
            flops = 4 * rx["lms_taps"] * (n_step // 2) * args.steps
        else:
            flops = None
        achieved = flops / (dom["ms"] / 1e3) / 1e12 if flops else None
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(name)
        roof = {"kernel_class": name, "bound": "alu", "achieved": achieved, "peak": peak_fp32,
                "unit": "TFLOP/s", "frac": (achieved / peak_fp32) if achieved else None,
                "traffic": traffic, "kernel_ms_per_step": dom["ms"] / args.steps,
                "share_of_step": dom["ms"] / res["ms"],
                "peak_note": "FP32 CUDA-core peak = 148 SMs x 128 lanes x 2 flop x max SM clock "
                             "(guide unit counts; the path is FP32/smem bound, SURVEY §8(d))",
                "live_note": "live = timed region, where the equaliser stage runs on the library's side "
                             "stream concurrently with the front-end (kernel times include that overlap); "
                             "isolated = the same classes with serial_equaliser=1 (untimed pass)"}
        roof["isolated"] = isolated_classes(torch, make_pam, ring, n_step, rx, False, dev, peak_fp32)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GSa/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (rxsynth, seeded C2: PAM-16 2 GBaud 2 sps, 91 km-like ISI, +20 ppm, SNR 32 dB)",
        "config": {"workload": "C2: PAM-16, 16,776,704 samples/step per GPU, 503-tap static EQ, "
                               "105-block clock recovery, 31-tap block-LMS, PRBS-15 BER",
                   "samples_per_step_per_gpu": n_step, "call_size": CHUNK,
                   "input": f"device ring {ring_samples * 2 / 2**30:.2f} GiB > L2 (fresh samples every step)",
                   "parallelism": f"{world} independent channel(s), 1 per GPU; NCCL all-reduce of counters per step"},
        "roofline": roof,
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "breakdown_ms_per_step": res["breakdown"],
        "host_enqueue_ms_per_step": round(res["host_ms"], 4),
        "hbm_roofline_frac_literal": round(value * 1e9 / world * 2.5 / 6537e9, 5),
        "x_paper_realtime": round(value / world / PAPER_REALTIME_GSA, 2),
        "quality_all_ranks": multi_summary(res["counters"]),
        "quality": {"ber": st["bit_errors"] / max(st["bits"], 1),
                    "evm_db": 10 * math.log10(st["evm_num"] / st["evm_den"]) if st["evm_den"] > 0 else None,
                    "sync_gamma": st["sync_gamma"], "flags": st["status_flags"]},
        "gen_seconds": round(t_gen, 1),
    }
    # ---- Q trace: BER in 21 ms sections, windows completed so far on this channel
    from paper_2011_13695_b200 import multi as _multi
    nwin = st["symbols_out"] // W21
    if nwin > 0:
        qe, qb = R.q_trace(0, int(nwin))
        line["quality"]["q_trace_21ms"] = {
            "window_symbols": W21, "windows": int(nwin),
            "q_db": [round(_multi.q_db_from_ber(int(e) / int(b)), 3) if b else None for e, b in zip(qe, qb)],
            "note": "the first window includes the warm-up symbols, which are not counted"}
    # ---- e2e through the public API with host buffers
    # (packed 12-bit input, the ADC's format: 1.5 B per sample over PCIe; u16 reported beside it)
    e_steps = max(5, args.steps)

    def e2e_value(Rx, packed):
        r = e2e_run(torch, Rx, n_step, rec.codes, e_steps, dev, packed=packed)
        e_ms = torch.tensor([r["ms"]], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        return {"value": round(world * n_step * e_steps / (float(e_ms.item()) / 1e3) / 1e9, 3),
                "unit": "GSa/s", "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]}
    Rp = make_pam(input_format=2)
    line["e2e"] = e2e_value(Rp, True)
    line["e2e"]["input"] = "pinned host, RX_IN_U12_PACKED (2 codes per 3 bytes)"
    line["e2e"]["x_paper_realtime"] = round(line["e2e"]["value"] / world / PAPER_REALTIME_GSA, 2)
    Rp.close()
    line["e2e_u16"] = e2e_value(R, False)
    R.close()
    del ring
    torch.cuda.empty_cache()
    # ---- CPU oracle baseline (rank 0, N = 1)
    if world == 1 and not args.no_cpu:
        v, dt, _ = cpu_oracle_rate(rec, rx, rec.n)
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "GSa/s", "cores": 1, "kind": "oracle",
                                "sample": f"one full C2 record ({rec.n} samples, one GPU step), fp64 "
                                          f"numpy oracle, 1 thread, {dt:.1f} s"}
    else:
        line["cpu_baseline"] = None
    # ---- KK-QAM mode (C4) at N = 1
    if world == 1 and not args.no_kk:
        rec4, rx4 = make_config("C4")
        ring4 = tiled_ring(rec4, max(1, int(args.ring_gib * (1 << 30) / 2 // N_C4)) * N_C4, dev)
        def make_kk(**kw):
            return Receiver(RX_QAM_KK, rec4.M, rec4.static_taps, device=local, dc_offset=rec4.dc_offset,
                            history_buffers=CALL_BUFFERS + 2,
                            **({"lms_batch_segments": args.lms_batch} if args.lms_batch else {}),
                            **rx_fields(rx4), **kw)
        R4 = make_kk()
        r4 = run_mode(torch, None, R4, ring4, N_C4, args.kk_steps, 2, 1, dev, None)
        s4 = r4["stats"]
        v4 = N_C4 * args.kk_steps / (r4["ms"] / 1e3) / 1e9
        dom4 = r4["dominant"]
        kk_roof = None
        if dom4 and (dom4["name"] in FLOPS_PER_UNIT or dom4["name"] == "LMS"):
            if dom4["name"] == "LMS":   # 16K flop per complex T/2 symbol + BPS 17 flop per test phase
                f4 = (16 * rx4["lms_taps"] + 17 * rx4["cpr_test_phases"]) * (N_C4 // 4)
            else:
                f4 = FLOPS_PER_UNIT[dom4["name"]] * (N_C4 // 512)
            a4 = f4 * args.kk_steps / (dom4["ms"] / 1e3) / 1e12
            kk_roof = {"kernel_class": dom4["name"], "bound": "alu", "achieved": a4, "peak": peak_fp32,
                       "isolated": isolated_classes(torch, make_kk, ring4, N_C4, rx4, True, dev, peak_fp32, 1),
                       "unit": "TFLOP/s", "frac": a4 / peak_fp32, "share_of_step": dom4["ms"] / r4["ms"]}
        elif dom4:
            kk_roof = {"kernel_class": dom4["name"], "share_of_step": dom4["ms"] / r4["ms"]}
        line["kk"] = {"workload": "C4: KK 64-QAM 1 GBaud 4 sps, 67,106,816 samples/step, CSPR 11 dB, "
                                  "ROADM-filtered, 10 kHz phase noise, 5 MHz CFO, BPS-32 CPR, 8-tap T/2 LMS",
                      "value": round(v4, 3), "unit": "GSa/s", "steps": args.kk_steps,
                      "ms_per_step": round(r4["ms"] / args.kk_steps, 4),
                      "breakdown_ms_per_step": r4["breakdown"], "roofline": kk_roof,
                      "host_enqueue_ms_per_step": round(r4["host_ms"], 4),
                      "gpu_launches": r4["launches"], "clocks": r4["clocks"],
                      "quality": {"ber": s4["bit_errors"] / max(s4["bits"], 1),
                                  "evm_db": 10 * math.log10(s4["evm_num"] / s4["evm_den"]) if s4["evm_den"] > 0 else None}}
        line["gpu_launches"] += r4["launches"]
        R4.close()
        del ring4
        torch.cuda.empty_cache()
    # ---- C3: CSPR sweep (N = 1)
    if world == 1 and not args.no_c3:
        line["c3_sweep"] = c3_sweep(torch, dev, local)
    # ---- C5: 8 mixed channels per GPU, concurrent streams (every N)
    if not args.no_c5:
        line["c5"] = c5_run(torch, dist, rank, world, dev, args.c5_steps, 2, args.ring_gib)
        line["gpu_launches"] += line["c5"]["gpu_launches"]
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
    rec, rx = make_config("C2", seed=2001)
    n = CHUNK
    for _ in range(args.warmup):
        cpu_oracle_rate(rec, rx, n)
    t = 0.0
    for _ in range(args.steps):
        _, dt, _ = cpu_oracle_rate(rec, rx, n)
        t += dt
    v = args.steps * n / t / 1e9
    sample = f"first {n} samples (one 2^22 buffer, P:116) of the C2 record per step, fp64 numpy oracle, 1 thread"
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GSa/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (rxsynth, seeded C2)",
            "config": {"workload": "C2: PAM-16 (bounded sample)", "samples_per_step": n},
            "cpu_baseline": {"value": round(v, 6), "unit": "GSa/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "GSa/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("gpu", "reference"), default="gpu")
    ap.add_argument("--no-kk", action="store_true")
    ap.add_argument("--kk-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--c5-steps", type=int, default=4)
    ap.add_argument("--ring-gib", type=float, default=1.0)
    ap.add_argument("--lms-batch", type=int, default=0,
                    help="segments per equaliser launch (rx_config.lms_batch_segments; 0 = library "
                         "default: D epochs, i.e. 4096 PAM / 2048 KK)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_main(args)
    else:
        gpu_main(args)


if __name__ == "__main__":
    main()
