"""The BASELINE.json configs C1-C5 as concrete generator calls + receiver parameters.

Plain data (SURVEY.md §8(d) "Per-config workloads"); no arithmetic. ``make_config(name,
n_samples=...)`` lets the parity tests shrink a config while keeping its structure.
"""
from __future__ import annotations

from .gen import kk_record, pam_record

# record lengths: 32767*512 keeps waveform and PRBS periodic (SURVEY §8(d) "Record length")
N_C2 = 32767 * 512          # 16,776,704  ("2^24")
N_C4 = 4 * 32767 * 512      # 67,106,816  ("2^26")

CONFIGS = {
    "C1": dict(gen=dict(kind="pam", M=2, n_samples=1 << 16, seed=1001, snr_db=9.0,
                        channel="b2b", ppm=0.0),
               rx=dict(lms_taps=15, lms_block=32, lms_segment=4096, lms_overlap=0,
                       mu=1e-3, train_symbols=4096, sync_start=4096, sync_window=2048,
                       warmup_symbols=0)),
    "C2": dict(gen=dict(kind="pam", M=16, n_samples=N_C2, seed=2001, snr_db=32.0,
                        channel="isi91", ppm=20.0),
               rx=dict(lms_taps=31, lms_block=32, lms_segment=4096, lms_overlap=0,
                       mu=1e-3, train_symbols=32768, sync_start=4096, sync_window=2048,
                       warmup_symbols=65536)),
    "C3": dict(gen=dict(kind="qam", M=4, n_samples=N_C2, seed=3001, cspr_db=6.0,
                        osnr_db=10.0, cfo_hz=20e6, linewidth_hz=100e3, rx_lpf=False),
               rx=dict(lms_taps=4, lms_block=32, lms_segment=4096, lms_overlap=256,
                       mu=2e-3, train_symbols=8192, sync_start=4096, sync_window=2048,
                       cpr_test_phases=0, warmup_symbols=16384)),
    "C4": dict(gen=dict(kind="qam", M=64, n_samples=N_C4, seed=4001, cspr_db=11.0,
                        osnr_db=30.0, cfo_hz=5e6, linewidth_hz=10e3, rx_lpf=False,
                        roadm_b3db=1.5e9),
               rx=dict(lms_taps=8, lms_block=32, lms_segment=4096, lms_overlap=256,
                       mu=2e-3, train_symbols=8192, sync_start=4096, sync_window=2048,
                       cpr_test_phases=32, warmup_symbols=16384)),
}

# C3 sweeps the CSPR (optimum 6 dB for QAM-4 at OSNR 10 dB)
C3_CSPR_DB = (2, 4, 6, 8, 10, 12, 14, 16)

# C5: 8 channels per GPU, C2/C4-style impairments per format (seed 5000 + channel)
C5_FORMATS = (("pam", 2), ("pam", 4), ("pam", 8), ("pam", 16),
              ("qam", 4), ("qam", 16), ("qam", 64), ("qam", 16))


def c5_channel(ch: int, n_samples: int = N_C2):
    fmt, M = C5_FORMATS[ch % 8]
    if fmt == "pam":
        return dict(gen=dict(kind="pam", M=M, n_samples=n_samples, seed=5000 + ch,
                             snr_db=32.0, channel="isi91", ppm=20.0),
                    rx=dict(CONFIGS["C2"]["rx"]))
    rx = dict(CONFIGS["C4"]["rx"])
    rx["cpr_test_phases"] = 0 if M == 4 else 32
    return dict(gen=dict(kind="qam", M=M, n_samples=n_samples, seed=5000 + ch,
                         cspr_db=6.0 if M == 4 else 11.0, osnr_db=30.0, cfo_hz=5e6,
                         linewidth_hz=10e3, rx_lpf=False, roadm_b3db=1.5e9, periodic=True),
                rx=rx)


def make_config(name: str, n_samples: int | None = None, **overrides):
    """Return (Record, rx_params) for config ``name`` (C1..C4 or "C5:<ch>")."""
    if name.startswith("C5:"):
        cfg = c5_channel(int(name[3:]))
    else:
        cfg = CONFIGS[name]
    g = dict(cfg["gen"])
    rx = dict(cfg["rx"])
    if n_samples is not None:
        g["n_samples"] = n_samples
    for k, v in overrides.items():
        if k in rx:
            rx[k] = v
        else:
            g[k] = v
    kind = g.pop("kind")
    rec = pam_record(**g) if kind == "pam" else kk_record(**g)
    return rec, rx
