"""Thin ctypes binding of librx (include/rx.h) — argument marshalling only.

Every step of the receiver chain runs in librx's CUDA kernels; this module only converts
Python arguments to the C ABI (device pointers from torch tensors, the current CUDA stream).
There is no CPU fallback: if librx.so is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "librx.so")

RX_PAM, RX_QAM_KK = 0, 1
RX_IN_U12_IN_U16, RX_IN_F32, RX_IN_U12_PACKED = 0, 1, 2
PROBES = dict(C=0, TAU=1, MB=2, U=3, UHAT=4, E=5, Z=6, CFO=7, Y=8, LEVEL=9, SEG=10, DEBUG=11)
FLAGS = dict(DOMAIN=1, SYNC=2, DIVERGE=4, CAPACITY=8)

_c_ll = ctypes.c_longlong
_c_dp = ctypes.POINTER(ctypes.c_double)


class RxConfig(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int), ("order", ctypes.c_int),
        ("baud", ctypes.c_double), ("sample_rate", ctypes.c_double),
        ("fft_size", ctypes.c_int), ("hop", ctypes.c_int), ("buffer_blocks", ctypes.c_int),
        ("static_taps", _c_dp), ("n_static_taps", ctypes.c_int),
        ("adc_gain", ctypes.c_double), ("clock_avg_half", ctypes.c_int),
        ("thresholds", _c_dp),
        ("carrier_offset_hz", ctypes.c_double), ("sideband", ctypes.c_int),
        ("dc_offset", ctypes.c_double),
        ("lms_taps", ctypes.c_int), ("lms_block", ctypes.c_int), ("lms_segment", ctypes.c_int),
        ("lms_overlap", ctypes.c_int), ("tap_lag_epochs", ctypes.c_int),
        ("widely_linear", ctypes.c_int),
        ("mu", ctypes.c_double), ("train_symbols", ctypes.c_int),
        ("cfo_enable", ctypes.c_int), ("cpr_test_phases", ctypes.c_int),
        ("cpr_anchor", ctypes.c_int),
        ("prbs_order", ctypes.c_uint), ("prbs_seed", ctypes.c_uint),
        ("sync_start", _c_ll), ("sync_window", ctypes.c_int), ("sync_min_corr", ctypes.c_double),
        ("warmup_symbols", _c_ll), ("history_buffers", ctypes.c_int),
        ("lms_batch_segments", ctypes.c_int),
        ("input_format", ctypes.c_int),
        ("serial_equaliser", ctypes.c_int),
        ("q_window_symbols", _c_ll),
        ("lms_mode", ctypes.c_int),
        ("equaliser_lag", ctypes.c_int),
        ("shard_count", ctypes.c_int), ("shard_index", ctypes.c_int),
        ("cuda_graphs", ctypes.c_int),
        ("fused_front_end", ctypes.c_int),
    ]


class RtStats(ctypes.Structure):
    _fields_ = [("calls", _c_ll), ("samples", _c_ll), ("overruns", _c_ll), ("busy_ms", ctypes.c_double),
                ("max_call_ms", ctypes.c_double), ("max_load", ctypes.c_double), ("realtime_ratio", ctypes.c_double)]


class TxConfig(ctypes.Structure):
    """include/tx.h tx_config (GPU transmitter + channel simulator)."""
    _fields_ = [
        ("family", ctypes.c_int), ("order", ctypes.c_int),
        ("baud", ctypes.c_double), ("sample_rate", ctypes.c_double),
        ("prbs_seed", ctypes.c_uint), ("symbol_offset", _c_ll),
        ("shaping_taps", _c_dp), ("n_shaping_taps", ctypes.c_int),
        ("clock_ppm", ctypes.c_double), ("tone_amp", ctypes.c_double), ("carrier_hz", ctypes.c_double),
        ("cfo_hz", ctypes.c_double), ("linewidth_hz", ctypes.c_double),
        ("iq_re", ctypes.c_double), ("iq_im", ctypes.c_double), ("noise_sigma", ctypes.c_double),
        ("adc_mean", ctypes.c_double), ("adc_full_scale", ctypes.c_double),
        ("noise_seed", ctypes.c_ulonglong),
    ]


class RxStats(ctypes.Structure):
    _fields_ = [
        ("samples_in", _c_ll), ("symbols_out", _c_ll),
        ("bit_errors", _c_ll), ("bits", _c_ll), ("symbols_counted", _c_ll),
        ("clipped", _c_ll), ("domain_errors", _c_ll), ("first_domain_error_index", _c_ll),
        ("evm_num", ctypes.c_double), ("evm_den", ctypes.c_double),
        ("sync_offset", ctypes.c_int), ("sync_phase", ctypes.c_int),
        ("sync_polarity", ctypes.c_int), ("synced", ctypes.c_int),
        ("sync_gamma", ctypes.c_double), ("sync_phi0", ctypes.c_double),
        ("status_flags", ctypes.c_int), ("launches", _c_ll),
    ]


EXPORTS = ("rx_config_default", "rx_create", "rx_process", "rx_flush", "rx_get_stats",
           "rx_reset_stats", "rx_get_taps", "rx_probe_read", "rx_destroy", "rx_strerror",
           "rx_version", "rx_profile_enable", "rx_profile_read", "rx_export_counters",
           "rx_set_taps", "rx_get_q_trace", "rx_calibrate_thresholds", "rx_calibrate_dc",
           "rx_design_static_eq", "rx_shard_process", "rx_shard_halo", "rx_carry_size", "rx_export_carry",
           "rx_import_carry", "rx_rt_enable", "rx_get_rt_stats", "tx_create", "tx_generate", "tx_destroy")
SHARD_PRE, SHARD_POST = 4096, 4096       # RX_SHARD_PRE / RX_SHARD_POST (include/rx.h; KK halos)
NCOUNTERS = 8
COUNTERS = ("bit_errors", "bits", "symbols_counted", "evm_num", "evm_den", "clipped",
            "domain_errors", "symbols_out")
KCLASSES = ("PAM_FE", "PAM_CLOCK", "PAM_BE", "NORM", "KK_S1", "KK_S2", "CFO", "SYNC", "LMS",
            "LMS_POST", "MISC", "KK_FE")

_lib = None


def load(path: str = SO_PATH):
    """Load librx.so (raises OSError if it is missing — no fallback). RX_SO overrides the path
    (kernel-variant experiments, tools/kk_variants.py)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("RX_SO", path)
    if not os.path.exists(path):
        raise OSError(f"librx.so not built at {path}; run paper_2011_13695_b200.build.build()")
    lib = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    lib.rx_config_default.argtypes = [ctypes.POINTER(RxConfig), ctypes.c_int, ctypes.c_int]
    lib.rx_config_default.restype = None
    lib.rx_create.argtypes = [ctypes.POINTER(RxConfig), ctypes.c_int, ctypes.POINTER(vp)]
    lib.rx_process.argtypes = [vp, vp, _c_ll, vp, _c_ll, vp]
    lib.rx_flush.argtypes = [vp, vp, _c_ll, vp]
    lib.rx_get_stats.argtypes = [vp, ctypes.POINTER(RxStats), vp]
    lib.rx_reset_stats.argtypes = [vp, vp]
    lib.rx_get_taps.argtypes = [vp, _c_dp, ctypes.c_int]
    lib.rx_set_taps.argtypes = [vp, _c_dp, ctypes.c_int]
    lib.rx_probe_read.argtypes = [vp, ctypes.c_int, _c_ll, _c_ll, vp, vp]
    lib.rx_destroy.argtypes = [vp]
    lib.rx_destroy.restype = None
    lib.rx_strerror.argtypes = [ctypes.c_int]
    lib.rx_strerror.restype = ctypes.c_char_p
    lib.rx_version.argtypes = []
    lib.rx_version.restype = ctypes.c_char_p
    lib.rx_profile_enable.argtypes = [vp, ctypes.c_int]
    lib.rx_export_counters.argtypes = [vp, vp, vp]
    lib.rx_export_counters.restype = ctypes.c_int
    lib.rx_profile_read.argtypes = [vp, _c_dp, ctypes.POINTER(_c_ll), ctypes.c_int]
    lib.rx_get_q_trace.argtypes = [vp, _c_ll, ctypes.c_int, ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll), vp]
    lib.rx_get_q_trace.restype = ctypes.c_int
    lib.rx_calibrate_thresholds.argtypes = [vp, _c_ll, _c_ll, _c_dp, _c_dp, vp]
    lib.rx_calibrate_thresholds.restype = ctypes.c_int
    lib.rx_calibrate_dc.argtypes = [ctypes.POINTER(RxConfig), ctypes.c_int, vp, _c_ll, _c_dp, ctypes.c_int,
                                    _c_dp, ctypes.POINTER(ctypes.c_int), vp]
    lib.rx_calibrate_dc.restype = ctypes.c_int
    lib.rx_design_static_eq.argtypes = [_c_dp, _c_dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _c_dp]
    lib.rx_design_static_eq.restype = ctypes.c_int
    lib.rx_shard_process.argtypes = [vp, _c_ll, vp, _c_ll, ctypes.c_int, vp, _c_ll, vp]
    lib.rx_carry_size.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    lib.rx_shard_halo.argtypes = [vp, ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll)]
    lib.rx_export_carry.argtypes = [vp, vp, vp]
    lib.rx_import_carry.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, vp]
    for f in ("rx_shard_process", "rx_shard_halo", "rx_carry_size", "rx_export_carry", "rx_import_carry"):
        getattr(lib, f).restype = ctypes.c_int
    lib.rx_rt_enable.argtypes = [vp, ctypes.c_int]
    lib.rx_rt_enable.restype = ctypes.c_int
    lib.rx_get_rt_stats.argtypes = [vp, ctypes.POINTER(RtStats)]
    lib.rx_get_rt_stats.restype = ctypes.c_int
    lib.tx_create.argtypes = [ctypes.POINTER(TxConfig), ctypes.c_int, ctypes.POINTER(vp)]
    lib.tx_create.restype = ctypes.c_int
    lib.tx_generate.argtypes = [vp, vp, _c_ll, vp]
    lib.tx_generate.restype = ctypes.c_int
    lib.tx_destroy.argtypes = [vp]
    lib.tx_destroy.restype = None
    for f in ("rx_create", "rx_process", "rx_flush", "rx_get_stats", "rx_reset_stats",
              "rx_get_taps", "rx_set_taps", "rx_probe_read", "rx_profile_enable", "rx_profile_read"):
        getattr(lib, f).restype = ctypes.c_int
    _lib = lib
    return lib


class RxError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: librx status {status} ({load().rx_strerror(status).decode()})")
        self.status = status


def _check(st: int, where: str):
    if st != 0:
        raise RxError(st, where)


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def default_config(family: int, order: int) -> RxConfig:
    cfg = RxConfig()
    load().rx_config_default(ctypes.byref(cfg), family, order)
    return cfg


class Receiver:
    """One receiver channel (one librx handle) on one CUDA device.

    Receiver(family, order, static_taps, device=0, **rx_config fields)
    """

    def __init__(self, family: int, order: int, static_taps, device: int = 0,
                 thresholds=None, **fields):
        lib = load()
        cfg = default_config(family, order)
        taps = np.ascontiguousarray(np.asarray(static_taps))
        if family == RX_QAM_KK:
            taps = np.ascontiguousarray(np.stack([taps.real, taps.imag], axis=-1).reshape(-1),
                                        dtype=np.float64)
            cfg.n_static_taps = taps.shape[0] // 2
        else:
            taps = np.ascontiguousarray(taps.real, dtype=np.float64)
            cfg.n_static_taps = taps.shape[0]
        self._taps = taps
        cfg.static_taps = taps.ctypes.data_as(_c_dp)
        if thresholds is not None:
            self._thr = np.ascontiguousarray(thresholds, dtype=np.float64)
            cfg.thresholds = self._thr.ctypes.data_as(_c_dp)
        for k, v in fields.items():
            if not hasattr(cfg, k):
                raise TypeError(f"unknown rx_config field {k}")
            setattr(cfg, k, v)
        self.cfg = cfg
        self.device = device
        h = ctypes.c_void_p()
        _check(lib.rx_create(ctypes.byref(cfg), device, ctypes.byref(h)), "rx_create")
        self._h = h
        self.family, self.order = family, order

    # -- streaming
    def process(self, samples, labels=None, stream=None):
        """samples: torch uint16/int16 CUDA tensor of u12 codes (RX_IN_U12_IN_U16), float32
        (RX_IN_F32) or uint8 bytes of packed 12-bit codes (RX_IN_U12_PACKED, 3 bytes per 2
        samples), per the handle's input_format; labels: uint8 CUDA tensor written at index
        m % len(labels)."""
        fmt = self.cfg.input_format
        want = {RX_IN_F32: 4, RX_IN_U12_PACKED: 1}.get(fmt, 2)
        if samples.element_size() != want:
            raise ValueError(f"input_format {fmt} needs {want}-byte elements")
        n = samples.numel() * 2 // 3 if fmt == RX_IN_U12_PACKED else samples.numel()
        lp, lc = (labels.data_ptr(), labels.numel()) if labels is not None else (None, 0)
        _check(load().rx_process(self._h, ctypes.c_void_p(samples.data_ptr()), n,
                                 ctypes.c_void_p(lp), lc, _stream_ptr(stream)), "rx_process")

    def process_ptr(self, ptr: int, n: int, labels_ptr: int = 0, labels_cap: int = 0, stream_ptr=None):
        _check(load().rx_process(self._h, ctypes.c_void_p(ptr), n, ctypes.c_void_p(labels_ptr),
                                 labels_cap, stream_ptr if stream_ptr is not None else _stream_ptr()),
               "rx_process")

    # -- time sharding of one stream (SURVEY §8(e) mode 2; include/rx.h rx_shard_process)
    def shard_process(self, buffer: int, samples, last: bool = False, labels=None, stream=None):
        """Stage A of paper buffer `buffer` (owned by this shard): `samples` = u16 codes of
        [max(0, buffer B4 - pre), (buffer + 1) B4 + post) of the stream, (pre, post) =
        shard_halo()."""
        lp, lc = (labels.data_ptr(), labels.numel()) if labels is not None else (None, 0)
        _check(load().rx_shard_process(self._h, int(buffer), ctypes.c_void_p(samples.data_ptr()),
                                       int(samples.numel()), int(bool(last)), ctypes.c_void_p(lp), lc,
                                       _stream_ptr(stream)), "rx_shard_process")

    def shard_halo(self) -> tuple[int, int]:
        """Input halos (samples before / after a buffer) its shard reads (rx_shard_halo)."""
        a, b = _c_ll(), _c_ll()
        _check(load().rx_shard_halo(self._h, ctypes.byref(a), ctypes.byref(b)), "rx_shard_halo")
        return a.value, b.value

    def carry_size(self) -> int:
        n = ctypes.c_int()
        _check(load().rx_carry_size(self._h, ctypes.byref(n)), "rx_carry_size")
        return n.value

    def export_carry(self, out, stream=None):
        """This round's carry record into `out` (uint8 CUDA tensor of carry_size() bytes)."""
        _check(load().rx_export_carry(self._h, ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
               "rx_export_carry")

    def import_carry(self, gathered, n_ranks: int, my_rank: int, stream=None):
        """All shards' records (rank order, one CUDA buffer): carries + the previous buffer's
        equaliser stage."""
        _check(load().rx_import_carry(self._h, ctypes.c_void_p(gathered.data_ptr()), int(n_ranks), int(my_rank),
                                      _stream_ptr(stream)), "rx_import_carry")

    def flush(self, labels=None, stream=None):
        lp, lc = (labels.data_ptr(), labels.numel()) if labels is not None else (None, 0)
        _check(load().rx_flush(self._h, ctypes.c_void_p(lp), lc, _stream_ptr(stream)), "rx_flush")

    def stats(self, stream=None) -> dict:
        st = RxStats()
        _check(load().rx_get_stats(self._h, ctypes.byref(st), _stream_ptr(stream)), "rx_get_stats")
        return {k: getattr(st, k) for k, _ in RxStats._fields_}

    def calibrate_thresholds(self, first: int, count: int, stream=None):
        """PAM decision thresholds from the equaliser output of finalised symbols
        [first, first + count) (rx_calibrate_thresholds): (thresholds [M-1], level means [M])."""
        thr = np.zeros(self.order - 1, dtype=np.float64)
        means = np.zeros(self.order, dtype=np.float64)
        _check(load().rx_calibrate_thresholds(self._h, first, count, thr.ctypes.data_as(_c_dp),
                                              means.ctypes.data_as(_c_dp), _stream_ptr(stream)),
               "rx_calibrate_thresholds")
        return thr, means

    def q_trace(self, first: int, n: int, stream=None):
        """Windowed (bit_errors, bits) of Q-trace windows [first, first + n) (rx_get_q_trace)."""
        err = np.zeros(n, dtype=np.int64)
        bits = np.zeros(n, dtype=np.int64)
        _check(load().rx_get_q_trace(self._h, first, n, err.ctypes.data_as(ctypes.POINTER(_c_ll)),
                                     bits.ctypes.data_as(ctypes.POINTER(_c_ll)), _stream_ptr(stream)),
               "rx_get_q_trace")
        return err, bits

    def export_counters(self, out, stream=None):
        """Enqueue a device copy of the counters into `out` (float64 CUDA tensor, >= 8)."""
        _check(load().rx_export_counters(self._h, ctypes.c_void_p(out.data_ptr()),
                                         _stream_ptr(stream)), "rx_export_counters")

    def reset_stats(self, stream=None):
        _check(load().rx_reset_stats(self._h, _stream_ptr(stream)), "rx_reset_stats")

    def train_taps(self) -> np.ndarray:
        """W_train (K real / complex); widely linear: (W_train, V_train)."""
        K = self.cfg.lms_taps
        wl = self.family == RX_QAM_KK and self.cfg.widely_linear
        n = (4 if wl else 2) * K if self.family == RX_QAM_KK else K
        out = np.zeros(n, dtype=np.float64)
        _check(load().rx_get_taps(self._h, out.ctypes.data_as(_c_dp), n), "rx_get_taps")
        if self.family != RX_QAM_KK:
            return out
        c = out[0::2] + 1j * out[1::2]
        return (c[:K], c[K:]) if wl else c

    def set_taps(self, w) -> None:
        """Start taps of the training pass (rx_set_taps); K real (PAM) or K complex (KK)."""
        w = np.asarray(w)
        if self.family == RX_QAM_KK:
            buf = np.empty(2 * w.size, dtype=np.float64)
            buf[0::2], buf[1::2] = w.real, w.imag
        else:
            buf = np.ascontiguousarray(w.real, dtype=np.float64)
        _check(load().rx_set_taps(self._h, buf.ctypes.data_as(_c_dp), int(buf.size)), "rx_set_taps")

    def probe(self, which: str, first: int, count: int, stream=None) -> np.ndarray:
        w = PROBES[which]
        dt, per = {
            "C": (np.float64, 2), "TAU": (np.float64, 1), "MB": (np.int64, 1), "U": (np.float32, 1),
            "UHAT": (np.float32, 1), "E": (np.float32, 2), "Z": (np.float32, 2), "CFO": (np.float64, 5),
            "Y": (np.float32, 2), "LEVEL": (np.uint8, 1), "SEG": (np.float64, 6), "DEBUG": (np.int64, 1),
        }[which]
        out = np.zeros(count * per, dtype=dt)
        _check(load().rx_probe_read(self._h, w, first, count, out.ctypes.data_as(ctypes.c_void_p),
                                    _stream_ptr(stream)), f"rx_probe_read({which})")
        if which in ("C", "E", "Z", "Y"):
            out = out.reshape(count, 2)
            return out[:, 0].astype(np.float64) + 1j * out[:, 1]
        if per > 1:
            return out.reshape(count, per)
        return out

    def rt_enable(self, on: bool = True):
        """Real-time monitor (rx_rt_enable): time every later rx_process call on its stream."""
        _check(load().rx_rt_enable(self._h, int(bool(on))), "rx_rt_enable")

    def rt_stats(self) -> dict:
        """rx_get_rt_stats: calls, samples, busy_ms, max_call_ms, max_load, overruns,
        realtime_ratio since the last read."""
        st = RtStats()
        _check(load().rx_get_rt_stats(self._h, ctypes.byref(st)), "rx_get_rt_stats")
        return {k: getattr(st, k) for k, _ in RtStats._fields_}

    def profile_enable(self, classes=KCLASSES):
        mask = 0
        for c in classes:
            mask |= 1 << KCLASSES.index(c)
        _check(load().rx_profile_enable(self._h, mask), "rx_profile_enable")

    def profile_read(self) -> dict:
        n = len(KCLASSES)
        ms = (ctypes.c_double * n)()
        cnt = (_c_ll * n)()
        _check(load().rx_profile_read(self._h, ms, cnt, n), "rx_profile_read")
        return {KCLASSES[i]: (ms[i], cnt[i]) for i in range(n) if cnt[i]}

    def close(self):
        if getattr(self, "_h", None):
            load().rx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def calibrate_dc(order: int, static_taps, samples, candidates, device: int = 0, stream=None, **fields):
    """KK DC-offset grid search through the chain (rx_calibrate_dc): ``samples`` is a
    device tensor holding the calibration record; returns (EVM dB per candidate, best index)."""
    lib = load()
    cfg = default_config(RX_QAM_KK, order)
    taps = np.asarray(static_taps)
    buf = np.ascontiguousarray(np.stack([taps.real, taps.imag], axis=-1).reshape(-1), dtype=np.float64)
    cfg.static_taps = buf.ctypes.data_as(_c_dp)
    cfg.n_static_taps = buf.shape[0] // 2
    for k, v in fields.items():
        if not hasattr(cfg, k):
            raise TypeError(f"unknown rx_config field {k}")
        setattr(cfg, k, v)
    cand = np.ascontiguousarray(candidates, dtype=np.float64)
    evm = np.zeros(cand.shape[0], dtype=np.float64)
    best = ctypes.c_int(-1)
    _check(lib.rx_calibrate_dc(ctypes.byref(cfg), device, ctypes.c_void_p(samples.data_ptr()),
                               int(samples.numel()), cand.ctypes.data_as(_c_dp), int(cand.shape[0]),
                               evm.ctypes.data_as(_c_dp), ctypes.byref(best), _stream_ptr(stream)),
           "rx_calibrate_dc")
    return evm, best.value


def design_static_eq(h_channel, h_target, lam: float, n_taps: int, real_taps: bool):
    """Static-equaliser design (rx_design_static_eq; host only): 1024-bin complex responses in,
    n_taps zero-phase taps out (real for PAM, complex for KK)."""
    lib = load()

    def inter(h):
        h = np.asarray(h, dtype=np.complex128)
        return np.ascontiguousarray(np.stack([h.real, h.imag], axis=-1).reshape(-1))
    a, b = inter(h_channel), inter(h_target)
    out = np.zeros(n_taps if real_taps else 2 * n_taps, dtype=np.float64)
    _check(lib.rx_design_static_eq(a.ctypes.data_as(_c_dp), b.ctypes.data_as(_c_dp), float(lam), int(n_taps),
                                   int(bool(real_taps)), out.ctypes.data_as(_c_dp)), "rx_design_static_eq")
    return out if real_taps else out[0::2] + 1j * out[1::2]


class Transmitter:
    """GPU transmitter + channel simulator (include/tx.h): generates the 12-bit
    ADC stream of the paper's PAM / KK-QAM set-ups on the device.

    Transmitter(family, order, shaping_taps, device=0, **tx_config fields)"""

    def __init__(self, family: int, order: int, shaping_taps, device: int = 0, **fields):
        lib = load()
        cfg = TxConfig()
        cfg.family, cfg.order = family, order
        cfg.baud = 2e9 if family == RX_PAM else 1e9
        cfg.sample_rate = 4e9
        cfg.prbs_seed = 0x7FFF
        cfg.carrier_hz = 0.547e9
        cfg.adc_full_scale = 1.0
        taps = np.asarray(shaping_taps)
        if family == RX_QAM_KK:
            buf = np.ascontiguousarray(np.stack([taps.real, taps.imag], axis=-1).reshape(-1), dtype=np.float64)
            cfg.n_shaping_taps = buf.shape[0] // 2
        else:
            buf = np.ascontiguousarray(taps.real, dtype=np.float64)
            cfg.n_shaping_taps = buf.shape[0]
        self._taps = buf
        cfg.shaping_taps = buf.ctypes.data_as(_c_dp)
        for k, v in fields.items():
            if not hasattr(cfg, k):
                raise TypeError(f"unknown tx_config field {k}")
            setattr(cfg, k, v)
        self.cfg = cfg
        h = ctypes.c_void_p()
        _check(lib.tx_create(ctypes.byref(cfg), device, ctypes.byref(h)), "tx_create")
        self._h = h

    def generate(self, out, stream=None):
        """Fill `out` (uint16 / int16 CUDA tensor, length a multiple of 512) with the next codes."""
        _check(load().tx_generate(self._h, ctypes.c_void_p(out.data_ptr()), int(out.numel()), _stream_ptr(stream)),
               "tx_generate")

    def close(self):
        if getattr(self, "_h", None):
            load().tx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
