"""The C-ABI library builds, loads and exports every symbol include/rx.h declares; calls that
need a GPU fail loudly (no CPU fallback). Runs without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2011_13695_b200 import build, rx
    build.build()
    return rx.load()


def _declared_functions():
    out = set()
    for hdr in ("rx.h", "tx.h"):
        src = open(os.path.join(ROOT, "include", hdr)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        out |= set(re.findall(r"\b((?:rx|tx)_[a-z_]+)\s*\(", src))
    return sorted(out)


def test_header_declares_the_north_star_calls():
    fns = _declared_functions()
    for f in ("rx_create", "rx_process", "rx_flush", "rx_get_stats", "rx_destroy"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    for f in _declared_functions():
        assert hasattr(lib, f), f"librx.so does not export {f}"
    from paper_2011_13695_b200 import rx
    assert set(rx.EXPORTS) <= set(_declared_functions())


def test_struct_layout_matches_header(lib):
    """ctypes mirrors must match the C structs (sizes checked against nvcc's layout)."""
    from paper_2011_13695_b200 import rx
    cfg = rx.default_config(rx.RX_PAM, 4)
    assert cfg.fft_size == 1024 and cfg.hop == 512 and cfg.buffer_blocks == 8192
    assert cfg.clock_avg_half == 52 and cfg.lms_block == 32 and cfg.history_buffers == 3
    assert abs(cfg.carrier_offset_hz - 0.547e9) < 1 and cfg.sideband == -1
    assert cfg.prbs_order == 15 and cfg.prbs_seed == 0x7FFF and cfg.sync_start == 4096
    kk = rx.default_config(rx.RX_QAM_KK, 64)
    assert kk.lms_taps == 4 and kk.lms_overlap == 256 and kk.cpr_test_phases == 32
    assert abs(kk.mu - 2e-3) < 1e-15 and abs(kk.sync_min_corr - 0.3) < 1e-15


def test_strerror_and_version(lib):
    assert lib.rx_strerror(0) == b"ok"
    assert b"invalid" in lib.rx_strerror(-1)
    assert lib.rx_version().startswith(b"librx sm_100a")


def test_create_rejects_bad_config_before_touching_the_gpu(lib):
    from paper_2011_13695_b200 import rx
    import numpy as np
    cfg = rx.default_config(rx.RX_PAM, 4)
    taps = np.ones(504)                      # even length -> invalid (A3)
    cfg.static_taps = taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    cfg.n_static_taps = 504
    h = ctypes.c_void_p()
    assert lib.rx_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == -1
    cfg.n_static_taps = 503
    cfg.order = 3
    assert lib.rx_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == -1


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2011_13695_b200 import rx
    import numpy as np
    with pytest.raises(rx.RxError) as e:
        rx.Receiver(rx.RX_PAM, 4, np.ones(503))
    assert e.value.status == -3          # RX_ECUDA: fails loudly


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2011_13695_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|oracle[/\\]|#include.*oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert not pat.search(txt), f


def test_new_config_fields_validated_before_touching_the_gpu(lib):
    """widely_linear (KK only), cpr_anchor, serial_equaliser (0/1), q_window_symbols (a
    multiple of lms_segment) are checked by rx_create before any CUDA call; calibration entry
    points reject wrong families / arguments synchronously."""
    from paper_2011_13695_b200 import rx
    import numpy as np
    taps = np.ones(503)
    h = ctypes.c_void_p()

    def pam():
        c = rx.default_config(rx.RX_PAM, 4)
        c.static_taps = taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        c.n_static_taps = 503
        return c
    for field, bad in (("widely_linear", 1), ("serial_equaliser", 2), ("cpr_anchor", 3),
                       ("q_window_symbols", 4097), ("q_window_symbols", -4096)):
        c = pam()
        setattr(c, field, bad)
        assert lib.rx_create(ctypes.byref(c), 0, ctypes.byref(h)) == -1, field
    c = pam()                                                # a PAM config is not a KK calibration
    cand = np.array([1.0])
    evm = np.zeros(1)
    best = ctypes.c_int(-1)
    dp = ctypes.POINTER(ctypes.c_double)
    assert lib.rx_calibrate_dc(ctypes.byref(c), 0, ctypes.c_void_p(16), 4096, cand.ctypes.data_as(dp), 1,
                               evm.ctypes.data_as(dp), ctypes.byref(best), None) == -1
    thr = np.zeros(3)
    assert lib.rx_calibrate_thresholds(None, 0, 10, thr.ctypes.data_as(dp), None, None) == -1
    e = np.zeros(1, dtype=np.int64)
    lp = ctypes.POINTER(ctypes.c_longlong)
    assert lib.rx_get_q_trace(None, 0, 1, e.ctypes.data_as(lp), e.ctypes.data_as(lp), None) == -1


def test_round2_config_fields_validated_before_touching_the_gpu(lib):
    """lms_mode (0/1), equaliser_lag (0..16) and time sharding (KK only, anchored quadrants,
    shard_count <= tap_lag_epochs, 0 <= shard_index < shard_count) are checked by rx_create
    before any CUDA call; the shard calls reject a NULL handle."""
    from paper_2011_13695_b200 import rx
    import numpy as np
    h = ctypes.c_void_p()
    taps = np.ones(2 * 203)

    def kk(**kw):
        c = rx.default_config(rx.RX_QAM_KK, 16)
        c.static_taps = taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        c.n_static_taps = 203
        for k, v in kw.items():
            setattr(c, k, v)
        return c
    for kw in (dict(lms_mode=3), dict(equaliser_lag=17), dict(equaliser_lag=-1), dict(cuda_graphs=2),
               dict(fused_front_end=2), dict(shard_count=9),   # 9 > D = 8
               dict(shard_count=4, shard_index=4), dict(shard_count=4, shard_index=-1),
               dict(shard_count=4, cpr_anchor=0), dict(shard_count=-1)):
        assert lib.rx_create(ctypes.byref(kk(**kw)), 0, ctypes.byref(h)) == -1, kw
    p = rx.default_config(rx.RX_PAM, 4)
    pt = np.ones(503)
    p.static_taps = pt.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    p.n_static_taps = 503
    p.shard_count = 7
    assert lib.rx_create(ctypes.byref(p), 0, ctypes.byref(h)) == -1           # PAM: N <= D - 2
    lo, hi = ctypes.c_longlong(), ctypes.c_longlong()
    assert lib.rx_shard_halo(None, ctypes.byref(lo), ctypes.byref(hi)) == -1
    n = ctypes.c_int()
    assert lib.rx_carry_size(None, ctypes.byref(n)) == -1
    assert lib.rx_shard_process(None, 0, None, 0, 0, None, 0, None) == -1
    assert lib.rx_export_carry(None, None, None) == -1
    assert lib.rx_import_carry(None, None, 2, 0, None) == -1


def test_struct_sizes_match_a_c_compiler(tmp_path):
    """The ctypes mirrors of rx_config / rx_stats have the C compiler's size and field offsets
    (gcc on include/rx.h), so no field is silently misaligned across the ABI."""
    from paper_2011_13695_b200 import rx
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "rx.h"\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu\\n", sizeof(rx_config), offsetof(rx_config, q_window_symbols),'
                   'offsetof(rx_config, shard_index), sizeof(rx_stats), offsetof(rx_stats, launches));return 0;}\n')
    exe = tmp_path / "sz"
    import subprocess
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    want = [ctypes.sizeof(rx.RxConfig), rx.RxConfig.q_window_symbols.offset, rx.RxConfig.shard_index.offset,
            ctypes.sizeof(rx.RxStats), rx.RxStats.launches.offset]
    assert got == want


def test_tx_struct_layout_and_validation(tmp_path, lib):
    """tx_config (include/tx.h) mirrors the C layout (gcc), and tx_create rejects bad configs
    before touching the GPU (odd / too long shaping FIR, wrong sps, KK with a clock offset)."""
    import subprocess
    import numpy as np
    from paper_2011_13695_b200 import rx
    src = tmp_path / "tx.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "tx.h"\nint main(void){'
                   'printf("%zu %zu %zu\\n", sizeof(tx_config), offsetof(tx_config, noise_sigma),'
                   'offsetof(tx_config, noise_seed));return 0;}\n')
    exe = tmp_path / "tx"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    assert got == [ctypes.sizeof(rx.TxConfig), rx.TxConfig.noise_sigma.offset, rx.TxConfig.noise_seed.offset]
    taps = np.ones(31)
    h = ctypes.c_void_p()
    for kw in (dict(n_shaping_taps=30), dict(n_shaping_taps=515), dict(baud=1e9), dict(order=3),
               dict(adc_full_scale=0.0), dict(family=1, order=16, clock_ppm=5.0)):
        c = rx.TxConfig()
        c.family, c.order, c.baud, c.sample_rate, c.prbs_seed = 0, 4, 2e9, 4e9, 0x7FFF
        c.shaping_taps = taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        c.n_shaping_taps, c.adc_full_scale = 31, 1.0
        for k, v in kw.items():
            setattr(c, k, v)
        if c.family == 1:
            c.baud = 1e9
        assert lib.tx_create(ctypes.byref(c), 0, ctypes.byref(h)) == -1, kw
