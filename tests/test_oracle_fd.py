"""Pins of the oracle's FD / framing / Hilbert / KK / DDS steps (CPU only).

Each test checks the oracle against something other than itself: a brute-force
definition (oracle/brute.py), a closed form, or an invariant — SURVEY.md §8(c)
"What pins each part".
"""
import math

import numpy as np
import pytest

from oracle import brute
from oracle import rx_oracle as O


def test_dft_matches_direct_definition():
    rng = np.random.default_rng(1)
    x = rng.normal(size=1024) + 1j * rng.normal(size=1024)
    X = np.fft.fft(x)
    Xd = brute.dft_direct(x)
    assert np.max(np.abs(X - Xd)) / np.max(np.abs(Xd)) < 1e-12
    # round trip and Hermitian symmetry of a real input
    xr = rng.normal(size=1024)
    Xr = brute.dft_direct(xr)
    assert np.allclose(Xr[1:][::-1], np.conj(Xr[1:]), atol=1e-9)
    assert np.max(np.abs(brute.idft_direct(Xr) - xr)) < 1e-11


def test_zero_phase_spectrum_is_real_for_symmetric_taps_and_matches_direct_dft():
    rng = np.random.default_rng(2)
    half = 251
    t = rng.normal(size=half + 1)
    taps = np.concatenate([t[::-1], t[1:]])               # symmetric, odd length 503
    H = O.zero_phase_spectrum(taps)
    hc = np.zeros(1024)
    for n in range(-half, half + 1):
        hc[n % 1024] = taps[half + n]
    assert np.max(np.abs(H - brute.dft_direct(hc))) < 1e-10
    assert np.max(np.abs(H.imag)) < 1e-10                  # zero-phase => real spectrum
    with pytest.raises(ValueError):
        O.zero_phase_spectrum(np.ones(515))
    with pytest.raises(ValueError):
        O.zero_phase_spectrum(np.ones(10))


@pytest.mark.parametrize("L", [1, 31, 503, 513])
def test_overlap_save_block_filter_equals_linear_convolution(L):
    """c-0 / A3: with zero-phase taps (L <= 513) and the central keep window, block FD
    filtering equals y_p = sum h[n] x_{p-n} exactly."""
    rng = np.random.default_rng(L)
    x = rng.normal(size=512 * 12)
    taps = rng.normal(size=L)
    Y, _ = O.pam_fd(x, taps)
    p_all, y_all = [], []
    for b in range(Y.shape[0]):
        y = np.fft.ifft(Y[b]).real
        p = np.arange(512 * b - 256, 512 * b + 256)
        ok = p >= 0
        p_all.append(p[ok]); y_all.append(y[256:768][ok])
    p = np.concatenate(p_all); y = np.concatenate(y_all)
    ref = brute.conv_direct(x, taps, p)
    assert np.max(np.abs(y - ref)) < 1e-11 * max(1, np.max(np.abs(ref)))
    # stream coverage: kept windows tile [0, 512 nb - 256) exactly once
    assert np.array_equal(p, np.arange(512 * Y.shape[0] - 256))


def test_clock_estimate_definition_matches_direct_sum():
    rng = np.random.default_rng(3)
    x = rng.normal(size=4096)
    taps = np.array([0.25, 0.5, 0.25])
    Y, C = O.pam_fd(x, taps)
    for b in range(Y.shape[0]):
        Yf = brute.dft_direct(O.frames(x, b, b + 1)[0]) * O.zero_phase_spectrum(taps)
        direct = sum(Yf[k] * np.conj(Yf[k + 512]) for k in range(512))
        assert abs(C[b] - direct) <= 1e-9 * abs(direct)


def test_hilbert_of_cosine_is_sine():
    """P:218 FD Hilbert: H{cos(2 pi k0 n/N)} = sin(2 pi k0 n/N) for an integer bin k0."""
    n = np.arange(1024)
    for k0 in (1, 37, 255, 511):
        ph = O.block_hilbert(np.cos(2 * math.pi * k0 * n / 1024))
        assert np.max(np.abs(ph - np.sin(2 * math.pi * k0 * n / 1024))) < 1e-12
    # DC and Nyquist are removed (A8)
    assert np.max(np.abs(O.block_hilbert(np.ones(1024)))) < 1e-14
    assert np.max(np.abs(O.block_hilbert((-1.0) ** n))) < 1e-14


def test_hilbert_equals_td_cot_kernel_and_is_an_anti_involution():
    rng = np.random.default_rng(4)
    h = rng.normal(size=1024)
    ph = O.block_hilbert(h)
    td = brute.hilbert_circular_td(h)
    assert np.max(np.abs(ph - td)) < 1e-11
    # H{H{x}} = -x for x without DC / Nyquist content
    x = h - h.mean()
    X = np.fft.fft(x); X[512] = 0; x = np.fft.ifft(X).real
    assert np.max(np.abs(O.block_hilbert(O.block_hilbert(x)) + x)) < 1e-12


def _min_phase_field(sigma, K=16, A=1.0, total=0.6, seed=0, n=512 * 8):
    rng = np.random.default_rng(seed)
    c = rng.normal(size=K) + 1j * rng.normal(size=K)
    c *= total * A / np.sum(np.abs(c))
    p = np.arange(n)
    E = A + sum(c[k - 1] * np.exp(1j * sigma * 2 * math.pi * k * p / 1024) for k in range(1, K + 1))
    return E


@pytest.mark.parametrize("sigma", [-1, +1])
def test_kk_exact_on_periodic_minimum_phase_field(sigma):
    """c-6 exact special case: a 1024-periodic one-sided field
    A + sum c_k e^{j sigma 2 pi k n/N}, sum|c_k| <= 0.6 A, is recovered exactly by
    sqrt(I) e^{j sigma H{1/2 ln I}}; the wrong sideband errs by >= 0.3."""
    E = _min_phase_field(sigma)
    I = np.abs(E) ** 2
    dc = 2.0
    Er, dom, _ = O.kk_stage1(I - dc, dc, carrier_hz=0.0, sideband=sigma, fs=4e9)
    assert dom == 0
    p = np.arange(768, Er.shape[0])                     # blocks >= 2: no zero-padding
    err = np.max(np.abs(Er[p] - E[p]))
    assert err < 1e-12
    Ew, _, _ = O.kk_stage1(I - dc, dc, carrier_hz=0.0, sideband=-sigma, fs=4e9)
    assert np.max(np.abs(Ew[p] - E[p])) > 0.3


def test_kk_domain_errors_are_counted_and_clamped():
    x = np.full(2048, 0.5)
    x[1000] = -3.0
    x[1500] = -2.0
    E, dom, first = O.kk_stage1(x, 1.0, 0.0, -1, 4e9)
    assert dom == 2 and first == 1000
    assert np.all(np.isfinite(E))


def test_downshift_is_a_pure_tone_with_exact_integer_phase():
    """Constant intensity I = 1 -> E_p = e^{-j psi(p; sigma f_c)} = e^{+j 2 pi f_c p / f_s}
    for sigma = -1. f_c/f_s = 547/4000 exactly, so the reference phase is computed
    from the integer (547 p) mod 4000 — independent of the 64-bit DDS."""
    n = 512 * 40
    E, _, _ = O.kk_stage1(np.zeros(n), 1.0, 0.547e9, -1, 4e9)
    p = np.arange(E.shape[0])
    ref = np.exp(2j * math.pi * ((547 * p) % 4000) / 4000.0)
    assert np.max(np.abs(E - ref)) < 1e-9
    # far into a stream the DDS stays exact (fp32 p*f/fs would be off by O(1) rad)
    # (inc approximates 547/4000 * 2^64 to ~2^8 units, i.e. 1e-14 rad/sample of drift)
    p_big = np.array([2 ** 31 + 12345], dtype=np.int64)
    w = O.dds_words(p_big, O.dds_increment(-0.547e9, 4e9))
    ph = O.dds_phase(w)[0]
    ref_ph = -2 * math.pi * ((547 * int(p_big[0])) % 4000) / 4000.0
    assert abs(math.remainder(ph - ref_ph, 2 * math.pi)) < 1e-5


def test_dds_increment_is_twos_complement_and_exact():
    inc = O.dds_increment(-0.547e9, 4e9)
    assert inc == (1 << 64) - round(0.13675 * 2 ** 64)
    assert O.dds_increment(1e9, 4e9) == 1 << 62


def test_stage2_equals_convolution_then_decimation_for_band_limited_field():
    """c-7 plain definition: with G vanishing outside kappa in [-256, 255] the decimating
    512-point IFFT equals z_q = sum_n h2[n] E_{2q-n}."""
    rng = np.random.default_rng(5)
    n = 512 * 12
    p = np.arange(n)
    E = np.zeros(n, dtype=np.complex128)
    for k in rng.integers(-200, 200, size=12):
        E += (rng.normal() + 1j * rng.normal()) * np.exp(2j * math.pi * k * p / 1024)
    taps2 = (rng.normal(size=203) + 1j * rng.normal(size=203)) * np.hanning(203)
    nb = n // 512
    z = O.kk_stage2(E, taps2, nb)
    q = np.arange(256 * 3, z.shape[0])                  # away from the p < 0 padding
    ref = brute.conv_direct(E, taps2, 2 * q)
    # the periodic E is exactly band-limited inside each frame only when the frame holds
    # whole periods: frames are 1024 long, E is 1024-periodic -> exact
    assert np.max(np.abs(z[q] - ref)) < 1e-10 * np.max(np.abs(ref))


def test_kk_reconstruction_fidelity_improves_with_cspr():
    """SPEC acceptance 11 (the reason for the CSPR trade-off of Fig. 7): noiseless,
    phase-noise-free SSB 16-QAM after square-law detection and the 12-bit ADC; the oracle's KK
    stage 1 (c-6) reconstructs the data field s = sqrt(fs) E - A e^{j 2 pi f_c p} with an error
    that strictly decreases over CSPR {3, 6, 9, 12, 15, 20} dB, below -25 dB at 20 dB (the
    generator's transmitted field is the reference)."""
    import math
    from rxsynth import gen
    evm = []
    for cspr in (3, 6, 9, 12, 15, 20):
        rec = gen.kk_record(16, 1 << 16, seed=5, cspr_db=cspr, osnr_db=None, keep_field=True)
        x, _ = O.ingest(rec.codes)
        E, _, _ = O.kk_stage1(x, rec.dc_offset, 0.547e9, -1, 4e9)
        fs, A = rec.meta["full_scale"], rec.meta["tone_amp"]
        n = np.arange(E.shape[0])
        s_rec = math.sqrt(fs) * E - A * np.exp(2j * math.pi * 0.547e9 / 4e9 * n)
        s = rec.meta["field"][:E.shape[0]]
        mid = slice(4096, E.shape[0] - 4096)
        evm.append(10 * math.log10(np.mean(np.abs(s_rec[mid] - s[mid]) ** 2) / np.mean(np.abs(s[mid]) ** 2)))
    assert all(b < a for a, b in zip(evm, evm[1:])), evm
    assert evm[-1] < -25, evm
