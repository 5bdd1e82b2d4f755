"""Pins of the oracle's PAM clock recovery, extraction and normalisation (CPU only).

SURVEY.md §8(c) pins: known fractional delay -> tau (A13, App. A-5); unwrap closed forms
(S:324-325); extraction under clock offset (A16, App. A-6); normalisation.
"""
import math

import numpy as np
import pytest

from oracle import rx_oracle as O
from rxsynth import gen


def _pam2_waveform(nsym, delay_sym=0.0, seed=0):
    """Noiseless 2-sps PAM-2 RRC(0.5) waveform delayed by delay_sym symbols (test-local)."""
    rng = np.random.default_rng(seed)
    a = rng.choice([-1.0, 1.0], size=nsym)
    n = 2 * nsym
    up = np.zeros(n)
    up[::2] = a
    f = np.fft.fftfreq(n, d=0.5)                 # in units of the baud rate
    F = np.fft.fft(up) * math.sqrt(2) * gen.rrc_amp(f, 0.5)
    F *= np.exp(-2j * math.pi * f * delay_sym)   # delay by d symbols
    return np.fft.ifft(F).real, a


@pytest.mark.parametrize("d", [0.0, 0.1, 0.25, -0.25, 0.4])
def test_clock_estimator_recovers_known_fractional_delay(d):
    """H3/H4 (A13): a signal delayed by d symbols gives tau = d (|err| <= 2e-3)."""
    x, _ = _pam2_waveform(512 * 64, d)
    taps = gen.static_taps_pam()
    _, C = O.pam_fd(x, taps)
    ck = O.clock_phase(C)
    tau = ck["tau"][60:-60]
    assert np.max(np.abs(tau - d)) < 2e-3


def test_average_and_unwrap_closed_forms():
    # constant C -> constant theta, tau
    C = np.full(300, 2.0 * np.exp(1j * 0.3))
    ck = O.clock_phase(C)
    assert np.allclose(ck["theta_u"], 0.3, atol=1e-14)
    # truncated window at the edges: Cbar_0 = sum of C_0..C_52 (53 terms)
    assert abs(ck["Cbar"][0] - 53 * C[0]) < 1e-12
    assert abs(ck["Cbar"][150] - 105 * C[0]) < 1e-12
    # wrapped [3.1, -3.1] -> [3.1, 3.1832]
    ck = O.clock_phase(np.exp(1j * np.array([3.1, -3.1])), half=0)
    assert np.allclose(ck["theta_u"], [3.1, 2 * math.pi - 3.1], atol=1e-12)
    # equals numpy's own unwrap on a random walk
    rng = np.random.default_rng(0)
    ph = np.cumsum(rng.normal(0, 0.8, size=5000))
    ck = O.clock_phase(np.exp(1j * ph), half=0)
    assert np.allclose(ck["theta_u"], np.unwrap(np.angle(np.exp(1j * ph))), atol=1e-10)
    # |Cbar| = 0 inherits the previous phase
    C = np.exp(1j * np.array([0.5, 0.7, 0.0, 0.9]))
    C[2] = 0
    ck = O.clock_phase(C, half=0)
    assert ck["theta"][2] == ck["theta"][1]


def test_linear_clock_ramp_gives_slope_256_eps():
    """A linear ppm ramp gives tau slope 256*eps symbols per block."""
    eps = 20e-6
    b = np.arange(2000)
    tau_true = 256 * eps * b
    C = np.exp(-2j * math.pi * tau_true)
    ck = O.clock_phase(C, half=0)
    assert np.allclose(np.diff(ck["tau"]), 256 * eps, rtol=1e-9)


@pytest.mark.parametrize("ppm", [0.0, 10.0, -10.0, 30.0, -30.0])
def test_extraction_under_clock_offset(ppm):
    """c-4 / A16 (App. A-6): noiseless PAM-2 at eps ppm: every m in [0, m_end) emitted once
    (the output is indexed by absolute symbol number), per-block counts in {255,256,257},
    long-run mean 256/(1+eps), and u_m decides to transmitted symbol m."""
    nsym = 512 * 96
    x, a = _pam2_waveform(nsym, 0.0, seed=7)
    if ppm:
        x = gen._resample_periodic(x, ppm, ntaps=48)
    taps = gen.static_taps_pam()
    Y, C = O.pam_fd(x, taps)
    ck = O.clock_phase(C)
    u, bos = O.pam_extract(Y, ck["tau"], ck["M"])
    counts = np.diff(ck["M"])[60:-60]
    assert set(np.unique(counts)) <= {255, 256, 257}
    eps = ppm * 1e-6
    mean = (ck["M"][-61] - ck["M"][60]) / (ck["M"].shape[0] - 121)
    assert abs(mean - 256 / (1 + eps)) < 0.05
    assert np.all(np.diff(bos) >= 0)
    m = np.arange(2000, u.shape[0] - 2000)
    assert np.all(np.sign(u[m]) == a[m]), "decision errors in a noiseless stream"


def test_normalisation_closed_form_and_homogeneity():
    """c-5: ideal equiprobable PAM-M -> dc = 0, A = 1; (a u + b) -> same u^."""
    for M in (2, 4, 8, 16):
        lv = O.pam_levels(M)
        u = np.tile(lv, 1000)
        uh, dc, A = O.pam_normalise(u, np.zeros(u.shape[0], np.int64), M)
        assert abs(dc[0]) < 1e-12 and abs(A[0] - 1) < 1e-12
        uh2, dc2, A2 = O.pam_normalise(3.7 * u - 0.8, np.zeros(u.shape[0], np.int64), M)
        assert np.allclose(uh2, uh, atol=1e-12)
    # buffers are normalised independently
    u = np.concatenate([np.tile(O.pam_levels(4), 10), 2 * np.tile(O.pam_levels(4), 10) + 1])
    b = np.concatenate([np.zeros(40, np.int64), np.full(40, 8192, np.int64)])
    uh, dc, A = O.pam_normalise(u, b, 4)
    assert np.allclose(dc, [0, 1]) and np.allclose(A, [1, 2])
    assert np.allclose(uh[:40], uh[40:])


def test_q_flat_across_static_and_time_varying_clock_offsets():
    """Fig. 4 / Fig. 5 behaviour: the Q factor of the PAM chain does
    not depend on a static clock offset within +-30 ppm (no 8-bit-counter cliff at 30.5 ppm:
    symbol indices are closed-form, A16) nor on a free-running clock whose offset swings
    +-20 ppm during the record; all within 0.5 dB of the 0 ppm Q."""
    from rxsynth import make_config
    from tests.gpu_util import run_oracle
    q = {}
    for name, kw in (("0", dict(ppm=0.0)), ("+30", dict(ppm=30.0)), ("-30", dict(ppm=-30.0)),
                     ("tri20", dict(ppm_triangle=20.0))):
        rec, rx = make_config("C2", n_samples=1 << 21, M=4, snr_db=17.0, **kw)
        out = run_oracle(rec, rx)
        assert 1e-3 < out["ber"] < 0.05
        q[name] = float(O.q_from_ber(out["ber"]))
    for k in ("+30", "-30", "tri20"):
        assert abs(q[k] - q["0"]) < 0.5, q
