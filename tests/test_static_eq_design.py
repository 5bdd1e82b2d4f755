"""Static-equaliser design (NEXT-3; P:150 / P:221 "optimized offline", SPEC S:299-307 reading,
DESIGN R-SEQ): the oracle's design pinned by its closed forms, and librx's host-side
rx_design_static_eq equal to it (no GPU needed)."""
import numpy as np

from oracle import rx_oracle as O
from rxsynth import gen

N = 1024


def _rrc_target(beta=0.1, sps=2):
    f = np.fft.fftfreq(N)                      # cycles per sample
    return gen.rrc_amp(f * sps, beta).astype(np.complex128)


def test_flat_channel_gives_the_windowed_target():
    """Flat channel, lambda = 0 -> the windowed, truncated impulse response of the target
    (SPEC: 'flat channel -> equalizer = matched RRC filter')."""
    t = _rrc_target()
    taps = O.design_static_eq(np.ones(N), t, 0.0, 503)
    h = np.fft.ifft(t)
    c = 251
    want = np.kaiser(503, 6.0) * np.array([h[(i - c) % N] for i in range(503)])   # brute index
    assert np.max(np.abs(taps - want)) < 1e-15
    assert np.max(np.abs(taps.imag)) < 1e-15          # real, even target -> real taps


def test_lowpass_channel_boost_and_regularisation_limit():
    """2nd-order low-pass channel: the per-bin MMSE magnitude rises with frequency inside the
    band (closed form |H_t| / |H_ch| for lambda = 0); lambda -> infinity drives the taps to 0."""
    f = np.fft.fftfreq(N)
    Hc = 1.0 / (1.0 + 1j * f / 0.15) ** 2
    t = _rrc_target()
    Heq = np.conj(Hc) * t / np.abs(Hc) ** 2
    band = (f > 0.0) & (f < 0.2)
    assert np.all(np.diff(np.abs(Heq[band]) / np.abs(t[band])) > 0)
    big = O.design_static_eq(Hc, t, 1e12, 203)
    assert np.max(np.abs(big)) < 1e-11


def test_librx_design_equals_oracle():
    from paper_2011_13695_b200 import build, rx
    build.build()
    f = np.fft.fftfreq(N)
    Hc = np.exp(-2j * np.pi * f * 0.3) / (1.0 + 1j * f / 0.2) ** 2
    t = _rrc_target(0.01, 4) * np.exp(-((f / 0.4) ** 8))
    for L, real in ((503, True), (203, False), (1, True)):
        want = O.design_static_eq(Hc, t, 1e-3, L)
        got = rx.design_static_eq(Hc, t, 1e-3, L, real)
        assert np.max(np.abs(got - (want.real if real else want))) < 1e-9 * max(1.0, np.max(np.abs(want)))
    import pytest
    with pytest.raises(rx.RxError):
        rx.design_static_eq(Hc, t, 1e-3, 504, True)
    with pytest.raises(rx.RxError):
        rx.design_static_eq(Hc, t, -1.0, 503, True)
