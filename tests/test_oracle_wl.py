"""Pins of the oracle's widely-linear equaliser (CPU only).

The paper's KK equaliser is a "4-tap adaptive widely-linear TD DDLMS" that also compensates
the transmitter's IQ imbalance. The build runs it as the widely-linear form of the
segmented block-LMS of SURVEY c-9: y = w^H u + v^H conj(u), v <- v + mu sum conj(u) conj(e)
(reading R-WL). Closed forms pinned here, none of which calls
the oracle's arithmetic to produce the expected value:

  * IQ imbalance z = alpha s + beta conj(s) of a proper unit-power QAM stream s has the exact
    widely-linear inverse s = conj(w_c) z + conj(v_c) conj(z) with
    w_c = alpha / (|alpha|^2 - |beta|^2),  v_c = -conj(beta) / (|alpha|^2 - |beta|^2);
    noiseless training converges to it (the Wiener solution with zero error).
  * The strictly linear MMSE solution is w_c = alpha / (|alpha|^2 + |beta|^2) and leaves the
    image: error power |beta|^2 / (|alpha|^2 + |beta|^2).
  * With a carrier phase phi (z = e^{j phi}(alpha s + beta s*)), every phase-equivalent WL
    solution has v_c / w_c = -e^{-2j phi} conj(beta) / alpha: the conjugate branch depends on the
    absolute carrier phase, which is why each decision-directed segment starts its v-branch at 0
    (reading R-WL) and converges to its own epoch's value.
"""
import math

import numpy as np

from oracle import rx_oracle as O

ALPHA = 1.0 * np.exp(0.05j)
BETA = 0.15 * np.exp(-0.6j)


def _qam16_stream(n, seed, phi0=0.0):
    """2-sps stream: even samples e^{j phi0}(alpha s + beta s*) of QAM-16 symbols s, odd samples
    independent (uncorrelated with every s_m, so the Wiener taps on them are 0)."""
    rng = np.random.default_rng(seed)
    sl = O._Slicer("qam", 16)
    idx = rng.integers(0, 4, size=(n, 2))
    s = sl.value(idx)
    z = np.empty(2 * n, dtype=np.complex128)
    z[0::2] = np.exp(1j * phi0) * (ALPHA * s + BETA * np.conj(s))
    z[1::2] = 0.3 * (rng.normal(size=n) + 1j * rng.normal(size=n))
    return z, s, idx, sl


def _train(z, s, wl, T=24576, mu=1e-3, K=4):
    lp = O.LmsParams(K=K, B=32, mu=mu, T_train=T, widely_linear=wl)
    m0 = 64
    return O.lms_train(z, 2, 0, s[m0:m0 + T], m0, lp, real=False)


def test_wl_training_converges_to_the_closed_form_iq_inverse():
    z, s, _, _ = _qam16_stream(32768, 1)
    w, v = _train(z, s, wl=True)
    den = abs(ALPHA) ** 2 - abs(BETA) ** 2
    w_c, v_c = ALPHA / den, -np.conj(BETA) / den
    c = 2
    assert abs(w[c] - w_c) < 2e-3 and abs(v[c] - v_c) < 2e-3
    others = [k for k in range(4) if k != c]
    assert np.max(np.abs(w[others])) < 2e-3 and np.max(np.abs(v[others])) < 2e-3
    # the equalised training data reproduces s (image rejected)
    m = np.arange(30000, 32000)
    U = O.tap_matrix(z, m, 2, 0, 4)
    y = U @ np.conj(w) + np.conj(U) @ np.conj(v)
    err_db = 10 * math.log10(np.mean(np.abs(y - s[m]) ** 2))
    assert err_db < -50


def test_linear_training_converges_to_linear_mmse_and_keeps_the_image():
    z, s, _, _ = _qam16_stream(32768, 2)
    w, v = _train(z, s, wl=False)
    assert np.all(v == 0)
    w_c = ALPHA / (abs(ALPHA) ** 2 + abs(BETA) ** 2)
    assert abs(w[2] - w_c) < 5e-3
    m = np.arange(30000, 32000)
    U = O.tap_matrix(z, m, 2, 0, 4)
    y = U @ np.conj(w)
    err = np.mean(np.abs(y - s[m]) ** 2)
    closed = abs(BETA) ** 2 / (abs(ALPHA) ** 2 + abs(BETA) ** 2)
    assert abs(10 * math.log10(err / closed)) < 0.5       # within 0.5 dB of the closed form
    # image rejection: WL >= 25 dB better than linear-only (SURVEY §8(f) NEXT-1 pin)
    w2, v2 = _train(z, s, wl=True)
    y2 = U @ np.conj(w2) + np.conj(U) @ np.conj(v2)
    err2 = np.mean(np.abs(y2 - s[m]) ** 2)
    assert 10 * math.log10(err / err2) > 25


E_T, S_T = 8192, 2048


def _full(wl, seed=3, n=10 * E_T, jump=0.6):
    """QAM-16 with IQ imbalance; the carrier phase is 0.7 rad up to epoch 2 (training) and then
    jumps by `jump` rad at every epoch boundary (piecewise constant; |jump| < pi/4 keeps the CPR
    quadrant unambiguous)."""
    z, s, idx, sl = _qam16_stream(n, seed)
    m = np.arange(n)
    e = m // E_T
    phi = 0.7 + jump * np.maximum(e - 2, 0)
    z[0::2] *= np.exp(1j * phi)
    lp = O.LmsParams(K=4, B=32, S=S_T, O=64, mu=1e-3, T_train=8192, D=2, E=E_T, cpr="bps", P_t=32,
                     widely_linear=wl)
    m0 = 256
    lm = O.lms_full(z, 2, 0, n, lambda m: idx[np.asarray(m)], lambda m: s[np.asarray(m)], sl, lp,
                    False, m0)
    return lm, s, idx, sl, lp, phi


def _abs_frame(lm):
    """z' of each segment rotated by its stitched quadrant j^{R_s} (c-9 'Stitching')."""
    return lm["z"] * (1j) ** lm["R"][lm["seg_of"]]


def test_wl_segments_follow_the_carrier_frame_and_decide_error_free():
    """Every decision-directed segment ends with v_c / w_c = -e^{-2j phi} conj(beta)/alpha for the
    carrier phase phi of its own epoch (the closed form), although phi jumps at every epoch;
    decisions after training are error free and the image is cancelled (reading R-WL)."""
    lm, s, idx, sl, lp, phi = _full(wl=True)
    n_seg = len(lm["seg_w"])
    assert abs(lm["v_train"][2] / lm["w_train"][2] + np.exp(-1.4j) * np.conj(BETA) / ALPHA) < 0.02
    for sg in range(8192 // S_T + 1, n_seg):
        ph = phi[sg * S_T]
        ratio = -np.exp(-2j * ph) * np.conj(BETA) / ALPHA
        got = lm["seg_v"][sg][2] / lm["seg_w"][sg][2]
        assert abs(got - ratio) < 0.03, (sg, got, ratio)
    lo = 8192 + 256
    assert np.array_equal(lm["idx"][lo:], idx[lo:])
    # after each segment's warm-up the image is gone (EVM far below the linear floor, -16.6 dB)
    late = np.concatenate([np.arange(k * S_T + S_T // 2, (k + 1) * S_T) for k in range(5, n_seg)])
    assert 10 * math.log10(np.mean(np.abs(_abs_frame(lm)[late] - s[late]) ** 2)) < -25


def test_linear_segmented_equaliser_is_image_limited():
    lm, s, idx, sl, lp, _ = _full(wl=False, jump=0.0)
    lo = 8192 + 256
    # the error sits near the linear-MMSE image floor (-16.6 dB here), far above the WL one
    err_db = 10 * math.log10(np.mean(np.abs(_abs_frame(lm)[lo:] - s[lo:]) ** 2))
    closed = 10 * math.log10(abs(BETA) ** 2 / (abs(ALPHA) ** 2 + abs(BETA) ** 2))
    assert closed - 2 < err_db < closed + 2


# ------------------------------------------------------------------ per-symbol DDLMS (NEXT-1)
# The paper's equaliser proper: a 4-tap widely-linear DDLMS updated every symbol
# (B = 1) that also does the symbol-phase recovery (no separate CPR; rx_config.lms_mode = 2,
# DESIGN reading R-DDLMS). Pinned by the same closed forms, now with a static carrier phase phi
# that only the taps can absorb: w_c = e^{j phi} alpha / den, v_c = -e^{-j phi} conj(beta) / den.

PHI = 0.3


def _ddlms_full(z, s, idx, sl, wl, n):
    lp = O.LmsParams(K=4, B=1, S=4096, O=256, mu=1e-3, T_train=8192, E=1 << 14, D=2, cpr="none",
                     widely_linear=wl, anchor_each=True)
    m0 = 64

    def ref_i(m):
        return idx[np.asarray(m)]

    def ref_v(m):
        return s[np.asarray(m)]
    return O.lms_full(z, 2, 0, n, ref_i, ref_v, sl, lp, False, m0)


def test_per_symbol_wl_ddlms_training_reaches_the_rotated_closed_form_inverse():
    """B = 1 training (e = r - y every symbol) on the IQ-imbalanced stream with carrier phase
    PHI converges to w_c = e^{j PHI} alpha / (|alpha|^2 - |beta|^2), v_c = -e^{-j PHI} conj(beta) /
    (|alpha|^2 - |beta|^2); the other taps vanish."""
    z, s, idx, sl = _qam16_stream(16384, 3, phi0=PHI)
    lp = O.LmsParams(K=4, B=1, mu=5e-4, T_train=16000, widely_linear=True)
    w, v = O.lms_train(z, 2, 0, s[64:64 + 16000], 64, lp, real=False)
    den = abs(ALPHA) ** 2 - abs(BETA) ** 2
    w_c, v_c = np.exp(1j * PHI) * ALPHA / den, -np.exp(-1j * PHI) * np.conj(BETA) / den
    assert abs(w[2] - w_c) < 2e-3 and abs(v[2] - v_c) < 2e-3
    assert np.max(np.abs(np.delete(w, 2))) < 2e-3 and np.max(np.abs(np.delete(v, 2))) < 2e-3


def test_per_symbol_wl_ddlms_tracks_phase_and_rejects_the_image():
    """Decision-directed B = 1 segments with no CPR: every segment ends at its phase-rotated
    closed-form ratio v/w = -e^{-2j PHI} conj(beta)/alpha, decodes error free, and the widely-linear
    equaliser's decision-referenced EVM beats the strictly linear one by >= 20 dB (the linear
    one sits at the closed-form image floor |beta|^2 / (|alpha|^2 + |beta|^2))."""
    n = 40000
    z, s, idx, sl = _qam16_stream(n, 4, phi0=PHI)
    out = _ddlms_full(z, s, idx, sl, True, n)
    assert np.all(out["idx"][64:] == idx[64:])
    ratio = -np.exp(-2j * PHI) * np.conj(BETA) / ALPHA
    for w, v in zip(out["seg_w"][1:], out["seg_v"][1:]):
        assert abs(v[2] / w[2] - ratio) < 1e-2          # v restarts at 0 per segment (R-WL)
    def evm(o):                          # second half of every segment (v has converged from 0)
        m = np.arange(8192, n)
        zz = o["z"][m[(m % 4096) >= 2048]]
        d = sl.value(sl.indices(zz))
        num, den = O.evm_sums(zz, d)
        return 10 * math.log10(num / den)
    lin = _ddlms_full(z, s, idx, sl, False, n)
    floor = 10 * math.log10(abs(BETA) ** 2 / (abs(ALPHA) ** 2 + abs(BETA) ** 2))
    assert abs(evm(lin) - floor) < 1.0
    assert evm(out) < evm(lin) - 20.0
