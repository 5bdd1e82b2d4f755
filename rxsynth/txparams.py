"""Parameters of the GPU transmitter + channel simulator (include/tx.h) for a config
of rxsynth: the shaping FIR (pulse shape x channel of gen.pam_record / gen.kk_record as one
513-tap filter at the sample rate) and the tone / noise / ADC mapping of a host reference record
with the same parameters. Host-side harness code (no receiver arithmetic)."""
from __future__ import annotations

import math

import numpy as np

from .configs import make_config
from .gen import FS, butterworth2, rrc_amp, super_gaussian

N_TX_TAPS = 513


def _fir(H_fn, n_taps: int = N_TX_TAPS, grid: int = 1 << 16, kaiser: float = 8.0) -> np.ndarray:
    """Zero-phase-centred FIR (taps[(n-1)/2 + t] = h[t]) of a frequency response H(f_hz) at FS,
    from a dense inverse DFT, Kaiser-windowed."""
    f = np.fft.fftfreq(grid, d=1.0 / FS)
    h = np.fft.fftshift(np.fft.ifft(H_fn(f)))
    c, half = grid // 2, (n_taps - 1) // 2
    return h[c - half:c + half + 1] * np.kaiser(n_taps, kaiser)


def tx_setup(name: str, n_ref: int = 1 << 18, noise_seed: int = 1, **overrides):
    """-> (family, order, shaping_taps, tx fields, reference Record, rx params). The reference
    record (rxsynth, n_ref samples, same parameters) supplies the symbol offset, the tone
    amplitude, the noise level and the ADC mapping; the returned fields feed
    paper_2011_13695_b200.Transmitter."""
    rec, rx = make_config(name, n_samples=n_ref, **overrides)
    m = rec.meta
    if rec.fmt == "pam":
        sps, baud = 2, 2e9

        def H(f):
            r = math.sqrt(sps) * rrc_amp(f / baud, 0.5).astype(np.complex128)
            if m["channel"] == "isi91":
                b2, L = -21.5e-27 * 1e-3, 91e3
                r = r * np.cos(2.0 * math.pi ** 2 * abs(b2) * L * f ** 2) * butterworth2(f, 1e9) ** 2
                e = np.zeros_like(r)
                for dd, cc in enumerate((1.0, 0.2, -0.1)):
                    e = e + cc * np.exp(-2j * math.pi * f * dd / baud)
                r = r * e
            return r
        taps = _fir(H).real
        fields = dict(symbol_offset=rec.offset, clock_ppm=float(rec.ppm), noise_sigma=math.sqrt(m["noise_var"]),
                      adc_mean=m["mean"], adc_full_scale=m["full_scale"], noise_seed=noise_seed)
        return 0, rec.M, taps, fields, rec, rx
    sps, baud = 4, 1e9

    def Hk(f):
        r = math.sqrt(sps) * rrc_amp(f / baud, 0.01).astype(np.complex128)
        if m.get("roadm_b3db") is not None:
            r = r * super_gaussian(f, m["roadm_b3db"])
        return r
    taps = _fir(Hk)
    A, Ps = m["tone_amp"], m["data_power"]
    sigma = 0.0
    if m.get("osnr_db") is not None:
        var = (A * A + Ps) / 10.0 ** (m["osnr_db"] / 10.0) * (FS / 12.5e9)
        sigma = math.sqrt(var / 2.0)
    iq = complex(m.get("iq_imbalance", 0.0))
    fields = dict(symbol_offset=rec.offset, tone_amp=A, carrier_hz=m["carrier_hz"], cfo_hz=m["cfo_hz"],
                  linewidth_hz=m["linewidth_hz"], iq_re=iq.real, iq_im=iq.imag, noise_sigma=sigma,
                  adc_mean=rec.dc_offset * m["full_scale"], adc_full_scale=m["full_scale"], noise_seed=noise_seed)
    return 1, rec.M, taps, fields, rec, rx
