"""Seeded transmitter + channel + 12-bit ADC models (numpy fp64).

Test/bench infrastructure only — see ``rxsynth/__init__.py``. No receiver arithmetic here.

Sources for the models (SURVEY.md §8(d) "Common synthetic-input definition"):
  * PAM: 2 GBaud, 2 sps, RRC roll-off 0.5, ADC 4 GSa/s 12 bit.
  * KK-QAM: 1 GBaud, 4 sps, RRC roll-off 0.01, digital carrier tone 0.547 GHz above the
    data, tone power sets the CSPR; square-law photodiode.
  * Receiver analog chain: two cascaded 2nd-order Butterworth sections at 1 GHz (P:116,
    P:174 "3 dB cut-off frequency of 1 GHz"), AC coupling, 12-bit quantisation
    with 4.5 sigma of the signal at full scale.
  * Data: PRBS-15 (x^15 + x^14 + 1, seed 0x7FFF), Gray-labelled.
"""
from __future__ import annotations

import dataclasses
import functools
import math

import numpy as np

FS = 4e9                 # ADC rate
PRBS_PERIOD = 32767      # 2^15 - 1


# --------------------------------------------------------------------------- data

@functools.lru_cache(maxsize=None)
def prbs_period_bits(order: int = 15, seed: int = 0x7FFF) -> np.ndarray:
    """One period of the transmitter PRBS (Fibonacci LFSR, x^15 + x^14 + 1).

    step: b = s[14] xor s[13]; s = (s << 1 | b) & 0x7FFF; emit b.
    """
    if order != 15:
        raise ValueError("only PRBS-15 is modelled")
    s = seed & 0x7FFF
    if s == 0:
        raise ValueError("PRBS seed must be non-zero")
    out = np.empty(PRBS_PERIOD, dtype=np.uint8)
    for i in range(PRBS_PERIOD):
        b = ((s >> 14) ^ (s >> 13)) & 1
        s = ((s << 1) | b) & 0x7FFF
        out[i] = b
    out.setflags(write=False)
    return out


def gray(i):
    return np.bitwise_xor(i, np.right_shift(i, 1))


def gray_inverse(g):
    g = np.asarray(g).astype(np.int64)
    i = g.copy()
    shift = 1
    while shift < 16:
        i ^= i >> shift
        shift <<= 1
    return i


def pam_levels(M: int) -> np.ndarray:
    """Unit-peak equally spaced PAM-M levels (2i - M + 1)/(M - 1)."""
    i = np.arange(M)
    return (2.0 * i - M + 1) / (M - 1)


def qam_axis_levels(M: int) -> np.ndarray:
    """Per-axis levels of square QAM-M scaled to unit mean power."""
    L = int(round(math.sqrt(M)))
    i = np.arange(L)
    return (2.0 * i - L + 1) * math.sqrt(3.0 / (2.0 * (M - 1)))


def reference_level_indices(fmt: str, M: int) -> np.ndarray:
    """Level indices of the periodic PRBS symbol sequence (period 32767 symbols).

    Symbol i takes bits [k i, k i + k) (mod 32767) MSB first as its Gray label, k = log2 M.
    PAM: returns int array [P] of level indices. QAM: int array [P, 2] of (i_I, i_Q), the
    label's high half being Gray(i_I).
    """
    k = int(round(math.log2(M)))
    bits = prbs_period_bits().astype(np.int64)
    idx = (np.arange(PRBS_PERIOD)[:, None] * k + np.arange(k)[None, :]) % PRBS_PERIOD
    labels = np.zeros(PRBS_PERIOD, dtype=np.int64)
    for t in range(k):
        labels = (labels << 1) | bits[idx[:, t]]
    if fmt == "pam":
        return gray_inverse(labels)
    b = k // 2
    return np.stack([gray_inverse(labels >> b), gray_inverse(labels & ((1 << b) - 1))], axis=1)


# --------------------------------------------------------------------------- filters

def rrc_amp(fnorm: np.ndarray, beta: float) -> np.ndarray:
    """Root-raised-cosine amplitude response, f normalised to the baud rate, H(0) = 1."""
    a = np.abs(fnorm)
    f1 = (1.0 - beta) / 2.0
    f2 = (1.0 + beta) / 2.0
    rc = np.where(a <= f1, 1.0, 0.0)
    mid = (a > f1) & (a <= f2)
    rc = np.where(mid, 0.5 * (1.0 + np.cos(np.pi / beta * (a - f1))), rc)
    return np.sqrt(rc)


def butterworth2(f_hz: np.ndarray, fc: float) -> np.ndarray:
    """Analog 2nd-order Butterworth low-pass H(s) = 1/(s^2 + sqrt2 s + 1), s = j f/fc."""
    s = 1j * f_hz / fc
    return 1.0 / (s * s + math.sqrt(2.0) * s + 1.0)


def super_gaussian(f_hz: np.ndarray, b3db: float, order: int = 2) -> np.ndarray:
    """Amplitude of a super-Gaussian band-pass, |H|^2 = exp(-ln2 (2f/B)^(2 order))."""
    return np.exp(-0.5 * math.log(2.0) * (2.0 * np.abs(f_hz) / b3db) ** (2 * order))


def _dense_taps(H_fn, n_taps: int, grid: int = 1 << 15) -> np.ndarray:
    k = np.fft.fftfreq(grid)               # cycles / sample
    h = np.fft.ifft(H_fn(k)).real
    h = np.fft.fftshift(h)
    c = grid // 2
    half = (n_taps - 1) // 2
    return h[c - half: c + half + 1].copy()


def static_taps_pam(n_taps: int = 503, sps: int = 2, beta: float = 0.5) -> np.ndarray:
    """Matched RRC for the PAM static equaliser input (503-tap offline FIR).

    Normalised so that transmitter RRC x receiver RRC is a raised cosine with unit peak.
    Zero-phase (symmetric, odd length). Bandwidth compensation is deliberately not included
    (SURVEY §8(d) "Static taps"), so the adaptive equaliser has work to do.
    """
    return _dense_taps(lambda k: math.sqrt(sps) * rrc_amp(k * sps, beta), n_taps)


def static_taps_kk(n_taps: int = 203, sps: int = 4, beta: float = 0.01,
                   kaiser_beta: float = 6.0) -> np.ndarray:
    """Matched RRC(0.01) for the KK static equaliser (203-tap offline FIR), Kaiser(6)
    windowed so the 0.547 GHz tone is rejected by > 50 dB.

    Returns complex taps (imaginary part zero) as complex128 [n_taps].
    """
    h = _dense_taps(lambda k: math.sqrt(sps) * rrc_amp(k * sps, beta), n_taps)
    h = h * np.kaiser(n_taps, kaiser_beta)
    return h.astype(np.complex128)


# --------------------------------------------------------------------------- helpers

_PHASES = 4096


@functools.lru_cache(maxsize=4)
def _polyphase_table(ntaps: int, phases: int = _PHASES, win_beta: float = 8.0) -> np.ndarray:
    """Kaiser(8)-windowed sinc interpolation kernels for `phases` fractional delays."""
    half = ntaps // 2
    j = np.arange(-half + 1, half + 1)
    fr = np.arange(phases + 1) / phases
    d = fr[:, None] - j[None, :]
    w = np.i0(win_beta * np.sqrt(np.clip(1.0 - (d / half) ** 2, 0.0, None))) / np.i0(win_beta)
    return np.sinc(d) * w


def _resample_periodic(x: np.ndarray, ppm: float, ntaps: int = 32,
                       n_out: int | None = None, p0: int = 0, positions=None) -> np.ndarray:
    """Band-limited resampling of a periodic sequence at positions p/(1+eps), eps = ppm*1e-6,
    p = p0 .. p0+n_out-1 (indices mod len(x): the periodic waveform makes a seamless ring).

    eps > 0 means the ADC takes more samples per symbol (SURVEY §8(c) extraction pin).
    Polyphase Kaiser(8)-windowed sinc over ``ntaps`` neighbours, 4096 fractional phases.
    """
    n = x.shape[0]
    n_out = n if n_out is None else n_out
    eps = ppm * 1e-6
    out = np.empty(n_out, dtype=x.dtype)
    half = ntaps // 2
    j = np.arange(-half + 1, half + 1)
    tab = _polyphase_table(ntaps)
    chunk = 1 << 18
    for s in range(0, n_out, chunk):
        p = np.arange(p0 + s, p0 + min(n_out, s + chunk), dtype=np.float64)
        t = p / (1.0 + eps) if positions is None else positions[s:s + p.shape[0]]
        t0 = np.floor(t)
        ph = np.rint((t - t0) * _PHASES).astype(np.int64)
        idx = (t0.astype(np.int64)[:, None] + j[None, :]) % n
        out[s:s + p.shape[0]] = np.einsum("ij,ij->i", x[idx], tab[ph])
    return out


def _quantise(x: np.ndarray, sigmas: float = 4.5):
    """AC-couple (remove the mean), scale 4.5 sigma to full scale, 12-bit mid-tread codes."""
    mean = float(np.mean(x))
    xac = x - mean
    fs = sigmas * float(np.std(xac))
    codes = np.rint(xac / fs * 2047.5 + 2047.5)
    clipped = int(np.count_nonzero((codes < 0) | (codes > 4095)))
    codes = np.clip(codes, 0, 4095).astype(np.uint16)
    return codes, mean, fs, clipped


@dataclasses.dataclass
class Record:
    """A generated ADC record plus the receiver parameters the harness derives for it."""
    codes: np.ndarray            # uint16 [n], u12 right-aligned
    fmt: str                     # "pam" | "qam"
    M: int
    baud: float
    sps: int
    offset: int                  # PRBS symbol index of transmitted symbol 0
    ppm: float
    static_taps: np.ndarray      # float64 (PAM) or complex128 (QAM)
    dc_offset: float = 0.0       # KK: removed mean in x units
    tx_index: np.ndarray | None = None   # transmitted level indices (PAM [n]; QAM [n, 2])
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.codes.shape[0])


def _tx_indices(fmt, M, nsym, offset):
    ref = reference_level_indices(fmt, M)
    return ref[(offset + np.arange(nsym)) % PRBS_PERIOD]


# --------------------------------------------------------------------------- PAM

def pam_record(M: int, n_samples: int, *, seed: int, snr_db: float | None = None,
               channel: str = "b2b", ppm: float = 0.0, offset: int | None = None,
               n_static_taps: int = 503, echo=(1.0, 0.2, -0.1), keep_tx: bool = False,
               ppm_triangle: float = 0.0) -> Record:
    """2 GBaud PAM-M at 2 sps, optional '91 km-like' ISI, clock offset, AWGN.

    channel "b2b": no filtering. "isi91": IM/DD CD response cos(2 pi^2 |b2| L f^2)
    (b2 = -21.5 ps^2/km, L = 91 km) x two 1 GHz Butterworth sections x symbol-spaced
    echo [1, 0.2, -0.1]. snr_db: electrical SNR at the matched-filter
    output relative to the ideal levels (C1: 9 dB -> BER Q(sqrt(7.94)) for PAM-2).
    ppm_triangle = A: a free-running, time-varying clock offset instead of a static one (the
    paper's Fig. 5 scenario): eps(p) is one triangle period over the record,
    0 -> +A -> 0 -> -A -> 0 ppm, and sample p is taken at t_p = sum_{i<p} 1/(1 + eps_i).
    """
    rng = np.random.default_rng(seed)
    sps, baud, beta = 2, 2e9, 0.5
    if n_samples % sps:
        raise ValueError("n_samples must be a multiple of sps")
    nsym = n_samples // sps
    if offset is None:
        offset = int(rng.integers(0, PRBS_PERIOD))
    idx = _tx_indices("pam", M, nsym, offset)
    a = pam_levels(M)[idx]
    up = np.zeros(n_samples)
    up[::sps] = a
    F = np.fft.fft(up)
    f_hz = np.fft.fftfreq(n_samples, d=1.0 / FS)
    F *= math.sqrt(sps) * rrc_amp(f_hz / baud, beta)
    if channel == "isi91":
        b2 = -21.5e-27 * 1e-3        # s^2/m  (-21.5 ps^2/km)
        L = 91e3
        F *= np.cos(2.0 * math.pi ** 2 * abs(b2) * L * f_hz ** 2)
        F *= butterworth2(f_hz, 1e9) ** 2
        T = 1.0 / baud
        e = np.zeros_like(F)
        for d, c in enumerate(echo):
            e = e + c * np.exp(-2j * math.pi * f_hz * d * T)
        F *= e
    elif channel != "b2b":
        raise ValueError(channel)
    x = np.fft.ifft(F).real
    x_tx = x if keep_tx else None            # periodic, pre-ADC-clock waveform (bench ring)
    if ppm_triangle != 0.0:
        ph = np.arange(n_samples, dtype=np.float64) / n_samples
        tri = np.where(ph < 0.25, 4 * ph, np.where(ph < 0.75, 2 - 4 * ph, 4 * ph - 4))
        step = 1.0 / (1.0 + ppm_triangle * 1e-6 * tri)
        pos = np.concatenate([[0.0], np.cumsum(step[:-1])])
        x = _resample_periodic(x, 0.0, positions=pos)
    elif ppm != 0.0:
        x = _resample_periodic(x, ppm)
    taps = static_taps_pam(n_static_taps, sps, beta)
    noise_var = 0.0
    if snr_db is not None:
        Ea2 = (M + 1.0) / (3.0 * (M - 1.0))
        noise_var = Ea2 / (10.0 ** (snr_db / 10.0) * float(np.sum(taps ** 2)))
        x = x + rng.normal(0.0, math.sqrt(noise_var), size=n_samples)
    codes, mean, fs, clipped = _quantise(x)
    return Record(codes=codes, fmt="pam", M=M, baud=baud, sps=sps, offset=offset, ppm=ppm,
                  static_taps=taps, tx_index=idx,
                  meta=dict(seed=seed, snr_db=snr_db, channel=channel, clipped=clipped, ppm_triangle=ppm_triangle,
                            full_scale=fs, mean=mean, noise_var=noise_var, x_tx=x_tx))


# --------------------------------------------------------------------------- KK-QAM

def kk_record(M: int, n_samples: int, *, seed: int, cspr_db: float, osnr_db: float | None,
              cfo_hz: float = 0.0, linewidth_hz: float = 0.0, rx_lpf: bool = False,
              roadm_b3db: float | None = None, offset: int | None = None,
              carrier_hz: float = 0.547e9, n_static_taps: int = 203,
              periodic: bool = False, iq_imbalance: complex = 0.0, keep_field: bool = False) -> Record:
    """1 GBaud QAM-M at 4 sps with a digital carrier tone 0.547 GHz above the data.

    Field in the tone's frame: E = A + s(t) e^{-j 2 pi f_c t}, |A|^2 = CSPR * mean|s|^2;
    s carries Wiener phase noise (linewidth) and a CFO between tone and data; optional
    super-Gaussian 'ROADM' filtering of the data term; complex AWGN at the given OSNR over
    12.5 GHz of total power; square-law detection; optional 1 GHz receiver LPF; AC coupling
    (the removed mean is returned as dc_offset in x units); 12-bit ADC.

    periodic=True makes the record exactly periodic, so a tiled ring of it is a seamless stream
    (bench inputs): the tone and CFO frequencies are rounded to whole cycles per record (a shift
    of at most FS/(2 n), 119 Hz at 2^24 samples) and the phase noise is a Wiener bridge (the
    walk minus its linear drift, so it ends where it starts).
    iq_imbalance = beta: transmitter IQ imbalance of the shaped data, s <- s + beta conj(s) (the
    impairment the paper's widely-linear equaliser compensates).
    """
    rng = np.random.default_rng(seed)
    sps, baud, beta = 4, 1e9, 0.01
    if n_samples % sps:
        raise ValueError("n_samples must be a multiple of sps")
    nsym = n_samples // sps
    if offset is None:
        offset = int(rng.integers(0, PRBS_PERIOD))
    idx = _tx_indices("qam", M, nsym, offset)
    lv = qam_axis_levels(M)
    sym = lv[idx[:, 0]] + 1j * lv[idx[:, 1]]
    up = np.zeros(n_samples, dtype=np.complex128)
    up[::sps] = sym
    F = np.fft.fft(up)
    f_hz = np.fft.fftfreq(n_samples, d=1.0 / FS)
    F *= math.sqrt(sps) * rrc_amp(f_hz / baud, beta)
    if roadm_b3db is not None:
        F *= super_gaussian(f_hz, roadm_b3db)
    s = np.fft.ifft(F)
    del F, up
    if iq_imbalance:
        s = s + complex(iq_imbalance) * np.conj(s)
    n = np.arange(n_samples, dtype=np.float64)
    if periodic:
        cfo_hz = round(cfo_hz * n_samples / FS) * FS / n_samples
        carrier_hz = round(carrier_hz * n_samples / FS) * FS / n_samples
    if linewidth_hz > 0:
        phi = np.cumsum(rng.normal(0.0, math.sqrt(2 * math.pi * linewidth_hz / FS), n_samples))
        if periodic:
            phi -= (n + 1.0) / n_samples * phi[-1]
        s *= np.exp(1j * phi)
    if cfo_hz != 0.0:
        s *= np.exp(2j * math.pi * cfo_hz / FS * n)
    Ps = float(np.mean(np.abs(s) ** 2))
    A = math.sqrt(10.0 ** (cspr_db / 10.0) * Ps)
    E = A + s * np.exp(-2j * math.pi * carrier_hz / FS * n)
    field = s if keep_field else None     # the transmitted data field (test reference)
    del s
    if osnr_db is not None:
        Ptot = A * A + Ps
        var = Ptot / 10.0 ** (osnr_db / 10.0) * (FS / 12.5e9)
        E += math.sqrt(var / 2.0) * (rng.normal(size=n_samples) + 1j * rng.normal(size=n_samples))
    I = E.real ** 2 + E.imag ** 2
    del E
    if rx_lpf:
        I = np.fft.ifft(np.fft.fft(I) * butterworth2(f_hz, 1e9) ** 2).real
    codes, mean, fs, clipped = _quantise(I)
    return Record(codes=codes, fmt="qam", M=M, baud=baud, sps=sps, offset=offset, ppm=0.0,
                  static_taps=static_taps_kk(n_static_taps, sps, beta), dc_offset=mean / fs,
                  tx_index=idx,
                  meta=dict(seed=seed, cspr_db=cspr_db, osnr_db=osnr_db, cfo_hz=cfo_hz,
                            linewidth_hz=linewidth_hz, rx_lpf=rx_lpf, roadm_b3db=roadm_b3db,
                            carrier_hz=carrier_hz, clipped=clipped, full_scale=fs,
                            iq_imbalance=complex(iq_imbalance), field=field,
                            tone_amp=A, data_power=Ps))


def tile_codes(codes: np.ndarray, n_total: int) -> np.ndarray:
    """Tile a (periodic) record into a longer ring, e.g. the >= 1 GiB bench input."""
    reps = -(-n_total // codes.shape[0])
    return np.tile(codes, reps)[:n_total]


def pack_u12(codes: np.ndarray) -> np.ndarray:
    """12-bit codes -> the packed ADC byte stream (2 codes per 3 bytes, little-endian bit
    stream: code k = bits [12k, 12k + 12)), the RX_IN_U12_PACKED input format."""
    c = np.asarray(codes, dtype=np.uint32).reshape(-1, 2)
    out = np.empty((c.shape[0], 3), dtype=np.uint8)
    out[:, 0] = c[:, 0] & 0xFF
    out[:, 1] = ((c[:, 0] >> 8) & 0x0F) | ((c[:, 1] & 0x0F) << 4)
    out[:, 2] = (c[:, 1] >> 4) & 0xFF
    return out.reshape(-1)
