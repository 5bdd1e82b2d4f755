"""fp64 CPU oracle of the block-wise receiver DSP chain — TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference). Shares no code with the CUDA path.

Each function cites the passage it follows:
  P:n  = /root/reference/PAPER.md line n (section given), S:n = SPEC.md line n,
  c-k  = SURVEY.md §8(c) step k (the restatement of the paper this build is held to),
  A-k  = SURVEY.md §8(c) "readings adopted" row k (also listed in DESIGN.md).

Parity status (see DESIGN.md §Readings/§Pins): every function has a non-self pin in
tests/test_oracle_*.py except the ones marked "parity unpinned" below, whose only check is
GPU == oracle (SURVEY §8(c) "Parity unpinned"): DD-mode segment trajectories, BPS on noisy
data, the last sub-bin of the CFO estimate on noisy data, absolute BER/EVM on C2/C4.

Conventions (c-0):
  * DFT X[k] = sum_n x[n] e^{-j2pi kn/N}; inverse carries 1/N (A1).
  * signed bin kappa(k) = k (k < N/2) else k - N.
  * absolute sample index p >= 0; x_p = 0 for p < 0.
  * block b uses x_p, p in [512b - 512, 512b + 512); keeps local [256, 768) -> stream
    positions [512b - 256, 512b + 256) (A2).
  * buffer beta = blocks [8192 beta, 8192 beta + 8192).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

N_FFT = 1024
HOP = 512
KEEP_LO, KEEP_HI = 256, 768
P_REF = 32767
TWO64 = float(2 ** 64)


# ============================================================================ c-0

def kappa(k, N=N_FFT):
    """Signed bin: k for k < N/2, k - N otherwise (Nyquist -> -N/2)."""
    k = np.asarray(k)
    return np.where(k < N // 2, k, k - N)


def zero_phase_spectrum(taps: np.ndarray, N: int = N_FFT) -> np.ndarray:
    """H = DFT_N(h_c), h_c[n mod N] = taps[(L-1)/2 + n] for |n| <= (L-1)/2 (c-0, A3).

    P:150 "optimized offline in TD using 503 taps, converted to a 1024-point FD version";
    L odd and L <= hop + 1 so the central keep window equals linear convolution.
    """
    L = taps.shape[0]
    if L % 2 != 1 or L > HOP + 1:
        raise ValueError("static taps: odd length <= hop+1 required (A3)")
    half = (L - 1) // 2
    hc = np.zeros(N, dtype=np.complex128)
    for n in range(-half, half + 1):
        hc[n % N] = taps[half + n]
    return np.fft.fft(hc)


def dds_increment(f_hz: float, fs_hz: float) -> int:
    """inc = round(f/f_s * 2^64) as a two's-complement 64-bit word (c-0 'DDS phase', A10)."""
    v = (f_hz / fs_hz) * TWO64          # exact power-of-two scaling of the fp64 ratio
    return int(round(v)) % (1 << 64)


def dds_words(p: np.ndarray, inc: int, origin: int = 0) -> np.ndarray:
    """u_p = (origin + p * inc) mod 2^64, exact (numpy uint64 arithmetic wraps mod 2^64)."""
    p = np.asarray(p).astype(np.uint64)
    with np.errstate(over="ignore"):
        return (np.uint64(origin) + p * np.uint64(inc)).astype(np.uint64)


def dds_phase(words: np.ndarray) -> np.ndarray:
    """psi = 2 pi u / 2^64 (fp64)."""
    return 2.0 * math.pi * (words.astype(np.float64) / TWO64)


# ============================================================================ c-1

def ingest(codes: np.ndarray, adc_gain: float = 1.0):
    """x_p = (code_p - 2047.5)/2047.5 * adc_gain (P:136 'converts … 12-bit unsigned
    integers to 32-bit floats'; scaling A5). Returns (x, clipped) with clipped =
    #codes in {0, 4095} (c-1)."""
    c = np.asarray(codes).astype(np.float64)
    x = (c - 2047.5) / 2047.5 * adc_gain
    clipped = int(np.count_nonzero((codes == 0) | (codes == 4095)))
    return x, clipped


def frames(sig: np.ndarray, b0: int, b1: int) -> np.ndarray:
    """Overlap-save frames of blocks b0..b1-1: frame b = sig[512b-512 : 512b+512], zeros for
    p < 0 and p >= len(sig) (P:136 'prepending a block'; P:150 '100% overlap-save')."""
    out = np.zeros((b1 - b0, N_FFT), dtype=sig.dtype)
    for i, b in enumerate(range(b0, b1)):
        lo = HOP * b - HOP
        a, e = max(lo, 0), min(lo + N_FFT, sig.shape[0])
        if e > a:
            out[i, a - lo:e - lo] = sig[a:e]
    return out


# ============================================================================ c-2

def pam_fd(x: np.ndarray, taps: np.ndarray, chunk: int = 4096):
    """Steps 1-3 of the IMDD chain (c-2):

      Y_b = DFT_1024(frame_b) * H_eq  (H_eq from the zero-phase static FIR)
      C_b = sum_{k=0}^{511} Y_b[k] conj(Y_b[k+512])  (FD clock-phase estimate, A13)

    Returns (Y [nb, 1024] complex, C [nb] complex). nb = n // 512 blocks (block b needs
    input up to 512b+512).
    """
    nb = x.shape[0] // HOP
    H = zero_phase_spectrum(np.asarray(taps, dtype=np.float64))
    Y = np.empty((nb, N_FFT), dtype=np.complex128)
    for b0 in range(0, nb, chunk):
        b1 = min(nb, b0 + chunk)
        Y[b0:b1] = np.fft.fft(frames(x, b0, b1), axis=1) * H[None, :]
    C = np.sum(Y[:, :512] * np.conj(Y[:, 512:]), axis=1)
    return Y, C


# ============================================================================ c-3

def wrap_pi(x):
    """w(x) = x - 2 pi round(x / 2 pi) (c-3)."""
    return x - 2.0 * math.pi * np.round(x / (2.0 * math.pi))


def clock_phase(C: np.ndarray, half: int = 52, sps_blocks: int = 256):
    """Steps 3-4 (c-3):

      Cbar_b = sum_{i=max(0,b-52)}^{min(nb-1,b+52)} C_i   (105-block vector average, A14)
      theta_b = atan2(Cbar_b); |Cbar_b| = 0 -> theta_{b-1}
      theta^u: theta^u_0 = theta_0, theta^u_b = theta^u_{b-1} + w(theta_b - theta_{b-1})
      tau_b = -theta^u_b / 2 pi   (symbols; sign per A13)
      M_b = ceil(256 b - 128 - tau_b)  (absolute index of block b's first symbol, A16)
    """
    nb = C.shape[0]
    Cbar = np.convolve(C, np.ones(2 * half + 1), mode="full")[half:half + nb]
    theta = np.empty(nb)
    prev = 0.0
    for b in range(nb):
        if Cbar[b] == 0:
            theta[b] = prev
        else:
            theta[b] = math.atan2(Cbar[b].imag, Cbar[b].real)
        prev = theta[b]
    theta_u = np.empty(nb)
    acc = theta[0] if nb else 0.0
    for b in range(nb):
        if b > 0:
            acc = acc + wrap_pi(theta[b] - theta[b - 1])
        theta_u[b] = acc
    tau = -theta_u / (2.0 * math.pi)
    b = np.arange(nb)
    M = np.ceil(sps_blocks * b - sps_blocks // 2 - tau).astype(np.int64)
    return dict(Cbar=Cbar, theta=theta, theta_u=theta_u, tau=tau, M=M)


# ============================================================================ c-4

def pam_extract(Y: np.ndarray, tau: np.ndarray, M: np.ndarray):
    """Steps 5-7 (P:167 'Clock recovery is performed by correcting for the unwrapped
    clock-phase in FD … extracted … variable rate symbol output'; c-4, A16):

      s_b = 2 tau_b; i_b = round_half_even(s_b); f_b = s_b - i_b
      Y'_b[k] = Y_b[k] e^{+j 2 pi kappa(k) f_b / 1024}; Nyquist bin: real part only
      y_b = IDFT(Y'_b)
      u_m = y_b[2m + i_b - 512 b + 512] for m in [max(M_b,0), M_{b+1})

    Block nb-1 only closes the range of block nb-2 (A16: emission needs M_{b+1}).
    Returns (u [m_end] fp64, block_of_symbol [m_end]).
    """
    nb = Y.shape[0]
    n_emit = nb - 1
    u_parts, b_parts = [], []
    kap = kappa(np.arange(N_FFT))
    for b in range(n_emit):
        s = 2.0 * tau[b]
        i_b = np.rint(s)
        f_b = s - i_b
        Yp = Y[b] * np.exp(2j * math.pi * kap * f_b / N_FFT)
        Yp[512] = Yp[512].real
        y = np.fft.ifft(Yp)
        assert np.max(np.abs(y.imag)) <= 1e-9 * max(1.0, np.max(np.abs(y.real)))
        y = y.real
        m = np.arange(max(M[b], 0), M[b + 1], dtype=np.int64)
        if m.shape[0] == 0:
            continue
        loc = 2 * m + int(i_b) - HOP * b + HOP
        assert loc.min() >= 0 and loc.max() < N_FFT, "clock step too large (|dtau| >= 1)"
        u_parts.append(y[loc])
        b_parts.append(np.full(m.shape[0], b, dtype=np.int64))
    if not u_parts:
        return np.zeros(0), np.zeros(0, dtype=np.int64)
    return np.concatenate(u_parts), np.concatenate(b_parts)


# ============================================================================ c-5

def pam_mean_abs_level(M: int) -> float:
    """Mean |level| of unit-peak equiprobable PAM-M: M / (2 (M - 1)) (c-5)."""
    return M / (2.0 * (M - 1))


def pam_normalise(u: np.ndarray, block_of_symbol: np.ndarray, M: int,
                  buffer_blocks: int = 8192):
    """Step 8, buffer-wise normalisation (P:167 'three kernels: initialization, estimation
    of the DC-offset, and estimation of the amplitude'; c-5, A18):
      dc = mean u, A = mean|u - dc| / (M/(2(M-1))), u^ = (u - dc)/A
    over the symbols emitted by the blocks of each buffer."""
    beta = block_of_symbol // buffer_blocks
    uh = np.empty_like(u)
    dcs, amps = [], []
    for bb in range(int(beta.max()) + 1 if beta.shape[0] else 0):
        sel = beta == bb
        if not np.any(sel):
            dcs.append(0.0); amps.append(1.0)
            continue
        dc = float(np.mean(u[sel]))
        A = float(np.mean(np.abs(u[sel] - dc))) / pam_mean_abs_level(M)
        uh[sel] = (u[sel] - dc) / A
        dcs.append(dc); amps.append(A)
    return uh, np.array(dcs), np.array(amps)


# ============================================================================ c-6

def block_hilbert(fr: np.ndarray) -> np.ndarray:
    """FD Hilbert transform of real 1024-sample frames (P:218 'The Hilbert transform is
    performed in FD'; c-6, A8): Phi = -j sgn(kappa) DFT(h), Phi at kappa in {0, -512} = 0,
    phi~ = IDFT(Phi), real (the imaginary residue is asserted < 1e-9 relative)."""
    sgn = np.sign(kappa(np.arange(N_FFT))).astype(np.float64)
    sgn[0] = 0.0
    sgn[N_FFT // 2] = 0.0
    ph = np.fft.ifft(-1j * sgn * np.fft.fft(fr, axis=-1), axis=-1)
    assert np.max(np.abs(ph.imag)) <= 1e-9 * max(1.0, np.max(np.abs(ph.real)))
    return ph.real


def kk_stage1(x: np.ndarray, dc: float, carrier_hz: float, sideband: int, fs: float,
              chunk: int = 4096):
    """KK steps 1-5 (c-6):

      I = x + dc (static offline DC offset, A6); I <= 0 -> domain count, clamp 1e-12 (A7)
      a = sqrt(I); h = 1/2 ln I (conventional KK front-end)
      Phi = -j sgn(kappa) DFT_1024(h_block), kappa in {0, -512} -> 0 (FD Hilbert, A8)
      phi~ = IDFT(Phi) (real)
      E_p = a_p e^{j sigma phi~_p} e^{-j psi(p; sigma f_c)} on the kept window (KK field
            reconstruction + downshift to DC, A9/A10)

    Returns (E [512 nb - 256] complex: positions p = 0 .. 512(nb-1)+255, domain, first_idx).
    """
    n = x.shape[0]
    nb = n // HOP
    I = x + dc
    bad = I <= 0.0
    domain = int(np.count_nonzero(bad))
    first = int(np.argmax(bad)) if domain else -1
    I = np.maximum(I, 1e-12)
    a = np.sqrt(I)
    h = 0.5 * np.log(I)
    h_pad_val = 0.5 * math.log(max(dc, 1e-12))      # x_p = 0 for p < 0 -> I_p = dc
    inc = dds_increment(sideband * carrier_hz, fs)
    n_keep = HOP * nb - 256
    E = np.zeros(n_keep, dtype=np.complex128)
    for b0 in range(0, nb, chunk):
        b1 = min(nb, b0 + chunk)
        fr = frames(h, b0, b1)
        for i, b in enumerate(range(b0, b1)):      # padding value for p < 0
            lo = HOP * b - HOP
            if lo < 0:
                fr[i, :-lo] = h_pad_val
        ph = block_hilbert(fr)[:, KEEP_LO:KEEP_HI]
        for i, b in enumerate(range(b0, b1)):
            p = np.arange(HOP * b - 256, HOP * b + 256)
            ok = p >= 0
            pk = p[ok]
            psi = dds_phase(dds_words(pk, inc))
            E[pk] = a[pk] * np.exp(1j * sideband * ph[i, ok]) * np.exp(-1j * psi)
    return E, domain, first


# ============================================================================ c-7

def kk_stage2(E: np.ndarray, taps2: np.ndarray, nb: int, chunk: int = 4096):
    """KK steps 6-8 (c-7, A12):

      F_b = DFT_1024(E_p, p in [512b-512, 512b+512)), E_p = 0 for p < 0
      G = F H_eq2  (static 203-tap FIR: matched RRC + bandwidth compensation)
      z_local = 1/2 IDFT_512(G'), G'[kappa mod 512] = G[kappa], kappa in [-256, 255]
                ('A 512-point IFFT both converts the signal to TD and downsamples it to 2 sps')
      keep local [128, 384) -> 2-sps positions q in [256b - 128, 256b + 128)

    Stage-2 blocks b = 0 .. nb-2 (block b needs stage-1 output of block b+1).
    Returns z [256 (nb-2) + 128] complex (q >= 0).
    """
    H2 = zero_phase_spectrum(np.asarray(taps2, dtype=np.complex128))
    nb2 = nb - 1
    q_end = 256 * (nb2 - 1) + 128
    z = np.zeros(max(q_end, 0), dtype=np.complex128)
    for b0 in range(0, nb2, chunk):
        b1 = min(nb2, b0 + chunk)
        G = np.fft.fft(frames(E, b0, b1), axis=1) * H2[None, :]
        Gp = np.concatenate([G[:, 0:256], G[:, 768:1024]], axis=1)
        zl = 0.5 * np.fft.ifft(Gp, axis=1)[:, 128:384]
        for i, b in enumerate(range(b0, b1)):
            q = np.arange(256 * b - 128, 256 * b + 128)
            ok = q >= 0
            z[q[ok]] = zl[i, ok]
    return z


# ============================================================================ c-8

def kk_norm_cfo(z: np.ndarray, fs2: float, buffer_len: int = 1 << 21, cfo_enable: bool = True):
    """Per-buffer power normalisation + coarse CFO estimate and removal (c-8; build
    addition X3/X6):

      P = mean|z|^2; z <- z / sqrt(P)
      S[k] = sum over complete non-overlapping 1024-blocks of |DFT_1024(z^4)[k]|^2
      k* = argmax S (lowest on ties); delta = 1/2 (ln S- - ln S+)/(ln S- - 2 ln S0 + ln S+)
      df_c = (kappa(k*) + delta) f_s2 / (4 * 1024)                 (coarse)
      fine stage (reading R-CFO): a_i = sum_{chunk i} (z_q e^{-j 2 pi df_c n/f_s2})^4,
      n = q - q_lo; rho = sum_i a_{i+1} conj(a_i); df = df_c + arg(rho) f_s2 / (2 pi 4 1024)
      z_q <- z_q e^{-j psi'_q}: 64-bit DDS at df whose phase word is carried across buffers

    The log-parabolic interpolation alone is biased by up to ~0.2 bin (~100 kHz), enough
    to defeat the training pass (no CPR, c-9); the phase-increment refinement removes it.
    A buffer without a complete 1024-block reuses the previous estimate (0 for buffer 0);
    with a single complete block the fine stage is skipped.
    """
    n = z.shape[0]
    nbuf = -(-n // buffer_len)
    out = np.empty_like(z)
    P_all, df_all, k_all, origin_all = [], [], [], []
    origin = 0
    df_prev = 0.0
    for bb in range(nbuf):
        lo, hi = bb * buffer_len, min(n, (bb + 1) * buffer_len)
        zb = z[lo:hi]
        P = float(np.mean(np.abs(zb) ** 2))
        zn = zb / math.sqrt(P)
        df, kstar = df_prev, -1
        if cfo_enable:
            nch = zn.shape[0] // 1024
            if nch > 0:
                blocks = zn[:nch * 1024].reshape(nch, 1024) ** 4
                S = np.sum(np.abs(np.fft.fft(blocks, axis=1)) ** 2, axis=0)
                kstar = int(np.argmax(S))
                Sm, S0, Sp = S[(kstar - 1) % 1024], S[kstar], S[(kstar + 1) % 1024]
                lm, l0, lp = math.log(Sm), math.log(S0), math.log(Sp)
                delta = 0.5 * (lm - lp) / (lm - 2.0 * l0 + lp)
                df = (float(kappa(kstar)) + delta) * fs2 / (4.0 * 1024.0)
                if nch >= 2:
                    n_ = np.arange(nch * 1024)
                    zc4 = (zn[:nch * 1024] * np.exp(-2j * math.pi * df / fs2 * n_)) ** 4
                    a = np.sum(zc4.reshape(nch, 1024), axis=1)
                    rho = np.sum(a[1:] * np.conj(a[:-1]))
                    df = df + math.atan2(rho.imag, rho.real) * fs2 / (2.0 * math.pi * 4.0 * 1024.0)
            inc = dds_increment(df, fs2)
            words = dds_words(np.arange(hi - lo), inc, origin)
            zn = zn * np.exp(-1j * dds_phase(words))
            origin_all.append(origin)
            origin = (origin + buffer_len * inc) % (1 << 64)
        else:
            df = 0.0
            origin_all.append(0)
        out[lo:hi] = zn
        P_all.append(P); df_all.append(df); k_all.append(kstar)
        df_prev = df
    return out, dict(P=np.array(P_all), df=np.array(df_all), kstar=np.array(k_all),
                     origin=origin_all)


# ============================================================================ c-10 / c-11 helpers

def prbs15(n: int, seed: int = 0x7FFF) -> np.ndarray:
    """PRBS-15 (x^15 + x^14 + 1) via its recurrence b[n] = b[n-15] xor b[n-14], with the
    15 bits preceding b[0] all equal to the seed's bits (seed 0x7FFF -> ones) (c-10)."""
    hist = [(seed >> (14 - i)) & 1 for i in range(15)]   # b[-15] .. b[-1]
    b = hist + [0] * n
    for i in range(15, 15 + n):
        b[i] = b[i - 15] ^ b[i - 14]
    return np.array(b[15:], dtype=np.uint8)


def gray(i):
    """Gray label of ascending level index i: i xor (i >> 1) (c-11, A20)."""
    i = np.asarray(i, dtype=np.int64)
    return i ^ (i >> 1)


def gray_decode(g):
    g = np.asarray(g, dtype=np.int64)
    i = np.zeros_like(g)
    for s in range(8):                                  # labels have <= 8 bits
        i ^= g >> s
    return i


def pam_levels(M: int) -> np.ndarray:
    """a_i = (2i - M + 1)/(M - 1) (c-11)."""
    return (2.0 * np.arange(M) - M + 1) / (M - 1)


def qam_axis(M: int) -> np.ndarray:
    """Per-axis sqrt(M)-PAM scaled to unit mean QAM power: a = (2i - L + 1) sqrt(3/(2(M-1)))
    (c-11)."""
    L = int(round(math.sqrt(M)))
    return (2.0 * np.arange(L) - L + 1) * math.sqrt(3.0 / (2.0 * (M - 1)))


def reference(fmt: str, M: int, seed: int = 0x7FFF):
    """The periodic reference: symbol i takes bits [k i, k i + k) mod 32767 of the PRBS, MSB
    first, as its Gray label (c-10). Returns (labels [P], level indices, values)."""
    k = int(round(math.log2(M)))
    bits = prbs15(P_REF, seed).astype(np.int64)
    labels = np.zeros(P_REF, dtype=np.int64)
    for t in range(k):
        labels = (labels << 1) | bits[(np.arange(P_REF) * k + t) % P_REF]
    if fmt == "pam":
        idx = gray_decode(labels)
        return labels, idx, pam_levels(M)[idx]
    b = k // 2
    iI = gray_decode(labels >> b)
    iQ = gray_decode(labels & ((1 << b) - 1))
    ax = qam_axis(M)
    return labels, np.stack([iI, iQ], axis=1), ax[iI] + 1j * ax[iQ]


def slice_axis(v: np.ndarray, thresholds: np.ndarray) -> np.ndarray:
    """Level index i = #{j : t_j <= v}; a value on a threshold goes up (c-11)."""
    return np.sum(v[..., None] >= thresholds, axis=-1).astype(np.int64)


def midpoints(levels: np.ndarray) -> np.ndarray:
    return 0.5 * (levels[1:] + levels[:-1])


# ============================================================================ c-10

def frame_sync(zeta_by_phase, ref_vals: np.ndarray, min_corr: float = 0.5):
    """Frame synchronisation against the periodic PRBS reference (c-10; build addition X1,
    S:533-541):

      Gamma(o, h) = |sum_i zeta_{m0+i} conj(r_{(o+i) mod P})| / (||zeta|| ||r_window||)
      (o*, h*) = argmax, lowest (o, h) on ties; Gamma < min_corr -> sync failure
      phi0 = arg of the correlation (reported, not applied); PAM: Re < 0 -> polarity flag

    zeta_by_phase: list over sampling phases h of the W-symbol window. The circular
    correlation over all o is computed with length-P FFTs (a library primitive).
    """
    P = ref_vals.shape[0]
    best = None
    for h, zeta in enumerate(zeta_by_phase):
        W = zeta.shape[0]
        zp = np.zeros(P, dtype=np.complex128)
        zp[:W] = zeta
        corr = np.conj(np.fft.ifft(np.fft.fft(ref_vals) * np.conj(np.fft.fft(zp))))
        r2 = np.abs(ref_vals) ** 2
        ones = np.zeros(P)
        ones[:W] = 1.0
        rnorm2 = np.real(np.fft.ifft(np.fft.fft(r2) * np.conj(np.fft.fft(ones))))
        gam = np.abs(corr) / (np.linalg.norm(zeta) * np.sqrt(np.maximum(rnorm2, 1e-300)))
        o = int(np.argmax(gam))
        if best is None or gam[o] > best[2]:
            best = (o, h, float(gam[o]), corr[o])
    o, h, g, c = best
    return dict(offset=o, phase=h, gamma=g, phi0=float(np.angle(c)),
                polarity=int(c.real < 0), ok=bool(g >= min_corr))


# ============================================================================ c-9

@dataclasses.dataclass
class LmsParams:
    K: int
    B: int = 32
    S: int = 4096
    O: int = 0
    mu: float = 1e-3
    T_train: int = 8192
    D: int = 8
    E: int = 1 << 21            # symbols per epoch (one buffer)
    cpr: str = "none"           # "none" (PAM) | "vv" | "bps"
    P_t: int = 32
    widely_linear: bool = False
    anchor_each: bool = False   # QAM: every segment's quadrant from the reference (DESIGN R-ANCHOR2)
    data_aided: bool = False    # every segment adapts like the training pass (e = r - y, no CPR)


def tap_matrix(v: np.ndarray, m: np.ndarray, stride: int, off: int, K: int) -> np.ndarray:
    """u_m[k] = v[stride*m + off + c - k], k = 0..K-1, c = K//2; zero outside v (c-9)."""
    c = K // 2
    idx = stride * m[..., None] + off + c - np.arange(K)
    ok = (idx >= 0) & (idx < v.shape[0])
    out = np.zeros(idx.shape, dtype=v.dtype)
    out[ok] = v[idx[ok]]
    return out


class _Slicer:
    """Decision d = slice(z) for PAM (real) or square QAM (per axis) (c-11)."""

    def __init__(self, fmt: str, M: int, thresholds=None):
        self.fmt, self.M = fmt, M
        if fmt == "pam":
            self.levels = pam_levels(M)
            self.t = midpoints(self.levels) if thresholds is None else np.asarray(thresholds, float)
        else:
            self.levels = qam_axis(M)
            self.t = midpoints(self.levels)
        self.L = self.levels.shape[0]

    def indices(self, z):
        if self.fmt == "pam":
            return slice_axis(np.real(z), self.t)
        return np.stack([slice_axis(z.real, self.t), slice_axis(z.imag, self.t)], axis=-1)

    def value(self, idx):
        if self.fmt == "pam":
            return self.levels[idx]
        return self.levels[idx[..., 0]] + 1j * self.levels[idx[..., 1]]


def rotate_indices(idx: np.ndarray, r: int, L: int) -> np.ndarray:
    """Indices of j^r * point: j (aI + j aQ) = -aQ + j aI -> (L-1-iQ, iI)."""
    out = idx.copy()
    for _ in range(r % 4):
        out = np.stack([L - 1 - out[..., 1], out[..., 0]], axis=-1)
    return out


def lms_train(v, stride, off, ref_vals, m0, lp: LmsParams, real: bool, w0=None,
              trajectory=None):
    """Training pass (c-9 'Training'): one sequential block-LMS pass over symbols
    [m0, m0 + T_train) from the centre spike, e_m = r_m - y_m, no CPR.
    ref_vals: reference symbol value for each m in that range. ``w0``/``trajectory`` are
    test hooks (start taps; list collecting the taps after every block)."""
    K = lp.K
    w = np.zeros(K, dtype=np.float64 if real else np.complex128)
    w[K // 2] = 1.0
    if w0 is not None:
        w = np.array(w0, dtype=w.dtype)
    v_ = np.zeros(K, dtype=w.dtype)
    for t in range(m0, m0 + lp.T_train, lp.B):
        m = np.arange(t, min(t + lp.B, m0 + lp.T_train))
        U = tap_matrix(v, m, stride, off, K)
        y = U @ np.conj(w)
        if lp.widely_linear:
            y = y + np.conj(U) @ np.conj(v_)
        e = ref_vals[m - m0] - y
        w = w + lp.mu * (U.T @ np.conj(e))
        if lp.widely_linear:
            v_ = v_ + lp.mu * (np.conj(U).T @ np.conj(e))
        if trajectory is not None:
            trajectory.append(w.copy())
    return w, v_


def _cpr_estimate(y, valid, slicer: _Slicer, lp: LmsParams):
    """Per block: VV theta = 1/4 arg(-sum y^4) or BPS argmin over P_t test phases
    phi_p = -pi/4 + (p + 1/2)(pi/2)/P_t of sum |y e^{-j phi} - slice(.)|^2 (c-9 step 2)."""
    if lp.cpr == "vv":
        s = np.sum(np.where(valid, y ** 4, 0.0), axis=-1)
        return 0.25 * np.angle(-s)
    phis = -math.pi / 4 + (np.arange(lp.P_t) + 0.5) * (math.pi / 2) / lp.P_t
    best = None
    for p, ph in enumerate(phis):
        zr = y * np.exp(-1j * ph)
        d = slicer.value(slicer.indices(zr))
        dist = np.sum(np.where(valid, np.abs(zr - d) ** 2, 0.0), axis=-1)
        if best is None:
            best, arg = dist, np.zeros(dist.shape, dtype=np.int64)
        else:
            upd = dist < best
            best = np.where(upd, dist, best)
            arg = np.where(upd, p, arg)
    return phis[arg]


SYM_INIT = 64              # symbols of the per-symbol DDLMS's seed rotation (DESIGN reading R-DDLMS)


def lms_segments(v, stride, off, m_end, seeds_fn, slicer: _Slicer, lp: LmsParams,
                 real: bool, segs, ref_val_fn=None):
    """Run segments ``segs`` of the segmented DD block-LMS (c-9 'Per block j'), in lockstep
    over block index (segments are independent). Returns per-segment dicts with the output
    level indices, z', warm-up decisions, final taps and final theta.

    lp.data_aided (rx_config.lms_mode = 1, DESIGN reading R-DA): every block adapts exactly as the
    training pass of c-9 does - e_m = r_m - y_m with the reference value r_m = ref_val_fn(m), no
    CPR (theta = 0) - and the decisions slice(y_m) only feed the outputs."""
    K, B, S, O = lp.K, lp.B, lp.S, lp.O
    segs = list(segs)
    ns = len(segs)
    t0 = np.array([max(s * S - O, 0) for s in segs], dtype=np.int64)
    s_lo = np.array([s * S for s in segs], dtype=np.int64)
    s_hi = np.array([min((s + 1) * S, m_end) for s in segs], dtype=np.int64)
    nblk = int(np.max(-(-(s_hi - t0) // B))) if ns else 0
    dt = np.float64 if real else np.complex128
    # seeds_fn(s) -> w, or (w, v) for the widely-linear equaliser (its v-branch is seeded like w)
    sd = [seeds_fn(s) for s in segs]
    if lp.widely_linear:
        W = np.stack([w for w, _ in sd]).astype(dt)
        Vw = np.stack([v_ for _, v_ in sd]).astype(dt)
    else:
        W = np.stack(sd).astype(dt)
        Vw = np.zeros_like(W)
    theta = np.zeros(ns)
    diverged = False
    L = slicer.L
    # per-symbol DDLMS without CPR (lms_mode 2, DESIGN reading R-DDLMS): its taps carry the carrier
    # phase, which a seed from D epochs back does not know, so each segment adapts on the known
    # reference during its O warm-up symbols (e = r - y, as the training pass and the quadrant
    # anchoring of R-ANCHOR2 use it) and decision-directed on its own output symbols
    ref_warm = lp.cpr == "none" and not real and not lp.data_aided and lp.B == 1
    if ref_warm:
        # ... and starts from its seed rotated onto the reference: theta_0 = arg sum_m y_m conj(r_m)
        # over its first SYM_INIT symbols (y from the seed taps), w <- w e^{j theta_0}
        m = t0[:, None] + np.arange(SYM_INIT)[None, :]
        ok = m < s_hi[:, None]
        y0 = np.einsum("sbk,sk->sb", tap_matrix(v, m, stride, off, K), np.conj(W))
        c0 = np.sum(np.where(ok, y0 * np.conj(ref_val_fn(np.minimum(m, m_end - 1))), 0.0), axis=1)
        W = W * np.exp(1j * np.angle(c0))[:, None]
    out_idx = [[] for _ in range(ns)]
    out_z = [[] for _ in range(ns)]
    out_m = [[] for _ in range(ns)]
    for j in range(nblk):
        m = t0[:, None] + j * B + np.arange(B)[None, :]
        valid = m < s_hi[:, None]
        if not np.any(valid):
            break
        U = tap_matrix(v, m, stride, off, K)                  # [ns, B, K]
        y = np.einsum("sbk,sk->sb", U, np.conj(W))
        if lp.widely_linear:
            y = y + np.einsum("sbk,sk->sb", np.conj(U), np.conj(Vw))
        if lp.cpr != "none" and not lp.data_aided:
            th_hat = _cpr_estimate(y, valid, slicer, lp)
            if j == 0:
                th = th_hat
            else:
                th = th_hat + (math.pi / 2) * np.round((theta - th_hat) / (math.pi / 2))
            active = valid[:, 0]
            theta = np.where(active, th, theta)
            zp = y * np.exp(-1j * theta)[:, None]
        else:
            zp = y
        idx = slicer.indices(zp)
        d = slicer.value(idx)
        if lp.data_aided:
            e = ref_val_fn(m) - y                              # c-9 'Training' error
        elif ref_warm:
            e = np.where(m < s_lo[:, None], ref_val_fn(np.minimum(m, m_end - 1)) - y, d - zp)
        else:
            e = d - zp
            if lp.cpr != "none":
                e = e * np.exp(1j * theta)[:, None]
        e = np.where(valid, e, 0.0)
        W = W + lp.mu * np.einsum("sbk,sb->sk", U, np.conj(e))
        if lp.widely_linear:
            Vw = Vw + lp.mu * np.einsum("sbk,sb->sk", np.conj(U), np.conj(e))
        if np.any(np.abs(W) > 1e3):        # DESIGN.md R-DIV: any tap beyond 1e3 ...
            diverged = True
        for i in range(ns):
            ok = valid[i]
            if np.any(ok):
                out_m[i].append(m[i, ok]); out_idx[i].append(idx[i, ok]); out_z[i].append(zp[i, ok])
    if np.any(np.linalg.norm(W, axis=1) > 1e3):   # ... or the tap norm at the end of the run
        diverged = True
    res = []
    for i, s in enumerate(segs):
        mm = np.concatenate(out_m[i]) if out_m[i] else np.zeros(0, np.int64)
        ii = np.concatenate(out_idx[i]) if out_idx[i] else np.zeros((0,) if real else (0, 2), np.int64)
        zz = np.concatenate(out_z[i]) if out_z[i] else np.zeros(0, dt)
        res.append(dict(s=s, m=mm, idx=ii, z=zz, w=W[i].copy(), v=Vw[i].copy(),
                        theta=float(theta[i]), lo=int(s_lo[i]), hi=int(s_hi[i])))
    return res, diverged


def lms_full(v, stride, off, m_end, ref_idx_fn, ref_val_fn, slicer: _Slicer, lp: LmsParams,
             real: bool, m0: int, seed_rotation=None, w_init=None):
    """The whole equaliser of c-9: training -> epoch waves of D epochs -> stitching ->
    canonical lag-D seeds. Returns dict with final level indices per m, z', R_s, taps.
    ``seed_rotation(s)`` (test hook) multiplies segment s's seed by j^r to force it into
    another quadrant (the stitching pin). ``w_init``: start taps of training (default spike)."""
    m_tr = np.arange(m0, m0 + lp.T_train)
    w_train, v_train = lms_train(v, stride, off, ref_val_fn(m_tr), m0, lp, real, w0=w_init)
    n_seg = -(-m_end // lp.S)
    seg_per_epoch = lp.E // lp.S
    n_epoch = -(-n_seg // seg_per_epoch)
    seeds = {}
    R = np.zeros(n_seg, dtype=np.int64)
    r_rel = np.zeros(n_seg, dtype=np.int64)
    results = [None] * n_seg
    diverged = False
    canon = np.zeros((n_seg, lp.K), dtype=np.float64 if real else np.complex128)
    s0 = m0 // lp.S
    L = slicer.L

    def seed(s):
        e = (s * lp.S) // lp.E
        w = w_train if e < lp.D else seeds[e]
        if seed_rotation is not None:
            w = w * (1j) ** int(seed_rotation(s))
        if lp.widely_linear:
            # (w, v): every decision-directed segment starts its v-branch at 0 (DESIGN R-WL): the
            # conjugate branch's value depends on the absolute carrier phase during the segment
            # (v/w = -e^{-2j phi} conj(beta)/alpha), which no earlier frame knows
            return w, np.zeros_like(w)
        return w

    for wave in range(0, n_epoch, lp.D):
        segs = range(wave * seg_per_epoch, min(n_seg, (wave + lp.D) * seg_per_epoch))
        res, dv = lms_segments(v, stride, off, m_end, seed, slicer, lp, real, segs, ref_val_fn)
        diverged |= dv
        for r in res:
            results[r["s"]] = r
        if not real and lp.anchor_each:
            # DESIGN reading R-ANCHOR2 (BER-tester mode): every segment is anchored to the known
            # reference like segment s0 (R-ANCHOR), R_s = argmax_r #{m in its first 256 output
            # symbols (from m0 for s0) : d_m j^r = ref_m}, lowest r on ties; no chain, so a
            # wrong quadrant decision cannot propagate into later segments
            for s in segs:
                cur = results[s]
                a0 = m0 if s == s0 else s * lp.S
                sel = (cur["m"] >= a0) & (cur["m"] < a0 + 256) & (cur["m"] >= cur["lo"])
                ref_i = ref_idx_fn(cur["m"][sel])
                counts = [int(np.sum(np.all(rotate_indices(cur["idx"][sel], r, L) == ref_i, axis=1)))
                          for r in range(4)]
                R[s] = int(np.argmax(counts))
                r_rel[s] = (R[s] - R[s - 1]) % 4 if s > 0 else 0
        elif lp.O > 0 and not real:
            # stitching (c-9 'Stitching'): r_s from the warm-up overlap with segment s-1
            for s in segs:
                if s == 0:
                    continue
                cur, prev = results[s], results[s - 1]
                ov = np.arange(max(s * lp.S - lp.O, 0), s * lp.S)
                ci = cur["idx"][np.isin(cur["m"], ov)]
                pi_ = prev["idx"][np.isin(prev["m"], ov)]
                counts = [int(np.sum(np.all(rotate_indices(ci, r, L) == pi_, axis=1))) for r in range(4)]
                r_rel[s] = int(np.argmax(counts))
            if wave == 0:
                cur = results[s0]
                sel = (cur["m"] >= m0) & (cur["m"] < m0 + 256)
                ref_i = ref_idx_fn(cur["m"][sel])
                counts = [int(np.sum(np.all(rotate_indices(cur["idx"][sel], r, L) == ref_i, axis=1)))
                          for r in range(4)]
                R[s0] = int(np.argmax(counts))
                for s in range(s0 - 1, -1, -1):
                    R[s] = (R[s + 1] - r_rel[s + 1]) % 4
            for s in segs:
                if s > s0:
                    R[s] = (R[s - 1] + r_rel[s]) % 4
        for s in segs:
            r = results[s]
            if real or lp.data_aided:
                canon[s] = r["w"]              # no CPR: the taps are in the absolute frame
            else:
                # DESIGN.md reading R-SEED: remove the common (carrier) phase before the epoch
                # average, phi_s = arg(sum_k w_k |w_k|); carrier phase noise decorrelates the
                # absolute frame across an epoch, and CPR + stitching absorb the common phase.
                w = r["w"]
                canon[s] = w * np.exp(-1j * np.angle(np.sum(w * np.abs(w))))
        for e in range(wave, min(n_epoch, wave + lp.D)):
            lo, hi = e * seg_per_epoch, min(n_seg, (e + 1) * seg_per_epoch)
            seeds[e + lp.D] = np.mean(canon[lo:hi], axis=0)
    # assemble outputs over m in [0, m_end)
    shape = (m_end,) if real else (m_end, 2)
    idx_out = np.zeros(shape, dtype=np.int64)
    z_out = np.zeros(m_end, dtype=np.float64 if real else np.complex128)
    seg_of = np.zeros(m_end, dtype=np.int64)
    for s, r in enumerate(results):
        sel = r["m"] >= r["lo"]
        mm = r["m"][sel]
        ii = r["idx"][sel]
        idx_out[mm] = ii if real else rotate_indices(ii, int(R[s]), L)
        z_out[mm] = r["z"][sel]
        seg_of[mm] = s
    return dict(idx=idx_out, z=z_out, R=R, r_rel=r_rel, w_train=w_train, v_train=v_train,
                canon=canon, diverged=diverged, seg_of=seg_of,
                seg_v=[r["v"] for r in results], seg_w=[r["w"] for r in results])


# ============================================================================ calibration

def calibrate_thresholds(y: np.ndarray, ref_level: np.ndarray, M: int):
    """PAM decision thresholds "optimized offline beforehand and uploaded", by SPEC's
    reading: level positions estimated on a calibration run - here data-aided, the mean
    equalised value of the symbols whose reference level is i - and thresholds at the midpoints
    between adjacent level means. Returns (thresholds [M-1], level means [M])."""
    y = np.real(np.asarray(y, dtype=np.float64))
    ref_level = np.asarray(ref_level)
    means = np.array([np.mean(y[ref_level == i]) for i in range(M)])
    return 0.5 * (means[:-1] + means[1:]), means


def design_static_eq(h_channel: np.ndarray, h_target: np.ndarray, lam: float, n_taps: int):
    """Static-EQ design, SPEC's reading of "optimized offline":
    H_eq = conj(H_ch) H_t / (|H_ch|^2 + lambda) per bin of the 1024 grid, h = IDFT(H_eq),
    zero-phase taps h[i - c] (c = (n_taps - 1)/2) times a Kaiser(beta = 6) window (DESIGN R-SEQ).
    Returns complex taps (take .real for a real design)."""
    H = np.conj(h_channel) * h_target / (np.abs(h_channel) ** 2 + lam)
    h = np.fft.ifft(H)
    c = (n_taps - 1) // 2
    return np.kaiser(n_taps, 6.0) * h[(np.arange(n_taps) - c) % h.shape[0]]


def calibrate_dc(codes: np.ndarray, p: "RxParams", candidates):
    """KK DC offset of the AC-coupled receiver (the DC is restored "using the method of
    [Luis:20]", which the paper does not restate): grid search - run the whole KK chain once per
    candidate dc and keep the one with the lowest decision-referenced EVM (lowest index on ties).
    Returns (EVM dB per candidate, best index)."""
    evm = []
    for dc in candidates:
        q = dataclasses.replace(p, dc_offset=float(dc))
        out = receive_kk(codes, q)
        evm.append(out["evm_db"] if out["sync"]["gamma"] >= q.sync_min_corr else float("inf"))
    evm = np.asarray(evm)
    return evm, int(np.argmin(evm))


# ============================================================================ c-11

def count_errors(fmt, M, idx, z, slicer: _Slicer, ref_labels_fn, m_lo, m_hi):
    """bit_errors += popcount(label xor ref_label), bits += log2 M, EVM sums (c-11, A24)."""
    k = int(round(math.log2(M)))
    m = np.arange(m_lo, m_hi)
    if fmt == "pam":
        lab = gray(idx[m])
    else:
        b = k // 2
        lab = (gray(idx[m, 0]) << b) | gray(idx[m, 1])
    ref = ref_labels_fn(m)
    errs = int(np.sum(popcount(np.bitwise_xor(lab, ref))))
    return lab, errs, k * m.shape[0], m.shape[0]


def evm_sums(z_seg_frame, d_seg_frame):
    return float(np.sum(np.abs(d_seg_frame - z_seg_frame) ** 2)), float(np.sum(np.abs(d_seg_frame) ** 2))


def q_from_ber(ber):
    """Q_dB = 20 log10(sqrt(2) erfcinv(2 BER)) (A25)."""
    from scipy.special import erfcinv
    return 20.0 * np.log10(math.sqrt(2.0) * erfcinv(2.0 * np.asarray(ber)))


def popcount(x):
    x = np.asarray(x, dtype=np.int64)
    c = np.zeros_like(x)
    for s in range(16):
        c += (x >> s) & 1
    return c


# ============================================================================ top level

@dataclasses.dataclass
class RxParams:
    fmt: str                   # "pam" | "qam"
    M: int
    static_taps: np.ndarray
    adc_gain: float = 1.0
    clock_avg_half: int = 52
    thresholds: np.ndarray | None = None
    buffer_blocks: int = 8192
    carrier_hz: float = 0.547e9
    sideband: int = -1
    dc_offset: float = 0.0
    fs: float = 4e9
    cfo_enable: bool = True
    lms_taps: int = 15
    lms_block: int = 32
    lms_segment: int = 4096
    lms_overlap: int = 0
    tap_lag_epochs: int = 8
    widely_linear: bool = False
    cpr_anchor: int = 1        # QAM: 1 = every segment anchored to the reference, 0 = c-9 chain
    lms_mode: int = 0          # 0 = decision directed (c-9), 1 = data aided (DESIGN reading R-DA),
                               # 2 = per-symbol DDLMS without CPR (lms_block = 1; DESIGN R-DDLMS)
    mu: float = 1e-3
    train_symbols: int = 8192
    cpr_test_phases: int = 0
    prbs_seed: int = 0x7FFF
    sync_start: int = 4096
    sync_window: int = 2048
    sync_min_corr: float = 0.3
    warmup_symbols: int = 0
    w_init: np.ndarray | None = None   # start taps of the training pass (rx_set_taps); None = spike


def _lms_params(p: RxParams) -> LmsParams:
    if p.fmt == "pam":
        E = p.buffer_blocks * 256
        cpr = "none"
    else:
        E = p.buffer_blocks * 128
        cpr = "vv" if p.cpr_test_phases == 0 else "bps"
    if p.lms_mode == 2:
        # the paper's equaliser (DESIGN reading R-DDLMS): per-symbol
        # (B = 1) decision-directed LMS, widely linear per rx_config, with no separate CPR - the
        # taps track the carrier phase ("symbol-phase recovery ... performed by the equalizer")
        cpr = "none"
    return LmsParams(K=p.lms_taps, B=p.lms_block, S=p.lms_segment, O=p.lms_overlap, mu=p.mu,
                     T_train=p.train_symbols, D=p.tap_lag_epochs, E=E, cpr=cpr,
                     P_t=max(p.cpr_test_phases, 1), widely_linear=p.widely_linear,
                     anchor_each=bool(p.cpr_anchor) and p.fmt != "pam",
                     data_aided=p.lms_mode == 1)


def _finish(p: RxParams, v, stride, off, m_end, sync, out):
    lp = _lms_params(p)
    labels_ref, idx_ref, vals_ref = reference(p.fmt, p.M, p.prbs_seed)
    m0 = p.sync_start
    o = sync["offset"]

    def ref_index(m):
        return (o + np.asarray(m) - m0) % P_REF

    slicer = _Slicer(p.fmt, p.M, p.thresholds)
    real = p.fmt == "pam"
    lm = lms_full(v, stride, off, m_end, lambda m: idx_ref[ref_index(m)],
                  lambda m: vals_ref[ref_index(m)], slicer, lp, real, m0, w_init=p.w_init)
    lo = min(max(p.warmup_symbols, 0), m_end)
    lab, errs, bits, nsym = count_errors(p.fmt, p.M, lm["idx"], lm["z"], slicer,
                                         lambda m: labels_ref[ref_index(m)], lo, m_end)
    # EVM in the segment frame (rotation invariant)
    d_rot = slicer.value(lm["idx"][lo:m_end]) if real else None
    if real:
        num, den = evm_sums(lm["z"][lo:m_end], d_rot)
    else:
        # undo the stitch rotation on the decision to compare in the segment frame
        Rm = lm["R"][lm["seg_of"][lo:m_end]]
        idx_abs = lm["idx"][lo:m_end]
        idx_seg = idx_abs.copy()
        for r in range(4):
            sel = Rm == r
            idx_seg[sel] = rotate_indices(idx_abs[sel], -r % 4, slicer.L)
        num, den = evm_sums(lm["z"][lo:m_end], slicer.value(idx_seg))
    all_labels = np.full(m_end, 0xFF, dtype=np.int64)
    k = int(round(math.log2(p.M)))
    if real:
        all_labels[:] = gray(lm["idx"])
    else:
        all_labels[:] = (gray(lm["idx"][:, 0]) << (k // 2)) | gray(lm["idx"][:, 1])
    out.update(lms=lm, labels=all_labels.astype(np.uint8), bit_errors=errs, bits=bits,
               symbols_counted=nsym, evm_num=num, evm_den=den,
               evm_db=10 * math.log10(num / den) if den > 0 else float("nan"),
               ber=errs / bits if bits else float("nan"), m_end=m_end, sync=sync)
    return out


def receive_pam(codes: np.ndarray, p: RxParams) -> dict:
    """The whole IMDD PAM-N chain (c-1..c-5, c-9..c-11) on one record."""
    x, clipped = ingest(codes, p.adc_gain)
    Y, C = pam_fd(x, p.static_taps)
    ck = clock_phase(C, p.clock_avg_half)
    u, bos = pam_extract(Y, ck["tau"], ck["M"])
    del Y
    uh, dc, A = pam_normalise(u, bos, p.M, p.buffer_blocks)
    m_end = uh.shape[0]
    _, _, vals_ref = reference("pam", p.M, p.prbs_seed)
    zeta = uh[p.sync_start:p.sync_start + p.sync_window]
    sync = frame_sync([zeta.astype(np.complex128)], vals_ref.astype(np.complex128), p.sync_min_corr)
    out = dict(x=x, clipped=clipped, C=C, clock=ck, u=u, block_of_symbol=bos, u_hat=uh,
               dc=dc, amp=A)
    return _finish(p, uh, 1, 0, m_end, sync, out)


def receive_kk(codes: np.ndarray, p: RxParams) -> dict:
    """The whole KK QAM-N chain (c-1, c-6..c-11) on one record."""
    x, clipped = ingest(codes, p.adc_gain)
    nb = x.shape[0] // HOP
    E, domain, first = kk_stage1(x, p.dc_offset, p.carrier_hz, p.sideband, p.fs)
    z = kk_stage2(E, p.static_taps, nb)
    zc, cfo = kk_norm_cfo(z, p.fs / 2, p.buffer_blocks * 256, p.cfo_enable)
    _, _, vals_ref = reference("qam", p.M, p.prbs_seed)
    m0, W = p.sync_start, p.sync_window
    zetas = [zc[2 * np.arange(m0, m0 + W) + h] for h in (0, 1)]
    sync = frame_sync(zetas, vals_ref, p.sync_min_corr)
    h = sync["phase"]
    m_end = (zc.shape[0] - h + 1) // 2
    out = dict(x=x, clipped=clipped, E=E, domain=domain, first_domain=first, z=z, zc=zc, cfo=cfo)
    return _finish(p, zc, 2, h, m_end, sync, out)
