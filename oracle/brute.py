"""Brute-force plain definitions used to pin the oracle (test infrastructure only).

None of these share code with ``rx_oracle``; each is the textbook definition written out.
"""
from __future__ import annotations

import math

import numpy as np


def dft_direct(x: np.ndarray) -> np.ndarray:
    """X[k] = sum_n x[n] e^{-j 2 pi k n / N}, O(N^2)."""
    x = np.asarray(x, dtype=np.complex128)
    N = x.shape[-1]
    n = np.arange(N)
    W = np.exp(-2j * math.pi * np.outer(n, n) / N)
    return x @ W.T


def idft_direct(X: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.complex128)
    N = X.shape[-1]
    n = np.arange(N)
    W = np.exp(2j * math.pi * np.outer(n, n) / N)
    return (X @ W.T) / N


def conv_direct(x: np.ndarray, taps: np.ndarray, p: np.ndarray) -> np.ndarray:
    """y_p = sum_n h[n] x_{p-n} with h centred (zero phase): h[n] = taps[(L-1)/2 + n],
    x_p = 0 outside [0, len(x))  (SURVEY §8(c) c-0 "Static filters")."""
    L = taps.shape[0]
    half = (L - 1) // 2
    out = np.zeros(p.shape[0], dtype=np.result_type(x, taps))
    for n in range(-half, half + 1):
        q = p - n
        ok = (q >= 0) & (q < x.shape[0])
        out[ok] += taps[half + n] * x[q[ok]]
    return out


def hilbert_kernel(N: int = 1024) -> np.ndarray:
    """g[n] = (2/N) cot(pi n / N) for odd n, 0 for even n — the closed-form discrete
    Hilbert kernel for even N with DC and Nyquist removed."""
    n = np.arange(N)
    g = np.zeros(N)
    odd = n % 2 == 1
    g[odd] = (2.0 / N) / np.tan(math.pi * n[odd] / N)
    return g


def hilbert_circular_td(h: np.ndarray) -> np.ndarray:
    """phi[l] = sum_n g[n] h[(l - n) mod N]: block-circular TD Hilbert transform."""
    N = h.shape[-1]
    g = hilbert_kernel(N)
    out = np.zeros(N)
    for n in range(1, N, 2):
        out += g[n] * np.roll(h, n)
    return out


def prbs15_fibonacci(n: int, seed: int = 0x7FFF) -> np.ndarray:
    """A third independent PRBS-15 (bitwise state machine, per-step loop)."""
    s = seed
    out = np.empty(n, dtype=np.uint8)
    for i in range(n):
        b = ((s >> 14) ^ (s >> 13)) & 1
        s = ((s << 1) | b) & 0x7FFF
        out[i] = b
    return out


def q_function(x):
    from scipy.special import erfc
    return 0.5 * erfc(np.asarray(x) / math.sqrt(2.0))


def pam_awgn_ber(levels: np.ndarray, thresholds: np.ndarray, labels: np.ndarray,
                 sigma: float) -> float:
    """Exact finite Q-sum BER of a 1-D slicer under AWGN (SURVEY §8(c) pin table):
    BER = 1/(M log2 M) sum_i sum_j d_H(g_i, g_j) [Q((t_j - a_i)/s) - Q((t_{j+1} - a_i)/s)],
    region j = [t_j, t_{j+1}), t_0 = -inf, t_M = +inf."""
    M = levels.shape[0]
    k = int(round(math.log2(M)))
    t = np.concatenate([[-np.inf], thresholds, [np.inf]])
    total = 0.0
    for i in range(M):
        for j in range(M):
            pj = q_function((t[j] - levels[i]) / sigma) - q_function((t[j + 1] - levels[i]) / sigma)
            total += bin(int(labels[i]) ^ int(labels[j])).count("1") * pj
    return float(total / (M * k))
