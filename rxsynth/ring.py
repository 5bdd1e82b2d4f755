"""Bench input rings (>= 1 GiB, larger than the 126 MB L2) built on the GPU with torch.

Test/bench infrastructure (no receiver arithmetic). A PAM ring continues the seeded C2 record
seamlessly: the transmitted waveform is periodic (32767*512 samples, a whole number of PRBS
periods), so sampling it at the ADC positions p/(1+eps) mod n for p up to the ring length is
a continuous stream with a continuous clock offset; fresh AWGN of the record's variance is
added and the record's AC-coupling / full-scale are reused. A KK ring tiles the record.
"""
from __future__ import annotations

import numpy as np

from .gen import _PHASES, _polyphase_table


def pam_ring(rec, n_ring: int, device, seed: int = 12345, chunk: int = 1 << 22, ntaps: int = 32,
             ppm: float | None = None, ppm_triangle: float = 0.0):
    """ppm: static clock offset (default: the record's); ppm_triangle = A: a free-running clock
    whose offset swings 0 -> +A -> 0 -> -A -> 0 ppm over the ring (Fig. 5), sample p at
    t_p = sum_{i<p} 1/(1 + eps_i)."""
    import torch
    x_tx = rec.meta.get("x_tx")
    if x_tx is None:
        raise ValueError("pam_record(..., keep_tx=True) required")
    n = x_tx.shape[0]
    x = torch.from_numpy(x_tx).to(device=device, dtype=torch.float64)
    tab = torch.from_numpy(_polyphase_table(ntaps)).to(device=device, dtype=torch.float64)
    half = ntaps // 2
    j = torch.arange(-half + 1, half + 1, device=device, dtype=torch.int64)
    eps = (rec.ppm if ppm is None else ppm) * 1e-6
    t_run = 0.0
    sigma = float(np.sqrt(rec.meta["noise_var"]))
    mean, fs = rec.meta["mean"], rec.meta["full_scale"]
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty(n_ring, dtype=torch.int16, device=device)
    for s in range(0, n_ring, chunk):
        e = min(n_ring, s + chunk)
        p = torch.arange(s, e, device=device, dtype=torch.float64)
        if ppm_triangle:
            ph = p / n_ring
            tri = torch.where(ph < 0.25, 4 * ph, torch.where(ph < 0.75, 2 - 4 * ph, 4 * ph - 4))
            step = 1.0 / (1.0 + ppm_triangle * 1e-6 * tri)
            t = t_run + torch.cumsum(step, 0) - step
            t_run = float(t[-1] + step[-1])
        else:
            t = p / (1.0 + eps)
        t0 = torch.floor(t)
        ph = torch.round((t - t0) * _PHASES).to(torch.int64)
        idx = torch.remainder(t0.to(torch.int64)[:, None] + j[None, :], n)
        v = (x[idx] * tab[ph]).sum(dim=1)
        if sigma > 0:
            v = v + sigma * torch.randn(e - s, generator=g, device=device, dtype=torch.float64)
        c = torch.clamp(torch.round((v - mean) / fs * 2047.5 + 2047.5), 0, 4095)
        out[s:e] = c.to(torch.int16)
    return out


def tiled_ring(rec, n_ring: int, device):
    import torch
    base = torch.from_numpy(rec.codes.view(np.int16)).to(device)
    reps = -(-n_ring // base.numel())
    return base.repeat(reps)[:n_ring].contiguous()
