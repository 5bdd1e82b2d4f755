"""GPU transmitter + channel simulator (include/tx.h) against host references.

  * exactness: with the noise off, the generated codes equal a numpy model of the same signal
    chain written here (PRBS symbols -> upsampled train -> linear convolution with the taps ->
    clock resampling / KK field -> ADC), to +-1 code (fp32 vs fp64 rounding at code boundaries);
  * noise statistics: the AWGN seen through the ADC has the configured variance;
  * determinism: the stream does not depend on how it is cut into tx_generate calls;
  * equivalence: C2- and C4-like streams from the GPU give the receiver (librx) the same quality
    as rxsynth's host records of the same parameters; noiseless streams of all seven formats
    decode error free with the configured symbol offset.
"""
import math

import numpy as np
import pytest

from oracle import rx_oracle as O
from rxsynth.txparams import tx_setup

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _gen(torch, fam, M, taps, n, chunk=None, **fields):
    from paper_2011_13695_b200 import Transmitter
    T = Transmitter(fam, M, taps, **fields)
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    chunk = chunk or n
    for o in range(0, n, chunk):
        T.generate(out[o:o + chunk])
    torch.cuda.synchronize()
    T.close()
    return out.cpu().numpy().view(np.uint16)


def _quant(x, mean, fs):
    return np.clip(np.rint((x - mean) / fs * 2047.5 + 2047.5), 0, 4095)


def _train(fmt, M, off, n, sps):
    """Upsampled symbol train of the PRBS reference (c-10 levels), written independently."""
    _, _, vals = O.reference(fmt, M)
    x = np.zeros(n, dtype=np.complex128)
    m = np.arange(n // sps)
    x[::sps] = vals[(off + m) % O.P_REF]
    return x


def test_pam_generator_equals_host_model_noiseless():
    """PAM-4 through a 63-tap FIR, without and with a +30 ppm ADC clock: codes equal the numpy
    model (np.convolve; Kaiser(8) windowed-sinc resampler at p / (1 + eps)) within one code."""
    torch = _torch()
    rng = np.random.default_rng(3)
    taps = rng.normal(size=63) * np.hanning(63)
    taps /= np.sum(np.abs(taps))
    n, off = 1 << 16, 1234
    x = _train("pam", 4, off, n + 256, 2).real
    half = 31
    y = np.convolve(x, taps)[half:half + n + 256]            # zero-phase centred: y[p] = sum h[t] x[p - t]
    for ppm in (0.0, 30.0):
        codes = _gen(torch, 0, 4, taps, n, symbol_offset=off, clock_ppm=ppm, noise_sigma=0.0,
                     adc_mean=0.0, adc_full_scale=2.0)
        if ppm == 0.0:
            ref = _quant(y[:n], 0.0, 2.0)
        else:
            eps = ppm * 1e-6
            t = np.arange(n) / (1.0 + eps)
            t0 = np.floor(t)
            ph = np.rint((t - t0) * 4096) / 4096
            jj = np.arange(-15, 17)
            d = ph[:, None] - jj[None, :]
            w = np.i0(8.0 * np.sqrt(np.clip(1.0 - (d / 16) ** 2, 0, None))) / np.i0(8.0)
            idx = t0.astype(np.int64)[:, None] + jj[None, :]
            vals = np.where(idx >= 0, y[np.clip(idx, 0, None)], 0.0)
            ref = _quant(np.sum(vals * np.sinc(d) * w, axis=1), 0.0, 2.0)
        diff = np.abs(codes.astype(np.int64) - ref.astype(np.int64))
        print(f"ppm {ppm}: max code diff {diff.max()}, {np.mean(diff > 0):.2e} differ")
        assert diff.max() <= 1 and np.mean(diff > 0) < 1e-3


def test_kk_generator_equals_host_model_noiseless():
    """QAM-16 KK field (tone A, data 0.547 GHz below it, CFO, Tx IQ imbalance, square law, ADC),
    no noise / phase noise: codes equal the numpy model within one code."""
    torch = _torch()
    rng = np.random.default_rng(4)
    taps = (rng.normal(size=101) + 1j * rng.normal(size=101)) * np.hanning(101)
    taps /= np.sum(np.abs(taps)) / 2
    n, off = 1 << 16, 777
    A, fc, cfo, beta = 1.3, 0.547e9, 3e6, 0.1 * np.exp(0.4j)
    x = _train("qam", 16, off, n + 512, 4)
    s = np.convolve(x, taps)[50:50 + n]
    s = s + beta * np.conj(s)
    p = np.arange(n)
    E = A + s * np.exp(2j * math.pi * cfo / 4e9 * p) * np.exp(-2j * math.pi * fc / 4e9 * p)
    I = np.abs(E) ** 2
    mean, fs = float(np.mean(I)), 4.5 * float(np.std(I))
    ref = _quant(I, mean, fs)
    codes = _gen(torch, 1, 16, taps, n, symbol_offset=off, tone_amp=A, carrier_hz=fc, cfo_hz=cfo,
                 iq_re=beta.real, iq_im=beta.imag, noise_sigma=0.0, adc_mean=mean, adc_full_scale=fs)
    diff = np.abs(codes.astype(np.int64) - ref.astype(np.int64))
    print(f"KK: max code diff {diff.max()}, {np.mean(diff > 0):.2e} differ")
    assert diff.max() <= 1 and np.mean(diff > 0) < 1e-3


def test_noise_statistics_and_call_chunking():
    """AWGN alone (taps ~ 0): code standard deviation = sigma 2047.5 / full_scale within 1%; the
    codes do not depend on the call sizes (counter-based generator)."""
    torch = _torch()
    taps = np.zeros(31)
    taps[15] = 1e-9
    n = 1 << 20
    a = _gen(torch, 0, 2, taps, n, noise_sigma=0.1, adc_mean=0.0, adc_full_scale=1.0, noise_seed=99)
    sd = np.std(a.astype(np.float64))
    assert abs(sd / (0.1 * 2047.5) - 1.0) < 0.01 and abs(np.mean(a) - 2047.5) < 1.0
    b = _gen(torch, 0, 2, taps, n, chunk=512 * 37, noise_sigma=0.1, adc_mean=0.0, adc_full_scale=1.0, noise_seed=99)
    assert np.array_equal(a, b)
    _, _, ktaps, kf, _, _ = tx_setup("C4", n_ref=1 << 18)
    c = _gen(torch, 1, 64, ktaps, 1 << 19, **kf)
    d = _gen(torch, 1, 64, ktaps, 1 << 19, chunk=512 * 129, **kf)
    assert np.array_equal(c, d)


def _receive(torch, rec, rx, codes):
    from paper_2011_13695_b200 import RX_PAM, RX_QAM_KK, Receiver
    fam = RX_PAM if rec.fmt == "pam" else RX_QAM_KK
    fields = {k: v for k, v in rx.items() if k in ("lms_taps", "lms_block", "lms_segment", "lms_overlap", "mu",
                                                   "train_symbols", "sync_start", "sync_window",
                                                   "warmup_symbols", "cpr_test_phases")}
    if fam == RX_QAM_KK:
        fields["dc_offset"] = rec.dc_offset
    R = Receiver(fam, rec.M, rec.static_taps, history_buffers=6, **fields)
    t = torch.from_numpy(codes.view(np.int16)).cuda()
    lab = torch.zeros(codes.size // 2 + 4096, dtype=torch.uint8, device="cuda")
    for o in range(0, codes.size, 4 << 22):
        R.process(t[o:o + (4 << 22)], lab)
    R.flush(lab)
    st = R.stats()
    R.close()
    return st


@pytest.mark.parametrize("name,over", [("C2", {}), ("C4", dict(linewidth_hz=0.0))])
def test_gpu_stream_matches_rxsynth_through_the_receiver(name, over):
    """C2 (PAM-16, 91 km-like ISI, +20 ppm, SNR 32 dB) and C4 (KK 64-QAM, ROADM, 5 MHz CFO,
    OSNR 30 dB): a 2^23-sample GPU stream and rxsynth's host record of the same parameters give the
    receiver the same quality (EVM within 1 dB, BER within a factor 3 or both < 1e-4) and the same
    frame-sync offset. (C4's 10 kHz phase noise is left out here: at that operating point the
    receiver's BER depends on the phase-noise realisation by more than an order of magnitude -
    a host record carrying the GPU's own realisation behaves like the GPU stream - so the Wiener
    path is pinned exactly instead, test_kk_phase_noise_path_equals_philox_model.)"""
    torch = _torch()
    from tests.gpu_util import run_gpu
    n = 1 << 23
    fam, M, taps, f, rec_ref, rx = tx_setup(name, n_ref=n, **over)
    codes = _gen(torch, fam, M, taps, n, **f)
    st_g = _receive(torch, rec_ref, rx, codes)
    _, _, st_h = run_gpu(rec_ref, rx, chunk=4 << 22, history_buffers=6)
    ev = lambda s: 10 * math.log10(s["evm_num"] / s["evm_den"])
    ber = lambda s: s["bit_errors"] / max(s["bits"], 1)
    print(f"{name}: GPU Tx BER {ber(st_g):.3e} EVM {ev(st_g):.2f} dB | rxsynth BER {ber(st_h):.3e} EVM {ev(st_h):.2f} dB")
    assert st_g["sync_offset"] == st_h["sync_offset"]
    assert abs(ev(st_g) - ev(st_h)) < 1.0
    assert (ber(st_g) < 1e-4 and ber(st_h) < 1e-4) or 1 / 3 < (ber(st_g) + 1e-9) / (ber(st_h) + 1e-9) < 3


@pytest.mark.parametrize("fmt,M", [("pam", 2), ("pam", 4), ("pam", 8), ("pam", 16),
                                   ("qam", 4), ("qam", 16), ("qam", 64)])
def test_noiseless_gpu_streams_decode_error_free(fmt, M):
    """Every format from the GPU transmitter, noiseless and offset free (back-to-back PAM, KK
    without phase noise / CFO / ROADM), decodes with zero bit errors at the configured symbol
    offset (SPEC acceptance 3 on the simulator's output)."""
    torch = _torch()
    if fmt == "pam":
        fam, _, taps, f, rec, rx = tx_setup("C2", n_ref=1 << 18, M=M, snr_db=None, channel="b2b", ppm=0.0)
    else:
        name = {4: "C5:4", 16: "C5:5", 64: "C5:6"}[M]
        fam, _, taps, f, rec, rx = tx_setup(name, n_ref=1 << 18, osnr_db=None, linewidth_hz=0.0, cfo_hz=0.0,
                                            roadm_b3db=None, cspr_db=14.0)
        rx["lms_taps"] = 8
    f["noise_sigma"] = 0.0
    codes = _gen(torch, fam, M, taps, 1 << 22, **f)
    st = _receive(torch, rec, rx, codes)
    print(f"{fmt}-{M}: {st['bit_errors']} errors in {st['bits']} bits, sync {st['sync_offset']}")
    assert st["sync_offset"] == (rec.offset + rx["sync_start"]) % O.P_REF
    assert st["bit_errors"] == 0 and st["bits"] > 500_000


def _philox_normals(p, tag, seed):
    """Philox-4x32-10 (Salmon et al. 2011; the Random123 round function and Weyl key schedule)
    keyed by seed, counter (p_lo, p_hi, tag, 0), then Box-Muller on the four words - written here
    independently of the CUDA generator, numpy uint64 arithmetic."""
    mask = np.uint64(0xFFFFFFFF)
    c0, c1 = (p & 0xFFFFFFFF).astype(np.uint64), (p >> 32).astype(np.uint64)
    c2, c3 = np.full_like(c0, tag), np.zeros_like(c0)
    k0, k1 = np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32)
    for _ in range(10):
        pr0, pr1 = np.uint64(0xD2511F53) * c0, np.uint64(0xCD9E8D57) * c2
        c0, c1, c2, c3 = ((pr1 >> np.uint64(32)) ^ c1 ^ k0) & mask, pr1 & mask, \
            ((pr0 >> np.uint64(32)) ^ c3 ^ k1) & mask, pr0 & mask
        k0, k1 = (k0 + np.uint64(0x9E3779B9)) & mask, (k1 + np.uint64(0xBB67AE85)) & mask
    u1 = (c0.astype(np.float64) + 1) * 2.0 ** -32
    u2 = c1.astype(np.float64) * 2.0 ** -32
    return np.sqrt(-2 * np.log(u1)) * np.cos(2 * np.pi * u2)


def test_kk_phase_noise_path_equals_philox_model():
    """The Wiener phase noise of the KK data (phi_p = sum_{i <= p} w_i, w_i = sqrt(2 pi dnu / fs)
    N(0,1) from the counter-based generator, carried across tx_generate calls): codes equal a numpy
    model built from an independent Philox implementation within one code, over several calls;
    the increments have unit variance and no lag-1 correlation."""
    torch = _torch()
    rng = np.random.default_rng(4)
    taps = (rng.normal(size=101) + 1j * rng.normal(size=101)) * np.hanning(101)
    taps /= np.sum(np.abs(taps)) / 2
    n, A, fc, lw, seed = 1 << 17, 1.3, 0.547e9, 1e6, 5
    x = _train("qam", 16, 0, n + 512, 4)
    s = np.convolve(x, taps)[50:50 + n]
    p = np.arange(n, dtype=np.int64)
    w = _philox_normals(p, 1, seed)
    assert abs(np.var(w) - 1) < 0.02 and abs(np.corrcoef(w[:-1], w[1:])[0, 1]) < 0.01
    phi = np.cumsum(w * math.sqrt(2 * math.pi * lw / 4e9))
    I = np.abs(A + s * np.exp(1j * phi) * np.exp(-2j * math.pi * fc / 4e9 * p)) ** 2
    mean, fs = float(np.mean(I)), 4.5 * float(np.std(I))
    codes = _gen(torch, 1, 16, taps, n, chunk=512 * 83, tone_amp=A, carrier_hz=fc, linewidth_hz=lw,
                 noise_sigma=0.0, adc_mean=mean, adc_full_scale=fs, noise_seed=seed)
    diff = np.abs(codes.astype(np.int64) - _quant(I, mean, fs).astype(np.int64))
    print(f"phase-noise path: max code diff {diff.max()}, {np.mean(diff > 0):.2e} differ")
    assert diff.max() <= 1 and np.mean(diff > 0) < 1e-3
