/*
 * tx.h — C ABI of the GPU transmitter + channel simulator, built into
 * librx.so next to the receiver (include/rx.h). It generates the 12-bit ADC stream the receiver
 * consumes, on the device and in stream order, so arbitrarily long workloads (>= 2^30 samples)
 * need neither host generation nor host-to-device copies. Test / bench infrastructure around the
 * hot path, not part of it.
 *
 * Signal model (the paper's set-ups; rxsynth/gen.py is the host reference it is tested against):
 *  - symbols: the PRBS-15 (x^15 + x^14 + 1, seed prbs_seed) reference sequence of c-10, Gray
 *    labels -> levels (PAM (2i - M + 1)/(M - 1); QAM per axis, unit mean power), symbol m = PRBS
 *    symbol (symbol_offset + m) mod 32767;
 *  - shaping: the upsampled symbol train (sps = sample_rate / baud: 2 PAM, 4 KK) through a
 *    zero-phase FIR at the sample rate (shaping_taps: pulse shape x channel, e.g. RRC x the
 *    "91 km-like" ISI for PAM; RRC(0.01) x ROADM filtering for KK), applied
 *    block-wise by 1024-point overlap-save (exact linear convolution for <= 513 taps);
 *  - PAM (IM/DD): ADC clock offset clock_ppm (band-limited resampling at p/(1+eps),
 *    32-tap Kaiser(8)-windowed sinc, 4096 phases: the free-running clock of Fig. 4/5),
 *    real AWGN of std noise_sigma at the ADC input;
 *  - KK: transmitter IQ imbalance s <- s + beta conj(s), Wiener phase noise of
 *    linewidth_hz and a CFO cfo_hz on the data, the carrier tone tone_amp with the data
 *    carrier_hz below it (E = A + s e^{-j 2 pi f_c t}, 64-bit DDS phase words), complex AWGN of
 *    std noise_sigma per dimension on the optical field, square-law photodetection I = |E|^2;
 *  - ADC: AC coupling and scaling x -> rint((x - adc_mean) / adc_full_scale * 2047.5 + 2047.5),
 *    clipped to 0..4095, u12 in uint16.
 * Noise and phase-noise increments come from a counter-based generator (Philox-4x32-10 keyed by
 * noise_seed, counter = absolute sample index), so the stream does not depend on how it is cut
 * into tx_generate calls. All calls return rx_status codes (RX_OK = 0, RX_EINVAL, RX_ECUDA ...).
 */
#ifndef TX_H
#define TX_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int family;                  /* RX_PAM (0) or RX_QAM_KK (1) */
  int order;                   /* PAM 2/4/8/16, QAM 4/16/64 */
  double baud, sample_rate;    /* sps = sample_rate / baud: 2 (PAM) or 4 (KK) */
  unsigned prbs_seed;          /* 0x7FFF */
  long long symbol_offset;     /* PRBS symbol index of transmitted symbol 0 (0 .. 32766) */
  const double *shaping_taps;  /* host, copied: zero-phase odd-length FIR at the sample rate, real
                                  (PAM, n values) or interleaved complex (KK, 2n), n <= 513 */
  int n_shaping_taps;
  double clock_ppm;            /* PAM: ADC clock offset eps = ppm 1e-6 (> 0: more samples per symbol) */
  double tone_amp;             /* KK: carrier tone amplitude A (CSPR = A^2 / mean|s|^2) */
  double carrier_hz;           /* KK: tone above the data, 0.547e9 */
  double cfo_hz;               /* KK: frequency offset of the data */
  double linewidth_hz;         /* KK: Wiener phase noise of the data */
  double iq_re, iq_im;         /* KK: transmitter IQ imbalance beta */
  double noise_sigma;          /* AWGN std per real dimension (PAM: ADC input; KK: optical field) */
  double adc_mean, adc_full_scale;   /* ADC mapping (AC coupling + 4.5 sigma full scale) */
  unsigned long long noise_seed;
} tx_config;

typedef struct tx_handle tx_handle;

/* Validate, allocate the device state and upload the shaping spectrum. RX_EINVAL on a bad
 * config, RX_ECUDA / RX_ENOMEM on device errors. */
int tx_create(const tx_config *cfg, int cuda_device, tx_handle **out);
/* The next n_samples (multiple of 512, <= 2^26 per call) of the stream as u12 codes into
 * d_codes (device, 16-byte aligned), asynchronously on cuda_stream. */
int tx_generate(tx_handle *h, unsigned short *d_codes, long long n_samples, void *cuda_stream);
void tx_destroy(tx_handle *h);

#ifdef __cplusplus
}
#endif
#endif /* TX_H */
