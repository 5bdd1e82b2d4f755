/*
 * rx.h — C ABI of librx: the B200 (sm_100a) block-wise receiver DSP chain of
 * van der Heide et al., "Field Trial of a Flexible Real-time Software-defined GPU-based
 * Optical Receiver" (arXiv 2011.13695, JLT 2021).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; SURVEY §8(x) = the build's
 * hot-path contract, whose step numbers H0..H25 / c-0..c-11 are used below.
 *
 * Shape of the API (BASELINE.json north_star): rx_create(format, baud, samples/symbol, taps,
 * block/overlap sizes) -> rx_process(device sample buffer, stream) -> decided bits, error
 * counts, EVM.  The paper's contract is the per-buffer hand-over of a filled GPU buffer to
 * the control program with ordered carries between buffers.
 *
 * General rules
 *  - C99, no C++ or torch types. All calls return rx_status (RX_OK = 0, errors < 0) unless
 *    stated. Argument/config errors are returned synchronously (RX_EINVAL) and change nothing.
 *  - Device pointers ("d_") must be device memory of the handle's CUDA device, 16-byte
 *    aligned. Host pointers ("host_") are plain host memory. `cuda_stream` is a cudaStream_t
 *    (NULL = legacy default stream).
 *  - The caller owns every buffer it passes; it must stay valid until the work enqueued on
 *    `cuda_stream` completes. The library owns all internal state (overlap halos, clock
 *    history, DDS phase words, normalisation partials, LMS taps and epoch seeds, CPR /
 *    stitch state, sync result, counters). A handle is not thread-safe; handles are
 *    independent (one handle = one channel).
 *  - rx_process / rx_flush are asynchronous and stream-ordered and never synchronise the host.
 *    Data-dependent errors (domain, divergence, sync failure, label capacity) set sticky
 *    device flags, reported by rx_get_stats() and returned by the next rx_process().
 *  - There is no CPU fallback: every step of the chain runs in the library's CUDA kernels.
 */
#ifndef RX_H
#define RX_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RX_OK = 0,
  RX_EINVAL = -1,     /* bad argument or configuration */
  RX_ENOMEM = -2,     /* device allocation failed */
  RX_ECUDA = -3,      /* a CUDA runtime call failed (no device, launch failure, ...) */
  RX_EDOMAIN = -4,    /* KK: I + dc <= 0 seen (counted, clamped to 1e-12) */
  RX_ESYNC = -5,      /* frame-sync correlation below sync_min_corr */
  RX_EDIVERGE = -6,   /* LMS tap norm > 1e3 */
  RX_ECAPACITY = -7,  /* internal history ring overrun (call larger than configured) */
  RX_ESTATE = -8      /* call order violated (e.g. rx_process after rx_flush) */
} rx_status;

typedef enum { RX_PAM = 0, RX_QAM_KK = 1 } rx_family;

/* Status flag bits (rx_stats.status_flags) */
#define RX_FLAG_DOMAIN   1
#define RX_FLAG_SYNC     2
#define RX_FLAG_DIVERGE  4
#define RX_FLAG_CAPACITY 8

typedef struct {
  int family;                 /* rx_family. PAM: IMDD PAM-N chain;
                                 RX_QAM_KK: Kramers-Kronig QAM-N chain */
  int order;                  /* PAM 2/4/8/16, QAM 4/16/64 */
  double baud;                /* symbols/s: 2e9 (PAM), 1e9 (KK) */
  double sample_rate;         /* ADC rate, 4e9. sps = sample_rate/baud must be 2 (PAM)
                                 or 4 (KK) */
  int fft_size;               /* 1024; only 1024 is built */
  int hop;                    /* 512 = fft_size/2: 100% overlap-save */
  int buffer_blocks;          /* 8192 blocks = 2^22 samples per buffer; unit of the
                                 normalisation, CFO and LMS epochs */
  const double *static_taps;  /* host, copied. Zero-phase odd-length FIR, n <= hop+1, placed
                                 centred. PAM: n real taps (503 in P:150).
                                 KK: n complex taps interleaved re,im (203 in P:221) */
  int n_static_taps;
  double adc_gain;            /* x = (code - 2047.5)/2047.5 * adc_gain */
  int clock_avg_half;         /* PAM: 52 -> 105-block clock-phase average */
  const double *thresholds;   /* PAM: M-1 ascending decision thresholds (P:167 'optimized
                                 offline'), host, copied; NULL = ideal midpoints */
  double carrier_offset_hz;   /* KK: 0.547e9 */
  int sideband;               /* KK: -1 = signal below the carrier (paper set-up) */
  double dc_offset;           /* KK: static DC restoring the AC-coupled intensity, x units */
  int lms_taps;               /* K: PAM T-spaced real taps (15/31), KK T/2-spaced complex (4..32) */
  int lms_block;              /* B symbols per tap update: 32; 1 with lms_mode = 2 */
  int lms_segment;            /* S symbols per parallel segment: 4096; divides the epoch */
  int lms_overlap;            /* O warm-up symbols per segment (KK 256, PAM 0); multiple of B */
  int tap_lag_epochs;         /* D: seeds of epoch e are the mean canonical taps of e-D (8) */
  int widely_linear;          /* KK only: 1 = widely-linear equaliser, y = w^H u + v^H conj(u)
                                 (the paper's "widely-linear TD DDLMS", compensating Tx
                                 IQ imbalance), run as the segmented block-LMS of SURVEY c-9: the
                                 v-branch is trained with w, and every decision-directed segment
                                 starts its v-branch at 0 (DESIGN reading R-WL); 0 = strictly
                                 linear. PAM: must be 0 */
  double mu;                  /* block-sum LMS step (1e-3 PAM, 2e-3 KK) */
  int train_symbols;          /* data-aided training symbols after sync (8192); multiple of B */
  int cfo_enable;             /* KK: per-buffer 4th-power CFO estimate + removal (1) */
  int cpr_test_phases;        /* KK: 0 = Viterbi-Viterbi (QAM-4), else BPS test phases (<= 64) */
  int cpr_anchor;             /* KK quadrant of each equaliser segment: 1 (default) = anchored to
                                 the known PRBS reference over its first 256 symbols (BER-tester
                                 mode, DESIGN reading R-ANCHOR2: a slip cannot propagate); 0 = the
                                 SURVEY c-9 stitch chain R_s = R_{s-1} + r_s from the warm-up
                                 overlap (no reference needed after segment s0) */
  unsigned prbs_order;        /* 15: PRBS x^15+x^14+1 reference (BER tester) */
  unsigned prbs_seed;         /* 0x7FFF */
  long long sync_start;       /* m0: first symbol of the sync window (4096); multiple of
                                 lms_segment is not required */
  int sync_window;            /* W_s symbols correlated (2048, <= 4096) */
  double sync_min_corr;       /* Gamma threshold (0.3) */
  long long warmup_symbols;   /* symbols below this index are not counted in BER/EVM */
  int history_buffers;        /* device rings keep this many buffers of each intermediate
                                 (>= 3; probes can read back only what is still held) */
  int lms_batch_segments;     /* equaliser launches wait until about this many segments are
                                 pending (more concurrent segment-warps per launch; results do
                                 not depend on it; adds latency); 0 = every call */
  int input_format;           /* rx_input_format of every rx_process call of this handle */
  int serial_equaliser;       /* 0 (default): each rx_process call forks the equaliser stage (sync,
                                 training, LMS rounds, stitching, labels, counters) on the data the
                                 earlier calls normalised onto an internal stream, concurrent with
                                 its own front-end; 1: everything in order on cuda_stream (for
                                 isolated kernel timing). Results are identical either way */
  long long q_window_symbols; /* > 0: also count bit errors / bits per window of this many
                                 symbols (window w = symbols [w W, (w+1) W)), the paper's "Q
                                 estimated from the BER in sections of 21 ms" (21 ms =
                                 42 M symbols at 2 GBaud); a multiple of lms_segment; 0 = off */
  int lms_mode;               /* 0 (default): decision-directed segments (SURVEY c-9 'Per block j');
                                 1: data aided - every segment adapts on the known PRBS reference
                                 exactly as the training pass does (c-9 'Training': e = r - y, no
                                 CPR), decisions slice(y) only feed labels / counters / EVM. The
                                 equaliser output then has no decision feedback, so it is compared
                                 with the oracle element by element (SURVEY §8(c) parity criterion
                                 'equaliser output in training mode'); a BER tester's reference-
                                 aided mode. Seeds: epoch means of the raw final taps (no R-SEED
                                 phase normalisation: no CPR, the frame is absolute);
                                 2: the paper's equaliser (KK only): a per-symbol
                                 (lms_block = 1, lms_taps <= 8) decision-directed LMS, widely linear
                                 per widely_linear, with NO separate CPR - the taps track the
                                 carrier ("symbol-phase recovery" by the equaliser); one serial
                                 recursion per segment (DESIGN reading R-DDLMS; raw-tap seeds) */
  int equaliser_lag;          /* side-stream equaliser (serial_equaliser = 0) only, 0..16. 0 (default):
                                 the work an rx_process call enqueues on cuda_stream ends with its own
                                 equaliser stage; L >= 1: with the stage forked L calls EARLIER, so a
                                 call's equaliser rounds overlap the next L calls' front-ends (the
                                 paper overlaps buffers across its five streams) - for small
                                 (one-buffer) calls, where a round runs only every
                                 lms_batch_segments / (segments per call) calls, L of about that
                                 ratio hides it. The rings grow by L calls. Labels of a call may then
                                 be written after its stream work completes: d_labels must stay
                                 valid until L more rx_process calls, or an rx_flush, rx_get_stats or
                                 rx_export_counters call, have been ordered behind it (the latter
                                 wait for every forked stage) */
  int shard_count;            /* time sharding of ONE stream (SURVEY §8(e) mode 2; KK chain): 0 or 1
                                 = off (rx_process); N > 1 = this handle is shard shard_index of N,
                                 fed with rx_shard_process (see below). Requires family KK,
                                 cpr_anchor = 1 and N <= tap_lag_epochs */
  int shard_index;
  int cuda_graphs;            /* 1 (default): a streaming equaliser round (segment recursion +
                                 stitching / labels / counters / seeds) is captured once as a CUDA
                                 graph and replayed per round (its kernels read every per-round
                                 quantity from device state); 0: launched kernel by kernel */
  int fused_front_end;        /* KK: 1 = both overlap-save stages (H11-H18) in one kernel (k_kk_fe),
                                 the 4-sps field E kept in shared memory (P:213 'to limit GPU memory
                                 access'; RX_PROBE_E then returns RX_EINVAL); 0 (default) = two
                                 kernels with E through an HBM ring (measured faster on B200, see
                                 DESIGN §6). z, labels and counters are bit-identical either way.
                                 Time shards (rx_shard_process) use the two kernels */
} rx_config;

/* Sample formats accepted by rx_process:
 *  RX_IN_U12_IN_U16: ADC codes 0..4095 right-aligned in uint16;
 *                    x = (code - 2047.5) / 2047.5 * adc_gain, codes 0 / 4095 count as clipped
 *  RX_IN_F32:        x = sample * adc_gain (already in x units; e.g. simulated or
 *                    pre-processed streams); nothing is counted as clipped */
/*  RX_IN_U12_PACKED: ADC codes packed 2 per 3 bytes, little-endian bit stream (sample k = bits
 *                    [12k, 12k + 12)), e.g. a digitiser's native 12-bit DMA format: 1.5 B per
 *                    sample over PCIe instead of 2. The library unpacks each call into an
 *                    internal u16 staging buffer (one HBM pass), then proceeds as RX_IN_U12_IN_U16 */
typedef enum { RX_IN_U12_IN_U16 = 0, RX_IN_F32 = 1, RX_IN_U12_PACKED = 2 } rx_input_format;

typedef struct rx_handle rx_handle;

typedef struct {
  long long samples_in;              /* samples accepted so far */
  long long symbols_out;             /* symbols with final labels (absolute m < symbols_out) */
  long long bit_errors, bits, symbols_counted;
  long long clipped;                 /* codes equal to 0 or 4095 */
  long long domain_errors, first_domain_error_index;   /* KK (A7); index -1 if none */
  double evm_num, evm_den;           /* sum |d - z'|^2, sum |d|^2 (decision-referenced) */
  int sync_offset, sync_phase, sync_polarity, synced;
  double sync_gamma, sync_phi0;
  int status_flags;                  /* RX_FLAG_* */
  long long launches;                /* kernels this handle has launched so far */
} rx_stats;

/* Set *cfg to the defaults for (family, order): PAM 2 GBaud 2 sps / KK 1 GBaud 4 sps. */
void rx_config_default(rx_config *cfg, int family, int order);

/* Validate cfg, allocate all device state on `cuda_device`, precompute the static-EQ spectra,
 * twiddles and PRBS reference tables. No allocation happens after this call. */
rx_status rx_create(const rx_config *cfg, int cuda_device, rx_handle **out);

/* Enqueue the chain on the next n_samples of the stream: uint16 u12 codes (the ADC format of
 * P:136 / S:602) or float32, as cfg.input_format says; d_samples 16-byte aligned device
 * memory on the handle's device. n_samples must be a multiple of hop and at most
 * (history_buffers - 2) * buffer_blocks * hop (one paper buffer with the default rings).
 * Samples are consumed in stream order (the overlap kernels are
 * chained). Outputs lag the input (held-back tail: 52 blocks of clock look-ahead for PAM,
 * one stage-2 block for KK, one buffer of normalisation, one LMS segment); everything that
 * becomes final is processed. The label of absolute symbol m is written to
 * d_labels[m % labels_capacity] (PAM: Gray label; QAM: Gray(i_I) << (k/2) | Gray(i_Q));
 * labels_capacity 0 = no labels. */
rx_status rx_process(rx_handle *h, const void *d_samples, long long n_samples,
                     unsigned char *d_labels, long long labels_capacity, void *cuda_stream);

/* End of stream: drain the tail with truncated windows (SURVEY c-3, A14) and finish every
 * symbol (the one call that synchronises cuda_stream, to run as many equaliser rounds as the
 * lag-D seed dependencies of the remaining segments need). After rx_flush only
 * rx_get_stats / rx_probe / rx_destroy are valid. */
rx_status rx_flush(rx_handle *h, unsigned char *d_labels, long long labels_capacity,
                   void *cuda_stream);

/* Synchronise `cuda_stream`, copy a snapshot of the cumulative counters to host_out. */
rx_status rx_get_stats(rx_handle *h, rx_stats *host_out, void *cuda_stream);

/* Enqueue on cuda_stream a copy of the cumulative counters into device memory d_out
 * (RX_NCOUNTERS doubles: bit_errors, bits, symbols_counted, evm_num, evm_den, clipped,
 * domain_errors, symbols_out) without synchronising the host, so a multi-GPU caller can
 * all-reduce them with NCCL on the same stream (one collective per round). */
#define RX_NCOUNTERS 8
rx_status rx_export_counters(rx_handle *h, double *d_out, void *cuda_stream);

/* Windowed BER counters (q_window_symbols > 0): synchronise cuda_stream and copy the bit errors
 * and counted bits of windows [first_window, first_window + n) to host_errors / host_bits
 * (n long longs each). Held: the window of the newest finalised symbol (still open: partial
 * counts) and the RX_Q_WINDOWS - 1 windows before it. RX_EINVAL if the trace is off or a
 * window is not held. rx_reset_stats does not clear the trace. */
#define RX_Q_WINDOWS 4096
rx_status rx_get_q_trace(rx_handle *h, long long first_window, int n, long long *host_errors,
                         long long *host_bits, void *cuda_stream);

/* PAM threshold calibration, the paper's "decision thresholds are optimized offline beforehand
 * and uploaded", read as in SPEC S:361: on finalised symbols [first_symbol,
 * first_symbol + count) still held in the device rings (after sync), the mean equaliser output
 * of the symbols whose PRBS reference level is i gives level i's position; the thresholds are
 * the midpoints between adjacent level means. Writes M-1 thresholds to host_thresholds and, if
 * not NULL, the M level means to host_level_means (pass the thresholds to rx_config.thresholds
 * of a new handle). Synchronises cuda_stream. RX_EINVAL: not PAM, range not finalised / held,
 * or a level without symbols; RX_ESTATE: not synced. */
rx_status rx_calibrate_thresholds(rx_handle *h, long long first_symbol, long long count,
                                  double *host_thresholds, double *host_level_means,
                                  void *cuda_stream);

/* KK DC-offset calibration. The paper restores the DC of the AC-coupled intensity "using the
 * method of [Luis:20]" without restating it; built as a grid search that reuses the
 * whole chain: for each of the n_candidates dc values a temporary handle with cfg (dc_offset
 * replaced) streams the n_samples of the calibration record at d_samples (device memory,
 * cfg->input_format) and is flushed; host_evm_db[i] gets its decision-referenced EVM (+inf if
 * frame sync failed), *best_index the lowest EVM (lowest index on ties). Synchronises
 * cuda_stream once per candidate. RX_EINVAL: not KK, bad sizes; other errors from rx_create /
 * rx_process are passed through. */
rx_status rx_calibrate_dc(const rx_config *cfg, int cuda_device, const void *d_samples,
                          long long n_samples, const double *candidates, int n_candidates,
                          double *host_evm_db, int *best_index, void *cuda_stream);

/* Static-equaliser design (host only, no GPU): the paper's static FIRs are "optimized offline"
 * (503 taps PAM; 203 taps KK) without a stated method; SPEC's reading:
 * per-bin regularised MMSE on the 1024-bin grid, H_eq[k] = conj(H_ch[k]) H_t[k] /
 * (|H_ch[k]|^2 + lambda), inverse DFT (1/N), zero-phase taps centred like rx_config.static_taps,
 * truncated to n_taps and re-windowed (Kaiser, beta = 6: DESIGN reading R-SEQ).
 * h_channel, h_target: 1024 complex bins interleaved (re, im), bin k = k/1024 of the sample rate.
 * real_taps = 1 writes the n_taps real parts (PAM), 0 writes 2 n_taps interleaved (KK).
 * RX_EINVAL: n_taps even or > 1023, lambda < 0, or a zero denominator. */
rx_status rx_design_static_eq(const double *h_channel, const double *h_target, double lambda,
                              int n_taps, int real_taps, double *taps_out);

/* Zero the BER/EVM/clip/domain counters (enqueued on cuda_stream). */
rx_status rx_reset_stats(rx_handle *h, void *cuda_stream);

/* Trained taps W_train (after sync + training): K values (PAM) or 2K interleaved (KK),
 * host_out capacity in doubles; a widely-linear handle also writes V_train (2K interleaved)
 * after W_train when capacity >= 4K. Synchronises the device. */
rx_status rx_get_taps(rx_handle *h, double *host_out, int capacity);

/* Start taps of the training pass, replacing the centre spike of SURVEY c-9 'Training':
 * a warm start from taps known for the channel (e.g. another handle's rx_get_taps).
 * host_in: n doubles, n = K (PAM, real) or 2K (KK, interleaved re/im), copied synchronously.
 * Returns RX_EINVAL on a size mismatch, RX_ESTATE once training has run (synchronises the
 * device to check). */
rx_status rx_set_taps(rx_handle *h, const double *host_in, int n);

/* Intermediate read-back for parity tests and tracing (synchronises `cuda_stream`).
 * Copies `count` elements starting at absolute index `first` of intermediate `which`
 * (still held in the device rings) to host_out. Returns RX_EINVAL if not held. */
typedef enum {
  RX_PROBE_C = 0,        /* PAM per block: C_b, complex double (re,im)          (H3) */
  RX_PROBE_TAU = 1,      /* PAM per block: tau_b, double                        (H4) */
  RX_PROBE_MB = 2,       /* PAM per block: M_b, int64                           (H4) */
  RX_PROBE_U = 3,        /* PAM per symbol: u_m, float                          (H7) */
  RX_PROBE_UHAT = 4,     /* PAM per symbol: normalised u_m, float               (H8) */
  RX_PROBE_E = 5,        /* KK per 4-sps sample: field E_p, complex float       (H15) */
  RX_PROBE_Z = 6,        /* KK per 2-sps sample: z_q, complex float             (H18) */
  RX_PROBE_CFO = 7,      /* KK per buffer: {P, df_hz, kstar, inc, origin} 5 doubles (H19-20) */
  RX_PROBE_Y = 8,        /* per symbol: equaliser output z'_m (after CPR), complex float
                            (PAM: imag 0)                                       (H9/H21-22) */
  RX_PROBE_LEVEL = 9,    /* per symbol: final level index (PAM i; QAM i_I | i_Q << 4), u8 */
  RX_PROBE_SEG = 10,     /* per segment: {R_s, r_s, theta_final, errors, evm_num, evm_den}
                            6 doubles                                           (H22) */
  RX_PROBE_DEBUG = 11    /* internal state words (int64), for diagnostics only */
} rx_probe;
rx_status rx_probe_read(rx_handle *h, int which, long long first, long long count,
                        void *host_out, void *cuda_stream);

/* Tracing (SURVEY §5 'tracing / profiling'; the paper reads its chain off profiler traces,
 * P:120). rx_profile_enable(h, mask) brackets every later launch of the kernel classes
 * in `mask` (bit i = class i below) with CUDA events on the launching stream; mask 0 stops.
 * rx_profile_read synchronises those events and returns, per class, the summed device time
 * (ms) and the launch count since the last read (arrays of RX_KCLASS_COUNT entries). */
typedef enum {
  RX_K_PAM_FE = 0,      /* H0-H3  ingest, R2C FFT, static EQ, C_b */
  RX_K_PAM_CLOCK = 1,   /* H4     105-block average, unwrap scan, tau_b, M_b */
  RX_K_PAM_BE = 2,      /* H1-H2, H5-H7 re-FFT, EQ, clock ramp, C2R IFFT, extraction */
  RX_K_NORM = 3,        /* H8     buffer normalisation */
  RX_K_KK_S1 = 4,       /* H0, H11-H15 KK front-end, Hilbert, reconstruction, downshift */
  RX_K_KK_S2 = 5,       /* H16-H18 C2C FFT, static EQ, decimating IFFT */
  RX_K_CFO = 6,         /* H19-H20 power, 4th-power periodogram, fine CFO */
  RX_K_SYNC = 7,        /* H24 frame sync + training */
  RX_K_LMS = 8,         /* H9, H21-H23 segment-parallel block-LMS + CPR + decisions */
  RX_K_LMS_POST = 9,    /* H22-H25 stitching, R_s scan, labels, counters, seeds */
  RX_K_MISC = 10,       /* history copy, bookkeeping */
  RX_K_KK_FE = 11,      /* H0, H11-H18 fused KK front-end (fused_front_end = 1): both stages, E on chip */
  RX_KCLASS_COUNT = 12
} rx_kernel_class;
rx_status rx_profile_enable(rx_handle *h, int mask);
rx_status rx_profile_read(rx_handle *h, double *host_ms, long long *host_counts, int n);

/* ---- Time-block sharding of one stream over GPUs (SURVEY §8(e) mode 2) -------------------------
 * The paper chains its buffers with ordered carries (the overlap kernel; the clock phase of
 * the previous buffer). Paper buffer b = input samples [b B4, (b+1) B4), B4 = 512
 * buffer_blocks; with shard_count = N, shard g owns the buffers b = g mod N and reads its input
 * halos itself: rx_shard_halo(h, &pre, &post) gives them (KK: RX_SHARD_PRE / RX_SHARD_POST; PAM:
 * the back-end look-back of the buffer's first segment plus the clock windows, 512 (PB + 2 + h) and
 * 512 (2 + h) with h = clock_avg_half, PB = (S + O + 2 floor(K/2) + 255) / 256 + 2).
 * What crosses a buffer boundary travels in one record per shard and round:
 *  KK: the CFO estimate (DDS phase origin = a prefix over all earlier buffers' estimates, c-8);
 *  PAM: the clock-phase wrap count of the buffer's own blocks (the unwrapped phase is theta_b -
 *    2 pi N_b, N_b an integer prefix over all earlier blocks; exact) and the buffer's
 *    normalisation scalars (dc, A; its neighbours normalise their look-back symbols with them);
 *  both: the frame-sync result and trained taps from the stream start, and the lag-D seed partial
 *    sums (c-9: 2^-32 fixed point, so an epoch split between shards gets the same seed).
 * Round r (buffers r N .. r N + N - 1):
 *  1. rx_shard_process(h, b = r N + g, ...): input samples [max(0, b B4 - pre), (b+1) B4 + post)
 *     (shorter only on the call holding the stream end, last = 1), device u16 codes. KK: stage 1 / 2
 *     over the blocks whose frames lie inside, CFO estimate of b. PAM: front-end and clock phases
 *     of b's blocks and their halo blocks. d_labels: where the labels of b's segments go (absolute
 *     symbol m at m % labels_capacity).
 *  2. rx_export_carry(h, d_rec): this round's record (rx_carry_size bytes, 16-byte aligned device
 *     memory); the caller all-gathers the N records in rank order into one device buffer (NCCL
 *     all-gather; no host staging).
 *  3. rx_import_carry(h, d_all, N, g): take the records. KK: DDS origin chain, sync / trained taps,
 *     seeds, then the equaliser, decisions, labels and counters of the shard's buffer of round
 *     r - 1 (its last segment needs z' of the next buffer, whose CFO estimate arrives now).
 *     PAM: the wrap base of b, scalars, sync / trained taps, seeds; the equaliser round of the
 *     shard's buffer of round r - 1 (segments s with (s + 1) S - 1 + floor(K/2) in its symbols,
 *     after normalising its look-back symbols with the previous buffer's scalars, which arrive
 *     now), then clock tau_b / M_b, back-end and normalisation of b (sync + training on b = 0).
 * After the round holding the stream end, one more export / gather / import without
 * rx_shard_process finishes every pending buffer. Labels are bit-identical and integer counters
 * (summed over shards) equal to one handle's on the same stream. Limits: KK needs cpr_anchor = 1
 * and N <= tap_lag_epochs; PAM N <= tap_lag_epochs - 2 (epochs drift against buffers with the
 * sampling clock; an epoch's seed can need the next round's partial). All calls are stream-ordered
 * and asynchronous; errors: RX_EINVAL (arguments, not a shard handle), RX_ESTATE (call order). */
#define RX_SHARD_PRE 4096
#define RX_SHARD_POST 4096
rx_status rx_shard_halo(const rx_handle *h, long long *pre, long long *post);
rx_status rx_shard_process(rx_handle *h, long long buffer, const void *d_samples, long long n_samples,
                           int last, unsigned char *d_labels, long long labels_capacity, void *cuda_stream);
rx_status rx_carry_size(const rx_handle *h, int *bytes);
rx_status rx_export_carry(rx_handle *h, void *d_buf, void *cuda_stream);
rx_status rx_import_carry(rx_handle *h, const void *d_gathered, int n_ranks, int my_rank, void *cuda_stream);

/* ---- Real-time monitor (the paper's real-time budget: one 2^22-sample
 * buffer per 1.049 ms at 4 GSa/s) -------------------------------------------------------
 * rx_rt_enable(h, 1) brackets every later rx_process call with CUDA events on its stream;
 * rx_get_rt_stats synchronises them and reports, over the calls since the last read: the count,
 * samples, summed span busy_ms, the longest call, max_load = max_k span_k / budget_k (budget =
 * n_k / sample_rate), overruns (calls slower than their budget) and realtime_ratio = (total
 * budget) / busy_ms (> 1: faster than real time). A call's span is its time on the caller's
 * stream (front end, the CFO / clock stages and the joined equaliser stage, per equaliser_lag). */
typedef struct {
  long long calls, samples, overruns;
  double busy_ms, max_call_ms, max_load, realtime_ratio;
} rx_rt_stats;
rx_status rx_rt_enable(rx_handle *h, int on);
rx_status rx_get_rt_stats(rx_handle *h, rx_rt_stats *host_out);

void rx_destroy(rx_handle *h);
const char *rx_strerror(int status);

/* Library build identification (e.g. "librx sm_100a <git>") */
const char *rx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RX_H */
