// rx_dev.cuh — device-resident state of one librx handle.
// Every ring is indexed by ABSOLUTE index (block b, sample p, 2-sps sample q, symbol m,
// segment s, buffer beta) modulo its power-of-two capacity, so results do not depend on how
// the caller chunks rx_process() calls (SURVEY §8(b) 'Ordering', §4 'Determinism').
#pragma once
#include "common.cuh"

#define RX_MAX_K 32
#define RX_MAX_PT 64
#define RX_MAX_O 512
#define RX_MAX_LAG 16        // rx_config.equaliser_lag upper bound

struct DevState {
  // ---- PAM clock recovery carries (unwrap needs the previous buffer's phase).
  // The unwrapped phase is theta^u_b = theta_b - 2 pi N_b with N_b = sum_{i <= b} rint((theta_i -
  // theta_{i-1}) / 2 pi) (the telescoped sum of the wrapped differences): wraps_prev = N of the
  // last block so far, an integer held in a double (exact), so it does not depend on how the
  // stream is cut into calls or shards.
  double theta_prev, wraps_prev;
  // ---- normalisation fronts
  long long v_front;        // PAM: uhat valid for m < v_front; KK: z' valid for q < v_front
  long long v_lms;          // the equaliser's snapshot of v_front, taken on the caller's stream
                            // before the call forks its equaliser work onto the side stream
  long long m_end;          // final symbol count (set at flush), else -1
  // ---- sync / training
  int synced, trained, sync_offset, sync_phase, sync_polarity, pad0;
  double sync_gamma, sync_phi0;
  // ---- LMS bookkeeping
  long long seg_next;       // first segment whose R_s is not yet known (= finalisation front)
  long long fin_lo, fin_hi; // segments finalised by the current round
  long long r_prefix;       // sum_{i <= seg_next-1} r_i (mod 4)
  int anchor_known, anchor_A;
  // ---- KK CFO DDS carry
  unsigned long long cfo_origin_next;
  double cfo_df_prev;
  // ---- counters (H25)
  long long bit_errors, bits, symbols_counted, clipped, domain_errors, first_domain;
  double evm_num, evm_den;
  long long symbols_out;
  int flags, pad1;
  // ---- PAM time shard (SURVEY §8(e) mode 2): local wrap count of the reference block
  // beta B - 1, wraps over the buffer's own blocks, the buffer's global base, the running
  // total over the buffers imported so far
  double sh_nref, sh_w, sh_nbase, wrap_total;
};

struct HostMirror {          // pinned, mapped: device writes hints the host reads lazily
  volatile long long seg_next;
  volatile int synced, trained;
};

struct CfoParam {            // per KK buffer (H19-H20)
  double P, df;
  unsigned long long inc, origin;
  float inv_sqrtP;
  int kstar;
};

#define RX_CARRY_SEEDS 3
struct SeedPart {            // one epoch's partial seed sum over the segments a round finalised
  long long epoch;           // -1: unused
  int n, pad;
  long long sum[RX_MAX_K][2];
};

struct RxDev {
  // ---- configuration
  int family, M, L;          // L = levels per axis (PAM: M, QAM: sqrt M)
  int kbits;                 // log2 M
  float scale;               // adc_gain / 2047.5
  float dc;                  // KK dc offset
  int sideband;
  unsigned long long carrier_inc;    // DDS increment of sigma * f_c (c-0)
  float2 carrier_st1, carrier_st128; // e^{-j psi} of 1 and 128 increments (host, fp64 -> fp32)
  double fs2;                // KK 2-sps rate
  int clock_half;
  int buffer_blocks;
  long long E_sym;           // symbols per LMS epoch
  int K, B, S, O, D, cpr, Pt;
  int anchor_each;           // KK: every segment's quadrant from the reference (R-ANCHOR2)
  int lms_mode;              // 0 decision directed (c-9), 1 data aided (reference-driven, no CPR)
  int shard_n, shard_g;      // time sharding (SURVEY §8(e) mode 2): buffers b = g mod n; 1, 0 = off
  float mu;
  int T_train;
  long long m0;
  int W_sync;
  float sync_min;
  long long warmup;
  int cfo_enable;
  int thr_default;           // PAM thresholds are the ideal midpoints (closed-form slicer)
  float qam_sc;              // QAM per-axis unit: levels (2i - L + 1) qam_sc
  // ---- constant tables (device)
  const float2 *tw;          // e^{-2 pi i k/1024}, k < 1024
  const float2 *H;           // static-EQ spectrum [1024]
  const float *Hr;           // its real part (used when the spectrum is real: H_real = 1)
  int H_real;
  const float *thr;          // PAM thresholds [M-1]
  const float *lvl;          // levels per axis [L]
  const float2 *ref_val;     // reference symbol values [P]
  const unsigned char *ref_lab;  // reference Gray labels [P]
  const unsigned char *ref_idx;  // reference level index (PAM i, QAM iI | iQ << 4) [P]
  const float2 *bps_rot;     // e^{-j phi_p}, p < Pt
  // ---- rings
  uint16_t *hist; float *histf; long long hist_cap;
  float2 *Xspec; long long xs_cap;      // PAM: R2C spectra of blocks [be_done, fe_done), 512 float2 each
  double2 *C; double *theta; double *tau; long long *Mb; double *blk_sum; double *blk_abs;
  long long blk_cap;
  float *u; float *uhat; long long sym_cap;
  double *norm_dc; double *norm_amp; long long *norm_cnt; long long buf_cap;
  double *norm_part; int *norm_tick;   // normalisation partials [16][NORM_G], tickets [16]
  double *clk_part, *clk_off, *clk_last; // unwrap tile totals / offsets / last phases
  long long *clk_flag;                   // fused clock: launch id that published each tile total
  int *clk_ticket;                       // fused clock: [0] tiles finished (the last one carries),
                                         // [1] tiles dispatched (dispatch-order tile index)
  float2 *E; long long E_cap;
  float2 *z; long long z_cap;
  int q_shift;                      // log2 of the 2-sps samples per buffer (buffer_blocks 256)
  CfoParam *cfo; float *cfo_part; double *cfo_pow; double2 *cfo_a; int *cfo_tick; int *cfo_tick_spec; int cfo_G;
  // ---- sync scratch
  float *sync_g; float2 *sync_c;
  // ---- LMS
  float2 *w_train;                 // [K]
  float2 *w_init;                  // [K] start taps of training (rx_set_taps)
  int has_winit;
  float2 *seed; int *seed_ready; long long seed_cap;   // per epoch [K]
  // lag-D seed accumulators per epoch (2^-32 fixed point, [seed_cap][RX_MAX_K][2]), segment
  // counts, tags (e + 1), and the partial sums of the latest round staged for the shard record
  long long *seed_acc; int *seed_cnt; long long *seed_tag;
  struct SeedPart *seed_xp;
  long long *buf_m;                // PAM shard: per buffer [4]: M of the pre-halo start, M_lo, M_hi
  int wl;                          // widely-linear equaliser (KK)
  float2 *v_train;                 // [K] trained v-branch (DD segments start theirs at 0)
  double *cal_part;                // PAM threshold calibration partials [CAL_G][16][2]
  long long q_segs;                // segments per Q-trace window (0 = off)
  unsigned long long *q_win;       // [RX_Q_WINDOWS][2]: bit errors, counted symbols
  float2 *seg_w; float *seg_theta; int *seg_done; int *seg_stitched; int *seg_r; int *seg_R;
  double *seg_evm; long long *seg_err; long long seg_cap;
  unsigned char *seg_warm;         // [seg_cap][O]
  unsigned char *level; unsigned char *level_fin; float2 *yout;   // per symbol rings (sym_cap)
  DevState *st;
  HostMirror *hm;                  // device pointer of the mapped host mirror
};

__device__ __forceinline__ long long rmod(long long i, long long cap) { return i & (cap - 1); }

__device__ __forceinline__ void set_flag(DevState *st, int f) { atomicOr(&st->flags, f); }
