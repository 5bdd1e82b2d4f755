// rx_api.cu — librx host side: the C ABI of include/rx.h, handle lifetime, constant tables,
// and the stream-ordered per-call orchestration of the kernels (no host synchronisation
// inside rx_process / rx_flush).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "rx.h"
#define RX_FLAG_SYNC_DEV RX_FLAG_SYNC
#include "k_pam.cuh"
#include "k_kk.cuh"
#include "k_lms.cuh"
#include "k_shard.cuh"

#ifndef RX_GIT
#define RX_GIT "dev"
#endif

// RX_SIDE_PRIO_LOW (experiments): the equaliser side stream at the lowest instead of the highest
// stream priority
static int g_side_low = getenv("RX_SIDE_PRIO_LOW") ? 1 : 0;
// KK CFO groups deferred on the side stream until this many buffers are pending (zp_due)
#ifndef CFO_DEFER_BUFS
#define CFO_DEFER_BUFS 4
#endif

// ------------------------------------------------------------------ small kernels
__global__ void k_pam_mend(RxDev d, long long be_done) {
  long long f = d.Mb[rmod(be_done, d.blk_cap)];
  if (f < 0) f = 0;
  d.st->v_front = f;
  d.st->m_end = f;
}
__global__ void k_kk_mend(RxDev d, long long q_end) {
  d.st->v_front = q_end;
  if (d.st->synced) {
    const long long h = d.st->sync_phase;
    long long me = (q_end - h + 1) / 2;
    d.st->m_end = me > 0 ? me : 0;
  } else {
    d.st->m_end = 0;
    set_flag(d.st, RX_FLAG_SYNC);
  }
}
__global__ void k_lms_snapshot(RxDev d) { d.st->v_lms = d.st->v_front; }

// RX_IN_U12_PACKED -> u16 codes: thread t turns bytes [12t, 12t + 12) (8 codes, sample k =
// bits [12k, 12k + 12) of the little-endian stream) into one 16-byte store
__global__ void __launch_bounds__(256) k_unpack12(const uint32_t *__restrict__ src, uint4 *__restrict__ dst,
                                                  long long n8) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n8; t += (long long)gridDim.x * blockDim.x) {
    const uint32_t w0 = __ldg(src + 3 * t), w1 = __ldg(src + 3 * t + 1), w2 = __ldg(src + 3 * t + 2);
    const uint32_t s0 = w0 & 0xFFFu, s1 = (w0 >> 12) & 0xFFFu, s2 = ((w0 >> 24) | (w1 << 8)) & 0xFFFu;
    const uint32_t s3 = (w1 >> 4) & 0xFFFu, s4 = (w1 >> 16) & 0xFFFu, s5 = ((w1 >> 28) | (w2 << 4)) & 0xFFFu;
    const uint32_t s6 = (w2 >> 8) & 0xFFFu, s7 = (w2 >> 20) & 0xFFFu;
    dst[t] = make_uint4(s0 | (s1 << 16), s2 | (s3 << 16), s4 | (s5 << 16), s6 | (s7 << 16));
  }
}

// PAM threshold calibration: per-CTA, per-reference-level sums and counts of the
// equaliser output over symbols [m0, m1), each thread in a fixed order, then a fixed-order CTA
// reduction (deterministic); the host adds the CTA partials in order
#define CAL_G 148
__global__ void __launch_bounds__(256) k_calib_levels(RxDev d, long long m0, long long m1) {
  __shared__ double ss[8][16], sc[8][16];
  double s[16], c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { s[i] = 0.0; c[i] = 0.0; }
  const long long o = d.st->sync_offset;
  for (long long m = m0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; m < m1;
       m += (long long)gridDim.x * blockDim.x) {
    const int lv = d.ref_idx[((o + m - d.m0) % RX_PREF + RX_PREF) % RX_PREF];
    const double y = (double)d.yout[rmod(m, d.sym_cap)].x;
#pragma unroll
    for (int i = 0; i < 16; ++i) if (i == lv) { s[i] += y; c[i] += 1.0; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double a = warp_sum_d(s[i]), b = warp_sum_d(c[i]);
    if (lane == 0) { ss[w][i] = a; sc[w][i] = b; }
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < 8; ++k) { a += ss[k][threadIdx.x]; b += sc[k][threadIdx.x]; }
    d.cal_part[(blockIdx.x * 16 + threadIdx.x) * 2] = a;
    d.cal_part[(blockIdx.x * 16 + threadIdx.x) * 2 + 1] = b;
  }
}
__global__ void k_export_counters(const DevState *st, double *o) {
  o[0] = (double)st->bit_errors; o[1] = (double)st->bits; o[2] = (double)st->symbols_counted;
  o[3] = st->evm_num; o[4] = st->evm_den; o[5] = (double)st->clipped;
  o[6] = (double)st->domain_errors; o[7] = (double)st->symbols_out;
}
__global__ void k_reset_counters(DevState *st) {
  st->bit_errors = st->bits = st->symbols_counted = st->clipped = st->domain_errors = 0;
  st->first_domain = 0x7fffffffffffffffLL;
  st->evm_num = st->evm_den = 0.0;
  st->flags = 0;
}

// ------------------------------------------------------------------ handle
struct rx_handle {
  rx_config cfg;
  int device;
  RxDev d;
  DevState *st_dev;
  HostMirror *hm_host;
  std::vector<void *> allocs;
  // host-known progress (absolute units)
  long long n_in, fe_done, clk_done, be_done, norm_done, s2_done, cfo_done;
  // Equaliser side stream: every streaming call forks the equaliser work on the data the
  // earlier calls normalised (sync, training, block-LMS rounds, stitching, labels, counters)
  // onto `side`, concurrently with its own front-end / clock / back-end / normalisation, and
  // joins it back before the call's work on the caller's stream ends.
  cudaStream_t side;
  cudaEvent_t ev_fork, ev_join[RX_MAX_LAG + 1];  // join of call k recorded in ev_join[k % (RX_MAX_LAG + 1)]
  long long ncall;                   // streaming rx_process calls so far
  long long lms_sym_ub;          // symbol upper bound of the data normalised by earlier calls
  uint16_t *unpacked;            // RX_IN_U12_PACKED: this call's codes unpacked to u16
  struct ZpJob { long long beta0, nb, q_front; int est; };
  std::vector<ZpJob> zp_pending; // KK: CFO groups deferred to the next call's side stream (est = 1:
                                 // estimate + carry, 0: carry only)
  long long clk_launch;          // fused clock launches so far (tags the tile totals)
  bool flushed;
  // time sharding (shard_count > 1): the buffer whose stage A ran last (awaiting export / stage B)
  // (PAM: c_lo / c_hi clock blocks, be_lo / be_hi back-end blocks of the buffer and its halo)
  struct ShardBuf { long long beta, qfront; int last, valid, exported; unsigned char *labels; long long cap;
                    long long c_lo, c_hi, be_lo, be_hi; };
  ShardBuf sh_cur, sh_pend;     // this round's stage A; the previous round's (stage B at import)
  long long sh_norm_beta;       // PAM: buffer normalised at the last import, for the next record
  long long sh_pre, sh_post;    // input halos (rx_shard_halo)
  long long sh_pb;              // PAM: back-end blocks before the buffer (equaliser look-back)
  long long launches;
  int sps;
  long long Q;   // 2-sps samples per buffer (KK)
  long long hist_cap;
  long long lms_launched_upto;   // segment estimate at the last equaliser launch
  long long lms_fin_est;         // host estimate of the finalised segment frontier (streaming)
  int n_sm;                      // SM count (persistent grids)
  int fe_slots;                  // resident k_kk_fe CTAs per GPU (occupancy x SMs)
  long long cfo_maxbuf;          // buffers per CFO launch (scratch rows)
  long long max_call;            // samples per rx_process call: (history_buffers - 2) buffers
  // tracing
  int prof_mask;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_free;
  // CUDA graph of one streaming equaliser round (cuda_graphs = 1): its kernels read every
  // per-round quantity from the device state, so one capture (fixed grid, the labels buffer
  // as captured) replays for every round
  cudaGraphExec_t lms_graph;
  unsigned char *lms_graph_labels;
  long long lms_graph_cap, lms_graph_nseg;
  int lms_graph_kernels;
  // real-time monitor (rx_rt_enable): per streaming call, events at its first and last operation
  // on the caller's stream and the call's sample count
  int rt_on;
  struct RtCall { cudaEvent_t a, b; long long n; };
  std::vector<RtCall> rt_pending;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> rt_free;
};

static void prof_begin(rx_handle *h, int cls, cudaStream_t s, cudaEvent_t *stop) {
  *stop = nullptr;
  if (!(h->prof_mask & (1 << cls))) return;
  std::pair<cudaEvent_t, cudaEvent_t> ev;
  if (!h->prof_free.empty()) { ev = h->prof_free.back(); h->prof_free.pop_back(); }
  else { cudaEventCreate(&ev.first); cudaEventCreate(&ev.second); }
  cudaEventRecord(ev.first, s);
  h->prof_pending.push_back({cls, ev});
  *stop = ev.second;
}

static long long next_pow2(long long x) {
  long long p = 1;
  while (p < x) p <<= 1;
  return p;
}

#define CK(x)                                      \
  do {                                             \
    cudaError_t e_ = (x);                          \
    if (e_ != cudaSuccess) {                       \
      fprintf(stderr, "librx: %s: %s\n", #x, cudaGetErrorString(e_)); \
      return RX_ECUDA;                             \
    }                                              \
  } while (0)

template <typename T>
static rx_status dalloc(rx_handle *h, T **p, long long n) {
  void *q = nullptr;
  size_t bytes = (size_t)(n > 0 ? n : 1) * sizeof(T);
  if (cudaMalloc(&q, bytes) != cudaSuccess) return RX_ENOMEM;
  if (cudaMemset(q, 0, bytes) != cudaSuccess) return RX_ECUDA;
  h->allocs.push_back(q);
  *p = (T *)q;
  return RX_OK;
}
template <typename T>
static rx_status dupload(rx_handle *h, const T **p, const std::vector<T> &v) {
  T *q;
  rx_status s = dalloc(h, &q, (long long)v.size());
  if (s) return s;
  if (cudaMemcpy(q, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return RX_ECUDA;
  *p = q;
  return RX_OK;
}

extern "C" void rx_config_default(rx_config *c, int family, int order) {
  memset(c, 0, sizeof(*c));
  c->family = family;
  c->order = order;
  c->baud = family == RX_PAM ? 2e9 : 1e9;
  c->sample_rate = 4e9;
  c->fft_size = 1024;
  c->hop = 512;
  c->buffer_blocks = 8192;
  c->adc_gain = 1.0;
  c->input_format = RX_IN_U12_IN_U16;
  c->clock_avg_half = 52;
  c->carrier_offset_hz = 0.547e9;
  c->sideband = -1;
  c->lms_taps = family == RX_PAM ? 15 : 4;
  c->lms_block = 32;
  c->lms_segment = 4096;
  c->lms_overlap = family == RX_PAM ? 0 : 256;
  c->tap_lag_epochs = 8;
  c->mu = family == RX_PAM ? 1e-3 : 2e-3;
  c->train_symbols = 8192;
  c->cfo_enable = 1;
  c->cpr_test_phases = order == 4 ? 0 : 32;
  c->cpr_anchor = 1;
  c->prbs_order = 15;
  c->prbs_seed = 0x7FFF;
  c->sync_start = 4096;
  c->sync_window = 2048;
  c->sync_min_corr = 0.3;
  c->history_buffers = 3;
  c->lms_batch_segments = family == RX_PAM ? 4096 : 2048;   // D epochs (one round each)
  c->cuda_graphs = 1;
  c->fused_front_end = 0;
}

extern "C" const char *rx_strerror(int s) {
  switch (s) {
    case RX_OK: return "ok";
    case RX_EINVAL: return "invalid argument or configuration";
    case RX_ENOMEM: return "device allocation failed";
    case RX_ECUDA: return "CUDA error";
    case RX_EDOMAIN: return "KK domain error (I + dc <= 0 seen)";
    case RX_ESYNC: return "frame synchronisation failed";
    case RX_EDIVERGE: return "equaliser diverged";
    case RX_ECAPACITY: return "capacity exceeded";
    case RX_ESTATE: return "call order violated";
    default: return "unknown status";
  }
}

extern "C" const char *rx_version(void) { return "librx sm_100a " RX_GIT; }

static bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }

static rx_status validate(const rx_config *c) {
  if (!c) return RX_EINVAL;
  if (c->family != RX_PAM && c->family != RX_QAM_KK) return RX_EINVAL;
  if (c->family == RX_PAM && !(c->order == 2 || c->order == 4 || c->order == 8 || c->order == 16)) return RX_EINVAL;
  if (c->family == RX_QAM_KK && !(c->order == 4 || c->order == 16 || c->order == 64)) return RX_EINVAL;
  if (!(c->baud > 0) || !(c->sample_rate > 0)) return RX_EINVAL;
  const double sps = c->sample_rate / c->baud;
  if (fabs(sps - (c->family == RX_PAM ? 2.0 : 4.0)) > 1e-9) return RX_EINVAL;
  if (c->fft_size != 1024 || c->hop != 512) return RX_EINVAL;
  if (c->buffer_blocks < 16 || !is_pow2(c->buffer_blocks)) return RX_EINVAL;
  if (!c->static_taps || c->n_static_taps < 1 || c->n_static_taps % 2 == 0 || c->n_static_taps > c->hop + 1)
    return RX_EINVAL;
  if (c->lms_taps < 1 || c->lms_taps > RX_MAX_K) return RX_EINVAL;
  // block LMS: B = 32; lms_mode 2 (per-symbol WL DDLMS, KK, K <= 8): B = 1
  if (c->lms_mode == 2 ? (c->lms_block != 1 || c->family != RX_QAM_KK || c->lms_taps > 8) : c->lms_block != 32)
    return RX_EINVAL;
  if (c->lms_segment < 64 || c->lms_segment % 32 || !is_pow2(c->lms_segment)) return RX_EINVAL;
  const long long E = (long long)c->buffer_blocks * (c->family == RX_PAM ? 256 : 128);
  if (E % c->lms_segment) return RX_EINVAL;
  if (c->lms_overlap < 0 || c->lms_overlap % 32 || c->lms_overlap > RX_MAX_O || c->lms_overlap > c->lms_segment) return RX_EINVAL;
  if (c->family == RX_PAM && c->lms_overlap != 0) return RX_EINVAL;
  if (c->tap_lag_epochs < 1 || c->tap_lag_epochs > 32) return RX_EINVAL;
  if (c->widely_linear != 0 && (c->widely_linear != 1 || c->family != RX_QAM_KK)) return RX_EINVAL;
  if (!(c->mu > 0) || c->mu > 1.0) return RX_EINVAL;
  if (c->train_symbols < 32 || c->train_symbols % 32) return RX_EINVAL;
  if (c->cpr_test_phases < 0 || c->cpr_test_phases > RX_MAX_PT) return RX_EINVAL;
  if (c->family == RX_QAM_KK && c->order > 4 && c->cpr_test_phases == 0) return RX_EINVAL;
  if (c->prbs_order != 15 || (c->prbs_seed & 0x7FFF) == 0) return RX_EINVAL;
  if (c->sync_start < 0 || c->sync_window < 64 || c->sync_window > 4096) return RX_EINVAL;
  if (c->clock_avg_half < 0 || c->clock_avg_half > 2048) return RX_EINVAL;
  if (c->history_buffers < 3 || c->history_buffers > 64) return RX_EINVAL;
  if (c->input_format != RX_IN_U12_IN_U16 && c->input_format != RX_IN_F32 && c->input_format != RX_IN_U12_PACKED)
    return RX_EINVAL;
  if (c->serial_equaliser != 0 && c->serial_equaliser != 1) return RX_EINVAL;
  if (c->cpr_anchor != 0 && c->cpr_anchor != 1) return RX_EINVAL;
  if (c->lms_mode < 0 || c->lms_mode > 2) return RX_EINVAL;
  if (c->equaliser_lag < 0 || c->equaliser_lag > RX_MAX_LAG) return RX_EINVAL;
  if (c->cuda_graphs != 0 && c->cuda_graphs != 1) return RX_EINVAL;
  if (c->fused_front_end != 0 && c->fused_front_end != 1) return RX_EINVAL;
  if (c->shard_count < 0 || c->shard_count > 64) return RX_EINVAL;
  if (c->shard_count > 1) {        // time sharding (SURVEY §8(e) mode 2)
    // KK: stage B of buffer b one round after its stage A, epochs = buffers: N <= D.
    // PAM: epochs drift against buffers with the clock, an epoch's last segments may finish a
    // round later on the next shard: N <= D - 2 keeps every lag-D seed ahead of its use.
    if (c->family == RX_QAM_KK && (c->cpr_anchor != 1 || c->shard_count > c->tap_lag_epochs)) return RX_EINVAL;
    if (c->family == RX_PAM && c->shard_count > c->tap_lag_epochs - 2) return RX_EINVAL;
    if (c->shard_index < 0 || c->shard_index >= c->shard_count) return RX_EINVAL;
  }
  if (c->q_window_symbols < 0 || (c->q_window_symbols > 0 && c->q_window_symbols % c->lms_segment)) return RX_EINVAL;
  if (c->lms_batch_segments < 0 || c->lms_batch_segments > (1 << 16)) return RX_EINVAL;
  if (c->family == RX_QAM_KK && !(c->sideband == 1 || c->sideband == -1)) return RX_EINVAL;
  if (c->family == RX_PAM && c->thresholds) {
    for (int i = 1; i < c->order - 1; ++i)
      if (!(c->thresholds[i] > c->thresholds[i - 1])) return RX_EINVAL;
  }
  return RX_OK;
}

// PRBS-15 (x^15 + x^14 + 1), library-side implementation: Galois-free Fibonacci register.
static void prbs_bits(unsigned seed, std::vector<int> &bits) {
  bits.resize(RX_PREF);
  unsigned s = seed & 0x7FFF;
  for (int i = 0; i < RX_PREF; ++i) {
    const unsigned b = ((s >> 14) ^ (s >> 13)) & 1u;
    s = ((s << 1) | b) & 0x7FFFu;
    bits[i] = (int)b;
  }
}
static int gray_dec(int g) {
  int i = 0;
  for (; g; g >>= 1) i ^= g;
  return i;
}

extern "C" void rx_destroy(rx_handle *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->side) cudaStreamSynchronize(h->side);   // equaliser work still reading the rings
  for (void *p : h->allocs) cudaFree(p);
  if (h->hm_host) cudaFreeHost(h->hm_host);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  for (int i = 0; i <= RX_MAX_LAG; ++i) if (h->ev_join[i]) cudaEventDestroy(h->ev_join[i]);
  for (auto &e : h->prof_pending) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
  for (auto &e : h->prof_free) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  if (h->lms_graph) cudaGraphExecDestroy(h->lms_graph);
  for (auto &e : h->rt_pending) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  for (auto &e : h->rt_free) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  delete h;
}

extern "C" rx_status rx_create(const rx_config *cfg, int cuda_device, rx_handle **out) {
  if (!out) return RX_EINVAL;
  *out = nullptr;
  rx_status vs = validate(cfg);
  if (vs) return vs;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) return RX_ECUDA;
  CK(cudaSetDevice(cuda_device));
  rx_handle *h = new rx_handle();
  h->cfg = *cfg;
  h->cfg.static_taps = nullptr;
  h->cfg.thresholds = nullptr;
  h->device = cuda_device;
  cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, cuda_device);
  const rx_config &c = *cfg;
  RxDev &d = h->d;
  memset(&d, 0, sizeof(d));
  const bool kk = c.family == RX_QAM_KK;
  d.family = c.family;
  d.M = c.order;
  d.L = kk ? (int)lround(sqrt((double)c.order)) : c.order;
  d.kbits = (int)lround(log2((double)c.order));
  d.scale = (float)(c.adc_gain / 2047.5);
  d.dc = (float)c.dc_offset;
  d.sideband = c.sideband;
  d.carrier_inc = (unsigned long long)llrint(ldexp((double)c.sideband * c.carrier_offset_hz / c.sample_rate, 64));
  {   // the kernels' per-thread DDS step rotations (dds_rot_neg of the top 32 bits, here in fp64)
    auto rot = [](unsigned long long u) {
      const double x = (double)(int)(u >> 32) * ldexp(1.0, -31) * 3.141592653589793;
      return make_float2((float)cos(x), (float)-sin(x));
    };
    d.carrier_st1 = rot(d.carrier_inc);
    d.carrier_st128 = rot(d.carrier_inc * 128ULL);
  }
  d.fs2 = c.sample_rate / 2.0;
  d.clock_half = c.clock_avg_half;
  d.buffer_blocks = c.buffer_blocks;
  d.E_sym = (long long)c.buffer_blocks * (kk ? 128 : 256);
  d.K = c.lms_taps; d.B = c.lms_block; d.S = c.lms_segment; d.O = c.lms_overlap;
  d.D = c.tap_lag_epochs;
  d.cpr = kk ? (c.cpr_test_phases == 0 ? 1 : 2) : 0;
  d.lms_mode = c.lms_mode;
  d.shard_n = c.shard_count > 1 ? c.shard_count : 1;
  d.shard_g = c.shard_count > 1 ? c.shard_index : 0;
  d.Pt = c.cpr_test_phases;
  d.anchor_each = kk && c.cpr_anchor;
  d.mu = (float)c.mu;
  d.T_train = c.train_symbols;
  d.m0 = c.sync_start;
  d.W_sync = c.sync_window;
  d.sync_min = (float)c.sync_min_corr;
  d.warmup = c.warmup_symbols;
  d.cfo_enable = kk ? c.cfo_enable : 0;
  d.thr_default = cfg->thresholds ? 0 : 1;
  d.qam_sc = kk ? (float)sqrt(3.0 / (2.0 * (c.order - 1))) : 0.f;
  h->sps = kk ? 4 : 2;
  const int HB = c.history_buffers;
  h->Q = (long long)c.buffer_blocks * 256;
  rx_status s = RX_OK;
#define TRY(x) do { s = (x); if (s) { rx_destroy(h); return s; } } while (0)
  // ---- constant tables
  std::vector<float2> tw(1024, make_float2(0.f, 0.f));   // layout: see fft.cuh
  auto w1024 = [](long long k) {
    const double a = -2.0 * M_PI * (double)(k % 1024) / 1024.0;
    return make_float2((float)cos(a), (float)sin(a));
  };
  for (int k = 0; k < 512; ++k) tw[k] = w1024(k);
  for (int r = 1; r < 8; ++r)
    for (int j = 0; j < 64; ++j) tw[TW_P3 + 64 * (r - 1) + j] = w1024(2LL * r * j);
  for (int r = 1; r < 8; ++r)
    for (int k = 0; k < 8; ++k) tw[TW_P2 + 8 * (r - 1) + k] = w1024(16LL * r * k);
  TRY(dupload(h, &d.tw, tw));
  // static EQ spectrum H = DFT_1024(h_c), h_c[n mod N] = taps[(L-1)/2 + n] (SURVEY c-0, A3)
  {
    std::vector<float2> H(1024);
    const int L = c.n_static_taps, half = (L - 1) / 2;
    for (int k = 0; k < 1024; ++k) {
      double re = 0.0, im = 0.0;
      for (int n = -half; n <= half; ++n) {
        const double tr = kk ? cfg->static_taps[2 * (half + n)] : cfg->static_taps[half + n];
        const double ti = kk ? cfg->static_taps[2 * (half + n) + 1] : 0.0;
        const double a = -2.0 * M_PI * (double)k * (double)n / 1024.0;
        const double cs = cos(a), sn = sin(a);
        re += tr * cs - ti * sn;
        im += tr * sn + ti * cs;
      }
      H[k] = make_float2((float)re, (float)im);
    }
    TRY(dupload(h, &d.H, H));
    std::vector<float> Hr(1024);
    bool real = true;
    for (int k = 0; k < 1024; ++k) { Hr[k] = H[k].x; if (H[k].y != 0.0f) real = false; }
    // symmetric real taps give an exactly real spectrum up to rounding: treat |imag| < 1e-6 max|H|
    float mx = 0.f;
    for (int k = 0; k < 1024; ++k) mx = fmaxf(mx, fabsf(H[k].x));
    real = true;
    for (int k = 0; k < 1024; ++k) if (fabsf(H[k].y) > 1e-7f * mx) real = false;
    d.H_real = real ? 1 : 0;
    TRY(dupload(h, &d.Hr, Hr));
  }
  // decision levels / thresholds (c-11)
  {
    std::vector<float> lv(d.L), th(d.M > 1 ? d.M - 1 : 1);
    if (!kk) {
      for (int i = 0; i < d.M; ++i) lv[i] = (float)((2.0 * i - d.M + 1) / (double)(d.M - 1));
      for (int i = 0; i < d.M - 1; ++i) {
        const double a = (2.0 * i - d.M + 1) / (double)(d.M - 1), b = (2.0 * (i + 1) - d.M + 1) / (double)(d.M - 1);
        th[i] = cfg->thresholds ? (float)cfg->thresholds[i] : (float)(0.5 * (a + b));
      }
    } else {
      const double sc = sqrt(3.0 / (2.0 * (d.M - 1)));
      for (int i = 0; i < d.L; ++i) lv[i] = (float)((2.0 * i - d.L + 1) * sc);
    }
    TRY(dupload(h, &d.lvl, lv));
    TRY(dupload(h, &d.thr, th));
  }
  // PRBS reference (c-10): symbol i = bits [k i, k i + k) mod P, MSB first, Gray label
  {
    std::vector<int> bits;
    prbs_bits(c.prbs_seed, bits);
    std::vector<float2> rv(RX_PREF);
    std::vector<unsigned char> rl(RX_PREF), ri(RX_PREF);
    const int k = d.kbits;
    std::vector<float> lvh(d.L);
    const double sc = kk ? sqrt(3.0 / (2.0 * (d.M - 1))) : 0.0;
    for (int i = 0; i < d.L; ++i) lvh[i] = kk ? (float)((2.0 * i - d.L + 1) * sc) : (float)((2.0 * i - d.M + 1) / (double)(d.M - 1));
    for (int i = 0; i < RX_PREF; ++i) {
      int lab = 0;
      for (int t = 0; t < k; ++t) lab = (lab << 1) | bits[((long long)i * k + t) % RX_PREF];
      rl[i] = (unsigned char)lab;
      if (!kk) {
        const int li = gray_dec(lab);
        ri[i] = (unsigned char)li;
        rv[i] = make_float2(lvh[li], 0.f);
      } else {
        const int b = k / 2;
        const int iI = gray_dec(lab >> b), iQ = gray_dec(lab & ((1 << b) - 1));
        ri[i] = (unsigned char)(iI | (iQ << 4));
        rv[i] = make_float2(lvh[iI], lvh[iQ]);
      }
    }
    TRY(dupload(h, &d.ref_val, rv));
    TRY(dupload(h, &d.ref_lab, rl));
    TRY(dupload(h, &d.ref_idx, ri));
    std::vector<float2> rot(RX_MAX_PT);
    for (int p = 0; p < RX_MAX_PT; ++p) {
      const int Pt = c.cpr_test_phases > 0 ? c.cpr_test_phases : 1;
      const double ph = -M_PI / 4 + (p + 0.5) * (M_PI / 2) / Pt;
      rot[p] = make_float2((float)cos(ph), (float)-sin(ph));
    }
    TRY(dupload(h, &d.bps_rot, rot));
  }
  // ---- rings
  h->max_call = (long long)(HB - 2) * c.buffer_blocks * 512;
  h->hist_cap = next_pow2(h->max_call + (1 << 18));   // > max call + clock lookback + kept tail
  d.hist_cap = h->hist_cap;
  if (c.input_format == RX_IN_U12_PACKED) TRY(dalloc(h, &h->unpacked, h->max_call));
  if (c.input_format == RX_IN_F32) TRY(dalloc(h, &d.histf, d.hist_cap));
  else TRY(dalloc(h, &d.hist, d.hist_cap));
  // PAM time shard: back-end blocks before the buffer so its first segment (whose last tap may sit
  // S - 1 symbols into the buffer) has its look-back O and taps; input halos for those blocks'
  // clock windows and overlap-save frames
  h->sh_pb = ((long long)c.lms_segment + c.lms_overlap + 2 * (c.lms_taps / 2) + 255) / 256 + 2;
  if (kk) { h->sh_pre = RX_SHARD_PRE; h->sh_post = RX_SHARD_POST; }
  else {
    h->sh_pre = 512 * (h->sh_pb + 2 + c.clock_avg_half);
    h->sh_post = 512 * (2 + (long long)c.clock_avg_half);
  }
  d.blk_cap = next_pow2((long long)HB * c.buffer_blocks + 256);
  if (!kk) {   // spectra from k_pam_fe to k_pam_be: one call + the clock look-ahead
    d.xs_cap = next_pow2((long long)(HB - 2) * c.buffer_blocks + 2 * c.clock_avg_half + 64);
    if (c.shard_count > 1 && d.xs_cap < next_pow2(c.buffer_blocks + h->sh_pb + 2 * c.clock_avg_half + 8))
      d.xs_cap = next_pow2(c.buffer_blocks + h->sh_pb + 2 * c.clock_avg_half + 8);
    TRY(dalloc(h, &d.Xspec, d.xs_cap * 512));
  }

  // equaliser batch + the seed-blocked tail that may wait for the next batch (<= D epochs)
  const long long E_sym = (long long)c.buffer_blocks * (kk ? 128 : 256);
  const long long tail_sym = (long long)c.tap_lag_epochs * E_sym;
  const long long bsym = (long long)c.lms_batch_segments * c.lms_segment;
  const long long batch_sym = bsym + (bsym > tail_sym ? tail_sym : bsym);
  // (HB + 1 buffers: the equaliser side stream reads the previous calls' symbols while the
  // current call writes up to one more call of them)
  // (equaliser_lag = L: the side stream may still read L more calls of them)
  const long long lag_calls = 1 + c.equaliser_lag;
  // per-buffer scalars (KK CFO parameters: z' is formed from them where the equaliser reads it;
  // PAM normalisation): every buffer the equaliser may still read - one batch + the seed-blocked
  // tail behind the front - plus the calls in flight on both streams
  {
    const long long need = batch_sym / E_sym + 2LL * HB + 4 + (long long)c.equaliser_lag * (HB - 2) + CFO_DEFER_BUFS;
    d.buf_cap = next_pow2(need > 64 ? need : 64);
  }
  d.sym_cap = next_pow2((long long)(HB + lag_calls * (HB - 2)) * c.buffer_blocks * (kk ? 128 : 260) + batch_sym);
  if (!kk && c.shard_count > 1) {   // buffers b and b + N (and halos) are held together
    const long long need = (long long)(c.shard_count + 2) * c.buffer_blocks * 260;
    if (d.sym_cap < next_pow2(need)) d.sym_cap = next_pow2(need);
    const long long nb = c.buffer_blocks + h->sh_pb + 2 * c.clock_avg_half + 8;
    if (d.blk_cap < next_pow2(nb)) d.blk_cap = next_pow2(nb);
  }
  if (!kk) {
    TRY(dalloc(h, &d.C, d.blk_cap));
    TRY(dalloc(h, &d.theta, d.blk_cap));
    TRY(dalloc(h, &d.tau, d.blk_cap));
    TRY(dalloc(h, &d.Mb, d.blk_cap));
    TRY(dalloc(h, &d.blk_sum, d.blk_cap));
    TRY(dalloc(h, &d.blk_abs, d.blk_cap));
    TRY(dalloc(h, &d.u, d.sym_cap));
    TRY(dalloc(h, &d.uhat, d.sym_cap));
    TRY(dalloc(h, &d.norm_dc, d.buf_cap));
    TRY(dalloc(h, &d.norm_amp, d.buf_cap));
    TRY(dalloc(h, &d.norm_cnt, d.buf_cap));
    TRY(dalloc(h, &d.norm_part, 16 * NORM_G));
    TRY(dalloc(h, &d.norm_tick, 16));
    long long maxtiles = ((long long)(HB - 2) * c.buffer_blocks + CLK_TILE - 1) / CLK_TILE + 2;
    if (c.shard_count > 1) maxtiles += (h->sh_pb + 4 + CLK_TILE - 1) / CLK_TILE + 1;
    TRY(dalloc(h, &d.clk_part, maxtiles));
    TRY(dalloc(h, &d.clk_off, maxtiles));
    TRY(dalloc(h, &d.clk_last, maxtiles));
    TRY(dalloc(h, &d.clk_flag, maxtiles));
    TRY(dalloc(h, &d.clk_ticket, 2));   // [0] tiles finished, [1] tiles dispatched
  } else {
    d.E_cap = next_pow2((long long)HB * c.buffer_blocks * 512);
    // z is read by the equaliser (z' on the fly, zp_value) up to one batch + D epochs after stage 2
    // wrote it, on the side stream while the current call writes one more call of it
    d.z_cap = next_pow2((long long)(HB + lag_calls * (HB - 2)) * c.buffer_blocks * 256 + 2 * batch_sym);
    if (c.shard_count > 1)   // a shard's buffers b and b + N (plus halos) are held together
      d.z_cap = next_pow2((long long)(c.shard_count + 2) * c.buffer_blocks * 256 + 2 * RX_SHARD_POST);
    if (!c.fused_front_end || c.shard_count > 1) TRY(dalloc(h, &d.E, d.E_cap));   // fused: E stays on chip
    TRY(dalloc(h, &d.z, d.z_cap));
    d.q_shift = 0;
    while ((1LL << d.q_shift) < (long long)c.buffer_blocks * 256) ++d.q_shift;
    TRY(dalloc(h, &d.cfo, d.buf_cap));
    d.cfo_G = CFO_ROWS + CFO_ROWS / CFO_GRP;             // spectrum rows per buffer (+ group rows)
    const long long maxbuf = HB > 8 ? HB : 8;              // buffers per CFO launch (a call's, or deferred groups)
    h->cfo_maxbuf = maxbuf;
    TRY(dalloc(h, &d.cfo_part, maxbuf * d.cfo_G * 1024));
    TRY(dalloc(h, &d.cfo_pow, maxbuf * d.cfo_G));
    TRY(dalloc(h, &d.cfo_tick, maxbuf));
    TRY(dalloc(h, &d.cfo_tick_spec, maxbuf * (CFO_ROWS / CFO_GRP + 1)));
    TRY(dalloc(h, &d.cfo_a, maxbuf * (h->Q / 1024 + 1)));
  }
  TRY(dalloc(h, &d.sync_g, 2 * RX_PREF));
  TRY(dalloc(h, &d.sync_c, 2 * RX_PREF));
  TRY(dalloc(h, &d.w_train, RX_MAX_K));
  TRY(dalloc(h, &d.w_init, RX_MAX_K));
  d.seed_cap = 64;
  TRY(dalloc(h, &d.seed, d.seed_cap * RX_MAX_K));
  if (c.shard_count > 1) {
    h->cfg.serial_equaliser = 1;   // a shard orders everything on the caller's stream
  }
  h->sh_cur.valid = h->sh_pend.valid = 0;
  h->sh_norm_beta = -1;
  d.wl = c.widely_linear;
  if (d.wl) TRY(dalloc(h, &d.v_train, RX_MAX_K));
  if (!kk) TRY(dalloc(h, &d.cal_part, (long long)CAL_G * 16 * 2));
  d.q_segs = c.q_window_symbols / c.lms_segment;
  if (d.q_segs > 0) TRY(dalloc(h, &d.q_win, 2 * RX_Q_WINDOWS));
  TRY(dalloc(h, &d.seed_ready, d.seed_cap));
  TRY(dalloc(h, &d.seed_acc, d.seed_cap * RX_MAX_K * 2));
  TRY(dalloc(h, &d.seed_cnt, d.seed_cap));
  TRY(dalloc(h, &d.seed_tag, d.seed_cap));
  TRY(dalloc(h, &d.seed_xp, RX_CARRY_SEEDS));
  TRY(cudaMemset(d.seed_xp, 0xFF, RX_CARRY_SEEDS * sizeof(SeedPart)) == cudaSuccess ? RX_OK : RX_ECUDA);   // epoch -1
  TRY(dalloc(h, &d.buf_m, d.buf_cap * 4));
  d.seg_cap = next_pow2(d.sym_cap / c.lms_segment + 8);
  TRY(dalloc(h, &d.seg_w, d.seg_cap * RX_MAX_K));
  TRY(dalloc(h, &d.seg_theta, d.seg_cap));
  TRY(dalloc(h, &d.seg_done, d.seg_cap));
  TRY(dalloc(h, &d.seg_stitched, d.seg_cap));
  TRY(dalloc(h, &d.seg_r, d.seg_cap));
  TRY(dalloc(h, &d.seg_R, d.seg_cap));
  TRY(dalloc(h, &d.seg_evm, 2 * d.seg_cap));
  TRY(dalloc(h, &d.seg_err, 2 * d.seg_cap));
  if (c.lms_overlap > 0) TRY(dalloc(h, &d.seg_warm, d.seg_cap * c.lms_overlap));
  TRY(dalloc(h, &d.level, d.sym_cap));
  if (kk) TRY(dalloc(h, &d.level_fin, d.sym_cap));
  else d.level_fin = d.level;            // PAM: R_s = 0, the segment frame is final
  TRY(dalloc(h, &d.yout, d.sym_cap));
  // ---- state
  TRY(dalloc(h, &h->st_dev, 1));
  {
    DevState st;
    memset(&st, 0, sizeof(st));
    st.m_end = -1;
    st.first_domain = 0x7fffffffffffffffLL;
    if (cudaMemcpy(h->st_dev, &st, sizeof(st), cudaMemcpyHostToDevice) != cudaSuccess) { rx_destroy(h); return RX_ECUDA; }
  }
  d.st = h->st_dev;
  if (cudaHostAlloc((void **)&h->hm_host, sizeof(HostMirror), cudaHostAllocMapped) != cudaSuccess) { rx_destroy(h); return RX_ENOMEM; }
  memset((void *)h->hm_host, 0, sizeof(HostMirror));
  if (cudaHostGetDevicePointer((void **)&d.hm, (void *)h->hm_host, 0) != cudaSuccess) { rx_destroy(h); return RX_ECUDA; }
  // kernels needing > 48 KB dynamic shared memory
  const size_t clk_smem = (CLK_TILE + 1 + 2 * c.clock_avg_half) * sizeof(double2);
  if (cudaFuncSetAttribute(k_pam_theta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)clk_smem) != cudaSuccess ||
      cudaFuncSetAttribute(k_pam_theta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)clk_smem) != cudaSuccess ||
      cudaFuncSetAttribute(k_sync_corr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536) != cudaSuccess ||
      cudaFuncSetAttribute(k_sync_corr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536) != cudaSuccess ||
      cudaFuncSetAttribute(k_kk_fe, cudaFuncAttributeMaxDynamicSharedMemorySize, KKFE_SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_cfo_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, CFO_STAGE_SMEM) != cudaSuccess) {
    rx_destroy(h);
    return RX_ECUDA;
  }
  {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kk_fe, 256, KKFE_SMEM) != cudaSuccess || per_sm < 1) {
      rx_destroy(h);
      return RX_ECUDA;
    }
    h->fe_slots = per_sm * h->n_sm;
  }
  {
    int lo = 0, hi = 0;   // the equaliser's latency-bound warps get the SM slots first
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, g_side_low ? lo : hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        [&] {
          for (int i = 0; i <= RX_MAX_LAG; ++i)
            if (cudaEventCreateWithFlags(&h->ev_join[i], cudaEventDisableTiming) != cudaSuccess) return true;
          return false;
        }()) {
      rx_destroy(h);
      return RX_ECUDA;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) { rx_destroy(h); return RX_ECUDA; }
#undef TRY
  *out = h;
  return RX_OK;
}

// ------------------------------------------------------------------ orchestration
#define KLAUNCH(h, cls, s, ...)          \
  do {                                   \
    cudaEvent_t stop_;                   \
    prof_begin((h), (cls), (s), &stop_); \
    __VA_ARGS__;                         \
    if (stop_) cudaEventRecord(stop_, (s)); \
    (h)->launches++;                     \
    if (g_rx_debug) {                    \
      fprintf(stderr, "librx: launch %s ...", #__VA_ARGS__); \
      cudaError_t e__ = cudaStreamSynchronize(s); \
      fprintf(stderr, " %s\n", cudaGetErrorString(e__)); \
    }                                    \
  } while (0)
static int g_rx_debug = getenv("RX_DEBUG_SYNC") ? 1 : 0;
// RX_CLK_FUSE_MAX (tests only): largest call, in clock tiles, that runs the fused one-pass clock
// kernel; larger calls take the three-launch path (default CLK_FUSE_MAX)
static long long g_clk_fuse_max = getenv("RX_CLK_FUSE_MAX") ? atoll(getenv("RX_CLK_FUSE_MAX")) : CLK_FUSE_MAX;

static rx_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "librx: launch failed: %s\n", cudaGetErrorString(e));
    return RX_ECUDA;
  }
  return RX_OK;
}

static unsigned gridc(long long n, int per) { return (unsigned)((n + per - 1) / per); }

// Programmatic dependent launch (sm_90+): the kernel may be scheduled while the previous kernel of
// the stream drains; it runs its independent prologue and then pdl_wait()s (common.cuh) before
// reading what that kernel produced. Only used for kernels that call pdl_wait() before any
// dependent access (KK stage 2, CFO periodogram and fine CFO; PAM clock and back-end; the
// equaliser's post-processing chain).
static bool g_no_pdl = getenv("RX_NO_PDL") != nullptr;
static long long g_fe_per_cta = getenv("RX_FE_PER_CTA") ? atoll(getenv("RX_FE_PER_CTA")) : 0;   // k_kk_fe experiments
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  if (g_no_pdl) { k<<<grid, block, smem, s>>>(args...); return; }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// tap padding KP in {4, 8, 16, 32} (compile-time) and the CPR flavour select the instance
typedef void (*lms_seg_fn)(RxDev, int, int, unsigned char *, long long);
typedef void (*lms_train_fn)(RxDev, int);
static int kp_of(int K) { return K <= 4 ? 4 : (K <= 8 ? 8 : (K <= 16 ? 16 : 32)); }
template <bool CPLX, int CPR, bool WL = false, int MODE = 1>
static lms_seg_fn seg_kp(int K) {
  switch (kp_of(K)) {
    case 4: return k_lms_seg<CPLX, CPR, 4, WL, MODE>;
    case 8: return k_lms_seg<CPLX, CPR, 8, WL, MODE>;
    case 16: return k_lms_seg<CPLX, CPR, 16, WL, MODE>;
    default: return k_lms_seg<CPLX, CPR, 32, WL, MODE>;
  }
}
static lms_seg_fn lms_seg_kernel(const RxDev &d) {
  if (d.lms_mode == 1) {   // data aided: reference-driven updates, no CPR (MODE 2)
    if (d.family == RX_PAM) return seg_kp<false, 0, false, 2>(d.K);
    return d.wl ? seg_kp<true, 0, true, 2>(d.K) : seg_kp<true, 0, false, 2>(d.K);
  }
  if (d.family == RX_PAM) return seg_kp<false, 0>(d.K);
  if (d.wl) return d.cpr == 1 ? seg_kp<true, 1, true>(d.K) : seg_kp<true, 2, true>(d.K);
  return d.cpr == 1 ? seg_kp<true, 1>(d.K) : seg_kp<true, 2>(d.K);
}
template <bool CPLX, bool WL = false>
static lms_train_fn lms_train_kp(int K) {
  switch (kp_of(K)) {
    case 4: return k_lms_train<CPLX, 4, WL>;
    case 8: return k_lms_train<CPLX, 8, WL>;
    case 16: return k_lms_train<CPLX, 16, WL>;
    default: return k_lms_train<CPLX, 32, WL>;
  }
}
template <bool CPLX>
static lms_train_fn lms_train_kernel(const RxDev &d) {
  if (CPLX && d.lms_mode == 2) {   // per-symbol DDLMS: B = 1 training pass
    if (d.wl) return d.K <= 4 ? k_lms_train_sym<4, true> : k_lms_train_sym<8, true>;
    return d.K <= 4 ? k_lms_train_sym<4, false> : k_lms_train_sym<8, false>;
  }
  if (CPLX && d.wl) return lms_train_kp<true, true>(d.K);
  return lms_train_kp<CPLX>(d.K);
}
static lms_seg_fn lms_sym_kernel(const RxDev &d) {
  if (d.wl) return d.K <= 4 ? k_lms_sym<4, true> : k_lms_sym<8, true>;
  return d.K <= 4 ? k_lms_sym<4, false> : k_lms_sym<8, false>;
}

template <bool CPLX>
static void launch_sync_train(rx_handle *h, cudaStream_t s, int flush) {
  RxDev &d = h->d;
  if (h->hm_host->trained) return;
  const int nh = CPLX ? 2 : 1;
  const size_t smem = (size_t)nh * d.W_sync * sizeof(float2);
  if (!h->hm_host->synced) {
    KLAUNCH(h, RX_K_SYNC, s, (k_sync_corr<CPLX><<<gridc((long long)nh * RX_PREF, 256), 256, smem, s>>>(d)));
    KLAUNCH(h, RX_K_SYNC, s, (k_sync_pick<CPLX><<<1, 1024, 0, s>>>(d, flush)));
  }
  KLAUNCH(h, RX_K_SYNC, s, (lms_train_kernel<CPLX>(d)<<<1, 32, 0, s>>>(d, flush)));
}

static void launch_lms_round(rx_handle *h, cudaStream_t s, unsigned char *labels, long long lab_cap,
                             int flush, long long nseg) {
  RxDev &d = h->d;
  const long long S = d.S;
  // segments per CTA: wpc warps, BPS segments on LMS_PAIR warps each (k_lms_seg); the
  // per-symbol DDLMS (lms_mode 2) runs one segment per thread (k_lms_sym)
  const int wpc = d.family == RX_PAM ? LMS_SPC_PAM : LMS_SPC_KK;   // warps per CTA
  const int spc = (d.cpr == 2 && d.lms_mode == 0) ? wpc / LMS_PAIR : wpc;
  if (d.lms_mode == 2)
    KLAUNCH(h, RX_K_LMS, s, (lms_sym_kernel(d)<<<gridc(nseg, 32), 32, 0, s>>>(d, flush, (int)nseg, labels, lab_cap)));
  else
    KLAUNCH(h, RX_K_LMS, s, (lms_seg_kernel(d)<<<gridc(nseg, spc), 32 * wpc, 0, s>>>(d, flush, (int)nseg, labels, lab_cap)));
  if (d.family == RX_PAM) {
    // PAM segments wrote their labels and error counts; the prefix also adds the counters
    KLAUNCH(h, RX_K_LMS_POST, s, launch_pdl(k_lms_prefix, 1, 1024, 0, s, d, flush, (int)nseg));
  } else {
    // anchored quadrants (R-ANCHOR2): k_lms_final takes each R_s itself; the c-9 chain stitches first
    if (!d.anchor_each) KLAUNCH(h, RX_K_LMS_POST, s, (k_lms_stitch<<<(unsigned)nseg, 256, 0, s>>>(d, (int)nseg)));
    KLAUNCH(h, RX_K_LMS_POST, s, launch_pdl(k_lms_prefix, 1, 1024, 0, s, d, flush, (int)nseg));
    KLAUNCH(h, RX_K_LMS_POST, s, launch_pdl(k_lms_final, (unsigned)nseg, LMS_FINAL_T, 0, s, d, labels, lab_cap, (int)nseg));
    KLAUNCH(h, RX_K_LMS_POST, s, launch_pdl(k_lms_counters, 1, 1024, 0, s, d));
  }
  const unsigned nseed = (unsigned)(nseg * S / d.E_sym + 2);
  KLAUNCH(h, RX_K_LMS_POST, s, launch_pdl(k_lms_seeds, nseed > RX_CARRY_SEEDS ? nseed : RX_CARRY_SEEDS, 1024, 0, s, d, flush));
}

// A streaming equaliser round as a CUDA graph (NEXT-2): captured once with a fixed grid that covers
// any streaming round's segments (the kernels take seg_next / fin_lo / fin_hi from the device
// state and skip what is not ready), then replayed with one cudaGraphLaunch per round. Not used
// while tracing (rx_profile_enable) or with RX_DEBUG_SYNC; re-captured if the labels buffer moves.
static bool lms_graph_round(rx_handle *h, cudaStream_t s, unsigned char *labels, long long lab_cap, long long nseg) {
  if (!h->cfg.cuda_graphs || h->prof_mask || g_rx_debug) return false;
  RxDev &d = h->d;
  if (!h->lms_graph || labels != h->lms_graph_labels || lab_cap != h->lms_graph_cap || nseg > h->lms_graph_nseg) {
    if (h->lms_graph) { cudaGraphExecDestroy(h->lms_graph); h->lms_graph = nullptr; }
    long long ng = nseg + (long long)d.E_sym / d.S;    // headroom over this round's grid
    if (ng > d.seg_cap / 2) ng = d.seg_cap / 2;
    if (ng < nseg) return false;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { cudaGetLastError(); return false; }
    const long long l0 = h->launches;
    launch_lms_round(h, s, labels, lab_cap, 0, ng);
    const int nk = (int)(h->launches - l0);
    h->launches = l0;
    if (cudaStreamEndCapture(s, &g) != cudaSuccess || !g) { cudaGetLastError(); return false; }
    const cudaError_t e = cudaGraphInstantiate(&h->lms_graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { cudaGetLastError(); h->lms_graph = nullptr; return false; }
    h->lms_graph_labels = labels;
    h->lms_graph_cap = lab_cap;
    h->lms_graph_nseg = ng;
    h->lms_graph_kernels = nk;
  }
  if (cudaGraphLaunch(h->lms_graph, s) != cudaSuccess) return false;
  h->launches += h->lms_graph_kernels;
  return true;
}

// Equaliser rounds. Streaming: one round per call once ~lms_batch_segments may be pending
// (a batch spans fewer than D epochs, so every lag-D seed it needs was finalised by an earlier
// round). Flush: rounds until every segment is final (each round can unlock the next D epochs;
// the end of stream is the one place the host synchronises).
static void launch_lms_rounds(rx_handle *h, cudaStream_t s, unsigned char *labels, long long lab_cap,
                              int flush, long long sym_ub) {
  RxDev &d = h->d;
  const long long S = d.S;
  const long long seg_ub = sym_ub / S + 1;
  if (!flush) {
    const long long est_ready = seg_ub - h->lms_launched_upto;
    if (h->cfg.lms_batch_segments > 0 && est_ready < h->cfg.lms_batch_segments) return;
    const long long prev_upto = h->lms_launched_upto;
    // grid: segments from the device's seg_next; pending ones are bounded by this batch plus
    // what could not run last time (data not yet normalised: at most one call of symbols)
    const long long call_segs = (h->max_call / h->sps) / S + 2;
    const long long tail = (long long)d.D * (d.E_sym / S);
    long long nseg = seg_ub - h->lms_launched_upto + call_segs + tail + 2;
    if (nseg > d.seg_cap / 2) nseg = d.seg_cap / 2;
    h->lms_launched_upto = seg_ub;
    // a round can finish at most D epochs in a row (each segment needs the seed of epoch
    // e - D): new segments beyond that need further rounds; a seed-blocked tail shorter than
    // a round rides along with the next batch (the rings hold one batch + D epochs)
    // Every round costs a full segment recursion however few segments it runs, so a short
    // remainder (e.g. the first segment of epoch e + D, whose seed this same round produces)
    // waits for the next batch; the host tracks an estimate of the finalised frontier and runs
    // a second round only when at least half a round more is pending. The backlog stays below
    // one batch + D epochs, which the rings hold (rx_create).
    (void)prev_upto;
    const long long per_round = (long long)d.D * (d.E_sym / S);
    if (h->lms_fin_est < seg_ub - 2 * per_round - call_segs) h->lms_fin_est = seg_ub - 2 * per_round - call_segs;
    const long long backlog = seg_ub - h->lms_fin_est;
    long long rounds = (backlog + per_round / 2) / per_round;
    if (rounds < 1) rounds = 1;
    for (long long r = 0; r < rounds; ++r)
      if (!lms_graph_round(h, s, labels, lab_cap, nseg)) launch_lms_round(h, s, labels, lab_cap, flush, nseg);
    h->lms_fin_est += rounds * per_round;
    if (h->lms_fin_est > seg_ub) h->lms_fin_est = seg_ub;
    return;
  }
  long long prev = -1;
  for (int it = 0; it < 4096; ++it) {
    DevState st;
    if (cudaStreamSynchronize(s) != cudaSuccess) return;
    if (cudaMemcpy(&st, h->st_dev, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    const long long total = st.m_end >= 0 ? (st.m_end + S - 1) / S : seg_ub;
    if (st.seg_next >= total || st.seg_next == prev) break;
    prev = st.seg_next;
    long long nseg = total - st.seg_next + 1;
    if (nseg > d.seg_cap / 2) nseg = d.seg_cap / 2;
    launch_lms_round(h, s, labels, lab_cap, flush, nseg);
  }
}

// H8: normalisation of every buffer whose symbols are complete (all of them at flush)
static void launch_norm_pam(rx_handle *h, cudaStream_t s, int flush) {
  RxDev &d = h->d;
  const long long BB = d.buffer_blocks;
  long long nbuf = 0;
  while ((h->norm_done + nbuf + 1) * BB <= h->be_done || (flush && (h->norm_done + nbuf) * BB < h->be_done)) ++nbuf;
  if (nbuf == 0) return;
  const long long beta0 = h->norm_done;
  const long long bend = h->be_done;
  for (long long b0 = 0; b0 < nbuf; b0 += 16) {
    const long long nb = nbuf - b0 < 16 ? nbuf - b0 : 16;
    KLAUNCH(h, RX_K_NORM, s, (k_norm_stats<<<dim3(NORM_G, (unsigned)nb), 1024, 0, s>>>(d, beta0 + b0, bend, flush)));
    KLAUNCH(h, RX_K_NORM, s, (k_norm_apply<<<dim3(NORM_AG, (unsigned)nb), 256, 0, s>>>(d, beta0 + b0, nb, bend, flush)));
  }
  h->norm_done += nbuf;
}

static void run_pam(rx_handle *h, cudaStream_t s, const InView &in, unsigned char *labels,
                    long long lab_cap, int flush) {
  RxDev &d = h->d;
  const long long fe_target = h->n_in / 512;
  if (fe_target > h->fe_done) {
    if (d.H_real) KLAUNCH(h, RX_K_PAM_FE, s, (k_pam_fe<true><<<gridc(fe_target - h->fe_done, FE_GROUPS), 256, 0, s>>>(d, in, h->fe_done, fe_target)));
    else KLAUNCH(h, RX_K_PAM_FE, s, (k_pam_fe<false><<<gridc(fe_target - h->fe_done, FE_GROUPS), 256, 0, s>>>(d, in, h->fe_done, fe_target)));
    h->fe_done = fe_target;
  }
  long long clk_target = flush ? h->fe_done : h->fe_done - d.clock_half;
  if (clk_target > h->clk_done) {
    const size_t smem = (CLK_TILE + 1 + 2 * d.clock_half) * sizeof(double2);
    const unsigned ntiles = gridc(clk_target - h->clk_done, CLK_TILE);
    if (ntiles <= g_clk_fuse_max && ntiles <= CLK_FUSE_MAX) {   // every tile co-resident: one pass + carry
      const long long id = ++h->clk_launch;
      KLAUNCH(h, RX_K_PAM_CLOCK, s, launch_pdl(k_pam_theta<true>, ntiles, CLK_TILE, smem, s, d, h->clk_done, clk_target, h->fe_done - 1, id));
    } else {
      KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_pam_theta<false><<<ntiles, CLK_TILE, smem, s>>>(d, h->clk_done, clk_target, h->fe_done - 1, 0)));
      KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_pam_carry<<<1, 1024, 0, s>>>(d, (int)ntiles)));
      KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_pam_tau<<<gridc(clk_target - h->clk_done, 256), 256, 0, s>>>(d, h->clk_done, clk_target)));
    }
    h->clk_done = clk_target;
  }
  long long be_target = flush ? h->fe_done - 1 : h->clk_done - 1;
  if (be_target > h->be_done) {
    if (d.H_real) KLAUNCH(h, RX_K_PAM_BE, s, launch_pdl(k_pam_be<true>, gridc(be_target - h->be_done, FE_GROUPS), 256, 0, s, d, h->be_done, be_target));
    else KLAUNCH(h, RX_K_PAM_BE, s, launch_pdl(k_pam_be<false>, gridc(be_target - h->be_done, FE_GROUPS), 256, 0, s, d, h->be_done, be_target));
    h->be_done = be_target;
  }
  // streaming: the buffer normalisation runs on the equaliser side stream at the start of the
  // next call (fork_equaliser), ahead of the equaliser that consumes it
  if (flush || h->cfg.serial_equaliser) launch_norm_pam(h, s, flush);
  if (flush) KLAUNCH(h, RX_K_MISC, s, (k_pam_mend<<<1, 1, 0, s>>>(d, h->be_done > 0 ? h->be_done : 0)));
  h->lms_sym_ub = 256 * h->be_done + h->be_done / 4 + 4096;
  if (flush) {
    KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
    launch_sync_train<false>(h, s, flush);
    launch_lms_rounds(h, s, labels, lab_cap, flush, h->lms_sym_ub);
  }
}

// KK: the deferred CFO carries, in buffer order (the DDS origin is a chain)
static void launch_zp_pending(rx_handle *h, cudaStream_t s) {
  RxDev &d = h->d;
  const int fine_ctas = (int)((h->Q / 1024 + 7) / 8);
  // contiguous deferred groups run as one launch set (up to cfo_maxbuf buffers): with one-buffer
  // calls the estimate of several buffers then shares one wave instead of a latency-bound launch
  // chain per buffer (results do not depend on the grouping: fixed spectrum rows per buffer, the
  // DDS carry runs over the buffers in order)
  size_t i = 0;
  const size_t n = h->zp_pending.size();
  while (i < n) {
    rx_handle::ZpJob j = h->zp_pending[i];
    size_t k = i + 1;
    while (k < n && h->zp_pending[k].est == j.est && h->zp_pending[k].beta0 == j.beta0 + j.nb &&
           j.nb + h->zp_pending[k].nb <= h->cfo_maxbuf) {
      j.nb += h->zp_pending[k].nb;
      j.q_front = h->zp_pending[k].q_front;
      ++k;
    }
    if (j.est) {   // plain launches: the producer (stage 2) is on the other stream (event order)
      KLAUNCH(h, RX_K_CFO, s, (k_cfo_spec<<<dim3(CFO_ROWS, (unsigned)j.nb), CFO_SPEC_T, CFO_STAGE_SMEM, s>>>(d, j.beta0, j.q_front)));
      if (d.cfo_enable) KLAUNCH(h, RX_K_CFO, s, (k_cfo_fine<<<dim3((unsigned)fine_ctas, (unsigned)j.nb), 256, 0, s>>>(d, j.beta0, j.q_front, fine_ctas)));
    }
    KLAUNCH(h, RX_K_CFO, s, (k_cfo_carry<<<1, 1, 0, s>>>(d, j.beta0, (int)j.nb, j.q_front)));
    i = k;
  }
  h->zp_pending.clear();
}

// Deferred KK CFO groups wait (streaming, after training) until CFO_DEFER_BUFS buffers are pending
// or an equaliser round is due - the only consumer of z' then (formed from the CFO parameters)
static bool zp_due(const rx_handle *h) {
  if (h->zp_pending.empty()) return false;
  if (!h->hm_host->trained) return true;       // sync / training read z' of the first buffers
  long long nb = 0;
  for (const auto &j : h->zp_pending) nb += j.nb;
  if (nb >= CFO_DEFER_BUFS) return true;
  const long long batch = h->cfg.lms_batch_segments;
  const long long seg_ub = h->lms_sym_ub / h->d.S + 1;
  return batch <= 0 || seg_ub - h->lms_launched_upto >= batch;   // the test of launch_lms_rounds
}

static void run_kk(rx_handle *h, cudaStream_t s, const InView &in, unsigned char *labels,
                   long long lab_cap, int flush) {
  RxDev &d = h->d;
  if (flush) launch_zp_pending(h, s);
  const long long s1_target = h->n_in / 512;
  if (h->cfg.fused_front_end && s1_target > h->fe_done) {
    // one kernel for both stages over the stage-2 blocks [s2_done, s1_target - 1) (stage 1 of
    // [fe_done, s1_target) counted). per_cta = 4 n - 2 stage-2 blocks per CTA (n iterations of
    // FE_GROUPS stage-1 blocks, 2 of them halos), n from the smallest per-CTA share that keeps the
    // grid within the resident CTA slots, or g_fe_per_cta (experiments)
    const long long x0 = h->s2_done, x1 = s1_target - 1;
    if (x1 > x0) {
      const long long L = x1 - x0;
      long long per = g_fe_per_cta;
      if (per <= 0) {
        const long long share = (L + h->fe_slots - 1) / h->fe_slots;
        per = FE_GROUPS * ((share + 2 + FE_GROUPS - 1) / FE_GROUPS) - 2;
      }
      KLAUNCH(h, RX_K_KK_FE, s, (k_kk_fe<<<gridc(L, (int)per), 256, KKFE_SMEM, s>>>(d, in, h->fe_done, x0, x1, (int)per)));
      h->s2_done = x1;
      h->fe_done = s1_target;   // (else: nothing computed or counted yet)
    }
  }
  if (!h->cfg.fused_front_end && s1_target > h->fe_done) {
    KLAUNCH(h, RX_K_KK_S1, s, (k_kk_s1<<<gridc(s1_target - h->fe_done, FE_GROUPS), 256, 0, s>>>(d, in, h->fe_done, s1_target)));
    h->fe_done = s1_target;
  }
  const long long s2_target = h->fe_done - 1;
  if (s2_target > h->s2_done) {
    KLAUNCH(h, RX_K_KK_S2, s, launch_pdl(k_kk_s2, gridc(s2_target - h->s2_done, FE_GROUPS), 256, 0, s, d, h->s2_done, s2_target));
    h->s2_done = s2_target;
  }
  const long long q_front = h->s2_done > 0 ? 256 * h->s2_done - 128 : 0;
  const long long Q = h->Q;
  {
    long long nbuf = 0;
    while ((h->cfo_done + nbuf + 1) * Q <= q_front || (flush && (h->cfo_done + nbuf) * Q < q_front)) ++nbuf;
    if (nbuf > 0) {
      const long long beta0 = h->cfo_done;
      const int fine_ctas = (int)((Q / 1024 + 7) / 8);
      for (long long b0 = 0; b0 < nbuf; b0 += h->cfg.history_buffers) {
        const long long nb = nbuf - b0 < h->cfg.history_buffers ? nbuf - b0 : h->cfg.history_buffers;
        if (flush || h->cfg.serial_equaliser) {
          KLAUNCH(h, RX_K_CFO, s, launch_pdl(k_cfo_spec, dim3(CFO_ROWS, (unsigned)nb), CFO_SPEC_T, CFO_STAGE_SMEM, s, d, beta0 + b0, q_front));
          if (d.cfo_enable) KLAUNCH(h, RX_K_CFO, s, launch_pdl(k_cfo_fine, dim3((unsigned)fine_ctas, (unsigned)nb), 256, 0, s, d, beta0 + b0, q_front, fine_ctas));
          KLAUNCH(h, RX_K_CFO, s, (k_cfo_carry<<<1, 1, 0, s>>>(d, beta0 + b0, (int)nb, q_front)));
        } else {
          // the CFO estimate and the DDS carry only feed the equaliser (z' where it is read):
          // they run at the next call on the side stream, concurrently with that call's
          // front-end (the paper overlaps consecutive buffers across streams)
          h->zp_pending.push_back({beta0 + b0, nb, q_front, 1});
        }
      }
      h->cfo_done += nbuf;
    }
  }
  h->lms_sym_ub = q_front / 2 + 1;
  if (flush) {   // m_end needs the sync phase: sync, then the end marker, then the rounds
    KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
    launch_sync_train<true>(h, s, flush);
    KLAUNCH(h, RX_K_MISC, s, (k_kk_mend<<<1, 1, 0, s>>>(d, q_front)));
    KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
    launch_lms_rounds(h, s, labels, lab_cap, flush, h->lms_sym_ub);
  }
}

// Streaming call: the equaliser stage (sync, training, LMS rounds and their post-processing)
// works on what earlier calls normalised (v_lms = v_front at the start of this call), on the
// side stream, while this call's front-end ... normalisation run on the caller's stream. Results
// do not depend on it (the equaliser output is independent of how its rounds are batched).
static void fork_equaliser(rx_handle *h, cudaStream_t s, unsigned char *labels, long long lab_cap) {
  RxDev &d = h->d;
  // The stages that only feed the equaliser move to the side stream too, ahead of the snapshot:
  // PAM: the normalisation of the earlier calls' buffers; KK: their CFO carry and z'.
  cudaEventRecord(h->ev_fork, s);
  cudaStreamWaitEvent(h->side, h->ev_fork, 0);
  if (d.family == RX_PAM) launch_norm_pam(h, h->side, 0);
  else if (zp_due(h)) launch_zp_pending(h, h->side);
  KLAUNCH(h, RX_K_MISC, h->side, (k_lms_snapshot<<<1, 1, 0, h->side>>>(d)));
  if (d.family == RX_PAM) launch_sync_train<false>(h, h->side, 0);
  else launch_sync_train<true>(h, h->side, 0);
  launch_lms_rounds(h, h->side, labels, lab_cap, 0, h->lms_sym_ub);
  cudaEventRecord(h->ev_join[h->ncall % (RX_MAX_LAG + 1)], h->side);
}

// Make `s` wait for every equaliser stage forked so far (the calls that read or report results).
static void join_side(rx_handle *h, cudaStream_t s) {
  if (h->ncall > 0) cudaStreamWaitEvent(s, h->ev_join[(h->ncall - 1) % (RX_MAX_LAG + 1)], 0);
}

static InView make_view(const rx_handle *h, const void *samples, long long n) {
  InView in;
  const bool f32 = h->cfg.input_format == RX_IN_F32;
  in.cur = f32 ? nullptr : (const uint16_t *)samples;
  in.curf = f32 ? (const float *)samples : nullptr;
  in.call_start = h->n_in;
  in.call_end = h->n_in + n;
  in.hist = h->d.hist;
  in.histf = h->d.histf;
  in.hist_cap = h->hist_cap;
  in.hist_w = h->d.hist;
  in.histf_w = h->d.histf;
  in.keep_from = n > 0 ? h->n_in + n - (1 << 16) : h->n_in;
  in.f32 = f32;
  in.gain = (float)h->cfg.adc_gain;
  in.cnt_lo = 0;
  in.cnt_hi = 0x7fffffffffffffffLL;
  return in;
}

extern "C" rx_status rx_process(rx_handle *h, const void *d_samples, long long n,
                                unsigned char *d_labels, long long labels_capacity, void *stream) {
  if (!h || n < 0 || (n > 0 && !d_samples) || n % 512 || labels_capacity < 0) return RX_EINVAL;
  if (n > h->max_call) return RX_EINVAL;
  if (labels_capacity > 0 && !d_labels) return RX_EINVAL;
  if (((uintptr_t)d_samples) & 15) return RX_EINVAL;
  if (h->flushed || h->d.shard_n > 1) return RX_ESTATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  std::pair<cudaEvent_t, cudaEvent_t> rt_ev(nullptr, nullptr);
  if (h->rt_on) {   // real-time monitor: the call's span on the caller's stream
    if (!h->rt_free.empty()) { rt_ev = h->rt_free.back(); h->rt_free.pop_back(); }
    else { CK(cudaEventCreate(&rt_ev.first)); CK(cudaEventCreate(&rt_ev.second)); }
    CK(cudaEventRecord(rt_ev.first, s));
  }
  if (h->cfg.input_format == RX_IN_U12_PACKED && n > 0) {   // unpack the call into the staging buffer
    KLAUNCH(h, RX_K_MISC, s, (k_unpack12<<<gridc(n / 8, 256) < 4096 ? gridc(n / 8, 256) : 4096, 256, 0, s>>>(
                                 (const uint32_t *)d_samples, (uint4 *)h->unpacked, n / 8)));
    d_samples = h->unpacked;
  }
  const InView in = make_view(h, d_samples, n);
  h->n_in += n;
  unsigned char *lab = labels_capacity ? d_labels : nullptr;
  const long long cap = labels_capacity ? labels_capacity : 1;
  const bool serial = h->cfg.serial_equaliser != 0;
  if (!serial) fork_equaliser(h, s, lab, cap);
  if (h->d.family == RX_PAM) run_pam(h, s, in, lab, cap, 0);
  else run_kk(h, s, in, lab, cap, 0);
  if (serial) {   // same stages, in order on the caller's stream, on everything normalised so far
    KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(h->d)));
    if (h->d.family == RX_PAM) launch_sync_train<false>(h, s, 0);
    else launch_sync_train<true>(h, s, 0);
    launch_lms_rounds(h, s, lab, cap, 0, h->lms_sym_ub);
  } else {
    // equaliser_lag = L: the call ends when the equaliser stage forked L calls earlier has (L = 0:
    // its own; L >= 1: this call's stage overlaps the next L calls' front-ends, as the paper's
    // buffers overlap across its five streams, P:146 - with small calls a round, which runs once
    // per lms_batch_segments, needs several calls of front-end to hide behind)
    const long long L = h->cfg.equaliser_lag;
    if (h->ncall >= L) CK(cudaStreamWaitEvent(s, h->ev_join[(h->ncall - L) % (RX_MAX_LAG + 1)], 0));
    h->ncall++;
  }
  if (rt_ev.first) {
    CK(cudaEventRecord(rt_ev.second, s));
    h->rt_pending.push_back({rt_ev.first, rt_ev.second, n});
  }
  return check_launch();
}

// ------------------------------------------------------------------ time sharding (mode 2)
// Stage A of buffer `beta` on its owning shard. The input covers [max(0, beta B - pre),
// (beta + 1) B + post) (rx_shard_halo; shorter at the stream end: last = 1).
//  KK: stage 1 / 2 over every block whose overlap-save frames lie inside it, then the CFO
//      estimate of the buffer.
//  PAM: front-end (spectra, C_b) of the buffer's blocks, its back-end look-back blocks and their
//      clock windows; the clock phases theta_b and their wrap counts relative to block beta B - 1
//      (the global count arrives with the records: rx_import_carry).
extern "C" rx_status rx_shard_process(rx_handle *h, long long beta, const void *d_samples, long long n, int last,
                                      unsigned char *d_labels, long long labels_capacity, void *stream) {
  if (!h || h->d.shard_n <= 1 || beta < 0 || n <= 0 || !d_samples || labels_capacity < 0 ||
      (labels_capacity > 0 && !d_labels))
    return RX_EINVAL;
  RxDev &d = h->d;
  if (beta % d.shard_n != d.shard_g || h->sh_cur.valid || h->flushed) return RX_ESTATE;
  if (h->cfg.input_format != RX_IN_U12_IN_U16 || (((uintptr_t)d_samples) & 15)) return RX_EINVAL;
  const long long BB = d.buffer_blocks, B4 = BB * 512;
  const long long P0 = beta * B4 - h->sh_pre > 0 ? beta * B4 - h->sh_pre : 0;
  const long long P1 = P0 + n;
  if (n % 512 || P1 <= beta * B4 || (!last && P1 < (beta + 1) * B4 + h->sh_post) || n > B4 + h->sh_pre + h->sh_post)
    return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  InView in = make_view(h, d_samples, 0);
  in.cur = (const uint16_t *)d_samples;
  in.call_start = P0;
  in.call_end = P1;
  in.keep_from = 0x7fffffffffffffffLL;           // nothing goes to the history ring
  in.cnt_lo = beta * BB;                          // the halos are counted by their owners
  in.cnt_hi = (beta + 1) * BB;
  rx_handle::ShardBuf &sb = h->sh_cur;
  if (d.family == RX_QAM_KK) {
    const long long s1_lo = P0 == 0 ? 0 : P0 / 512 + 1, s1_hi = P1 / 512;   // frames inside [P0, P1)
    const long long s2_lo = P0 == 0 ? 0 : s1_lo + 1, s2_hi = s1_hi - 1;
    KLAUNCH(h, RX_K_KK_S1, s, (k_kk_s1<<<gridc(s1_hi - s1_lo, FE_GROUPS), 256, 0, s>>>(d, in, s1_lo, s1_hi)));
    KLAUNCH(h, RX_K_KK_S2, s, (k_kk_s2<<<gridc(s2_hi - s2_lo, FE_GROUPS), 256, 0, s>>>(d, s2_lo, s2_hi)));
    const long long q_front = 256 * s2_hi - 128;
    const int fine_ctas = (int)((h->Q / 1024 + 7) / 8);
    KLAUNCH(h, RX_K_CFO, s, (k_cfo_spec<<<dim3(CFO_ROWS, 1), CFO_SPEC_T, CFO_STAGE_SMEM, s>>>(d, beta, q_front)));
    if (d.cfo_enable) KLAUNCH(h, RX_K_CFO, s, (k_cfo_fine<<<dim3((unsigned)fine_ctas, 1), 256, 0, s>>>(d, beta, q_front, fine_ctas)));
    sb.qfront = q_front;
  } else {
    // blocks: front-end [f_lo, f_hi) (block b's frame is samples [512 (b - 1), 512 (b + 1))),
    // clock [c_lo, c_hi) (windows of +-h blocks inside the front-end's), back-end [be_lo, be_hi)
    const long long hh = d.clock_half, pb = h->sh_pb;
    const long long f_lo = beta * BB - pb - 1 - hh > 0 ? beta * BB - pb - 1 - hh : 0;
    const long long f_hi = last ? P1 / 512 : (beta + 1) * BB + 2 + hh;
    sb.c_lo = beta * BB - pb > 0 ? beta * BB - pb : 0;
    sb.c_hi = last ? f_hi : (beta + 1) * BB + 1;
    sb.be_lo = sb.c_lo;
    sb.be_hi = last ? f_hi - 1 : (beta + 1) * BB;
    if (d.H_real) KLAUNCH(h, RX_K_PAM_FE, s, (k_pam_fe<true><<<gridc(f_hi - f_lo, FE_GROUPS), 256, 0, s>>>(d, in, f_lo, f_hi)));
    else KLAUNCH(h, RX_K_PAM_FE, s, (k_pam_fe<false><<<gridc(f_hi - f_lo, FE_GROUPS), 256, 0, s>>>(d, in, f_lo, f_hi)));
    // clock pass with a zero carry: N_loc (the first block's own count cancels out of every
    // difference N_loc(b) - N_loc(beta B - 1))
    const size_t smem = (CLK_TILE + 1 + 2 * d.clock_half) * sizeof(double2);
    const unsigned ntiles = gridc(sb.c_hi - sb.c_lo, CLK_TILE);
    KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_shard_clk_reset<<<1, 1, 0, s>>>(d)));
    KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_pam_theta<false><<<ntiles, CLK_TILE, smem, s>>>(d, sb.c_lo, sb.c_hi, f_hi - 1, 0)));
    KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_pam_carry<<<1, 1024, 0, s>>>(d, (int)ntiles)));
    const long long own_hi = (beta + 1) * BB < sb.c_hi ? (beta + 1) * BB : sb.c_hi;
    KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_shard_wraps<<<1, 1, 0, s>>>(d, beta, sb.c_lo, own_hi)));
  }
  sb.beta = beta;
  sb.last = last;
  sb.valid = 1;
  sb.exported = 0;
  sb.labels = labels_capacity ? d_labels : nullptr;
  sb.cap = labels_capacity ? labels_capacity : 1;
  h->n_in += P1 < (beta + 1) * B4 ? P1 - beta * B4 : B4;
  return check_launch();
}

extern "C" rx_status rx_shard_halo(const rx_handle *h, long long *pre, long long *post) {
  if (!h || !pre || !post) return RX_EINVAL;
  *pre = h->sh_pre;
  *post = h->sh_post;
  return RX_OK;
}

extern "C" rx_status rx_carry_size(const rx_handle *h, int *bytes) {
  if (!h || !bytes) return RX_EINVAL;
  *bytes = (int)sizeof(RxCarry);
  return RX_OK;
}

// This round's record (RxCarry, rx_carry_size bytes) into device memory d_buf, stream-ordered.
extern "C" rx_status rx_export_carry(rx_handle *h, void *d_buf, void *stream) {
  if (!h || !d_buf || h->d.shard_n <= 1 || (((uintptr_t)d_buf) & 15)) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const long long beta = (h->sh_cur.valid && !h->sh_cur.exported) ? h->sh_cur.beta : -1;
  KLAUNCH(h, RX_K_MISC, s, (k_carry_export<<<1, 1, 0, s>>>(h->d, (RxCarry *)d_buf, beta, h->sh_norm_beta)));
  if (h->sh_cur.valid) h->sh_cur.exported = 1;
  h->sh_norm_beta = -1;
  return check_launch();
}

// KK stage B of one buffer (the equaliser of its epoch): z' valid below the buffer's front, the
// finalisation front at the epoch's first segment, one round over the epoch's segments
static void shard_stage_b(rx_handle *h, cudaStream_t s, const rx_handle::ShardBuf &b) {
  RxDev &d = h->d;
  const long long spe = d.E_sym / d.S;
  KLAUNCH(h, RX_K_MISC, s, (k_shard_seek<<<1, 1, 0, s>>>(d, b.qfront, b.beta * spe)));
  if (b.last) KLAUNCH(h, RX_K_MISC, s, (k_kk_mend<<<1, 1, 0, s>>>(d, b.qfront)));   // stream end: m_end
  KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
  launch_lms_round(h, s, b.labels, b.cap, b.last ? 1 : 0, spe);
}

// PAM stage B of one buffer (one round after its stage A2: the previous buffer's normalisation
// scalars have arrived): its look-back symbols normalised with them, then one equaliser round
// over the segments whose last tap position lies in the buffer's symbols
static void shard_stage_b_pam(rx_handle *h, cudaStream_t s, const rx_handle::ShardBuf &b) {
  RxDev &d = h->d;
  KLAUNCH(h, RX_K_NORM, s, (k_shard_halo_norm<<<8, 256, 0, s>>>(d, b.beta)));
  KLAUNCH(h, RX_K_MISC, s, (k_shard_seek_pam<<<1, 1, 0, s>>>(d, b.beta)));
  KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
  launch_lms_round(h, s, b.labels, b.cap, b.last ? 1 : 0, d.E_sym / d.S + 4);
}

// PAM stage A2 of one buffer (after the exchange that gave its global wrap base): tau_b / M_b,
// the back-end (symbols u), the buffer's normalisation; frame sync + training at the stream start
static void shard_stage_a2_pam(rx_handle *h, cudaStream_t s, const rx_handle::ShardBuf &b) {
  RxDev &d = h->d;
  KLAUNCH(h, RX_K_PAM_CLOCK, s, (k_shard_tau<<<gridc(b.c_hi - b.c_lo, 256), 256, 0, s>>>(d, b.c_lo, b.c_hi)));
  if (d.H_real) KLAUNCH(h, RX_K_PAM_BE, s, (k_pam_be<true><<<gridc(b.be_hi - b.be_lo, FE_GROUPS), 256, 0, s>>>(d, b.be_lo, b.be_hi)));
  else KLAUNCH(h, RX_K_PAM_BE, s, (k_pam_be<false><<<gridc(b.be_hi - b.be_lo, FE_GROUPS), 256, 0, s>>>(d, b.be_lo, b.be_hi)));
  KLAUNCH(h, RX_K_NORM, s, (k_norm_stats<<<dim3(NORM_G, 1), 1024, 0, s>>>(d, b.beta, b.be_hi, b.last)));
  KLAUNCH(h, RX_K_NORM, s, (k_norm_apply<<<dim3(NORM_AG, 1), 256, 0, s>>>(d, b.beta, 1, b.be_hi, b.last)));
  KLAUNCH(h, RX_K_MISC, s, (k_shard_bufm<<<1, 1, 0, s>>>(d, b.beta, b.be_lo, b.be_hi)));
  if (b.beta == 0) {                 // the stream start: frame sync + training (c-10, c-9)
    KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
    launch_sync_train<false>(h, s, b.last);
  }
  h->sh_norm_beta = b.beta;
}

// The gathered records of all n_ranks shards (rank order). KK: CFO origin chain, sync /
// training, seeds; then stage B of this shard's previous buffer (and, on the shard holding the
// stream start, frame sync + training on buffer 0 as soon as its CFO estimate is known).
// PAM: wrap base, normalisation scalars, sync / training, seeds; stage B of the previous
// buffer, then stage A2 of this round's. A call with nothing new (every rank's buffers done)
// drains the last stage B.
extern "C" rx_status rx_import_carry(rx_handle *h, const void *d_gathered, int n_ranks, int my_rank, void *stream) {
  if (!h || !d_gathered || h->d.shard_n <= 1 || n_ranks != h->d.shard_n || my_rank != h->d.shard_g) return RX_EINVAL;
  if (h->flushed) return RX_ESTATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  RxDev &d = h->d;
  const RxCarry *g = (const RxCarry *)d_gathered;
  const long long my_beta = h->sh_cur.valid ? h->sh_cur.beta : -1;
  KLAUNCH(h, RX_K_MISC, s, (k_carry_import<<<1, 32, 0, s>>>(d, g, n_ranks, my_rank, my_beta)));
  if (d.family == RX_PAM) {
    if (h->sh_pend.valid) {
      shard_stage_b_pam(h, s, h->sh_pend);
      h->sh_pend.valid = 0;
    }
    if (h->sh_cur.valid) {
      shard_stage_a2_pam(h, s, h->sh_cur);
      h->sh_pend = h->sh_cur;
      h->sh_cur.valid = 0;
    }
    return check_launch();
  }
  KLAUNCH(h, RX_K_CFO, s, (k_carry_chain<<<1, 1, 0, s>>>(d, g, n_ranks)));
  if (h->sh_pend.valid) {
    shard_stage_b(h, s, h->sh_pend);
    h->sh_pend.valid = 0;
  }
  if (h->sh_cur.valid) {
    if (h->sh_cur.beta == 0) {       // the stream start: frame sync + training (c-10, c-9)
      KLAUNCH(h, RX_K_MISC, s, (k_shard_seek<<<1, 1, 0, s>>>(d, h->sh_cur.qfront, 0)));
      KLAUNCH(h, RX_K_MISC, s, (k_lms_snapshot<<<1, 1, 0, s>>>(d)));
      launch_sync_train<true>(h, s, h->sh_cur.last);
    }
    h->sh_pend = h->sh_cur;
    h->sh_cur.valid = 0;
    if (h->sh_pend.last) {           // nothing follows the stream end: finish it now
      shard_stage_b(h, s, h->sh_pend);
      h->sh_pend.valid = 0;
    }
  }
  return check_launch();
}

extern "C" rx_status rx_flush(rx_handle *h, unsigned char *d_labels, long long labels_capacity, void *stream) {
  if (!h || labels_capacity < 0 || (labels_capacity > 0 && !d_labels)) return RX_EINVAL;
  if (h->flushed || h->d.shard_n > 1) return RX_ESTATE;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  join_side(h, s);
  const InView in = make_view(h, nullptr, 0);
  if (h->d.family == RX_PAM) run_pam(h, s, in, labels_capacity ? d_labels : nullptr, labels_capacity ? labels_capacity : 1, 1);
  else run_kk(h, s, in, labels_capacity ? d_labels : nullptr, labels_capacity ? labels_capacity : 1, 1);
  h->flushed = true;
  return check_launch();
}

extern "C" rx_status rx_get_stats(rx_handle *h, rx_stats *o, void *stream) {
  if (!h || !o) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  join_side(h, (cudaStream_t)stream);
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  DevState st;
  CK(cudaMemcpy(&st, h->st_dev, sizeof(st), cudaMemcpyDeviceToHost));
  memset(o, 0, sizeof(*o));
  o->samples_in = h->n_in;
  o->symbols_out = st.symbols_out;
  o->bit_errors = st.bit_errors;
  o->bits = st.bits;
  o->symbols_counted = st.symbols_counted;
  o->clipped = st.clipped;
  o->domain_errors = st.domain_errors;
  o->first_domain_error_index = st.domain_errors ? st.first_domain : -1;
  o->evm_num = st.evm_num;
  o->evm_den = st.evm_den;
  o->sync_offset = st.sync_offset;
  o->sync_phase = st.sync_phase;
  o->sync_polarity = st.sync_polarity;
  o->synced = st.synced;
  o->sync_gamma = st.sync_gamma;
  o->sync_phi0 = st.sync_phi0;
  o->status_flags = st.flags | (st.domain_errors ? RX_FLAG_DOMAIN : 0);
  o->launches = h->launches;
  return RX_OK;
}

extern "C" rx_status rx_reset_stats(rx_handle *h, void *stream) {
  if (!h) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  KLAUNCH(h, RX_K_MISC, (cudaStream_t)stream, (k_reset_counters<<<1, 1, 0, (cudaStream_t)stream>>>(h->st_dev)));
  return check_launch();
}

extern "C" rx_status rx_get_taps(rx_handle *h, double *out, int capacity) {
  if (!h || !out) return RX_EINVAL;
  const bool kk = h->d.family == RX_QAM_KK;
  const int need = kk ? 2 * h->d.K : h->d.K;
  if (capacity < need) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  float2 w[RX_MAX_K];
  CK(cudaMemcpy(w, h->d.w_train, sizeof(float2) * h->d.K, cudaMemcpyDeviceToHost));
  for (int k = 0; k < h->d.K; ++k) {
    if (kk) { out[2 * k] = w[k].x; out[2 * k + 1] = w[k].y; }
    else out[k] = w[k].x;
  }
  if (h->d.wl && capacity >= 2 * need) {   // widely linear: V_train follows W_train
    CK(cudaMemcpy(w, h->d.v_train, sizeof(float2) * h->d.K, cudaMemcpyDeviceToHost));
    for (int k = 0; k < h->d.K; ++k) { out[need + 2 * k] = w[k].x; out[need + 2 * k + 1] = w[k].y; }
  }
  return RX_OK;
}

extern "C" rx_status rx_set_taps(rx_handle *h, const double *in, int n) {
  if (!h || !in) return RX_EINVAL;
  const bool kk = h->d.family == RX_QAM_KK;
  if (n != (kk ? 2 * h->d.K : h->d.K)) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  DevState st;
  CK(cudaMemcpy(&st, h->st_dev, sizeof(st), cudaMemcpyDeviceToHost));
  if (st.trained) return RX_ESTATE;
  float2 w[RX_MAX_K];
  for (int k = 0; k < h->d.K; ++k) w[k] = kk ? make_float2((float)in[2 * k], (float)in[2 * k + 1]) : make_float2((float)in[k], 0.f);
  CK(cudaMemcpy(h->d.w_init, w, sizeof(float2) * h->d.K, cudaMemcpyHostToDevice));
  h->d.has_winit = 1;
  return RX_OK;
}

// copy [first, first+count) of a ring with capacity cap (elements of size es) to host
static rx_status ring_read(const void *ring, long long cap, size_t es, long long first, long long count, void *out) {
  if (first < 0 || count < 0 || count > cap) return RX_EINVAL;
  const char *r = (const char *)ring;
  char *o = (char *)out;
  long long done = 0;
  while (done < count) {
    const long long i = (first + done) & (cap - 1);
    long long chunk = cap - i;
    if (chunk > count - done) chunk = count - done;
    if (cudaMemcpy(o + done * es, r + i * es, (size_t)chunk * es, cudaMemcpyDeviceToHost) != cudaSuccess) return RX_ECUDA;
    done += chunk;
  }
  return RX_OK;
}

extern "C" rx_status rx_probe_read(rx_handle *h, int which, long long first, long long count, void *out,
                                   void *stream) {
  if (!h || !out) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  join_side(h, (cudaStream_t)stream);
  // deferred KK CFO groups (zp_due) run now, in buffer order after every forked stage, so the
  // CFO / z' probes see every completed buffer
  if (!h->zp_pending.empty()) launch_zp_pending(h, (cudaStream_t)stream);
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  RxDev &d = h->d;
  const bool kk = d.family == RX_QAM_KK;
  switch (which) {
    case RX_PROBE_C: if (kk) return RX_EINVAL; return ring_read(d.C, d.blk_cap, sizeof(double2), first, count, out);
    case RX_PROBE_TAU: if (kk) return RX_EINVAL; return ring_read(d.tau, d.blk_cap, sizeof(double), first, count, out);
    case RX_PROBE_MB: if (kk) return RX_EINVAL; return ring_read(d.Mb, d.blk_cap, sizeof(long long), first, count, out);
    case RX_PROBE_U: if (kk) return RX_EINVAL; return ring_read(d.u, d.sym_cap, sizeof(float), first, count, out);
    case RX_PROBE_UHAT: if (kk) return RX_EINVAL; return ring_read(d.uhat, d.sym_cap, sizeof(float), first, count, out);
    case RX_PROBE_E: if (!kk || !d.E) return RX_EINVAL; return ring_read(d.E, d.E_cap, sizeof(float2), first, count, out);
    case RX_PROBE_Z: if (!kk) return RX_EINVAL; return ring_read(d.z, d.z_cap, sizeof(float2), first, count, out);
    case RX_PROBE_CFO: {
      if (!kk) return RX_EINVAL;
      std::vector<CfoParam> cp((size_t)count);
      rx_status st = ring_read(d.cfo, d.buf_cap, sizeof(CfoParam), first, count, cp.data());
      if (st) return st;
      double *o = (double *)out;
      for (long long i = 0; i < count; ++i) {
        o[5 * i] = cp[i].P; o[5 * i + 1] = cp[i].df; o[5 * i + 2] = cp[i].kstar;
        o[5 * i + 3] = (double)cp[i].inc; o[5 * i + 4] = (double)cp[i].origin;
      }
      return RX_OK;
    }
    case RX_PROBE_Y: return ring_read(d.yout, d.sym_cap, sizeof(float2), first, count, out);
    case RX_PROBE_LEVEL: return ring_read(d.level_fin, d.sym_cap, 1, first, count, out);
    case RX_PROBE_SEG: {
      std::vector<int> R(count), r(count);
      std::vector<float> th(count);
      std::vector<double> evm(2 * count);
      std::vector<long long> err(2 * count);
      for (long long i = 0; i < count; ++i) {
        const long long si = (first + i) & (d.seg_cap - 1);
        CK(cudaMemcpy(&R[i], d.seg_R + si, sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&r[i], d.seg_r + si, sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&th[i], d.seg_theta + si, sizeof(float), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&evm[2 * i], d.seg_evm + 2 * si, 2 * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&err[2 * i], d.seg_err + 2 * si, 2 * sizeof(long long), cudaMemcpyDeviceToHost));
      }
      double *o = (double *)out;
      for (long long i = 0; i < count; ++i) {
        o[6 * i] = R[i]; o[6 * i + 1] = r[i]; o[6 * i + 2] = th[i];
        o[6 * i + 3] = (double)err[2 * i]; o[6 * i + 4] = evm[2 * i]; o[6 * i + 5] = evm[2 * i + 1];
      }
      return RX_OK;
    }
    case RX_PROBE_DEBUG: {
      DevState st;
      CK(cudaMemcpy(&st, h->st_dev, sizeof(st), cudaMemcpyDeviceToHost));
      long long v[16] = {h->n_in, h->fe_done, h->clk_done, h->be_done, h->norm_done, h->s2_done, h->cfo_done,
                         st.v_front, st.m_end, st.seg_next, st.fin_lo, st.fin_hi, st.synced, st.trained,
                         st.anchor_known, st.anchor_A};
      long long n = count < 16 ? count : 16;
      memcpy(out, v, (size_t)n * sizeof(long long));
      return RX_OK;
    }
    default: return RX_EINVAL;
  }
}

extern "C" rx_status rx_profile_enable(rx_handle *h, int mask) {
  if (!h || mask < 0 || mask >= (1 << RX_KCLASS_COUNT)) return RX_EINVAL;
  h->prof_mask = mask;
  return RX_OK;
}

extern "C" rx_status rx_profile_read(rx_handle *h, double *ms, long long *counts, int n) {
  if (!h || !ms || !counts || n < RX_KCLASS_COUNT) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  for (int i = 0; i < RX_KCLASS_COUNT; ++i) { ms[i] = 0.0; counts[i] = 0; }
  for (auto &e : h->prof_pending) {
    CK(cudaEventSynchronize(e.second.second));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e.second.first, e.second.second));
    ms[e.first] += t;
    counts[e.first] += 1;
    h->prof_free.push_back(e.second);
  }
  h->prof_pending.clear();
  return RX_OK;
}

extern "C" rx_status rx_calibrate_thresholds(rx_handle *h, long long first, long long count, double *thr,
                                             double *means, void *stream) {
  if (!h || !thr || first < 0 || count <= 0 || h->d.family != RX_PAM) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  join_side(h, s);
  CK(cudaStreamSynchronize(s));
  DevState st;
  CK(cudaMemcpy(&st, h->st_dev, sizeof(st), cudaMemcpyDeviceToHost));
  if (!st.synced) return RX_ESTATE;
  // finalised and still held by the symbol rings (with a one-call margin for the writers)
  const long long held_lo = st.symbols_out - h->d.sym_cap / 2;
  if (first + count > st.symbols_out || first < held_lo) return RX_EINVAL;
  KLAUNCH(h, RX_K_MISC, s, (k_calib_levels<<<CAL_G, 256, 0, s>>>(h->d, first, first + count)));
  if (check_launch() != RX_OK) return RX_ECUDA;
  std::vector<double> part((size_t)CAL_G * 16 * 2);
  CK(cudaMemcpyAsync(part.data(), h->d.cal_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int M = h->d.M;
  std::vector<double> mu(M);
  for (int i = 0; i < M; ++i) {
    double a = 0.0, b = 0.0;
    for (int g = 0; g < CAL_G; ++g) { a += part[(g * 16 + i) * 2]; b += part[(g * 16 + i) * 2 + 1]; }
    if (b <= 0.0) return RX_EINVAL;
    mu[i] = a / b;
  }
  for (int i = 0; i + 1 < M; ++i) thr[i] = 0.5 * (mu[i] + mu[i + 1]);
  if (means) for (int i = 0; i < M; ++i) means[i] = mu[i];
  return RX_OK;
}

extern "C" rx_status rx_calibrate_dc(const rx_config *cfg, int dev, const void *d_samples, long long n,
                                     const double *cands, int ncand, double *evm, int *best, void *stream) {
  if (!cfg || !cands || !evm || !best || ncand <= 0 || n <= 0 || n % 512 || !d_samples) return RX_EINVAL;
  if (cfg->family != RX_QAM_KK) return RX_EINVAL;
  const size_t es = cfg->input_format == RX_IN_F32 ? 4 : 2;   // bytes per sample (x 3/4 packed)
  int bi = -1;
  for (int i = 0; i < ncand; ++i) {
    rx_config c = *cfg;
    c.dc_offset = cands[i];
    rx_handle *h = nullptr;
    rx_status st = rx_create(&c, dev, &h);
    if (st) return st;
    for (long long off = 0; off < n && st == RX_OK; off += h->max_call) {
      const long long k = n - off < h->max_call ? n - off : h->max_call;
      const long long boff = cfg->input_format == RX_IN_U12_PACKED ? off / 2 * 3 : off * (long long)es;
      st = rx_process(h, (const char *)d_samples + boff, k, nullptr, 0, stream);
    }
    if (st == RX_OK) st = rx_flush(h, nullptr, 0, stream);
    rx_stats s;
    if (st == RX_OK) st = rx_get_stats(h, &s, stream);
    rx_destroy(h);
    if (st != RX_OK && st != RX_ESYNC && st != RX_EDOMAIN && st != RX_EDIVERGE) return st;
    const bool ok = st == RX_OK || st == RX_EDOMAIN || st == RX_EDIVERGE;
    evm[i] = (ok && s.synced && !(s.status_flags & RX_FLAG_SYNC) && s.evm_den > 0.0)
                 ? 10.0 * log10(s.evm_num / s.evm_den) : INFINITY;
    if (bi < 0 || evm[i] < evm[bi]) bi = i;
  }
  *best = bi;
  return RX_OK;
}

// modified Bessel function of the first kind, order 0 (series; Kaiser window)
static double bessel_i0(double x) {
  double s = 1.0, t = 1.0;
  for (int k = 1; k < 64; ++k) {
    t *= (x / (2.0 * k)) * (x / (2.0 * k));
    s += t;
    if (t < 1e-18 * s) break;
  }
  return s;
}

extern "C" rx_status rx_design_static_eq(const double *hc, const double *ht, double lambda, int L, int real_taps,
                                         double *out) {
  const int N = 1024;
  if (!hc || !ht || !out || L < 1 || L % 2 == 0 || L > N - 1 || !(lambda >= 0.0)) return RX_EINVAL;
  std::vector<double> er(N), ei(N);
  for (int k = 0; k < N; ++k) {   // per-bin regularised MMSE
    const double cr = hc[2 * k], ci = hc[2 * k + 1], tr = ht[2 * k], ti = ht[2 * k + 1];
    const double den = cr * cr + ci * ci + lambda;
    if (den <= 0.0) {
      if (tr == 0.0 && ti == 0.0) { er[k] = ei[k] = 0.0; continue; }
      return RX_EINVAL;
    }
    er[k] = (cr * tr + ci * ti) / den;   // conj(H_ch) H_t / den
    ei[k] = (cr * ti - ci * tr) / den;
  }
  const int c = (L - 1) / 2;
  const double beta = 6.0, i0b = bessel_i0(beta);
  for (int i = 0; i < L; ++i) {
    const int n = ((i - c) % N + N) % N;   // zero-phase: tap i is time index i - c
    double sr = 0.0, si = 0.0;
    for (int k = 0; k < N; ++k) {          // h[n] = (1/N) sum_k H[k] e^{+j 2 pi k n / N}
      const int ph = (int)(((long long)k * n) % N);
      const double a = 2.0 * M_PI * ph / N, ca = cos(a), sa = sin(a);
      sr += er[k] * ca - ei[k] * sa;
      si += er[k] * sa + ei[k] * ca;
    }
    const double r = L > 1 ? (2.0 * i) / (L - 1) - 1.0 : 0.0;
    const double w = bessel_i0(beta * sqrt(fmax(0.0, 1.0 - r * r))) / i0b;
    if (real_taps) out[i] = w * sr / N;
    else { out[2 * i] = w * sr / N; out[2 * i + 1] = w * si / N; }
  }
  return RX_OK;
}

extern "C" rx_status rx_get_q_trace(rx_handle *h, long long first, int n, long long *err, long long *bits,
                                    void *stream) {
  if (!h || n < 0 || (n > 0 && (!err || !bits)) || first < 0 || h->d.q_segs <= 0) return RX_EINVAL;
  if (n > RX_Q_WINDOWS) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  join_side(h, (cudaStream_t)stream);
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  DevState st;
  CK(cudaMemcpy(&st, h->st_dev, sizeof(st), cudaMemcpyDeviceToHost));
  // held: the window of the newest finalised segment (possibly still open) and the
  // RX_Q_WINDOWS - 1 before it (older slots have been reused)
  const long long newest = st.seg_next > 0 ? (st.seg_next - 1) / h->d.q_segs : -1;
  if (n > 0 && (first + n - 1 > newest || first < newest - RX_Q_WINDOWS + 1)) return RX_EINVAL;
  std::vector<unsigned long long> q(2 * (size_t)RX_Q_WINDOWS);
  CK(cudaMemcpy(q.data(), h->d.q_win, q.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) {
    const long long w = (first + i) & (RX_Q_WINDOWS - 1);
    err[i] = (long long)q[2 * w];
    bits[i] = (long long)q[2 * w + 1] * h->d.kbits;
  }
  return RX_OK;
}

extern "C" rx_status rx_export_counters(rx_handle *h, double *d_out, void *stream) {
  if (!h || !d_out) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  join_side(h, s);
  KLAUNCH(h, RX_K_MISC, s, (k_export_counters<<<1, 1, 0, s>>>(h->st_dev, d_out)));
  return check_launch();
}

// ------------------------------------------------------------------ real-time monitor (NEXT-2)
extern "C" rx_status rx_rt_enable(rx_handle *h, int on) {
  if (!h || (on != 0 && on != 1)) return RX_EINVAL;
  h->rt_on = on;
  return RX_OK;
}

// Per streaming call k: span d_k (ms) between its first and last operation on the caller's stream
// (CUDA events) against its real-time budget n_k / sample_rate; overrun when d_k exceeds it.
extern "C" rx_status rx_get_rt_stats(rx_handle *h, rx_rt_stats *o) {
  if (!h || !o) return RX_EINVAL;
  CK(cudaSetDevice(h->device));
  memset(o, 0, sizeof(*o));
  double busy = 0.0, budget = 0.0;
  for (auto &c : h->rt_pending) {
    CK(cudaEventSynchronize(c.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c.a, c.b));
    const double bud = (double)c.n / h->cfg.sample_rate * 1e3;
    o->calls += 1;
    o->samples += c.n;
    busy += ms;
    budget += bud;
    if (ms > o->max_call_ms) o->max_call_ms = ms;
    if (bud > 0.0 && ms / bud > o->max_load) o->max_load = ms / bud;
    if (ms > bud) o->overruns += 1;
    h->rt_free.push_back({c.a, c.b});
  }
  h->rt_pending.clear();
  o->busy_ms = busy;
  o->realtime_ratio = busy > 0.0 ? budget / busy : 0.0;
  return RX_OK;
}
