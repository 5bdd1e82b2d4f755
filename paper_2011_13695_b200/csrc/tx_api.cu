// tx_api.cu — GPU transmitter + channel simulator (C ABI in include/tx.h).
// Generates the ADC stream of the paper's PAM and KK-QAM set-ups
// on the device, block-wise and stream-ordered; tested against rxsynth (the host generator) and
// through the receiver (tests/test_tx.py). Build: compiled into librx.so with rx_api.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "rx.h"
#include "tx.h"
#include "fft.cuh"

#define TX_BLK 512                // output samples per overlap-save block
#define TX_PHASES 4096            // polyphase resampler phases
#define TX_NTAP 32                // resampler taps

struct TxDev {
  int kk, M, L, sps;
  const float2 *tw;               // FFT twiddles (fft.cuh layout)
  const float2 *H;                // DFT_1024 of the zero-phase shaping FIR
  const float2 *sym;              // level values of the 32767 PRBS symbols
  long long sym_off;
  double eps;                     // PAM clock offset
  float sigma, pn_sigma, A;
  float2 iq;
  unsigned long long inc_c, inc_cfo;   // DDS increments of -f_c and +cfo
  float mean, gain;               // ADC: (x - mean) * gain + 2047.5, gain = 2047.5 / full_scale
  unsigned seed_lo, seed_hi;
  float2 *s; long long s_cap;     // shaped data waveform ring (absolute sample index)
  double *pn_part, *pn_base, *pn_carry;
  const float *ptab;              // [TX_PHASES + 1][TX_NTAP] resampler kernels
};

// ------------------------------------------------------------------ Philox-4x32-10 + Box-Muller
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
// four standard normals of absolute sample p (counter = p, stream tag)
__device__ __forceinline__ float4 tx_normals(const TxDev &d, long long p, unsigned tag) {
  const uint4 r = philox4x32(make_uint4((unsigned)p, (unsigned)((unsigned long long)p >> 32), tag, 0u),
                             make_uint2(d.seed_lo, d.seed_hi));
  const float u1 = ((float)r.x + 1.0f) * 2.3283064365386963e-10f, u2 = (float)r.y * 2.3283064365386963e-10f;
  const float u3 = ((float)r.z + 1.0f) * 2.3283064365386963e-10f, u4 = (float)r.w * 2.3283064365386963e-10f;
  const float a = sqrtf(-2.0f * logf(u1)), b = sqrtf(-2.0f * logf(u3));
  float s1, c1, s2, c2;
  sincospif(2.0f * u2, &s1, &c1);
  sincospif(2.0f * u4, &s2, &c2);
  return make_float4(a * c1, a * s1, b * c2, b * s2);
}
// e^{+j 2 pi u / 2^64} of a 64-bit phase word (exact word, accurate sin/cos of the top 32 bits)
__device__ __forceinline__ float2 tx_dds(unsigned long long u) {
  float s, c;
  sincospif((float)(int)(u >> 32) * 4.656612873077393e-10f, &s, &c);
  return make_float2(c, s);
}

__device__ __forceinline__ float2 tx_symbol(const TxDev &d, long long n) {   // upsampled train
  if (n < 0 || n % d.sps) return make_float2(0.f, 0.f);
  const long long m = n / d.sps;
  return __ldg(d.sym + (d.sym_off + m) % RX_PREF);
}

// ------------------------------------------------------------------ shaping (overlap-save)
// One 64-thread group per 512-sample block c: frame [512c - 256, 512c + 768) of the upsampled
// symbol train (odd samples are zero for sps >= 2: one FFT-512 of the even samples gives the
// 1024-point spectrum, X[k] = X[k + 512] = Ev[k]), times H, then the 1024-point inverse as two
// IFFT-512s of the even / odd outputs; the central 512 samples are s_p, p in [512c, 512c + 512).
__global__ void __launch_bounds__(256) k_tx_shape(TxDev d, long long c0, long long c1) {
  __shared__ float2 tw[1024];
  __shared__ float2 buf[4][FFT_PAD_N];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = d.tw[i];
  __syncthreads();
  const long long c = c0 + (long long)blockIdx.x * 4 + g;
  const bool act = c < c1;
  const long long F0 = TX_BLK * c - 256;
  float2 ev[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) ev[r] = act ? tx_symbol(d, F0 + 2 * (j + 64 * r)) : make_float2(0.f, 0.f);
  fft512_regs<false>(buf[g], j, tw, ev);            // Ev[k], k = j + 64 r
  float2 ye[8], yo[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int k = j + 64 * r;
    const float2 a = cmul(ev[r], __ldg(d.H + k)), b = cmul(ev[r], __ldg(d.H + k + 512));
    ye[r] = cadd(a, b);                               // spectrum of x[2m]
    yo[r] = cmulc(csub(a, b), tw[k]);                 // of x[2m + 1]: (A - B) W^{-k}
  }
  fft512_regs<true>(buf[g], j, tw, ye);
  fft512_regs<true>(buf[g], j, tw, yo);
  if (act) {
#pragma unroll
    for (int r = 2; r < 6; ++r) {                     // local 2m, 2m + 1 in [256, 768)
      const long long p = F0 + 2 * (j + 64 * r);
      const float4 v = make_float4(ye[r].x * (1.f / 1024.f), ye[r].y * (1.f / 1024.f),
                                   yo[r].x * (1.f / 1024.f), yo[r].y * (1.f / 1024.f));
      *reinterpret_cast<float4 *>(d.s + (p & (d.s_cap - 1))) = v;
    }
  }
}

// ------------------------------------------------------------------ Wiener phase noise
// phi_p = sum_{i <= p} w_i, w_i = pn_sigma N(0,1) (normal 0 of sample i, tag 1): per-block sums
// (one warp per block, fixed order), an exclusive scan of the block sums with the carry of
// earlier calls, and the in-block prefix in k_tx_kk
__global__ void __launch_bounds__(256) k_tx_pn_sums(TxDev d, long long c0, long long c1) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long c = c0 + (long long)blockIdx.x * 8 + w;
  if (c >= c1) return;
  float acc = 0.f;
  for (int i = 0; i < TX_BLK / 32; ++i) acc += tx_normals(d, TX_BLK * c + 16 * lane + i, 1u).x;
  double s = (double)acc * d.pn_sigma;
  s = warp_sum_d(s);
  if (lane == 0) d.pn_part[c - c0] = s;
}
__global__ void k_tx_pn_scan(TxDev d, long long n) {
  double run = *d.pn_carry;
  for (long long i = 0; i < n; ++i) { d.pn_base[i] = run; run += d.pn_part[i]; }
  *d.pn_carry = run;
}

__device__ __forceinline__ unsigned short tx_quantise(const TxDev &d, float x) {
  const float q = rintf(fmaf(x - d.mean, d.gain, 2047.5f));
  return (unsigned short)fminf(fmaxf(q, 0.f), 4095.f);
}

// ------------------------------------------------------------------ KK field + PD + ADC
// Thread j of a block's group takes its 8 consecutive samples p = 512c + 8j .. + 7 (in-block
// phase-noise prefix: sequential over its 8, a scan over the 64 threads)
__global__ void __launch_bounds__(256) k_tx_kk(TxDev d, long long c0, long long c1, long long call_p0,
                                               unsigned short *out) {
  __shared__ float tsum[4][64];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  const long long c = c0 + (long long)blockIdx.x * 4 + g;
  const bool act = c < c1;
  const long long p0 = TX_BLK * c + 8 * j;
  float4 nz[8];
  float inc[8], loc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    nz[i] = act ? tx_normals(d, p0 + i, 1u) : make_float4(0.f, 0.f, 0.f, 0.f);
    inc[i] = nz[i].x * d.pn_sigma;
    loc += inc[i];
  }
  // exclusive prefix of the threads' sums within the block (fixed order: tsum over j)
  tsum[g][j] = loc;
  __syncthreads();
  float before = 0.f;
  for (int t = 0; t < j; ++t) before += tsum[g][t];
  const double base = (act && d.pn_sigma > 0.f) ? d.pn_base[c - c0] : 0.0;
  if (!act) return;
  float phi = before;
  const unsigned long long uc = (unsigned long long)p0 * d.inc_c, uf = (unsigned long long)p0 * d.inc_cfo;
  unsigned short q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long p = p0 + i;
    phi += inc[i];
    const float2 s = d.s[p & (d.s_cap - 1)];
    float2 dv = make_float2(s.x + d.iq.x * s.x + d.iq.y * s.y, s.y + d.iq.y * s.x - d.iq.x * s.y);  // s + beta s*
    // phase noise (double base + float in-block prefix) and CFO, then the data's offset below
    // the tone; exact 64-bit DDS phase words
    float sp, cp;
    const double ph = base + (double)phi;
    const float phr = (float)(ph - 6.283185307179586 * rint(ph * 0.15915494309189535));
    sincosf(phr, &sp, &cp);
    dv = cmul(dv, make_float2(cp, sp));
    dv = cmul(dv, tx_dds(uf + (unsigned long long)i * d.inc_cfo));
    const float2 e = cadd(make_float2(d.A, 0.f), cmul(dv, tx_dds(uc + (unsigned long long)i * d.inc_c)));
    const float2 en = make_float2(fmaf(d.sigma, nz[i].y, e.x), fmaf(d.sigma, nz[i].z, e.y));
    q[i] = tx_quantise(d, en.x * en.x + en.y * en.y);                                 // |E|^2
  }
  const long long o = p0 - call_p0;
  *reinterpret_cast<uint4 *>(out + o) = make_uint4(q[0] | (q[1] << 16), q[2] | (q[3] << 16), q[4] | (q[5] << 16),
                                                   q[6] | ((unsigned)q[7] << 16));
}

// ------------------------------------------------------------------ PAM clock + AWGN + ADC
// y_p = sum_i s[t0 + i] h_ph[i] (t_p = p / (1 + eps), t0 = floor t_p, ph = rint(frac 4096)),
// x_p = y_p + sigma N(0,1) (normal 0 of sample p, tag 2)
__global__ void __launch_bounds__(256) k_tx_pam(TxDev d, long long p_lo, long long n, unsigned short *out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long p = p_lo + i;
  float y;
  if (d.eps == 0.0) {
    y = d.s[p & (d.s_cap - 1)].x;
  } else {
    const double t = (double)p / (1.0 + d.eps);
    const double t0 = floor(t);
    const int ph = (int)rint((t - t0) * TX_PHASES);
    const long long b = (long long)t0 - TX_NTAP / 2 + 1;
    const float *h = d.ptab + (long long)ph * TX_NTAP;
    y = 0.f;
#pragma unroll 8
    for (int k = 0; k < TX_NTAP; ++k) {
      const long long n2 = b + k;
      if (n2 >= 0) y = fmaf(d.s[n2 & (d.s_cap - 1)].x, __ldg(h + k), y);
    }
  }
  const float x = fmaf(d.sigma, tx_normals(d, p, 2u).x, y);
  out[i] = tx_quantise(d, x);
}

// ------------------------------------------------------------------ handle
struct tx_handle {
  tx_config cfg;
  int device;
  TxDev d;
  std::vector<void *> allocs;
  long long n_out;      // samples generated so far
  long long s_done;     // shaped blocks computed so far (absolute)
};

template <typename T>
static int tx_alloc(tx_handle *h, T **p, long long n) {
  void *q = nullptr;
  if (cudaMalloc(&q, (size_t)(n > 0 ? n : 1) * sizeof(T)) != cudaSuccess) return RX_ENOMEM;
  cudaMemset(q, 0, (size_t)(n > 0 ? n : 1) * sizeof(T));
  h->allocs.push_back(q);
  *p = (T *)q;
  return RX_OK;
}
template <typename T>
static int tx_upload(tx_handle *h, const T **p, const std::vector<T> &v) {
  T *q;
  int s = tx_alloc(h, &q, (long long)v.size());
  if (s) return s;
  if (cudaMemcpy(q, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return RX_ECUDA;
  *p = q;
  return RX_OK;
}

extern "C" void tx_destroy(tx_handle *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (void *p : h->allocs) cudaFree(p);
  delete h;
}

static double tx_i0(double x) {
  double s = 1.0, t = 1.0;
  for (int k = 1; k < 64; ++k) {
    t *= (x / (2.0 * k)) * (x / (2.0 * k));
    s += t;
    if (t < 1e-18 * s) break;
  }
  return s;
}

#define TX_MAX_CALL (1LL << 26)

extern "C" int tx_create(const tx_config *c, int dev, tx_handle **out) {
  if (!c || !out) return RX_EINVAL;
  *out = nullptr;
  const bool kk = c->family == RX_QAM_KK;
  if (c->family != RX_PAM && !kk) return RX_EINVAL;
  if (!kk && !(c->order == 2 || c->order == 4 || c->order == 8 || c->order == 16)) return RX_EINVAL;
  if (kk && !(c->order == 4 || c->order == 16 || c->order == 64)) return RX_EINVAL;
  if (!(c->baud > 0) || !(c->sample_rate > 0)) return RX_EINVAL;
  const double sps = c->sample_rate / c->baud;
  if (fabs(sps - (kk ? 4.0 : 2.0)) > 1e-9) return RX_EINVAL;
  if (!c->shaping_taps || c->n_shaping_taps < 1 || c->n_shaping_taps % 2 == 0 || c->n_shaping_taps > 513) return RX_EINVAL;
  if (c->symbol_offset < 0 || c->symbol_offset >= RX_PREF || (c->prbs_seed & 0x7FFF) == 0) return RX_EINVAL;
  if (!(c->adc_full_scale > 0) || c->noise_sigma < 0 || c->linewidth_hz < 0 || fabs(c->clock_ppm) > 1e4) return RX_EINVAL;
  if (kk && c->clock_ppm != 0.0) return RX_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || dev < 0 || dev >= ndev) return RX_ECUDA;
  if (cudaSetDevice(dev) != cudaSuccess) return RX_ECUDA;
  tx_handle *h = new tx_handle();
  h->cfg = *c;
  h->cfg.shaping_taps = nullptr;
  h->device = dev;
  TxDev &d = h->d;
  memset(&d, 0, sizeof(d));
  d.kk = kk;
  d.M = c->order;
  d.L = kk ? (int)lround(sqrt((double)c->order)) : c->order;
  d.sps = kk ? 4 : 2;
  d.sym_off = c->symbol_offset;
  d.eps = c->clock_ppm * 1e-6;
  d.sigma = (float)c->noise_sigma;
  d.pn_sigma = (float)sqrt(2.0 * M_PI * c->linewidth_hz / c->sample_rate);
  d.A = (float)c->tone_amp;
  d.iq = make_float2((float)c->iq_re, (float)c->iq_im);
  d.inc_c = (unsigned long long)llrint(ldexp(-c->carrier_hz / c->sample_rate, 64));
  d.inc_cfo = (unsigned long long)llrint(ldexp(c->cfo_hz / c->sample_rate, 64));
  d.mean = (float)c->adc_mean;
  d.gain = (float)(2047.5 / c->adc_full_scale);
  d.seed_lo = (unsigned)c->noise_seed;
  d.seed_hi = (unsigned)(c->noise_seed >> 32);
  int s = RX_OK;
#define TTRY(x) do { s = (x); if (s) { tx_destroy(h); return s; } } while (0)
  {   // FFT twiddles, fft.cuh layout (the receiver's table construction, restated)
    std::vector<float2> tw(1024, make_float2(0.f, 0.f));
    auto w = [](long long k) { const double a = -2.0 * M_PI * (double)(k % 1024) / 1024.0; return make_float2((float)cos(a), (float)sin(a)); };
    for (int k = 0; k < 512; ++k) tw[k] = w(k);
    for (int r = 1; r < 8; ++r) for (int jj = 0; jj < 64; ++jj) tw[TW_P3 + 64 * (r - 1) + jj] = w(2LL * r * jj);
    for (int r = 1; r < 8; ++r) for (int k = 0; k < 8; ++k) tw[TW_P2 + 8 * (r - 1) + k] = w(16LL * r * k);
    TTRY(tx_upload(h, &d.tw, tw));
  }
  {   // H = DFT_1024 of the zero-phase FIR (taps[(L-1)/2 + n] at time n)
    std::vector<float2> H(1024);
    const int L = c->n_shaping_taps, half = (L - 1) / 2;
    for (int k = 0; k < 1024; ++k) {
      double re = 0.0, im = 0.0;
      for (int n = -half; n <= half; ++n) {
        const double tr = kk ? c->shaping_taps[2 * (half + n)] : c->shaping_taps[half + n];
        const double ti = kk ? c->shaping_taps[2 * (half + n) + 1] : 0.0;
        const double a = -2.0 * M_PI * (double)k * (double)n / 1024.0;
        re += tr * cos(a) - ti * sin(a);
        im += tr * sin(a) + ti * cos(a);
      }
      H[k] = make_float2((float)re, (float)im);
    }
    TTRY(tx_upload(h, &d.H, H));
  }
  {   // PRBS-15 reference symbols (c-10): Gray labels of consecutive log2 M-bit groups -> levels
    std::vector<int> bits(RX_PREF);
    unsigned st = c->prbs_seed & 0x7FFF;
    for (int i = 0; i < RX_PREF; ++i) { const unsigned b = ((st >> 14) ^ (st >> 13)) & 1u; st = ((st << 1) | b) & 0x7FFFu; bits[i] = (int)b; }
    const int kb = (int)lround(log2((double)c->order));
    auto gdec = [](int g) { int i = 0; for (; g; g >>= 1) i ^= g; return i; };
    std::vector<float2> sym(RX_PREF);
    const double sc = kk ? sqrt(3.0 / (2.0 * (c->order - 1))) : 0.0;
    for (int i = 0; i < RX_PREF; ++i) {
      int lab = 0;
      for (int t = 0; t < kb; ++t) lab = (lab << 1) | bits[((long long)i * kb + t) % RX_PREF];
      if (!kk) {
        const int li = gdec(lab);
        sym[i] = make_float2((float)((2.0 * li - c->order + 1) / (double)(c->order - 1)), 0.f);
      } else {
        const int hb = kb / 2, iI = gdec(lab >> hb), iQ = gdec(lab & ((1 << hb) - 1));
        sym[i] = make_float2((float)((2.0 * iI - d.L + 1) * sc), (float)((2.0 * iQ - d.L + 1) * sc));
      }
    }
    TTRY(tx_upload(h, &d.sym, sym));
  }
  if (!kk && d.eps != 0.0) {   // Kaiser(8)-windowed sinc kernels, 4097 fractional delays
    std::vector<float> tab((size_t)(TX_PHASES + 1) * TX_NTAP);
    const int half = TX_NTAP / 2;
    for (int ph = 0; ph <= TX_PHASES; ++ph)
      for (int k = 0; k < TX_NTAP; ++k) {
        const double x = (double)ph / TX_PHASES - (double)(k - half + 1);
        const double r = x / half, wv = fabs(r) < 1.0 ? tx_i0(8.0 * sqrt(1.0 - r * r)) / tx_i0(8.0) : 0.0;
        const double sn = fabs(x) < 1e-12 ? 1.0 : sin(M_PI * x) / (M_PI * x);
        tab[(size_t)ph * TX_NTAP + k] = (float)(sn * wv);
      }
    TTRY(tx_upload(h, &d.ptab, tab));
  }
  long long cap = 1;
  while (cap < 2 * TX_MAX_CALL + (1 << 16)) cap <<= 1;
  d.s_cap = cap;
  TTRY(tx_alloc(h, &d.s, d.s_cap));
  const long long maxblk = TX_MAX_CALL / TX_BLK + 8;
  TTRY(tx_alloc(h, &d.pn_part, maxblk));
  TTRY(tx_alloc(h, &d.pn_base, maxblk));
  TTRY(tx_alloc(h, &d.pn_carry, 1));
#undef TTRY
  if (cudaDeviceSynchronize() != cudaSuccess) { tx_destroy(h); return RX_ECUDA; }
  *out = h;
  return RX_OK;
}

extern "C" int tx_generate(tx_handle *h, unsigned short *out, long long n, void *stream) {
  if (!h || !out || n <= 0 || n % TX_BLK || n > TX_MAX_CALL || (((unsigned long long)out) & 15)) return RX_EINVAL;
  if (cudaSetDevice(h->device) != cudaSuccess) return RX_ECUDA;
  cudaStream_t s = (cudaStream_t)stream;
  TxDev &d = h->d;
  const long long P0 = h->n_out, P1 = h->n_out + n;
  // shaped waveform needed: samples [P0, P1), or around t_p = p / (1 + eps) for the resampler
  long long need_hi = P1;
  if (!d.kk && d.eps != 0.0) need_hi = (long long)ceil((double)(P1 - 1) / (1.0 + d.eps)) + TX_NTAP;
  const long long c_hi = (need_hi + TX_BLK - 1) / TX_BLK;
  if (c_hi > h->s_done) {
    const long long c0 = h->s_done;
    k_tx_shape<<<(unsigned)((c_hi - c0 + 3) / 4), 256, 0, s>>>(d, c0, c_hi);
    h->s_done = c_hi;
  }
  if (d.kk) {
    const long long c0 = P0 / TX_BLK, c1 = P1 / TX_BLK;
    if (d.pn_sigma > 0.f) {
      k_tx_pn_sums<<<(unsigned)((c1 - c0 + 7) / 8), 256, 0, s>>>(d, c0, c1);
      k_tx_pn_scan<<<1, 1, 0, s>>>(d, c1 - c0);
    }
    k_tx_kk<<<(unsigned)((c1 - c0 + 3) / 4), 256, 0, s>>>(d, c0, c1, P0, out);
  } else {
    k_tx_pam<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d, P0, n, out);
  }
  h->n_out = P1;
  return cudaGetLastError() == cudaSuccess ? RX_OK : RX_ECUDA;
}
