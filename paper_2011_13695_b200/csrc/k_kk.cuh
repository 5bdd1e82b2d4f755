// k_kk.cuh — Kramers-Kronig QAM-N chain kernels (§IV).
//
//  k_kk_s1   H0, H11-H15  ingest + dc + sqrt / 1/2 ln + R2C FFT-1024 + FD Hilbert + C2R +
//                         KK field reconstruction + 64-bit-DDS downshift  -> E ring (4 sps)
//  k_kk_s2   H16-H18      C2C FFT-1024 (2 x FFT-512 + radix-2) + 203-tap FD EQ + decimating
//                         512-point IFFT -> z ring (2 sps)
//  k_cfo_*   H19-H20      per-buffer power + 4th-power periodogram, argmax, parabolic
//                         interpolation, DDS carry
#pragma once
#include "fft.cuh"
#include "rx_dev.cuh"
#include "k_pam.cuh"

// Twiddle source per kernel: 1 = the 8 KiB table read from global memory (L1 / L2), 0 = staged into
// shared memory by every CTA (cp.async). Measured (C4, isolated): k_kk_s1 0.387 -> 0.370 ms with the
// global table (the staging loop was 5 % of its stall samples); k_kk_s2 0.402 -> 0.395 ms with the
// global table and without the register copy of the pass-3 twiddles (KK_S2_T3 = 0: no spill)
#ifndef KK_S1_TW_GLOBAL
#define KK_S1_TW_GLOBAL 1
#endif
#ifndef KK_S2_T3
#define KK_S2_T3 0          // 1: k_kk_s2 loads the pass-3 twiddles once per block for its three transforms
#endif
#ifndef KK_S2_TW_GLOBAL
#define KK_S2_TW_GLOBAL 1
#endif

// ------------------------------------------------------------------ H0, H11-H15
// Stage 1 of block b by the 64-thread group j = 0..63 (every thread of the CTA calls it: the FFT
// barriers are CTA-wide). act = 0: the group idles through the barriers; count: the block's owned
// samples are counted (clipped / domain errors; the fused front-end recomputes halo blocks
// uncounted). wait_tw: the twiddle table's cp.async staging is waited for before the first FFT.
// The reconstructed pairs (E_p, E_{p+1}), p = 512 b - 512 + 2 (j + 64 r), r = 2..5, p >= 0, go to
// sink(r, p, pair).
#ifndef KK_S1_T3
#define KK_S1_T3 0          // measured: 48 -> 72 registers, KK_S1 0.395 -> 0.438 ms (not kept)
#endif
template <class Sink>
__device__ __forceinline__ void kk_s1_block(const RxDev &d, const InView &in, long long b, bool act, bool count,
                                            bool wait_tw, int j, const float2 *tw, float2 *buf, Sink sink) {
  int clip = 0, dom = 0;
  long long first_dom = 0x7fffffffffffffffLL;
  float2 v[8];
  float amp[4][2];                                      // sqrt(I) of the kept samples (r = 2..5)
  if (act) {
    clip = load_block_regs(in, b, d.scale, j, v);       // x_p = 0 for p < 0 (c-0) -> I = dc
    const long long p0 = 512 * b - 512;
    const float2 dc2 = make_float2(d.dc, d.dc);
    const float2 hl = make_float2(0.5f * 0.693147182f, 0.5f * 0.693147182f);   // 1/2 ln 2 (exact halving)
    unsigned fail = 0;                                  // I + dc <= 0 among the owned samples (r >= 4)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float2 I = __fadd2_rn(v[r], dc2);                 // P:215 static DC offset
      if (r >= 4) fail |= ((unsigned)(I.x <= 0.0f) | ((unsigned)(I.y <= 0.0f) << 1)) << (2 * (r - 4));
      I = make_float2(fmaxf(I.x, 1e-12f), fmaxf(I.y, 1e-12f));
      // P:215 logarithm for the phase: 1/2 ln I = log2(I) (ln 2 / 2) (MUFU lg2, one FMUL2)
      const float2 hh = __fmul2_rn(make_float2(__log2f(I.x), __log2f(I.y)), hl);
      if (r >= 2 && r < 6) {                            // P:215 square root: amplitude
        const float2 a = __fmul2_rn(I, make_float2(rsqrtf(I.x), rsqrtf(I.y)));
        amp[r - 2][0] = a.x;
        amp[r - 2][1] = a.y;
      }
      v[r] = hh;
    }
    if (fail) {                                         // owned samples counted once (A7)
      dom = __popc(fail);
      const int k = __ffs(fail) - 1;                    // the first in index order
      first_dom = p0 + 2 * (j + 64 * (4 + (k >> 1))) + (k & 1);
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 4; ++r) amp[r][0] = amp[r][1] = 0.f;
  }
  if (!count || b < in.cnt_lo || b >= in.cnt_hi) {   // a time shard's halo block: counted by its owner
    clip = 0;
    dom = 0;
    first_dom = 0x7fffffffffffffffLL;
  }
  block_reduce_clip(d.st, clip);
  dom = __reduce_add_sync(0xffffffffu, dom);
  if ((threadIdx.x & 31) == 0 && dom) atomicAdd((unsigned long long *)&d.st->domain_errors, (unsigned long long)dom);
  if (first_dom != 0x7fffffffffffffffLL) atomicMin(&d.st->first_domain, first_dom);
  if (wait_tw) tw_wait();
#if KK_S1_T3
  const FftT3 t3 = fft_t3_load(tw, j);          // shared by the forward and inverse transforms
  const FftT3 *t3p = &t3;
#else
  const FftT3 *t3p = nullptr;
#endif
  fft512_regs<false>(buf, j, tw, v, t3p);
  fft512_publish_upper(buf, j, v);
  // FD Hilbert (c-6, A8): Phi = -j sgn(kappa) H, Phi[0] = Phi[512] = 0
  float2 Zk[4], Zn[4];
  const float2 *pm = fft_mirror_base(buf, j);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = j + 64 * r;
    float2 Xk, Xn;
    // (both packings without their 1/2 scalings: Z is exactly 4x, folded into the phase scale below)
    r2c_pair<false>(v[r], fft_partner(pm, j, r, v), tw[k], Xk, Xn);
    float2 Pk = cmul_mi(Xk), Pn = cmul_mi(Xn);
    if (k == 0) { Pk = make_float2(0.f, 0.f); Pn = make_float2(0.f, 0.f); }
    c2r_pair<false>(Pk, Pn, tw[k], Zk[r], Zn[r]);
  }
  const float2 Z256 = cscale(cconj(cmul_mi(cconj(v[4]))), 4.0f);
  __syncthreads();
  {
    float2 *paw = buf + j;                      // natural layout
    float2 *pmw = buf + (512 - j);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      paw[64 * r] = Zk[r];
      if (!(j == 0 && r == 0)) pmw[-64 * r] = Zn[r];
    }
    if (j == 0) buf[256] = Z256;
  }
  __syncthreads();
  {
    const float2 *const pa = buf + j;
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = pa[64 * r];
  }
  fft512_regs<true>(buf, j, tw, v, t3p);
  // v[r] = 2048 (phi[2n] + i phi[2n+1]) (512 of the unnormalised IFFT, 4 of the unscaled
  // packings), n = j + 64 r; kept local [256, 768) <=> r = 2..5
  if (act) {
    const float sg = (float)d.sideband;
    // downshift to DC: e^{-j psi(p; sigma f_c)}, 64-bit DDS from the absolute index for
    // the thread's first sample, then exact-phase-word steps of 1 and 128 samples as rotations
    // (|error| ~ 1e-7 after the 3 steps)
    const long long pa = 512 * b - 512 + 2 * (j + 128);
    float2 rp = dds_rot_neg((unsigned long long)pa * d.carrier_inc);
    const float2 st1 = d.carrier_st1, st128 = d.carrier_st128;   // (rx_create)
#pragma unroll
    for (int r = 2; r < 6; ++r) {
      const int n = j + 64 * r;
      const long long p = 512 * b - 512 + 2 * n;
      const float2 r0 = rp, r1 = cmul(rp, st1);
      rp = cmul(rp, st128);
      if (p < 0) continue;
      // sigma phi in [-pi, pi] first, then the MUFU sin/cos (accurate there); the pair of samples
      // on the packed pipe (sigma / 512 and the 2 pi multiples exact, as in the scalar form)
      float2 ph = __fmul2_rn(v[r], make_float2(sg * (1.0f / 2048.0f), sg * (1.0f / 2048.0f)));
      const float2 k2 = __fmul2_rn(ph, make_float2(0.15915494309189535f, 0.15915494309189535f));
      ph = __ffma2_rn(make_float2(rintf(k2.x), rintf(k2.y)), make_float2(-6.283185307179586f, -6.283185307179586f), ph);
      float s0, c0, s1, c1;
      __sincosf(ph.x, &s0, &c0);
      __sincosf(ph.y, &s1, &c1);
      const float2 e0 = cmul(__fmul2_rn(make_float2(c0, s0), make_float2(amp[r - 2][0], amp[r - 2][0])), r0);
      const float2 e1 = cmul(__fmul2_rn(make_float2(c1, s1), make_float2(amp[r - 2][1], amp[r - 2][1])), r1);
      sink(r, p, make_float4(e0.x, e0.y, e1.x, e1.y));
    }
  }
}

__global__ void __launch_bounds__(256, 5) k_kk_s1(RxDev d, InView in, long long b0, long long b1) {   // 5 CTAs / SM: <= 51 registers
  __shared__ float2 buf[FE_GROUPS][FFT_PAD_N];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
#if KK_S1_TW_GLOBAL
  const float2 *const tw = d.tw;   // the 8 KiB table from L1 / L2 (no per-CTA staging)
#else
  __shared__ float2 tws[1024];
  const float2 *const tw = tws;
  tw_stage_async(tws, d.tw);  // waited for (tw_wait) before the first FFT pass
#endif
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  float2 *const E = d.E;
  const long long Ecap = d.E_cap;
  kk_s1_block(d, in, b, b < b1, true, !KK_S1_TW_GLOBAL, j, tw, buf[g], [=](int, long long p, float4 e) {
    *reinterpret_cast<float4 *>(E + rmod(p, Ecap)) = e;
  });
}

// ------------------------------------------------------------------ H16-H18
// One block per 64-thread group, entirely in registers between the FFT passes:
//   F = DFT_1024(E frame) from the two half-size FFTs of the even / odd samples, whose pass-1
//   operands (E[p0 + 2n], E[p0 + 2n + 1], n = j + 64 r) are one float4 load each;
//   G'[k'] = (Ev[k'] + W^k' Od[k']) H2[k'],        k' in [0, 256)   (kappa = k')
//   G'[k'] = (Ev[k'] - W^k' Od[k']) H2[k' + 512],  k' in [256, 512) (kappa = k' - 512)
//   — bin k' = j + 64 r is exactly the IFFT's pass-1 operand of thread j, so the band-selected
//   spectrum feeds the decimating IFFT-512 without a shared-memory round trip.
// The block's overlapped E frame (1024 cf32, 8 KiB, contiguous in the E ring) is staged by one TMA
// bulk copy per group into shared memory (the north_star's "TMA staging of overlapped blocks"),
// completed on an mbarrier; the staging area then serves as the group's FFT scratch. Frames at
// the stream start (p < 0) or across the ring's end are loaded by the threads instead.
// Stage 2 of block b from its frame's even / odd samples in registers (ve[r] = E[p0 + 2n],
// vo[r] = E[p0 + 2n + 1], n = j + 64 r, p0 = 512 b - 512): every thread of the CTA calls it.
// W16^r = e^{-2 pi i r / 16} (r < 8) as literals
__device__ __forceinline__ float2 w16c(int r) {
  switch (r) {
    case 1: return make_float2(0.92387953251128674f, -0.38268343236508977f);
    case 2: return make_float2(0.70710678118654752f, -0.70710678118654752f);
    case 3: return make_float2(0.38268343236508977f, -0.92387953251128674f);
    case 4: return make_float2(0.0f, -1.0f);
    case 5: return make_float2(-0.38268343236508977f, -0.92387953251128674f);
    case 6: return make_float2(-0.70710678118654752f, -0.70710678118654752f);
    case 7: return make_float2(-0.92387953251128674f, -0.38268343236508977f);
    default: return make_float2(1.0f, 0.0f);
  }
}
__device__ __forceinline__ void kk_s2_block(const RxDev &d, long long b, bool act, int j, const float2 *tw,
                                            float2 *buf, float2 (&ve)[8], float2 (&vo)[8]) {
#if KK_S2_T3
  const FftT3 t3 = fft_t3_load(tw, j);        // shared by the three transforms
  const FftT3 *const t3p = &t3;
#else
  const FftT3 *const t3p = nullptr;
#endif
  fft512_regs<false>(buf, j, tw, ve, t3p);
  fft512_regs<false>(buf, j, tw, vo, t3p);
  // radix-2 combination, W1024^k for k = j + 64 r: W1024^j W16^r (one shared load, the W16^r
  // are constants; |error| ~ 1e-7)
  const float2 w0 = tw[j];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int k = j + 64 * r;
    const float2 wk = r == 0 ? w0 : cmul(w0, w16c(r));
    const float2 od = cmul(vo[r], wk);
    ve[r] = r < 4 ? cmul(cadd(ve[r], od), __ldg(d.H + k)) : cmul(csub(ve[r], od), __ldg(d.H + k + 512));
  }
  fft512_regs<true>(buf, j, tw, ve, t3p);
  // z_local[n] = 1/2 * IDFT512 = v / 1024; keep n in [128, 384) <=> r = 2..5
  if (act) {
#pragma unroll
    for (int r = 2; r < 6; ++r) {
      const long long q = 256 * b - 256 + j + 64 * r;
      if (q >= 0) d.z[rmod(q, d.z_cap)] = cscale(ve[r], 1.0f / 1024.0f);
    }
  }
}

#ifndef KK_S2_TMA
#define KK_S2_TMA 1
#endif
__global__ void __launch_bounds__(256, 4) k_kk_s2(RxDev d, long long b0, long long b1) {   // 4 CTAs / SM: <= 64 registers
#if KK_S2_TW_GLOBAL
  const float2 *const tw = d.tw;   // the 8 KiB table from L1 / L2 (no per-CTA staging)
#else
  __shared__ __align__(16) float2 tws[1024];
  const float2 *const tw = tws;
#endif
  __shared__ __align__(128) float2 stage[FE_GROUPS][1024];   // E frames (TMA), then FFT scratch
  __shared__ __align__(8) uint64_t fbar[FE_GROUPS];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  float2 *const buf = stage[g];                               // FFT_PAD_N <= 1024
  if (threadIdx.x < FE_GROUPS) mbar_init(&fbar[threadIdx.x], 1);
  mbar_fence_init();
#if !KK_S2_TW_GLOBAL
  tw_stage_async(tws, d.tw);  // waited for (tw_wait) before the first FFT pass
#endif
  __syncthreads();            // barrier inits visible to every thread
  pdl_wait();                 // E from k_kk_s1
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  const bool act = b < b1;
  const long long p0 = 512 * b - 512;                         // frame [p0, p0 + 1024)
  const long long r0 = rmod(p0, d.E_cap);
  const bool tma = KK_S2_TMA && act && p0 >= 0 && r0 + 1024 <= d.E_cap;    // group-uniform
  if (tma && j == 0) {
    mbar_expect_tx(&fbar[g], 1024 * sizeof(float2));
    bulk_g2s(stage[g], d.E + r0, 1024 * sizeof(float2), &fbar[g]);
  }
  float2 ve[8], vo[8];
  {
    float4 e[8];
    if (tma) {
      mbar_wait(&fbar[g], 0);
      const float4 *sf = reinterpret_cast<const float4 *>(stage[g]);
#pragma unroll
      for (int r = 0; r < 8; ++r) e[r] = sf[j + 64 * r];    // E[p0 + 2n], E[p0 + 2n + 1], n = j + 64 r
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) {         // E_p = 0 for p < 0
        const long long p = p0 + 2 * (j + 64 * r);
        e[r] = (act && p >= 0) ? *reinterpret_cast<const float4 *>(d.E + rmod(p, d.E_cap))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) { ve[r] = make_float2(e[r].x, e[r].y); vo[r] = make_float2(e[r].z, e[r].w); }
  }
#if KK_S2_TW_GLOBAL
  __syncthreads();            // every thread's frame is in registers before the FFT scratch use
#else
  tw_wait();                  // (also: every thread's frame is in registers before the FFT scratch use)
#endif
  kk_s2_block(d, b, act, j, tw, buf, ve, vo);
}

// ------------------------------------------------------------------ H0, H11-H18 fused
// k_kk_fe: both overlap-save stages in one kernel, the 4-sps field E never leaving the SM
// (P:213 'to limit GPU memory access'; only the 2-sps field z touches HBM).
// CTA c owns the stage-2 blocks [x_c, x_c + per_cta) of [x0, x1) and walks them in steps of
// FE_GROUPS: iteration k computes stage 1 of the blocks y = x_c - 1 + 4k + g (one per group) into
// a shared ring of KKFE_SLOTS x 512 E samples (slot y mod KKFE_SLOTS), then, after one CTA barrier,
// stage 2 of the blocks x = x_c - 2 + 4k + g, whose frames [512x - 512, 512x + 512) are the
// upper half of slot x - 1, slot x and the lower half of slot x + 1 (all written by now).
// The CTA recomputes the stage-1 blocks x_c - 1 and x_c + per_cta at its edges (halos, not
// counted); a stage-1 block is counted by the CTA whose stage-2 range holds it (the last CTA
// also counts x1), and only if it is new in this call (y >= f0). The arithmetic of both stages
// is kk_s1_block / kk_s2_block, so z is bit-identical to the k_kk_s1 -> E -> k_kk_s2 path.
#define KKFE_SLOTS 6
#define KKFE_SMEM (KKFE_SLOTS * 256 * 16)   // dynamic shared memory of k_kk_fe (static: 25.6 KB)
__global__ void __launch_bounds__(256, 4) k_kk_fe(RxDev d, InView in, long long f0, long long x0, long long x1,
                                                  int per_cta) {
  __shared__ __align__(16) float2 tw[1024];
  __shared__ __align__(16) float2 buf[FE_GROUPS][FFT_PAD_N];
  extern __shared__ __align__(16) float4 ring_dyn[];          // [KKFE_SLOTS][256]: 512 E samples per slot
  float4 (*const ring)[256] = reinterpret_cast<float4 (*)[256]>(ring_dyn);
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  const long long xc0 = x0 + (long long)blockIdx.x * per_cta;
  if (xc0 >= x1) return;                                      // CTA-uniform
  const long long xc1 = xc0 + per_cta < x1 ? xc0 + per_cta : x1;
  const bool last = xc1 == x1;
  tw_stage_async(tw, d.tw);
  const int niter = (int)((xc1 - xc0 + 2 + FE_GROUPS - 1) / FE_GROUPS);
  for (int k = 0; k < niter; ++k) {
    // ---- stage 1 of y into slot y mod KKFE_SLOTS
    const long long y = xc0 - 1 + (long long)FE_GROUPS * k + g;
    const bool act1 = y >= 0 && y <= xc1;
    const bool cnt = y >= f0 && ((y >= xc0 && y < xc1) || (last && y >= xc1));
    float4 *const slot = ring[(int)(y % KKFE_SLOTS + KKFE_SLOTS) % KKFE_SLOTS];
    kk_s1_block(d, in, y, act1, cnt, k == 0, j, tw, buf[g], [=](int r, long long, float4 e) {
      slot[j + 64 * (r - 2)] = e;
    });
    __syncthreads();
    // ---- stage 2 of x from slots x - 1, x, x + 1
    const long long x = xc0 - 2 + (long long)FE_GROUPS * k + g;
    const bool act2 = x >= xc0 && x < xc1;
    float2 ve[8], vo[8];
    {
      const int sm = (int)((x - 1) % KKFE_SLOTS + KKFE_SLOTS) % KKFE_SLOTS;
      const int s0 = sm + 1 == KKFE_SLOTS ? 0 : sm + 1, sp = s0 + 1 == KKFE_SLOTS ? 0 : s0 + 1;
      const long long p0 = 512 * x - 512;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        // frame offset m = 2 (j + 64 r): slot x - 1 + (r + 2) / 4 at pair index j + 64 ((r + 2) % 4)
        const int sl = r < 2 ? sm : (r < 6 ? s0 : sp);
        float4 e = ring[sl][j + 64 * ((r + 2) & 3)];
        if (!act2 || p0 + 2 * (j + 64 * r) < 0) e = make_float4(0.f, 0.f, 0.f, 0.f);   // E_p = 0 for p < 0
        ve[r] = make_float2(e.x, e.y);
        vo[r] = make_float2(e.z, e.w);
      }
    }
    kk_s2_block(d, x, act2, j, tw, buf[g], ve, vo);
  }
}

// ------------------------------------------------------------------ H19-H20
// Per-buffer power normalisation and coarse + fine CFO (c-8, reading R-CFO), batched over the
// buffers that complete in one call (blockIdx.y = buffer of the call):
//  k_cfo_spec   CFO_ROWS CTAs per buffer, 4 chunks of 1024 per CTA step (one per 64-thread
//               group): |DFT_1024(z^4)|^2 summed over the CTA's chunks in a fixed order -> one
//               partial row; power partials
//  (final)      the last k_cfo_spec CTA of each buffer: rows -> S[k] (fixed order), P, k* (lowest on ties), delta,
//               coarse df and its DDS increment
//  k_cfo_fine   one warp per chunk: a_i = sum (z e^{-j psi_c})^4; the last CTA of a buffer forms
//               rho = sum a_{i+1} conj(a_i) in index order -> fine df
//  k_cfo_carry  one thread: DDS increments and phase origins carried across buffers
//  zp_value     z' = z / sqrt(P) e^{-j psi'}, evaluated where the equaliser stages read it
__device__ __forceinline__ void buf_range(const RxDev &d, long long beta, long long qfront,
                                          long long &qlo, long long &qhi) {
  const long long Q = (long long)d.buffer_blocks * 256;
  qlo = beta * Q;
  qhi = qlo + Q < qfront ? qlo + Q : qfront;
}

// e^{-j 2 pi u / 2^64} of a 64-bit phase word from its top 32 bits as an angle in [-pi, pi),
// MUFU sin / cos (|error| ~ 1e-6 rad); the exact-libm variant is dds_rot_neg (common.cuh)
__device__ __forceinline__ float2 dds_rot_neg_fast(unsigned long long u) {
  const float x = (float)(int)(u >> 32) * 1.4629180792671596e-9f;   // pi 2^-31
  float sn, cs;
  __sincosf(x, &sn, &cs);
  return make_float2(cs, -sn);
}

// Per-buffer periodogram argmax + log-parabolic interpolation + power (c-8): the CTA that finishes
// a buffer's spectrum rows (last-CTA ticket in k_cfo_spec) reduces them in fixed row order
// (CFO_SPEC_T threads, each owning the bins k = t + CFO_SPEC_T i)
#define CFO_SPEC_T 256
// spectrum rows (CTAs) per buffer and the resident CTAs per SM the register allocation must
// allow: 3 x 148 SMs hold a 4-buffer call's 416 CTAs in one wave with 80 registers (no spills;
// 4 CTAs per SM capped them at 64 with 48 B of stack)
#ifndef CFO_ROWS
#define CFO_ROWS 104
#endif
#ifndef CFO_MINB
#define CFO_MINB 3
#endif
#define CFO_GRP 8              // rows summed per group in the two-level row reduction
static_assert(CFO_ROWS % CFO_GRP == 0, "CFO_ROWS must be a multiple of CFO_GRP");
#define CFO_KPT (1024 / CFO_SPEC_T)
__device__ __forceinline__ void cfo_final_block(const RxDev &d, long long beta, long long qfront, long long rb, int nrows) {
  __shared__ double Sd[1024];
  __shared__ double wv[CFO_SPEC_T / 32];
  __shared__ int wi[CFO_SPEC_T / 32];
  __shared__ double pws[CFO_SPEC_T / 32];
  const int t = threadIdx.x;
  long long qlo, qhi;
  buf_range(d, beta, qfront, qlo, qhi);
  double bv = -1.0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < CFO_KPT; ++i) {
    const int k = t + CFO_SPEC_T * i;
    double sk = 0.0;
    int r = 0;
    for (; r + 16 <= nrows; r += 16) {        // 16 independent loads in flight, summed in row order
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(d.cfo_part + (rb + r + u) * 1024 + k);
#pragma unroll
      for (int u = 0; u < 16; ++u) sk += (double)v[u];
    }
    for (; r < nrows; ++r) sk += (double)__ldcg(d.cfo_part + (rb + r) * 1024 + k);
    Sd[k] = sk;
    if (sk > bv) { bv = sk; bi = k; }         // k increasing: strict > keeps the lowest on ties
  }
  double pw = 0.0;
  for (int r = t; r < nrows; r += blockDim.x) pw += __ldcg(d.cfo_pow + rb + r);
  pw = warp_sum_d(pw);
  if ((t & 31) == 0) pws[t >> 5] = pw;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if ((t & 31) == 0) { wv[t >> 5] = bv; wi[t >> 5] = bi; }
  __syncthreads();
  if (t == 0) {
    double P = 0.0;
    for (int w = 0; w < CFO_SPEC_T / 32; ++w) P += pws[w];
    const long long n = qhi - qlo;
    P = n > 0 ? P / (double)n : 1.0;
    if (!(P > 0.0)) P = 1.0;
    double best = wv[0];
    int k = wi[0];
    for (int w = 1; w < CFO_SPEC_T / 32; ++w)
      if (wv[w] > best || (wv[w] == best && wi[w] < k)) { best = wv[w]; k = wi[w]; }
    const long long nch = n / 1024;
    double df = 0.0;
    const bool have = nch > 0;
    if (have) {
      const double lm = log(Sd[(k + 1023) & 1023]), l0 = log(Sd[k]), lp = log(Sd[(k + 1) & 1023]);
      const double delta = 0.5 * (lm - lp) / (lm - 2.0 * l0 + lp);
      const double kap = (double)(k < 512 ? k : k - 1024);
      df = (kap + delta) * d.fs2 / (4.0 * 1024.0);
    } else {
      k = -1;
    }
    CfoParam cp;
    cp.P = P;
    cp.inv_sqrtP = (float)(1.0 / sqrt(P));
    cp.kstar = k;
    cp.df = df;                      // coarse (refined by k_cfo_fine; kstar < 0: reuse previous)
    cp.inc = (unsigned long long)llrint(ldexp(df / d.fs2, 64));
    cp.origin = 0ull;
    d.cfo[rmod(beta, d.buf_cap)] = cp;
  }
}

// |DFT_1024(z^4)|^2 periodogram rows + power partials. Grid (CFO_ROWS, buffers of the call),
// CFO_SPEC_T threads = 4 groups of 64, one FFT-1024 (2 x FFT-512 + radix-2) per group at a time:
// CTA x takes chunks c = 4 (x + CFO_ROWS it) + g, it = 0, 1, ... (4 consecutive chunks per CTA
// step, every CTA resident in one wave), accumulates |X[k]|^2 of its chunks per thread in
// registers (chunk order), then sums the 4 groups in fixed order into row x. The power partial
// sums the same samples (plus, in CTA 0, the tail beyond the last complete chunk).
// CFO_STAGE: each group's next chunk (1024 z, 8 KiB, contiguous in the ring: chunks start at
// multiples of 1024 from a buffer start) is fetched by one TMA bulk copy into dynamic shared memory
// while the group transforms the current one (mbarrier completion, one phase per chunk)
#ifndef CFO_STAGE
#define CFO_STAGE 1
#endif
#define CFO_STAGE_SMEM (CFO_STAGE ? (CFO_SPEC_T / 64) * 1024 * 8 : 0)
__global__ void __launch_bounds__(CFO_SPEC_T, CFO_MINB) k_cfo_spec(RxDev d, long long beta0, long long qfront) {
  __shared__ float2 tw[1024];
  __shared__ float2 bufs[CFO_SPEC_T / 64][FFT_PAD_N];   // FFT scratch; later acc[4][1024] floats
  __shared__ double red[CFO_SPEC_T / 32];
  __shared__ __align__(8) uint64_t fbar[CFO_SPEC_T / 64];
  extern __shared__ __align__(128) float4 cfo_stage_dyn[];  // [NG][512]: 1024 z per group
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  long long qlo, qhi;
  buf_range(d, beta0 + blockIdx.y, qfront, qlo, qhi);
  tw_stage_async(tw, d.tw);   // waited for before the first FFT (tw_wait, iteration 0)
  constexpr int NG = CFO_SPEC_T / 64;
  if (CFO_STAGE && threadIdx.x < NG) mbar_init(&fbar[threadIdx.x], 1);
  if (CFO_STAGE) mbar_fence_init();
  __syncthreads();
  pdl_wait();                 // z from k_kk_s2
  const long long nch = (qhi - qlo) / 1024;
  float4 *const stage = cfo_stage_dyn + 512 * g;
  auto chunk_of = [&](long long it) { return (long long)NG * (blockIdx.x + (long long)gridDim.x * it) + g; };
  auto fetch = [&](long long c) {   // one thread per group
    mbar_expect_tx(&fbar[g], 1024 * sizeof(float2));
    bulk_g2s(stage, d.z + rmod(qlo + 1024 * c, d.z_cap), 1024 * sizeof(float2), &fbar[g]);
  };
  if (CFO_STAGE && j == 0 && chunk_of(0) < nch) fetch(chunk_of(0));
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  double pw = 0.0;
  const long long steps = (nch + (long long)NG * gridDim.x - 1) / ((long long)NG * gridDim.x);
  FftT3 t3;
  for (long long it = 0; it < steps; ++it) {   // uniform trip count (the FFT barriers are CTA-wide)
    const long long c = chunk_of(it);
    const bool act = c < nch;
    float2 ve[8], vo[8];
    float p0 = 0.f;
    if (CFO_STAGE && act) mbar_wait(&fbar[g], (unsigned)(it & 1));
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
      if (act) zz = CFO_STAGE ? stage[j + 64 * r]
                              : *reinterpret_cast<const float4 *>(d.z + rmod(qlo + 1024 * c + 2 * (j + 64 * r), d.z_cap));
      p0 += zz.x * zz.x + zz.y * zz.y + zz.z * zz.z + zz.w * zz.w;
      const float2 a = make_float2(zz.x, zz.y), bq = make_float2(zz.z, zz.w);
      const float2 a2 = cmul(a, a), b2 = cmul(bq, bq);
      ve[r] = cmul(a2, a2);
      vo[r] = cmul(b2, b2);
    }
    pw += (double)p0;
    if (it == 0) {                              // uniform over the CTA
      tw_wait();
      t3 = fft_t3_load(tw, j);
    }
    fft512_regs<false, 0>(bufs[g], j, tw, ve, &t3);
    // every thread of the CTA has passed the transform's barriers, so the group's staged chunk
    // has been read: the next one goes into the same stage (async-proxy write after generic reads)
    if (CFO_STAGE && j == 0 && chunk_of(it + 1) < nch) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      fetch(chunk_of(it + 1));
    }
    fft512_regs<false, 0>(bufs[g], j, tw, vo, &t3);   // same buffer: fft512_regs syncs before its first store
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float2 od = cmul(vo[r], tw[j + 64 * r]);
      acc[r] += act ? cabs2(cadd(ve[r], od)) : 0.f;        // X[k],       k = j + 64 r
      acc[8 + r] += act ? cabs2(csub(ve[r], od)) : 0.f;    // X[k + 512]
    }
  }
  if (blockIdx.x == 0)                          // power of the tail beyond the complete chunks
    for (long long q = qlo + 1024 * nch + threadIdx.x; q < qhi; q += blockDim.x) pw += (double)cabs2(d.z[rmod(q, d.z_cap)]);
  __syncthreads();                              // every group done with its FFT buffer
  float *accs = reinterpret_cast<float *>(&bufs[0][0]);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    accs[g * 1024 + j + 64 * r] = acc[r];
    accs[g * 1024 + j + 64 * r + 512] = acc[8 + r];
  }
  __syncthreads();
  const long long row = (long long)blockIdx.y * d.cfo_G + blockIdx.x;   // CFO_ROWS rows + group rows per buffer
#pragma unroll
  for (int i = 0; i < CFO_KPT; ++i) {
    const int k = threadIdx.x + CFO_SPEC_T * i;
    float sk = 0.f;
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) sk += accs[gg * 1024 + k];
    d.cfo_part[row * 1024 + k] = sk;
  }
  pw = warp_sum_d(pw);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < CFO_SPEC_T / 32; ++i) t += red[i];
    d.cfo_pow[row] = t;
  }
  // two-level fixed-order reduction of the rows: the last CTA of each group of CFO_GRP rows sums
  // them (row order) into a group row, the last group finisher reduces the group rows (group
  // order) and takes the argmax / interpolation / power (cfo_final_block)
  __shared__ int ticket;
  const int ngrp = CFO_ROWS / CFO_GRP, grp = blockIdx.x / CFO_GRP;
  int *tick = d.cfo_tick_spec + blockIdx.y * (ngrp + 1);
  const long long rb = (long long)blockIdx.y * d.cfo_G;        // this buffer's rows
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(tick + grp, 1);
  __syncthreads();
  if (ticket != CFO_GRP - 1) return;
  __threadfence();
#pragma unroll
  for (int i = 0; i < CFO_KPT; ++i) {
    const int k = threadIdx.x + CFO_SPEC_T * i;
    float v[CFO_GRP];
#pragma unroll
    for (int r = 0; r < CFO_GRP; ++r) v[r] = __ldcg(d.cfo_part + (rb + grp * CFO_GRP + r) * 1024 + k);
    float sk = 0.f;
#pragma unroll
    for (int r = 0; r < CFO_GRP; ++r) sk += v[r];
    d.cfo_part[(rb + CFO_ROWS + grp) * 1024 + k] = sk;
  }
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < CFO_GRP; ++r) t += __ldcg(d.cfo_pow + rb + grp * CFO_GRP + r);
    d.cfo_pow[rb + CFO_ROWS + grp] = t;
    tick[grp] = 0;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(tick + ngrp, 1);
  __syncthreads();
  if (ticket != ngrp - 1) return;
  __threadfence();
  cfo_final_block(d, beta0 + blockIdx.y, qfront, rb + CFO_ROWS, ngrp);
  if (threadIdx.x == 0) tick[ngrp] = 0;
}


__global__ void __launch_bounds__(256) k_cfo_fine(RxDev d, long long beta0, long long qfront, int cta_per_buf) {
  __shared__ int ticket;
  pdl_wait();                 // the coarse estimate from k_cfo_spec
  const long long beta = beta0 + blockIdx.y;
  long long qlo, qhi;
  buf_range(d, beta, qfront, qlo, qhi);
  const long long nch = (qhi - qlo) / 1024;
  CfoParam *cpp = &d.cfo[rmod(beta, d.buf_cap)];
  const unsigned long long inc = cpp->inc;
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  double2 *abuf = d.cfo_a + (long long)blockIdx.y * (d.buffer_blocks / 4 + 1);
  if (i < nch) {
    float2 zz[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) zz[u] = d.z[rmod(qlo + 1024 * i + lane + 32 * u, d.z_cap)];
    float ax = 0.f, ay = 0.f;
    // DDS rotation: exact phase word every 8th sample of the lane (MUFU sin/cos of the top 32
    // bits), 32-sample step rotations in between (|error| ~ 1e-6 rad)
    const float2 st32 = dds_rot_neg_fast(32ULL * inc);
    float2 rot = make_float2(1.f, 0.f);
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const long long n = 1024 * i + lane + 32 * u;
      rot = (u & 7) == 0 ? dds_rot_neg_fast((unsigned long long)n * inc) : cmul(rot, st32);
      const float2 w = cmul(zz[u], rot);
      const float2 w2 = cmul(w, w), w4 = cmul(w2, w2);
      ax += w4.x;
      ay += w4.y;
    }
    const double sx = warp_sum_d((double)ax), sy = warp_sum_d((double)ay);
    if (lane == 0) abuf[i] = make_double2(sx, sy);
  }
  // last CTA of this buffer: rho in index order -> fine df (stored in the coarse slot)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(&d.cfo_tick[blockIdx.y], 1);
  __syncthreads();
  if (ticket != cta_per_buf - 1) return;
  __threadfence();
  double rx = 0.0, ry = 0.0;
  for (long long k = threadIdx.x; k + 1 < nch; k += blockDim.x) {
    volatile const double *vb = reinterpret_cast<volatile const double *>(abuf);
    const double ax = vb[2 * k], ay = vb[2 * k + 1], bx = vb[2 * k + 2], by = vb[2 * k + 3];
    rx += bx * ax + by * ay;
    ry += by * ax - bx * ay;
  }
  rx = warp_sum_d(rx);
  ry = warp_sum_d(ry);
  __shared__ double2 red[8];
  if (lane == 0) red[threadIdx.x >> 5] = make_double2(rx, ry);
  __syncthreads();
  if (threadIdx.x == 0) {
    double sx = 0.0, sy = 0.0;
    for (int w = 0; w < 8; ++w) { sx += red[w].x; sy += red[w].y; }
    if (nch >= 2) cpp->df = cpp->df + atan2(sy, sx) * d.fs2 / (2.0 * 3.141592653589793 * 4.0 * 1024.0);
    d.cfo_tick[blockIdx.y] = 0;
  }
}

// DDS increments and phase origins, carried across buffers (sequential, tiny); then z' is valid
// (computed on the fly by zp_value) for q < min((beta0 + nbuf) Q, qfront)
__global__ void k_cfo_carry(RxDev d, long long beta0, int nbuf, long long qfront) {
  for (int i = 0; i < nbuf; ++i) {
    CfoParam cp = d.cfo[rmod(beta0 + i, d.buf_cap)];
    double df = cp.kstar >= 0 ? cp.df : d.st->cfo_df_prev;   // no complete chunk: reuse
    if (d.cfo_enable) {
      cp.df = df;
      cp.inc = (unsigned long long)llrint(ldexp(df / d.fs2, 64));
      cp.origin = d.st->cfo_origin_next;
      d.st->cfo_origin_next = cp.origin + (unsigned long long)((long long)d.buffer_blocks * 256) * cp.inc;
      d.st->cfo_df_prev = df;
    } else {
      cp.df = 0.0; cp.inc = 0ull; cp.origin = 0ull;
    }
    d.cfo[rmod(beta0 + i, d.buf_cap)] = cp;
  }
  const long long q1 = (beta0 + nbuf) * (long long)d.buffer_blocks * 256;
  d.st->v_front = q1 < qfront ? q1 : qfront;   // consumed by later launches (stream order)
}

// z'_q = z_q / sqrt(P_beta) e^{-j psi'_q} (c-8), psi' the carried per-buffer CFO DDS: evaluated
// where it is consumed (the equaliser's shared-memory staging, frame sync, training) instead of
// being materialised as a ring (the former k_kk_zprime pass: one HBM read + write of the 2-sps
// field saved). The phase word is exact (64-bit, absolute index); the rotation takes the MUFU
// sin/cos of the top 32 bits as an angle in [-pi, pi) (|error| ~ 1e-6 rad).
struct ZpCache {
  long long beta;
  unsigned long long origin, inc;
  float s;
};
__device__ __forceinline__ float2 zp_rotate(const RxDev &d, float2 v, long long q, ZpCache &c) {
  const long long beta = q >> d.q_shift;
  if (beta != c.beta) {
    const CfoParam &cp = d.cfo[rmod(beta, d.buf_cap)];
    c.beta = beta;
    c.origin = cp.origin;
    c.inc = cp.inc;
    c.s = cp.inv_sqrtP;
  }
  v = cscale(v, c.s);
  if (d.cfo_enable) v = cmul(v, dds_rot_neg_fast(c.origin + (unsigned long long)(q - (beta << d.q_shift)) * c.inc));
  return v;
}
// Equaliser staging: a lane stages the samples q, q + 64, q + 128, ... (one per block); its z'
// rotation advances by the exact-phase-word step e^{-j psi'(64 inc)} (one complex multiply) and is
// re-anchored on the exact 64-bit phase word every ZP_REANCHOR samples and at every buffer change
// (fp32 drift <= ZP_REANCHOR x ~1e-7 rad)
#define ZP_REANCHOR 32
struct ZpStep {
  long long beta;
  long long qlim;                  // the phasor steps hold for q < qlim (same buffer, < ZP_REANCHOR
                                   // steps since the anchor, q < vend)
  float2 rot, step;                // includes 1 / sqrt(P_beta)
};
// z'_q of the staging lane's next sample q (q advances by 64 per call): one complex multiply and
// one phasor step while q < qlim, else the exact-phase-word re-anchor (or 0 outside [0, vend))
__device__ __forceinline__ float2 zp_step(const RxDev &d, float2 v, long long q, ZpStep &z, long long vend) {
  if (!(q >= 0 && q < z.qlim)) {
    if (q < 0 || q >= vend) return make_float2(0.f, 0.f);
    const long long beta = q >> d.q_shift;
    const CfoParam &cp = d.cfo[rmod(beta, d.buf_cap)];
    const float s = cp.inv_sqrtP;
    if (d.cfo_enable) {
      z.rot = cscale(dds_rot_neg_fast(cp.origin + (unsigned long long)(q - (beta << d.q_shift)) * cp.inc), s);
      z.step = dds_rot_neg_fast(64ULL * cp.inc);
    } else {
      z.rot = make_float2(s, 0.f);
      z.step = make_float2(1.f, 0.f);
    }
    z.beta = beta;
    long long lim = (beta + 1) << d.q_shift;
    if (q + 64LL * ZP_REANCHOR < lim) lim = q + 64LL * ZP_REANCHOR;
    z.qlim = lim < vend ? lim : vend;
  }
  const float2 out = cmul(v, z.rot);
  z.rot = cmul(z.rot, z.step);
  return out;
}
__device__ __forceinline__ float2 zp_rotate_or_zero(const RxDev &d, float2 v, long long q, long long vend, ZpCache &c) {
  if (q < 0 || q >= vend) return make_float2(0.f, 0.f);
  return zp_rotate(d, v, q, c);
}
__device__ __forceinline__ float2 zp_value(const RxDev &d, long long q, long long vend, ZpCache &c) {
  if (q < 0 || q >= vend) return make_float2(0.f, 0.f);
  return zp_rotate(d, d.z[rmod(q, d.z_cap)], q, c);
}
