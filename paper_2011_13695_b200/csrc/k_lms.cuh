// k_lms.cuh — frame sync, segmented block-LMS equaliser with in-loop CPR, quadrant
// stitching, decisions, Gray labels and BER/EVM counters (c-9..c-11).
//
// The paper's KK equaliser is a serial 4-tap widely-linear DDLMS using warp shuffles
// and its PAM decision uses offline thresholds. The build's equaliser is
// the segment-parallel block-LMS of SURVEY c-9: one warp owns one segment of S symbols,
// lane i owns symbol i of each B = 32 block, lane k owns tap k; CPR and decisions are fused.
#pragma once
#include <type_traits>
#include "k_kk.cuh"


template <bool CPLX>
__device__ __forceinline__ float2 lms_in(const RxDev &d, long long i, long long vend) {
  if (i < 0 || i >= vend) return make_float2(0.f, 0.f);
  if (CPLX) {
    ZpCache c;
    c.beta = -1;
    return zp_value(d, i, vend, c);            // z' on the fly (c-8)
  }
  return make_float2(d.uhat[rmod(i, d.sym_cap)], 0.f);
}

// level index per axis: #{thresholds <= v} (c-11; ties go up)
__device__ __forceinline__ int slice_pam(const RxDev &d, float v) {
  int i = 0;
  for (int t = 0; t < d.M - 1; ++t) i += (__ldg(d.thr + t) <= v);
  return i;
}
__device__ __forceinline__ int slice_axis(float v, float inv2s, int L) {
  int i = (int)floorf(fmaf(v, inv2s, 0.5f * (float)L));
  return i < 0 ? 0 : (i > L - 1 ? L - 1 : i);
}

// rotate a QAM level pair by j^r: j (aI + j aQ) = -aQ + j aI -> (L-1-iQ, iI)
__device__ __forceinline__ int qam_rot(int code, int r, int L) {
  int iI = code & 15, iQ = code >> 4;
  for (int t = 0; t < (r & 3); ++t) { int nI = L - 1 - iQ; iQ = iI; iI = nI; }
  return iI | (iQ << 4);
}
__device__ __forceinline__ int gray(int i) { return i ^ (i >> 1); }

__device__ __forceinline__ long long seg_end_of(const RxDev &d, long long s) {
  long long hi = (s + 1) * (long long)d.S;
  const long long me = d.st->m_end;
  if (me >= 0 && hi > me) hi = me;
  return hi;
}

// ------------------------------------------------------------------ H24 frame sync
// Gamma(o,h) = |sum_i zeta_{m0+i,h} conj(r_{(o+i) mod P})| / (||zeta_h|| ||r_window||) (c-10)
template <bool CPLX>
__device__ __forceinline__ bool sync_ready(const RxDev &d) {
  const long long need = CPLX ? 2 * (d.m0 + d.W_sync) + 2 : d.m0 + d.W_sync;
  return d.st->v_lms >= need;
}

template <bool CPLX>
__global__ void __launch_bounds__(256) k_sync_corr(RxDev d) {
  extern __shared__ float2 zeta[];   // [nh][W]
  if (d.st->synced || !sync_ready<CPLX>(d)) return;
  const int nh = CPLX ? 2 : 1, W = d.W_sync;
  const long long vend = d.st->v_lms;
  for (int i = threadIdx.x; i < nh * W; i += blockDim.x) {
    const int h = i / W, k = i % W;
    zeta[i] = CPLX ? lms_in<true>(d, 2 * (d.m0 + k) + h, vend) : lms_in<false>(d, d.m0 + k, vend);
  }
  __syncthreads();
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nh * RX_PREF) return;
  const int h = gid / RX_PREF, o = gid % RX_PREF;
  float ar = 0.f, ai = 0.f, rn = 0.f;
  int idx = o;
  for (int i = 0; i < W; ++i) {
    const float2 r = __ldg(d.ref_val + idx);
    const float2 zz = zeta[h * W + i];
    ar = fmaf(zz.x, r.x, fmaf(zz.y, r.y, ar));
    ai = fmaf(zz.y, r.x, fmaf(-zz.x, r.y, ai));
    rn = fmaf(r.x, r.x, fmaf(r.y, r.y, rn));
    if (++idx == RX_PREF) idx = 0;
  }
  d.sync_c[gid] = make_float2(ar, ai);
  d.sync_g[gid] = sqrtf(ar * ar + ai * ai) * rsqrtf(fmaxf(rn, 1e-30f));
}

template <bool CPLX>
__global__ void __launch_bounds__(1024) k_sync_pick(RxDev d, int flush) {
  __shared__ double zn[2];
  __shared__ float bv[32];
  __shared__ int bi[32];
  DevState *st = d.st;
  if (st->synced) return;
  if (!sync_ready<CPLX>(d)) {
    if (flush && threadIdx.x == 0) set_flag(st, RX_FLAG_SYNC_DEV);
    return;
  }
  const int nh = CPLX ? 2 : 1, W = d.W_sync;
  const long long vend = st->v_lms;
  for (int h = 0; h < nh; ++h) {
    double s = 0.0;
    for (int k = threadIdx.x; k < W; k += blockDim.x) {
      const float2 zz = CPLX ? lms_in<true>(d, 2 * (d.m0 + k) + h, vend) : lms_in<false>(d, d.m0 + k, vend);
      s += (double)cabs2(zz);
    }
    s = warp_sum_d(s);
    __shared__ double wsum[32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 32; ++w) t += wsum[w];
      zn[h] = sqrt(t);
    }
    __syncthreads();
  }
  // argmax in (h, o) order, lowest on ties (as the oracle scans h outer, o inner)
  float best = -1.f;
  int bidx = 0x7fffffff;
  for (int gid = threadIdx.x; gid < nh * RX_PREF; gid += blockDim.x) {
    const int h = gid / RX_PREF;
    const float g = d.sync_g[gid] / (float)fmax(zn[h], 1e-30);
    if (g > best || (g == best && gid < bidx)) { best = g; bidx = gid; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = bidx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 32; ++w)
      if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) { bv[0] = bv[w]; bi[0] = bi[w]; }
    const int gid = bi[0];
    const float2 c = d.sync_c[gid];
    st->sync_offset = gid % RX_PREF;
    st->sync_phase = gid / RX_PREF;
    st->sync_gamma = bv[0];
    st->sync_phi0 = atan2((double)c.y, (double)c.x);
    st->sync_polarity = c.x < 0.f;
    if (bv[0] < d.sync_min) set_flag(st, RX_FLAG_SYNC_DEV);
    __threadfence();
    st->synced = 1;
    d.hm->synced = 1;
  }
}

// ------------------------------------------------------------------ H9/H21 LMS core
// One warp runs block-LMS over symbols [t_begin, t_end) starting from tap wk (lane k).
// MODE 0: training (e = r - y, no CPR), MODE 1: decision directed with CPR `CPR`
// (0 none, 1 VV, 2 BPS). Outputs for m >= out_lo go to the level / yout rings,
// warm-up decisions (m < out_lo) to warm[]. Returns final theta; accumulates EVM.
//
// Layout: taps are padded to KP = 4 ceil(K/4) (zero taps, exact) so the K-term dot products
// run with 4 independent accumulators; lane i owns symbol i of the block, lane k tap k; the
// sliding window of inputs lives in shared memory (double-buffered, next block prefetched
// into registers while the current block computes).
#define LMS_RING 512        // per-warp input ring (power of two), mirrored: element i lives at
                            // (i & (RING-1)) and (i & (RING-1)) + RING, so every block window is
                            // contiguous and read with compile-time offsets
#define LMS_AHEAD 4         // blocks of lookahead staged by cp.async

template <bool CPLX> struct LmsElem { using T = float; };    // PAM: real
template <> struct LmsElem<true> { using T = float2; };     // KK: complex

template <bool CPLX>
struct LmsSmemT {
  using T = typename LmsElem<CPLX>::T;
  alignas(16) T ring[2 * LMS_RING];
  alignas(16) T w[32];
  alignas(16) T v[32];      // widely-linear branch (KK, widely_linear = 1)
  alignas(16) T e[32];
  alignas(16) float2 y[32];
};

__device__ __forceinline__ void cp_async_elem(float *dst, const float *src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(src), "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async_elem(float2 *dst, const float2 *src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// stage input samples [i0, i1) (absolute index of u^ (PAM) or z' (KK)) into the mirrored ring;
// zero outside [0, vend). PAM: cp.async (zero-fill); KK: z' is formed from z on the way in
// (zp_value: normalisation + CFO rotation, c-8) and stored by the warp
template <bool CPLX>
__device__ __forceinline__ void lms_stage(const RxDev &d, LmsSmemT<CPLX> &sm, long long i0, long long i1,
                                          long long vend, long long base, ZpCache *zc = nullptr) {
  const int lane = threadIdx.x & 31;
  for (long long i = i0 + lane; i < i1; i += 32) {
    const bool ok = i >= 0 && i < vend;
    const int slot = (int)((i - base) & (LMS_RING - 1));   // block windows start 128 B aligned
    if constexpr (CPLX) {
      const float2 v = zp_value(d, i, vend, *zc);
      sm.ring[slot] = v;
      sm.ring[slot + LMS_RING] = v;
    } else {
      const float *src = ok ? d.uhat + rmod(i, d.sym_cap) : d.uhat;
      cp_async_elem(&sm.ring[slot], src, ok);
      cp_async_elem(&sm.ring[slot + LMS_RING], src, ok);
    }
  }
}

// BPS rounding: two FADDs with the 1.5 2^23 shift (round to nearest even, exact for |u| < 2^22)
// instead of FRND (measured: C4 +1-2 %, the FRND pipe is shared with the concurrent front-end).
// Beyond 2^22 both forms clamp to the same level, so the distances are identical for every input.
#ifndef BPS_MAGIC
#define BPS_MAGIC 1
#endif
__device__ __forceinline__ float bps_rint(float u) {
#if BPS_MAGIC
  return __fadd_rn(__fadd_rn(u, 12582912.f), -12582912.f);
#else
  return rintf(u);
#endif
}

// Blind phase search partial sums over symbols [i0, i1) of a block (lane p: test phases p and
// p + 32). Distances are in units of the level spacing 2s: u = y e^{-j phi_p} / 2s + (L - 1)/2
// puts the levels on the integers 0..L-1, so |z - slice(z)|^2 = (2s)^2 sum (u - clamp(rint u))^2
// (the common factor (2s)^2 does not move the argmin). Fixed summation order.
// acc += |u - clamp(rint(u))|^2 over both axes of y e^{-j phi} / 2s + (L - 1)/2 (two FFMA
// accumulations, no separate product)
__device__ __forceinline__ void bps_acc(float2 yi, float2 r, float cst, float Lm1, float &acc) {
  const float ux = fmaf(yi.x, r.x, fmaf(-yi.y, r.y, cst));
  const float uy = fmaf(yi.x, r.y, fmaf(yi.y, r.x, cst));
  const float ex = ux - fminf(fmaxf(bps_rint(ux), 0.f), Lm1);
  const float ey = uy - fminf(fmaxf(bps_rint(uy), 0.f), Lm1);
  acc = fmaf(ex, ex, acc);
  acc = fmaf(ey, ey, acc);
}
template <bool TWO>
__device__ __forceinline__ void bps_partial_t(const float2 *ys, int i0, int i1, float2 rsA, float2 rsB, int L,
                                              float &dA, float &dB) {
  const float cst = 0.5f * (float)(L - 1), Lm1 = (float)(L - 1);
  float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
  const float4 *y4 = reinterpret_cast<const float4 *>(ys);
  if (i0 == 0 && i1 == 32) {         // a full block (the common case): straight-line code
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float4 yy = y4[i];
      bps_acc(make_float2(yy.x, yy.y), rsA, cst, Lm1, a0);
      bps_acc(make_float2(yy.z, yy.w), rsA, cst, Lm1, a1);
      if (TWO) {
        bps_acc(make_float2(yy.x, yy.y), rsB, cst, Lm1, b0);
        bps_acc(make_float2(yy.z, yy.w), rsB, cst, Lm1, b1);
      }
    }
  } else {
    const int n2 = (i1 - i0) >> 1;   // i0 even
#pragma unroll 4
    for (int i = 0; i < n2; ++i) {
      const float4 yy = y4[(i0 >> 1) + i];
      bps_acc(make_float2(yy.x, yy.y), rsA, cst, Lm1, a0);
      bps_acc(make_float2(yy.z, yy.w), rsA, cst, Lm1, a1);
      if (TWO) {
        bps_acc(make_float2(yy.x, yy.y), rsB, cst, Lm1, b0);
        bps_acc(make_float2(yy.z, yy.w), rsB, cst, Lm1, b1);
      }
    }
    if ((i1 - i0) & 1) {
      const float2 yi = ys[i1 - 1];
      bps_acc(yi, rsA, cst, Lm1, a0);
      if (TWO) bps_acc(yi, rsB, cst, Lm1, b0);
    }
  }
  dA += a0 + a1;
  dB += b0 + b1;
}
// (the summation order is the same on both paths: even / odd symbol chains, then their sum)
__device__ __forceinline__ void bps_partial(const float2 *ys, int i0, int i1, float2 rsA, float2 rsB, int L,
                                            bool two, float &dA, float &dB) {
  if (two) bps_partial_t<true>(ys, i0, i1, rsA, rsB, L, dA, dB);
  else bps_partial_t<false>(ys, i0, i1, rsA, rsB, L, dA, dB);
}
__device__ __forceinline__ void named_bar(int id) {   // the 64 threads of a segment's warp pair
  asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory");
}

// 4 x 8 register tile of a 32 x 32 Toeplitz contraction (TILED path of lms_run): x4 -> 12
// consecutive window samples X, v4 -> 8 coefficients V; FILTER: acc[a] = sum_b V[b] X[a + 7 - b]
// (outputs a, taps b), else acc[a] = sum_b V[b] X[b + 3 - a] (taps a, outputs b)
__device__ __forceinline__ void lms_tile(const float4 *x4, const float4 *v4, float acc[4], bool filter) {
  const float4 xa = x4[0], xb = x4[1], xc = x4[2], va = v4[0], vb = v4[1];
  const float X[12] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w, xc.x, xc.y, xc.z, xc.w};
  const float V[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    float s = 0.f;
#pragma unroll
    for (int b = 0; b < 8; ++b) s = fmaf(V[b], filter ? X[a + 7 - b] : X[b + 3 - a], s);
    acc[a] = s;
  }
}
// reduce-scatter of acc[0..3] over the four lane quarters q: returns sum_q' acc_q'[q]
__device__ __forceinline__ float lms_tile_reduce(const float acc[4], int q) {
  const bool h = q & 2, l = q & 1;
  const float s0 = h ? acc[0] : acc[2], s1 = h ? acc[1] : acc[3];
  const float k0 = (h ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, s0, 16);
  const float k1 = (h ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, s1, 16);
  return (l ? k1 : k0) + __shfl_xor_sync(0xffffffffu, l ? k0 : k1, 8);
}

// PAM fast staging: 16-byte cp.async of 4 consecutive u^ (needs i0 = 0 mod 4, (i1 - i0) = 0 mod 4;
// a chunk never straddles index 0 or the ring wrap); zero-fill beyond vend / below 0
__device__ __forceinline__ void lms_stage_vec(const RxDev &d, LmsSmemT<false> &sm, long long i0, long long i1,
                                              long long vend, long long base) {
  const int lane = threadIdx.x & 31;
  for (long long i = i0 + 4 * lane; i < i1; i += 128) {
    long long nv = vend - i;
    nv = i < 0 ? 0 : (nv < 0 ? 0 : (nv > 4 ? 4 : nv));
    const int slot = (int)((i - base) & (LMS_RING - 1));
    const float *src = nv ? d.uhat + rmod(i, d.sym_cap) : d.uhat;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(&sm.ring[slot]);
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&sm.ring[slot + LMS_RING]);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"((int)(4 * nv)));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sb), "l"(src), "r"((int)(4 * nv)));
  }
}
template <bool CPLX>
__device__ __forceinline__ void lms_stage_any(const RxDev &d, LmsSmemT<CPLX> &sm, long long i0, long long i1,
                                              long long vend, long long base, bool vec, ZpCache *zc = nullptr) {
  if constexpr (!CPLX) {
    if (vec) { lms_stage_vec(d, sm, i0, i1, vend, base); return; }
  }
  lms_stage<CPLX>(d, sm, i0, i1, vend, base, zc);
}

__device__ __forceinline__ float2 as_c(float v) { return make_float2(v, 0.f); }
__device__ __forceinline__ float2 as_c(float2 v) { return v; }

// decision level value of index i: PAM (2i - M + 1)/(M - 1); QAM axis (2i - L + 1) sc
__device__ __forceinline__ float level_of(int i, float two_s, float off) { return fmaf((float)i, two_s, off); }

// One warp runs block-LMS over symbols [t_begin, t_end) starting from tap wk (lane k).
// MODE 0: training (e = r - y, no CPR, no outputs), MODE 1: decision directed with CPR `CPR`
// (0 none, 1 VV, 2 BPS), MODE 2: data aided (rx_config.lms_mode = 1: e = r - y, no CPR, as in
// training, with decisions slice(y) and outputs). Outputs for m >= out_lo go to the level /
// yout rings, warm-up decisions (m < out_lo) to warm[]. Returns final theta; accumulates EVM.
//
// Layout: taps are padded to KP in {4, 8, 16, 32} (zero taps, exact); lane i owns symbol i of
// the block, lane k tap k; the inputs stream through a per-warp mirrored shared-memory ring
// filled LMS_AHEAD blocks ahead with cp.async, so the serial block recursion never waits on
// HBM and every window access is an immediate offset.
//
// WLIN (KK): widely-linear form of c-9, y = w^H u + v^H conj(u), v <- v + mu sum conj(u) conj(e)
// (the paper's "widely-linear TD DDLMS"; DESIGN reading R-WL); lane k also owns v_k.
template <bool CPLX, int CPR, int MODE, int KP, bool WLIN = false>
__device__ float lms_run(const RxDev &d, LmsSmemT<CPLX> &sm, long long t_begin, long long t_end,
                         long long out_lo, float2 &wk, float2 &vk, unsigned char *warm, double &evn,
                         double &evd, long long vend, int bps_bar = 0, float2 *bps_part = nullptr) {
  using T = typename LmsElem<CPLX>::T;
  const int lane = threadIdx.x & 31;
  const int K = d.K, c = K >> 1;
  constexpr int stride = CPLX ? 2 : 1;
  const int off = CPLX ? d.st->sync_phase : 0;
  constexpr int WL = stride * 31 + KP;      // window of one block
  constexpr int DS = stride * 32;           // window shift per block
  const float mu = d.mu;
  const int L = d.L;
  const float two_s = CPLX ? 2.0f * d.qam_sc : 2.0f / (float)(d.M - 1);
  const float lvl0 = CPLX ? -(float)(L - 1) * d.qam_sc : -1.0f;
  const float inv2s = 1.0f / two_s;
  const float Lh = 0.5f * (float)L, Lm1 = (float)(L - 1);
  const long long o_ref = d.st->sync_offset;
  const int ref0 = MODE != 1 ? (int)(((o_ref + t_begin - d.m0) % RX_PREF + RX_PREF) % RX_PREF) : 0;
  float2 rotA = make_float2(1.f, 0.f), rotB = make_float2(1.f, 0.f);
  if (CPR == 2) {
    if (lane < d.Pt) rotA = __ldg(d.bps_rot + lane);
    if (lane + 32 < d.Pt) rotB = __ldg(d.bps_rot + lane + 32);
  }
  float theta = 0.f;
  // BPS over full 32-phase blocks: lane l scores the phase pair (q, 31 - q), q = l & 15; its
  // rotation e^{-j phi_q} / 2s is loaded once per run, not per block
  float bq_c = 0.f, bq_s = 0.f;
  if (CPR == 2 && d.Pt == 32) {
    const float2 rq = __ldg(d.bps_rot + (lane & 15));         // e^{-j phi_q} = (cos, -sin)
    bq_c = rq.x * inv2s;
    bq_s = -rq.y * inv2s;
  }
  float wmax = 0.f;   // max |w_k|^2 over the run's blocks (R-DIV: any tap beyond 1e3 at any block)
  // TILED (PAM, KP = 32): lane (q, r) = (lane >> 3, lane & 7) owns output / tap io = 4r + q and
  // computes a 4 x 8 register tile of each contraction from 128-bit shared loads, reduced over q
  // with two shuffle stages; otherwise lane i owns output i and tap i
  constexpr bool TILED = !CPLX && KP == 32;
  const int tq = lane >> 3, tr = lane & 7;
  const int io = TILED ? 4 * tr + tq : lane;
  if (lane >= K) wk = make_float2(0.f, 0.f);
  if constexpr (WLIN) {
    if (lane >= K) vk = make_float2(0.f, 0.f);
    reinterpret_cast<float2 *>(sm.v)[lane] = vk;
  }
  if (CPLX) reinterpret_cast<float2 *>(sm.w)[lane] = wk;
  else reinterpret_cast<float *>(sm.w)[lane] = wk.x;
  if (TILED) {
    __syncwarp();
    wk.x = reinterpret_cast<const float *>(sm.w)[io];
  }
  const long long wb0 = (long long)stride * t_begin + off + c - (KP - 1);
  const long long nblk = (t_end - t_begin + 31) / 32;
  constexpr int WLa = (WL + 3) & ~3;        // first stage rounded up: later stages stay 4-aligned
  const bool vec = !CPLX && (wb0 & 3) == 0;
  // PAM fast staging: every staged index of the run lies in [0, vend): 16-byte copies with
  // 32-bit ring arithmetic, the mirror copy only for the slots a window can wrap onto (< 64)
  const bool fast = vec && wb0 >= 0 && wb0 + WLa + DS * nblk <= vend;
  const int gbase = (int)(wb0 & (d.sym_cap - 1)), gmask = (int)(d.sym_cap - 1);
  ZpCache zc;                               // KK: CFO parameters of the buffer last staged
  zc.beta = -1;
  ZpStep zs[2];                             // KK: per-lane z' phasors of the two staged samples
  zs[0].qlim = zs[1].qlim = -1;                 // (re-anchor at the first use)
  lms_stage_any<CPLX>(d, sm, wb0, wb0 + WLa, vend, wb0, vec, &zc);
  cp_async_commit();
#pragma unroll 1
  for (int g = 1; g < LMS_AHEAD; ++g) {
    if (g < nblk) lms_stage_any<CPLX>(d, sm, wb0 + WLa + (long long)(g - 1) * DS, wb0 + WLa + (long long)g * DS, vend, wb0, vec, &zc);
    cp_async_commit();
  }
  bool first = true;
  // 32-bit offsets relative to t_begin inside the loop (a run spans < 2^31 symbols)
  const int nsym = (int)(t_end - t_begin);
  auto rel_of = [&](long long a) -> int {
    const long long r = a - t_begin;
    return r < -(1 << 30) ? -(1 << 30) : (r > (1 << 30) ? (1 << 30) : (int)r);
  };
  const int olo = rel_of(out_lo), wmr = rel_of(d.warmup), wlo = olo - d.O;
  const int smask = (int)(d.sym_cap - 1), mb0 = (int)(t_begin & (d.sym_cap - 1));
  float evn_f = 0.f, evd_f = 0.f;
  const int nblk32 = (int)nblk;
#pragma unroll 1
  for (int jb = 0; jb < nblk32; ++jb) {
    const int rb = 32 * jb;                  // block start relative to t_begin
    // KK: the z samples of block jb + AHEAD are loaded now and turned into z' at the end of this
    // block (the load latency hides behind the block's recursion; DS = 64 = 2 per lane)
    float2 zr[2];
    long long zq[2];
    if constexpr (CPLX) {
      const int jn = jb + LMS_AHEAD;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        zq[u] = wb0 + WLa + (long long)(jn - 1) * DS + lane + 32 * u;
        zr[u] = (jn < nblk && zq[u] >= 0 && zq[u] < vend) ? d.z[rmod(zq[u], d.z_cap)] : make_float2(0.f, 0.f);
      }
    }
    cp_async_wait<LMS_AHEAD - 1>();
    __syncwarp();
    const int nvalid = nsym - rb < 32 ? nsym - rb : 32;
    const bool valid = io < nvalid;
    const int mr = rb + io;                  // this lane's symbol, relative
    const T *win = sm.ring + ((DS * jb) & (LMS_RING - 1));   // contiguous window (mirror)
    // y_i = w^H u_i, u_i[k] = win[stride i + KP-1-k]
    float2 y;
    if constexpr (TILED) {
      // y_i = sum_k w_k win[i + 31 - k]; lane: i = 4r + a, k = 8q + b -> win[4r + 24 - 8q + (a + 7 - b)]
      const float *wf = reinterpret_cast<const float *>(win);
      const float4 *x4 = reinterpret_cast<const float4 *>(wf + 4 * tr + 24 - 8 * tq);
      const float4 *w4 = reinterpret_cast<const float4 *>(sm.w) + 2 * tq;
      float acc[4];
      lms_tile(x4, w4, acc, true);
      y = make_float2(lms_tile_reduce(acc, tq), 0.f);
    } else {
      const T *ub = win + stride * lane + KP - 1;
      float2 a[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      if (CPLX) {
        const float4 *w4 = reinterpret_cast<const float4 *>(sm.w);
#pragma unroll
        for (int k = 0; k < KP; k += 2) {
          const float4 ww = w4[k >> 1];                         // taps k, k+1 (broadcast)
          const float2 u0 = as_c(ub[-k]), u1 = as_c(ub[-k - 1]);
          float2 &A = a[(k >> 1) & 3];
          // A += conj(w) u as two packed FFMA2 (inner products first, as the scalar form:
          // A.x = fma(w.x, u.x, fma(w.y, u.y, A.x)), A.y = fma(w.x, u.y, fma(-w.y, u.x, A.y)))
          A = __ffma2_rn(make_float2(ww.x, ww.x), u0, __ffma2_rn(make_float2(ww.y, -ww.y), make_float2(u0.y, u0.x), A));
          A = __ffma2_rn(make_float2(ww.z, ww.z), u1, __ffma2_rn(make_float2(ww.w, -ww.w), make_float2(u1.y, u1.x), A));
        }
        if constexpr (WLIN) {   // + sum_k conj(v_k u_k): (vx ux - vy uy) - j (vx uy + vy ux)
          const float4 *v4 = reinterpret_cast<const float4 *>(sm.v);
#pragma unroll
          for (int k = 0; k < KP; k += 2) {
            const float4 vv = v4[k >> 1];
            const float2 u0 = as_c(ub[-k]), u1 = as_c(ub[-k - 1]);
            float2 &A = a[(k >> 1) & 3];
            A.x = fmaf(vv.x, u0.x, fmaf(-vv.y, u0.y, A.x));
            A.y = fmaf(-vv.x, u0.y, fmaf(-vv.y, u0.x, A.y));
            A.x = fmaf(vv.z, u1.x, fmaf(-vv.w, u1.y, A.x));
            A.y = fmaf(-vv.z, u1.y, fmaf(-vv.w, u1.x, A.y));
          }
        }
      } else {
        const float4 *w4 = reinterpret_cast<const float4 *>(sm.w);
#pragma unroll
        for (int k = 0; k < KP; k += 4) {
          const float4 ww = w4[k >> 2];                         // taps k..k+3 (broadcast)
          float2 &A = a[(k >> 2) & 3];
          A.x = fmaf(ww.x, as_c(ub[-k]).x, A.x);
          A.x = fmaf(ww.y, as_c(ub[-k - 1]).x, A.x);
          A.x = fmaf(ww.z, as_c(ub[-k - 2]).x, A.x);
          A.x = fmaf(ww.w, as_c(ub[-k - 3]).x, A.x);
        }
      }
      y = make_float2((a[0].x + a[1].x) + (a[2].x + a[3].x), CPLX ? (a[0].y + a[1].y) + (a[2].y + a[3].y) : 0.f);
    }
    float2 e, zp = y;
    int code = 0;
    if (MODE != 1) {        // training / data aided: the reference symbol drives the update
      int ri = ref0 + mr;
      while (ri >= RX_PREF) ri -= RX_PREF;
      const float2 r = __ldg(d.ref_val + ri);
      e = CPLX ? csub(r, y) : make_float2(r.x - y.x, 0.f);
    }
    if (MODE != 0) {
      float cth = 1.f, sth = 0.f;
      if (CPLX && CPR != 0 && MODE == 1) {
        float th_hat;
        if (CPR == 1) {   // Viterbi-Viterbi: 1/4 arg(-sum y^4)
          const float2 y2 = cmul(y, y);
          float2 y4 = cmul(y2, y2);
          if (!valid) y4 = make_float2(0.f, 0.f);
          const float sx = warp_sum(y4.x), sy = warp_sum(y4.y);
          th_hat = 0.25f * atan2f(-sy, -sx);
        } else {           // blind phase search: lane p scores test phases p and p + 32
          // distance in units of the level spacing 2s: u = y e^{-j phi_p} / 2s + (L - 1)/2 puts
          // the levels on the integers 0..L-1, so |z - slice(z)|^2 = (2s)^2 sum (u - clamp(rint u))^2
          // (the common factor (2s)^2 does not move the argmin)
          const float2 rsA = make_float2(rotA.x * inv2s, rotA.y * inv2s);
          const float2 rsB = make_float2(rotB.x * inv2s, rotB.y * inv2s);
          float dA = 0.f, dB = 0.f;
          sm.y[lane] = y;
          if (bps_bar) {   // helper warp scores symbols 16..31 (bps_helper)
            named_bar(bps_bar);
            bps_partial(sm.y, 0, nvalid < 16 ? nvalid : 16, rsA, rsB, L, d.Pt > 32, dA, dB);
            named_bar(bps_bar);
            const float2 pb = bps_part[lane];
            dA += pb.x;
            dB += pb.y;
          } else if (d.Pt == 32 && nvalid == 32) {
            // 32 test phases over a full block: the grid is symmetric (phi_{31-q} = -phi_q), so
            // lane l scores the pair (q, 31 - q), q = l & 15, on symbols 16 (l >> 4) .. + 15 with
            // shared products (3 instead of 4 rotation FMAs per evaluation), the two halves are
            // added by one shuffle, and lane l < 16 then holds phase l, lane l >= 16 phase 47 - l
            __syncwarp();
            const int hh = lane >> 4;
            const float cq = bq_c, sq = bq_s, cst = 0.5f * (float)(L - 1);
            const float4 *y4 = reinterpret_cast<const float4 *>(sm.y) + 8 * hh;
            // packed FP32x2 (FFMA2 / FADD2; the clamps stay scalar FMNMX): the pair (phase q,
            // phase 31 - q) of one axis shares an instruction, roundings identical to the scalar
            // form, 19 instead of 30 instructions per symbol and phase pair
            const float2 cq2 = make_float2(cq, cq), cst2 = make_float2(cst, cst);
            const float2 sqpm = make_float2(sq, -sq), sqmp = make_float2(-sq, sq);
            const float2 mg = make_float2(12582912.f, 12582912.f), mgn = make_float2(-12582912.f, -12582912.f);
            float2 pm0 = make_float2(0.f, 0.f), pm1 = make_float2(0.f, 0.f);   // (P, M) per symbol parity
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 yy = y4[i];
#pragma unroll
              for (int hsym = 0; hsym < 2; ++hsym) {
                const float yx = hsym ? yy.z : yy.x, yq = hsym ? yy.w : yy.y;
                const float2 AC = __ffma2_rn(make_float2(yx, yq), cq2, cst2);               // (A, C)
                // (sq, -sq) yq + A, (-sq, sq) yx + C: the symbol and A / C enter as broadcast operands
                const float2 ux = __ffma2_rn(sqpm, make_float2(yq, yq), make_float2(AC.x, AC.x));   // phase q / 31 - q
                const float2 uy = __ffma2_rn(sqmp, make_float2(yx, yx), make_float2(AC.y, AC.y));
#if BPS_MAGIC
                const float2 rx = __fadd2_rn(__fadd2_rn(ux, mg), mgn), ry = __fadd2_rn(__fadd2_rn(uy, mg), mgn);
#else
                const float2 rx = make_float2(rintf(ux.x), rintf(ux.y)), ry = make_float2(rintf(uy.x), rintf(uy.y));
#endif
                const float2 ex = __fadd2_rn(ux, make_float2(-fminf(fmaxf(rx.x, 0.f), Lm1), -fminf(fmaxf(rx.y, 0.f), Lm1)));
                const float2 ey = __fadd2_rn(uy, make_float2(-fminf(fmaxf(ry.x, 0.f), Lm1), -fminf(fmaxf(ry.y, 0.f), Lm1)));
                float2 &PM = hsym ? pm1 : pm0;
                PM = __ffma2_rn(ex, ex, PM);
                PM = __ffma2_rn(ey, ey, PM);
              }
            }
            float dp = pm0.x + pm1.x, dm = pm0.y + pm1.y;
            dp += __shfl_xor_sync(0xffffffffu, dp, 16);
            dm += __shfl_xor_sync(0xffffffffu, dm, 16);
            dA = hh ? dm : dp;
          } else {
            __syncwarp();
            bps_partial(sm.y, 0, nvalid, rsA, rsB, L, d.Pt > 32, dA, dB);
          }
          // argmin over the test phases, lowest p on ties (c-9 step 2): the distances are sums of
          // squares (>= +0), so their IEEE bit patterns order like the values and one warp-wide
          // integer min (redux.sync) finds the minimum; the lowest phase holding it is p
          float bd = lane < d.Pt ? dA : 3.4e38f;
          int bp = lane;
          if (lane + 32 < d.Pt && dB < bd) { bd = dB; bp = lane + 32; }
          const unsigned bits = __float_as_uint(bd);
          const unsigned mn = __reduce_min_sync(0xffffffffu, bits);
          if (d.Pt == 32 && nvalid == 32 && !bps_bar) {   // lanes hold phases 0..15, then 31..16
            const unsigned m = __ballot_sync(0xffffffffu, bits == mn);
            bp = (m & 0xFFFFu) ? __ffs(m & 0xFFFFu) - 1 : 47 - (31 - __clz(m));
          } else {
            const unsigned lo = __ballot_sync(0xffffffffu, bits == mn && bp < 32);
            bp = lo ? __ffs(lo) - 1 : __ffs(__ballot_sync(0xffffffffu, bits == mn)) - 1 + 32;
          }
          th_hat = -0.78539816339744831f + ((float)bp + 0.5f) * (1.5707963267948966f / (float)d.Pt);
        }
        if (first) theta = th_hat;
        else theta = th_hat + 1.5707963267948966f * rintf((theta - th_hat) * 0.63661977236758134f);
        // theta reduced to [-pi, pi] first: the fast sincos is accurate there (no local-memory
        // range reduction in the serial loop)
        __sincosf(theta - 6.283185307179586f * rintf(theta * 0.15915494309189535f), &sth, &cth);
        zp = cmul(y, make_float2(cth, -sth));
      }
      // slicing in the float domain (level index = clamp(floor(v / 2s + L/2)), same value as
      // slice_axis) keeps the integer conversion off the error's dependency chain
      float2 dv;
      if (CPLX) {
        const float fI = fminf(fmaxf(floorf(fmaf(zp.x, inv2s, Lh)), 0.f), Lm1);
        const float fQ = fminf(fmaxf(floorf(fmaf(zp.y, inv2s, Lh)), 0.f), Lm1);
        dv = make_float2(fmaf(fI, two_s, lvl0), fmaf(fQ, two_s, lvl0));
        if (MODE == 1) e = cmul(csub(dv, zp), make_float2(cth, sth));
        code = (int)fI | ((int)fQ << 4);
      } else if (d.thr_default) {
        const float fi = fminf(fmaxf(floorf(fmaf(zp.x, inv2s, Lh)), 0.f), Lm1);
        dv = make_float2(fmaf(fi, two_s, lvl0), 0.f);
        if (MODE == 1) e = make_float2(dv.x - zp.x, 0.f);
        code = (int)fi;
      } else {
        const int i = slice_pam(d, zp.x);
        code = i;
        dv = make_float2(level_of(i, two_s, lvl0), 0.f);
        if (MODE == 1) e = make_float2(dv.x - zp.x, 0.f);
      }
      if (valid && mr >= olo) {
        const int ix = (mb0 + mr) & smask;
        d.level[ix] = (unsigned char)code;
        d.yout[ix] = zp;
        if (mr >= wmr) {
          const float ex = dv.x - zp.x, ey = dv.y - zp.y;
          evn_f = fmaf(ex, ex, fmaf(ey, ey, evn_f));
          evd_f = fmaf(dv.x, dv.x, fmaf(dv.y, dv.y, evd_f));
        }
      } else if (valid && warm) {
        warm[mr - wlo] = (unsigned char)code;
      }
    }
    if (!valid) e = make_float2(0.f, 0.f);
    if (CPLX) reinterpret_cast<float2 *>(sm.e)[lane] = e;
    else reinterpret_cast<float *>(sm.e)[io] = e.x;
    __syncwarp();
    // gradient: lane k: g_k = sum_i u_i[k] conj(e_i); w <- w + mu g   (c-9 step 7)
    if constexpr (TILED) {
      // g_k = sum_i win[i + 31 - k] e_i; lane: k = 4r + a, i = 8q + b -> win[8q + 28 - 4r + (b + 3 - a)]
      const float *wf = reinterpret_cast<const float *>(win);
      const float4 *x4 = reinterpret_cast<const float4 *>(wf + 8 * tq + 28 - 4 * tr);
      const float4 *e4 = reinterpret_cast<const float4 *>(sm.e) + 2 * tq;
      float acc[4];
      lms_tile(x4, e4, acc, false);
      const float g = lms_tile_reduce(acc, tq);
      if (io < K) {
        wk.x = fmaf(mu, g, wk.x);
        wmax = fmaxf(wmax, wk.x * wk.x);          // (|w_k| > 1e3 <=> w_k^2 > 1e6; flagged after the loop)
      }
    } else {
      // lane = (group, tap kt): tap kt = lane % KP sums the block's symbols i in [i0, i0 + KP),
      // i0 = KP * group; the 32 / KP group partials are combined by xor shuffles, so no lane
      // works on a padding tap and every lane ends with its tap's full sum
      const int kt = lane & (KP - 1), i0 = lane & ~(KP - 1);
      const T *ug = win + KP - 1 - kt + stride * i0;
      float2 g[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      float2 hh[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};   // WLIN: sum_i u_i[k] e_i
      if (CPLX) {
        // (KP < 32) the group takes the symbol pairs t = group + (32 / KP) m, m < KP / 2, instead of
        // a contiguous run: the T/2-spaced window reads of one half-warp then cover distinct banks
        // (contiguous runs put groups 8 symbols = 16 samples apart, a 2-way conflict in ncu)
        constexpr int NGR = 32 / KP;
        const int grp = lane / KP;
        const T *ugc = win + KP - 1 - kt;
        const float4 *e4 = reinterpret_cast<const float4 *>(sm.e);
#pragma unroll
        for (int i = 0; i < KP; i += 2) {
          const int t = grp + NGR * (i >> 1);                   // symbols 2t, 2t + 1
          const float4 ee = e4[t];                              // e_2t, e_2t+1 (group broadcast)
          const float2 u0 = as_c(ugc[2 * stride * t]), u1 = as_c(ugc[2 * stride * t + stride]);
          float2 &G = g[(i >> 1) & 1];
          // G += u conj(e), packed (G.x = fma(u.x, e.x, fma(u.y, e.y, G.x)), G.y = fma(u.y, e.x, fma(-u.x, e.y, G.y)))
          G = __ffma2_rn(u0, make_float2(ee.x, ee.x), __ffma2_rn(make_float2(u0.y, -u0.x), make_float2(ee.y, ee.y), G));
          G = __ffma2_rn(u1, make_float2(ee.z, ee.z), __ffma2_rn(make_float2(u1.y, -u1.x), make_float2(ee.w, ee.w), G));
          if constexpr (WLIN) {
            float2 &H = hh[(i >> 1) & 1];
            H.x = fmaf(u0.x, ee.x, fmaf(-u0.y, ee.y, H.x));
            H.y = fmaf(u0.x, ee.y, fmaf(u0.y, ee.x, H.y));
            H.x = fmaf(u1.x, ee.z, fmaf(-u1.y, ee.w, H.x));
            H.y = fmaf(u1.x, ee.w, fmaf(u1.y, ee.z, H.y));
          }
        }
      } else {
        const float4 *e4 = reinterpret_cast<const float4 *>(sm.e) + (i0 >> 2);
#pragma unroll
        for (int i = 0; i < KP; i += 4) {
          const float4 ee = e4[i >> 2];
          float2 &G = g[(i >> 2) & 1];
          G.x = fmaf(as_c(ug[i]).x, ee.x, G.x);
          G.x = fmaf(as_c(ug[i + 1]).x, ee.y, G.x);
          G.x = fmaf(as_c(ug[i + 2]).x, ee.z, G.x);
          G.x = fmaf(as_c(ug[i + 3]).x, ee.w, G.x);
        }
      }
      float gx = g[0].x + g[1].x, gy = g[0].y + g[1].y;
      float hx = hh[0].x + hh[1].x, hy = hh[0].y + hh[1].y;
#pragma unroll
      for (int o = KP; o < 32; o <<= 1) {
        gx += __shfl_xor_sync(0xffffffffu, gx, o);
        if (CPLX) gy += __shfl_xor_sync(0xffffffffu, gy, o);
        if (WLIN) {
          hx += __shfl_xor_sync(0xffffffffu, hx, o);
          hy += __shfl_xor_sync(0xffffffffu, hy, o);
        }
      }
      if constexpr (WLIN) {   // v_k <- v_k + mu conj(h_k)
        if (lane < K) {
          vk.x = fmaf(mu, hx, vk.x);
          vk.y = fmaf(-mu, hy, vk.y);
        }
        reinterpret_cast<float2 *>(sm.v)[lane] = vk;
      }
      if (lane < K) {
        wk.x = fmaf(mu, gx, wk.x);
        if (CPLX) wk.y = fmaf(mu, gy, wk.y);
        // divergence (reading R-DIV): any single tap beyond 1e3 at any block - tracked
        // as the running max of |w_k|^2 (flagged after the loop), the full norm at the end
        wmax = fmaxf(wmax, cabs2(wk));
      }
    }
    if (CPLX) reinterpret_cast<float2 *>(sm.w)[lane] = wk;
    else reinterpret_cast<float *>(sm.w)[io] = wk.x;
    __syncwarp();
    // stage the new samples of block jb + AHEAD (the slots of block jb are no longer read)
    const int jn = jb + LMS_AHEAD;
    if constexpr (!CPLX) {
      if (fast) {
        if (jn < nblk && lane < 8) {
          const int rel = WLa + (jn - 1) * DS + 4 * lane;
          const int slot = rel & (LMS_RING - 1);
          const float *src = d.uhat + ((gbase + rel) & gmask);
          const unsigned sa = (unsigned)__cvta_generic_to_shared(&sm.ring[slot]);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
          if (slot < 64) {
            const unsigned sb = (unsigned)__cvta_generic_to_shared(&sm.ring[slot + LMS_RING]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb), "l"(src));
          }
        }
      } else if (jn < nblk) {
        lms_stage_any<CPLX>(d, sm, wb0 + WLa + (long long)(jn - 1) * DS, wb0 + WLa + (long long)jn * DS, vend, wb0, vec);
      }
    } else if (jn < nblk) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float2 v = zp_step(d, zr[u], zq[u], zs[u], vend);
        const int slot = (int)((zq[u] - wb0) & (LMS_RING - 1));
        sm.ring[slot] = v;
        sm.ring[slot + LMS_RING] = v;
      }
    }
    cp_async_commit();
    first = false;
  }
  cp_async_wait<0>();
  evn += (double)evn_f;
  evd += (double)evd_f;
  if (TILED) wk.x = reinterpret_cast<const float *>(sm.w)[lane];   // back to lane = tap order
  const float nrm = warp_sum(lane < K ? cabs2(wk) : 0.f);
  if (__any_sync(0xffffffffu, wmax > 1e6f) && lane == 0) set_flag(d.st, RX_FLAG_DIVERGE);
  if (lane == 0 && nrm > 1e6f) set_flag(d.st, RX_FLAG_DIVERGE);
  return theta;
}

// ------------------------------------------------------------------ training (1 warp)
template <bool CPLX, int KP, bool WLIN = false>
__global__ void __launch_bounds__(32) k_lms_train(RxDev d, int flush) {
  __shared__ LmsSmemT<CPLX> sm;
  DevState *st = d.st;
  if (!st->synced || st->trained) return;
  const int lane = threadIdx.x;
  const int K = d.K, c = K >> 1, stride = CPLX ? 2 : 1;
  const long long vend = st->v_lms;
  const long long last = (long long)stride * (d.m0 + d.T_train - 1) + (CPLX ? st->sync_phase : 0) + c;
  if (last >= vend && !flush) return;
  float2 wk = make_float2(lane == c ? 1.f : 0.f, 0.f);    // centre spike ...
  if (d.has_winit) wk = lane < K ? d.w_init[lane] : make_float2(0.f, 0.f);   // ... or rx_set_taps
  double en = 0.0, ed = 0.0;
  float2 vk = make_float2(0.f, 0.f);                      // widely-linear branch starts at 0
  lms_run<CPLX, 0, 0, KP, WLIN>(d, sm, d.m0, d.m0 + d.T_train, 0, wk, vk, nullptr, en, ed, vend);
  if (lane < K) d.w_train[lane] = wk;
  if (WLIN && lane < K) d.v_train[lane] = vk;
  __threadfence();
  if (lane == 0) { st->trained = 1; d.hm->trained = 1; }
}

// PAM labels and bit errors of output symbols [lo, hi) from the level ring (written by this warp)
__device__ __forceinline__ void pam_finalise(const RxDev &d, long long lo, long long hi, unsigned char *labels,
                                             long long lab_cap, int &err, int &cnt) {
  const int lane = threadIdx.x & 31;
  const DevState *st = d.st;
  const int r0 = (int)(((st->sync_offset + lo - d.m0) % RX_PREF + RX_PREF) % RX_PREF);
  const bool vec = labels && (((unsigned long long)labels | (unsigned long long)lab_cap | (unsigned long long)lo) & 15) == 0;
  const long long n = hi - lo;
  for (long long v = 16LL * lane; v < n; v += 512) {
    const long long m0v = lo + v;
    const int nv = n - v < 16 ? (int)(n - v) : 16;
    unsigned char code[16];
    if (nv == 16 && (m0v & 15) == 0) {
      const uint4 q = *reinterpret_cast<const uint4 *>(d.level + rmod(m0v, d.sym_cap));
      const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) code[j] = (unsigned char)(w[j >> 2] >> (8 * (j & 3)));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) code[j] = j < nv ? d.level[rmod(m0v + j, d.sym_cap)] : 0;
    }
    unsigned char lab[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) lab[j] = (unsigned char)(code[j] ^ (code[j] >> 1));
    if (labels) {
      const long long li0 = m0v % lab_cap;
      if (vec && nv == 16) {
        unsigned w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j >> 2] |= (unsigned)lab[j] << (8 * (j & 3));
        *reinterpret_cast<uint4 *>(labels + li0) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        long long li = li0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < nv) labels[li] = lab[j];
          if (++li == lab_cap) li = 0;
        }
      }
    }
    int ri = r0 + (int)v % RX_PREF;    // (v < 2^31: 32-bit modulo)
    if (ri >= RX_PREF) ri -= RX_PREF;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < nv && m0v + j >= d.warmup) {
        err += __popc((int)lab[j] ^ (int)__ldg(d.ref_lab + ri));
        ++cnt;
      }
      if (++ri == RX_PREF) ri = 0;
    }
  }
}

// BPS helper warp (KK, CPR = BPS): per block, waits for the block's y, scores symbols 16..31
// for every test phase and hands the partial sums to the segment's LMS warp (c-9 step 2)
__device__ void bps_helper(const RxDev &d, const float2 *ys, long long t_begin, long long t_end, int bar,
                           float2 *part) {
  const int lane = threadIdx.x & 31, L = d.L;
  const float two_s = 2.0f * d.qam_sc, inv2s = 1.0f / two_s;
  float2 rotA = make_float2(1.f, 0.f), rotB = make_float2(1.f, 0.f);
  if (lane < d.Pt) rotA = __ldg(d.bps_rot + lane);
  if (lane + 32 < d.Pt) rotB = __ldg(d.bps_rot + lane + 32);
  const float2 rsA = make_float2(rotA.x * inv2s, rotA.y * inv2s);
  const float2 rsB = make_float2(rotB.x * inv2s, rotB.y * inv2s);
  const long long nblk = (t_end - t_begin + 31) / 32;
#pragma unroll 1
  for (long long jb = 0; jb < nblk; ++jb) {
    const long long t = t_begin + 32 * jb;
    const int nvalid = (int)((t_end - t) < 32 ? (t_end - t) : 32);
    named_bar(bar);
    float dA = 0.f, dB = 0.f;
    if (nvalid > 16) bps_partial(ys, 16, nvalid, rsA, rsB, L, d.Pt > 32, dA, dB);
    part[lane] = make_float2(dA, dB);
    named_bar(bar);
  }
}

// ------------------------------------------------------------------ segments (1 warp each)
// Segment s outputs [sS, min((s+1)S, m_end)), recursion starts O symbols early (c-9).
// warps per CTA of k_lms_seg: KK 1 (finest CTA balance over the SMs for its 2048-segment rounds:
// measured 4 -> 1 warps, C4 equaliser 0.89 -> 0.72 ms per step), PAM 4 (its shorter rounds of
// 4096 segments: 4 -> 1 measured 0.081 -> 0.090 ms per C2 step)
#ifndef LMS_SPC_KK
#define LMS_SPC_KK 1
#endif
#ifndef LMS_SPC_PAM
#define LMS_SPC_PAM 4
#endif
#define LMS_SPC_OF(CPLX) ((CPLX) ? LMS_SPC_KK : LMS_SPC_PAM)
// minimum resident CTAs per SM the register allocation must allow (0: the compiler default)
#ifndef LMS_MINB_KK
#define LMS_MINB_KK 0
#endif
#define LMS_MINB_OF(CPLX) ((CPLX) ? LMS_MINB_KK : 0)
#ifndef LMS_PAIR
#define LMS_PAIR 1          // BPS segments: 2 = a helper warp scores half of each block's symbols
#endif
template <bool CPLX, int CPR, int KP, bool WLIN = false, int MODE = 1>
__global__ void __launch_bounds__(32 * LMS_SPC_OF(CPLX), LMS_MINB_OF(CPLX)) k_lms_seg(RxDev d, int flush, int nseg, unsigned char *labels,
                                                 long long lab_cap) {
  // BPS segments run on a warp pair (LMS warp + BPS helper), others on one warp
  constexpr int PAIR = (CPR == 2) ? LMS_PAIR : 1, SPC = LMS_SPC_OF(CPLX) / PAIR;   // PAIR = 2: BPS helper warp
  static_assert(SPC >= 1 && SPC * PAIR == LMS_SPC_OF(CPLX), "LMS_SPC_* must be a multiple of LMS_PAIR");
  __shared__ LmsSmemT<CPLX> sm[SPC];
  __shared__ float2 bps_part[SPC][32];
  DevState *st = d.st;
  if (!st->trained) return;
  const int slot = (threadIdx.x >> 5) / PAIR, role = (threadIdx.x >> 5) % PAIR, lane = threadIdx.x & 31;
  const int warp = slot;
  const long long s = st->seg_next + (long long)blockIdx.x * SPC + slot;
  if (blockIdx.x * SPC + slot >= nseg) return;
  if (d.seg_done[rmod(s, d.seg_cap)] == s + 1) return;
  const long long S = d.S;
  const long long lo = s * S;
  const long long me = st->m_end;
  if (me >= 0 && lo >= me) return;
  const long long hi = seg_end_of(d, s);
  const int K = d.K, c = K >> 1, stride = CPLX ? 2 : 1;
  const long long vend = st->v_lms;
  if (me < 0) {   // streaming: all taps of the last symbol must be available
    const long long lastidx = (long long)stride * (hi - 1) + (CPLX ? st->sync_phase : 0) + c;
    if (lastidx >= vend) return;
  }
  // seed: W_train for e < D, else the mean canonical taps of epoch e - D (c-9 'Seed')
  const long long e = lo / d.E_sym;
  // widely linear: the v-branch of every decision-directed segment starts at 0 (reading R-WL:
  // its value depends on the absolute carrier phase during the segment, v/w = -e^{-2j phi} b*/a)
  float2 wk = make_float2(0.f, 0.f), vk = make_float2(0.f, 0.f);
  if (e < d.D) {
    if (lane < K) wk = d.w_train[lane];
  } else {
    if (d.seed_ready[rmod(e, d.seed_cap)] != e + 1) return;
    if (lane < K) wk = d.seed[rmod(e, d.seed_cap) * RX_MAX_K + lane];
  }
  long long t0 = lo - d.O;
  if (t0 < 0) t0 = 0;
  double en = 0.0, ed = 0.0;
  unsigned char *warm = d.O > 0 ? d.seg_warm + rmod(s, d.seg_cap) * d.O : nullptr;
  if (PAIR == 2 && role == 1) {
    bps_helper(d, sm[warp].y, t0, hi, 1 + slot, bps_part[slot]);
    return;
  }
  const float th = lms_run<CPLX, CPR, MODE, KP, WLIN>(d, sm[warp], t0, hi, lo, wk, vk, warm, en, ed, vend,
                                                   PAIR == 2 ? 1 + slot : 0, bps_part[slot]);
  en = warp_sum_d(en);
  ed = warp_sum_d(ed);
  const long long si = rmod(s, d.seg_cap);
  if (lane < K) d.seg_w[si * RX_MAX_K + lane] = wk;
  if (!CPLX) {
    // PAM finalises its own symbols (R_s = 0): Gray labels + reference comparison (H10/H25)
    // over the segment's level codes, 16 per lane-step, off the serial recursion
    __syncwarp();
    int er = 0, ct = 0;
    pam_finalise(d, lo, hi, labels, lab_cap, er, ct);
    er = __reduce_add_sync(0xffffffffu, (unsigned)er);
    ct = __reduce_add_sync(0xffffffffu, (unsigned)ct);
    if (lane == 0) { d.seg_err[2 * si] = er; d.seg_err[2 * si + 1] = ct; }
  }
  if (lane == 0) {
    d.seg_theta[si] = th;
    d.seg_evm[2 * si] = en;
    d.seg_evm[2 * si + 1] = ed;
    __threadfence();
    d.seg_done[si] = (int)(s + 1);
  }
}

// ------------------------------------------------------------------ per-symbol WL DDLMS (NEXT-1)
// The paper's KK equaliser proper: a K-tap (4 in the paper) widely-linear TD DDLMS
// updated after EVERY symbol (B = 1), which also does the symbol-phase recovery (no separate
// CPR; rx_config.lms_mode = 2, DESIGN reading R-DDLMS). The recursion is serial per symbol, so
// each thread runs one segment's recursion with its taps, window and error in registers (the
// paper's "serial in nature" kernel: few processing units, long time); the segment-parallel
// structure of c-9 (seeds, warm-up, anchored quadrants) supplies the parallelism.
//   y_m = sum_k conj(w_k) u_m[k] (+ conj(v_k) conj(u_m[k])),  u_m[k] = z'[2m + h* + c - k]
//   MODE 1: d_m = slice(y_m), e_m = d_m - y_m (reference r_m - y_m on the warm-up symbols, the
//           seed first rotated onto the reference: DESIGN reading R-DDLMS);
//   MODE 0 (training): e_m = r_m - y_m
//   w_k += mu u_m[k] conj(e_m);  v_k += mu conj(u_m[k]) conj(e_m)
#define SYM_PF 8            // symbols of z prefetched ahead of the recursion (registers)
#define SYM_INIT 64         // symbols of a DDLMS segment's seed rotation onto the reference (R-DDLMS)
template <int KP, bool WLIN, int MODE>
__device__ void lms_sym_run(const RxDev &d, long long t_begin, long long t_end, long long out_lo, float2 (&w)[KP],
                            float2 (&v)[KP], unsigned char *warm, double &evn, double &evd, long long vend) {
  const int K = d.K, c = K >> 1, h = d.st->sync_phase;
  const float mu = d.mu;
  const int L = d.L;
  const float two_s = 2.0f * d.qam_sc, lvl0 = -(float)(L - 1) * d.qam_sc, inv2s = 1.0f / two_s;
  const float Lh = 0.5f * (float)L, Lm1 = (float)(L - 1);
  // reference index of t_begin: training (MODE 0) adapts on it throughout; DD segments (MODE 1)
  // on their warm-up symbols m < out_lo (R-DDLMS)
  int ri = (int)(((d.st->sync_offset + t_begin - d.m0) % RX_PREF + RX_PREF) % RX_PREF);
  ZpCache zc;
  zc.beta = -1;
  // window u_{t_begin}[k] = z'[2 t_begin + h + c - k]
  float2 U[KP];
  const long long qb = 2 * t_begin + h + c;
#pragma unroll
  for (int k = 0; k < KP; ++k) U[k] = zp_value(d, qb - k, vend, zc);
  if (MODE == 1) {
    // the seed rotated onto the reference: c0 = sum_m y_m conj(r_m) over the first SYM_INIT
    // symbols (y from the seed taps, v = 0), w <- w c0 / |c0| (R-DDLMS)
    float2 c0 = make_float2(0.f, 0.f);
    int rj = ri;
    for (long long m = t_begin; m < t_begin + SYM_INIT && m < t_end; ++m) {
      const long long q = 2 * m + h + c;
      float2 y = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const float2 u = zp_value(d, q - k, vend, zc);
        y.x = fmaf(w[k].x, u.x, fmaf(w[k].y, u.y, y.x));
        y.y = fmaf(w[k].x, u.y, fmaf(-w[k].y, u.x, y.y));
      }
      c0 = cadd(c0, cmulc(y, __ldg(d.ref_val + rj)));
      if (++rj == RX_PREF) rj = 0;
    }
    const float a = sqrtf(cabs2(c0));
    if (a > 0.f) {
      const float2 rot = make_float2(c0.x / a, c0.y / a);
#pragma unroll
      for (int k = 0; k < KP; ++k) w[k] = cmul(w[k], rot);
    }
  }
  // raw z of the two samples entering at symbol m + 1 + i (i < SYM_PF), loaded SYM_PF ahead
  float2 pf[SYM_PF][2];
#pragma unroll
  for (int i = 0; i < SYM_PF; ++i) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const long long q = qb + 2 * (i + 1) - 1 + e;
      pf[i][e] = (q >= 0 && q < vend) ? d.z[rmod(q, d.z_cap)] : make_float2(0.f, 0.f);
    }
  }
  float evn_f = 0.f, evd_f = 0.f;
  const long long n = t_end - t_begin;
  for (long long m0 = 0; m0 < n; m0 += SYM_PF) {
#pragma unroll
    for (int i = 0; i < SYM_PF; ++i) {
      const long long rel = m0 + i;
      if (rel < n) {
        const long long m = t_begin + rel;
        float2 y = make_float2(0.f, 0.f), y2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          float2 &A = (k & 1) ? y2 : y;
          A.x = fmaf(w[k].x, U[k].x, fmaf(w[k].y, U[k].y, A.x));
          A.y = fmaf(w[k].x, U[k].y, fmaf(-w[k].y, U[k].x, A.y));
          if (WLIN) {
            A.x = fmaf(v[k].x, U[k].x, fmaf(-v[k].y, U[k].y, A.x));
            A.y = fmaf(-v[k].x, U[k].y, fmaf(-v[k].y, U[k].x, A.y));
          }
        }
        y = cadd(y, y2);
        const float fI = fminf(fmaxf(floorf(fmaf(y.x, inv2s, Lh)), 0.f), Lm1);
        const float fQ = fminf(fmaxf(floorf(fmaf(y.y, inv2s, Lh)), 0.f), Lm1);
        const float2 dv = make_float2(fmaf(fI, two_s, lvl0), fmaf(fQ, two_s, lvl0));
        float2 e;
        const float2 rv = __ldg(d.ref_val + ri);
        if (++ri == RX_PREF) ri = 0;
        if (MODE == 0) {
          e = csub(rv, y);
        } else {
          e = m < out_lo ? csub(rv, y) : csub(dv, y);       // reference-aided warm-up (R-DDLMS)
          const int code = (int)fI | ((int)fQ << 4);
          if (m >= out_lo) {
            const long long ix = rmod(m, d.sym_cap);
            d.level[ix] = (unsigned char)code;
            d.yout[ix] = y;
            if (m >= d.warmup) {                            // decision-referenced: e = d - y here
              evn_f = fmaf(e.x, e.x, fmaf(e.y, e.y, evn_f));
              evd_f = fmaf(dv.x, dv.x, fmaf(dv.y, dv.y, evd_f));
            }
          } else if (warm) {
            warm[m - (out_lo - d.O)] = (unsigned char)code;
          }
        }
        // w_k += mu u_k conj(e); v_k += mu conj(u_k) conj(e)
        const float ex = mu * e.x, ey = mu * e.y;
        float nrm = 0.f;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          if (k < K) {
            w[k].x = fmaf(U[k].x, ex, fmaf(U[k].y, ey, w[k].x));
            w[k].y = fmaf(U[k].y, ex, fmaf(-U[k].x, ey, w[k].y));
            if (WLIN) {
              v[k].x = fmaf(U[k].x, ex, fmaf(-U[k].y, ey, v[k].x));
              v[k].y = fmaf(-U[k].y, ex, fmaf(-U[k].x, ey, v[k].y));
            }
            nrm = fmaxf(nrm, cabs2(w[k]));
          }
        }
        if (nrm > 1e6f) set_flag(d.st, RX_FLAG_DIVERGE);   // R-DIV: any tap beyond 1e3
        // slide the window by one symbol (two T/2 samples enter) and refill the prefetch slot
#pragma unroll
        for (int k = KP - 1; k >= 2; --k) U[k] = U[k - 2];
        const long long qn = qb + 2 * (rel + 1);
        U[1] = zp_rotate_or_zero(d, pf[i][0], qn - 1, vend, zc);
        if (KP > 0) U[0] = zp_rotate_or_zero(d, pf[i][1], qn, vend, zc);
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const long long q = qn + 2 * SYM_PF - 1 + e2;
          pf[i][e2] = (q >= 0 && q < vend) ? d.z[rmod(q, d.z_cap)] : make_float2(0.f, 0.f);
        }
      }
    }
  }
  evn += (double)evn_f;
  evd += (double)evd_f;
}

template <int KP, bool WLIN>
__global__ void __launch_bounds__(32) k_lms_train_sym(RxDev d, int flush) {
  DevState *st = d.st;
  if (!st->synced || st->trained || threadIdx.x != 0) return;
  const int K = d.K, c = K >> 1;
  const long long vend = st->v_lms;
  const long long last = 2 * (d.m0 + d.T_train - 1) + st->sync_phase + c;
  if (last >= vend && !flush) return;
  float2 w[KP], v[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    w[k] = make_float2(k == c ? 1.f : 0.f, 0.f);                       // centre spike ...
    if (d.has_winit) w[k] = k < K ? d.w_init[k] : make_float2(0.f, 0.f); // ... or rx_set_taps
    v[k] = make_float2(0.f, 0.f);
  }
  double en = 0.0, ed = 0.0;
  lms_sym_run<KP, WLIN, 0>(d, d.m0, d.m0 + d.T_train, 0, w, v, nullptr, en, ed, vend);
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (k < K) {
      d.w_train[k] = w[k];
      if (WLIN) d.v_train[k] = v[k];
    }
  }
  __threadfence();
  st->trained = 1;
  d.hm->trained = 1;
}

// one thread per segment (32 per CTA); outputs, counters and taps as k_lms_seg's
template <int KP, bool WLIN>
__global__ void __launch_bounds__(32) k_lms_sym(RxDev d, int flush, int nseg, unsigned char *labels, long long lab_cap) {
  DevState *st = d.st;
  if (!st->trained) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseg) return;
  const long long s = st->seg_next + t;
  const long long si = rmod(s, d.seg_cap);
  if (d.seg_done[si] == s + 1) return;
  const long long lo = s * (long long)d.S;
  const long long me = st->m_end;
  if (me >= 0 && lo >= me) return;
  const long long hi = seg_end_of(d, s);
  const int K = d.K, c = K >> 1;
  const long long vend = st->v_lms;
  if (me < 0 && 2 * (hi - 1) + st->sync_phase + c >= vend) return;   // streaming: data not there yet
  const long long e = lo / d.E_sym;
  float2 w[KP], v[KP];
  if (e >= d.D && d.seed_ready[rmod(e, d.seed_cap)] != e + 1) return;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    w[k] = k < K ? (e < d.D ? d.w_train[k] : d.seed[rmod(e, d.seed_cap) * RX_MAX_K + k]) : make_float2(0.f, 0.f);
    v[k] = make_float2(0.f, 0.f);                  // R-WL: every DD segment's v-branch from 0
  }
  long long t0 = lo - d.O;
  if (t0 < 0) t0 = 0;
  double en = 0.0, ed = 0.0;
  unsigned char *warm = d.O > 0 ? d.seg_warm + si * d.O : nullptr;
  lms_sym_run<KP, WLIN, 1>(d, t0, hi, lo, w, v, warm, en, ed, vend);
  float nrm = 0.f;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (k < K) {
      d.seg_w[si * RX_MAX_K + k] = w[k];
      nrm += cabs2(w[k]);
    }
  }
  if (nrm > 1e6f) set_flag(st, RX_FLAG_DIVERGE);
  d.seg_theta[si] = 0.f;
  d.seg_evm[2 * si] = en;
  d.seg_evm[2 * si + 1] = ed;
  __threadfence();
  d.seg_done[si] = (int)(s + 1);
}

// ------------------------------------------------------------------ H22 stitching
// r_s = argmax_r #{m in warm-up overlap : d^(s) j^r = d^(s-1)}, lowest r on ties (c-9)
__global__ void __launch_bounds__(256) k_lms_stitch(RxDev d, int nseg) {
  __shared__ int cnt[4];
  const long long s = d.st->seg_next + blockIdx.x;
  if (blockIdx.x >= nseg) return;
  const long long si = rmod(s, d.seg_cap);
  if (d.seg_done[si] != s + 1 || d.seg_stitched[si] == s + 1) return;
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  if (d.anchor_each) {
    // R-ANCHOR2: R_s = argmax_r #{m in the segment's first 256 outputs (from m0 for s0) :
    // d_m j^r = ref_m}, lowest r on ties; stored as the absolute quadrant (no prefix chain)
    __syncthreads();
    const long long a0 = (s == d.m0 / d.S) ? d.m0 : s * (long long)d.S;
    long long a1 = a0 + 256;
    const long long hi = seg_end_of(d, s);
    if (a1 > hi) a1 = hi;
    int c4[4] = {0, 0, 0, 0};
    for (long long m = a0 + threadIdx.x; m < a1; m += blockDim.x) {
      const int cur = d.level[rmod(m, d.sym_cap)];
      const long long ri = ((d.st->sync_offset + m - d.m0) % RX_PREF + RX_PREF) % RX_PREF;
      const int ref = d.ref_idx[ri];
#pragma unroll
      for (int r = 0; r < 4; ++r) c4[r] += (qam_rot(cur, r, d.L) == ref);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int v = __reduce_add_sync(0xffffffffu, c4[r]);
      if ((threadIdx.x & 31) == 0) atomicAdd(&cnt[r], v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int best = 0;
      for (int r = 1; r < 4; ++r) if (cnt[r] > cnt[best]) best = r;
      d.seg_r[si] = best;
      __threadfence();
      d.seg_stitched[si] = (int)(s + 1);
    }
    return;
  }
  if (s > 0 && d.seg_done[rmod(s - 1, d.seg_cap)] != s) return;
  __syncthreads();
  const bool doit = (d.family == 1) && d.O > 0 && s > 0;
  if (doit) {
    int c4[4] = {0, 0, 0, 0};
    const long long base = s * (long long)d.S - d.O;
    for (int x = threadIdx.x; x < d.O; x += blockDim.x) {
      const int cur = d.seg_warm[si * d.O + x];
      const int prev = d.level[rmod(base + x, d.sym_cap)];
#pragma unroll
      for (int r = 0; r < 4; ++r) c4[r] += (qam_rot(cur, r, d.L) == prev);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int v = __reduce_add_sync(0xffffffffu, c4[r]);
      if ((threadIdx.x & 31) == 0) atomicAdd(&cnt[r], v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int best = 0;
    for (int r = 1; r < 4; ++r) if (cnt[r] > cnt[best]) best = r;
    d.seg_r[si] = doit ? best : 0;
    __threadfence();
    d.seg_stitched[si] = (int)(s + 1);
  }
}

// Counters in fixed order (one CTA of 1024 threads) over finalised segments [lo, hi)
__device__ __forceinline__ void lms_add_counters(const RxDev &d, long long lo, long long hi) {
  __shared__ double sh[32], sh2[32];
  __shared__ long long shl[32], shl2[32];
  DevState *st = d.st;
  const int t = threadIdx.x;
  double en = 0.0, ed = 0.0;
  long long er = 0, ct = 0;
  for (long long s0 = lo + t; s0 < hi; s0 += 4 * (long long)blockDim.x) {   // 4 segments in flight
    double2 ev[4];
    longlong2 eg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long s = s0 + u * (long long)blockDim.x;
      const long long si = rmod(s, d.seg_cap);
      ev[u] = s < hi ? reinterpret_cast<const double2 *>(d.seg_evm)[si] : make_double2(0.0, 0.0);
      eg[u] = s < hi ? reinterpret_cast<const longlong2 *>(d.seg_err)[si] : make_longlong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { en += ev[u].x; ed += ev[u].y; er += eg[u].x; ct += eg[u].y; }
  }
  if (d.q_segs > 0) {
    // Q-trace windows. Segments are finalised once each, in increasing order, by this
    // single CTA: a window's ring slot is cleared in the round that finalises its first segment,
    // then segments with the same window combine per warp, one atomic each
    for (long long w = (lo + d.q_segs - 1) / d.q_segs + t; w * d.q_segs < hi; w += blockDim.x) {
      unsigned long long *q = d.q_win + 2 * (w & (RX_Q_WINDOWS - 1));
      q[0] = 0ull;
      q[1] = 0ull;
    }
    __syncthreads();
    for (long long b = lo; b < hi; b += blockDim.x) {
      const long long s = b + t;
      const unsigned act = __ballot_sync(0xffffffffu, s < hi);
      if (s < hi) {
        const long long w = s / d.q_segs;
        const longlong2 eg = reinterpret_cast<const longlong2 *>(d.seg_err)[rmod(s, d.seg_cap)];
        const unsigned m = __match_any_sync(act, w);
        const unsigned e = __reduce_add_sync(m, (unsigned)eg.x), c = __reduce_add_sync(m, (unsigned)eg.y);
        if ((t & 31) == __ffs(m) - 1) {
          unsigned long long *q = d.q_win + 2 * (w & (RX_Q_WINDOWS - 1));
          atomicAdd(q, (unsigned long long)e);
          atomicAdd(q + 1, (unsigned long long)c);
        }
      }
    }
  }
  en = warp_sum_d(en);
  ed = warp_sum_d(ed);
  for (int o = 16; o > 0; o >>= 1) {
    er += __shfl_xor_sync(0xffffffffu, er, o);
    ct += __shfl_xor_sync(0xffffffffu, ct, o);
  }
  if ((t & 31) == 0) { sh[t >> 5] = en; sh2[t >> 5] = ed; shl[t >> 5] = er; shl2[t >> 5] = ct; }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    long long x = 0, y = 0;
    for (int w = 0; w < 32; ++w) { a += sh[w]; b += sh2[w]; x += shl[w]; y += shl2[w]; }
    st->evm_num += a;
    st->evm_den += b;
    st->bit_errors += x;
    st->symbols_counted += y;
    st->bits += y * d.kbits;
    long long so = hi * (long long)d.S;
    if (st->m_end >= 0 && so > st->m_end) so = st->m_end;
    if (hi > lo) st->symbols_out = so;
  }
}

// ------------------------------------------------------------------ R_s prefix + anchor
// R_s = (A + sum_{i<=s} r_i) mod 4 with A fixed by anchoring the segment containing m0 to
// the known reference over [m0, m0 + 256) (c-9 'Stitching').
__global__ void __launch_bounds__(1024) k_lms_prefix(RxDev d, int flush, int maxn) {
  pdl_wait();                 // the previous kernel of the round (programmatic dependent launch)
  __shared__ int firstbad;
  __shared__ int acnt[4];
  DevState *st = d.st;
  const long long base = st->seg_next;
  const int t = threadIdx.x;
  if (t == 0) firstbad = maxn;
  if (t < 4) acnt[t] = 0;
  __syncthreads();
  // PAM: no stitching (R_s = 0); anchored QAM: R_s is taken by k_lms_final itself (R-ANCHOR2)
  const int *ready = (d.family == 1 && !d.anchor_each) ? d.seg_stitched : d.seg_done;
  for (int i0 = t; i0 < maxn; i0 += 4 * blockDim.x) {          // 4 loads in flight per thread
    int v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < maxn ? ready[rmod(base + i, d.seg_cap)] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < maxn && v[u] != base + i + 1) atomicMin(&firstbad, i);
    }
  }
  __syncthreads();
  int n = firstbad;
  // anchor
  const long long s0 = d.m0 / d.S;
  __shared__ int A_sh, known_sh;
  if (t == 0) {
    A_sh = st->anchor_A;
    known_sh = st->anchor_known;
    if (!known_sh && d.anchor_each) { A_sh = 0; known_sh = 1; }   // R-ANCHOR2: every R_s is absolute
  }
  __syncthreads();
  const int known0 = known_sh;        // block-uniform copy: thread 0 may update known_sh below
  __syncthreads();
  if (!known0) {
    const long long me = st->m_end;
    const bool s0_exists = !(me >= 0 && s0 * (long long)d.S >= me);
    if (d.family == 0) {
      if (t == 0) { A_sh = 0; known_sh = 1; }
    } else if (!s0_exists) {
      if (t == 0) { A_sh = 0; known_sh = 1; }
    } else if (s0 < base + n) {
      const long long hi0 = seg_end_of(d, s0);
      long long mend = d.m0 + 256;
      if (mend > hi0) mend = hi0;
      int c4[4] = {0, 0, 0, 0};
      for (long long m = d.m0 + t; m < mend; m += blockDim.x) {
        const int cur = d.level[rmod(m, d.sym_cap)];
        const long long ri = ((st->sync_offset + m - d.m0) % RX_PREF + RX_PREF) % RX_PREF;
        const int ref = d.ref_idx[ri];
#pragma unroll
        for (int r = 0; r < 4; ++r) c4[r] += (qam_rot(cur, r, d.L) == ref);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int v = __reduce_add_sync(0xffffffffu, c4[r]);
        if ((t & 31) == 0) atomicAdd(&acnt[r], v);
      }
      __syncthreads();
      if (t == 0) {
        int best = 0;
        for (int r = 1; r < 4; ++r) if (acnt[r] > acnt[best]) best = r;
        // P_{s0} = r_prefix + sum_{i=base}^{s0} r_i
        int p = (int)(st->r_prefix & 3);
        for (long long s = base; s <= s0; ++s) p += (s == 0) ? 0 : d.seg_r[rmod(s, d.seg_cap)];
        A_sh = ((best - p) % 4 + 4) % 4;
        known_sh = 1;
      }
    }
  }
  __syncthreads();
  if (!known_sh) n = 0;
  // prefix of r over [base, base + n) in chunks of 1024 (QAM; PAM has R_s = 0): warp shuffle
  // scans + one scan of the 32 warp totals
  int carry = (int)(st->r_prefix & 3);
  if (d.family == 1 && d.anchor_each) {
    // (R_s = r_s, both written by k_lms_final)
  } else if (d.family == 1) {
    __shared__ int wsum[32];
    const int lane = t & 31, warp = t >> 5;
    for (int c0 = 0; c0 < n; c0 += 1024) {
      const long long s = base + c0 + t;
      int x = 0;
      if (c0 + t < n && s > 0) x = d.seg_r[rmod(s, d.seg_cap)];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int v = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += y;
        }
        wsum[lane] = v;
      }
      __syncthreads();
      const int incl = x + (warp > 0 ? wsum[warp - 1] : 0);
      if (c0 + t < n) d.seg_R[rmod(s, d.seg_cap)] = (A_sh + carry + incl) & 3;
      const int tot = wsum[31];
      __syncthreads();
      carry = (carry + tot) & 3;
    }
  } else {
    lms_add_counters(d, base, base + n);   // PAM: the segments counted their own errors
  }
  if (t == 0) {
    st->anchor_known = known_sh;
    st->anchor_A = A_sh;
    st->fin_lo = base;
    st->fin_hi = base + n;
    st->seg_next = base + n;
    st->r_prefix = carry;
    d.hm->seg_next = base + n;
  }
}

// ------------------------------------------------------------------ H10/H23/H25 finalise
// Final labels (rotated by j^{R_s}), reference comparison, per-segment error counts,
// canonical absolute-frame taps w~_s = w e^{j theta} j^{-R_s} (c-9 'Seed').
#ifndef LMS_FINAL_T
#define LMS_FINAL_T 64      // threads per segment CTA of k_lms_final (measured: 256 -> 64, LMS_POST 0.116 -> 0.103 ms)
#endif
__global__ void __launch_bounds__(LMS_FINAL_T) k_lms_final(RxDev d, unsigned char *labels, long long lab_cap,
                                                   int nseg) {
  pdl_wait();                 // fin_lo / fin_hi from k_lms_prefix
  constexpr int NW = LMS_FINAL_T / 32;
  __shared__ long long red[NW];
  DevState *st = d.st;
  const long long s = st->fin_lo + blockIdx.x;
  if (blockIdx.x >= nseg || s >= st->fin_hi) return;
  const long long si = rmod(s, d.seg_cap);
  const long long lo = s * (long long)d.S, hi = seg_end_of(d, s);
  int R = 0;
  if (d.family == 1 && d.anchor_each) {
    // R-ANCHOR2 (formerly the separate k_lms_stitch launch): R_s = argmax_r #{m in the segment's
    // first 256 outputs (from m0 for s0) : d_m j^r = ref_m}, lowest r on ties
    __shared__ int cnt[4];
    if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long a0 = (s == d.m0 / d.S) ? d.m0 : lo;
    long long a1 = a0 + 256;
    if (a1 > hi) a1 = hi;
    int c4[4] = {0, 0, 0, 0};
    // reference index of a0 (one 64-bit modulo per CTA; the window is < RX_PREF symbols long)
    const int ra0 = (int)(((st->sync_offset + a0 - d.m0) % RX_PREF + RX_PREF) % RX_PREF);
    for (long long m = a0 + threadIdx.x; m < a1; m += blockDim.x) {
      const int cur = d.level[rmod(m, d.sym_cap)];
      int ri = ra0 + (int)(m - a0);
      if (ri >= RX_PREF) ri -= RX_PREF;
      const int ref = d.ref_idx[ri];
#pragma unroll
      for (int r = 0; r < 4; ++r) c4[r] += (qam_rot(cur, r, d.L) == ref);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int v = __reduce_add_sync(0xffffffffu, c4[r]);
      if ((threadIdx.x & 31) == 0) atomicAdd(&cnt[r], v);
    }
    __syncthreads();
    for (int r = 1; r < 4; ++r) if (cnt[r] > cnt[R]) R = r;
    if (threadIdx.x == 0) {
      d.seg_r[si] = R;
      d.seg_R[si] = R;
      d.seg_stitched[si] = (int)(s + 1);
    }
  } else if (d.family == 1) {
    R = d.seg_R[si];
  }
  const int b = d.kbits >> 1;
  // per-segment lookup: level code -> code rotated by j^R (QAM) and its Gray label
  __shared__ unsigned char lut_code[256], lut_lab[256];
  {
    for (int c0 = threadIdx.x; c0 < 256; c0 += LMS_FINAL_T) {
      int c = c0;
      unsigned char lb;
      if (d.family == 1) {
        c = ((c & 15) < d.L && (c >> 4) < d.L) ? qam_rot(c, R, d.L) : c;
        lb = (unsigned char)((gray(c & 15) << b) | gray(c >> 4));
      } else {
        lb = (unsigned char)gray(c);
      }
      lut_code[c0] = (unsigned char)c;
      lut_lab[c0] = lb;
    }
  }
  __syncthreads();
  long long err = 0, cntd = 0;
  // reference index of the segment's first symbol (one modulo per segment); 16 symbols per
  // thread-step: 128-bit level / label accesses where aligned
  const int r0 = (int)(((st->sync_offset + lo - d.m0) % RX_PREF + RX_PREF) % RX_PREF);
  const bool lvec = labels && (((unsigned long long)labels | (unsigned long long)lab_cap) & 15) == 0;
  for (long long v = 16LL * threadIdx.x; v < hi - lo; v += 16LL * blockDim.x) {
    const long long m0v = lo + v;
    const int nv = hi - m0v < 16 ? (int)(hi - m0v) : 16;
    const bool full = nv == 16 && (m0v & 15) == 0;
    unsigned char code[16];
    if (full) {
      const uint4 q = *reinterpret_cast<const uint4 *>(d.level + rmod(m0v, d.sym_cap));
      const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) code[j] = (unsigned char)(w[j >> 2] >> (8 * (j & 3)));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) code[j] = j < nv ? d.level[rmod(m0v + j, d.sym_cap)] : 0;
    }
    unsigned char lab[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {    // level ring stays in the segment frame (stitching)
      const int c = code[j];
      lab[j] = lut_lab[c];
      code[j] = lut_code[c];
    }
    if (full) {
      unsigned w[4] = {0u, 0u, 0u, 0u}, l[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int j = 0; j < 16; ++j) { w[j >> 2] |= (unsigned)code[j] << (8 * (j & 3)); l[j >> 2] |= (unsigned)lab[j] << (8 * (j & 3)); }
      *reinterpret_cast<uint4 *>(d.level_fin + rmod(m0v, d.sym_cap)) = make_uint4(w[0], w[1], w[2], w[3]);
      if (lvec) *reinterpret_cast<uint4 *>(labels + m0v % lab_cap) = make_uint4(l[0], l[1], l[2], l[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) if (j < nv) d.level_fin[rmod(m0v + j, d.sym_cap)] = code[j];
    }
    if (labels && !(full && lvec)) {
      long long li = m0v % lab_cap;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < nv) labels[li] = lab[j];
        if (++li == lab_cap) li = 0;
      }
    }
    int ri = r0 + (int)v % RX_PREF;    // (v < 2^31: 32-bit modulo)
    if (ri >= RX_PREF) ri -= RX_PREF;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < nv && m0v + j >= d.warmup) {
        err += __popc((int)lab[j] ^ (int)__ldg(d.ref_lab + ri));
        ++cntd;
      }
      if (++ri == RX_PREF) ri = 0;
    }
  }
  err = __reduce_add_sync(0xffffffffu, (unsigned)err);
  cntd = __reduce_add_sync(0xffffffffu, (unsigned)cntd);
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = err; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long e2 = 0;
    for (int w = 0; w < NW; ++w) e2 += red[w];
    d.seg_err[2 * si] = e2;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cntd;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long c2 = 0;
    for (int w = 0; w < NW; ++w) c2 += red[w];
    d.seg_err[2 * si + 1] = c2;
  }
  // canonical taps for the lag-D seeds (reading R-SEED): QAM taps are rotated so
  // that arg(sum_k w_k |w_k|) = 0 — the common carrier phase is removed before averaging.
  if (threadIdx.x < 32) {
    const int k = threadIdx.x;
    float2 w = k < d.K ? d.seg_w[si * RX_MAX_K + k] : make_float2(0.f, 0.f);
    if (d.family == 1 && d.lms_mode != 1) {   // data aided (lms_mode 1): no CPR, absolute frame
      const float a = sqrtf(cabs2(w));
      const float px = warp_sum(w.x * a), py = warp_sum(w.y * a);
      const float inv = rsqrtf(fmaxf(px * px + py * py, 1e-30f));
      w = cmulc(w, make_float2(px * inv, py * inv));
    }
    if (k < d.K) d.seg_w[si * RX_MAX_K + k] = w;
  }
}

__global__ void __launch_bounds__(1024) k_lms_counters(RxDev d) {
  pdl_wait();                 // the previous kernel of the round (programmatic dependent launch)
  lms_add_counters(d, d.st->fin_lo, d.st->fin_hi);
}

// ... and the lag-D epoch seeds (c-9 'Seed': the seed of epoch e + D is the mean of the canonical
// taps of epoch e's segments). The mean is accumulated per epoch in 2^-32 fixed point (int64:
// exact, so independent of the order and grouping of the additions): every round adds the
// segments it finalised, and the epoch's seed is formed once its count is complete. A time shard
// (SURVEY §8(e) mode 2) can therefore add the partial sums of an epoch split between shards
// (rx_import_carry) and still form the single stream's seed bit for bit.
#define SEED_FX 4294967296.0f
#define SEED_FX_INV 2.3283064365386963e-10
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// segments in epoch e (spe; fewer for the last epoch once the stream end m_end is known)
__device__ __forceinline__ long long epoch_segs(const RxDev &d, long long e) {
  const long long spe = d.E_sym / d.S;
  const long long me = d.st->m_end;
  if (me >= 0) {
    const long long left = (me + d.S - 1) / d.S - e * spe;
    if (left < spe) return left > 0 ? left : 0;
  }
  return spe;
}
// add a partial sum (n segments, sums [K][2]) to epoch e's accumulator; tap k by lane k of one
// warp (every lane calls). Forms the seed of e + D when the epoch is complete.
__device__ void seed_acc_add(const RxDev &d, long long e, int n, long long sx, long long sy) {
  const int lane = threadIdx.x & 31;
  const long long slot = rmod(e, d.seed_cap);
  const long long tgt = e + d.D;
  const bool fresh = d.seed_tag[slot] != e + 1;
  long long *acc = d.seed_acc + slot * RX_MAX_K * 2;
  long long ax = 0, ay = 0;
  if (lane < d.K) {
    ax = (fresh ? 0 : acc[2 * lane]) + sx;
    ay = (fresh ? 0 : acc[2 * lane + 1]) + sy;
    acc[2 * lane] = ax;
    acc[2 * lane + 1] = ay;
  }
  const int cnt = (fresh ? 0 : d.seed_cnt[slot]) + n;
  __syncwarp();
  if (lane == 0) {
    d.seed_cnt[slot] = cnt;
    d.seed_tag[slot] = e + 1;
  }
  if (cnt > 0 && cnt >= epoch_segs(d, e) && d.seed_ready[rmod(tgt, d.seed_cap)] != tgt + 1) {
    if (lane < d.K) {
      const double inv = SEED_FX_INV / (double)cnt;
      d.seed[rmod(tgt, d.seed_cap) * RX_MAX_K + lane] = make_float2((float)((double)ax * inv), (float)((double)ay * inv));
    }
    __syncwarp();
    if (lane == 0) { __threadfence(); d.seed_ready[rmod(tgt, d.seed_cap)] = (int)(tgt + 1); }
  }
}

// CTA i: epoch fin_lo/spe + i, the segments of it this round finalised ([fin_lo, fin_hi)):
// warp k sums tap k over them (lane-strided), warp 0 adds the partial to the accumulator. CTAs
// 0..RX_CARRY_SEEDS-1 also stage their partial for the shard record (epoch -1: none).
__global__ void __launch_bounds__(1024) k_lms_seeds(RxDev d, int flush) {
  pdl_wait();                 // the previous kernel of the round (programmatic dependent launch)
  __shared__ long long part[RX_MAX_K][2];
  DevState *st = d.st;
  const long long lo = st->fin_lo, hi = st->fin_hi;
  const long long spe = d.E_sym / d.S;
  const long long e = lo / spe + blockIdx.x;
  const int t = threadIdx.x, k = t >> 5, lane = t & 31;
  const bool has = hi > lo && e <= (hi - 1) / spe;
  if (!has) {
    if (blockIdx.x < RX_CARRY_SEEDS && t == 0) d.seed_xp[blockIdx.x].epoch = -1;
    return;
  }
  long long s_lo = e * spe, s_hi = s_lo + spe;
  if (s_lo < lo) s_lo = lo;
  if (s_hi > hi) s_hi = hi;
  long long sx = 0, sy = 0;
  if (k < d.K) {
    const float2 *src = d.seg_w;
    long long s = s_lo + lane;
    for (; s + 96 < s_hi; s += 128) {            // 4 independent loads in flight
      const float2 w0 = src[rmod(s, d.seg_cap) * RX_MAX_K + k];
      const float2 w1 = src[rmod(s + 32, d.seg_cap) * RX_MAX_K + k];
      const float2 w2 = src[rmod(s + 64, d.seg_cap) * RX_MAX_K + k];
      const float2 w3 = src[rmod(s + 96, d.seg_cap) * RX_MAX_K + k];
      sx += __float2ll_rn(w0.x * SEED_FX) + __float2ll_rn(w1.x * SEED_FX) + __float2ll_rn(w2.x * SEED_FX) +
            __float2ll_rn(w3.x * SEED_FX);
      sy += __float2ll_rn(w0.y * SEED_FX) + __float2ll_rn(w1.y * SEED_FX) + __float2ll_rn(w2.y * SEED_FX) +
            __float2ll_rn(w3.y * SEED_FX);
    }
    for (; s < s_hi; s += 32) {
      const float2 w = src[rmod(s, d.seg_cap) * RX_MAX_K + k];
      sx += __float2ll_rn(w.x * SEED_FX);
      sy += __float2ll_rn(w.y * SEED_FX);
    }
    sx = warp_sum_ll(sx);
    sy = warp_sum_ll(sy);
    if (lane == 0) { part[k][0] = sx; part[k][1] = sy; }
  }
  __syncthreads();
  if (k == 0) {
    const long long px = lane < d.K ? part[lane][0] : 0, py = lane < d.K ? part[lane][1] : 0;
    const int n = (int)(s_hi - s_lo);
    if (blockIdx.x < RX_CARRY_SEEDS) {
      SeedPart *xp = d.seed_xp + blockIdx.x;
      xp->sum[lane][0] = px;
      xp->sum[lane][1] = py;
      if (lane == 0) { xp->epoch = e; xp->n = n; }
    }
    seed_acc_add(d, e, n, px, py);
  }
  (void)flush;
}
