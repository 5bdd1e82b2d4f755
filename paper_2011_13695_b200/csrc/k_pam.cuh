// k_pam.cuh — IMDD PAM-N chain kernels (§III).
//
//  k_pam_fe     H0-H3  ingest + overlap framing + R2C FFT-1024 + static FD EQ + C_b
//  k_pam_theta  H4a    105-block complex average + atan2 (parallel, shared-memory C tiles)
//  k_pam_unwrap H4b    unwrap as a prefix sum of wrapped differences -> tau_b, M_b (one CTA)
//  k_pam_be     H1,H2,H5-H7  re-FFT + EQ + FD clock correction + C2R IFFT + extraction
//  k_norm_coop  H8     buffer-wise DC / amplitude normalisation (one cooperative launch)
#pragma once
#include "fft.cuh"
#include "rx_dev.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define FE_GROUPS 4

// Load block b's 1024 samples (input [512b-512, 512b+512)) into buf as packed complex
// z[n] = x[2n] + i x[2n+1]; returns clipped count of the samples the block owns
// ([512b, 512b+512), so every sample is counted once).
__device__ __forceinline__ int load_block_packed(const InView &in, long long b, float scale,
                                                 float2 *buf, int j) {
  long long p = 512 * b - 512 + 16 * j;
  float x[16];
  int clip = 0;
  load16(in, p, scale, 0.f, x, 512 * b, clip);
#pragma unroll
  for (int i = 0; i < 8; ++i) buf[P8(8 * j + i)] = make_float2(x[2 * i], x[2 * i + 1]);
  return clip;
}

__device__ __forceinline__ void block_reduce_clip(DevState *st, int clip) {
  clip = __reduce_add_sync(0xffffffffu, clip);
  if ((threadIdx.x & 31) == 0 && clip) atomicAdd((unsigned long long *)&st->clipped, (unsigned long long)clip);
}

// ------------------------------------------------------------------ H0-H3
__global__ void __launch_bounds__(256) k_pam_fe(RxDev d, InView in, long long b0, long long b1) {
  __shared__ float2 tw[1024];
  __shared__ float2 buf[FE_GROUPS][FFT_PAD_N];
  __shared__ double2 red[FE_GROUPS][2];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = d.tw[i];
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  const bool act = b < b1;
  int clip = 0;
  if (act) clip = load_block_packed(in, b, d.scale, buf[g], j);
  block_reduce_clip(d.st, clip);
  __syncthreads();
  float2 v[8];
  fft512<false>(buf[g], j, tw, v);
  fft512_store(buf[g], j, v);
  // C_b = sum_{k<512} Y[k] conj(Y[k+512]) = Y0 conj(Y512) + Y256^2 + 2 sum_{k=1}^{255} Y[k] Y[512-k]
  double cr = 0.0, ci = 0.0;
  if (act) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = j + 64 * r;
      float2 Xk, Xn;
      r2c_pair(buf[g][P8(k)], buf[g][P8((512 - k) & 511)], tw[k], Xk, Xn);
      const float2 Yk = cmul(Xk, __ldg(d.H + k)), Yn = cmul(Xn, __ldg(d.H + 512 - k));
      const double ar = Yk.x, ai = Yk.y, br = Yn.x, bi = Yn.y;
      if (k == 0) { cr += ar * br + ai * bi; ci += ai * br - ar * bi; }   // Y0 conj(Y512)
      else { cr += 2.0 * (ar * br - ai * bi); ci += 2.0 * (ar * bi + ai * br); }
    }
    if (j == 0) {
      const float2 Y = cmul(cconj(buf[g][P8(256)]), __ldg(d.H + 256));
      cr += (double)Y.x * Y.x - (double)Y.y * Y.y;
      ci += 2.0 * (double)Y.x * Y.y;
    }
  }
  cr = warp_sum_d(cr);
  ci = warp_sum_d(ci);
  if ((threadIdx.x & 31) == 0) red[g][(threadIdx.x >> 5) & 1] = make_double2(cr, ci);
  __syncthreads();
  if (act && j == 0)
    d.C[rmod(b, d.blk_cap)] = make_double2(red[g][0].x + red[g][1].x, red[g][0].y + red[g][1].y);
}

// ------------------------------------------------------------------ H4
// One CTA of 1024 threads per call, blocks [b0, b1) in chunks of 8192 (c-3):
//   Cbar_b = sum_{i=max(0,b-h)}^{min(blast,b+h)} C_i   (105-block vector average, from a
//            shared-memory tile of C, each thread sliding its window over 8 blocks)
//   theta_b = atan2(Cbar_b) ; |Cbar| = 0 inherits the previous phase
//   theta^u_b = theta^u_{b-1} + w(theta_b - theta_{b-1}), w(x) = x - 2 pi rint(x / 2 pi):
//            the paper's serial single-warp unwrap as a warp-shuffle block scan
//   tau_b = -theta^u_b / 2 pi ; M_b = ceil(256 b - 128 - tau_b)
#define CLK_CHUNK 8192
__device__ __forceinline__ double warp_incl_scan_d(double v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ long long warp_incl_max_ll(long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o && t > v) v = t;
  }
  return v;
}

// (a) theta_b for blocks [b0, b1): one CTA per 256 blocks, C tile (+ 2h halo) in shared
//     memory, each thread sums its own 105-term window (consecutive lanes, conflict-free).
__global__ void __launch_bounds__(256) k_pam_theta(RxDev d, long long b0, long long b1, long long blast) {
  extern __shared__ double2 Ct[];                 // [256 + 2 h]
  const int t = threadIdx.x, hh = d.clock_half;
  const long long base = b0 + (long long)blockIdx.x * 256;
  for (int i = t; i < 256 + 2 * hh; i += blockDim.x) {
    const long long b = base - hh + i;
    Ct[i] = (b >= 0 && b <= blast) ? d.C[rmod(b, d.blk_cap)] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const long long b = base + t;
  if (b >= b1) return;
  double sr = 0.0, si = 0.0;
  for (int i = 0; i <= 2 * hh; ++i) { const double2 c = Ct[t + i]; sr += c.x; si += c.y; }
  d.theta[rmod(b, d.blk_cap)] = (sr == 0.0 && si == 0.0) ? __longlong_as_double(0x7ff8000000000000LL)
                                                         : atan2(si, sr);
}

// (b) one CTA: |Cbar| = 0 inherits the previous phase (max-scan of the last valid block),
//     wrapped differences, prefix sum (warp-shuffle block scan), tau_b and M_b.
__global__ void __launch_bounds__(1024) k_pam_unwrap(RxDev d, long long b0, long long b1) {
  __shared__ double wsum[32];
  __shared__ long long wmax[32];
  __shared__ double carry_theta, carry_u;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double TWO_PI = 6.283185307179586476925;
  if (t == 0) { carry_theta = d.st->theta_prev; carry_u = d.st->thetau_prev; }
  __syncthreads();
  for (long long base = b0; base < b1; base += CLK_CHUNK) {
    const long long nb = (b1 - base) < CLK_CHUNK ? (b1 - base) : CLK_CHUNK;
    double th[8];
    long long last = -1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long j = 8 * t + q;
      th[q] = __longlong_as_double(0x7ff8000000000000LL);
      if (j < nb) th[q] = d.theta[rmod(base + j, d.blk_cap)];
      if (j < nb && !isnan(th[q])) last = base + j;
    }
    const long long lw = warp_incl_max_ll(last);
    if (lane == 31) wmax[warp] = lw;
    __syncthreads();
    if (warp == 0) wmax[lane] = warp_incl_max_ll(wmax[lane]);
    __syncthreads();
    long long excl = __shfl_up_sync(0xffffffffu, lw, 1);
    if (lane == 0) excl = -1;
    if (warp > 0 && wmax[warp - 1] > excl) excl = wmax[warp - 1];
    const double prev0 = excl >= 0 ? d.theta[rmod(excl, d.blk_cap)] : carry_theta;
    double diff[8], run = 0.0;
    {
      double cur = prev0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        diff[q] = 0.0;
        if (8 * t + q < nb) {
          const double x = isnan(th[q]) ? cur : th[q];
          const double dd = x - cur;
          diff[q] = dd - TWO_PI * rint(dd / TWO_PI);
          cur = x;
        }
        run += diff[q];
      }
    }
    const double incl = warp_incl_scan_d(run);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) wsum[lane] = warp_incl_scan_d(wsum[lane]);
    __syncthreads();
    double acc = carry_u + (incl - run) + (warp > 0 ? wsum[warp - 1] : 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long j = 8 * t + q;
      acc += diff[q];
      if (j < nb) {
        const long long b = base + j;
        const double tau = -acc / TWO_PI;
        d.tau[rmod(b, d.blk_cap)] = tau;
        d.Mb[rmod(b, d.blk_cap)] = (long long)ceil(256.0 * (double)b - 128.0 - tau);
      }
    }
    const double total = wsum[31];
    const long long lastall = wmax[31];
    __syncthreads();
    if (t == 0) {
      carry_u += total;
      if (lastall >= 0) carry_theta = d.theta[rmod(lastall, d.blk_cap)];
    }
    __syncthreads();
  }
  if (t == 0) { d.st->theta_prev = carry_theta; d.st->thetau_prev = carry_u; }
}

// ------------------------------------------------------------------ H1, H2, H5-H7
__global__ void __launch_bounds__(256) k_pam_be(RxDev d, InView in, long long b0, long long b1) {
  __shared__ float2 tw[1024];
  __shared__ float2 buf[FE_GROUPS][FFT_PAD_N];
  __shared__ double red[FE_GROUPS][2];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = d.tw[i];
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  const bool act = b < b1;
  if (act) load_block_packed(in, b, d.scale, buf[g], j);
  __syncthreads();
  float2 v[8];
  fft512<false>(buf[g], j, tw, v);
  fft512_store(buf[g], j, v);
  // clock phase of this block: s = 2 tau, i_b = rint(s), f_b = s - i_b   (c-4)
  double tau = act ? d.tau[rmod(b, d.blk_cap)] : 0.0;
  const double s = 2.0 * tau;
  const double ibd = rint(s);
  const float f = (float)(s - ibd);
  float2 Zk[4], Zn[4], Z256;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = j + 64 * r;
    float2 Xk, Xn;
    r2c_pair(buf[g][P8(k)], buf[g][P8((512 - k) & 511)], tw[k], Xk, Xn);
    float2 Yk = cmul(Xk, __ldg(d.H + k)), Yn = cmul(Xn, __ldg(d.H + 512 - k));
    // Y'[k] = Y[k] e^{+j 2 pi kappa(k) f / 1024}; kappa(k) = k, kappa(512-k) = 512-k,
    // Nyquist (k = 0 partner): Re(Y[512] e^{-j pi f})
    float sk, ck, sn, cn;
    sincospif((float)k * f * (1.0f / 512.0f), &sk, &ck);
    Yk = cmul(Yk, make_float2(ck, sk));
    if (k == 0) {
      sincospif(f, &sn, &cn);
      Yn = make_float2(Yn.x * cn + Yn.y * sn, 0.0f);
    } else {
      sincospif((float)(512 - k) * f * (1.0f / 512.0f), &sn, &cn);
      Yn = cmul(Yn, make_float2(cn, sn));
    }
    c2r_pair(Yk, Yn, tw[k], Zk[r], Zn[r]);
  }
  {
    float2 Y = cmul(cconj(buf[g][P8(256)]), __ldg(d.H + 256));
    float s2, c2;
    sincospif(256.0f * f * (1.0f / 512.0f), &s2, &c2);
    Y = cmul(Y, make_float2(c2, s2));
    Z256 = cconj(Y);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = j + 64 * r;
    buf[g][P8(k)] = Zk[r];
    if (k != 0) buf[g][P8(512 - k)] = Zn[r];
  }
  if (j == 0) buf[g][P8(256)] = Z256;
  __syncthreads();
  fft512<true>(buf[g], j, tw, v);
  fft512_store(buf[g], j, v);
  // variable-rate extraction (c-4): u_m = y[2m + i_b - 512b + 512], m in [max(M_b,0), M_{b+1})
  double part = 0.0;
  if (act) {
    const long long Mb = d.Mb[rmod(b, d.blk_cap)], Mb1 = d.Mb[rmod(b + 1, d.blk_cap)];
    const long long lo = Mb > 0 ? Mb : 0;
    const long long ib = (long long)ibd;
    for (long long m = lo + j; m < Mb1; m += 64) {
      long long loc = 2 * m + ib - 512 * b + 512;
      if (loc < 0 || loc >= 1024) { set_flag(d.st, 8); loc = loc < 0 ? 0 : 1023; }
      const float2 zz = buf[g][P8((int)(loc >> 1))];
      const float y = ((loc & 1) ? zz.y : zz.x) * (1.0f / 512.0f);
      d.u[rmod(m, d.sym_cap)] = y;
      part += (double)y;
    }
  }
  part = warp_sum_d(part);
  if ((threadIdx.x & 31) == 0) red[g][(threadIdx.x >> 5) & 1] = part;
  __syncthreads();
  if (act && j == 0) d.blk_sum[rmod(b, d.blk_cap)] = red[g][0] + red[g][1];
}

// ------------------------------------------------------------------ H8 normalisation
// One cooperative kernel per buffer (P:167 'three kernels: initialization, estimation of the
// DC-offset, and estimation of the amplitude'; c-5):
//   dc = mean u, A = mean|u - dc| / (M / (2 (M-1))), u^ = (u - dc) / A
// over the symbols emitted by blocks [blo, bhi). Each CTA owns a contiguous block range; the
// two buffer-wide reductions are fixed-order (per-CTA partials, then every CTA sums the
// partials in index order) separated by grid-wide syncs, so results are deterministic.
__device__ __forceinline__ double block_sum_det(double v, double *sh) {
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) r += sh[w];
  __syncthreads();
  return r;   // identical in all threads
}
__device__ __forceinline__ long long sym_lo_of(const RxDev &d, long long b) {
  const long long m = d.Mb[rmod(b, d.blk_cap)];
  return m > 0 ? m : 0;
}

__global__ void __launch_bounds__(1024) k_norm_coop(RxDev d, long long beta, long long blo, long long bhi,
                                                   int last) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  const int G = gridDim.x, g = blockIdx.x, t = threadIdx.x;
  const long long nb = bhi - blo;
  const long long cb0 = blo + nb * g / G, cb1 = blo + nb * (g + 1) / G;
  const long long m0 = sym_lo_of(d, cb0), m1 = sym_lo_of(d, cb1) > m0 ? sym_lo_of(d, cb1) : m0;
  // phase 1: sum u over the CTA's symbols (from the per-block sums written by k_pam_be)
  double s = 0.0;
  for (long long b = cb0 + t; b < cb1; b += blockDim.x) s += d.blk_sum[rmod(b, d.blk_cap)];
  s = block_sum_det(s, sh);
  if (t == 0) { d.norm_part[2 * g] = s; d.norm_part[2 * g + 1] = (double)(m1 - m0); }
  grid.sync();
  __shared__ double bc[3];
  if (t < 32) {   // fixed order: lane l sums partials l, l+32, ..., then a fixed shuffle tree
    double ps = 0.0, pc = 0.0;
    for (int i = t; i < G; i += 32) { ps += d.norm_part[2 * i]; pc += d.norm_part[2 * i + 1]; }
    ps = warp_sum_d(ps);
    pc = warp_sum_d(pc);
    if (t == 0) { bc[0] = ps; bc[1] = pc; }
  }
  __syncthreads();
  const double S = bc[0], Cn = bc[1];
  const double dc = Cn > 0.0 ? S / Cn : 0.0;
  // phase 2: sum |u - dc|
  double a = 0.0;
  for (long long m = m0 + t; m < m1; m += blockDim.x) a += fabs((double)d.u[rmod(m, d.sym_cap)] - dc);
  a = block_sum_det(a, sh);
  grid.sync();                                   // everyone has read phase-1 partials
  if (t == 0) d.norm_part[2 * G + g] = a;
  grid.sync();
  if (t < 32) {
    double pa = 0.0;
    for (int i = t; i < G; i += 32) pa += d.norm_part[2 * G + i];
    pa = warp_sum_d(pa);
    if (t == 0) bc[2] = pa;
  }
  __syncthreads();
  const double Aa = bc[2];
  const double mal = (double)d.M / (2.0 * (double)(d.M - 1));
  double A = Cn > 0.0 ? (Aa / Cn) / mal : 1.0;
  if (!(A > 0.0)) A = 1.0;
  // phase 3: apply
  const float dcf = (float)dc, inv = (float)(1.0 / A);
  for (long long m = m0 + t; m < m1; m += blockDim.x) {
    const long long i = rmod(m, d.sym_cap);
    d.uhat[i] = (d.u[i] - dcf) * inv;
  }
  if (g == 0 && t == 0) {
    d.norm_dc[rmod(beta, d.buf_cap)] = dc;
    d.norm_amp[rmod(beta, d.buf_cap)] = A;
    d.norm_cnt[rmod(beta, d.buf_cap)] = (long long)Cn;
    long long f = sym_lo_of(d, bhi);
    d.st->v_front = f;
    if (last) d.st->m_end = f;
  }
}
