// k_pam.cuh — IMDD PAM-N chain kernels (§III).
//
//  k_pam_fe     H0-H3  ingest + overlap framing + R2C FFT-1024 + static FD EQ + C_b
//  k_pam_theta  H4a    105-block complex average + atan2          (parallel over blocks)
//  k_pam_unwrap H4b    unwrap as a prefix sum of wrapped differences, tau_b, M_b (1 CTA)
//  k_pam_be     H1,H2,H5-H7  re-FFT + EQ + FD clock correction + C2R IFFT + extraction
//  k_norm_*     H8     buffer-wise DC / amplitude normalisation (fixed-order reductions)
#pragma once
#include "fft.cuh"
#include "rx_dev.cuh"

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

// ------------------------------------------------------------------ H4 (a)
// Cbar_b = sum_{i=max(0,b-h)}^{min(blast,b+h)} C_i ; theta_b = atan2(Cbar_b) (NaN if 0).
__global__ void k_pam_theta(RxDev d, long long b0, long long b1, long long blast) {
  const long long b = b0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= b1) return;
  long long lo = b - d.clock_half, hi = b + d.clock_half;
  if (lo < 0) lo = 0;
  if (hi > blast) hi = blast;
  double sr = 0.0, si = 0.0;
  for (long long i = lo; i <= hi; ++i) {
    const double2 c = d.C[rmod(i, d.blk_cap)];
    sr += c.x; si += c.y;
  }
  d.theta[rmod(b, d.blk_cap)] = (sr == 0.0 && si == 0.0) ? __longlong_as_double(0x7ff8000000000000LL)
                                                         : atan2(si, sr);
}

// ------------------------------------------------------------------ H4 (b)
// One CTA of 1024 threads. theta^u_b = theta^u_{b-1} + w(theta_b - theta_{b-1}),
// w(x) = x - 2 pi rint(x / 2 pi): a prefix sum of wrapped differences (SURVEY c-3, A15) —
// the paper's single-warp serial unwrap as a block scan. |Cbar| = 0 inherits the
// previous phase via a max-scan of the last valid index.
__global__ void __launch_bounds__(1024) k_pam_unwrap(RxDev d, long long b0, long long b1) {
  __shared__ double sd[1024];
  __shared__ long long si[1024];
  __shared__ double carry_theta, carry_u;
  const int t = threadIdx.x;
  const double TWO_PI = 6.283185307179586476925;
  if (t == 0) { carry_theta = d.st->theta_prev; carry_u = d.st->thetau_prev; }
  __syncthreads();
  for (long long base = b0; base < b1; base += 8192) {
    double th[8];
    long long vi[8];
    long long last = -1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long b = base + 8 * t + i;
      double x = 0.0;
      bool valid = false;
      if (b < b1) { x = d.theta[rmod(b, d.blk_cap)]; valid = !isnan(x); }
      th[i] = x;
      if (valid) last = b;
      vi[i] = last;
    }
    // inclusive max-scan of the last valid index
    si[t] = last;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      long long o = (t >= off) ? si[t - off] : -1;
      __syncthreads();
      if (o > si[t]) si[t] = o;
      __syncthreads();
    }
    const long long excl = (t > 0) ? si[t - 1] : -1;
    __syncthreads();
    // resolve inherited phases: theta_b = theta[last valid <= b] or the carry
    double prev_local;
    {
      long long src = excl;
      prev_local = (src >= 0) ? d.theta[rmod(src, d.blk_cap)] : carry_theta;
    }
    double diff[8];
    double run = 0.0;
    double prevth = prev_local;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long b = base + 8 * t + i;
      double x;
      if (vi[i] >= 0 && vi[i] == b) x = th[i];
      else if (vi[i] >= 0) x = d.theta[rmod(vi[i], d.blk_cap)];
      else x = prev_local;
      // for inherited entries with no valid in this thread's run, vi < 0 -> prev_local
      if (vi[i] < 0) x = prev_local;
      const double dd = x - prevth;
      diff[i] = (b < b1) ? dd - TWO_PI * rint(dd / TWO_PI) : 0.0;
      run += diff[i];
      th[i] = x;
      prevth = x;
    }
    // exclusive prefix sum of the per-thread totals (Hillis-Steele in double)
    sd[t] = run;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      double o = (t >= off) ? sd[t - off] : 0.0;
      __syncthreads();
      sd[t] += o;
      __syncthreads();
    }
    double acc = carry_u + ((t > 0) ? sd[t - 1] : 0.0);
    const double total = sd[1023];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long b = base + 8 * t + i;
      acc += diff[i];
      if (b < b1) {
        const double tau = -acc / TWO_PI;
        d.tau[rmod(b, d.blk_cap)] = tau;
        d.Mb[rmod(b, d.blk_cap)] = (long long)ceil(256.0 * (double)b - 128.0 - tau);
      }
    }
    __syncthreads();
    // carries for the next chunk: last resolved theta and the running unwrapped phase
    if (t == 1023) {
      carry_u = carry_u + total;
    }
    long long nlast = si[1023];
    __syncthreads();
    if (t == 0 && nlast >= 0) carry_theta = d.theta[rmod(nlast, d.blk_cap)];
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
// fixed-order block reduction of doubles (deterministic)
__device__ __forceinline__ double block_sum_1024(double v, double *sh) {
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
    r = warp_sum_d(r);
  }
  __syncthreads();
  return r;   // valid in warp 0
}

// dc_beta = sum u / count over the symbols emitted by blocks [blo, bhi)
__global__ void __launch_bounds__(1024) k_norm_dc(RxDev d, long long beta, long long blo, long long bhi) {
  __shared__ double sh[32];
  double s = 0.0, c = 0.0;
  for (long long b = blo + threadIdx.x; b < bhi; b += blockDim.x) {
    s += d.blk_sum[rmod(b, d.blk_cap)];
    const long long Mb = d.Mb[rmod(b, d.blk_cap)], Mb1 = d.Mb[rmod(b + 1, d.blk_cap)];
    const long long lo = Mb > 0 ? Mb : 0;
    c += (double)(Mb1 > lo ? Mb1 - lo : 0);
  }
  s = block_sum_1024(s, sh);
  c = block_sum_1024(c, sh);
  if (threadIdx.x == 0) {
    d.norm_dc[rmod(beta, d.buf_cap)] = c > 0 ? s / c : 0.0;
    d.norm_cnt[rmod(beta, d.buf_cap)] = (long long)c;
  }
}

// per-block sum |u - dc|
__global__ void __launch_bounds__(256) k_norm_abs(RxDev d, long long beta, long long blo, long long bhi) {
  __shared__ double sh[8];
  const long long b = blo + blockIdx.x;
  if (b >= bhi) return;
  const double dc = d.norm_dc[rmod(beta, d.buf_cap)];
  const long long Mb = d.Mb[rmod(b, d.blk_cap)], Mb1 = d.Mb[rmod(b + 1, d.blk_cap)];
  const long long lo = Mb > 0 ? Mb : 0;
  double s = 0.0;
  for (long long m = lo + threadIdx.x; m < Mb1; m += blockDim.x)
    s += fabs((double)d.u[rmod(m, d.sym_cap)] - dc);
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    d.blk_abs[rmod(b, d.blk_cap)] = t;
  }
}

// A = mean|u - dc| / (M / (2 (M-1)))   (c-5)
__global__ void __launch_bounds__(1024) k_norm_amp(RxDev d, long long beta, long long blo, long long bhi) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long b = blo + threadIdx.x; b < bhi; b += blockDim.x) s += d.blk_abs[rmod(b, d.blk_cap)];
  s = block_sum_1024(s, sh);
  if (threadIdx.x == 0) {
    const long long c = d.norm_cnt[rmod(beta, d.buf_cap)];
    const double mal = (double)d.M / (2.0 * (double)(d.M - 1));
    double A = c > 0 ? (s / (double)c) / mal : 1.0;
    if (!(A > 0.0)) A = 1.0;
    d.norm_amp[rmod(beta, d.buf_cap)] = A;
  }
}

// u^ = (u - dc) / A; advances the v_front to M_{bhi} (or m_end at flush)
__global__ void __launch_bounds__(256) k_norm_apply(RxDev d, long long beta, long long blo, long long bhi,
                                                   int last) {
  const long long b = blo + blockIdx.x;
  if (b < bhi) {
    const float dc = (float)d.norm_dc[rmod(beta, d.buf_cap)];
    const float inv = (float)(1.0 / d.norm_amp[rmod(beta, d.buf_cap)]);
    const long long Mb = d.Mb[rmod(b, d.blk_cap)], Mb1 = d.Mb[rmod(b + 1, d.blk_cap)];
    const long long lo = Mb > 0 ? Mb : 0;
    for (long long m = lo + threadIdx.x; m < Mb1; m += blockDim.x) {
      const long long i = rmod(m, d.sym_cap);
      d.uhat[i] = (d.u[i] - dc) * inv;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long f = d.Mb[rmod(bhi, d.blk_cap)];
    if (f < 0) f = 0;
    d.st->v_front = f;
    if (last) d.st->m_end = f;
  }
}
