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

// ------------------------------------------------------------------ H0, H11-H15
__global__ void __launch_bounds__(256) k_kk_s1(RxDev d, InView in, long long b0, long long b1) {
  __shared__ float2 tw[1024];
  __shared__ float2 buf[FE_GROUPS][FFT_PAD_N];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = d.tw[i];
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  const bool act = b < b1;
  int clip = 0, dom = 0;
  long long first_dom = 0x7fffffffffffffffLL;
  float2 v[8];
  float amp[4][2];                                      // sqrt(I) of the kept samples (r = 2..5)
  if (act) {
    clip = load_block_regs(in, b, d.scale, j, v);       // x_p = 0 for p < 0 (c-0) -> I = dc
    const long long p0 = 512 * b - 512;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float hh[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float I = (e ? v[r].y : v[r].x) + d.dc;         // P:215 static DC offset
        const long long p = p0 + 2 * (j + 64 * r) + e;
        if (I <= 0.0f && r >= 4) {                      // owned samples counted once (A7)
          ++dom;
          if (p < first_dom) first_dom = p;
        }
        I = fmaxf(I, 1e-12f);
        hh[e] = 0.5f * logf(I);                         // P:215 logarithm for the phase
        if (r >= 2 && r < 6) amp[r - 2][e] = sqrtf(I);  // P:215 square root: amplitude
      }
      v[r] = make_float2(hh[0], hh[1]);
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 4; ++r) amp[r][0] = amp[r][1] = 0.f;
  }
  block_reduce_clip(d.st, clip);
  dom = __reduce_add_sync(0xffffffffu, dom);
  if ((threadIdx.x & 31) == 0 && dom) atomicAdd((unsigned long long *)&d.st->domain_errors, (unsigned long long)dom);
  if (first_dom != 0x7fffffffffffffffLL) atomicMin(&d.st->first_domain, first_dom);
  fft512_regs<false>(buf[g], j, tw, v);
  fft512_publish_upper(buf[g], j, v);
  // FD Hilbert (c-6, A8): Phi = -j sgn(kappa) H, Phi[0] = Phi[512] = 0
  float2 Zk[4], Zn[4];
  const float2 *pm = fft_mirror_base(buf[g], j);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = j + 64 * r;
    float2 Xk, Xn;
    r2c_pair(v[r], fft_partner(pm, j, r, v), tw[k], Xk, Xn);
    float2 Pk = cmul_mi(Xk), Pn = cmul_mi(Xn);
    if (k == 0) { Pk = make_float2(0.f, 0.f); Pn = make_float2(0.f, 0.f); }
    c2r_pair(Pk, Pn, tw[k], Zk[r], Zn[r]);
  }
  const float2 Z256 = cconj(cmul_mi(cconj(v[4])));
  __syncthreads();
  {
    float2 *paw = buf[g] + j + (j >> 4);
    float2 *pmw = buf[g] + (512 - j) + ((512 - j) >> 4);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      paw[68 * r] = Zk[r];
      if (!(j == 0 && r == 0)) pmw[-68 * r] = Zn[r];
    }
    if (j == 0) buf[g][256 + (256 >> 4)] = Z256;
  }
  __syncthreads();
  fft512<true>(buf[g], j, tw, v);
  // v[r] = 512 (phi[2n] + i phi[2n+1]), n = j + 64 r; kept local [256, 768) <=> r = 2..5
  if (act) {
    const float sg = (float)d.sideband;
#pragma unroll
    for (int r = 2; r < 6; ++r) {
      const int n = j + 64 * r;
      const long long p = 512 * b - 512 + 2 * n;
      if (p < 0) continue;
      const float ph0 = v[r].x * (1.0f / 512.0f), ph1 = v[r].y * (1.0f / 512.0f);
      float s0, c0, s1, c1;
      sincosf(sg * ph0, &s0, &c0);
      sincosf(sg * ph1, &s1, &c1);
      const float a0 = amp[r - 2][0], a1 = amp[r - 2][1];
      // downshift to DC: e^{-j psi(p; sigma f_c)}, 64-bit DDS from the absolute index
      const float2 r0 = dds_rot_neg((unsigned long long)p * d.carrier_inc);
      const float2 r1 = dds_rot_neg((unsigned long long)(p + 1) * d.carrier_inc);
      const float2 e0 = cmul(make_float2(a0 * c0, a0 * s0), r0);
      const float2 e1 = cmul(make_float2(a1 * c1, a1 * s1), r1);
      *reinterpret_cast<float4 *>(d.E + rmod(p, d.E_cap)) = make_float4(e0.x, e0.y, e1.x, e1.y);
    }
  }
}

// ------------------------------------------------------------------ H16-H18
// 4 blocks per CTA: pass A runs 8 half-size FFTs (evens / odds of each block) on the 4 groups,
// pass B the 4 decimating IFFT-512s.
__global__ void __launch_bounds__(256) k_kk_s2(RxDev d, long long b0, long long b1) {
  extern __shared__ float2 sm[];
  float2 *tw = sm;                               // 1024
  float2 *bufs = sm + 1024;                      // [4 blocks][2][FFT_PAD_N]
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tw[i] = d.tw[i];
  // load E for the 4 blocks: frame p in [512b - 512, 512b + 512), E_p = 0 for p < 0
  for (int bl = 0; bl < 4; ++bl) {
    const long long b = b0 + (long long)blockIdx.x * 4 + bl;
    float2 *be = bufs + (bl * 2) * FFT_PAD_N, *bo = bufs + (bl * 2 + 1) * FFT_PAD_N;
    for (int n = threadIdx.x; n < 512; n += blockDim.x) {
      const long long p = 512 * b - 512 + 2 * n;
      float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
      if (b < b1 && p >= 0) e = *reinterpret_cast<const float4 *>(d.E + rmod(p, d.E_cap));
      be[P8(n)] = make_float2(e.x, e.y);
      bo[P8(n)] = make_float2(e.z, e.w);
    }
  }
  __syncthreads();
  float2 v[8];
  // pass A: group g transforms half-buffers 2g and 2g+1 ... (blocks g/2 ... ) -> 8 halves on 4 groups
  for (int rep = 0; rep < 2; ++rep) {
    float2 *hb = bufs + (g * 2 + rep) * FFT_PAD_N;
    fft512<false>(hb, j, tw, v);
    fft512_store(hb, j, v);
  }
  // combine + EQ + band select: for block bl = g:
  //   G'[k'] = (Ev[k'] + W^k' Od[k']) H2[k'],        k' in [0, 256)   (kappa = k')
  //   G'[k'] = (Ev[k'] - W^k' Od[k']) H2[k' + 512],  k' in [256, 512) (kappa = k' - 512)
  {
    float2 *be = bufs + (g * 2) * FFT_PAD_N, *bo = bufs + (g * 2 + 1) * FFT_PAD_N;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int k = j + 64 * r;
      const float2 ev = be[P8(k)], od = cmul(bo[P8(k)], tw[k]);
      float2 G;
      if (k < 256) G = cmul(cadd(ev, od), __ldg(d.H + k));
      else G = cmul(csub(ev, od), __ldg(d.H + k + 512));
      be[P8(k)] = G;
    }
  }
  __syncthreads();
  {
    float2 *be = bufs + (g * 2) * FFT_PAD_N;
    fft512<true>(be, j, tw, v);
    // z_local[n] = 1/2 * IDFT512 = v / 1024; keep n in [128, 384) <=> r = 2..5
    const long long b = b0 + (long long)blockIdx.x * 4 + g;
    if (b < b1) {
#pragma unroll
      for (int r = 2; r < 6; ++r) {
        const int n = j + 64 * r;
        const long long q = 256 * b - 256 + n;
        if (q >= 0) d.z[rmod(q, d.z_cap)] = cscale(v[r], 1.0f / 1024.0f);
      }
    }
  }
}

// ------------------------------------------------------------------ H19-H20
// Partial sums over the complete 1024-sample chunks of buffer beta:
//   pow_part[cta] = sum |z|^2 (all samples of [qlo, qhi)),
//   S_part[cta][k] = sum_chunks |DFT_1024(z^4)[k]|^2
__global__ void __launch_bounds__(256) k_cfo_partial(RxDev d, long long qlo, long long qhi) {
  extern __shared__ float2 sm[];
  float2 *tw = sm;
  float2 *bufs = sm + 1024;                    // [4 groups][2][FFT_PAD_N]
  float *S = reinterpret_cast<float *>(bufs + 8 * FFT_PAD_N);   // [1024]
  __shared__ double red[8];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { tw[i] = d.tw[i]; S[i] = 0.f; }
  const long long n = qhi - qlo;
  const long long nch = n / 1024;
  double pw = 0.0;
  for (long long q = qlo + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < qhi;
       q += (long long)gridDim.x * blockDim.x)
    pw += (double)cabs2(d.z[rmod(q, d.z_cap)]);
  __syncthreads();
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  const long long per = (nch + gridDim.x - 1) / gridDim.x;   // chunks per CTA (contiguous)
  const long long c0 = (long long)blockIdx.x * per;
  const long long c1 = c0 + per < nch ? c0 + per : nch;
  for (long long cb = c0; cb < c1; cb += 4) {
    const long long c = cb + g;
    float2 *be = bufs + (g * 2) * FFT_PAD_N, *bo = bufs + (g * 2 + 1) * FFT_PAD_N;
    const bool act = c < c1;
    for (int t = j; t < 512; t += 64) {
      float2 a = make_float2(0.f, 0.f), bq = a;
      if (act) {
        const long long q = qlo + 1024 * c + 2 * t;
        a = d.z[rmod(q, d.z_cap)];
        bq = d.z[rmod(q + 1, d.z_cap)];
      }
      float2 a2 = cmul(a, a), b2 = cmul(bq, bq);
      be[P8(t)] = cmul(a2, a2);
      bo[P8(t)] = cmul(b2, b2);
    }
    __syncthreads();
    float2 ve[8], vo[8];
    fft512<false>(be, j, tw, ve);
    __syncthreads();
    fft512<false>(bo, j, tw, vo);
    if (act) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int k = j + 64 * r;
        const float2 od = cmul(vo[r], tw[k]);
        acc[r] += cabs2(cadd(ve[r], od));        // X[k]
        acc[8 + r] += cabs2(csub(ve[r], od));    // X[k + 512]
      }
    }
    __syncthreads();
  }
  // combine the 4 groups' accumulators in fixed order
  for (int gg = 0; gg < 4; ++gg) {
    if (g == gg) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        S[j + 64 * r] += acc[r];
        S[j + 64 * r + 512] += acc[8 + r];
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) d.cfo_part[(long long)blockIdx.x * 1024 + i] = S[i];
  pw = warp_sum_d(pw);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    d.cfo_pow[blockIdx.x] = t;
  }
}

// P, k* = argmax S (lowest on ties), delta, df, DDS increment and carried origin (c-8).
__global__ void __launch_bounds__(1024) k_cfo_final(RxDev d, long long beta, long long qlo, long long qhi) {
  __shared__ double Sd[1024];
  __shared__ double wv[32];
  __shared__ int wi[32];
  const int t = threadIdx.x;
  const int G = d.cfo_G;
  double s = 0.0;
  int c = 0;
  for (; c + 8 <= G; c += 8) {          // 8 independent loads in flight, summed in index order
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = d.cfo_part[(long long)(c + i) * 1024 + t];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += (double)v[i];
  }
  for (; c < G; ++c) s += (double)d.cfo_part[(long long)c * 1024 + t];
  Sd[t] = s;
  // argmax, lowest index on ties
  double bv = s;
  int bi = t;
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
    for (int c = 0; c < G; ++c) P += d.cfo_pow[c];
    const long long n = qhi - qlo;
    P = n > 0 ? P / (double)n : 1.0;
    if (!(P > 0.0)) P = 1.0;
    double best = wv[0];
    int k = wi[0];
    for (int w = 1; w < 32; ++w)
      if (wv[w] > best || (wv[w] == best && wi[w] < k)) { best = wv[w]; k = wi[w]; }
    const long long nch = n / 1024;
    double df = d.st->cfo_df_prev;
    if (nch > 0) {
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
    cp.df = df;                      // coarse; refined by k_cfo_fine_final
    cp.inc = (unsigned long long)llrint(ldexp(df / d.fs2, 64));
    cp.origin = 0ull;
    d.cfo[rmod(beta, d.buf_cap)] = cp;
  }
}

// Fine stage (reading R-CFO): a_i = sum_{chunk i} (z_q e^{-j 2 pi df_c n / f_s2})^4,
// n = q - q_lo, the coarse rotation from a 64-bit DDS word n * inc_c.
__global__ void __launch_bounds__(256) k_cfo_fine(RxDev d, long long beta, long long qlo, long long qhi) {
  __shared__ double2 red[8];
  const long long nch = (qhi - qlo) / 1024;
  const CfoParam cp = d.cfo[rmod(beta, d.buf_cap)];
  for (long long i = blockIdx.x; i < nch; i += gridDim.x) {
    float ax = 0.f, ay = 0.f;
    for (int t = threadIdx.x; t < 1024; t += blockDim.x) {
      const long long n = 1024 * i + t;
      float2 zz = cmul(d.z[rmod(qlo + n, d.z_cap)], dds_rot_neg((unsigned long long)n * cp.inc));
      float2 z2 = cmul(zz, zz);
      float2 z4 = cmul(z2, z2);
      ax += z4.x; ay += z4.y;
    }
    double sx = warp_sum_d((double)ax), sy = warp_sum_d((double)ay);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(sx, sy);
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 a = make_double2(0.0, 0.0);
      for (int w = 0; w < 8; ++w) { a.x += red[w].x; a.y += red[w].y; }
      d.cfo_a[i] = a;
    }
    __syncthreads();
  }
}

// rho = sum_i a_{i+1} conj(a_i); df = df_c + arg(rho) f_s2 / (2 pi 4 1024); DDS increment and
// carried phase origin (c-8); z' becomes valid up to qhi.
__global__ void __launch_bounds__(1024) k_cfo_fine_final(RxDev d, long long beta, long long qlo, long long qhi) {
  __shared__ double2 red[32];
  const long long nch = (qhi - qlo) / 1024;
  double rx = 0.0, ry = 0.0;
  for (long long i = threadIdx.x; i + 1 < nch; i += blockDim.x) {
    const double2 a = d.cfo_a[i], b = d.cfo_a[i + 1];
    rx += b.x * a.x + b.y * a.y;
    ry += b.y * a.x - b.x * a.y;
  }
  rx = warp_sum_d(rx);
  ry = warp_sum_d(ry);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(rx, ry);
  __syncthreads();
  if (threadIdx.x == 0) {
    double sx = 0.0, sy = 0.0;
    for (int w = 0; w < 32; ++w) { sx += red[w].x; sy += red[w].y; }
    CfoParam cp = d.cfo[rmod(beta, d.buf_cap)];
    double df = cp.df;
    if (nch >= 2) df += atan2(sy, sx) * d.fs2 / (2.0 * 3.141592653589793 * 4.0 * 1024.0);
    if (d.cfo_enable) {
      cp.df = df;
      cp.inc = (unsigned long long)llrint(ldexp(df / d.fs2, 64));
      cp.origin = d.st->cfo_origin_next;
      d.st->cfo_origin_next = cp.origin + (unsigned long long)((long long)d.buffer_blocks * 256) * cp.inc;
      d.st->cfo_df_prev = df;
    } else {
      cp.df = 0.0; cp.inc = 0ull; cp.origin = 0ull;
    }
    d.cfo[rmod(beta, d.buf_cap)] = cp;
  }
}

// z'_q = z_q / sqrt(P_beta) e^{-j psi'_q}, psi' the carried per-buffer CFO DDS (c-8),
// materialised once per buffer into the z' ring that the sync / LMS stages read.
__global__ void __launch_bounds__(256) k_kk_zprime(RxDev d, long long beta, long long qlo, long long qhi) {
  const CfoParam cp = d.cfo[rmod(beta, d.buf_cap)];
  if (blockIdx.x == 0 && threadIdx.x == 0) d.st->v_front = qhi;   // consumed by later launches
  for (long long q = qlo + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < qhi;
       q += (long long)gridDim.x * blockDim.x) {
    float2 zz = cscale(d.z[rmod(q, d.z_cap)], cp.inv_sqrtP);
    if (d.cfo_enable) zz = cmul(zz, dds_rot_neg(cp.origin + (unsigned long long)(q - qlo) * cp.inc));
    d.zp[rmod(q, d.zp_cap)] = zz;
  }
}
