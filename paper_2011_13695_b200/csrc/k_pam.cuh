// k_pam.cuh — IMDD PAM-N chain kernels (§III).
//
//  k_pam_fe     H0-H3  ingest + overlap framing + R2C FFT-1024 + static FD EQ + C_b
//  k_pam_theta/carry/tau  H4  105-block complex average + atan2 + unwrap as a prefix sum of
//                      wrapped differences (tile-local scans, one-CTA carry scan) -> tau_b, M_b
//  k_pam_be     H2,H5-H7  stored spectrum + EQ + FD clock correction + C2R IFFT + extraction
//  k_norm_*     H8     buffer-wise DC / amplitude normalisation (stats + apply)
#pragma once
#include "fft.cuh"
#include "rx_dev.cuh"

// PAM_TW_GLOBAL = 1: k_pam_fe / k_pam_be read the twiddle table from global memory (L1) instead of
// staging 8 KiB into shared memory per CTA of 4 blocks
#ifndef PAM_TW_GLOBAL
#define PAM_TW_GLOBAL 1      // measured: C2 67.7 -> 71.9 GSa/s, u / u^ / labels bit-identical
#endif
#if PAM_TW_GLOBAL
#define PAM_TW_WAIT() __syncthreads()
#else
#define PAM_TW_WAIT() tw_wait()
#endif
#ifndef FE_GROUPS
#define FE_GROUPS 4
#endif

__device__ __forceinline__ float code_lo(uint32_t w) {     // exact float of the low 16 bits
  return __uint_as_float((w & 0xFFFFu) | 0x4B000000u) - 8388608.0f;
}
__device__ __forceinline__ float code_hi(uint32_t w) {
  return __uint_as_float((w >> 16) | 0x4B000000u) - 8388608.0f;
}

// Thread j of a block's group receives v[r] = (x[2(j + 64 r)], x[2(j + 64 r) + 1]) of block b's
// frame (input [512b-512, 512b+512)) directly in registers: the FFT's pass-1 operands. The
// block owns the frame's second half (r >= 4): those samples are counted for clipping and
// appended to the history ring when they are the call's tail.
__device__ __forceinline__ int load_block_regs(const InView &in, long long b, float scale, int j,
                                               float2 (&v)[8]) {
  const long long p0 = 512 * b - 512;
  const float off = -2047.5f * scale;
  int clip = 0;
  if (in.f32) {   // RX_IN_F32: x = sample * gain, no clip count; float history ring
    if (p0 >= in.call_start && p0 + 1024 <= in.call_end) {
      const float2 *src = reinterpret_cast<const float2 *>(in.curf + (p0 - in.call_start));
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float2 w = __ldg(src + j + 64 * r);
        v[r] = make_float2(w.x * in.gain, w.y * in.gain);
        const long long p = p0 + 2 * (j + 64 * r);
        if (r >= 4 && p >= in.keep_from)
          reinterpret_cast<float2 *>(in.histf_w)[(p & (in.hist_cap - 1)) >> 1] = w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const long long p = p0 + 2 * (j + 64 * r);
        v[r] = make_float2(in_xf(in, p), in_xf(in, p + 1));
        if (r >= 4 && p >= in.keep_from && p >= in.call_start)   // (the call's own samples)
          reinterpret_cast<float2 *>(in.histf_w)[(p & (in.hist_cap - 1)) >> 1] =
              make_float2(in.curf[p - in.call_start], in.curf[p + 1 - in.call_start]);
      }
    }
    return 0;
  }
  if (p0 >= in.call_start && p0 + 1024 <= in.call_end) {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(in.cur + (p0 - in.call_start));
    uint32_t w[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) w[r] = __ldg(src + j + 64 * r);
#pragma unroll
    for (int r = 0; r < 8; ++r) {   // (code - 2047.5) scale as one FADD2 (exact codes) + one FFMA2
      const float2 c = __fadd2_rn(make_float2(__uint_as_float((w[r] & 0xFFFFu) | 0x4B000000u),
                                              __uint_as_float((w[r] >> 16) | 0x4B000000u)),
                                  make_float2(-8388608.0f, -8388608.0f));
      v[r] = __ffma2_rn(c, make_float2(scale, scale), make_float2(off, off));
    }
    // clipped codes (0 or 4095) per 16-bit half: (c + 1) & 0xFFE is 0 exactly for those, and
    // adding 0x7FFF sets bit 15 of every other half (no carry between halves: halves < 0x1000)
#pragma unroll
    for (int r = 4; r < 8; ++r) {
      const uint32_t u = (w[r] + 0x00010001u) & 0x0FFE0FFEu;
      clip += 2 - __popc((u + 0x7FFF7FFFu) & 0x80008000u);
    }
    if (p0 + 1024 > in.keep_from) {   // the call's tail: append the owned half to the history ring
#pragma unroll
      for (int r = 4; r < 8; ++r) {
        const long long p = p0 + 2 * (j + 64 * r);
        if (p >= in.keep_from)
          reinterpret_cast<uint32_t *>(in.hist_w)[(p & (in.hist_cap - 1)) >> 1] = w[r];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float x[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long long p = p0 + 2 * (j + 64 * r) + e;
        bool pad;
        const int c = in_code(in, p, pad);
        x[e] = pad ? 0.f : fmaf((float)c, scale, off);
        if (!pad && r >= 4) clip += (c == 0 || c == 4095);
        // every owned sample of the call reaches the history ring, also when its block's frame
        // starts in an earlier call (k_kk_fe recomputes stage-1 blocks up to 1536 samples back)
        if (r >= 4 && p >= in.keep_from && p >= in.call_start) in.hist_w[p & (in.hist_cap - 1)] = (uint16_t)c;
      }
      v[r] = make_float2(x[0], x[1]);
    }
  }
  return clip;
}

__device__ __forceinline__ void block_reduce_clip(DevState *st, int clip) {
  clip = __reduce_add_sync(0xffffffffu, clip);
  if ((threadIdx.x & 31) == 0 && clip) atomicAdd((unsigned long long *)&st->clipped, (unsigned long long)clip);
}

// ------------------------------------------------------------------ H0-H3
// HREAL: the static-EQ spectrum is real (zero-phase symmetric real taps, the PAM case) and is
// applied as a real scale per bin.
template <bool HREAL>
__global__ void __launch_bounds__(256, 6) k_pam_fe(RxDev d, InView in, long long b0, long long b1) {   // 6 CTAs / SM: <= 40 registers
#if PAM_TW_GLOBAL
  const float2 *const tw = d.tw;   // twiddles from L1 / L2 (no per-CTA staging)
#else
  __shared__ float2 tws[1024];
  const float2 *const tw = tws;
#endif
  __shared__ float2 buf[FE_GROUPS][FFT_PAD_N];
  __shared__ double2 red[FE_GROUPS][2];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
#if !PAM_TW_GLOBAL
  tw_stage_async(tws, d.tw);   // waited for (tw_wait) before the first FFT pass
#endif
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  const bool act = b < b1;
  int clip = 0;
  float2 v[8];
  if (act) clip = load_block_regs(in, b, d.scale, j, v);
  else {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = make_float2(0.f, 0.f);
  }
  if (b < in.cnt_lo || b >= in.cnt_hi) clip = 0;   // a time shard's halo block: counted by its owner
  block_reduce_clip(d.st, clip);
  PAM_TW_WAIT();
  fft512_regs<false>(buf[g], j, tw, v);
  fft512_publish_upper(buf[g], j, v);
  // C_b = sum_{k<512} Y[k] conj(Y[k+512]) = Y0 conj(Y512) + Y256^2 + 2 sum_{k=1}^{255} Y[k] Y[512-k]
  // (per-thread fp32 partials of 4-5 terms, fp64 across threads)
  float cr = 0.f, ci = 0.f;
  if (act) {
    const float2 *pm = fft_mirror_base(buf[g], j);
    float2 *xs = d.Xspec + rmod(b, d.xs_cap) * 512;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = j + 64 * r;
      float2 Xk, Xn;
      r2c_pair(v[r], fft_partner(pm, j, r, v), tw[k], Xk, Xn);
      // X for k_pam_be (slot 0 packs the real X[0], X[512]; slot k < 512 holds X[k])
      if (k == 0) xs[0] = make_float2(Xk.x, Xn.x);
      else { xs[k] = Xk; xs[512 - k] = Xn; }
      float2 Yk, Yn;
      if (HREAL) { Yk = cscale(Xk, __ldg(d.Hr + k)); Yn = cscale(Xn, __ldg(d.Hr + 512 - k)); }
      else { Yk = cmul(Xk, __ldg(d.H + k)); Yn = cmul(Xn, __ldg(d.H + 512 - k)); }
      if (k == 0) { cr = fmaf(Yk.x, Yn.x, fmaf(Yk.y, Yn.y, cr)); ci = fmaf(Yk.y, Yn.x, fmaf(-Yk.x, Yn.y, ci)); }
      else {
        cr = fmaf(2.f * Yk.x, Yn.x, fmaf(-2.f * Yk.y, Yn.y, cr));
        ci = fmaf(2.f * Yk.x, Yn.y, fmaf(2.f * Yk.y, Yn.x, ci));
      }
    }
    if (j == 0) {
      const float2 Z = v[4];                                   // X[256] = conj Z[256]
      xs[256] = cconj(Z);
      const float2 Y = HREAL ? cscale(cconj(Z), __ldg(d.Hr + 256)) : cmul(cconj(Z), __ldg(d.H + 256));
      cr = fmaf(Y.x, Y.x, fmaf(-Y.y, Y.y, cr));
      ci = fmaf(2.f * Y.x, Y.y, ci);
    }
  }
  const double dr = warp_sum_d((double)cr), di = warp_sum_d((double)ci);
  if ((threadIdx.x & 31) == 0) red[g][(threadIdx.x >> 5) & 1] = make_double2(dr, di);
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
//            the paper's serial single-warp unwrap, telescoped: theta^u_b = theta_b -
//            2 pi N_b, N_b = sum_{i<=b} rint((theta_i - theta_{i-1}) / 2 pi), an integer scan
//            (exact in any order: call and shard boundaries cannot change it, DESIGN R-UNWRAP)
//   tau_b = -theta^u_b / 2 pi = N_b - theta_b / 2 pi ; M_b = ceil(256 b - 128 - tau_b)
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

// Three launches, all but (b) fully parallel:
// (a) k_pam_theta: one CTA per 256 blocks. Cbar_b from a shared-memory C tile (+2h halo),
//     theta_b = atan2(Cbar_b) (|Cbar| = 0 inherits the previous phase), the wrap counts
//     n_b = rint((theta_b - theta_{b-1}) / 2 pi) and their CTA-local inclusive prefix.
// (b) k_pam_carry: one CTA scans the CTA totals -> per-CTA offsets (+ the call's carry).
// (c) k_pam_tau: N_b = offset + local prefix, tau_b = N_b - theta_b / 2 pi, M_b.
#define CLK_TILE 256
// tau_b and M_b from the integer wrap count N_b and the resolved phase theta_b: one expression
// for every path (fused, three-launch, time shard), so all of them give identical bits
__device__ __forceinline__ double clk_tau(double N, double th) {
  return __fma_rn(-th, 0.15915494309189533577, N);
}
__device__ __forceinline__ long long clk_mb(long long b, double tau) {
  return (long long)ceil(__dsub_rn(__dsub_rn(256.0 * (double)b, 128.0), tau));
}
__device__ __forceinline__ double theta_of(const double2 *Ct, int i, int hh) {   // window at tile i
  // 4 interleaved partial sums (independent add chains), combined in a fixed order
  double sr[4] = {0.0, 0.0, 0.0, 0.0}, si[4] = {0.0, 0.0, 0.0, 0.0};
  const int n = 2 * hh + 1;
  int k = 0;
  for (; k + 4 <= n; k += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) { const double2 c = Ct[i + k + u]; sr[u] += c.x; si[u] += c.y; }
  }
  for (; k < n; ++k) { const double2 c = Ct[i + k]; sr[0] += c.x; si[0] += c.y; }
  const double r = (sr[0] + sr[1]) + (sr[2] + sr[3]), m = (si[0] + si[1]) + (si[2] + si[3]);
  return (r == 0.0 && m == 0.0) ? __longlong_as_double(0x7ff8000000000000LL) : atan2(m, r);
}

// FUSED = true: one launch does (a)-(c). Tile t publishes its total (tagged with the launch id),
// then forms its offset from the call carry plus the totals of tiles 0..t-1 summed in a fixed
// order (deterministic; every tile waits only for totals, so nothing is chained), and finishes
// tau / M itself. Needs every tile co-resident (the host falls back to three launches for
// more than CLK_FUSE_MAX tiles).
#define CLK_FUSE_MAX 512
template <bool FUSED>
__global__ void __launch_bounds__(CLK_TILE) k_pam_theta(RxDev d, long long b0, long long b1, long long blast,
                                                        long long launch_id) {
  extern __shared__ double2 Ct[];                 // [CLK_TILE + 1 + 2 h]: blocks base-1-h ..
  pdl_wait();                                     // C_b from k_pam_fe
  __shared__ double th_sh[CLK_TILE + 1];
  __shared__ double wsum[CLK_TILE / 32];
  __shared__ long long wmax[CLK_TILE / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, hh = d.clock_half;
  const double INV_2PI = 0.15915494309189533577;
  // FUSED: the tile index is taken in dispatch order from a counter (clk_ticket[1]), not from
  // blockIdx, so a tile only ever waits on tiles that are already resident (decoupled look-back
  // ordering; no reliance on blockIdx-ordered CTA dispatch)
  __shared__ int tile_sh;
  if (FUSED) {
    if (t == 0) tile_sh = atomicAdd(d.clk_ticket + 1, 1);
    __syncthreads();
  }
  const int tile = FUSED ? tile_sh : (int)blockIdx.x;
  const long long base = b0 + (long long)tile * CLK_TILE;
  for (int i = t; i < CLK_TILE + 1 + 2 * hh; i += blockDim.x) {
    const long long b = base - 1 - hh + i;
    Ct[i] = (b >= 0 && b <= blast) ? d.C[rmod(b, d.blk_cap)] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // theta of blocks base-1+i, i = 0..CLK_TILE (entry 0 = the previous block, for the difference)
  th_sh[t + 1] = (base + t < b1) ? theta_of(Ct, t + 1, hh) : __longlong_as_double(0x7ff8000000000000LL);
  if (t == 0) {
    double p = __longlong_as_double(0x7ff8000000000000LL);
    if (base - 1 >= b0) p = theta_of(Ct, 0, hh);
    th_sh[0] = p;
  }
  __syncthreads();
  const long long b = base + t;
  // resolve inherited phases: last valid theta at or before each entry (max-scan of indices)
  long long last = isnan(th_sh[t + 1]) ? -1 : t + 1;
  long long inc = last;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o && v > inc) inc = v;
  }
  if (lane == 31) wmax[warp] = inc;
  __syncthreads();
  long long pre = -1;
  for (int w = 0; w < warp; ++w) pre = wmax[w] > pre ? wmax[w] : pre;
  long long excl = __shfl_up_sync(0xffffffffu, inc, 1);   // all lanes shuffle
  if (lane == 0) excl = -1;
  long long src_prev = excl > pre ? excl : pre;          // last valid entry before t+1 in tile
  long long src_cur = inc > pre ? inc : pre;             // last valid entry at or before t+1
  // entry 0 (previous block) and anything before the tile: walk back through global theta
  auto resolve_before = [&](void) -> double {
    if (!isnan(th_sh[0])) return th_sh[0];
    for (long long q = base - 2; q >= b0; --q) {         // rare: |Cbar| = 0 runs; recompute
      double sr = 0.0, si = 0.0;                         // from C (other tiles may not have
      for (long long k = q - hh; k <= q + hh; ++k)       // written theta yet)
        if (k >= 0 && k <= blast) { const double2 c = d.C[rmod(k, d.blk_cap)]; sr += c.x; si += c.y; }
      if (!(sr == 0.0 && si == 0.0)) return atan2(si, sr);
    }
    return d.st->theta_prev;                             // resolved phase before this call
  };
  const double tprev = src_prev >= 1 ? th_sh[src_prev] : resolve_before();
  const double tcur = src_cur >= 1 ? th_sh[src_cur] : resolve_before();
  double diff = 0.0;                                     // n_b (an integer, held in a double)
  if (b < b1) {
    const double dd = tcur - tprev;
    diff = rint(dd * INV_2PI);
    if (b == 0) diff = 0.0;                              // theta^u_0 = theta_0: N_0 = 0
  }
  // CTA-local inclusive prefix of the wrap counts (integer sums: exact)
  double incl = diff;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  double off = 0.0;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  if (!FUSED && b < b1) {                                // local prefix (finished by k_pam_tau)
    d.tau[rmod(b, d.blk_cap)] = off + incl;
    d.theta[rmod(b, d.blk_cap)] = tcur;
  }
  if (t == CLK_TILE - 1) {
    double tot = 0.0;
    for (int w = 0; w < CLK_TILE / 32; ++w) tot += wsum[w];
    d.clk_part[tile] = tot;
    d.clk_last[tile] = tcur;                             // resolved phase of the tile's last block
    if (FUSED) {
      __threadfence();
      atomicExch((unsigned long long *)&d.clk_flag[tile], (unsigned long long)launch_id);
    }
  }
  if constexpr (FUSED) {
    // tile offset = carry + sum_{t' < tile} tot_t' (lane-strided then fixed tree: deterministic)
    __shared__ double tile_off;
    if (warp == 0) {
      double acc = 0.0;
      for (int i = lane; i < tile; i += 32) {
        while (((volatile long long *)d.clk_flag)[i] != launch_id) { }
        __threadfence();
        acc += ((volatile double *)d.clk_part)[i];
      }
      acc = warp_sum_d(acc);
      if (lane == 0) tile_off = d.st->wraps_prev + acc;
    }
    __syncthreads();
    const double Nb = tile_off + off + incl;
    if (b < b1) {
      const double tau = clk_tau(Nb, tcur);
      d.tau[rmod(b, d.blk_cap)] = tau;
      d.Mb[rmod(b, d.blk_cap)] = clk_mb(b, tau);
    }
    // the last tile to finish (every tile has read the call's carry by then) advances the carry:
    // wraps_prev += sum of the tile totals, theta_prev = the call's last resolved phase
    __shared__ int last_tile;
    __syncthreads();
    if (t == 0) {
      __threadfence();
      last_tile = atomicAdd(d.clk_ticket, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last_tile && warp == 0) {
      __threadfence();
      double acc = 0.0;
      for (int i = lane; i < (int)gridDim.x; i += 32) acc += ((volatile double *)d.clk_part)[i];
      acc = warp_sum_d(acc);
      if (lane == 0) {
        d.st->wraps_prev += acc;
        d.st->theta_prev = ((volatile double *)d.clk_last)[gridDim.x - 1];
        d.clk_ticket[0] = 0;
        d.clk_ticket[1] = 0;                             // every tile has taken its index
      }
    }
  }
  (void)INV_2PI;
}

// (b) offsets of the tiles (exclusive scan of the tile totals, plus the carried unwrapped phase)
__global__ void __launch_bounds__(1024) k_pam_carry(RxDev d, int ntiles) {
  __shared__ double ws[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double carry = d.st->wraps_prev;
  for (int c0 = 0; c0 < ntiles; c0 += 1024) {
    const int i = c0 + t;
    const double v = i < ntiles ? d.clk_part[i] : 0.0;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    double off = 0.0;
    for (int w = 0; w < warp; ++w) off += ws[w];
    double tot = 0.0;
    for (int w = 0; w < 32; ++w) tot += ws[w];
    if (i < ntiles) d.clk_off[i] = carry + off + incl - v;
    __syncthreads();
    carry += tot;
  }
  if (t == 0) {
    d.st->wraps_prev = carry;
    d.st->theta_prev = d.clk_last[ntiles - 1];
  }
}

// (c) tau_b and M_b
__global__ void __launch_bounds__(256) k_pam_tau(RxDev d, long long b0, long long b1) {
  const long long b = b0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= b1) return;
  const int tile = (int)((b - b0) / CLK_TILE);
  const double Nb = d.clk_off[tile] + d.tau[rmod(b, d.blk_cap)];
  const double tau = clk_tau(Nb, d.theta[rmod(b, d.blk_cap)]);
  d.tau[rmod(b, d.blk_cap)] = tau;
  d.Mb[rmod(b, d.blk_cap)] = clk_mb(b, tau);
}

// ------------------------------------------------------------------ H1, H2, H5-H7
template <bool HREAL>
__global__ void __launch_bounds__(256) k_pam_be(RxDev d, long long b0, long long b1) {
#if PAM_TW_GLOBAL
  const float2 *const tw = d.tw;   // twiddles from L1 / L2 (no per-CTA staging)
#else
  __shared__ float2 tws[1024];
  const float2 *const tw = tws;
#endif
  __shared__ float2 buf[FE_GROUPS][FFT_PAD_N];
  __shared__ double red[FE_GROUPS][2];
  const int g = threadIdx.x >> 6, j = threadIdx.x & 63;
#if !PAM_TW_GLOBAL
  tw_stage_async(tws, d.tw);   // waited for (tw_wait) before the first FFT pass
#endif
  pdl_wait();                 // tau_b / M_b from the clock stage
  const long long b = b0 + (long long)blockIdx.x * FE_GROUPS + g;
  const bool act = b < b1;
  // the block's spectrum X stored by k_pam_fe (SURVEY §8(a) 'read back spectra' option):
  // thread j owns the pairs (k, 512 - k), k = j + 64 r, r < 4, and thread 0 also X[256]
  float2 Xk_[4], Xn_[4], X256 = make_float2(0.f, 0.f);
  {
    const float2 *xs = d.Xspec + rmod(act ? b : b0, d.xs_cap) * 512;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = j + 64 * r;
      const float2 a = act ? xs[k] : make_float2(0.f, 0.f);
      const float2 c = act ? xs[(512 - k) & 511] : make_float2(0.f, 0.f);
      if (k == 0) { Xk_[r] = make_float2(a.x, 0.f); Xn_[r] = make_float2(a.y, 0.f); }
      else { Xk_[r] = a; Xn_[r] = c; }
    }
    if (j == 0 && act) X256 = xs[256];
  }
  // clock phase of this block: s = 2 tau, i_b = rint(s), f_b = s - i_b   (c-4)
  const double tau = act ? d.tau[rmod(b, d.blk_cap)] : 0.0;
  const double sd = 2.0 * tau;
  const double ibd = rint(sd);
  const float f = (float)(sd - ibd);
  // FD clock correction Y'[k] = Y[k] e^{+j pi kappa(k) f / 512}: rotations for k = j + 64 r from
  // base e^{j pi j f/512} and step e^{j pi f/8}; the partner 512-k is e^{j pi f} conj(rot(k))
  float2 rot, step, nyq;
  sincospif((float)j * f * (1.0f / 512.0f), &rot.y, &rot.x);
  sincospif(f * 0.125f, &step.y, &step.x);
  sincospif(f, &nyq.y, &nyq.x);
  float2 Zk[4], Zn[4], Z256;
  PAM_TW_WAIT();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = j + 64 * r;
    const float2 Xk = Xk_[r], Xn = Xn_[r];
    float2 Yk, Yn;
    if (HREAL) { Yk = cscale(Xk, __ldg(d.Hr + k)); Yn = cscale(Xn, __ldg(d.Hr + 512 - k)); }
    else { Yk = cmul(Xk, __ldg(d.H + k)); Yn = cmul(Xn, __ldg(d.H + 512 - k)); }
    Yk = cmul(Yk, rot);
    if (k == 0) Yn = make_float2(Yn.x * nyq.x + Yn.y * nyq.y, 0.0f);   // Nyquist: Re(Y e^{-j pi f})
    else Yn = cmul(Yn, cmulc(nyq, rot));
    c2r_pair<false>(Yk, Yn, tw[k], Zk[r], Zn[r]);   // without its exact 1/2 (x2 folded into 1/1024 below)
    rot = cmul(rot, step);
  }
  {
    float2 Y = HREAL ? cscale(X256, __ldg(d.Hr + 256)) : cmul(X256, __ldg(d.H + 256));
    float2 r256;
    sincospif(0.5f * f, &r256.y, &r256.x);
    Z256 = cscale(cconj(cmul(Y, r256)), 2.0f);      // (the packing's x2)
  }
  {
    float2 *paw = buf[g] + j;                   // natural layout
    float2 *pmw = buf[g] + (512 - j);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      paw[64 * r] = Zk[r];
      if (!(j == 0 && r == 0)) pmw[-64 * r] = Zn[r];
    }
    if (j == 0) buf[g][256] = Z256;
  }
  __syncthreads();
  float2 v[8];
  fft512<true>(buf[g], j, tw, v);
  fft512_store(buf[g], j, v);
  // variable-rate extraction (c-4): u_m = y[2m + i_b - 512b + 512], m in [max(M_b,0), M_{b+1})
  double part = 0.0;
  if (act) {
    const long long Mb = d.Mb[rmod(b, d.blk_cap)], Mb1 = d.Mb[rmod(b + 1, d.blk_cap)];
    const long long lo = Mb > 0 ? Mb : 0;
    const int base2 = (int)(2 * lo + (long long)ibd - 512 * b + 512);   // local index of m = lo
    const int cnt = (int)(Mb1 - lo);
    float ps = 0.f;
    for (int t = j; t < cnt; t += 64) {
      const long long m = lo + t;
      int loc = base2 + 2 * t;                                        // 2m + i_b - 512b + 512
      if (loc < 0 || loc >= 1024) { set_flag(d.st, 8); loc = loc < 0 ? 0 : 1023; }
      const int n = loc >> 1;
      const float2 zz = buf[g][n];                 // natural layout
      const float y = ((loc & 1) ? zz.y : zz.x) * (1.0f / 1024.0f);
      d.u[rmod(m, d.sym_cap)] = y;
      ps += y;
    }
    part = (double)ps;
  }
  part = warp_sum_d(part);
  if ((threadIdx.x & 31) == 0) red[g][(threadIdx.x >> 5) & 1] = part;
  __syncthreads();
  if (act && j == 0) d.blk_sum[rmod(b, d.blk_cap)] = red[g][0] + red[g][1];
}

// Buffer-wise normalisation (P:167 'three kernels: initialization, estimation of the DC-offset,
// and estimation of the amplitude'; c-5): dc = mean u, A = mean|u - dc| / (M / (2 (M-1))),
// u^ = (u - dc) / A over the symbols emitted by each buffer's blocks. Reductions are fixed
// order (deterministic).
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

// (1) k_norm_stats: grid (nbuf x G). CTA (buffer bi, part g): dc from the buffer's per-block
//     sums (every CTA reduces them in the same fixed order), then the partial sum |u - dc| over
//     its contiguous symbol range; the last CTA of the buffer (atomic ticket) reduces the
//     partials in index order -> A. (2) k_norm_apply: u^ = (u - dc)/A, elementwise.
#define NORM_G 64
__global__ void __launch_bounds__(1024) k_norm_stats(RxDev d, long long beta0, long long be_done, int flush) {
  __shared__ double sh[32];
  __shared__ int ticket;
  const int g = blockIdx.x, t = threadIdx.x;
  const long long beta = beta0 + blockIdx.y;
  const long long blo = beta * d.buffer_blocks;
  long long bhi = blo + d.buffer_blocks;
  if (bhi > be_done) bhi = be_done;
  // dc over the whole buffer (fixed order: thread-strided, then the fixed block tree)
  double s = 0.0;
  for (long long b = blo + t; b < bhi; b += blockDim.x) s += d.blk_sum[rmod(b, d.blk_cap)];
  s = block_sum_det(s, sh);
  const long long mlo = sym_lo_of(d, blo), mhi0 = sym_lo_of(d, bhi);
  const long long mhi = mhi0 > mlo ? mhi0 : mlo;
  const double Cn = (double)(mhi - mlo);
  const double dc = Cn > 0.0 ? s / Cn : 0.0;
  // partial |u - dc| over this CTA's share of the symbols
  const long long n = mhi - mlo;
  const long long m0 = mlo + n * g / NORM_G, m1 = mlo + n * (g + 1) / NORM_G;
  double a = 0.0;
  {
    const long long a0 = (m0 + 3) & ~3LL, a1 = m1 & ~3LL;
    const long long h1 = a0 < m1 ? a0 : m1;
    if (m0 + t < h1) a += fabs((double)d.u[rmod(m0 + t, d.sym_cap)] - dc);
    const long long tl = a1 > h1 ? a1 : h1;
    if (tl + t < m1) a += fabs((double)d.u[rmod(tl + t, d.sym_cap)] - dc);
    double a2 = 0.0;
    for (long long q = a0 / 4 + t; q < a1 / 4; q += blockDim.x) {
      const float4 x = *reinterpret_cast<const float4 *>(d.u + rmod(4 * q, d.sym_cap));
      a += fabs((double)x.x - dc) + fabs((double)x.y - dc);
      a2 += fabs((double)x.z - dc) + fabs((double)x.w - dc);
    }
    a += a2;
  }
  a = block_sum_det(a, sh);
  double *part = d.norm_part + (blockIdx.y % 16) * NORM_G;
  if (t == 0) {
    part[g] = a;
    __threadfence();
    ticket = atomicAdd(&d.norm_tick[blockIdx.y % 16], 1);
  }
  __syncthreads();
  if (ticket != NORM_G - 1) return;
  __threadfence();
  if (t < 32) {
    double pa = 0.0;
    for (int i = t; i < NORM_G; i += 32) pa += ((volatile double *)part)[i];
    pa = warp_sum_d(pa);
    if (t == 0) {
      const double mal = (double)d.M / (2.0 * (double)(d.M - 1));
      double A = Cn > 0.0 ? (pa / Cn) / mal : 1.0;
      if (!(A > 0.0)) A = 1.0;
      d.norm_dc[rmod(beta, d.buf_cap)] = dc;
      d.norm_amp[rmod(beta, d.buf_cap)] = A;
      d.norm_cnt[rmod(beta, d.buf_cap)] = (long long)Cn;
      d.norm_tick[blockIdx.y % 16] = 0;
    }
  }
  (void)flush;
}

// u^ over the symbols of buffers [beta0, beta0 + nbuf): grid (NORM_AG, nbuf), CTA (g, y) scales
// its share of buffer beta0 + y with that buffer's (dc, 1/A), 4 symbols per thread-step (float4
// where the absolute index is 4-aligned); advances the front (and m_end at flush)
#define NORM_AG 128
__global__ void __launch_bounds__(256) k_norm_apply(RxDev d, long long beta0, long long nbuf, long long be_done,
                                                   int flush) {
  const long long beta = beta0 + blockIdx.y;
  const long long blo = beta * d.buffer_blocks;
  long long bhi = blo + d.buffer_blocks;
  if (bhi > be_done) bhi = be_done;
  const long long mlo = sym_lo_of(d, blo);
  const long long mhi = sym_lo_of(d, bhi) > mlo ? sym_lo_of(d, bhi) : mlo;
  const float dc = (float)d.norm_dc[rmod(beta, d.buf_cap)];
  const float inv = (float)(1.0 / d.norm_amp[rmod(beta, d.buf_cap)]);
  const long long a0 = (mlo + 3) & ~3LL, a1 = mhi & ~3LL;
  const int t = threadIdx.x;
  if (blockIdx.x == 0) {   // unaligned head / tail
    const long long h1 = a0 < mhi ? a0 : mhi;
    if (mlo + t < h1) { const long long i = rmod(mlo + t, d.sym_cap); d.uhat[i] = (d.u[i] - dc) * inv; }
    const long long tl = a1 > h1 ? a1 : h1;
    if (tl + t < mhi) { const long long i = rmod(tl + t, d.sym_cap); d.uhat[i] = (d.u[i] - dc) * inv; }
  }
  for (long long q = a0 / 4 + (long long)blockIdx.x * blockDim.x + t; q < a1 / 4;
       q += (long long)gridDim.x * blockDim.x) {
    const long long i = rmod(4 * q, d.sym_cap);
    const float4 x = *reinterpret_cast<const float4 *>(d.u + i);
    *reinterpret_cast<float4 *>(d.uhat + i) =
        make_float4((x.x - dc) * inv, (x.y - dc) * inv, (x.z - dc) * inv, (x.w - dc) * inv);
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && t == 0) {
    long long bend = (beta0 + nbuf) * d.buffer_blocks;
    if (bend > be_done) bend = be_done;
    const long long mend = sym_lo_of(d, bend) > mlo ? sym_lo_of(d, bend) : mlo;
    d.st->v_front = mend;
    if (flush && bend == be_done) d.st->m_end = mend;
  }
}
