// k_shard.cuh — time sharding of one stream (SURVEY §8(e) mode 2): the per-round carry record
// of a shard and the small kernels around it. Shard g of N owns paper buffers beta = g mod N
// (2^22-sample buffers), reads its input halos itself and exchanges one record per round
// (rx_export_carry -> NCCL all-gather by the caller -> rx_import_carry). The record carries
// exactly the quantities that cross buffer boundaries in the chain:
//  KK (c-7, c-8): the CFO estimate (P, df, k*) of the buffer estimated this round; every shard
//    rebuilds the DDS origin chain origin_{b+1} = origin_b + Q inc_b from all of them;
//  PAM (c-3, c-5): the clock-phase wrap count over the buffer's own blocks (the
//    unwrap carries the previous buffer's phase; with theta^u_b = theta_b - 2 pi N_b the carry
//    is the integer N, an exclusive scan over the buffers) and the normalisation scalars (dc, A)
//    of the buffer normalised at the previous import (its neighbours' halo symbols use them);
//  both: the frame-sync result and the trained taps from the shard holding the stream start
//    (c-10, c-9 'Training'), and the lag-D seed partial sums (c-9 'Seed') of the segments the
//    shard finalised in its last round (exact fixed-point sums: an epoch split between shards
//    gets the single stream's seed, k_lms.cuh seed_acc_add).
#pragma once
#include "k_lms.cuh"

struct RxCarry {
  long long beta;                       // buffer whose stage A ran this round (-1: none)
  double P, df;                         // KK: its CFO estimate
  int kstar, flags;                     // flags bit 0: sync + training valid; bit 1: norm valid
  int sync_offset, sync_phase, sync_polarity, pad;
  double sync_gamma, sync_phi0;
  float2 w_train[RX_MAX_K], v_train[RX_MAX_K];
  double wraps;                         // PAM: sum of n_b over the buffer's own blocks
  long long norm_beta;                  // PAM: the buffer normalised at the previous import
  double norm_dc, norm_amp;
  long long norm_cnt;
  SeedPart part[RX_CARRY_SEEDS];        // seed partials of the last stage B round
};

// one thread: the shard's record of this round (and the seed partials are consumed)
__global__ void k_carry_export(RxDev d, RxCarry *out, long long beta, long long norm_beta) {
  RxCarry *c = out;
  c->beta = beta;
  c->P = c->df = 0.0;
  c->kstar = 0;
  c->flags = 0;
  c->wraps = 0.0;
  if (beta >= 0) {
    if (d.family == 1) {
      const CfoParam cp = d.cfo[rmod(beta, d.buf_cap)];
      c->P = cp.P;
      c->df = cp.df;
      c->kstar = cp.kstar;
    } else {
      c->wraps = d.st->sh_w;
    }
  }
  c->norm_beta = norm_beta;
  if (norm_beta >= 0) {
    c->flags |= 2;
    c->norm_dc = d.norm_dc[rmod(norm_beta, d.buf_cap)];
    c->norm_amp = d.norm_amp[rmod(norm_beta, d.buf_cap)];
    c->norm_cnt = d.norm_cnt[rmod(norm_beta, d.buf_cap)];
  }
  const DevState *st = d.st;
  if (st->synced && st->trained) {
    c->flags |= 1;
    c->sync_offset = st->sync_offset;
    c->sync_phase = st->sync_phase;
    c->sync_polarity = st->sync_polarity;
    c->sync_gamma = st->sync_gamma;
    c->sync_phi0 = st->sync_phi0;
    for (int k = 0; k < RX_MAX_K; ++k) {
      c->w_train[k] = d.w_train[k];
      c->v_train[k] = d.wl ? d.v_train[k] : make_float2(0.f, 0.f);
    }
  }
  for (int i = 0; i < RX_CARRY_SEEDS; ++i) {
    c->part[i] = d.seed_xp[i];
    d.seed_xp[i].epoch = -1;
  }
}

// one warp: every shard's record of the round, in rank order (= buffer order). KK CFO
// parameters go to the per-buffer table as cfo_final_block / k_cfo_fine leave them (the origin
// chain is then advanced by k_carry_chain); PAM wrap counts advance the running total (this
// shard's buffer my_beta takes the total before it as its base); normalisation scalars, sync /
// training and the other shards' seed partials are taken over.
__global__ void k_carry_import(RxDev d, const RxCarry *g, int n, int me, long long my_beta) {
  DevState *st = d.st;
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < n; ++i) {
    const RxCarry &c = g[i];
    if (lane == 0) {
      if (c.beta >= 0) {
        if (d.family == 1) {
          CfoParam cp;
          cp.P = c.P;
          cp.df = c.df;
          cp.kstar = c.kstar;
          cp.inv_sqrtP = (float)(1.0 / sqrt(c.P));
          cp.inc = (unsigned long long)llrint(ldexp(c.df / d.fs2, 64));
          cp.origin = 0ull;
          d.cfo[rmod(c.beta, d.buf_cap)] = cp;
        } else {
          if (c.beta == my_beta) st->sh_nbase = st->wrap_total;
          st->wrap_total += c.wraps;           // integers held in doubles: exact
        }
      }
      if (c.flags & 2) {
        d.norm_dc[rmod(c.norm_beta, d.buf_cap)] = c.norm_dc;
        d.norm_amp[rmod(c.norm_beta, d.buf_cap)] = c.norm_amp;
        d.norm_cnt[rmod(c.norm_beta, d.buf_cap)] = c.norm_cnt;
      }
      if ((c.flags & 1) && !st->trained) {
        st->sync_offset = c.sync_offset;
        st->sync_phase = c.sync_phase;
        st->sync_polarity = c.sync_polarity;
        st->sync_gamma = c.sync_gamma;
        st->sync_phi0 = c.sync_phi0;
        for (int k = 0; k < RX_MAX_K; ++k) {
          d.w_train[k] = c.w_train[k];
          if (d.wl) d.v_train[k] = c.v_train[k];
        }
        if (c.sync_gamma < d.sync_min) set_flag(st, RX_FLAG_SYNC_DEV);
        __threadfence();
        st->synced = 1;
        st->trained = 1;
        d.hm->synced = 1;
        d.hm->trained = 1;
      }
    }
    __syncwarp();
    if (i == me) continue;                   // this shard added its own partials already
    for (int j = 0; j < RX_CARRY_SEEDS; ++j) {
      const SeedPart &p = c.part[j];
      if (p.epoch < 0 || p.n <= 0) continue;
      seed_acc_add(d, p.epoch, p.n, p.sum[lane][0], p.sum[lane][1]);
      __syncwarp();
    }
  }
}

// KK: the DDS origin chain over the round's buffers in buffer order (k_cfo_carry's arithmetic)
__global__ void k_carry_chain(RxDev d, const RxCarry *g, int n) {
  for (int i = 0; i < n; ++i) {
    const long long b = g[i].beta;
    if (b < 0) continue;
    CfoParam cp = d.cfo[rmod(b, d.buf_cap)];
    const double df = cp.kstar >= 0 ? cp.df : d.st->cfo_df_prev;
    if (d.cfo_enable) {
      cp.df = df;
      cp.inc = (unsigned long long)llrint(ldexp(df / d.fs2, 64));
      cp.origin = d.st->cfo_origin_next;
      d.st->cfo_origin_next = cp.origin + (unsigned long long)((long long)d.buffer_blocks * 256) * cp.inc;
      d.st->cfo_df_prev = df;
    } else {
      cp.df = 0.0; cp.inc = 0ull; cp.origin = 0ull;
    }
    d.cfo[rmod(b, d.buf_cap)] = cp;
  }
}

// KK stage B of a time shard: z' valid below q_valid, finalisation front at the epoch's first segment
__global__ void k_shard_seek(RxDev d, long long q_valid, long long seg0) {
  d.st->v_front = q_valid;
  d.st->seg_next = seg0;
  d.hm->seg_next = seg0;
}

// ---- PAM
// N_loc(b) of the shard's clock pass over blocks [c_lo, ...) (k_pam_theta<false> + k_pam_carry
// with a zero carry): tile offset + local prefix
__device__ __forceinline__ double shard_nloc(const RxDev &d, long long c_lo, long long b) {
  return d.clk_off[(int)((b - c_lo) / CLK_TILE)] + d.tau[rmod(b, d.blk_cap)];
}
// after the clock pass of stage A: the reference (block beta B - 1) and the buffer's own wraps
__global__ void k_shard_wraps(RxDev d, long long beta, long long c_lo, long long own_hi) {
  const long long BB = d.buffer_blocks;
  const double nref = beta > 0 ? shard_nloc(d, c_lo, beta * BB - 1) : 0.0;
  d.st->sh_nref = nref;
  d.st->sh_w = own_hi > beta * BB ? shard_nloc(d, c_lo, own_hi - 1) - nref : 0.0;
}
// stage A2 (after the exchange): N_b = base + N_loc(b) - N_ref (exact integers), tau_b, M_b
// with the single stream's expressions (clk_tau / clk_mb)
__global__ void __launch_bounds__(256) k_shard_tau(RxDev d, long long c_lo, long long c_hi) {
  const long long b = c_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= c_hi) return;
  const double Nb = d.st->sh_nbase + (shard_nloc(d, c_lo, b) - d.st->sh_nref);
  const double tau = clk_tau(Nb, d.theta[rmod(b, d.blk_cap)]);   // (each thread reads and
  d.tau[rmod(b, d.blk_cap)] = tau;                                // rewrites its own block only)
  d.Mb[rmod(b, d.blk_cap)] = clk_mb(b, tau);
}
// the buffer's symbol bounds for its stage B: [0] first symbol of the pre-halo blocks, [1] M_lo,
// [2] M_hi (symbols of blocks [be_lo, beta B) / [beta B, be_hi))
__global__ void k_shard_bufm(RxDev d, long long beta, long long be_lo, long long be_hi) {
  long long *m = d.buf_m + rmod(beta, d.buf_cap) * 4;
  const long long BB = d.buffer_blocks;
  long long a = d.Mb[rmod(be_lo, d.blk_cap)], b = d.Mb[rmod(beta * BB, d.blk_cap)], c = d.Mb[rmod(be_hi, d.blk_cap)];
  a = a > 0 ? a : 0;
  b = b > 0 ? b : 0;
  c = c > b ? c : b;
  m[0] = a < b ? a : b;
  m[1] = b;
  m[2] = c;
}
// stage B: u^ of the pre-halo symbols [m0, M_lo) with the previous buffer's scalars (k_norm_apply's
// expression), then the finalisation front / readiness bound: segment s is this buffer's when
// its last tap position (s + 1) S - 1 + c lies in [M_lo, M_hi) (the single stream's readiness
// rule with v_front = M_hi: the previous buffer's shard ran every segment below M_lo)
__global__ void __launch_bounds__(256) k_shard_halo_norm(RxDev d, long long beta) {
  if (beta <= 0) return;
  const long long *m = d.buf_m + rmod(beta, d.buf_cap) * 4;
  const long long m0 = m[0], m1 = m[1];
  const float dc = (float)d.norm_dc[rmod(beta - 1, d.buf_cap)];
  const float inv = (float)(1.0 / d.norm_amp[rmod(beta - 1, d.buf_cap)]);
  for (long long q = m0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < m1; q += (long long)gridDim.x * blockDim.x) {
    const long long i = rmod(q, d.sym_cap);
    d.uhat[i] = (d.u[i] - dc) * inv;
  }
}
__global__ void k_shard_seek_pam(RxDev d, long long beta) {
  const long long *m = d.buf_m + rmod(beta, d.buf_cap) * 4;
  const long long S = d.S, c = d.K >> 1;
  long long s0 = 0;
  if (beta > 0) {
    const long long num = m[1] - c + 1;                  // s >= num / S - 1
    s0 = (num > 0 ? (num + S - 1) / S : 0) - 1;
    if (s0 < 0) s0 = 0;
  }
  d.st->v_front = m[2];
  d.st->seg_next = s0;
  d.hm->seg_next = s0;
}
// stage A clock pass of a PAM shard: zero carry (the local wrap counts are relative)
__global__ void k_shard_clk_reset(RxDev d) {
  d.st->wraps_prev = 0.0;
  d.st->theta_prev = 0.0;
}
