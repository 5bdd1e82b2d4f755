// fft.cuh — shared-memory radix-8 Stockham FFT-512 and the real<->complex packing that
// turns it into the 1024-point R2C/C2R transforms of the overlap-save stages
// (P:150 '100% overlap-save 1024-point FFT', P:218 'real-to-complex FFT', P:221 '512-point
// IFFT'). No cuFFT (north_star). One transform = 64 threads x 8 points, 3 radix-8 passes,
// natural-order output (Stockham autosort). Unnormalised in both directions.
#pragma once
#include "common.cuh"

#define FFT_PAD_N 576   // 512 float2 + padding. Three layouts, one per exchange: P8(i) = i + i/16
                        // between passes 1 and 2 (stride-8 stores), Q(i) = i + 2 (i/16) between
                        // passes 2 and 3 (max 573), and the natural (unpadded) layout for the
                        // transforms' inputs / outputs and the real-FFT packing (contiguous runs,
                        // ascending or mirrored): under the half-warp bank model every access is
                        // conflict-free (tools/banks.py; ncu measured 4 wavefronts per pass-2
                        // store and per mirror load with P8 there)

__device__ __forceinline__ int P8(int i) { return i + (i >> 4); }

// Twiddle table (1024 float2, staged in shared memory by every FFT kernel), laid out so that
// each pass reads consecutive entries:
//   tw[k]                      = W1024^k,            k < 512   (R2C / C2R packing, radix-2)
//   tw[512 + 64 (r-1) + j]     = W512^(r j),         r = 1..7, j < 64   (pass 3)
//   tw[960 + 8 (r-1) + k]      = W512^(8 r k),       r = 1..7, k < 8    (pass 2)
#define TW_P3 512
#define TW_P2 960
// Every FFT CTA stages the 8 KiB twiddle table into shared memory. The copy is issued with
// cp.async (16-byte LDGSTS, no register round trip) BEFORE the CTA loads its own blocks, and
// waited for (tw_wait: wait_all + CTA barrier) just before the first FFT pass, so the table's L2
// latency hides behind the block loads instead of stalling the CTA at its start.
__device__ __forceinline__ void tw_stage_async(float2 *tw, const float2 *src) {
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(tw + 2 * i);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + 2 * i));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void tw_wait() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
}

template <bool INV>
__device__ __forceinline__ float2 twv(const float2 *tw, int idx) {
  const float2 w = tw[idx];
  return INV ? make_float2(w.x, -w.y) : w;
}

template <bool INV>
__device__ __forceinline__ void dft8(float2 (&v)[8]) {
  const float r = 0.70710678118654752f;
  // stage 1 (span 4): a_{4+r} = (v_r - v_{r+4}) W8^r
  float2 a0 = cadd(v[0], v[4]), a4 = csub(v[0], v[4]);
  float2 a1 = cadd(v[1], v[5]), a5 = csub(v[1], v[5]);
  float2 a2 = cadd(v[2], v[6]), a6 = csub(v[2], v[6]);
  float2 a3 = cadd(v[3], v[7]), a7 = csub(v[3], v[7]);
  // (packed: one FADD2 on the swapped / half-negated operand, one FMUL2; same roundings as
  // the scalar (x +- y) * r)
  const float2 rr = make_float2(r, r);
  if (!INV) {
    a5 = __fmul2_rn(__fadd2_rn(a5, make_float2(a5.y, -a5.x)), rr);            // * (1 - i)/sqrt2
    a6 = cmul_mi(a6);                                                       // * -i
    a7 = __fmul2_rn(__fadd2_rn(make_float2(a7.y, -a7.x), make_float2(-a7.x, -a7.y)), rr);   // * (-1 - i)/sqrt2
  } else {
    a5 = __fmul2_rn(__fadd2_rn(a5, make_float2(-a5.y, a5.x)), rr);            // * (1 + i)/sqrt2
    a6 = cmul_i(a6);
    a7 = __fmul2_rn(__fadd2_rn(make_float2(-a7.x, a7.x), make_float2(-a7.y, -a7.y)), rr);   // * (-1 + i)/sqrt2
  }
  // stage 2 (span 2)
  float2 b0 = cadd(a0, a2), b2 = csub(a0, a2);
  float2 b1 = cadd(a1, a3), b3 = csub(a1, a3);
  float2 b4 = cadd(a4, a6), b6 = csub(a4, a6);
  float2 b5 = cadd(a5, a7), b7 = csub(a5, a7);
  if (!INV) { b3 = cmul_mi(b3); b7 = cmul_mi(b7); }
  else { b3 = cmul_i(b3); b7 = cmul_i(b7); }
  // stage 3 (span 1), outputs in natural order
  v[0] = cadd(b0, b1); v[4] = csub(b0, b1);
  v[2] = cadd(b2, b3); v[6] = csub(b2, b3);
  v[1] = cadd(b4, b5); v[5] = csub(b4, b5);
  v[3] = cadd(b6, b7); v[7] = csub(b6, b7);
}

// In-place FFT-512 of buf (padded, FFT_PAD_N float2) by the 64 threads j = 0..63 of a group.
// All threads of the group (GB = 1) or CTA (GB = 0) must call it.
// On return thread j holds X[j + 64 r] in v[r]; fft512_store() writes them back.
// Padded addresses are formed from one per-thread base plus compile-time offsets:
//   P8(j + 64 r)   = (j + j/16) + 68 r
//   P8(8 j + r)    = (8 j + j/2) + r                     (r < 8)
//   Q(B + 8 r)     = (72 (j/8) + j%8) + 8 r + 2 (r/2), Q(j + 64 r) = (j + 2 (j/16)) + 72 r  (passes 2 -> 3)
// Barrier of one transform: GB = 0 -> __syncthreads (default); GB = 1 -> only the 64 threads of
// the group (named barrier 1 + group; measured 3-5% slower on k_pam_fe / k_pam_be than the CTA
// barrier, kept for experiments; kernels then need a CTA barrier after staging shared tables).
template <int GB>
__device__ __forceinline__ void fft_sync() {
  if constexpr (GB != 0) asm volatile("bar.sync %0, 64;\n" ::"r"(1 + (int)(threadIdx.x >> 6)) : "memory");
  else __syncthreads();
}

// The pass-3 twiddles W512^(r j), r = 1..7, of thread j are the same for every transform the thread
// runs (conjugated for the inverse): kernels that run several FFT-512s per block load them once
// (fft_t3_load) and pass them in registers, saving 7 shared loads (14 wavefronts per warp) per
// transform - the FFT kernels are shared-memory-bandwidth bound (ncu: 0.66-0.81 wavefronts per
// SM cycle).
struct FftT3 { float2 w[7]; };
__device__ __forceinline__ FftT3 fft_t3_load(const float2 *tw, int j) {
  FftT3 t;
#pragma unroll
  for (int r = 1; r < 8; ++r) t.w[r - 1] = tw[TW_P3 + j + 64 * (r - 1)];
  return t;
}

template <bool INV, int GB = 0>
__device__ __forceinline__ void fft512_regs(float2 *buf, int j, const float2 *tw, float2 (&v)[8],
                                            const FftT3 *t3r = nullptr) {
  // pass-1 input already in registers: v[r] = z[j + 64 r]
  float2 *const pa = buf + j + (j >> 4);
  float2 *const pw1 = buf + 8 * j + (j >> 1);
  // pass-2 outputs go to Q(B + 8 r), Q(i) = i + 2 (i >> 4), B = 64 (j / 8) + j % 8:
  //   Q(B + 8 r) = (72 (j / 8) + j % 8) + 8 r + 2 (r / 2);   pass 3 reads Q(j + 64 r) = (j + 2 (j / 16)) + 72 r
  float2 *const pw2 = buf + 72 * (j >> 3) + (j & 7);
  const float2 *const pq = buf + j + 2 * (j >> 4);
  dft8<INV>(v);
  fft_sync<GB>();
#pragma unroll
  for (int r = 0; r < 8; ++r) pw1[r] = v[r];
  fft_sync<GB>();
  // pass 2: Ns = 8, twiddle W512^(r k), k = j % 8
  {
    const float2 *t2 = tw + TW_P2 + (j & 7);
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = pa[68 * r];
#pragma unroll
    for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], twv<INV>(t2, 8 * (r - 1)));
    dft8<INV>(v);
    fft_sync<GB>();
#pragma unroll
    for (int r = 0; r < 8; ++r) pw2[8 * r + 2 * (r >> 1)] = v[r];
    fft_sync<GB>();
  }
  // pass 3: Ns = 64, twiddle W512^(r j)
  const float2 *t3 = tw + TW_P3 + j;
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = pq[72 * r];
#pragma unroll
  for (int r = 1; r < 8; ++r) {
    float2 w;
    if (t3r) w = INV ? cconj(t3r->w[r - 1]) : t3r->w[r - 1];
    else w = twv<INV>(t3, 64 * (r - 1));
    v[r] = cmul(v[r], w);
  }
  dft8<INV>(v);
  // result: v[r] = X[j + 64 r]
}

template <bool INV, int GB = 0>
__device__ __forceinline__ void fft512(float2 *buf, int j, const float2 *tw, float2 (&v)[8]) {
  const float2 *const pa = buf + j;            // natural (unpadded) layout, see FFT_PAD_N
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = pa[64 * r];
  fft512_regs<INV, GB>(buf, j, tw, v);
}

// Real-FFT pairing without a full store: bin k = j + 64 r (r < 4) is v[r] of thread j, its
// partner 512 - k is v[7 - r] of thread (64 - j) % 64, so only v[4..7] are published.
template <int GB = 0>
__device__ __forceinline__ void fft512_publish_upper(float2 *buf, int j, const float2 (&v)[8]) {
  float2 *const pa = buf + j;
  fft_sync<GB>();
#pragma unroll
  for (int q = 4; q < 8; ++q) pa[64 * q] = v[q];
  fft_sync<GB>();
}
__device__ __forceinline__ float2 fft_partner(const float2 *pm, int j, int r, const float2 (&v)[8]) {
  return (j == 0 && r == 0) ? v[0] : pm[-64 * r];
}

// Store the pass-3 result back (natural order) — only needed when other threads read it.
template <int GB = 0>
__device__ __forceinline__ void fft512_store(float2 *buf, int j, const float2 (&v)[8]) {
  float2 *const pa = buf + j;
  fft_sync<GB>();
#pragma unroll
  for (int r = 0; r < 8; ++r) pa[64 * r] = v[r];
  fft_sync<GB>();
}

// Mirror addresses used by the real-FFT packing: for k = j + 64 r (r = 0..3) thread j needs
// buf[P8(k)] = pa[68 r] and buf[P8(512 - k)] = pm[-68 r] with pm = P8(512 - j) (j >= 1);
// j = 0, r = 0 pairs bin 0 with itself (index 0).
__device__ __forceinline__ const float2 *fft_mirror_base(const float2 *buf, int j) {
  return buf + (512 - j);     // j = 0: buf + 512 (inside FFT_PAD_N; its r = 0 partner is v[0])
}
__device__ __forceinline__ float2 fft_mirror(const float2 *buf, const float2 *pm, int j, int r) {
  return (j == 0 && r == 0) ? buf[0] : pm[-64 * r];
}

// ---------------------------------------------------------------------------------------
// Real 1024-point transforms through the packed 512-point complex FFT.
// Forward: z[n] = x[2n] + i x[2n+1]; Z = FFT512(z);
//   X[k] = Xe + W^k Xo, Xe = (Z[k] + conj Z[512-k])/2, Xo = -i (Z[k] - conj Z[512-k])/2,
//   X[512-k] = conj(Xe - W^k Xo)   (W = e^{-2 pi i/1024}).
// Thread j of a group owns the bin pairs (k, 512-k) for k = j + 64 r, r = 0..3; thread 0
// additionally owns k = 256 (X[256] = conj Z[256]); k = 0 pairs with 512.
// HALF = false: the same pair without the two exact 1/2 scalings (outputs exactly 2x; callers fold
// the power of two into a later scale - bit-identical results, two FMUL2 fewer per pair)
template <bool HALF = true>
__device__ __forceinline__ void r2c_pair(float2 Zk, float2 Zn, float2 w, float2 &Xk, float2 &Xn) {
  float2 Xe = cadd(Zk, cconj(Zn));
  float2 Xo = cmul_mi(csub(Zk, cconj(Zn)));
  if (HALF) { Xe = cscale(Xe, 0.5f); Xo = cscale(Xo, 0.5f); }
  float2 t = cmul(w, Xo);
  Xk = cadd(Xe, t);
  Xn = cconj(csub(Xe, t));
}
// Inverse packing: given Hermitian half-spectrum pair (Y[k], Y[512-k]) produce Z[k], Z[512-k]
// such that IFFT512(Z)[n] = (y[2n] + i y[2n+1]) * 512 / 1024 * 2 ... i.e. y = IFFT1024(Y)
// satisfies y[2n] + i y[2n+1] = IFFT512(Z)[n] / 512 (unnormalised IFFT512 used).
//   Xe = (Y[k] + conj Y[512-k])/2, Xo = (Y[k] - conj Y[512-k])/2 * conj(W^k)
//   Z[k] = Xe + i Xo, Z[512-k] = conj(Xe) + i conj(Xo)
template <bool HALF = true>
__device__ __forceinline__ void c2r_pair(float2 Yk, float2 Yn, float2 w, float2 &Zk, float2 &Zn) {
  float2 Xe = cadd(Yk, cconj(Yn));
  float2 Xo = cmulc(csub(Yk, cconj(Yn)), w);
  if (HALF) { Xe = cscale(Xe, 0.5f); Xo = cscale(Xo, 0.5f); }
  Zk = cadd(Xe, cmul_i(Xo));
  Zn = cadd(cconj(Xe), cmul_i(cconj(Xo)));
}
