// common.cuh — shared device helpers of librx (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RX_FFT_N 1024
#define RX_HOP 512
#define RX_PREF 32767

// ------------------------------------------------------------------ complex helpers
// Complex arithmetic on the sm_100 packed FP32x2 pipe (FADD2 / FMUL2 / FFMA2: two IEEE fp32
// operations per instruction, each rounded exactly like its scalar form; the operand swaps,
// broadcasts and single-half negations these need are free SASS modifiers). The FP32 throughput is
// unchanged (a packed op occupies the FMA pipe for two cycles) but the issue slots of the FFT
// butterflies, twiddle products and BPS distances halve - the chain's kernels are issue-bound.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a b = (fma(a.x, b.x, -a.y b.y), fma(a.x, b.y, a.y b.x)): one FMUL2 + one FFMA2
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x));
  return __ffma2_rn(make_float2(a.x, a.x), b, make_float2(-t.x, t.y));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b) = (fma(a.x, b.x, a.y b.y), fma(a.y, b.x, -a.x b.y))
  const float2 t = __fmul2_rn(make_float2(a.y, a.x), make_float2(b.y, b.y));
  return __ffma2_rn(a, make_float2(b.x, b.x), make_float2(t.x, -t.y));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
__device__ __forceinline__ float2 cmul_i(float2 a) { return make_float2(-a.y, a.x); }    // i a
__device__ __forceinline__ float2 cmul_mi(float2 a) { return make_float2(a.y, -a.x); }   // -i a
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

// ------------------------------------------------------------------ DDS (SURVEY c-0, A10)
// phase word u = origin + p * inc (mod 2^64); e^{-j 2 pi u / 2^64} from the top 32 bits:
// x = (int32)(u >> 32) / 2^31 in [-1, 1), sincospi in fp32 (error <= pi 2^-24).
__device__ __forceinline__ float2 dds_rot_neg(uint64_t u) {
  int32_t top = (int32_t)(u >> 32);
  float x = (float)top * 4.656612873077393e-10f;   // 2^-31
  float s, c;
  sincospif(x, &s, &c);
  return make_float2(c, -s);
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels launched with the PDL attribute (rx_api.cu launch_pdl) start their independent prologue
// (twiddle staging) while the previous kernel of the stream drains, and wait here before touching
// anything it produced (griddepcontrol.wait returns once the preceding grid has completed and its
// memory is visible; a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// ------------------------------------------------------------------ TMA bulk copies + mbarrier
// 1-D bulk global -> shared copies by the async (TMA) engine (cp.async.bulk, SASS UBLKCP) with
// transaction-count completion on a shared-memory mbarrier: one elected thread arms the barrier
// with the byte count and issues the copy, the consumers spin on the barrier's phase.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {   // make the init visible to the async proxy
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// ------------------------------------------------------------------ warp reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ virtual input
// Sample p of the stream: from the current call's buffer when p >= call_start, else from
// the history ring (the tail of earlier calls, P:136 'prepending a block … stored
// elsewhere'), 0 for p < 0 (SURVEY c-0).
struct InView {
  const uint16_t *cur;      // this call's samples (RX_IN_U12_IN_U16) ...
  const float *curf;        // ... or (RX_IN_F32)
  long long call_start;
  long long call_end;
  const uint16_t *hist;     // history ring of earlier calls' samples (u16 codes or floats)
  const float *histf;
  long long hist_cap;       // power of two, > max call size + lookback + keep
  uint16_t *hist_w;         // front-end kernels append the call's last samples here
  float *histf_w;
  long long keep_from;      // samples p >= keep_from of this call are kept in the history ring
  int f32;                  // input format RX_IN_F32
  float gain;               // adc_gain (f32 input)
  long long cnt_lo, cnt_hi; // blocks whose owned samples are counted (clipped / domain); a
                            // time shard counts only its own buffer's blocks (its halos belong
                            // to its neighbours)
};
__device__ __forceinline__ int in_code(const InView &v, long long p, bool &pad) {
  pad = p < 0;
  if (p < 0) return -1;
  if (p >= v.call_start) return __ldg(v.cur + (p - v.call_start));
  return __ldg(v.hist + (p & (v.hist_cap - 1)));
}
// x_p of an f32 stream (0 for p < 0)
__device__ __forceinline__ float in_xf(const InView &v, long long p) {
  if (p < 0) return 0.f;
  if (p >= v.call_start) return __ldg(v.curf + (p - v.call_start)) * v.gain;
  return __ldg(v.histf + (p & (v.hist_cap - 1))) * v.gain;
}

