// common.cuh — shared device helpers of librx (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RX_FFT_N 1024
#define RX_HOP 512
#define RX_PREF 32767

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
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
  const uint16_t *cur;
  long long call_start;
  long long call_end;
  const uint16_t *hist;
  long long hist_cap;   // power of two, > max call size + lookback + keep
  uint16_t *hist_w;     // front-end kernels append the call's last samples here
  long long keep_from;  // samples p >= keep_from of this call are kept in the history ring
};
__device__ __forceinline__ int in_code(const InView &v, long long p, bool &pad) {
  pad = p < 0;
  if (p < 0) return -1;
  if (p >= v.call_start) return __ldg(v.cur + (p - v.call_start));
  return __ldg(v.hist + (p & (v.hist_cap - 1)));
}

// Load 16 consecutive codes starting at p (p multiple of 16) as floats x = (c-2047.5)*scale;
// `pad` entries (p < 0) get value `padval`. Also counts clipped codes (0 or 4095) among
// entries with p >= count_from.
__device__ __forceinline__ void load16(const InView &v, long long p, float scale, float padval,
                                       float (&x)[16], long long count_from, int &clip) {
  if (p >= v.call_start && p + 16 <= v.call_end) {
    const uint4 *src = reinterpret_cast<const uint4 *>(v.cur + (p - v.call_start));
    uint4 a = __ldg(src), b = __ldg(src + 1);
    // owned (new) samples of the call's tail go to the history ring for later calls
    if (p >= count_from && p >= v.keep_from) {
      uint4 *dst = reinterpret_cast<uint4 *>(v.hist_w + (p & (v.hist_cap - 1)));
      dst[0] = a;
      dst[1] = b;
    }
    uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const float off = -2047.5f * scale;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int c0 = (int)(w[i] & 0xffffu), c1 = (int)(w[i] >> 16);
      x[2 * i] = fmaf((float)c0, scale, off);
      x[2 * i + 1] = fmaf((float)c1, scale, off);
      if (p + 2 * i >= count_from) clip += (c0 == 0 || c0 == 4095);
      if (p + 2 * i + 1 >= count_from) clip += (c1 == 0 || c1 == 4095);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      bool pad;
      int c = in_code(v, p + i, pad);
      x[i] = pad ? padval : fmaf((float)c, scale, -2047.5f * scale);   // same rounding as fast paths
      if (!pad && p + i >= count_from) clip += (c == 0 || c == 4095);
    }
  }
}
