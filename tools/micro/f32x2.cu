// Throughput of scalar FFMA / FADD vs the sm_100 packed FFMA2 / FADD2 (fma.rn.f32x2 /
// add.rn.f32x2): 16 independent chains per thread, 148 x 8 CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 o; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o) : "l"(a), "l"(b), "l"(c)); return o; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 o; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(o) : "l"(a), "l"(b)); return o; }
template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, int iters, float b, float c) {
  float x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = threadIdx.x * 1e-3f + i;
  if (MODE == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = fmaf(x[i], b, c);
  } else if (MODE == 1) {
    u64 *y = reinterpret_cast<u64 *>(x);
    float2 bb = make_float2(b, b), cc = make_float2(c, c);
    u64 B = *reinterpret_cast<u64 *>(&bb), C = *reinterpret_cast<u64 *>(&cc);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = ffma2(y[i], B, C);
  } else if (MODE == 2) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = x[i] + c;
  } else if (MODE == 3) {
    u64 *y = reinterpret_cast<u64 *>(x);
    float2 cc = make_float2(c, c);
    u64 C = *reinterpret_cast<u64 *>(&cc);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = fadd2(y[i], C);
  } else if (MODE == 4) {   // mix: 16 FFMA2 + 16 integer ops (does the packed op free issue slots?)
    u64 *y = reinterpret_cast<u64 *>(x);
    float2 bb = make_float2(b, b), cc = make_float2(c, c);
    u64 B = *reinterpret_cast<u64 *>(&bb), C = *reinterpret_cast<u64 *>(&cc);
    unsigned s[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) { y[i] = ffma2(y[i], B, C); s[i] = s[i] * 0x9E3779B9u + (unsigned)it; }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] += (float)s[i];
  } else {                  // mix: 32 FFMA + 16 integer ops
    unsigned s[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = fmaf(x[i], b, c);
#pragma unroll
      for (int i = 0; i < 16; ++i) s[i] = s[i] * 0x9E3779B9u + (unsigned)it;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] += (float)s[i];
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char *name, double ops_per_iter) {
  float *o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE><<<148 * 8, 256>>>(o, iters, 0.999f, 1e-3f);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<MODE><<<148 * 8, 256>>>(o, iters, 0.999f, 1e-3f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  double n = 148.0 * 8 * 256 * iters;
  printf("%-28s %8.3f ms  %8.2f T fp32-lane-ops/s  %8.2f T warp-instr/s(x32)\n", name, best, n * ops_per_iter / best / 1e9,
         0.0);
  cudaFree(o);
}
int main() {
  run<0>("FFMA x32", 32); run<1>("FFMA2 x16 (32 lanes-ops)", 32);
  run<2>("FADD x32", 32); run<3>("FADD2 x16 (32 lane-ops)", 32);
  run<4>("FFMA2 x16 + 16 IMAD", 32); run<5>("FFMA x32 + 16 IMAD", 32);
  return 0;
}
