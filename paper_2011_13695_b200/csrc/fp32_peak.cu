// fp32_peak.cu — measurement helper for bench.py (not part of the receiver ABI): the FP32
// CUDA-core FFMA throughput this B200 actually sustains, the denominator of the "alu" roofline
// (MEASURED_PEAKS.json has HBM and bf16 tensor peaks only).
//
// Every thread runs 16 independent FFMA chains (enough ILP to cover the 4-cycle FMA latency at
// any occupancy), 148 x 8 CTAs of 256 threads; the result is conditionally stored so nothing is
// dead code. flop = 2 per FFMA.
#include <cuda_runtime.h>

#define CHAINS 16

__global__ void __launch_bounds__(256) k_fp32_ffma(float *out, int iters, float b, float c) {
  float a[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) a[i] = (float)(threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) a[i] = fmaf(a[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += a[i];
  if (s == 1234.5678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Measured FP32 FFMA peak in TFLOP/s (best of `reps` timed launches after a warm-up) and the
// launch's duration. Returns 0 on success, the cudaError_t otherwise.
extern "C" int fp32_peak_tflops(int device, int reps, double *tflops, double *ms_best) {
  if (cudaSetDevice(device) != cudaSuccess) return 1;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const int blocks = nsm * 8, threads = 256, iters = 8192;
  float *out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp32_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);   // warm-up (clocks ramp)
  k_fp32_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    k_fp32_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return (int)err;
  const double flop = 2.0 * CHAINS * (double)iters * blocks * threads;
  *tflops = flop / (best * 1e-3) / 1e12;
  *ms_best = best;
  return 0;
}
