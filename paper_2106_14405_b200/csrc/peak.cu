// peak.cu -- FP32 / FP64 FMA-pipe microbenchmark used as the roofline
// denominator for the (non-tensor) step kernels.  MEASURED_PEAKS.json only
// carries HBM and bf16 tensor peaks (SURVEY.md §8d asks for a measured
// FMA peak).  Not part of the reference-facing ABI (include/rsim_bench.h).
#include <cuda_runtime.h>

#include "../../include/rsim_bench.h"

namespace {

template <typename T>
__global__ void fma_kernel(T *out, int iters, T seed) {
  T a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const T b = (T)0.999999, c = (T)1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  T s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == (T)-1.2345) out[blockIdx.x] = s;  // never true; keeps the chain live
}

template <typename T>
int run(double *tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T *out = nullptr;
  if (cudaMalloc(&out, sizeof(T) * sms * 64) != cudaSuccess) return 2;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_kernel<T><<<blocks, threads>>>(out, 64, (T)1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    fma_kernel<T><<<blocks, threads>>>(out, iters, (T)1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 2;
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return 0;
}

}  // namespace

int rsim_bench_fma_peak(int fp64, double *tflops) {
  if (!tflops) return 1;
  return fp64 ? run<double>(tflops) : run<float>(tflops);
}
