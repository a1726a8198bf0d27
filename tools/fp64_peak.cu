// fp64_peak.cu -- measured FP64 peak of this B200:
// the roofline's FP64 term.  Every thread runs 8 independent dependency
// chains (enough ILP to cover the DFMA latency at full occupancy), so the
// FP64 pipe, not latency, bounds the rate.
//   dfma:      a = fma(a, x, y)             -> 2 flops per DFMA
//   dmul+dadd: a = a * x; a = a + y          -> 1 flop each (the bitwise sweeps'
//                                              uncontracted form)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_fp64_peak tools/fp64_peak.cu
// Prints one JSON line; the numbers come from CUDA events around the kernel
// after a warm-up launch, best of 5.
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double x, double y) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = __fma_rn(a[c], x, y);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

__global__ void dmul_dadd_kernel(double* out, double x, double y) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = __dadd_rn(__dmul_rn(a[c], x), y);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == 12345.678) out[0] = s;
}

template <class K>
float best_ms(K kernel, int blocks, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int threads = 256, blocks = sms * 8;
  const double ops = (double)blocks * threads * kIters * kChains;  // instructions of each kind
  const float ms_fma = best_ms(dfma_kernel, blocks, threads, out);
  const float ms_md = best_ms(dmul_dadd_kernel, blocks, threads, out);
  const double dfma_per_s = ops / (ms_fma * 1e-3);
  const double md_per_s = 2 * ops / (ms_md * 1e-3);  // DMUL + DADD instructions
  const cudaError_t e = cudaGetLastError();
  std::printf(
      "{\"dfma_tflops\": %.4f, \"dfma_ginstr_per_s\": %.2f, \"dmul_dadd_ginstr_per_s\": %.2f, "
      "\"dmul_dadd_tflops\": %.4f, \"lanes_per_sm_per_clk_at_max\": %.2f, \"sms\": %d, "
      "\"max_clock_mhz\": %.0f, \"ms_dfma\": %.4f, \"ms_dmul_dadd\": %.4f, \"status\": \"%s\", "
      "\"how\": \"%d blocks x %d threads x %d iterations x %d independent chains; CUDA events, "
      "best of 5 after a warm-up\"}\n",
      2 * dfma_per_s / 1e12, dfma_per_s / 1e9, md_per_s / 1e9, md_per_s / 1e12,
      dfma_per_s / (sms * (clk * 1e3)), sms, clk / 1e3, ms_fma, ms_md, cudaGetErrorString(e),
      blocks, threads, kIters, kChains);
  cudaFree(out);
  return e == cudaSuccess ? 0 : 1;
}
