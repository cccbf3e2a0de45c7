// FP64 FMA throughput of this GPU (the ionic kernel's compute roofline):
// 8 independent DFMA chains per thread, full occupancy, CUDA-event timed.
// Prints one JSON line: {"fp64_tflops": ..., "dfma_per_clk_per_sm": ..., ...}
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 123.456) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  dfma_loop<<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fmas = (double)blocks * threads * iters * 8;
  const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  const double per_clk = fmas / (best * 1e-3) / sms / (clk_khz * 1e3);
  printf("{\"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_max_clock\": %.2f, \"sms\": %d, "
         "\"max_clock_mhz\": %.0f, \"ms\": %.4f}\n", tflops, per_clk, sms, clk_khz / 1e3, best);
  return 0;
}
