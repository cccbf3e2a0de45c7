// Microbenchmarks for the persistent-PCG building blocks on B200:
// grid-barrier latency vs grid size and fence flavour, and one streaming
// phase over n nodes.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o mb scripts/microbench.cu ; run: ./mb
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void bar_release(unsigned long long* bar, unsigned nb, bool fence) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (fence) __threadfence();
    unsigned long long old, cur;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
    const unsigned long long target = (old / nb + 1) * nb;
    do {
      asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
    } while (cur < target);
    if (fence) __threadfence();
  }
  __syncthreads();
}

__global__ void barriers(unsigned long long* bar, int reps, int fence) {
  for (int r = 0; r < reps; ++r) bar_release(bar, gridDim.x, fence);
}

__global__ void stream_phase(const double* a, const double* b, double* c, long n, int reps,
                             unsigned long long* bar) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride)
      c[i] = a[i] * 1.0001 + b[i];
    bar_release(bar, gridDim.x, false);
  }
}

__global__ void stencil_phase(const double* v, double* out, long n, int nx, int ny, int reps,
                              unsigned long long* bar) {
  const long stride = (long)gridDim.x * blockDim.x;
  const long sz = (long)nx * ny;
  for (int r = 0; r < reps; ++r) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride) {
      double acc = 0.0;
      if (i >= sz + nx + 1 && i < n - sz - nx - 1) {
#pragma unroll
        for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx)
              acc = __dadd_rn(acc, __dmul_rn(0.1 * (dz + 2) * (dy + 3), v[i + dz * sz + dy * nx + dx]));
      }
      out[i] = acc;
    }
    bar_release(bar, gridDim.x, false);
  }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long* bar;
  cudaMalloc(&bar, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 2000;
  for (int fence = 0; fence < 2; ++fence)
    for (int nb : {1, 9, 74, 148, 296}) {
      for (int bs : {256, 512, 1024}) {
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, barriers, bs, 0);
        if (nb > per * sms) continue;
        cudaMemset(bar, 0, 8);
        barriers<<<nb, bs>>>(bar, 10, fence);
        cudaEventRecord(e0);
        barriers<<<nb, bs>>>(bar, reps, fence);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("barrier fence=%d blocks=%4d threads=%4d : %.3f us/barrier\n", fence, nb, bs,
               ms * 1e3 / reps);
      }
    }
  const long n = 442401;
  double *a, *b, *c;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&c, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaMemset(b, 0, n * 8);
  for (int nb : {148, 296, 592}) {
    for (int bs : {256, 512}) {
      int per1 = 0, per2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, stream_phase, bs, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, stencil_phase, bs, 0);
      if (nb > per1 * sms || nb > per2 * sms) continue;
      const int r2 = 200;
      cudaMemset(bar, 0, 8);
      stream_phase<<<nb, bs>>>(a, b, c, n, 5, bar);
      cudaEventRecord(e0);
      stream_phase<<<nb, bs>>>(a, b, c, n, r2, bar);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("stream phase n=%ld blocks=%d threads=%d : %.3f us/phase (%.0f GB/s)\n", n, nb, bs,
             ms * 1e3 / r2, 24.0 * n / (ms / r2 * 1e-3) / 1e9);
      cudaMemset(bar, 0, 8);
      stencil_phase<<<nb, bs>>>(a, c, n, 201, 71, 5, bar);
      cudaEventRecord(e0);
      stencil_phase<<<nb, bs>>>(a, c, n, 201, 71, r2, bar);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("stencil phase n=%ld blocks=%d threads=%d : %.3f us/phase\n", n, nb, bs,
             ms * 1e3 / r2);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
