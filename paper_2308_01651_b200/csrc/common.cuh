// Shared helpers for the sm_100a kernels behind include/mdx.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mdx.h"

namespace mdx {

// Thread-local error text reported through mdx_last_error().
void set_error(const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return MDX_ERR_CUDA;
  }
  return MDX_OK;
}

int num_sms();

// IEEE round-to-nearest multiply/add that nvcc may not contract into an FMA.
// Used wherever the reference (numba, no fastmath) evaluates a*b + c as two
// rounded operations and we want bit-identical results (operators, CG
// vector updates, BDF history combinations).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double madd_rn(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}

// Warp-level sum with a fixed shuffle tree (deterministic for a fixed launch).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV values; result valid in thread 0. `scratch` holds
// NV * 32 doubles. Warp partials are combined in warp order.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[k * 32 + warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += scratch[k * 32 + w];
      v[k] = s;
    }
  }
  __syncthreads();
}

// Software grid barrier for a launch whose blocks are all co-resident
// (cooperative launch).  bar is a monotonic 64-bit arrival counter whose
// value is a multiple of the grid size between barriers: a block arrives
// with one release atomic and spins (acquire loads) until the count reaches
// the end of its epoch.  The gpu-scope fences make every write issued before
// the barrier visible to every block after it (and invalidate stale L1).
__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned int nblocks) {
  __syncthreads();
  if (nblocks == 1) return;
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long old;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
    const unsigned long long target = (old / nblocks + 1) * nblocks;
    unsigned long long cur;
    do {
      asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
    } while (cur < target);
    __threadfence();
  }
  __syncthreads();
}

// Coherent (L2) loads for values other blocks wrote earlier in this launch.
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

}  // namespace mdx
