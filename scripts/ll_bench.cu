// Grid-reduction latency microbenchmark (B200): R back-to-back 4-value grid
// sums by a cooperative grid of G blocks x 512 threads.
//   mode 0: arrival counter (atom.add.release + one poller) + partial loads
//   mode 1: LL words (fenced publish), every block reads all slots, thread b
//           reading slot b
//   mode 2: as 1 without fences
//   mode 3: as 1, but only warp 0 polls, one ld.v2 x4 per slot, all slots of
//           a lane issued before any spin
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ll_bench scripts/ll_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int NT = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ int g_st_kind;
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  const int kind = g_st_kind;
  if (kind == 0) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else if (kind == 1) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else if (kind == 2) asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else if (kind == 3) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  } else {
    unsigned long long old;
    asm volatile("atom.exch.relaxed.gpu.global.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  }
}
__device__ __forceinline__ void ld_relaxed_v2(const unsigned long long* p, unsigned long long& a,
                                              unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p)
               : "memory");
}

__global__ void __launch_bounds__(NT, 1)
bench(int mode, int rounds, unsigned long long* bar, double* part, unsigned long long* ll,
      double* out) {
  __shared__ double sh[300];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[4] = {1.0 + threadIdx.x, 2.0, 3.0, 4.0};
  for (int r = 0; r < rounds; ++r) {
    const uint32_t ep = (uint32_t)r + 1u;
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = warp_sum(v[k] * 1e-9);
    if (lane == 0)
      for (int k = 0; k < 4; ++k) sh[k * 32 + warp] = v[k];
    __syncthreads();
    double t[4];
    if (warp == 0)
      for (int k = 0; k < 4; ++k) t[k] = warp_sum(lane < NT / 32 ? sh[k * 32 + lane] : 0.0);
    if (mode == 0) {
      double* pp = part + (size_t)(r & 1) * gridDim.x * 4;
      if (warp == 0 && lane == 0) {
        for (int k = 0; k < 4; ++k) pp[blockIdx.x * 4 + k] = t[k];
        unsigned long long old;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
        if (old + 1 != target) {
          unsigned long long cur;
          do {
            asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
          } while (cur < target);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
      double acc[4] = {0, 0, 0, 0};
      for (unsigned b = threadIdx.x; b < gridDim.x; b += NT)
        for (int k = 0; k < 4; ++k) acc[k] += __ldcg(pp + b * 4 + k);
      for (int k = 0; k < 4; ++k) {
        acc[k] = warp_sum(acc[k]);
        if (lane == 0) sh[128 + k * 32 + warp] = acc[k];
      }
    } else {
      unsigned long long* slotb = ll + (size_t)(ep & 1) * gridDim.x * 8;
      if (warp == 0) {
        if (mode == 1 || mode == 3 || mode == 4 || mode == 9) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (lane < 8) {
          double x = t[lane >> 1];
          const uint32_t h = (lane & 1) ? (uint32_t)__double2loint(x) : (uint32_t)__double2hiint(x);
          if (mode == 6)
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(slotb + blockIdx.x * 8 + lane),
                         "l"(((unsigned long long)ep << 32) | h) : "memory");
          else if ((mode == 7 || mode == 8) && lane == 0) {
            unsigned long long old;
            asm volatile("atom.exch.release.gpu.global.b64 %0, [%1], %2;" : "=l"(old)
                         : "l"(slotb + blockIdx.x * 8 + lane), "l"(((unsigned long long)ep << 32) | h)
                         : "memory");
          }
          else
            st_relaxed_u64(slotb + blockIdx.x * 8 + lane, ((unsigned long long)ep << 32) | h);
        }
      }
      if (mode == 8 || mode == 9) __syncthreads();
      double acc[4] = {0, 0, 0, 0};
      if (mode == 3) {
        if (warp == 0) {
          for (unsigned b0 = 0; b0 < gridDim.x; b0 += 32 * 4) {
            unsigned long long wd[4][8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const unsigned b = b0 + q * 32 + lane;
              if (b < gridDim.x)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  ld_relaxed_v2(slotb + b * 8 + 2 * k, wd[q][2 * k], wd[q][2 * k + 1]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const unsigned b = b0 + q * 32 + lane;
              if (b < gridDim.x)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  while ((uint32_t)(wd[q][2 * k] >> 32) != ep ||
                         (uint32_t)(wd[q][2 * k + 1] >> 32) != ep)
                    ld_relaxed_v2(slotb + b * 8 + 2 * k, wd[q][2 * k], wd[q][2 * k + 1]);
                  acc[k] += __hiloint2double((int)wd[q][2 * k], (int)wd[q][2 * k + 1]);
                }
            }
          }
        }
      } else {
        for (unsigned b = threadIdx.x; b < gridDim.x; b += NT) {
          unsigned long long wd[8];
          bool ok;
          do {
#pragma unroll
            for (int k = 0; k < 4; ++k) ld_relaxed_v2(slotb + b * 8 + 2 * k, wd[2 * k], wd[2 * k + 1]);
            ok = true;
#pragma unroll
            for (int k = 0; k < 8; ++k) ok = ok && (uint32_t)(wd[k] >> 32) == ep;
          } while (!ok);
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] += __hiloint2double((int)wd[2 * k], (int)wd[2 * k + 1]);
        }
      }
      if (mode == 1 || mode == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (mode == 5 || mode == 7 || mode == 8 || mode == 9) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      for (int k = 0; k < 4; ++k) {
        acc[k] = warp_sum(acc[k]);
        if (lane == 0) sh[128 + k * 32 + warp] = acc[k];
      }
    }
    __syncthreads();
    if (warp == 0)
      for (int k = 0; k < 4; ++k) {
        const double s = warp_sum(lane < NT / 32 ? sh[128 + k * 32 + lane] : 0.0);
        if (lane == 0) sh[256 + k] = s;
      }
    __syncthreads();
    for (int k = 0; k < 4; ++k) v[k] = sh[256 + k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = v[0];
}

int main(int argc, char** argv) {
  int rounds = 2000;
  int grids[2] = {289, 148};
  unsigned long long *bar, *ll;
  double *part, *out;
  cudaMalloc(&bar, 8);
  cudaMalloc(&ll, 2 * 1024 * 8 * 8);
  cudaMalloc(&part, 2 * 1024 * 4 * 8);
  cudaMalloc(&out, 8);
  printf("{");
  for (int gi = 1; gi < 2; ++gi) {
    int G = grids[gi];
    for (int mode = 0; mode < 10; ++mode) {
      int kind = 0;
      int mreal = mode;
      cudaMemcpyToSymbol(g_st_kind, &kind, sizeof(int));
      cudaMemset(bar, 0, 8);
      cudaMemset(ll, 0, 2 * 1024 * 8 * 8);
      void* args[] = {&mreal, &rounds, &bar, &part, &ll, &out};
      int r0 = 10;
      void* args0[] = {&mreal, &r0, &bar, &part, &ll, &out};
      cudaLaunchCooperativeKernel((void*)bench, G, NT, args0, 0, 0);
      cudaDeviceSynchronize();
      cudaMemset(bar, 0, 8);
      cudaMemset(ll, 0, 2 * 1024 * 8 * 8);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)bench, G, NT, args, 0, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s\"G%d_mode%d_kind%d_us\": %.3f", mode ? ", " : "", G, mreal, kind,
             err == cudaSuccess ? 1000.0 * ms / rounds : -1.0);
    }
  }
  printf("}\n");
  return 0;
}
