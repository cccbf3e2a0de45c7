// Stand-alone timing of the three sweeps of the reference-recurrence PCG on the
// config-4 diagonal operator (7 symmetric offsets, n = 10,276,240), each as its
// own kernel, to see what each sweep reaches of HBM in isolation and how the
// launch shape (persistent grid-stride vs one-shot, block size, nodes per thread)
// changes it.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/sb scripts/sweep_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

constexpr int NP = 7;
struct Dia { long n, ld; long off[NP]; };

template <int NPT>
__global__ void __launch_bounds__(512, 2)
sweepP(long n, const double* __restrict__ r, const double* __restrict__ dinv, double* __restrict__ p,
       double* __restrict__ x, double alpha, double beta) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long base = blockIdx.x * (long)blockDim.x + threadIdx.x; base < n; base += stride * NPT) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long i = base + k * stride;
      if (i < n) {
        const double zi = dinv[i] * r[i];
        const double pi = p[i];
        x[i] = fma(alpha, pi, x[i]);
        p[i] = fma(beta, pi, zi);
      }
    }
  }
}

template <int NPT>
__global__ void __launch_bounds__(512, 2)
sweepR(long n, double* __restrict__ r, const double* __restrict__ q, const double* __restrict__ dinv,
       double alpha, double* out) {
  const long stride = (long)gridDim.x * blockDim.x;
  double s0 = 0, s1 = 0;
  for (long base = blockIdx.x * (long)blockDim.x + threadIdx.x; base < n; base += stride * NPT) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long i = base + k * stride;
      if (i < n) {
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        const double zi = dinv[i] * ri;
        s0 = fma(ri, ri, s0);
        s1 = fma(ri, zi, s1);
      }
    }
  }
  if (s0 == 123.456) out[0] = s0 + s1;
}

__device__ __forceinline__ double dia_row(const Dia& op, const double* __restrict__ vals,
                                          const double* v, long i) {
  const long ld = op.ld, last = op.n - 1;
  double cl[NP], vl[NP], cu[NP], vu[NP];
#pragma unroll
  for (int s = 0; s < NP; ++s) {
    const long d = op.off[s];
    const double* cs = vals + (1 + s) * ld;
    const long jl = i - d, jlc = jl < 0 ? 0 : jl, ju = i + d;
    cl[s] = __ldg(cs + jlc);
    vl[s] = v[jlc];
    cu[s] = __ldg(cs + i);
    vu[s] = v[ju > last ? last : ju];
    if (jl < 0) cl[s] = 0.0;
  }
  const double dg = __ldg(vals + i), vc = v[i];
  double acc = 0.0;
#pragma unroll
  for (int s = NP - 1; s >= 0; --s) acc = fma(cl[s], vl[s], acc);
  acc = fma(dg, vc, acc);
#pragma unroll
  for (int s = 0; s < NP; ++s) acc = fma(cu[s], vu[s], acc);
  return acc;
}

template <int NPT, int BLK, int MINB>
__global__ void __launch_bounds__(BLK, MINB)
sweepQ(Dia op, const double* __restrict__ vals, const double* p, double* __restrict__ q, double* out) {
  const long n = op.n;
  const long stride = (long)gridDim.x * blockDim.x;
  double s0 = 0;
  for (long base = blockIdx.x * (long)blockDim.x + threadIdx.x; base < n; base += stride * NPT) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long i = base + k * stride;
      if (i < n) {
        const double qi = dia_row(op, vals, p, i);
        q[i] = qi;
        s0 = fma(p[i], qi, s0);
      }
    }
  }
  if (s0 == 123.456) out[0] = s0;
}

// contiguous tile per block iteration: block handles BLK*NPT consecutive nodes
template <int NPT, int BLK, int MINB>
__global__ void __launch_bounds__(BLK, MINB)
sweepQ_tile(Dia op, const double* __restrict__ vals, const double* p, double* __restrict__ q, double* out) {
  const long n = op.n;
  double s0 = 0;
  const long ntiles = (n + BLK * NPT - 1) / (BLK * NPT);
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long i = t * (BLK * NPT) + k * BLK + threadIdx.x;
      if (i < n) {
        const double qi = dia_row(op, vals, p, i);
        q[i] = qi;
        s0 = fma(p[i], qi, s0);
      }
    }
  }
  if (s0 == 123.456) out[0] = s0;
}

// theta-strips marched along phi: the block's rows of consecutive planes sit one
// plane (nx*nth rows) apart, so the phi-neighbours' p values and the mirrored
// coefficients of the previous plane are still in L1 when the next plane needs them
struct Strips { int nx, nth, nph, S; int th0[40]; long unit0[700]; };   // unit0: per-block first unit

template <int NPT, int BLK, int MINB>
__global__ void __launch_bounds__(BLK, MINB)
sweepQ_strip(Dia op, Strips g, const double* __restrict__ vals, const double* p,
             double* __restrict__ q, double* out) {
  double s0 = 0;
  const long u0 = g.unit0[blockIdx.x], u1 = g.unit0[blockIdx.x + 1];
  const long plane = (long)g.nx * g.nth;
  for (long u = u0; u < u1; u += NPT) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long uu = u + k;
      if (uu < u1) {
        const int s = (int)(uu / g.nph), ph = (int)(uu % g.nph);
        const int t0 = g.th0[s], rows = g.nx * (g.th0[s + 1] - t0);
        const long base = (long)g.nx * t0 + plane * ph;
        for (int r = threadIdx.x; r < rows; r += BLK) {
          const long i = base + r;
          const double qi = dia_row(op, vals, p, i);
          q[i] = qi;
          s0 = fma(p[i], qi, s0);
        }
      }
    }
  }
  if (s0 == 123.456) out[0] = s0;
}

__global__ void fill(double* a, long n, double v) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    a[i] = v * (1.0 + 1e-3 * (i % 977));
}

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  const long n = 10276240;
  Dia op; op.n = n; op.ld = n;
  const long nx = 41, nxy = 41 * 241;
  const long offs[NP] = {1, nx, nx + 1, nxy, nxy + 1, nxy + nx, nxy + nx + 1};
  for (int s = 0; s < NP; ++s) op.off[s] = offs[s];
  double *vals, *r, *p, *q, *x, *dinv, *out;
  cudaMalloc(&vals, sizeof(double) * n * (NP + 1));
  cudaMalloc(&r, sizeof(double) * n); cudaMalloc(&p, sizeof(double) * n);
  cudaMalloc(&q, sizeof(double) * n); cudaMalloc(&x, sizeof(double) * n);
  cudaMalloc(&dinv, sizeof(double) * n); cudaMalloc(&out, 64);
  fill<<<1024, 256>>>(vals, n * (NP + 1), 1e-3);
  fill<<<1024, 256>>>(r, n, 1.0); fill<<<1024, 256>>>(p, n, 0.5); fill<<<1024, 256>>>(q, n, 0.25);
  fill<<<1024, 256>>>(x, n, 0.1); fill<<<1024, 256>>>(dinv, n, 2.0);
  cudaDeviceSynchronize();
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double GB = 1e-9 * n;
  float ms;
  printf("SMs %d\n", sms);
  for (int g : {sms * 2}) {
    ms = timeit([&] { sweepP<4><<<g, 512>>>(n, r, dinv, p, x, 1e-9, 0.5); });
    printf("P  npt4 grid %6d: %.3f ms  %.0f GB/s (48 B)\n", g, ms, 48 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepR<4><<<g, 512>>>(n, r, q, dinv, 1e-9, out); });
    printf("R  npt4 grid %6d: %.3f ms  %.0f GB/s (32 B)\n", g, ms, 32 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ<4, 512, 2><<<g, 512>>>(op, vals, p, q, out); });
    printf("Q  npt4 b512 grid %6d: %.3f ms  %.0f GB/s (80 B)\n", g, ms, 80 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ<2, 512, 2><<<g, 512>>>(op, vals, p, q, out); });
    printf("Q  npt2 b512 grid %6d: %.3f ms  %.0f GB/s\n", g, ms, 80 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ<1, 512, 2><<<g, 512>>>(op, vals, p, q, out); });
    printf("Q  npt1 b512 grid %6d: %.3f ms  %.0f GB/s\n", g, ms, 80 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ<1, 256, 4><<<g * 2, 256>>>(op, vals, p, q, out); });
    printf("Q  npt1 b256x4 grid %6d: %.3f ms  %.0f GB/s\n", g * 2, ms, 80 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ<2, 256, 6><<<g * 3, 256>>>(op, vals, p, q, out); });
    printf("Q  npt2 b256x6 grid %6d: %.3f ms  %.0f GB/s\n", g * 3, ms, 80 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ_tile<4, 512, 2><<<g, 512>>>(op, vals, p, q, out); });
    printf("Qt npt4 b512 grid %6d: %.3f ms  %.0f GB/s\n", g, ms, 80 * GB / (ms * 1e-3));
    ms = timeit([&] { sweepQ_tile<2, 256, 6><<<g * 3, 256>>>(op, vals, p, q, out); });
    printf("Qt npt2 b256x6 grid %6d: %.3f ms  %.0f GB/s\n", g * 3, ms, 80 * GB / (ms * 1e-3));
  }
  for (int S : {21, 31, 16, 41}) {
    for (int G : {sms * 2, sms * 4}) {
      Strips g; g.nx = 41; g.nth = 241; g.nph = 1040; g.S = S;
      for (int k = 0; k <= S; ++k) g.th0[k] = (int)((long)k * g.nth / S);
      // units (strip-major, phi) split over the blocks at equal cumulative rows
      std::vector<long> cum((size_t)S * g.nph + 1, 0);
      for (long u = 0; u < (long)S * g.nph; ++u)
        cum[u + 1] = cum[u] + g.nx * (g.th0[u / g.nph + 1] - g.th0[u / g.nph]);
      long u = 0;
      for (int b = 0; b <= G; ++b) {
        const long target = cum.back() * b / G;
        while (u < (long)S * g.nph && cum[u] < target) ++u;
        g.unit0[b] = u;
      }
      g.unit0[G] = (long)S * g.nph;
      if (G == sms * 2) {
        ms = timeit([&] { sweepQ_strip<1, 512, 2><<<G, 512>>>(op, g, vals, p, q, out); });
        printf("Qs S=%d npt1 b512 grid %d: %.3f ms  %.0f GB/s\n", S, G, ms, 80 * GB / (ms * 1e-3));
        ms = timeit([&] { sweepQ_strip<2, 512, 2><<<G, 512>>>(op, g, vals, p, q, out); });
        printf("Qs S=%d npt2 b512 grid %d: %.3f ms  %.0f GB/s\n", S, G, ms, 80 * GB / (ms * 1e-3));
      } else {
        ms = timeit([&] { sweepQ_strip<1, 256, 4><<<G, 256>>>(op, g, vals, p, q, out); });
        printf("Qs S=%d npt1 b256x4 grid %d: %.3f ms  %.0f GB/s\n", S, G, ms, 80 * GB / (ms * 1e-3));
        ms = timeit([&] { sweepQ_strip<2, 256, 4><<<G, 256>>>(op, g, vals, p, q, out); });
        printf("Qs S=%d npt2 b256x4 grid %d: %.3f ms  %.0f GB/s\n", S, G, ms, 80 * GB / (ms * 1e-3));
      }
    }
  }
  // the whole iteration back to back (L2 carry-over between sweeps)
  ms = timeit([&] {
    sweepP<4><<<sms * 2, 512>>>(n, r, dinv, p, x, 1e-9, 0.5);
    sweepQ<4, 512, 2><<<sms * 2, 512>>>(op, vals, p, q, out);
    sweepR<4><<<sms * 2, 512>>>(n, r, q, dinv, 1e-9, out);
  });
  printf("P+Q+R persistent-shape: %.3f ms  %.0f GB/s (160 B)\n", ms, 160 * GB / (ms * 1e-3));
  ms = timeit([&] {
    sweepP<4><<<20071, 512>>>(n, r, dinv, p, x, 1e-9, 0.5);
    sweepQ<1, 256, 4><<<40142, 256>>>(op, vals, p, q, out);
    sweepR<4><<<20071, 512>>>(n, r, q, dinv, 1e-9, out);
  });
  printf("P+Q+R one-shot: %.3f ms  %.0f GB/s (160 B)\n", ms, 160 * GB / (ms * 1e-3));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
