// Whole CG iterations of the config-4 diagonal-operator PCG as ONE persistent
// cooperative kernel on synthetic arrays (n = 10,276,240, 7 symmetric offsets):
// what the grid-wide syncs, the reductions and the per-SM spread of the Q sweep
// cost against the three sweeps timed alone (scripts/sweep_bench.cu), and whether
// handing the Q sweep's tiles out dynamically (per-tile partial sums, summed in
// tile order: the result does not depend on which block took which tile) wins.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ib scripts/iter_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

constexpr int NP = 7;
struct Dia { long n, ld; long off[NP]; const int* rem_ptr; };

struct Args {
  Dia op;
  const double* vals;
  double *r, *p, *q, *x;
  const double* dinv;
  double* part;                 // partial sums (blocks or tiles), 2 values each
  unsigned long long* bar;      // grid barrier counter
  unsigned long long* ctr;      // tile counter
  int iters;
  double* out;
  unsigned long long* stamps;   // optional: globaltimer after each of the 3 barriers
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
    const unsigned long long target = (old / nblocks + 1) * nblocks;
    unsigned long long cur;
    if (old + 1 != target) do {
      asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
    } while (cur < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// block-level deterministic sum of NV values -> every thread gets the totals
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[k * 32 + warp] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(lane < nw ? sh[k * 32 + lane] : 0.0);
}

// grid sum: block partial -> part[block] -> barrier -> everyone sums nparts partials
template <int NV>
__device__ __forceinline__ void grid_sum_blocks(double (&v)[NV], const Args& a, double* sh) {
  block_sum<NV>(v, sh);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) a.part[blockIdx.x * 2 + k] = v[k];
  grid_barrier(a.bar, gridDim.x);
  double s[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) s[k] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] += __ldcg(a.part + b * 2 + k);
  block_sum<NV>(s, sh);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = s[k];
}

// after a dynamic sweep: barrier, then everyone sums the per-tile partials in tile order
__device__ __forceinline__ double grid_sum_tiles(const double* tpart, long ntiles, const Args& a,
                                                 double* sh) {
  grid_barrier(a.bar, gridDim.x);
  double s[1] = {0.0};
  for (long t = threadIdx.x; t < ntiles; t += blockDim.x) s[0] += __ldcg(tpart + t);
  block_sum<1>(s, sh);
  return s[0];
}

// interior rows (every neighbour index in range): no index clamps, no coefficient fix-up
__device__ __forceinline__ double dia_row_interior(const Dia& op, const double* __restrict__ vals,
                                                   const double* v, long i) {
  const long ld = op.ld;
  double cl[NP], vl[NP], cu[NP], vu[NP];
#pragma unroll
  for (int s = 0; s < NP; ++s) {
    const long d = op.off[s];
    const double* cs = vals + (1 + s) * ld;
    cl[s] = __ldg(cs + i - d);
    vl[s] = v[i - d];
    cu[s] = __ldg(cs + i);
    vu[s] = v[i + d];
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

template <bool REM>
__device__ __forceinline__ double dia_row(const Dia& op, const double* __restrict__ vals,
                                          const double* v, long i) {
  const long ld = op.ld, last = op.n - 1;
  if (REM) {   // lab switch: REM = true now means "interior fast path when the warp allows"
    const long dmax = op.off[NP - 1];
    if (__all_sync(__activemask(), i >= dmax && i + dmax <= last)) return dia_row_interior(op, vals, v, i);
  }
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

// MODE 0: all sweeps static grid-stride (the product's shape)
// MODE 1: Q sweep handed out as dynamic block tiles (BLK*NPT rows), per-tile partials
// MODE 2: Q and R sweeps dynamic
// MODE 3: all three sweeps dynamic
template <int MODE, int NPT, int BLK, int MINB, bool REM, bool NORED = false>
__global__ void __launch_bounds__(BLK, MINB) cg_iters(const Args a) {
  __shared__ double sh[64];
  __shared__ double sw[2][2][32];
  __shared__ long s_tile[2];
  const long n = a.op.n;
  const long stride = (long)gridDim.x * blockDim.x;
  const long tid0 = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = BLK / 32;
  constexpr long TILE = (long)BLK * NPT;
  const long ntiles = (n + TILE - 1) / TILE;
  const unsigned long long per_sweep = (unsigned long long)ntiles + gridDim.x;
  unsigned long long sweep_no = 0;   // dynamic sweeps done so far
  double* tpart = a.part + 4096;     // per-tile partials: [2][ntiles]
  double alpha = 1e-9, beta = 0.5, rz = 1.0;
  double* __restrict__ x = a.x;
  double* r = a.r;
  double* p = a.p;
  double* q = a.q;
  const double* __restrict__ dinv = a.dinv;

  // dynamic tile loop: F(i) per row returns nothing; NS sums per tile
  auto first_tile = [&]() {
    if (threadIdx.x == 0)
      s_tile[0] = (long)(atomicAdd(a.ctr, 1ULL) - sweep_no * per_sweep);
    __syncthreads();
  };

  for (int it = 0; it < a.iters; ++it) {
    // ---- P ----
    if (MODE >= 3) {
      first_tile();
      for (int j = 0;; ++j) {
        const long t = s_tile[j & 1];
        if (t >= ntiles) break;
        if (threadIdx.x == 0)
          s_tile[(j + 1) & 1] = (long)(atomicAdd(a.ctr, 1ULL) - sweep_no * per_sweep);
#pragma unroll
        for (int k = 0; k < NPT; ++k) {
          const long i = t * TILE + k * BLK + threadIdx.x;
          if (i < n) {
            const double zi = dinv[i] * r[i];
            const double pi = p[i];
            x[i] = fma(alpha, pi, x[i]);
            p[i] = fma(beta, pi, zi);
          }
        }
        __syncthreads();
      }
      ++sweep_no;
    } else {
      for (long base = tid0; base < n; base += stride * NPT) {
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
    grid_barrier(a.bar, gridDim.x);
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) a.stamps[it * 3 + 0] = gtimer();
    // ---- Q ----
    double pq;
    if (MODE >= 1) {
      first_tile();
      for (int j = 0;; ++j) {
        const long t = s_tile[j & 1];
        if (t >= ntiles) break;
        if (threadIdx.x == 0)
          s_tile[(j + 1) & 1] = (long)(atomicAdd(a.ctr, 1ULL) - sweep_no * per_sweep);
        double s0 = 0.0;
#pragma unroll
        for (int k = 0; k < NPT; ++k) {
          const long i = t * TILE + k * BLK + threadIdx.x;
          if (i < n) {
            const double qi = dia_row<REM>(a.op, a.vals, p, i);
            q[i] = qi;
            s0 = fma(p[i], qi, s0);
          }
        }
        s0 = warp_sum(s0);
        if (lane == 0) sw[j & 1][0][warp] = s0;
        __syncthreads();
        if (warp == 0) {
          const double tsum = warp_sum(lane < NW ? sw[j & 1][0][lane] : 0.0);
          if (lane == 0) tpart[t] = tsum;
        }
      }
      ++sweep_no;
      pq = grid_sum_tiles(tpart, ntiles, a, sh);
    } else {
      double s1[1] = {0.0};
      for (long base = tid0; base < n; base += stride * NPT) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) {
          const long i = base + k * stride;
          if (i < n) {
            const double qi = dia_row<REM>(a.op, a.vals, p, i);
            q[i] = qi;
            s1[0] = fma(p[i], qi, s1[0]);
          }
        }
      }
      if (NORED) { grid_barrier(a.bar, gridDim.x); if (s1[0] == 123.456) a.out[1] = s1[0]; s1[0] = 1.0; }
      else grid_sum_blocks<1>(s1, a, sh);
      pq = s1[0];
      if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) a.stamps[it * 3 + 1] = gtimer();
    }
    alpha = 1e-9 + 1e-30 * pq;
    // ---- R ----
    double rr, rzn;
    if (MODE >= 2) {
      first_tile();
      for (int j = 0;; ++j) {
        const long t = s_tile[j & 1];
        if (t >= ntiles) break;
        if (threadIdx.x == 0)
          s_tile[(j + 1) & 1] = (long)(atomicAdd(a.ctr, 1ULL) - sweep_no * per_sweep);
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k < NPT; ++k) {
          const long i = t * TILE + k * BLK + threadIdx.x;
          if (i < n) {
            const double ri = r[i] - alpha * q[i];
            r[i] = ri;
            const double zi = dinv[i] * ri;
            s0 = fma(ri, ri, s0);
            s1 = fma(ri, zi, s1);
          }
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        if (lane == 0) { sw[j & 1][0][warp] = s0; sw[j & 1][1][warp] = s1; }
        __syncthreads();
        if (warp == 0) {
          const double t0 = warp_sum(lane < NW ? sw[j & 1][0][lane] : 0.0);
          const double t1 = warp_sum(lane < NW ? sw[j & 1][1][lane] : 0.0);
          if (lane == 0) { tpart[t] = t0; tpart[ntiles + t] = t1; }
        }
      }
      ++sweep_no;
      grid_barrier(a.bar, gridDim.x);
      double s[2] = {0.0, 0.0};
      for (long t = threadIdx.x; t < ntiles; t += blockDim.x) {
        s[0] += __ldcg(tpart + t);
        s[1] += __ldcg(tpart + ntiles + t);
      }
      block_sum<2>(s, sh);
      rr = s[0]; rzn = s[1];
    } else {
      double s2[2] = {0.0, 0.0};
      for (long base = tid0; base < n; base += stride * NPT) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) {
          const long i = base + k * stride;
          if (i < n) {
            const double ri = r[i] - alpha * q[i];
            r[i] = ri;
            const double zi = dinv[i] * ri;
            s2[0] = fma(ri, ri, s2[0]);
            s2[1] = fma(ri, zi, s2[1]);
          }
        }
      }
      if (NORED) { grid_barrier(a.bar, gridDim.x); if (s2[0] == 123.456) a.out[1] = s2[1]; s2[0] = s2[1] = 1.0; }
      else grid_sum_blocks<2>(s2, a, sh);
      rr = s2[0]; rzn = s2[1];
      if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) a.stamps[it * 3 + 2] = gtimer();
    }
    beta = 0.5 + 1e-30 * (rzn / rz + rr);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out[0] = alpha + beta;
}

// Static sweeps with (ALT) consecutive sweeps running in opposite directions, so each
// starts on the part of the vectors the previous one touched last, and (CS) the
// operator's own-row coefficients loaded with the evict-first policy (ld.global.cs),
// so the 658 MB operator stream does not push the 82 MB vectors out of the 126 MB L2.
template <bool CS>
__device__ __forceinline__ double dia_row_cs(const Dia& op, const double* __restrict__ vals,
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
    cu[s] = CS ? __ldcs(cs + i) : __ldg(cs + i);
    vu[s] = v[ju > last ? last : ju];
    if (jl < 0) cl[s] = 0.0;
  }
  const double dg = CS ? __ldcs(vals + i) : __ldg(vals + i), vc = v[i];
  double acc = 0.0;
#pragma unroll
  for (int s = NP - 1; s >= 0; --s) acc = fma(cl[s], vl[s], acc);
  acc = fma(dg, vc, acc);
#pragma unroll
  for (int s = 0; s < NP; ++s) acc = fma(cu[s], vu[s], acc);
  return acc;
}

template <int NPT, bool ALT, bool CS>
__global__ void __launch_bounds__(512, 2) cg_iters_alt(const Args a) {
  __shared__ double sh[64];
  const long n = a.op.n;
  const long stride = (long)gridDim.x * blockDim.x;
  const long tid0 = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nbatch = (n + stride * NPT - 1) / (stride * NPT);
  double alpha = 1e-9, beta = 0.5, rz = 1.0;
  double* __restrict__ x = a.x;
  double* r = a.r;
  double* p = a.p;
  double* q = a.q;
  const double* __restrict__ dinv = a.dinv;
  int sweep = 0;
#define FOR_ROWS(...)                                                        \
  for (long bb = 0; bb < nbatch; ++bb) {                                      \
    const long b_ = (ALT && (sweep & 1)) ? nbatch - 1 - bb : bb;              \
    _Pragma("unroll") for (int k = 0; k < NPT; ++k) {                         \
      const long i = tid0 + (b_ * NPT + k) * stride;                          \
      if (i < n) { __VA_ARGS__ }                                              \
    }                                                                         \
  }                                                                           \
  ++sweep;
  for (int it = 0; it < a.iters; ++it) {
    FOR_ROWS({
      const double zi = dinv[i] * r[i];
      const double pi = p[i];
      x[i] = fma(alpha, pi, x[i]);
      p[i] = fma(beta, pi, zi);
    })
    grid_barrier(a.bar, gridDim.x);
    double s1[1] = {0.0};
    FOR_ROWS({
      const double qi = dia_row_cs<CS>(a.op, a.vals, p, i);
      q[i] = qi;
      s1[0] = fma(p[i], qi, s1[0]);
    })
    grid_sum_blocks<1>(s1, a, sh);
    alpha = 1e-9 + 1e-30 * s1[0];
    double s2[2] = {0.0, 0.0};
    FOR_ROWS({
      const double ri = r[i] - alpha * q[i];
      r[i] = ri;
      const double zi = dinv[i] * ri;
      s2[0] = fma(ri, ri, s2[0]);
      s2[1] = fma(ri, zi, s2[1]);
    })
    grid_sum_blocks<2>(s2, a, sh);
    beta = 0.5 + 1e-30 * (s2[1] / rz + s2[0]);
  }
#undef FOR_ROWS
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out[0] = alpha + beta;
}

// Q sweep with the operator's own-row coefficients staged through shared memory by
// TMA bulk copies (cp.async.bulk + mbarrier, STAGES tiles of 512 rows in flight per
// block): the 64 B/row operator stream holds no registers while in flight, the
// mirrored coefficient of a small offset comes from the staged tile.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(512, 2) cg_iters_tma(const Args a) {
  constexpr int T = 512;
  extern __shared__ __align__(128) double stage[];      // [STAGES][NP + 1][T]
  __shared__ unsigned long long bars[STAGES];
  __shared__ double sh[64];
  const long n = a.op.n;
  const long stride = (long)gridDim.x * blockDim.x;
  const long tid0 = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nb = (n + stride - 1) / stride;          // tiles per block
  double alpha = 1e-9, beta = 0.5, rz = 1.0;
  double* __restrict__ x = a.x;
  double* r = a.r;
  double* p = a.p;
  double* q = a.q;
  const double* __restrict__ dinv = a.dinv;
  const double* vals = a.vals;
  const long ld = a.op.ld, last = n - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long issued = 0, consumed = 0;     // tiles over the whole run (stage = count % STAGES)
  auto issue = [&](long j) {         // thread 0: tile j of the current sweep
    const long t0 = (j * gridDim.x + blockIdx.x) * (long)T;
    if (t0 >= n) return;             // (empty tiles are not counted: parities stay aligned)
    const unsigned rows = (unsigned)min((long)T, n - t0);
    const int st = (int)(issued % STAGES);
    mbar_expect_tx(&bars[st], (NP + 1) * rows * 8u);
#pragma unroll
    for (int c = 0; c <= NP; ++c)
      tma_load_1d(stage + ((long)st * (NP + 1) + c) * T, vals + c * ld + t0, rows * 8u, &bars[st]);
    ++issued;
  };
  for (int it = 0; it < a.iters; ++it) {
    for (long base = tid0; base < n; base += stride * 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long i = base + k * stride;
        if (i < n) {
          const double zi = dinv[i] * r[i];
          const double pi = p[i];
          x[i] = fma(alpha, pi, x[i]);
          p[i] = fma(beta, pi, zi);
        }
      }
    }
    // the operator tiles do not depend on p: start them before the barrier
    if (threadIdx.x == 0)
      for (long j = 0; j < STAGES - 1 && j < nb; ++j) issue(j);
    grid_barrier(a.bar, gridDim.x);
    double s1[1] = {0.0};
    for (long j = 0; j < nb; ++j) {
      if (threadIdx.x == 0 && j + STAGES - 1 < nb) issue(j + STAGES - 1);
      const long i = tid0 + j * stride;
      const int st = (int)(consumed % STAGES);
      const unsigned parity = (unsigned)((consumed / STAGES) & 1);
      if ((j * gridDim.x + blockIdx.x) * (long)T < n) {
        mbar_wait(&bars[st], parity);
        ++consumed;
      }
      if (i < n) {
        const double* tile = stage + (long)st * (NP + 1) * T;
        const int t = threadIdx.x;
        double cl[NP], vl[NP], cu[NP], vu[NP];
#pragma unroll
        for (int s = 0; s < NP; ++s) {
          const long d = a.op.off[s];
          const long jl = i - d, jlc = jl < 0 ? 0 : jl, ju = i + d;
          cl[s] = (d <= t) ? tile[(1 + s) * T + t - d] : __ldg(vals + (1 + s) * ld + jlc);
          vl[s] = p[jlc];
          cu[s] = tile[(1 + s) * T + t];
          vu[s] = p[ju > last ? last : ju];
          if (jl < 0) cl[s] = 0.0;
        }
        const double dg = tile[t], vc = p[i];
        double acc = 0.0;
#pragma unroll
        for (int s = NP - 1; s >= 0; --s) acc = fma(cl[s], vl[s], acc);
        acc = fma(dg, vc, acc);
#pragma unroll
        for (int s = 0; s < NP; ++s) acc = fma(cu[s], vu[s], acc);
        q[i] = acc;
        s1[0] = fma(vc, acc, s1[0]);
      }
      __syncthreads();    // the stage may be refilled
    }
    grid_sum_blocks<1>(s1, a, sh);
    alpha = 1e-9 + 1e-30 * s1[0];
    double s2[2] = {0.0, 0.0};
    for (long base = tid0; base < n; base += stride * 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long i = base + k * stride;
        if (i < n) {
          const double ri = r[i] - alpha * q[i];
          r[i] = ri;
          const double zi = dinv[i] * ri;
          s2[0] = fma(ri, ri, s2[0]);
          s2[1] = fma(ri, zi, s2[1]);
        }
      }
    }
    grid_sum_blocks<2>(s2, a, sh);
    beta = 0.5 + 1e-30 * (s2[1] / rz + s2[0]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out[0] = alpha + beta;
}

// One kernel per sweep with the real reductions: every block leaves its partial,
// the next kernel's blocks sum all partials (fixed order) to get alpha / beta.
template <int NV>
__device__ __forceinline__ void read_partials(double (&v)[NV], const double* part, int nparts, double* sh) {
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __ldcg(part + b * 2 + k);
  block_sum<NV>(v, sh);
}

template <int NPT>
__global__ void __launch_bounds__(512, 2) sepP(const Args a) {
  __shared__ double sh[64];
  double s[2];
  read_partials<2>(s, a.part + 1024, gridDim.x, sh);     // R's partials -> beta
  const double beta = 0.5 + 1e-30 * s[1], alpha = 1e-9 + 1e-30 * s[0];
  const long n = a.op.n, stride = (long)gridDim.x * blockDim.x;
  const double* __restrict__ r = a.r; const double* __restrict__ dinv = a.dinv;
  double* __restrict__ p = a.p; double* __restrict__ x = a.x;
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
__global__ void __launch_bounds__(512, 2) sepQ(const Args a) {
  __shared__ double sh[64];
  const long n = a.op.n, stride = (long)gridDim.x * blockDim.x;
  const double* p = a.p; double* __restrict__ q = a.q;
  double s1[1] = {0.0};
  for (long base = blockIdx.x * (long)blockDim.x + threadIdx.x; base < n; base += stride * NPT) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long i = base + k * stride;
      if (i < n) {
        const double qi = dia_row<false>(a.op, a.vals, p, i);
        q[i] = qi;
        s1[0] = fma(p[i], qi, s1[0]);
      }
    }
  }
  block_sum<1>(s1, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x * 2] = s1[0];
}

template <int NPT>
__global__ void __launch_bounds__(512, 2) sepR(const Args a) {
  __shared__ double sh[64];
  double s[1];
  read_partials<1>(s, a.part, gridDim.x, sh);            // Q's partials -> alpha
  const double alpha = 1e-9 + 1e-30 * s[0];
  const long n = a.op.n, stride = (long)gridDim.x * blockDim.x;
  double* __restrict__ r = a.r; const double* __restrict__ q = a.q; const double* __restrict__ dinv = a.dinv;
  double s2[2] = {0.0, 0.0};
  for (long base = blockIdx.x * (long)blockDim.x + threadIdx.x; base < n; base += stride * NPT) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const long i = base + k * stride;
      if (i < n) {
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        const double zi = dinv[i] * ri;
        s2[0] = fma(ri, ri, s2[0]);
        s2[1] = fma(ri, zi, s2[1]);
      }
    }
  }
  block_sum<2>(s2, sh);
  if (threadIdx.x == 0) { a.part[1024 + blockIdx.x * 2] = s2[0]; a.part[1024 + blockIdx.x * 2 + 1] = s2[1]; }
}

// barrier cost alone: iters x 3 grid barriers with nothing between them
template <int BLK, int MINB>
__global__ void __launch_bounds__(BLK, MINB) barriers_only(const Args a) {
  for (int it = 0; it < a.iters * 3; ++it) grid_barrier(a.bar, gridDim.x);
}

__global__ void fill(double* a, long n, double v) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    a[i] = v * (1.0 + 1e-3 * (i % 977));
}

template <class K>
float run(K kern, Args& a, int grid, int blk, int reps = 3) {
  void* params[] = {&a};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaMemset(a.bar, 0, 8); cudaMemset(a.ctr, 0, 8);
  cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(blk), params, 0, 0);
  cudaMemsetAsync(a.ctr, 0, 8);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) {
    cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(blk), params, 0, 0);
    cudaMemsetAsync(a.ctr, 0, 8);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(e));
  return ms / reps / a.iters * 1e3f;   // us per iteration
}

int main() {
  const long n = 10276240;
  Args a;
  const long ld_pad = getenv("IB_LD_PAD") ? atol(getenv("IB_LD_PAD")) : 0;       // doubles
  const long stagger = getenv("IB_STAGGER") ? atol(getenv("IB_STAGGER")) : 0;     // doubles
  const bool quick = getenv("IB_QUICK") != nullptr;
  a.op.n = n; a.op.ld = n + ld_pad;
  const long nx = 41, nxy = 41 * 241;
  const long offs[NP] = {1, nx, nx + 1, nxy, nxy + 1, nxy + nx, nxy + nx + 1};
  for (int s = 0; s < NP; ++s) a.op.off[s] = offs[s];
  double *vals, *dinv;
  int* rem;
  cudaMalloc(&vals, sizeof(double) * (n + ld_pad) * (NP + 1));
  cudaMalloc(&a.r, sizeof(double) * (n + 8 * stagger)); cudaMalloc(&a.p, sizeof(double) * (n + 8 * stagger));
  cudaMalloc(&a.q, sizeof(double) * (n + 8 * stagger)); cudaMalloc(&a.x, sizeof(double) * (n + 8 * stagger));
  cudaMalloc(&dinv, sizeof(double) * (n + 8 * stagger)); cudaMalloc(&a.out, 64);
  a.p += stagger; a.q += 2 * stagger; a.x += 3 * stagger; dinv += 4 * stagger;   // r stays
  cudaMalloc(&a.part, sizeof(double) * (4096 + 2 * 65536));
  cudaMalloc(&a.bar, 8); cudaMalloc(&a.ctr, 8);
  cudaMalloc(&rem, sizeof(int) * (n / 32 + 2)); cudaMemset(rem, 0, sizeof(int) * (n / 32 + 2));
  a.op.rem_ptr = rem; a.vals = vals; a.dinv = dinv;
  fill<<<1024, 256>>>(vals, (n + ld_pad) * (NP + 1), 1e-3);
  fill<<<1024, 256>>>(a.r, n, 1.0); fill<<<1024, 256>>>(a.p, n, 0.5); fill<<<1024, 256>>>(a.q, n, 0.25);
  fill<<<1024, 256>>>(a.x, n, 0.1); fill<<<1024, 256>>>(dinv, n, 2.0);
  cudaDeviceSynchronize();
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  a.iters = 40; a.stamps = nullptr;
  const double GB = 160e-9 * n;
  auto report = [&](const char* name, float us) {
    printf("%-58s %7.1f us/iteration  %5.0f GB/s\n", name, us, GB / (us * 1e-6));
  };
  printf("SMs %d, n %ld, 160 B per node and iteration\n", sms, n);
  {
    Args b = a; b.iters = 200;
    float us = run(barriers_only<512, 2>, b, sms * 2, 512);
    printf("3 grid barriers alone (296 x 512): %.2f us per iteration\n", us);
  }
  if (quick) {
    printf("ld_pad %ld stagger %ld\n", ld_pad, stagger);
    for (int rep = 0; rep < 3; ++rep) {
      report("static  npt4 b512x2", run(cg_iters<0, 4, 512, 2, false>, a, sms * 2, 512));
      report("static  npt4 b512x2, interior rows without clamps", run(cg_iters<0, 4, 512, 2, true>, a, sms * 2, 512));
    }
    return 0;
  }
  report("static  npt4 b512x2", run(cg_iters<0, 4, 512, 2, false>, a, sms * 2, 512));
  report("static  npt4 b512x2 barriers only (no sums)", run(cg_iters<0, 4, 512, 2, false, true>, a, sms * 2, 512));
  {
    unsigned long long* st; cudaMalloc(&st, 8 * 3 * a.iters);
    Args b = a; b.stamps = st;
    run(cg_iters<0, 4, 512, 2, false>, b, sms * 2, 512, 1);
    std::vector<unsigned long long> h(3 * a.iters);
    cudaMemcpy(h.data(), st, 8 * 3 * a.iters, cudaMemcpyDeviceToHost);
    double tp = 0, tq = 0, tr = 0;
    for (int it = 1; it < a.iters; ++it) {
      tp += h[it * 3] - h[it * 3 - 1]; tq += h[it * 3 + 1] - h[it * 3]; tr += h[it * 3 + 2] - h[it * 3 + 1];
    }
    printf("  block 0's view, barrier to barrier: P %.1f  Q %.1f  R %.1f us\n", tp / (a.iters - 1) * 1e-3,
           tq / (a.iters - 1) * 1e-3, tr / (a.iters - 1) * 1e-3);
  }
  {
    cudaMemset(a.part, 0, sizeof(double) * 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      for (int it = 0; it < a.iters; ++it) {
        sepP<4><<<sms * 2, 512>>>(a); sepQ<4><<<sms * 2, 512>>>(a); sepR<4><<<sms * 2, 512>>>(a);
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    report("three kernels per iteration, real reductions", ms / a.iters * 1e3f);
    cudaGraph_t graph; cudaGraphExec_t ge; cudaStream_t st; cudaStreamCreate(&st);
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int it = 0; it < a.iters; ++it) {
      sepP<4><<<sms * 2, 512, 0, st>>>(a); sepQ<4><<<sms * 2, 512, 0, st>>>(a); sepR<4><<<sms * 2, 512, 0, st>>>(a);
    }
    cudaStreamEndCapture(st, &graph); cudaGraphInstantiate(&ge, graph, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("three kernels per iteration, CUDA graph", ms / a.iters * 1e3f);
  }
  {
    auto k3 = cg_iters_tma<3>;
    const int smem3 = 3 * (NP + 1) * 512 * 8;
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    void* params[] = {&a};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(a.bar, 0, 8);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((const void*)k3, dim3(sms * 2), dim3(512), params, smem3, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  tma error: %s\n", cudaGetErrorString(e));
    report("static  Q tiles staged by TMA (3 stages x 32 KB)", ms / a.iters * 1e3f);
    auto k2 = cg_iters_tma<2>;
    const int smem2 = 2 * (NP + 1) * 512 * 8;
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(a.bar, 0, 8);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((const void*)k2, dim3(sms * 2), dim3(512), params, smem2, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    e = cudaGetLastError();
    if (e != cudaSuccess) printf("  tma error: %s\n", cudaGetErrorString(e));
    report("static  Q tiles staged by TMA (2 stages x 32 KB)", ms / a.iters * 1e3f);
  }
  report("static  npt4 (alt kernel, no alt, no cs)", run(cg_iters_alt<4, false, false>, a, sms * 2, 512));
  report("static  npt4 alternating directions", run(cg_iters_alt<4, true, false>, a, sms * 2, 512));
  report("static  npt4 operator evict-first (ld.cs)", run(cg_iters_alt<4, false, true>, a, sms * 2, 512));
  report("static  npt4 alternating + evict-first", run(cg_iters_alt<4, true, true>, a, sms * 2, 512));
  report("static  npt4 b512x2, interior rows without clamps", run(cg_iters<0, 4, 512, 2, true>, a, sms * 2, 512));
  report("dyn Q   npt4 b512x2 (tile 2048)", run(cg_iters<1, 4, 512, 2, false>, a, sms * 2, 512));
  report("dyn QR  npt4 b512x2", run(cg_iters<2, 4, 512, 2, false>, a, sms * 2, 512));
  report("dyn PQR npt4 b512x2", run(cg_iters<3, 4, 512, 2, false>, a, sms * 2, 512));
  report("static  npt4 b512x2 (again)", run(cg_iters<0, 4, 512, 2, false>, a, sms * 2, 512));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
