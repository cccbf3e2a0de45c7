// Ionic-model kernels: the pointwise module protocol, the fused tissue
// update and the register-resident 0D pacing batch.
//
// Replaces (see include/mdx.h for the per-entry citations):
//   <model>.advance_kernel / current_kernel / point_rates  (numba prange)
//   TissueSolver.step ionic section + BDF combinations     (simulation.py:433-461)
//   pace_single_cell                                        (ionic/__init__.py:119-167)
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"
#include "ionic_models.cuh"

// 3 x 128 threads per SM: 168 registers, no spills.  Since the kernel lost
// its inlined library log and per-variable index math, 3 spill-free warps per
// SM sub-partition beat 4 at 128 registers (76.8 vs 78.1 us on config 2) and
// 5 at 96 (83.1 us)
#ifndef MDX_IONIC_MINB
#define MDX_IONIC_MINB 3
#endif
#ifndef MDX_IONIC_BLOCK
#define MDX_IONIC_BLOCK 128
#endif

namespace mdx {

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// ---------------------------------------------------------------------------
// Module-protocol kernels on strided state: element (i, v) at W[i*cs + v*vs].
// AoS numpy arrays use (cs, vs) = (nv, 1); the tissue SoA store uses (1, ld).
// ---------------------------------------------------------------------------
template <class M>
__global__ void __launch_bounds__(128)
advance_strided(int64_t n, const double* __restrict__ u_ext,
                const double* __restrict__ W_ext, const double* __restrict__ W_bdf,
                int64_t cs, int64_t vs, double alpha, double dt,
                const typename M::Params P, double* __restrict__ W_out,
                double* __restrict__ I_out, unsigned long long* clamp_count) {
  int local_clamp = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double we[M::NV], wb[M::NV], wo[M::NV];
#pragma unroll
    for (int v = 0; v < M::NV; ++v) {
      wb[v] = W_bdf[i * cs + v * vs];
      we[v] = M::NEEDS_WEXT ? W_ext[i * cs + v * vs] : 0.0;
    }
    double I;
    M::advance(u_ext[i], we, wb, alpha, dt, P, wo, I, local_clamp);
#pragma unroll
    for (int v = 0; v < M::NV; ++v) W_out[i * cs + v * vs] = wo[v];
    I_out[i] = I;
  }
  if (clamp_count) {
    // one atomic per warp that saw any clamp
    int tot = __reduce_add_sync(0xffffffffu, local_clamp);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(clamp_count, (unsigned long long)tot);
  }
}

// Rush-Larsen one-step update (M::advance_rl) on strided state.
template <class M>
__global__ void __launch_bounds__(128)
advance_rl_strided(int64_t n, const double* __restrict__ u, const double* __restrict__ W_n,
                   int64_t cs, int64_t vs, double dt, const typename M::Params P,
                   double* __restrict__ W_out, double* __restrict__ I_out,
                   unsigned long long* clamp_count) {
  int local_clamp = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double wn[M::NV], wo[M::NV];
#pragma unroll
    for (int v = 0; v < M::NV; ++v) wn[v] = W_n[i * cs + v * vs];
    double I;
    M::advance_rl(u[i], wn, dt, P, wo, I, local_clamp);
#pragma unroll
    for (int v = 0; v < M::NV; ++v) W_out[i * cs + v * vs] = wo[v];
    I_out[i] = I;
  }
  if (clamp_count) {
    int tot = __reduce_add_sync(0xffffffffu, local_clamp);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(clamp_count, (unsigned long long)tot);
  }
}

template <class M>
__global__ void __launch_bounds__(128)
current_strided(int64_t n, const double* __restrict__ u, const double* __restrict__ W,
                int64_t cs, int64_t vs, const typename M::Params P,
                double* __restrict__ I_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double w[M::NV];
#pragma unroll
    for (int v = 0; v < M::NV; ++v) w[v] = W[i * cs + v * vs];
    I_out[i] = M::current(u[i], w, P);
  }
}

template <class M>
__global__ void __launch_bounds__(128)
rates_aos(int64_t n, const double* __restrict__ u, const double* __restrict__ W,
          const typename M::Params P, double* __restrict__ I_out,
          double* __restrict__ dW) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double w[M::NV], dw[M::NV], I;
#pragma unroll
    for (int v = 0; v < M::NV; ++v) w[v] = W[i * M::NV + v];
    M::rates(u[i], w, P, I, dw);
#pragma unroll
    for (int v = 0; v < M::NV; ++v) dW[i * M::NV + v] = dw[v];
    I_out[i] = I;
  }
}

// ---------------------------------------------------------------------------
// BDF combinations, evaluated exactly like HistoryRing.weighted_sum
// (timestepping.py:89-102): acc = w0*v0, then acc = acc + wk*vk, each a
// separately rounded operation.
// ---------------------------------------------------------------------------
struct Bdf {
  double alpha, h[3], e[3];
  int order;
};

__device__ __forceinline__ Bdf bdf_of(int order) {
  Bdf b;
  b.order = order;
  if (order == 1) {
    b.alpha = 1.0; b.h[0] = 1.0; b.e[0] = 1.0;
    b.h[1] = b.h[2] = b.e[1] = b.e[2] = 0.0;
  } else if (order == 2) {
    b.alpha = 1.5; b.h[0] = 2.0; b.h[1] = -0.5; b.e[0] = 2.0; b.e[1] = -1.0;
    b.h[2] = b.e[2] = 0.0;
  } else {
    b.alpha = 11.0 / 6.0; b.h[0] = 3.0; b.h[1] = -1.5; b.h[2] = 1.0 / 3.0;
    b.e[0] = 3.0; b.e[1] = -3.0; b.e[2] = 1.0;
  }
  return b;
}

// BDF1/BDF2 weights are 1, 2, -1/2, -1: every product is exact, so the FMA
// form rounds once exactly where the reference's separately rounded
// multiply-then-add does (bitwise equal), costs half the FP64 work, and lets
// the compiler share 2*w_n between the BDF and the extrapolation sums.
template <int ORDER>
__device__ __forceinline__ double combine(const double (&x)[ORDER], const double* wts) {
  if (ORDER <= 2) {
    double acc = wts[0] * x[0];
#pragma unroll
    for (int k = 1; k < ORDER; ++k) acc = fma(wts[k], x[k], acc);
    return acc;
  }
  double acc = mul_rn(wts[0], x[0]);
#pragma unroll
  for (int k = 1; k < ORDER; ++k) acc = madd_rn(acc, wts[k], x[k]);
  return acc;
}

// ---------------------------------------------------------------------------
// Tissue ionic update for one volume (one launch per volume per step).
// Reads u_n..u_{n-order+1} and W_n..W_{n-order+1} from the device rings,
// writes W_{n+1} into the ring's next slot and I^v at the volume's DOFs.
// With `prep` set (single volume covering every DOF, identity map) it also
// emits the RHS nodal term combo = u_BDF/dt + I_app and the CG warm start
// x0 = u_EXT into the u ring's next slot, so no separate nodal pass runs.
// RL (gate_scheme = MDX_GATES_RUSH_LARSEN): the states advance in one step from
// W_n alone (M::advance_rl at u_EXT), so only the newest state slot is read.
// ---------------------------------------------------------------------------
template <class M, int ORDER, bool RL>
__global__ void __launch_bounds__(MDX_IONIC_BLOCK, MDX_IONIC_MINB)
tissue_ionic(mdx_tissue_ionic_args a, const typename M::Params P) {
  if (a.status && *(volatile const int32_t*)a.status) return;
  const Bdf b = bdf_of(ORDER);
  const int S = a.ring_slots;
  const int nslot = (a.head + 1) % S;
  // ring slots of this step, resolved once: u and W history bases (newest
  // first) and the slot W_{n+1} goes to; a node then walks its variables with
  // one pointer increment per access
  const double* ub[ORDER];
  const double* wbase[ORDER];
#pragma unroll
  for (int k = 0; k < ORDER; ++k) {
    const int slot = (a.head - k + 3 * S) % S;
    ub[k] = a.u_ring + (int64_t)slot * a.ldu;
    wbase[k] = a.w_ring + (int64_t)slot * M::NV * a.ldw;
  }
  double* const wout = a.w_ring + (int64_t)nslot * M::NV * a.ldw;
  const int64_t ldw = a.ldw;
  int local_clamp = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = a.dofs ? (int64_t)a.dofs[i] : i;
    double uh[ORDER];
#pragma unroll
    for (int k = 0; k < ORDER; ++k) uh[k] = ub[k][node];
    const double u_ext = combine<ORDER>(uh, b.e);

    double I;
    double wo[M::NV];
    if (RL) {
      double wn[M::NV];
      const double* p0 = wbase[0] + i;
#pragma unroll
      for (int v = 0; v < M::NV; ++v) {
        wn[v] = *p0;
        p0 += ldw;
      }
      M::advance_rl(u_ext, wn, a.dt, P, wo, I, local_clamp);
    } else {
      double we[M::NV], wb[M::NV];
      const double* p[ORDER];
#pragma unroll
      for (int k = 0; k < ORDER; ++k) p[k] = wbase[k] + i;
#pragma unroll
      for (int v = 0; v < M::NV; ++v) {
        double wh[ORDER];
#pragma unroll
        for (int k = 0; k < ORDER; ++k) {
          wh[k] = *p[k];
          p[k] += ldw;
        }
        wb[v] = combine<ORDER>(wh, b.h);
        we[v] = M::NEEDS_WEXT ? combine<ORDER>(wh, b.e) : 0.0;
      }
      M::advance(u_ext, we, wb, b.alpha, a.dt, P, wo, I, local_clamp);
    }
    {
      double* po = wout + i;
#pragma unroll
      for (int v = 0; v < M::NV; ++v) {
        *po = wo[v];
        po += ldw;
      }
    }
    a.i_out[node] = I;

    if (a.prep) {
      const double u_bdf = combine<ORDER>(uh, b.h);
      double combo = u_bdf / a.dt;
      if (a.active_mask) {
        double app = 0.0;
        bool first = true;
        for (int k = 0; k < a.n_impulses; ++k) {
          if (!((a.active_mask >> k) & 1ull)) continue;
          const double pv = a.profiles[(int64_t)k * a.ldp + node];
          app = first ? pv : add_rn(app, pv);
          first = false;
        }
        combo = add_rn(combo, app);
      }
      a.combo[node] = combo;
      a.u_ring[nslot * a.ldu + node] = u_ext;
    }
  }
  if (a.clamp_count) {
    int tot = __reduce_add_sync(0xffffffffu, local_clamp);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(a.clamp_count, (unsigned long long)tot);
  }
}

// Nodal RHS term and warm start for multi-volume meshes (identity over all n).
template <int ORDER>
__global__ void __launch_bounds__(256)
tissue_prep(mdx_tissue_ionic_args a) {
  if (a.status && *(volatile const int32_t*)a.status) return;
  const Bdf b = bdf_of(ORDER);
  const int S = a.ring_slots;
  const int nslot = (a.head + 1) % S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double uh[ORDER];
#pragma unroll
    for (int k = 0; k < ORDER; ++k) uh[k] = a.u_ring[((a.head - k + 3 * S) % S) * a.ldu + i];
    const double u_ext = combine<ORDER>(uh, b.e);
    const double u_bdf = combine<ORDER>(uh, b.h);
    double combo = u_bdf / a.dt;
    if (a.active_mask) {
      double app = 0.0;
      bool first = true;
      for (int k = 0; k < a.n_impulses; ++k) {
        if (!((a.active_mask >> k) & 1ull)) continue;
        const double pv = a.profiles[(int64_t)k * a.ldp + i];
        app = first ? pv : add_rn(app, pv);
        first = false;
      }
      combo = add_rn(combo, app);
    }
    a.combo[i] = combo;
    a.u_ring[nslot * a.ldu + i] = u_ext;
  }
}

// ---------------------------------------------------------------------------
// 0D pacing batch: every thread integrates one cell for all steps with its
// state and BDF history in registers (pace_single_cell's splitting,
// ionic/__init__.py:140-163, with t_{k+1} = (k+1)*dt).
// ---------------------------------------------------------------------------
// RL: Rush-Larsen states (M::advance_rl from W_n at u_n) with the order-1
// potential update u+ = u_n + dt (I_app - I_ion(u_n, W+)).
template <class M, int ORDER, bool RL>
__global__ void __launch_bounds__(128)
pace_cells(mdx_pace_args a, const typename M::Params P) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= a.n_cells) return;
  double uh[3], wh[3][M::NV];
  uh[0] = a.u[c];
#pragma unroll
  for (int v = 0; v < M::NV; ++v) wh[0][v] = a.W[(int64_t)v * a.ldw + c];
  double peak = uh[0];
  const bool stim = c < a.n_stim_cells;
  int nclamp = 0;
  bool finite = true;
  int64_t row = 0;
  const bool traced = c < a.n_trace_cells;
  const int rowlen = 2 + M::NV;
  if (traced) {
    double* t = a.trace + c * a.trace_rows * rowlen;
    t[0] = 0.0;
    t[1] = uh[0];
    for (int v = 0; v < M::NV; ++v) t[2 + v] = wh[0][v];
    row = 1;
  }
  for (int64_t k = 0; k < a.n_steps; ++k) {
    const int ord = k + 1 < ORDER ? (int)(k + 1) : ORDER;
    const Bdf b = bdf_of(ord);
    double ub = mul_rn(b.h[0], uh[0]);
    double ue = mul_rn(b.e[0], uh[0]);
    for (int q = 1; q < ord; ++q) {
      ub = madd_rn(ub, b.h[q], uh[q]);
      ue = madd_rn(ue, b.e[q], uh[q]);
    }
    double wb[M::NV], we[M::NV], wo[M::NV];
#pragma unroll
    for (int v = 0; v < M::NV; ++v) {
      double sb = mul_rn(b.h[0], wh[0][v]);
      double se = mul_rn(b.e[0], wh[0][v]);
      for (int q = 1; q < ord; ++q) {
        sb = madd_rn(sb, b.h[q], wh[q][v]);
        se = madd_rn(se, b.e[q], wh[q][v]);
      }
      wb[v] = sb;
      we[v] = se;
    }
    double I;
    if (RL) M::advance_rl(ue, wh[0], a.dt, P, wo, I, nclamp);
    else M::advance(ue, we, wb, b.alpha, a.dt, P, wo, I, nclamp);
    const double t_next = (double)(k + 1) * a.dt;
    double iapp = 0.0;
    if (stim) {
      for (int s = 0; s < a.n_pulses; ++s) {
        double sd = t_next - a.pulse_t0[s];
        if (sd < 0.0) continue;
        if (a.period > 0.0) sd -= a.period * floor(sd / a.period);
        if (sd < a.pulse_dur[s]) iapp += a.pulse_amp[s];
      }
    }
    const double un = (ub + a.dt * (iapp - I)) / b.alpha;
    // shift histories (newest first)
#pragma unroll
    for (int q = ORDER - 1; q > 0; --q) {
      uh[q] = uh[q - 1];
#pragma unroll
      for (int v = 0; v < M::NV; ++v) wh[q][v] = wh[q - 1][v];
    }
    uh[0] = un;
    bool ok = isfinite(un);
#pragma unroll
    for (int v = 0; v < M::NV; ++v) {
      wh[0][v] = wo[v];
      ok = ok && isfinite(wo[v]);
    }
    peak = fmax(peak, un);
    if (!ok) {
      finite = false;
      break;
    }
    if (traced && a.stride > 0 && ((k + 1) % a.stride) == 0 && row < a.trace_rows) {
      double* t = a.trace + (c * a.trace_rows + row) * rowlen;
      t[0] = t_next;
      t[1] = un;
      for (int v = 0; v < M::NV; ++v) t[2 + v] = wo[v];
      ++row;
    }
  }
  a.u[c] = uh[0];
#pragma unroll
  for (int v = 0; v < M::NV; ++v) a.W[(int64_t)v * a.ldw + c] = wh[0][v];
  if (a.peak) a.peak[c] = peak;
  if (!finite && a.status) atomicOr(a.status, 1);
  if (a.clamp_count && nclamp) atomicAdd(a.clamp_count, (unsigned long long)nclamp);
}

// One output row of run() (simulation.py:670-681): u_min, u_max, u[probes].
// Multi-block min/max: every block writes its partial, the last block to
// finish (completion counter) combines them in block order and resets the
// counter; block 0 gathers the probes.
constexpr int ROW_MAX_BLOCKS = (MDX_ROW_SCRATCH - 8) / 2;
__global__ void __launch_bounds__(256)
record_row(const double* __restrict__ u, int64_t n, const int64_t* __restrict__ probes,
           int nprobes, double* __restrict__ row, double* scratch) {
  __shared__ double smin[8], smax[8];
  __shared__ bool last;
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = u[i];
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = lo;
    smax[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  unsigned int* counter = reinterpret_cast<unsigned int*>(scratch + 2 * ROW_MAX_BLOCKS);
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, smin[w]);
      hi = fmax(hi, smax[w]);
    }
    scratch[2 * blockIdx.x] = lo;
    scratch[2 * blockIdx.x + 1] = hi;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < nprobes; k += blockDim.x) row[2 + k] = u[probes[k]];
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    lo = INFINITY;
    hi = -INFINITY;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      lo = fmin(lo, __ldcg(scratch + 2 * b));
      hi = fmax(hi, __ldcg(scratch + 2 * b + 1));
    }
    row[0] = lo;
    row[1] = hi;
    *counter = 0u;
  }
}

template <class M>
static typename M::Params load_params(const double* P, int np, int* err) {
  typename M::Params p;
  memset(&p, 0, sizeof(p));
  if (np != M::NP) {
    set_error("model expects %d packed parameters, got %d", M::NP, np);
    *err = MDX_ERR_ARG;
    return p;
  }
  memcpy(p.p, P, sizeof(double) * M::NP);
  M::derive(p);
  *err = MDX_OK;
  return p;
}

static inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

template <class M>
static int advance_impl(int64_t n, const double* u, const double* We, const double* Wb,
                        int64_t cs, int64_t vs, double alpha, double dt, const double* P,
                        int np, double* Wo, double* Io, unsigned long long* clamp,
                        cudaStream_t st) {
  int err;
  auto p = load_params<M>(P, np, &err);
  if (err) return err;
  if (n <= 0) return MDX_OK;
  advance_strided<M><<<grid_for(n, 128), 128, 0, st>>>(n, u, We, Wb, cs, vs, alpha, dt, p,
                                                       Wo, Io, clamp);
  return check_launch("mdx_ionic_advance");
}

template <class M>
static int advance_rl_impl(int64_t n, const double* u, const double* Wn, int64_t cs,
                           int64_t vs, double dt, const double* P, int np, double* Wo,
                           double* Io, unsigned long long* clamp, cudaStream_t st) {
  int err;
  auto p = load_params<M>(P, np, &err);
  if (err) return err;
  if (n <= 0) return MDX_OK;
  advance_rl_strided<M><<<grid_for(n, 128), 128, 0, st>>>(n, u, Wn, cs, vs, dt, p, Wo, Io,
                                                          clamp);
  return check_launch("mdx_ionic_advance_rl");
}

template <class M>
static int current_impl(int64_t n, const double* u, const double* W, int64_t cs, int64_t vs,
                        const double* P, int np, double* Io, cudaStream_t st) {
  int err;
  auto p = load_params<M>(P, np, &err);
  if (err) return err;
  if (n <= 0) return MDX_OK;
  current_strided<M><<<grid_for(n, 128), 128, 0, st>>>(n, u, W, cs, vs, p, Io);
  return check_launch("mdx_ionic_current");
}

template <class M>
static int rates_impl(int64_t n, const double* u, const double* W, const double* P, int np,
                      double* Io, double* dW, cudaStream_t st) {
  int err;
  auto p = load_params<M>(P, np, &err);
  if (err) return err;
  if (n <= 0) return MDX_OK;
  rates_aos<M><<<grid_for(n, 128), 128, 0, st>>>(n, u, W, p, Io, dW);
  return check_launch("mdx_ionic_point_rates");
}

template <class M>
static int tissue_impl(const mdx_tissue_ionic_args* a, const double* P, int np,
                       cudaStream_t st) {
  int err;
  auto p = load_params<M>(P, np, &err);
  if (err) return err;
  if (a->n <= 0) return MDX_OK;
  constexpr int B = MDX_IONIC_BLOCK;
  const int g = grid_for(a->n, B);
  if (a->gate_scheme != MDX_GATES_BDF && a->gate_scheme != MDX_GATES_RUSH_LARSEN) {
    set_error("gate scheme %d", a->gate_scheme);
    return MDX_ERR_ARG;
  }
  const bool rl = a->gate_scheme == MDX_GATES_RUSH_LARSEN;
  switch (a->order) {
    case 1:
      if (rl) tissue_ionic<M, 1, true><<<g, B, 0, st>>>(*a, p);
      else tissue_ionic<M, 1, false><<<g, B, 0, st>>>(*a, p);
      break;
    case 2:
      if (rl) tissue_ionic<M, 2, true><<<g, B, 0, st>>>(*a, p);
      else tissue_ionic<M, 2, false><<<g, B, 0, st>>>(*a, p);
      break;
    case 3:
      if (rl) tissue_ionic<M, 3, true><<<g, B, 0, st>>>(*a, p);
      else tissue_ionic<M, 3, false><<<g, B, 0, st>>>(*a, p);
      break;
    default: set_error("BDF order %d", a->order); return MDX_ERR_ARG;
  }
  return check_launch("mdx_tissue_ionic");
}

template <class M>
static int pace_impl(const mdx_pace_args* a, const double* P, int np, cudaStream_t st) {
  int err;
  auto p = load_params<M>(P, np, &err);
  if (err) return err;
  if (a->n_cells <= 0) return MDX_OK;
  const int g = (int)((a->n_cells + 127) / 128);
  if (a->gate_scheme == MDX_GATES_RUSH_LARSEN) {
    if (a->order != 1) {
      set_error("Rush-Larsen pacing is a one-step scheme: order must be 1, got %d", a->order);
      return MDX_ERR_ARG;
    }
    pace_cells<M, 1, true><<<g, 128, 0, st>>>(*a, p);
    return check_launch("mdx_pace_cells");
  }
  if (a->gate_scheme != MDX_GATES_BDF) {
    set_error("gate scheme %d", a->gate_scheme);
    return MDX_ERR_ARG;
  }
  switch (a->order) {
    case 1: pace_cells<M, 1, false><<<g, 128, 0, st>>>(*a, p); break;
    case 2: pace_cells<M, 2, false><<<g, 128, 0, st>>>(*a, p); break;
    case 3: pace_cells<M, 3, false><<<g, 128, 0, st>>>(*a, p); break;
    default: set_error("BDF order %d", a->order); return MDX_ERR_ARG;
  }
  return check_launch("mdx_pace_cells");
}

}  // namespace mdx

using namespace mdx;

#define MDX_DISPATCH(model, CALL)                                       \
  switch (model) {                                                      \
    case MDX_MODEL_ALIEV_PANFILOV: { using M = AlievPanfilov; return CALL; } \
    case MDX_MODEL_BUENO_OROVIO: { using M = BuenoOrovio; return CALL; }     \
    case MDX_MODEL_TTP06: { using M = TTP06; return CALL; }                  \
    default: set_error("unknown model id %d", model); return MDX_ERR_ARG;    \
  }

extern "C" {

const char* mdx_last_error(void) { return g_err; }

int mdx_abi_version(void) { return MDX_ABI_VERSION; }

int mdx_ionic_num_vars(int model) {
  switch (model) {
    case MDX_MODEL_ALIEV_PANFILOV: return AlievPanfilov::NV;
    case MDX_MODEL_BUENO_OROVIO: return BuenoOrovio::NV;
    case MDX_MODEL_TTP06: return TTP06::NV;
    default: return -1;
  }
}

int mdx_ionic_num_params(int model) {
  switch (model) {
    case MDX_MODEL_ALIEV_PANFILOV: return AlievPanfilov::NP;
    case MDX_MODEL_BUENO_OROVIO: return BuenoOrovio::NP;
    case MDX_MODEL_TTP06: return TTP06::NP;
    default: return -1;
  }
}

int mdx_ionic_advance(int model, int64_t n, const double* u_ext, const double* W_ext,
                      const double* W_bdf, int64_t cs, int64_t vs, double alpha, double dt,
                      const double* P, int np, double* W_out, double* I_out,
                      unsigned long long* clamp_count, void* stream) {
  MDX_DISPATCH(model, (advance_impl<M>(n, u_ext, W_ext, W_bdf, cs, vs, alpha, dt, P, np,
                                       W_out, I_out, clamp_count, (cudaStream_t)stream)))
}

int mdx_ionic_advance_rl(int model, int64_t n, const double* u, const double* W_n, int64_t cs,
                         int64_t vs, double dt, const double* P, int np, double* W_out,
                         double* I_out, unsigned long long* clamp_count, void* stream) {
  MDX_DISPATCH(model, (advance_rl_impl<M>(n, u, W_n, cs, vs, dt, P, np, W_out, I_out,
                                          clamp_count, (cudaStream_t)stream)))
}

int mdx_ionic_current(int model, int64_t n, const double* u, const double* W, int64_t cs,
                      int64_t vs, const double* P, int np, double* I_out, void* stream) {
  MDX_DISPATCH(model, (current_impl<M>(n, u, W, cs, vs, P, np, I_out, (cudaStream_t)stream)))
}

int mdx_ionic_point_rates(int model, int64_t n, const double* u, const double* W,
                          const double* P, int np, double* I_out, double* dW, void* stream) {
  MDX_DISPATCH(model, (rates_impl<M>(n, u, W, P, np, I_out, dW, (cudaStream_t)stream)))
}

int mdx_tissue_ionic(int model, const mdx_tissue_ionic_args* args, const double* P, int np,
                     void* stream) {
  MDX_DISPATCH(model, (tissue_impl<M>(args, P, np, (cudaStream_t)stream)))
}

int mdx_tissue_prep(const mdx_tissue_ionic_args* a, void* stream) {
  if (a->n <= 0) return MDX_OK;
  const int g = grid_for(a->n, 256);
  cudaStream_t st = (cudaStream_t)stream;
  switch (a->order) {
    case 1: tissue_prep<1><<<g, 256, 0, st>>>(*a); break;
    case 2: tissue_prep<2><<<g, 256, 0, st>>>(*a); break;
    case 3: tissue_prep<3><<<g, 256, 0, st>>>(*a); break;
    default: set_error("BDF order %d", a->order); return MDX_ERR_ARG;
  }
  return check_launch("mdx_tissue_prep");
}

int mdx_record_row(const double* u, int64_t n, const int64_t* probes, int nprobes,
                   double* row, double* scratch, void* stream) {
  if (n <= 0) return MDX_OK;
  int64_t g = (n + 256 * 8 - 1) / (256 * 8);
  const int64_t cap = std::min<int64_t>(ROW_MAX_BLOCKS, 2 * (int64_t)num_sms());
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  record_row<<<(int)g, 256, 0, (cudaStream_t)stream>>>(u, n, probes, nprobes, row, scratch);
  return check_launch("mdx_record_row");
}

int mdx_pace_cells(int model, const mdx_pace_args* args, const double* P, int np,
                   void* stream) {
  MDX_DISPATCH(model, (pace_impl<M>(args, P, np, (cudaStream_t)stream)))
}

}  // extern "C"
