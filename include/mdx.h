/*
 * mdx.h - C ABI of the B200 (sm_100a) monodomain hot path.
 *
 * Every data pointer is a DEVICE pointer owned by the caller; `stream` is a
 * cudaStream_t (NULL = legacy default stream). Calls are stream-ordered and
 * asynchronous; none allocates device memory or synchronises. Return value:
 * MDX_OK (0) or a negative MDX_ERR_* code with text in mdx_last_error().
 * Numerical failures detected on the device (CG divergence, non-finite
 * solution) are reported through the caller's `status` word, never by
 * return code, so launches stay asynchronous.
 *
 * The reference (lifex-ep re-implementation, /root/reference/pkg) is
 * Python + numba; each entry point below names the reference function it
 * replaces. The Python package paper_2308_01651_b200 binds this header with
 * ctypes (see INTEGRATION.md for the binding a reference maintainer adds).
 */
#ifndef MDX_H
#define MDX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDX_ABI_VERSION 5

#define MDX_OK 0
#define MDX_ERR_ARG (-1)
#define MDX_ERR_CUDA (-2)
#define MDX_ERR_SIZE (-3)

/* ionic/__init__.py:40-49 model_module(kind) */
#define MDX_MODEL_ALIEV_PANFILOV 0
#define MDX_MODEL_BUENO_OROVIO 1
#define MDX_MODEL_TTP06 2

/* Ionic time integrator.  MDX_GATES_BDF is the reference's scheme (closed-form
 * implicit BDF gate solve, explicit BDF non-gates: <model>.advance_kernel).
 * MDX_GATES_RUSH_LARSEN is the mode BASELINE.json's north_star / config 1 name
 * and the reference does not have: from W_n alone,
 * gates w+ = w_inf + (w_n - w_inf) exp(-dt/tau), non-gates explicit Euler, with
 * the reference's own targets/currents/rates (ten_tusscher.py:175-350,
 * bueno_orovio.py:101-132) and the same [0,1] clamp. */
#define MDX_GATES_BDF 0
#define MDX_GATES_RUSH_LARSEN 1

/* bits of the status word the step kernels raise (mdx_cg_args.status) */
#define MDX_STATUS_DIVERGED 1
#define MDX_STATUS_NONFINITE 2
#define MDX_STATUS_STOPPED 4

#define MDX_OP_STENCIL27 1 /* structured hex slab, node-class tables */
#define MDX_OP_CSR 2       /* assembled CSR, int64 indptr / int32 indices */
#define MDX_OP_SELL 3      /* SELL-32: rows in chunks of 32, entries column-major per chunk;
                              indptr = chunk offsets (nchunks+1), indices = padded columns,
                              padding entries have value 0 and column = the row itself */
#define MDX_OP_DIASYM 4    /* symmetric diagonal storage (any mesh whose node numbering puts
                              most couplings at a few index offsets: structured hex/tet
                              slabs, the logical-grid ventricle): value block
                              [1 + dia_np][dia_ld] = diag, then c_s[i] = A[i, i + dia_off[s]]
                              (0 where absent); A[i, i - d] is read as c_s[i - d].
                              Couplings at other offsets (the ventricle's periodic seam)
                              are a row-sorted remainder list, rem_n values appended after
                              the block, found per 32-row chunk through rem_ptr */
#define MDX_DIA_MAX 16

#define MDX_MAX_LIFT 8 /* volumes in the ICI lift (simulation.py:342-352) */

const char* mdx_last_error(void);
int mdx_abi_version(void);

/* --------------------------------------------------------------------- */
/* Ionic-model module protocol (ionic/__init__.py:1-11)                   */
/* State element (i, v) lives at W[i*cs + v*vs]: AoS (cs=nv, vs=1) as the */
/* reference's (N, nv) arrays, or SoA (cs=1, vs=ld).                      */
/* --------------------------------------------------------------------- */
int mdx_ionic_num_vars(int model);   /* <model>.NUM_VARS */
int mdx_ionic_num_params(int model); /* len(<model>.pack(...)) */

/* <model>.advance_kernel(u_ext, W_ext, W_bdf, alpha, dt, P, W_out, I_out)
 *   bueno_orovio.py:152-186, ten_tusscher.py:374-403, aliev_panfilov.py:82-95.
 * P is a HOST array of np doubles (it is passed by value to the kernel).
 * clamp_count (device, may be NULL) accumulates the returned clamp count. */
int mdx_ionic_advance(int model, int64_t n, const double* u_ext, const double* W_ext,
                      const double* W_bdf, int64_t cs, int64_t vs, double alpha, double dt,
                      const double* P, int np, double* W_out, double* I_out,
                      unsigned long long* clamp_count, void* stream);

/* Rush-Larsen counterpart of advance_kernel (MDX_GATES_RUSH_LARSEN above): W_out from
 * W_n at potential u, I_out = I_ion(u, W_out).  Same layout/ownership rules. */
int mdx_ionic_advance_rl(int model, int64_t n, const double* u, const double* W_n, int64_t cs,
                         int64_t vs, double dt, const double* P, int np, double* W_out,
                         double* I_out, unsigned long long* clamp_count, void* stream);

/* <model>.current_kernel(u, W, P, I_out)
 *   bueno_orovio.py:146-149, ten_tusscher.py:368-371, aliev_panfilov.py:75-79 */
int mdx_ionic_current(int model, int64_t n, const double* u, const double* W, int64_t cs,
                      int64_t vs, const double* P, int np, double* I_out, void* stream);

/* <model>.point_rates(u, w, P) -> (I, dw) for n points, AoS W and dW
 *   bueno_orovio.py:135-143, ten_tusscher.py:353-365, aliev_panfilov.py:62-72 */
int mdx_ionic_point_rates(int model, int64_t n, const double* u, const double* W,
                          const double* P, int np, double* I_out, double* dW, void* stream);

/* --------------------------------------------------------------------- */
/* Tissue step, part 1: ionic update of one volume                        */
/*   TissueSolver.step ionic section, simulation.py:440-455, plus the      */
/*   HistoryRing.weighted_sum combinations it consumes (timestepping.py:89) */
/* Rings: slot s of the potential at u_ring + s*ldu; slot s of a volume's  */
/* state, variable v, at w_ring + (s*nv + v)*ldw. `head` is the slot of    */
/* the newest entry; the update writes slot (head+1) % ring_slots.         */
/* --------------------------------------------------------------------- */
typedef struct mdx_tissue_ionic_args {
  int64_t n;             /* DOFs of this volume (or all nodes for prep) */
  const int32_t* dofs;   /* volume DOF -> node id; NULL = identity */
  double* u_ring;        /* potential ring */
  int64_t ldu;
  double* w_ring;        /* ionic state ring of this volume (SoA) */
  int64_t ldw;
  int32_t ring_slots;    /* >= order + 1 */
  int32_t head;
  int32_t order;         /* BDF order of this step, min(step+1, bdf_order) */
  int32_t prep;          /* 1: also write combo and x0 (identity map only) */
  double dt;
  double* i_out;         /* full-length current of this volume (by node id) */
  unsigned long long* clamp_count; /* may be NULL */
  /* prep outputs: combo = u_BDF/dt + I_app (simulation.py:457-461) and the
   * CG warm start x0 = u_EXT written into the u ring's next slot */
  double* combo;
  const double* profiles; /* [n_impulses][ldp] applied-current profiles / C_m */
  int64_t ldp;
  uint64_t active_mask;  /* impulses whose window is open at t_{n+1} */
  int32_t n_impulses;
  int32_t gate_scheme;   /* MDX_GATES_BDF (reference) or MDX_GATES_RUSH_LARSEN */
  const int32_t* status; /* nonzero => an earlier step failed: no-op */
} mdx_tissue_ionic_args;

int mdx_tissue_ionic(int model, const mdx_tissue_ionic_args* args, const double* P, int np,
                     void* stream);
/* combo/x0 pass over all nodes when several volumes share the mesh */
int mdx_tissue_prep(const mdx_tissue_ionic_args* args, void* stream);

/* --------------------------------------------------------------------- */
/* Tissue step, part 2 / linear solver: persistent Jacobi PCG             */
/*   JacobiCg.solve + _cg_kernel (linalg.py:34-105); in tissue mode also   */
/*   the RHS assembly (simulation.py:457-465, fem.py:489-504), the         */
/*   finiteness check (:473-476) and _update_activation (:485-494).        */
/* --------------------------------------------------------------------- */
typedef struct mdx_operator {
  int32_t kind;          /* MDX_OP_STENCIL27, MDX_OP_CSR or MDX_OP_SELL */
  int32_t ncls;          /* stencil: number of node classes */
  int64_t n;             /* rows = nodes */
  int32_t nx1, ny1, nz1; /* stencil: nodes per axis (x fastest) */
  int32_t _pad;
  const uint32_t* meta;  /* stencil: class id | neighbour mask << 16, per node */
  const int64_t* indptr; /* csr */
  const int32_t* indices;
  int64_t nnz;
  /* MDX_OP_DIASYM (ABI v4) */
  int32_t dia_np;        /* positive offsets stored (<= MDX_DIA_MAX) */
  int32_t _pad1;
  int64_t dia_ld;        /* stride of the value block (>= n) */
  int64_t dia_off[MDX_DIA_MAX]; /* ascending positive offsets */
  int64_t rem_n;         /* remainder entries */
  const int32_t* rem_ptr;  /* [ceil(n/32) + 1] remainder range of each 32-row chunk */
  const int32_t* rem_row;  /* [rem_n] row of each remainder entry */
  const int32_t* rem_col;  /* [rem_n] column of each remainder entry */
} mdx_operator;

typedef struct mdx_cg_args {
  mdx_operator op;
  /* operator values: stencil -> [ncls][27] class tables; csr -> [nnz];
     diasym -> [(1 + dia_np) * dia_ld + rem_n] */
  const double* a_val;   /* (alpha/dt) M + K, inactive rows = identity */
  const double* dinv;    /* 1/diag(A): stencil [ncls], csr [n] */
  /* right-hand side: plain solve */
  const double* b;
  /* right-hand side: tissue (b == NULL) */
  const double* m_val;   /* M */
  const double* combo;   /* u_BDF/dt + I_app */
  int32_t n_lift;        /* ICI lift terms sum_v M^v I^v */
  int32_t step;          /* step index recorded on failure */
  const double* lift_val[MDX_MAX_LIFT];
  const double* lift_cur[MDX_MAX_LIFT];
  const uint8_t* inactive; /* stencil: per class; csr: per node; NULL = none */
  const double* rest;      /* pinned value of inactive rows */
  const double* thr;       /* activation threshold */
  /* vectors */
  double* x;             /* in: warm start (u_EXT); out: solution */
  double* p;             /* work vectors, n doubles each */
  double* q;
  double* r;
  double* z;             /* variants 1, 2 */
  /* variant 2 (pipelined CG) only: w = A u, s = A p, m = D^-1 w (2n: two
     buffers alternating between iterations) */
  double* w;
  double* s;
  double* m;
  /* activation map (tissue; act_time NULL = skip) */
  const double* u_prev;
  double* act_time;
  double* best_slope;
  uint8_t* frozen;
  double t_next, dt;
  double tol;
  int32_t max_iter;
  int32_t partials_capacity; /* blocks the partials buffer can hold */
  double* partials;      /* [2][partials_capacity][4] (double-buffered) */
  unsigned long long* barrier; /* grid-barrier counter, zero-initialised, reused */
  int32_t* iters_out;    /* iterations (reference convention: -max_iter) */
  double* relres_out;
  int32_t* status;       /* nonzero on entry => no-op; bit0 diverged, bit1 non-finite,
                            bit2 (MDX_STATUS_STOPPED) fully activated, see below */
  int32_t* fail_step;    /* receives `step` when status is raised */
  int32_t variant;       /* 0: reference recurrences (3 syncs/iter); 1: q = A z + beta q (2);
                            2: pipelined PCG (1 reduction/iter) */
  int32_t dom_class1;    /* stencil: 1 + id of the dominant interior class whose
                            coefficients are staged in constant memory (0 = none) */
  /* distributed phases (mdx_pcg_phase): rows [row_begin, row_end) are the
     rank-owned local rows; 0/0 = all rows */
  int64_t row_begin, row_end;
  /* optional run() output row of the solved potential, written by the solve
     itself (mdx_pcg_solve, tissue=1): row_out = [min x, max x, x[row_probes]]
     (device-accessible memory, e.g. mapped pinned host memory); NULL = none */
  double* row_out;
  const int64_t* row_probes;
  int32_t row_nprobes;
  int32_t _pad2;
  /* optional HOST copy of the 27 coefficients of class dom_class1 - 1 of
     a_val (the brick-streaming solver passes them as kernel parameters);
     read at launch time only; NULL = use the device table */
  const double* dom_row_host;
  /* optional HOST copy of the 27 coefficients of class dom_class1 - 1 of
     m_val (tissue RHS); with dom_row_host it lets the resident solver take
     both dominant rows as kernel parameters; NULL = fetched from m_val */
  const double* dom_m_row_host;
  /* distributed phases (ABI v4): when row_mask is set, mdx_pcg_phase[_dev]
     processes (and sums) only the rows i of [row_begin, row_end) with
     row_mask[i] & row_select != 0 (1 = owned interior, 2 = owned next to a
     ghost, 0 = ghost); NULL = every row of the range */
  const uint8_t* row_mask;
  int32_t row_select;
  int32_t _pad3;
  /* ABI v5, optional (NULL = off): 4 globaltimer stamps [ns] written by block 0 of
     mdx_pcg_solve: kernel start, RHS + initial residual done ("Monodomain
     assembly", simulation.py:457-465), CG loop done ("Linear solver"), activation
     and output row done ("Other") - the reference's per-step sections
     (simulation.py:225-254, 432-483) from inside the fused kernel */
  unsigned long long* tstamps;
  /* ABI v5, optional (NULL = off): *frozen_count accumulates the nodes whose
     activation time froze (simulation.py:485-494).  With stop_when_full != 0 the
     step that brings it to frozen_target stores its index in *fail_step and sets
     bit 2 (MDX_STATUS_STOPPED) of *status: later launches on the stream are
     no-ops, which is run(stop_when_fully_activated=True) (simulation.py:702-703)
     without a host synchronisation per step */
  unsigned long long* frozen_count;
  int64_t frozen_target;
  int32_t stop_when_full;
  int32_t _pad4;
} mdx_cg_args;

/* blocks_hint: grid size override (0 = automatic, capped at one co-resident wave) */
int mdx_pcg_solve(const mdx_cg_args* args, int tissue, int blocks_hint, void* stream);
/* One phase of the distributed (multi-GPU) pipelined PCG: phase 0 init,
 * 1 w0 = A u0, 2 sweep with host-supplied alpha/beta, 3 x = 0, 4 activation.
 * mbuf selects the m buffer read (the other one is written). When sums_out
 * is given, the phase's 4 partial sums are reduced (fixed order) into it.
 * Rows [row_begin, row_end) of the local (owned + ghost) numbering. */
int mdx_pcg_phase(const mdx_cg_args* args, int phase, int tissue, double alpha, double beta,
                  int first, int mbuf, double* sums_out, void* stream);

/* Device-resident scalar state of the distributed pipelined PCG: the host
 * enqueues phases without reading anything back; every rank's scalar
 * kernel sees the same all-reduced sums and takes the same decisions
 * (same formulas and order as the host driver, distributed.py). */
typedef struct {
  double b_norm, res, gamma, delta, gamma_prev, alpha_prev, alpha, beta, nonfinite;
  int32_t it;     /* sweeps consumed */
  int32_t state;  /* 0 iterating, 1 converged, 2 zero right-hand side, 3 max_iter reached */
  int32_t first;  /* the next sweep is the first */
  int32_t _pad;
} mdx_pcg_scal;

enum { MDX_SC_INIT = 0, MDX_SC_W0 = 1, MDX_SC_SWEEP = 2 };

/* scal <- f(scal, sums) after phase MDX_SC_*: one thread, stream-ordered */
int mdx_pcg_scalars(const double* sums, mdx_pcg_scal* scal, int phase, double tol,
                    int max_iter, void* stream);
/* mdx_pcg_phase with alpha/beta/first read from scal on the device; phases
 * gate themselves on scal->state (w0/sweep only while iterating, x = 0 only
 * for a zero right-hand side, activation only after a finite solve). */
int mdx_pcg_phase_dev(const mdx_cg_args* args, int phase, int tissue, const mdx_pcg_scal* scal,
                      int mbuf, double* sums_out, void* stream);
/* Halo packing of the distributed solver: dst[k] = src[idx[k]] (gather)
   and dst[idx[k]] = src[k] (scatter), k < n */
int mdx_gather(int64_t n, const int64_t* idx, const double* src, double* dst, void* stream);
int mdx_scatter(int64_t n, const int64_t* idx, const double* src, double* dst, void* stream);
/* y = A x with the same row arithmetic (csr_matvec, linalg.py:17-23) */
int mdx_spmv(const mdx_cg_args* args, const double* x, double* y, void* stream);

/* --------------------------------------------------------------------- */
/* Setup: operator assembly (fem.py:280-426, bit-identical)               */
/* --------------------------------------------------------------------- */
typedef struct mdx_assembly_args {
  int64_t n_elem;
  int32_t nl;            /* 8 hex, 4 tet */
  int32_t nq;
  const double* nodes;   /* [n][3] */
  const int32_t* elements; /* [n_elem][nl] */
  const double* quad_w;    /* HOST [nq] */
  const double* quad_basis;/* HOST [nq][nl] */
  const double* quad_grad; /* HOST [nq][nl][3] */
  const int32_t* sigma_row;/* [n_elem], -1 = no conduction; NULL = mass only */
  const double* sigmas;    /* [rows][3] (sigma_l, sigma_t, sigma_n) */
  const double* f0;        /* [n][3] */
  const double* s0;        /* [n][3] */
  double* K_local;         /* [n_elem][nl][nl] or NULL */
  double* M_local;         /* [n_elem][nl][nl] or NULL */
} mdx_assembly_args;

int mdx_assemble_local(const mdx_assembly_args* args, void* stream);
int mdx_scatter_csr(int64_t n, int nl, const int32_t* elements, const int64_t* inc_ptr,
                    const int32_t* inc_elem, const int8_t* inc_local, const uint8_t* include,
                    const double* local, const int64_t* indptr, const int32_t* indices,
                    double* data, void* stream);
int mdx_stencil_rows(int nx, int ny, int nz, const uint8_t* include, const double* local,
                     double* rows, void* stream);
/* Node classes of the stencil operator: rows are [nblk x 27 coefficients |
 * nextra exact columns]; coefficients are compared to 36 bits relative to
 * each block's largest entry (element matrices built from node coordinates
 * differ in the last bits between analytically equal elements).
 * mismatches[0] counts rows off their class representative, mismatches[1]
 * receives the largest relative deviation (as the bits of a double). */
int mdx_hash_rows(int64_t n, int nblk, int nextra, const double* rows,
                  unsigned long long* out, void* stream);
int mdx_verify_classes(int64_t n, int nblk, int nextra, const double* rows,
                       const uint16_t* cls, const int64_t* rep,
                       unsigned long long* mismatches, void* stream);
/* A = c*M + K entrywise (simulation.py:398) */
int mdx_combine_system(int64_t m, double c, const double* M, const double* K, double* A,
                       void* stream);

/* --------------------------------------------------------------------- */
/* 0D pacing batch: pace_single_cell (ionic/__init__.py:119-167) for many  */
/* cells at once, state and BDF history register-resident (config 1).     */
/* --------------------------------------------------------------------- */
typedef struct mdx_pace_args {
  int64_t n_cells;
  double* u;             /* [n_cells] in: initial, out: final */
  double* W;             /* [nv][ldw] SoA, in/out */
  int64_t ldw;
  double* peak;          /* [n_cells] running max of u, or NULL */
  int32_t order;         /* target BDF order (ramped from 1) */
  int32_t n_pulses;
  int64_t n_steps;
  double dt;
  int64_t n_stim_cells;  /* cells [0, n_stim_cells) receive the protocol */
  double period;
  double pulse_t0[8];
  double pulse_dur[8];
  double pulse_amp[8];
  int64_t n_trace_cells; /* cells [0, n_trace_cells) record a trace */
  int64_t trace_rows;
  int64_t stride;
  double* trace;         /* [n_trace_cells][trace_rows][2+nv] */
  unsigned long long* clamp_count;
  int32_t* status;       /* bit0: a cell lost finiteness */
  int32_t gate_scheme;   /* MDX_GATES_BDF, or MDX_GATES_RUSH_LARSEN (order must be 1) */
  int32_t _pad;
} mdx_pace_args;

int mdx_pace_cells(int model, const mdx_pace_args* args, const double* P, int np,
                   void* stream);

/* One run() output row (simulation.py:670-681): row = [min u, max u, u[probes]].
   scratch: MDX_ROW_SCRATCH doubles, zero-initialised once, reused (per-block
   partials + a completion counter); one call at a time per scratch buffer. */
#define MDX_ROW_SCRATCH 1024
int mdx_record_row(const double* u, int64_t n, const int64_t* probes, int nprobes,
                   double* row, double* scratch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MDX_H */
