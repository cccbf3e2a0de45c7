// Setup-time operator assembly on the device.
//
// Compiled with --fmad=false: every product and sum is rounded separately,
// as in the reference's numba kernels (no fastmath), so element matrices and
// the assembled operator entries are bit-identical to
//   _assemble_mass_kernel       `/root/reference/pkg/src/monodomain/fem.py:280-314`
//   _assemble_stiffness_kernel  `fem.py:317-426`
// scattered in ascending element order like `_csr_add` (`fem.py:267-277`).
//
// Two destinations: CSR rows (any mesh) and 27-point stencil rows for
// structured hex slabs, from which the host derives the node-class tables of
// the matrix-free operator.
#include "common.cuh"

namespace mdx {

// Quadrature tables are tiny; they ride in the kernel parameter block.
struct QuadTables {
  int nq, nl;
  double w[8];
  double basis[8][8];
  double grad[8][8][3];
};

__global__ void __launch_bounds__(128)
element_matrices(int64_t ne, const double* __restrict__ nodes,
                 const int32_t* __restrict__ elems, const QuadTables T,
                 const int32_t* __restrict__ sigma_row, const double* __restrict__ sigmas,
                 const double* __restrict__ f0, const double* __restrict__ s0,
                 double* __restrict__ Ke, double* __restrict__ Me) {
  const int nl = T.nl, nq = T.nq;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* conn = elems + e * nl;
    double X[8][3];
    for (int a = 0; a < nl; ++a)
      for (int i = 0; i < 3; ++i) X[a][i] = nodes[(int64_t)conn[a] * 3 + i];
    const int srow = sigma_row ? sigma_row[e] : -1;
    double sl = 0.0, st = 0.0, sn = 0.0;
    if (srow >= 0) {
      sl = sigmas[srow * 3 + 0];
      st = sigmas[srow * 3 + 1];
      sn = sigmas[srow * 3 + 2];
    }
    double Kl[8][8], Ml[8][8];
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) Kl[a][b] = Ml[a][b] = 0.0;

    for (int q = 0; q < nq; ++q) {
      double jac[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      for (int a = 0; a < nl; ++a)
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) jac[i][j] += X[a][i] * T.grad[q][a][j];
      const double det = jac[0][0] * (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) -
                         jac[0][1] * (jac[1][0] * jac[2][2] - jac[1][2] * jac[2][0]) +
                         jac[0][2] * (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]);
      const double scale = T.w[q] * det;
      // consistent mass
      for (int a = 0; a < nl; ++a) {
        const double va = T.basis[q][a] * scale;
        for (int b = 0; b < nl; ++b) Ml[a][b] += va * T.basis[q][b];
      }
      if (srow < 0) continue;
      // anisotropic stiffness with the fiber frame re-orthonormalised per QP
      const double idet = 1.0 / det;
      double inv[3][3];
      inv[0][0] = (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) * idet;
      inv[0][1] = (jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2]) * idet;
      inv[0][2] = (jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1]) * idet;
      inv[1][0] = (jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2]) * idet;
      inv[1][1] = (jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0]) * idet;
      inv[1][2] = (jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2]) * idet;
      inv[2][0] = (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]) * idet;
      inv[2][1] = (jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1]) * idet;
      inv[2][2] = (jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0]) * idet;
      double g[8][3];
      for (int a = 0; a < nl; ++a)
        for (int i = 0; i < 3; ++i)
          g[a][i] = inv[0][i] * T.grad[q][a][0] + inv[1][i] * T.grad[q][a][1] +
                    inv[2][i] * T.grad[q][a][2];
      double fq[3] = {0.0, 0.0, 0.0}, sq[3] = {0.0, 0.0, 0.0}, nq3[3];
      for (int a = 0; a < nl; ++a) {
        const double w = T.basis[q][a];
        const int64_t nd = conn[a];
        for (int i = 0; i < 3; ++i) {
          fq[i] += w * f0[nd * 3 + i];
          sq[i] += w * s0[nd * 3 + i];
        }
      }
      const double fn = sqrt(fq[0] * fq[0] + fq[1] * fq[1] + fq[2] * fq[2]);
      for (int i = 0; i < 3; ++i) fq[i] /= fn;
      const double dot = fq[0] * sq[0] + fq[1] * sq[1] + fq[2] * sq[2];
      for (int i = 0; i < 3; ++i) sq[i] -= dot * fq[i];
      const double snn = sqrt(sq[0] * sq[0] + sq[1] * sq[1] + sq[2] * sq[2]);
      for (int i = 0; i < 3; ++i) sq[i] /= snn;
      nq3[0] = fq[1] * sq[2] - fq[2] * sq[1];
      nq3[1] = fq[2] * sq[0] - fq[0] * sq[2];
      nq3[2] = fq[0] * sq[1] - fq[1] * sq[0];
      double D[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          D[i][j] = sl * fq[i] * fq[j] + st * sq[i] * sq[j] + sn * nq3[i] * nq3[j];
      for (int a = 0; a < nl; ++a) {
        const double d0 = D[0][0] * g[a][0] + D[0][1] * g[a][1] + D[0][2] * g[a][2];
        const double d1 = D[1][0] * g[a][0] + D[1][1] * g[a][1] + D[1][2] * g[a][2];
        const double d2 = D[2][0] * g[a][0] + D[2][1] * g[a][1] + D[2][2] * g[a][2];
        for (int b = 0; b < nl; ++b)
          Kl[a][b] += scale * (d0 * g[b][0] + d1 * g[b][1] + d2 * g[b][2]);
      }
    }
    const int64_t base = e * nl * nl;
    for (int a = 0; a < nl; ++a)
      for (int b = 0; b < nl; ++b) {
        if (Ke) Ke[base + a * nl + b] = Kl[a][b];
        if (Me) Me[base + a * nl + b] = Ml[a][b];
      }
  }
}

// CSR rows in ascending element order. inc_ptr/inc_elem/inc_local list, for
// each row, the incident (element, local corner) pairs sorted by element.
__global__ void __launch_bounds__(128)
scatter_csr(int64_t n, int nl, const int32_t* __restrict__ elems,
            const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc_elem,
            const int8_t* __restrict__ inc_local, const uint8_t* __restrict__ include,
            const double* __restrict__ local, const int64_t* __restrict__ indptr,
            const int32_t* __restrict__ indices, double* __restrict__ data) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo0 = indptr[row], hi0 = indptr[row + 1];
    for (int64_t k = lo0; k < hi0; ++k) data[k] = 0.0;
    for (int64_t t = inc_ptr[row]; t < inc_ptr[row + 1]; ++t) {
      const int64_t e = inc_elem[t];
      if (include && !include[e]) continue;
      const int a = inc_local[t];
      for (int b = 0; b < nl; ++b) {
        const int32_t col = elems[e * nl + b];
        int64_t lo = lo0, hi = hi0;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (indices[mid] < col) lo = mid + 1; else hi = mid;
        }
        data[lo] += local[(e * nl + a) * nl + b];
      }
    }
  }
}

// 27-point stencil rows of a structured hex lattice (nx, ny, nz cells),
// cells visited in ascending element id (z, then y, then x).
__global__ void __launch_bounds__(128)
stencil_rows(int nx, int ny, int nz, const uint8_t* __restrict__ include,
             const double* __restrict__ local, double* __restrict__ rows) {
  const int nx1 = nx + 1, ny1 = ny + 1, nz1 = nz + 1;
  const int64_t n = (int64_t)nx1 * ny1 * nz1;
  // VTK corner -> lattice offset
  const int ox[8] = {0, 1, 1, 0, 0, 1, 1, 0};
  const int oy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
  const int oz[8] = {0, 0, 0, 0, 1, 1, 1, 1};
  for (int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; node < n;
       node += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(node / ((int64_t)nx1 * ny1));
    const int64_t rem = node - (int64_t)k * nx1 * ny1;
    const int j = (int)(rem / nx1);
    const int i = (int)(rem - (int64_t)j * nx1);
    double acc[27];
    for (int o = 0; o < 27; ++o) acc[o] = 0.0;
    for (int ck = k - 1; ck <= k; ++ck) {
      if (ck < 0 || ck >= nz) continue;
      for (int cj = j - 1; cj <= j; ++cj) {
        if (cj < 0 || cj >= ny) continue;
        for (int ci = i - 1; ci <= i; ++ci) {
          if (ci < 0 || ci >= nx) continue;
          const int64_t e = ci + (int64_t)nx * (cj + (int64_t)ny * ck);
          if (include && !include[e]) continue;
          int a = 0;
          for (int c = 0; c < 8; ++c)
            if (ci + ox[c] == i && cj + oy[c] == j && ck + oz[c] == k) a = c;
          for (int b = 0; b < 8; ++b) {
            const int dx = ci + ox[b] - i, dy = cj + oy[b] - j, dz = ck + oz[b] - k;
            const int o = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
            acc[o] += local[(e * 8 + a) * 8 + b];
          }
        }
      }
    }
    for (int o = 0; o < 27; ++o) rows[node * 27 + o] = acc[o];
  }
}

// Row classes for the stencil operator.  The reference assembles every
// element from its own node coordinates, so rows that are analytically equal
// differ in the last bits (i*h is not exactly uniform); classes therefore
// group rows that agree to QUANT_BITS bits relative to the largest entry of
// each 27-wide block.  Trailing `nextra` columns (flags, rest potential,
// threshold) must match exactly.
constexpr int QUANT_BITS = 36;

__device__ __forceinline__ int block_exponent(const double* r) {
  double m = 0.0;
  for (int k = 0; k < 27; ++k) m = fmax(m, fabs(r[k]));
  return m > 0.0 ? ilogb(m) : -2000;
}

__device__ __forceinline__ void fnv(unsigned long long& h, unsigned long long v) {
  for (int byte = 0; byte < 8; ++byte) {
    h ^= (v >> (8 * byte)) & 0xffull;
    h *= 1099511628211ull;
  }
}

__global__ void hash_rows(int64_t n, int nblk, int nextra, const double* __restrict__ rows,
                          unsigned long long* __restrict__ out) {
  const int width = 27 * nblk + nextra;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = 1469598103934665603ull;
    const double* r = rows + i * (int64_t)width;
    for (int b = 0; b < nblk; ++b) {
      const double* blk = r + 27 * b;
      const int e = block_exponent(blk);
      fnv(h, (unsigned long long)(e + 4096));
      for (int k = 0; k < 27; ++k) {
        const double qv = e > -2000 ? rint(ldexp(blk[k], QUANT_BITS - e)) : 0.0;
        fnv(h, (unsigned long long)(long long)qv);
      }
    }
    for (int k = 27 * nblk; k < width; ++k) fnv(h, __double_as_longlong(r[k]));
    out[i] = h;
  }
}

// Counts rows farther than 4 quanta from their class representative (or
// with different exact columns); also records the largest relative
// deviation |row - rep| / max|rep block| in dev_bits (as ordered bits).
__global__ void verify_classes(int64_t n, int nblk, int nextra,
                               const double* __restrict__ rows,
                               const uint16_t* __restrict__ cls,
                               const int64_t* __restrict__ rep,
                               unsigned long long* __restrict__ mismatches) {
  const int width = 27 * nblk + nextra;
  unsigned long long bad = 0;
  double worst = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* a = rows + i * (int64_t)width;
    const double* b = rows + rep[cls[i]] * (int64_t)width;
    bool ok = true;
    for (int blk = 0; blk < nblk; ++blk) {
      double m = 0.0;
      for (int k = 0; k < 27; ++k) m = fmax(m, fabs(b[27 * blk + k]));
      const double tol = m > 0.0 ? ldexp(m, 2 - QUANT_BITS) : 0.0;
      for (int k = 0; k < 27; ++k) {
        const double d = fabs(a[27 * blk + k] - b[27 * blk + k]);
        if (d > tol) ok = false;
        if (m > 0.0) worst = fmax(worst, d / m);
      }
    }
    for (int k = 27 * nblk; k < width; ++k)
      if (__double_as_longlong(a[k]) != __double_as_longlong(b[k])) ok = false;
    if (!ok) ++bad;
  }
  if (bad) atomicAdd(mismatches, bad);
  // non-negative doubles order like their bit patterns
  atomicMax(mismatches + 1, (unsigned long long)__double_as_longlong(worst));
}

// y = c*M + K entrywise (scipy's scalar-times-matrix then matrix add, each
// rounded), with optional unit diagonal overrides; then inv_diag = 1/diag.
__global__ void combine_system(int64_t m, double c, const double* __restrict__ M,
                               const double* __restrict__ K, double* __restrict__ A) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    A[i] = c * M[i] + K[i];
}

static inline int grid1(int64_t n, int b) {
  int64_t g = (n + b - 1) / b;
  const int64_t cap = (int64_t)num_sms() * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace mdx

using namespace mdx;

extern "C" {

int mdx_assemble_local(const mdx_assembly_args* a, void* stream) {
  if (a->n_elem <= 0) return MDX_OK;
  if (a->nl != 4 && a->nl != 8) {
    mdx::set_error("element must have 4 or 8 nodes, got %d", a->nl);
    return MDX_ERR_ARG;
  }
  QuadTables T;
  T.nq = a->nq;
  T.nl = a->nl;
  for (int q = 0; q < 8; ++q) {
    T.w[q] = q < a->nq ? a->quad_w[q] : 0.0;
    for (int l = 0; l < 8; ++l) {
      const bool ok = q < a->nq && l < a->nl;
      T.basis[q][l] = ok ? a->quad_basis[q * a->nl + l] : 0.0;
      for (int d = 0; d < 3; ++d)
        T.grad[q][l][d] = ok ? a->quad_grad[(q * a->nl + l) * 3 + d] : 0.0;
    }
  }
  element_matrices<<<grid1(a->n_elem, 128), 128, 0, (cudaStream_t)stream>>>(
      a->n_elem, a->nodes, a->elements, T, a->sigma_row, a->sigmas, a->f0, a->s0, a->K_local,
      a->M_local);
  return check_launch("mdx_assemble_local");
}

int mdx_scatter_csr(int64_t n, int nl, const int32_t* elements, const int64_t* inc_ptr,
                    const int32_t* inc_elem, const int8_t* inc_local, const uint8_t* include,
                    const double* local, const int64_t* indptr, const int32_t* indices,
                    double* data, void* stream) {
  if (n <= 0) return MDX_OK;
  scatter_csr<<<grid1(n, 128), 128, 0, (cudaStream_t)stream>>>(
      n, nl, elements, inc_ptr, inc_elem, inc_local, include, local, indptr, indices, data);
  return check_launch("mdx_scatter_csr");
}

int mdx_stencil_rows(int nx, int ny, int nz, const uint8_t* include, const double* local,
                     double* rows, void* stream) {
  const int64_t n = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  stencil_rows<<<grid1(n, 128), 128, 0, (cudaStream_t)stream>>>(nx, ny, nz, include, local,
                                                                 rows);
  return check_launch("mdx_stencil_rows");
}

int mdx_hash_rows(int64_t n, int nblk, int nextra, const double* rows,
                  unsigned long long* out, void* stream) {
  if (n <= 0) return MDX_OK;
  hash_rows<<<grid1(n, 256), 256, 0, (cudaStream_t)stream>>>(n, nblk, nextra, rows, out);
  return check_launch("mdx_hash_rows");
}

int mdx_verify_classes(int64_t n, int nblk, int nextra, const double* rows,
                       const uint16_t* cls, const int64_t* rep,
                       unsigned long long* mismatches, void* stream) {
  if (n <= 0) return MDX_OK;
  verify_classes<<<grid1(n, 256), 256, 0, (cudaStream_t)stream>>>(n, nblk, nextra, rows, cls,
                                                                  rep, mismatches);
  return check_launch("mdx_verify_classes");
}

int mdx_combine_system(int64_t m, double c, const double* M, const double* K, double* A,
                       void* stream) {
  if (m <= 0) return MDX_OK;
  combine_system<<<grid1(m, 256), 256, 0, (cudaStream_t)stream>>>(m, c, M, K, A);
  return check_launch("mdx_combine_system");
}

}  // extern "C"
