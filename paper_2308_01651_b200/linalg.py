"""Jacobi-preconditioned CG on the device.

Mirror of `/root/reference/pkg/src/monodomain/linalg.py`: `csr_matvec`
(`:17-23`), `JacobiCg` (`:76-105`) and `solve_cg` (`:108-113`).  The whole
solve is one persistent cooperative launch of `mdx_pcg_solve`
(`csrc/solver.cu`): SpMV, vector updates, dot products and the convergence
test never leave the device.  Error behaviour is the reference's:
`ValueError` for a non-positive diagonal, `SolverDivergence(iters, rel)`
when the iteration cap is hit, `NonFiniteSolution` for NaN/inf output.
"""

import numpy as np

from . import _native as N
from .errors import NonFiniteSolution, SolverDivergence


def _torch():
    import torch

    return torch


class CgWorkspace:
    """Device scratch shared by every solve of one operator size."""

    def __init__(self, n, max_blocks=None):
        torch = _torch()
        if max_blocks is None:
            props = torch.cuda.get_device_properties(0)
            max_blocks = props.multi_processor_count * 8
        self.capacity = int(max_blocks)
        self.partials = torch.zeros(self.capacity * 8, dtype=torch.float64, device="cuda")
        self.barrier = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.p = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
        self.q = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
        self.r = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
        self.z = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
        self.w = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
        self.s = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
        self.m = torch.zeros(2 * max(n, 1), dtype=torch.float64, device="cuda")
        self.iters = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.relres = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.fail_step = torch.full((1,), -1, dtype=torch.int32, device="cuda")

    def fill(self, a):
        a.partials_capacity = self.capacity
        a.partials = N.ptr(self.partials)
        a.barrier = N.ptr(self.barrier)
        a.p = N.ptr(self.p)
        a.q = N.ptr(self.q)
        a.r = N.ptr(self.r)
        a.z = N.ptr(self.z)
        a.w = N.ptr(self.w)
        a.s = N.ptr(self.s)
        a.m = N.ptr(self.m)
        a.iters_out = N.ptr(self.iters)
        a.relres_out = N.ptr(self.relres)
        a.status = N.ptr(self.status)
        a.fail_step = N.ptr(self.fail_step)


class DeviceCsr:
    """CSR operator resident on the device (int64 indptr, int32 indices)."""

    def __init__(self, matrix):
        torch = _torch()
        m = matrix.tocsr()
        m.sort_indices()
        self.n = m.shape[0]
        self.indptr = torch.from_numpy(m.indptr.astype(np.int64)).cuda()
        self.indices = torch.from_numpy(m.indices.astype(np.int32)).cuda()
        self.data = torch.from_numpy(np.ascontiguousarray(m.data, np.float64)).cuda()
        self.nnz = int(m.nnz)

    def operator(self):
        op = N.Operator()
        op.kind = N.OP_CSR
        op.n = self.n
        op.indptr = N.ptr(self.indptr)
        op.indices = N.ptr(self.indices)
        op.nnz = self.nnz
        return op


def csr_matvec(indptr, indices, data, x, out):
    """out = A @ x with row-serial accumulation (linalg.py:17-23)."""
    import scipy.sparse as sp

    torch = _torch()
    n = len(indptr) - 1
    A = sp.csr_matrix((np.asarray(data), np.asarray(indices), np.asarray(indptr)),
                      shape=(n, len(x)))
    dev = DeviceCsr(A)
    a = N.CgArgs()
    a.op = dev.operator()
    a.a_val = N.ptr(dev.data)
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
    yd = torch.empty(n, dtype=torch.float64, device="cuda")
    N.check(N.lib().mdx_spmv(N.C.byref(a), N.ptr(xd), N.ptr(yd), N.stream_handle()),
            "mdx_spmv")
    out[...] = yd.cpu().numpy()


class JacobiCg:
    """CG bound to one CSR matrix and its inverse diagonal."""

    def __init__(self, matrix, tolerance=1e-10, max_iterations=2000):
        torch = _torch()
        self.matrix = matrix.tocsr()
        self.tolerance = float(tolerance)
        self.max_iterations = int(max_iterations)
        diag = self.matrix.diagonal()
        if (diag <= 0).any():
            raise ValueError("system matrix has non-positive diagonal")
        self.inv_diag = 1.0 / diag
        self._dev = DeviceCsr(self.matrix)
        self._dinv = torch.from_numpy(self.inv_diag).cuda()
        self._ws = CgWorkspace(self._dev.n)

    def solve_device(self, b, x):
        """Solve in place on device tensors; returns (iters, rel) lazily
        as device scalars (no synchronisation)."""
        a = N.CgArgs()
        a.op = self._dev.operator()
        a.a_val = N.ptr(self._dev.data)
        a.dinv = N.ptr(self._dinv)
        a.b = N.ptr(b)
        a.x = N.ptr(x)
        a.tol = self.tolerance
        a.max_iter = self.max_iterations
        self._ws.status.zero_()
        self._ws.fill(a)
        N.check(N.lib().mdx_pcg_solve(N.C.byref(a), 0, 0, N.stream_handle()),
                "mdx_pcg_solve")
        return self._ws.iters, self._ws.relres

    def solve(self, rhs, initial_guess=None):
        torch = _torch()
        rhs = np.asarray(rhs, dtype=np.float64)
        b = torch.from_numpy(np.ascontiguousarray(rhs)).cuda()
        x0 = np.zeros_like(rhs) if initial_guess is None else \
            np.asarray(initial_guess, dtype=np.float64)
        x = torch.from_numpy(np.array(x0, copy=True)).cuda()
        it_d, rel_d = self.solve_device(b, x)
        iters = int(it_d.item())
        rel = float(rel_d.item())
        if iters < 0:
            raise SolverDivergence(-iters, rel)
        xh = x.cpu().numpy()
        if not np.isfinite(xh).all():
            raise NonFiniteSolution("linear solve produced non-finite entries")
        return xh, iters, rel


def solve_cg(matrix, rhs, tolerance=1e-10, max_iterations=2000, initial_guess=None):
    return JacobiCg(matrix, tolerance, max_iterations).solve(rhs, initial_guess)
