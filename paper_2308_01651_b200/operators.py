"""Device-resident tissue operators: class-table stencil and CSR.

The tissue step needs, per node row i: the system matrix A = (alpha/dt) M + K
for each BDF phase, the mass M for the RHS, the per-volume masses M^v of the
ICI lift, the inactive flag with its pinned resting value, the activation
threshold, and 1/A_ii (`/root/reference/pkg/src/monodomain/simulation.py:
327-413`).

`StencilOperator` (structured hex slabs): every node row has at most 27
entries at fixed lattice offsets, and rows repeat: a uniform slab has 27
distinct row patterns (interior, faces, edges, corners); a slab with a scar
has a few hundred.  The device computes every node's row from the element
matrices, hashes it (coefficients to 36 bits relative to the row block's
largest entry: the reference integrates each element from its own node
coordinates, so analytically equal rows differ in the last bits), and the
host groups rows into classes whose table row is one representative node's
exact row.  A node then costs 2 bytes (its class id) and the operator
streams no matrix data - a matrix-free apply whose entries match the
reference's to ~1e-15 relative (`max_rel_dev`).  `CsrOperator` is the
bit-exact alternative (`TissueSolver(..., operator="csr")`).

`CsrOperator` (any mesh): the reference pattern with device-assembled values.

`DiaOperator` (any mesh whose numbering puts most couplings at a few index
offsets - every structured slab and the logical-grid ventricle of config 4):
the CSR values re-laid as symmetric diagonals.  Row i keeps its diagonal and
its couplings at the positive offsets d_s (c_s[i] = A[i, i + d_s]); the
coupling A[i, i - d_s] is read from row i - d_s's copy, so a P1-tet row of 15
entries costs 8 doubles per node and no column indices (120 + 60 B on CSR).
Couplings at any other offset (the ventricle's periodic seam) stay in a small
row-sorted remainder list.  The assembled matrices are symmetric up to the
last bit (the reference sums K_ab and K_ba in different orders): the relative
deviation introduced by reading the mirror is recorded in `max_rel_dev`
(~1e-16) and anything above 1e-10 is refused.
"""

import numpy as np

from . import _native as N
from .timestepping import ALPHA

STENCIL_CENTER = 13
MAX_CLASSES = 65535


def _torch():
    import torch

    return torch


def _combine_host(c, M, K):
    """c*M + K with two roundings (numpy never fuses), scipy's arithmetic."""
    return c * M + K


class StencilOperator:
    kind = N.OP_STENCIL27

    def __init__(self, dm, lattice, K_local, M_local, include_k, include_m,
                 lift_includes, inactive, rest, thr, dt, orders):
        torch = _torch()
        nx, ny, nz = lattice
        self.lattice = lattice
        self.n = dm.n
        rows_k = dm.stencil_rows(lattice, K_local, include_k)
        rows_m = dm.stencil_rows(lattice, M_local, include_m)
        lift_rows = [rows_m if inc is None else dm.stencil_rows(lattice, M_local, inc)
                     for inc in lift_includes]
        extra = torch.from_numpy(np.column_stack([
            inactive.astype(np.float64), rest.astype(np.float64),
            thr.astype(np.float64)])).cuda()
        key = torch.cat([rows_k, rows_m, *lift_rows, extra], dim=1).contiguous()
        nblk = 2 + len(lift_rows)
        hashes = torch.empty(self.n, dtype=torch.int64, device="cuda")
        N.check(N.lib().mdx_hash_rows(self.n, nblk, 3, N.ptr(key), N.ptr(hashes),
                                      N.stream_handle()), "mdx_hash_rows")
        h = hashes.cpu().numpy()
        uniq, first, inverse = np.unique(h, return_index=True, return_inverse=True)
        if uniq.size > MAX_CLASSES:
            raise OverflowError(f"{uniq.size} stencil classes exceed {MAX_CLASSES}")
        self.ncls = int(uniq.size)
        self.cls = torch.from_numpy(inverse.astype(np.uint16)).cuda()
        # per-node operator word: class id | neighbour-validity mask << 16
        k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1),
                              indexing="ij")
        i, j, k = i.ravel(), j.ravel(), k.ravel()
        mask = ((i > 0) * 1 | (i < nx) * 2 | (j > 0) * 4 | (j < ny) * 8 | (k > 0) * 16
                | (k < nz) * 32).astype(np.uint32)
        self.meta = torch.from_numpy(inverse.astype(np.uint32) | (mask << 16)).cuda()
        # the most frequent class among nodes with all 26 neighbours (the
        # solver stages its row in the constant bank); -1 when there is none
        full = inverse[mask == 63]
        self.dom_class = int(np.bincount(full).argmax()) if full.size else -1
        rep = torch.from_numpy(first.astype(np.int64)).cuda()
        bad = torch.zeros(2, dtype=torch.int64, device="cuda")
        N.check(N.lib().mdx_verify_classes(self.n, nblk, 3, N.ptr(key), N.ptr(self.cls),
                                           N.ptr(rep), N.ptr(bad), N.stream_handle()),
                "mdx_verify_classes")
        badh = bad.cpu().numpy()
        if int(badh[0]):
            raise OverflowError(f"{int(badh[0])} stencil rows off their class")
        # largest |row - class row| / max|class row| over all nodes and blocks
        self.max_rel_dev = float(badh[1:2].view(np.float64)[0])
        tab = key[rep].cpu().numpy()
        nl = len(lift_rows)
        self.tab_k = np.ascontiguousarray(tab[:, 0:27])
        self.tab_m = np.ascontiguousarray(tab[:, 27:54])
        self.tab_lift = [np.ascontiguousarray(tab[:, 54 + 27 * v: 81 + 27 * v])
                         for v in range(nl)]
        base = 54 + 27 * nl
        self.cls_inactive = tab[:, base] != 0.0
        self.cls_rest = np.ascontiguousarray(tab[:, base + 1])
        self.cls_thr = np.ascontiguousarray(tab[:, base + 2])
        del key, rows_k, rows_m, lift_rows

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).cuda()

        self.d_m = up(self.tab_m.ravel())
        self.d_lift = [self.d_m if inc is None else up(t.ravel())
                       for inc, t in zip(lift_includes, self.tab_lift)]
        self.d_inactive = up(self.cls_inactive.astype(np.uint8))
        self.d_rest = up(self.cls_rest)
        self.d_thr = up(self.cls_thr)
        self.a_tables, self.dinv = {}, {}
        self.host_a = {}
        for order in orders:
            c = ALPHA[order] / dt
            A = _combine_host(c, self.tab_m, self.tab_k)
            diag = A[:, STENCIL_CENTER].copy()
            diag[self.cls_inactive] = 1.0
            A[:, STENCIL_CENTER] = diag
            if (diag <= 0).any():
                raise ValueError("system matrix has non-positive diagonal")
            self.host_a[order] = A
            self.a_tables[order] = up(A.ravel())
            self.dinv[order] = up(1.0 / diag)

    def operator(self):
        op = N.Operator()
        op.kind = N.OP_STENCIL27
        op.ncls = self.ncls
        op.n = self.n
        op.nx1, op.ny1, op.nz1 = (d + 1 for d in self.lattice)
        op.meta = N.ptr(self.meta)
        return op

    def device_bytes(self):
        return 2 * self.n


class CsrOperator:
    """Reference pattern, device-assembled values; SELL-32 layout by default."""

    kind = N.OP_CSR

    def __init__(self, dm, space, K_local, M_local, include_k, include_m,
                 lift_includes, inactive, rest, thr, dt, orders, sell=True):
        torch = _torch()
        indptr, indices = space.pattern()
        self.n = dm.n
        self.nnz = int(indices.size)
        self.indptr = torch.from_numpy(indptr).cuda()
        self.indices = torch.from_numpy(indices).cuda()
        vk = dm.csr_values(space, K_local, include_k)
        self.d_m = dm.csr_values(space, M_local, include_m)
        self.d_lift = [self.d_m if inc is None else dm.csr_values(space, M_local, inc)
                       for inc in lift_includes]
        diag_pos = np.full(self.n, -1, dtype=np.int64)
        rows = np.repeat(np.arange(self.n), np.diff(indptr))
        on_diag = np.flatnonzero(rows == indices)
        diag_pos[rows[on_diag]] = on_diag
        if (diag_pos < 0).any():
            raise ValueError("system matrix has non-positive diagonal")
        dpos = torch.from_numpy(diag_pos).cuda()
        inact = torch.from_numpy(inactive.astype(np.bool_)).cuda()
        self.d_inactive = torch.from_numpy(inactive.astype(np.uint8)).cuda()
        self.d_rest = torch.from_numpy(np.ascontiguousarray(rest, np.float64)).cuda()
        self.d_thr = torch.from_numpy(np.ascontiguousarray(thr, np.float64)).cuda()
        self.a_tables, self.dinv = {}, {}
        for order in orders:
            c = ALPHA[order] / dt
            A = torch.empty(self.nnz, dtype=torch.float64, device="cuda")
            N.check(N.lib().mdx_combine_system(self.nnz, c, N.ptr(self.d_m), N.ptr(vk),
                                               N.ptr(A), N.stream_handle()),
                    "mdx_combine_system")
            diag = A[dpos]
            diag = torch.where(inact, torch.ones_like(diag), diag)
            A[dpos] = diag
            if bool((diag <= 0).any()):
                raise ValueError("system matrix has non-positive diagonal")
            self.a_tables[order] = A
            self.dinv[order] = 1.0 / diag
        if sell:
            self._to_sell(indptr, indices)

    def _to_sell(self, indptr, indices):
        """Re-layout every value array as SELL-32 (coalesced warp loads).

        Row order and the ascending-column order inside a row are kept, so
        the row sums round exactly as on CSR; padding entries are (0, row).
        """
        torch = _torch()
        n = self.n
        lens = np.diff(indptr)
        nch = (n + 31) // 32
        padded = np.zeros(nch * 32, dtype=np.int64)
        padded[:n] = lens
        width = padded.reshape(nch, 32).max(axis=1)
        cptr = np.zeros(nch + 1, dtype=np.int64)
        np.cumsum(32 * width, out=cptr[1:])
        rows = np.repeat(np.arange(n), lens)
        j = np.arange(indices.size) - indptr[rows]
        pos = cptr[rows // 32] + j * 32 + (rows % 32)
        total = int(cptr[-1])
        # column of every SELL slot: its own row for padding, then the real ones
        within = np.arange(total) - np.repeat(cptr[:-1], 32 * width)
        slot_row = (np.repeat(np.arange(nch), 32 * width) * 32 + within % 32)
        cols = np.minimum(slot_row, n - 1).astype(np.int32)
        cols[pos] = indices
        dpos = torch.from_numpy(pos).cuda()

        def relayout(vals):
            out = torch.zeros(total, dtype=torch.float64, device="cuda")
            out[dpos] = vals
            return out

        self.a_tables = {k: relayout(v) for k, v in self.a_tables.items()}
        m_new = relayout(self.d_m)
        self.d_lift = [m_new if v is self.d_m else relayout(v) for v in self.d_lift]
        self.d_m = m_new
        self.indptr = torch.from_numpy(cptr).cuda()
        self.indices = torch.from_numpy(cols).cuda()
        self.kind = N.OP_SELL
        self.sell_slots = total

    def operator(self):
        op = N.Operator()
        op.kind = self.kind
        op.n = self.n
        op.indptr = N.ptr(self.indptr)
        op.indices = N.ptr(self.indices)
        op.nnz = self.nnz
        return op

    def device_bytes(self):
        return 12 * self.nnz + 8 * (self.n + 1)


class DiaOperator:
    """Symmetric diagonal layout of a CsrOperator's values (MDX_OP_DIASYM)."""

    kind = N.OP_DIASYM
    MIN_FRACTION = 0.25           # an offset is stored as a diagonal when this
    MAX_REMAINDER = 0.05          # fraction of the rows couple there

    @staticmethod
    def plan(d_indptr, d_indices, n, max_np=N.DIA_MAX):
        """Diagonal offsets and entry classes of a CSR pattern on the device.

        Returns None when the pattern does not compress (too many offsets or
        too large a remainder, or an unsymmetric pattern)."""
        torch = _torch()
        dev = d_indices.device
        lens = d_indptr[1:] - d_indptr[:-1]
        rows = torch.repeat_interleave(torch.arange(n, device=dev), lens)
        off = d_indices.long() - rows
        uniq, cnt = torch.unique(off, return_counts=True)
        cnt_of = dict(zip(uniq.tolist(), cnt.tolist()))
        cand = [(c, d) for d, c in cnt_of.items()
                if d > 0 and c >= max(1, int(n * DiaOperator.MIN_FRACTION))]
        cand.sort(reverse=True)
        pos = sorted(d for _, d in cand[:max_np])
        if any(cnt_of.get(-d, 0) != cnt_of[d] for d in pos):
            return None
        if not pos:
            pos = [1]
        d_pos = torch.tensor(pos, dtype=torch.int64, device=dev)
        aoff = off.abs()
        slot = torch.searchsorted(d_pos, aoff).clamp_(max=len(pos) - 1)
        main = (d_pos[slot] == aoff) & (off != 0)
        diag = off == 0
        rem = ~(main | diag)
        if int(diag.sum()) != n:
            return None
        nrem = int(rem.sum())
        if nrem > DiaOperator.MAX_REMAINDER * off.numel():
            return None
        return dict(rows=rows, off=off, slot=slot, upper=main & (off > 0),
                    lower=main & (off < 0), diag=diag, rem=rem, nrem=nrem, pos=pos)

    def __init__(self, csr, plan):
        """Convert every value array of `csr` (a CsrOperator built with
        sell=False) with the plan from `DiaOperator.plan`."""
        torch = _torch()
        self.n = n = csr.n
        self.pos = plan["pos"]
        self.np_ = len(self.pos)
        self.ld = ld = ((n + 31) // 32) * 32
        rows, slot = plan["rows"], plan["slot"]
        up, lo, dg, rm = plan["upper"], plan["lower"], plan["diag"], plan["rem"]
        cols = csr.indices.long()
        self.nrem = plan["nrem"]
        self._up_idx = (1 + slot[up]) * ld + rows[up]
        self._lo_mirror = (1 + slot[lo]) * ld + cols[lo]
        self._dg_idx = rows[dg]
        self._dg, self._up, self._lo, self._rm = dg, up, lo, rm
        self.rem_row = rows[rm].to(torch.int32).contiguous()
        self.rem_col = csr.indices[rm].contiguous()
        nch = (n + 31) // 32
        cnt = torch.bincount(rows[rm] >> 5, minlength=nch) if self.nrem else \
            torch.zeros(nch, dtype=torch.int64, device=rows.device)
        self.rem_ptr = torch.zeros(nch + 1, dtype=torch.int32, device=rows.device)
        self.rem_ptr[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        self.max_rel_dev = 0.0
        self.a_tables = {k: self._convert(v) for k, v in csr.a_tables.items()}
        m_new = self._convert(csr.d_m)
        self.d_lift = [m_new if v is csr.d_m else self._convert(v) for v in csr.d_lift]
        self.d_m = m_new
        self.dinv = csr.dinv
        self.d_inactive, self.d_rest, self.d_thr = csr.d_inactive, csr.d_rest, csr.d_thr
        self.nnz = csr.nnz
        del self._up_idx, self._lo_mirror, self._dg_idx, self._dg, self._up, self._lo, self._rm
        if self.max_rel_dev > 1e-10:
            raise ValueError(f"operator is not symmetric (relative deviation "
                             f"{self.max_rel_dev:.3g})")

    def _convert(self, vals):
        torch = _torch()
        blk = torch.zeros((1 + self.np_) * self.ld + self.nrem, dtype=torch.float64,
                          device=vals.device)
        blk[self._dg_idx] = vals[self._dg]
        blk[self._up_idx] = vals[self._up]
        if self.nrem:
            blk[(1 + self.np_) * self.ld:] = vals[self._rm]
        lo = vals[self._lo]
        if lo.numel():
            mirror = blk[self._lo_mirror]
            scale = torch.maximum(lo.abs(), mirror.abs()).clamp_min(1e-300)
            dev = float(((lo - mirror).abs() / scale).max())
            self.max_rel_dev = max(self.max_rel_dev, dev)
        return blk

    def operator(self):
        op = N.Operator()
        op.kind = N.OP_DIASYM
        op.n = self.n
        op.nnz = self.nnz
        op.dia_np = self.np_
        op.dia_ld = self.ld
        for s, d in enumerate(self.pos):
            op.dia_off[s] = d
        op.rem_n = self.nrem
        op.rem_ptr = N.ptr(self.rem_ptr)
        op.rem_row = N.ptr(self.rem_row)
        op.rem_col = N.ptr(self.rem_col)
        return op

    def device_bytes(self):
        return 8 * (1 + self.np_) * self.ld + 16 * self.nrem
