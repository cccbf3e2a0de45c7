"""CPU implementation of the DistributedTissueSolver hooks - TEST INFRASTRUCTURE.

Runs the product's distributed host logic (slab partition, halo exchange,
pipelined-PCG driver, step bookkeeping) over gloo with numpy/oracle local
kernels, so tests/test_distributed.py can check the multi-rank algorithm on
a machine without GPUs.  Mirrors mdx_tissue_ionic / mdx_pcg_phase.
"""

import numpy as np
import scipy.sparse as sp
import torch

from oracle import monodomain_oracle as O
from paper_2308_01651_b200.distributed import (PH_ACT, PH_INIT, PH_SWEEP, PH_W0, PH_ZERO,
                                               DistributedTissueSolver, SlabComm,
                                               slab_partition)
from paper_2308_01651_b200.fem import detect_lattice
from paper_2308_01651_b200.simulation import RING_SLOTS

_ALPHA = {1: 1.0, 2: 1.5, 3: 11.0 / 6.0}
_HIST = {1: (1.0,), 2: (2.0, -0.5), 3: (3.0, -1.5, 1.0 / 3.0)}
_EXT = {1: (1.0,), 2: (2.0, -1.0), 3: (3.0, -3.0, 1.0)}


def _wsum(vs, ws):
    acc = ws[0] * vs[0]
    for w, v in zip(ws[1:], vs[1:]):
        acc = acc + w * v
    return acc


class _Scal:
    """Fields of mdx_pcg_scal (include/mdx.h)."""

    def __init__(self):
        self.b_norm = self.res = self.gamma = self.delta = self.gamma_prev = 0.0
        self.alpha_prev = self.alpha = self.beta = self.nonfinite = 0.0
        self.it = self.state = self.first = 0


def _scalars(s, c, phase, tol, max_iter):
    """Restatement of pcg_scalars_kernel (csrc/solver.cu) for the CPU backend."""
    if phase == 0:
        c.b_norm, c.res, c.gamma, c.nonfinite = np.sqrt(s[0]), np.sqrt(s[1]), s[2], s[3]
        c.it, c.first, c.gamma_prev, c.alpha_prev, c.alpha, c.beta = 0, 1, 0.0, 1.0, 0.0, 0.0
        if c.b_norm == 0.0:
            c.state, c.nonfinite, c.res = 2, 0.0, 0.0
        elif c.res <= tol * c.b_norm:
            c.state = 1
        else:
            c.state = 0
    elif c.state == 0 and phase == 1:
        c.delta, c.beta = s[0], 0.0
        c.alpha = c.gamma / c.delta
        c.first = 1
        if max_iter < 1:
            c.state = 3
    elif c.state == 0 and phase == 2:
        c.it += 1
        c.nonfinite, c.res = s[3], np.sqrt(s[2])
        if c.res <= tol * c.b_norm:
            c.state = 1
        elif c.it >= max_iter:
            c.state = 3
        else:
            c.gamma_prev, c.alpha_prev, c.gamma, c.delta = c.gamma, c.alpha, s[0], s[1]
            c.beta = c.gamma / c.gamma_prev
            c.alpha = c.gamma / (c.delta - c.beta * c.gamma / c.alpha_prev)
            c.first = 0


class CpuSlabTissue(DistributedTissueSolver):
    def __init__(self, config, group=None, device_scalars=False):
        import torch.distributed as dist

        self.device_scalars = device_scalars
        self.sums = torch.zeros(4, dtype=torch.float64)
        self.sum_parts = torch.zeros((3, 4), dtype=torch.float64)
        self.sweep_rows_seen = set()
        self._scal = _Scal()
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.slab = slab_partition(detect_lattice(config.mesh), self.nranks)[self.rank]
        self.comm = SlabComm(self.slab, group)
        orc = O.OracleTissue(config)
        self._orc = orc
        sl = self.slab
        gb, nl = sl.global_begin, sl.n_local
        self.gb, self.nl = gb, nl
        self.dt = config.dt
        self.step_index, self.time = 0, 0.0
        self.bdf_order = config.bdf_order
        self.tol = config.linear_solver.tolerance
        self.max_iter = config.linear_solver.max_iterations
        self.iters = []
        f = dict(dtype=torch.float64)
        self.u_ring = torch.zeros((RING_SLOTS, nl), **f)
        self.u_ring[0] = torch.from_numpy(orc.u_ring[0][gb:gb + nl].copy())
        self.head = 0
        self.u_hist = [orc.u_ring[0][gb:gb + nl].copy()]
        o0, o1 = sl.own_begin, sl.own_end
        self.o0, self.o1 = o0, o1
        (vol, Mv), = orc.vol_mass
        self.vol = vol
        self.w_hist = [vol.ring[0][gb + o0 - 0: gb + o1].copy()]  # owned AoS
        self.currents = torch.zeros(nl, **f)
        self.combo = torch.zeros(nl, **f)
        self.r, self.z_, self.w_, self.s_, self.p_ = (torch.zeros(nl, **f) for _ in range(5))
        self.m_ = torch.zeros(2 * nl, **f)
        self.act = orc.act[gb:gb + nl].copy()
        self.best = orc.best[gb:gb + nl].copy()
        self.frozen = orc.frozen[gb:gb + nl].copy()
        self.thr = orc.thr[gb:gb + nl]
        self._impulses = [(p, i) for p, i, _ in orc.impulses]
        self._profiles = [prof[gb:gb + nl] for _, _, prof in orc.impulses]

        def local_rows(csr):
            m = sp.csr_matrix((csr.data, csr.indices, csr.indptr), shape=(orc.n, orc.n))
            return m[gb + o0: gb + o1][:, gb: gb + nl].tocsr()

        self.M_loc = local_rows(orc.M)
        self.A_loc, self.dinv_loc = {}, {}
        for order in {min(k + 1, self.bdf_order) for k in range(self.bdf_order)}:
            orc._alpha = None
            orc._system(_ALPHA[order])
            self.A_loc[order] = local_rows(orc.A)
            self.dinv_loc[order] = orc.inv_diag[gb + o0: gb + o1].copy()
        self.x = None

    # backend protocol ----------------------------------------------------------
    def lift_currents(self):
        return (self.currents,)

    def m_buffer(self, k):
        return self.m_[k * self.nl:(k + 1) * self.nl]

    @property
    def z(self):
        return self.z_

    def potential_local(self):
        return self.u_ring[self.head]

    def _ionic(self, order, t_next, head, nslot, mask):
        o0, o1 = self.o0, self.o1
        uh = [h[o0:o1] for h in self.u_hist]
        u_ext = _wsum(uh, _EXT[order])
        u_bdf = _wsum(uh, _HIST[order])
        wb = _wsum(self.w_hist, _HIST[order])
        we = _wsum(self.w_hist, _EXT[order])
        wo = np.empty_like(we)
        io = np.empty(o1 - o0)
        O.advance(self.vol.model, u_ext, we, wb, _ALPHA[order], self.dt, self.vol.P, wo, io)
        self._w_new = wo
        cur = self.currents.numpy()
        cur[:] = 0.0
        cur[o0:o1] = io
        combo = u_bdf / self.dt
        app = None
        for k, prof in enumerate(self._profiles):
            if (mask >> k) & 1:
                app = prof[o0:o1].copy() if app is None else app + prof[o0:o1]
        if app is not None:
            combo = combo + app
        self.combo.numpy()[o0:o1] = combo
        self.u_ring[nslot] = 0.0
        self.u_ring[nslot, o0:o1] = torch.from_numpy(u_ext)
        self._order, self._t_next, self._uprev = order, t_next, self.u_ring[head].numpy()

    def _prepare_solve(self, order, t_next, head, nslot):
        self.x = self.u_ring[nslot]

    # DevicePcgDriver protocol: the phases gate on the scalar state exactly as
    # pcg_phase_kernel does with a non-null scal
    def phase_dev(self, kind, mbuf=0, rows=None, part=None):
        c = self._scal
        if kind in (PH_W0, PH_SWEEP) and c.state != 0:
            return
        if kind == PH_ZERO and c.state != 2:
            return
        if kind == PH_ACT and (c.state in (0, 3) or c.nonfinite != 0.0):
            return
        out = self.sums if part is None else self.sum_parts[part]
        out.copy_(self.phase(kind, c.alpha, c.beta, c.first, mbuf, rows=rows))

    def combine_parts(self, k):
        torch.sum(self.sum_parts[:k], 0, out=self.sums)

    def scalars(self, phase):
        _scalars(self.sums.numpy().copy(), self._scal, phase, self.tol, self.max_iter)

    def read_scalars(self):
        import copy

        return copy.copy(self._scal)

    def phase(self, kind, alpha=0.0, beta=0.0, first=0, mbuf=0, rows=None):
        o0, o1 = self.o0, self.o1
        A = self.A_loc[self._order]
        di = self.dinv_loc[self._order]
        if rows is not None:        # the sweep over a sub-range of the owned rows
            assert kind == PH_SWEEP and self.o0 <= rows[0] < rows[1] <= self.o1
            o0, o1 = rows
            A = A[o0 - self.o0:o1 - self.o0]
            di = di[o0 - self.o0:o1 - self.o0]
            self.sweep_rows_seen.add((o0, o1))
        x, r, z = self.x.numpy(), self.r.numpy(), self.z_.numpy()
        w, s, p = self.w_.numpy(), self.s_.numpy(), self.p_.numpy()
        out = np.zeros(4)
        if kind == PH_INIT:
            b = self.M_loc @ self.combo.numpy() - self.M_loc @ self.currents.numpy()
            rr = b - A @ x
            zz = di * rr
            r[o0:o1], z[o0:o1] = rr, zz
            out[:] = (b @ b, rr @ rr, rr @ zz, float((~np.isfinite(x[o0:o1])).sum()))
        elif kind == PH_W0:
            ww = A @ z
            w[o0:o1] = ww
            self.m_buffer((mbuf + 1) & 1).numpy()[o0:o1] = di * ww
            out[0] = ww @ z[o0:o1]
        elif kind == PH_SWEEP:
            mc = self.m_buffer(mbuf & 1).numpy()
            mn = self.m_buffer((mbuf + 1) & 1).numpy()
            nn = A @ mc
            r0, w0 = r[o0:o1].copy(), w[o0:o1].copy()
            u0 = di * r0
            zz = nn if first else beta * z[o0:o1] + nn
            ss = w0 if first else beta * s[o0:o1] + w0
            pp = u0 if first else beta * p[o0:o1] + u0
            xx = x[o0:o1] + alpha * pp
            rn = r0 - alpha * ss
            wn = w0 - alpha * zz
            z[o0:o1], s[o0:o1], p[o0:o1] = zz, ss, pp
            x[o0:o1], r[o0:o1], w[o0:o1] = xx, rn, wn
            mn[o0:o1] = di * wn
            un = di * rn
            out[:] = (rn @ un, wn @ un, rn @ rn, float((~np.isfinite(xx)).sum()))
        elif kind == PH_ZERO:
            x[o0:o1] = 0.0
        elif kind == PH_ACT:
            xn = x[o0:o1]
            up = self._uprev[o0:o1]
            slope = (xn - up) / self.dt
            unfrozen = ~self.frozen[o0:o1]
            better = unfrozen & (slope > self.best[o0:o1])
            self.best[o0:o1][better] = slope[better]
            self.act[o0:o1][better] = self._t_next
            crossed = unfrozen & (up <= self.thr[o0:o1]) & (xn > self.thr[o0:o1])
            self.frozen[o0:o1][crossed] = True
            # histories advance after a successful step
            self.u_hist = [self.x.numpy().copy()] + self.u_hist[:2]
            self.w_hist = [self._w_new] + self.w_hist[:2]
        return torch.from_numpy(out)
