"""CPU implementation of the DistributedTissueSolver hooks - TEST INFRASTRUCTURE.

Runs the product's distributed host logic (RCB partition, rank-local
problem, halo plans and exchange, pipelined-PCG drivers, step bookkeeping)
over gloo with numpy/oracle local kernels, so tests/test_distributed.py can
check the multi-rank algorithm on a machine without GPUs.  Each rank's local
operators and ionic kernels come from the oracle (pinned bit-for-bit to the
reference) run on the rank's local config; the phases restate
pcg_phase_kernel (csrc/solver.cu) in numpy, row classes included.
"""

import copy

import numpy as np
import torch

from oracle import monodomain_oracle as O
from paper_2308_01651_b200.distributed import (PH_ACT, PH_INIT, PH_SWEEP, PH_W0, PH_ZERO,
                                               ROW_BOUNDARY, ROW_INTERIOR,
                                               DistributedTissueSolver, HaloComm,
                                               local_config, row_classes)
from paper_2308_01651_b200.partition import build_part, partition, send_lists

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


class CpuPartTissue(DistributedTissueSolver):
    def __init__(self, config, group=None, device_scalars=False, owner=None):
        import torch.distributed as dist

        self.device_scalars = device_scalars
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.launches = 0
        mesh = config.mesh
        self.owner = partition(mesh, self.nranks) if owner is None else np.asarray(owner)
        part = build_part(mesh, self.owner, self.rank)
        part.send = send_lists(mesh, self.owner, part)
        self.part = part
        self.n_global = mesh.nodes.shape[0]
        self.comm = HaloComm(part, group, device="cpu")
        self.cls = row_classes(part)
        self.has_interior = bool((self.cls == ROW_INTERIOR).any())
        self.sel_seen = set()
        self.config = config
        orc = O.OracleTissue(local_config(config, part))
        self._orc = orc
        n = orc.n
        self.n_local = n
        self.dt = config.dt
        self._step, self._time = 0, 0.0
        self.bdf_order = config.bdf_order
        self.tol = config.linear_solver.tolerance
        self.max_iter = config.linear_solver.max_iterations
        self.iters = []
        self.sums = torch.zeros(4, dtype=torch.float64)
        self.sum_parts = torch.zeros((2, 4), dtype=torch.float64)
        self._scal = _Scal()
        f = dict(dtype=torch.float64)
        u0 = torch.from_numpy(orc.u_ring[0].copy())
        self.comm.halo(u0)                    # ghosts take their owner's initial u
        self.u_hist = [u0.numpy().copy()]
        self.w_hist = {id(v): [v.ring[0].copy()] for v, _ in orc.vol_mass}
        self.currents = torch.zeros((len(orc.vol_mass), n), **f)
        self._zero_lift = torch.zeros((len(config.volumes), n), **f)
        self.combo_ = torch.zeros(n, **f)
        self.x_ = torch.zeros(n, **f)
        self.r, self.z_, self.w_, self.s_, self.p_ = (torch.zeros(n, **f) for _ in range(5))
        self.m_ = torch.zeros(2 * n, **f)
        self.act = orc.act.copy()
        self.best = orc.best.copy()
        self.frozen = orc.frozen.copy()
        self.thr = orc.thr
        self._impulses = [(p, i) for p, i, _ in orc.impulses]
        self._profiles = [prof for _, _, prof in orc.impulses]
        self.A_loc, self.dinv_loc = {}, {}
        for order in {min(k + 1, self.bdf_order) for k in range(self.bdf_order)}:
            orc._alpha = None
            orc._system(_ALPHA[order])
            self.A_loc[order] = orc.A
            self.dinv_loc[order] = orc.inv_diag.copy()

    # -- state -----------------------------------------------------------------
    @property
    def step_index(self):
        return self._step

    @property
    def time(self):
        return self._time

    @property
    def x(self):
        return self.x_

    @property
    def combo(self):
        return self.combo_

    def lift_currents(self):
        """Per GLOBAL conducting volume (zeros where absent locally), as the
        product's backend."""
        labels = [v.cfg.label for v, _ in self._orc.vol_mass]
        return tuple(self.currents[labels.index(v.label)] if v.label in labels
                     else self._zero_lift[k]
                     for k, v in enumerate(x for x in self.config.volumes if not x.disabled))

    @property
    def z(self):
        return self.z_

    def m_buffer(self, k):
        return self.m_[k * self.n_local:(k + 1) * self.n_local]

    def potential_local(self):
        return torch.from_numpy(self.u_hist[0])

    def gather_potential(self):
        return self._gather(self.u_hist[0])

    def gather_activation_map(self):
        return self._gather(np.where(self.frozen, self.act, -1.0))

    def _gather(self, local):
        import torch.distributed as dist

        idx = self.part.owned_local()
        k = torch.tensor([idx.size])
        sizes = [torch.zeros_like(k) for _ in range(self.nranks)]
        dist.all_gather(sizes, k)
        width = int(max(int(s) for s in sizes))
        buf = torch.zeros((2, width), dtype=torch.float64)
        buf[0, :idx.size] = torch.from_numpy(self.part.nodes[idx].astype(np.float64))
        buf[1, :idx.size] = torch.from_numpy(np.asarray(local)[idx])
        parts = [torch.empty_like(buf) for _ in range(self.nranks)]
        dist.all_gather(parts, buf)
        out = np.empty(self.n_global)
        for p, s in zip(parts, sizes):
            m = int(s)
            out[p[0, :m].numpy().astype(np.int64)] = p[1, :m].numpy()
        return out

    # -- step (the product's step with CPU hooks) -------------------------------
    def step(self, device_scalars=None):
        from paper_2308_01651_b200.distributed import DevicePcgDriver, PipelinedPcgDriver

        dev = self.device_scalars if device_scalars is None else device_scalars
        order = min(self._step + 1, self.bdf_order)
        t_next = self._time + self.dt
        mask = 0
        for k, (protocol, i) in enumerate(self._impulses):
            if protocol.window_active(i, t_next):
                mask |= 1 << k
        self._ionic(order, t_next, mask)
        if dev:
            it, rel, nonfinite = DevicePcgDriver(
                self.comm, self, self.tol, self.max_iter,
                predict=max(self.iters[-1] - 1, 1) if self.iters else 8).solve()
        else:
            it, rel, nonfinite = PipelinedPcgDriver(self.comm, self, self.tol,
                                                    self.max_iter).solve()
        assert it >= 0 and not nonfinite
        if dev:
            self.phase_dev(PH_ACT)
        else:
            self.phase(PH_ACT)
        self.iters.append(it)
        self._step += 1
        self._time = t_next
        return it

    def _ionic(self, order, t_next, mask):
        orc = self._orc
        u_ext = _wsum(self.u_hist, _EXT[order])
        u_bdf = _wsum(self.u_hist, _HIST[order])
        self._w_new = {}
        cur = self.currents.numpy()
        cur[:] = 0.0
        for k, (v, _) in enumerate(orc.vol_mass):
            wh = self.w_hist[id(v)]
            wb = _wsum(wh, _HIST[order])
            we = _wsum(wh, _EXT[order])
            wo = np.empty_like(we)
            io = np.empty(v.dofs.size)
            O.advance(v.model, u_ext[v.dofs], we, wb, _ALPHA[order], self.dt, v.P, wo, io)
            self._w_new[id(v)] = wo
            cur[k, v.dofs] = io
        combo = u_bdf / self.dt
        for k, prof in enumerate(self._profiles):
            if (mask >> k) & 1:
                combo = combo + prof
        self.combo_.numpy()[:] = combo
        self.x_.numpy()[:] = u_ext
        self._order, self._t_next = order, t_next
        self._uprev = self.u_hist[0]

    # DevicePcgDriver protocol: the phases gate on the scalar state exactly as
    # pcg_phase_kernel does with a non-null scal
    def phase_dev(self, kind, mbuf=0, sel=3, part=None):
        c = self._scal
        if kind in (PH_W0, PH_SWEEP) and c.state != 0:
            return
        if kind == PH_ZERO and c.state != 2:
            return
        if kind == PH_ACT and (c.state in (0, 3) or c.nonfinite != 0.0):
            return
        out = self.sums if part is None else self.sum_parts[part]
        out.copy_(self.phase(kind, c.alpha, c.beta, c.first, mbuf, sel=sel))

    def combine_parts(self, k):
        torch.sum(self.sum_parts[:k], 0, out=self.sums)

    def scalars(self, phase):
        _scalars(self.sums.numpy().copy(), self._scal, phase, self.tol, self.max_iter)

    def read_scalars(self):
        return copy.copy(self._scal)

    def phase(self, kind, alpha=0.0, beta=0.0, first=0, mbuf=0, sel=3):
        rows = np.flatnonzero(self.cls & sel)
        if kind == PH_SWEEP:
            self.sel_seen.add(sel)
        A = self.A_loc[self._order]
        import scipy.sparse as sp

        Ar = sp.csr_matrix((A.data, A.indices, A.indptr),
                           shape=(self.n_local, self.n_local))[rows]
        di = self.dinv_loc[self._order][rows]
        x, r, z = self.x_.numpy(), self.r.numpy(), self.z_.numpy()
        w, s, p = self.w_.numpy(), self.s_.numpy(), self.p_.numpy()
        out = np.zeros(4)
        orc = self._orc
        if kind == PH_INIT:
            lift = np.zeros(rows.size)
            for k, (v, Mv) in enumerate(orc.vol_mass):
                Mr = sp.csr_matrix((Mv.data, Mv.indices, Mv.indptr),
                                   shape=(self.n_local, self.n_local))[rows]
                lift = lift + Mr @ self.currents[k].numpy()
            Mr = sp.csr_matrix((orc.M.data, orc.M.indices, orc.M.indptr),
                               shape=(self.n_local, self.n_local))[rows]
            b = Mr @ self.combo_.numpy() - lift
            inact = orc.inactive[rows]
            b[inact] = orc.rest[rows][inact]
            rr = b - Ar @ x
            zz = di * rr
            r[rows], z[rows] = rr, zz
            out[:] = (b @ b, rr @ rr, rr @ zz, float((~np.isfinite(x[rows])).sum()))
        elif kind == PH_W0:
            ww = Ar @ z
            w[rows] = ww
            self.m_buffer((mbuf + 1) & 1).numpy()[rows] = di * ww
            out[0] = ww @ z[rows]
        elif kind == PH_SWEEP:
            mc = self.m_buffer(mbuf & 1).numpy()
            mn = self.m_buffer((mbuf + 1) & 1).numpy()
            nn = Ar @ mc
            r0, w0 = r[rows].copy(), w[rows].copy()
            u0 = di * r0
            zz = nn if first else beta * z[rows] + nn
            ss = w0 if first else beta * s[rows] + w0
            pp = u0 if first else beta * p[rows] + u0
            xx = x[rows] + alpha * pp
            rn = r0 - alpha * ss
            wn = w0 - alpha * zz
            z[rows], s[rows], p[rows] = zz, ss, pp
            x[rows], r[rows], w[rows] = xx, rn, wn
            mn[rows] = di * wn
            un = di * rn
            out[:] = (rn @ un, wn @ un, rn @ rn, float((~np.isfinite(xx)).sum()))
        elif kind == PH_ZERO:
            x[rows] = 0.0
        elif kind == PH_ACT:
            xn = x[rows]
            up = self._uprev[rows]
            slope = (xn - up) / self.dt
            unfrozen = ~self.frozen[rows]
            better = unfrozen & (slope > self.best[rows])
            bi = rows[better]
            self.best[bi] = slope[better]
            self.act[bi] = self._t_next
            crossed = unfrozen & (up <= self.thr[rows]) & (xn > self.thr[rows])
            self.frozen[rows[crossed]] = True
            # histories advance after a successful step (owned entries are the
            # solution; ghost entries are refreshed by the next step's halo)
            self.u_hist = [x.copy()] + self.u_hist[:2]
            for v, _ in orc.vol_mass:
                self.w_hist[id(v)] = [self._w_new[id(v)]] + self.w_hist[id(v)][:2]
        return torch.from_numpy(out)
