"""CPU oracle for the monodomain hot path - TEST INFRASTRUCTURE ONLY.

Restates the reference's time step (`/root/reference/pkg/src/monodomain/
simulation.py:305-494`) with numpy on the host and the per-cell / per-row
kernels in `mdx_oracle.c` (OpenMP, no FMA contraction).  It is pinned
against the reference's own outputs in `tests/golden/` (see
tests/test_oracle.py) and then used as (a) the live checker of the CUDA path
in the GPU tests, (b) `__graft_entry__.smoke()`'s checker and (c) the CPU
baseline of `bench.py` (`--impl reference` and the `cpu_baseline` field).
The product package never imports this module.

Input: any config object with the reference's SimulationConfig fields
(mesh, fibers, volumes, stimuli, dt, bdf_order, ...), e.g. one built by
`paper_2308_01651_b200.configs`.
"""

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "mdx_oracle.c"
LIB = HERE / "_build" / "liboracle.so"

_ALPHA = {1: 1.0, 2: 1.5, 3: 11.0 / 6.0}
_HIST = {1: (1.0,), 2: (2.0, -0.5), 3: (3.0, -1.5, 1.0 / 3.0)}
_EXT = {1: (1.0,), 2: (2.0, -1.0), 3: (3.0, -3.0, 1.0)}
_MODEL_ID = {"Aliev-Panfilov": 0, "Bueno-Orovio": 1, "TTP06": 2}


def build(force=False):
    """gcc -O2 -fopenmp -ffp-contract=off -> oracle/_build/liboracle.so"""
    LIB.parent.mkdir(exist_ok=True)
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", str(SRC), "-o", str(LIB), "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        P = C.c_void_p
        _lib.orc_advance.argtypes = [C.c_int, C.c_long, P, P, P, C.c_double, C.c_double,
                                     P, P, P]
        _lib.orc_advance.restype = C.c_long
        _lib.orc_advance_rl.argtypes = [C.c_int, C.c_long, P, P, C.c_double, P, P, P]
        _lib.orc_advance_rl.restype = C.c_long
        _lib.orc_current.argtypes = [C.c_int, C.c_long, P, P, P, P]
        _lib.orc_csr_matvec.argtypes = [C.c_long, P, P, P, P, P]
        _lib.orc_cg.argtypes = [C.c_long, P, P, P, P, P, P, C.c_double, C.c_long, P, P]
        _lib.orc_cg.restype = C.c_long
        _lib.orc_assemble_mass.argtypes = [C.c_long, C.c_int, C.c_int, P, P, P, P, P, P,
                                           P, P, P]
        _lib.orc_assemble_stiffness.argtypes = [C.c_long, C.c_int, C.c_int, P, P, P, P,
                                                P, P, P, P, P, P, P, P]
        _lib.orc_num_threads.restype = C.c_int
        _lib.orc_incidence.argtypes = [C.c_long, C.c_long, C.c_int, P, P, P]
        _lib.orc_pattern_rows.argtypes = [C.c_long, C.c_int, P, P, P, P, P]
        _lib.orc_assemble_par.argtypes = [C.c_int, C.c_long, C.c_long, C.c_int, C.c_int,
                                          P, P, P, P, P, P, P, P, P, P, P, P, P, P, P]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def num_threads():
    return int(lib().orc_num_threads())


# ---------------------------------------------------------------------------
# ionic kernels (AoS (n, nv) arrays, the reference layout)
# ---------------------------------------------------------------------------


def advance(model_name, u_ext, W_ext, W_bdf, alpha, dt, P, W_out, I_out):
    u_ext = np.ascontiguousarray(u_ext, np.float64)
    W_ext = np.ascontiguousarray(W_ext, np.float64)
    W_bdf = np.ascontiguousarray(W_bdf, np.float64)
    P = np.ascontiguousarray(P, np.float64)
    return int(lib().orc_advance(_MODEL_ID[model_name], u_ext.shape[0], _p(u_ext),
                                 _p(W_ext), _p(W_bdf), alpha, dt, _p(P), _p(W_out),
                                 _p(I_out)))


def advance_rl(model_name, u, W_n, dt, P, W_out, I_out):
    """Rush-Larsen one-step update (mdx_oracle.c: ttp_rl1 / bo_rl1 / apf_rl1):
    only the integrator differs from `advance`; pinned by tests/golden/rl_kat.npz."""
    u = np.ascontiguousarray(u, np.float64)
    W_n = np.ascontiguousarray(W_n, np.float64)
    P = np.ascontiguousarray(P, np.float64)
    return int(lib().orc_advance_rl(_MODEL_ID[model_name], u.shape[0], _p(u), _p(W_n), dt,
                                    _p(P), _p(W_out), _p(I_out)))


def current(model_name, u, W, P, I_out):
    u = np.ascontiguousarray(u, np.float64)
    W = np.ascontiguousarray(W, np.float64)
    P = np.ascontiguousarray(P, np.float64)
    lib().orc_current(_MODEL_ID[model_name], u.shape[0], _p(u), _p(W), _p(P), _p(I_out))


# ---------------------------------------------------------------------------
# sparse algebra
# ---------------------------------------------------------------------------


class Csr:
    def __init__(self, indptr, indices, data):
        self.indptr = np.ascontiguousarray(indptr, np.int64)
        self.indices = np.ascontiguousarray(indices, np.int32)
        self.data = np.ascontiguousarray(data, np.float64)
        self.n = self.indptr.size - 1

    @classmethod
    def from_scipy(cls, m):
        m = m.tocsr()
        return cls(m.indptr, m.indices, m.data)

    def matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.n)
        lib().orc_csr_matvec(self.n, _p(self.indptr), _p(self.indices), _p(self.data),
                             _p(x), _p(out))
        return out

    def diagonal(self):
        d = np.zeros(self.n)
        rows = np.repeat(np.arange(self.n), np.diff(self.indptr))
        on = rows == self.indices
        d[rows[on]] = self.data[on]
        return d


def cg(A, inv_diag, b, x0, tol, max_iter):
    """_cg_kernel (linalg.py:34-73): returns (x, iters, relres)."""
    x = np.array(x0, dtype=np.float64, copy=True)
    b = np.ascontiguousarray(b, np.float64)
    work = np.empty(4 * A.n)
    rel = C.c_double(0.0)
    it = lib().orc_cg(A.n, _p(A.indptr), _p(A.indices), _p(A.data),
                      _p(np.ascontiguousarray(inv_diag)), _p(b), _p(x), tol, max_iter,
                      _p(work), C.byref(rel))
    return x, int(it), rel.value


# ---------------------------------------------------------------------------
# FE assembly (fem.py:36-486)
# ---------------------------------------------------------------------------


def _tables(kind):
    if kind == "Hex8":
        g = 1.0 / np.sqrt(3.0)
        signs = np.array([(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1),
                          (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)], np.float64)
        pts = np.array([(x, y, z) for z in (-g, g) for y in (-g, g) for x in (-g, g)])
        vals = np.empty((8, 8))
        grads = np.empty((8, 8, 3))
        for p, xi in enumerate(pts):
            for a, s in enumerate(signs):
                fac = (1.0 + s * xi) / 2.0
                vals[p, a] = fac[0] * fac[1] * fac[2]
                grads[p, a, 0] = s[0] / 2.0 * fac[1] * fac[2]
                grads[p, a, 1] = s[1] / 2.0 * fac[0] * fac[2]
                grads[p, a, 2] = s[2] / 2.0 * fac[0] * fac[1]
        return np.ones(8), vals, grads
    a, b = 0.5854101966249685, 0.1381966011250105
    vals = np.array([(a, b, b, b), (b, a, b, b), (b, b, a, b), (b, b, b, a)])
    g = np.array([(-1.0, -1.0, -1.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)])
    return np.full(4, 1.0 / 24.0), vals, np.broadcast_to(g, (4, 4, 3)).copy()


class Pattern(tuple):
    """(indptr, indices) of FeSpace.pattern (fem.py:242-259) plus the node ->
    incident-element lists the parallel assembly walks."""

    incidence = None


def pattern(n, elements):
    """Sorted unique node pairs sharing an element, rows in parallel (C)."""
    el = np.ascontiguousarray(elements, np.int32)
    ne, nl = el.shape
    ptr = np.empty(n + 1, np.int64)
    elem = np.empty(ne * nl, np.int32)
    lib().orc_incidence(n, ne, nl, _p(el), _p(ptr), _p(elem))
    indptr = np.empty(n + 1, np.int64)
    lib().orc_pattern_rows(n, nl, _p(el), _p(ptr), _p(elem), _p(indptr), None)
    indices = np.empty(int(indptr[-1]), np.int32)
    lib().orc_pattern_rows(n, nl, _p(el), _p(ptr), _p(elem), _p(indptr), _p(indices))
    pat = Pattern((indptr, indices))
    pat.incidence = (ptr, elem)
    return pat


def _assemble(kind, mesh, pat, include=None, sigma_rows=None, sigmas=None, fibers=None):
    """Element-order sums of fem.py:280-426, element matrices in parallel and
    each row scattered in ascending element order (identical sums)."""
    w, basis, grad = _tables(mesh.element_kind.value)
    indptr, indices = pat
    ptr, elem = pat.incidence
    data = np.zeros(indices.size)
    nodes = np.ascontiguousarray(mesh.nodes, np.float64)
    el = np.ascontiguousarray(mesh.elements, np.int32)
    inc = sr = sg = f0 = s0 = None
    if kind == 0:
        inc = np.ascontiguousarray(include, np.uint8)
    else:
        sr = np.ascontiguousarray(sigma_rows, np.int64)
        sg = np.ascontiguousarray(np.asarray(sigmas, np.float64).reshape(-1, 3))
        f0 = np.ascontiguousarray(fibers.f0, np.float64)
        s0 = np.ascontiguousarray(fibers.s0, np.float64)

    def pp(a):
        return None if a is None else _p(a)

    lib().orc_assemble_par(kind, nodes.shape[0], el.shape[0], el.shape[1], w.size, _p(nodes),
                           _p(el), pp(inc), pp(sr), pp(sg), pp(f0), pp(s0), _p(w), _p(basis),
                           _p(grad), _p(indptr), _p(indices), _p(ptr), _p(elem), _p(data))
    return Csr(indptr, indices, data)


def assemble_mass(mesh, include, pat):
    return _assemble(0, mesh, pat, include=include)


def assemble_stiffness(mesh, sigma_rows, sigmas, fibers, pat):
    return _assemble(1, mesh, pat, sigma_rows=sigma_rows, sigmas=sigmas, fibers=fibers)


def add_scaled(c, M, K):
    """(c*M + K) on a shared pattern, dropping exact zeros like scipy."""
    data = c * M.data + K.data
    return Csr(M.indptr, M.indices, data)


# ---------------------------------------------------------------------------
# Tissue solver (simulation.py:262-494)
# ---------------------------------------------------------------------------


class _Vol:
    pass


class OracleTissue:
    """Reference time loop on the CPU (numpy + mdx_oracle.c)."""

    def __init__(self, config, gate_scheme="bdf"):
        cfg = config
        self.cfg = cfg
        assert gate_scheme in ("bdf", "rush_larsen")
        self.gate_scheme = gate_scheme
        mesh = cfg.mesh
        n = mesh.nodes.shape[0]
        self.n = n
        self.dt = cfg.dt
        self.step_index = 0
        self.time = 0.0
        self.pat = pattern(n, mesh.elements)
        vols = []
        for vc in cfg.volumes:
            v = _Vol()
            v.cfg = vc
            from paper_2308_01651_b200.ionic import model_module  # metadata only
            from paper_2308_01651_b200.ionic.base import ModelKind, CellType

            kind = ModelKind.from_name(vc.ionic.kind.value)
            ct = (None if vc.ionic.cell_type is None
                  else CellType.from_name(vc.ionic.cell_type.value))
            mod = model_module(kind)
            v.model = kind.value
            v.nv = mod.NUM_VARS
            v.P = mod.pack(vc.ionic.parameters, ct)
            mats = np.isin(mesh.material_ids, np.array(vc.material_ids))
            v.dofs = np.unique(mesh.elements[mats].ravel())
            v.rest_u = float(vc.ionic.initial_state.u)
            th = cfg.activation.threshold
            v.threshold = mod.ACTIVATION_THRESHOLD if th is None else th
            v.ring = []
            vols.append(v)
        self.vols = vols
        scale = 1.0 / (cfg.chi_m * cfg.membrane_capacitance)
        sig = {}
        active = set()
        disabled = set()
        for v in vols:
            for m in v.cfg.material_ids:
                sig[m] = (v.cfg.sigma_l * scale, v.cfg.sigma_t * scale,
                          v.cfg.sigma_n * scale)
                if v.cfg.disabled:
                    disabled.add(m)
                else:
                    active.add(m)
        present = [int(m) for m in np.unique(mesh.material_ids)]
        table, row_of = [], {}
        for m in present:
            if m in disabled:
                row_of[m] = -1
            else:
                row_of[m] = len(table)
                table.append(sig[m])
        srows = np.array([row_of[int(m)] for m in mesh.material_ids], np.int64)
        self.M = assemble_mass(mesh, np.isin(mesh.material_ids, list(active)), self.pat)
        self.K = assemble_stiffness(mesh, srows, table, cfg.fibers, self.pat)
        # inactive DOFs: attached only to disabled materials (fem.py:225-239)
        touches = np.zeros(n, bool)
        attached = np.zeros(n, bool)
        el = mesh.elements
        attached[el.ravel()] = True
        act_el = np.isin(mesh.material_ids, list(active))
        touches[el[act_el].ravel()] = True
        self.inactive = attached & ~touches if disabled else np.zeros(n, bool)
        self.vol_mass = []
        for v in vols:
            if v.cfg.disabled:
                continue
            mats = set(v.cfg.material_ids)
            if mats == active:
                self.vol_mass.append((v, self.M))
            else:
                self.vol_mass.append((v, assemble_mass(
                    mesh, np.isin(mesh.material_ids, list(mats)), self.pat)))
        u0 = np.zeros(n)
        self.rest = np.zeros(n)
        self.thr = np.zeros(n)
        for v in sorted(vols, key=lambda v: min(v.cfg.material_ids), reverse=True):
            st = v.cfg.ionic.initial_state
            v.ring = [np.broadcast_to(np.asarray(st.w, np.float64),
                                      (v.dofs.size, v.nv)).copy()]
            u0[v.dofs] = st.u
            self.rest[v.dofs] = v.rest_u
            self.thr[v.dofs] = v.threshold
        u0[self.inactive] = self.rest[self.inactive]
        self.u_ring = [u0]
        self.impulses = []
        for prot in cfg.stimuli:
            for i in range(len(prot.sites)):
                prof = prot.spatial_factor(mesh.nodes, i) / cfg.membrane_capacitance
                prof[self.inactive] = 0.0
                self.impulses.append((prot, i, prof))
        self.act = np.full(n, -1.0)
        self.best = np.full(n, -np.inf)
        self.frozen = self.inactive.copy()
        self._alpha = None
        self.last_iterations = 0
        self.iters = []
        self.clamps = 0

    def _system(self, alpha):
        if self._alpha == alpha:
            return
        A = add_scaled(alpha / self.dt, self.M, self.K)
        diag = A.diagonal()
        diag[self.inactive] = 1.0
        rows = np.repeat(np.arange(self.n), np.diff(A.indptr))
        on = rows == A.indices
        A.data[on] = diag[rows[on]]
        self.A = A
        self.inv_diag = 1.0 / diag
        self._alpha = alpha

    @staticmethod
    def _wsum(ring, weights):
        acc = weights[0] * ring[0]
        for w, v in zip(weights[1:], ring[1:]):
            acc = acc + w * v
        return acc

    def step(self):
        order = min(self.step_index + 1, self.cfg.bdf_order)
        alpha, hw, ew = _ALPHA[order], _HIST[order], _EXT[order]
        t_next = self.time + self.dt
        self._system(alpha)
        u_bdf = self._wsum(self.u_ring, hw)
        u_ext = self._wsum(self.u_ring, ew)
        new_states, lift = [], None
        for v, Mv in self.vol_mass:
            wb = self._wsum(v.ring, hw)
            we = self._wsum(v.ring, ew)
            wo = np.empty_like(we)
            io = np.empty(v.dofs.size)
            if self.gate_scheme == "rush_larsen":     # one step from W_n at u_EXT
                self.clamps += advance_rl(v.model, u_ext[v.dofs], v.ring[0], self.dt, v.P,
                                          wo, io)
            else:
                self.clamps += advance(v.model, u_ext[v.dofs], we, wb, alpha, self.dt, v.P,
                                       wo, io)
            full = np.zeros(self.n)
            full[v.dofs] = io
            term = Mv.matvec(full)
            lift = term if lift is None else lift + term
            new_states.append((v, wo))
        combo = u_bdf / self.dt
        app = None
        for prot, i, prof in self.impulses:
            if prot.window_active(i, t_next):
                app = prof.copy() if app is None else app + prof
        if app is not None:
            combo = combo + app
        rhs = self.M.matvec(combo)
        if lift is not None:
            rhs = rhs - lift
        rhs[self.inactive] = self.rest[self.inactive]
        tol = self.cfg.linear_solver.tolerance
        mx = self.cfg.linear_solver.max_iterations
        u_new, it, rel = cg(self.A, self.inv_diag, rhs, u_ext, tol, mx)
        if it < 0:
            raise RuntimeError(f"oracle CG diverged (rel {rel:.3e})")
        self.last_iterations = it
        self.iters.append(it)
        u_prev = self.u_ring[0]
        slope = (u_new - u_prev) / self.dt
        unfrozen = ~self.frozen
        better = unfrozen & (slope > self.best)
        self.best[better] = slope[better]
        self.act[better] = t_next
        crossed = unfrozen & (u_prev <= self.thr) & (u_new > self.thr)
        self.frozen[crossed] = True
        for v, wo in new_states:
            v.ring = [wo] + v.ring[:2]
        self.u_ring = [u_new] + self.u_ring[:2]
        self.step_index += 1
        self.time = t_next
        return u_new

    @property
    def potential(self):
        return self.u_ring[0]

    @property
    def activation_map(self):
        return np.where(self.frozen, self.act, -1.0)


def pace_batch(model_name, P, u0, W0, dt, steps, order, n_stim, amp, t_end,
               gate_scheme="bdf"):
    """0D splitting for many cells (ionic/__init__.py:140-163), cfg-1 oracle.
    gate_scheme="rush_larsen": order 1 with the Rush-Larsen state update."""
    if gate_scheme == "rush_larsen":
        assert order == 1
    n = u0.size
    uh, wh = [u0.copy()], [W0.copy()]
    peak = u0.copy()
    W_out = np.empty_like(W0)
    I_out = np.empty(n)
    clamps = 0
    for k in range(steps):
        o = min(k + 1, order)
        ub = OracleTissue._wsum(uh, _HIST[o])
        ue = OracleTissue._wsum(uh, _EXT[o])
        wb = OracleTissue._wsum(wh, _HIST[o])
        we = OracleTissue._wsum(wh, _EXT[o])
        if gate_scheme == "rush_larsen":
            clamps += advance_rl(model_name, ue, wh[0], dt, P, W_out, I_out)
        else:
            clamps += advance(model_name, ue, we, wb, _ALPHA[o], dt, P, W_out, I_out)
        t_next = (k + 1) * dt
        iapp = np.zeros(n)
        if t_next < t_end:
            iapp[:n_stim] = amp
        un = (ub + dt * (iapp - I_out)) / _ALPHA[o]
        uh = [un] + uh[:2]
        wh = [W_out.copy()] + wh[:2]
        peak = np.maximum(peak, un)
    return uh[0], wh[0], peak, clamps


if __name__ == "__main__":
    build(force=True)
    print(LIB, num_threads(), "threads", os.cpu_count(), "cores")
