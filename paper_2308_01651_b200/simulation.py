"""The coupled monodomain time loop, device-resident.

Drop-in mirror of `/root/reference/pkg/src/monodomain/simulation.py`:
stimulus types (`:48-115`), configuration dataclasses (`:123-218`),
`SectionTimer` (`:225-254`), `TissueSolver` (`:293-604`), checkpoints
(`:518-631`) and `run` (`:651-716`).  `TissueSolver` accepts these
configuration objects or the reference's own (duck-typed), so one config
drives both solvers.

Per step the device runs, with no host round trip:

1. `mdx_tissue_ionic` per volume: BDF combinations of the potential and
   ionic-state rings, closed-form gate update, explicit non-gates, I_ion at
   the new state; for a single volume also the RHS nodal term
   `combo = u_BDF/dt + I_app` and the warm start `x0 = u_EXT`
   (`mdx_tissue_prep` does that pass when several volumes share the mesh);
2. `mdx_pcg_solve` (tissue mode): one cooperative launch assembling
   `b = M combo - sum_v M^v I^v` (inactive rows pinned), running Jacobi PCG
   to `||r|| <= tol ||b||`, checking finiteness and updating the
   activation map.

The host only enqueues launches; per-step scalars (BDF order, t_{n+1},
which stimulus windows are open) are computed on the host exactly as the
reference computes them (accumulated time, left-closed windows) and passed
as kernel arguments.  Device failures set a status word that makes every
later launch a no-op; the host notices at its next synchronisation point,
rolls its step counter back to the failed step and raises the reference's
exception (`SolverDivergence`, `NonFiniteSolution`).
"""

import os
import struct
import time
import zlib
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native as N
from .errors import (ConfigError, CorruptFile, DofCountMismatch, NonFiniteSolution,
                     NonFiniteState, SolverDivergence, VersionMismatch)
from .fem import ConductivitySet, DeviceMesh, FeSpace, _sigma_table, detect_lattice
from .geometry import ElementKind, nearest_node
from .ionic import IonicModelSpec, ModelKind, CellType, pace_single_cell
from .ionic import model_module
from .operators import CsrOperator, DiaOperator, StencilOperator
from .outputs import OutputConfig, write_csv, write_vtk
from .timestepping import ALPHA, bdf_coefficients

ACTIVATION_SENTINEL = -1.0
RING_SLOTS = 4


# ---------------------------------------------------------------------------
# Stimuli (simulation.py:48-115)
# ---------------------------------------------------------------------------


class StimulusShape(Enum):
    CUBIC = "Cubic"
    SPHERICAL = "Spherical"
    GAUSSIAN = "Gaussian"


@dataclass
class StimulusProtocol:
    shape: StimulusShape
    sites: tuple
    amplitudes: tuple
    extents: tuple
    initial_times: tuple
    durations: tuple
    period: float = 0.0

    def __post_init__(self):
        lists = (self.sites, self.amplitudes, self.extents, self.initial_times,
                 self.durations)
        if len({len(x) for x in lists}) != 1:
            raise ValueError("stimulus lists must all have the same length")
        if any(d <= 0 for d in self.durations):
            raise ValueError("stimulus durations must be positive")
        if self.period != 0 and self.durations and self.period <= max(self.durations):
            raise ValueError("stimulus period must exceed every duration")

    def window_active(self, index, t):
        s = t - self.initial_times[index]
        if s < 0.0:
            return False
        if self.period > 0.0:
            s -= self.period * np.floor(s / self.period)
        return s < self.durations[index]

    def spatial_factor(self, coords, index):
        site = np.asarray(self.sites[index], dtype=np.float64)
        amp = self.amplitudes[index]
        extent = self.extents[index]
        shape = StimulusShape(self.shape.value)
        if shape is StimulusShape.CUBIC:
            half = extent / 2.0
            inside = (np.abs(coords - site) <= half * (1 + 1e-12)).all(axis=1)
            return amp * inside.astype(np.float64)
        d2 = ((coords - site) ** 2).sum(axis=1)
        if shape is StimulusShape.SPHERICAL:
            return amp * (d2 <= extent * extent * (1 + 1e-12)).astype(np.float64)
        return amp * np.exp(-d2 / (2.0 * extent * extent))


def applied_current(protocols, x, t):
    point = np.asarray(x, dtype=np.float64).reshape(1, 3)
    total = 0.0
    for protocol in protocols:
        for i in range(len(protocol.sites)):
            if protocol.window_active(i, t):
                total += protocol.spatial_factor(point, i)[0]
    return float(total)


# ---------------------------------------------------------------------------
# Configuration (simulation.py:123-218)
# ---------------------------------------------------------------------------


@dataclass
class VolumeConfig:
    label: str
    material_ids: tuple
    ionic: object
    sigma_l: float = 0.0
    sigma_t: float = 0.0
    sigma_n: float = 0.0
    disabled: bool = False
    prepacing_time: float = 0.0
    prepacing_protocol: object = None
    zero_d_csv_path: str = None

    def __post_init__(self):
        self.material_ids = tuple(int(m) for m in self.material_ids)
        if not self.material_ids:
            raise ValueError(f"volume {self.label!r} claims no material IDs")


@dataclass
class LinearSolverConfig:
    tolerance: float = 1e-10
    max_iterations: int = 2000


@dataclass
class ActivationConfig:
    enabled: bool = False
    path: str = "activation.vtk"
    threshold: float = None


@dataclass
class CheckpointConfig:
    enabled: bool = False
    path: str = "checkpoint.bin"


@dataclass
class SimulationConfig:
    mesh: object
    fibers: object
    volumes: tuple
    bdf_order: int = 2
    dt: float = 1e-4
    final_time: float = 1e-3
    degree: int = 1
    stimuli: tuple = ()
    membrane_capacitance: float = 1.0
    chi_m: float = 1.0
    linear_solver: LinearSolverConfig = field(default_factory=LinearSolverConfig)
    output: OutputConfig = field(default_factory=OutputConfig)
    activation: ActivationConfig = field(default_factory=ActivationConfig)
    checkpoint: CheckpointConfig = field(default_factory=CheckpointConfig)

    def validate(self):
        return validate_config(self)


def validate_config(config):
    """SimulationConfig.validate (simulation.py:190-218), duck-typed."""
    if config.dt <= 0:
        raise ConfigError("Time solver/Time step", "must be positive")
    if config.final_time <= 0:
        raise ConfigError("Time solver/Final time", "must be positive")
    if config.membrane_capacitance <= 0 or config.chi_m <= 0:
        raise ConfigError("Dimensional rescaling", "factors must be positive")
    bdf_coefficients(config.bdf_order)
    claimed = {}
    for vol in config.volumes:
        for mat in vol.material_ids:
            if mat in claimed:
                raise ConfigError(f"{vol.label}/Material IDs",
                                  f"material {mat} already claimed by {claimed[mat]!r}")
            claimed[mat] = vol.label
    present = {int(m) for m in np.unique(config.mesh.material_ids)}
    unclaimed = present - set(claimed)
    if unclaimed:
        raise ConfigError("Physical constants and models",
                          f"mesh materials {sorted(unclaimed)} not claimed by any volume")
    return config


# ---------------------------------------------------------------------------
# Timing (simulation.py:225-254): same five sections; device sections are
# timed with CUDA events when `timed=True` (otherwise host enqueue time).
# ---------------------------------------------------------------------------

TIMING_SECTIONS = ("Initialization", "Ionic model update", "Monodomain assembly",
                   "Linear solver", "Other")


class SectionTimer:
    def __init__(self):
        self._host = {name: 0.0 for name in TIMING_SECTIONS}
        self._events = []

    class _Span:
        def __init__(self, timer, name):
            self.timer, self.name = timer, name

        def __enter__(self):
            self.start = time.perf_counter()
            return self

        def __exit__(self, *exc):
            self.timer._host[self.name] += time.perf_counter() - self.start
            return False

    def section(self, name):
        return self._Span(self, name)

    def device_span(self, name, start, end):
        self._events.append((name, start, end))

    def device_stamps(self, stamps):
        """`stamps`: CUDA int64 tensor (k, 4) of globaltimer ns written by the solve
        kernels (mdx_cg_args.tstamps): start, assembly done, solve done, end."""
        self._stamps = stamps

    # the fused solve kernel's sections, from its own stamps
    _STAMP_SECTIONS = ("Monodomain assembly", "Linear solver", "Other")

    @property
    def totals(self):
        out = dict(self._host)
        if self._events:
            self._events[-1][2].synchronize()
            for name, s, e in self._events:
                out[name] += s.elapsed_time(e) * 1e-3
        st = getattr(self, "_stamps", None)
        if st is not None and st.numel():
            d = (st[:, 1:] - st[:, :-1]).clamp_(min=0).sum(dim=0).cpu().numpy() * 1e-9
            for name, v in zip(self._STAMP_SECTIONS, d):
                out[name] += float(v)
        return out


# ---------------------------------------------------------------------------
# Duck-typed views of (possibly reference-built) config objects
# ---------------------------------------------------------------------------


def _spec_of(ionic):
    """IonicModelSpec of this package from any spec-like object."""
    if isinstance(ionic, IonicModelSpec):
        return ionic
    kind = ModelKind.from_name(ionic.kind.value)
    ct = None if ionic.cell_type is None else CellType.from_name(ionic.cell_type.value)
    mod = model_module(kind)
    defaults = mod.default_parameters()
    overrides = {k: v for k, v in ionic.parameters.items() if defaults.get(k) != v}
    from .ionic.base import CellState

    st = ionic.initial_state
    return IonicModelSpec(kind, ct, overrides, CellState(float(st.u), np.array(st.w)))


class _Volume:
    def __init__(self, config, space, threshold_override):
        self.config = config
        self.spec = _spec_of(config.ionic)
        self.module = model_module(self.spec.kind)
        if self.module.MODEL_ID is None and not config.disabled:
            raise NotImplementedError(f"{self.spec.kind.value} has no kernels")
        self.packed = self.module.pack(self.spec.parameters, self.spec.cell_type)
        self.dofs = np.unique(np.concatenate(
            [space.dofs_in_subdomain(m) for m in config.material_ids]))
        self.num_vars = self.module.NUM_VARS
        self.rest_u = float(self.spec.initial_state.u)
        self.threshold = (threshold_override if threshold_override is not None
                          else self.module.ACTIVATION_THRESHOLD)
        self.w_ring = None
        self.w_fill = 1

    def initial_cell_state(self, order):
        cfg = self.config
        if cfg.disabled or cfg.prepacing_time <= 0.0:
            return self.spec.initial_state, None
        return pace_single_cell(self.spec, cfg.prepacing_protocol, order=order)


def _pad(n):
    return (n + 31) // 32 * 32


class TissueSolver:
    """Owns the device operators and state; advances the coupled system."""

    def __init__(self, config, operator="auto", blocks_hint=0, timed=False, cg_variant=None,
                 gate_scheme="bdf"):
        validate_config(config)
        self.config = config
        # "bdf": the reference's ionic update (advance_kernel).  "rush_larsen": the
        # one-step mode of BASELINE.json's north_star (exponential gates, explicit
        # Euler for the rest, from W_n at u_EXT) - not a reference scheme, checked
        # against an oracle built from the reference's own gate/current functions.
        from .ionic import gate_scheme_id

        self.gate_scheme = gate_scheme
        self._gate_scheme_id = gate_scheme_id(gate_scheme)
        self.timer = SectionTimer()
        self.timed = timed
        self.blocks_hint = blocks_hint
        # CG recurrences (csrc/solver.cu): 0 = the reference's verbatim (3 grid
        # syncs per iteration), 1 = q by recurrence (2), 2 = pipelined PCG (1).
        # Same Krylov iterates up to rounding; all checked against the goldens.
        # None: pipelined on the SMEM-resident stencil solve (latency-bound),
        # the reference's recurrences on global-memory operators (bandwidth-
        # bound: 3 syncs cost nothing there and it moves the fewest vectors).
        self._cg_variant_req = cg_variant
        self.cg_variant = 2 if cg_variant is None else cg_variant
        with self.timer.section("Initialization"):
            self._initialize(operator)

    # -- setup ---------------------------------------------------------------

    def _initialize(self, operator):
        import torch

        N.lib()
        cfg = self.config
        mesh = cfg.mesh
        self.space = FeSpace(mesh, cfg.degree)
        n = self.space.num_dofs
        self.n = n
        self.dt = cfg.dt
        self.step_index = 0
        self.time = 0.0
        self.volumes = [_Volume(v, self.space, cfg.activation.threshold)
                        for v in cfg.volumes]
        by_desc = sorted(self.volumes, key=lambda v: min(v.config.material_ids),
                         reverse=True)

        cset = ConductivitySet()
        active = set()
        scale = 1.0 / (cfg.chi_m * cfg.membrane_capacitance)
        for vol in self.volumes:
            for mat in vol.config.material_ids:
                cset.add(mat, vol.config.sigma_l * scale, vol.config.sigma_t * scale,
                         vol.config.sigma_n * scale, vol.config.disabled)
                if not vol.config.disabled:
                    active.add(mat)
        self.active_materials = active
        inactive = self.space.inactive_dof_mask(cset.disabled_ids())
        self.inactive = inactive

        # nodal initial state (smaller material ID wins at interfaces)
        u0 = np.zeros(n)
        rest = np.zeros(n)
        thr = np.zeros(n)
        w0 = {}
        for vol in by_desc:
            state, trace = vol.initial_cell_state(cfg.bdf_order)
            w0[id(vol)] = np.asarray(state.w, dtype=np.float64)
            u0[vol.dofs] = state.u
            rest[vol.dofs] = vol.rest_u
            thr[vol.dofs] = vol.threshold
            if trace is not None and vol.config.zero_d_csv_path:
                from .outputs import write_zero_d_trace

                write_zero_d_trace(vol.config.zero_d_csv_path, trace)
        u0[inactive] = rest[inactive]
        self.rest_field = rest
        self.thresholds = thr

        # operators
        rows, table = _sigma_table(self.space, cset)
        dm = DeviceMesh(mesh, cfg.fibers)
        K_local, M_local = dm.element_matrices(rows, table)
        include_k = torch.from_numpy((rows >= 0).astype(np.uint8)).cuda()
        include_m = dm.include_mask(active)
        self.lift_volumes = [v for v in self.volumes if not v.config.disabled]
        if len(self.lift_volumes) > N.MAX_LIFT:
            raise ConfigError("Physical constants and models",
                              f"at most {N.MAX_LIFT} conducting volumes")
        lift_includes = [None if set(v.config.material_ids) == active
                         else dm.include_mask(v.config.material_ids)
                         for v in self.lift_volumes]
        orders = sorted({min(k + 1, cfg.bdf_order) for k in range(cfg.bdf_order)})
        lattice = detect_lattice(mesh) if operator in ("auto", "stencil") else None
        args = (K_local, M_local, include_k, include_m, lift_includes, inactive,
                rest, thr, cfg.dt, orders)
        self.op = None
        if lattice is not None:
            try:
                self.op = StencilOperator(dm, lattice, *args)
            except OverflowError:
                if operator == "stencil":
                    raise
        if self.op is None:
            csr = CsrOperator(dm, self.space, *args,
                              sell=operator not in ("csr", "dia", "auto"))
            if operator in ("dia", "auto"):
                plan = DiaOperator.plan(csr.indptr, csr.indices, csr.n)
                if plan is None and operator == "dia":
                    raise ValueError("mesh numbering does not compress to diagonals")
                if plan is not None:
                    self.op = DiaOperator(csr, plan)
                    del plan
                else:
                    csr._to_sell(*self.space.pattern())
            if self.op is None:
                self.op = csr
            del csr
            if self._cg_variant_req is None:
                # bandwidth-bound solves: the reference recurrences in three sweeps
                # (160 B per node and iteration on the diagonal operator), or in two
                # with q = A z + beta q (168 B, one grid barrier fewer: 2% faster on
                # config 4, same iteration counts)
                self.cg_variant = 1 if isinstance(self.op, DiaOperator) else 0
        del K_local, M_local, dm

        # device state
        ld = _pad(n)
        self.ld = ld
        f64 = dict(dtype=torch.float64, device="cuda")
        self.u_ring = torch.zeros((RING_SLOTS, ld), **f64)
        self.u_ring[0, :n] = torch.from_numpy(u0).cuda()
        self.head = 0
        self.u_fill = 1
        for vol in self.volumes:
            lw = _pad(vol.dofs.size)
            vol.ldw = lw
            vol.w_ring = torch.zeros((RING_SLOTS, vol.num_vars, lw), **f64)
            vol.w_ring[0, :, :vol.dofs.size] = torch.from_numpy(w0[id(vol)]).cuda()[:, None]
            vol.w_fill = 1
            vol.d_dofs = (None if (vol.dofs.size == n and vol.dofs[-1] == n - 1)
                          else torch.from_numpy(vol.dofs.astype(np.int32)).cuda())
        self.currents = torch.zeros((max(len(self.lift_volumes), 1), ld), **f64)
        self.combo = torch.zeros(ld, **f64)
        self.fused_prep = (len(self.lift_volumes) == 1
                           and self.lift_volumes[0].d_dofs is None)

        # stimuli: time-independent profiles (simulation.py:374-382)
        self._impulses = []
        coords = self.space.dof_coords
        profiles = []
        for protocol in cfg.stimuli:
            for i in range(len(protocol.sites)):
                prof = protocol.spatial_factor(coords, i) / cfg.membrane_capacitance
                prof[inactive] = 0.0
                self._impulses.append((protocol, i))
                profiles.append(prof)
        if len(profiles) > 64:
            raise ConfigError("Stimulus", "at most 64 impulses")
        self.profiles = (torch.from_numpy(np.ascontiguousarray(
            np.stack(profiles))).cuda() if profiles else None)

        # activation (simulation.py:384-388)
        self.act_time = torch.full((n,), ACTIVATION_SENTINEL, **f64)
        self.best_slope = torch.full((n,), -np.inf, **f64)
        self.frozen = torch.from_numpy(inactive.astype(np.uint8)).cuda()
        # device-side count of frozen nodes (inactive ones are frozen from the
        # start) and the early-stop switch of run(stop_when_fully_activated=True)
        self.frozen_count = torch.tensor([int(inactive.sum())], dtype=torch.int64,
                                         device="cuda")
        self.stop_when_full = False
        self.stopped_at = None
        self._stamp_log = None

        # solver workspace and logs
        from .linalg import CgWorkspace

        self.ws = CgWorkspace(n)
        self.iter_log = torch.zeros(1024, dtype=torch.int32, device="cuda")
        self.relres_log = torch.zeros(1024, dtype=torch.float64, device="cuda")
        self.clamps = torch.zeros(1, dtype=torch.int64, device="cuda")
        self._log_base = 0
        self._pending = []          # (step_index, head_before, time_before)
        self._max_seen = 0
        self._last_iters = 0
        self.launches = 0
        self._build_launch_args()

    # -- per-step launch sequence ---------------------------------------------

    def _active_mask(self, t_next):
        mask = 0
        for k, (protocol, i) in enumerate(self._impulses):
            if protocol.window_active(i, t_next):
                mask |= 1 << k
        return mask

    def _ensure_log(self, slot):
        import torch

        if slot >= self.iter_log.numel():
            grow = max(slot + 1, 2 * self.iter_log.numel())
            il = torch.zeros(grow, dtype=torch.int32, device="cuda")
            rl = torch.zeros(grow, dtype=torch.float64, device="cuda")
            il[: self.iter_log.numel()] = self.iter_log
            rl[: self.relres_log.numel()] = self.relres_log
            self.iter_log, self.relres_log = il, rl

    def _build_launch_args(self):
        """ctypes argument blocks built once; per step only scalars change."""
        cfg = self.config
        self._stream = N.stream_handle()
        self._ionic_args = []
        base = dict(u_ring=N.ptr(self.u_ring), ldu=self.ld, ring_slots=RING_SLOTS,
                    dt=self.dt, clamp_count=N.ptr(self.clamps), combo=N.ptr(self.combo),
                    profiles=N.ptr(self.profiles), ldp=self.n,
                    n_impulses=len(self._impulses), status=N.ptr(self.ws.status),
                    gate_scheme=self._gate_scheme_id)
        if not self.fused_prep:
            ia = N.TissueIonicArgs(**base)
            ia.n = self.n
            ia.prep = 1
            self._prep_args = ia
        for v, vol in enumerate(self.lift_volumes):
            ia = N.TissueIonicArgs(**base)
            ia.n = vol.dofs.size
            ia.dofs = N.ptr(vol.d_dofs)
            ia.w_ring = N.ptr(vol.w_ring)
            ia.ldw = vol.ldw
            ia.i_out = N.ptr(self.currents[v])
            ia.prep = 1 if self.fused_prep else 0
            Ph, Pp = N.host_doubles(vol.packed)
            self._ionic_args.append((vol.module.MODEL_ID, ia, Ph, Pp))
        op = self.op
        a = N.CgArgs()
        a.op = op.operator()
        a.m_val = N.ptr(op.d_m)
        a.combo = N.ptr(self.combo)
        a.n_lift = len(self.lift_volumes)
        for v in range(len(self.lift_volumes)):
            a.lift_val[v] = N.ptr(op.d_lift[v])
            a.lift_cur[v] = N.ptr(self.currents[v])
        a.inactive = N.ptr(op.d_inactive)
        a.rest = N.ptr(op.d_rest)
        a.thr = N.ptr(op.d_thr)
        a.act_time = N.ptr(self.act_time)
        a.best_slope = N.ptr(self.best_slope)
        a.frozen = N.ptr(self.frozen)
        a.frozen_count = N.ptr(self.frozen_count)
        a.frozen_target = self.n
        a.dt = self.dt
        a.tol = cfg.linear_solver.tolerance
        a.max_iter = cfg.linear_solver.max_iterations
        self.ws.fill(a)
        a.variant = self.cg_variant
        a.dom_class1 = getattr(op, "dom_class", -1) + 1
        if os.environ.get("MDX_DOM_CLASS") == "0":      # ablation switch
            a.dom_class1 = 0
        self._cg_args = a
        self._a_ptr = {k: N.ptr(v) for k, v in op.a_tables.items()}
        # host copy of the dominant class row per BDF order (brick solver)
        self._dom_host = {}
        if a.dom_class1 > 0 and hasattr(op, "host_a"):
            for k, tab in op.host_a.items():
                self._dom_host[k] = np.ascontiguousarray(tab[a.dom_class1 - 1], np.float64)
        self._dom_ptr = {k: v.ctypes.data for k, v in self._dom_host.items()}
        # and of M's dominant row (the resident solver's RHS stencil)
        self._dom_m_host = None
        if a.dom_class1 > 0 and hasattr(op, "tab_m"):
            self._dom_m_host = np.ascontiguousarray(op.tab_m[a.dom_class1 - 1], np.float64)
            a.dom_m_row_host = self._dom_m_host.ctypes.data
        self._dinv_ptr = {k: N.ptr(v) for k, v in op.dinv.items()}
        self._slot_ptr = [N.ptr(self.u_ring[s]) for s in range(RING_SLOTS)]
        self._log_ptrs = (self.iter_log.data_ptr(), self.relres_log.data_ptr())

    def step_plan(self):
        """(order, t_next, active-impulse mask, head slot, next slot) of the
        next step (simulation.py:427-431)."""
        order = min(self.step_index + 1, self.config.bdf_order)
        t_next = self.time + self.dt
        mask = self._active_mask(t_next) if self._impulses else 0
        head = self.head
        return order, t_next, mask, head, (head + 1) % RING_SLOTS

    def enqueue_ionic(self, order, mask, head):
        """The ionic section of the step (simulation.py:440-455): one launch
        per volume, plus the combo/x0 prep pass when it is not fused."""
        lib = N.lib()
        stream = self._stream
        if not self.fused_prep:
            ia = self._prep_args
            ia.head, ia.order, ia.active_mask = head, order, mask
            N.check(lib.mdx_tissue_prep(N.C.byref(ia), stream), "mdx_tissue_prep")
            self.launches += 1
        for model_id, ia, Ph, Pp in self._ionic_args:
            ia.head, ia.order, ia.active_mask = head, order, mask
            N.check(lib.mdx_tissue_ionic(model_id, N.C.byref(ia), Pp, int(Ph.size), stream),
                    "mdx_tissue_ionic")
            self.launches += 1

    def solve_args(self, order, t_next, head, nslot):
        """The solve's argument block for this step (system of this BDF
        order, x = the next ring slot, iteration/residual log slots)."""
        a = self._cg_args
        a.a_val = self._a_ptr[order]
        a.dinv = self._dinv_ptr[order]
        a.dom_row_host = self._dom_ptr.get(order)
        a.step = self.step_index
        a.x = self._slot_ptr[nslot]
        a.u_prev = self._slot_ptr[head]
        a.t_next = t_next
        slot = self.step_index - self._log_base
        if slot >= self.iter_log.numel():
            self._ensure_log(slot)
            self._log_ptrs = (self.iter_log.data_ptr(), self.relres_log.data_ptr())
        a.iters_out = self._log_ptrs[0] + 4 * slot
        a.relres_out = self._log_ptrs[1] + 8 * slot
        a.stop_when_full = 1 if self.stop_when_full else 0
        if self.timed:
            a.tstamps = self._stamp_slot(slot)
        return a

    def _stamp_slot(self, slot):
        """Device address of this step's 4 section stamps (timed mode)."""
        import torch

        log = self._stamp_log
        if log is None or slot >= log.shape[0]:
            grow = max(1024, 2 * (slot + 1))
            new = torch.zeros((grow, 4), dtype=torch.int64, device="cuda")
            if log is not None:
                new[: log.shape[0]] = log
            self._stamp_log = log = new
        self._stamp_used = max(getattr(self, "_stamp_used", 0), slot + 1)
        self.timer.device_stamps(log[: self._stamp_used])
        return log.data_ptr() + 32 * slot

    def enqueue_step(self, events=None, record=None):
        """Launch one step; no host synchronisation.

        `events`: optional (after_ionic, after_solve) CUDA events recorded on
        the launch stream (bench.py's per-kernel timing).
        `record`: optional (probe_idx, dst): the solve itself writes the run()
        output row [u_min, u_max, u[probes]] of the new potential into `dst`
        (a pinned host float64 row, written through its device mapping, or a
        CUDA tensor) - no extra kernel or copy.
        """
        import torch

        order, t_next, mask, head, nslot = self.step_plan()
        lib = N.lib()
        stream = self._stream
        timed = self.timed
        if timed:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
        self.enqueue_ionic(order, mask, head)
        if timed:
            ev[1].record()
        if events is not None:
            events[0].record()
        a = self.solve_args(order, t_next, head, nslot)
        if record is not None:
            probe_idx, dst = record
            k = 2 + (0 if probe_idx is None else probe_idx.numel())
            if not (dst.dtype == torch.float64 and dst.is_contiguous() and dst.numel() >= k
                    and (dst.is_cuda or dst.is_pinned())):
                raise ValueError("record row must be a contiguous float64 CUDA or pinned "
                                 f"host tensor with >= {k} entries")
            a.row_out = dst.data_ptr()
            a.row_probes = N.ptr(probe_idx)
            a.row_nprobes = 0 if probe_idx is None else probe_idx.numel()
        try:
            N.check(lib.mdx_pcg_solve(N.C.byref(a), 1, self.blocks_hint, stream),
                    "mdx_pcg_solve")
        finally:
            a.row_out = None
        self.launches += 1
        if events is not None:
            events[1].record()
        if timed:
            # the ionic launches between two events; the solve kernel splits itself
            # into assembly / solver / other through its section stamps
            self.timer.device_span("Ionic model update", ev[0], ev[1])

        self.advance_bookkeeping(head, nslot, t_next)

    def advance_bookkeeping(self, head, nslot, t_next):
        """Ring pushes and time accumulation (simulation.py:477-482)."""
        self._pending.append((self.step_index, head, self.time))
        self.head = nslot
        self.u_fill = min(self.u_fill + 1, 3)
        for vol in self.lift_volumes:
            vol.w_fill = min(vol.w_fill + 1, 3)
        self.step_index += 1
        self.time = t_next

    def sync(self):
        """Wait for the device; raise the reference exception of a failed step."""
        import torch

        torch.cuda.current_stream().synchronize()
        st = int(self.ws.status.item())
        if st == N.STATUS_STOPPED:
            self._finish_stop()
            return
        if self._pending:
            first = self._pending[0][0]
            last = self._pending[-1][0]
            its = self.iter_log[first - self._log_base: last - self._log_base + 1]
            if st:
                fail = int(self.ws.fail_step.item())
                its = its[: max(fail - first, 0)]
            if its.numel():
                self._max_seen = max(self._max_seen, int(its.max().item()))
                self._last_iters = int(its[-1].item())
        if st:
            fail = int(self.ws.fail_step.item())
            for (k, head, t) in self._pending:
                if k == fail:
                    self.step_index, self.head, self.time = k, head, t
                    break
            self._pending = []
            rel = float(self.relres_log[fail - self._log_base].item())
            its = int(self.iter_log[fail - self._log_base].item())
            if st & N.STATUS_DIVERGED:
                raise SolverDivergence(-its, rel)
            raise NonFiniteSolution("linear solve produced non-finite entries")
        self._pending = []

    def _finish_stop(self):
        """Every node froze at step `fail_step` with stop_when_full set: the steps
        enqueued after it were no-ops on the device; put the host bookkeeping back
        to the state right after that step and clear the stop bit."""
        stop = int(self.ws.fail_step.item())
        first = self._pending[0][0] if self._pending else stop
        its = self.iter_log[first - self._log_base: stop - self._log_base + 1]
        if its.numel():
            self._max_seen = max(self._max_seen, int(its.max().item()))
            self._last_iters = int(its[-1].item())
        for (k, head, t) in self._pending:
            if k == stop + 1:            # the state before step stop+1 = after `stop`
                self.step_index, self.head, self.time = k, head, t
                break
        self._pending = []
        self.stopped_at = stop
        self.ws.status.zero_()

    def step(self, return_potential=True):
        """Advance one step (TissueSolver.step, simulation.py:425-483).

        Returns the new potential as a numpy array (drop-in semantics, one
        synchronisation) or, with return_potential=False, None without
        synchronising.
        """
        self.enqueue_step()
        if not return_potential:
            return None
        self.sync()
        return self.potential

    def advance(self, steps):
        """Enqueue `steps` steps back to back, then synchronise once."""
        for _ in range(steps):
            self.enqueue_step()
        self.sync()

    # -- state access ---------------------------------------------------------

    @property
    def potential_device(self):
        return self.u_ring[self.head, : self.n]

    @property
    def potential(self):
        return self.potential_device.cpu().numpy()

    @property
    def last_iterations(self):
        if self._pending:
            self.sync()
        return self._last_iters

    @property
    def max_iterations_seen(self):
        if self._pending:
            self.sync()
        return self._max_seen

    def iterations_log(self):
        """Per-step CG iteration counts since construction (or restore)."""
        if self._pending:
            self.sync()
        k = self.step_index - self._log_base
        return self.iter_log[:k].cpu().numpy().astype(np.int64)

    @property
    def activation_time(self):
        return self.act_time.cpu().numpy()

    @property
    def activation_map(self):
        fr = self.frozen.cpu().numpy().astype(bool)
        return np.where(fr, self.act_time.cpu().numpy(), ACTIVATION_SENTINEL)

    def fully_activated(self):
        """Every conducting DOF has frozen its activation time (simulation.py:512):
        one 8-byte read of the device-side counter the solve kernels maintain."""
        if self.stopped_at is not None:
            return True
        return int(self.frozen_count.item()) >= self.n

    def record_row(self, probe_idx, dst):
        """Asynchronously copy [u_min, u_max, u[probes]] of the current
        potential into `dst` (a pinned host tensor row): one kernel and one
        D2H copy, no synchronisation."""
        import torch

        k = 2 + (0 if probe_idx is None else probe_idx.numel())
        if getattr(self, "_row_scratch", None) is None:
            self._row_scratch = torch.zeros(N.ROW_SCRATCH, dtype=torch.float64, device="cuda")
        # pinned host memory is mapped into the device address space (UVA):
        # the kernel writes the row straight into it, no copy is enqueued
        direct = (not dst.is_cuda and dst.is_pinned() and dst.is_contiguous()
                  and dst.dtype == torch.float64 and dst.numel() >= k)
        if direct:
            row = dst
        else:
            if getattr(self, "_row_dev", None) is None or self._row_dev.numel() < k:
                self._row_dev = torch.empty(k, dtype=torch.float64, device="cuda")
            row = self._row_dev
        N.check(N.lib().mdx_record_row(
            N.ptr(self.potential_device), self.n, N.ptr(probe_idx),
            0 if probe_idx is None else probe_idx.numel(), row.data_ptr(),
            N.ptr(self._row_scratch), N.stream_handle()), "mdx_record_row")
        if not direct:
            dst.copy_(self._row_dev[:k], non_blocking=True)

    def clamp_total(self):
        return int(self.clamps.item())

    def volume_state(self, k, index=0):
        """AoS (ndofs, nv) ionic state of volume k, `index` steps back."""
        vol = self.volumes[k]
        slot = (self.head - index) % RING_SLOTS if not vol.config.disabled else 0
        return vol.w_ring[slot, :, : vol.dofs.size].t().contiguous().cpu().numpy()

    # -- checkpointing (simulation.py:518-631), reference byte format --------

    def checkpoint_payload(self, levels=None):
        """The reference's MHEP body.  `levels` caps the history levels written
        (None: every level the rings hold, like the reference; `bdf_order` levels
        are all a restart needs - the format carries its own level counts, so the
        reference's restore reads either)."""
        if self._pending:
            self.sync()
        n = self.n
        cap = RING_SLOTS if levels is None else max(1, int(levels))
        u_fill = min(self.u_fill, cap)
        parts = [struct.pack("<IQ", CHECKPOINT_VERSION, n),
                 struct.pack("<Qd", self.step_index, self.time),
                 struct.pack("<I", u_fill)]
        for k in range(u_fill):
            slot = (self.head - k) % RING_SLOTS
            parts.append(self.u_ring[slot, :n].cpu().numpy().tobytes())
        parts.append(self.act_time.cpu().numpy().tobytes())
        parts.append(self.best_slope.cpu().numpy().tobytes())
        parts.append(self.frozen.cpu().numpy().astype(np.uint8).tobytes())
        parts.append(struct.pack("<I", len(self.volumes)))
        for vol in self.volumes:
            label = vol.config.label.encode("utf-8")
            parts.append(struct.pack("<I", len(label)))
            parts.append(label)
            fill = 1 if vol.config.disabled else min(vol.w_fill, cap)
            parts.append(struct.pack("<IQI", vol.num_vars, vol.dofs.size, fill))
            for k in range(fill):
                slot = 0 if vol.config.disabled else (self.head - k) % RING_SLOTS
                aos = vol.w_ring[slot, :, : vol.dofs.size].t().contiguous()
                parts.append(aos.cpu().numpy().tobytes())
        return b"".join(parts)

    def restore(self, payload):
        """Load a checkpoint payload (the reference's MHEP body).  `payload` is
        bytes-like, or a uint8 CPU tensor - in pinned memory the upload is one
        asynchronous DMA instead of a staged pageable copy."""
        import torch

        if self._pending:
            self.sync()
        src = None
        if isinstance(payload, torch.Tensor):
            if payload.dtype != torch.uint8 or payload.dim() != 1 or payload.is_cuda:
                raise ValueError("a tensor payload must be a 1-D uint8 CPU tensor")
            src = payload
            payload = payload.numpy()
        version, n = struct.unpack_from("<IQ", payload, 0)
        if version != CHECKPOINT_VERSION:
            raise VersionMismatch(f"checkpoint version {version}, expected "
                                  f"{CHECKPOINT_VERSION}")
        if n != self.n:
            raise DofCountMismatch(f"checkpoint has {n} DOFs, mesh has {self.n}")
        off = struct.calcsize("<IQ")
        step_index, t = struct.unpack_from("<Qd", payload, off)
        off += struct.calcsize("<Qd")

        # parse the layout on the host (header fields only), upload the whole
        # payload in one H2D copy and cut the arrays out on the device
        segs = []

        def take(count, dtype=np.float64):
            nonlocal off
            segs.append((off, count, np.dtype(dtype)))
            off += count * np.dtype(dtype).itemsize
            return len(segs) - 1

        (fill,) = struct.unpack_from("<I", payload, off)
        off += 4
        us = [take(n) for _ in range(fill)]
        act = take(n)
        best = take(n)
        frozen = take(n, np.uint8)
        (nvols,) = struct.unpack_from("<I", payload, off)
        off += 4
        if nvols != len(self.volumes):
            raise CorruptFile(f"checkpoint has {nvols} volumes, config has "
                              f"{len(self.volumes)}")
        vol_states = []
        for vol in self.volumes:
            (ll,) = struct.unpack_from("<I", payload, off)
            off += 4
            label = bytes(payload[off: off + ll]).decode("utf-8")
            off += ll
            if label != vol.config.label:
                raise CorruptFile(f"checkpoint volume {label!r} does not match "
                                  f"{vol.config.label!r}")
            nv, nd, wf = struct.unpack_from("<IQI", payload, off)
            off += struct.calcsize("<IQI")
            if nv != vol.num_vars or nd != vol.dofs.size:
                raise DofCountMismatch(f"checkpoint volume {label!r} shape mismatch")
            vol_states.append([(take(nd * nv), nd, nv) for _ in range(wf)])
        if off > len(payload):
            raise CorruptFile("checkpoint payload truncated")
        import warnings

        if src is not None:
            dev = src[:off].to("cuda", non_blocking=src.is_pinned())
        else:
            with warnings.catch_warnings():      # read-only bytes: never written
                warnings.simplefilter("ignore", UserWarning)
                raw = torch.frombuffer(payload, dtype=torch.uint8, count=off)
            dev = raw.to("cuda")
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8}

        def seg(k):
            o, count, dt = segs[k]
            nb = count * dt.itemsize
            b = dev[o: o + nb]
            if o % dt.itemsize:
                b = b.clone()                     # re-align on the device
            return b.view(tdt[dt])

        # newest first -> slots head, head-1, ...
        self.head = 0
        for k, u in enumerate(us):
            self.u_ring[(-k) % RING_SLOTS, :n] = seg(u)
        self.u_fill = fill
        for vol, states in zip(self.volumes, vol_states):
            for k, (w, nd, nv) in enumerate(states):
                # the reference's AoS block, transposed to SoA on the device
                vol.w_ring[(-k) % RING_SLOTS, :, :nd] = seg(w).view(nd, nv).t()
            vol.w_fill = len(states)
        self.act_time.copy_(seg(act))
        self.best_slope.copy_(seg(best))
        self.frozen.copy_(seg(frozen).view(self.frozen.dtype))
        self.frozen_count.copy_(self.frozen.ne(0).sum().view(1))
        self.stopped_at = None
        self.step_index, self.time = int(step_index), float(t)
        self._log_base = self.step_index
        self.ws.status.zero_()


CHECKPOINT_MAGIC = b"MHEP"
CHECKPOINT_VERSION = 1


def save_checkpoint(solver, path):
    payload = solver.checkpoint_payload()
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(payload)
        fh.write(struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF))


def load_checkpoint(path):
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < len(CHECKPOINT_MAGIC) + 4 or not blob.startswith(CHECKPOINT_MAGIC):
        raise CorruptFile(f"{path} is not a checkpoint file")
    payload = blob[len(CHECKPOINT_MAGIC): -4]
    (stored,) = struct.unpack("<I", blob[-4:])
    if zlib.crc32(payload) & 0xFFFFFFFF != stored:
        raise CorruptFile(f"{path} failed its checksum")
    return payload


# ---------------------------------------------------------------------------
# Run loop (simulation.py:634-716)
# ---------------------------------------------------------------------------


@dataclass
class RunReport:
    activation_times: np.ndarray
    final_potential: np.ndarray
    timings: dict
    steps: int
    max_cg_iterations: int
    csv_path: str = None
    vtk_paths: tuple = ()
    solver: TissueSolver = None
    rows: list = None


def run(config, stop_when_fully_activated=False, resume_from=None, **solver_kw):
    """Execute a configured simulation to its final time on the device.

    Steps are enqueued back to back; the host synchronises only to record an
    output row (every `output.stride` steps, a 2+P-value read-back) or to
    test full activation.
    """
    import torch

    solver = TissueSolver(config, **solver_kw)
    if resume_from is not None:
        solver.restore(load_checkpoint(resume_from))
    n_steps = int(round(config.final_time / config.dt))
    out = getattr(config, "output", None) or OutputConfig()
    vtk_paths = []
    probes = [nearest_node(config.mesh, p) for p in out.probe_points]
    probe_idx = torch.tensor(probes, dtype=torch.int64, device="cuda") if probes else None
    n_rec = (n_steps - solver.step_index) // out.stride + 2
    pinned = torch.empty((n_rec, 2 + len(probes)), dtype=torch.float64, pin_memory=True)
    times = []
    row_steps = []
    # early stop on the device: the step that freezes the last node turns the
    # steps enqueued after it into no-ops; the host looks every CHECK steps
    solver.stop_when_full = bool(stop_when_fully_activated)
    CHECK = 64

    def record():
        with solver.timer.section("Other"):
            if out.enable_csv or not out.enable_field_output:
                solver.record_row(probe_idx, pinned[len(times)])   # async D2H
                times.append(solver.time)
                row_steps.append(solver.step_index)
            if out.enable_field_output:
                path = f"{out.field_stem}_{solver.step_index:06d}.vtk"
                write_vtk(path, config.mesh, {"transmembrane_potential": solver.potential})
                vtk_paths.append(path)

    if solver.step_index == 0:
        record()
    row_only = out.enable_csv or not out.enable_field_output
    while solver.step_index < n_steps:
        k = solver.step_index + 1
        if (k % out.stride == 0 or k == n_steps) and row_only and not out.enable_field_output:
            # the row is written by the step's own solve kernel
            with solver.timer.section("Other"):
                solver.enqueue_step(record=(probe_idx, pinned[len(times)]))
                times.append(solver.time)
                row_steps.append(solver.step_index)
        else:
            solver.enqueue_step()
            k = solver.step_index
            if k % out.stride == 0 or k == n_steps:
                record()
        if stop_when_fully_activated and (solver.step_index % CHECK == 0
                                          or out.enable_field_output):
            solver.sync()
            if solver.stopped_at is not None:
                break
    solver.sync()
    if solver.stopped_at is not None:
        # rows of the no-op steps after the stop were never written
        keep = [i for i, k in enumerate(row_steps) if k <= solver.step_index]
        times = [times[i] for i in keep]
        rows = [(t, *pinned[i].tolist()) for i, t in zip(keep, times)]
    else:
        rows = [(t, *pinned[i].tolist()) for i, t in enumerate(times)]
    with solver.timer.section("Other"):
        csv_path = None
        if out.enable_csv:
            write_csv(out.csv_path, rows, probe_count=len(probes))
            csv_path = out.csv_path
        act_cfg = getattr(config, "activation", None)
        if act_cfg is not None and act_cfg.enabled:
            write_vtk(act_cfg.path, config.mesh, {"activation_time": solver.activation_map})
            vtk_paths.append(act_cfg.path)
        ck = getattr(config, "checkpoint", None)
        if ck is not None and ck.enabled:
            save_checkpoint(solver, ck.path)
    return RunReport(
        activation_times=solver.activation_map,
        final_potential=solver.potential.copy(),
        timings=dict(solver.timer.totals),
        steps=solver.step_index,
        max_cg_iterations=solver.max_iterations_seen,
        csv_path=csv_path,
        vtk_paths=tuple(vtk_paths),
        solver=solver,
        rows=rows,
    )
