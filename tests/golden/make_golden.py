"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in the build container (the reference is importable only here):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_golden.py [name ...]

Every fixture is produced by the UNMODIFIED reference package
(`/root/reference/pkg/src/monodomain`) on inputs built by
`paper_2308_01651_b200.configs` with the reference's own types, so the GPU
path and the oracle are checked against the reference's numbers, not against
each other.  Nothing here runs on the GPU box.
"""

import hashlib
import struct
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def _ref():
    import monodomain  # noqa: F401

    from paper_2308_01651_b200 import configs

    return configs, configs.reference_namespace()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------


def ionic_kat():
    """advance_kernel / current_kernel / point_rates on seeded random states."""
    from monodomain.ionic import IonicModelSpec, ModelKind, model_module

    rng = np.random.default_rng(7)
    out = {}
    cases = {
        "ttp06": (ModelKind.TTP06, (-0.09, 0.045), (2e-5, 1e-5)),
        "bo": (ModelKind.BUENO_OROVIO, (-0.1, 1.5), (5e-5, 1e-3)),
        "apf": (ModelKind.ALIEV_PANFILOV, (-0.05, 1.2), (1e-4, 1e-3)),
    }
    for name, (kind, (ulo, uhi), dts) in cases.items():
        for ct_name in (["epi", "endo", "myo"] if kind is ModelKind.TTP06 else ["-"]):
            from monodomain.ionic import CellType

            ct = {"epi": CellType.EPICARDIUM, "endo": CellType.ENDOCARDIUM,
                  "myo": CellType.MYOCARDIUM}.get(ct_name)
            spec = IonicModelSpec(kind, cell_type=ct)
            mod = model_module(kind)
            P = mod.pack(spec.parameters, spec.cell_type)
            n = 512
            rest = spec.initial_state.w
            u = rng.uniform(ulo, uhi, n)
            scale = 1.0 + 0.05 * rng.standard_normal((n, rest.size))
            base = np.where(rest == 0.0, 0.05, rest)
            W_ext = base * scale
            W_bdf = base * (1.0 + 0.05 * rng.standard_normal((n, rest.size)))
            if kind is not ModelKind.ALIEV_PANFILOV:
                # some wild gates to exercise clamping
                ng = sum(mod.GATES)
                W_bdf[:16, :ng] = rng.uniform(-0.5, 1.5, (16, ng))
            tag = f"{name}_{ct_name}"
            out[f"{tag}_P"] = P
            out[f"{tag}_u"] = u
            out[f"{tag}_Wext"] = W_ext
            out[f"{tag}_Wbdf"] = W_bdf
            for alpha in (1.0, 1.5):
                for dt in dts:
                    W_out = np.empty_like(W_ext)
                    I_out = np.empty(n)
                    c = mod.advance_kernel(u, W_ext, W_bdf, alpha, dt, P, W_out, I_out)
                    key = f"{tag}_a{alpha}_dt{dt:g}"
                    out[f"{key}_Wout"] = W_out
                    out[f"{key}_Iout"] = I_out
                    out[f"{key}_clamped"] = np.array(c)
            I_cur = np.empty(n)
            mod.current_kernel(u, W_ext, P, I_cur)
            out[f"{tag}_current"] = I_cur
            rates_I = np.empty(8)
            rates_dw = np.empty((8, rest.size))
            for k in range(8):
                rates_I[k], rates_dw[k] = mod.point_rates(u[k], W_ext[k], P)
            out[f"{tag}_rates_I"] = rates_I
            out[f"{tag}_rates_dw"] = rates_dw
    # known-answer values pinned by the reference tests
    from monodomain.ionic import ion_current

    spec = IonicModelSpec(ModelKind.TTP06)
    out["kat_ttp06_rest_current"] = np.array(
        ion_current(spec, spec.initial_state.u, spec.initial_state.w))
    np.savez_compressed(OUT / "ionic_kat.npz", **out)


def pace0d():
    """pace_single_cell traces (0D splitting) for the three models."""
    from monodomain.ionic import IonicModelSpec, ModelKind, PacingProtocol0D, pace_single_cell

    out = {}
    apf_listing = PacingProtocol0D((0.0,), (4e-3,), (1.1628e3,), 0.8, 0.8, 2.5e-5)
    _, tr = pace_single_cell(IonicModelSpec(ModelKind.ALIEV_PANFILOV), apf_listing,
                             order=2, stride=40)
    out["apf_trace"] = tr
    bo = PacingProtocol0D((0.0,), (4e-3,), (1.1628e3,), 0.8, 0.4, 5e-5)
    for order in (1, 2, 3):
        _, tr = pace_single_cell(IonicModelSpec(ModelKind.BUENO_OROVIO), bo,
                                 order=order, stride=20)
        out[f"bo_trace_o{order}"] = tr
    ttp = PacingProtocol0D((0.0,), (2e-3,), (35.714,), 0.0, 0.05, 2.5e-5)
    for order in (1, 2):
        st, tr = pace_single_cell(IonicModelSpec(ModelKind.TTP06), ttp, order=order,
                                  stride=40)
        out[f"ttp_trace_o{order}"] = tr
    np.savez_compressed(OUT / "pace0d.npz", **out)


def operators():
    """Assembled M and K: full CSR for small meshes, hashes for cfg-0 size."""
    from monodomain.fem import ConductivitySet, FeSpace, assemble_mass, assemble_stiffness
    from monodomain.geometry import ElementKind, Mesh, SlabSpec, build_slab_mesh, slab_fiber_field

    out = {}
    meshes = {
        "unit_hex": (SlabSpec((1.0, 1.0, 1.0), 1.0, ElementKind.HEX8), (0, 0.0, 0.0)),
        "hex27": (SlabSpec((1e-3, 1e-3, 1e-3), 0.5e-3, ElementKind.HEX8), (0, 60.0, -60.0)),
        "tet_slab": (SlabSpec((2e-3, 3e-3, 4e-3), 0.5e-3, ElementKind.TET4), (2, 60.0, -60.0)),
        "hex_slab": (SlabSpec((2e-3, 3e-3, 4e-3), 0.5e-3, ElementKind.HEX8), (2, 60.0, -60.0)),
        "cfg0_hex": (SlabSpec((20e-3, 7e-3, 3e-3), 0.5e-3, ElementKind.HEX8), (2, 0.0, 0.0)),
        "cfg0_tet": (SlabSpec((20e-3, 7e-3, 3e-3), 0.5e-3, ElementKind.TET4), (2, 0.0, 0.0)),
    }
    for name, (spec, fib) in meshes.items():
        mesh = build_slab_mesh(spec)
        if name in ("tet_slab", "hex_slab"):
            mats = mesh.material_ids.copy()
            zc = mesh.nodes[mesh.elements].mean(axis=1)[:, 2]
            mats[zc > 2e-3] = 2
            mesh = Mesh(mesh.nodes, mesh.elements, mesh.element_kind, mats)
        fibers = slab_fiber_field(mesh, *fib)
        space = FeSpace(mesh)
        cs = ConductivitySet().add(1, 1.2e-4, 3e-5, 1.5e-5)
        if name in ("tet_slab", "hex_slab"):
            cs.add(2, 2e-4, 1e-5, 1e-5)
        K = assemble_stiffness(space, cs, fibers)
        M = assemble_mass(space)
        out[f"{name}_K_indptr_sha"] = np.array(sha(K.indptr.astype(np.int64)))
        out[f"{name}_K_indices_sha"] = np.array(sha(K.indices.astype(np.int32)))
        out[f"{name}_K_data_sha"] = np.array(sha(K.data))
        out[f"{name}_M_data_sha"] = np.array(sha(M.data))
        if name in ("tet_slab", "hex_slab"):
            M1 = assemble_mass(space, {1})
            out[f"{name}_M1_data_sha"] = np.array(sha(M1.data))
        if mesh.num_nodes <= 400:
            out[f"{name}_K_indptr"] = K.indptr.astype(np.int64)
            out[f"{name}_K_indices"] = K.indices.astype(np.int32)
            out[f"{name}_K_data"] = K.data
            out[f"{name}_M_data"] = M.data
    np.savez_compressed(OUT / "operators.npz", **out)


def cg_kat():
    """JacobiCg on the benchmark-sized system of tests/test_linalg.py:33-45."""
    from monodomain.fem import ConductivitySet, FeSpace, assemble_mass, assemble_stiffness
    from monodomain.geometry import ElementKind, SlabSpec, build_slab_mesh, slab_fiber_field
    from monodomain.linalg import JacobiCg

    mesh = build_slab_mesh(SlabSpec((3e-3, 7e-3, 20e-3), 0.5e-3, ElementKind.HEX8))
    space = FeSpace(mesh)
    fibers = slab_fiber_field(mesh, 0, 0.0, 0.0)
    K = assemble_stiffness(space, ConductivitySet().add(1, 0.95298e-4, 0.12576e-4,
                                                       0.12576e-4), fibers)
    A = ((1.5 / 5e-5) * assemble_mass(space) + K).tocsr()
    b = np.random.default_rng(1).standard_normal(space.num_dofs) * 1e-8
    x, it, rel = JacobiCg(A, 1e-10, 2000).solve(b)
    x12, it12, rel12 = JacobiCg(A, 1e-12, 2000).solve(b)
    x0 = np.random.default_rng(2).standard_normal(space.num_dofs) * 1e-9
    xw, itw, relw = JacobiCg(A, 1e-10, 2000).solve(b, initial_guess=x0)
    np.savez_compressed(OUT / "cg_kat.npz", b=b, x=x, iters=np.array(it),
                        relres=np.array(rel), x12=x12, iters12=np.array(it12),
                        x0=x0, xw=xw, itersw=np.array(itw),
                        A_data_sha=np.array(sha(A.data)))


def _drive(solver, steps, probes, snap_every=None, payload_at=()):
    """Step the reference solver, recording what the parity tests compare."""
    its = np.empty(steps, dtype=np.int32)
    pr = np.empty((steps, len(probes)))
    umin = np.empty(steps)
    umax = np.empty(steps)
    snaps, payloads = {}, {}
    t0 = time.perf_counter()
    for k in range(steps):
        u = solver.step()
        its[k] = solver.last_iterations
        pr[k] = u[probes]
        umin[k], umax[k] = u.min(), u.max()
        if snap_every and (k + 1) % snap_every == 0:
            snaps[k + 1] = u.copy()
        if (k + 1) in payload_at:
            payloads[k + 1] = np.frombuffer(solver.checkpoint_payload(), dtype=np.uint8).copy()
    wall = time.perf_counter() - t0
    return its, pr, umin, umax, snaps, payloads, wall


def tissue(name, build, steps, snap_every=None, payload_at=(), subsample=None, lean=False,
           act_steps=False):
    configs, ns = _ref()
    from monodomain.simulation import TissueSolver

    cfg = build(configs, ns)
    if cfg.mesh.element_kind.value == "Tet4" and cfg.mesh.nodes[:, 2].min() < -1e-3:
        # ventricle: apex, base ring points, mid-wall equator
        pts = [(0, 0, -45e-3), (0, 0, -55e-3), (30e-3, 0, 0), (0, 30e-3, 0),
               (-30e-3, 0, 0), (0, -30e-3, 0), (25e-3, 0, -20e-3), (0, 32e-3, -30e-3),
               (-27e-3, 0, -10e-3)]
    else:
        pts = configs.corner_probes() + [(10e-3, 3.5e-3, 1.5e-3)]
    probes = [ns.nearest_node(cfg.mesh, p) for p in pts]
    solver = TissueSolver(cfg)
    its, pr, umin, umax, snaps, payloads, wall = _drive(solver, steps, probes,
                                                        snap_every, payload_at)
    out = dict(iters=its, probes=np.asarray(probes), probe_u=pr, umin=umin, umax=umax,
               steps=np.array(steps), wall=np.array(wall),
               activation=solver.activation_map)
    out["frozen"] = solver.frozen.astype(np.uint8)
    if act_steps:
        # activation times as step numbers (t_{n+1} is accumulated dt: exact
        # after rounding); the parity bar is one dt, so this is lossless for it
        act = solver.activation_map
        out["activation"] = np.where(act < 0, -1, np.rint(act / cfg.dt)).astype(np.int32)
        out["act_steps"] = np.array(1)
    if not lean:               # lean: full-size fixtures drop the best-slope field
        out["best_slope"] = solver.best_slope
    u = solver.potential
    out["final_u_sha"] = np.array(sha(u))
    if subsample:
        out["final_u_sub"] = u[::subsample]
        out["subsample"] = np.array(subsample)
    else:
        out["final_u"] = u
        for v, vol in enumerate(solver.volumes):
            out[f"final_w{v}"] = vol.ring[0]
    for k, s in snaps.items():
        out[f"snap_{k}"] = s if not subsample else s[::subsample]
    for k, p in payloads.items():
        out[f"payload_{k}"] = p
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: {steps} steps in {wall:.1f} s, iters {its.min()}..{its.max()}")


def tissue_segmented(name, build, steps, seg=500, subsample=97, work="/tmp/golden_seg"):
    """Long full-size runs (config 3: 25,000 steps, hours of CPU): the unmodified
    reference stepped in segments of `seg` steps; after each segment the records so
    far and the reference's own checkpoint payload go to `work`, so an interrupted
    run resumes through `TissueSolver.restore` (bit-exact: the payload carries every
    history ring and the activation fields, reference simulation.py:518-607).
    Records: per-step CG iterations / probe potentials / u_min / u_max, snapshots
    every `seg` steps (every `subsample`-th node), activation map as step numbers."""
    configs, ns = _ref()
    from monodomain.simulation import TissueSolver

    cfg = build(configs, ns)
    pts = configs.corner_probes() + [(10e-3, 3.5e-3, 1.5e-3)]
    probes = [ns.nearest_node(cfg.mesh, p) for p in pts]
    solver = TissueSolver(cfg)
    wdir = Path(work) / name
    wdir.mkdir(parents=True, exist_ok=True)
    its = np.zeros(steps, dtype=np.int16)
    pr = np.zeros((steps, len(probes)))
    umin = np.zeros(steps)
    umax = np.zeros(steps)
    snaps = {}
    done = 0
    state = wdir / "state.npz"
    if state.exists():
        z = np.load(state)
        done = int(z["done"])
        its[:done], pr[:done] = z["iters"][:done], z["probe_u"][:done]
        umin[:done], umax[:done] = z["umin"][:done], z["umax"][:done]
        snaps = {int(k[5:]): z[k] for k in z.files if k.startswith("snap_")}
        solver.restore((wdir / "payload.bin").read_bytes())
        assert solver.step_index == done
        print(f"{name}: resumed at step {done}", flush=True)
    t0 = time.perf_counter()
    while done < steps:
        for k in range(done, min(done + seg, steps)):
            u = solver.step()
            its[k] = solver.last_iterations
            pr[k] = u[probes]
            umin[k], umax[k] = u.min(), u.max()
        done = k + 1
        snaps[done] = u[::subsample].copy()
        (wdir / "payload.tmp").write_bytes(solver.checkpoint_payload())
        np.savez(wdir / "state.tmp.npz", done=np.array(done), iters=its, probe_u=pr,
                 umin=umin, umax=umax, **{f"snap_{s}": v for s, v in snaps.items()})
        (wdir / "payload.tmp").rename(wdir / "payload.bin")
        (wdir / "state.tmp.npz").rename(state)
        _write_segmented(name, cfg, solver, done, its, pr, umin, umax, snaps, probes,
                         subsample)
        print(f"{name}: step {done}/{steps}, {time.perf_counter() - t0:.0f} s, "
              f"iters {its[done - seg:done].min()}..{its[done - seg:done].max()}, "
              f"frozen {int(solver.frozen.sum())}", flush=True)


def _write_segmented(name, cfg, solver, done, its, pr, umin, umax, snaps, probes, subsample):
    act = solver.activation_map
    u = solver.potential
    out = dict(iters=its[:done], probes=np.asarray(probes), probe_u=pr[:done],
               umin=umin[:done], umax=umax[:done], steps=np.array(done),
               activation=np.where(act < 0, -1, np.rint(act / cfg.dt)).astype(np.int32),
               act_steps=np.array(1), frozen=solver.frozen.astype(np.uint8),
               final_u_sha=np.array(sha(u)), final_u_sub=u[::subsample],
               subsample=np.array(subsample))
    for s, v in snaps.items():
        out[f"snap_{s}"] = v
    tmp = OUT / f"{name}.tmp.npz"
    np.savez_compressed(tmp, **out)
    tmp.rename(OUT / f"{name}.npz")


def cfg1_subset():
    """Config 1 parity subset: seeded TTP06 cells, 0D splitting, BDF1/BDF2."""
    from monodomain.ionic import IonicModelSpec, ModelKind, model_module
    from monodomain.timestepping import bdf_coefficients

    from paper_2308_01651_b200 import configs

    n, steps, dt = 512, 2000, 1e-5
    u0, W0 = configs.config1_initial(n)
    spec = IonicModelSpec(ModelKind.TTP06)
    mod = model_module(ModelKind.TTP06)
    P = mod.pack(spec.parameters, spec.cell_type)
    n_stim = n // 100
    out = {"u0": u0, "W0": W0, "n_stim": np.array(n_stim)}
    for order in (1, 2):
        uh = [u0.copy()]
        wh = [W0.copy()]
        peak = u0.copy()
        clamps = 0
        W_out = np.empty_like(W0)
        I_out = np.empty(n)
        for k in range(steps):
            s = bdf_coefficients(min(k + 1, order))
            ub = s.history_weights[0] * uh[0]
            ue = s.ext_weights[0] * uh[0]
            wb = s.history_weights[0] * wh[0]
            we = s.ext_weights[0] * wh[0]
            for q in range(1, len(s.history_weights)):
                ub = ub + s.history_weights[q] * uh[q]
                ue = ue + s.ext_weights[q] * uh[q]
                wb = wb + s.history_weights[q] * wh[q]
                we = we + s.ext_weights[q] * wh[q]
            clamps += mod.advance_kernel(ue, we, wb, s.alpha, dt, P, W_out, I_out)
            t_next = (k + 1) * dt
            iapp = np.zeros(n)
            if t_next < 1e-3:
                iapp[:n_stim] = 52.0
            un = (ub + dt * (iapp - I_out)) / s.alpha
            uh = [un] + uh[:2]
            wh = [W_out.copy()] + wh[:2]
            peak = np.maximum(peak, un)
        out[f"o{order}_u"] = uh[0]
        out[f"o{order}_W"] = wh[0]
        out[f"o{order}_peak"] = peak
        out[f"o{order}_clamps"] = np.array(clamps)
    np.savez_compressed(OUT / "cfg1_subset.npz", **out)


# ---------------------------------------------------------------------------
# Rush-Larsen mode (BASELINE.json north_star / config 1; not a reference scheme,
# SPEC.md:201).  The fixtures below replace ONLY the integrator: the targets,
# currents and rates are the reference's own jitted functions
# (ten_tusscher._gate_targets/_currents/_conc_rates/_total,
# bueno_orovio._gate_pieces/_current, aliev_panfilov.advance_kernel), and the
# tissue/0D drivers are the reference's TissueSolver / pace_single_cell at BDF
# order 1 (where W_ext = W_bdf = W_n, alpha = 1) with <model>.advance_kernel
# swapped for that integrator.
# ---------------------------------------------------------------------------


def _rl_kernels():
    from numba import njit, prange

    from monodomain.ionic import aliev_panfilov as ap
    from monodomain.ionic import bueno_orovio as bo
    from monodomain.ionic import ten_tusscher as tt

    tt_targets, tt_currents, tt_conc, tt_total = (tt._gate_targets, tt._currents,
                                                  tt._conc_rates, tt._total)
    bo_pieces, bo_current = bo._gate_pieces, bo._current

    @njit(parallel=True)
    def ttp_rl(u, W_n, dt, P, W_out, I_out):
        dt_ms = dt * 1.0e3
        clamped = 0
        for i in prange(u.shape[0]):
            v = u[i] * 1.0e3
            w = W_n[i]
            targets = tt_targets(v, w[14], P[49])
            nclamp = 0
            for g in range(12):
                inf = targets[2 * g]
                gval = inf + (w[g] - inf) * np.exp(-dt_ms / targets[2 * g + 1])
                if gval < 0.0:
                    gval = 0.0
                    nclamp += 1
                elif gval > 1.0:
                    gval = 1.0
                    nclamp += 1
                W_out[i, g] = gval
            rates = tt_conc(w, tt_currents(v, w, P), P)
            for c in range(6):
                W_out[i, 12 + c] = w[12 + c] + dt_ms * rates[c]
            I_out[i] = tt_total(tt_currents(v, W_out[i], P))
            clamped += nclamp
        return clamped

    @njit(parallel=True)
    def bo_rl(u, W_n, dt, P, W_out, I_out):
        dt_ms = dt * 1.0e3
        clamped = 0
        for i in prange(u.shape[0]):
            pieces = bo_pieces(u[i], P)
            nclamp = 0
            for g in range(3):
                src, rate = pieces[2 * g], pieces[2 * g + 1]
                inf = src / rate
                gval = inf + (W_n[i, g] - inf) * np.exp(-dt_ms * rate)
                if gval < 0.0:
                    gval = 0.0
                    nclamp += 1
                elif gval > 1.0:
                    gval = 1.0
                    nclamp += 1
                W_out[i, g] = gval
            I_out[i] = bo_current(u[i], W_out[i, 0], W_out[i, 1], W_out[i, 2], P)
            clamped += nclamp
        return clamped

    def apf_rl(u, W_n, dt, P, W_out, I_out):
        return ap.advance_kernel(u, W_n, W_n, 1.0, dt, P, W_out, I_out)

    return {"ttp06": (tt, ttp_rl), "bo": (bo, bo_rl), "apf": (ap, apf_rl)}


class _RlPatch:
    """Swap <module>.advance_kernel for the Rush-Larsen integrator (order-1 callers
    pass W_ext = W_bdf = W_n and alpha = 1, checked)."""

    def __init__(self, mod, rl):
        self.mod, self.rl = mod, rl

    def __enter__(self):
        self.orig = self.mod.advance_kernel
        rl = self.rl

        def patched(u_ext, W_ext, W_bdf, alpha, dt, P, W_out, I_out):
            assert alpha == 1.0 and np.array_equal(W_ext, W_bdf)
            return rl(np.ascontiguousarray(u_ext), np.ascontiguousarray(W_bdf), dt, P,
                      W_out, I_out)

        self.mod.advance_kernel = patched
        return self

    def __exit__(self, *exc):
        self.mod.advance_kernel = self.orig
        return False


def rl_kat():
    """RL step on the ionic_kat inputs; cfg-1 subset in RL mode; 0D traces; two
    small tissue runs (reference TissueSolver, BDF1, RL ionic update)."""
    import dataclasses

    from monodomain.ionic import (CellType, IonicModelSpec, ModelKind, PacingProtocol0D,
                                  model_module, pace_single_cell)
    from monodomain.simulation import TissueSolver

    from paper_2308_01651_b200 import configs

    K = _rl_kernels()
    kat = np.load(OUT / "ionic_kat.npz")
    out = {}
    for tag, name in (("ttp06_epi", "ttp06"), ("ttp06_endo", "ttp06"), ("ttp06_myo", "ttp06"),
                      ("bo_-", "bo"), ("apf_-", "apf")):
        P, u, Wn = kat[f"{tag}_P"], kat[f"{tag}_u"], kat[f"{tag}_Wext"].copy()
        if name != "apf":
            ng = 12 if name == "ttp06" else 3
            Wn[:16, :ng] = kat[f"{tag}_Wbdf"][:16, :ng]      # out-of-range gates: clamps
        out[f"{tag}_Wn"] = Wn
        for dt in ((2e-5, 1e-5) if name == "ttp06" else (5e-5, 1e-3)):
            W_out, I_out = np.empty_like(Wn), np.empty(u.size)
            c = K[name][1](u, Wn, dt, P, W_out, I_out)
            out[f"{tag}_dt{dt:g}_Wout"] = W_out
            out[f"{tag}_dt{dt:g}_Iout"] = I_out
            out[f"{tag}_dt{dt:g}_clamped"] = np.array(c)
    # config-1 subset, RL mode: u+ = u_n + dt (I_app - I_ion(u_n, W+))
    n, steps, dt = 512, 2000, 1e-5
    u, W = configs.config1_initial(n)
    spec = IonicModelSpec(ModelKind.TTP06)
    P = model_module(ModelKind.TTP06).pack(spec.parameters, spec.cell_type)
    n_stim = n // 100
    peak, clamps = u.copy(), 0
    W_out, I_out = np.empty_like(W), np.empty(n)
    for k in range(steps):
        clamps += K["ttp06"][1](u, W, dt, P, W_out, I_out)
        iapp = np.zeros(n)
        if (k + 1) * dt < 1e-3:
            iapp[:n_stim] = 52.0
        u = (u + dt * (iapp - I_out)) / 1.0
        W = W_out.copy()
        peak = np.maximum(peak, u)
    out.update(cfg1_u=u, cfg1_W=W, cfg1_peak=peak, cfg1_clamps=np.array(clamps),
               cfg1_n_stim=np.array(n_stim))
    # 0D traces through the reference's pace_single_cell at order 1
    ttp = PacingProtocol0D((0.0,), (2e-3,), (35.714,), 0.0, 0.05, 2.5e-5)
    with _RlPatch(*K["ttp06"]):
        _, tr = pace_single_cell(IonicModelSpec(ModelKind.TTP06), ttp, order=1, stride=40)
    out["ttp_trace"] = tr
    bop = PacingProtocol0D((0.0,), (4e-3,), (1.1628e3,), 0.8, 0.4, 5e-5)
    with _RlPatch(*K["bo"]):
        _, tr = pace_single_cell(IonicModelSpec(ModelKind.BUENO_OROVIO), bop, order=1,
                                 stride=20)
    out["bo_trace"] = tr
    # tissue: the reference solver at BDF1 with the RL ionic update
    ns = configs.reference_namespace()
    for key, name, cfg, steps in (
            ("tissue_bo", "bo", configs.config0(ns), 400),
            ("tissue_ttp", "ttp06", configs.config2(ns, h=0.5e-3), 1000)):
        cfg = dataclasses.replace(cfg, bdf_order=1)
        pts = configs.corner_probes() + [(10e-3, 3.5e-3, 1.5e-3)]
        probes = [ns.nearest_node(cfg.mesh, p) for p in pts]
        with _RlPatch(*K[name]):
            solver = TissueSolver(cfg)
            its, pr, umin, umax, _, _, wall = _drive(solver, steps, probes)
        out[f"{key}_iters"] = its
        out[f"{key}_probes"] = np.asarray(probes)
        out[f"{key}_probe_u"] = pr
        out[f"{key}_final_u"] = solver.potential
        out[f"{key}_final_w"] = solver.volumes[0].ring[0]
        out[f"{key}_activation"] = solver.activation_map
        print(f"rl {key}: {steps} steps in {wall:.1f} s, iters {its.min()}..{its.max()}")
    np.savez_compressed(OUT / "rl_kat.npz", **out)


JOBS = {
    "ionic_kat": ionic_kat,
    "pace0d": pace0d,
    "operators": operators,
    "cg_kat": cg_kat,
    "cfg1_subset": cfg1_subset,
    "rl_kat": rl_kat,
    "tissue_cfg0": lambda: tissue("tissue_cfg0", lambda c, ns: c.config0(ns), 800,
                                  snap_every=100, payload_at=(400,)),
    "tissue_ttp_h05": lambda: tissue("tissue_ttp_h05",
                                     lambda c, ns: c.config2(ns, h=0.5e-3), 2000,
                                     snap_every=250, payload_at=(1000,)),
    "tissue_tet": lambda: tissue("tissue_tet",
                                 lambda c, ns: c.config0(ns, kind="Tet4"), 400,
                                 snap_every=100),
    "tissue_cfg3_h05": lambda: tissue("tissue_cfg3_h05",
                                      lambda c, ns: c.config3(ns, h=0.5e-3), 25000,
                                      snap_every=2500, payload_at=(15000,)),
    "tissue_cfg4_small": lambda: tissue(
        "tissue_cfg4_small",
        lambda c, ns: __import__("paper_2308_01651_b200.ventricle", fromlist=["config4"])
        .config4(ns, n_xi=4, n_th=24, n_ph=64, final_time=30e-3), 1500,
        snap_every=500),
    "tissue_cfg2_head": lambda: tissue("tissue_cfg2_head", lambda c, ns: c.config2(ns),
                                       40, snap_every=20, subsample=97),
    # config 2 at full size through the first 10 ms of propagation: iteration
    # counts, probe traces and the full activation map of ~1/4 of the slab
    "tissue_cfg2_500": lambda: tissue("tissue_cfg2_500", lambda c, ns: c.config2(ns),
                                      500, subsample=97, lean=True),
    # round 2: full-length parity at the stated sizes (VERDICT r1 "next" #1)
    "tissue_cfg2_full": lambda: tissue("tissue_cfg2_full", lambda c, ns: c.config2(ns),
                                       5000, snap_every=500, subsample=97, lean=True,
                                       act_steps=True),
    "tissue_cfg4_100k": lambda: tissue(
        "tissue_cfg4_100k",
        lambda c, ns: __import__("paper_2308_01651_b200.ventricle", fromlist=["config4"])
        .config4(ns, *__import__("paper_2308_01651_b200.ventricle",
                                 fromlist=["size_for_nodes"]).size_for_nodes(100_000),
                 final_time=60e-3), 3000, snap_every=250, subsample=7, lean=True,
        act_steps=True),
    # resumable: `python make_golden.py tissue_cfg3_full` again continues from the
    # last finished segment; the fixture on disk always holds the steps done so far
    "tissue_cfg3_full": lambda: tissue_segmented("tissue_cfg3_full",
                                                 lambda c, ns: c.config3(ns), 25000),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(JOBS)
    for name in names:
        t = time.perf_counter()
        JOBS[name]()
        print(f"[{name}] {time.perf_counter() - t:.1f} s", flush=True)
