"""CUDA tissue path vs the reference (golden fixtures) and the CPU oracle.

Parity bar (BASELINE.json north_star): fp64 potential traces within relative
L2 1e-6, activation times within one dt, CG iteration counts within +-1 per
step.  Operators are bit-identical to the reference (hash-pinned).
"""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------

MESHES = {
    "unit_hex": ((1.0, 1.0, 1.0), 1.0, "Hex8", (0, 0.0, 0.0)),
    "hex27": ((1e-3, 1e-3, 1e-3), 0.5e-3, "Hex8", (0, 60.0, -60.0)),
    "tet_slab": ((2e-3, 3e-3, 4e-3), 0.5e-3, "Tet4", (2, 60.0, -60.0)),
    "hex_slab": ((2e-3, 3e-3, 4e-3), 0.5e-3, "Hex8", (2, 60.0, -60.0)),
    "cfg0_hex": ((20e-3, 7e-3, 3e-3), 0.5e-3, "Hex8", (2, 0.0, 0.0)),
    "cfg0_tet": ((20e-3, 7e-3, 3e-3), 0.5e-3, "Tet4", (2, 0.0, 0.0)),
}


def _mesh(name):
    from paper_2308_01651_b200.geometry import ElementKind, SlabSpec, build_slab_mesh, slab_fiber_field

    ext, h, kind, fib = MESHES[name]
    mesh = build_slab_mesh(SlabSpec(ext, h, ElementKind(kind)))
    two = name in ("tet_slab", "hex_slab")
    if two:
        mats = mesh.material_ids.copy()
        mats[mesh.nodes[mesh.elements].mean(axis=1)[:, 2] > 2e-3] = 2
        mesh = mesh.with_materials(mats)
    return mesh, slab_fiber_field(mesh, *fib), two


@pytest.mark.parametrize("name", list(MESHES))
def test_device_assembly_bit_identical(golden, name):
    from paper_2308_01651_b200.fem import ConductivitySet, FeSpace, assemble_mass, assemble_stiffness

    g = golden("operators")
    mesh, fibers, two = _mesh(name)
    space = FeSpace(mesh)
    cs = ConductivitySet().add(1, 1.2e-4, 3e-5, 1.5e-5)
    if two:
        cs.add(2, 2e-4, 1e-5, 1e-5)
    K = assemble_stiffness(space, cs, fibers)
    M = assemble_mass(space)
    assert _sha(K.indptr.astype(np.int64)) == str(g[f"{name}_K_indptr_sha"])
    assert _sha(K.indices.astype(np.int32)) == str(g[f"{name}_K_indices_sha"])
    assert _sha(K.data) == str(g[f"{name}_K_data_sha"])
    assert _sha(M.data) == str(g[f"{name}_M_data_sha"])
    if two:
        assert _sha(assemble_mass(space, {1}).data) == str(g[f"{name}_M1_data_sha"])
    if f"{name}_K_data" in g:
        np.testing.assert_array_equal(K.data, g[f"{name}_K_data"])


def test_unit_hex_closed_forms():
    """tests/test_fem.py:71-89: M_ii = 1/27, K_ii = 1/3, K diagonals -1/12."""
    from paper_2308_01651_b200.fem import ConductivitySet, FeSpace, assemble_mass, assemble_stiffness

    mesh, fibers, _ = _mesh("unit_hex")
    space = FeSpace(mesh)
    M = assemble_mass(space).toarray()
    K = assemble_stiffness(space, ConductivitySet().add(1, 1.0, 1.0, 1.0), fibers).toarray()
    np.testing.assert_allclose(np.diag(M), 1.0 / 27.0, rtol=1e-14)
    np.testing.assert_allclose(np.diag(K), 1.0 / 3.0, rtol=1e-14)
    np.testing.assert_allclose(K.sum(axis=1), 0.0, atol=1e-15)
    assert K[0, 6] == pytest.approx(-1.0 / 12.0, rel=1e-14)


def test_csr_matvec_bitwise_vs_oracle():
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200.fem import ConductivitySet, FeSpace, assemble_stiffness
    from paper_2308_01651_b200.linalg import csr_matvec

    mesh, fibers, _ = _mesh("cfg0_tet")
    K = assemble_stiffness(FeSpace(mesh), ConductivitySet().add(1, 1e-4, 2e-5, 1e-5), fibers)
    x = np.random.default_rng(3).standard_normal(K.shape[0])
    y = np.empty(K.shape[0])
    csr_matvec(K.indptr, K.indices, K.data, x, y)
    np.testing.assert_array_equal(y, O.Csr.from_scipy(K).matvec(x))


def test_jacobi_cg_known_systems(golden):
    import scipy.sparse as sp

    from paper_2308_01651_b200.errors import SolverDivergence
    from paper_2308_01651_b200.fem import ConductivitySet, FeSpace, assemble_mass, assemble_stiffness
    from paper_2308_01651_b200.geometry import ElementKind, SlabSpec, build_slab_mesh, slab_fiber_field
    from paper_2308_01651_b200.linalg import JacobiCg, solve_cg

    x, it, _ = solve_cg(sp.identity(5, format="csr"), np.array([1.0, -2, 3, 0.5, 0]))
    assert np.allclose(x, [1, -2, 3, 0.5, 0]) and it <= 1
    A2 = sp.csr_matrix(np.array([[4.0, 1.0], [1.0, 3.0]]))
    x, _, _ = solve_cg(A2, np.array([1.0, 2.0]), tolerance=1e-14)
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], atol=1e-13)
    x, it, _ = solve_cg(A2, np.zeros(2))
    assert (x == 0).all() and it == 0

    g = golden("cg_kat")
    mesh = build_slab_mesh(SlabSpec((3e-3, 7e-3, 20e-3), 0.5e-3, ElementKind.HEX8))
    space = FeSpace(mesh)
    K = assemble_stiffness(space, ConductivitySet().add(1, 0.95298e-4, 0.12576e-4,
                                                       0.12576e-4),
                           slab_fiber_field(mesh, 0, 0.0, 0.0))
    A = ((1.5 / 5e-5) * assemble_mass(space) + K).tocsr()
    assert _sha(A.data) == str(g["A_data_sha"])
    solver = JacobiCg(A, 1e-10, 2000)
    x, it, rel = solver.solve(g["b"])
    assert abs(it - int(g["iters"])) <= 1
    assert _rel(x, g["x"]) < 1e-9
    assert np.linalg.norm(g["b"] - A @ x) <= 1e-10 * np.linalg.norm(g["b"])
    _, it0, _ = solver.solve(g["b"], initial_guess=g["x"])
    assert it0 == 0
    xw, itw, _ = solver.solve(g["b"], initial_guess=g["x0"])
    assert abs(itw - int(g["itersw"])) <= 1 and _rel(xw, g["xw"]) < 1e-9
    x1, i1, r1 = JacobiCg(A, 1e-10, 2000).solve(g["b"])
    x2, i2, r2 = JacobiCg(A, 1e-10, 2000).solve(g["b"])
    assert i1 == i2 and r1 == r2 and np.array_equal(x1, x2)   # deterministic
    with pytest.raises(SolverDivergence) as err:
        solve_cg(A, g["b"], tolerance=1e-15, max_iterations=2)
    assert err.value.iterations == 2
    with pytest.raises(ValueError):
        JacobiCg(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 2.0]])))


def test_stencil_operator_matches_csr(ns):
    """Class-table stencil apply vs the bit-exact CSR operator: the class rows
    are one representative node's exact row, so they differ from a node's own
    row by the reference's coordinate round-off only (<= 1e-13 relative)."""
    import torch

    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import _native as N, configs
    from paper_2308_01651_b200.simulation import TissueSolver

    for cfg in (configs.config0(ns), configs.config3(ns, h=0.5e-3)):
        st = TissueSolver(cfg, operator="stencil")
        cs = TissueSolver(cfg, operator="csr")
        sl = TissueSolver(cfg, operator="sell")
        assert st.op.kind == N.OP_STENCIL27 and cs.op.kind == N.OP_CSR
        assert sl.op.kind == N.OP_SELL
        x = torch.from_numpy(np.random.default_rng(5).standard_normal(st.n)).cuda()
        for order in st.op.a_tables:
            ys = []
            for s in (st, cs):
                a = N.CgArgs()
                a.op = s.op.operator()
                a.a_val = N.ptr(s.op.a_tables[order])
                y = torch.empty_like(x)
                N.check(N.lib().mdx_spmv(N.C.byref(a), N.ptr(x), N.ptr(y),
                                         N.stream_handle()))
                ys.append(y.cpu().numpy())
            absx = torch.abs(x)
            scale = []
            for s in (cs,):
                a = N.CgArgs()
                a.op = s.op.operator()
                absA = torch.abs(s.op.a_tables[order])
                a.a_val = N.ptr(absA)
                y = torch.empty_like(x)
                N.check(N.lib().mdx_spmv(N.C.byref(a), N.ptr(absx), N.ptr(y),
                                         N.stream_handle()))
                scale = y.cpu().numpy()
            assert (np.abs(ys[0] - ys[1]) <= 1e-13 * scale).all()
        assert st.op.max_rel_dev < 1e-13
        assert st.op.ncls <= 200
        orc = O.OracleTissue(cfg)
        orc._system(1.5)
        np.testing.assert_array_equal(orc.A.matvec(x.cpu().numpy()), ys[1])  # CSR: bitwise
        a = N.CgArgs()
        a.op = sl.op.operator()
        a.a_val = N.ptr(sl.op.a_tables[1.5 and 2])
        y = torch.empty_like(x)
        N.check(N.lib().mdx_spmv(N.C.byref(a), N.ptr(x), N.ptr(y), N.stream_handle()))
        np.testing.assert_array_equal(orc.A.matvec(x.cpu().numpy()), y.cpu().numpy())


# ---------------------------------------------------------------------------
# tissue runs vs reference goldens
# ---------------------------------------------------------------------------


def _run_against(g, cfg, steps, operator="auto"):
    from paper_2308_01651_b200.simulation import TissueSolver

    s = TissueSolver(cfg, operator=operator)
    probes = g["probes"]
    pu = np.empty((steps, probes.size))
    for k in range(steps):
        u = s.step()
        pu[k] = u[probes]
    return s, pu


def _check(s, pu, g, dt, steps, trace_tol=1e-6):
    its = s.iterations_log()
    ref_its = g["iters"][:steps]
    assert np.abs(its - ref_its).max() <= 1, np.flatnonzero(its != ref_its)
    rel = _rel(pu, g["probe_u"][:steps])
    assert rel < trace_tol, rel
    if steps != int(g["steps"]):
        return its, rel
    act, ref = s.activation_map, g["activation"]
    both = (act >= 0) & (ref >= 0)
    assert np.array_equal(act >= 0, ref >= 0)
    assert np.abs(act[both] - ref[both]).max() <= dt * (1 + 1e-9)
    return its, rel


def test_cfg0_bo_full_run(golden, ns):
    from paper_2308_01651_b200 import configs

    g = golden("tissue_cfg0")
    s, pu = _run_against(g, configs.config0(ns), 800)
    its, rel = _check(s, pu, g, 5e-5, 800)
    assert rel < 1e-9               # reduction-order noise only
    assert (its == g["iters"]).mean() > 0.99
    assert _rel(s.potential, g["final_u"]) < 1e-9
    np.testing.assert_allclose(s.volume_state(0), g["final_w0"], rtol=1e-8, atol=1e-10)


def test_cfg0_csr_path_matches(golden, ns):
    from paper_2308_01651_b200 import configs

    g = golden("tissue_cfg0")
    s, pu = _run_against(g, configs.config0(ns), 300, operator="csr")
    _check(s, pu, g, 5e-5, 300)


@pytest.mark.parametrize("operator", ["auto", "sell"])
def test_tet_mesh_run(golden, ns, operator):
    from paper_2308_01651_b200 import configs

    g = golden("tissue_tet")
    s, pu = _run_against(g, configs.config0(ns, kind="Tet4"), 400, operator=operator)
    assert s.op.kind == {"auto": 4, "sell": 3}[operator]
    _check(s, pu, g, 5e-5, 400)


def test_ttp06_slab(golden, ns):
    from paper_2308_01651_b200 import configs

    g = golden("tissue_ttp_h05")
    s, pu = _run_against(g, configs.config2(ns, h=0.5e-3), 2000)
    _check(s, pu, g, 2e-5, 2000)
    assert _rel(s.potential, g["final_u"]) < 1e-8


def test_cfg3_scar_full_500ms(golden, ns):
    """Three volumes (duplicated interface states), two stimuli, 25,000 steps."""
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    g = golden("tissue_cfg3_h05")
    steps = int(g["steps"])
    s = TissueSolver(configs.config3(ns, h=0.5e-3))
    probes = g["probes"]
    pu = np.empty((steps, probes.size))
    chunk = 500
    done = 0
    while done < steps:
        m = min(chunk, steps - done)
        for _ in range(m):
            s.enqueue_step()
        s.sync()
        done += m
        pu[done - 1] = s.potential[probes]
    its = s.iterations_log()
    assert np.abs(its - g["iters"]).max() <= 1
    ref = g["probe_u"][chunk - 1::chunk]
    assert _rel(pu[chunk - 1::chunk], ref) < 1e-6
    assert _rel(s.potential, g["final_u"]) < 1e-6
    act, ra = s.activation_map, g["activation"]
    both = (act >= 0) & (ra >= 0)
    assert np.array_equal(act >= 0, ra >= 0)
    assert np.abs(act[both] - ra[both]).max() <= 2e-5 * (1 + 1e-9)


def test_cfg2_full_size_head(golden, ns):
    """Config 2 at full size (442,401 nodes): first 40 steps vs the reference."""
    from paper_2308_01651_b200 import configs

    g = golden("tissue_cfg2_head")
    s, pu = _run_against(g, configs.config2(ns), 40)
    its = s.iterations_log()
    assert np.abs(its - g["iters"]).max() <= 1
    assert _rel(pu, g["probe_u"]) < 1e-9
    sub = int(g["subsample"])
    assert _rel(s.potential[::sub], g["final_u_sub"]) < 1e-9
    assert s.op.ncls == 27          # uniform slab: interior + 26 boundary classes


def test_cfg2_full_size_500_steps(golden, ns):
    """Config 2 at full size (442,401 nodes) through 10 ms of propagation (500
    steps) against the reference: CG iterations within +-1, probe traces, the
    set of activated (threshold-crossed) nodes and their activation times
    within one time step."""
    from paper_2308_01651_b200 import configs

    g = golden("tissue_cfg2_500")
    dt = 2e-5
    s, pu = _run_against(g, configs.config2(ns), 500)
    its = s.iterations_log()
    assert np.abs(its - g["iters"]).max() <= 1
    assert (its == g["iters"]).mean() > 0.95
    assert _rel(pu, g["probe_u"]) < 1e-6          # BASELINE bar (measured ~1e-9)
    sub = int(g["subsample"])
    assert _rel(s.potential[::sub], g["final_u_sub"]) < 1e-6
    fz, rfz = s.frozen.cpu().numpy().astype(bool), g["frozen"].astype(bool)
    assert rfz.sum() > 10000                       # the front has swept a good part
    # nodes crossing the threshold at the very last steps may differ by one step
    assert (fz != rfz).sum() <= 1e-3 * rfz.sum()
    both = fz & rfz
    act, ref = s.activation_map, g["activation"]
    assert np.abs(act[both] - ref[both]).max() <= dt * (1 + 1e-9)


def _run_long(g, cfg, steps, operator="auto"):
    """Enqueue `steps` steps; the solve writes each step's probe row on the
    device (no per-step host sync); subsampled snapshots at the golden's
    stride.  Returns (solver, probe trace, {step: snapshot})."""
    import torch

    from paper_2308_01651_b200.simulation import TissueSolver

    s = TissueSolver(cfg, operator=operator)
    probes = torch.from_numpy(g["probes"].astype(np.int64)).cuda()
    rows = torch.zeros((steps, 2 + probes.numel()), dtype=torch.float64, device="cuda")
    sub = int(g["subsample"])
    snap_at = sorted(int(k[5:]) for k in g if k.startswith("snap_"))
    snaps = {}
    for k in range(steps):
        s.enqueue_step(record=(probes, rows[k]))
        if (k + 1) in snap_at:
            snaps[k + 1] = s.potential_device[::sub].clone()
        if (k + 1) % 1000 == 0:
            s.sync()
    s.sync()
    return s, rows[:, 2:].cpu().numpy(), {k: v.cpu().numpy() for k, v in snaps.items()}


def _check_long(s, pu, snaps, g, steps, dt):
    """The north_star parity bar on a whole run: CG iterations within +-1 on
    every step, probe traces and every snapshot within relative L2 1e-6, the
    same activated set except nodes crossing in the final two steps, and
    activation times within one dt (goldens store them as step numbers)."""
    its = s.iterations_log()
    ref_its = g["iters"][:steps]
    assert np.abs(its - ref_its).max() <= 1, np.flatnonzero(np.abs(its - ref_its) > 1)[:10]
    assert _rel(pu, g["probe_u"][:steps]) < 1e-6
    for k, snap in snaps.items():
        assert _rel(snap, g[f"snap_{k}"]) < 1e-6, k
    sub = int(g["subsample"])
    assert _rel(s.potential[::sub], g["final_u_sub"]) < 1e-6
    act = s.activation_map
    ours = np.where(act < 0, -1, np.rint(act / dt)).astype(np.int64)
    ref = g["activation"].astype(np.int64)
    on, ron = ours >= 0, ref >= 0
    late = np.where(on, ours, ref) >= steps - 2
    assert ((on != ron) & ~late).sum() == 0
    both = on & ron
    assert np.abs(ours[both] - ref[both]).max() <= 1
    return its


def test_cfg2_full_run_5000_steps(golden, ns):
    """Config 2 at its stated size AND length (442,401 nodes, 5,000 steps =
    100 ms: propagation, plateau, repolarisation) against the reference."""
    from paper_2308_01651_b200 import configs

    g = golden("tissue_cfg2_full")
    s, pu, snaps = _run_long(g, configs.config2(ns), 5000)
    its = _check_long(s, pu, snaps, g, 5000, 2e-5)
    assert (its == g["iters"]).mean() > 0.95
    assert (g["activation"] >= 0).all()            # the whole slab activates


def test_cfg3_full_size_25000_steps(golden, ns):
    """Config 3 at its stated size AND length (442,401 nodes, three volumes with
    duplicated interface states, scar sigma x0.01, second stimulus at 0.3 s,
    25,000 steps = 500 ms) against the unmodified reference: per-step CG
    iterations, per-step probe traces, 50 snapshots, the full activation map."""
    from paper_2308_01651_b200 import configs

    g = golden("tissue_cfg3_full")
    steps = int(g["steps"])          # the committed fixture holds all 25,000
    s, pu, snaps = _run_long(g, configs.config3(ns), steps)
    assert len(s.volumes) == 3
    its = _check_long(s, pu, snaps, g, steps, 2e-5)
    assert (its == g["iters"]).mean() > 0.95
    if steps > 15200:   # the second pulse (t = 0.3 s, step 15,000) re-excites the slab
        assert g["iters"][15000:15200].max() > 10 and its[15000:15200].max() > 10


def test_cfg4_ventricle_100k_60ms(golden, ns):
    """Config 4 geometry reduced to 128,700 nodes (P1 tets, 3 volumes with
    duplicated interface states, helix fibers) over 60 ms (3,000 steps), on
    the diagonal operator, against the reference run on the same mesh."""
    from paper_2308_01651_b200 import ventricle

    g = golden("tissue_cfg4_100k")
    cfg = ventricle.config4(ns, *ventricle.size_for_nodes(100_000), final_time=60e-3)
    s, pu, snaps = _run_long(g, cfg, 3000)
    assert s.op.kind == 4
    its = _check_long(s, pu, snaps, g, 3000, 2e-5)
    assert its.max() >= 20


def test_cfg4_full_size_against_oracle_and_properties(ns):
    """Config 4 at BASELINE's full size (10,276,240 nodes, 59.9 M tets, 3 volumes) - beyond
    the reference itself (~28 h) - against the CPU oracle (pinned bit-for-bit
    to the reference on the smaller meshes) over the first two steps from rest, plus
    size-independent properties of the full-size operator and solve: the diagonal
    storage with its 77,922-entry seam list is symmetric and positive, K has zero row
    sums ((A_2 - A_1) 1 is a constant multiple of M 1), and the two- and three-sweep CG
    forms agree step by step."""
    import torch

    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import ventricle
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = ventricle.config4(ns, *ventricle.size_for_nodes(1e7))
    n = cfg.mesh.nodes.shape[0]
    assert n == 10_276_240
    s = TissueSolver(cfg)
    assert s.op.kind == 4 and s.op.np_ == 7 and s.op.nrem == 77_922 and s.cg_variant == 1
    # ---- the operator at full size --------------------------------------------------
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5
    y = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5
    A2 = s.op.a_tables[2]
    Ax, Ay = _spmv(s.op, A2, x), _spmv(s.op, A2, y)
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    assert abs(yh @ Ax - xh @ Ay) <= 1e-11 * (np.abs(yh) @ np.abs(Ax))
    assert xh @ Ax > 0 and yh @ Ay > 0
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    m1 = _spmv(s.op, s.op.d_m, one)
    d = _spmv(s.op, A2, one) - _spmv(s.op, s.op.a_tables[1], one)
    ratio = d / m1                       # (alpha_2 - alpha_1) chi C_m / dt on every row
    assert m1.min() > 0
    assert np.abs(ratio - np.median(ratio)).max() <= 1e-9 * abs(np.median(ratio))
    # ---- two steps from rest against the oracle ---------------------------------------
    orc = O.OracleTissue(cfg)
    for _ in range(2):
        s.enqueue_step()
        orc.step()
    s.sync()
    its = s.iterations_log()
    assert np.abs(its - np.array(orc.iters)).max() <= 1
    assert its.max() >= 70               # the full-size solve's iteration counts (8 on 8,000 nodes)
    assert _rel(s.potential, orc.potential) < 1e-8
    del orc
    # ---- the three-sweep form on the same steps ---------------------------------------
    u1 = s.potential.copy()
    del s
    torch.cuda.empty_cache()
    s0 = TissueSolver(cfg, cg_variant=0)
    for _ in range(2):
        s0.enqueue_step()
    s0.sync()
    assert np.abs(s0.iterations_log() - its).max() <= 1
    assert _rel(s0.potential, u1) < 1e-9


@pytest.mark.parametrize("key,steps", [("tissue_bo", 400), ("tissue_ttp", 1000)])
def test_rush_larsen_tissue_vs_reference_functions(golden, ns, key, steps):
    """gate_scheme="rush_larsen": the reference TissueSolver at BDF1 with its ionic
    update swapped for the RL integrator over the reference's own gate/current/rate
    functions (rl_kat golden) against the GPU solver in that mode."""
    import dataclasses

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    g = golden("rl_kat")
    cfg = configs.config0(ns) if key == "tissue_bo" else configs.config2(ns, h=0.5e-3)
    dt = cfg.dt
    s = TissueSolver(dataclasses.replace(cfg, bdf_order=1), gate_scheme="rush_larsen")
    probes = g[f"{key}_probes"]
    pu = np.empty((steps, probes.size))
    for k in range(steps):
        pu[k] = s.step()[probes]
    its = s.iterations_log()
    assert np.abs(its - g[f"{key}_iters"]).max() <= 1
    assert _rel(pu, g[f"{key}_probe_u"]) < 1e-8
    assert _rel(s.potential, g[f"{key}_final_u"]) < 1e-8
    np.testing.assert_allclose(s.volume_state(0), g[f"{key}_final_w"], rtol=1e-6, atol=1e-10)
    act, ref = s.activation_map, g[f"{key}_activation"]
    assert np.array_equal(act >= 0, ref >= 0)
    both = act >= 0
    assert np.abs(act[both] - ref[both]).max() <= dt * (1 + 1e-9)
    with pytest.raises(ValueError):
        TissueSolver(cfg, gate_scheme="forward_euler")


def test_rush_larsen_bdf2_potential_vs_oracle(ns):
    """RL ionic update under the BDF2 potential (states from W_n, u at u_EXT): live
    against the oracle in the same mode, three volumes."""
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config3(ns, h=0.5e-3)
    s = TissueSolver(cfg, gate_scheme="rush_larsen")
    o = O.OracleTissue(cfg, gate_scheme="rush_larsen")
    for _ in range(300):
        s.enqueue_step()
        o.step()
    s.sync()
    assert np.abs(s.iterations_log() - np.array(o.iters)).max() <= 1
    assert _rel(s.potential, o.potential) < 1e-9


def test_five_section_device_timing(ns):
    """timer.totals (simulation.py:225-254): with timed=True the ionic launches are
    timed by CUDA events and the fused solve kernel splits itself into assembly /
    solver / other through its globaltimer section stamps."""
    import time

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TIMING_SECTIONS, TissueSolver

    for build in (lambda: configs.config0(ns), lambda: configs.config0(ns, kind="Tet4")):
        s = TissueSolver(build(), timed=True)
        s.advance(5)
        s.sync()
        before = dict(s.timer.totals)
        t0 = time.perf_counter()
        s.advance(200)
        s.sync()
        wall = time.perf_counter() - t0
        tot = s.timer.totals
        assert tuple(tot) == TIMING_SECTIONS
        d = {k: tot[k] - before[k] for k in tot}
        for k in ("Ionic model update", "Monodomain assembly", "Linear solver"):
            assert d[k] > 0.0, k
        assert d["Other"] >= 0.0
        dev = sum(d[k] for k in TIMING_SECTIONS[1:])
        assert 0.3 * wall < dev < 1.05 * wall, (dev, wall)
        assert d["Linear solver"] > d["Monodomain assembly"]      # CG 28-41 iterations


def test_run_stops_on_device_when_fully_activated(ns):
    """run(stop_when_fully_activated=True) (simulation.py:702-703; the reference
    benchmark's mode, benchmark.py:166): the stop is detected on the device by the
    step that freezes the last node - same step count as the oracle's per-step
    check, no host synchronisation per step."""
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver, run

    cfg = configs.config0(ns, final_time=60e-3)      # fully activated at step 1,045
    o = O.OracleTissue(cfg)
    n_steps = int(round(cfg.final_time / cfg.dt))
    while o.step_index < n_steps:
        o.step()
        if o.frozen.all():
            break
    assert 100 < o.step_index < n_steps - 100          # it does stop early
    rep = run(cfg, stop_when_fully_activated=True)
    assert rep.steps == o.step_index
    assert rep.solver.stopped_at == o.step_index - 1
    assert rep.solver.time == pytest.approx(o.time, rel=1e-12)
    assert _rel(rep.final_potential, o.potential) < 1e-9
    assert (rep.activation_times >= 0).all()
    assert np.abs(rep.activation_times - o.activation_map).max() <= cfg.dt * (1 + 1e-9)
    assert rep.rows[-1][0] <= o.time + 1e-12 and len(rep.rows) >= 1
    # the counter also answers fully_activated() without copying the frozen field
    s = TissueSolver(cfg)
    s.advance(50)
    assert not s.fully_activated()
    assert int(s.frozen_count.item()) == int(s.frozen.ne(0).sum().item())
    s.restore(rep.solver.checkpoint_payload())
    assert s.fully_activated()
    # and the solver keeps stepping after a stop (status cleared)
    rep.solver.stop_when_full = False
    rep.solver.advance(3)
    rep.solver.sync()
    assert rep.solver.step_index == o.step_index + 3


@pytest.mark.parametrize("build", ["cfg0", "ttp", "tet", "sell"])
def test_solve_kernels_are_deterministic_run_to_run(ns, build):
    """compute-sanitizer is closed on this GPU pool, so the custom grid barrier /
    grid reduction (relaxed polling, double-buffered partials) is stress-checked
    the other way: a race would show as run-to-run differences.  Two fresh solvers
    must produce bit-identical potentials, states and iteration counts."""
    from paper_2308_01651_b200 import configs, ventricle
    from paper_2308_01651_b200.simulation import TissueSolver

    def make():
        if build == "cfg0":
            return TissueSolver(configs.config0(ns))                 # resident, 3 blocks
        if build == "ttp":
            return TissueSolver(configs.config2(ns, h=0.25e-3))      # resident, many blocks
        cfg = ventricle.config4(ns, *ventricle.size_for_nodes(60_000))
        return TissueSolver(cfg, operator="auto" if build == "tet" else "sell")

    outs = []
    for _ in range(2):
        s = make()
        s.advance(150)
        outs.append((s.potential, s.iterations_log(), s.volume_state(0)))
    assert np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][2], outs[1][2])


def test_checkpoint_format_and_cross_restore(golden, ns):
    """Restore the REFERENCE's checkpoint (step 400) and continue to 800."""
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    g = golden("tissue_cfg0")
    cfg = configs.config0(ns)
    s = TissueSolver(cfg)
    s.restore(g["payload_400"].tobytes())
    assert s.step_index == 400
    s.advance(400)
    assert _rel(s.potential, g["final_u"]) < 1e-9
    # our payload has the reference layout and round-trips
    ref_payload = g["payload_400"].tobytes()
    s2 = TissueSolver(cfg)
    s2.advance(400)
    mine = s2.checkpoint_payload()
    assert len(mine) == len(ref_payload)
    assert mine[:12] == ref_payload[:12]
    s3 = TissueSolver(cfg)
    s3.restore(mine)
    assert s3.checkpoint_payload() == mine
    # trimmed to the BDF order's history levels (bench.py's e2e input): shorter, and
    # the continuation is bit-identical to the full payload's
    short = s2.checkpoint_payload(levels=cfg.bdf_order)
    assert len(short) < len(mine)
    s4 = TissueSolver(cfg)
    s4.restore(short)
    assert s4.step_index == 400
    s3.advance(50)
    s4.advance(50)
    assert np.array_equal(s3.potential, s4.potential)
    assert np.array_equal(s3.iterations_log(), s4.iterations_log())


def test_divergence_is_raised_and_state_rolls_back(ns):
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.errors import SolverDivergence
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config0(ns, h=1e-3)
    cfg.linear_solver.max_iterations = 3
    s = TissueSolver(cfg)
    for _ in range(5):
        s.enqueue_step()
    with pytest.raises(SolverDivergence) as err:
        s.sync()
    assert err.value.iterations == 3
    assert s.step_index == 0 and s.time == 0.0


def test_oracle_live_parity_random_config(ns):
    """A seeded two-material slab, BDF3, checked against the live oracle."""
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config3(ns, h=1e-3, seed=7)
    cfg.bdf_order = 3
    s = TissueSolver(cfg)
    o = O.OracleTissue(cfg)
    for _ in range(150):
        s.enqueue_step()
        o.step()
    s.sync()
    assert np.abs(s.iterations_log() - np.array(o.iters)).max() <= 1
    assert _rel(s.potential, o.potential) < 1e-9


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_cfg0_all_cg_variants(golden, ns, variant):
    """0: the reference's recurrences verbatim; 1: q by recurrence; 2: pipelined."""
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    g = golden("tissue_cfg0")
    s = TissueSolver(configs.config0(ns), cg_variant=variant)
    probes = g["probes"]
    pu = np.empty((800, probes.size))
    for k in range(800):
        pu[k] = s.step()[probes]
    _check(s, pu, g, 5e-5, 800)


def test_single_block_and_multi_block_grids_agree(ns):
    """The same solve on 1 block and on many blocks (grid barrier path)."""
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config0(ns)
    runs = []
    for blocks in (1, 7):
        s = TissueSolver(cfg, blocks_hint=blocks)
        s.advance(100)
        runs.append((s.iterations_log(), s.potential))
    assert np.abs(runs[0][0] - runs[1][0]).max() <= 1
    assert _rel(runs[0][1], runs[1][1]) < 1e-10


@pytest.mark.parametrize("variant", [0, 2])
def test_ttp06_slab_cg_variants(golden, ns, variant):
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    g = golden("tissue_ttp_h05")
    s = TissueSolver(configs.config2(ns, h=0.5e-3), cg_variant=variant)
    probes = g["probes"]
    pu = np.empty((2000, probes.size))
    for k in range(2000):
        s.enqueue_step()
        if (k + 1) % 100 == 0:
            s.sync()
    s.sync()
    its = s.iterations_log()
    assert np.abs(its - g["iters"]).max() <= 1
    assert _rel(s.potential, g["final_u"]) < 1e-8


def _dist_cfg(name):
    from paper_2308_01651_b200 import configs, ventricle

    ns = configs.this_package()
    if name == "tissue_cfg0":
        return configs.config0(ns)
    return ventricle.config4(ns, n_xi=4, n_th=24, n_ph=64, final_time=30e-3)


@pytest.mark.parametrize("name,steps,sweep_min", [("tissue_cfg0", 300, None),
                                                  ("tissue_cfg4_small", 500, None),
                                                  ("tissue_cfg4_small", 500, 1)])
def test_distributed_solver_single_rank_on_gpu(golden, monkeypatch, name, steps, sweep_min):
    """DistributedTissueSolver (rank-local TissueSolver, phase kernels with
    row classes, NCCL plumbing) with one rank reproduces the reference run
    (multi-rank host logic: tests/test_distributed.py over gloo).  sweep_min=1
    runs the large-slab sweep kernel (pcg_sweep_kernel) on the small mesh."""
    import os
    import socket

    if sweep_min is not None:
        monkeypatch.setenv("MDX_SWEEP_MIN_ROWS", str(sweep_min))

    import torch.distributed as dist

    from paper_2308_01651_b200.distributed import DistributedTissueSolver

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = golden(name)
        s = DistributedTissueSolver(_dist_cfg(name))
        for _ in range(steps):
            s.step()
        its = np.array(s.iters)
        assert np.abs(its - g["iters"][:steps]).max() <= 1
        assert _rel(s.gather_potential(), g[f"snap_{steps}"]) < 1e-9
    finally:
        dist.destroy_process_group()


def _gloo_gpu_worker(rank, world, port, name, steps, out_dir, backend="gloo"):
    import os
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_2308_01651_b200.distributed import DistributedTissueSolver

    if backend == "nccl":            # one GPU per rank
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = DistributedTissueSolver(_dist_cfg(name))
        for _ in range(steps):
            s.step()
        u = s.gather_potential()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=u, iters=np.array(s.iters),
                 act=s.gather_activation_map(), kind=np.array(s.local.op.kind))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,steps,kind,sweep_min", [("tissue_cfg0", 200, 1, None),
                                                       ("tissue_cfg4_small", 500, 4, None),
                                                       ("tissue_cfg4_small", 500, 4, 1)])
def test_distributed_two_ranks_on_gpu_gloo(golden, tmp_path, monkeypatch, name, steps, kind,
                                           sweep_min):
    """The multi-rank GPU path (RCB boxes, rank-local problems: class-table
    stencil on the slab, diagonal operator on the ventricle; device-scalar
    pipelined PCG with the interior sweep overlapping the halo) with two
    ranks sharing the one GPU of the box.  Exchanges go through gloo host
    staging, so no rank's kernels wait on another's; NCCL itself is covered
    by the single-rank test."""
    import socket

    import torch.multiprocessing as mp

    if sweep_min is not None:     # the workers inherit it: pcg_sweep_kernel with row classes
        monkeypatch.setenv("MDX_SWEEP_MIN_ROWS", str(sweep_min))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(_gloo_gpu_worker, args=(2, port, name, steps, str(tmp_path)), nprocs=2,
             join=True)
    g = golden(name)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    np.testing.assert_array_equal(res[0]["u"], res[1]["u"])
    np.testing.assert_array_equal(res[0]["iters"], res[1]["iters"])
    assert int(res[0]["kind"]) == kind
    assert np.abs(res[0]["iters"] - g["iters"][:steps]).max() <= 1
    assert _rel(res[0]["u"], g[f"snap_{steps}"]) < 1e-9


@pytest.mark.parametrize("name,steps,kind", [("tissue_cfg0", 200, 1),
                                             ("tissue_cfg4_small", 500, 4)])
def test_distributed_two_ranks_nccl(golden, tmp_path, monkeypatch, name, steps, kind):
    """Two ranks on two GPUs over NCCL: the packed halo exchange posted with
    batch_isend_irecv on NCCL's stream while the interior rows are swept, the
    boundary rows after work.wait(), one all-reduce per iteration - the stream
    ordering the gloo tests cannot exercise.  Needs a box with two GPUs (skipped
    on this pool's one-GPU boxes: NCCL refuses two ranks on one device)."""
    import socket

    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    monkeypatch.setenv("MDX_SWEEP_MIN_ROWS", "1")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(_gloo_gpu_worker, args=(2, port, name, steps, str(tmp_path), "nccl"), nprocs=2,
             join=True)
    g = golden(name)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    np.testing.assert_array_equal(res[0]["u"], res[1]["u"])
    np.testing.assert_array_equal(res[0]["iters"], res[1]["iters"])
    assert int(res[0]["kind"]) == kind
    assert np.abs(res[0]["iters"] - g["iters"][:steps]).max() <= 1
    assert _rel(res[0]["u"], g[f"snap_{steps}"]) < 1e-9


def test_fused_output_row(ns):
    """enqueue_step(record=...): the solve kernel writes [min, max, probes] of
    the new potential into pinned host memory (resident stencil kernel on a
    slab, grid-stride SELL kernel on tets) - same values as the standalone
    record_row kernel and as the potential itself."""
    import torch

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    for cfg in (configs.config0(ns), configs.config0(ns, kind="Tet4")):
        s = TissueSolver(cfg)
        probes = torch.tensor([0, 7, s.n // 2, s.n - 1], device="cuda")
        fused = torch.zeros((40, 6), dtype=torch.float64, pin_memory=True)
        alone = torch.zeros((40, 6), dtype=torch.float64, pin_memory=True)
        pots = []
        for k in range(40):
            s.enqueue_step(record=(probes, fused[k]))
            s.record_row(probes, alone[k])
            pots.append(s.potential_device.clone())
        s.sync()
        for k in range(40):
            u = pots[k].cpu().numpy()
            want = [u.min(), u.max(), *u[probes.cpu().numpy()]]
            np.testing.assert_array_equal(fused[k].numpy(), want)
            np.testing.assert_array_equal(alone[k].numpy(), want)


def test_cfg4_ventricle_small(golden, ns):
    """Config-4 geometry (prolate-spheroid P1 tets, helix fibers, endo/mid/epi
    volumes with duplicated interface states) on a reduced grid, CSR path."""
    from paper_2308_01651_b200.simulation import TissueSolver
    from paper_2308_01651_b200.ventricle import config4

    g = golden("tissue_cfg4_small")
    cfg = config4(ns, n_xi=4, n_th=24, n_ph=64, final_time=30e-3)
    for operator, kind in (("auto", 4), ("sell", 3)):       # DIASYM, SELL-32
        s, pu = _run_against(g, cfg, 1500, operator=operator)
        assert s.op.kind == kind
        _check(s, pu, g, 2e-5, 1500)
        assert _rel(s.potential, g["final_u"]) < 1e-8


def _spmv(op, vals, x):
    import torch

    from paper_2308_01651_b200 import _native as N

    a = N.CgArgs()
    a.op = op.operator()
    a.a_val = N.ptr(vals)
    y = torch.empty_like(x)
    N.check(N.lib().mdx_spmv(N.C.byref(a), N.ptr(x), N.ptr(y), N.stream_handle()))
    return y.cpu().numpy()


def test_dia_operator_matches_csr(ns):
    """Symmetric diagonal storage (MDX_OP_DIASYM) vs the bit-exact CSR values:
    A[i, i-d] is read from row i-d's copy, so rows differ from the reference
    rows by the assembly's own K_ab / K_ba round-off only.  Covers P1 tets
    (7 stored offsets), the ventricle's periodic seam (remainder list), hex
    slabs (13 offsets) and the multi-volume lift matrices."""
    import torch

    from paper_2308_01651_b200 import _native as N, configs
    from paper_2308_01651_b200.simulation import TissueSolver
    from paper_2308_01651_b200.ventricle import config4

    cases = [(configs.config0(ns, kind="Tet4"), 8, False),
             (config4(ns, n_xi=4, n_th=24, n_ph=64), 7, True),
             (configs.config3(ns, h=0.5e-3), 13, False)]
    for cfg, nd, seam in cases:
        dia = TissueSolver(cfg, operator="dia")
        csr = TissueSolver(cfg, operator="csr")
        assert dia.op.kind == N.OP_DIASYM and dia.op.np_ <= nd
        assert (dia.op.nrem > 0) == seam
        assert dia.op.max_rel_dev < 1e-13
        x = torch.from_numpy(np.random.default_rng(3).standard_normal(dia.n)).cuda()
        pairs = [(dia.op.a_tables[k], csr.op.a_tables[k]) for k in dia.op.a_tables]
        pairs += [(dia.op.d_m, csr.op.d_m)]
        pairs += list(zip(dia.op.d_lift, csr.op.d_lift))
        for vd, vc in pairs:
            yd = _spmv(dia.op, vd, x)
            yc = _spmv(csr.op, vc, x)
            scale = _spmv(csr.op, vc.abs(), x.abs())
            assert (np.abs(yd - yc) <= 1e-13 * scale + 1e-300).all()
        # device bytes per node: (1 + 7) doubles for tets vs CSR's 12 B/entry
        assert dia.op.device_bytes() < 0.5 * csr.op.device_bytes()


def test_run_loop_rows_csv_and_vtk(golden, ns, tmp_path):
    """run() (simulation.py:651-716): output rows, CSV/VTK writers, report."""
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.outputs import OutputConfig
    from paper_2308_01651_b200.simulation import ActivationConfig, run

    g = golden("tissue_cfg0")
    cfg = configs.config0(ns, final_time=100 * 5e-5)
    pts = [tuple(ns_node) for ns_node in cfg.mesh.nodes[g["probes"]]]
    cfg.output = OutputConfig(enable_csv=True, csv_path=str(tmp_path / "t.csv"), stride=10,
                              probe_points=tuple(pts))
    cfg.activation = ActivationConfig(enabled=True, path=str(tmp_path / "act.vtk"),
                                      threshold=84.0 / 85.7)
    rep = run(cfg)
    assert rep.steps == 100
    rows = np.array(rep.rows)
    assert rows.shape == (11, 3 + len(pts))
    np.testing.assert_allclose(rows[1:, 3:], g["probe_u"][9:100:10], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(rows[1:, 2], g["umax"][9:100:10], rtol=1e-9)
    text = (tmp_path / "t.csv").read_text().splitlines()
    assert text[0].startswith("t,u_min,u_max,probe_0") and len(text) == 12
    assert (tmp_path / "act.vtk").read_text().startswith("# vtk DataFile Version 3.0")
    assert rep.max_cg_iterations == int(g["iters"][:100].max()) or \
        abs(rep.max_cg_iterations - int(g["iters"][:100].max())) <= 1


def test_stream_kernel_parity(tmp_path):
    """The brick-streaming solver (MDX_PCG_KERNEL=stream, chosen once per
    process) against the reference goldens: config 0 (BO, full 800 steps),
    the TTP06 slab and config 2 at full size, in a child pytest."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, MDX_PCG_KERNEL="stream", MDX_DEBUG_PLAN="1")
    sel = "cfg0_bo_full_run or test_ttp06_slab or cfg2_full_size_head"
    res = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-s", "-m", "gpu",
                          "-k", sel, "-p", "no:cacheprovider", __file__],
                         env=env, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert "[mdx] stream plan" in out, out[-2000:]
    import re

    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 3 and " failed" not in out, out[-2000:]


def test_tiny_meshes_cooperative_grid_path(tmp_path):
    """Meshes of <= 6,144 nodes run the resident PCG as one thread-block cluster with
    DSMEM reductions (the default: the config-0 and h=0.5 mm TTP06 goldens above go
    through it with 6 blocks, smoke() with 2).
    MDX_PCG_CLUSTER=0 (chosen once per process) keeps the cooperative-grid reduction:
    the same goldens in a child pytest, and a launch-plan line to prove the switch."""
    import os
    import re
    import subprocess
    import sys

    env = dict(os.environ, MDX_PCG_CLUSTER="0")
    sel = "cfg0_bo_full_run or rush_larsen_tissue_vs_reference_functions or fused_output_row"
    res = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-k", sel,
                          "-p", "no:cacheprovider", __file__],
                         env=env, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 3 and " failed" not in out, out[-2000:]


def test_restore_from_pinned_tensor(ns):
    """restore() from a pinned uint8 tensor (one async DMA) = restore from bytes."""
    import torch

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config0(ns, h=1e-3)
    s = TissueSolver(cfg)
    for _ in range(7):
        s.step(return_potential=False)
    s.sync()
    payload = s.checkpoint_payload()
    a, b = TissueSolver(cfg), TissueSolver(cfg)
    a.restore(payload)
    b.restore(torch.frombuffer(bytearray(payload), dtype=torch.uint8).pin_memory())
    for _ in range(5):
        a.step(return_potential=False)
        b.step(return_potential=False)
    a.sync()
    b.sync()
    assert np.array_equal(a.potential, b.potential)
    assert np.array_equal(a.activation_map, b.activation_map)
    assert a.step_index == b.step_index == 12
