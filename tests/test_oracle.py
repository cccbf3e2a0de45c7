"""Pin the CPU oracle to the reference's own outputs (tests/golden/).

The oracle (oracle/mdx_oracle.c + oracle/monodomain_oracle.py) is only
trusted as the checker of the CUDA path after it reproduces the golden
vectors produced by the unmodified reference (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from oracle import monodomain_oracle as O

MODELS = {"ttp06": "TTP06", "bo": "Bueno-Orovio", "apf": "Aliev-Panfilov"}


def _cases(g):
    for key in g:
        if key.endswith("_Wout"):
            tag = key[: -len("_Wout")]
            model_tag = tag.split("_a")[0]
            yield tag, model_tag


@pytest.mark.parametrize("model", ["ttp06", "bo", "apf"])
def test_oracle_advance_matches_reference(golden, model):
    g = golden("ionic_kat")
    seen = 0
    for tag, mt in _cases(g):
        if not mt.startswith(model + "_"):
            continue
        rest = tag[len(mt) + 2:]           # "1.0_dt2e-05"
        alpha = float(rest.split("_dt")[0])
        dt = float(rest.split("_dt")[1])
        u, We, Wb, P = g[f"{mt}_u"], g[f"{mt}_Wext"], g[f"{mt}_Wbdf"], g[f"{mt}_P"]
        Wo = np.empty_like(We)
        Io = np.empty(u.size)
        c = O.advance(MODELS[model], u, We, Wb, alpha, dt, P, Wo, Io)
        np.testing.assert_allclose(Wo, g[f"{tag}_Wout"], rtol=1e-13, atol=1e-300)
        np.testing.assert_allclose(Io, g[f"{tag}_Iout"], rtol=1e-11, atol=1e-12)
        assert c == int(g[f"{tag}_clamped"])
        seen += 1
    assert seen >= 4


def test_oracle_current_and_rest_kat(golden):
    g = golden("ionic_kat")
    for mt in ("ttp06_epi", "bo_-", "apf_-"):
        model = MODELS[mt.split("_")[0]]
        Io = np.empty(g[f"{mt}_u"].size)
        O.current(model, g[f"{mt}_u"], g[f"{mt}_Wext"], g[f"{mt}_P"], Io)
        np.testing.assert_allclose(Io, g[f"{mt}_current"], rtol=1e-11, atol=1e-12)
    # TTP06 rest current, tests/test_ionic.py:119-125
    from paper_2308_01651_b200.ionic import ten_tusscher as T

    st = T.default_initial_state()
    P = T.pack(T.default_parameters())
    Io = np.empty(1)
    O.current("TTP06", np.array([st.u]), st.w.reshape(1, -1), P, Io)
    assert Io[0] == pytest.approx(0.0017519776588273556, rel=1e-12)
    assert Io[0] == pytest.approx(float(g["kat_ttp06_rest_current"]), rel=1e-14)


def test_oracle_cfg1_subset(golden):
    """0D splitting over a seeded TTP06 batch (config 1 parity subset)."""
    g = golden("cfg1_subset")
    from paper_2308_01651_b200.ionic import ten_tusscher as T

    P = T.pack(T.default_parameters())
    for order in (1, 2):
        u, W, peak, clamps = O.pace_batch("TTP06", P, g["u0"], g["W0"], 1e-5, 2000, order,
                                          int(g["n_stim"]), 52.0, 1e-3)
        np.testing.assert_allclose(u, g[f"o{order}_u"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(W, g[f"o{order}_W"], rtol=1e-8, atol=1e-14)
        np.testing.assert_allclose(peak, g[f"o{order}_peak"], rtol=1e-9, atol=1e-12)
        assert clamps == int(g[f"o{order}_clamps"])


def _mesh(name, ns):
    from paper_2308_01651_b200.geometry import ElementKind, Mesh, SlabSpec, build_slab_mesh

    spec = {
        "unit_hex": ((1.0, 1.0, 1.0), 1.0, "Hex8", (0, 0.0, 0.0)),
        "hex27": ((1e-3, 1e-3, 1e-3), 0.5e-3, "Hex8", (0, 60.0, -60.0)),
        "tet_slab": ((2e-3, 3e-3, 4e-3), 0.5e-3, "Tet4", (2, 60.0, -60.0)),
        "hex_slab": ((2e-3, 3e-3, 4e-3), 0.5e-3, "Hex8", (2, 60.0, -60.0)),
        "cfg0_hex": ((20e-3, 7e-3, 3e-3), 0.5e-3, "Hex8", (2, 0.0, 0.0)),
        "cfg0_tet": ((20e-3, 7e-3, 3e-3), 0.5e-3, "Tet4", (2, 0.0, 0.0)),
    }[name]
    mesh = build_slab_mesh(SlabSpec(spec[0], spec[1], ElementKind(spec[2])))
    two = name in ("tet_slab", "hex_slab")
    if two:
        mats = mesh.material_ids.copy()
        zc = mesh.nodes[mesh.elements].mean(axis=1)[:, 2]
        mats[zc > 2e-3] = 2
        mesh = mesh.with_materials(mats)
    return mesh, spec[3], two


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["unit_hex", "hex27", "tet_slab", "hex_slab",
                                  "cfg0_hex", "cfg0_tet"])
def test_oracle_assembly_bit_identical(golden, ns, name):
    from paper_2308_01651_b200.geometry import slab_fiber_field

    g = golden("operators")
    mesh, fib, two = _mesh(name, ns)
    fibers = slab_fiber_field(mesh, *fib)
    pat = O.pattern(mesh.nodes.shape[0], mesh.elements)
    assert _sha(pat[0]) == str(g[f"{name}_K_indptr_sha"])
    assert _sha(pat[1]) == str(g[f"{name}_K_indices_sha"])
    table = [(1.2e-4, 3e-5, 1.5e-5)] + ([(2e-4, 1e-5, 1e-5)] if two else [])
    rows = (mesh.material_ids - 1).astype(np.int64)
    K = O.assemble_stiffness(mesh, rows, table, fibers, pat)
    M = O.assemble_mass(mesh, np.ones(mesh.elements.shape[0], np.uint8), pat)
    assert _sha(K.data) == str(g[f"{name}_K_data_sha"])
    assert _sha(M.data) == str(g[f"{name}_M_data_sha"])
    if two:
        M1 = O.assemble_mass(mesh, mesh.material_ids == 1, pat)
        assert _sha(M1.data) == str(g[f"{name}_M1_data_sha"])


def test_oracle_cg_known_system(golden):
    from paper_2308_01651_b200.geometry import ElementKind, SlabSpec, build_slab_mesh, slab_fiber_field

    g = golden("cg_kat")
    mesh = build_slab_mesh(SlabSpec((3e-3, 7e-3, 20e-3), 0.5e-3, ElementKind.HEX8))
    fibers = slab_fiber_field(mesh, 0, 0.0, 0.0)
    pat = O.pattern(mesh.nodes.shape[0], mesh.elements)
    K = O.assemble_stiffness(mesh, np.zeros(mesh.elements.shape[0], np.int64),
                             [(0.95298e-4, 0.12576e-4, 0.12576e-4)], fibers, pat)
    M = O.assemble_mass(mesh, np.ones(mesh.elements.shape[0], np.uint8), pat)
    A = O.add_scaled(1.5 / 5e-5, M, K)
    assert _sha(A.data) == str(g["A_data_sha"])
    inv = 1.0 / A.diagonal()
    x, it, rel = O.cg(A, inv, g["b"], np.zeros_like(g["b"]), 1e-10, 2000)
    assert it == int(g["iters"])
    np.testing.assert_array_equal(x, g["x"])       # same serial algorithm: bitwise
    xw, itw, _ = O.cg(A, inv, g["b"], g["x0"], 1e-10, 2000)
    assert itw == int(g["itersw"])
    np.testing.assert_array_equal(xw, g["xw"])
    _, it0, _ = O.cg(A, inv, g["b"], g["x"], 1e-10, 2000)
    assert it0 == 0                                 # warm start (test_linalg.py:55-60)


@pytest.mark.parametrize("name,build,steps", [
    ("tissue_cfg0", lambda c, ns: c.config0(ns), 800),
    ("tissue_tet", lambda c, ns: c.config0(ns, kind="Tet4"), 400),
])
def test_oracle_tissue_matches_reference(golden, ns, name, build, steps):
    from paper_2308_01651_b200 import configs

    g = golden(name)
    cfg = build(configs, ns)
    orc = O.OracleTissue(cfg)
    probes = g["probes"]
    pu = np.empty((steps, probes.size))
    for k in range(steps):
        u = orc.step()
        pu[k] = u[probes]
    assert np.array_equal(np.array(orc.iters), g["iters"])
    np.testing.assert_array_equal(pu, g["probe_u"])   # serial oracle: bitwise
    np.testing.assert_array_equal(orc.activation_map, g["activation"])
    np.testing.assert_array_equal(orc.potential, g["final_u"])


@pytest.mark.slow
def test_oracle_tissue_ttp_h05(golden, ns):
    from paper_2308_01651_b200 import configs

    g = golden("tissue_ttp_h05")
    orc = O.OracleTissue(configs.config2(ns, h=0.5e-3))
    steps = int(g["steps"])
    for k in range(steps):
        orc.step()
    assert np.array_equal(np.array(orc.iters), g["iters"])
    np.testing.assert_allclose(orc.potential, g["final_u"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(orc.activation_map, g["activation"])


def test_oracle_cfg4_ventricle_small(golden, ns):
    from paper_2308_01651_b200.ventricle import config4

    g = golden("tissue_cfg4_small")
    orc = O.OracleTissue(config4(ns, n_xi=4, n_th=24, n_ph=64, final_time=30e-3))
    for _ in range(300):
        orc.step()
    assert np.array_equal(np.array(orc.iters), g["iters"][:300])


# ---------------------------------------------------------------------------
# Rush-Larsen mode: the oracle's integrator over the restated reference functions
# against fixtures built from the reference's OWN jitted functions with the same
# integrator (tests/golden/make_golden.py: rl_kat)
# ---------------------------------------------------------------------------

RL_CASES = [("ttp06_epi", "TTP06"), ("ttp06_endo", "TTP06"), ("ttp06_myo", "TTP06"),
            ("bo_-", "Bueno-Orovio"), ("apf_-", "Aliev-Panfilov")]


@pytest.mark.parametrize("tag,model", RL_CASES)
def test_oracle_rush_larsen_step(golden, tag, model):
    g, kat = golden("rl_kat"), golden("ionic_kat")
    u, P, Wn = kat[f"{tag}_u"], kat[f"{tag}_P"], g[f"{tag}_Wn"]
    seen = 0
    for key in g:
        if key.startswith(f"{tag}_dt") and key.endswith("_Wout"):
            dt = float(key[len(tag) + 3: -len("_Wout")])
            Wo, Io = np.empty_like(Wn), np.empty(u.size)
            c = O.advance_rl(model, u, Wn, dt, P, Wo, Io)
            np.testing.assert_allclose(Wo, g[f"{tag}_dt{dt:g}_Wout"], rtol=1e-13, atol=1e-300)
            np.testing.assert_allclose(Io, g[f"{tag}_dt{dt:g}_Iout"], rtol=1e-11, atol=1e-12)
            assert c == int(g[f"{tag}_dt{dt:g}_clamped"])
            if model != "Aliev-Panfilov":
                assert c > 0                      # the out-of-range gates were clamped
            seen += 1
    assert seen == 2


def test_oracle_rush_larsen_cfg1_subset(golden):
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.ionic import ten_tusscher as T

    g = golden("rl_kat")
    u0, W0 = configs.config1_initial(512)
    P = T.pack(T.default_parameters())
    u, W, peak, clamps = O.pace_batch("TTP06", P, u0, W0, 1e-5, 2000, 1, int(g["cfg1_n_stim"]),
                                      52.0, 1e-3, gate_scheme="rush_larsen")
    np.testing.assert_allclose(u, g["cfg1_u"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(W, g["cfg1_W"], rtol=1e-8, atol=1e-14)
    np.testing.assert_allclose(peak, g["cfg1_peak"], rtol=1e-9, atol=1e-12)
    assert clamps == int(g["cfg1_clamps"])


@pytest.mark.parametrize("key,steps", [("tissue_bo", 400), ("tissue_ttp", 1000)])
def test_oracle_rush_larsen_tissue(golden, ns, key, steps):
    """Reference TissueSolver at BDF1 with the RL ionic update vs the oracle in
    gate_scheme="rush_larsen" mode: same iterations, probes, activation map."""
    import dataclasses

    from paper_2308_01651_b200 import configs

    g = golden("rl_kat")
    cfg = configs.config0(ns) if key == "tissue_bo" else configs.config2(ns, h=0.5e-3)
    orc = O.OracleTissue(dataclasses.replace(cfg, bdf_order=1), gate_scheme="rush_larsen")
    probes = g[f"{key}_probes"]
    pu = np.empty((steps, probes.size))
    for k in range(steps):
        pu[k] = orc.step()[probes]
    assert np.array_equal(np.array(orc.iters), g[f"{key}_iters"])
    np.testing.assert_allclose(pu, g[f"{key}_probe_u"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(orc.potential, g[f"{key}_final_u"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(orc.activation_map, g[f"{key}_activation"])
