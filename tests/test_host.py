"""Host-side logic that needs no GPU: BDF tables, history ring, geometry,
fiber fields, stimulus windows, configuration validation, CSR pattern and
incidence, lattice detection, config-4 generator.  Mirrors the reference's
own tests where they apply (tests/test_timestepping.py, test_geometry.py)."""

import numpy as np
import pytest

from paper_2308_01651_b200 import configs
from paper_2308_01651_b200.errors import (ConfigError, HistoryTooShort, InvertedElement,
                                          NonDivisibleExtent, UnsupportedOrder, ZeroSpacing)
from paper_2308_01651_b200.fem import FeSpace, detect_lattice
from paper_2308_01651_b200.geometry import (ElementKind, Mesh, SlabSpec, build_slab_mesh,
                                            nearest_node, slab_fiber_field)
from paper_2308_01651_b200.simulation import StimulusProtocol, StimulusShape, validate_config
from paper_2308_01651_b200.timestepping import (HistoryRing, bdf_coefficients, ring_slot,
                                                startup_schedule)


def test_bdf_tables_and_errors():
    s = bdf_coefficients(2)
    assert (s.alpha, s.history_weights, s.ext_weights) == (1.5, (2.0, -0.5), (2.0, -1.0))
    assert bdf_coefficients(3).alpha == 11.0 / 6.0
    for bad in (0, 4, -1, "2", None, 2.5, True):
        with pytest.raises(UnsupportedOrder):
            bdf_coefficients(bad)
    assert startup_schedule(3, 6) == [1, 2, 3, 3, 3, 3]
    for order in (1, 2, 3):
        sc = bdf_coefficients(order)
        assert sum(sc.history_weights) == pytest.approx(sc.alpha, abs=1e-15)
        assert sum(sc.ext_weights) == pytest.approx(1.0, abs=1e-15)


def test_history_ring_semantics():
    ring = HistoryRing(3)
    for v in (1.0, 2.0, 3.0, 4.0):
        ring.push(np.array([v]))
    assert ring.fill == 3 and [ring[k][0] for k in range(3)] == [4.0, 3.0, 2.0]
    np.testing.assert_array_equal(ring.weighted_sum((2.0, -1.0)), [5.0])
    with pytest.raises(ValueError):
        ring.push(np.zeros(2))
    short = HistoryRing()
    short.push(np.zeros(1))
    with pytest.raises(HistoryTooShort):
        short.weighted_sum((1.0, 1.0))
    # device ring slot arithmetic: k pushes back from head, modulo 4 slots
    assert [ring_slot(0, k) for k in range(3)] == [0, 2, 1]


def test_slab_mesh_counts_numbering_and_errors():
    m = build_slab_mesh(SlabSpec((20e-3, 7e-3, 3e-3), 0.5e-3))
    assert m.num_nodes == 41 * 15 * 7 and m.num_elements == 40 * 14 * 6
    assert m.lattice == (40, 14, 6)
    i, j, k = 3, 5, 2
    assert np.allclose(m.nodes[i + 41 * (j + 15 * k)], (i * 0.5e-3, j * 0.5e-3, k * 0.5e-3))
    t = build_slab_mesh(SlabSpec((2e-3, 3e-3, 4e-3), 0.5e-3, ElementKind.TET4))
    assert t.num_elements == 6 * 4 * 6 * 8
    with pytest.raises(NonDivisibleExtent):
        SlabSpec((1e-3, 1e-3, 1.1e-3), 0.5e-3).cells_per_axis()
    with pytest.raises(ZeroSpacing):
        SlabSpec((1e-3, 1e-3, 1e-3), 0.0)
    bad = Mesh(m.nodes, m.elements[:, [1, 0, 2, 3, 5, 4, 6, 7]], m.element_kind, m.material_ids)
    with pytest.raises(InvertedElement):
        bad.validate()
    assert nearest_node(m, (20e-3, 7e-3, 3e-3)) == m.num_nodes - 1


def test_fiber_field_rotation_and_frame():
    m = build_slab_mesh(SlabSpec((2e-3, 3e-3, 4e-3), 0.5e-3))
    f = slab_fiber_field(m, 2, 60.0, -60.0)
    top = m.nodes[:, 2] == m.nodes[:, 2].max()
    ang = np.rad2deg(np.arctan2(f.f0[top, 0], f.f0[top, 1]))
    # long in-plane axis is y (3 mm > 2 mm); e_perp = z x y = -x, so the epi
    # angle of -60 deg puts f0 at +60 deg from y toward x
    assert np.allclose(ang, 60.0)
    np.testing.assert_allclose(np.einsum("ij,ij->i", f.f0, f.s0), 0.0, atol=1e-14)
    np.testing.assert_allclose(np.linalg.norm(np.cross(f.f0, f.s0), axis=1), 1.0)


def test_stimulus_windows_left_closed_and_periodic():
    p = StimulusProtocol(StimulusShape.CUBIC, ((0.0, 0.0, 0.0),), (1.0,), (1e-3,), (1e-3,),
                         (2e-3,))
    assert not p.window_active(0, 0.5e-3)
    assert p.window_active(0, 1e-3)
    assert p.window_active(0, 3e-3 - 1e-12)
    assert not p.window_active(0, 3e-3)
    q = StimulusProtocol(StimulusShape.CUBIC, ((0.0, 0.0, 0.0),), (1.0,), (1e-3,), (0.0,),
                         (2e-3,), period=0.5)
    assert q.window_active(0, 0.5) and not q.window_active(0, 0.5 + 2e-3)
    # the accumulated-time trap: step 40 of config 0 is still stimulated
    t = 0.0
    for _ in range(40):
        t += 5e-5
    assert t < 2e-3 and p.window_active(0, t + 1e-3)
    pts = np.array([[0.0, 0.0, 0.0], [0.5e-3, 0.5e-3, 0.5e-3], [0.6e-3, 0.0, 0.0]])
    np.testing.assert_array_equal(p.spatial_factor(pts, 0), [1.0, 1.0, 0.0])
    with pytest.raises(ValueError):
        StimulusProtocol(StimulusShape.CUBIC, ((0, 0, 0),), (1.0, 2.0), (1e-3,), (0.0,), (1e-3,))


def test_config_validation_errors():
    ns = configs.this_package()
    cfg = configs.config0(ns, h=1e-3)
    validate_config(cfg)
    cfg.dt = 0.0
    with pytest.raises(ConfigError):
        validate_config(cfg)
    cfg = configs.config3(ns, h=1e-3)
    vols = list(cfg.volumes)
    cfg.volumes = tuple(vols[:-1])              # a material left unclaimed
    with pytest.raises(ConfigError):
        validate_config(cfg)
    cfg.volumes = tuple(vols + [vols[0]])       # a material claimed twice
    with pytest.raises(ConfigError):
        validate_config(cfg)


def test_pattern_and_incidence_match_element_connectivity():
    m = build_slab_mesh(SlabSpec((2e-3, 1.5e-3, 1e-3), 0.5e-3, ElementKind.TET4))
    sp = FeSpace(m)
    indptr, indices = sp.pattern()
    pairs = {(int(a), int(b)) for e in m.elements for a in e for b in e}
    got = {(r, int(c)) for r in range(sp.num_dofs) for c in indices[indptr[r]:indptr[r + 1]]}
    assert got == pairs
    ptr, elem, loc = sp.incidence()
    for node in (0, 7, sp.num_dofs - 1):
        es = elem[ptr[node]:ptr[node + 1]]
        assert np.all(np.diff(es) > 0)                      # ascending element order
        assert all(m.elements[e][l] == node for e, l in zip(es, loc[ptr[node]:ptr[node + 1]]))


def test_lattice_detection():
    m = build_slab_mesh(SlabSpec((2e-3, 1.5e-3, 1e-3), 0.5e-3))
    assert detect_lattice(m) == (4, 3, 2)
    bare = Mesh(m.nodes, m.elements, m.element_kind, m.material_ids)   # no lattice attribute
    assert detect_lattice(bare) == (4, 3, 2)
    perm = Mesh(m.nodes, m.elements[::-1].copy(), m.element_kind, m.material_ids)
    assert detect_lattice(perm) is None
    t = build_slab_mesh(SlabSpec((2e-3, 1.5e-3, 1e-3), 0.5e-3, ElementKind.TET4))
    assert detect_lattice(t) is None


def test_config4_generator_geometry():
    from paper_2308_01651_b200.ventricle import WALL, prolate_ventricle

    mesh, fib, xi = prolate_ventricle(3, 12, 32)
    assert mesh.num_nodes == 4 * 13 * 32
    assert set(np.unique(mesh.material_ids)) == {1, 2, 3}
    assert mesh.nodes[:, 2].max() == pytest.approx(0.0, abs=1e-12)     # base plane
    np.testing.assert_allclose(np.linalg.norm(fib.f0, axis=1), 1.0)
    np.testing.assert_allclose(np.einsum("ij,ij->i", fib.f0, fib.n0), 0.0, atol=1e-12)
    # helix angle: +60 deg at the endocardium, -60 deg at the epicardium
    # (on the base ring the longitudinal direction is +z, so f0_z = sin(helix))
    eq = np.isclose(mesh.nodes[:, 2], 0.0, atol=1e-12)
    np.testing.assert_allclose(fib.f0[eq & (xi == 0.0), 2], np.sin(np.deg2rad(60.0)))
    np.testing.assert_allclose(fib.f0[eq & (xi == 1.0), 2], np.sin(np.deg2rad(-60.0)))
    # wall thickness at the equator
    r = np.hypot(mesh.nodes[:, 0], mesh.nodes[:, 1])
    assert r[eq].max() - r[eq].min() == pytest.approx(WALL, rel=1e-9)


def test_msh_round_trip_and_reference_reader(tmp_path):
    """write_msh/read_msh (the reference's MSH 2.2 dialect): exact round trip of
    a slab and of a reduced config-4 ventricle; where the reference package
    is importable (build container only) its own reader parses our file to
    the same arrays."""
    import importlib
    import sys

    from paper_2308_01651_b200.geometry import read_msh, write_msh
    from paper_2308_01651_b200.ventricle import prolate_ventricle

    slab = build_slab_mesh(SlabSpec((2e-3, 1.5e-3, 1e-3), 0.5e-3))
    vent, _, _ = prolate_ventricle(2, 8, 16)
    for mesh, name in ((slab, "slab.msh"), (vent, "vent.msh")):
        path = tmp_path / name
        write_msh(mesh, path)
        back = read_msh(path)
        assert back.element_kind is mesh.element_kind
        np.testing.assert_array_equal(back.nodes, mesh.nodes)
        np.testing.assert_array_equal(back.elements, mesh.elements)
        np.testing.assert_array_equal(back.material_ids, mesh.material_ids)
    ref_src = "/root/reference/pkg/src"
    try:
        sys.path.insert(0, ref_src)
        rgeo = importlib.import_module("monodomain.geometry")
    except Exception:
        pytest.skip("reference package not importable here")
    finally:
        if sys.path and sys.path[0] == ref_src:
            sys.path.pop(0)
    for name, mesh in (("slab.msh", slab), ("vent.msh", vent)):
        r = rgeo.import_msh(str(tmp_path / name))
        np.testing.assert_array_equal(np.asarray(r.nodes), mesh.nodes)
        np.testing.assert_array_equal(np.asarray(r.elements), mesh.elements)
        np.testing.assert_array_equal(np.asarray(r.material_ids), mesh.material_ids)


def test_msh_errors(tmp_path):
    from paper_2308_01651_b200.errors import CorruptFile
    from paper_2308_01651_b200.geometry import read_msh

    bad = tmp_path / "bad.msh"
    bad.write_text("$MeshFormat\n4.1 0 8\n$EndMeshFormat\n$Nodes\n0\n$EndNodes\n")
    with pytest.raises(CorruptFile):
        read_msh(bad)
    bad.write_text("$Nodes\n1\n1 0 0 0\n$EndNodes\n$Elements\n1\n1 4 1 1 1 2 3 9\n$EndElements\n")
    with pytest.raises(CorruptFile):
        read_msh(bad)


def _dia_apply_host(op, blk, x):
    """numpy restatement of the MDX_OP_DIASYM row (csrc/solver.cu dia_row)."""
    n, ld = op.n, op.ld
    b = blk.numpy()
    y = b[:n] * x
    for s, d in enumerate(op.pos):
        c = b[(1 + s) * ld:(1 + s) * ld + n]
        y[:n - d] += c[:n - d] * x[d:]          # upper: c_s[i] x[i + d]
        y[d:] += c[:n - d] * x[:n - d]          # lower: c_s[i - d] x[i - d]
    if op.nrem:
        rv = b[(1 + op.np_) * ld:]
        np.add.at(y, op.rem_row.numpy(), rv * x[op.rem_col.numpy()])
    return y


def test_dia_layout_ventricle_seam():
    """DiaOperator.plan/convert on the host (torch CPU tensors): the 7 Kuhn
    offsets of the xi-fastest ventricle numbering become diagonals, the
    periodic ph seam goes to the remainder, and the symmetric apply equals
    the CSR product."""
    import types

    import scipy.sparse as sp
    import torch

    from paper_2308_01651_b200.operators import DiaOperator
    from paper_2308_01651_b200.ventricle import prolate_ventricle

    n_xi, n_th, n_ph = 3, 6, 40
    mesh, _, _ = prolate_ventricle(n_xi, n_th, n_ph)
    n = mesh.num_nodes
    rng = np.random.default_rng(0)
    e = mesh.elements
    rows = np.repeat(e, 4, axis=1).ravel()
    cols = np.tile(e, (1, 4)).ravel()
    A = sp.coo_matrix((rng.uniform(0.1, 1.0, rows.size), (rows, cols)), shape=(n, n)).tocsr()
    A = (A + A.T).tocsr()
    A.sort_indices()
    # locality of the numbering: every non-seam coupling within (n_xi+1)(n_th+2)+1
    coo = A.tocoo()
    off = np.abs(coo.col - coo.row)
    seam = off > (n_xi + 1) * (n_th + 2) + 1
    ph_r = coo.row // ((n_xi + 1) * (n_th + 1))
    ph_c = coo.col // ((n_xi + 1) * (n_th + 1))
    assert np.all(np.abs(ph_r - ph_c)[seam] == n_ph - 1)
    csr = types.SimpleNamespace(
        n=n, nnz=A.nnz, indices=torch.from_numpy(A.indices.astype(np.int32)),
        a_tables={2: torch.from_numpy(A.data.copy())}, d_lift=[], dinv={},
        d_inactive=None, d_rest=None, d_thr=None)
    csr.d_m = csr.a_tables[2]
    plan = DiaOperator.plan(torch.from_numpy(A.indptr.astype(np.int64)), csr.indices, n)
    assert plan is not None
    op = DiaOperator(csr, plan)
    assert op.np_ == 7 and op.nrem > 0 and op.max_rel_dev == 0.0
    x = rng.standard_normal(n)
    np.testing.assert_allclose(_dia_apply_host(op, op.a_tables[2], x), A @ x, rtol=1e-13)
    # remainder rows are the two seam planes only, chunk pointers consistent
    rr = op.rem_row.numpy()
    assert set(rr // ((n_xi + 1) * (n_th + 1))) == {0, n_ph - 1}
    ptr = op.rem_ptr.numpy()
    for c in range(ptr.size - 1):
        assert np.all(rr[ptr[c]:ptr[c + 1]] // 32 == c)
    # sorted by row: the kernels find a row's entries by a lower-bound search
    assert np.all(np.diff(rr) >= 0)
