"""Config 4 geometry: truncated prolate-spheroid ventricle, P1 tets, helix fibers.

BASELINE.json configs[4]; the reference has no generator for it (SURVEY.md
D8), so this module builds one and the reference is fed the same arrays
(through its own `Mesh`/`FiberField` types) for the reduced-size parity run.

Geometry: nested prolate spheroids x = a(xi) sin(th) cos(ph),
y = a(xi) sin(th) sin(ph), z = -c(xi) cos(th) with a = a_in + wall*xi,
c = c_in + wall*xi, xi in [0, 1] (endocardium -> epicardium), th from a small
apical angle (a ~1 mm apical opening keeps every element non-degenerate)
to pi/2 (the base plane z = 0), ph periodic.  The logical (ph, th, xi) grid
is split into tets with the Kuhn six-tet rule (conforming across cells).

Fibers: helix angle +60 deg (endo) to -60 deg (epi), linear in xi, measured
from the circumferential direction towards the apex-to-base direction in the
wall's tangent plane; n0 = transmural normal, s0 = n0 x f0 (as
`slab_fiber_field`, geometry.py:299-331).  Cell types: element centroid
depth xi in thirds -> materials 1 (endo), 2 (mid), 3 (epi).
"""

import numpy as np

from .geometry import ElementKind, FiberField, KUHN_TETS, Mesh, tet_volumes6

INNER_A, INNER_C, WALL = 25e-3, 45e-3, 10e-3


def _coords(xi, th, ph):
    a = INNER_A + WALL * xi
    c = INNER_C + WALL * xi
    return np.stack([a * np.sin(th) * np.cos(ph), a * np.sin(th) * np.sin(ph),
                     -c * np.cos(th)], axis=-1)


def prolate_ventricle(n_xi, n_th, n_ph, apex_opening=1e-3):
    """(mesh, fibers, xi_of_node) for an n_xi x n_th x n_ph logical grid.

    Nodes are numbered xi fastest, then th, then ph (node (i_xi, i_th, i_ph) =
    i_xi + (n_xi+1) (i_th + (n_th+1) i_ph)), cells likewise: every coupling
    of a node then sits within (n_xi+1)(n_th+2) + 1 indices of it except
    across the periodic ph seam, which keeps the vectors an operator apply
    gathers inside a window of a few MB (L2-resident at 10 M nodes).
    """
    th0 = np.arcsin(apex_opening / INNER_A)
    xi = np.linspace(0.0, 1.0, n_xi + 1)
    th = np.linspace(th0, np.pi / 2, n_th + 1)
    ph = np.arange(n_ph) * (2 * np.pi / n_ph)
    PH, TH, XI = np.meshgrid(ph, th, xi, indexing="ij")        # node (i_ph, i_th, i_xi)
    nodes = _coords(XI, TH, PH).reshape(-1, 3)
    nx1, nt1 = n_xi + 1, n_th + 1

    def nid(i_xi, i_th, i_ph):
        return i_xi + nx1 * (i_th + nt1 * (i_ph % n_ph))

    cp, ct, cx = np.meshgrid(np.arange(n_ph, dtype=np.int64), np.arange(n_th, dtype=np.int64),
                             np.arange(n_xi, dtype=np.int64), indexing="ij")
    cx, ct, cp = cx.ravel(), ct.ravel(), cp.ravel()
    # Kuhn corner q = a + 2b + 4c with offsets (ph: a, th: b, xi: c)
    corner = np.column_stack([nid(cx + ((q >> 2) & 1), ct + ((q >> 1) & 1), cp + (q & 1))
                              for q in range(8)]).astype(np.int32)
    del cx, ct, cp
    tets = np.stack([corner[:, list(t)] for t in KUHN_TETS], axis=1).reshape(-1, 4)
    del corner
    # orient every tet positively
    flip = np.flatnonzero(tet_volumes6(nodes, tets) < 0)
    tets[flip, 1], tets[flip, 2] = tets[flip, 2].copy(), tets[flip, 1].copy()
    # material by centroid depth: the four corners' xi indices
    xi_idx = (tets % nx1).sum(axis=1)                       # 4 * centroid_xi * n_xi
    cxi = xi_idx / (4.0 * n_xi)
    mats = np.where(cxi < 1.0 / 3.0, 1, np.where(cxi < 2.0 / 3.0, 2, 3)).astype(np.int32)
    mesh = Mesh(nodes, tets, ElementKind.TET4, mats,
                grid=((nx1, nt1, n_ph), (False, False, True)))

    # fiber frame from the analytic tangents
    a = INNER_A + WALL * XI
    c = INNER_C + WALL * XI
    e_c = np.stack([-np.sin(PH), np.cos(PH), np.zeros_like(PH)], axis=-1)
    e_l = np.stack([a * np.cos(TH) * np.cos(PH), a * np.cos(TH) * np.sin(PH),
                    c * np.sin(TH)], axis=-1)
    e_l /= np.linalg.norm(e_l, axis=-1, keepdims=True)
    e_t = np.cross(e_l, e_c)                       # outward normal of the wall
    e_t /= np.linalg.norm(e_t, axis=-1, keepdims=True)
    helix = np.deg2rad(60.0 - 120.0 * XI)[..., None]
    f0 = np.cos(helix) * e_c + np.sin(helix) * e_l
    f0 /= np.linalg.norm(f0, axis=-1, keepdims=True)
    n0 = e_t
    s0 = np.cross(n0, f0)
    fibers = FiberField(f0.reshape(-1, 3), s0.reshape(-1, 3), n0.reshape(-1, 3))
    return mesh.validate(), fibers.validate(), XI.reshape(-1)


def apex_point():
    """Endocardial apex (centre of the apical stimulus sphere)."""
    return (0.0, 0.0, -INNER_C)


def size_for_nodes(target):
    """Logical grid (n_xi, n_th, n_ph) with ~target nodes and ~isotropic cells."""
    n_xi = max(2, int(round((target / 156.0) ** (1.0 / 3.0))))
    n_th = 6 * n_xi
    n_ph = 26 * n_xi
    return n_xi, n_th, n_ph


def config4(ns, n_xi=40, n_th=240, n_ph=1040, dt=2e-5, final_time=200e-3):
    """Config 4 as a SimulationConfig of namespace `ns` (ours or the reference's)."""
    from . import configs

    mesh, fibers, _ = prolate_ventricle(n_xi, n_th, n_ph)
    if ns.Mesh is not Mesh:
        mesh = ns.Mesh(mesh.nodes, mesh.elements, ns.ElementKind("Tet4"), mesh.material_ids)
        fibers = ns.FiberField(fibers.f0, fibers.s0, fibers.n0)
    sl, st, sn = configs.SIGMA
    CT = ns.CellType
    vols = tuple(
        ns.VolumeConfig(label, (mat,), ns.IonicModelSpec(ns.ModelKind.TTP06, cell_type=ct),
                        sigma_l=sl, sigma_t=st, sigma_n=sn)
        for label, mat, ct in (("Endocardium", 1, CT.ENDOCARDIUM),
                               ("Midmyocardium", 2, CT.MYOCARDIUM),
                               ("Epicardium", 3, CT.EPICARDIUM)))
    stim = ns.StimulusProtocol(ns.StimulusShape.SPHERICAL, (apex_point(),),
                               (configs.TTP_AMPLITUDE,), (3e-3,), (0.0,), (2e-3,))
    return ns.SimulationConfig(
        mesh=mesh, fibers=fibers, volumes=vols, bdf_order=2, dt=dt, final_time=final_time,
        stimuli=(stim,), membrane_capacitance=configs.CM, chi_m=configs.CHI,
        linear_solver=ns.LinearSolverConfig(1e-10, 2000),
        activation=ns.ActivationConfig(threshold=0.0))
