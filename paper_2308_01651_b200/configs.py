"""Builders for the BASELINE.json configurations.

Each builder takes a namespace `ns` exposing the reference's type names
(SlabSpec, build_slab_mesh, slab_fiber_field, ElementKind, Mesh,
VolumeConfig, IonicModelSpec, ModelKind, StimulusProtocol, StimulusShape,
SimulationConfig, LinearSolverConfig, ActivationConfig, nearest_node).
`this_package()` gives ours; the golden-fixture script passes the
reference's, so both solvers see identical inputs (SURVEY.md §8(d),
Appendix B).

* cfg 0: BO slab 20x7x3 mm, h=0.5 mm, dt=5e-5 s, 40 ms (800 steps).
* cfg 2: TTP06 slab, h=0.1 mm (442,401 nodes), dt=2e-5 s, 100 ms.
* cfg 3: cfg-2 slab + seeded ellipsoidal scar (sigma x0.01) and 1 mm border
  zone (GNa x0.38, GCaL x0.31, Gkr x0.3), second stimulus at t=0.3 s, 500 ms.
* ladder: the reference N-version benchmark slab (benchmark.py:67-101).

Stimulus amplitudes follow SURVEY.md D6: BO amplitude 0.5 A/m^2 / 0.0857 V
in model units with C_m = 1e-2 F/m^2, chi = 1.4e5 1/m; TTP06 0.5 A/m^2.
Activation thresholds are the 0 mV equivalents (D5).
"""

import types

import numpy as np

SLAB = (20e-3, 7e-3, 3e-3)
SIGMA = (0.17, 0.019, 0.019)
CHI = 1.4e5
CM = 1e-2
STIM_SITE = (0.75e-3, 0.75e-3, 0.75e-3)
STIM_EDGE = 1.5e-3
BO_AMPLITUDE = 0.5 / 85.7e-3
TTP_AMPLITUDE = 0.5


def this_package():
    from . import geometry, simulation
    from .ionic import IonicModelSpec, ModelKind, CellType

    ns = types.SimpleNamespace()
    for mod in (geometry, simulation):
        for k in dir(mod):
            if not k.startswith("_"):
                setattr(ns, k, getattr(mod, k))
    ns.IonicModelSpec, ns.ModelKind, ns.CellType = IonicModelSpec, ModelKind, CellType
    return ns


def reference_namespace():
    """The reference package's types (importable in the build container only)."""
    import monodomain.geometry as g
    import monodomain.simulation as s
    from monodomain.ionic import CellType, IonicModelSpec, ModelKind

    ns = types.SimpleNamespace()
    for mod in (g, s):
        for k in dir(mod):
            if not k.startswith("_"):
                setattr(ns, k, getattr(mod, k))
    ns.IonicModelSpec, ns.ModelKind, ns.CellType = IonicModelSpec, ModelKind, CellType
    return ns


def corner_probes(extent=SLAB):
    return [(x, y, z) for z in (0.0, extent[2]) for y in (0.0, extent[1])
            for x in (0.0, extent[0])]


def _slab(ns, h, kind="Hex8"):
    mesh = ns.build_slab_mesh(ns.SlabSpec(SLAB, h, ns.ElementKind(kind)))
    fibers = ns.slab_fiber_field(mesh, 2, 0.0, 0.0)   # f0 = x (D4)
    return mesh, fibers


def config0(ns, h=0.5e-3, final_time=40e-3, dt=5e-5, kind="Hex8"):
    mesh, fibers = _slab(ns, h, kind)
    vol = ns.VolumeConfig("Volumetric parameters", (1,),
                          ns.IonicModelSpec(ns.ModelKind.BUENO_OROVIO),
                          sigma_l=SIGMA[0], sigma_t=SIGMA[1], sigma_n=SIGMA[2])
    stim = ns.StimulusProtocol(ns.StimulusShape.CUBIC, (STIM_SITE,), (BO_AMPLITUDE,),
                               (STIM_EDGE,), (0.0,), (2e-3,))
    return ns.SimulationConfig(
        mesh=mesh, fibers=fibers, volumes=(vol,), bdf_order=2, dt=dt,
        final_time=final_time, stimuli=(stim,), membrane_capacitance=CM, chi_m=CHI,
        linear_solver=ns.LinearSolverConfig(1e-10, 2000),
        activation=ns.ActivationConfig(threshold=84.0 / 85.7))


def config2(ns, h=0.1e-3, final_time=100e-3, dt=2e-5, kind="Hex8"):
    mesh, fibers = _slab(ns, h, kind)
    vol = ns.VolumeConfig("Volumetric parameters", (1,),
                          ns.IonicModelSpec(ns.ModelKind.TTP06),
                          sigma_l=SIGMA[0], sigma_t=SIGMA[1], sigma_n=SIGMA[2])
    stim = ns.StimulusProtocol(ns.StimulusShape.CUBIC, (STIM_SITE,), (TTP_AMPLITUDE,),
                               (STIM_EDGE,), (0.0,), (2e-3,))
    return ns.SimulationConfig(
        mesh=mesh, fibers=fibers, volumes=(vol,), bdf_order=2, dt=dt,
        final_time=final_time, stimuli=(stim,), membrane_capacitance=CM, chi_m=CHI,
        linear_solver=ns.LinearSolverConfig(1e-10, 2000),
        activation=ns.ActivationConfig(threshold=0.0))


def scar_materials(mesh, seed=1234, extent=SLAB, border=1e-3):
    """Per-element material IDs: 1 healthy, 2 scar, 3 border zone."""
    rng = np.random.default_rng(seed)
    semi = rng.uniform(2e-3, 4e-3, 3)
    centre = rng.uniform(np.zeros(3), np.asarray(extent))
    cent = mesh.nodes[mesh.elements].mean(axis=1)
    r_scar = (((cent - centre) / semi) ** 2).sum(axis=1)
    r_bz = (((cent - centre) / (semi + border)) ** 2).sum(axis=1)
    mats = np.ones(mesh.elements.shape[0], dtype=np.int32)
    mats[r_bz <= 1.0] = 3
    mats[r_scar <= 1.0] = 2
    return mats


def config3(ns, h=0.1e-3, final_time=500e-3, dt=2e-5, seed=1234, kind="Hex8"):
    mesh, fibers = _slab(ns, h, kind)
    mats = scar_materials(mesh, seed)
    mesh = ns.Mesh(mesh.nodes, mesh.elements, mesh.element_kind, mats)
    sl, st, sn = SIGMA
    healthy = ns.VolumeConfig("Healthy", (1,), ns.IonicModelSpec(ns.ModelKind.TTP06),
                              sigma_l=sl, sigma_t=st, sigma_n=sn)
    scar = ns.VolumeConfig("Scar", (2,), ns.IonicModelSpec(ns.ModelKind.TTP06),
                           sigma_l=sl * 0.01, sigma_t=st * 0.01, sigma_n=sn * 0.01)
    base = ns.IonicModelSpec(ns.ModelKind.TTP06).parameters
    bz_spec = ns.IonicModelSpec(ns.ModelKind.TTP06, parameters={
        "GNa": base["GNa"] * 0.38, "GCaL": base["GCaL"] * 0.31,
        "Gkr": base["Gkr"] * 0.3})
    border = ns.VolumeConfig("Border Zone", (3,), bz_spec, sigma_l=sl, sigma_t=st,
                             sigma_n=sn)
    far = tuple(e - c for e, c in zip(SLAB, STIM_SITE))
    stim = ns.StimulusProtocol(ns.StimulusShape.CUBIC, (STIM_SITE, far),
                               (TTP_AMPLITUDE, TTP_AMPLITUDE), (STIM_EDGE, STIM_EDGE),
                               (0.0, 0.3), (2e-3, 2e-3))
    vols = tuple(v for v, m in ((healthy, 1), (scar, 2), (border, 3))
                 if (mats == m).any())
    return ns.SimulationConfig(
        mesh=mesh, fibers=fibers, volumes=vols, bdf_order=2, dt=dt,
        final_time=final_time, stimuli=(stim,), membrane_capacitance=CM, chi_m=CHI,
        linear_solver=ns.LinearSolverConfig(1e-10, 2000),
        activation=ns.ActivationConfig(threshold=0.0))


def ladder_config(ns, dx_mm, dt_ms, kind="Hex8", final_time=150e-3):
    """The reference benchmark slab (benchmark.py:67-101)."""
    mesh = ns.build_slab_mesh(ns.SlabSpec((3e-3, 7e-3, 20e-3), dx_mm * 1e-3,
                                          ns.ElementKind(kind)))
    fibers = ns.slab_fiber_field(mesh, 0, 0.0, 0.0)
    vol = ns.VolumeConfig("Volumetric parameters", (1,),
                          ns.IonicModelSpec(ns.ModelKind.TTP06),
                          sigma_l=0.95298e-4, sigma_t=0.12576e-4, sigma_n=0.12576e-4)
    stim = ns.StimulusProtocol(ns.StimulusShape.CUBIC, (STIM_SITE,), (35.714,),
                               (STIM_EDGE,), (0.0,), (2e-3,))
    return ns.SimulationConfig(mesh=mesh, fibers=fibers, volumes=(vol,), bdf_order=2,
                               dt=dt_ms * 1e-3, final_time=final_time, stimuli=(stim,))


def config1_initial(n_cells, seed=20261019):
    """Config 1: TTP06 epicardial rest state x (1 + 0.01 N(0,1)), seeded."""
    from .ionic import ten_tusscher

    st = ten_tusscher.default_initial_state()
    x0 = np.concatenate([[st.u], st.w])
    rng = np.random.default_rng(seed)
    x = x0[None, :] * (1.0 + 0.01 * rng.standard_normal((n_cells, x0.size)))
    return x[:, 0].copy(), np.ascontiguousarray(x[:, 1:])
