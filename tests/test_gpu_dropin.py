"""Drop-in checks with the REFERENCE's own objects on the GPU box.

The unmodified reference package travels as `baseline/_ref` (installed by
`__graft_entry__.build()` from /root/reference in the build container; it is
Python + numba, both importable on the box).  Two claims of INTEGRATION.md:

 1. `paper_2308_01651_b200.simulation.TissueSolver` / `run` accept the reference's
    `SimulationConfig` / `VolumeConfig` / `Mesh` / `StimulusProtocol` objects
    unchanged (reference simulation.py:123-218) and reproduce the reference's
    `TissueSolver` run on those same objects.
 2. the kernel-level binding (tests/ref_binding.py = INTEGRATION.md section 2)
    works inside the reference's own `TissueSolver.step` (simulation.py:440-455).
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def refns():
    if not (REF / "monodomain").is_dir():
        pytest.skip("baseline/_ref not installed (run __graft_entry__.build() where "
                    "/root/reference exists)")
    pytest.importorskip("numba")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_mdx")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from paper_2308_01651_b200 import configs

    return configs.reference_namespace()


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


@pytest.mark.parametrize("name,steps", [("cfg0", 120), ("cfg3_h05", 60), ("tet", 60)])
def test_reference_config_objects_run_unchanged(refns, name, steps):
    """Reference-built config objects through the GPU TissueSolver and through the
    reference's TissueSolver: same iterations (+-1), potentials, activation."""
    import monodomain.simulation as ref_sim

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = {"cfg0": lambda: configs.config0(refns),
           "cfg3_h05": lambda: configs.config3(refns, h=0.5e-3),
           "tet": lambda: configs.config0(refns, kind="Tet4")}[name]()
    assert type(cfg).__module__ == "monodomain.simulation"
    assert type(cfg.mesh).__module__ == "monodomain.geometry"
    gpu = TissueSolver(cfg)
    ref = ref_sim.TissueSolver(cfg)
    its_ref = []
    for _ in range(steps):
        u_ref = ref.step()
        its_ref.append(ref.last_iterations)
        u_gpu = gpu.step()
    assert np.abs(gpu.iterations_log() - np.array(its_ref)).max() <= 1
    assert _rel(u_gpu, u_ref) < 1e-9
    assert gpu.last_iterations in (its_ref[-1] - 1, its_ref[-1], its_ref[-1] + 1)
    assert gpu.step_index == ref.step_index and gpu.time == ref.time
    a, b = gpu.activation_map, ref.activation_map
    assert np.array_equal(a >= 0, b >= 0)
    if (b >= 0).any():
        assert np.abs(a[b >= 0] - b[b >= 0]).max() <= cfg.dt * (1 + 1e-9)
    # checkpoints cross both ways (MHEP payload)
    ref2 = ref_sim.TissueSolver(cfg)
    ref2.restore(gpu.checkpoint_payload())
    gpu2 = TissueSolver(cfg)
    gpu2.restore(ref.checkpoint_payload())
    assert _rel(ref2.step(), gpu2.step()) < 1e-9
    # a payload trimmed to the BDF order's levels is still one the reference reads
    ref3 = ref_sim.TissueSolver(cfg)
    ref3.restore(gpu.checkpoint_payload(levels=cfg.bdf_order))
    gpu3 = TissueSolver(cfg)
    gpu3.restore(gpu.checkpoint_payload())
    assert _rel(ref3.step(), gpu3.step()) < 1e-9


def test_reference_run_function_with_reference_config(refns, tmp_path):
    """`run(config)` on a reference SimulationConfig with the reference's
    OutputConfig: same rows, same activation map, same five timing sections."""
    import dataclasses

    import monodomain.simulation as ref_sim
    from monodomain.outputs import OutputConfig

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TIMING_SECTIONS, run

    cfg = configs.config0(refns, h=1e-3, final_time=4e-3)
    out = OutputConfig(enable_csv=True, csv_path=str(tmp_path / "ref.csv"), stride=10,
                               probe_points=((10e-3, 3.5e-3, 1.5e-3), (0.0, 0.0, 0.0)))
    cfg_ref = dataclasses.replace(cfg, output=out)
    cfg_gpu = dataclasses.replace(cfg, output=dataclasses.replace(
        out, csv_path=str(tmp_path / "gpu.csv")))
    rr = ref_sim.run(cfg_ref)
    rg = run(cfg_gpu, timed=True)
    assert rg.steps == rr.steps == 80
    assert _rel(rg.final_potential, rr.final_potential) < 1e-9
    ref_rows = np.loadtxt(tmp_path / "ref.csv", delimiter=",", skiprows=1)
    gpu_rows = np.loadtxt(tmp_path / "gpu.csv", delimiter=",", skiprows=1)
    assert ref_rows.shape == gpu_rows.shape
    np.testing.assert_allclose(gpu_rows, ref_rows, rtol=2e-8, atol=1e-10)   # 9-digit CSV
    assert set(rg.timings) == set(rr.timings) == set(TIMING_SECTIONS)
    for section in ("Ionic model update", "Monodomain assembly", "Linear solver"):
        assert rg.timings[section] > 0.0, section


@pytest.mark.parametrize("model,steps", [("bo", 40), ("ttp06", 25)])
def test_reference_step_with_cabi_advance_kernel(refns, model, steps):
    """The reference's own TissueSolver.step with its numba advance_kernel swapped
    for the C-ABI binding of INTEGRATION.md section 2 (tests/ref_binding.py)."""
    import monodomain.simulation as ref_sim
    from monodomain.ionic import bueno_orovio, ten_tusscher

    import ref_binding
    from paper_2308_01651_b200 import configs

    if model == "bo":
        cfg, mod, mid = configs.config0(refns, h=1e-3), bueno_orovio, 1
    else:
        cfg, mod, mid = configs.config2(refns, h=1e-3), ten_tusscher, 2
    plain = ref_sim.TissueSolver(cfg)
    for _ in range(steps):
        u_plain = plain.step()
    its_plain = plain.last_iterations
    with ref_binding.bound(mod, mid):
        swapped = ref_sim.TissueSolver(cfg)
        for _ in range(steps):
            u_swapped = swapped.step()
    assert mod.advance_kernel.__module__.startswith("monodomain")   # restored
    assert swapped.last_iterations == its_plain
    assert _rel(u_swapped, u_plain) < 1e-10
    np.testing.assert_allclose(swapped.volumes[0].ring[0], plain.volumes[0].ring[0],
                               rtol=1e-9, atol=1e-12)
