"""CUDA ionic kernels vs the reference's golden vectors and the CPU oracle.

Tolerances: the device evaluates exp/log/tanh with CUDA's fp64 libm
(<= 2 ulp) and contracts a*b+c into FMAs, so results differ from the
reference's numba/glibc values at the 1e-15..1e-12 relative level; clamp
counts must match exactly.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODELS = {"ttp06": "ten_tusscher", "bo": "bueno_orovio", "apf": "aliev_panfilov"}


def _module(tag):
    import importlib

    return importlib.import_module(
        f"paper_2308_01651_b200.ionic.{MODELS[tag.split('_')[0]]}")


def _cases(g, model):
    for key in g:
        if key.endswith("_Wout") and key.startswith(model + "_"):
            tag = key[: -len("_Wout")]
            mt = tag.split("_a")[0]
            rest = tag[len(mt) + 2:]
            yield tag, mt, float(rest.split("_dt")[0]), float(rest.split("_dt")[1])


@pytest.mark.parametrize("model", ["ttp06", "bo", "apf"])
@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_advance_kernel_matches_reference(golden, model, layout):
    import torch

    g = golden("ionic_kat")
    n_cases = 0
    for tag, mt, alpha, dt in _cases(g, model):
        mod = _module(mt)
        u, We, Wb, P = g[f"{mt}_u"], g[f"{mt}_Wext"], g[f"{mt}_Wbdf"], g[f"{mt}_P"]
        if layout == "aos":
            Wo = np.empty_like(We)
            Io = np.empty(u.size)
            c = mod.advance_kernel(u, We, Wb, alpha, dt, P, Wo, Io)
        else:   # SoA device tensors: (nv, n) storage viewed as (n, nv)
            def soa(a):
                return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()

            wo_d = torch.empty((We.shape[1], u.size), dtype=torch.float64,
                               device="cuda").t()
            io_d = torch.empty(u.size, dtype=torch.float64, device="cuda")
            c = mod.advance_kernel(torch.from_numpy(u).cuda(), soa(We), soa(Wb), alpha,
                                   dt, P, wo_d, io_d)
            Wo, Io = wo_d.cpu().numpy(), io_d.cpu().numpy()
        np.testing.assert_allclose(Wo, g[f"{tag}_Wout"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(Io, g[f"{tag}_Iout"], rtol=1e-9, atol=1e-10)
        assert c == int(g[f"{tag}_clamped"]), tag
        n_cases += 1
    assert n_cases >= 4


def test_current_kernel_and_rest_kat(golden):
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, ion_current

    g = golden("ionic_kat")
    for mt in ("ttp06_epi", "ttp06_endo", "ttp06_myo", "bo_-", "apf_-"):
        mod = _module(mt)
        Io = np.empty(g[f"{mt}_u"].size)
        mod.current_kernel(g[f"{mt}_u"], g[f"{mt}_Wext"], g[f"{mt}_P"], Io)
        np.testing.assert_allclose(Io, g[f"{mt}_current"], rtol=1e-10, atol=1e-11)
    spec = IonicModelSpec(ModelKind.TTP06)
    rest = ion_current(spec, spec.initial_state.u, spec.initial_state.w)
    assert rest == pytest.approx(0.0017519776588273556, rel=1e-12)  # test_ionic.py:119


def test_point_rates(golden):
    g = golden("ionic_kat")
    for mt in ("ttp06_epi", "bo_-", "apf_-"):
        mod = _module(mt)
        for k in range(8):
            I, dw = mod.point_rates(g[f"{mt}_u"][k], g[f"{mt}_Wext"][k], g[f"{mt}_P"])
            assert I == pytest.approx(g[f"{mt}_rates_I"][k], rel=1e-10, abs=1e-11)
            np.testing.assert_allclose(dw, g[f"{mt}_rates_dw"][k], rtol=1e-10,
                                       atol=1e-11)


def test_gates_read_history_not_extrapolation():
    """tests/test_ionic.py:169-182 semantics, including the fCass quirk: the
    fCass target reads CaSS from w_ext, so exactly one gate moves too."""
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, advance_ionic, model_module
    from paper_2308_01651_b200.timestepping import HistoryRing, bdf_coefficients

    spec = IonicModelSpec(ModelKind.TTP06)
    mod = model_module(ModelKind.TTP06)
    rest = spec.initial_state.w
    ring = HistoryRing()
    ring.push(rest)
    ring.push(rest * 1.0001)
    s = bdf_coefficients(2)
    base = advance_ionic(spec, -0.02, rest, ring, 2.5e-5, s)
    pert = advance_ionic(spec, -0.02, rest * 1.01, ring, 2.5e-5, s)
    gates = np.array(mod.GATES)
    changed = np.flatnonzero(base[gates] != pert[gates])
    assert changed.tolist() == [11]          # fCass only
    assert not np.array_equal(base[~gates], pert[~gates])


def test_gate_clamping_counts():
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, model_module

    mod = model_module(ModelKind.BUENO_OROVIO)
    P = mod.pack(IonicModelSpec(ModelKind.BUENO_OROVIO).parameters)
    w = np.array([[1.8, -0.5, 0.3]])
    wo = np.empty((1, 3))
    io = np.empty(1)
    c = mod.advance_kernel(np.array([0.4]), w.copy(), w * 3.0, 1.0, 5.0, P, wo, io)
    assert c > 0 and (wo >= 0).all() and (wo <= 1).all()


def test_pace_single_cell_traces(golden):
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, PacingProtocol0D, pace_single_cell

    g = golden("pace0d")
    apf = PacingProtocol0D((0.0,), (4e-3,), (1.1628e3,), 0.8, 0.8, 2.5e-5)
    _, tr = pace_single_cell(IonicModelSpec(ModelKind.ALIEV_PANFILOV), apf, order=2,
                             stride=40)
    np.testing.assert_allclose(tr, g["apf_trace"], rtol=1e-9, atol=1e-12)
    _, full = pace_single_cell(IonicModelSpec(ModelKind.ALIEV_PANFILOV), apf, order=2)
    assert full[:, 1].max() == pytest.approx(1.6735286, rel=1e-6)  # test_ionic.py:348
    bo = PacingProtocol0D((0.0,), (4e-3,), (1.1628e3,), 0.8, 0.4, 5e-5)
    for order in (1, 2, 3):
        _, tr = pace_single_cell(IonicModelSpec(ModelKind.BUENO_OROVIO), bo,
                                 order=order, stride=20)
        ref = g[f"bo_trace_o{order}"]
        rel = np.linalg.norm(tr[:, 1] - ref[:, 1]) / np.linalg.norm(ref[:, 1])
        assert rel < 1e-9
    ttp = PacingProtocol0D((0.0,), (2e-3,), (35.714,), 0.0, 0.05, 2.5e-5)
    for order in (1, 2):
        _, tr = pace_single_cell(IonicModelSpec(ModelKind.TTP06), ttp, order=order,
                                 stride=40)
        ref = g[f"ttp_trace_o{order}"]
        rel = np.linalg.norm(tr[:, 1] - ref[:, 1]) / np.linalg.norm(ref[:, 1])
        assert rel < 1e-9, rel


def test_phenomenological_rest_exact():
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, PacingProtocol0D, pace_single_cell

    for kind in (ModelKind.ALIEV_PANFILOV, ModelKind.BUENO_OROVIO):
        _, tr = pace_single_cell(IonicModelSpec(kind),
                                 PacingProtocol0D((), (), (), 0.0, 1.0, 1e-3), stride=50)
        assert np.abs(tr[:, 1]).max() == 0.0


def test_cfg1_batch_vs_reference_and_oracle(golden):
    """Config 1 (0D TTP06 batch) parity subset: reference golden + live oracle."""
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, PacingProtocol0D, pace_cells

    g = golden("cfg1_subset")
    spec = IonicModelSpec(ModelKind.TTP06)
    proto = PacingProtocol0D((0.0,), (1e-3,), (52.0,), 0.0, 2000 * 1e-5, 1e-5)
    for order in (1, 2):
        u, W, peak, clamps, _ = pace_cells(spec, proto, g["u0"], g["W0"], order=order,
                                           n_stim_cells=int(g["n_stim"]))
        np.testing.assert_allclose(u, g[f"o{order}_u"], rtol=1e-7, atol=1e-9)
        np.testing.assert_allclose(peak, g[f"o{order}_peak"], rtol=1e-7, atol=1e-9)
        np.testing.assert_allclose(W, g[f"o{order}_W"], rtol=1e-6, atol=1e-12)
        assert clamps == int(g[f"o{order}_clamps"])
    # a second seeded subset checked live against the oracle
    u0, W0 = configs.config1_initial(256, seed=99)
    P = spec and __import__("paper_2308_01651_b200.ionic.ten_tusscher",
                            fromlist=["pack"]).pack(spec.parameters)
    proto = PacingProtocol0D((0.0,), (1e-3,), (52.0,), 0.0, 300 * 1e-5, 1e-5)
    u, W, peak, _, _ = pace_cells(spec, proto, u0, W0, order=2, n_stim_cells=3)
    ur, Wr, pr, _ = O.pace_batch("TTP06", P, u0, W0, 1e-5, 300, 2, 3, 52.0, 1e-3)
    np.testing.assert_allclose(u, ur, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(peak, pr, rtol=1e-9, atol=1e-12)


# ---------------------------------------------------------------------------
# Rush-Larsen mode (gate_scheme="rush_larsen"; north_star / config 1).  Fixtures:
# the reference's own gate/current/rate functions under the RL integrator
# (tests/golden/make_golden.py: rl_kat).
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("tag", ["ttp06_epi", "ttp06_endo", "ttp06_myo", "bo_-", "apf_-"])
@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_rush_larsen_kernel_matches_reference_functions(golden, tag, layout):
    import torch

    g, kat = golden("rl_kat"), golden("ionic_kat")
    mod = _module(tag)
    u, P, Wn = kat[f"{tag}_u"], kat[f"{tag}_P"], g[f"{tag}_Wn"]
    seen = 0
    for key in g:
        if not (key.startswith(f"{tag}_dt") and key.endswith("_Wout")):
            continue
        dt = float(key[len(tag) + 3: -len("_Wout")])
        if layout == "aos":
            Wo, Io = np.empty_like(Wn), np.empty(u.size)
            c = mod.rush_larsen_kernel(u, Wn, dt, P, Wo, Io)
        else:
            wn_d = torch.from_numpy(np.ascontiguousarray(Wn.T)).cuda().t()
            wo_d = torch.empty((Wn.shape[1], u.size), dtype=torch.float64, device="cuda").t()
            io_d = torch.empty(u.size, dtype=torch.float64, device="cuda")
            c = mod.rush_larsen_kernel(torch.from_numpy(u).cuda(), wn_d, dt, P, wo_d, io_d)
            Wo, Io = wo_d.cpu().numpy(), io_d.cpu().numpy()
        np.testing.assert_allclose(Wo, g[f"{tag}_dt{dt:g}_Wout"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(Io, g[f"{tag}_dt{dt:g}_Iout"], rtol=1e-9, atol=1e-10)
        assert c == int(g[f"{tag}_dt{dt:g}_clamped"])
        seen += 1
    assert seen == 2


def test_rush_larsen_cfg1_subset_and_traces(golden):
    """Config 1 as BASELINE words it (Rush-Larsen on gates): the 512-cell subset and
    the 0D traces of the reference's pace_single_cell with the RL integrator."""
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.ionic import (IonicModelSpec, ModelKind, PacingProtocol0D,
                                             pace_cells, pace_single_cell)

    g = golden("rl_kat")
    u0, W0 = configs.config1_initial(512)
    spec = IonicModelSpec(ModelKind.TTP06)
    proto = PacingProtocol0D((0.0,), (1e-3,), (52.0,), 0.0, 2000 * 1e-5, 1e-5)
    u, W, peak, clamps, _ = pace_cells(spec, proto, u0, W0, order=1,
                                       n_stim_cells=int(g["cfg1_n_stim"]),
                                       gate_scheme="rush_larsen")
    np.testing.assert_allclose(u, g["cfg1_u"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(peak, g["cfg1_peak"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(W, g["cfg1_W"], rtol=1e-6, atol=1e-12)
    assert clamps == int(g["cfg1_clamps"])
    with pytest.raises(ValueError):
        pace_cells(spec, proto, u0, W0, order=2, gate_scheme="rush_larsen")
    with pytest.raises(ValueError):
        pace_cells(spec, proto, u0, W0, order=1, gate_scheme="euler")
    ttp = PacingProtocol0D((0.0,), (2e-3,), (35.714,), 0.0, 0.05, 2.5e-5)
    _, tr = pace_single_cell(spec, ttp, order=1, stride=40, gate_scheme="rush_larsen")
    ref = g["ttp_trace"]
    assert np.linalg.norm(tr[:, 1] - ref[:, 1]) / np.linalg.norm(ref[:, 1]) < 1e-9
    bo = PacingProtocol0D((0.0,), (4e-3,), (1.1628e3,), 0.8, 0.4, 5e-5)
    _, tr = pace_single_cell(IonicModelSpec(ModelKind.BUENO_OROVIO), bo, order=1, stride=20,
                             gate_scheme="rush_larsen")
    ref = g["bo_trace"]
    assert np.linalg.norm(tr[:, 1] - ref[:, 1]) / np.linalg.norm(ref[:, 1]) < 1e-9


def test_empty_and_ragged_inputs_through_the_abi():
    """Edge cases at the C-ABI: zero-length batches are no-ops that return MDX_OK
    (the reference's prange kernels accept empty arrays), a batch that is not a
    multiple of the block or warp size is handled to the last cell, a wrong
    parameter count is refused with a message, and a non-finite state is reported."""
    import torch

    from paper_2308_01651_b200 import _native as N
    from paper_2308_01651_b200.errors import NonFiniteState
    from paper_2308_01651_b200.ionic import (IonicModelSpec, ModelKind, PacingProtocol0D,
                                             pace_cells, ten_tusscher as T)

    lib = N.lib()
    spec = IonicModelSpec(ModelKind.TTP06)
    P = T.pack(spec.parameters)
    Ph, Pp = N.host_doubles(P)
    st = N.stream_handle()
    assert lib.mdx_ionic_advance(N.MODEL_TTP06, 0, None, None, None, 18, 1, 1.0, 1e-5, Pp,
                                 int(Ph.size), None, None, None, st) == 0
    assert lib.mdx_ionic_advance_rl(N.MODEL_TTP06, 0, None, None, 18, 1, 1e-5, Pp, int(Ph.size),
                                    None, None, None, st) == 0
    assert lib.mdx_ionic_current(N.MODEL_TTP06, 0, None, None, 18, 1, Pp, int(Ph.size), None,
                                 st) == 0
    assert lib.mdx_record_row(None, 0, None, 0, None, None, st) == 0
    # wrong packed-parameter length: refused, with the reason in mdx_last_error
    assert lib.mdx_ionic_advance(N.MODEL_TTP06, 1, None, None, None, 18, 1, 1.0, 1e-5, Pp, 7,
                                 None, None, None, st) != 0
    assert b"50" in lib.mdx_last_error()
    assert lib.mdx_ionic_advance(99, 1, None, None, None, 18, 1, 1.0, 1e-5, Pp, int(Ph.size),
                                 None, None, None, st) != 0
    # ragged batch sizes: every cell equals the single-cell result
    st0 = spec.initial_state
    proto = PacingProtocol0D((0.0,), (1e-3,), (52.0,), 0.0, 50e-5, 1e-5)
    for n in (1, 31, 33, 129, 1000):
        u0 = np.full(n, st0.u)
        W0 = np.tile(st0.w, (n, 1))
        u, W, peak, _, _ = pace_cells(spec, proto, u0, W0, order=2)
        assert u.shape == (n,) and W.shape == (n, 18)
        assert np.all(u == u[0]) and np.all(W == W[0])
    u, W, _, _, _ = pace_cells(spec, proto, np.empty(0), np.empty((0, 18)), order=2)
    assert u.size == 0 and W.shape == (0, 18)
    bad = np.tile(st0.w, (4, 1))
    bad[2, 12] = np.nan                      # Cai of one cell
    with pytest.raises(NonFiniteState):
        pace_cells(spec, proto, np.full(4, st0.u), bad, order=2)
    torch.cuda.synchronize()
