"""Ionic membrane models and 0D pacing on the device.

Mirror of `/root/reference/pkg/src/monodomain/ionic/__init__.py`:
`model_module` (`:40-49`), `num_variables`, `to_millivolts` (`:52-60`),
`ion_current` (`:67-85`), `advance_ionic` (`:88-116`) and `pace_single_cell`
(`:119-167`).  `pace_cells` is the batched form of `pace_single_cell`
(config 1: many independent cells, one register-resident device thread per
cell for the whole protocol).
"""

import numpy as np

from .. import _native as N
from ..errors import NonFiniteState
from ..timestepping import HistoryRing, bdf_coefficients
from .base import CellState, CellType, IonicModelSpec, ModelKind, PacingProtocol0D

__all__ = [
    "CellState", "CellType", "IonicModelSpec", "ModelKind", "PacingProtocol0D",
    "advance_ionic", "ion_current", "model_module", "num_variables",
    "pace_single_cell", "pace_cells", "to_millivolts",
]


def model_module(kind):
    from . import aliev_panfilov, bueno_orovio, courtemanche, ten_tusscher

    return {
        ModelKind.ALIEV_PANFILOV: aliev_panfilov,
        ModelKind.BUENO_OROVIO: bueno_orovio,
        ModelKind.TTP06: ten_tusscher,
        ModelKind.CRN_SLOT: courtemanche,
    }[kind]


def num_variables(kind):
    return model_module(kind).NUM_VARS


def to_millivolts(kind, u):
    mod = model_module(kind)
    return mod.MILLIVOLT_GAIN * u + mod.MILLIVOLT_OFFSET


def _check_finite(u, w):
    if not (np.all(np.isfinite(u)) and np.all(np.isfinite(w))):
        raise NonFiniteState("membrane state contains non-finite entries")


def ion_current(spec, u, w):
    """I_ion(u, w) with du/dt = -I_ion + I_app (V/s or 1/s)."""
    mod = model_module(spec.kind)
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (mod.NUM_VARS,):
        raise ValueError(f"{spec.kind.value} expects {mod.NUM_VARS} ionic "
                         f"variables, got shape {w.shape}")
    _check_finite(u, w)
    P = mod.pack(spec.parameters, spec.cell_type)
    out = np.empty(1)
    mod.current_kernel(np.array([float(u)]), w.reshape(1, -1), P, out)
    return float(out[0])


def advance_ionic(spec, u_ext, w_ext, w_history, dt, scheme):
    """One IMEX step of the ionic variables (gates implicit, rest explicit)."""
    mod = model_module(spec.kind)
    w_ext = np.asarray(w_ext, dtype=np.float64)
    w_bdf = w_history.weighted_sum(scheme.history_weights)
    _check_finite(u_ext, w_ext)
    if dt <= 0:
        raise ValueError("dt must be positive")
    P = mod.pack(spec.parameters, spec.cell_type)
    w_out = np.empty((1, mod.NUM_VARS))
    i_out = np.empty(1)
    mod.advance_kernel(np.array([float(u_ext)]), w_ext.reshape(1, -1),
                       w_bdf.reshape(1, -1), scheme.alpha, dt, P, w_out, i_out)
    if not np.all(np.isfinite(w_out)):
        raise NonFiniteState("ionic update produced non-finite values")
    return w_out[0]


GATE_SCHEMES = {"bdf": N.GATES_BDF, "rush_larsen": N.GATES_RUSH_LARSEN}


def gate_scheme_id(name):
    """"bdf" (the reference's IMEX-BDF ionic update) or "rush_larsen" (exponential
    gates + explicit Euler from W_n; BASELINE.json north_star / config 1)."""
    try:
        return GATE_SCHEMES[name]
    except KeyError:
        raise ValueError(f"gate_scheme must be one of {sorted(GATE_SCHEMES)}, got {name!r}")


def pace_cells(spec, protocol, u0, W0, order=2, n_stim_cells=None,
               trace_cells=0, stride=1, return_device=False, gate_scheme="bdf"):
    """Integrate many independent cells under one 0D protocol on the device.

    gate_scheme="rush_larsen" is the one-step mode (order must be 1):
    u+ = u_n + dt (I_app - I_ion(u_n, W+)).

    u0: (n,), W0: (n, nv) host arrays or CUDA tensors (SoA (nv, n) tensors
    are accepted too).  Cells [0, n_stim_cells) receive the protocol's
    pulses (all cells by default).  Returns (u, W (n, nv), peak, clamps,
    trace) with trace shaped (trace_cells, rows, 2+nv) when requested.
    """
    import torch

    mod = model_module(spec.kind)
    if mod.MODEL_ID is None:
        raise NotImplementedError(f"{spec.kind.value} has no kernels")
    nv = mod.NUM_VARS
    bdf_coefficients(order)
    scheme_id = gate_scheme_id(gate_scheme)
    if scheme_id == N.GATES_RUSH_LARSEN and order != 1:
        raise ValueError("Rush-Larsen pacing is a one-step scheme: order must be 1")
    u = torch.as_tensor(np.asarray(u0, dtype=np.float64) if not
                        hasattr(u0, "is_cuda") else u0).to("cuda", torch.float64).contiguous().clone()
    n = u.shape[0]
    W = torch.as_tensor(W0 if hasattr(W0, "is_cuda") else np.asarray(W0, dtype=np.float64))
    W = W.to("cuda", torch.float64)
    if W.shape == (n, nv):
        W = W.t()
    W = W.contiguous().clone()                       # (nv, n) SoA
    if len(protocol.initial_times) > 8:
        raise ValueError("at most 8 pulses per 0D protocol")
    n_steps = int(round(protocol.total_time / protocol.dt))
    peak = torch.empty(n, dtype=torch.float64, device="cuda")
    clamp = torch.zeros(1, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    rows = (n_steps // stride + 1) if trace_cells else 0
    trace = (torch.empty((trace_cells, rows, 2 + nv), dtype=torch.float64,
                         device="cuda") if trace_cells else None)
    a = N.PaceArgs()
    a.n_cells = n
    a.u = N.ptr(u)
    a.W = N.ptr(W)
    a.ldw = n
    a.peak = N.ptr(peak)
    a.order = order
    a.n_pulses = len(protocol.initial_times)
    a.n_steps = n_steps
    a.dt = protocol.dt
    a.n_stim_cells = n if n_stim_cells is None else int(n_stim_cells)
    a.period = protocol.period
    for k, (t0, d, amp) in enumerate(zip(protocol.initial_times,
                                         protocol.durations,
                                         protocol.amplitudes)):
        a.pulse_t0[k], a.pulse_dur[k], a.pulse_amp[k] = t0, d, amp
    a.n_trace_cells = trace_cells
    a.trace_rows = rows
    a.stride = stride
    a.trace = N.ptr(trace)
    a.clamp_count = N.ptr(clamp)
    a.status = N.ptr(status)
    a.gate_scheme = scheme_id
    P = mod.pack(spec.parameters, spec.cell_type)
    Ph, Pp = N.host_doubles(P)
    N.check(N.lib().mdx_pace_cells(mod.MODEL_ID, N.C.byref(a), Pp, int(Ph.size),
                                   N.stream_handle()), "mdx_pace_cells")
    if int(status.item()):
        raise NonFiniteState("0D integration lost finiteness")
    if return_device:
        return u, W, peak, int(clamp.item()), trace
    tr = trace.cpu().numpy() if trace is not None else None
    return (u.cpu().numpy(), W.t().contiguous().cpu().numpy(),
            peak.cpu().numpy(), int(clamp.item()), tr)


def pace_single_cell(spec, protocol, order=2, stride=1, gate_scheme="bdf"):
    """0D integration of one cell; returns (CellState, trace rows (t,u,w..))."""
    state = spec.initial_state
    u, W, _, _, trace = pace_cells(
        spec, protocol, np.array([float(state.u)]),
        state.w.reshape(1, -1), order=order, trace_cells=1, stride=stride,
        gate_scheme=gate_scheme)
    return CellState(float(u[0]), W[0].copy()), trace[0]
