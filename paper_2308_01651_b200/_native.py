"""ctypes binding of `include/mdx.h` (the C-ABI of libmdx.so).

This module is the only place that knows the struct layouts; everything else
passes torch CUDA tensors and lets the helpers here turn them into device
pointers.  There is no CPU fallback: `lib()` raises `NativeUnavailable` when
the shared library is missing or no CUDA device is visible.
"""

import ctypes as C
from pathlib import Path

import numpy as np

from .errors import NativeUnavailable

import os

_LIB_PATH = Path(os.environ.get("MDX_LIB", Path(__file__).resolve().parent / "libmdx.so"))
_lib = None

MDX_OK = 0
MODEL_ALIEV_PANFILOV = 0
MODEL_BUENO_OROVIO = 1
MODEL_TTP06 = 2
OP_STENCIL27 = 1
OP_CSR = 2
OP_SELL = 3
OP_DIASYM = 4
DIA_MAX = 16
ROW_SCRATCH = 1024        # MDX_ROW_SCRATCH
MAX_LIFT = 8
ABI_VERSION = 5   # include/mdx.h MDX_ABI_VERSION
GATES_BDF, GATES_RUSH_LARSEN = 0, 1   # MDX_GATES_*

STATUS_DIVERGED = 1
STATUS_NONFINITE = 2
STATUS_STOPPED = 4

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double


class TissueIonicArgs(C.Structure):
    _fields_ = [
        ("n", _i64), ("dofs", _p), ("u_ring", _p), ("ldu", _i64),
        ("w_ring", _p), ("ldw", _i64), ("ring_slots", _i32), ("head", _i32),
        ("order", _i32), ("prep", _i32), ("dt", _d), ("i_out", _p),
        ("clamp_count", _p), ("combo", _p), ("profiles", _p), ("ldp", _i64),
        ("active_mask", C.c_uint64), ("n_impulses", _i32), ("gate_scheme", _i32),
        ("status", _p),
    ]


class Operator(C.Structure):
    _fields_ = [
        ("kind", _i32), ("ncls", _i32), ("n", _i64), ("nx1", _i32),
        ("ny1", _i32), ("nz1", _i32), ("_pad", _i32), ("meta", _p),
        ("indptr", _p), ("indices", _p), ("nnz", _i64),
        ("dia_np", _i32), ("_pad1", _i32), ("dia_ld", _i64), ("dia_off", _i64 * DIA_MAX),
        ("rem_n", _i64), ("rem_ptr", _p), ("rem_row", _p), ("rem_col", _p),
    ]


class CgArgs(C.Structure):
    _fields_ = [
        ("op", Operator), ("a_val", _p), ("dinv", _p), ("b", _p),
        ("m_val", _p), ("combo", _p), ("n_lift", _i32), ("step", _i32),
        ("lift_val", _p * MAX_LIFT), ("lift_cur", _p * MAX_LIFT),
        ("inactive", _p), ("rest", _p), ("thr", _p), ("x", _p), ("p", _p),
        ("q", _p), ("r", _p), ("z", _p), ("w", _p), ("s", _p),
        ("m", _p),
        ("u_prev", _p), ("act_time", _p), ("best_slope", _p), ("frozen", _p),
        ("t_next", _d), ("dt", _d), ("tol", _d), ("max_iter", _i32),
        ("partials_capacity", _i32), ("partials", _p), ("barrier", _p),
        ("iters_out", _p), ("relres_out", _p), ("status", _p),
        ("fail_step", _p), ("variant", _i32), ("dom_class1", _i32),
        ("row_begin", _i64), ("row_end", _i64),
        ("row_out", _p), ("row_probes", _p), ("row_nprobes", _i32), ("_pad2", _i32),
        ("dom_row_host", _p), ("dom_m_row_host", _p),
        ("row_mask", _p), ("row_select", _i32), ("_pad3", _i32),
        ("tstamps", _p), ("frozen_count", _p), ("frozen_target", _i64),
        ("stop_when_full", _i32), ("_pad4", _i32),
    ]


class PcgScal(C.Structure):
    _fields_ = [
        ("b_norm", _d), ("res", _d), ("gamma", _d), ("delta", _d), ("gamma_prev", _d),
        ("alpha_prev", _d), ("alpha", _d), ("beta", _d), ("nonfinite", _d),
        ("it", _i32), ("state", _i32), ("first", _i32), ("_pad", _i32),
    ]


SC_INIT, SC_W0, SC_SWEEP = 0, 1, 2


class AssemblyArgs(C.Structure):
    _fields_ = [
        ("n_elem", _i64), ("nl", _i32), ("nq", _i32), ("nodes", _p),
        ("elements", _p), ("quad_w", _p), ("quad_basis", _p),
        ("quad_grad", _p), ("sigma_row", _p), ("sigmas", _p), ("f0", _p),
        ("s0", _p), ("K_local", _p), ("M_local", _p),
    ]


class PaceArgs(C.Structure):
    _fields_ = [
        ("n_cells", _i64), ("u", _p), ("W", _p), ("ldw", _i64), ("peak", _p),
        ("order", _i32), ("n_pulses", _i32), ("n_steps", _i64), ("dt", _d),
        ("n_stim_cells", _i64), ("period", _d), ("pulse_t0", _d * 8),
        ("pulse_dur", _d * 8), ("pulse_amp", _d * 8), ("n_trace_cells", _i64),
        ("trace_rows", _i64), ("stride", _i64), ("trace", _p),
        ("clamp_count", _p), ("status", _p), ("gate_scheme", _i32), ("_pad", _i32),
    ]


_SIGNATURES = {
    "mdx_last_error": ([], C.c_char_p),
    "mdx_abi_version": ([], C.c_int),
    "mdx_ionic_num_vars": ([C.c_int], C.c_int),
    "mdx_ionic_num_params": ([C.c_int], C.c_int),
    "mdx_ionic_advance": ([C.c_int, _i64, _p, _p, _p, _i64, _i64, _d, _d, _p,
                           C.c_int, _p, _p, _p, _p], C.c_int),
    "mdx_ionic_advance_rl": ([C.c_int, _i64, _p, _p, _i64, _i64, _d, _p, C.c_int, _p, _p,
                              _p, _p], C.c_int),
    "mdx_ionic_current": ([C.c_int, _i64, _p, _p, _i64, _i64, _p, C.c_int, _p,
                           _p], C.c_int),
    "mdx_ionic_point_rates": ([C.c_int, _i64, _p, _p, _p, C.c_int, _p, _p, _p],
                              C.c_int),
    "mdx_tissue_ionic": ([C.c_int, C.POINTER(TissueIonicArgs), _p, C.c_int, _p],
                         C.c_int),
    "mdx_tissue_prep": ([C.POINTER(TissueIonicArgs), _p], C.c_int),
    "mdx_pcg_solve": ([C.POINTER(CgArgs), C.c_int, C.c_int, _p], C.c_int),
    "mdx_pcg_phase": ([C.POINTER(CgArgs), C.c_int, C.c_int, _d, _d, C.c_int, C.c_int, _p,
                       _p], C.c_int),
    "mdx_pcg_phase_dev": ([C.POINTER(CgArgs), C.c_int, C.c_int, _p, C.c_int, _p, _p],
                          C.c_int),
    "mdx_pcg_scalars": ([_p, _p, C.c_int, _d, C.c_int, _p], C.c_int),
    "mdx_spmv": ([C.POINTER(CgArgs), _p, _p, _p], C.c_int),
    "mdx_gather": ([_i64, _p, _p, _p, _p], C.c_int),
    "mdx_scatter": ([_i64, _p, _p, _p, _p], C.c_int),
    "mdx_assemble_local": ([C.POINTER(AssemblyArgs), _p], C.c_int),
    "mdx_scatter_csr": ([_i64, C.c_int, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
                        C.c_int),
    "mdx_stencil_rows": ([C.c_int, C.c_int, C.c_int, _p, _p, _p, _p], C.c_int),
    "mdx_hash_rows": ([_i64, C.c_int, C.c_int, _p, _p, _p], C.c_int),
    "mdx_verify_classes": ([_i64, C.c_int, C.c_int, _p, _p, _p, _p, _p], C.c_int),
    "mdx_combine_system": ([_i64, _d, _p, _p, _p, _p], C.c_int),
    "mdx_pace_cells": ([C.c_int, C.POINTER(PaceArgs), _p, C.c_int, _p],
                       C.c_int),
    "mdx_record_row": ([_p, _i64, _p, C.c_int, _p, _p, _p], C.c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def load_library(path=_LIB_PATH):
    """dlopen libmdx.so and attach signatures (no CUDA device needed)."""
    if not Path(path).exists():
        raise NativeUnavailable(
            f"{path} is missing: run `python -m paper_2308_01651_b200.native_build`"
        )
    handle = C.CDLL(str(path))
    for name, (argtypes, restype) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = argtypes
        fn.restype = restype
    return handle


def lib():
    """The loaded library, after checking a CUDA device is usable."""
    global _lib
    if _lib is None:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable(
                "no CUDA device: the monodomain kernels run only on sm_100a "
                "(there is no CPU fallback)")
        _lib = load_library()
        if _lib.mdx_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libmdx.so ABI version mismatch")
    return _lib


def check(rc, what=""):
    if rc != MDX_OK:
        msg = lib().mdx_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def host_doubles(values):
    """Contiguous float64 numpy array + its ctypes pointer (kept alive)."""
    arr = np.ascontiguousarray(values, dtype=np.float64)
    return arr, arr.ctypes.data_as(C.c_void_p)
