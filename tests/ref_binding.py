"""The kernel-level binding of INTEGRATION.md section 2, as a maintainer of the
reference would add it: plain ctypes over libmdx.so, no import of this package.

`bind(module, model_id)` swaps `<module>.advance_kernel` (reference
ionic/ten_tusscher.py:374-403, bueno_orovio.py:152-186) for the C-ABI call
`mdx_ionic_advance`; `unbind` restores the numba kernel.  Used by
tests/test_gpu_dropin.py inside the reference's own TissueSolver.step.
"""

import ctypes
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parents[1] / "paper_2308_01651_b200" / "libmdx.so"
MDX_MODEL_BUENO_OROVIO, MDX_MODEL_TTP06 = 1, 2

_mdx = None


def _lib():
    global _mdx
    if _mdx is None:
        _mdx = ctypes.CDLL(str(LIB))
        _mdx.mdx_ionic_advance.argtypes = (
            [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 +
            [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
             ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4)
        _mdx.mdx_ionic_advance.restype = ctypes.c_int
        _mdx.mdx_last_error.restype = ctypes.c_char_p
    return _mdx


def make_advance_kernel(model_id):
    import torch

    def advance_kernel(u_ext, W_ext, W_bdf, alpha, dt, P, W_out, I_out):
        def dev(a):
            return torch.from_numpy(np.ascontiguousarray(a)).cuda()

        u, we, wb = dev(u_ext), dev(W_ext), dev(W_bdf)
        wo = torch.empty_like(we)
        io = torch.empty_like(u)
        clamp = torch.zeros(1, dtype=torch.int64, device="cuda")
        P = np.ascontiguousarray(P, dtype=np.float64)        # host array, passed by value
        rc = _lib().mdx_ionic_advance(
            model_id, u.numel(), u.data_ptr(), we.data_ptr(), wb.data_ptr(),
            W_ext.shape[1], 1,                                # AoS (N, nv): cs = nv, vs = 1
            alpha, dt, P.ctypes.data, P.size, wo.data_ptr(), io.data_ptr(),
            clamp.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0, _lib().mdx_last_error()
        W_out[...] = wo.cpu().numpy()
        I_out[...] = io.cpu().numpy()
        return int(clamp.item())

    return advance_kernel


class bound:
    """Context manager: <module>.advance_kernel -> the C-ABI kernel."""

    def __init__(self, module, model_id):
        self.module, self.model_id = module, model_id

    def __enter__(self):
        self.orig = self.module.advance_kernel
        self.module.advance_kernel = make_advance_kernel(self.model_id)
        return self

    def __exit__(self, *exc):
        self.module.advance_kernel = self.orig
        return False
