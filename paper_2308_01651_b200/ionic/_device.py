"""Shared device dispatch for the ionic module protocol.

Each model module exposes `advance_kernel`, `current_kernel` and
`point_rates` with the reference signatures
(`/root/reference/pkg/src/monodomain/ionic/__init__.py:1-11`). Inputs may be
numpy arrays (the reference's AoS `(N, nv)` layout; copied to the device,
computed, copied back into the caller's output arrays) or torch CUDA tensors
(computed in place, no host round trip). Both go through libmdx.so.
"""

import numpy as np

from .. import _native as N


def _torch():
    import torch

    return torch


def _is_cuda_tensor(x):
    return hasattr(x, "is_cuda") and x.is_cuda


def _as_device(x, torch, dtype=None):
    if _is_cuda_tensor(x):
        return x
    arr = np.ascontiguousarray(x, dtype=np.float64 if dtype is None else dtype)
    return torch.from_numpy(arr).cuda()


def _layout(W, nv):
    """(cs, vs) element strides of a 2-D state array of shape (N, nv)."""
    if W.ndim != 2 or W.shape[1] != nv:
        raise ValueError(f"state array must have shape (N, {nv}), got {tuple(W.shape)}")
    s0, s1 = (W.stride() if _is_cuda_tensor(W)
              else tuple(s // W.itemsize for s in W.strides))
    if nv == 1:
        s1 = 0          # a single variable: the variable stride is never used
    if W.shape[0] == 1:
        s0 = 0
    return s0, s1


def advance(model_id, nv, u_ext, W_ext, W_bdf, alpha, dt, P, W_out, I_out):
    """Run <model>.advance_kernel on the device; returns the clamp count."""
    torch = _torch()
    lib = N.lib()
    n = int(u_ext.shape[0])
    host_out = not _is_cuda_tensor(W_out)
    u_d = _as_device(u_ext, torch)
    we_d = _as_device(W_ext, torch)
    wb_d = _as_device(W_bdf, torch)
    if host_out:
        wo_d = torch.empty((n, nv), dtype=torch.float64, device="cuda")
        io_d = torch.empty(n, dtype=torch.float64, device="cuda")
    else:
        wo_d, io_d = W_out, I_out
    cs, vs = _layout(wb_d, nv)
    if _layout(we_d, nv) != (cs, vs) or _layout(wo_d, nv) != (cs, vs):
        raise ValueError("W_ext, W_bdf and W_out must share one layout")
    clamp = torch.zeros(1, dtype=torch.int64, device="cuda")
    Ph, Pp = N.host_doubles(P)
    N.check(lib.mdx_ionic_advance(
        model_id, n, N.ptr(u_d), N.ptr(we_d), N.ptr(wb_d), cs, vs,
        float(alpha), float(dt), Pp, int(Ph.size), N.ptr(wo_d), N.ptr(io_d),
        N.ptr(clamp), N.stream_handle()), "mdx_ionic_advance")
    if host_out:
        W_out[...] = wo_d.cpu().numpy()
        I_out[...] = io_d.cpu().numpy()
    return int(clamp.item())


def advance_rl(model_id, nv, u, W_n, dt, P, W_out, I_out):
    """Rush-Larsen one-step update (`mdx_ionic_advance_rl`); returns the clamp count."""
    torch = _torch()
    lib = N.lib()
    n = int(u.shape[0])
    host_out = not _is_cuda_tensor(W_out)
    u_d = _as_device(u, torch)
    wn_d = _as_device(W_n, torch)
    if host_out:
        wo_d = torch.empty((n, nv), dtype=torch.float64, device="cuda")
        io_d = torch.empty(n, dtype=torch.float64, device="cuda")
    else:
        wo_d, io_d = W_out, I_out
    cs, vs = _layout(wn_d, nv)
    if _layout(wo_d, nv) != (cs, vs):
        raise ValueError("W_n and W_out must share one layout")
    clamp = torch.zeros(1, dtype=torch.int64, device="cuda")
    Ph, Pp = N.host_doubles(P)
    N.check(lib.mdx_ionic_advance_rl(
        model_id, n, N.ptr(u_d), N.ptr(wn_d), cs, vs, float(dt), Pp, int(Ph.size),
        N.ptr(wo_d), N.ptr(io_d), N.ptr(clamp), N.stream_handle()), "mdx_ionic_advance_rl")
    if host_out:
        W_out[...] = wo_d.cpu().numpy()
        I_out[...] = io_d.cpu().numpy()
    return int(clamp.item())


def current(model_id, nv, u, W, P, I_out):
    torch = _torch()
    lib = N.lib()
    n = int(u.shape[0])
    host_out = not _is_cuda_tensor(I_out)
    u_d = _as_device(u, torch)
    w_d = _as_device(W, torch)
    io_d = torch.empty(n, dtype=torch.float64, device="cuda") if host_out else I_out
    cs, vs = _layout(w_d, nv)
    Ph, Pp = N.host_doubles(P)
    N.check(lib.mdx_ionic_current(model_id, n, N.ptr(u_d), N.ptr(w_d), cs, vs,
                                  Pp, int(Ph.size), N.ptr(io_d),
                                  N.stream_handle()), "mdx_ionic_current")
    if host_out:
        I_out[...] = io_d.cpu().numpy()


def point_rates(model_id, nv, u, w, P):
    """(I_ion, dw/dt) at one point, evaluated on the device."""
    torch = _torch()
    lib = N.lib()
    u_d = torch.tensor([float(u)], dtype=torch.float64, device="cuda")
    w_d = _as_device(np.asarray(w, dtype=np.float64).reshape(1, nv), torch)
    i_d = torch.empty(1, dtype=torch.float64, device="cuda")
    dw_d = torch.empty((1, nv), dtype=torch.float64, device="cuda")
    Ph, Pp = N.host_doubles(P)
    N.check(lib.mdx_ionic_point_rates(model_id, 1, N.ptr(u_d), N.ptr(w_d), Pp,
                                      int(Ph.size), N.ptr(i_d), N.ptr(dw_d),
                                      N.stream_handle()), "mdx_ionic_point_rates")
    return float(i_d.item()), dw_d.cpu().numpy()[0]
