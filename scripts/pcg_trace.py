"""Per-block timeline of one persistent PCG launch (debug build with
-DMDX_PCG_TRACE): phase time = arrive(k) - release(k-1), wait = release -
arrive, per reduction k.  Usage: MDX_LIB=<trace .so> python scripts/pcg_trace.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2308_01651_b200 import _native as N, configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config2(configs.this_package())
    blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    s = TissueSolver(cfg, blocks_hint=blocks, cg_variant=int(sys.argv[2]) if len(sys.argv) > 2 else 2)
    for _ in range(6):
        s.enqueue_step()
    s.sync()
    lib = N.lib()
    lib.mdx_debug_trace.argtypes = [C.c_void_p]
    buf = np.zeros((512, 256, 2), dtype=np.uint64)
    lib.mdx_debug_trace(buf.ctypes.data_as(C.c_void_p))
    its = s.iterations_log()[-1]
    used = buf[:, :, 0].any(axis=1)
    nb = int(used.sum())
    ne = int((buf[0, :, 0] > 0).sum())
    t = buf[:nb, :ne, :].astype(np.int64)
    t0 = t[:, 0, 0].min()
    arrive = t[:, :, 0] - t0
    release = t[:, :, 1] - t0
    X = None
    if hasattr(lib, "mdx_debug_trace_x"):
        lib.mdx_debug_trace_x.argtypes = [C.c_void_p]
        bx = np.zeros((512, 256, 2), dtype=np.uint64)
        lib.mdx_debug_trace_x(bx.ctypes.data_as(C.c_void_p))
        X = bx[:nb, :ne, :].astype(np.int64) - t0
    print(f"blocks {nb}, reductions {ne}, CG iterations {its}")
    print(f"kernel span {release.max() / 1e3:.1f} us")
    for k in range(min(ne, 12)):
        ph = arrive[:, k] - (release[:, k - 1] if k else arrive[:, 0] * 0)
        wait = release[:, k] - arrive[:, k]
        if X is not None and k > 1 and k < ne:
            fx = X[:, k, 0] - arrive[:, k]      # arrival -> neighbour flags seen
            sx = X[:, k, 1] - X[:, k, 0]            # stencil
            print(f"        flags-wait min/med/max {fx.min()/1e3:6.2f} {np.median(fx)/1e3:6.2f} "
                  f"{fx.max()/1e3:6.2f} us | stencil {sx.min()/1e3:6.2f} {np.median(sx)/1e3:6.2f} "
                  f"{sx.max()/1e3:6.2f} us")
        print(f"red {k:2d}: phase min/med/max {ph.min()/1e3:6.2f} {np.median(ph)/1e3:6.2f} "
              f"{ph.max()/1e3:6.2f} us | wait min/med/max {wait.min()/1e3:6.2f} "
              f"{np.median(wait)/1e3:6.2f} {wait.max()/1e3:6.2f} us")


if __name__ == "__main__":
    main()
