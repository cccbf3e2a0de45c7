"""Per-block timeline of one persistent PCG launch (debug build with
-DMDX_PCG_TRACE): per reduction k, phase = arrive(k) - release(k-1) and
wait = release(k) - arrive(k); inside the wait: block sums + publish,
arrival atomic, spin until the last arrival, partial loads.
Usage: MDX_LIB=<trace .so> python scripts/pcg_trace.py [blocks] [variant]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def stats(x):
    return f"{np.min(x) / 1e3:6.2f} {np.median(x) / 1e3:6.2f} {np.max(x) / 1e3:6.2f}"


def main():
    from paper_2308_01651_b200 import _native as N, configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config2(configs.this_package())
    blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    variant = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    s = TissueSolver(cfg, blocks_hint=blocks, cg_variant=variant)
    for _ in range(6):
        s.enqueue_step()
    s.sync()
    lib = N.lib()

    def grab(name, shape):
        fn = getattr(lib, name)
        fn.argtypes = [C.c_void_p]
        buf = np.zeros(shape, dtype=np.uint64)
        fn(buf.ctypes.data_as(C.c_void_p))
        return buf

    buf = grab("mdx_debug_trace", (512, 256, 2))
    bx = grab("mdx_debug_trace_x", (512, 256, 2))
    by = grab("mdx_debug_trace_y", (512, 256))
    its = s.iterations_log()[-1]
    nb = int(buf[:, :, 0].any(axis=1).sum())
    ne = int((buf[0, :, 0] > 0).sum())
    t = buf[:nb, :ne, :].astype(np.int64)
    t0 = t[:, 0, 0].min()
    arrive, release = t[:, :, 0] - t0, t[:, :, 1] - t0
    pub, cnt = bx[:nb, :ne, 0].astype(np.int64) - t0, bx[:nb, :ne, 1].astype(np.int64) - t0
    rel = by[:nb, :ne].astype(np.int64) - t0
    print(f"blocks {nb}, reductions {ne}, CG iterations {its}")
    print(f"kernel span {release.max() / 1e3:.1f} us   (min/med/max in us)")
    for k in range(1, min(ne, 12)):
        ph = arrive[:, k] - release[:, k - 1]
        last = int(np.argmax(arrive[:, k]))
        print(f"red {k:2d}: phase {stats(ph)} | wait {stats(release[:, k] - arrive[:, k])} | "
              f"blocksum {stats(pub[:, k] - arrive[:, k])} | atomic {stats(cnt[:, k] - pub[:, k])}"
              f" | spin(last block) {(rel[last, k] - cnt[last, k]) / 1e3:5.2f} | "
              f"last-arrival->release {stats(rel[:, k] - pub[:, k].max())} | "
              f"loads {stats(release[:, k] - rel[:, k])}")


    # which blocks publish last (sweep + intra-block skew), averaged over reductions
    done = (pub[:, 2:min(ne, 12)] - release[:, 1:min(ne, 12) - 1]).mean(axis=1)
    order = np.argsort(-done)
    print("slowest blocks (mean release->publish us):",
          ", ".join(f"{b}:{done[b] / 1e3:.2f}" for b in order[:12]))
    print("fastest blocks:", ", ".join(f"{b}:{done[b] / 1e3:.2f}" for b in order[-6:]))
    q = np.percentile(done, [10, 50, 90]) / 1e3
    print(f"release->publish p10/p50/p90 {q[0]:.2f} {q[1]:.2f} {q[2]:.2f} us")


if __name__ == "__main__":
    main()
