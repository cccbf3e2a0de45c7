"""Per-block timeline of the config-4 PCG launch (trace build, -DMDX_PCG_TRACE):
the reference-recurrence loop has two traced reductions per iteration - after the
Q sweep (q = A p) and after the R sweep (r -= alpha q) - so
  phase(Q event) = P sweep + grid_sync + Q sweep,  phase(R event) = R sweep,
and wait = time a block spends in the reduction (publish, arrive, spin, loads).
Usage: MDX_LIB=<trace .so> python scripts/pcg_trace4.py [nodes]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2308_01651_b200 import _native as N, configs, ventricle
    from paper_2308_01651_b200.simulation import TissueSolver

    nodes = float(sys.argv[1]) if len(sys.argv) > 1 else 1e7
    ns = configs.this_package()
    cfg = ventricle.config4(ns, *ventricle.size_for_nodes(nodes))
    s = TissueSolver(cfg)
    for _ in range(12):
        s.enqueue_step()
    s.sync()
    lib = N.lib()
    fn = lib.mdx_debug_trace
    fn.argtypes = [C.c_void_p]
    buf = np.zeros((512, 256, 2), dtype=np.uint64)
    fn(buf.ctypes.data_as(C.c_void_p))
    its = s.iterations_log()[-1]
    nb = int(buf[:, :, 0].any(axis=1).sum())
    ne = int((buf[0, :, 0] > 0).sum())
    t = buf[:nb, :ne, :].astype(np.int64)
    t0 = t[:, 0, 0].min()
    arrive, release = (t[:, :, 0] - t0) / 1e3, (t[:, :, 1] - t0) / 1e3
    print(f"n {s.n} blocks {nb} traced reductions {ne} CG iterations {its}")
    out = Path(__file__).resolve().parents[1] / "gpurun_out"
    out.mkdir(exist_ok=True)
    np.savez_compressed(out / "trace_cfg4.npz", arrive=arrive, release=release)
    print(f"kernel span to last traced event {release.max():.1f} us")
    # event 0: RHS/r0 pass; then per iteration (Q event, R event)
    ph = arrive[:, 1:] - release[:, :-1]
    wait = release - arrive
    # critical path per event = last arrival - previous (common) release
    crit = arrive[:, 1:].max(axis=0) - release[:, :-1].min(axis=0)
    q_ev = np.arange(1, ne - 1, 2) - 1      # indices into ph (event k -> ph[k-1])
    r_ev = q_ev + 1
    r_ev = r_ev[r_ev < ph.shape[1]]

    def line(name, idx):
        p = ph[:, idx]
        print(f"{name}: per-block phase min/med/max {p.min():7.1f} {np.median(p):7.1f} "
              f"{p.max():7.1f} us | critical path mean {crit[idx].mean():7.1f} us | "
              f"wait med {np.median(wait[:, idx + 1]):6.1f} max {wait[:, idx + 1].max():6.1f}")

    line("P+sync+Q", q_ev)
    line("R       ", r_ev)
    per_it = (release[:, 2:ne - 1:2].max(axis=0)[1:] - release[:, 2:ne - 1:2].max(axis=0)[:-1])
    print(f"per-iteration span {per_it.mean():.1f} us (sum of the two critical paths "
          f"{crit[q_ev].mean() + crit[r_ev].mean():.1f})")
    spread_q = arrive[:, 1:][:, q_ev].max(axis=0) - arrive[:, 1:][:, q_ev].min(axis=0)
    spread_r = arrive[:, 1:][:, r_ev].max(axis=0) - arrive[:, 1:][:, r_ev].min(axis=0)
    print(f"arrival spread (last - first block): Q {spread_q.mean():.1f} us, R {spread_r.mean():.1f} us")


if __name__ == "__main__":
    main()
