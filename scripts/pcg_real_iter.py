"""Per-iteration cost of pcg_kernel<DIASYM7> on the REAL config-4 operator.

    python scripts/pcg_real_iter.py [--nodes 1e7] [--steps 3]

Builds the config-4 solver, advances a few steps, then runs capped solves
(tolerance out of reach, K1 and K2 iterations) on the solver's own operator,
workspace and vectors: cost per iteration = (T2 - T1) / (K2 - K1).  Variants:
the plain (non-tissue) instantiation with a random right-hand side, the same
with the seam's remainder list detached (wrong operator, timing only), and the
tissue instantiation on the solver's state.  Beside scripts/pcg_synth.py (the
same kernel on a synthetic operator) this separates code from data effects.
The solver is left in a meaningless state: timing only.
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=float, default=1e7)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()

    import torch

    from paper_2308_01651_b200 import _native as N
    from paper_2308_01651_b200 import configs, ventricle
    from paper_2308_01651_b200.simulation import TissueSolver

    ns = configs.this_package()
    cfg = ventricle.config4(ns, *ventricle.size_for_nodes(args.nodes))
    s = TissueSolver(cfg)
    for _ in range(args.steps):
        s.enqueue_step()
    s.sync()
    n = s.n
    print(f"n={n} operator kind {s.op.kind} np {getattr(s.op, 'np_', None)} "
          f"nrem {getattr(s.op, 'nrem', None)} iterations so far {s.iterations_log().tolist()}")
    order, t_next, mask, head, nslot = s.step_plan()
    base = s.solve_args(order, t_next, head, nslot)
    g = torch.Generator(device="cuda").manual_seed(1)
    b = torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    xs = torch.zeros(n, dtype=torch.float64, device="cuda")

    def timed(a, tissue, k):
        a.tol = 1e-300
        a.max_iter = k
        s.ws.status.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(N.lib().mdx_pcg_solve(N.C.byref(a), tissue, 0, N.stream_handle()),
                "mdx_pcg_solve")
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    def variant(name, tissue, norem=False, own_x=True):
        a = type(base).from_buffer_copy(base)
        if not tissue:
            a.b = N.ptr(b)
        if own_x:
            a.x = N.ptr(xs)
        if norem:
            a.op.rem_n = 0
        a.act_time = None if not tissue else a.act_time
        a.row_out = None
        a.tstamps = None
        a.frozen_count = None
        k1, k2 = 20, 100
        timed(a, tissue, 5)
        for _ in range(2):
            xs.zero_()
            t1 = timed(a, tissue, k1)
            xs.zero_()
            t2 = timed(a, tissue, k2)
            per = (t2 - t1) / (k2 - k1) * 1e3
            print(f"{name:34s}: {k1} it {t1:.3f} ms, {k2} it {t2:.3f} ms -> {per:.1f} us/iteration "
                  f"{160e-9 * n / (per * 1e-6):.0f} GB/s at 160 B")

    variant("plain, random b, scratch x", 0)
    variant("plain, random b, no remainder", 0, norem=True)
    variant("plain, random b, x = ring slot", 0, own_x=False)
    variant("tissue, solver state, scratch x", 1)
    variant("tissue, no remainder", 1, norem=True)
    s.ws.status.zero_()


if __name__ == "__main__":
    main()
