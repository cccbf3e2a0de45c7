"""Minimal driver for profiling: build a config, run W + K steps, print timing.

    python scripts/step_driver.py [--config 2|0|3] [--steps K] [--warmup W]

Used under ncu (launch lists and --set full captures); the numbers it prints
are not bench values.
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--h", type=float, default=None)
    ap.add_argument("--operator", default="auto")
    ap.add_argument("--blocks", type=int, default=0)
    ap.add_argument("--variant", type=int, default=None)
    ap.add_argument("--nodes", type=float, default=1e6, help="config 4 target size")
    args = ap.parse_args()

    import torch

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    ns = configs.this_package()
    kw = {} if args.h is None else {"h": args.h}
    if args.config == "4":
        from paper_2308_01651_b200 import ventricle

        t0 = time.perf_counter()
        cfg = ventricle.config4(ns, *ventricle.size_for_nodes(args.nodes))
        print(f"config 4 mesh: {cfg.mesh.nodes.shape[0]} nodes, "
              f"{cfg.mesh.elements.shape[0]} tets, {time.perf_counter() - t0:.1f} s")
    else:
        cfg = {"0": configs.config0, "2": configs.config2, "3": configs.config3}[args.config](
            ns, **kw)
    t0 = time.perf_counter()
    s = TissueSolver(cfg, operator=args.operator, blocks_hint=args.blocks,
                     cg_variant=args.variant)
    print(f"setup {time.perf_counter() - t0:.1f} s")
    for _ in range(args.warmup):
        s.enqueue_step()
    s.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.enqueue_step()
    ev[1].record()
    s.sync()
    wall = time.perf_counter() - t0
    ms = ev[0].elapsed_time(ev[1])
    its = s.iterations_log()[-args.steps:]
    print(f"n={s.n} op={ {1: 'stencil', 2: 'csr', 3: 'sell', 4: 'dia'}[s.op.kind]} variant={s.cg_variant} steps={args.steps} "
          f"device {ms / args.steps:.3f} ms/step host {wall / args.steps * 1e3:.3f} ms/step "
          f"iters {its.min()}..{its.max()} mean {its.mean():.2f} "
          f"DoF*steps/s {s.n * args.steps / (ms * 1e-3):.3e}")
    if args.steps <= 16:
        print("iterations of every step since rest:", s.iterations_log().tolist())


if __name__ == "__main__":
    main()
