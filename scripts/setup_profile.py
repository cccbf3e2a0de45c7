"""cProfile of config-4 generation + TissueSolver setup (where setup time goes).

    python scripts/setup_profile.py [--nodes 1e7]
"""

import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=float, default=1e7)
    args = ap.parse_args()
    import torch

    from paper_2308_01651_b200 import configs, ventricle
    from paper_2308_01651_b200.simulation import TissueSolver

    ns = configs.this_package()
    torch.zeros(1, device="cuda")
    t0 = time.perf_counter()
    cfg = ventricle.config4(ns, *ventricle.size_for_nodes(args.nodes))
    print(f"mesh {time.perf_counter() - t0:.1f} s", flush=True)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    s = TissueSolver(cfg)
    torch.cuda.synchronize()
    pr.disable()
    print(f"setup {time.perf_counter() - t0:.1f} s, op kind {s.op.kind}", flush=True)
    pstats.Stats(pr).sort_stats("cumtime").print_stats(30)


if __name__ == "__main__":
    main()
