"""Config 1 (BASELINE.json configs[1]): 2^26 independent TTP06 epicardial cells.

Initial state = rest x (1 + 0.01 N(0,1)) per variable (seeded), cells with
index < N/100 paced at 52 V/s for 1 ms, dt = 1e-5 s, 2,000 steps, in either
ionic scheme: `--scheme bdf` the reference's IMEX-BDF splitting (parity mode),
`--scheme rush_larsen` the config as BASELINE words it (Rush-Larsen on gates,
explicit Euler elsewhere; not a reference scheme).  One register-resident device thread per cell for
all steps (`mdx_pace_cells`).  A 256-cell prefix is re-run with the CPU
oracle and compared.

    python scripts/config1_batch.py [--cells N] [--steps K] [--order 2] [--scheme bdf|rush_larsen]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=2 ** 26)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--check", type=int, default=256)
    ap.add_argument("--scheme", default="bdf", choices=["bdf", "rush_larsen"])
    args = ap.parse_args()
    if args.scheme == "rush_larsen":
        args.order = 1

    import torch

    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.ionic import (IonicModelSpec, ModelKind, PacingProtocol0D,
                                             pace_cells, ten_tusscher)

    n = args.cells
    u0, W0 = configs.config1_initial(n)
    spec = IonicModelSpec(ModelKind.TTP06)
    dt = 1e-5
    proto = PacingProtocol0D((0.0,), (1e-3,), (52.0,), 0.0, args.steps * dt, dt)
    u_d = torch.from_numpy(u0).cuda()
    W_d = torch.from_numpy(np.ascontiguousarray(W0.T)).cuda()      # SoA (18, n)
    # warm-up on a small batch (module load, JIT-free)
    pace_cells(spec, proto, u0[:1024], W0[:1024], order=args.order, n_stim_cells=10,
               gate_scheme=args.scheme)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    u, W, peak, clamps, _ = pace_cells(spec, proto, u_d, W_d, order=args.order,
                                       n_stim_cells=n // 100, return_device=True,
                                       gate_scheme=args.scheme)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    k = args.check
    P = ten_tusscher.pack(spec.parameters)
    ur, Wr, pr, _ = O.pace_batch("TTP06", P, u0[:k], W0[:k], dt, args.steps, args.order,
                                 min(k, n // 100), 52.0, 1e-3, gate_scheme=args.scheme)
    ug = u[:k].cpu().numpy()
    pg = peak[:k].cpu().numpy()
    rel = float(np.linalg.norm(ug - ur) / np.linalg.norm(ur))
    fired = int((pg > 0.0).sum())
    print(json.dumps({
        "workload": f"config1 TTP06 batch, {n} cells x {args.steps} steps, "
                    + (f"BDF{args.order}" if args.scheme == "bdf" else "Rush-Larsen"),
        "cell_steps_per_s": n * args.steps / (ms * 1e-3), "ms": ms,
        "state_bytes_per_cell_step_streaming_equiv": 8 * (1 + 18) * 2,
        "oracle_prefix_rel_l2_u": rel, "oracle_prefix_cells": k,
        "fired_in_prefix": fired, "clamps": clamps}))


if __name__ == "__main__":
    main()
