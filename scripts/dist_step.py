"""Time DistributedTissueSolver steps (config 2) under torchrun or alone.

    python scripts/dist_step.py [--steps K] [--host-scalars]
    torchrun --nproc-per-node N scripts/dist_step.py ...
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--host-scalars", action="store_true")
    ap.add_argument("--config", default="2")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.distributed import DistributedTissueSolver

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ns = configs.this_package()
    cfg = {"0": configs.config0, "2": configs.config2}[args.config](ns)
    s = DistributedTissueSolver(cfg, device_scalars=not args.host_scalars)
    for _ in range(args.warmup):
        s.step()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.steps
    its = np.array(s.iters[-args.steps:])
    if dist.get_rank() == 0:
        print(f"world {dist.get_world_size()} {'host' if args.host_scalars else 'device'} "
              f"scalars: {dt * 1e3:.3f} ms/step, CG {its.mean():.2f} it/step, "
              f"{dt / its.mean() * 1e6:.1f} us/iteration")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
