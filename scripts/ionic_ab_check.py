"""Bitwise A/B of two libmdx builds on a tissue run (same config, same steps).

    MDX_LIB=<lib> python scripts/ionic_ab_check.py --config 2 --steps 60 --out f.npz
    python scripts/ionic_ab_check.py --compare a.npz b.npz

Dumps the potential, every volume's newest ionic state, the CG iteration log
and the activation map; --compare reports the number of differing entries.
"""

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--out")
    ap.add_argument("--compare", nargs=2)
    args = ap.parse_args()
    if args.compare:
        a, b = (np.load(f) for f in args.compare)
        bad = 0
        for k in a.files:
            d = int(np.count_nonzero(a[k].view(np.uint8) != b[k].view(np.uint8)))
            print(f"{k}: {a[k].shape} differing bytes {d}")
            bad += d
        print("BITWISE EQUAL" if bad == 0 else "DIFFERENT")
        return
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    ns = configs.this_package()
    cfg = {"0": configs.config0, "2": configs.config2, "3": configs.config3}[args.config](ns)
    s = TissueSolver(cfg)
    for _ in range(args.steps):
        s.enqueue_step()
    s.sync()
    out = {"u": np.asarray(s.potential), "iters": np.asarray(s.iterations_log()),
           "act": np.asarray(s.activation_map),
           "clamps": np.array([s.clamp_total()])}
    for k, vol in enumerate(s.volumes):
        out[f"w{k}"] = s.volume_state(k)
    np.savez(args.out, **out)
    print("saved", args.out, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
