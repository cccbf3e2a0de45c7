"""Time the tissue ionic kernel alone on config 2 for several libmdx variants.

    python scripts/kbench.py variant1 variant2 ...   (paper_2308_01651_b200/_build/variants)
Each variant runs in a subprocess (MDX_LIB selects the .so).
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child():
    sys.path.insert(0, str(ROOT))
    import torch

    from paper_2308_01651_b200 import _native as N, configs
    from paper_2308_01651_b200.simulation import TissueSolver

    cfg = configs.config2(configs.this_package())
    s = TissueSolver(cfg)
    for _ in range(3):
        s.enqueue_step()
    s.sync()
    model_id, ia, Ph, Pp = s._ionic_args[0]
    ia.head = s.head
    ia.order = 2
    lib = N.lib()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        lib.mdx_tissue_ionic(model_id, N.C.byref(ia), Pp, int(Ph.size), s._stream)
    ev[0].record()
    reps = 20
    for _ in range(reps):
        lib.mdx_tissue_ionic(model_id, N.C.byref(ia), Pp, int(Ph.size), s._stream)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    nbytes = s.n * 8 * (2 + 2 * 18 + 18 + 3)
    print(f"{os.environ.get('MDX_LIB', 'default')}: {ms * 1e3:.1f} us/launch, "
          f"{nbytes / ms / 1e6:.0f} GB/s algorithmic, {s.n / ms / 1e3:.3e} nodes/s")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        names = sys.argv[1:] or ["default"]
        for nm in names:
            env = dict(os.environ)
            if nm != "default":
                env["MDX_LIB"] = str(ROOT / "paper_2308_01651_b200" / "_build" / "variants"
                                     / f"libmdx_{nm}.so")
            subprocess.run([sys.executable, __file__, "--child"], env=env)
