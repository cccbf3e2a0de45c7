"""B200-native monodomain hot path (lifex-ep, arXiv 2308.01651).

Python host mirror of the reference package's ionic-model, mesh, FE,
linear-solver and tissue-solver interfaces (`/root/reference/pkg/src/
monodomain`), running every per-node and per-iteration computation in the
hand-written sm_100a kernels of `libmdx.so` (C-ABI: `include/mdx.h`).
There is no CPU fallback.
"""

from . import errors  # noqa: F401
from .timestepping import BdfScheme, HistoryRing, bdf_coefficients, startup_schedule  # noqa: F401

__version__ = "0.1.0"
