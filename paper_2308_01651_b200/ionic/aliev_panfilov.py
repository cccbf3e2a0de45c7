"""Aliev-Panfilov two-variable model (u + explicit recovery w).

Module protocol of `/root/reference/pkg/src/monodomain/ionic/aliev_panfilov.py`
(metadata `:20-29`, parameters `:32-41`, `pack` `:52-57`, kernels `:62-95`).
The arithmetic runs in `csrc/ionic_models.cuh` (struct AlievPanfilov).
"""

import numpy as np

from . import _device
from .base import CellState

NAME = "Aliev-Panfilov"
NUM_VARS = 1
VAR_NAMES = ("w",)
GATES = (False,)
MILLIVOLT_GAIN = 100.0
MILLIVOLT_OFFSET = -80.0
ACTIVATION_THRESHOLD = 0.6
MODEL_ID = 0


def default_parameters():
    return {"a": 0.01, "b": 0.15, "k": 8.0, "eps0": 0.002, "mu1": 0.2,
            "mu2": 0.3, "Time constant": 12.9e-3}


def default_initial_state():
    return CellState(0.0, np.zeros(1))


def default_initial_conditions():
    return {"Transmembrane potential": 0.0, "w": 0.0}


def pack(parameters, cell_type=None):
    keys = ("a", "b", "k", "eps0", "mu1", "mu2", "Time constant")
    return np.array([parameters[k] for k in keys], dtype=np.float64)


def advance_kernel(u_ext, W_ext, W_bdf, alpha, dt, P, W_out, I_out):
    return _device.advance(MODEL_ID, NUM_VARS, u_ext, W_ext, W_bdf, alpha, dt,
                           P, W_out, I_out)


def rush_larsen_kernel(u, W_n, dt, P, W_out, I_out):
    """Rush-Larsen mode (not in the reference): gates exponential,
    the rest explicit Euler, from W_n at potential u; I_out at (u, W_out)."""
    return _device.advance_rl(MODEL_ID, NUM_VARS, u, W_n, dt, P, W_out, I_out)


def current_kernel(u, W, P, I_out):
    _device.current(MODEL_ID, NUM_VARS, u, W, P, I_out)


def point_rates(u, w, P):
    return _device.point_rates(MODEL_ID, NUM_VARS, u, w, P)
