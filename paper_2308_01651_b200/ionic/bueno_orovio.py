"""Bueno-Orovio minimal ventricular model (u + gates v, w, s).

Module protocol of `/root/reference/pkg/src/monodomain/ionic/bueno_orovio.py`:
metadata `:18-27`, EPI parameter set `:30-61` (Bueno-Orovio, Cherry & Fenton,
J. Theor. Biol. 253, 2008, Table 1), `pack` `:72-73`, kernels `:135-186`.
The arithmetic runs in `csrc/ionic_models.cuh` (struct BuenoOrovio).
"""

import numpy as np

from . import _device
from .base import CellState

NAME = "Bueno-Orovio"
NUM_VARS = 3
VAR_NAMES = ("v", "w", "s")
GATES = (True, True, True)
MILLIVOLT_GAIN = 85.7
MILLIVOLT_OFFSET = -84.0
ACTIVATION_THRESHOLD = 0.6
MODEL_ID = 1

_EPI = (
    ("u_o", 0.0), ("u_u", 1.55), ("theta_v", 0.3), ("theta_w", 0.13),
    ("theta_v_minus", 0.006), ("theta_o", 0.006), ("tau_v1_minus", 60.0),
    ("tau_v2_minus", 1150.0), ("tau_v_plus", 1.4506), ("tau_w1_minus", 60.0),
    ("tau_w2_minus", 15.0), ("k_w_minus", 65.0), ("u_w_minus", 0.03),
    ("tau_w_plus", 200.0), ("tau_fi", 0.11), ("tau_o1", 400.0),
    ("tau_o2", 6.0), ("tau_so1", 30.0181), ("tau_so2", 0.9957),
    ("k_so", 2.0458), ("u_so", 0.65), ("tau_s1", 2.7342), ("tau_s2", 16.0),
    ("k_s", 2.0994), ("u_s", 0.9087), ("tau_si", 1.8875),
    ("tau_w_inf", 0.07), ("w_inf_star", 0.94),
)
_ORDER = tuple(k for k, _ in _EPI)


def default_parameters():
    return dict(_EPI)


def default_initial_state():
    return CellState(0.0, np.array([1.0, 1.0, 0.0]))


def default_initial_conditions():
    return {"Transmembrane potential": 0.0, "v": 1.0, "w": 1.0, "s": 0.0}


def pack(parameters, cell_type=None):
    return np.array([parameters[k] for k in _ORDER], dtype=np.float64)


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
