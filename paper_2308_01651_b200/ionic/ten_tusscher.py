"""ten Tusscher-Panfilov 2006 human ventricular model (u + 18 variables).

Module protocol of `/root/reference/pkg/src/monodomain/ionic/ten_tusscher.py`:
metadata `:28-41`, parameters `:44-104` (ten Tusscher & Panfilov, Am. J.
Physiol. 291, 2006), packed layout `:107-128`, `pack` `:131-138`, paced
epicardial initial state `:141-163`, kernels `:175-403`.  The arithmetic runs
in `csrc/ionic_models.cuh` (struct TTP06).
"""

import numpy as np

from . import _device
from .base import CellState, CellType

NAME = "TTP06"
NUM_VARS = 18
VAR_NAMES = ("m", "h", "j", "Xr1", "Xr2", "Xs", "s", "r", "d", "f", "f2",
             "fCass", "Cai", "CaSR", "CaSS", "Nai", "Ki", "Rbar")
GATES = (True,) * 12 + (False,) * 6
MILLIVOLT_GAIN = 1.0e3
MILLIVOLT_OFFSET = 0.0
ACTIVATION_THRESHOLD = -0.020
MODEL_ID = 2

_DEFAULTS = (
    # conductances (nS/pF) and permeabilities
    ("GNa", 14.838), ("GK1", 5.405), ("Gto_endo", 0.073), ("Gto_myo", 0.294),
    ("Gto_epi", 0.294), ("Gkr", 0.153), ("Gks_endo", 0.392),
    ("Gks_myo", 0.098), ("Gks_epi", 0.392), ("GCaL", 3.98e-5),
    ("GpCa", 0.1238), ("KpCa", 0.0005), ("GpK", 0.0146), ("GbNa", 0.00029),
    ("GbCa", 0.000592),
    # pump and exchanger
    ("PNaK", 2.724), ("KmK", 1.0), ("KmNa", 40.0), ("KNaCa", 1000.0),
    ("KmNai", 87.5), ("KmCa", 1.38), ("Ksat", 0.1), ("Alpha", 2.5),
    ("Gamma", 0.35),
    # extracellular concentrations (mM) and physical constants
    ("Ko", 5.4), ("Nao", 140.0), ("Cao", 2.0), ("PkNa", 0.03), ("Cm", 0.185),
    ("F", 96485.3415), ("R", 8314.472), ("T", 310.0), ("Vc", 0.016404),
    ("Vsr", 0.001094), ("Vss", 5.468e-5),
    # buffering
    ("Bufc", 0.2), ("Kbufc", 0.001), ("Bufsr", 10.0), ("Kbufsr", 0.3),
    ("Bufss", 0.4), ("Kbufss", 0.00025),
    # SR fluxes and release
    ("Vmaxup", 0.006375), ("Kup", 0.00025), ("Vrel", 0.102),
    ("Vleak", 0.00036), ("Vxfer", 0.0038), ("k1_prime", 0.15),
    ("k2_prime", 0.045), ("k3", 0.06), ("k4", 0.005), ("EC", 1.5),
    ("max_sr", 2.5), ("min_sr", 1.0),
)

# packed order seen by the kernel (enum TTP06 in ionic_models.cuh); the
# cell-type-specific Gto/Gks are resolved, the endocardial flag appended
PACKED = ("GNa", "GK1", "Gto", "Gkr", "Gks", "GCaL", "GpCa", "KpCa", "GpK",
          "GbNa", "GbCa", "PNaK", "KmK", "KmNa", "KNaCa", "KmNai", "KmCa",
          "Ksat", "Alpha", "Gamma", "Ko", "Nao", "Cao", "PkNa", "Cm", "F",
          "R", "T", "Vc", "Vsr", "Vss", "Bufc", "Kbufc", "Bufsr", "Kbufsr",
          "Bufss", "Kbufss", "Vmaxup", "Kup", "Vrel", "Vleak", "Vxfer",
          "k1_prime", "k2_prime", "k3", "k4", "EC", "max_sr", "min_sr")

_SUFFIX = {CellType.ENDOCARDIUM: "endo", CellType.MYOCARDIUM: "myo",
           CellType.EPICARDIUM: "epi"}


def default_parameters():
    return dict(_DEFAULTS)


def pack(parameters, cell_type=CellType.EPICARDIUM):
    if cell_type is None:
        cell_type = CellType.EPICARDIUM
    sfx = _SUFFIX[cell_type]
    resolved = dict(parameters)
    resolved["Gto"] = parameters[f"Gto_{sfx}"]
    resolved["Gks"] = parameters[f"Gks_{sfx}"]
    vals = [resolved[k] for k in PACKED]
    vals.append(1.0 if cell_type is CellType.ENDOCARDIUM else 0.0)
    return np.array(vals, dtype=np.float64)


def default_initial_state():
    w = np.array([0.00172, 0.7444, 0.7045, 0.00621, 0.4712, 0.00095, 0.999998,
                  2.42e-8, 3.373e-5, 0.7888, 0.9755, 0.9953, 0.000126, 3.64,
                  0.00036, 8.604, 136.89, 0.9073])
    return CellState(-85.23e-3, w)


def default_initial_conditions():
    state = default_initial_state()
    out = {"Transmembrane potential": state.u}
    names = ("M", "H", "J", "Xr1", "Xr2", "Xs", "S", "R", "D", "F", "F2",
             "FCass", "Cai", "CaSR", "CaSS", "Nai", "Ki", "RR")
    out.update(zip(names, state.w))
    return out


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
