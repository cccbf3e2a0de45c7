"""Courtemanche-Ramirez-Nattel atrial model: interface slot only.

The reference ships parameters and state metadata but no kernels
(`/root/reference/pkg/src/monodomain/ionic/courtemanche.py:87-94` raise
NotImplementedError, pinned by `tests/test_ionic.py:100-105`). With no
reference arithmetic there is no oracle, so this build keeps the slot
(the same metadata names) and raises the same way. SURVEY.md D2.
"""

import numpy as np

from .base import CellState

NAME = "CRN"
NUM_VARS = 20
VAR_NAMES = ("m", "h", "j", "oa", "oi", "ua", "ui", "xr", "xs", "d", "f",
             "fCa", "u_rel", "v_rel", "w_rel", "Nai", "Ki", "Cai", "CaUp",
             "CaRel")
GATES = (True,) * 15 + (False,) * 5
MILLIVOLT_GAIN = 1.0e3
MILLIVOLT_OFFSET = 0.0
ACTIVATION_THRESHOLD = -0.020
MODEL_ID = None

_PARAMETERS = (
    ("gNa", 7.8), ("gK1", 0.09), ("gto", 0.1652), ("gKur_fix", 0.005),
    ("gKur_var", 0.05), ("gKr", 0.029411765), ("gKs", 0.12941176),
    ("gCaL", 0.12375), ("gbNa", 0.0006744375), ("gbCa", 0.001131),
)


def default_parameters():
    return dict(_PARAMETERS)


def default_initial_state():
    w = np.array([2.91e-3, 0.965, 0.978, 3.04e-2, 0.999, 4.96e-3, 0.999,
                  3.29e-5, 1.87e-2, 1.37e-4, 0.999, 0.775, 0.0, 1.0, 0.999,
                  11.17, 139.0, 1.013e-4, 1.488, 1.488])
    return CellState(-81.18e-3, w)


def default_initial_conditions():
    s = default_initial_state()
    out = {"Transmembrane potential": s.u}
    out.update(zip(VAR_NAMES, s.w))
    return out


def pack(parameters, cell_type=None):
    return np.array([parameters[k] for k, _ in _PARAMETERS], dtype=np.float64)


def _missing(*_args, **_kwargs):
    raise NotImplementedError(
        "the CRN slot has no kernels (reference courtemanche.py:87-94)")


current_kernel = _missing
advance_kernel = _missing
point_rates = _missing
