"""The ionic kernels' exp / log restated in exact rational arithmetic from
the tables and constants in csrc/ionic_models.cuh, checked against
high-precision values: the error bounds DESIGN.md quotes (CPU only)."""

import math
import random
import re
import struct
from fractions import Fraction
from pathlib import Path

import pytest

mpmath = pytest.importorskip("mpmath")

SRC = (Path(__file__).resolve().parents[1] / "paper_2308_01651_b200" / "csrc"
       / "ionic_models.cuh").read_text()


def _table(name):
    m = re.search(r"MDX_TABLE double " + name + r"\[64\] = \{(.*?)\};", SRC, re.S)
    return [float(x) for x in m.group(1).replace("\n", " ").split(",") if x.strip()]


def _fma(a, b, c):                      # one rounding, like the device DFMA
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _bits(x):
    return struct.unpack("<q", struct.pack("<d", x))[0]


def _dbl(b):
    return struct.unpack("<d", struct.pack("<q", b))[0]


def _mexp(x, t2):
    n = float(round(x * 92.33248261689366))
    r = _fma(n, -0.01083042468962958, x)
    r = _fma(n, -6.619564634077006e-12, r)
    ni = int(n)
    t = t2[ni & 63]
    r2 = r * r
    a = _fma(r, 1 / 6, 0.5)
    b = _fma(r, 1 / 120, 1 / 24)
    q = _fma(r2, _fma(r2, b, a), r)
    return _dbl(_bits(_fma(t, q, t)) + ((ni >> 6) << 52))


def _mlog(x, inv, lt):
    b = _bits(x)
    e = (b >> 52) - 1023
    j = (b >> 46) & 63
    m = _dbl((b & 0x000FFFFFFFFFFFFF) | 0x3FF0000000000000)
    f = _fma(m, inv[j], -1.0)
    f2 = f * f
    a = _fma(f, 1 / 7, -1 / 6)
    c = _fma(f, 0.2, -0.25)
    d = _fma(f, 1 / 3, -0.5)
    q = _fma(f2, _fma(f2, a, c), d)
    hi = _fma(float(e), 0.6931467056274414, lt[j])
    lo = _fma(float(e), 4.7493250390316726e-07, _fma(f2, q, f))
    return hi + lo


def test_tables_match_their_definitions():
    mpmath.mp.prec = 120
    t2 = _table("c_exp2j")
    inv, lt = _table("c_log_inv"), _table("c_log_t")
    for j in range(64):
        assert t2[j] == float(mpmath.mpf(2) ** (mpmath.mpf(j) / 64))
        assert inv[j] == float(1 / (1 + (mpmath.mpf(j) + 0.5) / 64))
        assert lt[j] == float(-mpmath.log(mpmath.mpf(inv[j])))


def test_exp_and_log_error_bounds():
    mpmath.mp.prec = 120
    t2 = _table("c_exp2j")
    inv, lt = _table("c_log_inv"), _table("c_log_t")
    rng = random.Random(7)
    worst_e = worst_l = 0.0
    for _ in range(3000):
        x = rng.uniform(-700, 700) if rng.random() < 0.5 else rng.uniform(-30, 30)
        ex = mpmath.e ** mpmath.mpf(x)
        worst_e = max(worst_e, float(abs(mpmath.mpf(_mexp(x, t2)) - ex) / math.ulp(float(ex))))
        z = 10 ** rng.uniform(-8, 8)
        if 0.6 < z < 1.65:                       # the library log covers this window
            continue
        lx = mpmath.log(mpmath.mpf(z))
        worst_l = max(worst_l, float(abs(mpmath.mpf(_mlog(z, inv, lt)) - lx)
                                     / math.ulp(float(lx))))
    assert worst_e < 1.5 and worst_l < 1.5
