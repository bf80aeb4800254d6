"""Pins for O3 (the contract's exp) against libm and closed forms.

O3 is the exponential both sides use for Eq.1's softmax numerator.
Pins: exp(0) = 1 exactly; the cutoff returns 0 below -87; the EXHAUSTIVE sweep
over every float in [-87, -0] stays within 1 ulp of double-precision libm
exp and never produces a subnormal or non-finite value; exp(-n ln2) ~ 2^-n.
"""
import math
import struct
from concurrent.futures import ThreadPoolExecutor

import pytest


def fbits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_exp_closed_forms(oracle):
    assert oracle.spc_exp(0.0) == 1.0
    assert oracle.spc_exp(-0.0) == 1.0
    assert oracle.spc_exp(-87.5) == 0.0
    assert oracle.spc_exp(-1000.0) == 0.0
    for n in range(0, 120, 7):
        x = -n * math.log(2.0)
        x32 = struct.unpack("<f", struct.pack("<f", x))[0]  # the float actually passed
        y = oracle.spc_exp(x32)
        # exp(x32) = 2^-n * exp(x32 - x): input rounding plus <= 1 ulp
        assert abs(y / 2.0 ** -n - math.exp(x32 - x)) < 2.0 ** -23, n
    # a few ordinary points against libm (the whole range is swept below)
    for x in (-1e-7, -0.5, -1.0, -2.302585, -10.0, -50.0, -86.9):
        x = struct.unpack("<f", struct.pack("<f", x))[0]
        assert abs(oracle.spc_exp(x) - math.exp(x)) <= 1.2e-7 * math.exp(x), x


def test_exp_exhaustive_ulp(oracle):
    """Every float in [-87, -0] (1,118,699,521 values): <= 1 ulp, no subnormal."""
    lo, hi = fbits(-0.0), fbits(-87.0)
    assert (lo, hi) == (0x80000000, 0xC2AE0000)
    nchunk = 64
    step = (hi - lo + nchunk) // nchunk
    ranges = [(lo + i * step, min(hi, lo + (i + 1) * step - 1)) for i in range(nchunk)]
    with ThreadPoolExecutor(max_workers=8) as ex:  # ctypes drops the GIL
        res = list(ex.map(lambda r: oracle.exp_max_ulp(*r), ranges))
    worst = max(r[0] for r in res)
    n_sub = sum(r[1] for r in res)
    assert worst <= 1.0, worst
    assert n_sub == 0


@pytest.mark.parametrize("x", [-0.34657359, -0.34657360, -0.6931472, -43.6682, -86.99])
def test_exp_reduction_boundaries(oracle, x):
    """Points where rint(x*log2e) switches n: the Cody-Waite split must hold there too."""
    for k in range(-3, 4):
        xx = struct.unpack("<f", struct.pack("<I", fbits(x) + k))[0]
        y = oracle.spc_exp(xx)
        assert abs(y - math.exp(xx)) <= 1.0 * 2.0 ** (math.frexp(math.exp(xx))[1] - 24)
