"""Pins for the oracle's correctly rounded sums (reading Q17).

Independent references: Python's math.fsum (CPython's own C implementation)
and exact rational arithmetic with fractions.Fraction, whose float() rounds
correctly (int/int true division is correctly rounded).
"""
import math
from fractions import Fraction

import numpy as np
import pytest


def exact_dot(a, b):
    return float(sum((Fraction(x) * Fraction(y) for x, y in zip(a, b)), Fraction(0)))


@pytest.mark.parametrize("seed", range(6))
def test_fsum_matches_math_fsum(orc, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=3000) * 10.0 ** rng.integers(-30, 30, 3000)
    x = np.concatenate([x, -x[:1500] * (1 + 1e-15)])  # heavy cancellation
    rng.shuffle(x)
    assert orc.fsum(x) == math.fsum(x)


@pytest.mark.parametrize("seed", range(8))
def test_dot_is_correctly_rounded(orc, seed):
    rng = np.random.default_rng(100 + seed)
    n = 200
    a = rng.normal(size=n) * 10.0 ** rng.integers(-8, 8, n)
    b = rng.normal(size=n)
    if seed % 2:  # ill-conditioned: make the dot nearly cancel
        b[-1] = 0.0
        partial = exact_dot(a[:-1], b[:-1])
        b[-1] = -partial / a[-1]
    assert orc.dot(a, b) == exact_dot(a, b)


def test_dot_half_way_rounding(orc):
    # exact value 1 + 2^-53 is a tie between 1 and 1+2^-52: round-half-even gives 1.0
    a = np.array([1.0, 2.0 ** -27])
    b = np.array([1.0, 2.0 ** -26])
    assert orc.dot(a, b) == 1.0
    # 1 + 2^-53 + 2^-80 is above the tie: rounds up
    a = np.array([1.0, 2.0 ** -27, 2.0 ** -40])
    b = np.array([1.0, 2.0 ** -26, 2.0 ** -40])
    assert orc.dot(a, b) == 1.0 + 2.0 ** -52


def test_dot_zero_and_sign(orc):
    assert math.copysign(1.0, orc.dot(np.array([-0.0]), np.array([1.0]))) == 1.0
    assert orc.dot(np.zeros(0), np.zeros(0)) == 0.0
    a = np.array([1e300, 1.0, -1e300])
    assert orc.dot(a, np.ones(3)) == 1.0


def test_sumabs(orc):
    rng = np.random.default_rng(7)
    x = rng.normal(size=5000) * 10.0 ** rng.integers(-10, 10, 5000)
    assert orc.sumabs(x) == math.fsum(np.abs(x))
