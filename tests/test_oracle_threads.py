"""The oracle's OpenMP parallelisation changes no bit (oracle/oracle.c header:
row loops split over threads, exact sums merged from per-thread exact
expansions before the single rounding).  Pinned against the serial run and
against math.fsum on sizes above the parallel threshold."""
import math

import numpy as np
import pytest

import synth
from synth import Params


@pytest.fixture
def threads(orc):
    n = orc.max_threads()
    yield n
    orc.set_mode(n, False)


def test_exact_sums_any_thread_count(orc, threads):
    rng = np.random.default_rng(4)
    a = rng.normal(size=200_003) * np.exp(rng.uniform(-30, 30, 200_003))
    b = rng.normal(size=200_003)
    for t in (1, 2, 3, max(threads, 4)):
        orc.set_mode(t, False)
        assert orc.fsum(a) == math.fsum(a)
        assert orc.sumabs(a) == math.fsum(np.abs(a))
        d = orc.dot(a, b)
        if t == 1:
            d1 = d
        assert d == d1
    # the correctly rounded dot against its definition: exact rational sum, rounded once
    from fractions import Fraction
    exact = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))
    assert d1 == float(exact)


def test_solver_and_simple_bitwise_across_threads(orc, threads):
    g = synth.make_grid(40, 32, 30)          # 38,400 cells: above the parallel threshold
    pr = Params(lin_maxit_pp=300)
    st = synth.make_state(g, 55, pr, n_scalars=1)
    out = []
    for t in (1, max(threads, 3)):
        orc.set_mode(t, False)
        s2 = {k: v.copy() for k, v in st.items()}
        ref_state, R, iters, status, rc = orc.simple_iter(g, pr, s2, n_scalars=1)
        out.append((ref_state, R, iters, status, rc))
    (a, Ra, ia, sa, _), (b, Rb, ib, sb, _) = out
    assert ia == ib and sa == sb and list(Ra) == list(Rb)
    for k in ("u", "v", "w", "p", "phi0"):
        assert np.array_equal(a[k], b[k]), k


def test_naive_mode_is_plain_sum(orc, threads):
    x = np.random.default_rng(1).normal(size=100_000)
    orc.set_mode(1, True)
    s = orc.fsum(x)
    acc = 0.0
    for v in x:
        acc += v
    assert s == acc
    orc.set_mode(threads, False)
    assert orc.fsum(x) == math.fsum(x)
