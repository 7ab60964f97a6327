"""Pins of the oracle's time loop (NEXT-3; PAPER.md:111,
PAPER.md:165; SPEC.md:388-396 adapt_dt examples)."""
import numpy as np
import pytest

import synth


def test_adapt_dt_spec_examples(orc):
    tc = orc.time_ctrl(dt=4.8e-4, dt_max=5e-4, grow=1.1, grow_threshold=3)
    assert orc.adapt_dt(tc, 2, True) and tc.dt == 5e-4            # S:393 capped at dt_max
    tc = orc.time_ctrl(dt=1e-3, shrink=0.5)
    assert not orc.adapt_dt(tc, 10, False) and tc.dt == 5e-4        # S:394 rejected, retry at half
    tc = orc.time_ctrl(dt=3e-4, grow_threshold=3)
    assert orc.adapt_dt(tc, 4, True) and tc.dt == 3e-4              # S:395 threshold + 1: unchanged
    tc = orc.time_ctrl(dt=1e-5, dt_min=1e-5)
    assert orc.adapt_dt(tc, 10, False) and tc.dt == 1e-5            # accepted at dt_min (flagged)


def test_growth_sequence_to_dt_max(orc):
    """'initially set to 1e-4 ... gradually increased to the maximum
    timestep of 5e-4': repeated fast convergence multiplies dt by `grow`."""
    tc = orc.time_ctrl(dt=1e-4, dt_max=5e-4, grow=1.1)
    seq = []
    for _ in range(25):
        orc.adapt_dt(tc, 1, True)
        seq.append(tc.dt)
    expect = []
    d = 1e-4
    for _ in range(25):
        d = min(d * 1.1, 5e-4)
        expect.append(d)
    assert seq == expect and seq[-1] == 5e-4


def small():
    g = synth.make_grid(8, 6, 10)
    pr = synth.Params(lin_maxit_pp=2000)
    st = synth.make_state(g, 21, pr)
    return g, pr, st


def test_time_step_updates_old_fields_and_time(orc):
    g, pr, st = small()
    pr.tol = 1e30                                                   # converges after one outer iteration
    tc = orc.time_ctrl(dt=2e-4, dt_max=5e-4, grow=1.25, max_outer=5)
    new, its, R, rc = orc.time_step(g, pr, st, tc)
    assert rc == 0 and its == 1 and tc.steps == 1 and tc.rejected == 0
    assert tc.time == 2e-4 and tc.dt == 2.5e-4
    for a, b in (("u", "u_old"), ("v", "v_old"), ("w", "w_old"), ("eps", "eps_old")):
        assert np.array_equal(new[a], new[b])
    ref, R1, it1, s1, rc1 = orc.simple_iter(g, synth.Params(**{**pr.__dict__, "dt": 2e-4}), st)
    assert np.array_equal(new["u"], ref["u"]) and np.array_equal(new["p"], ref["p"])


def test_rejected_attempts_leave_no_trace(orc):
    """A step rejected down to dt_min equals a step started at dt_min (the
    state is restored before every retry)."""
    g, pr, st = small()
    pr.tol = 0.0                                                    # never converged
    tc = orc.time_ctrl(dt=4e-4, dt_min=1e-4, shrink=0.5, max_outer=2)
    new, its, R, rc = orc.time_step(g, pr, st, tc)
    assert rc == 1 and tc.rejected == 2 and tc.dt == 1e-4 and tc.time == 1e-4
    tc2 = orc.time_ctrl(dt=1e-4, dt_min=1e-4, max_outer=2)
    ref, its2, R2, rc2 = orc.time_step(g, pr, st, tc2)
    for k in ("u", "v", "w", "p", "u_old"):
        assert np.array_equal(new[k], ref[k]), k
