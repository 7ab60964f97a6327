"""Pins for the oracle's 7-point operator and BiCGSTAB.

The 7-point operator is pinned against a dense matrix assembled directly from
the coefficient arrays in numpy (brute force, independent indexing); BiCGSTAB
against numpy.linalg.solve, the SPEC worked examples and
the k-distinct-eigenvalue termination property of Krylov methods.
"""
import json
import os

import numpy as np
import pytest

import synth
from synth import Grid

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def dense_from_arrays(g, s, sym=False):
    """A[n,n] = aP, A[n,nb] = -a_nb, built with numpy index arithmetic."""
    nx, ny, nz = g.nx, g.ny, g.nz
    n = g.n
    A = np.zeros((n, n))
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    idx = i + nx * (j + ny * k)
    A[idx, idx] = s["aP"][idx]
    offs = {"W": (-1, 0, 0), "E": (1, 0, 0), "S": (0, -1, 0), "N": (0, 1, 0), "B": (0, 0, -1), "T": (0, 0, 1)}
    for name, (di, dj, dk) in offs.items():
        ii, jj, kk = i + di, j + dj, k + dk
        ok = (ii >= 0) & (ii < nx) & (jj >= 0) & (jj < ny) & (kk >= 0) & (kk < nz)
        src = idx[ok]
        dst = (ii + nx * (jj + ny * kk))[ok]
        if sym:
            # a_E(n) = c_x[n], a_W(n) = c_x[n-1]
            arr = {"E": "aE", "N": "aN", "T": "aT", "W": "aE", "S": "aN", "B": "aT"}[name]
            coef = s[arr][src] if name in "ENT" else s[arr][dst]
        else:
            coef = s["a" + name][src]
        A[src, dst] = -coef
    return A


def random_mom_system(g, seed, dominance=1.0):
    rng = np.random.default_rng(seed)
    n = g.n
    s = {k: rng.uniform(0.1, 1.0, n) for k in ("aE", "aW", "aN", "aS", "aT", "aB")}
    tot = sum(s[k] for k in ("aE", "aW", "aN", "aS", "aT", "aB"))
    s["aP"] = tot * (1.0 + dominance) + rng.uniform(0, 0.1, n)
    s["b"] = rng.normal(size=n)
    s["d"] = np.zeros(n)
    return s


def random_pp_system(g, seed):
    rng = np.random.default_rng(seed)
    n = g.n
    s = {k: rng.uniform(0.1, 1.0, n) for k in ("aE", "aN", "aT")}
    nx, ny = g.nx, g.ny
    k, j, i = np.meshgrid(np.arange(g.nz), np.arange(ny), np.arange(nx), indexing="ij")
    s["aE"][(i == nx - 1).ravel()] = 0.0
    s["aN"][(j == ny - 1).ravel()] = 0.0
    cx, cy, cz = (s["aE"].reshape(g.nz, ny, nx), s["aN"].reshape(g.nz, ny, nx), s["aT"].reshape(g.nz, ny, nx))
    ap = cx + cy + cz
    ap[:, :, 1:] += cx[:, :, :-1]
    ap[:, 1:, :] += cy[:, :-1, :]
    ap[1:, :, :] += cz[:-1, :, :]
    s["aP"] = ap.ravel()
    s["b"] = rng.normal(size=n)
    return s


@pytest.mark.parametrize("shape", [(2, 2, 2), (5, 3, 4), (4, 6, 3)])
def test_spmv_dense_brute_force(orc, shape):
    g = Grid(*shape, 1.0, 1.0, 1.0)
    s = random_mom_system(g, 1)
    x = np.random.default_rng(2).normal(size=g.n)
    y = orc.spmv(g, s, x)
    ref = dense_from_arrays(g, s) @ x
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-13 * np.abs(s["aP"]).max())


@pytest.mark.parametrize("shape", [(3, 4, 5), (6, 2, 3)])
def test_spmv_symmetric_storage(orc, shape):
    g = Grid(*shape, 1.0, 1.0, 1.0)
    s = random_pp_system(g, 3)
    x = np.random.default_rng(4).normal(size=g.n)
    y = orc.spmv(g, s, x)
    A = dense_from_arrays(g, s, sym=True)
    assert np.array_equal(A, A.T)
    assert np.allclose(y, A @ x, rtol=1e-13, atol=1e-13 * s["aP"].max())
    # the oracle's own unit-vector matrix agrees exactly with the numpy one
    assert np.array_equal(orc.dense_matrix(g, s), A)


@pytest.mark.parametrize("shape,seed", [((4, 4, 4), 0), ((8, 8, 8), 1), ((5, 7, 3), 2)])
def test_bicgstab_vs_dense_lu(orc, shape, seed):
    g = Grid(*shape, 1.0, 1.0, 1.0)
    s = random_mom_system(g, seed, dominance=0.05)
    A = dense_from_arrays(g, s)
    xe = np.linalg.solve(A, s["b"])
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-13, 1000)
    assert res["status"] == 0
    kappa = np.linalg.cond(A)
    assert np.linalg.norm(res["x"] - xe) <= 10 * kappa * 1e-13 * np.linalg.norm(xe)
    # the returned (recursive) residual obeys the stopping rule
    assert res["rel_resid"] <= 1e-13


def test_bicgstab_symmetric_vs_dense_lu(orc):
    g = Grid(6, 5, 4, 1.0, 1.0, 1.0)
    s = random_pp_system(g, 9)
    # make it nonsingular like the outlet p' system: extra diagonal on top layer
    k = np.arange(g.n) // (g.nx * g.ny)
    s["aP"] = s["aP"] + np.where(k == g.nz - 1, 0.5, 0.0)
    A = dense_from_arrays(g, s, sym=True)
    xe = np.linalg.solve(A, s["b"])
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-12, 2000)
    assert res["status"] == 0
    assert np.linalg.norm(res["x"] - xe) <= 10 * np.linalg.cond(A) * 1e-12 * np.linalg.norm(xe)


def test_bicgstab_identity_one_iteration(orc):
    """identity stencil -> x = b in <= 1 iteration."""
    g = Grid(3, 3, 3, 1.0, 1.0, 1.0)
    n = g.n
    s = {k: np.zeros(n) for k in ("aE", "aW", "aN", "aS", "aT", "aB", "d")}
    s["aP"] = np.ones(n)
    s["b"] = np.random.default_rng(0).normal(size=n)
    res = orc.bicgstab(g, s, np.zeros(n), 1e-10, 50)
    assert res["iters"] <= GOLD["bicgstab_identity"]["max_iters"]
    assert np.array_equal(res["x"], s["b"])


def test_bicgstab_2x2(orc):
    """[[2,-1],[-1,2]] x = (1,1) -> x = (1,1); pairs of cells along x."""
    gold = GOLD["bicgstab_2x2"]
    g = Grid(2, 2, 2, 1.0, 1.0, 1.0)
    n = g.n
    s = {k: np.zeros(n) for k in ("aE", "aW", "aN", "aS", "aT", "aB", "d")}
    i = np.arange(n) % 2
    s["aP"] = np.full(n, gold["A"][0][0])
    s["aE"] = np.where(i == 0, -gold["A"][0][1], 0.0)
    s["aW"] = np.where(i == 1, -gold["A"][1][0], 0.0)
    s["b"] = np.full(n, gold["b"][0])
    res = orc.bicgstab(g, s, np.zeros(n), 1e-14, 10)
    assert res["status"] == 0
    assert np.allclose(res["x"], gold["x"][0], rtol=0, atol=1e-15)


def test_bicgstab_zero_rhs(orc):
    """b = 0 -> x = 0 in 0 iterations (even from a nonzero x0)."""
    g = Grid(3, 2, 2, 1.0, 1.0, 1.0)
    s = random_mom_system(g, 5)
    s["b"] = np.zeros(g.n)
    res = orc.bicgstab(g, s, np.ones(g.n), 1e-6, 10)
    assert res["iters"] == GOLD["bicgstab_zero_rhs"]["iters"] and res["status"] == 0
    assert np.all(res["x"] == 0.0)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_bicgstab_k_eigenvalues(orc, k):
    """A diagonal A with k distinct eigenvalues: the Krylov space has dimension
    k, so BiCGSTAB (exact arithmetic) hits s = 0 at the half step of iteration k."""
    g = Grid(4, 4, 4, 1.0, 1.0, 1.0)
    n = g.n
    rng = np.random.default_rng(k)
    s = {kk: np.zeros(n) for kk in ("aE", "aW", "aN", "aS", "aT", "aB", "d")}
    eig = np.array([1.0, 2.5, 4.0, 7.0])[:k]
    s["aP"] = eig[rng.integers(0, k, n)]
    s["aP"][:k] = eig  # every eigenvalue present
    s["b"] = rng.normal(size=n)
    res = orc.bicgstab(g, s, np.zeros(n), 1e-10, 50)
    assert res["status"] == 0
    assert res["iters"] == k
    assert np.allclose(res["x"], s["b"] / s["aP"], rtol=1e-9)


def test_bicgstab_manufactured(orc):
    g = Grid(6, 5, 7, 1.0, 1.0, 1.0)
    s = random_mom_system(g, 11, dominance=0.2)
    xe = np.random.default_rng(12).normal(size=g.n)
    s["b"] = orc.spmv(g, s, xe)
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-12, 500)
    assert res["status"] == 0
    assert np.linalg.norm(res["x"] - xe) <= 1e-10 * np.linalg.norm(xe)


def test_bicgstab_deterministic(orc):
    g = Grid(6, 5, 7, 1.0, 1.0, 1.0)
    s = random_pp_system(g, 13)
    s["aP"] = s["aP"] * 1.001
    r1 = orc.bicgstab(g, s, np.zeros(g.n), 1e-9, 300, trace=True)
    r2 = orc.bicgstab(g, s, np.zeros(g.n), 1e-9, 300, trace=True)
    assert r1["iters"] == r2["iters"]
    assert np.array_equal(r1["x"], r2["x"]) and np.array_equal(r1["trace"], r2["trace"])


def test_bicgstab_breakdown_restart_once(orc):
    """sigma = <r^,A p> = 0 for the rotation [[0,1],[-1,0]] with b = (1,0):
    restart once (r^ <- r), meet sigma = 0 again -> BREAKDOWN after 2 iterations
    (reading Q4)."""
    g = Grid(2, 2, 2, 1.0, 1.0, 1.0)
    n = g.n
    i = np.arange(n) % 2
    s = {k: np.zeros(n) for k in ("aE", "aW", "aN", "aS", "aT", "aB", "d")}
    s["aP"] = np.zeros(n)
    s["aE"] = np.where(i == 0, -1.0, 0.0)   # A[0,1] = -aE = +1
    s["aW"] = np.where(i == 1, 1.0, 0.0)    # A[1,0] = -aW = -1
    s["b"] = np.where(i == 0, 1.0, 0.0)
    res = orc.bicgstab(g, s, np.zeros(n), 1e-8, 20)
    assert res["status"] == -4 and res["iters"] == 2 and res["restarts"] == 1


def test_bicgstab_not_converged_returns_last_iterate(orc):
    g = Grid(8, 8, 8, 1.0, 1.0, 1.0)
    s = random_pp_system(g, 21)
    s["aP"] = s["aP"] * 1.0001
    r5 = orc.bicgstab(g, s, np.zeros(g.n), 1e-14, 5)
    r6 = orc.bicgstab(g, s, np.zeros(g.n), 1e-14, 6, trace=True)
    assert r5["status"] == 1 and r5["iters"] == 5
    assert not np.array_equal(r5["x"], r6["x"])
