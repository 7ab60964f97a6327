"""GPU parity: libmfx.so (through the C ABI) vs the CPU oracle on identical
seeded inputs.  Gate (BASELINE.json north_star): relative L2 <= 1e-9 in the
solution and the same iteration count +-1; under the arithmetic contract of
DESIGN.md §3 the results are expected to be bitwise identical, which is
asserted for the assembly, the 7-point apply and the correction.
"""
import numpy as np
import pytest

import synth
from synth import Grid, Params, BC_WALL, BC_INLET, BC_OUTLET, BC_DIRICHLET_TEST

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL_L2 = 1e-9


@pytest.fixture(scope="module")
def mfx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15605_b200 as m
    return m


@pytest.fixture(params=["tma", "cluster", "cluster8", "v1", "grid", "persist"])
def solver_path(request, mfx):
    """cluster: the single-cluster solver at its default size (16 CTAs where the
    device places such a cluster); cluster8: the same kernel on 8 CTAs."""
    v = {"tma": mfx.PATH_TMA, "cluster": mfx.PATH_CLUSTER, "cluster8": mfx.PATH_CLUSTER, "v1": mfx.PATH_V1,
         "grid": mfx.PATH_GRID, "persist": mfx.PATH_PERSIST}[request.param]
    cl = mfx.get_option("cluster_size")
    if request.param == "cluster8":
        mfx.set_option("cluster_size", 8)
    mfx.set_option("solver_path", v)
    yield "cluster" if request.param == "cluster8" else request.param
    mfx.set_option("solver_path", mfx.PATH_AUTO)
    mfx.set_option("cluster_size", cl)


def cluster_fits(g, sym):
    # bicg_cluster.cu: (NA + 8) slab arrays + 5 planes (fp64) + slab flags (int32) <= 200 KiB
    import paper_2211_15605_b200 as m_
    cl = m_.get_option("cluster_size")
    plane = g.nx * g.ny
    m = plane * -(-g.nz // cl)
    return ((11 if sym else 15) * m + 5 * plane) * 8 + 4 * m <= 200 * 1024


def need_path(solver_path, g, sym):
    if solver_path == "cluster" and not cluster_fits(g, sym):
        pytest.skip("system does not fit the single-cluster solver")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def state_dev(st):
    return {k: dev(v) for k, v in st.items()}


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# grids: named configs plus ragged shapes (ny, nz odd / not tile multiples;
# "odd": odd nx, rows not 16-byte aligned -> grid-stride kernels, same bits)
GRIDS = {
    "c1": (16, 16, 32),
    "rag1": (10, 7, 9),
    "rag2": (34, 19, 23),
    "thin": (2, 2, 2),
    "tall": (6, 5, 41),
    "tiles": (70, 21, 45),     # several 32x8 assembly tiles with ragged x/y tails
    "odd": (9, 7, 13),
}


@pytest.fixture(params=["tma", "gridstride"])
def asm_path(request, mfx):
    mfx.set_option("asm_tma", 1 if request.param == "tma" else 0)
    yield request.param
    mfx.set_option("asm_tma", 1)


def case(name, seed=0, n_scalars=1, bc_zhi=BC_OUTLET):
    nx, ny, nz = GRIDS[name]
    g = synth.make_grid(nx, ny, nz, bc_zhi=bc_zhi)
    pr = Params()
    st = synth.make_state(g, 1000 + seed + nx * 7 + nz, pr, n_scalars=n_scalars)
    if n_scalars:
        rng = np.random.default_rng(seed)
        st["phi0"] = rng.uniform(0, 1, g.n)
        st["phi_old0"] = rng.uniform(0, 1, g.n)
    return g, pr, st


# ---------------------------------------------------------------- a-1/a-2/a-3 assembly
@pytest.mark.parametrize("name", list(GRIDS))
@pytest.mark.parametrize("comp", [0, 1, 2])
def test_assemble_momentum_bitwise(mfx, orc, name, comp, asm_path):
    g, pr, st = case(name)
    ref, r2, rc = orc.assemble_mom(g, pr, comp, st)
    ws = mfx.Workspace(g)
    out, res2 = mfx.assemble_eq(comp, g, pr, state_dev(st), ws)
    ws.check()
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d"):
        assert np.array_equal(host(out[k]), ref[k]), k
    assert np.array_equal(host(res2), r2)


@pytest.mark.parametrize("name", ["c1", "rag2", "thin", "tiles"])
@pytest.mark.parametrize("bc_zhi", [BC_OUTLET, BC_WALL])
def test_assemble_momentum_bc_variants(mfx, orc, name, bc_zhi, asm_path):
    g, pr, st = case(name, bc_zhi=bc_zhi)
    for comp in range(3):
        ref, r2, _ = orc.assemble_mom(g, pr, comp, st)
        ws = mfx.Workspace(g)
        out, res2 = mfx.assemble_eq(comp, g, pr, state_dev(st), ws)
        for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d"):
            assert np.array_equal(host(out[k]), ref[k]), (comp, k)


@pytest.mark.parametrize("name", list(GRIDS))
def test_assemble_pp_bitwise(mfx, orc, name):
    g, pr, st = case(name)
    rng = np.random.default_rng(1)
    star = [st["u"] + rng.normal(0, 1e-3, g.n), st["v"], st["w"] * 1.01]
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    ref, cont, rc = orc.assemble_pp(g, pr, st, star, dv)
    ws = mfx.Workspace(g)
    out, res2 = mfx.assemble_eq(mfx.EQ_PP, g, pr, state_dev(st), ws, star=[dev(a) for a in star + dv])
    for k in ("aP", "aE", "aN", "aT", "b"):
        assert np.array_equal(host(out[k]), ref[k]), k
    assert host(res2)[0] == cont


@pytest.mark.parametrize("name", list(GRIDS))
@pytest.mark.parametrize("bc_zhi", [BC_OUTLET, BC_DIRICHLET_TEST])
def test_assemble_scalar_bitwise(mfx, orc, name, bc_zhi):
    g, pr, st = case(name, bc_zhi=bc_zhi)
    ref, r2, _ = orc.assemble_scalar(g, pr, 0, st)
    ws = mfx.Workspace(g)
    out, res2 = mfx.assemble_eq(mfx.EQ_SCALAR, g, pr, state_dev(st), ws, scalar_id=0)
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b"):
        assert np.array_equal(host(out[k]), ref[k]), k
    assert np.array_equal(host(res2), r2)


# ---------------------------------------------------------------- a-4 apply
@pytest.mark.parametrize("name", list(GRIDS))
def test_spmv_bitwise(mfx, orc, name):
    g, pr, st = case(name)
    ref, _, _ = orc.assemble_mom(g, pr, 2, st)
    x = np.random.default_rng(3).normal(size=g.n)
    y = mfx.spmv(mfx.EQ_W, g, {k: dev(v) for k, v in ref.items()}, dev(x))
    assert np.array_equal(host(y), orc.spmv(g, ref, x))
    dv = [np.random.default_rng(4 + a).uniform(1e-4, 1e-3, g.n) for a in range(3)]
    pp, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    y = mfx.spmv(mfx.EQ_PP, g, {k: dev(v) for k, v in pp.items()}, dev(x))
    assert np.array_equal(host(y), orc.spmv(g, pp, x))


# ---------------------------------------------------------------- a-5/a-6 BiCGSTAB
def solve_both(mfx, orc, g, kind, sysd, x0, tol, maxit):
    ref = orc.bicgstab(g, sysd, x0, tol, maxit)
    ws = mfx.Workspace(g)
    x = dev(x0)
    info = mfx.bicgstab_solve(kind, g, {k: dev(v) for k, v in sysd.items()}, x, tol, maxit, ws)
    return ref, info, host(x)


def assert_solve_parity(ref, info, x):
    assert abs(info["iters"] - ref["iters"]) <= 1, (info, ref["iters"])
    assert info["status"] == ref["status"]
    assert rel_l2(x, ref["x"]) <= REL_L2
    # expected under the arithmetic contract: bitwise
    assert info["iters"] == ref["iters"] and np.array_equal(x, ref["x"])


@pytest.mark.parametrize("name", list(GRIDS))
@pytest.mark.parametrize("comp", [0, 2])
def test_bicgstab_momentum_parity(mfx, orc, name, comp, solver_path):
    g, pr, st = case(name)
    need_path(solver_path, g, False)
    sysd, _, _ = orc.assemble_mom(g, pr, comp, st)
    x0 = [st["u"], st["v"], st["w"]][comp]
    ref, info, x = solve_both(mfx, orc, g, comp, sysd, x0, 1e-10, 200)
    assert_solve_parity(ref, info, x)


def test_bicgstab_pp_c1_parity(mfx, orc, solver_path):
    """Configuration 1 (BASELINE.json): p' BiCGSTAB on 16x16x32 with bed contrast,
    tol 1e-6, maxit 5000 (SURVEY §8d c1 procedure)."""
    g, pr, st = synth.config_case(1)
    pr.lin_maxit_pp = 5000
    star, dv = [], []
    for c in range(3):
        s, _, _ = orc.assemble_mom(g, pr, c, st)
        star.append(orc.bicgstab(g, s, [st["u"], st["v"], st["w"]][c], pr.lin_tol_mom, pr.lin_maxit_mom)["x"])
        dv.append(s["d"])
    sysd, _, _ = orc.assemble_pp(g, pr, st, star, dv)
    ref, info, x = solve_both(mfx, orc, g, mfx.EQ_PP, sysd, np.zeros(g.n), pr.lin_tol_pp, 5000)
    assert ref["status"] == 0 and ref["iters"] > 50
    assert_solve_parity(ref, info, x)


@pytest.mark.parametrize("name", ["rag1", "rag2", "tall"])
def test_bicgstab_pp_ragged_parity(mfx, orc, name, solver_path):
    g, pr, st = case(name)
    need_path(solver_path, g, True)
    dv = [np.random.default_rng(9 + a).uniform(1e-4, 1e-3, g.n) for a in range(3)]
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    ref, info, x = solve_both(mfx, orc, g, mfx.EQ_PP, sysd, np.zeros(g.n), 1e-8, 3000)
    assert_solve_parity(ref, info, x)


def test_pp_diagonal_derived_not_read(mfx, orc, solver_path):
    """p' kind: every path rebuilds a_P as the ordered row sum
    and never reads A->aP -- a NaN-poisoned or absent aP changes no bit."""
    g, pr, st = case("rag2")
    need_path(solver_path, g, True)
    dv = [np.random.default_rng(21 + a).uniform(1e-4, 1e-3, g.n) for a in range(3)]
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    ref = orc.bicgstab(g, sysd, np.zeros(g.n), 1e-9, 400)
    x = np.random.default_rng(5).normal(size=g.n)
    yref = orc.spmv(g, sysd, x)
    for variant in ("nan", "absent"):
        d = {k: dev(v) for k, v in sysd.items()}
        if variant == "nan":
            d["aP"] = torch.full_like(d["aP"], float("nan"))
        else:
            del d["aP"]
        assert np.array_equal(host(mfx.spmv(mfx.EQ_PP, g, d, dev(x))), yref), variant
        ws = mfx.Workspace(g)
        xs = torch.zeros(g.n, dtype=torch.float64, device="cuda")
        info = mfx.bicgstab_solve(mfx.EQ_PP, g, d, xs, 1e-9, 400, ws)
        assert info["iters"] == ref["iters"] and np.array_equal(host(xs), ref["x"]), variant


@pytest.mark.parametrize("maxit", [0, 1, 2, 7])
def test_bicgstab_not_converged_last_iterate(mfx, orc, maxit, solver_path):
    g, pr, st = case("rag2")
    need_path(solver_path, g, True)
    dv = [np.full(g.n, 5e-4)] * 3
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    ref, info, x = solve_both(mfx, orc, g, mfx.EQ_PP, sysd, np.zeros(g.n), 1e-14, maxit)
    assert ref["status"] == 1 and info["status"] == 1 and info["iters"] == maxit
    assert np.array_equal(x, ref["x"])


def test_bicgstab_edge_cases(mfx, orc, solver_path):
    g = Grid(4, 2, 2, 1.0, 1.0, 1.0)
    n = g.n
    z = {k: np.zeros(n) for k in ("aE", "aW", "aN", "aS", "aT", "aB", "d")}
    # b = 0 from nonzero x0 -> x = 0, 0 iterations
    s = dict(z, aP=np.full(n, 2.0), b=np.zeros(n))
    ref, info, x = solve_both(mfx, orc, g, 0, s, np.ones(n), 1e-6, 10)
    assert info["iters"] == 0 and info["status"] == 0 and np.all(x == 0.0)
    # identity -> x = b in 1 iteration
    s = dict(z, aP=np.ones(n), b=np.arange(n, dtype=float) + 1)
    ref, info, x = solve_both(mfx, orc, g, 0, s, np.zeros(n), 1e-10, 10)
    assert info["iters"] == 1 and np.array_equal(x, s["b"])
    # rotation pairs: sigma = 0 -> restart -> BREAKDOWN after 2 iterations
    i = np.arange(n) % 2
    s = dict(z, aP=np.zeros(n), aE=np.where(i == 0, -1.0, 0.0), aW=np.where(i == 1, 1.0, 0.0),
             b=np.where(i == 0, 1.0, 0.0))
    ref, info, x = solve_both(mfx, orc, g, 0, s, np.zeros(n), 1e-8, 20)
    assert (info["status"], info["iters"], info["restarts"]) == (ref["status"], ref["iters"], ref["restarts"]) == (-4, 2, 1)
    # x0 already the solution -> 0 iterations
    s = dict(z, aP=np.full(n, 3.0), b=np.full(n, 3.0))
    ref, info, x = solve_both(mfx, orc, g, 0, s, np.ones(n), 1e-6, 10)
    assert info["iters"] == 0 and np.array_equal(x, np.ones(n))


def test_bicgstab_deterministic(mfx, orc, solver_path):
    g, pr, st = case("rag2")
    need_path(solver_path, g, True)
    dv = [np.full(g.n, 5e-4)] * 3
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    d = {k: dev(v) for k, v in sysd.items()}
    ws = mfx.Workspace(g)
    xs = []
    for _ in range(3):
        x = torch.zeros(g.n, dtype=torch.float64, device="cuda")
        mfx.bicgstab_solve(mfx.EQ_PP, g, d, x, 1e-8, 500, ws)
        xs.append(host(x))
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[0], xs[2])


# ---------------------------------------------------------------- a-7 correction
@pytest.mark.parametrize("name", list(GRIDS))
def test_correct_bitwise(mfx, orc, name):
    g, pr, st = case(name)
    rng = np.random.default_rng(5)
    star = [st["u"], st["v"], st["w"]]
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    pp = rng.normal(size=g.n)
    ref = orc.correct(g, pr, star, dv, pp, st["p"])
    out = mfx.correct(g, pr, [dev(a) for a in star + dv], dev(pp), dev(st["p"]))
    for a, b in zip(out, ref):
        assert np.array_equal(host(a), b)


# ---------------------------------------------------------------- a-9 SIMPLE
@pytest.mark.parametrize("name,n_scalars", [("c1", 0), ("rag2", 1), ("tall", 2), ("odd", 1)])
def test_simple_iter_111_parity(mfx, orc, name, n_scalars, solver_path):
    g, pr, st = case(name, n_scalars=n_scalars)
    need_path(solver_path, g, False)
    pr.lin_maxit_pp = 2000
    asg = "111[1]" + "1" * n_scalars
    ctx = mfx.SimpleContext(asg, g, pr)
    sd = state_dev(st)
    ref_state = st
    for it in range(2):
        ref_state, R, iters, status, rc = orc.simple_iter(g, pr, ref_state, n_scalars=n_scalars)
        out = ctx.step(sd)
        assert out["iters"][:4] == iters[:4], (out["iters"], iters)
        assert np.array_equal(np.array(out["R"]), R)
        for k in ("u", "v", "w", "p") + tuple(f"phi{s}" for s in range(n_scalars)):
            a, b = host(sd[k]), ref_state[k]
            assert rel_l2(a, b) <= REL_L2
            assert np.array_equal(a, b), k
    times = ctx.phase_times()
    assert times["total"] > 0
    ctx.close()


# ---------------------------------------------------------------- errors
def test_argument_errors(mfx):
    g = Grid(1, 4, 4, 1.0, 1.0, 1.0)        # extent < 2
    with pytest.raises(mfx.MfxError) as e:
        mfx.Workspace(synth.make_grid(4, 4, 4))  # fine
        mfx.spmv(0, g, {k: torch.zeros(16, dtype=torch.float64, device="cuda") for k in mfx.SYS_KEYS},
                 torch.zeros(16, dtype=torch.float64, device="cuda"))
    assert e.value.status == mfx.ERR_ARG and ">= 2" in str(e.value)


def test_misaligned_arrays_refused_on_tma_path(mfx, orc):
    """TMA tensor maps need 16-byte aligned arrays: an 8-byte aligned view is
    refused before any launch (even nx); with odd nx the grid-stride kernels
    accept it and give the oracle's bits."""
    g, pr, st = case("rag2")
    ref, _, _ = orc.assemble_mom(g, pr, 0, st)
    sysd = {k: torch.from_numpy(ref[k]).cuda() for k in mfx.SYS_KEYS}
    x = np.random.default_rng(5).normal(size=g.n)
    buf = torch.zeros(g.n + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(x).cuda()
    with pytest.raises(mfx.MfxError) as e:
        mfx.spmv(0, g, sysd, buf[1:])
    assert e.value.status == mfx.ERR_ARG and "aligned" in str(e.value)
    go, pro, sto = case("odd")
    refo, _, _ = orc.assemble_mom(go, pro, 0, sto)
    sysd = {k: torch.from_numpy(refo[k]).cuda() for k in mfx.SYS_KEYS}
    xo = np.random.default_rng(6).normal(size=go.n)
    bufo = torch.zeros(go.n + 1, dtype=torch.float64, device="cuda")
    bufo[1:] = torch.from_numpy(xo).cuda()
    assert np.array_equal(host(mfx.spmv(0, go, sysd, bufo[1:])), orc.spmv(go, refo, xo))


def test_nonfinite_latched(mfx):
    g, pr, st = case("rag1")
    st = dict(st)
    st["eps"] = st["eps"].copy()
    st["eps"][37] = np.nan
    ws = mfx.Workspace(g)
    mfx.assemble_eq(0, g, pr, state_dev(st), ws)
    with pytest.raises(mfx.MfxError) as e:
        ws.check()
    assert e.value.status == mfx.ERR_NONFINITE
    ws.check()  # latch cleared


@pytest.mark.parametrize("bc_zlo,w_in", [(BC_INLET, 0.15), (BC_WALL, 0.0)])
def test_simple_outer_loop_parity(mfx, orc, bc_zlo, w_in):
    """Ten consecutive SIMPLE outer iterations (state m -> m+10) on GPU and oracle:
    bitwise identical states, residual records and iteration counts at every
    iteration, with an inlet or a bottom wall (top outlet in both: the p'
    system needs the outlet's Dirichlet ghost)."""
    g = synth.make_grid(12, 10, 16, bc_zlo=bc_zlo, w_in=w_in)
    pr = Params(lin_maxit_pp=3000, lin_tol_pp=1e-8)
    st = synth.make_state(g, 777, pr)
    ctx = mfx.SimpleContext("111[1]", g, pr)
    sd = state_dev(st)
    ref = st
    Rs = []
    for it in range(10):
        ref, R, iters, status, rc = orc.simple_iter(g, pr, ref)
        out = ctx.step(sd)
        assert out["iters"][:4] == iters[:4], (it, out["iters"], iters)
        assert np.array_equal(np.array(out["R"]), R), it
        for k in ("u", "v", "w", "p"):
            assert np.array_equal(host(sd[k]), ref[k]), (it, k)
        Rs.append(max(R))
    assert all(np.isfinite(Rs))
    ctx.close()


def test_simple_thin_grid(mfx, orc):
    """Degenerate extents: 2 x 2 x 2 cells (every row touches a boundary)."""
    g = synth.make_grid(2, 2, 2)
    pr = Params()
    st = synth.make_state(g, 31, pr)
    ref, R, iters, status, rc = orc.simple_iter(g, pr, st)
    ctx = mfx.SimpleContext("111[1]", g, pr)
    sd = state_dev(st)
    out = ctx.step(sd)
    assert out["iters"][:4] == iters[:4]
    for k in ("u", "v", "w", "p"):
        assert np.array_equal(host(sd[k]), ref[k]), k
    ctx.close()


def test_simple_iter_reports_nonfinite(mfx):
    """A NaN in the void fraction is latched by the assembly and reported by
    mfx_simple_iter as MFX_ERR_NONFINITE with the cell index."""
    g, pr, st = case("rag1")
    st = dict(st)
    st["eps"] = st["eps"].copy()
    st["eps"][50] = np.nan
    ctx = mfx.SimpleContext("111[1]", g, pr)
    with pytest.raises(mfx.MfxError) as e:
        ctx.step(state_dev(st))
    assert e.value.status == mfx.ERR_NONFINITE and "cell" in str(e.value)
    ctx.close()


# ---------------------------------------------------------------- graph cache and exit residual
def _pp_system(orc, g, seed):
    pr = Params()
    st = synth.make_state(g, seed, pr)
    dv = [np.random.default_rng(seed + a).uniform(1e-4, 1e-3, g.n) for a in range(3)]
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    return sysd


def test_graph_cache_same_n_different_shape(mfx, orc):
    """Two p' systems with equal N and different shapes solved back to back in
    the SAME device buffers, with enough iterations that the 16-iteration CUDA
    graphs engage: each must equal the oracle bitwise (the cached graph bakes
    in tensor maps and tiles, so it must be keyed on the shape)."""
    shapes = [(64, 32, 40), (32, 64, 40), (64, 32, 40)]
    n = 64 * 32 * 40
    bufs = {k: torch.empty(n, dtype=torch.float64, device="cuda") for k in ("aP", "aE", "aN", "aT", "b")}
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = mfx.Workspace(synth.make_grid(*shapes[0]))
    mfx.set_option("graphs", 1)
    for q, shp in enumerate(shapes):
        g = synth.make_grid(*shp)
        sysd = _pp_system(orc, g, 300 + q)
        for k in bufs:
            bufs[k].copy_(torch.from_numpy(sysd[k]))
        x.zero_()
        ref = orc.bicgstab(g, sysd, np.zeros(n), 1e-12, 48)
        info = mfx.bicgstab_solve(mfx.EQ_PP, g, bufs, x, 1e-12, 48, ws)
        assert ref["iters"] == 48 and info["iters"] == 48, (shp, ref["iters"], info["iters"])
        assert np.array_equal(host(x), ref["x"]), shp
    assert mfx.graph_cache_size() >= 2
    mfx.graph_cache_clear()
    assert mfx.graph_cache_size() == 0


def test_true_rel_resid_matches_oracle(mfx, orc):
    """mfx_solve_info.true_rel_resid = ||b - A x|| / ||b|| of the returned
    iterate (reading Q2), computed once at exit with the canonical operator and
    correctly rounded dots: bitwise the oracle's composition of the same
    definitions; for a capped solve it differs from the recursive residual."""
    g = synth.make_grid(34, 19, 23)
    sysd = _pp_system(orc, g, 77)
    for tol, maxit in ((1e-8, 3000), (0.0, 40)):
        ref = orc.bicgstab(g, sysd, np.zeros(g.n), tol, maxit)
        x = torch.zeros(g.n, dtype=torch.float64, device="cuda")
        info = mfx.bicgstab_solve(mfx.EQ_PP, g, {k: dev(v) for k, v in sysd.items()}, x, tol, maxit,
                                  mfx.Workspace(g))
        r = sysd["b"] - orc.spmv(g, sysd, ref["x"])
        want = np.sqrt(orc.dot(r, r)) / np.sqrt(orc.dot(sysd["b"], sysd["b"]))
        assert info["true_rel_resid"] == want, (info, want)
        assert info["true_rel_resid"] > 0.0


@pytest.mark.parametrize("cl", [16, 8])
def test_cluster_solver_back_to_back_shapes(mfx, orc, cl):
    """Single-cluster solver: different systems back to back (shared memory
    left over from the previous launch holds another system's slabs -- a
    missing barrier after a shared-memory fill reads those stale values
    instead of failing loudly), each bitwise vs the oracle; ragged slab splits
    (nz not a multiple of the cluster size) included."""
    prev = mfx.get_option("cluster_size")
    mfx.set_option("cluster_size", cl)
    mfx.set_option("solver_path", mfx.PATH_CLUSTER)
    try:
        for (nx, ny, nz) in ((16, 16, 32), (8, 8, 48), (16, 16, 20), (16, 16, 32), (12, 10, 37)):
            g = synth.make_grid(nx, ny, nz)
            pr = Params()
            st = synth.make_state(g, 77 + nx + nz, pr, n_scalars=0)
            if not cluster_fits(g, True):
                continue
            dv = [np.random.default_rng(3 + a).uniform(1e-4, 1e-3, g.n) for a in range(3)]
            sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
            for maxit in (1, 2, 7):
                ref, info, x = solve_both(mfx, orc, g, mfx.EQ_PP, sysd, np.zeros(g.n), 1e-30, maxit)
                assert info["iters"] == ref["iters"] and np.array_equal(x, ref["x"]), ((nx, ny, nz), maxit)
            sysm, _, _ = orc.assemble_mom(g, pr, 2, st)
            ref, info, x = solve_both(mfx, orc, g, 2, sysm, st["w"], 1e-10, 60)
            assert_solve_parity(ref, info, x)
    finally:
        mfx.set_option("solver_path", mfx.PATH_AUTO)
        mfx.set_option("cluster_size", prev)
