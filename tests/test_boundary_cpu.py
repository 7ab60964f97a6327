"""CPU-only checks of the C-ABI boundary: libmfx.so loads without a GPU, exports
every function include/mfx.h declares, and its host logic (assignment parsing,
exchange plan, workspace sizing, argument validation) behaves as specified
(PAPER.md:95 assignment notation)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mfx.h")


@pytest.fixture(scope="module")
def mfx(mfx_built):
    import paper_2211_15605_b200 as m
    return m


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mfx_[a-z_]+)\s*\(", text)))


def test_exports_every_declared_symbol(mfx):
    so = os.path.join(ROOT, "paper_2211_15605_b200", "libmfx.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = set(re.findall(r" T (mfx_[a-z_]+)$", out, flags=re.M))
    decl = declared_functions()
    assert len(decl) >= 20
    missing = [f for f in decl if f not in exported]
    assert not missing, missing
    lib = mfx.lib()
    for f in decl:
        assert getattr(lib, f) is not None
    assert set(mfx.EXPORTED) == set(decl)


def test_no_driver_link_dependency():
    so = os.path.join(ROOT, "paper_2211_15605_b200", "libmfx.so")
    out = subprocess.check_output(["ldd", so], text=True)
    assert "libcuda.so" not in out and "libnccl" not in out and "libtorch" not in out


def test_version(mfx):
    assert "sm_100a" in mfx.version()


@pytest.mark.parametrize("text,n,owner", [
    ("111[1]", 1, [0, 0, 0, 0, -1, -1, -1, -1]),          # PAPER.md:95 single GPU
    ("234[1]", 4, [1, 2, 3, 0, -1, -1, -1, -1]),          # Fig. 2b with single-GPU P
    ("222[1]", 2, [1, 1, 1, 0, -1, -1, -1, -1]),
    ("234[1]5678", 8, [1, 2, 3, 0, 4, 5, 6, 7]),          # extra scalar equations
    ("111[1]1111", 1, [0, 0, 0, 0, 0, 0, 0, 0]),
    ("234[1234]", 4, [1, 2, 3, 0, -1, -1, -1, -1]),       # Fig. 2b: multi-GPU pressure
    ("222[12]1", 2, [1, 1, 1, 0, 0, -1, -1, -1]),
    ("234[23]", 4, [1, 2, 3, 1, -1, -1, -1, -1]),         # a subset of the devices solves p'
    ("123[31]", 3, [0, 1, 2, 2, -1, -1, -1, -1]),         # ... in any order: P0 is its first entry
])
def test_parse_assignment(mfx, text, n, owner):
    a = mfx.parse_assignment(text, n)
    assert a["owner"] == owner
    assert a["n_scalars"] == sum(o >= 0 for o in owner[4:])


@pytest.mark.parametrize("text,n", [
    ("123[45]", 4),        # SPEC.md:448 id 5 out of range
    ("12[1]", 4),          # malformed
    ("111", 1),
    ("111[]", 1),
    ("111[1]x", 1),
    ("234[122]", 4),       # a device twice in the pressure list
    ("234[125]", 4),       # pressure-list device out of range
    ("111[1]11111", 1),    # > 4 scalars
])
def test_parse_assignment_errors(mfx, text, n):
    with pytest.raises(mfx.MfxError) as e:
        mfx.parse_assignment(text, n)
    assert e.value.status == mfx.ERR_ARG
    assert mfx.last_error()


def _plan_all(mfx, text, n, nz=16):
    return {r: (mfx.exchange_plan(text, n, r, 0, nz), mfx.exchange_plan(text, n, r, 1, nz)) for r in range(n)}


@pytest.mark.parametrize("text,n", [("234[1]", 4), ("222[1]", 2), ("234[1]5678", 8), ("211[2]3", 3),
                                    ("111[1]", 1), ("111[1]", 3), ("234[1234]", 4), ("222[12]1", 2),
                                    ("234[23]", 4), ("234[413]", 4), ("235[35]1", 5)])
def test_exchange_plan_consistency(mfx, text, n):
    plans = _plan_all(mfx, text, n)
    a = mfx.parse_assignment(text, n)
    P = a["owner"][3]
    prs = a["p_rank"] if a["n_p"] > 1 else [P]
    assert prs[0] == P
    # GATHER: every send has exactly one matching recv on the peer, same buffer
    sends = [(r, o["peer"], o["buf"], o["slot"]) for r, (g, _) in plans.items() for o in g if o["op"] == mfx.OP_SEND]
    recvs = [(o["peer"], r, o["buf"], o["slot"]) for r, (g, _) in plans.items() for o in g if o["op"] == mfx.OP_RECV]
    assert sorted(sends) == sorted(recvs)
    for (src, dst, buf, slot) in sends:
        assert dst in prs and src != dst
    # every p' rank ends up with every momentum component (u*, d, meta)
    for pr in prs:
        got = {"uvw".index(b) for (_, d, b, _) in sends if b in ("u", "v", "w") and d == pr}
        assert got == {c for c in range(3) if a["owner"][c] != pr}
    # PSLAB (multi-GPU p'): slabs tile [0, nz) and all go to P0
    if a["n_p"] > 1:
        slabs = sorted((o["k0"], o["k1"]) for r in range(n) for o in mfx.exchange_plan(text, n, r, 2, 16)
                       if o["op"] == mfx.OP_RECV)
        sends = {r: [o for o in mfx.exchange_plan(text, n, r, 2, 16) if o["op"] == mfx.OP_SEND] for r in range(n)}
        for r in range(n):   # slab i travels from p_rank[i]; ranks outside the list have no PSLAB ops
            if r in prs[1:]:
                i = prs.index(r)
                assert [(o["k0"], o["k1"]) for o in sends[r]] == [mfx.dist_slab(16, i, a["n_p"])]
            else:
                assert not sends[r]
        own = mfx.dist_slab(16, 0, a["n_p"])
        cover = sorted(slabs + [own])
        assert cover[0][0] == 0 and cover[-1][1] == 16
        assert all(cover[i][1] == cover[i + 1][0] for i in range(len(cover) - 1))
    # BCAST: identical op list on every rank (collective order must match)
    b0 = plans[0][1]
    for r in range(n):
        assert plans[r][1] == b0
    roots = {o["buf"]: o["peer"] for o in b0 if o["buf"] != "meta"}
    assert roots["u"] == roots["v"] == roots["w"] == roots["p"] == P
    for s in range(a["n_scalars"]):
        assert roots[f"phi{s}"] == a["owner"][4 + s]


def test_exchange_plan_counts(mfx):
    g = mfx.exchange_plan("234[1]", 4, 0, 0)
    assert len(g) == 9                      # recv u*,d,meta from 3 owners
    assert len(mfx.exchange_plan("234[1]", 4, 2, 0)) == 3
    assert len(mfx.exchange_plan("111[1]", 1, 0, 0)) == 0


def test_workspace_bytes_scale(mfx):
    import synth
    g1 = synth.make_grid(16, 16, 32)
    g2 = synth.make_grid(32, 16, 32)
    b1 = mfx.lib().mfx_workspace_bytes(C.byref(mfx.c_grid(g1)), 0)
    b2 = mfx.lib().mfx_workspace_bytes(C.byref(mfx.c_grid(g2)), 0)
    assert b2 - b1 == 7 * 8 * 16 * 16 * 32


def test_no_unresolved_library_symbols():
    """Every symbol libmfx.so needs at load time comes from libc/libstdc++/libm
    (a missing definition would only surface at dlopen on the GPU box)."""
    so = os.path.join(ROOT, "paper_2211_15605_b200", "libmfx.so")
    out = subprocess.check_output(["nm", "-D", "--undefined-only", so], text=True)
    bad = [l for l in out.splitlines() if l.strip() and not re.search(r"@(GLIBC|GLIBCXX|CXXABI|GCC)", l)
           and "__gmon_start__" not in l and "_ITM_" not in l and "__cxa_finalize" not in l]
    assert not bad, bad


@pytest.mark.parametrize("text,n", [("234[1]", 4), ("111[1]", 1), ("234[1]5678", 8)])
def test_exchange_plan_pic_phase(mfx, text, n):
    """Phase 3 (PIC): the PIC device (rank 0) broadcasts the four
    drag fields; identical op list on every rank (collective order)."""
    plans = [mfx.exchange_plan(text, n, r, 3) for r in range(n)]
    assert all(p == plans[0] for p in plans)
    assert [o["buf"] for o in plans[0]] == ["beta", "sbeta_u", "sbeta_v", "sbeta_w", "meta"]
    assert plans[0][-1]["slot"] == 8 and plans[0][-1]["nslots"] == 1    # the PIC error record
    assert all(o["op"] == mfx.OP_BCAST and o["peer"] == 0 for o in plans[0])


def test_exchange_plan_bad_phase(mfx):
    with pytest.raises(mfx.MfxError):
        mfx.exchange_plan("234[1]", 4, 0, 4)


def test_pic_entry_points_reject_bad_args(mfx):
    """Argument errors return MFX_ERR_ARG before any launch (no GPU needed)."""
    import ctypes as C
    import synth
    g = synth.make_grid(16, 16, 32)
    cg = mfx.c_grid(g)
    pp = mfx.PicParams(0.0, 0.35)                     # d_p <= 0
    pc = mfx.Parcels(None, None, None, None, None, None, None, 0)
    assert mfx.lib().mfx_pic_deposit_eps(C.byref(cg), C.byref(pp), C.byref(pc), None, None, 0, None) == mfx.ERR_ARG
    assert "d_p" in mfx.last_error()
    pp = mfx.PicParams(200e-6, 0.35)
    pc = mfx.Parcels(None, None, None, None, None, None, None, 5)   # n > 0 with NULL arrays
    assert mfx.lib().mfx_pic_deposit_eps(C.byref(cg), C.byref(pp), C.byref(pc), C.c_void_p(8), C.c_void_p(8),
                                         1 << 20, None) == mfx.ERR_ARG
    assert mfx.lib().mfx_ctx_set_pic(None, None, None, 2) == mfx.ERR_ARG


def test_adapt_dt_matches_spec_examples(mfx):
    """mfx_adapt_dt is host logic: SPEC.md:393-395 examples without a GPU."""
    tc = mfx.time_ctrl(dt=4.8e-4, dt_max=5e-4, grow=1.1, grow_threshold=3)
    assert mfx.adapt_dt(tc, 2, True) and tc.dt == 5e-4
    tc = mfx.time_ctrl(dt=1e-3, shrink=0.5)
    assert not mfx.adapt_dt(tc, 10, False) and tc.dt == 5e-4
    tc = mfx.time_ctrl(dt=3e-4, grow_threshold=3)
    assert mfx.adapt_dt(tc, 4, True) and tc.dt == 3e-4
    tc = mfx.time_ctrl(dt=1e-5, dt_min=1e-5)
    assert mfx.adapt_dt(tc, 10, False) and tc.dt == 1e-5


def test_adapt_dt_same_decisions_as_oracle(mfx, orc):
    rng = __import__("numpy").random.default_rng(4)
    for _ in range(200):
        args = dict(dt=float(rng.uniform(1e-5, 2e-3)), dt_min=1e-5, dt_max=float(rng.uniform(1e-4, 1e-3)),
                    grow=float(rng.uniform(1.0, 1.5)), shrink=float(rng.uniform(0.2, 0.9)),
                    grow_threshold=int(rng.integers(1, 5)), max_outer=10)
        a, b = mfx.time_ctrl(**args), orc.time_ctrl(**args)
        its, conv = int(rng.integers(1, 11)), bool(rng.integers(0, 2))
        assert mfx.adapt_dt(a, its, conv) == orc.adapt_dt(b, its, conv)
        assert a.dt == b.dt


def test_time_and_sort_entry_points_reject_bad_args(mfx):
    """Argument errors of the time-loop and parcel-sort entry points return
    MFX_ERR_ARG before any device work (no GPU needed)."""
    import ctypes as C
    import synth
    for bad in (dict(shrink=1.0), dict(shrink=0.0), dict(shrink=float("nan")), dict(grow=0.9),
                dict(dt_max=float("inf"))):
        tc = mfx.time_ctrl(**bad)
        acc = C.c_int()
        assert mfx.lib().mfx_adapt_dt(C.byref(tc), 1, 0, C.byref(acc)) == mfx.ERR_ARG, bad
    tc = mfx.time_ctrl(dt=-1.0)
    acc = C.c_int()
    assert mfx.lib().mfx_adapt_dt(C.byref(tc), 1, 1, C.byref(acc)) == mfx.ERR_ARG
    assert mfx.lib().mfx_time_step(None, None, None, None, None, None) == mfx.ERR_ARG
    g = synth.make_grid(16, 16, 32)
    cg = mfx.c_grid(g)
    assert mfx.lib().mfx_pic_sort_scratch_bytes(C.byref(cg), 1000) > 4 * 2 * g.n
    pp = mfx.PicParams(200e-6, 0.35)
    pc = mfx.Parcels(C.c_void_p(8), C.c_void_p(8), C.c_void_p(8), C.c_void_p(8), C.c_void_p(8), C.c_void_p(8),
                     C.c_void_p(8), 10)
    outs = (C.c_void_p * 7)(*([8] * 7))                       # aliases the input
    assert mfx.lib().mfx_pic_sort(C.byref(cg), C.byref(pp), C.byref(pc), outs, None, None, None, 0,
                                  None) == mfx.ERR_ARG
    assert "in place" in mfx.last_error()


def test_state_load_rejects_missing_file(mfx, tmp_path):
    import ctypes as C
    import synth
    g = synth.make_grid(8, 6, 10)
    st = mfx.State()
    rc = mfx.lib().mfx_state_load(str(tmp_path / "nope.mpxd").encode(), C.byref(mfx.c_grid(g)), C.byref(st), 0,
                                  None, 0, None, None, None, None)
    assert rc == mfx.ERR_ARG and "cannot open" in mfx.last_error()


def test_grid_validation_before_any_launch(mfx):
    """Grid checks run before any launch (no GPU needed): an extent below 2 is
    refused with its own message; an odd nx passes grid validation (it runs the
    grid-stride kernels on a GPU) and the call stops at the next check, the
    NULL system arrays."""
    import synth
    eq = mfx.Eqsys()
    for nx, ok in ((1, False), (9, True), (10, True)):
        cg = mfx.c_grid(synth.make_grid(nx, 6, 8))
        st = mfx.lib().mfx_spmv(0, C.byref(cg), C.byref(eq), None, None, None)
        assert st == mfx.ERR_ARG
        msg = mfx.last_error()
        if ok:
            assert ">= 2" not in msg and "even" not in msg, msg
        else:
            assert ">= 2" in msg, msg


def test_runtime_option_validation(mfx):
    """mfx_set_option refuses out-of-range values and unknown keys before any
    device work (include/mfx.h "Runtime options")."""
    lib = mfx.lib()
    lib.mfx_set_option.restype = C.c_int
    lib.mfx_set_option.argtypes = [C.c_char_p, C.c_int]
    assert lib.mfx_set_option(b"cluster_size", 7) != 0
    assert lib.mfx_set_option(b"cluster_size", 32) != 0
    assert lib.mfx_set_option(b"solver_path", 6) != 0
    assert lib.mfx_set_option(b"no_such_option", 1) != 0
    assert lib.mfx_get_option(b"no_such_option") == -1
    assert lib.mfx_set_option(b"solver_path", 0) == 0
