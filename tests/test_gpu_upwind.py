"""GPU parity of the upwinded convective face eps: every
assembly (both momentum paths), and SIMPLE iterations, bitwise vs the
oracle with face_eps_upwind = 1."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mfx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15605_b200 as m
    return m


def dev(st):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in st.items()}


def host(t):
    return t.detach().cpu().numpy()


def case(shape=(34, 19, 23), seed=3):
    g = synth.make_grid(*shape)
    pr = synth.Params(face_eps_upwind=1, lin_maxit_pp=3000)
    st = synth.make_state(g, seed, pr, n_scalars=1)
    rng = np.random.default_rng(seed)
    st["phi_old0"] = rng.uniform(0, 1, g.n)
    st["phi0"] = st["phi_old0"].copy()
    return g, pr, st


@pytest.mark.parametrize("asm", [1, 0])
@pytest.mark.parametrize("shape", [(34, 19, 23), (70, 21, 45)])
def test_upwind_assembly_bitwise(mfx, orc, asm, shape):
    g, pr, st = case(shape)
    sd = dev(st)
    ws = mfx.Workspace(g)
    mfx.set_option("asm_tma", asm)
    try:
        for comp in range(3):
            ref, r2, _ = orc.assemble_mom(g, pr, comp, st)
            out, res2 = mfx.assemble_eq(comp, g, pr, sd, ws)
            for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d"):
                assert np.array_equal(host(out[k]), ref[k]), (comp, k)
            assert np.array_equal(host(res2), r2)
    finally:
        mfx.set_option("asm_tma", 1)
    rng = np.random.default_rng(7)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    star = [rng.normal(size=g.n) for _ in range(3)]
    ref, cont, _ = orc.assemble_pp(g, pr, st, star, dv)
    out, res2 = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=[dev({"a": a})["a"] for a in star + dv])
    for k in ("aP", "aE", "aN", "aT", "b"):
        assert np.array_equal(host(out[k]), ref[k]), k
    sref, _, _ = orc.assemble_scalar(g, pr, 0, st)
    sout, _ = mfx.assemble_eq(mfx.EQ_SCALAR, g, pr, sd, ws, scalar_id=0)
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b"):
        assert np.array_equal(host(sout[k]), sref[k]), k


def test_upwind_simple_iterations_bitwise(mfx, orc):
    g, pr, st = case((16, 12, 20), seed=9)
    sd = dev(st)
    ctx = mfx.SimpleContext("111[1]1", g, pr)
    s = st
    for _ in range(2):
        o = ctx.step(sd)
        s, R, it, stt, rc = orc.simple_iter(g, pr, s, n_scalars=1)
        assert o["iters"][:5] == it[:5]
    ctx.close()
    for k in ("u", "v", "w", "p", "phi0"):
        assert np.array_equal(host(sd[k]), s[k]), k
