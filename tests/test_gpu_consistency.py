"""GPU parity on the smooth manufactured fields of test_oracle_consistency.py
(anisotropic spacing dx != dy != dz, every term of every row active, central
and upwinded face eps): the GPU rows equal the oracle's bitwise, so the
consistency pins of the oracle carry over to the CUDA path."""
import numpy as np
import pytest

from synth import Params
from test_oracle_consistency import F, PR, VEL, make_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mfx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15605_b200 as m
    return m


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("n", [16, 34])
@pytest.mark.parametrize("upwind", [0, 1])
@pytest.mark.parametrize("asm", [1, 0])
def test_manufactured_rows_bitwise(mfx, orc, n, upwind, asm):
    g, h, cc, st, _ = make_case(n)
    p = Params(rho=PR["rho"], mu=PR["mu"], g=PR["g"], dt=PR["dt"], urf_mom=PR["urf_mom"],
               gamma_phi=PR["gamma_phi"], urf_phi=1.0, face_eps_upwind=upwind)
    sd = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in st.items()}
    ws = mfx.Workspace(g)
    mfx.set_option("asm_tma", asm)
    try:
        for comp in range(3):
            ref, r2, _ = orc.assemble_mom(g, p, comp, st)
            out, res2 = mfx.assemble_eq(comp, g, p, sd, ws)
            for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d"):
                assert np.array_equal(host(out[k]), ref[k]), (comp, k)
            assert np.array_equal(host(res2), r2)
    finally:
        mfx.set_option("asm_tma", 1)
    ref, r2, _ = orc.assemble_scalar(g, p, 0, st)
    out, res2 = mfx.assemble_eq(mfx.EQ_SCALAR, g, p, sd, ws, scalar_id=0)
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b"):
        assert np.array_equal(host(out[k]), ref[k]), ("phi", k)
    dv = []
    for c in range(3):
        X = cc.copy()
        X[c] += 0.5 * h[c]
        dv.append(F["d%d" % c](*X))
    star = [st[vn] for vn in VEL]
    ref, cont, _ = orc.assemble_pp(g, p, st, star, dv)
    out, res2 = mfx.assemble_eq(mfx.EQ_PP, g, p, sd, ws,
                                star=[sd[vn] for vn in VEL] + [torch.from_numpy(a).cuda() for a in dv])
    for k in ("aP", "aE", "aN", "aT", "b"):
        assert np.array_equal(host(out[k]), ref[k]), ("pp", k)
    assert host(res2)[0] == cont
