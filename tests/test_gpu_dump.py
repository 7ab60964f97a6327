"""GPU side of NEXT-4: MPXD dumps of
device state through the C ABI, restart transparency, and the paper-style
Eq. 6 digits report of the GPU state against the oracle's (Fig. 5: the
expected result under the arithmetic contract is the single 16-digit bar).
With MFX_REPORT_DIR set, the report is written there as JSON."""
import json
import os

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


def case(n_scalars=1):
    g = synth.make_grid(24, 14, 30)
    pr = synth.Params(lin_maxit_pp=1500)
    st = synth.make_state(g, 97, pr, n_scalars=n_scalars)
    rng = np.random.default_rng(8)
    for s in range(n_scalars):
        st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
        st[f"phi{s}"] = st[f"phi_old{s}"].copy()
    return g, pr, st


def dev(st):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in st.items()}


def test_dump_load_dump_bytewise(mfx, tmp_path):
    g, pr, st = case()
    sd = dev(st)
    pc = {k: torch.from_numpy(v).cuda() for k, v in synth.make_parcels(g, 3, 500, st["eps"]).items()}
    a, b = tmp_path / "a.mpxd", tmp_path / "b.mpxd"
    mfx.state_dump(str(a), g, sd, n_scalars=1, parcels=pc, time=0.125, dt=5e-4)
    sd2 = {k: torch.empty_like(v) for k, v in sd.items()}
    pc2 = {k: torch.empty_like(v) for k, v in pc.items()}
    info = mfx.state_load(str(a), g, sd2, n_scalars=1, parcels=pc2)
    assert info["n_parcels"] == 500 and info["time"] == 0.125 and info["dt"] == 5e-4
    for k in sd:
        assert torch.equal(sd[k], sd2[k]), k
    for k in pc:
        assert torch.equal(pc[k], pc2[k]), k
    mfx.state_dump(str(b), g, sd2, n_scalars=1, parcels=pc2, time=0.125, dt=5e-4)
    assert a.read_bytes() == b.read_bytes()


def test_load_rejects_mismatch(mfx, tmp_path):
    g, pr, st = case()
    sd = dev(st)
    p = tmp_path / "a.mpxd"
    mfx.state_dump(str(p), g, sd, n_scalars=1)
    g2 = synth.make_grid(24, 14, 31)
    sd2 = dev(synth.make_state(g2, 1, pr, n_scalars=1))
    with pytest.raises(mfx.MfxError, match="does not match"):
        mfx.state_load(str(p), g2, sd2, n_scalars=1)
    with pytest.raises(mfx.MfxError, match="missing"):
        mfx.state_load(str(p), g, dev(case(2)[2]), n_scalars=2)     # dump holds one scalar
    raw = p.read_bytes()
    # a rejected file leaves the caller's buffers untouched (validated before any copy)
    for bad in (raw[: len(raw) // 2], raw + b"\0" * 8):
        p.write_bytes(bad)
        nan = {k: torch.full_like(v, float("nan")) for k, v in dev(st).items()}
        with pytest.raises(mfx.MfxError, match="payload"):
            mfx.state_load(str(p), g, nan, n_scalars=1)
        assert all(bool(torch.isnan(v).all()) for v in nan.values())


def test_restart_transparency(mfx, tmp_path):
    """dump/load inserted between SIMPLE iterations never changes
    the subsequent state (bitwise)."""
    g, pr, st = case()
    ref = dev(st)
    ctx = mfx.SimpleContext("111[1]1", g, pr)
    for _ in range(3):
        ctx.step(ref)
    ctx.close()
    sd = dev(st)
    ctx = mfx.SimpleContext("111[1]1", g, pr)
    for _ in range(2):
        ctx.step(sd)
    ctx.close()
    p = tmp_path / "r.mpxd"
    mfx.state_dump(str(p), g, sd, n_scalars=1, time=2 * pr.dt, dt=pr.dt)
    del sd
    fresh = {k: torch.full_like(v, float("nan")) for k, v in ref.items()}
    mfx.state_load(str(p), g, fresh, n_scalars=1)
    ctx = mfx.SimpleContext("111[1]1", g, pr)
    ctx.step(fresh)
    ctx.close()
    for k in ("u", "v", "w", "p", "phi0"):
        assert torch.equal(fresh[k], ref[k]), k


def test_digits_report_gpu_vs_oracle(mfx, orc, tmp_path):
    """PAPER.md:121 / Fig. 5 methodology on one SIMPLE iteration: GPU dump vs
    oracle dump, Eq. 6 histogram per field; expected: every non-zero entry in
    the 16-digit bar (bitwise parity under DESIGN.md §3)."""
    from paper_2211_15605_b200 import verify
    g, pr, st = case()
    sd = dev(st)
    ctx = mfx.SimpleContext("111[1]1", g, pr)
    ctx.step(sd)
    ctx.close()
    gpu = tmp_path / "gpu.mpxd"
    mfx.state_dump(str(gpu), g, sd, n_scalars=1)
    new, R, iters, status, rc = orc.simple_iter(g, pr, st, n_scalars=1)
    names = {"eps": "eps", "eps_old": "eps_old", "u": "u", "v": "v", "w": "w", "u_old": "u_old", "v_old": "v_old",
             "w_old": "w_old", "p": "p", "beta": "beta", "sbu": "sbeta_u", "sbv": "sbeta_v", "sbw": "sbeta_w",
             "phi0": "phi0", "phio0": "phi_old0"}
    ora = tmp_path / "oracle.mpxd"
    verify.write_dump(str(ora), (g.nx, g.ny, g.nz), {k: new[v] for k, v in names.items()})
    rep = verify.compare_dumps(str(ora), str(gpu))
    out_dir = os.environ.get("MFX_REPORT_DIR")
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "digits_report.json"), "w") as f:
            json.dump({"grid": [g.nx, g.ny, g.nz], "assignment": "111[1]1", "fields": rep}, f, indent=1)
    for k in ("u", "v", "w", "p", "phi0"):
        h = rep[k]["hist"]
        assert sum(h.values()) == h[16], (k, h)
