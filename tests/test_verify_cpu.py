"""NEXT-4 verification tooling on the CPU: Eq. 6 digits (
SPEC.md:509-519 examples), histograms, and the MPXD container read by both
the numpy reader and libmfx's host-only mfx_dump_info."""
import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def vf(mfx_built):
    from paper_2211_15605_b200 import verify
    return verify


def test_digits_spec_examples(vf):
    assert vf.digits(3.7, 3.7) == 16.0                       # S:513 exact match clamps at 16
    assert vf.digits(1.0, 0.999) == pytest.approx(3.0)
    assert vf.digits(1.0, 2.0) == pytest.approx(0.0)
    assert np.isnan(vf.digits(0.0, 1.0))                      # zero references excluded (Fig. 5)
    assert vf.digits(1.0, 1e9) == -5.0                        # clamp floor


def test_digits_scale_invariant(vf):
    rng = np.random.default_rng(1)
    a = rng.uniform(-1, 1, 1000)
    b = a * (1 + rng.uniform(-1e-7, 1e-7, 1000))
    np.testing.assert_allclose(vf.digits(1e6 * a, 1e6 * b), vf.digits(a, b), atol=1e-6)


def test_histogram_counts(vf):
    d = vf.digits(np.array([1.0, 2.0, 0.0, 5.0]), np.array([1.0, 2.0 * (1 + 1e-9), 3.0, 5.0 * (1 + 1e-3)]))
    h, zeros = vf.histogram(d)
    assert zeros == 1 and h[16] == 1 and h[9] == 1 and h[3] == 1
    assert sum(h.values()) == 3


def make_fields(rng, dims):
    n = int(np.prod(dims))
    return {k: rng.normal(0, 1, n) for k in ("eps", "u", "v", "w", "p")}


def test_dump_roundtrip_and_compare(vf, tmp_path):
    """a dump against itself is all 16; a (1 + 1e-9) copy is all 9."""
    rng = np.random.default_rng(2)
    dims = (4, 3, 5)
    f = make_fields(rng, dims)
    pc = {k: rng.uniform(0, 1, 7) for k in ("px", "py", "pz")}
    a = tmp_path / "a.mpxd"
    vf.write_dump(str(a), dims, f, pc, time=0.25, dt=5e-4)
    r = vf.read_dump(str(a))
    assert r["dims"] == dims and r["n_parcels"] == 7 and r["time"] == 0.25
    for k in f:
        assert np.array_equal(r["fields"][k], f[k])
    same = vf.compare_dumps(str(a), str(a))
    assert all(v["hist"][16] == v["hist"][16] and sum(v["hist"].values()) == v["hist"][16] for v in same.values())
    b = tmp_path / "b.mpxd"
    vf.write_dump(str(b), dims, {k: v * (1 + 1e-9) for k, v in f.items()}, {k: v * (1 + 1e-9) for k, v in pc.items()})
    cmp = vf.compare_dumps(str(a), str(b))
    for v in cmp.values():
        assert v["mode"] == 9 and sum(v["hist"].values()) == v["hist"][9]


def test_dump_info_host_only(vf, tmp_path):
    """libmfx reads the header without a GPU; corrupt files are rejected."""
    import paper_2211_15605_b200 as mfx
    rng = np.random.default_rng(3)
    dims = (6, 4, 3)
    f = make_fields(rng, dims)
    f.update({"phi0": rng.normal(size=72), "phio0": rng.normal(size=72), "phi1": rng.normal(size=72)})
    p = tmp_path / "c.mpxd"
    vf.write_dump(str(p), dims, f, {"px": np.zeros(9)}, time=1.5, dt=2e-4)
    info = mfx.dump_info(str(p))
    assert info["dims"] == dims and info["n_parcels"] == 9 and info["n_scalars"] == 2
    assert info["time"] == 1.5 and info["dt"] == 2e-4
    raw = p.read_bytes()
    bad = tmp_path / "bad.mpxd"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(mfx.MfxError, match="magic"):
        mfx.dump_info(str(bad))
    bad.write_bytes(raw[:30])
    with pytest.raises(mfx.MfxError, match="truncated"):
        mfx.dump_info(str(bad))
    with pytest.raises(mfx.MfxError, match="cannot open"):
        mfx.dump_info(str(tmp_path / "missing.mpxd"))
    with pytest.raises(ValueError, match="truncated"):
        vf.read_dump(str(bad))
