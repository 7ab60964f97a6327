"""Host-side pieces of bench.py that the driver's multi-GPU runs depend on."""
import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("n", range(1, 9))
def test_assignment_for_every_gpu_count(n, mfx_built):
    import paper_2211_15605_b200 as mfx
    b = load_bench()
    a = mfx.parse_assignment(b.assignment_for(n), n)
    used = {o for o in a["owner"] if o >= 0}
    assert used == set(range(n)), (n, b.assignment_for(n))   # every rank owns an equation
    assert a["owner"][3] == 0                                 # p' on GPU 1


def test_byte_model_matches_design():
    b = load_bench()
    bpc = b.BYTES_PER_CELL
    # SURVEY §8d p' iteration is 200 B/cell with aP streamed; the solver
    # rebuilds the p' diagonal from c_x, c_y, c_z: 184.
    assert bpc["K1_pp"] + bpc["K2_pp"] + bpc["K3"] == 184
    assert bpc["K1_mom"] + bpc["K2_mom"] + bpc["K3"] == 248      # momentum iteration


def test_peaks_file_used():
    b = load_bench()
    peak, kind = b.load_peaks()
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        assert kind == "measured" and peak == json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    else:
        assert "fallback" in kind


@pytest.mark.parametrize("n", range(1, 9))
def test_assignment_multi_p_every_gpu_count(n):
    import paper_2211_15605_b200 as mfx
    b = load_bench()
    a = mfx.parse_assignment(b.assignment_multi_p(n), n)
    assert a["n_p"] == n and a["owner"][3] == 0
    assert a["owner"][:3] == mfx.parse_assignment(b.assignment_for(n), n)["owner"][:3]
