"""CPU tests of the plan models: the paper's Eq. 2 planner (fusion.plan_linear,
fusion.cpp:199-224) and the B200 roofline planner (fusion.plan_linear_device)
against the committed measurements of the complexity sweep
(profiles/round1/complexity_sweep.json, BASELINE configs[4])."""
import json
import os

import pytest

from paper_2306_08367_b200 import fusion

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SWEEP = os.path.join(ROOT, "profiles", "round1", "complexity_sweep.json")


def test_device_costs_monotone():
    base = fusion.device_plan_costs(10**6, 64, 64, [10**5])
    assert fusion.device_plan_costs(10**6, 64, 4096, [10**5])[1] > base[1]  # wider model costs more
    assert fusion.device_plan_costs(10**6, 64, 64, [10**7])[0] > base[0]    # bigger dim costs the fused plan
    assert fusion.device_plan_costs(10**7, 64, 64, [10**5])[1] > base[1]    # more fact rows cost the non-fused plan


def test_cfg3_plan_is_nonfused_under_both_models():
    # k/l = 64/256 -> Eq. 2 ratio 0.25 < 1; the FFN's layer 1 cannot be pushed down profitably
    assert fusion.plan_linear(60_000_000, 64, 256, [300_000, 800_000]) == "nonfused"
    assert fusion.plan_linear_device(60_000_000, 64, 256, [300_000, 800_000]) == "nonfused"


@pytest.mark.skipif(not os.path.exists(SWEEP), reason="sweep not committed")
def test_device_planner_tracks_measurements():
    d = json.load(open(SWEEP))
    cells = [c for c in d["cells"] if "skipped" not in c]
    dev = sum(fusion.plan_linear_device(10**6, c["k"], c["l"], [c["r"]]) == c["measured_winner"] for c in cells)
    paper = sum(c["planner_right"] for c in cells)
    assert dev >= 0.9 * len(cells)
    assert dev > paper
    for c in cells:  # the sweep's accuracy record: condition-aware 1e-5
        assert c["cond_err_fused"] <= 1e-5 and c["cond_err_nonfused"] <= 1e-5


def test_device_plan_model_c_abi_equals_python():
    """laq_plan_linear_device (the C-ABI a C++ host calls) == fusion.device_plan_costs
    on the sweep and hold-out grids; no device needed."""
    from paper_2306_08367_b200 import fusion
    peaks = (1628e12, 6548e9)
    for r in (1_000, 3_000, 100_000, 3_000_000, 10_000_000):
        for k in (8, 16, 64, 256, 1024):
            for l in (1, 2, 32, 512, 4096):
                for dims in ([r], [r, r // 3 + 1]):
                    tf, tn = fusion.device_plan_costs(1_000_000, k, l, dims, peaks)
                    cf, cn, fused = fusion.device_plan_costs_abi(1_000_000, k, l, dims, peaks)
                    assert abs(cf - tf) <= 1e-12 * tf and abs(cn - tn) <= 1e-12 * tn
                    assert fused == (tf < tn)
