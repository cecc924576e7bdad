"""Plan-level decision replay (north star: given identical bounds, branching and pruning
decisions and selected subdomain indices are bit-exact).

The device planner runs a whole plan() with its plan log on (bp_set_plan_log): every searched
child's box, search report (uf, best, top list, samples) and lower bound, in creation order.  The
oracle's plan() (bab.cpp:266-415) is then replayed on those reports and bounds
(Objective.plan_replay): its own pick_out, split, merge_report, incumbent updates and prune run on
identical inputs.  The boxes it splits out must equal the device's bit for bit (so every pick and
split axis / midpoint agreed), and the two traces -- incumbent, min lf, pruned and selected
volume, pool size, samples per iteration -- and the results must be identical.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2412_09584_b200 import workloads
from paper_2412_09584_b200.config import from_json

pytestmark = pytest.mark.gpu

CASES = [
    ("c1", '{"batch": 8, "seed": 3, "search": {"samples_per_iter": 128, "iterations": 4, "top_capacity": 32},'
           ' "termination": {"max_iterations": 7}}'),
    ("c1", '{"batch": 5, "seed": 9, "eta": 0.4, "temperature": 0.5, "split_rule": "width",'
           ' "search": {"samples_per_iter": 96, "iterations": 3, "top_capacity": 8}, "termination": {"max_iterations": 6}}'),
    ("c2", '{"batch": 6, "seed": 4, "top_percent": 5.0, "search": {"samples_per_iter": 128, "iterations": 3,'
           ' "top_capacity": 48}, "termination": {"max_iterations": 5}}'),
]


@pytest.mark.parametrize("name,cfg_json", CASES)
def test_plan_decisions_replay_bit_exact(device, name, cfg_json):
    wl = workloads.ALL[name](glorot=True)
    dev = device.load(wl.spec)
    cfg = from_json(cfg_json)
    dev.plan_log(True)
    try:
        res = dev.plan(cfg)
        log = dev.plan_log()
    finally:
        dev.plan_log(False)
    assert log["iter"][0] == 0 and np.all(np.diff(log["iter"]) >= 0)  # root first, children in creation order
    ref = orc.Objective(wl.spec).plan_replay(cfg, log)
    assert ref["order_mismatch"] == 0 and ref["box_mismatch"] == 0
    for k in ("iter", "uf", "min_lf", "pruned_vol", "selected_vol", "pool_size", "samples"):
        assert res["trace"][k] == ref["trace"][k], k
    assert res["objective"] == ref["objective"] and np.array_equal(res["action"], ref["action"])
    assert res["lower_bound"] == ref["lower_bound"] and res["iterations"] == ref["iterations"]
    assert res["stop_reason"] == ref["stop_reason"] and res["samples"] == ref["samples"]
    # the replay exercised real branching: several iterations, pruning or retirement somewhere
    assert res["iterations"] >= 3 and len(log["lf"]) > 2 * cfg["batch"]
