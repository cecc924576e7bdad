"""The planner loop over the device pool (pool.cu + host heads): the paths of
plan() (bab.cpp:266-415) that the throughput configs do not reach -- retirement of
boxes narrower than min_width, tiny and zero top-list capacities, the width split
rule, batches larger than the pool, the stop reasons -- checked through plan()'s own
invariants (bab.hpp:136-148): the incumbent never worsens, the certified bound never
exceeds it, pruned + pool volume never exceeds the root's, every box is searched
once, and runs are deterministic."""
import json

import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import objective as objmod

pytestmark = pytest.mark.gpu


def ref_linear():
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = [0.4, 0.4], [0.0, 0.0], [0.0, 0.0]
    s.horizon = 3
    s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
    return objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(1, [4, 2]), s))


def config(**kw):
    cfg = json.loads(bp.default_config())
    cfg["batch"] = 8
    cfg["termination"]["max_iterations"] = 12
    cfg["search"]["samples_per_iter"] = 64
    cfg["search"]["iterations"] = 3
    for k, v in kw.items():
        if k in cfg["search"]:
            cfg["search"][k] = v
        elif k in cfg["termination"] or k == "target_objective":
            cfg["termination"][k] = v
        else:
            cfg[k] = v
    return cfg


def check_invariants(res, cfg):
    tr = res["trace"]
    uf = np.asarray(tr["uf"])
    assert np.all(np.diff(uf) <= 0), "incumbent got worse"
    assert res["lower_bound"] <= res["objective"] + 1e-9
    vol = np.asarray(tr["pruned_vol"])
    assert np.all(np.diff(vol) >= -1e-12) and vol[-1] <= 1.0 + 1e-9
    rows = cfg["search"]["samples_per_iter"] // cfg["search"]["cem"]["agents"] * cfg["search"]["cem"]["agents"] + 1
    assert res["samples"] % (rows * cfg["search"]["iterations"]) == 0  # whole searches only
    assert res["objective"] == pytest.approx(float(uf[-1]))


@pytest.mark.parametrize("kw", [
    {"min_width": 0.26},                 # boxes retire after two halvings of every axis
    {"top_capacity": 1},
    {"top_capacity": 0},
    {"split_rule": "width"},
    {"batch": 64},                       # more picks than the pool holds
    {"eta": 0.0, "temperature": 1e-9},   # pure softmax picks, degenerate temperature
    {"top_percent": 100.0},
])
def test_planner_paths_keep_invariants_and_are_deterministic(device, kw):
    dev = device.load(ref_linear())
    cfg = config(**kw)
    a = dev.plan(cfg)
    check_invariants(a, cfg)
    b = dev.plan(cfg)
    assert a["objective"] == b["objective"] and np.array_equal(a["action"], b["action"])
    assert a["trace"]["pool_size"] == b["trace"]["pool_size"] and a["trace"]["min_lf"] == b["trace"]["min_lf"]


def test_retirement_exhausts_the_pool(device):
    """With a width floor above the box the root retires at once; just below it the
    pool runs dry after a few splits (pool-exhausted), and the retired bounds stay in
    the certified lower bound."""
    dev = device.load(ref_linear())
    res = dev.plan(config(min_width=2.0))
    assert res["iterations"] == 1 and res["stop_reason"] == "pool-exhausted"
    assert res["trace"]["pool_size"][-1] == 0
    res = dev.plan(config(min_width=0.51, batch=64, max_iterations=50))  # every axis split once: 64 leaves
    assert res["stop_reason"] == "pool-exhausted"
    assert np.isfinite(res["lower_bound"]) and res["lower_bound"] <= res["objective"] + 1e-9


def test_stop_reasons(device):
    dev = device.load(ref_linear())
    assert dev.plan(config(max_iterations=2))["stop_reason"] == "max-iterations"
    assert dev.plan(config(target_objective=1e30))["stop_reason"] == "target"
    res = dev.plan(config(max_iterations=10**6, wall_clock_ms=50.0))
    assert res["stop_reason"] in ("wall-clock", "pool-exhausted")
