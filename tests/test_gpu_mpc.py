"""Receding-horizon MPC over the device planner (the reference's
run_mpc, proj/tools/babplan_cli.cpp:333-420)."""
import json
import math

import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import mpc_driver as mpcmod

pytestmark = pytest.mark.gpu


def scenario(obstacles=False, H=6):
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = [0.4, -0.3, 0.1, 0.2], [0.0, 0.0, 0.1, 0.1], [0.0, 0.0]
    s.horizon = H
    s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
    if obstacles:
        s.obstacles = [bp.Obstacle([0.2, 0.1], 0.3)]
        s.cost_form = "tracking_obstacles"
        s.lam = 50.0
    return s


def config(seed=3):
    cfg = json.loads(bp.default_config())
    cfg["seed"] = seed
    cfg["termination"]["max_iterations"] = 4
    cfg["search"]["samples_per_iter"] = 128
    cfg["search"]["iterations"] = 4
    return json.dumps(cfg)


@pytest.mark.parametrize("obstacles", [False, True])
def test_single_plan_executed_open_loop_realises_its_objective(obstacles):
    """replan = H: the plant is the model, so executing the plan reproduces its
    objective (device FP32 rollout vs the FP64 host plant: 1e-5 relative)."""
    m = bp.generate_model(3, [6, 16, 16, 4])
    s = scenario(obstacles)
    r = bp.mpc(m, s, config(), replan=s.horizon)
    assert r["replans"] == 1 and r["steps"] == s.horizon and len(r["trace"]["step"]) == s.horizon
    assert math.isclose(r["realized_objective"], r["open_loop_objective"], rel_tol=1e-5, abs_tol=1e-6)


@pytest.mark.parametrize("replan,method", [(1, "babnd"), (2, "babnd"), (1, "cem")])
def test_receding_horizon_trace(replan, method):
    m = bp.generate_model(3, [6, 16, 16, 4])
    s = scenario(True)
    r = bp.mpc(m, s, config(), method=method, replan=replan)
    assert r["replans"] == math.ceil(s.horizon / replan)
    assert r["trace"]["step"] == list(range(1, s.horizon + 1))
    assert np.isclose(np.sum(r["trace"]["cost"]), r["realized_objective"])
    assert np.all(np.diff(r["trace"]["samples"]) >= 0) and r["samples"] > 0
    assert len(r["replan_ms"]) == r["replans"]
    assert r["final_step_cost"] == r["trace"]["cost"][-1]


def test_plant_step_matches_reference_rollout():
    """The host plant (make_features + Model.forward) equals bp.rollout's states."""
    m = bp.generate_model(3, [6, 16, 16, 4])
    s = scenario()
    act = np.random.default_rng(0).uniform(-0.5, 0.5, size=2 * s.horizon)
    x, p = s.x0.copy(), s.p0.copy()
    states = bp.rollout(m, s, act)
    for t in range(s.horizon):
        u = act[2 * t:2 * t + 2]
        x = m.forward(mpcmod.make_features(s, x, p, u)[None])[0]
        p = p + u
        assert np.allclose(states[t], x, rtol=1e-5, atol=1e-6)


def test_mix_seed_matches_reference_kat():
    # splitmix64 (rng.cpp:37-42); the planner's pick stream seed for seed 0
    assert mpcmod.mix_seed(0, 0) == 0xE220A8397B1DCDAF


def test_rejects_bad_replan():
    with pytest.raises(ValueError):
        bp.mpc(bp.generate_model(3, [6, 4]), scenario(), config(), replan=0)
