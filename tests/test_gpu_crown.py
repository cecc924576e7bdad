"""GPU parity of full CROWN (crown_node_bounds + the stop-free output pass,
proj/src/crown.cpp:379-469) against the FP64 oracle, and the
reference's own smoke test for network_lower_bound (test_smoke.py:79-85).

Both sides are FP64 with the same relaxations; the device sums in a different
order (per-thread partials and a fixed block reduction), so the bar is 1e-8
relative to max(1, |bound|).
"""
import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import objective as objmod, workloads

pytestmark = pytest.mark.gpu

TOL = 1e-8


def close(a, b):
    return abs(a - b) <= TOL * max(1.0, abs(b))


def short(spec, H):
    """The same objective over the first H steps (keeps the FP64 oracle's full CROWN,
    quadratic in depth, to seconds)."""
    return objmod.ObjectiveSpec(**{**spec.__dict__, "horizon": H, "step_weight": spec.step_weight[:H],
                                   "custom_stop_steps": [t for t in spec.custom_stop_steps if t <= H]})


def spec_of(name):
    if name == "ref-obstacles":  # relative features; hinges on keypoint slices and on p_t
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, -0.3, 0.1, 0.2], [0.0, 0.0, 0.1, 0.1], [0.0, 0.0]
        s.horizon = 4
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        s.obstacles = [bp.Obstacle([0.2, 0.1], 0.3), bp.Obstacle([-0.1, 0.2], 0.25)]
        s.cost_form = "tracking_obstacles"
        s.lam = 50.0
        return objmod.build_objective(bp.generate_model(3, [6, 16, 16, 4]), s)
    if name == "ref-linear":  # zero hidden layers
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, 0.4], [0.0, 0.0], [0.0, 0.0]
        s.horizon = 3
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        return objmod.build_objective(bp.generate_model(1, [4, 2]), s)
    if name == "c1":  # action penalty: SquaredDistance on the u_t slice
        return short(workloads.c1(glorot=True).spec, 3)
    if name == "c2":  # squared-radius obstacle ReLUs (SqDist -> ScalarAffine -> ReLU)
        return short(workloads.c2(glorot=True).spec, 2)
    if name == "c4":  # L1 goal and state-bound penalty (Linear / ReLU cost ops)
        return short(workloads.c4(glorot=True).spec, 2)
    raise KeyError(name)


@pytest.mark.parametrize("name", ["ref-linear", "ref-obstacles", "c1", "c2", "c4"])
@pytest.mark.parametrize("alpha", ["adaptive", "zero", "one"])
def test_full_crown_matches_oracle(device, name, alpha):
    spec = spec_of(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    rng = np.random.default_rng(7)
    c = rng.uniform(lo, hi)
    los = np.stack([lo, np.minimum(c, hi), lo])
    his = np.stack([hi, hi, np.maximum(c, lo)])
    lf = dev.bound_boxes(los, his, "full-crown", alpha)
    ob = orc.Objective(spec)
    for i in range(3):
        ref = ob.lower_bound(los[i], his[i], mode="full-crown", alpha=alpha)
        assert close(lf[i], ref), (name, alpha, i, lf[i], ref)
    # sound: below every sampled value of its box
    for i in range(3):
        pts = rng.uniform(los[i], his[i], size=(256, spec.d)).astype(np.float32)
        vals = ob.evaluate(pts.astype(np.float64))
        assert lf[i] <= vals.min() + 1e-9


@pytest.mark.parametrize("name", ["ref-linear", "ref-obstacles", "c1", "c2", "c4"])
def test_full_crown_node_bounds_match_oracle(device, name):
    """Every intermediate bound of the device's node passes against crown_node_bounds."""
    spec = spec_of(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    c = np.random.default_rng(8).uniform(lo, hi)
    los, his = np.stack([lo, np.minimum(c, hi)]), np.stack([hi, hi])
    dev.bound_boxes(los, his, "full-crown")
    nlo, nhi = dev.node_bounds(2)
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    for i in range(2):
        st = ob.crown_node_stats(los[i], his[i], ob.watch_set())
        rlo, rhi = ob.stats_in_layout(st, layout, spec.horizon)
        seen = ~np.isnan(rlo)
        assert seen.any()
        bad = np.argwhere(seen & ~(np.abs(nlo[i] - np.nan_to_num(rlo)) <= TOL * np.maximum(1, np.abs(np.nan_to_num(rlo)))))
        assert bad.size == 0, (name, i, bad[:5], nlo[i][tuple(bad[0])], rlo[tuple(bad[0])])
        bad = np.argwhere(seen & ~(np.abs(nhi[i] - np.nan_to_num(rhi)) <= TOL * np.maximum(1, np.abs(np.nan_to_num(rhi)))))
        assert bad.size == 0, (name, i, bad[:5], nhi[i][tuple(bad[0])], rhi[tuple(bad[0])])


def test_full_crown_is_tighter_than_intervals(device):
    spec = spec_of("c1")
    dev = device.load(spec)
    lo, hi = spec.box()
    full = dev.bound_boxes(lo[None], hi[None], "full-crown")[0]
    ivl = dev.bound_boxes(lo[None], hi[None], "early-stop-interval")[0]
    assert full >= ivl - 1e-9


def test_scenario_lower_bound_defaults_to_full_crown():
    """pymodule.cpp:180-190 through the drop-in: mode defaults to full-crown."""
    m = bp.generate_model(seed=4, widths=[4, 8, 2])
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = np.full(2, 0.4), np.zeros(2), np.zeros(2)
    s.horizon = 3
    s.u_lower, s.u_upper = np.full(2, -0.5), np.full(2, 0.5)
    lb = bp.lower_bound(m, s)
    spec = objmod.build_objective(m, s)
    lo, hi = spec.box()
    assert close(lb, orc.Objective(spec).lower_bound(lo, hi, mode="full-crown"))


def oracle_network_bound(m, lo, hi, mode, alpha="adaptive"):
    """build_network_objective (model.cpp:389-405) on the oracle's graph."""
    g = orc.Graph()
    h = g.input(m.input_dim)
    last_relu = -1
    for W, b, r in zip(m.W, m.b, m.relu):
        h = g.linear(h, W, b)
        if r:
            h = g.relu(h)
            last_relu = h
    g.set_output(h)
    g.finalize()
    return g.objective(final_step_last_relu=last_relu).lower_bound(lo, hi, mode=mode, alpha=alpha)


@pytest.mark.parametrize("widths", [[3, 12, 12, 1], [5, 32, 1], [2, 1], [4, 16, 16, 16, 1]])
@pytest.mark.parametrize("mode", ["full-crown", "early-stop-interval"])
def test_network_lower_bound_matches_oracle(widths, mode):
    m = bp.generate_model(seed=21, widths=widths)
    rng = np.random.default_rng(3)
    for _ in range(3):
        a, b = rng.uniform(-1, 1, size=(2, widths[0]))
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        lb = bp.network_lower_bound(m, lo, hi, mode=mode)
        assert close(lb, oracle_network_bound(m, lo, hi, mode))


def test_reference_smoke_lower_bound_sound_on_samples():
    """proj/tests/python/test_smoke.py:79-85, unchanged apart from the module name."""
    m = bp.generate_model(seed=21, widths=[3, 12, 12, 1])
    lo, hi = np.full(3, -1.0), np.full(3, 1.0)
    lb = bp.network_lower_bound(m, lo, hi, mode="full-crown")
    pts = np.random.default_rng(1).uniform(-1, 1, size=(2000, 3))
    vals = m.forward(pts)[:, 0]
    assert lb <= vals.min() + 1e-9


def test_network_lower_bound_rejects_bad_inputs():
    m = bp.generate_model(seed=21, widths=[3, 12, 2])
    with pytest.raises(ValueError):
        bp.network_lower_bound(m, np.zeros(3), np.ones(3))  # output not scalar
    m = bp.generate_model(seed=21, widths=[3, 12, 1])
    with pytest.raises(ValueError):
        bp.network_lower_bound(m, np.zeros(2), np.ones(2))  # box dim mismatch
    with pytest.raises(ValueError):
        bp.network_lower_bound(m, np.ones(3), np.zeros(3))  # inverted box


def test_plan_with_full_crown_is_certified(device):
    """plan() in the sound full-CROWN mode: a certified bracket (bab.cpp:410, crown.cpp:326)."""
    import json
    from paper_2412_09584_b200.config import from_json
    spec = spec_of("c1")
    dev = device.load(spec)
    cfg = json.loads(bp.default_config())
    cfg["bound_mode"] = "full-crown"
    cfg["batch"] = 4
    cfg["termination"]["max_iterations"] = 3
    cfg["search"]["samples_per_iter"] = 64
    cfg["search"]["iterations"] = 3
    res = dev.plan(from_json(json.dumps(cfg)))
    assert res["certified"] and res["lower_bound"] <= res["objective"] + 1e-9
    lo, hi = spec.box()
    assert res["lower_bound"] >= orc.Objective(spec).lower_bound(lo, hi, mode="full-crown") - 1e-9
