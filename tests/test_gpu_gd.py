"""GD searcher on the device: the reverse-mode gradient of the
unrolled objective against the FP64 oracle (graph.cpp:403-564 restated), and GD
search / planning against the reference's run_gd (search.cpp:214-245).

Bars: the gradient is FP64 on both sides and returned in FP32: 2e-5 relative to
max(1, |g|) (also absorbs the FP32 inputs' kinks being identical).  A single-start
GD trajectory from a warm start is deterministic on both sides: its best value
within 1e-4 relative after 10 steps (FP32 iterates on the device, FP64 in the
reference).
"""
import json

import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import objective as objmod, workloads
from paper_2412_09584_b200.config import from_json

pytestmark = pytest.mark.gpu


def spec_of(name):
    if name == "ref-obstacles":
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, -0.3, 0.1, 0.2], [0.0, 0.0, 0.1, 0.1], [0.0, 0.0]
        s.horizon = 5
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        s.obstacles = [bp.Obstacle([0.2, 0.1], 0.3), bp.Obstacle([-0.1, 0.2], 0.25)]
        s.cost_form = "tracking_obstacles"
        s.lam = 50.0
        return objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(3, [6, 16, 16, 4]), s))
    if name == "ref-linear":
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, 0.4], [0.0, 0.0], [0.0, 0.0]
        s.horizon = 3
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        return objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(1, [4, 2]), s))
    return {"c1": workloads.c1, "c2": workloads.c2, "c3": workloads.c3, "c4": workloads.c4}[name](glorot=True).spec


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


@pytest.mark.parametrize("name", ["ref-linear", "ref-obstacles", "c1", "c2", "c3", "c4"])
def test_gradient_matches_oracle(device, name):
    spec = spec_of(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    acts = np.random.default_rng(4).uniform(lo, hi, size=(9, spec.d)).astype(np.float32)
    g = dev.gradient(acts)
    ref = orc.Objective(spec).gradient(acts.astype(np.float64))
    assert rel(g, ref) < 2e-5, name


@pytest.mark.parametrize("d", [1, 7, 64])
def test_synthetic_gradient_matches_oracle(device, d):
    dev = device.load_synthetic(d)
    acts = np.random.default_rng(d).uniform(-1, 1, size=(5, d)).astype(np.float32)
    assert rel(dev.gradient(acts), orc.Objective(synthetic_dim=d).gradient(acts.astype(np.float64))) < 2e-5


def gd_config(starts, iters=10):
    return from_json(json.dumps({"search": {"method": "gd", "samples_per_iter": starts, "iterations": iters}}))


@pytest.mark.parametrize("name", ["ref-obstacles", "c1"])
def test_single_start_gd_trajectory_matches_reference(device, name):
    spec = spec_of(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    warm = np.random.default_rng(9).uniform(lo, hi).astype(np.float32).astype(np.float64)
    cfg = gd_config(1)
    rep = dev.batch_search(lo[None], hi[None], warm[None], cfg, seed=5)
    ref = orc.Objective(spec).batch_search(lo[None], hi[None], warm[None], cfg, seed=5)
    assert rep["ok"].all()
    assert abs(rep["uf"][0] - ref.get(0)["uf"]) <= 1e-4 * max(1.0, abs(ref.get(0)["uf"]))
    assert rep["samples"][0] == 10


def test_synthetic_single_start_gd_matches_reference(device):
    d = 6
    dev = device.load_synthetic(d)
    lo, hi = -np.ones(d), np.ones(d)
    warm = np.random.default_rng(2).uniform(-1, 1, size=d).astype(np.float32).astype(np.float64)
    cfg = gd_config(1, 20)
    rep = dev.batch_search(lo[None], hi[None], warm[None], cfg, seed=1)
    ref = orc.Objective(synthetic_dim=d).batch_search(lo[None], hi[None], warm[None], cfg, seed=1)
    assert abs(rep["uf"][0] - ref.get(0)["uf"]) <= 1e-4 * max(1.0, abs(ref.get(0)["uf"]))


def test_gd_search_improves_and_plans(device):
    """Multi-start GD over several boxes: incumbents never worse than the warm start's
    value, and BaB with the GD searcher keeps a valid bracket."""
    spec = spec_of("c1")
    dev = device.load(spec)
    lo, hi = spec.box()
    rep = dev.batch_search(np.stack([lo, lo]), np.stack([hi, hi]), None, gd_config(64, 6), seed=2)
    ob = orc.Objective(spec)
    centre = ob.evaluate(((lo + hi) / 2)[None].astype(np.float32).astype(np.float64))[0]
    assert rep["ok"].all() and np.all(rep["uf"] <= centre * (1 + 1e-5) + 1e-6)
    cfg = json.loads(bp.default_config())
    cfg["search"]["method"] = "gd"
    cfg["search"]["samples_per_iter"] = 64
    cfg["search"]["iterations"] = 5
    cfg["termination"]["max_iterations"] = 3
    res = dev.plan(from_json(json.dumps(cfg)))
    assert res["lower_bound"] <= res["objective"] + 1e-9
    uf = res["trace"]["uf"]
    assert all(a >= b for a, b in zip(uf, uf[1:]))
    res2 = dev.plan(from_json(json.dumps(cfg)), method="gd")  # the sampler alone
    assert res2["stop_reason"] == "sampler-budget"
