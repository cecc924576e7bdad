"""GPU parity of the separable synthetic objective and its exact bounder
 against the FP64 oracle, and the reference's own smoke test
for plan_synthetic (proj/tests/python/test_smoke.py:45-57) through the drop-in.

Bars: objective values are FP64 on the device, rounded to FP32 for the planner's
cost buffer: 1e-6 relative.  Bounds are FP64 on both sides (CUDA vs glibc cos):
1e-12 relative.
"""
import json

import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [1, 4, 50, 300])
def test_synthetic_objective_matches_oracle(device, d):
    dev = device.load_synthetic(d)
    assert dev.rollout_kernel() == "synthetic"
    acts = np.random.default_rng(d).uniform(-1, 1, size=(3, 41, d)).astype(np.float32)
    costs, _, _, _, bad = dev.rollout(acts, want_stats=False)
    assert not bad.any()
    ob = orc.Objective(synthetic_dim=d)
    for s in range(3):
        ref = ob.evaluate(acts[s].astype(np.float64))
        assert np.max(np.abs(costs[s] - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-6


def test_synthetic_rows_are_batch_invariant(device):
    dev = device.load_synthetic(64)
    acts = np.random.default_rng(5).uniform(-1, 1, size=(1, 300, 64)).astype(np.float32)
    whole = dev.rollout(acts, want_stats=False)[0]
    for i in (0, 7, 299):
        assert dev.rollout(acts[:, i:i + 1], want_stats=False)[0][0, 0] == whole[0, i]


@pytest.mark.parametrize("d", [1, 3, 50])
def test_separable_bound_matches_oracle(device, d):
    """bab.cpp:70-83 on random sub-boxes, degenerate intervals and the full domain."""
    dev = device.load_synthetic(d)
    rng = np.random.default_rng(10 + d)
    a = rng.uniform(-1, 1, size=(40, d))
    b = rng.uniform(-1, 1, size=(40, d))
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    lo[0], hi[0] = -1.0, 1.0           # the whole domain: d * global minimum
    lo[1] = hi[1] = a[1]               # points
    lf = dev.bound_boxes(lo, hi, "full-crown", "adaptive")
    for i in range(len(lo)):
        ref = sum(orc.separable_term_min(float(lo[i, j]), float(hi[i, j])) for j in range(d))
        assert abs(lf[i] - ref) <= 1e-12 * max(1.0, abs(ref))
    assert abs(lf[0] - d * -0.980339434486584) < 1e-9 * d  # SyntheticObjective::kUnitMinimum
    # a bound never exceeds any sample of its box
    for i in range(2, 10):
        pts = rng.uniform(lo[i], hi[i], size=(500, d))
        vals = np.sum(5 * pts ** 2 + np.cos(50 * pts), axis=1)
        assert lf[i] <= vals.min() + 1e-12


def test_reference_smoke_plan_synthetic_babnd_beats_default_sampler():
    """proj/tests/python/test_smoke.py:45-57, unchanged apart from the module name."""
    cfg = json.loads(bp.default_config())
    cfg["seed"] = 5
    cfg["termination"]["max_iterations"] = 8
    cfg["search"]["samples_per_iter"] = 200
    cfg["search"]["iterations"] = 10
    res = bp.plan_synthetic(4, json.dumps(cfg), method="babnd")
    assert res["objective"] <= 4 * -0.9  # near 4 * global minimum
    assert res["lower_bound"] <= res["objective"]
    assert res["stop_reason"] in {"max-iterations", "pool-exhausted", "target", "wall-clock"}
    assert len(res["trace"]["uf"]) >= 1
    uf = res["trace"]["uf"]
    assert all(a >= b for a, b in zip(uf, uf[1:]))  # incumbent never worsens


@pytest.mark.parametrize("d", [8, 50])
def test_plan_synthetic_matches_or_beats_cpu_reference(d):
    """Same or better best objective than the CPU planner (oracle) at equal iteration
    count on the paper's separable benchmark, with a certified bracket.  The device
    samples with Philox, the reference with mt19937_64 + Box-Muller, so single runs
    differ; the bar is on the mean over 12 seeds, within ~2 standard errors of the
    difference (measured over 24 seeds: d=8 -6.987 vs -6.983, d=50 -9.37 vs -9.28).
    Deterministic: fixed seeds give identical runs."""
    from paper_2412_09584_b200.config import from_json
    g, c = [], []
    for seed in range(1, 13):
        cfg = json.loads(bp.default_config())
        cfg["seed"] = seed
        cfg["termination"]["max_iterations"] = 6
        cfg["search"]["samples_per_iter"] = 256
        gpu = bp.plan_synthetic(d, json.dumps(cfg))
        cpu = orc.Objective(synthetic_dim=d).plan(from_json(json.dumps(cfg)))
        assert gpu["iterations"] == cpu["iterations"] == 6
        assert gpu["lower_bound"] <= gpu["objective"] + 1e-9
        assert gpu["lower_bound"] >= d * -0.980339434486584 - 1e-9  # never below the global minimum
        g.append(gpu["objective"])
        c.append(cpu["objective"])
    print(f"d={d}: gpu mean {np.mean(g):.4f} cpu mean {np.mean(c):.4f}")
    assert np.mean(g) <= np.mean(c) + 0.02 * d


def test_plan_synthetic_rejects_bad_dimension():
    with pytest.raises(ValueError):
        bp.plan_synthetic(0)
