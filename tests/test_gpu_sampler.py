"""The device sampler's distributions against the reference's (search.cpp:87-155): the streams
differ (Philox vs mt19937_64), so the checks are statistical, over many boxes at once.

* CEM initial means: agent 0 at the box centre (no warm start), agents 1.. uniform in the box
  (search.cpp:105-112).  With init_sigma and jitter ~0 every agent's single sample is its mean;
  over 4096 boxes the agents' samples must be uniform on each axis (mean, spread, range).
* The best value after one CEM iteration, and after one and ten MPPI iterations, over 96 seeds
  against the oracle's: the same distribution (medians within 12 %; measured 3 %, 0.2 %, 3.4 %).  Round 2 found agents 1.. starting in the box's lower
  corner (a 53-bit uniform built from two shifted words: u < 2^-11), which this bar catches
  (median 384 vs 268 on C1) and the first test pins directly.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2412_09584_b200 import workloads

pytestmark = pytest.mark.gpu


def test_cem_initial_means_are_uniform_in_the_box(device):
    wl = workloads.c1(glorot=True)
    dev = device.load(wl.spec)
    lo, hi = wl.spec.box()
    n = 4096
    cfg = wl.planner_config()
    cfg["search"].update({"samples_per_iter": 4, "iterations": 1, "top_capacity": 8})
    cfg["search"]["cem"].update({"agents": 4, "elites": 1, "jitter": 1e-9, "init_sigma": 1e-9})
    rep = dev.batch_search(np.tile(lo, (n, 1)), np.tile(hi, (n, 1)), None, cfg, seed=11)
    assert rep["ok"].all()
    # each box's top list holds its 4 agent samples and the incumbent row (the centre)
    centre = 0.5 * (lo + hi)
    agents = []
    for b in range(0, n, 8):
        _, acts = dev.report_top(b, 5)
        far = [a for a in acts if np.max(np.abs(a - centre) / (hi - lo)) > 1e-3]
        agents.extend(far)
    agents = np.array(agents)
    assert len(agents) >= 2.5 * (n // 8), len(agents)  # three uniform agents per box (a few may sit near the centre)
    u = (agents - lo) / (hi - lo)
    assert np.all(u >= -1e-6) and np.all(u <= 1 + 1e-6)
    assert np.all(np.abs(u.mean(axis=0) - 0.5) < 0.05), u.mean(axis=0)
    assert np.all(np.abs(u.std(axis=0) - np.sqrt(1 / 12)) < 0.04), u.std(axis=0)
    assert np.all(u.min(axis=0) < 0.02) and np.all(u.max(axis=0) > 0.98)


@pytest.mark.parametrize("method,iters", [("cem", 1), ("mppi", 1), ("mppi", 10)])
def test_search_matches_the_reference_distribution(device, method, iters):
    wl = workloads.c1()
    dev = device.load(wl.spec)
    ob = orc.Objective(wl.spec)
    lo, hi = wl.spec.box()
    cfg = wl.planner_config()
    cfg["search"]["samples_per_iter"] = 256
    cfg["search"]["iterations"] = iters
    cfg["search"]["method"] = method
    g = [dev.batch_search(lo[None], hi[None], None, cfg, seed=s)["uf"][0] for s in range(100, 196)]
    c = [ob.batch_search(lo[None], hi[None], None, cfg, seed=s).get(0)["uf"] for s in range(100, 196)]
    mg, mc = np.median(g), np.median(c)
    assert abs(mg / mc - 1) < 0.12, (mg, mc)
