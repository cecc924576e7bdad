"""Sampler-update parity on identical samples.

The device sampler is Philox and the reference's is mt19937_64 + Box-Muller, so
whole search trajectories are not comparable.  Here both sides consume the SAME
injected rows and values: the oracle runs the reference's run_cem / run_mppi
with its sampled rows replaced and a table objective (oracle SearchHooks), the
device runs its update kernel (bp_search_update) on the same rows.  After every
iteration the incumbent, the top-K list, the CEM elite refit (mu, var) and the
MPPI weighted means must agree:

* incumbent value / action, top-K values (and the actions of values that are
  neither tied nor at the list's boundary, where the reference's heap keeps an
  unspecified one of the equal values): bit-exact -- SampleSink::consume,
  search.cpp:41-74;
* CEM mu: bit-exact after rounding the oracle's FP64 mean to FP32 (same elites
  by partial_sort's (value, index) order, same FP64 summation order) -- run_cem,
  search.cpp:131-149; var within 1e-6 relative (the variance floor is formed
  from the FP32 jitter and box width on the device);
* MPPI mu within 1e-6 relative (device exp vs glibc exp) -- search.cpp:192-205.

Costs are drawn from a coarse grid so that ties between elites, between top-K
entries and against the incumbent occur and the tie rules are exercised.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2412_09584_b200 import workloads
from paper_2412_09584_b200.config import from_json

pytestmark = pytest.mark.gpu


def _run(device, cfg_json, method, T=6, seed=0, warm=True):
    wl = workloads.c1(glorot=True)
    dev = device.load(wl.spec)
    d = wl.spec.d
    rng = np.random.default_rng(seed)
    lo = np.full(d, -1.0)
    hi = np.full(d, 1.0)
    lo[:4], hi[:4] = -0.5, 0.25  # a sub-box on some axes (dyadic, FP32-exact centre)
    cfg = from_json(cfg_json)
    s = cfg["search"]
    if s["method"] == "cem":
        G = s["cem"]["agents"]
    else:
        G = len(s["mppi"]["noise_ratios"]) * len(s["mppi"]["temperature_ratios"])
    n_samp = G * (s["samples_per_iter"] // G)
    R = n_samp + 1
    K = s["top_capacity"]
    w = rng.uniform(lo, hi).astype(np.float32).astype(np.float64) if warm else None
    rows = rng.uniform(lo, hi, size=(T, n_samp, d)).astype(np.float32).astype(np.float64)
    costs = (np.round(rng.normal(size=(T, R)) * 6) / 8).astype(np.float32).astype(np.float64)
    # the incumbent row's value: any value at it=0, the incumbent's own value afterwards (a deterministic
    # objective re-evaluates it to uf, the minimum of everything consumed so far)
    uf = np.inf
    for t in range(T):
        if t > 0:
            costs[t, -1] = uf
        uf = min(uf, costs[t].min())
    ref = orc.search_injected(lo, hi, w, cfg, rows, costs)

    inc0 = np.clip(w, lo, hi) if warm else 0.5 * (lo + hi)
    st = {"mu": np.zeros((1, G, d)), "var": np.zeros((1, G, d)), "uf": np.full(1, np.inf), "best": inc0[None],
          "top_n": np.zeros(1), "top_val": np.zeros((1, K)), "top_seq": np.zeros((1, K)), "top_act": np.zeros((1, K, d))}
    for t in range(T):
        r = ref[t]
        st = dev.search_update(cfg, lo[None], hi[None], t, r["batch"][None], costs[t][None], st)
        # incumbent (first row attaining the minimum, strict improvement)
        assert st["uf"][0] == r["uf"], t
        assert np.array_equal(st["best"][0].astype(np.float64), r["best"]), t
        # top-K: the kept values, ascending; actions where the value is not tied
        n = int(st["top_n"][0])
        assert n == r["top_n"] == min(K, (t + 1) * R), t
        dv = st["top_val"][0, :n].astype(np.float64)
        assert np.array_equal(dv, r["top_val"][:n]), t
        # a value below the list's last one has all its instances in the list; unique there = unique
        vals, counts = np.unique(dv, return_counts=True)
        single = np.isin(dv, vals[counts == 1]) & (dv < dv[-1])
        assert np.array_equal(st["top_act"][0, :n][single].astype(np.float64), r["top_act"][:n][single]), t
        # the refit
        if s["method"] == "cem":
            assert np.array_equal(st["mu"][0], r["mu"].astype(np.float32)), t
            assert np.allclose(st["var"][0], r["var"], rtol=1e-6, atol=0), t
        else:
            assert np.allclose(st["mu"][0], r["mu"], rtol=1e-6, atol=1e-7), t
    return ref


def test_cem_update_matches_oracle_on_identical_samples(device):
    _run(device, '{"search": {"samples_per_iter": 64, "top_capacity": 24, "cem": {"elites": 5}}}', "cem")


def test_cem_update_more_elites_than_rows_and_no_warm(device):
    # elites > rows per agent (n_el = min(agent rows, elites); agent 0 owns the incumbent row)
    _run(device, '{"search": {"samples_per_iter": 20, "top_capacity": 8, "cem": {"elites": 9}}}', "cem", warm=False)


def test_cem_update_large_capacity(device):
    # capacity above the rows of one iteration: the list fills over iterations
    _run(device, '{"search": {"samples_per_iter": 40, "top_capacity": 150, "cem": {"agents": 3, "elites": 4}}}', "cem")


def test_mppi_update_matches_oracle_on_identical_samples(device):
    _run(device, '{"search": {"method": "mppi", "samples_per_iter": 60, "top_capacity": 16, '
                 '"mppi": {"temperature": 0.7}}}', "mppi")


def test_mppi_update_instances_grid(device):
    _run(device, '{"search": {"method": "mppi", "samples_per_iter": 48, "top_capacity": 32, '
                 '"mppi": {"noise_ratios": [0.5, 2.0], "temperature_ratios": [0.1, 1.0, 3.0]}}}', "mppi", warm=False)
