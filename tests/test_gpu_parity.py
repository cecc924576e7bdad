"""GPU parity: the sm_100a kernels (through the C-ABI) against the FP64 oracle
on identical FP32-representable inputs.

Tolerances (north star): rollout costs and empirical bounds within 1e-5
relative in FP32 (relative to max(|ref|, 1) for bounds near zero); CROWN lower
bounds from identical extrema within 1e-9 of the bound's term magnitude (the
bound kernel runs in FP64); branching decisions bit-exact.
"""
import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import objective as objmod, workloads
from paper_2412_09584_b200.config import from_json

pytestmark = pytest.mark.gpu

RTOL = 1e-5
# The tcgen05 path computes every Linear layer in 3xTF32 (~2^-21 per product
# instead of FP32's 2^-24).  Costs meet the FP32 bar (1e-5; measured <= 6e-6);
# sample extrema and states get the stated looser tensor-core bar, 2.5e-5 (measured
# <= 1.3e-5: a relative-feature pre-activation x - p cancels), well inside the
# north star's 5e-5 allowance for the TF32 path.
RTOL_TC_COST = 1e-5
RTOL_TC = 2.5e-5


def rtol_for(dev):
    return RTOL_TC if dev.rollout_path() == "tcgen05" else RTOL


def rel_err(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0))) if got.size else 0.0


def small_spec(name):
    if name == "c1":
        return workloads.c1(glorot=True).spec
    if name == "c2":
        return workloads.c2(glorot=True).spec
    if name == "c4":
        return workloads.c4(glorot=True).spec
    if name == "c3":
        return workloads.c3(glorot=True).spec
    if name == "c5":
        return workloads.c5(glorot=True).spec
    if name == "ref-obstacles":  # reference build_objective, relative features, hinges on keypoints and p_t
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, -0.3, 0.1, 0.2], [0.0, 0.0, 0.1, 0.1], [0.0, 0.0]
        s.horizon = 6
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        s.obstacles = [bp.Obstacle([0.2, 0.1], 0.3), bp.Obstacle([-0.1, 0.2], 0.25)]
        s.cost_form = "tracking_obstacles"
        s.lam = 50.0
        return objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(3, [6, 32, 32, 4]), s))
    if name == "ref-linear":  # test_smoke.py's zero-hidden-layer model, relative features
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, 0.4], [0.0, 0.0], [0.0, 0.0]
        s.horizon = 3
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        return objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(1, [4, 2]), s))
    raise KeyError(name)


CASES = ["c1", "c2", "c4", "ref-obstacles", "ref-linear", "c3", "c5"]


@pytest.mark.parametrize("name", CASES)
def test_rollout_costs_and_extrema_match_oracle(device, name):
    spec = small_spec(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    rows = 37 if name not in ("c3", "c5") else 9
    acts = np.random.default_rng(1).uniform(lo, hi, size=(3, rows, spec.d)).astype(np.float32)
    costs, _, elo, ehi, bad = dev.rollout(acts)
    assert not bad.any()
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    for s in range(3):
        st = orc.Stats()
        ref = ob.evaluate(acts[s].astype(np.float64), st)
        tol = rtol_for(dev)
        assert rel_err(costs[s], ref) < (RTOL_TC_COST if dev.rollout_path() == "tcgen05" else RTOL), name
        rlo, rhi = ob.stats_in_layout(st, layout, spec.horizon)
        # the device records x_t at every step; the oracle watches it only where
        # a bound reads it (stop steps, quadratic / ReLU arguments)
        seen = ~np.isnan(rlo)
        assert seen.mean() > 0.5
        assert rel_err(elo[s][seen], rlo[seen]) < tol and rel_err(ehi[s][seen], rhi[seen]) < tol, name


KERNEL_CASES = [("c1", 2), ("c2", 2), ("c4", 1), ("ref-obstacles", 2), ("ref-linear", 2), ("c3", 1)]


@pytest.mark.parametrize("name,tiles", KERNEL_CASES)
@pytest.mark.parametrize("shape", [(3, 37), (2, 300), (1, 700)])
def test_tcgen05_v2_matches_oracle(device, name, tiles, shape):
    """rollout_tc2.cu (two ping-pong tiles per CTA at widths <= 128, one 256-wide tile
    for C3) against the FP64 oracle: subdomains straddling warps and tiles (37 rows),
    a CTA with one live tile (300 rows), several CTAs (700 rows)."""
    spec = small_spec(name)
    dev = device.load(spec)
    # the default for widths in (128, 256]; selectable wherever every width <= 256
    assert dev.rollout_kernel() == "tc2" if name in ("c3", "c4") else "tc1"  # C4: v1's smem does not fit
    assert dev.rollout_path("tc2") == "tcgen05" and dev.rollout_kernel() == "tc2"
    assert dev.rollout_tiles() == tiles  # C4's wide cost scratch leaves room for one tile
    n_sub, rows = shape
    if name == "c3":
        rows = min(rows, 140)  # the FP64 oracle is slow at width 256
    lo, hi = spec.box()
    acts = np.random.default_rng(11).uniform(lo, hi, size=(n_sub, rows, spec.d)).astype(np.float32)
    costs, states, elo, ehi, bad = dev.rollout(acts, want_states=True)
    assert not bad.any()
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    for s in range(n_sub):
        st = orc.Stats()
        ref = ob.evaluate(acts[s].astype(np.float64), st)
        assert rel_err(costs[s], ref) < RTOL_TC_COST, name
        rlo, rhi = ob.stats_in_layout(st, layout, spec.horizon)
        seen = ~np.isnan(rlo)
        assert rel_err(elo[s][seen], rlo[seen]) < RTOL_TC and rel_err(ehi[s][seen], rhi[seen]) < RTOL_TC, name
    # the v2 kernel and the SIMT FP32 kernel see the same rollouts
    dev.rollout_path("simt")
    c_s, st_s, lo_s, hi_s, _ = dev.rollout(acts, want_states=True)
    dev.rollout_path("auto")
    assert rel_err(costs, c_s) < RTOL_TC_COST and rel_err(states, st_s) < RTOL_TC
    assert rel_err(elo, lo_s) < RTOL_TC and rel_err(ehi, hi_s) < RTOL_TC


@pytest.mark.parametrize("shape", [(3, 37), (1, 300), (3, 130)])
def test_tcgen05_v2_cta_pair_matches_one_cta(device, shape, monkeypatch):
    """The CTA-pair form of the 256-wide v2 kernel (BP_TC2_PAIR=1: clusters of two CTAs,
    cta_group::2 MMAs with M = 256, B's rows split between the CTAs) computes the same
    rollouts as the one-CTA form -- bit for bit (the same MMA terms in the same order per
    row) -- and matches the oracle; odd tile counts leave a CTA of the last pair empty."""
    spec = small_spec("c3")
    lo, hi = spec.box()
    n_sub, rows = shape
    acts = np.random.default_rng(5).uniform(lo, hi, size=(n_sub, rows, spec.d)).astype(np.float32)
    one = device.load(spec).rollout(acts, want_states=True)
    monkeypatch.setenv("BP_TC2_PAIR", "1")
    dev = device.load(spec)
    assert dev.rollout_kernel() == "tc2"
    pair = dev.rollout(acts, want_states=True)
    for x, y in zip(one, pair):
        assert np.array_equal(x, y)
    ob = orc.Objective(spec)
    ref = ob.evaluate(acts[0].astype(np.float64))
    assert rel_err(pair[0][0], ref) < RTOL_TC_COST


def v3_spec(name):
    """Objectives for rollout_tc3.cu: C5 itself, ragged widths (two N chunks of 256 + 160
    columns, padded N-blocks), relative features with a 16 + 4 input."""
    if name == "c5":
        return small_spec("c5")
    s = bp.Scenario()
    s.horizon = 5
    if name == "ragged":
        s.x0, s.x_target, s.p0 = [0.4, -0.3, 0.1, 0.2, 0.0, 0.3], [0.0] * 6, [0.0, 0.0]
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        widths = [8, 300, 400, 6]
    else:  # "rel16": relative feature mode, keypoints over a 16-dim state
        s.x0 = list(np.linspace(-0.5, 0.5, 16))
        s.x_target = [0.1] * 16
        s.p0 = [0.0, 0.0, 0.0, 0.0]
        s.u_lower, s.u_upper = [-0.5] * 4, [0.5] * 4
        widths = [20, 512, 288, 16]
    return objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(9, widths), s))


@pytest.mark.parametrize("name", ["c5", "ragged", "rel16"])
@pytest.mark.parametrize("shape", [(3, 37), (2, 300), (1, 700)])
def test_tcgen05_v3_matches_oracle(device, name, shape):
    """rollout_tc3.cu (512-wide hidden layers: layer 1 in N chunks with layer 0 recomputed
    per chunk, layer 2 accumulated across chunks) against the FP64 oracle and the SIMT
    FP32 kernel: costs, states and the recorded extrema."""
    spec = v3_spec(name)
    dev = device.load(spec)
    assert dev.rollout_kernel() == "tc3" and dev.rollout_path() == "tcgen05"
    n_sub, rows = shape
    if name == "c5":
        rows = min(rows, 120)  # the FP64 oracle is slow at width 512
    lo, hi = spec.box()
    acts = np.random.default_rng(13).uniform(lo, hi, size=(n_sub, rows, spec.d)).astype(np.float32)
    costs, states, elo, ehi, bad = dev.rollout(acts, want_states=True)
    assert not bad.any()
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    for s in range(n_sub):
        st = orc.Stats()
        ref = ob.evaluate(acts[s].astype(np.float64), st)
        assert rel_err(costs[s], ref) < RTOL_TC_COST, name
        rlo, rhi = ob.stats_in_layout(st, layout, spec.horizon)
        seen = ~np.isnan(rlo)
        assert rel_err(elo[s][seen], rlo[seen]) < RTOL_TC and rel_err(ehi[s][seen], rhi[seen]) < RTOL_TC, name
    dev.rollout_path("simt")
    c_s, st_s, lo_s, hi_s, _ = dev.rollout(acts, want_states=True)
    dev.rollout_path("auto")
    assert rel_err(costs, c_s) < RTOL_TC_COST and rel_err(states, st_s) < RTOL_TC
    assert rel_err(elo, lo_s) < RTOL_TC and rel_err(ehi, hi_s) < RTOL_TC


@pytest.mark.parametrize("name", ["c5", "ragged"])
@pytest.mark.parametrize("shape", [(3, 37), (1, 300), (3, 130)])
def test_tcgen05_v3_cta_pair_matches_one_cta(device, name, shape, monkeypatch):
    """rollout_tc3.cu's CTA-pair form (BP_TC3_PAIR=1: clusters of two, cta_group::2 MMAs with
    M = 256, each CTA streaming half of every weight block) computes the same rollouts as one
    CTA per tile bit for bit; odd tile counts leave the last pair's second CTA empty."""
    spec = v3_spec(name)
    lo, hi = spec.box()
    n_sub, rows = shape
    acts = np.random.default_rng(6).uniform(lo, hi, size=(n_sub, rows, spec.d)).astype(np.float32)
    dev = device.load(spec)
    one = dev.rollout(acts, want_states=True)
    monkeypatch.setenv("BP_TC3_PAIR", "1")
    pair = dev.rollout(acts, want_states=True)
    for x, y in zip(one, pair):
        assert np.array_equal(x, y)


def test_tcgen05_v3_rows_are_batch_invariant(device):
    spec = v3_spec("ragged")
    dev = device.load(spec)
    lo, hi = spec.box()
    acts = np.random.default_rng(4).uniform(lo, hi, size=(1, 300, spec.d)).astype(np.float32)
    whole, _, _, _, _ = dev.rollout(acts)
    for i in (0, 1, 127, 128, 299):
        one, _, _, _, _ = dev.rollout(acts[:, i:i + 1])
        assert whole[0, i] == one[0, 0]
    split, _, _, _, _ = dev.rollout(acts.reshape(3, 100, spec.d))
    assert np.array_equal(split.reshape(-1), whole.reshape(-1))


@pytest.mark.parametrize("name", ["c1", "c2", "ref-obstacles"])
def test_tcgen05_v1_still_matches_oracle(device, name):
    """The v1 kernel (rollout_tc.cu) stays selectable (BP_ROLLOUT=tc1) and parity-green."""
    spec = small_spec(name)
    dev = device.load(spec)
    assert dev.rollout_path("tc1") == "tcgen05" and dev.rollout_kernel() == "tc1"
    lo, hi = spec.box()
    acts = np.random.default_rng(12).uniform(lo, hi, size=(2, 300, spec.d)).astype(np.float32)
    costs, _, elo, ehi, _ = dev.rollout(acts)
    dev.rollout_path("auto")
    c2, _, lo2, hi2, _ = dev.rollout(acts)
    ob = orc.Objective(spec)
    for s in range(2):
        ref = ob.evaluate(acts[s].astype(np.float64))
        assert rel_err(costs[s], ref) < RTOL_TC_COST
    assert rel_err(costs, c2) < RTOL_TC_COST and rel_err(elo, lo2) < RTOL_TC and rel_err(ehi, hi2) < RTOL_TC


def test_rollout_rows_are_batch_invariant(device):
    spec = small_spec("c2")
    dev = device.load(spec)
    lo, hi = spec.box()
    acts = np.random.default_rng(2).uniform(lo, hi, size=(1, 300, spec.d)).astype(np.float32)
    whole, _, _, _, _ = dev.rollout(acts)
    for i in (0, 1, 127, 128, 129, 299):
        one, _, _, _, _ = dev.rollout(acts[:, i:i + 1])
        assert whole[0, i] == one[0, 0]
    split, _, _, _, _ = dev.rollout(acts.reshape(3, 100, spec.d))
    assert np.array_equal(split.reshape(-1), whole.reshape(-1))


def test_states_match_reference_rollout(device):
    m = bp.generate_model(1, [4, 2])
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = [0.4, 0.4], [0.0, 0.0], [0.0, 0.0]
    s.horizon = 3
    s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
    act = np.array([0.1, -0.2, 0.3, 0.05, -0.4, 0.2])
    states = bp.rollout(m, s, act)
    x, p = s.x0.copy(), s.p0.copy()
    for t in range(3):
        u = act[2 * t:2 * t + 2]
        x = m.forward(np.concatenate([x - p, u]))[0]
        p = p + u
        assert np.allclose(states[t], x, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "ref-obstacles", "ref-linear"])
@pytest.mark.parametrize("alpha", ["adaptive", "zero"])
def test_empirical_bound_matches_oracle_on_identical_extrema(device, name, alpha):
    spec = small_spec(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    c = 0.5 * (lo + hi)
    los = np.stack([lo, np.minimum(c, hi), lo])
    his = np.stack([hi, hi, np.maximum(c, lo)])
    cfg = from_json('{"search": {"samples_per_iter": 64, "iterations": 3}}')
    rep = dev.batch_search(los, his, None, cfg, seed=5)
    lf = dev.batch_bound(3, "early-stop-empirical", alpha)
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    for i in range(3):
        assert rep["ok"][i]
        elo, ehi = dev.report_stats(i)
        st = ob.stats_from_layout(elo.astype(np.float64), ehi.astype(np.float64), layout, spec.horizon)
        ref = ob.lower_bound(los[i], his[i], "early-stop-empirical", st, alpha)
        assert abs(lf[i] - ref) <= 1e-9 * max(1.0, abs(ref)), (name, i, lf[i], ref)
        assert lf[i] <= rep["uf"][i] + 1e-6 * max(1.0, abs(rep["uf"][i]))


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "ref-obstacles", "ref-linear"])
def test_interval_bound_matches_oracle(device, name):
    spec = small_spec(name)
    dev = device.load(spec)
    lo, hi = spec.box()
    lf = dev.bound_boxes(lo[None], hi[None], "early-stop-interval")
    ref = orc.Objective(spec).lower_bound(lo, hi, "early-stop-interval")
    assert abs(lf[0] - ref) <= 1e-9 * max(1.0, abs(ref))


@pytest.mark.parametrize("width", [100, 128, 200, 256, 300, 500, 512])
def test_bound_width_classes_match_oracle(device, width):
    """The bound kernel is instantiated per width class (128 / 256 / 512 scratch doubles
    for the widest layer or cost-scratch row); objectives in each class bound like the
    oracle, full CROWN included."""
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = [0.4, -0.3, 0.1, 0.2], [0.0, 0.0, 0.1, 0.1], [0.0, 0.0]
    s.horizon = 3
    s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
    spec = objmod.round_spec_to_f32(objmod.build_objective(bp.generate_model(7, [6, width, 4]), s))
    dev = device.load(spec)
    lo, hi = spec.box()
    ob = orc.Objective(spec)
    for mode in ("early-stop-interval", "full-crown"):
        lf = dev.bound_boxes(lo[None], hi[None], mode)
        ref = ob.lower_bound(lo, hi, mode)
        assert abs(lf[0] - ref) <= 1e-8 * max(1.0, abs(ref)), (width, mode)


def test_search_properties(device):
    spec = small_spec("c1")
    dev = device.load(spec)
    lo, hi = spec.box()
    cfg = from_json('{"search": {"samples_per_iter": 200, "iterations": 6, "top_capacity": 64}}')
    warm = np.random.default_rng(0).uniform(lo, hi)[None]
    rep = dev.batch_search(lo[None], hi[None], warm, cfg, seed=11)
    warm_val = bp.api.default_device()  # noqa: F841 (keeps the default device alive)
    ob = orc.Objective(spec)
    wv = ob.evaluate(warm.astype(np.float32).astype(np.float64))[0]
    assert rep["ok"][0] and rep["uf"][0] <= wv * (1 + 1e-5) + 1e-6
    v, a = dev.report_top(0, rep["n_top"][0])
    assert 0 < len(v) <= 64 and v[0] == rep["uf"][0] and np.all(np.diff(v) >= 0)
    assert np.all(a >= lo - 1e-7) and np.all(a <= hi + 1e-7)
    assert np.array_equal(a[0], rep["best"][0])
    assert rep["samples"][0] == 6 * (4 * 50 + 1)
    # the device values of the kept samples are the oracle's objective at those points
    ref = ob.evaluate(a.astype(np.float32).astype(np.float64))
    assert rel_err(v, ref) < rtol_for(dev)


def test_search_large_batch_sorts_in_global_memory(device):
    """samples_per_iter + top_capacity above the shared-memory sort (P = 32768 keys, 384 KB):
    search_update sorts in a global scratch instead of failing; the kept list is the oracle's
    objective at the kept points, ascending, and the incumbent is its head."""
    spec = small_spec("c1")
    dev = device.load(spec)
    lo, hi = spec.box()
    cfg = from_json('{"search": {"samples_per_iter": 20000, "iterations": 2, "top_capacity": 512}}')
    rep = dev.batch_search(np.stack([lo, lo]), np.stack([hi, hi]), None, cfg, seed=5)
    ob = orc.Objective(spec)
    for b in range(2):
        assert rep["ok"][b] and rep["samples"][b] == 2 * 20001
        v, a = dev.report_top(b, rep["n_top"][b])
        assert len(v) == 512 and v[0] == rep["uf"][b] and np.all(np.diff(v) >= 0)
        assert rel_err(v, ob.evaluate(a.astype(np.float32).astype(np.float64))) < rtol_for(dev)


def test_search_is_seeded_per_box(device):
    """batch_search equals independent runs with seed ^ index (test_search.cpp:171-188)."""
    spec = small_spec("c1")
    dev = device.load(spec)
    lo, hi = spec.box()
    los = np.stack([lo, lo * 0.5, lo])
    his = np.stack([hi, hi * 0.5, hi * 0.25])
    cfg = from_json('{"search": {"samples_per_iter": 100, "iterations": 4}}')
    batch = dev.batch_search(los, his, None, cfg, seed=99)
    for i in range(3):
        solo = dev.batch_search(los[i:i + 1], his[i:i + 1], None, cfg, seed=99 ^ i)
        assert batch["uf"][i] == solo["uf"][0] and np.array_equal(batch["best"][i], solo["best"][0])
    again = dev.batch_search(los, his, None, cfg, seed=99)
    assert np.array_equal(again["uf"], batch["uf"])


def test_mppi_search_runs(device):
    spec = small_spec("c1")
    dev = device.load(spec)
    lo, hi = spec.box()
    cfg = from_json('{"search": {"method": "mppi", "samples_per_iter": 120, "iterations": 5}}')
    rep = dev.batch_search(lo[None], hi[None], None, cfg, seed=1, method="mppi")
    center = orc.Objective(spec).evaluate((0.5 * (lo + hi))[None])[0]
    assert rep["ok"][0] and rep["uf"][0] <= center * (1 + 1e-5)
    assert rep["samples"][0] == 5 * (3 * 40 + 1)


def test_reference_smoke_plan_reaches_target():
    """proj/tests/python/test_smoke.py:60-76 through the drop-in module."""
    import json
    import math

    m = bp.generate_model(seed=1, widths=[4, 2])
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = np.full(2, 0.4), np.zeros(2), np.zeros(2)
    s.horizon = 3
    s.u_lower, s.u_upper = np.full(2, -0.5), np.full(2, 0.5)
    s.validate()
    cfg = json.loads(bp.default_config())
    cfg["seed"] = 11
    cfg["termination"]["max_iterations"] = 5
    cfg["search"]["samples_per_iter"] = 48
    cfg["search"]["iterations"] = 3
    res = bp.plan(m, s, json.dumps(cfg), method="babnd")
    act = np.asarray(res["action"])
    assert act.shape == (6,)
    assert bp.rollout(m, s, act).shape == (3, 2)
    vals = bp.objective_value(m, s, act.reshape(1, -1))
    assert math.isclose(vals[0], res["objective"], rel_tol=0, abs_tol=1e-9)
    uf = res["trace"]["uf"]
    assert all(a >= b for a, b in zip(uf, uf[1:]))
    assert res["lower_bound"] <= res["objective"] + 1e-9
    assert res["stop_reason"] in {"max-iterations", "pool-exhausted", "target", "wall-clock"}


def test_plan_matches_or_beats_cpu_reference_objective(device):
    """Best objective against the CPU planner (the oracle's bab.cpp restatement) at equal
    iteration count and batch on C1, over 8 seeds.  The samplers differ (Philox on the device,
    mt19937_64 + Box-Muller in the reference), so single runs differ by the seed-to-seed spread
    (~3 % here); the bar is on the median over the seeds: no worse than the CPU's by 1 %, and the
    device's best run no worse than the CPU's best by 1 %.  Both sides are deterministic per seed."""
    wl = workloads.c1()
    dev = device.load(wl.spec)
    ob = orc.Objective(wl.spec)
    gpu, cpu = [], []
    for seed in range(2, 10):
        cfg = wl.planner_config()
        cfg["termination"]["max_iterations"] = 6
        cfg["seed"] = seed
        g = dev.plan(cfg)
        c = ob.plan(cfg)
        assert g["iterations"] == c["iterations"] == 6
        assert g["trace"]["pool_size"][0] == 1
        gpu.append(g["objective"])
        cpu.append(c["objective"])
    gpu, cpu = np.array(gpu), np.array(cpu)
    assert np.median(gpu) <= np.median(cpu) * 1.01, (gpu, cpu)
    assert gpu.min() <= cpu.min() * 1.01, (gpu, cpu)


def test_plan_sample_only_method(device):
    spec = small_spec("c1")
    dev = device.load(spec)
    cfg = from_json('{"search": {"samples_per_iter": 100, "iterations": 4}}')
    res = dev.plan(cfg, method="cem")
    assert res["stop_reason"] == "sampler-budget" and res["iterations"] == 4
    assert res["lower_bound"] == -np.inf and not res["certified"]
    assert len(res["trace"]["uf"]) == 4


def test_nonfinite_rollouts_fail_the_box_not_the_batch(device):
    """search.cpp:273-278 failure isolation: a box whose rollouts overflow is reported failed."""
    spec = small_spec("ref-linear")
    big = objmod.ObjectiveSpec(**{**spec.__dict__, "W": [spec.W[0] * 1e30]})
    dev = device.load(big)
    lo, hi = big.box()
    cfg = from_json('{"search": {"samples_per_iter": 32, "iterations": 2}}')
    rep = dev.batch_search(np.stack([lo, lo]), np.stack([hi, hi]), None, cfg, seed=1)
    assert not rep["ok"].any()
    lf = dev.batch_bound(2)  # no valid samples: the bound falls back to intervals (bab.cpp)
    ref = orc.Objective(big).lower_bound(lo, hi, "early-stop-empirical", None)
    assert lf.shape == (2,)
    for v in lf:
        assert v == ref or abs(v - ref) <= 1e-9 * max(1.0, abs(ref)), (lf, ref)


@pytest.mark.parametrize("name", ["c1", "c2", "ref-obstacles", "ref-linear"])
def test_tcgen05_and_simt_rollouts_agree(device, name):
    """The tcgen05 3xTF32 kernel and the SIMT FP32 kernel against the oracle and each other."""
    spec = small_spec(name)
    dev = device.load(spec)
    assert dev.rollout_path("auto") == "tcgen05"
    lo, hi = spec.box()
    acts = np.random.default_rng(3).uniform(lo, hi, size=(2, 300, spec.d)).astype(np.float32)
    c_tc, _, lo_tc, hi_tc, _ = dev.rollout(acts)
    assert dev.rollout_path("simt") == "simt"
    c_simt, _, lo_s, hi_s, _ = dev.rollout(acts)
    dev.rollout_path("auto")
    ob = orc.Objective(spec)
    for s in range(2):
        ref = ob.evaluate(acts[s].astype(np.float64))
        assert rel_err(c_tc[s], ref) < RTOL_TC_COST and rel_err(c_simt[s], ref) < RTOL
    assert rel_err(lo_tc, lo_s) < RTOL_TC and rel_err(hi_tc, hi_s) < RTOL_TC


def fold_spec(name):
    """Objectives whose cost program reads x_t through LINEAR ops (folded into the v2 output
    layer's MMA, host.cu): C4, and a 160-wide model whose 70 folded columns plus x_t span
    three 32-column chunks, with a folded op feeding a SUM, a SLICE and a RELU."""
    if name == "c4":
        return workloads.c4(glorot=True).spec
    from paper_2412_09584_b200.objective import Op, X, op_id
    from paper_2412_09584_b200._capi import BP_OP_LINEAR, BP_OP_RELU, BP_OP_SLICE, BP_OP_SUM
    r = np.random.default_rng(3)
    W1 = (r.standard_normal((70, 12)) / 4).astype(np.float32)
    W2 = (r.standard_normal((12, 12)) / 4).astype(np.float32)
    ops = [Op(BP_OP_LINEAR, X, dim=70, W=W1, b=r.standard_normal(70).astype(np.float32)),
           Op(BP_OP_RELU, op_id(0)),
           Op(BP_OP_LINEAR, op_id(1), dim=1, W=np.ones((1, 70)), b=np.zeros(1), is_term=True),
           Op(BP_OP_LINEAR, X, dim=12, W=W2, b=np.zeros(12)),
           Op(BP_OP_SLICE, op_id(3), begin=2, dim=5),
           Op(BP_OP_SUM, op_id(4), src1=op_id(4)),
           Op(BP_OP_RELU, op_id(5)),
           Op(BP_OP_LINEAR, op_id(6), dim=1, W=np.ones((1, 5)), b=np.zeros(1), is_term=True)]
    return workloads._spec([14, 160, 160, 12], 12, 2, 7, ops, glorot=True)


@pytest.mark.parametrize("name", ["c4", "wide"])
def test_v2_folded_cost_linears_match_oracle_and_unfolded(device, name, monkeypatch):
    """Cost-program LINEARs on x_t computed as extra N columns of the v2 output layer's MMA
    (W_op W_L, W_op b_L + b_op): the same costs and extrema as the oracle and as the
    unfolded kernel (BP_NO_FOLD=1) within the 3xTF32 tolerance."""
    spec = fold_spec(name)
    lo, hi = spec.box()
    acts = np.random.default_rng(12).uniform(lo, hi, size=(2, 300, spec.d)).astype(np.float32)
    dev = device.load(spec)
    assert dev.rollout_kernel() == "tc2"
    costs, states, elo, ehi, bad = dev.rollout(acts, want_states=True)
    assert not bad.any()
    monkeypatch.setenv("BP_NO_FOLD", "1")
    dev2 = bp.Device(0).load(spec)
    assert dev2.rollout_kernel() == "tc2"
    c2, s2, lo2, hi2, _ = dev2.rollout(acts, want_states=True)
    assert rel_err(costs, c2) < RTOL_TC_COST and rel_err(states, s2) < RTOL_TC
    assert rel_err(elo, lo2) < RTOL_TC and rel_err(ehi, hi2) < RTOL_TC
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    for s in range(2):
        st = orc.Stats()
        ref = ob.evaluate(acts[s].astype(np.float64), st)
        assert rel_err(costs[s], ref) < RTOL_TC_COST, name
        rlo, rhi = ob.stats_in_layout(st, layout, spec.horizon)
        seen = ~np.isnan(rlo)
        assert rel_err(elo[s][seen], rlo[seen]) < RTOL_TC and rel_err(ehi[s][seen], rhi[seen]) < RTOL_TC, name
