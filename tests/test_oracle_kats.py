"""Pins the FP64 oracle to the reference's own known-answer tests and property
checks (proj/tests/test_graph.cpp, test_crown.cpp, test_model.cpp,
test_search.cpp, test_bab.cpp).  CPU only."""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2412_09584_b200 import objective as objmod
from paper_2412_09584_b200.model import Obstacle, Scenario
from paper_2412_09584_b200.workloads import f32


def small_graph():
    """y = sqdist(relu(Wx+b)) + hinge(x[0:2]) (test_graph.cpp:36-48)."""
    g = orc.Graph()
    i = g.input(3)
    lin = g.linear(i, [[1.0, -2.0, 0.5], [0.0, 1.0, 1.0]], [0.1, -0.2])
    act = g.relu(lin)
    sq = g.squared_distance(act, [0.0, 0.0], [1.0, 2.0])
    sl = g.slice(i, 0, 2)
    h = g.penalty_hinge(sl, [0.5, 0.5], 0.3, 10.0)
    g.set_output(g.sum([sq, h]))
    g.finalize()
    return g


def by_hand(x):
    z0 = x[0] - 2 * x[1] + 0.5 * x[2] + 0.1
    z1 = x[1] + x[2] - 0.2
    a0, a1 = max(0.0, z0), max(0.0, z1)
    return a0 * a0 + 2 * a1 * a1 + 10.0 * max(0.0, 0.3 - math.hypot(x[0] - 0.5, x[1] - 0.5))


def test_mt19937_64_known_answer():
    # The C++ standard fixes the 10000th output of a default-seeded mt19937_64.
    r = orc.Rng(5489)
    for _ in range(9999):
        r.bits()
    assert r.bits() == 9981545732273789042


def test_mix_seed_matches_splitmix_restatement():
    M = 2**64 - 1
    for m, s in [(0, 0), (1, 1), (2, 7), (2**63 + 5, 3)]:
        z = (m + 0x9E3779B97F4A7C15 * (s + 1)) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        assert orc.mix_seed(m, s) == z ^ (z >> 31)


def test_rng_uniform_and_normal_mapping():
    a, b = orc.Rng(7), orc.Rng(7)
    for _ in range(100):
        assert a.uniform() == (b.bits() >> 11) * 2.0**-53
    r, s = orc.Rng(3), orc.Rng(3)
    x = [r.normal() for _ in range(4)]
    u1, u2 = s.uniform(), s.uniform()
    rad = math.sqrt(-2 * math.log(u1))
    assert x[0] == rad * math.cos(2 * math.pi * u2) and x[1] == rad * math.sin(2 * math.pi * u2)


def test_evaluate_matches_hand_computed():  # test_graph.cpp:52-61
    g = small_graph()
    r = orc.Rng(7)
    batch = np.array([[r.uniform() * 4 - 2 for _ in range(3)] for _ in range(40)])
    got = g.evaluate(batch)
    for i in range(40):
        assert got[i] == pytest.approx(by_hand(batch[i]), rel=1e-12)


def test_evaluate_bitwise_batch_invariant():  # test_graph.cpp:71-82
    g = small_graph()
    batch = np.random.default_rng(11).uniform(-1, 1, (33, 3))
    whole = g.evaluate(batch)
    for i in range(33):
        assert whole[i] == g.evaluate(batch[i:i + 1])[0]


def test_watch_stats_exact_extrema():  # test_graph.cpp:84-98
    g = small_graph()
    st = orc.Stats()
    g.evaluate(np.eye(3), watch=[1], stats=st)
    mn, mx, cnt = st.get(1, 2)
    assert cnt == 3
    assert mn[0] == pytest.approx(-1.9) and mx[0] == pytest.approx(1.1)
    assert mn[1] == pytest.approx(-0.2) and mx[1] == pytest.approx(0.8)


def test_watch_stats_merge_like_one_pass():  # test_graph.cpp:100-116
    g = small_graph()
    batch = np.random.default_rng(3).uniform(-2, 2, (20, 3))
    whole, split = orc.Stats(), orc.Stats()
    g.evaluate(batch, [1, 2], whole)
    g.evaluate(batch[:7], [1, 2], split)
    g.evaluate(batch[7:], [1, 2], split)
    for node in (1, 2):
        a, b = whole.get(node, 2), split.get(node, 2)
        assert a[2] == b[2] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_gradient_matches_central_differences():  # test_graph.cpp:118-137
    g = small_graph()
    rng = np.random.default_rng(5)
    checked = 0
    while checked < 12:
        x = rng.uniform(-2, 2, 3)
        z0, z1 = x[0] - 2 * x[1] + 0.5 * x[2] + 0.1, x[1] + x[2] - 0.2
        dist = math.hypot(x[0] - 0.5, x[1] - 0.5)
        if min(abs(z0), abs(z1), abs(dist - 0.3), dist) < 1e-3:
            continue
        got = g.gradient(x[None])[0]
        for j in range(3):
            e = np.zeros(3)
            e[j] = 1e-6
            fd = (g.evaluate((x + e)[None])[0] - g.evaluate((x - e)[None])[0]) / 2e-6
            assert got[j] == pytest.approx(fd, rel=1e-5, abs=1e-6)
        checked += 1


def test_interval_encloses_samples():  # test_graph.cpp:139-158
    g = small_graph()
    lo, hi = np.array([-1.0, -0.5, 0.0]), np.array([1.0, 0.5, 2.0])
    batch = np.random.default_rng(9).uniform(lo, hi, (200, 3))
    st = orc.Stats()
    g.evaluate(batch, list(range(g.size())), st)
    for node in range(g.size()):
        a, b = g.interval(lo, hi, node)
        mn, mx, _ = st.get(node, g.dim(node))
        assert np.all(a <= mn + 1e-12) and np.all(b >= mx - 1e-12)


def test_builder_rejects_malformed_graphs():  # test_graph.cpp:160-173
    g = orc.Graph()
    i = g.input(2)
    with pytest.raises(ValueError):
        g.slice(i, 1, 5)
    lin = g.linear(i, np.eye(2), np.zeros(2))
    with pytest.raises(ValueError):
        g.set_output(lin)
    with pytest.raises(ValueError):
        g.finalize()


def relax(l, u, pol):
    import ctypes as C
    L = orc.lib()
    out = [np.zeros(len(l)) for _ in range(4)]
    l, u = np.asarray(l, float), np.asarray(u, float)
    orc.ck(L.or_relax_relu(l.ctypes.data_as(orc.dp), u.ctypes.data_as(orc.dp), C.c_int(len(l)), C.c_int(pol),
                           *[o.ctypes.data_as(orc.dp) for o in out]))
    return out


def test_relu_relaxation_sandwich_and_kats():  # test_crown.cpp:49-82
    rng = np.random.default_rng(101)
    for _ in range(300):
        l, u = sorted(rng.uniform(-4, 4, 2))
        for pol in (0, 1, 2):
            ls, lo, us, uo = relax([l], [u], pol)
            for z in np.linspace(l, u, 21):
                y = max(0.0, z)
                assert ls[0] * z + lo[0] <= y + 1e-12 and us[0] * z + uo[0] >= y - 1e-12
    ls, lo, us, uo = relax([0.5], [2.0], 0)
    assert (ls[0], lo[0], us[0]) == (1.0, 0.0, 1.0)
    ls, lo, us, uo = relax([-2.0], [-0.5], 0)
    assert (ls[0], us[0], uo[0]) == (0.0, 0.0, 0.0)
    assert relax([-1.0], [3.0], 0)[0][0] == 1.0
    assert relax([-3.0], [1.0], 0)[0][0] == 0.0


def test_concretize_kat():  # test_crown.cpp:169-187
    import ctypes as C
    L = orc.lib()
    dims = np.array([2], dtype=np.int32)
    c = np.array([2.0, -3.0])
    lo, hi = np.array([-1.0, -2.0]), np.array([0.5, 4.0])
    out = C.c_double()
    for lower, want in ((1, 1.5 + 2.0 * -1.0 + -3.0 * 4.0), (0, 1.5 + 2.0 * 0.5 + -3.0 * -2.0)):
        orc.ck(L.or_concretize(C.c_double(1.5), 1, dims.ctypes.data_as(orc.ip), c.ctypes.data_as(orc.dp),
                               lo.ctypes.data_as(orc.dp), hi.ctypes.data_as(orc.dp), lower, C.byref(out)))
        assert out.value == pytest.approx(want)


def network(seed, widths, affine=False):
    """build_network_objective(generate_model(seed, widths)) (model.cpp:389-405)."""
    p = orc.generate_model_params(seed, widths)
    g = orc.Graph()
    h = g.input(widths[0])
    off, last_relu = 0, -1
    for i in range(len(widths) - 1):
        a, b = widths[i], widths[i + 1]
        W = p[off:off + a * b].reshape(b, a)
        off += a * b
        bias = p[off:off + b]
        off += b
        h = g.linear(h, W, bias)
        if i + 2 < len(widths) and not affine:
            h = g.relu(h)
            last_relu = h
    g.set_output(h)
    g.finalize()
    return g, g.objective((), last_relu)


def random_net(seed, rng, max_layers=4, max_width=32, max_dim=4):
    d = 1 + rng.uniform_int(max_dim)
    layers = 1 + rng.uniform_int(max_layers)
    widths = [d] + [2 + rng.uniform_int(max_width - 1) for _ in range(layers)] + [1]
    return network(seed, widths)


def random_box(d, rng, max_half=2.0):
    lo = np.array([-(0.1 + (max_half - 0.1) * rng.uniform()) for _ in range(d)])
    hi = np.array([0.1 + (max_half - 0.1) * rng.uniform() for _ in range(d)])
    return lo, hi


def test_sound_bounds_on_random_networks():  # test_crown.cpp:84-96
    rng = orc.Rng(7)
    for t in range(20):
        g, obj = random_net(1000 + t, rng)
        lo, hi = random_box(obj.dim, rng)
        pts = np.random.default_rng(t).uniform(lo, hi, (500, obj.dim))
        truth = obj.evaluate(pts).min()
        for pol in ("adaptive", "zero", "one"):
            assert obj.lower_bound(lo, hi, "full-crown", None, pol) <= truth + 1e-9
        assert obj.lower_bound(lo, hi, "early-stop-interval") <= truth + 1e-9


def test_affine_networks_are_exact():  # test_crown.cpp:98-111
    rng = orc.Rng(19)
    for t in range(15):
        d = 1 + rng.uniform_int(5)
        g, obj = network(2000 + t, [d, 3 + rng.uniform_int(5), 1], affine=True)
        lo, hi = random_box(d, rng)
        verts = np.array(np.meshgrid(*[[lo[j], hi[j]] for j in range(d)])).reshape(d, -1).T
        truth = obj.evaluate(verts).min()
        assert obj.lower_bound(lo, hi, "full-crown") == pytest.approx(truth, rel=1e-12, abs=1e-12)
        assert obj.lower_bound(lo, hi, "early-stop-interval") == pytest.approx(truth, rel=1e-12, abs=1e-12)


def test_empirical_never_exceeds_samples_and_can_beat_sound():  # test_crown.cpp:113-147
    rng = orc.Rng(43)
    tighter = 0
    for t in range(20):
        g, obj = random_net(4000 + t, rng, 3, 16, 3)
        lo, hi = random_box(obj.dim, rng, 3.0)
        c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
        pts = np.random.default_rng(t).uniform(c - h / 3, c + h / 3, (300, obj.dim))
        st = orc.Stats()
        vals = obj.evaluate(pts, st)
        emp = obj.lower_bound(lo, hi, "early-stop-empirical", st)
        sound = obj.lower_bound(lo, hi, "early-stop-interval")
        assert emp <= vals.min() + 1e-9
        tighter += emp > sound + 1e-12
    assert tighter > 0


def test_interval_zero_alpha_monotone_under_shrink():  # test_crown.cpp:149-167
    rng = orc.Rng(47)
    for t in range(15):
        g, obj = random_net(5000 + t, rng, 3, 12, 3)
        lo, hi = random_box(obj.dim, rng)
        w = hi - lo
        ilo = lo + 0.25 * w * np.array([rng.uniform() for _ in range(obj.dim)])
        ihi = hi - 0.25 * w * np.array([rng.uniform() for _ in range(obj.dim)])
        assert obj.lower_bound(ilo, ihi, "early-stop-interval", None, "zero") >= \
            obj.lower_bound(lo, hi, "early-stop-interval", None, "zero") - 1e-9


def model_params(seed, widths):
    from paper_2412_09584_b200.model import Model
    p = orc.generate_model_params(seed, widths)
    Ws, bs, off = [], [], 0
    for i in range(len(widths) - 1):
        a, b = widths[i], widths[i + 1]
        Ws.append(p[off:off + a * b].reshape(b, a))
        off += a * b
        bs.append(p[off:off + b])
        off += b
    return Model(widths, Ws, bs)


def two_step():
    s = Scenario()
    s.x0, s.x_target, s.p0 = [0.4, -0.3], [0.0, 0.0], [0.0, 0.0]
    s.horizon = 2
    s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
    return s


def test_unrolled_objective_equals_manual_rollout():  # test_model.cpp:131-185
    for obstacles in (False, True):
        s = two_step()
        if obstacles:
            s.obstacles = [Obstacle([0.1, 0.1], 0.4)]
            s.cost_form = "tracking_obstacles"
        m = model_params(17 if not obstacles else 29, [4, 10 if not obstacles else 8, 2])
        obj = orc.Objective(objmod.build_objective(m, s))
        lo, hi = obj.box()
        assert np.array_equal(lo, [-0.5] * 4) and np.array_equal(hi, [0.5] * 4)
        for u in np.random.default_rng(23).uniform(-0.5, 0.5, (20, 4)):
            x, p, want = s.x0.copy(), s.p0.copy(), 0.0
            for step in range(2):
                us = u[2 * step:2 * step + 2]
                x = m.forward(np.concatenate([x - p, us]))[0]
                p = p + us
                want += s.tracking_weight(step + 1) * np.sum((x - s.x_target) ** 2)
                if obstacles:
                    for o in s.obstacles:
                        for pt in (x, p):
                            want += s.lam * max(0.0, o.size - np.linalg.norm(pt - o.center))
            assert obj.evaluate(u[None])[0] == pytest.approx(want, rel=1e-10)


def test_scenario_bound_sound_across_modes():  # test_crown.cpp:202-219
    s = Scenario()
    s.x0, s.x_target, s.p0 = [0.3, -0.2], [0.0, 0.0], [0.0, 0.0]
    s.horizon = 2
    s.u_lower, s.u_upper = [-0.4, -0.4], [0.4, 0.4]
    s.obstacles = [Obstacle([0.15, 0.0], 0.1)]
    s.cost_form = "tracking_obstacles"
    obj = orc.Objective(objmod.build_objective(model_params(77, [4, 12, 12, 2]), s))
    lo, hi = obj.box()
    truth = obj.evaluate(np.random.default_rng(53).uniform(lo, hi, (2000, 4))).min()
    assert obj.lower_bound(lo, hi, "full-crown") <= truth + 1e-9
    assert obj.lower_bound(lo, hi, "early-stop-interval") <= truth + 1e-9


def bowl(at):
    g = orc.Graph()
    i = g.input(len(at))
    g.set_output(g.squared_distance(i, at, np.ones(len(at))))
    g.finalize()
    return g, g.objective()


def small_cfg(method, iters=12, spi=60, cap=32):
    from paper_2412_09584_b200.config import from_json
    c = from_json("{}")
    c["search"].update(method=method, samples_per_iter=spi, iterations=iters, top_capacity=cap)
    return c


def test_search_improves_bowl_and_keeps_warm_start():  # test_search.cpp:58-91
    g, obj = bowl([0.4, -0.6, 0.2])
    for m in ("cem", "mppi", "gd"):
        rep = obj.batch_search(-np.ones(3), np.ones(3), None, small_cfg(m), seed=3).get(0)
        assert rep["ok"] and rep["uf"] < 0.05 and np.all(np.abs(rep["best"]) <= 1 + 1e-12)
    g, obj = bowl([2.0, 2.0])
    for m in ("cem", "mppi", "gd"):
        rep = obj.batch_search(-np.ones(2), np.ones(2), np.array([[5.0, 5.0]]), small_cfg(m), seed=7).get(0)
        assert rep["uf"] == pytest.approx(2.0, rel=1e-9)


def test_search_top_sorted_and_batch_equals_solo():  # test_search.cpp:130-188
    obj = orc.Objective(synthetic_dim=2)
    cfg = small_cfg("cem", cap=9)
    rep = obj.batch_search(-np.ones(2), np.ones(2), None, cfg, seed=31).get(0)
    tv = rep["top_values"]
    assert 0 < len(tv) <= 9 and tv[0] == rep["uf"] and np.all(np.diff(tv) >= 0)
    los = np.array([[-1.0, -1.0], [0.0, -1.0], [-0.5, -0.5]])
    his = np.array([[0.0, 1.0], [1.0, 1.0], [0.5, 0.5]])
    batch = obj.batch_search(los, his, None, small_cfg("cem"), seed=99)
    for i in range(3):
        solo = obj.batch_search(los[i:i + 1], his[i:i + 1], None, small_cfg("cem"), seed=99 ^ i).get(0)
        b = batch.get(i)
        assert b["uf"] == solo["uf"] and np.array_equal(b["best"], solo["best"])


def test_pick_out_kats():  # test_bab.cpp:68-106
    meta = [(-10.0 + i, float(i), i, 0.0) for i in range(8)]
    assert orc.pick_out(meta, 4, 1.0, 0.05, orc.Rng(5)) == [0, 1, 2, 3]
    low = sum(orc.pick_out([(-100.0 if i == 3 else 0.0, 1.0, i, 0.0) for i in range(6)], 1, 0.0, 0.05,
                           orc.Rng(100 + t)) == [3] for t in range(50))
    assert low >= 48
    assert sorted(orc.pick_out([(-math.inf, 0.5, 0, 0.0), (-1.0, 0.25, 1, 0.0)], 10, 0.5, 0.05, orc.Rng(9))) == [0, 1]


def test_split_kats():  # test_bab.cpp:108-164
    top = np.array([[x, 0.5] for x in (0.5, 0.6, 0.7, 0.8)])
    axis, mid, route = orc.split([0, 0], [4, 1], [0.5, 0.6, 0.7, 0.8], top, 4, 100.0)
    assert axis == 0 and mid == 2.0 and list(route) == [0, 0, 0, 0]
    top = np.array([[x, 3 * x] for x in (0.2, 0.8)])
    assert orc.split([0, 0], [1, 3], [0.2, 0.8], top, 2, 100.0)[0] == 1
    assert orc.split([0, 0], [1e-9, 5], [], None, 0, 100.0)[0] == 1


def test_prune_kat():  # test_bab.cpp:166-180
    keep, removed = orc.prune([(1.0, 2.0, 0, math.log(0.25)), (0.0, 2.0, 1, math.log(0.5)),
                               (-1.0, 2.0, 2, math.log(0.25))], 0.0)
    assert keep == [1, 2] and removed == pytest.approx(0.25)


def test_planner_separable_bracket_and_determinism():  # test_bab.cpp:182-234
    obj = orc.Objective(synthetic_dim=2)
    from paper_2412_09584_b200.config import from_json
    cfg = from_json('{"seed": 7, "search": {"samples_per_iter": 48, "iterations": 4, "top_capacity": 48},'
                    ' "termination": {"max_iterations": 12}}')
    a = obj.plan(cfg)
    truth = 2 * -0.980339434486584
    assert a["certified"] and a["lower_bound"] <= truth + 1e-9 <= a["objective"] + 2e-9
    assert a["objective"] <= truth + 0.5 and a["stop_reason"] == "max-iterations"
    uf = a["trace"]["uf"]
    assert all(x >= y for x, y in zip(uf, uf[1:]))
    b = obj.plan(cfg)
    assert a["objective"] == b["objective"] and a["trace"]["min_lf"] == b["trace"]["min_lf"]


def test_graph_objective_plan_properties():  # test_bab.cpp:274-295
    s = Scenario()
    s.x0, s.x_target, s.p0 = [0.3, -0.2], [0.0, 0.0], [0.0, 0.0]
    s.horizon = 2
    s.u_lower, s.u_upper = [-0.4, -0.4], [0.4, 0.4]
    obj = orc.Objective(objmod.build_objective(model_params(5, [4, 10, 2]), s))
    from paper_2412_09584_b200.config import from_json
    cfg = from_json('{"seed": 51, "search": {"samples_per_iter": 48, "iterations": 4, "top_capacity": 48},'
                    ' "termination": {"max_iterations": 12}}')
    emp = obj.plan(cfg)
    assert not emp["certified"] and emp["lower_bound"] <= emp["objective"] + 1e-9
    cfg["bound_mode"] = "full-crown"
    sound = obj.plan(cfg)
    assert sound["certified"] and sound["lower_bound"] <= sound["objective"] + 1e-9


def test_search_injection_hooks_restate_the_sink_and_refit():
    """The oracle's injection hooks (used by the device sampler-update parity tests) leave run_cem's
    own logic in charge: after each iteration uf / best are the first minimum so far, the top list is
    the K smallest values consumed, and agent g's mean is the mean of its n_el best rows in (value,
    row) order (search.cpp:41-74, 131-149)."""
    from paper_2412_09584_b200.config import from_json

    cfg = from_json('{"search": {"samples_per_iter": 24, "top_capacity": 10, "cem": {"agents": 3, "elites": 4}}}')
    d, T = 5, 3
    rng = np.random.default_rng(1)
    lo, hi = -np.ones(d), np.ones(d)
    rows = rng.uniform(lo, hi, size=(T, 24, d))
    costs = np.round(rng.normal(size=(T, 25)) * 4) / 8
    ref = orc.search_injected(lo, hi, None, cfg, rows, costs)
    seen = []
    for t in range(T):
        b = ref[t]["batch"]
        assert np.array_equal(b[:24], rows[t])
        seen += list(costs[t])
        assert ref[t]["uf"] == min(seen)
        assert np.array_equal(ref[t]["top_val"][:ref[t]["top_n"]], np.sort(seen)[:10])
        for g in range(3):
            idx = list(range(8 * g, 8 * g + 8)) + ([24] if g == 0 else [])
            el = sorted(idx, key=lambda i: (costs[t][i], i))[:4]
            m = np.zeros(d)
            for i in el:
                m += b[i]
            assert np.array_equal(ref[t]["mu"][g], m / 4)
