"""Branching on the device (pool.cu): split and merge_report over the device slab
against the oracle's restatement of the reference (bab.cpp:155-223, 245-262).

Both are comparisons, integer counts and copies, so the bar is bit-exact: the axis,
the midpoint, the child boxes, the routed top lists (order included) and the merged
lists / incumbents.  Inputs are FP32-representable, as on the device."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def random_parents(rng, n, d, K, degenerate=False, tied=False):
    lo = rng.uniform(-2, 0, (n, d))
    hi = lo + rng.uniform(0.01, 2, (n, d))
    if degenerate:
        hi[:, 0] = lo[:, 0]  # an axis below the width floor
    n_top = rng.integers(0, K + 1, n)
    n_top[0] = 0
    n_top[-1] = K
    tv = np.zeros((n, K), np.float32)
    ta = np.zeros((n, K, d), np.float32)
    for i in range(n):
        k = n_top[i]
        v = rng.integers(0, 5, k) if tied else rng.normal(size=k)
        tv[i, :k] = np.sort(v).astype(np.float32)
        if tied:  # samples exactly on the midpoint of every axis
            ta[i, :k] = (0.5 * (lo[i] + hi[i])).astype(np.float32)
            ta[i, :k:3] = rng.uniform(lo[i], hi[i], (len(range(0, k, 3)), d)).astype(np.float32)
        else:
            ta[i, :k] = rng.uniform(lo[i], hi[i], (k, d)).astype(np.float32)
    lo, hi = lo.astype(np.float32).astype(np.float64), hi.astype(np.float32).astype(np.float64)
    samples = rng.integers(0, 5000, n)
    samples[1 % n] = 0
    return lo, hi, tv, ta, n_top, samples


@pytest.mark.parametrize("d,K,rule,tp", [(1, 8, 0, 1.0), (6, 40, 0, 1.0), (6, 40, 1, 1.0), (24, 300, 0, 5.0),
                                          (200, 512, 0, 1.0), (33, 17, 0, 50.0)])
@pytest.mark.parametrize("tied", [False, True])
def test_split_matches_oracle(device, d, K, rule, tp, tied):
    rng = np.random.default_rng(d * 1000 + K + rule + 7 * tied)
    n = 24
    lo, hi, tv, ta, n_top, samples = random_parents(rng, n, d, K, degenerate=d > 1, tied=tied)
    axis, clo, chi, cn, cv, ca = device.pool_split(lo, hi, tv, ta, n_top, samples, tp, 1e-6, rule)
    for i in range(n):
        k = n_top[i]
        ref_axis, ref_mid, route = orc.split(lo[i], hi[i], tv[i, :k].astype(np.float64), ta[i, :k].astype(np.float64),
                                             int(samples[i]), tp, 1e-6, rule)
        assert axis[i] == ref_axis, i
        exp_lo_hi = hi[i].copy()
        exp_lo_hi[ref_axis] = ref_mid
        exp_hi_lo = lo[i].copy()
        exp_hi_lo[ref_axis] = ref_mid
        assert np.array_equal(clo[2 * i], lo[i]) and np.array_equal(chi[2 * i], exp_lo_hi)
        assert np.array_equal(clo[2 * i + 1], exp_hi_lo) and np.array_equal(chi[2 * i + 1], hi[i])
        for b in (0, 1):
            sel = np.flatnonzero(route == b)
            c = 2 * i + b
            assert cn[c] == len(sel)
            assert np.array_equal(cv[c, :len(sel)], tv[i, sel])
            assert np.array_equal(ca[c, :len(sel)], ta[i, sel])


def test_split_without_axis_raises(device):
    lo = np.zeros((2, 3))
    hi = np.ones((2, 3))
    hi[1] = lo[1]  # nothing above the floor
    with pytest.raises(ValueError, match="no axis above the width floor"):
        device.pool_split(lo, hi, np.zeros((2, 4)), np.zeros((2, 4, 3)), [0, 0], [0, 0])


def random_lists(rng, n, K, d, tied):
    cnt = rng.integers(0, K + 1, n)
    val = np.zeros((n, K), np.float32)
    act = rng.uniform(-1, 1, (n, K, d)).astype(np.float32)
    for i in range(n):
        v = rng.integers(0, 6, cnt[i]) if tied else rng.normal(size=cnt[i])
        val[i, :cnt[i]] = np.sort(v).astype(np.float32)
    return cnt, val, act


@pytest.mark.parametrize("d,K,cap", [(1, 4, 4), (7, 32, 32), (7, 32, 20), (200, 512, 512), (5, 1, 0)])
@pytest.mark.parametrize("tied", [False, True])
def test_merge_matches_oracle(device, d, K, cap, tied):
    rng = np.random.default_rng(d + K + cap + 3 * tied)
    n = 30
    a_n, a_val, a_act = random_lists(rng, n, K, d, tied)
    b_n, b_val, b_act = random_lists(rng, n, K, d, tied)
    a_n[0], b_n[1], a_n[2], b_n[2] = 0, 0, 0, 0
    b_uf = np.where(b_n > 0, b_val[:, 0], np.float32(np.inf)).astype(np.float32)
    b_uf[3] = np.float32(-10.0)  # a search incumbent below its own stored list
    b_best = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    failed = np.zeros(n, np.int32)
    failed[4] = 1
    on, ov, oa, ou, oh, ob = device.pool_merge(cap, a_n, a_val, a_act, b_n, b_val, b_act, b_uf, b_best, failed)
    for i in range(n):
        na, nb = a_n[i], (0 if failed[i] else b_n[i])
        a_uf = float(a_val[i, 0]) if na else np.inf
        a_best = a_act[i, 0] if na else None
        r_uf = np.inf if failed[i] else float(b_uf[i])
        r_best = None if failed[i] else b_best[i]
        rv, ra, uf, best = orc.merge_report(cap, a_val[i, :na], a_act[i, :na], a_uf, a_best, b_val[i, :nb],
                                            b_act[i, :nb], r_uf, r_best)
        assert on[i] == len(rv), i
        assert np.array_equal(ov[i, :on[i]], rv.astype(np.float32)), i
        assert np.array_equal(oa[i, :on[i]], ra.astype(np.float32)), i
        assert ou[i] == np.float32(uf), i
        assert oh[i] == (best is not None), i
        if best is not None:
            assert np.array_equal(ob[i], best.astype(np.float32)), i


def test_search_after_plan_sees_its_own_boxes():
    """A plan sizes the context's search buffers for its children per step; a later
    batch_search on the same context (fewer boxes, a warm start) must give exactly what
    a fresh context gives (regression: buffers reallocated between upload and use)."""
    import paper_2412_09584_b200 as bp
    from paper_2412_09584_b200 import workloads

    wl = workloads.c1(glorot=True)
    cfg = wl.planner_config()
    cfg["batch"] = 64
    cfg["termination"]["max_iterations"] = 2
    cfg["search"]["samples_per_iter"] = 128
    cfg["search"]["iterations"] = 3
    lo, hi = wl.spec.box()
    warm = np.random.default_rng(3).uniform(lo, hi).astype(np.float32).astype(np.float64)
    used = bp.Device(0).load(wl.spec)
    used.plan(cfg)
    a = used.batch_search(lo[None], hi[None], warm[None], cfg, seed=11)
    b = bp.Device(0).load(wl.spec).batch_search(lo[None], hi[None], warm[None], cfg, seed=11)
    assert a["uf"][0] == b["uf"][0] and np.array_equal(a["best"], b["best"])
