"""CPU checks of the C-ABI library: it loads, exports every symbol the header
declares, and its host-side restatements (Rng stream, generate_model,
pick_out) agrees bit-for-bit with the oracle (split / merge_report run on the
device: tests/test_gpu_pool.py).  No GPU compute."""
import ctypes as C
import json
import math
import os
import re

import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import _capi, config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "babplan_cuda.h")).read()
    return sorted(set(re.findall(r"^\s*(?:bp_status|uint64_t|size_t)\s+(bp_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    syms = header_symbols()
    assert len(syms) >= 30
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTS) == sorted(syms)


def test_rng_stream_matches_oracle():
    lib = _capi.load()
    h = C.c_void_p()
    _capi.check(lib.bp_rng_new(123, C.byref(h)))
    r = orc.Rng(123)
    out = C.c_double()
    for i in range(200):
        if i % 3 == 0:
            _capi.check(lib.bp_rng_normal(h, C.byref(out)))
            assert out.value == r.normal()
        else:
            _capi.check(lib.bp_rng_uniform(h, C.byref(out)))
            assert out.value == r.uniform()
    lib.bp_rng_free(h)
    assert lib.bp_mix_seed(7, 3) == orc.mix_seed(7, 3)


def test_generate_model_matches_oracle_and_reference_smoke():
    for seed, widths in ((7, [4, 8, 2]), (21, [3, 12, 12, 1])):
        m = bp.generate_model(seed, widths)
        flat = np.concatenate([np.concatenate([W.ravel(), b]) for W, b in zip(m.W, m.b)])
        assert np.array_equal(flat, orc.generate_model_params(seed, widths))
    # proj/tests/python/test_smoke.py:28-35
    a, b, c = (bp.generate_model(s, [4, 8, 2]) for s in (7, 7, 8))
    assert a.digest == b.digest and a.digest != c.digest
    assert a.parameter_count() == 4 * 8 + 8 + 8 * 2 + 2
    for W in a.W:  # Glorot envelope (test_model.cpp:47-53)
        assert np.abs(W).max() <= math.sqrt(6.0 / (W.shape[0] + W.shape[1]))


def test_forward_shapes():  # test_smoke.py:37-42
    m = bp.generate_model(seed=3, widths=[5, 16, 16, 3])
    y = m.forward(np.random.default_rng(0).uniform(-1, 1, size=(11, 5)))
    assert y.shape == (11, 3) and np.isfinite(y).all()


def product_pick(meta, n, eta, temperature, seed):
    lib = _capi.load()
    arr = (_capi.PoolMeta * len(meta))(*[_capi.PoolMeta(*m) for m in meta])
    h = C.c_void_p()
    _capi.check(lib.bp_rng_new(seed, C.byref(h)))
    picked = np.zeros(len(meta), dtype=np.int32)
    k = C.c_int()
    _capi.check(lib.bp_pick_out(arr, len(meta), n, eta, temperature, h, _capi.iptr(picked), C.byref(k)))
    lib.bp_rng_free(h)
    return [int(x) for x in picked[:k.value]]


def test_pick_out_bit_exact_vs_oracle():
    rng = np.random.default_rng(4)
    for trial in range(40):
        n_pool = int(rng.integers(1, 60))
        lf = rng.normal(size=n_pool) * 3
        uf = lf + rng.exponential(size=n_pool)
        uf[rng.random(n_pool) < 0.2] = uf[0]  # ties in uf
        if trial % 5 == 0:
            lf[0] = -math.inf
        meta = [(float(lf[i]), float(uf[i]), i, -0.7 * i) for i in range(n_pool)]
        for n, eta, T in ((4, 0.75, 0.05), (10, 0.0, 0.5), (n_pool + 3, 0.5, 1e-13)):
            assert product_pick(meta, n, eta, T, 99 + trial) == orc.pick_out(meta, n, eta, T, orc.Rng(99 + trial))


def test_config_defaults_and_round_trip():
    d = json.loads(bp.default_config())
    assert d["batch"] == 4 and d["eta"] == 0.75 and d["bound_mode"] == "early-stop-empirical"
    assert d["search"]["cem"] == {"agents": 4, "elites": 10, "jitter": 1e-3, "init_sigma": 0.5}
    c = config.from_json('{"seed": 5, "search": {"samples_per_iter": 48}, "termination": {"max_iterations": 8}}')
    assert c["seed"] == 5 and c["search"]["samples_per_iter"] == 48 and c["search"]["iterations"] == 10
    assert config.from_json(config.to_json(c)) == c
    for bad in ('{"bound_mode": "nope"}', '{"alpha": "x"}', '{"search": {"method": "sgd"}}', "[1]"):
        with pytest.raises(ValueError):
            config.from_json(bad)


def test_scenario_round_trip(tmp_path):  # test_smoke.py:88-97
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = np.full(2, 0.4), np.zeros(2), np.zeros(2)
    s.horizon = 4
    s.u_lower, s.u_upper = np.full(2, -0.5), np.full(2, 0.5)
    s.obstacles = [bp.Obstacle(center=np.array([0.3, 0.1]), size=0.2)]
    s.cost_form = "tracking_obstacles"
    path = str(tmp_path / "scenario.json")
    s.save(path)
    t = bp.load_scenario(path)
    assert t.digest == s.digest and t.cost_form == "tracking_obstacles" and np.allclose(t.x0, s.x0)
    m = bp.generate_model(9, [4, 6, 2])
    m.save(str(tmp_path / "m.json"))
    r = bp.load_model(str(tmp_path / "m.json"))
    assert r.digest == m.digest and r.widths == m.widths


def test_scenario_validation():  # test_model.cpp:109-122
    def two():
        s = bp.Scenario()
        s.x0, s.x_target, s.p0 = [0.4, -0.3], [0.0, 0.0], [0.0, 0.0]
        s.horizon = 2
        s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
        return s
    s = two()
    s.u_lower = [-0.5]
    with pytest.raises(ValueError):
        s.validate()
    s = two()
    s.horizon = 0
    with pytest.raises(ValueError):
        s.validate()
    s = two()
    s.u_lower, s.u_upper = [0.5, 0.5], [-0.5, -0.5]
    with pytest.raises(ValueError):
        s.validate()


def test_objective_program_matches_oracle_graph_order():
    """The descriptor for the reference forms builds the reference's node order."""
    from paper_2412_09584_b200.objective import build_objective
    s = bp.Scenario()
    s.x0, s.x_target, s.p0 = [0.3, -0.2, 0.1, 0.0], [0.0] * 4, [0.0, 0.0]
    s.horizon = 2
    s.u_lower, s.u_upper = [-0.4, -0.4], [0.4, 0.4]
    s.obstacles = [bp.Obstacle([0.15, 0.0], 0.1)]
    s.cost_form = "tracking_obstacles"
    ob = orc.Objective(build_objective(bp.generate_model(77, [6, 12, 4]), s))
    # nodes: U, x0, p0, then per step: slice, tile linear, sum, concat, linear, relu, linear, sum(p),
    # sqdist, slice, hinge, slice, hinge, hinge(p)
    sn = ob.step_nodes(0)
    assert (sn["u"], sn["preact"], sn["x"], sn["p"]) == (3, [7], 9, 10)
    assert sn["ops"] == [11, 12, 13, 14, 15, 16]
    # kLastRelu: the final step's last ReLU (22) plus every hinge (objective.cpp:45-63)
    assert ob.stop_set() == [13, 15, 16, 22, 27, 29, 30]


def test_pick_out_bit_exact_on_large_pools():
    """Pools of a throughput run's size (the weights are reused between softmax picks
    unless a pick moves the lf range; picks of the extreme records force recomputes)."""
    rng = np.random.default_rng(12)
    for trial, n_pool in enumerate((700, 2500)):
        lf = rng.normal(size=n_pool) * 5
        lf[rng.random(n_pool) < 0.05] = -math.inf
        uf = lf + rng.exponential(size=n_pool)
        meta = [(float(lf[i]), float(uf[i]), i, -0.1 * i) for i in range(n_pool)]
        for n, eta, T in ((256, 0.75, 0.05), (120, 0.0, 5.0), (64, 0.0, 1e-4)):
            assert product_pick(meta, n, eta, T, 7 + trial) == orc.pick_out(meta, n, eta, T, orc.Rng(7 + trial))


def test_pick_out_bit_exact_on_multi_gpu_sized_pools():
    """Pools above the threaded weight recompute (>= 32768 records: each w_i computed on a host
    thread, the running sums kept in the reference's order with removed records at weight 0),
    with tied uf / lf values and +-inf bounds, and picks that drain the low end (lo moves)."""
    rng = np.random.default_rng(21)
    n_pool = 40000
    lf = np.round(rng.normal(size=n_pool) * 8, 1)  # many ties
    lf[rng.random(n_pool) < 0.02] = -math.inf
    lf[rng.random(n_pool) < 0.01] = math.inf
    uf = np.round(lf + rng.exponential(size=n_pool), 1)
    uf[~np.isfinite(uf)] = math.inf
    meta = [(float(lf[i]), float(uf[i]), i, -0.1 * i) for i in range(n_pool)]
    for n, eta, T in ((1024, 0.75, 0.05), (300, 0.0, 1e-3)):
        assert product_pick(meta, n, eta, T, 3) == orc.pick_out(meta, n, eta, T, orc.Rng(3))


def test_workloads_rng_is_the_reference_stream_without_the_cuda_library():
    """workloads.Rng (pure Python mt19937_64 + Box-Muller) draws the reference Rng stream bit for
    bit (rng.hpp:12-35, rng.cpp:20-35; std::mt19937_64 10000th-output KAT), so the bench's
    reference arm builds its fixtures without loading libbabplan_cuda.so."""
    import subprocess
    import sys

    from paper_2412_09584_b200 import workloads

    assert workloads.Rng(5489).bits(10000)[-1] == np.uint64(9981545732273789042)
    for seed in (0, 1, 2, 2**63 + 12345):
        a, b = workloads.Rng(seed), orc.Rng(seed)
        assert np.array_equal(a.bits(700), np.array([b.bits() for _ in range(700)], dtype=np.uint64))
        assert np.array_equal(a.uniform(333, -1, 1), np.array([-1 + 2 * b.uniform() for _ in range(333)]))
        assert np.array_equal(a.normal(501), np.array([b.normal() for _ in range(501)]))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2412_09584_b200 import workloads\n"
            "from oracle import oracle as orc\n"
            "w = workloads.c2(); orc.Objective(w.spec)\n"
            "print('libbabplan_cuda' in open('/proc/self/maps').read())" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "False", r.stderr
