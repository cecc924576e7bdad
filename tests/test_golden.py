"""Golden fixtures (tests/golden/oracle_golden.json, made by make_golden.py):
the oracle must keep reproducing them bit-for-bit (CPU), and the device must
match them within the FP32 bar without building the oracle (GPU)."""
import json
import os

import numpy as np
import pytest

from paper_2412_09584_b200 import workloads

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_golden.json")))
MK = {"c1": workloads.c1, "c2": workloads.c2, "c4": workloads.c4}


@pytest.mark.parametrize("name", sorted(G))
def test_oracle_reproduces_golden(name):
    from oracle import oracle as orc
    spec = MK[name](glorot=True).spec
    g = G[name]
    ob = orc.Objective(spec)
    st = orc.Stats()
    assert ob.evaluate(np.array(g["actions"]), st).tolist() == g["costs"]
    lo, hi = spec.box()
    assert ob.lower_bound(lo, hi, "early-stop-empirical", st) == g["lf_empirical"]
    assert ob.lower_bound(lo, hi, "early-stop-interval") == g["lf_interval"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(G))
def test_device_matches_golden(device, name):
    spec = MK[name](glorot=True).spec
    g = G[name]
    dev = device.load(spec)
    costs, _, _, _, bad = dev.rollout(np.array(g["actions"], dtype=np.float32)[None])
    ref = np.array(g["costs"])
    assert not bad.any()
    tol = 1e-5  # the FP32 bar, on the SIMT and the 3xTF32 tensor-core paths alike
    assert np.max(np.abs(costs[0] - ref) / np.maximum(np.abs(ref), 1.0)) < tol
    lo, hi = spec.box()
    lf = dev.bound_boxes(lo[None], hi[None], "early-stop-interval")[0]
    assert abs(lf - g["lf_interval"]) <= 1e-9 * max(1.0, abs(g["lf_interval"]))
