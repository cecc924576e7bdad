"""The device-direct NCCL exchange (bp_set_nccl, parallel.NcclLink) on one GPU: the library
dlopens NCCL, builds its own communicator and moves all-gathers and all-to-all-v segments
device to device (bp_nccl_selftest checks every byte); a planner with the link attached plans
as without it.  More ranks need more GPUs (NCCL refuses two ranks on one device): the
planner's exchange sequence itself is covered by the gloo multi-rank tests, which drive the
same host code with the staged hooks."""
import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import parallel, workloads

pytestmark = pytest.mark.gpu


def test_nccl_link_selftest_moves_every_byte():
    dev = bp.Device(0)
    dev.load(workloads.c1(glorot=True).spec)
    link = parallel.nccl_single(dev)
    for n in (1, 7, 4096, 1 << 20):
        assert link.selftest(n), n


def test_planner_with_nccl_link_plans_as_without():
    wl = workloads.c1(glorot=True)
    cfg = wl.planner_config()
    cfg["termination"]["max_iterations"] = 4
    cfg["batch"] = 8
    out = []
    for use_link in (False, True):
        dev = bp.Device(0)
        dev.load(wl.spec)
        if use_link:
            parallel.nccl_single(dev)
        r = dev.plan(cfg)
        out.append(r)
    a, b = out
    assert a["objective"] == b["objective"]
    assert np.array_equal(np.asarray(a["action"]), np.asarray(b["action"]))
