"""The C-ABI consumed from compiled C++ (tests/native/capi_consumer.cpp): it builds and links
against the in-tree library here; on a B200 it plans the reference smoke-test scenario through
bp_plan and checks objective_value(action) == objective and the exception mapping."""
import json
import os
import subprocess

import pytest

from paper_2412_09584_b200 import _build


def test_consumer_builds_and_links():
    exe = _build.build_consumer()
    assert os.access(exe, os.X_OK)
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libbabplan_cuda.so" in out and "not found" not in out.split("libbabplan_cuda.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_consumer_plans_the_reference_smoke_scenario():
    exe = _build.build_consumer()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["same"] and res["incumbent_monotone"] and res["lower_bound"] <= res["objective"] + 1e-9
    assert res["stop_reason"] in {"max-iterations", "pool-exhausted", "target", "wall-clock"}
    assert "null argument" in res["invalid_argument"]
