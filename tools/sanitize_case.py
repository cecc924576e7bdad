"""Small invocations of every hand-written kernel family for compute-sanitizer (dev helper):
the three tcgen05 rollouts (v1 rollout_tc.cu, v2 rollout_tc2.cu incl. the CTA pair, v3
rollout_tc3.cu incl. the CTA pair), the SIMT rollout, search (sample / update), bound (empirical,
interval, full CROWN), the pool kernels (split / merge) and a short plan.
  compute-sanitizer --tool memcheck python tools/sanitize_case.py
(one tool per gpurun call; see profiles/r02_sanitizer.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2412_09584_b200 as bp  # noqa: E402
from paper_2412_09584_b200.config import from_json  # noqa: E402
from test_gpu_parity import small_spec, v3_spec  # noqa: E402

dev = bp.Device(0)
rng = np.random.default_rng(0)
cases = [("c1", "tc1"), ("c2", "tc1"), ("c2", "tc2"), ("c3", "tc2"), ("c4", "tc2"), ("c1", "simt")]
for name, path in cases:
    spec = small_spec(name)
    dev.load(spec)
    dev.rollout_path(path)
    lo, hi = spec.box()
    acts = rng.uniform(lo, hi, size=(2, 130, spec.d)).astype(np.float32)
    dev.rollout(acts, want_states=True)
    print(name, path, dev.rollout_kernel(), flush=True)
dev.rollout_path("auto")
os.environ["BP_TC2_PAIR"] = "1"
dev.load(small_spec("c3"))
dev.rollout(rng.uniform(-1, 1, size=(1, 300, small_spec("c3").d)).astype(np.float32))
os.environ.pop("BP_TC2_PAIR")
print("c3 tc2 pair", flush=True)
for pair in ("0", "1"):
    os.environ["BP_TC3_PAIR"] = pair
    spec = v3_spec("ragged")
    dev.load(spec)
    lo, hi = spec.box()
    dev.rollout(rng.uniform(lo, hi, size=(2, 200, spec.d)).astype(np.float32), want_states=True)
    print("v3 ragged pair", pair, dev.rollout_kernel(), flush=True)
os.environ.pop("BP_TC3_PAIR")
dev.rollout_path("auto")
spec = small_spec("c1")
dev.load(spec)
lo, hi = spec.box()
cfg = from_json('{"search": {"samples_per_iter": 64, "iterations": 2, "top_capacity": 16}}')
rep = dev.batch_search(np.stack([lo, lo]), np.stack([hi, hi]), None, cfg, seed=1)
for mode in ("early-stop-empirical", "early-stop-interval"):
    dev.batch_bound(2, mode)
dev.bound_boxes(lo[None], hi[None], "full-crown")
cfg = from_json('{"batch": 4, "search": {"samples_per_iter": 64, "iterations": 2, "top_capacity": 16},'
                ' "termination": {"max_iterations": 3}}')
res = dev.plan(cfg)
print("search / bound / plan ok", res["objective"], flush=True)
