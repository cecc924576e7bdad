"""Dev helper: one steady-state rollout launch of a workload (for ncu captures).
python tools/rollout_once.py c2 [n_sub] [kernel]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = workloads.ALL[name]()
n_sub = int(sys.argv[2]) if len(sys.argv) > 2 else 512
dev = bp.Device(0).load(wl.spec)
if len(sys.argv) > 3:
    dev.rollout_path(sys.argv[3])
print(dev.rollout_info())
lo, hi = wl.spec.box()
acts = np.random.default_rng(0).uniform(lo, hi, size=(n_sub, wl.rows_per_search_iter, wl.spec.d)).astype(np.float32)
for _ in range(2):
    dev.rollout(acts, want_stats=True)
