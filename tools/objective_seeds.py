"""Best objective of the device planner vs the CPU oracle planner over many seeds (dev helper).

usage: python tools/objective_seeds.py c2 12 [iters] [batch]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import workloads

name = sys.argv[1]
n = int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 4
wl = workloads.ALL[name]()
dev = bp.Device(0)
dev.load(wl.spec)
ob = orc.Objective(wl.spec)
rows = []
for seed in range(2, 2 + n):
    cfg = wl.planner_config(batch=batch)
    cfg["seed"] = seed
    cfg["termination"]["max_iterations"] = iters
    dev.rollout_path("auto")
    g = dev.plan(cfg)["objective"]
    dev.rollout_path("simt")
    gs = dev.plan(cfg)["objective"]
    t0 = time.time()
    c = ob.plan(cfg)["objective"]
    rows.append((seed, g, gs, c))
    print(f"seed {seed}: gpu tc {g:.6g}  gpu simt {gs:.6g}  cpu {c:.6g}  ({time.time()-t0:.1f} s)", flush=True)
a = np.array(rows)
for k, nm in ((1, "tc"), (2, "simt")):
    gap = (a[:, k] - a[:, 3]) / np.abs(a[:, 3])
    print(f"{nm}: gpu<=cpu {int((a[:, k] <= a[:, 3]).sum())}/{n}, median gap {np.median(gap):+.4f}, mean gap {gap.mean():+.4f}")
