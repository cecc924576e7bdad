"""Planner trace statistics, device vs CPU oracle, over seeds (dev helper): final objective, min lf,
pruned volume, pool size and certification at equal iterations.

usage: python tools/trace_seeds.py c1 8 [iters] [batch]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import workloads

name, n = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else None
batch = int(sys.argv[4]) if len(sys.argv) > 4 else None
wl = workloads.ALL[name]()
dev = bp.Device(0)
dev.load(wl.spec)
ob = orc.Objective(wl.spec)
rows = {"gpu": [], "cpu": []}
for seed in range(2, 2 + n):
    cfg = wl.planner_config(**({"batch": batch} if batch else {}))
    cfg["seed"] = seed
    if iters:
        cfg["termination"]["max_iterations"] = iters
    for side, r in (("gpu", dev.plan(cfg)), ("cpu", ob.plan(cfg))):
        tr = r["trace"]
        rows[side].append((r["objective"], r["lower_bound"], tr["pruned_vol"][-1], tr["pool_size"][-1],
                           float(r["certified"]), r["samples"]))
    print(seed, "gpu", rows["gpu"][-1], "cpu", rows["cpu"][-1], flush=True)
for k, nm in enumerate(["objective", "min_lf", "pruned_vol", "pool_size", "certified", "samples"]):
    g = np.array([r[k] for r in rows["gpu"]]); c = np.array([r[k] for r in rows["cpu"]])
    print(f"{nm:12s} gpu median {np.median(g):.6g} mean {g.mean():.6g} | cpu median {np.median(c):.6g} mean {c.mean():.6g}")
