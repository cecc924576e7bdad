"""Distribution of the root-box search's best value, device vs CPU oracle, over many seeds (dev helper):
a systematic gap would point at a sampler difference (the update is bit-exact on identical samples).

usage: python tools/search_seeds.py c2 32 [M] [iters] [method]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from paper_2412_09584_b200 import workloads

name, n = sys.argv[1], int(sys.argv[2])
M = int(sys.argv[3]) if len(sys.argv) > 3 else 256
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 10
method = sys.argv[5] if len(sys.argv) > 5 else "cem"
wl = workloads.ALL[name]()
lo, hi = wl.spec.box()
dev = bp.Device(0)
dev.load(wl.spec)
ob = orc.Objective(wl.spec)
cfg = wl.planner_config()
cfg["search"]["samples_per_iter"] = M
cfg["search"]["iterations"] = iters
cfg["search"]["method"] = method
g, c = [], []
t0 = time.time()
for seed in range(100, 100 + n):
    g.append(dev.batch_search(lo[None], hi[None], None, cfg, seed=seed)["uf"][0])
gt = time.time() - t0
t0 = time.time()
for seed in range(100, 100 + n):
    c.append(ob.batch_search(lo[None], hi[None], None, cfg, seed=seed).get(0)["uf"])
print("gpu s", gt, "cpu s", time.time() - t0)
g, c = np.array(g), np.array(c)
print("gpu", np.sort(g))
print("cpu", np.sort(c))
print(f"median gpu {np.median(g):.6g} cpu {np.median(c):.6g}; mean gpu {g.mean():.6g} cpu {c.mean():.6g}")
