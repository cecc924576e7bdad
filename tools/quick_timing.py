"""Quick device timing of the rollout / search / bound on a BASELINE config (dev helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
D = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = workloads.ALL[name]() if name != "c5" else workloads.c5(D or 1024)
D = D or wl.children
dev = bp.Device(0).load(wl.spec)
if len(sys.argv) > 3: dev.rollout_path(sys.argv[3])
print("rollout path:", dev.rollout_path(), flush=True)
los, his = workloads.presplit_boxes(wl.spec, D)
cfg = wl.planner_config()
for it in range(3):
    t0 = time.time()
    rep = dev.batch_search(los, his, None, cfg, seed=it)
    lf = dev.batch_bound(D)
    t1 = time.time()
    tm = dev.timing()
    rows = wl.rows_per_search_iter
    flops = D * rows * wl.spec.horizon * wl.flops_per_sample_step * cfg["search"]["iterations"]
    print(f"{wl.name} D={D} iter {it}: wall {1e3*(t1-t0):.1f} ms, rollout {tm['rollout_ms']:.1f} ms over "
          f"{tm['rollout_launches']} launches -> {flops/tm['rollout_ms']/1e9:.1f} TFLOP/s, bound {tm['bound_ms']:.2f} ms, "
          f"ok {rep['ok'].mean():.2f}, uf min {rep['uf'].min():.4g}, lf min {lf.min():.4g}", flush=True)
