"""Per-step wall vs device-search time of the steady-state BaB iteration (dev helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import workloads

wl = workloads.ALL[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
dev = bp.Device(0).load(wl.spec)
cfg = wl.planner_config()
cfg["termination"]["max_iterations"] = 10**6
pl = dev.planner(cfg)
for i in range(14):
    dev.timing()
    t0 = time.perf_counter()
    ok, ch, pool = pl.step()
    wall = 1e3 * (time.perf_counter() - t0)
    tm = dev.timing()
    print(f"step {i}: children {ch} pool {pool} wall {wall:.1f} ms  search+bound {tm['search_ms']:.1f} ms  "
          f"rollout {tm['rollout_ms']:.1f} ms  bound {tm['bound_ms']:.2f} ms", flush=True)
