"""Wall time per planner step from the root on a fresh Device (diagnostic)."""
import sys
import time

import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import workloads

wl = getattr(workloads, sys.argv[1] if len(sys.argv) > 1 else "c2")()
for rep in range(2):
    dev = bp.Device(0)
    t0 = time.perf_counter()
    dev.load(wl.spec)
    t1 = time.perf_counter()
    cfg = wl.planner_config()
    cfg["termination"]["max_iterations"] = 16
    p = dev.planner(cfg)
    t2 = time.perf_counter()
    rows = []
    while True:
        ts = time.perf_counter()
        ok, ch, pool = p.step()
        if not ok:
            break
        rows.append((ch, pool, (time.perf_counter() - ts) * 1e3))
    print(f"rep {rep}: load {1e3*(t1-t0):.1f} ms, root {1e3*(t2-t1):.1f} ms, steps:",
          " ".join(f"{c}/{q}:{ms:.1f}" for c, q, ms in rows), flush=True)
    dev.close()
