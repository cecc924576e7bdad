"""Max relative error of the tcgen05 and SIMT rollouts against the oracle (dev helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from test_gpu_parity import small_spec, rel_err

dev = bp.Device(0)
for name in ["c1", "c2", "ref-obstacles", "c4", "c5"]:
    spec = small_spec(name)
    dev.load(spec)
    lo, hi = spec.box()
    acts = np.random.default_rng(3).uniform(lo, hi, size=(2, 300, spec.d)).astype(np.float32)
    out = {}
    for path in ("auto", "simt"):
        p = dev.rollout_path(path)
        c, _, l, h, _ = dev.rollout(acts)
        out[p] = (c, l, h)
    dev.rollout_path("auto")
    ob = orc.Objective(spec)
    ref = np.stack([ob.evaluate(acts[s].astype(np.float64)) for s in range(2)])
    msg = [f"{name:14s}"]
    for p, (c, l, h) in out.items():
        ok = np.isfinite(ref)
        msg.append(f"{p}: cost {rel_err(c[ok], ref[ok]):.2e}")
    if "tcgen05" in out:
        msg.append(f"bounds tc-vs-simt {max(rel_err(out['tcgen05'][1], out['simt'][1]), rel_err(out['tcgen05'][2], out['simt'][2])):.2e}")
    print("  ".join(msg), flush=True)
