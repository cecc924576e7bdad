"""Localise a rollout mismatch: per recorded node kind and step, the max error of the
device extrema / states against the oracle (dev helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2412_09584_b200 as bp
from oracle import oracle as orc
from test_gpu_parity import v3_spec, small_spec

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
path = sys.argv[2] if len(sys.argv) > 2 else "auto"
spec = v3_spec(name) if name in ("c5", "ragged", "rel16") else small_spec(name)
dev = bp.Device(0).load(spec)
print("kernel", dev.rollout_path(path), dev.rollout_kernel())
lo, hi = spec.box()
acts = np.random.default_rng(13).uniform(lo, hi, size=(1, 9, spec.d)).astype(np.float32)
costs, states, elo, ehi, bad = dev.rollout(acts, want_states=True)
ob = orc.Objective(spec)
st = orc.Stats()
ref = ob.evaluate(acts[0].astype(np.float64), st)
print("costs", costs[0][:4], ref[:4])
per, slots = dev.stat_layout()
rlo, rhi = ob.stats_in_layout(st, (per, slots), spec.horizon)
for t in range(min(3, spec.horizon)):
    for kind, index, dim, off in slots:
        g, w = elo[0][t, off:off + dim], rlo[t, off:off + dim]
        if np.isnan(w).all():
            continue
        e = np.nanmax(np.abs(g - w) / np.maximum(np.abs(w), 1))
        print(f"t={t} kind={kind} index={index} dim={dim}: max err {e:.3e}  dev {g[:3]} ref {w[:3]}")
        if t == 0:
            blk = [float(np.nanmax(np.abs(g[b:b + 32] - w[b:b + 32]))) for b in range(0, dim, 32)]
            print("   per 32-block:", " ".join(f"{x:.1e}" for x in blk))
