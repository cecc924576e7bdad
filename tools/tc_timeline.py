import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BP_TC_TIMELINE"] = "1"
# the marks are compiled in only in the timeline variant:
#   python -c "from paper_2412_09584_b200 import _build; _build.build_variant('timeline', ['-DBP_TC_TIMELINE'])"
_v = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2412_09584_b200", "_lib", "variant_timeline.so")
if os.path.exists(_v):
    os.environ.setdefault("BP_LIB_PATH", _v)
import numpy as np
import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import workloads
wl = workloads.ALL[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
dev = bp.Device(0).load(wl.spec)
if len(sys.argv) > 2:
    dev.rollout_path(sys.argv[2])
lo, hi = wl.spec.box()
acts = np.random.default_rng(0).uniform(lo, hi, size=(512 if wl.spec.d < 100 else 128, 1025, wl.spec.d)).astype(np.float32)
for _ in range(2):
    dev.rollout(acts, want_stats=True)
