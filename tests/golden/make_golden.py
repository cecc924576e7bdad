"""Regenerates tests/golden/*.json from the FP64 oracle (test infrastructure).

The reference itself does not build in this container (Eigen3 and proj/vendor
are absent), so the fixtures are oracle outputs on FP32-representable inputs;
the oracle is pinned to the reference's KATs by tests/test_oracle_kats.py.
Run: python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2412_09584_b200 import workloads  # noqa: E402


def main():
    out = {}
    for name, mk in (("c1", workloads.c1), ("c2", workloads.c2), ("c4", workloads.c4)):
        wl = mk(glorot=True)
        spec = wl.spec
        lo, hi = spec.box()
        acts = np.random.default_rng(7).uniform(lo, hi, size=(6, spec.d)).astype(np.float32).astype(np.float64)
        ob = orc.Objective(spec)
        st = orc.Stats()
        costs = ob.evaluate(acts, st)
        lf_emp = ob.lower_bound(lo, hi, "early-stop-empirical", st)
        lf_ivl = ob.lower_bound(lo, hi, "early-stop-interval")
        x1 = ob.step_nodes(0)["x"]
        mn, mx, _ = st.get(x1, spec.ks) if st.get(x1, spec.ks) else (np.zeros(0), np.zeros(0), 0)
        out[name] = {"actions": acts.tolist(), "costs": costs.tolist(), "lf_empirical": lf_emp,
                     "lf_interval": lf_ivl, "x1_min": list(mn), "x1_max": list(mx)}
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "oracle_golden.json"))


if __name__ == "__main__":
    main()
