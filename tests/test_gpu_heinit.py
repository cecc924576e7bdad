"""Rollout error on the weights the bench times (He-init, BASELINE.json wording).

The parity suite pins the kernels on the reference's Glorot generator; here the
bench's own He-normal fixtures (workloads.c1() ... c5(), zero bias) are rolled
out on every kernel path and compared with the FP64 oracle on identical
FP32-representable inputs.  He-init rollouts are expansive (|x_H|
up to 1e7 on C5, 1e16 on C4), so FP32 rounding in the state is amplified by the
dynamics Jacobian whatever the kernel does; the bars below are per config and
path, set from measurements (DESIGN.md 5 lists max and p99), and the SIMT FP32
kernel is the reference point for what FP32 arithmetic itself costs.

Costs: |dev - ref| / max(|ref|, 1) per row (a sum of non-negative terms, no
cancellation).  Sample extrema: normwise per recorded node and step, |dev - ref|
/ max(max |ref| over the node's coordinates at that step, 1) -- a pre-activation
is a dot product whose terms can cancel to far below their own magnitude, so
elementwise relative error there measures the cancellation, not the kernel
(SURVEY 7.3).  Actions: uniform in the box plus box corners (the searches
sample clamped Gaussians, so corners are common).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2412_09584_b200 import workloads

pytestmark = pytest.mark.gpu

# (config, rows per subdomain): the FP64 oracle bounds the sample size at width 256 / 512
ROWS = {"c1": 96, "c2": 64, "c3": 24, "c4": 48, "c5": 16}
# stated bars (max relative error over the sample), per config and kernel family: about twice
# the measured maximum (DESIGN.md 5 lists max and p99 per config and path).  The tensor-core
# paths sit 10-80x above FP32 here: the tensor pipe accumulates each 8-deep k-step into the FP32
# accumulator with truncation, a bias of ~2^-24 |D| per MMA that a contractive (Glorot) network
# forgets (<= 1e-5 there) and an expansive He-init rollout amplifies step over step.
BAR = {
    ("c1", "simt"): 2e-5, ("c1", "tcgen05"): 5e-5,
    ("c2", "simt"): 2e-5, ("c2", "tcgen05"): 2.5e-4,
    ("c3", "simt"): 2e-5, ("c3", "tcgen05"): 7e-4,
    ("c4", "simt"): 2e-5, ("c4", "tcgen05"): 4e-4,
    ("c5", "simt"): 2e-5, ("c5", "tcgen05"): 1.2e-3,
}
_RESULTS = {}


def _errs(got, ref):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_he_init_rollout_error_is_within_stated_bar(device, name):
    wl = workloads.ALL[name]()
    spec = wl.spec
    dev = device.load(spec)
    lo, hi = spec.box()
    rng = np.random.default_rng(5)
    n_sub, rows = 2, ROWS[name]
    acts = rng.uniform(lo, hi, size=(n_sub, rows, spec.d))
    corners = rng.integers(0, 2, size=(n_sub, rows // 4, spec.d))
    acts[:, : rows // 4] = np.where(corners == 1, hi, lo)
    acts = acts.astype(np.float32)
    ob = orc.Objective(spec)
    layout = dev.stat_layout()
    refs = []
    for s in range(n_sub):
        st = orc.Stats()
        refs.append((ob.evaluate(acts[s].astype(np.float64), st), ob.stats_in_layout(st, layout, spec.horizon)))
    paths = ["auto", "simt"]
    out = {}
    for path in paths:
        fam = dev.rollout_path(path)
        kern = dev.rollout_kernel()
        costs, _, elo, ehi, bad = dev.rollout(acts)
        ce, ee = [], []
        for s in range(n_sub):
            ref, (rlo, rhi) = refs[s]
            finite = np.abs(ref) < 3e38  # rows beyond FP32 range are flagged, not compared
            if not finite.all():
                assert bad[s], "a row beyond FP32 range must mark its subdomain failed"
                continue
            ce.append(_errs(costs[s], ref))
            per, slots = layout
            for _, _, dim, off in slots:
                for got, want in ((elo[s], rlo), (ehi[s], rhi)):
                    g, w = got[:, off:off + dim].astype(float), want[:, off:off + dim]
                    seen = ~np.isnan(w).any(axis=1)
                    if not seen.any():
                        continue
                    scale = np.maximum(np.abs(w[seen]).max(axis=1, keepdims=True), 1.0)
                    ee.append((np.abs(g[seen] - w[seen]) / scale).ravel())
        ce = np.concatenate(ce) if ce else np.zeros(1)
        ee = np.concatenate(ee) if ee else np.zeros(1)
        out[kern] = {"family": fam, "cost_max": float(ce.max()), "cost_p99": float(np.percentile(ce, 99)),
                     "extrema_max": float(ee.max()), "extrema_p99": float(np.percentile(ee, 99)),
                     "rows": int(n_sub * rows)}
    dev.rollout_path("auto")
    _RESULTS[name] = out
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(d):
        json.dump(_RESULTS, open(os.path.join(d, "he_init_errors.json"), "w"), indent=1)
    for kern, r in out.items():
        bar = BAR[(name, r["family"])]
        assert r["cost_max"] < bar and r["extrema_max"] < bar, (name, kern, r)
