"""The reference's soundness audit and its negative control (babplan_cli.cpp run_audit, :431-527), on
the device: for random networks and scenarios, the sound bound modes (full CROWN, early-stop interval)
over the root box never exceed the best of uniform samples over that box, and bounds computed on a
corrupted (shrunk, off-centre) box do -- the audit must notice the corruption.  Empirical mode: the
device bound from a search's own extrema never exceeds the search's best sample (lf <= uf)."""
import numpy as np
import pytest

import paper_2412_09584_b200 as bp
from paper_2412_09584_b200 import objective as objmod
from paper_2412_09584_b200.config import from_json

pytestmark = pytest.mark.gpu
TOL = 1e-6


def _scenario(rng, ks, horizon):
    s = bp.Scenario()
    s.x0 = list(rng.uniform(-1, 1, ks))
    s.x_target = list(rng.uniform(-1, 1, ks))
    s.p0 = [0.0, 0.0]
    s.horizon = horizon
    s.u_lower, s.u_upper = [-0.5, -0.5], [0.5, 0.5]
    return s


def _corrupt(lo, hi, rng):  # babplan_cli.cpp:431-439
    a, b = rng.uniform(0.2, 0.45, lo.shape), rng.uniform(0.2, 0.45, lo.shape)
    w = hi - lo
    return lo + a * w, hi - b * w


@pytest.mark.parametrize("widths", [[6, 16, 16, 4], [6, 32, 4]])
def test_sound_modes_hold_and_the_corruption_control_fires(device, widths):
    rng = np.random.default_rng(17)
    cases = violations = corrupt_cases = corrupt_violations = 0
    for trial in range(12):
        model = bp.generate_model(100 + trial, widths)
        spec = objmod.round_spec_to_f32(objmod.build_objective(model, _scenario(rng, widths[-1], 3)))
        dev = device.load(spec)
        lo, hi = spec.box()
        acts = rng.uniform(lo, hi, size=(1, 2048, spec.d)).astype(np.float32)
        costs, _, _, _, bad = dev.rollout(acts, want_stats=False)
        assert not bad.any()
        vmin = float(costs.min())
        mode = "full-crown" if trial % 2 == 0 else "early-stop-interval"
        lf = dev.bound_boxes(lo[None], hi[None], mode)[0]
        cases += 1
        violations += lf > vmin + TOL * max(1.0, abs(vmin))
        clo, chi = _corrupt(lo, hi, rng)
        lfc = dev.bound_boxes(clo[None], chi[None], mode)[0]
        corrupt_cases += 1
        corrupt_violations += lfc > vmin + TOL * max(1.0, abs(vmin))
    assert violations == 0, (violations, cases)
    assert corrupt_violations > 0, (corrupt_violations, corrupt_cases)  # the negative control fires


def test_empirical_bound_never_exceeds_the_search_best(device):
    rng = np.random.default_rng(3)
    for trial in range(6):
        model = bp.generate_model(200 + trial, [6, 32, 32, 4])
        spec = objmod.round_spec_to_f32(objmod.build_objective(model, _scenario(rng, 4, 4)))
        dev = device.load(spec)
        lo, hi = spec.box()
        c = 0.5 * (lo + hi)
        los = np.stack([lo, np.minimum(c, hi)])
        his = np.stack([hi, hi])
        rep = dev.batch_search(los, his, None, from_json('{"search": {"samples_per_iter": 256, "iterations": 4}}'),
                               seed=trial)
        lf = dev.batch_bound(2, "early-stop-empirical")
        for i in range(2):
            assert rep["ok"][i]
            assert lf[i] <= rep["uf"][i] + 1e-6 * max(1.0, abs(rep["uf"][i])), (trial, i, lf[i], rep["uf"][i])
