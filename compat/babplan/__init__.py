"""`babplan` alias of paper_2412_09584_b200 (the reference module name, bindings/__init__.py).

Putting `compat/` on PYTHONPATH lets code written against the reference's Python module -- its
own tests included (proj/tests/python/test_smoke.py, run unmodified: tools/run_reference_smoke.sh)
-- import this implementation as `babplan`.
"""
import os as _os
import sys as _sys

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
if _ROOT not in _sys.path:
    _sys.path.insert(0, _ROOT)

from paper_2412_09584_b200 import (  # noqa: E402,F401
    Model, Obstacle, Scenario, default_config, generate_model, load_model, load_scenario, lower_bound,
    network_lower_bound, objective_value, plan, plan_synthetic, prm_plan, rollout, rrt_plan)

__all__ = [
    "Model", "Obstacle", "Scenario", "default_config", "generate_model", "load_model", "load_scenario",
    "lower_bound", "network_lower_bound", "objective_value", "plan", "plan_synthetic", "prm_plan", "rollout",
    "rrt_plan",
]
