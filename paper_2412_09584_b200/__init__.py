"""B200-native BaB-ND planner hot path (arXiv 2412.09584).

Drop-in for the reference's `babplan` Python module: the same 15 names
(bindings/__init__.py:3-19), backed by hand-written sm_100a kernels behind
the C-ABI in include/babplan_cuda.h.
"""
from .api import (Device, default_config, lower_bound, network_lower_bound, objective_value, plan,
                  plan_synthetic, prm_plan, rollout, rrt_plan)
from .model import Model, Obstacle, Scenario, generate_model, load_model, load_scenario
from .mpc_driver import mpc

__all__ = [
    "Model", "Obstacle", "Scenario", "default_config", "generate_model", "load_model", "load_scenario",
    "lower_bound", "network_lower_bound", "objective_value", "plan", "plan_synthetic", "prm_plan", "rollout",
    "rrt_plan", "Device", "mpc",
]
