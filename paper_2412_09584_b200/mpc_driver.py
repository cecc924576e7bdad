"""Receding-horizon MPC over the device planner.

Restates the reference's closed-loop driver `run_mpc` (proj/tools/babplan_cli.cpp:
333-420): at every replan the suffix scenario (state and effector from the plant,
horizon H - executed, the original per-step tracking weights) is planned with
plan() (or the sampler for another method) warm-started from the previous plan's
unexecuted tail, the first `replan` actions are applied to the plant -- the same
MLP, in FP64 on the host (MlpModel::forward, model.cpp:60-69, the reference's
simulator) -- and the realised step cost (tracking + collision_penalty,
baselines.cpp:12-26) accumulates.  The planning itself (search, bound, BaB) runs
on the device through the C-ABI; per-replan wall time is the replan latency.
"""
from __future__ import annotations

import copy
import math
import time
from typing import Optional

import numpy as np

from . import config as _config
from .api import Device, default_device
from .model import Model, Scenario
from .objective import build_objective

_M64 = (1 << 64) - 1


def mix_seed(master: int, salt: int) -> int:
    """splitmix64 finalizer over master + golden * (salt + 1) (rng.cpp:37-42)."""
    z = (master + 0x9E3779B97F4A7C15 * (salt + 1)) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def make_features(s: Scenario, x: np.ndarray, p: np.ndarray, u: np.ndarray) -> np.ndarray:
    """make_features (model.cpp:294-308): concat(x [- tile(p)], u)."""
    f = x.astype(np.float64).copy()
    if s.feature_mode == "relative":
        kd = p.size
        for k in range(x.size // kd):
            f[k * kd:(k + 1) * kd] -= p
    return np.concatenate([f, u])


def collision_penalty(s: Scenario, x: np.ndarray, p: np.ndarray) -> float:
    """baselines.cpp:12-26: lambda * max(0, size - |pos - center|) per keypoint
    (tracking_obstacles) and for the effector, summed over obstacles."""
    if s.cost_form == "tracking" or not s.obstacles:
        return 0.0
    kd = s.workspace_dim()
    hinge = lambda pos, o: s.lam * max(0.0, o.size - float(np.linalg.norm(pos - o.center)))
    total = 0.0
    for o in s.obstacles:
        if s.cost_form == "tracking_obstacles":
            for k in range(s.keypoints()):
                total += hinge(x[k * kd:(k + 1) * kd], o)
        total += hinge(p, o)
    return total


def mpc(model: Model, scenario: Scenario, config: str = "", method: str = "babnd", replan: int = 1,
        device: Optional[Device] = None) -> dict:
    """Closed-loop planning (run_mpc).  Returns the reference's mpc summary
    (open_loop_objective, realized_objective, final_step_cost, final_state_distance,
    steps, replans, samples) plus the per-step trace {step, cost, cumulative, plan_uf,
    samples, wall_ms} and the per-replan latency in ms."""
    if replan < 1:
        raise ValueError("replan period must be at least 1")
    s = scenario
    s.validate()
    base = _config.from_json(config)
    dev = device or default_device()
    H, ka = s.horizon, s.action_dim()
    axis = s.axis_weights if s.axis_weights.size else np.ones(s.state_dim())
    x, p = s.x0.astype(np.float64).copy(), s.p0.astype(np.float64).copy()
    open_loop = math.inf
    cumulative = final_step_cost = 0.0
    samples = replans = 0
    prev_best: Optional[np.ndarray] = None
    trace = {k: [] for k in ("step", "cost", "cumulative", "plan_uf", "samples", "wall_ms")}
    latency = []
    t0 = time.perf_counter()
    execd = 0
    while execd < H:
        suffix = copy.deepcopy(s)
        suffix.x0, suffix.p0 = x.copy(), p.copy()
        suffix.horizon = H - execd
        suffix.weights = [s.tracking_weight(execd + t) for t in range(1, H - execd + 1)]
        spec = build_objective(model, suffix)
        pc = copy.deepcopy(base)
        pc["seed"] = mix_seed(int(base["seed"]), replans)
        warm = prev_best if prev_best is not None and prev_best.size == spec.d else None
        r0 = time.perf_counter()
        res = dev.load(spec).plan(pc, warm, method)
        latency.append(1e3 * (time.perf_counter() - r0))
        samples += res["samples"]
        replans += 1
        if replans == 1:
            open_loop = res["objective"]
        best = np.asarray(res["action"], dtype=np.float64)
        steps = min(replan, H - execd)
        for r in range(steps):
            u = best[r * ka:(r + 1) * ka]
            x = model.forward(make_features(s, x, p, u)[None])[0]
            p = p + u
            execd += 1
            track = float(np.sum(axis * (x - s.x_target) ** 2))
            cost = s.tracking_weight(execd) * track + collision_penalty(s, x, p)
            cumulative += cost
            final_step_cost = cost
            for k, v in (("step", execd), ("cost", cost), ("cumulative", cumulative), ("plan_uf", res["objective"]),
                         ("samples", samples), ("wall_ms", 1e3 * (time.perf_counter() - t0))):
                trace[k].append(v)
        prev_best = best[steps * ka:] if best.size >= (steps + 1) * ka else None
    return {"open_loop_objective": open_loop, "realized_objective": cumulative, "final_step_cost": final_step_cost,
            "final_state_distance": float(np.linalg.norm(x - s.x_target)), "steps": H, "replans": replans,
            "samples": samples, "trace": trace, "replan_ms": latency}
