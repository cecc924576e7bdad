"""Planner configuration JSON (planner_config_to_json / _from_json,
reference src/bench.cpp:170-258): every field explicit when serialised,
partial objects accepted on parse with the defaults of bab.hpp:51-62 and
search.hpp:18-46.  Unknown keys are ignored, unknown enum names raise
ValueError.  A `split_rule` key ("samples" | "width") is added for the
width-only split of the BASELINE.json tiny config.
"""
from __future__ import annotations

import copy
import ctypes as C
import json
import math

import numpy as np

from . import _capi

BOUND_MODES = {"full-crown": _capi.BP_BOUND_FULL_CROWN, "early-stop-empirical": _capi.BP_BOUND_EMPIRICAL,
               "early-stop-interval": _capi.BP_BOUND_INTERVAL}
ALPHAS = {"adaptive": _capi.BP_ALPHA_ADAPTIVE, "zero": _capi.BP_ALPHA_ZERO, "one": _capi.BP_ALPHA_ONE}
METHODS = {"cem": _capi.BP_SEARCH_CEM, "mppi": _capi.BP_SEARCH_MPPI, "gd": _capi.BP_SEARCH_GD}
SPLITS = {"samples": _capi.BP_SPLIT_SAMPLES, "width": _capi.BP_SPLIT_WIDTH}

DEFAULTS = {
    "batch": 4, "eta": 0.75, "temperature": 0.05, "top_percent": 1.0, "min_width": 1e-6,
    "bound_mode": "early-stop-empirical", "alpha": "adaptive", "seed": 0,
    "search": {
        "method": "cem", "samples_per_iter": 1000, "iterations": 10, "top_capacity": 512,
        "cem": {"agents": 4, "elites": 10, "jitter": 1e-3, "init_sigma": 0.5},
        "mppi": {"noise_frac": 0.25, "temperature": 10.0, "noise_ratios": [0.5, 1.0, 2.0],
                 "temperature_ratios": [1.0]},
        "gd": {"base_step": 0.01, "step_ratios": [0.05, 0.1, 0.25, 0.5, 0.75, 1.0, 1.5, 2.0, 5.0, 10.0]},
    },
    "termination": {"max_iterations": 50, "wall_clock_ms": 0.0},
}


def _parse_enum(table, name, what):
    if name not in table:
        raise ValueError(f"unknown {what} '{name}'")
    return name


def from_json(text: str) -> dict:
    """Resolved config dict from a (partial) JSON object."""
    try:
        j = json.loads(text if text else "{}")
    except json.JSONDecodeError as e:
        raise ValueError(f"planner config: {e}") from e
    if not isinstance(j, dict):
        raise ValueError("planner config: expected an object")
    c = copy.deepcopy(DEFAULTS)
    for k in ("batch", "eta", "temperature", "top_percent", "min_width", "seed"):
        if k in j:
            c[k] = j[k]
    if "bound_mode" in j:
        c["bound_mode"] = _parse_enum(BOUND_MODES, j["bound_mode"], "bound mode")
    if "alpha" in j:
        c["alpha"] = _parse_enum(ALPHAS, j["alpha"], "alpha policy")
    if "split_rule" in j:
        c["split_rule"] = _parse_enum(SPLITS, j["split_rule"], "split rule")
    s = j.get("search", {})
    if "method" in s:
        c["search"]["method"] = _parse_enum(METHODS, s["method"], "search method")
    for k in ("samples_per_iter", "iterations", "top_capacity"):
        if k in s:
            c["search"][k] = s[k]
    for sub in ("cem", "mppi", "gd"):
        for k, v in s.get(sub, {}).items():
            if k in c["search"][sub]:
                c["search"][sub][k] = v
    t = j.get("termination", {})
    for k in ("max_iterations", "wall_clock_ms"):
        if k in t:
            c["termination"][k] = t[k]
    if "target_objective" in t:
        c["termination"]["target_objective"] = float(t["target_objective"])
    return c


def to_json(c: dict) -> str:
    out = copy.deepcopy(c)
    tgt = out["termination"].get("target_objective")
    if tgt is not None and not math.isfinite(tgt):
        del out["termination"]["target_objective"]
    return json.dumps(out)


def default_config() -> str:
    return to_json(DEFAULTS)


class PackedConfig:
    """ctypes bp_planner_config for a resolved dict (keeps its arrays alive)."""

    def __init__(self, c: dict, method: str = "babnd"):
        s = c["search"]
        meth = s["method"] if method in ("", "babnd") else _parse_enum(METHODS, method, "search method")
        self._nr = np.asarray(s["mppi"]["noise_ratios"], dtype=np.float64)
        self._tr = np.asarray(s["mppi"]["temperature_ratios"], dtype=np.float64)
        self._gr = np.asarray(s["gd"]["step_ratios"], dtype=np.float64)
        sc = _capi.SearchConfig(
            method=METHODS[meth], samples_per_iter=int(s["samples_per_iter"]), iterations=int(s["iterations"]),
            top_capacity=int(s["top_capacity"]), seed=0, cem_agents=int(s["cem"]["agents"]),
            cem_elites=int(s["cem"]["elites"]), cem_jitter=float(s["cem"]["jitter"]),
            cem_init_sigma=float(s["cem"]["init_sigma"]), mppi_noise_frac=float(s["mppi"]["noise_frac"]),
            mppi_temperature=float(s["mppi"]["temperature"]), mppi_n_noise=len(self._nr),
            mppi_n_temp=len(self._tr), mppi_noise_ratios=_capi.dptr(self._nr) if len(self._nr) else None,
            mppi_temperature_ratios=_capi.dptr(self._tr) if len(self._tr) else None,
            gd_base_step=float(s["gd"]["base_step"]), gd_n_ratios=len(self._gr),
            gd_step_ratios=_capi.dptr(self._gr) if len(self._gr) else None)
        self.cfg = _capi.PlannerConfig(
            batch=int(c["batch"]), eta=float(c["eta"]), temperature=float(c["temperature"]),
            top_percent=float(c["top_percent"]), min_width=float(c["min_width"]),
            bound_mode=BOUND_MODES[c["bound_mode"]], alpha=ALPHAS[c["alpha"]],
            split_rule=SPLITS[c.get("split_rule", "samples")], seed=int(c["seed"]) & (2**64 - 1), search=sc,
            max_iterations=int(c["termination"]["max_iterations"]),
            wall_clock_ms=float(c["termination"]["wall_clock_ms"]),
            target_objective=float(c["termination"].get("target_objective", -math.inf)))

    def ref(self):
        return C.byref(self.cfg)

    def search_ref(self, seed: int):
        self.cfg.search.seed = seed & (2**64 - 1)
        return C.byref(self.cfg.search)
