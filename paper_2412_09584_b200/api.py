"""The reference's Python API (bindings/pymodule.cpp:85-252, bindings/__init__.py)
on top of the C-ABI in include/babplan_cuda.h.

`Device` is the per-process handle (one CUDA device per process, like the
one-rank-per-GPU runtime); the module-level functions use a lazily created
default `Device` on LOCAL_RANK.  Every compute call goes through the CUDA
library; there is no host fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional

import numpy as np

from . import _capi, config as _config
from ._capi import check
from .model import Model, Scenario
from .objective import ObjectiveSpec, build_network_objective, build_objective

_BOUND = _config.BOUND_MODES
_ALPHA = _config.ALPHAS


class SyntheticSpec:
    """The separable synthetic objective on [-1, 1]^d (objective.hpp:73-95) as the
    Device sees it: a one-step "rollout" of d actions, no MLP, no recorded statistics."""

    def __init__(self, dim: int):
        if dim <= 0:
            raise ValueError("SyntheticObjective: dimension must be positive")
        self.d = self.ka = int(dim)
        self.horizon, self.ks = 1, 0

    def box(self):
        return np.full(self.d, -1.0), np.full(self.d, 1.0)


class Device:
    """One bp_ctx bound to a CUDA device, plus the objective loaded on it."""

    def __init__(self, device: Optional[int] = None):
        self.lib = _capi.load()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        h = C.c_void_p()
        check(self.lib.bp_init(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self.spec: Optional[ObjectiveSpec] = None
        self._packed = None
        self._layout = None

    def close(self):
        if self.h:
            self.lib.bp_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- objective
    def load(self, spec: ObjectiveSpec) -> "Device":
        if spec is self.spec:
            return self
        packed = spec.to_c()
        check(self.lib.bp_load_objective(self.h, packed.ref()))
        self.spec, self._packed, self._layout = spec, packed, None
        return self

    def load_synthetic(self, dim: int) -> "Device":
        """The separable benchmark objective (model.cpp:407-409) with its exact bounder."""
        spec = SyntheticSpec(dim)
        check(self.lib.bp_load_synthetic(self.h, spec.d))
        self.spec, self._packed, self._layout = spec, None, None
        return self

    def stat_layout(self):
        """(per_step, [(kind, index, dim, offset), ...]); kind 0 preact(layer),
        1 x_t, 2 u_t, 3 p_t, 4 cost op(index)."""
        if self._layout is None:
            cap = 64
            per, n = C.c_int(), C.c_int()
            arrs = [np.zeros(cap, dtype=np.int32) for _ in range(4)]
            check(self.lib.bp_stat_layout(self.h, C.byref(per), C.byref(n), *[_capi.iptr(a) for a in arrs], cap))
            self._layout = (per.value, [tuple(int(a[i]) for a in arrs) for i in range(n.value)])
        return self._layout

    # ------------------------------------------------------------------ rollout
    def rollout(self, actions: np.ndarray, want_states: bool = False, want_stats: bool = True):
        """actions: (n_sub, rows, d) -> costs (n_sub, rows), states, emp lo/hi (n_sub, H, per_step), nonfinite.
        The rollout kernels compute in FP32 (3xTF32 on the tensor cores); actions are taken as FP32
        (FP64 input is rounded here, as bp_rollout's float* interface requires)."""
        a = np.ascontiguousarray(actions, dtype=np.float32)
        if a.ndim == 2:
            a = a[None]
        n_sub, rows, d = a.shape
        if d != self.spec.d:
            raise ValueError("evaluate: batch width does not match the input dimension")
        per, _ = self.stat_layout()
        H, ks = self.spec.horizon, self.spec.ks
        costs = np.zeros((n_sub, rows), dtype=np.float32)
        states = np.zeros((n_sub, rows, H, ks), dtype=np.float32) if want_states else None
        lo = np.zeros((n_sub, H, per), dtype=np.float32) if want_stats else None
        hi = np.zeros((n_sub, H, per), dtype=np.float32) if want_stats else None
        bad = np.zeros(n_sub, dtype=np.int32)
        check(self.lib.bp_rollout(self.h, n_sub, rows, _capi.fptr(a), _capi.fptr(costs), _capi.fptr(states),
                                  _capi.fptr(lo), _capi.fptr(hi), _capi.iptr(bad)))
        return costs, states, lo, hi, bad

    # ------------------------------------------------------------------- search
    def batch_search(self, lo: np.ndarray, hi: np.ndarray, warm: Optional[np.ndarray], cfg: dict, seed: int,
                     method: str = "babnd"):
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        n, d = lo.shape
        w = None if warm is None else np.ascontiguousarray(warm, dtype=np.float64)
        packed = _config.PackedConfig(cfg, method)
        check(self.lib.bp_batch_search(self.h, n, _capi.dptr(lo), _capi.dptr(hi), _capi.dptr(w),
                                       packed.search_ref(seed)))
        uf = np.zeros(n)
        best = np.zeros((n, d))
        samples = np.zeros(n, dtype=np.int64)
        ok = np.zeros(n, dtype=np.int32)
        ntop = np.zeros(n, dtype=np.int32)
        check(self.lib.bp_report_summary(self.h, _capi.dptr(uf), _capi.dptr(best),
                                         samples.ctypes.data_as(C.POINTER(C.c_int64)), _capi.iptr(ok),
                                         _capi.iptr(ntop)))
        return {"uf": uf, "best": best, "samples": samples, "ok": ok.astype(bool), "n_top": ntop}

    def search_update(self, cfg: dict, lo: np.ndarray, hi: np.ndarray, it: int, rows: np.ndarray, costs: np.ndarray,
                      state: dict, method: str = "babnd") -> dict:
        """One device sampler update (bp_search_update) on given rows [n][R][d] and costs [n][R]:
        incumbent + top-K + CEM refit / MPPI mean.  state (and the result): mu, var, uf, best,
        top_n, top_val, top_seq, top_act as float32 / int32 arrays."""
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        n = lo.shape[0]
        packed = _config.PackedConfig(cfg, method)
        st = {k: np.ascontiguousarray(v, dtype=np.int32 if k in ("top_n", "top_seq") else np.float32).copy()
              for k, v in state.items()}
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        costs = np.ascontiguousarray(costs, dtype=np.float32)
        check(self.lib.bp_search_update(self.h, n, packed.search_ref(0), _capi.dptr(lo), _capi.dptr(hi), int(it),
                                        _capi.fptr(rows), _capi.fptr(costs), _capi.fptr(st["mu"]),
                                        _capi.fptr(st.get("var")), _capi.fptr(st["uf"]), _capi.fptr(st["best"]),
                                        _capi.iptr(st["top_n"]), _capi.fptr(st["top_val"]), _capi.iptr(st["top_seq"]),
                                        _capi.fptr(st["top_act"])))
        return st

    def report_top(self, box: int, n_top: int):
        d = self.spec.d
        v = np.zeros(max(n_top, 1))
        a = np.zeros((max(n_top, 1), d))
        check(self.lib.bp_report_top(self.h, box, _capi.dptr(v), _capi.dptr(a), n_top))
        return v[:n_top], a[:n_top]

    def report_stats(self, box: int):
        per, _ = self.stat_layout()
        lo = np.zeros((self.spec.horizon, per), dtype=np.float32)
        hi = np.zeros((self.spec.horizon, per), dtype=np.float32)
        check(self.lib.bp_report_stats(self.h, box, _capi.fptr(lo), _capi.fptr(hi)))
        return lo, hi

    def batch_bound(self, n: int, mode: str = "early-stop-empirical", alpha: str = "adaptive") -> np.ndarray:
        lf = np.zeros(n)
        check(self.lib.bp_batch_bound(self.h, _BOUND[mode], _ALPHA[alpha], _capi.dptr(lf)))
        return lf

    def bound_boxes(self, lo, hi, mode: str = "early-stop-interval", alpha: str = "adaptive") -> np.ndarray:
        lo = np.ascontiguousarray(np.atleast_2d(lo), dtype=np.float64)
        hi = np.ascontiguousarray(np.atleast_2d(hi), dtype=np.float64)
        lf = np.zeros(lo.shape[0])
        check(self.lib.bp_bound_boxes(self.h, lo.shape[0], _capi.dptr(lo), _capi.dptr(hi), _BOUND[mode],
                                      _ALPHA[_config._parse_enum(_ALPHA, alpha, "alpha policy")], _capi.dptr(lf)))
        return lf

    def gradient(self, actions: np.ndarray) -> np.ndarray:
        """d objective / d actions per row (Objective::gradient), FP64 on the device."""
        a = np.ascontiguousarray(np.atleast_2d(actions), dtype=np.float32)
        g = np.zeros_like(a)
        check(self.lib.bp_gradient(self.h, a.shape[0], _capi.fptr(a), _capi.fptr(g)))
        return g

    def node_bounds(self, n_boxes: int):
        """The intermediate bounds of the last bound call, (n_boxes, H, per_step) lo / hi."""
        per, _ = self.stat_layout()
        lo = np.zeros((n_boxes, self.spec.horizon, per))
        hi = np.zeros((n_boxes, self.spec.horizon, per))
        check(self.lib.bp_node_bounds(self.h, _capi.dptr(lo), _capi.dptr(hi)))
        return lo, hi

    # ---------------------------------------------------------- pool operations
    def pool_split(self, lo, hi, top_val, top_act, n_top, samples, top_percent=1.0, min_width=1e-6, split_rule=0):
        """split() (bab.cpp:155-223) of n parents on the device (pool.cu split_kernel).

        lo / hi (n, d); top_val (n, K) and top_act (n, K, d) hold n_top[i] ascending
        entries each.  Returns (axis (n,), child_lo / child_hi (2n, d), child_n (2n,),
        child_val (2n, K), child_act (2n, K, d)); child 2i is the lower half."""
        lo, hi = np.ascontiguousarray(lo, np.float64), np.ascontiguousarray(hi, np.float64)
        n, d = lo.shape
        tv = np.ascontiguousarray(top_val, np.float32)
        K = tv.shape[1]
        ta = np.ascontiguousarray(top_act, np.float32).reshape(n, K, d)
        nt = np.ascontiguousarray(n_top, np.int32)
        sm = np.ascontiguousarray(samples, np.int64)
        axis = np.zeros(n, np.int32)
        clo, chi = np.zeros((2 * n, d)), np.zeros((2 * n, d))
        cn = np.zeros(2 * n, np.int32)
        cv, ca = np.zeros((2 * n, K), np.float32), np.zeros((2 * n, K, d), np.float32)
        check(self.lib.bp_pool_split(self.h, n, d, K, _capi.dptr(lo), _capi.dptr(hi), _capi.iptr(nt), _capi.fptr(tv),
                                     _capi.fptr(ta), sm.ctypes.data_as(C.POINTER(C.c_int64)), float(top_percent),
                                     float(min_width), int(split_rule), _capi.iptr(axis), _capi.dptr(clo),
                                     _capi.dptr(chi), _capi.iptr(cn), _capi.fptr(cv), _capi.fptr(ca)))
        return axis, clo, chi, cn, cv, ca

    def pool_merge(self, capacity, a_n, a_val, a_act, b_n, b_val, b_act, b_uf, b_best, b_failed):
        """merge_report() (bab.cpp:245-262) of n records on the device (pool.cu merge_kernel);
        the record's incumbent is its list's front.  Returns (n, val, act, uf, has_best, best)."""
        a_val = np.ascontiguousarray(a_val, np.float32)
        n, K = a_val.shape
        a_act = np.ascontiguousarray(a_act, np.float32)
        d = a_act.shape[2]
        f = lambda x: np.ascontiguousarray(x, np.float32)
        i32 = lambda x: np.ascontiguousarray(x, np.int32)
        on, ov, oa = np.zeros(n, np.int32), np.zeros((n, K), np.float32), np.zeros((n, K, d), np.float32)
        ou, oh, ob = np.zeros(n, np.float32), np.zeros(n, np.int32), np.zeros((n, d), np.float32)
        an, bn, bf = i32(a_n), i32(b_n), i32(b_failed)
        bv, ba, bu, bb = f(b_val), f(b_act), f(b_uf), f(b_best)
        check(self.lib.bp_pool_merge(self.h, n, d, K, int(capacity), _capi.iptr(an), _capi.fptr(a_val),
                                     _capi.fptr(a_act), _capi.iptr(bn), _capi.fptr(bv), _capi.fptr(ba),
                                     _capi.fptr(bu), _capi.fptr(bb), _capi.iptr(bf), _capi.iptr(on), _capi.fptr(ov),
                                     _capi.fptr(oa), _capi.fptr(ou), _capi.iptr(oh), _capi.fptr(ob)))
        return on, ov, oa, ou, oh, ob

    # --------------------------------------------------------------------- plan
    def plan(self, cfg: dict, warm: Optional[np.ndarray] = None, method: str = "babnd") -> dict:
        packed = _config.PackedConfig(cfg, method)
        w = None if warm is None else np.ascontiguousarray(warm, dtype=np.float64)
        res = C.c_void_p()
        check(self.lib.bp_plan(self.h, packed.ref(), _capi.dptr(w), 1 if method == "babnd" else 0, C.byref(res)))
        return _result_dict(self.lib, res)

    def planner(self, cfg: dict, warm: Optional[np.ndarray] = None) -> "Planner":
        """plan() driven one BaB iteration at a time (the bench steps it)."""
        return Planner(self, cfg, warm)

    def set_stream(self, stream_handle: Optional[int]) -> None:
        """Run on an external CUDA stream (e.g. torch.cuda.current_stream().cuda_stream)."""
        check(self.lib.bp_set_stream(self.h, C.c_void_p(stream_handle) if stream_handle else None))

    def rollout_path(self, path: Optional[str] = None) -> str:
        """Select ("auto" | "simt" | "tc1" | "tc2" | "tc3") and report ("tcgen05" | "simt") the
        rollout kernel family; rollout_kernel() names the exact kernel."""
        code = {None: -1, "auto": 0, "simt": 1, "tc1": 2, "tc2": 3, "tc3": 5}[path]
        active = C.c_int()
        check(self.lib.bp_set_rollout_path(self.h, code, C.byref(active)))
        return "tcgen05" if active.value in (2, 3, 5) else "simt"

    def rollout_kernel(self) -> str:
        """The rollout kernel the loaded objective runs: "tc3" (tcgen05 v3, rollout_tc3.cu), "tc2"
        (tcgen05 v2, rollout_tc2.cu), "tc1" (tcgen05 v1, rollout_tc.cu) or "simt" (FP32 FFMA, rollout.cu)."""
        active = C.c_int()
        check(self.lib.bp_set_rollout_path(self.h, -1, C.byref(active)))
        return {1: "simt", 2: "tc1", 3: "tc2", 4: "synthetic", 5: "tc3"}[active.value]

    def rollout_info(self) -> dict:
        """Rollout kernel, 128-row tiles per CTA, rows per CTA and shared memory per CTA."""
        k, t, r, sm = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        check(self.lib.bp_rollout_info(self.h, C.byref(k), C.byref(t), C.byref(r), C.byref(sm)))
        return {"kernel": {1: "simt", 2: "tc1", 3: "tc2", 4: "synthetic", 5: "tc3"}[k.value], "tiles_per_cta": t.value,
                "rows_per_cta": r.value, "smem_bytes": sm.value}

    def rollout_tiles(self) -> int:
        return self.rollout_info()["tiles_per_cta"]

    @staticmethod
    def io_bytes():
        """(h2d, d2h) bytes copied by the library since the previous call."""
        lib = _capi.load()
        a, b = C.c_int64(), C.c_int64()
        check(lib.bp_io_bytes(C.byref(a), C.byref(b)))
        return a.value, b.value

    def timing(self) -> dict:
        """Device time since the previous call: rollout ms and launches, bound ms, search wall ms."""
        r, b, s = C.c_double(), C.c_double(), C.c_double()
        rl, l = C.c_int64(), C.c_int64()
        check(self.lib.bp_timing(self.h, C.byref(r), C.byref(rl), C.byref(b), C.byref(s), C.byref(l)))
        return {"rollout_ms": r.value, "rollout_launches": rl.value, "bound_ms": b.value, "search_ms": s.value,
                "launches": l.value}


    def plan_log(self, enable: Optional[bool] = None) -> Optional[dict]:
        """Decision-replay log of the plans run on this device (bp_set_plan_log): enable / disable
        with a bool; with no argument, the log of the last plan as arrays in child order."""
        if enable is not None:
            check(self.lib.bp_set_plan_log(self.h, 1 if enable else 0))
            return None
        n, tot = C.c_int(), C.c_int()
        check(self.lib.bp_plan_log_size(self.h, C.byref(n), C.byref(tot)))
        n, tot, d = n.value, tot.value, self.spec.d
        out = {"iter": np.zeros(n, np.int32), "lo": np.zeros((n, d)), "hi": np.zeros((n, d)), "lf": np.zeros(n),
               "uf": np.zeros(n), "best": np.zeros((n, d)), "n_top": np.zeros(n, np.int32),
               "top_val": np.zeros(max(tot, 1)), "top_act": np.zeros((max(tot, 1), d)),
               "samples": np.zeros(n, np.int64), "ok": np.zeros(n, np.int32)}
        check(self.lib.bp_plan_log_get(self.h, _capi.iptr(out["iter"]), _capi.dptr(out["lo"]), _capi.dptr(out["hi"]),
                                       _capi.dptr(out["lf"]), _capi.dptr(out["uf"]), _capi.dptr(out["best"]),
                                       _capi.iptr(out["n_top"]), _capi.dptr(out["top_val"]), _capi.dptr(out["top_act"]),
                                       out["samples"].ctypes.data_as(C.POINTER(C.c_int64)), _capi.iptr(out["ok"])))
        return out

    def search_counters(self) -> dict:
        """Boxes searched and boxes whose search failed (non-finite rollout) since the previous call."""
        b, f = C.c_int64(), C.c_int64()
        check(self.lib.bp_search_counters(self.h, C.byref(b), C.byref(f)))
        return {"boxes": b.value, "failed": f.value}


def _result_dict(lib, res) -> dict:
    try:
        uf, mlf = C.c_double(), C.c_double()
        cert, iters, ntr, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        samples = C.c_int64()
        stop = C.create_string_buffer(64)
        check(lib.bp_result_summary(res, C.byref(uf), C.byref(mlf), C.byref(cert), C.byref(samples),
                                    C.byref(iters), stop, 64, C.byref(ntr), C.byref(d)))
        best = np.zeros(d.value)
        check(lib.bp_result_best(res, _capi.dptr(best)))
        rows = (_capi.TraceRow * max(1, ntr.value))()
        check(lib.bp_result_trace(res, rows, ntr.value))
    finally:
        lib.bp_result_free(res)
    tr = rows[:ntr.value]
    trace = {k: [getattr(r, k) for r in tr] for k in
             ("iter", "uf", "min_lf", "pruned_vol", "selected_vol", "pool_size", "samples", "wall_ms")}
    return {"objective": uf.value, "action": best, "lower_bound": mlf.value, "certified": bool(cert.value),
            "samples": samples.value, "iterations": iters.value, "stop_reason": stop.value.decode(),
            "trace": trace}


class Planner:
    """bp_planner handle: root search + bound on creation, then step()."""

    def __init__(self, dev: Device, cfg: dict, warm=None):
        self.dev, self.lib = dev, dev.lib
        self._packed = _config.PackedConfig(cfg)
        self._w = None if warm is None else np.ascontiguousarray(warm, dtype=np.float64)
        self.h = C.c_void_p()
        check(self.lib.bp_planner_create(dev.h, self._packed.ref(), _capi.dptr(self._w), C.byref(self.h)))

    def step(self):
        """One BaB iteration -> (stepped, children searched+bounded, pool size)."""
        st, ch, ps = C.c_int(), C.c_int(), C.c_int()
        check(self.lib.bp_planner_step(self.h, C.byref(st), C.byref(ch), C.byref(ps)))
        return bool(st.value), ch.value, ps.value

    def finish(self) -> dict:
        res = C.c_void_p()
        check(self.lib.bp_planner_finish(self.h, C.byref(res)))
        return _result_dict(self.lib, res)

    def close(self):
        if self.h:
            self.lib.bp_planner_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Device] = None


def default_device() -> Device:
    global _default
    if _default is None:
        _default = Device()
    return _default


# ----------------------------------------------------------- reference API
def default_config() -> str:
    return _config.default_config()


def plan(model: Model, scenario: Scenario, config: str = "", method: str = "babnd") -> dict:
    """pymodule.cpp:152-160: build the unrolled objective, then plan() or sample_only_plan()."""
    cfg = _config.from_json(config)
    dev = default_device().load(build_objective(model, scenario))
    return dev.plan(cfg, None, method)


def objective_value(model: Model, scenario: Scenario, actions) -> np.ndarray:
    """pymodule.cpp:171-178: objective per row of flattened action sequences.  The device
    evaluates in FP32 (3xTF32 on the tensor-core kernels): the FP64 actions are rounded to FP32
    here, and the result agrees with the reference's FP64 evaluation within the stated bars
    (1e-5 relative to max(|value|, 1) on the SIMT and tensor-core kernels)."""
    a = np.asarray(actions, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if not np.all(np.isfinite(a)):
        raise ValueError("evaluate batch: non-finite values")
    dev = default_device().load(build_objective(model, scenario))
    costs, _, _, _, bad = dev.rollout(a[None].astype(np.float32), want_stats=False)
    if bad[0]:
        raise RuntimeError("evaluate: non-finite objective value (malformed weights?)")
    return costs[0].astype(np.float64)


def lower_bound(model: Model, scenario: Scenario, mode: str = "full-crown", alpha: str = "adaptive") -> float:
    """pymodule.cpp:180-190: bound over the whole action box without samples."""
    if mode not in _BOUND:
        raise ValueError(f"unknown bound mode '{mode}'")
    if alpha not in _ALPHA:
        raise ValueError(f"unknown alpha policy '{alpha}'")
    spec = build_objective(model, scenario)
    dev = default_device().load(spec)
    lo, hi = spec.box()
    return float(dev.bound_boxes(lo[None], hi[None], mode, alpha)[0])


def network_lower_bound(model: Model, lower, upper, mode: str = "full-crown", alpha: str = "adaptive") -> float:
    """pymodule.cpp:192-202: certified lower bound of a scalar-output network over an
    input box (build_network_objective, model.cpp:389-405), on the device."""
    if mode not in _BOUND:
        raise ValueError(f"unknown bound mode '{mode}'")
    if alpha not in _ALPHA:
        raise ValueError(f"unknown alpha policy '{alpha}'")
    spec = build_network_objective(model, lower, upper)
    dev = default_device().load(spec)
    lo, hi = spec.box()
    if not (np.all(np.isfinite(lo)) and np.all(np.isfinite(hi)) and np.all(lo <= hi)):
        raise ValueError("BoxDomain: invalid bounds")
    return float(dev.bound_boxes(lo[None], hi[None], mode, alpha)[0])


def rollout(model: Model, scenario: Scenario, action) -> np.ndarray:
    """pymodule.cpp:204-223: states x_1..x_H of one flattened action sequence (H x ks)."""
    a = np.asarray(action, dtype=np.float64).reshape(-1)
    if a.size != scenario.action_dim() * scenario.horizon:
        raise ValueError("action length must be horizon * action_dim")
    dev = default_device().load(build_objective(model, scenario))
    _, states, _, _, _ = dev.rollout(a.reshape(1, 1, -1).astype(np.float32), want_states=True, want_stats=False)
    return states[0, 0].astype(np.float64)


def plan_synthetic(d: int, config: str = "", method: str = "babnd") -> dict:
    """pymodule.cpp:162-169: minimise the separable benchmark objective on [-1, 1]^d;
    babnd uses the exact SeparableBounder (bab.cpp:275-283), on the device."""
    cfg = _config.from_json(config)
    return default_device().load_synthetic(int(d)).plan(cfg, None, method)


def rrt_plan(*args, **kwargs):
    raise NotImplementedError("RRT/PRM graph-planner baselines are out of scope (SURVEY 2, row 11)")


def prm_plan(*args, **kwargs):
    raise NotImplementedError("RRT/PRM graph-planner baselines are out of scope (SURVEY 2, row 11)")
