"""TEST INFRASTRUCTURE ONLY -- ctypes driver of the FP64 oracle (oracle/*.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / the timed CPU implementation;
the product path (paper_2412_09584_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import Optional

import numpy as np

from paper_2412_09584_b200 import _capi
from paper_2412_09584_b200.config import ALPHAS, BOUND_MODES, PackedConfig

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
_lib = None
_lock = threading.Lock()
vp = C.c_void_p
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


def build() -> str:
    srcs = [os.path.join(HERE, f) for f in ("oracle.cpp", "oracle_capi.cpp", "oracle.hpp")]
    if not os.path.exists(LIB) or any(os.path.getmtime(s) > os.path.getmtime(LIB) for s in srcs):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.or_last_error.restype = C.c_size_t
            for name in ("or_rng_new", "or_graph_new", "or_stats_new", "or_report_stats"):
                getattr(L, name).restype = vp
            L.or_rng_new.argtypes = [C.c_uint64]
            for name in ("or_rng_uniform", "or_rng_normal"):
                getattr(L, name).restype = C.c_double
                getattr(L, name).argtypes = [vp]
            L.or_rng_bits.restype = C.c_uint64
            L.or_rng_bits.argtypes = [vp]
            L.or_mix_seed.restype = C.c_uint64
            L.or_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
            L.or_separable_term_min.restype = C.c_double
            L.or_separable_term_min.argtypes = [C.c_double, C.c_double]
            L.or_report_stats.argtypes = [vp, C.c_int]
            L.or_generate_model.argtypes = [C.c_uint64, C.c_int, ip, dp]
            _lib = L
        return _lib


def ck(status: int):
    if status != 0:
        buf = C.create_string_buffer(1024)
        lib().or_last_error(buf, 1024)
        msg = buf.value.decode()
        raise {1: ValueError, 2: RuntimeError, 3: RuntimeError}.get(status, RuntimeError)(msg)


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def thread_count() -> int:
    return lib().or_thread_count()


def mix_seed(m: int, s: int) -> int:
    return lib().or_mix_seed(m, s)


class Rng:
    def __init__(self, seed: int):
        self.h = lib().or_rng_new(seed & (2**64 - 1))

    def __del__(self):
        try:
            lib().or_rng_free(vp(self.h))
        except Exception:
            pass

    def uniform(self):
        return lib().or_rng_uniform(vp(self.h))

    def normal(self):
        return lib().or_rng_normal(vp(self.h))

    def bits(self):
        return lib().or_rng_bits(vp(self.h))

    def uniform_int(self, n):
        return lib().or_rng_uniform_int(vp(self.h), int(n))


def generate_model_params(seed: int, widths) -> np.ndarray:
    w = np.asarray(widths, dtype=np.int32)
    n = sum(int(w[i]) * int(w[i + 1]) + int(w[i + 1]) for i in range(len(w) - 1))
    out = np.zeros(n)
    ck(lib().or_generate_model(seed, len(w), w.ctypes.data_as(ip), out.ctypes.data_as(dp)))
    return out


class Stats:
    def __init__(self, handle=None, owned=True):
        self.h = handle if handle is not None else lib().or_stats_new()
        self.owned = owned

    def __del__(self):
        if self.owned:
            try:
                lib().or_stats_free(vp(self.h))
            except Exception:
                pass

    def get(self, node: int, dim: int):
        mn, mx = np.zeros(dim), np.zeros(dim)
        cnt = C.c_int64()
        n = lib().or_stats_get(vp(self.h), node, mn.ctypes.data_as(dp), mx.ctypes.data_as(dp), C.byref(cnt))
        if n < 0:
            return None
        return mn[:n], mx[:n], cnt.value

    def set(self, node: int, mn, mx, count: int = 1):
        mn, mx = _d(mn), _d(mx)
        lib().or_stats_set(vp(self.h), node, mn.ctypes.data_as(dp), mx.ctypes.data_as(dp), mn.size,
                           C.c_int64(count))

    def ids(self):
        n = lib().or_stats_ids(vp(self.h), None, 0)
        out = np.zeros(max(n, 1), dtype=np.int32)
        lib().or_stats_ids(vp(self.h), out.ctypes.data_as(ip), n)
        return [int(x) for x in out[:n]]


class Graph:
    """CompGraph builder (graph.hpp:52-88) for hand-written KAT graphs."""

    def __init__(self):
        self.h = lib().or_graph_new()

    def __del__(self):
        try:
            lib().or_graph_free(vp(self.h))
        except Exception:
            pass

    def _id(self, fn, *args):
        out = C.c_int()
        ck(fn(vp(self.h), *args, C.byref(out)))
        return out.value

    def input(self, dim):
        return self._id(lib().or_graph_add_input, C.c_int(dim))

    def constant(self, v):
        v = _d(v)
        return self._id(lib().or_graph_add_constant, v.ctypes.data_as(dp), C.c_int(v.size))

    def linear(self, arg, W, b):
        W, b = _d(W), _d(b)
        return self._id(lib().or_graph_add_linear, C.c_int(arg), W.ctypes.data_as(dp), C.c_int(W.shape[0]),
                        C.c_int(W.shape[1]), b.ctypes.data_as(dp))

    def relu(self, arg):
        return self._id(lib().or_graph_add_relu, C.c_int(arg))

    def sum(self, args):
        a = np.asarray(args, dtype=np.int32)
        return self._id(lib().or_graph_add_sum, a.ctypes.data_as(ip), C.c_int(a.size))

    def scalar_affine(self, arg, s, o):
        return self._id(lib().or_graph_add_scalar_affine, C.c_int(arg), C.c_double(s), C.c_double(o))

    def squared_distance(self, arg, t, w):
        t, w = _d(t), _d(w)
        return self._id(lib().or_graph_add_squared_distance, C.c_int(arg), t.ctypes.data_as(dp),
                        w.ctypes.data_as(dp), C.c_int(t.size))

    def penalty_hinge(self, arg, c, r, p):
        c = _d(c)
        return self._id(lib().or_graph_add_penalty_hinge, C.c_int(arg), c.ctypes.data_as(dp), C.c_int(c.size),
                        C.c_double(r), C.c_double(p))

    def concat(self, args):
        a = np.asarray(args, dtype=np.int32)
        return self._id(lib().or_graph_add_concat, a.ctypes.data_as(ip), C.c_int(a.size))

    def slice(self, arg, begin, length):
        return self._id(lib().or_graph_add_slice, C.c_int(arg), C.c_int(begin), C.c_int(length))

    def set_output(self, node):
        ck(lib().or_graph_set_output(vp(self.h), C.c_int(node)))

    def finalize(self):
        ck(lib().or_graph_finalize(vp(self.h)))

    def size(self):
        return lib().or_graph_size(vp(self.h))

    def dim(self, node):
        return lib().or_graph_node_dim(vp(self.h), C.c_int(node))

    def evaluate(self, batch, watch=None, stats: Optional[Stats] = None):
        b = _d(np.atleast_2d(batch))
        out = np.zeros(b.shape[0])
        w = np.asarray(watch or [0], dtype=np.int32)
        ck(lib().or_graph_evaluate(vp(self.h), b.ctypes.data_as(dp), C.c_int(b.shape[0]), C.c_int(b.shape[1]),
                                   out.ctypes.data_as(dp), w.ctypes.data_as(ip), C.c_int(len(watch or [])),
                                   vp(stats.h) if stats else None))
        return out

    def gradient(self, batch):
        b = _d(np.atleast_2d(batch))
        out = np.zeros_like(b)
        ck(lib().or_graph_gradient(vp(self.h), b.ctypes.data_as(dp), C.c_int(b.shape[0]), C.c_int(b.shape[1]),
                                   out.ctypes.data_as(dp)))
        return out

    def interval(self, lo, hi, node):
        lo, hi = _d(lo), _d(hi)
        n = self.dim(node)
        a, b = np.zeros(n), np.zeros(n)
        ck(lib().or_graph_interval(vp(self.h), lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), C.c_int(lo.size),
                                   C.c_int(node), a.ctypes.data_as(dp), b.ctypes.data_as(dp)))
        return a, b

    def objective(self, step_states=(), final_step_last_relu=-1) -> "Objective":
        ss = np.asarray(list(step_states) or [0], dtype=np.int32)
        h = vp()
        ck(lib().or_objective_from_graph(vp(self.h), ss.ctypes.data_as(ip), C.c_int(len(step_states)),
                                         C.c_int(final_step_last_relu), C.byref(h)))
        return Objective(handle=h)


class Objective:
    """GraphObjective (or the synthetic objective) on the oracle side."""

    def __init__(self, spec=None, handle=None, synthetic_dim: Optional[int] = None):
        if handle is not None:
            self.h = handle
        elif synthetic_dim is not None:
            self.h = vp()
            ck(lib().or_objective_synthetic(C.c_int(synthetic_dim), C.byref(self.h)))
        else:
            self.spec = spec
            self._packed = spec.to_c()
            self.h = vp()
            ck(lib().or_objective_from_desc(self._packed.ref(), C.byref(self.h)))

    def __del__(self):
        try:
            lib().or_objective_free(self.h)
        except Exception:
            pass

    @property
    def dim(self):
        return lib().or_objective_dim(self.h)

    def box(self):
        d = self.dim
        lo, hi = np.zeros(d), np.zeros(d)
        lib().or_objective_box(self.h, lo.ctypes.data_as(dp), hi.ctypes.data_as(dp))
        return lo, hi

    def _set(self, which):
        n = lib().or_objective_sets(self.h, which, None, 0)
        out = np.zeros(max(n, 1), dtype=np.int32)
        lib().or_objective_sets(self.h, which, out.ctypes.data_as(ip), n)
        return [int(x) for x in out[:n]]

    def stop_set(self):
        return self._set(0)

    def watch_set(self):
        return self._set(1)

    def relu_nodes(self):
        return self._set(2)

    def set_stop_rule(self, rule: int, ids=()):
        a = np.asarray(list(ids) or [0], dtype=np.int32)
        ck(lib().or_objective_set_stop_rule(self.h, rule, a.ctypes.data_as(ip), len(ids)))

    def step_nodes(self, t: int):
        uxp = np.zeros(3, dtype=np.int32)
        pre = np.zeros(16, dtype=np.int32)
        ops = np.zeros(64, dtype=np.int32)
        code = lib().or_objective_step_nodes(self.h, t, uxp.ctypes.data_as(ip), pre.ctypes.data_as(ip), 16,
                                             ops.ctypes.data_as(ip), 64)
        n_pre, n_ops = code // 1000, code % 1000
        return {"u": int(uxp[0]), "x": int(uxp[1]), "p": int(uxp[2]), "preact": [int(x) for x in pre[:n_pre]],
                "ops": [int(x) for x in ops[:n_ops]]}

    def node_dim(self, node):
        return lib().or_objective_node_dim(self.h, node)

    def evaluate(self, batch, stats: Optional[Stats] = None):
        b = _d(np.atleast_2d(batch))
        out = np.zeros(b.shape[0])
        ck(lib().or_objective_evaluate(self.h, b.ctypes.data_as(dp), C.c_int(b.shape[0]), C.c_int(b.shape[1]),
                                       out.ctypes.data_as(dp), vp(stats.h) if stats else None))
        return out

    def lower_bound(self, lo, hi, mode="early-stop-empirical", stats: Optional[Stats] = None, alpha="adaptive"):
        lo, hi = _d(lo), _d(hi)
        out = C.c_double()
        ck(lib().or_lower_bound(self.h, lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), BOUND_MODES[mode],
                                vp(stats.h) if stats else None, ALPHAS[alpha], C.byref(out)))
        return out.value

    def gradient(self, batch):
        b = _d(np.atleast_2d(batch))
        out = np.zeros_like(b)
        ck(lib().or_objective_gradient(self.h, b.ctypes.data_as(dp), C.c_int(b.shape[0]), out.ctypes.data_as(dp)))
        return out

    def crown_node_stats(self, lo, hi, ids, alpha="adaptive") -> Stats:
        """crown_node_bounds (crown.cpp:379-412) for the given nodes, as watch stats."""
        lo, hi = _d(lo), _d(hi)
        ids = np.asarray(list(ids), dtype=np.int32)
        h = vp()
        ck(lib().or_crown_node_stats(self.h, lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), ALPHAS[alpha],
                                     ids.ctypes.data_as(ip), C.c_int(len(ids)), C.byref(h)))
        return Stats(handle=h.value)

    def stats_in_layout(self, stats: Stats, layout, horizon: int):
        """Oracle watch stats rearranged into the device record layout (H x per_step)."""
        per, slots = layout
        lo = np.full((horizon, per), np.nan)
        hi = np.full((horizon, per), np.nan)
        relu_layers = None
        for t in range(horizon):
            sn = self.step_nodes(t)
            for kind, index, dim, off in slots:
                if kind == 0:
                    if relu_layers is None:
                        relu_layers = [l for l in range(len(self.spec.relu)) if self.spec.relu[l]]
                    node = sn["preact"][relu_layers.index(index)]
                else:
                    node = {1: sn["x"], 2: sn["u"], 3: sn["p"]}.get(kind)
                    if kind == 4:
                        node = sn["ops"][index]
                r = stats.get(node, dim)
                if r is not None:
                    lo[t, off:off + dim], hi[t, off:off + dim] = r[0], r[1]
        return lo, hi

    def stats_from_layout(self, lo, hi, layout, horizon: int) -> Stats:
        """Device-layout extrema (H x per_step) as oracle WatchStats on the matching nodes."""
        per, slots = layout
        st = Stats()
        relu_layers = [l for l in range(len(self.spec.relu)) if self.spec.relu[l]]
        for t in range(horizon):
            sn = self.step_nodes(t)
            for kind, index, dim, off in slots:
                if kind == 0:
                    node = sn["preact"][relu_layers.index(index)]
                    # the ReLU node itself: extrema are relu(extrema of its argument)
                    st.set(node + 1, np.maximum(lo[t, off:off + dim], 0), np.maximum(hi[t, off:off + dim], 0))
                elif kind == 4:
                    node = sn["ops"][index]
                else:
                    node = {1: sn["x"], 2: sn["u"], 3: sn["p"]}[kind]
                st.set(node, lo[t, off:off + dim], hi[t, off:off + dim])
        return st

    def batch_search(self, lo, hi, warm, cfg: dict, seed: int, method: str = "babnd") -> "Reports":
        lo, hi = _d(np.atleast_2d(lo)), _d(np.atleast_2d(hi))
        w = None if warm is None else _d(warm)
        packed = PackedConfig(cfg, method)
        h = vp()
        ck(lib().or_batch_search(self.h, C.c_int(lo.shape[0]), lo.ctypes.data_as(dp), hi.ctypes.data_as(dp),
                                 w.ctypes.data_as(dp) if w is not None else None, packed.search_ref(seed),
                                 C.byref(h)))
        return Reports(h, self, lo, hi)

    def plan_replay(self, cfg: dict, log: dict) -> dict:
        """plan() (bab.cpp:266-415) taking every child's search report and bound from a device plan
        log (Device.plan_log()) instead of searching and bounding: the decisions (pick_out, split,
        merge_report, prune, the incumbent and the trace) are the oracle's own.  Adds box_mismatch
        (children whose box differs from the device's) and order_mismatch to the plan dict."""
        packed = PackedConfig(cfg, "babnd")
        n = len(log["lf"])
        n_top = np.ascontiguousarray(log["n_top"], dtype=np.int32)
        off = np.zeros(n, dtype=np.int32)
        if n > 1:
            off[1:] = np.cumsum(n_top)[:-1]
        arrs = {k: np.ascontiguousarray(log[k], dtype=np.float64) for k in ("lo", "hi", "lf", "uf", "best", "top_val", "top_act")}
        it = np.ascontiguousarray(log["iter"], dtype=np.int32)
        samples = np.ascontiguousarray(log["samples"], dtype=np.int64)
        ok = np.ascontiguousarray(log["ok"], dtype=np.int32)
        bm, om = C.c_int(), C.c_int()
        h = vp()
        ck(lib().or_plan_replay(self.h, packed.ref(), C.c_int(n), it.ctypes.data_as(ip), *[arrs[k].ctypes.data_as(dp) for k in ("lo", "hi", "lf", "uf", "best")],
                                n_top.ctypes.data_as(ip), off.ctypes.data_as(ip), arrs["top_val"].ctypes.data_as(dp),
                                arrs["top_act"].ctypes.data_as(dp), samples.ctypes.data_as(C.POINTER(C.c_int64)),
                                ok.ctypes.data_as(ip), C.byref(bm), C.byref(om), C.byref(h)))
        res = self._plan_result(h)
        res["box_mismatch"], res["order_mismatch"] = bm.value, om.value
        return res

    def plan(self, cfg: dict, warm=None, method: str = "babnd") -> dict:
        packed = PackedConfig(cfg, method)
        w = _d(warm)
        h = vp()
        ck(lib().or_plan(self.h, packed.ref(), w.ctypes.data_as(dp) if w is not None else None,
                         1 if method == "babnd" else 0, C.byref(h)))
        return self._plan_result(h)

    def _plan_result(self, h) -> dict:
        try:
            uf, mlf = C.c_double(), C.c_double()
            cert, iters = C.c_int(), C.c_int()
            samples = C.c_int64()
            stop = C.create_string_buffer(64)
            best = np.zeros(self.dim)
            n = lib().or_plan_summary(h, C.byref(uf), C.byref(mlf), C.byref(cert), C.byref(samples), C.byref(iters),
                                      stop, 64, best.ctypes.data_as(dp))
            rows = (_capi.TraceRow * max(n, 1))()
            lib().or_plan_trace(h, rows, n)
        finally:
            lib().or_plan_free(h)
        tr = rows[:n]
        return {"objective": uf.value, "action": best, "lower_bound": mlf.value, "certified": bool(cert.value),
                "samples": samples.value, "iterations": iters.value, "stop_reason": stop.value.decode(),
                "trace": {k: [getattr(r, k) for r in tr] for k in
                          ("iter", "uf", "min_lf", "pruned_vol", "selected_vol", "pool_size", "samples", "wall_ms")}}


def search_injected(lo, hi, warm, cfg: dict, rows, costs, method: str = "babnd") -> list:
    """run_cem / run_mppi (search.cpp:87-209) on injected samples rows[it][n_samp][d] and values
    costs[it][R] (R = n_samp + 1; the incumbent row is the searcher's own).  Per iteration the
    state after the refit: batch, mu, var, uf, best, top values / actions (value order)."""
    lo, hi = _d(lo), _d(hi)
    d = lo.shape[0]
    rows, costs = _d(rows), _d(costs)
    T, n_samp = rows.shape[0], rows.shape[1]
    R = n_samp + 1
    packed = PackedConfig(cfg, method)
    s = packed.cfg.search
    G = s.cem_agents if s.method == 0 else max(1, s.mppi_n_noise) * max(1, s.mppi_n_temp)
    K = max(1, s.top_capacity)
    out = {"batch": np.zeros((T, R, d)), "mu": np.zeros((T, G, d)), "var": np.zeros((T, G, d)), "uf": np.zeros(T),
           "best": np.zeros((T, d)), "top_n": np.zeros(T, dtype=np.int32), "top_val": np.zeros((T, K)),
           "top_act": np.zeros((T, K, d))}
    w = _d(warm)
    ck(lib().or_search_injected(C.c_int(d), lo.ctypes.data_as(dp), hi.ctypes.data_as(dp),
                                w.ctypes.data_as(dp) if w is not None else None, packed.search_ref(0), C.c_int(T),
                                C.c_int(n_samp),
                                rows.ctypes.data_as(dp), costs.ctypes.data_as(dp),
                                *[out[k].ctypes.data_as(dp) for k in ("batch", "mu", "var", "uf", "best")],
                                out["top_n"].ctypes.data_as(ip), out["top_val"].ctypes.data_as(dp),
                                out["top_act"].ctypes.data_as(dp)))
    return [{k: v[t] for k, v in out.items()} for t in range(T)]


class Reports:
    def __init__(self, h, obj: Objective, lo, hi):
        self.h, self.obj, self.lo, self.hi = h, obj, lo, hi

    def __del__(self):
        try:
            lib().or_reports_free(self.h)
        except Exception:
            pass

    def __len__(self):
        return self.lo.shape[0]

    def get(self, i: int) -> dict:
        d = self.lo.shape[1]
        uf = C.c_double()
        best = np.zeros(d)
        samples = C.c_int64()
        ok, ntop = C.c_int(), C.c_int()
        lib().or_report_get(self.h, i, C.byref(uf), best.ctypes.data_as(dp), C.byref(samples), C.byref(ok),
                            C.byref(ntop))
        vals = np.zeros(max(ntop.value, 1))
        acts = np.zeros((max(ntop.value, 1), d))
        lib().or_report_top(self.h, i, vals.ctypes.data_as(dp), acts.ctypes.data_as(dp))
        return {"uf": uf.value, "best": best, "samples": samples.value, "ok": bool(ok.value),
                "top_values": vals[:ntop.value], "top_actions": acts[:ntop.value]}

    def stats(self, i: int) -> Stats:
        return Stats(lib().or_report_stats(self.h, i), owned=False)

    def bound(self, i: int, mode="early-stop-empirical", alpha="adaptive") -> float:
        out = C.c_double()
        ck(lib().or_report_bound(self.obj.h, self.h, i, self.lo[i].ctypes.data_as(dp),
                                 self.hi[i].ctypes.data_as(dp), BOUND_MODES[mode], ALPHAS[alpha], C.byref(out)))
        return out.value

    def bound_all(self, mode="early-stop-empirical", alpha="adaptive") -> np.ndarray:
        out = np.zeros(len(self))
        ck(lib().or_reports_bound_all(self.obj.h, self.h, C.c_int(len(self)), self.lo.ctypes.data_as(dp),
                                      self.hi.ctypes.data_as(dp), BOUND_MODES[mode], ALPHAS[alpha],
                                      out.ctypes.data_as(dp)))
        return out


def pick_out(meta, n, eta, temperature, rng: Rng):
    arr = (_capi.PoolMeta * max(1, len(meta)))(*[_capi.PoolMeta(*m) for m in meta])
    picked = np.zeros(max(1, len(meta)), dtype=np.int32)
    k = C.c_int()
    ck(lib().or_pick_out(arr, C.c_int(len(meta)), C.c_int(n), C.c_double(eta), C.c_double(temperature), vp(rng.h),
                         picked.ctypes.data_as(ip), C.byref(k)))
    return [int(x) for x in picked[:k.value]]


def split(lo, hi, top_values, top_u, samples, top_percent=1.0, min_width=1e-6, split_rule=0):
    lo, hi = _d(lo), _d(hi)
    tu = _d(np.atleast_2d(top_u)) if len(top_values) else np.zeros((0, lo.size))
    tv = _d(top_values) if len(top_values) else np.zeros(1)
    axis, mid = C.c_int(), C.c_double()
    route = np.zeros(max(1, len(top_values)), dtype=np.uint8)
    ck(lib().or_split(C.c_int(lo.size), lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), C.c_int(len(top_values)),
                      tv.ctypes.data_as(dp), np.ascontiguousarray(tu).ctypes.data_as(dp), C.c_int64(samples),
                      C.c_double(top_percent), C.c_double(min_width), C.c_int(split_rule), C.byref(axis),
                      C.byref(mid), route.ctypes.data_as(C.POINTER(C.c_ubyte))))
    return axis.value, mid.value, route[:len(top_values)]


def merge_report(capacity, a_val, a_act, a_uf, a_best, b_val, b_act, b_uf, b_best):
    """merge_report (bab.cpp:245-262): returns (values, actions, uf, best or None)."""
    a_act, b_act = np.atleast_2d(a_act), np.atleast_2d(b_act)
    d = a_act.shape[1] if a_act.size else b_act.shape[1]
    na, nb = len(a_val), len(b_val)
    n = C.c_int()
    out_v = np.zeros(max(1, na + nb))
    out_a = np.zeros((max(1, na + nb), d))
    uf, has = C.c_double(), C.c_int()
    best = np.zeros(d)
    opt = lambda x: _d(x).ctypes.data_as(dp) if x is not None else None
    ck(lib().or_merge_report(C.c_int(d), C.c_int(capacity), C.c_int(na), opt(np.asarray(a_val) if na else np.zeros(1)),
                             opt(a_act if na else np.zeros((1, d))), C.c_double(a_uf), opt(a_best),
                             C.c_int(nb), opt(np.asarray(b_val) if nb else np.zeros(1)), opt(b_act if nb else np.zeros((1, d))),
                             C.c_double(b_uf), opt(b_best), C.byref(n), out_v.ctypes.data_as(dp),
                             out_a.ctypes.data_as(dp), C.byref(uf), C.byref(has), best.ctypes.data_as(dp)))
    return out_v[:n.value], out_a[:n.value], uf.value, (best if has.value else None)


def prune(meta, incumbent):
    arr = (_capi.PoolMeta * max(1, len(meta)))(*[_capi.PoolMeta(*m) for m in meta])
    keep = np.zeros(max(1, len(meta)), dtype=np.int32)
    k = C.c_int()
    removed = C.c_double()
    ck(lib().or_prune(arr, C.c_int(len(meta)), C.c_double(incumbent), keep.ctypes.data_as(ip), C.byref(k),
                      C.byref(removed)))
    return [int(x) for x in keep[:k.value]], removed.value


def separable_term_min(a, b):
    return lib().or_separable_term_min(a, b)
