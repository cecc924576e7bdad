"""The BASELINE.json configurations as objective specs + planner configs.

Synthetic, seeded stand-ins (there is no dataset in the reference): weights
He-normal N(0, 2/fan_in) with zero bias from the reference Rng stream
(mt19937_64 + Box-Muller, seed 0); x0 / goals / obstacles from seed 1;
planner seed 2.  Every parameter is rounded to FP32 so the
FP64 oracle and the FP32 device see identical values.  Cost programs follow
SURVEY.md Appendix A.  `glorot=True` swaps in generate_model-style weights
(the reference's own generator), which keeps rollouts bounded for parity.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass

import numpy as np

from . import config as _config
from ._capi import (BP_FEATURE_ABSOLUTE, BP_OP_LINEAR, BP_OP_RELU, BP_OP_SCALAR_AFFINE, BP_OP_SLICE,
                    BP_OP_SQDIST, BP_STOP_CUSTOM, BP_STOP_LAST_RELU)
from .objective import ObjectiveSpec, Op, P, U, X, op_id


class Rng:
    """The reference Rng stream (rng.hpp:12-35, rng.cpp:20-35) on the host, in Python.

    std::mt19937_64 (the C++ standard's parameters; the twist is vectorised with numpy
    uint64 arithmetic), uniform = (bits >> 11) * 2^-53, Box-Muller with a cached spare
    using the C library's log / sqrt / sin / cos (Python's math module) so every draw is
    the reference's bit for bit.  Fixture generation needs no GPU library: the bench's
    reference arm builds its fixtures through this class without loading the CUDA .so.
    """

    _N, _M = 312, 156
    _A = np.uint64(0xB5026F5AA96619E9)
    _UM, _LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, self._N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = np.array(mt, dtype=np.uint64)
        self.out = np.zeros(0, dtype=np.uint64)
        self.pos = 0
        self.spare = None

    def _twist(self):
        mt, N, M = self.mt, self._N, self._M
        one = np.uint64(1)

        def step(i0, i1, nxt, far):  # mt[i] = mt[i+M] ^ (y >> 1) ^ (y & 1) * A, y = hi(mt[i]) | lo(mt[i+1])
            y = (mt[i0:i1] & self._UM) | (nxt & self._LM)
            mt[i0:i1] = far ^ (y >> one) ^ ((y & one) * self._A)

        step(0, N - M, mt[1:N - M + 1].copy(), mt[M:N].copy())      # mt[i + M]: not yet updated
        step(N - M, N - 1, mt[N - M + 1:N].copy(), mt[0:M - 1].copy())  # mt[i + M - N]: updated above
        step(N - 1, N, mt[0:1].copy(), mt[M - 1:M].copy())
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.out = y
        self.pos = 0

    def bits(self, n: int) -> np.ndarray:
        parts = []
        while n > 0:
            if self.pos == self._N:
                self._twist()
            if self.out.size == 0:
                self._twist()
            take = min(n, self._N - self.pos)
            parts.append(self.out[self.pos:self.pos + take])
            self.pos += take
            n -= take
        return np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint64)

    def _uniform01(self, n: int) -> np.ndarray:
        return (self.bits(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53

    def uniform(self, n, lo=0.0, hi=1.0):
        return lo + (hi - lo) * self._uniform01(int(n))

    def normal(self, n):
        import math

        out = np.empty(int(n))
        for i in range(int(n)):
            if self.spare is not None:
                out[i], self.spare = self.spare, None
                continue
            u1 = self._uniform01(1)[0]
            while u1 <= 0.0:
                u1 = self._uniform01(1)[0]
            u2 = self._uniform01(1)[0]
            r = math.sqrt(-2.0 * math.log(u1))
            a = 6.283185307179586476925286766559 * u2
            self.spare = r * math.sin(a)
            out[i] = r * math.cos(a)
        return out


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def mlp_weights(widths, seed=0, glorot=False):
    r = Rng(seed)
    Ws, bs = [], []
    for i in range(len(widths) - 1):
        fin, fout = widths[i], widths[i + 1]
        if glorot:
            a = np.sqrt(6.0 / (fin + fout))
            Ws.append(f32(r.uniform(fin * fout, -a, a).reshape(fout, fin)))
            bs.append(f32(r.uniform(fout, -a, a)))
        else:
            Ws.append(f32(r.normal(fin * fout).reshape(fout, fin) * np.sqrt(2.0 / fin)))
            bs.append(np.zeros(fout))
    relu = [i + 2 < len(widths) for i in range(len(widths) - 1)]
    return Ws, bs, relu


@dataclass
class Workload:
    name: str
    spec: ObjectiveSpec
    samples_per_iter: int  # M
    children: int          # D (= 2 * batch)
    iterations: int        # BaB iterations
    split_rule: str = "samples"

    def planner_config(self, **over) -> dict:
        c = copy.deepcopy(_config.DEFAULTS)
        c["batch"] = max(1, self.children // 2)
        c["seed"] = 2
        c["split_rule"] = self.split_rule
        c["search"]["samples_per_iter"] = self.samples_per_iter
        c["termination"]["max_iterations"] = self.iterations
        for k, v in over.items():
            c[k] = v
        return c

    @property
    def flops_per_sample_step(self) -> int:
        w = self.spec.widths
        return 2 * sum(w[i] * w[i + 1] for i in range(len(w) - 1))

    @property
    def rows_per_search_iter(self) -> int:
        agents = 4
        return agents * (self.samples_per_iter // agents) + 1


def _spec(widths, ks, ka, H, ops, seed_w=0, glorot=False, stop_rule=BP_STOP_LAST_RELU, stops=(), x0=None):
    Ws, bs, relu = mlp_weights(widths, seed_w, glorot)
    r = Rng(1)
    x0 = f32(r.uniform(ks, -1.0, 1.0)) if x0 is None else f32(x0)
    return ObjectiveSpec(ks=ks, ka=ka, kd=ka, horizon=H, feature_mode=BP_FEATURE_ABSOLUTE, W=Ws, b=bs, relu=relu,
                         x0=x0, p0=np.zeros(ka), u_lower=-np.ones(ka), u_upper=np.ones(ka),
                         step_weight=np.ones(H), ops=ops, stop_rule=stop_rule, custom_stop_steps=list(stops))


def c1(glorot=False) -> Workload:
    """Tiny: [6,64,64,4], H=10, |x-g|^2 + 0.01|u|^2, M=256, D=64, 20 iterations, width split."""
    r = Rng(1)
    x0 = f32(r.uniform(4, -1, 1))
    g = f32(r.uniform(4, -1, 1))
    ops = [Op(BP_OP_SQDIST, X, target=g, weight=np.ones(4), weight_by_step=True, is_term=True),
           Op(BP_OP_SQDIST, U, target=np.zeros(2), weight=f32(np.full(2, 0.01)), is_term=True)]
    return Workload("C1-tiny", _spec([6, 64, 64, 4], 4, 2, 10, ops, glorot=glorot, x0=x0), 256, 64, 20, "width")


def c2(glorot=False) -> Workload:
    """Mid: [12,128,128,128,10], H=20, goal + 4 squared-radius obstacle ReLUs on x_t[0:2]."""
    r = Rng(1)
    x0 = f32(r.uniform(10, -1, 1))
    g = f32(r.uniform(10, -1, 1))
    ops = [Op(BP_OP_SQDIST, X, target=g, weight=np.ones(10), weight_by_step=True, is_term=True),
           Op(BP_OP_SLICE, X, begin=0, dim=2)]
    for _ in range(4):
        o = f32(r.uniform(2, -1, 1))
        rad = float(f32(r.uniform(1, 0.1, 0.3))[0])
        ops.append(Op(BP_OP_SQDIST, op_id(1), target=o, weight=np.ones(2)))
        ops.append(Op(BP_OP_SCALAR_AFFINE, op_id(len(ops) - 1), scale=-1.0, offset=float(np.float32(rad * rad))))
        ops.append(Op(BP_OP_RELU, op_id(len(ops) - 1), is_term=True))
    return Workload("C2-mid", _spec([12, 128, 128, 128, 10], 10, 2, 20, ops, glorot=glorot, x0=x0), 1024, 512, 50)


def c3(glorot=False) -> Workload:
    """Wide: [36,256,256,256,32], H=30, quadratic goal g ~ N(0,1)^32, M=4096, D=2048."""
    r = Rng(1)
    x0 = f32(r.uniform(32, -1, 1))
    g = f32(r.normal(32))
    ops = [Op(BP_OP_SQDIST, X, target=g, weight=np.ones(32), weight_by_step=True, is_term=True)]
    return Workload("C3-wide", _spec([36, 256, 256, 256, 32], 32, 4, 30, ops, glorot=glorot, x0=x0), 4096, 2048, 50)


def c4(glorot=False) -> Workload:
    """Long: [22,128,128,20], H=80, L1 goal + 10 relu(|x_t[0]| - 0.8), stops every 5 steps."""
    r = Rng(1)
    x0 = f32(r.uniform(20, -1, 1))
    g = f32(r.uniform(20, -1, 1))
    I = np.eye(20)
    e0 = np.zeros((2, 20))
    e0[0, 0], e0[1, 0] = 1.0, -1.0
    ops = [Op(BP_OP_LINEAR, X, dim=40, W=np.vstack([I, -I]), b=np.concatenate([-g, g])),
           Op(BP_OP_RELU, op_id(0)),
           Op(BP_OP_LINEAR, op_id(1), dim=1, W=np.ones((1, 40)), b=np.zeros(1), is_term=True),
           Op(BP_OP_LINEAR, X, dim=2, W=e0, b=np.zeros(2)),
           Op(BP_OP_RELU, op_id(3)),
           Op(BP_OP_LINEAR, op_id(4), dim=1, W=np.ones((1, 2)), b=f32([-0.8])),
           Op(BP_OP_RELU, op_id(5)),
           Op(BP_OP_SCALAR_AFFINE, op_id(6), scale=10.0, offset=0.0, is_term=True)]
    spec = _spec([22, 128, 128, 20], 20, 2, 80, ops, glorot=glorot, x0=x0, stop_rule=BP_STOP_CUSTOM,
                 stops=range(5, 81, 5))
    return Workload("C4-long", spec, 2048, 1024, 100)


def c5(D=1024, glorot=False) -> Workload:
    """Sweep: [20,512,512,16], H=40, quadratic; D pre-split boxes, one search + one bound pass."""
    r = Rng(1)
    x0 = f32(r.uniform(16, -1, 1))
    g = f32(r.uniform(16, -1, 1))
    ops = [Op(BP_OP_SQDIST, X, target=g, weight=np.ones(16), weight_by_step=True, is_term=True)]
    return Workload(f"C5-sweep-D{D}", _spec([20, 512, 512, 16], 16, 4, 40, ops, glorot=glorot, x0=x0), 1024, D, 1)


ALL = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def presplit_boxes(spec: ObjectiveSpec, n: int):
    """n leaves of recursive widest-axis bisection of the root box."""
    lo, hi = spec.box()
    boxes = [(lo.copy(), hi.copy())]
    while len(boxes) < n:
        nxt = []
        for l, h in boxes:
            j = int(np.argmax(h - l))
            m = 0.5 * (l[j] + h[j])
            a_hi, b_lo = h.copy(), l.copy()
            a_hi[j], b_lo[j] = m, m
            nxt += [(l, a_hi), (b_lo, h)]
        boxes = nxt
    boxes = boxes[:n]
    return np.array([b[0] for b in boxes]), np.array([b[1] for b in boxes])
