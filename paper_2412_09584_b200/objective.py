"""Objective descriptor: the unrolled-rollout objective the device evaluates,
bounds and searches (bp_objective_desc in include/babplan_cuda.h).

`build_objective(model, scenario)` restates the reference's build_objective
(src/model.cpp:310-387): per step t the cost program is
  SquaredDistance(x_t, x_target, w_t * axis)                       (model.cpp:358-359)
  + for each obstacle: PenaltyHinge(Slice(x_t, k*kd, kd)) per keypoint
    (tracking_obstacles) and PenaltyHinge(p_t)                     (model.cpp:360-370)
in exactly the node order the reference creates, so the oracle's graph built
from the same descriptor has the reference's node ids.  Other cost programs
(the BASELINE.json configs) use the same op vocabulary.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import (BP_FEATURE_ABSOLUTE, BP_FEATURE_NETWORK, BP_FEATURE_RELATIVE, BP_OP_HINGE, BP_OP_LINEAR, BP_OP_RELU,
                    BP_OP_SCALAR_AFFINE, BP_OP_SLICE, BP_OP_SQDIST, BP_OP_SUM, BP_STOP_CUSTOM,
                    BP_STOP_LAST_RELU, BP_VAL_OP0, BP_VAL_P, BP_VAL_U, BP_VAL_X)

X, U, P = BP_VAL_X, BP_VAL_U, BP_VAL_P


@dataclass
class Op:
    kind: int
    src0: int
    src1: int = -1
    dim: int = 0
    begin: int = 0
    W: Optional[np.ndarray] = None
    b: Optional[np.ndarray] = None
    scale: float = 1.0
    offset: float = 0.0
    target: Optional[np.ndarray] = None
    weight: Optional[np.ndarray] = None
    weight_by_step: bool = False
    center: Optional[np.ndarray] = None
    radius: float = 0.0
    penalty: float = 1.0
    is_term: bool = False


def op_id(i: int) -> int:
    """Value id of the output of cost op i."""
    return BP_VAL_OP0 + i


@dataclass
class ObjectiveSpec:
    ks: int
    ka: int
    kd: int
    horizon: int
    feature_mode: int
    W: List[np.ndarray]
    b: List[np.ndarray]
    relu: List[bool]
    x0: np.ndarray
    p0: np.ndarray
    u_lower: np.ndarray
    u_upper: np.ndarray
    step_weight: np.ndarray
    ops: List[Op]
    stop_rule: int = BP_STOP_LAST_RELU
    custom_stop_steps: List[int] = field(default_factory=list)

    @property
    def d(self) -> int:
        return self.ka * self.horizon

    @property
    def widths(self) -> List[int]:
        return [self.W[0].shape[1]] + [w.shape[0] for w in self.W]

    def box(self):
        lo = np.tile(self.u_lower, self.horizon)
        hi = np.tile(self.u_upper, self.horizon)
        return lo, hi

    def value_dims(self) -> List[int]:
        dims = [self.ks, self.ka, self.kd]
        for op in self.ops:
            src = dims[op.src0]
            if op.kind in (BP_OP_RELU, BP_OP_SUM, BP_OP_SCALAR_AFFINE):
                dims.append(src)
            elif op.kind in (BP_OP_SQDIST, BP_OP_HINGE):
                dims.append(1)
            else:
                dims.append(op.dim)
        return dims

    def to_c(self) -> "PackedObjective":
        return PackedObjective(self)


class PackedObjective:
    """Owns the numpy buffers behind a ctypes bp_objective_desc."""

    def __init__(self, s: ObjectiveSpec):
        keep = []

        def dp(a):
            if a is None:
                return None
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
            keep.append(a)
            return _capi.dptr(a)

        L = len(s.W)
        widths = np.asarray(s.widths, dtype=np.int32)
        relu = np.asarray([1 if r else 0 for r in s.relu], dtype=np.int32)
        keep += [widths, relu]
        Wp = (C.POINTER(C.c_double) * L)(*[dp(w) for w in s.W])
        bp = (C.POINTER(C.c_double) * L)(*[dp(b) for b in s.b])
        dims = s.value_dims()
        ops = (_capi.CostOp * max(1, len(s.ops)))()
        for i, op in enumerate(s.ops):
            c = ops[i]
            c.kind, c.src0, c.src1 = op.kind, op.src0, op.src1
            c.in_dim = dims[op.src0]
            c.dim = dims[BP_VAL_OP0 + i]
            c.begin = op.begin
            c.W, c.b = dp(op.W), dp(op.b)
            c.scale, c.offset = float(op.scale), float(op.offset)
            c.target, c.weight = dp(op.target), dp(op.weight)
            c.weight_by_step = 1 if op.weight_by_step else 0
            c.center = dp(op.center)
            c.radius, c.penalty = float(op.radius), float(op.penalty)
            c.is_term = 1 if op.is_term else 0
        stops = np.asarray(s.custom_stop_steps or [0], dtype=np.int32)
        keep.append(stops)
        self.desc = _capi.ObjectiveDesc(
            ks=s.ks, ka=s.ka, kd=s.kd, horizon=s.horizon, feature_mode=s.feature_mode, n_layers=L,
            widths=_capi.iptr(widths), W=Wp, b=bp, relu_after=_capi.iptr(relu),
            x0=dp(s.x0), p0=dp(s.p0), u_lower=dp(s.u_lower), u_upper=dp(s.u_upper),
            step_weight=dp(s.step_weight), n_ops=len(s.ops), ops=ops, stop_rule=s.stop_rule,
            n_custom_stops=len(s.custom_stop_steps), custom_stop_steps=_capi.iptr(stops))
        self._keep = (keep, Wp, bp, ops)

    def ref(self):
        return C.byref(self.desc)


def build_objective(model, s) -> ObjectiveSpec:
    """build_objective (model.cpp:310-387) for a Model and a Scenario."""
    s.validate()
    ks, ka, kd, H = s.state_dim(), s.action_dim(), s.workspace_dim(), s.horizon
    if model.input_dim != ks + ka:
        raise ValueError("build_objective: model input must take state plus action")
    if model.output_dim != ks:
        raise ValueError("build_objective: model output must be the state")
    axis = s.axis_weights if s.axis_weights.size else np.ones(ks)
    ops = [Op(BP_OP_SQDIST, X, target=s.x_target, weight=axis, weight_by_step=True, is_term=True)]
    if s.cost_form != "tracking":
        for o in s.obstacles:
            if s.cost_form == "tracking_obstacles":
                for k in range(s.keypoints()):
                    ops.append(Op(BP_OP_SLICE, X, begin=k * kd, dim=kd))
                    ops.append(Op(BP_OP_HINGE, op_id(len(ops) - 1), center=o.center, radius=o.size,
                                  penalty=s.lam, is_term=True))
            ops.append(Op(BP_OP_HINGE, P, center=o.center, radius=o.size, penalty=s.lam, is_term=True))
    return ObjectiveSpec(
        ks=ks, ka=ka, kd=kd, horizon=H,
        feature_mode=BP_FEATURE_RELATIVE if s.feature_mode == "relative" else BP_FEATURE_ABSOLUTE,
        W=list(model.W), b=list(model.b), relu=list(model.relu), x0=s.x0, p0=s.p0,
        u_lower=s.u_lower, u_upper=s.u_upper,
        step_weight=np.array([s.tracking_weight(t) for t in range(1, H + 1)]), ops=ops)


def build_network_objective(model, lower, upper) -> ObjectiveSpec:
    """build_network_objective (model.cpp:389-405): the bare network over an input box,
    its scalar output the objective -- one step, the MLP reads the box only."""
    if model.output_dim != 1:
        raise ValueError("build_network_objective: network output must be scalar")
    lo = np.asarray(lower, dtype=np.float64).reshape(-1)
    hi = np.asarray(upper, dtype=np.float64).reshape(-1)
    if lo.size != model.input_dim or hi.size != model.input_dim:
        raise ValueError("lower_bound: box dim mismatch")
    n = model.input_dim
    return ObjectiveSpec(ks=1, ka=n, kd=n, horizon=1, feature_mode=BP_FEATURE_NETWORK,
                         W=list(model.W), b=list(model.b), relu=list(model.relu), x0=np.zeros(1), p0=np.zeros(n),
                         u_lower=lo, u_upper=hi, step_weight=np.ones(1), ops=[Op(BP_OP_SUM, X, dim=1, is_term=True)])


def round_spec_to_f32(spec: ObjectiveSpec) -> ObjectiveSpec:
    """Same objective with every parameter rounded to FP32, so the FP64 oracle
    and the FP32 device evaluate identical inputs."""
    f = lambda a: None if a is None else np.asarray(a, dtype=np.float32).astype(np.float64)
    ops = []
    for op in spec.ops:
        ops.append(Op(op.kind, op.src0, op.src1, op.dim, op.begin, f(op.W), f(op.b),
                      float(np.float32(op.scale)), float(np.float32(op.offset)), f(op.target), f(op.weight),
                      op.weight_by_step, f(op.center), float(np.float32(op.radius)),
                      float(np.float32(op.penalty)), op.is_term))
    return ObjectiveSpec(spec.ks, spec.ka, spec.kd, spec.horizon, spec.feature_mode,
                         [f(w) for w in spec.W], [f(b) for b in spec.b], list(spec.relu), f(spec.x0), f(spec.p0),
                         f(spec.u_lower), f(spec.u_upper), f(spec.step_weight), ops, spec.stop_rule,
                         list(spec.custom_stop_steps))
