"""Tensor-core (tcgen05, scaled fp16x2 split) forms of the dense contractions for the wide
shapes of the paper's complexity analysis (BASELINE configs[4]; csrc/gemm_tc.cu).

  prefuse_linear_tc      P_j = B_j (M_j L)                 fusion.cpp:31-36, 50-62
  apply_fused_linear_tc  Y = ((P_0[i_0] + P_1[i_1]) + ...)  fusion.cpp:64-77
  predict_nonfused_tc    Y = materialize(I_j, B_j) L         laqops.cpp:338-374 + mlops.cpp:248-250
                         (the gathered T never leaves shared memory)

fp32 outputs, fp16x2 split (3 MMAs per product) with fp32 accumulation: checked condition-aware at
1e-5 (|err| <= 1e-5 * (|T| |L|)) against the fp64 reference functions.  The
fp64 bit-exact forms (fusion.prefuse_linear / predict_linear) remain the
drop-in for the reference's own 1e-9 tests; the planner picks between the two
plans with the paper's cost model (fusion.plan_linear).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import errors
from .device import context, dev, ptrs
from .fusion import _placements_arg

f64 = torch.float64
f32 = torch.float32


class TCFeatures:
    """Dims' feature tables in the split block layout (laq_tc_features)."""

    def __init__(self, dims, placements, k: int):
        self.ctx = ctx = context()
        B = [dev(d, f64) for d in dims]
        if len(B) == 0 or len(B) != len(placements):
            raise errors.ShapeError("tc features: dim/map list lengths")
        for b, p in zip(B, placements):
            if b.shape[1] != len(p):
                raise errors.ShapeError("fusion: column map does not fit dim table")
        keep, plp = _placements_arg(placements)
        rows = (C.c_int64 * len(B))(*[b.shape[0] for b in B])
        cols = (C.c_int64 * len(B))(*[b.shape[1] for b in B])
        h = C.c_void_p()
        ctx.check(ctx.lib.laq_tc_features_create(ctx.h, len(B), ptrs(B), rows, cols, C.cast(plp, C.c_void_p), k,
                                                 C.byref(h)))
        self.h = h
        self.k = k
        self.n_dims = len(B)
        self.rows = [int(b.shape[0]) for b in B]

    def gemm(self, W, row_maps=None, m=None, out=None):
        ctx = self.ctx
        Wd = dev(W, f64)
        if Wd.shape[0] != self.k:
            raise errors.ShapeError(f"dense_matmul: T has {self.k} columns, W has {Wd.shape[0]} rows")
        n = int(Wd.shape[1])
        if row_maps is None:
            m = self.rows[0]
            rp = None
        else:
            idx = [dev(r, torch.int32) for r in row_maps]
            m = int(idx[0].numel())
            rp = ptrs(idx)
        if out is None:
            out = torch.empty((m, n), dtype=f32, device="cuda")
        ctx.bind_stream()
        ctx.check(ctx.lib.laq_tc_gemm(ctx.h, self.h, rp, m, Wd.data_ptr(), n, out.data_ptr()))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.laq_tc_features_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_placements(placements, k):
    """fusion.cpp:11-25: placements tile [0, k) exactly."""
    seen = np.zeros(k, bool)
    total = 0
    for p in placements:
        for t in np.asarray(p, np.int64):
            if t < 0 or t >= k:
                raise errors.MappingError(f"column map: target index {t} out of range")
            if seen[t]:
                raise errors.MappingError(f"fusion: overlapping target column {t}")
            seen[t] = True
            total += 1
    if total != k:
        raise errors.ShapeError(f"fusion: placements claim {total} of {k} feature columns")


def prefuse_linear_tc(dims, placements, L):
    """P_j = B_j (M_j L) per dim on the tensor cores; fp32 device tensors."""
    Ld = dev(L, f64)
    k = int(Ld.shape[0])
    _check_placements(placements, k)
    parts = []
    for d, p in zip(dims, placements):
        f = TCFeatures([d], [p], k)
        parts.append(f.gemm(Ld))
        f.close()
    return parts


def apply_fused_linear_tc(i_maps, partials):
    """Y = ((P_0[i_0] + P_1[i_1]) + ...), fp32 partials and output."""
    ctx = context()
    idx = [dev(i, torch.int32) for i in i_maps]
    P = [dev(p, f32) for p in partials]
    if len(idx) == 0 or len(idx) != len(P):
        raise errors.ShapeError("apply_fused_linear: map/partial list lengths")
    rows, l = int(idx[0].numel()), int(P[0].shape[1])
    out = torch.empty((rows, l), dtype=f32, device="cuda")
    ctx.bind_stream()
    ctx.check(ctx.lib.laq_apply_fused_linear_f32(ctx.h, len(idx), ptrs(idx), rows, ptrs(P), l, out.data_ptr()))
    return out


def predict_nonfused_tc(i_maps, dims, placements, L, features: TCFeatures | None = None):
    """Y = materialize(I_j, B_j, placements) L with T gathered tile by tile."""
    Ld = dev(L, f64)
    k = int(Ld.shape[0])
    f = features or TCFeatures(dims, placements, k)
    try:
        return f.gemm(Ld, row_maps=i_maps)
    finally:
        if features is None:
            f.close()



def predict_star_linear(i_maps, dims, placements, L, planner: str = "device", threshold: float = 1.0,
                        features: TCFeatures | None = None, plan: str | None = None):
    """The planner-driven linear predict over a star join on the tensor cores:
    the plan (fused: prefuse P_j = B_j (M_j L) + gather-apply; non-fused: one
    GEMM over the gathered rows) is CHOSEN by a cost model, as the paper
    prescribes (fusion.cpp:199-224 decide_fusion; cli.cpp:648-652 leaves the
    choice to the user):

      planner="device": laq_plan_linear_device (the B200 roofline model);
      planner="paper":  speedup_ratio_linear (Eq. 2) + decide_fusion(threshold);
      plan="fused"|"nonfused" forces one.

    Returns (Y [rows x l] fp32 device tensor, the plan taken)."""
    from . import fusion
    Ld = dev(L, f64)
    k, l = int(Ld.shape[0]), int(Ld.shape[1])
    rows = int(len(i_maps[0])) if len(i_maps) else 0
    dim_rows = [int(d.shape[0]) for d in dims]
    if plan is None:
        if planner == "device":
            fused = fusion.device_plan_costs_abi(rows, k, l, dim_rows)[2]
        elif planner == "paper":
            r = fusion.speedup_ratio_linear(fusion.CostInputs(rows, k, l, k, dim_rows))
            fused = fusion.decide_fusion(r, threshold)
        else:
            raise errors.ShapeError(f"unknown planner {planner!r}")
        plan = "fused" if fused else "nonfused"
    if plan == "fused":
        return apply_fused_linear_tc(i_maps, prefuse_linear_tc(dims, placements, Ld)), plan
    if plan == "nonfused":
        return predict_nonfused_tc(i_maps, dims, placements, Ld, features), plan
    raise errors.ShapeError(f"unknown plan {plan!r}")
