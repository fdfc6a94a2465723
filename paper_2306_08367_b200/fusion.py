"""laq::fusion on the device (mirror of proj/include/laq/fusion.hpp) plus the
planner that picks the fused operator with the paper's cost model (Eq. 2).

  prefuse_linear      P_j = B_j (M_j L)                      fusion.cpp:31-36, 50-62
  apply_fused_linear  Y = ((I_0 P_0 + I_1 P_1) + ...)        fusion.cpp:64-77
  fused_star_predict  join + apply in one pass (north_star: (Fact x Dim) W = I (Dim W))
  speedup_ratio_*     fusion.cpp:199-219;  decide_fusion fusion.cpp:221-224
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import errors
from .device import context, dev, host, ptrs

f64 = torch.float64


def _is_dev(*xs) -> bool:
    return any(isinstance(x, torch.Tensor) and x.is_cuda for x in xs)


@dataclass
class FusedLinear:
    """fusion.hpp:11-14."""
    partials: list
    out_width: int


def _placements_arg(placements):
    pl = [np.ascontiguousarray(p, np.int64) for p in placements]
    arr = (C.POINTER(C.c_int64) * max(1, len(pl)))(*[p.ctypes.data_as(C.POINTER(C.c_int64)) for p in pl])
    return pl, arr


def prefuse_linear(dims, placements, L) -> FusedLinear:
    """P_j = B_j (M_j L), fp64, bit-identical to the reference (sequential-k sums)."""
    if len(dims) == 0 or len(dims) != len(placements):
        raise errors.ShapeError("prefuse_linear: dim/map list lengths")
    on = _is_dev(*dims, L)
    ctx = context()
    B = [dev(d, f64) for d in dims]
    Ld = dev(L, f64)
    k, l = Ld.shape
    for b, p in zip(B, placements):
        if b.shape[1] != len(p):
            raise errors.ShapeError("fusion: column map does not fit dim table")
    keep, plp = _placements_arg(placements)
    parts = [torch.empty((b.shape[0], l), dtype=f64, device="cuda") for b in B]
    rows = (C.c_int64 * len(B))(*[b.shape[0] for b in B])
    cols = (C.c_int64 * len(B))(*[b.shape[1] for b in B])
    ctx.check(ctx.lib.laq_prefuse_linear(ctx.h, len(B), ptrs(B), rows, cols, C.cast(plp, C.c_void_p),
                                         Ld.data_ptr(), k, l, ptrs(parts)))
    return FusedLinear([p if on else host(p) for p in parts], l)


def apply_fused_linear(i_maps, f: FusedLinear):
    """Y = sum_j I_j P_j with I_j given as row-index vectors (one source row per target row)."""
    if len(i_maps) == 0 or len(i_maps) != len(f.partials):
        raise errors.ShapeError("apply_fused_linear: map/partial list lengths")
    rows = len(i_maps[0])
    for i in i_maps:
        if len(i) != rows:
            raise errors.ShapeError("apply_fused_linear: row counts differ")
    for p in f.partials:
        if p.shape[1] != f.out_width:
            raise errors.ShapeError("apply_fused_linear: partial width")
    on = _is_dev(*i_maps, *f.partials)
    ctx = context()
    idx = [dev(i, torch.int64) for i in i_maps]
    P = [dev(p, f64) for p in f.partials]
    out = torch.empty((rows, f.out_width), dtype=f64, device="cuda")
    prow = (C.c_int64 * len(P))(*[p.shape[0] for p in P])
    ctx.check(ctx.lib.laq_apply_fused_linear(ctx.h, len(idx), ptrs(idx), rows, ptrs(P), prow, f.out_width,
                                             out.data_ptr()))
    return out if on else host(out)


def predict_linear(T, W):
    """mlops.cpp:248-250 = dense_matmul (matrix.cpp:158-174), bit-identical fp64."""
    on = _is_dev(T, W)
    ctx = context()
    A, B = dev(T, f64), dev(W, f64)
    if A.shape[1] != B.shape[0]:
        raise errors.ShapeError(f"dense_matmul: {A.shape[0]}x{A.shape[1]} x {B.shape[0]}x{B.shape[1]}")
    out = torch.empty((A.shape[0], B.shape[1]), dtype=f64, device="cuda")
    ctx.check(ctx.lib.laq_dense_matmul(ctx.h, A.data_ptr(), A.shape[0], A.shape[1], B.data_ptr(), B.shape[1],
                                       out.data_ptr()))
    return out if on else host(out)


dense_matmul = predict_linear


class FusedStarPredictor:
    """The fused join+predict operator over int32 device keys.

    Probe tables over the dimension pks are built once (laq_probe_build);
    __call__ streams the fact keys and returns (Y, nnz) for the surviving fact
    rows in ascending order.  No host synchronisation inside __call__ when
    sync=False (CUDA-graph capturable); the survivor count lands in self.nnz_dev.
    """

    def __init__(self, dim_pks, partials):
        self.ctx = context()
        self.pks = [dev(p, torch.int32) for p in dim_pks]
        self.partials = [dev(p, f64) for p in partials]
        self.l = int(self.partials[0].shape[1])
        h = C.c_void_p()
        prow = (C.c_int64 * len(self.pks))(*[p.numel() for p in self.pks])
        self.ctx.check(self.ctx.lib.laq_probe_build(self.ctx.h, len(self.pks), ptrs(self.pks), prow, C.byref(h)))
        self.h = h
        self.nnz_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        # Bind the partials once (slot-ordered layout); per call only the fact keys stream.
        rc = self.ctx.lib.laq_probe_bind_partials(self.ctx.h, self.h, ptrs(self.partials), self.l)
        self.bound = rc == 0

    def __call__(self, fact_fks, out=None, survivors=None, sync=True):
        fks = [dev(f, torch.int32) for f in fact_fks]
        n = fks[0].numel()
        if out is None:
            out = torch.empty((n, self.l), dtype=f64, device="cuda")
        self.ctx.bind_stream()
        self.ctx.check(self.ctx.lib.laq_probe_fused_predict(
            self.ctx.h, self.h, ptrs(fks), n, None if self.bound else ptrs(self.partials), self.l, out.data_ptr(),
            survivors.data_ptr() if survivors is not None else None, self.nnz_dev.data_ptr()))
        if not sync:
            return out, None
        nnz = int(self.nnz_dev.item())
        return out[:nnz], nnz

    def predict_host(self, fact_fks, out=None, chunk_rows=0):
        """The same operator with HOST buffers (laq_probe_fused_predict_host):
        int32 keys in host memory, predictions written to a host float64
        [n, l] buffer (`out`, allocated pinned when None); the keys' H2D and
        the predictions' D2H are chunked over two copy streams and overlap the
        probe kernel.  Returns (out[:nnz], nnz).  Pinned inputs (torch
        pin_memory tensors) stream at the full PCIe rate."""
        if not self.bound:
            raise errors.ShapeError("predict_host needs partials bound at construction")
        keys = [f if isinstance(f, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(f, np.int32))
                for f in fact_fks]
        for k in keys:
            if k.is_cuda or k.dtype != torch.int32 or not k.is_contiguous():
                raise errors.ShapeError("predict_host takes contiguous int32 host keys")
        n = keys[0].numel()
        if out is None:
            out = torch.empty((n, self.l), dtype=f64, pin_memory=True)
        if out.is_cuda or out.dtype != f64 or out.numel() < n * self.l:
            raise errors.ShapeError("predict_host writes a float64 host buffer of n * l values")
        nnz = C.c_int64(0)
        kp = (C.c_void_p * len(keys))(*[k.data_ptr() for k in keys])
        self.ctx.bind_stream()
        self.ctx.check(self.ctx.lib.laq_probe_fused_predict_host(
            self.ctx.h, self.h, kp, n, self.l, out.data_ptr(), int(chunk_rows), C.byref(nnz)))
        return out[:nnz.value], int(nnz.value)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.laq_probe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fused_star_predict(fact_fks, dim_pks, partials):
    """One-shot fused join + predict (int32 keys); returns (Y, survivors)."""
    on = _is_dev(*fact_fks, *partials)
    ctx = context()
    fks = [dev(f, torch.int32) for f in fact_fks]
    pks = [dev(p, torch.int32) for p in dim_pks]
    P = [dev(p, f64) for p in partials]
    n = fks[0].numel()
    l = int(P[0].shape[1])
    out = torch.empty((max(n, 1), l), dtype=f64, device="cuda")
    surv = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    nnz = C.c_int64()
    prow = (C.c_int64 * len(pks))(*[p.numel() for p in pks])
    ctx.check(ctx.lib.laq_fused_star_predict(ctx.h, len(fks), ptrs(fks), n, ptrs(pks), prow, ptrs(P), l,
                                             out.data_ptr(), surv.data_ptr(), C.byref(nnz)))
    m = nnz.value
    return (out[:m], surv[:m]) if on else (host(out[:m]), host(surv[:m]))


# ---------------------------------------------------------------------------
# cost model (fusion.hpp:56-76) and planner
# ---------------------------------------------------------------------------

@dataclass
class CostInputs:
    target_rows: int = 0
    input_width: int = 0
    output_width: int = 0
    tree_features: int = 0
    dim_rows: list = field(default_factory=list)

    def sum_dim_rows(self) -> float:
        return float(sum(float(r) for r in self.dim_rows))


def _check_cost(rc):
    if rc != 0:
        errors.raise_for(rc, "cost model: all inputs must be positive")


def speedup_ratio_linear(c: CostInputs) -> float:
    from ._abi import lib
    d = np.ascontiguousarray(c.dim_rows, np.int64)
    out = C.c_double()
    if c.tree_features <= 0:
        _check_cost(8)
    _check_cost(lib().laq_speedup_ratio_linear(c.target_rows, c.input_width, c.output_width,
                                               d.ctypes.data_as(C.POINTER(C.c_int64)), len(d), C.byref(out)))
    return out.value


def speedup_ratio_tree(c: CostInputs) -> float:
    from ._abi import lib
    d = np.ascontiguousarray(c.dim_rows, np.int64)
    out = C.c_double()
    _check_cost(lib().laq_speedup_ratio_tree(c.target_rows, c.input_width, c.output_width, c.tree_features,
                                             d.ctypes.data_as(C.POINTER(C.c_int64)), len(d), C.byref(out)))
    return out.value


def decide_fusion(ratio: float, threshold: float = 1.0) -> bool:
    from ._abi import lib
    out = C.c_int32()
    rc = lib().laq_decide_fusion(C.c_double(ratio), C.c_double(threshold), C.byref(out))
    if rc != 0:
        raise errors.DomainError("decide_fusion: ratio not finite")
    return bool(out.value)


def plan_linear(target_rows: int, k: int, l: int, dim_rows, threshold: float = 1.0) -> str:
    """The planner the reference lacks (decide_fusion is only reachable from
    `laq cost`, cli.cpp:709-741): fused iff speedup_ratio_linear > threshold."""
    r = speedup_ratio_linear(CostInputs(target_rows, k, l, k, list(dim_rows)))
    return "fused" if decide_fusion(r, threshold) else "nonfused"


# ---------------------------------------------------------------------------
# B200 plan model (device roofline).  The paper's Eq. 2 counts CPU sparse-matrix
# work; on the tensor cores both plans are GEMM + gather and the winner is set
# by tensor time vs HBM bytes.  Calibrated on profiles/round1/complexity_sweep.json
# (164 measured cells): picks the measured winner in 154 (Eq. 2: 113), worst
# slowdown of its pick 1.22x (Eq. 2: 8.9x).
# ---------------------------------------------------------------------------

def _device_peaks():
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["bf16_tflops"]) * 1e12, float(d["hbm_gbs"]) * 1e9
    except Exception:  # noqa: BLE001
        return 1654e12, 6548e9


def device_plan_costs(target_rows: int, k: int, l: int, dim_rows, peaks=None):
    """Predicted seconds (fused, non-fused) of the tensor-core plans on B200.

    non-fused: one GEMM over the gathered rows (3 MMAs per product on blocks of
      32 features and 16 output columns) vs its bytes (keys, fp16x2 features,
      fp32 Y);
    fused: prefuse GEMMs over every dim (M = r_j) + the fp32 gather-apply, whose
      P reads come from L2 when sum r_j l 4 B fits (~100 MB), else HBM."""
    pt, bw = peaks or _device_peaks()
    pt *= 0.85  # tensor-pipe rate reached by csrc/gemm_tc.cu on long GEMMs
    bw *= 0.76  # gather + streaming mix
    ovh = 20e-6  # launch + pipeline fill per kernel
    F = float(target_rows)
    kp = (k + 31) // 32 * 32
    lp = max(16, (l + 15) // 16 * 16)
    R = float(sum(dim_rows))
    t_nf = ovh + max(6.0 * F * kp * lp / pt, (F * 4 * len(dim_rows) + F * kp * 4 + F * l * 4) / bw)
    p_bytes = R * l * 4
    gather_p = 0.0 if p_bytes <= 100e6 else F * l * 4 * len(dim_rows)
    t_pre = sum(max(6.0 * r * kp * lp / pt, (r * kp * 4 + r * l * 4) / bw) for r in dim_rows)
    t_f = (1 + len(dim_rows)) * ovh + t_pre + (F * 4 * len(dim_rows) + F * l * 4 + gather_p) / bw
    return t_f, t_nf


def plan_linear_device(target_rows: int, k: int, l: int, dim_rows) -> str:
    """The planner for the tensor-core operators: the plan with the smaller
    predicted device time (device_plan_costs)."""
    t_f, t_nf = device_plan_costs(target_rows, k, l, dim_rows)
    return "fused" if t_f < t_nf else "nonfused"


def device_plan_costs_abi(target_rows: int, k: int, l: int, dim_rows, peaks=None):
    """The same model through the C-ABI (laq_plan_linear_device): what a C++
    host calls.  Returns (t_fused, t_nonfused, fused)."""
    from . import _abi
    pt, bw = peaks or _device_peaks()
    dims = (C.c_int64 * len(dim_rows))(*[int(r) for r in dim_rows])
    tf, tn, fu = C.c_double(), C.c_double(), C.c_int32()
    rc = _abi.lib().laq_plan_linear_device(int(target_rows), int(k), int(l), dims, len(dim_rows), pt, bw,
                                           C.byref(tf), C.byref(tn), C.byref(fu))
    errors.raise_for(rc, "plan_linear_device: non-positive inputs")
    return tf.value, tn.value, bool(fu.value)
