"""Non-fused 2-layer FFN over a star join on the tensor cores (BASELINE configs[2]).

    Y = ReLU(T W1) W2,   T = materialize(I_j, B_j, placements)

The reference has no FFN model: configs[2] composes its pinned operators
materialize (laqops.cpp:338-374) and predict_linear (mlops.cpp:248-250) with an
elementwise ReLU.  Only layer 1 could be pushed through
the join (P_j = B_j W1_j); the cost model (fusion.cpp:199-208) rejects that for
k/l = 64/256, so the planner runs this non-fused operator, which never writes T:
tiles of T are gathered into shared memory and multiplied by tcgen05 MMAs
(csrc/ffn.cu).

Numerics: scaled fp16x2 split (hi.hi + hi.lo + lo.hi), fp32 accumulation, fp32 output; checked
condition-aware at 1e-5 against oracle.laq_oracle.ffn_predict.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import errors
from .device import context, dev, ptrs
from .fusion import _placements_arg

f64 = torch.float64


class StarFFN:
    """Feature tables (fp16x2 split, device layout) + W1/W2 bound once; __call__ runs
    join + FFN over fact keys (probe tables built once) or explicit row maps."""

    def __init__(self, dims, placements, W1, W2, dim_pks=None):
        self.ctx = ctx = context()
        B = [dev(d, f64) for d in dims]
        if len(B) == 0 or len(B) != len(placements):
            raise errors.ShapeError("ffn: dim/map list lengths")
        for b, p in zip(B, placements):
            if b.shape[1] != len(p):
                raise errors.ShapeError("ffn: column map does not fit dim table")
        W1d, W2d = dev(W1, f64), dev(W2, f64)
        k, h = W1d.shape
        if W2d.shape[0] != h:
            raise errors.ShapeError(f"ffn: W1 {k}x{h} then W2 {W2d.shape[0]}x{W2d.shape[1]}")
        self.k, self.h, self.l = int(k), int(h), int(W2d.shape[1])
        keep, plp = _placements_arg(placements)
        rows = (C.c_int64 * len(B))(*[b.shape[0] for b in B])
        cols = (C.c_int64 * len(B))(*[b.shape[1] for b in B])
        hdl = C.c_void_p()
        ctx.check(ctx.lib.laq_ffn_create(ctx.h, len(B), ptrs(B), rows, cols, C.cast(plp, C.c_void_p), self.k,
                                         W1d.data_ptr(), self.h, W2d.data_ptr(), self.l, C.byref(hdl)))
        self.hf = hdl
        self.n_dims = len(B)
        self.probe = None
        if dim_pks is not None:
            self.pks = [dev(p, torch.int32) for p in dim_pks]
            ph = C.c_void_p()
            prow = (C.c_int64 * len(self.pks))(*[p.numel() for p in self.pks])
            ctx.check(ctx.lib.laq_probe_build(ctx.h, len(self.pks), ptrs(self.pks), prow, C.byref(ph)))
            self.probe = ph

    def predict_rows(self, row_maps, out=None):
        """Y for explicit join row maps (one dim row per target row, int32)."""
        idx = [dev(r, torch.int32) for r in row_maps]
        n = idx[0].numel()
        if out is None:
            out = torch.empty((n, self.l), dtype=torch.float32, device="cuda")
        self.ctx.bind_stream()
        self.ctx.check(self.ctx.lib.laq_ffn_predict_rows(self.ctx.h, self.hf, ptrs(idx), n, out.data_ptr()))
        return out

    def __call__(self, fact_fks, out=None, survivors=None):
        """Join (probe tables) + FFN; returns (Y[:nnz], nnz) for surviving fact rows, ascending."""
        if self.probe is None:
            raise errors.ShapeError("ffn: built without dimension keys (use predict_rows)")
        fks = [dev(f, torch.int32) for f in fact_fks]
        n = fks[0].numel()
        if out is None:
            out = torch.empty((max(n, 1), self.l), dtype=torch.float32, device="cuda")
        nnz = C.c_int64()
        self.ctx.bind_stream()
        self.ctx.check(self.ctx.lib.laq_ffn_predict_star(
            self.ctx.h, self.hf, self.probe, ptrs(fks), n, out.data_ptr(),
            survivors.data_ptr() if survivors is not None else None, C.byref(nnz)))
        return out[:nnz.value], nnz.value

    def close(self):
        if getattr(self, "hf", None):
            self.ctx.lib.laq_ffn_destroy(self.hf)
            self.hf = None
        if getattr(self, "probe", None):
            self.ctx.lib.laq_probe_destroy(self.probe)
            self.probe = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cfg3_inputs(g, seed=42, feat=32, hidden=256, out=1):
    """SURVEY.md §8d cfg3 on a generated SSB star `g`: 32 fp64 unit() feature
    columns on customer and on part (derive_seed(seed, "customer_f"/"part_f")),
    W1 = gen_linear(64, 256, 11), W2 = gen_linear(256, 1, 12), no bias.
    Returns (fact fks [custkey, partkey], dim pks, dim features, placements, W1, W2)."""
    from . import gen
    t = g.tables
    cust, part = t["customer"], t["part"]
    fc = gen.unit_matrix(seed, "customer_f", len(cust["c_key"]), feat)
    fp = gen.unit_matrix(seed, "part_f", len(part["p_key"]), feat)
    W1 = gen.gen_linear(2 * feat, hidden, 11)
    W2 = gen.gen_linear(hidden, out, 12)
    fks = [g.fact["lo_customer"], g.fact["lo_part"]]
    pks = [cust["c_key"], part["p_key"]]
    placements = [np.arange(feat), np.arange(feat, 2 * feat)]
    return fks, pks, [fc, fp], placements, W1, W2
