"""tcgen05 GEMM (K5/K7, csrc/gemm_tc.cu) throughput on the complexity-sweep
shapes, W tiles by TMA (default) vs cp.async (LAQ_GEMM_NO_TMA=1): device ms
(CUDA events, median of 5; prefuse = identity rows: A tiles by TMA too unless
LAQ_GEMM_NO_TMA_A=1), algorithmic TFLOP/s (2 m k n) and the tensor-pipe
rate (x3: the hi.hi + hi.lo + lo.hi fp16 split); results must be bit-identical."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08367_b200 import tc_ops  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    xs = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        xs.append(e0.elapsed_time(e1))
    return float(np.median(xs))


out = {}
g = torch.Generator(device="cuda")
g.manual_seed(5)
F = 1_000_000
for r, k, l in [(1_000_000, 1024, 4096), (1_000_000, 512, 1024), (100_000, 1024, 4096), (1_000_000, 128, 256)]:
    B = torch.rand((r, k), dtype=torch.float64, device="cuda", generator=g)
    fk = torch.randint(0, r, (F,), dtype=torch.int32, device="cuda", generator=g)
    W = torch.rand((k, l), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    feats = tc_ops.TCFeatures([B], [np.arange(k)], k)
    P = torch.empty((r, l), dtype=torch.float32, device="cuda")
    Y = torch.empty((F, l), dtype=torch.float32, device="cuda")
    cell = {}
    for name, env in (("tma", {}), ("tma_w_only", {"LAQ_GEMM_NO_TMA_A": "1"}), ("cp_async", {"LAQ_GEMM_NO_TMA": "1"})):
        for key in ("LAQ_GEMM_NO_TMA", "LAQ_GEMM_NO_TMA_A"):
            os.environ.pop(key, None)
        os.environ.update(env)
        ms_p = timed(lambda: feats.gemm(W, out=P))
        ms_n = timed(lambda: feats.gemm(W, row_maps=[fk], out=Y))
        cell[name] = {"prefuse_ms": round(ms_p, 3), "prefuse_alg_tflops": round(2 * r * k * l / ms_p / 1e9, 1),
                      "nonfused_ms": round(ms_n, 3), "nonfused_alg_tflops": round(2 * F * k * l / ms_n / 1e9, 1),
                      "nonfused_pipe_tflops": round(6 * F * k * l / ms_n / 1e9, 1),
                      "P_sum": float(P.double().sum()), "Y_sum": float(Y.double().sum())}
    for key in ("LAQ_GEMM_NO_TMA", "LAQ_GEMM_NO_TMA_A"):
        os.environ.pop(key, None)
    cell["bit_identical"] = all(cell[v]["P_sum"] == cell["cp_async"]["P_sum"] and
                                cell[v]["Y_sum"] == cell["cp_async"]["Y_sum"] for v in ("tma", "tma_w_only"))
    out[f"r={r} k={k} l={l}"] = cell
    print(json.dumps({f"r={r} k={k} l={l}": cell}), flush=True)
    del B, fk, W, feats, P, Y
    torch.cuda.empty_cache()
