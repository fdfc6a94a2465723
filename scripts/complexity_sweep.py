"""BASELINE configs[4]: the paper's complexity sweep on one B200 -- fused (pushdown:
prefuse P = B L, then Y = I P) vs non-fused (Y = (I B) L, T gathered inside the
GEMM) over dim cardinality r x feature width k x model width l, F = 1e6 fact rows,
one dimension, uniform foreign keys.

For every cell: device time of both plans (CUDA events, median of 3 after a
warm-up), the cost model's ratio (speedup_ratio_linear, fusion.cpp:199-208, the
paper's Eq. 2) and decision (decide_fusion, threshold 1), and whether the
decision picked the measured winner.  Cells whose P (r l 4 B), B (r k 8 B) or Y
(F l 4 B) exceed 64 GB are skipped as CapacityError, as the survey specifies.
A 512-row sample of every cell is checked against an fp64 product (cond-aware 1e-5).

usage: python scripts/complexity_sweep.py [out.json] [--quick | --holdout]

--holdout: a grid disjoint from the one the B200 planner's constants were
fitted on (r in 3e3..3e6, k in 16/64/256, l in 2..2048): an out-of-sample check
of fusion.plan_linear_device (constants unchanged).
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08367_b200 import fusion, tc_ops  # noqa: E402

F = 1_000_000
R = [1_000, 10_000, 100_000, 1_000_000, 10_000_000]
K = [8, 32, 128, 512, 1024]
L = [1, 4, 16, 64, 256, 1024, 4096]
CAP = 64 << 30
if "--quick" in sys.argv:
    R, K, L = [1_000, 100_000], [8, 128], [1, 64, 1024]
if "--holdout" in sys.argv:
    R, K, L = [3_000, 30_000, 300_000, 3_000_000], [16, 64, 256], [2, 8, 32, 128, 512, 2048]
out_path = next((a for a in sys.argv[1:] if a.endswith(".json")), "gpurun_out/complexity_sweep.json")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


gen = torch.Generator(device="cuda")
rows = []
t_start = time.time()
for r in R:
    for k in K:
        if r * k * 8 > CAP:
            for l in L:
                rows.append({"r": r, "k": k, "l": l, "skipped": "CapacityError: B"})
            continue
        gen.manual_seed(r * 7919 + k)
        B = torch.rand((r, k), dtype=torch.float64, device="cuda", generator=gen)
        fk = torch.randint(0, r, (F,), dtype=torch.int32, device="cuda", generator=gen)
        feats = tc_ops.TCFeatures([B], [np.arange(k)], k)
        sample = torch.arange(0, F, F // 512, device="cuda")[:512]
        for l in L:
            cell = {"r": r, "k": k, "l": l}
            if r * l * 4 > CAP or F * l * 4 > CAP:
                cell["skipped"] = "CapacityError: P or Y"
                rows.append(cell)
                continue
            W = torch.rand((k, l), dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
            P = torch.empty((r, l), dtype=torch.float32, device="cuda")
            Y = torch.empty((F, l), dtype=torch.float32, device="cuda")

            def fused():
                feats.gemm(W, out=P)
                return tc_ops.apply_fused_linear_tc([fk], [P])

            def nonfused():
                return feats.gemm(W, row_maps=[fk], out=Y)

            cell["ms_prefuse"] = timed(lambda: feats.gemm(W, out=P))
            cell["ms_fused"] = timed(fused)
            cell["ms_nonfused"] = timed(nonfused)
            # accuracy on a row sample, both plans vs an fp64 product
            T = B[fk[sample].long()]
            ref = (T @ W).cpu().numpy()
            bound = (T.abs() @ W.abs()).cpu().numpy()
            yf = fused()[sample].double().cpu().numpy()
            yn = nonfused()[sample].double().cpu().numpy()
            cell["cond_err_fused"] = float(np.max(np.abs(yf - ref) / np.maximum(bound, 1e-300)))
            cell["cond_err_nonfused"] = float(np.max(np.abs(yn - ref) / np.maximum(bound, 1e-300)))
            ratio = fusion.speedup_ratio_linear(fusion.CostInputs(F, k, l, k, [r]))
            cell["cost_ratio"] = ratio
            cell["planner"] = "fused" if fusion.decide_fusion(ratio, 1.0) else "nonfused"
            cell["measured_winner"] = "fused" if cell["ms_fused"] < cell["ms_nonfused"] else "nonfused"
            cell["planner_right"] = cell["planner"] == cell["measured_winner"]
            cell["device_planner"] = fusion.plan_linear_device(F, k, l, [r])
            pick = cell["ms_fused"] if cell["device_planner"] == "fused" else cell["ms_nonfused"]
            cell["device_planner_slowdown"] = pick / min(cell["ms_fused"], cell["ms_nonfused"])
            pick = cell["ms_fused"] if cell["planner"] == "fused" else cell["ms_nonfused"]
            cell["planner_slowdown"] = pick / min(cell["ms_fused"], cell["ms_nonfused"])
            flop = 2.0 * F * k * l
            cell["nonfused_alg_tflops"] = flop / (cell["ms_nonfused"] / 1e3) / 1e12
            cell["prefuse_alg_tflops"] = 2.0 * r * k * l / (cell["ms_prefuse"] / 1e3) / 1e12
            rows.append(cell)
            print(json.dumps(cell), flush=True)
            del P, Y, W
        feats.close()
        del B, fk
        torch.cuda.empty_cache()

done = [c for c in rows if "skipped" not in c]
summary = {
    "cells": len(rows), "measured": len(done), "skipped": len(rows) - len(done),
    "planner_agrees_with_measurement": sum(c["planner_right"] for c in done),
    "device_planner_agrees": sum(c["device_planner"] == c["measured_winner"] for c in done),
    "device_planner_max_slowdown": max([c["device_planner_slowdown"] for c in done], default=1.0),
    "planner_max_slowdown": max([c["planner_slowdown"] for c in done], default=1.0),
    "grid": {"r": R, "k": K, "l": L, "F": F},
    "max_cond_err": max([max(c["cond_err_fused"], c["cond_err_nonfused"]) for c in done], default=0.0),
    "best_nonfused_alg_tflops": max([c["nonfused_alg_tflops"] for c in done], default=0.0),
    "best_prefuse_alg_tflops": max([c["prefuse_alg_tflops"] for c in done], default=0.0),
    "wall_s": time.time() - t_start,
}
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
json.dump({"summary": summary, "cells": rows}, open(out_path, "w"), indent=1)
print(json.dumps(summary))
