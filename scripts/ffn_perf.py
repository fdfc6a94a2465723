"""cfg3 timing: SSB SF=10 lineorder x customer x part + 2-layer FFN (h=256) on one B200.
Prints per-call ms for the join+FFN (probe mode) and the FFN over precomputed row maps,
algorithmic TFLOP/s and the tensor-pipe rate (x3 for the bf16x3 split)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_08367_b200 import ffn, gen  # noqa: E402

sf = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10
t0 = time.time()
g = gen.gen_star("Ssb", sf, 42, narrow=True)
fks, pks, dims, pl, W1, W2 = ffn.cfg3_inputs(g)
print(f"gen {time.time() - t0:.1f}s rows={len(fks[0])}", flush=True)
m = ffn.StarFFN(dims, pl, W1, W2, dim_pks=pks)
fd = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in fks]
n = fd[0].numel()
out = torch.empty((n, 1), dtype=torch.float32, device="cuda")
rows = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(2)]
nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
import ctypes as C  # noqa: E402
from paper_2306_08367_b200.device import ptrs  # noqa: E402
ctx = m.ctx
ctx.check(ctx.lib.laq_probe_join_rows(ctx.h, m.probe, ptrs(fd), n, ptrs(rows), None, nnz.data_ptr()))
torch.cuda.synchronize()


if "--profile" in sys.argv:  # one launch of each form, for ncu
    m(fd, out=out)
    m.predict_rows(rows, out=out)
    torch.cuda.synchronize()
    sys.exit(0)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms_star = timed(lambda: m(fd, out=out))
ms_rows = timed(lambda: m.predict_rows(rows, out=out))
ms_join = timed(lambda: ctx.check(ctx.lib.laq_probe_join_rows(ctx.h, m.probe, ptrs(fd), n, ptrs(rows), None,
                                                               nnz.data_ptr())))
flop = n * (2 * 64 * 256 + 2 * 256)
res = {"rows": n, "ms_join_ffn_probe": ms_star, "ms_ffn_rows": ms_rows, "ms_join_rows": ms_join,
       "rows_per_s": n / ms_star * 1e3, "alg_tflops": flop / ms_star / 1e9,
       "tensor_tflops_x3": 3 * n * 2 * 64 * 256 / ms_star / 1e9,
       "gather_bytes": n * 256, "gather_gbs": n * 256 / ms_star / 1e6}
print(json.dumps(res))
