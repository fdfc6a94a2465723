"""ncu driver for the fused join+predict kernel (cfg1 shape at 1e8 fact rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08367_b200 import fusion, gen
fk, pk, feats, W = gen.cfg1_inputs(1_000_000, 10_000, 16, 1)
f = fusion.prefuse_linear([feats], [np.arange(16)], W)
pred = fusion.FusedStarPredictor([pk], f.partials)
n = int(os.environ.get("N", "100000000"))
fkd = torch.randint(0, 10_000, (n,), dtype=torch.int32, device="cuda")
y = torch.empty((n, 1), dtype=torch.float64, device="cuda")
for _ in range(3):
    pred([fkd], out=y, sync=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    pred([fkd], out=y, sync=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"n={n} ms={ms:.4f} GB/s={12*n/ms/1e6:.1f} nnz={int(pred.nnz_dev.item())}")
