"""Bandwidth reference points for the fused predict traffic mix (4 B read + 8 B write per row)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = 100_000_000
k = torch.randint(0, 10_000, (n,), dtype=torch.int32, device="cuda")
P = torch.rand(10_000, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: y.copy_(k)); print(f"copy int32->f64: {ms:.3f} ms  {12*n/ms/1e6:.0f} GB/s")
ms = t(lambda: torch.index_select(P, 0, k, out=y)); print(f"index_select gather: {ms:.3f} ms  {12*n/ms/1e6:.0f} GB/s")
z = torch.empty(n, dtype=torch.int32, device="cuda")
ms = t(lambda: z.copy_(k)); print(f"copy int32: {ms:.3f} ms  {8*n/ms/1e6:.0f} GB/s")
ms = t(lambda: y.fill_(1.0)); print(f"fill f64: {ms:.3f} ms  {8*n/ms/1e6:.0f} GB/s")
ms = t(lambda: k.sum()); print(f"sum int32: {ms:.3f} ms  {4*n/ms/1e6:.0f} GB/s")
