"""configs[0] end to end with host buffers: plain copies vs the serial
H2D -> predict -> D2H sequence vs laq_probe_fused_predict_host at several
chunk sizes (host clock, median of 20)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08367_b200 import fusion, gen  # noqa: E402

fk, pk, feats, W = gen.cfg1_inputs(1_000_000, 10_000, 16, 1)
f = fusion.prefuse_linear([feats], [np.arange(16)], W)
pred = fusion.FusedStarPredictor([pk], f.partials)
fk_pin = torch.from_numpy(fk.astype(np.int32)).pin_memory()
y_pin = torch.empty((1_000_000, 1), dtype=torch.float64).pin_memory()
fkd = torch.empty(1_000_000, dtype=torch.int32, device="cuda")
yd = torch.empty((1_000_000, 1), dtype=torch.float64, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    xs = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        xs.append((time.perf_counter() - t0) * 1e6)
    return round(float(np.median(xs)), 1)


print("h2d 4MB us", t(lambda: fkd.copy_(fk_pin, non_blocking=True)))
print("d2h 8MB us", t(lambda: y_pin.copy_(yd, non_blocking=True)))
print("predict device us", t(lambda: pred([fkd], out=yd, sync=False)))
print("serial us", t(lambda: (fkd.copy_(fk_pin, non_blocking=True), pred([fkd], out=yd, sync=False),
                              y_pin.copy_(yd, non_blocking=True))))
for c in (0, 500_000, 250_000, 125_000):
    print("predict_host chunk", c, "us", t(lambda: pred.predict_host([fk_pin], out=y_pin, chunk_rows=c)))
# 1e8 rows: 400 MB of keys up, 800 MB of predictions down
big = torch.randint(0, 10_000, (100_000_000,), dtype=torch.int32).pin_memory()
ybig = torch.empty((100_000_000, 1), dtype=torch.float64).pin_memory()
bd = torch.empty(100_000_000, dtype=torch.int32, device="cuda")
ybd = torch.empty((100_000_000, 1), dtype=torch.float64, device="cuda")
print("1e8 serial ms", t(lambda: (bd.copy_(big, non_blocking=True), pred([bd], out=ybd, sync=False),
                                  ybig.copy_(ybd, non_blocking=True)), reps=5) / 1e3)
for c in (100_000_000, 0, 4_000_000):
    print("1e8 predict_host chunk", c, "ms", t(lambda: pred.predict_host([big], out=ybig, chunk_rows=c), reps=5) / 1e3)
