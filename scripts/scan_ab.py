"""A/B timing of the K4 scan variants on the six bench queries (SSB SF=10).
LAQ_SCAN=ldg forces the vectorised-load fallback, =pipe the TMA pipeline, =stream the
generic stream kernel; default (direct) is the direct-probe stream kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_08367_b200 import gen, query as Q, star  # noqa: E402

DIALS = {(1, 0): 222, (1, 1): 200, (1, 2): 133, (2, 0): 500, (2, 1): 199, (2, 2): 516}
g = gen.gen_star("Ssb", int(os.environ.get("LAQ_SF", "10")), 42, narrow=True)
ds = star.upload_gen_star(g)
res = {}
for variant in ("direct", "stream", "pipe", "ldg"):
    os.environ["LAQ_SCAN"] = variant
    plans = [ds.prepare(Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)) for (gr, qi), d in DIALS.items()]
    out = []
    for p in plans:
        p.build_codes()
        for _ in range(3):
            p.scan()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            p.scan()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        r = p.emit(p.acc.cpu().numpy())
        out.append((p.q.id, round(ms, 4), round(p.bytes_per_row * len(g.fact["lo_part"]) / ms / 1e6, 1), r.shape[0],
                    float(r[:, -1].sum())))
    res[variant] = out
    print(variant, out, flush=True)
bad = 0
for a, b in list(zip(res["pipe"], res["ldg"])) + list(zip(res["stream"], res["ldg"])) + list(zip(res["direct"], res["ldg"])):
    if a[3:] != b[3:]:
        bad += 1
        print("MISMATCH", a, b)
print("mismatches", bad)
for a, b in []:
    assert a[3:] == b[3:], (a, b)
print("variants agree")
