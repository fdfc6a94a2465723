"""A/B timing of the SF=100 Q3.x/Q4.x scans under env switches (LAQ_PREFETCH,
LAQ_NOSMEMTAB, LAQ_SCAN).  Usage: python scripts/q34_ab.py [sf]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2306_08367_b200 import gen, query as Q, star  # noqa: E402

sf = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = gen.gen_star("Ssb", sf, 42, narrow=True, max_bytes=64 << 30)
ds = star.upload_gen_star(g)
qs = [q for gr in (3, 4) for q in ds.gen_queries(gr)]
for env in ({}, {"LAQ_PREFETCH": "2"}, {"LAQ_PREFETCH": "1"}, {"LAQ_NOSMEMTAB": "1"}):
    for k in ("LAQ_PREFETCH", "LAQ_NOSMEMTAB"):
        os.environ.pop(k, None)
    os.environ.update(env)
    out = []
    for q in qs:
        p = ds.prepare(q)
        p.build_codes()
        for _ in range(2):
            p.scan()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            p.scan()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out.append((q.id, round(ms, 3), round(p.bytes_per_row * ds.rows["lineorder"] / ms / 1e6)))
    print(env, out, flush=True)
