import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08367_b200 import gen, query as Q, star
g = gen.gen_star("Ssb", int(os.environ.get("LAQ_SF", "10")), 42, narrow=True)
ds = star.upload_gen_star(g)
DIALS = {(1, 0): 222, (1, 1): 200, (1, 2): 133, (2, 0): 500, (2, 1): 199, (2, 2): 516}
for env in ({}, {"LAQ_SCAN": "ldg"}):
    for k in ("LAQ_STAGES", "LAQ_NOSMEMTAB", "LAQ_SCAN"):
        os.environ.pop(k, None)
    os.environ.update(env)
    plans = [ds.prepare(Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)) for (gr, qi), d in DIALS.items()]
    for p in plans:
        p.build_codes()
        accs = [torch.zeros_like(p.acc) for _ in range(12)]
        for a in accs:
            p.scan(a)
        torch.cuda.synchronize()
        sums = [int(a.cpu().numpy()[1::2].sum()) for a in accs]
        print(env, p.q.id, len(set(sums)), sums[:4], flush=True)
