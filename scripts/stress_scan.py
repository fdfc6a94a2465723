"""Stress the pipelined scan against the ldg fallback: many back-to-back scans
per query and per stage count; report mismatch counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_08367_b200 import gen, query as Q, star
g = gen.gen_star("Ssb", int(os.environ.get("LAQ_SF", "10")), 42, narrow=True)
ds = star.upload_gen_star(g)
DIALS = {(1, 0): 222, (1, 1): 200, (1, 2): 133, (2, 0): 500, (2, 1): 199, (2, 2): 516,
         (3, 0): 90, (4, 0): 50}
reps = int(os.environ.get("REPS", "50"))
os.environ["LAQ_SCAN"] = "ldg"
want = {}
for (gr, qi), d in DIALS.items():
    p = ds.prepare(Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d))
    p.build_codes()
    want[(gr, qi)] = p.scan().cpu().numpy().copy()
os.environ.pop("LAQ_SCAN")
for stages in ("8", "2", "3"):
    os.environ["LAQ_STAGES"] = stages
    for (gr, qi), d in DIALS.items():
        p = ds.prepare(Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d))
        p.build_codes()
        accs = [torch.zeros_like(p.acc) for _ in range(reps)]
        for a in accs:
            p.scan(a)
        torch.cuda.synchronize()
        bad = [i for i, a in enumerate(accs) if not np.array_equal(a.cpu().numpy(), want[(gr, qi)])]
        diff = [int(accs[i].cpu().numpy()[1::2].sum() - want[(gr, qi)][1::2].sum()) for i in bad[:3]]
        print(f"S<={stages} Q{gr}.{qi+1}: {len(bad)}/{reps} mismatches {diff}", flush=True)
