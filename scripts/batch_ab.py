"""A/B of the batched scan's layout knobs on the headline data (SSB SF=100,
600M rows, the bench's dials): L2 prefetch distance, decode-table replication,
(count, sum) vs sum-only bins.  Knobs are read when a batch is prepared, so
each setting prepares its own batch.  Prints one JSON object.

  python scripts/batch_ab.py [--sf 100] [--only default,vec=2,...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_08367_b200 import gen, query as Q, star  # noqa: E402

SF = int(sys.argv[sys.argv.index("--sf") + 1]) if "--sf" in sys.argv else 100
DIALS = {3: (105, 79, 43), 4: (249, 199, 284)} if SF == 100 else None


def main():
    g = gen.gen_star("Ssb", SF, 42, narrow=True, max_bytes=64 << 30)
    ds = star.upload_gen_star(g)
    dials = DIALS or {grp: [int(q.filters[-1].pred.lo) for q in Q.gen_queries(ds.measure_selectivity, grp)]
                      for grp in (3, 4)}
    settings = [("default", {}), ("prefetch=0", {"LAQ_PREFETCH": "0"}), ("prefetch=1", {"LAQ_PREFETCH": "1"}),
                ("prefetch=2", {"LAQ_PREFETCH": "2"}), ("prefetch=4", {"LAQ_PREFETCH": "4"}),
                ("dec_rep=1", {"LAQ_BATCH_DEC_REP": "1"}), ("count_bins", {"LAQ_BATCH_COUNT_BINS": "1"}),
                ("bitmap_first", {"LAQ_BATCH_BITMAP_FIRST": "1"}),
                ("bitmap_first+pipe", {"LAQ_BATCH_BITMAP_FIRST": "1", "LAQ_BATCH_PIPE": "1"}),
                ("pipe", {"LAQ_BATCH_PIPE": "1"}), ("dec64", {"LAQ_BATCH_DEC64": "1"}), ("nojoint", {"LAQ_BATCH_NOJOINT": "1"}), ("jgather=0", {"LAQ_BATCH_JOINT_GATHER_MAX": "0"}),
                ("jgather=1024", {"LAQ_BATCH_JOINT_GATHER_MAX": "1024"}),
                ("nojoint+dec64", {"LAQ_BATCH_NOJOINT": "1", "LAQ_BATCH_DEC64": "1"}),
                ("bulkpf=-1", {"LAQ_PREFETCH": "-1"}), ("bulkpf=-2", {"LAQ_PREFETCH": "-2"}),
                ("bulkpf=-4", {"LAQ_PREFETCH": "-4"})]
    if "--only" in sys.argv:
        keep = sys.argv[sys.argv.index("--only") + 1].split(",")
        settings = [s for s in settings if s[0] in keep]
    out = {"sf": SF}
    for grp in (3, 4):
        qs = [Q.spec_with_dial(d, grp, x) for d, x in zip(Q.group_defs(grp), dials[grp])]
        plans = [ds.prepare(q) for q in qs]
        ref = None
        for name, env in settings:
            for k, v in env.items():
                os.environ[k] = v
            b = star.Batch(plans)
            for k in env:
                del os.environ[k]
            b.build()
            accs = [torch.zeros(2 * p.n_groups, dtype=torch.int64, device="cuda") for p in plans]
            ts = []
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b.scan(accs)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            rows = [p.emit(a.cpu().numpy()) for p, a in zip(plans, accs)]
            if ref is None:
                ref = rows
            same = all(np.array_equal(x, y) for x, y in zip(rows, ref))
            out[f"Q{grp} {name}"] = {"ms": round(float(np.median(ts[1:])), 4), "same_result": same, "fused": b.fused}
            b.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
