"""Goldens for the benchmark-size SSB configurations (run in the dev container,
where /root/reference exists; the GPU box only reads the committed JSON):

  ssb_sf10.json   BASELINE configs[1]: SF=10, seed 42, Q1.1-Q2.3.  Data from the
                  REFERENCE generator (ref.gen_star), dials from the REFERENCE
                  tuner (ref.gen_queries, benchgen.cpp:413-457), results from the
                  REFERENCE run_query_laq (cli.cpp:73-138) on the full 60M rows.
  ssb_sf100.json  BASELINE configs[3]: SF=100, seed 42, Q3.1-Q4.3.  The reference
                  needs ~130 GB and ~10 min per query here, so:
                  data from the bit-exact generator restatement (pinned column by
                  column against the reference in tests/test_gen.py), dials from
                  the restated tuner (query.gen_queries, pinned against the
                  reference's dials in tests/test_oracle_golden.py) over exact
                  selectivities, whole-table results from the C checker
                  oracle/fast_query (pinned against the reference's goldens in
                  tests/test_oracle_fast.py), AND the reference's own
                  run_query_laq on the first SAMPLE_ROWS lineorder rows (the
                  sample bench.py's reference arm runs).

    make -C oracle && python tests/golden/make_golden_large.py [sf10] [sf100]
"""
from __future__ import annotations

import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import fast_query as F  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2306_08367_b200 import gen, query as Q  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SAMPLE_ROWS = 3_000_000


def fx(a):
    return [float(v).hex() for v in np.asarray(a, np.float64).ravel()]


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name, flush=True)


def entry(qid, grp, dial, m):
    return {"id": qid, "group": grp, "dial": int(dial), "rows": m.shape[0], "cols": m.shape[1], "result": fx(m),
            "checksum": str(ref.checksum_rows(m))}


def parallel(fns):
    out = [None] * len(fns)

    def run(i):
        out[i] = fns[i]()
    th = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def sf10():
    t0 = time.time()
    s = ref.gen_star("Ssb", sf=10, seed=42, max_bytes=64 << 30)
    print(f"ref gen sf=10 {time.time() - t0:.1f}s", flush=True)
    tuned = parallel([lambda g=g: ref.gen_queries(s, g) for g in (1, 2)])
    print(f"ref gen_queries {time.time() - t0:.1f}s", flush=True)
    qs = []
    for grp, (dials, _) in zip((1, 2), tuned):
        for qi, d in enumerate(Q.group_defs(grp)):
            qs.append((d.id, grp, int(dials[qi]), Q.spec_with_dial(d, grp, int(dials[qi]))))
    res = []
    for half in (qs[:3], qs[3:]):  # three concurrent run_query_laq at a time (host RAM)
        res += parallel([lambda q=q: ref.run_query(s, q[3]) for q in half])
    print(f"ref run_query_laq x6 {time.time() - t0:.1f}s", flush=True)
    dump("ssb_sf10.json", {"setting": "Ssb", "sf": 10, "seed": 42, "lineorder_rows": len(s.fact["lo_part"]),
                           "source": "reference gen_star + gen_queries + run_query_laq (oracle/_ref)",
                           "queries": [dict(entry(a, b, c, m), ref_seconds=secs)
                                       for (a, b, c, _), (m, secs) in zip(qs, res)]})


def sf100():
    t0 = time.time()
    g = gen.gen_star("Ssb", 100, 42, narrow=True, max_bytes=64 << 30)
    n = len(g.fact["lo_part"])
    print(f"gen sf=100 {time.time() - t0:.1f}s", flush=True)

    def selectivity(q):
        c, _ = F.Prepared(g.tables, q).partial()
        return float(c.sum()) / float(n)
    qs = []
    for grp in (3, 4):
        for qi, q in enumerate(Q.gen_queries(selectivity, grp)):
            qs.append((q.id, grp, int(q.filters[-1].pred.lo), q))
    print(f"tuned {[x[2] for x in qs]} {time.time() - t0:.1f}s", flush=True)
    full = [F.run_query(g.tables, q[3]) for q in qs]
    print(f"checked whole table {time.time() - t0:.1f}s", flush=True)
    sm = gen.gen_star("Ssb", 100, 42, narrow=False, max_bytes=64 << 30, row_range=(0, SAMPLE_ROWS))
    tables = [("lineorder", dict(sm.fact))] + [(t, dict(c)) for t, c in sm.tables.items() if t != "lineorder"]
    rs = ref.star_from_tables(tables, sm.links())
    sample = parallel([lambda q=q: ref.run_query(rs, q[3]) for q in qs])
    for q, (m, _) in zip(qs, sample):
        assert np.array_equal(m, F.run_query(g.tables, q[3], row_range=(0, SAMPLE_ROWS))), q[0]
    print(f"reference sample {time.time() - t0:.1f}s", flush=True)
    dump("ssb_sf100.json", {
        "setting": "Ssb", "sf": 100, "seed": 42, "lineorder_rows": n, "sample_rows": SAMPLE_ROWS,
        "source": "whole table: oracle/fast_query over the generator restatement, dials from query.gen_queries "
                  "over exact selectivities; sample: the reference's run_query_laq (oracle/_ref) on lineorder "
                  f"rows [0, {SAMPLE_ROWS})",
        "queries": [entry(a, b, c, m) for (a, b, c, _), m in zip(qs, full)],
        "sample": [dict(entry(a, b, c, m), ref_seconds=secs) for (a, b, c, _), (m, secs) in zip(qs, sample)]})


if __name__ == "__main__":
    what = sys.argv[1:] or ["sf10", "sf100"]
    if "sf10" in what:
        sf10()
    if "sf100" in what:
        sf100()
