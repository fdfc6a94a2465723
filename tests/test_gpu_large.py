"""Slow GPU parity at the benchmark sizes (marked slow => also gpu).

* SF=10 Q1.1-Q2.3 (BASELINE configs[1]) with the bench's dials through the
  bench's kernels -- the batched pass (laq_batch_*, one pass per query group)
  and the per-query scans -- equal to the REFERENCE's own run_query_laq on the full
  60M-row table (tests/golden/ssb_sf10.json) and to the C checker.
* SF=100 Q3.1-Q4.3 (BASELINE configs[3], the metric's config): every query on
  the 600M-row table, through the bench's batched passes, equals the whole-table goldens (tests/golden/ssb_sf100.json)
  and the live C checker (oracle/fast_query); the first 3M rows, scanned alone,
  equal the reference's own run_query_laq on those rows (golden "sample").
Tolerance 0, as acceptance.cpp:78-103.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, fa, load_golden

pytestmark = [pytest.mark.slow, pytest.mark.gpu]


def _rows(x):
    return fa(x["result"], (x["rows"], x["cols"]))


def _specs(G):
    from paper_2306_08367_b200 import query as Q
    return [Q.spec_with_dial(Q.group_defs(x["group"])[int(x["id"][1]) - 1], x["group"], x["dial"])
            for x in G["queries"]]


def _bench_step(ds, queries, batched=True):
    """The bench's step: per query group (Q1/Q2 at SF=10, Q3/Q4 at SF=100) one
    batched pass (laq_batch_*: code tables + link dictionaries + one scan), or
    one scan per query; then emit."""
    import torch
    from paper_2306_08367_b200 import star
    plans = [ds.prepare(q) for q in queries]
    accs = [torch.zeros(2 * p.n_groups, dtype=torch.int64, device="cuda") for p in plans]
    flags = []
    for grp in (range(0, 3), range(3, 6)):
        if batched:
            b = star.Batch([plans[i] for i in grp])
            b.build()
            b.scan([accs[i] for i in grp])
            flags.append(b.fused)
        else:
            star.build_codes_batch([plans[i] for i in grp])
            for i in grp:
                plans[i].scan(accs[i])
    out = [p.emit(a.cpu().numpy()) for p, a in zip(plans, accs)]
    return out, flags, plans


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "ssb_sf10.json")), reason="sf10 goldens missing")
def test_sf10_bench_queries_vs_reference(gpu_ctx):
    from oracle import fast_query as F
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_sf10.json")
    g = gen.gen_star("Ssb", 10, 42, narrow=True, max_bytes=64 << 30)
    assert len(g.fact["lo_part"]) == G["lineorder_rows"]
    ds = star.upload_gen_star(g)
    queries = _specs(G)
    shared, flags, _ = _bench_step(ds, queries, batched=True)
    assert flags == [True, True]  # the bench's SF=10 groups take the fused batched pass
    single, _, _ = _bench_step(ds, queries, batched=False)
    for q, x, a, b in zip(queries, G["queries"], shared, single):
        want = _rows(x)  # the reference's run_query_laq on the full table
        assert np.array_equal(a, want), x["id"]
        assert np.array_equal(b, want), x["id"]
        assert np.array_equal(F.run_query(g.tables, q), want), x["id"]


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "ssb_sf100.json")), reason="sf100 goldens missing")
def test_sf100_q3q4_vs_oracle_and_reference_sample(gpu_ctx):
    import torch
    from oracle import fast_query as F
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_sf100.json")
    g = gen.gen_star("Ssb", 100, 42, narrow=True, max_bytes=64 << 30)
    assert len(g.fact["lo_part"]) == G["lineorder_rows"] == 600_000_000
    ds = star.upload_gen_star(g)
    queries = _specs(G)
    got, flags, plans = _bench_step(ds, queries, batched=True)
    assert flags == [True, True]  # the bench's SF=100 groups take the fused batched pass
    for q, x, a in zip(queries, G["queries"], got):
        want = _rows(x)
        assert np.array_equal(a, want), x["id"]
        assert np.array_equal(ds.run_query(q), want), x["id"]  # laq_run_query, one call
        assert np.array_equal(F.run_query(g.tables, q), want), x["id"]  # live C checker
    m = G["sample_rows"]
    for p, x in zip(plans, G["sample"]):
        acc = torch.zeros(2 * p.n_groups, dtype=torch.int64, device="cuda")
        p.scan_range(0, m, acc)
        assert np.array_equal(p.emit(acc.cpu().numpy()), _rows(x)), x["id"]  # the reference on these rows
