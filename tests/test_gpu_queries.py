"""GPU parity for the query plan driver (run_query_laq, cli.cpp:73-138) and
the device-tuned workload (gen_queries, benchgen.cpp:413-457).

Integer aggregates: tolerance 0 (acceptance.cpp:78-103 uses tolerance 0 too).
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, fa, load_golden
from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu


def _star(setting, sf, seed, narrow=False, row_range=None):
    from paper_2306_08367_b200 import gen, star
    g = gen.gen_star(setting, sf, seed, narrow=narrow)
    return g, star.upload_gen_star(g, row_range=row_range)


def _q(group, qid, dial):
    from paper_2306_08367_b200 import query as Q
    return Q.spec_with_dial(Q.group_defs(group)[int(qid[1]) - 1], group, dial)


@pytest.mark.parametrize("narrow", [False, True])
def test_queries_s2_golden(gpu_ctx, narrow):
    G = load_golden("ssb_s2_sf2.json")
    g, ds = _star(G["setting"], G["sf"], G["seed"], narrow)
    for qg in G["queries"]:
        q = _q(qg["group"], qg["id"], qg["dial"])
        m = ds.run_query(q)
        assert m.shape == (qg["rows"], qg["cols"]), qg["id"]
        assert np.array_equal(m.ravel(), fa(qg["result"])), qg["id"]
        assert str(O.checksum_rows(m)) == qg["checksum"]
        assert ds.measure_selectivity(q) == float.fromhex(qg["selectivity"])


def test_device_gen_queries_pick_reference_dials(gpu_ctx):
    G = load_golden("ssb_s2_sf2.json")
    g, ds = _star(G["setting"], G["sf"], G["seed"])
    for grp in (1, 2, 3, 4):
        qs = ds.gen_queries(grp)
        want = [x for x in G["queries"] if x["group"] == grp]
        assert [q.filters[-1].pred.lo for q in qs] == [w["dial"] for w in want]
        assert [q.realized_selectivity for q in qs] == [float.fromhex(w["realized"]) for w in want]


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "ssb_sf1.json")), reason="sf1 goldens not generated")
def test_queries_ssb_sf1_reference_checksums(gpu_ctx):
    """all 12 SSB sf=1 (seed 42) queries, reference checksums."""
    G = load_golden("ssb_sf1.json")
    g, ds = _star("Ssb", 1, 42, narrow=True)
    for qg in G["queries"]:
        m = ds.run_query(_q(qg["group"], qg["id"], qg["dial"]))
        assert m.shape == (qg["rows"], qg["cols"]), qg["id"]
        assert np.array_equal(m.ravel(), fa(qg["result"])), qg["id"]
        assert str(O.checksum_rows(m)) == qg["checksum"], qg["id"]


def test_sharded_accumulators_sum_to_whole(gpu_ctx):
    """Row shards (multi-GPU layout): per-shard accumulators add up
    to the whole-table accumulator, and emit() of the sum equals the full query."""
    import torch
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_s2_sf2.json")
    g = gen.gen_star(G["setting"], G["sf"], G["seed"], narrow=True)
    n = len(g.fact["lo_part"])
    full = star.upload_gen_star(g)
    shards = [star.upload_gen_star(g, row_range=(n * k // 3, n * (k + 1) // 3)) for k in range(3)]
    for qg in G["queries"]:
        q = _q(qg["group"], qg["id"], qg["dial"])
        plans = [s.prepare(q) for s in shards]
        acc = sum(p.execute().clone() for p in plans)
        m = plans[0].emit(acc.cpu().numpy())
        assert np.array_equal(m, full.run_query(q)), qg["id"]


def test_query_errors(gpu_ctx):
    from paper_2306_08367_b200 import errors, query as Q
    G = load_golden("ssb_s2_sf2.json")
    g, ds = _star(G["setting"], G["sf"], G["seed"])
    q = _q(2, "21", 100)
    bad = Q.QuerySpec(id="x", group=2, joins=q.joins, filters=[Q.FilterSpec(1, "s_nope", Q.Pred.eq(1))],
                      group_by=q.group_by, order_by=True)
    with pytest.raises(errors.NameError_):
        ds.run_query(bad)
    bad2 = Q.QuerySpec(id="x", group=2, joins=[Q.StarLink("lo_part", "nodim", "p_key")], filters=[])
    with pytest.raises(errors.NameError_):
        ds.run_query(bad2)
    f = Q.FilterSpec(-1, "lo_quantity", Q.Pred(Q.LT, 3, is_float=True))
    with pytest.raises(errors.TypeError_):
        ds.run_query(Q.QuerySpec(id="x", group=1, joins=[Q.ORDERDATE], filters=[f]))


def test_duplicate_pk_is_rejected(gpu_ctx):
    from paper_2306_08367_b200 import errors, star
    ds = star.DeviceStar()
    ds.add_table("lineorder", {"f": np.array([0, 1, 2])}, {"f": 0}, is_fact=True)
    ds.add_table("d", {"k": np.array([0, 0, 1]), "a": np.array([1, 2, 3])}, {"k": 0, "a": 1})
    with pytest.raises(errors.DuplicateKeyError):
        ds.add_link("f", "d", "k")
    with pytest.raises(errors.FormatError):
        ds.add_table("neg", {"k": np.array([-1, 2])}, {"k": 0})


@pytest.mark.slow
def test_sf10_q21_against_oracle(gpu_ctx):
    """Full-size property check at BASELINE cfg2 scale (SF=10, 60M rows)."""
    from paper_2306_08367_b200 import query as Q
    g, ds = _star("Ssb", 10, 42, narrow=True)
    for grp, qi, dial in ((1, 0, 30), (2, 0, 100), (3, 0, 90), (4, 0, 50)):
        q = Q.spec_with_dial(Q.group_defs(grp)[qi], grp, dial)
        assert np.array_equal(ds.run_query(q), O.run_query(g.tables, q))


@pytest.mark.parametrize("dangling", [0.0, 0.05])
def test_link_elision_respects_inner_join(gpu_ctx, dangling):
    """Q3.x joins part with no filter / group column.  With every lo_part key
    present the link is left out of the scan (one 4-byte column less per row);
    with dangling keys (fact rows whose part is missing must drop, inner join,
    laqops.cpp:283-298) it must stay.  Both must equal the oracle exactly."""
    from paper_2306_08367_b200 import gen, star
    g = gen.gen_star("Ssb", 1, 42, dangling=dangling, narrow=True)
    ds = star.upload_gen_star(g)
    for grp in (3, 4):
        for q in ds.gen_queries(grp):
            p = ds.prepare(q)
            if dangling == 0.0 and grp == 3:
                assert p.scanned_links == len(q.joins) - 1  # part link elided
            if dangling > 0.0:
                assert p.scanned_links == len(q.joins)
            assert np.array_equal(ds.run_query(q), O.run_query(g.tables, q))


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "ssb_sf1.json")), reason="sf1 goldens not generated")
def test_packed_fact_table_reference_checksums(gpu_ctx):
    """The compact transfer format (star.pack_columns: uint8/uint16 offsets from the
    column minimum) registered in place with laq_star_add_table_device_packed:
    all 12 SSB sf=1 queries still reproduce the reference checksums."""
    import torch
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_sf1.json")
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    packed = star.pack_columns(g.fact)
    assert {w for _, w, _ in packed.values()} >= {1, 2}  # discount/quantity bytes, dates/supplier halves
    ds = star.DeviceStar()
    dev = {c: (torch.from_numpy(b).cuda(), w, off) for c, (b, w, off) in packed.items()}
    ds.add_table_device_packed("lineorder", dev, g.kinds["lineorder"], is_fact=True)
    for t, cols in g.tables.items():
        if t != "lineorder":
            ds.add_table(t, cols, g.kinds[t])
    for l in g.links():
        ds.add_link(*l)
    for qg in G["queries"]:
        m = ds.run_query(_q(qg["group"], qg["id"], qg["dial"]))
        assert np.array_equal(m.ravel(), fa(qg["result"])), qg["id"]
        assert str(O.checksum_rows(m)) == qg["checksum"], qg["id"]


def test_scan_ranges_sum_to_whole(gpu_ctx):
    """laq_plan_scan_range over consecutive row chunks (the chunked-upload path of
    bench.py's e2e) accumulates to exactly the whole-table scan."""
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_s2_sf2.json")
    g = gen.gen_star(G["setting"], G["sf"], G["seed"], narrow=True)
    ds = star.upload_gen_star(g)
    n = len(g.fact["lo_part"])
    cuts = [0, (n // 7) // 4 * 4, (n // 2) // 4 * 4, n]
    for qg in G["queries"]:
        p = ds.prepare(_q(qg["group"], qg["id"], qg["dial"]))
        whole = p.execute().clone()
        p.build_codes()
        acc = None
        for k in range(3):
            acc = p.scan_range(cuts[k], cuts[k + 1] - cuts[k], acc=None if acc is None else acc, accumulate=k > 0)
        assert np.array_equal(acc.cpu().numpy(), whole.cpu().numpy()), qg["id"]


def test_batched_code_tables_equal_per_plan(gpu_ctx):
    """laq_plans_build_codes: one launch for a batch of plans (and the per-plan
    fallback beyond 24 links) gives the same accumulators as per-plan builds."""
    from paper_2306_08367_b200 import gen, query as Q, star
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    ds = star.upload_gen_star(g)
    qs = [Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)
          for (gr, qi), d in {(1, 0): 222, (2, 1): 199, (3, 0): 90, (4, 2): 20, (2, 0): 500, (4, 0): 50,
                              (3, 2): 40, (4, 1): 30, (1, 2): 133}.items()]
    want = []
    for q in qs:
        p = ds.prepare(q)
        want.append(p.execute().cpu().numpy().copy())
    for batch in (qs[:6], qs):  # <= 24 links: one launch; all nine: per-plan fallback
        plans = [ds.prepare(q) for q in batch]
        star.build_codes_batch(plans)
        for p, w in zip(plans, want):
            assert np.array_equal(p.scan().cpu().numpy(), w), p.q.id


def test_shared_scan_equals_individual_scans(gpu_ctx):
    """laq_plans_scan_shared: Q1.1-Q1.3, Q2.1-Q2.3, Q3.x and Q4.x batches in one
    pass over the fact table equal the queries scanned one by one; a batch
    mixing column sets falls back to one-by-one scans with the same results."""
    import torch
    from paper_2306_08367_b200 import gen, query as Q, star
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    ds = star.upload_gen_star(g)
    dials = {1: (222, 200, 133), 2: (500, 199, 516), 3: (90, 60, 40), 4: (50, 30, 20)}
    batches = [[(gr, qi) for qi in range(3)] for gr in (1, 2, 3, 4)] + [[(2, 0), (2, 2)], [(1, 0), (2, 0)]]
    for batch in batches:
        qs = [Q.spec_with_dial(Q.group_defs(gr)[qi], gr, dials[gr][qi]) for gr, qi in batch]
        plans = [ds.prepare(q) for q in qs]
        want = [p.execute().cpu().numpy().copy() for p in plans]
        star.build_codes_batch(plans)
        accs = [torch.full_like(p.acc, 7) for p in plans]
        shared = star.scan_shared(plans, accs)
        torch.cuda.synchronize()
        if len({gr for gr, _ in batch}) > 1:
            assert not shared, batch  # different column sets: one by one
        if batch[0][0] == 1 and len(batch) == 3:
            assert shared  # Q1.x: same columns, small tables -> one pass
        for a, w, q in zip(accs, want, qs):
            assert np.array_equal(a.cpu().numpy(), w), (batch, q.id)
