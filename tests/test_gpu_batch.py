"""GPU: the batched scan (laq_batch_*, csrc/ssb_batch.cuh) -- a batch of
queries in one pass with one dictionary-encoded probe per link -- equals each
query run alone by the reference semantics (run_query_laq, cli.cpp:73-138),
exactly (integer aggregates: tolerance 0, as acceptance.cpp:78-103).

Covers: the SSB query groups (every group fused), the committed SF=1 / SF=10 /
SF=100 goldens, random stars with random query batches (fused and plan-by-plan
fallback batches), queries of a batch joining different link sets, empty fact
intervals, dangling keys, mixed plain-sum / group-by batches."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, fa, load_golden
from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu


def _q(group, i, dial):
    from paper_2306_08367_b200 import query as Q
    return Q.spec_with_dial(Q.group_defs(group)[i], group, dial)


def _run_batch(ds, qs):
    from paper_2306_08367_b200 import star
    plans = [ds.prepare(q) for q in qs]
    b = star.Batch(plans)
    got = b.run()
    again = b.run()  # rebuild + rescan: same answer (dictionaries rebuilt each step)
    for x, y in zip(got, again):
        assert np.array_equal(x, y)
    return b, got


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "ssb_sf1.json")), reason="sf1 goldens not generated")
def test_ssb_sf1_groups_fused_match_goldens(gpu_ctx):
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_sf1.json")
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    ds = star.upload_gen_star(g)
    for grp in (1, 2, 3, 4):
        qg = [x for x in G["queries"] if x["group"] == grp]
        qs = [_q(grp, int(x["id"][1]) - 1, x["dial"]) for x in qg]
        b, got = _run_batch(ds, qs)
        assert b.fused, (grp, b.why)
        for m, x in zip(got, qg):
            assert m.shape == (x["rows"], x["cols"]), x["id"]
            assert np.array_equal(m.ravel(), fa(x["result"])), x["id"]
            assert str(O.checksum_rows(m)) == x["checksum"], x["id"]


def test_all_twelve_queries_in_batches_of_any_mix(gpu_ctx):
    """Batches mixing groups (different link sets, plain sums with group-bys,
    fact filters only some queries have) vs the oracle."""
    from paper_2306_08367_b200 import gen, star
    g = gen.gen_star("S2", 2, 42, narrow=True)
    ds = star.upload_gen_star(g)
    qs = []
    for grp in (1, 2, 3, 4):
        qs += ds.gen_queries(grp)
    want = [O.run_query(g.tables, q) for q in qs]
    rng = np.random.default_rng(3)
    for trial in range(8):
        k = int(rng.integers(1, 5))
        pick = rng.choice(len(qs), k, replace=False)
        b, got = _run_batch(ds, [qs[i] for i in pick])
        for i, m in zip(pick, got):
            assert m.shape == want[i].shape and np.array_equal(m, want[i]), (trial, qs[i].id, b.fused, b.why)


def _random_star(rng, n, dense=True, dangling=0.0, positive=False):
    from paper_2306_08367_b200 import query as Q
    fact = {"lo_measure": rng.integers(1 if positive else 0, 10_000, n).astype(np.int64),
            "lo_a": rng.integers(0, 50, n).astype(np.int64),
            "lo_b": rng.integers(-20, 20, n).astype(np.int64)}
    fk_kinds = {"lo_measure": 1, "lo_a": 1, "lo_b": 1}
    tables, kinds, links = {}, {}, []
    for d in range(int(rng.integers(1, 5))):
        rows = int(rng.integers(1, 40_000))
        pk = np.arange(rows) if dense else np.sort(rng.choice(5_000_000, rows, replace=False))
        pk = pk.astype(np.int64)
        rng.shuffle(pk)
        name = f"dim{d}"
        tables[name] = {"pk": pk, "x": rng.integers(0, 7, rows).astype(np.int64),
                        "y": rng.integers(0, 40, rows).astype(np.int64),
                        "z": rng.integers(0, 1000, rows).astype(np.int64)}
        kinds[name] = {"pk": 0, "x": 1, "y": 1, "z": 1}
        fk = rng.choice(pk, n)
        if dangling:
            miss = rng.random(n) < dangling
            fk[miss] = pk.max() + 1 + rng.integers(0, 100, miss.sum())
        fact[f"lo_fk{d}"] = fk
        fk_kinds[f"lo_fk{d}"] = 0
        links.append((f"lo_fk{d}", name, "pk"))
    tables = {"lineorder": fact, **tables}
    kinds = {"lineorder": fk_kinds, **kinds}
    return tables, kinds, links, [Q.StarLink(*l) for l in links]


def _random_query(rng, joins, i):
    from paper_2306_08367_b200 import query as Q
    use = [j for j in range(len(joins)) if rng.random() < 0.8] or [0]
    sub = [joins[j] for j in use]
    filters, group = [], []
    for t in range(len(sub)):
        r = rng.random()
        if r < 0.35:
            filters.append(Q.FilterSpec(t, "x", Q.Pred.lt(int(rng.integers(0, 8)))))
        elif r < 0.55:
            filters.append(Q.FilterSpec(t, "z", Q.Pred.between(int(rng.integers(0, 600)), int(rng.integers(300, 1000)))))
        elif r < 0.65:
            filters.append(Q.FilterSpec(t, "y", Q.Pred.in_set(rng.choice(40, int(rng.integers(1, 10)), replace=False))))
        if rng.random() < 0.45:
            group.append(Q.GroupRef(t, "x" if rng.random() < 0.6 else "y"))
    r = rng.random()
    if r < 0.3:
        filters.append(Q.FilterSpec(-1, "lo_a", Q.Pred.between(int(rng.integers(0, 30)), int(rng.integers(10, 50)))))
    elif r < 0.4:
        filters.append(Q.FilterSpec(-1, "lo_b", Q.Pred.gt(int(rng.integers(-25, 25)))))
    elif r < 0.45:
        filters.append(Q.FilterSpec(-1, "lo_b", Q.Pred.in_set(rng.choice(np.arange(-20, 20), 5, replace=False))))
    return Q.QuerySpec(id=f"r{i}", group=0, joins=sub, filters=filters, measure="lo_measure", group_by=group,
                       order_by=bool(group) and rng.random() < 0.5)


@pytest.mark.parametrize("seed", range(24))
def test_random_batches_match_oracle(gpu_ctx, seed):
    from paper_2306_08367_b200 import star
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 400_000))
    # positive measures (every other seed): sum-only bins and the joint pair decode
    tables, kinds, links, joins = _random_star(rng, n, dense=seed % 4 != 3, dangling=0.03 if seed % 5 == 1 else 0.0,
                                               positive=seed % 2 == 0)
    ds = star.DeviceStar.from_tables(tables, kinds, links)
    qs = [_random_query(rng, joins, i) for i in range(int(rng.integers(1, 5)))]
    b, got = _run_batch(ds, qs)
    for q, m in zip(qs, got):
        want = O.run_query(tables, q)
        assert m.shape == want.shape and np.array_equal(m, want), (seed, q, b.fused, b.why)


def test_empty_interval_and_tail_rows(gpu_ctx):
    """A fact interval that matches nothing (lo > hi) rejects every row for that
    query only; row counts not a multiple of the 4096-row step."""
    from paper_2306_08367_b200 import query as Q, star
    rng = np.random.default_rng(7)
    for n in (1, 5, 4097, 4096 * 148 + 3):
        tables, kinds, links, joins = _random_star(rng, n)
        ds = star.DeviceStar.from_tables(tables, kinds, links)
        qs = [Q.QuerySpec(id="e", group=0, joins=joins[:1], filters=[Q.FilterSpec(-1, "lo_a", Q.Pred.between(30, 10))],
                          measure="lo_measure", group_by=[Q.GroupRef(0, "x")]),
              Q.QuerySpec(id="f", group=0, joins=joins[:1], filters=[], measure="lo_measure",
                          group_by=[Q.GroupRef(0, "x")]),
              Q.QuerySpec(id="g", group=0, joins=joins[:1], filters=[Q.FilterSpec(-1, "lo_a", Q.Pred.lt(25))],
                          measure="lo_measure", group_by=[])]
        b, got = _run_batch(ds, qs)
        assert b.fused, b.why
        for q, m in zip(qs, got):
            want = O.run_query(tables, q)
            assert m.shape == want.shape and np.array_equal(m, want), (n, q.id)


@pytest.mark.slow
def test_sf10_bench_groups_fused_vs_golden(gpu_ctx):
    """The q1q2 bench workload (SF=10 Q1.1-Q2.3, its dials) through the batched
    scan vs the committed whole-table goldens (tests/golden/make_golden_large.py)."""
    from paper_2306_08367_b200 import gen, star
    G = load_golden("ssb_sf10.json")
    g = gen.gen_star("Ssb", 10, 42, narrow=True)
    ds = star.upload_gen_star(g)
    qg = G["queries"]
    for grp in (1, 2):
        sel = [x for x in qg if x["group"] == grp]
        qs = [_q(grp, int(x["id"][1]) - 1, x["dial"]) for x in sel]
        b, got = _run_batch(ds, qs)
        assert b.fused, b.why
        for m, x in zip(got, sel):
            assert m.shape == (x["rows"], x["cols"]) and np.array_equal(m.ravel(), fa(x["result"])), x["id"]


@pytest.mark.parametrize("env", [{"LAQ_NOSMEMTAB": "1"}, {"LAQ_NOSMEMTAB": "1", "LAQ_BATCH_PIPE": "1"},
                                 {"LAQ_BATCH_COUNT_BINS": "1"}, {"LAQ_BATCH_COUNT_BINS": "1", "LAQ_NOSMEMTAB": "1"},
                                 {"LAQ_BATCH_DEC64": "1"}, {"LAQ_BATCH_DEC64": "1", "LAQ_NOSMEMTAB": "1"},
                                 {"LAQ_BATCH_NOJOINT": "1"}, {"LAQ_BATCH_NOJOINT": "1", "LAQ_BATCH_DEC64": "1"}])
def test_layout_variants_match_oracle(gpu_ctx, monkeypatch, env):
    """Every kernel form the layout can pick: all links gathered through L2
    (the software-pipelined 2-row kernel for the last link, synchronous
    gathers for the others), the unpipelined form, (count, sum) vs sum-only
    bins, narrow (4-byte, 10-bit lanes) vs wide (8-byte, 16-bit lanes) decode,
    with and without the joint decode table of the first two staged links --
    same results as the oracle on the SSB groups and random batches."""
    from paper_2306_08367_b200 import gen, star
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = gen.gen_star("S2", 2, 42, narrow=True)
    ds = star.upload_gen_star(g)
    for grp in (2, 3, 4):
        qs = ds.gen_queries(grp)
        b, got = _run_batch(ds, qs)
        assert b.fused, b.why
        for q, m in zip(qs, got):
            assert np.array_equal(m, O.run_query(g.tables, q)), (env, q.id)
    rng = np.random.default_rng(77)
    for trial in range(6):
        tables, kinds, links, joins = _random_star(rng, int(rng.integers(1, 300_000)), dangling=0.02 * (trial % 2),
                                                   positive=trial % 3 == 0)
        dsr = star.DeviceStar.from_tables(tables, kinds, links)
        qs = [_random_query(rng, joins, i) for i in range(int(rng.integers(2, 5)))]
        b, got = _run_batch(dsr, qs)
        for q, m in zip(qs, got):
            assert np.array_equal(m, O.run_query(tables, q)), (env, trial, q, b.fused, b.why)


def test_wide_dictionaries_and_fallbacks(gpu_ctx):
    """uint16 tuple ids (> 256 distinct tuples on a link: ~4,900 here), a group
    space above 4096 (plan-by-plan fallback) and more than 65,535 distinct
    tuples on a link (dictionary overflow -> fallback): every case equals the
    oracle."""
    from paper_2306_08367_b200 import query as Q, star
    rng = np.random.default_rng(11)
    n, r = 300_000, 300_000  # a, b, c: 48 values each -> ~103K distinct (a, b, c) tuples
    dim = {"pk": np.arange(r, dtype=np.int64), "a": rng.integers(0, 48, r).astype(np.int64),
           "b": rng.integers(0, 48, r).astype(np.int64), "c": rng.integers(0, 48, r).astype(np.int64),
           "w": rng.integers(0, 100, r).astype(np.int64), "big": rng.integers(0, 5000, r).astype(np.int64)}
    fact = {"fk": rng.integers(0, r, n).astype(np.int64), "m": rng.integers(1, 100, n).astype(np.int64)}
    tables = {"lineorder": fact, "d": dim}
    kinds = {"lineorder": {"fk": 0, "m": 1}, "d": {k: (0 if k == "pk" else 1) for k in dim}}
    ds = star.DeviceStar.from_tables(tables, kinds, [("fk", "d", "pk")])
    j = [Q.StarLink("fk", "d", "pk")]

    def q(i, group, flt=None):
        return Q.QuerySpec(id=f"w{i}", group=0, joins=j, filters=[] if flt is None else [flt], measure="m",
                           group_by=[Q.GroupRef(0, g) for g in group], order_by=True)

    cases = {
        "u16 ids": ([q(0, ["w"]), q(1, ["a"], Q.FilterSpec(0, "b", Q.Pred.lt(20)))], True),
        "G > 4096": ([q(2, ["big"]), q(3, ["a"])], False),
        "> 65535 tuples": ([q(4, ["a"]), q(5, ["b"]), q(6, ["c"])], False),
    }
    for name, (qs, fused) in cases.items():
        b, got = _run_batch(ds, qs)
        assert b.fused == fused, (name, b.why)
        for qq, m in zip(qs, got):
            assert np.array_equal(m, O.run_query(tables, qq)), (name, qq.id)


def test_four_link_batches(gpu_ctx, monkeypatch, capfd):
    """SSB Q4.x's shape: three queries over four links with a 175-group space,
    dangling keys (miss tuples fail every link) and a ragged tail; a second
    four-link batch with an empty fact interval (one more fail in the initial
    lane) and small group spaces.  Both run fused; every result equals the
    oracle."""
    from paper_2306_08367_b200 import query as Q, star
    monkeypatch.setenv("LAQ_BATCH_VERBOSE", "1")
    rng = np.random.default_rng(404)
    n = 4096 * 148 * 2 + 777
    sizes = (3000, 20000, 1400, 2555)
    fact = {"lo_m": rng.integers(1, 10_000, n).astype(np.int64), "lo_a": rng.integers(0, 50, n).astype(np.int64)}
    tables, kinds, links = {}, {}, []
    fk_kinds = {"lo_m": 1, "lo_a": 1}
    for d, rows in enumerate(sizes):
        name = f"d{d}"
        tables[name] = {"pk": np.arange(rows, dtype=np.int64), "x": rng.integers(0, 7, rows).astype(np.int64),
                        "y": rng.integers(0, 25, rows).astype(np.int64),
                        "z": rng.integers(0, 1000, rows).astype(np.int64)}
        kinds[name] = {"pk": 0, "x": 1, "y": 1, "z": 1}
        fk = rng.integers(0, rows, n).astype(np.int64)
        miss = rng.random(n) < 0.01
        fk[miss] = rows + rng.integers(0, 50, miss.sum())
        fact[f"lo_fk{d}"] = fk
        fk_kinds[f"lo_fk{d}"] = 0
        links.append((f"lo_fk{d}", name, "pk"))
    tables = {"lineorder": fact, **tables}
    kinds = {"lineorder": fk_kinds, **kinds}
    joins = [Q.StarLink(*l) for l in links]
    ds = star.DeviceStar.from_tables(tables, kinds, links)

    def q4(i, dial):
        return Q.QuerySpec(id=f"n{i}", group=0, joins=joins,
                           filters=[Q.FilterSpec(0, "z", Q.Pred.lt(dial)), Q.FilterSpec(1, "x", Q.Pred.lt(5)),
                                    Q.FilterSpec(3, "z", Q.Pred.between(100, 900))],
                           measure="lo_m", group_by=[Q.GroupRef(3, "x"), Q.GroupRef(1, "y")], order_by=True)

    batches = [[q4(0, 300), q4(1, 500), q4(2, 700)],
               [Q.QuerySpec(id="e", group=0, joins=joins, filters=[Q.FilterSpec(-1, "lo_a", Q.Pred.between(30, 10))],
                            measure="lo_m", group_by=[Q.GroupRef(2, "x")]),
                Q.QuerySpec(id="f", group=0, joins=joins, filters=[Q.FilterSpec(0, "x", Q.Pred.lt(3))],
                            measure="lo_m", group_by=[Q.GroupRef(2, "x")]),
                Q.QuerySpec(id="g", group=0, joins=joins, filters=[Q.FilterSpec(-1, "lo_a", Q.Pred.lt(25))],
                            measure="lo_m", group_by=[Q.GroupRef(1, "x")])]]
    for qs in batches:
        capfd.readouterr()
        b, got = _run_batch(ds, qs)
        assert b.fused, b.why
        err = capfd.readouterr().err
        assert "nl=4" in err, err
        for q, m in zip(qs, got):
            want = O.run_query(tables, q)
            assert m.shape == want.shape and np.array_equal(m, want), q.id
