"""The full-size query checker (oracle/fast_query.py + oracle/ssb_oracle.c,
a multi-threaded restatement of run_query_oracle, cli.cpp:140-225) pinned
against the reference's own goldens and the numpy restatement -- before it is
trusted at SF=10 / SF=100 in the slow GPU tests and in bench.py."""
import numpy as np
import pytest

from conftest import fa, load_golden
from oracle import fast_query as F
from oracle import laq_oracle as O


def _q(group, qid, dial):
    from paper_2306_08367_b200 import query as Q
    return Q.spec_with_dial(Q.group_defs(group)[int(qid[1]) - 1], group, dial)


@pytest.fixture(scope="module")
def sf1():
    from paper_2306_08367_b200 import gen
    return gen.gen_star("Ssb", 1, 42, narrow=True)


def test_ssb_sf1_reference_goldens(sf1):
    """all 12 SSB sf=1 queries equal the reference's results."""
    G = load_golden("ssb_sf1.json")
    for qg in G["queries"]:
        q = _q(qg["group"], qg["id"], qg["dial"])
        F.Prepared(sf1.tables, q)  # every SSB query takes the fast form (no fallback)
        m = F.run_query(sf1.tables, q, threads=4)
        assert m.shape == (qg["rows"], qg["cols"]), qg["id"]
        assert np.array_equal(m.ravel(), fa(qg["result"])), qg["id"]
        assert str(O.checksum_rows(m)) == qg["checksum"], qg["id"]


def test_row_ranges_merge_exactly(sf1):
    """partial() over row shards sums to the whole table (the multi-GPU check)."""
    n = len(sf1.fact["lo_part"])
    for grp, qi, dial in [(3, 0, 105), (4, 2, 284), (1, 0, 222)]:
        p = F.Prepared(sf1.tables, _q(grp, f"{grp}{qi + 1}", dial))
        c0, s0 = p.partial()
        cs, ss = zip(*[p.partial(n * k // 5, n * (k + 1) // 5 - n * k // 5, threads=3) for k in range(5)])
        assert np.array_equal(sum(cs), c0) and np.array_equal(sum(ss), s0)
        assert np.array_equal(p.emit(c0, s0), O.run_query(sf1.tables, p.q))


def test_row_range_equals_sliced_numpy_oracle(sf1):
    t = dict(sf1.tables)
    t["lineorder"] = {c: a[1_000_000:2_500_000] for c, a in sf1.fact.items()}
    for grp, qi, dial in [(2, 0, 50), (3, 2, 43)]:
        q = _q(grp, f"{grp}{qi + 1}", dial)
        assert np.array_equal(F.run_query(sf1.tables, q, row_range=(1_000_000, 2_500_000)), O.run_query(t, q))


def test_random_stars_match_numpy_oracle():
    from test_gpu_query_fuzz import _random_case
    fast = 0
    for seed in range(80):
        tables, kinds, links, q = _random_case(seed)
        try:
            F.Prepared(tables, q)
            fast += 1
        except F.Unsupported:
            pass
        assert np.array_equal(F.run_query(tables, q, threads=3), O.run_query(tables, q)), seed
    assert fast >= 10
