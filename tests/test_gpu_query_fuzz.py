"""GPU: random star schemas and queries vs the oracle (run_query_laq
semantics, cli.cpp:73-138), exactly.  Covers every scan variant the planner
can pick: direct (dense keys), generic stream / plain-load (hash-probed sparse
keys, fact InSet filters, fact group-by columns), dangling foreign keys
(inner join drops them), empty results, wide group spaces."""
import numpy as np
import pytest

from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu


def _random_case(seed):
    from paper_2306_08367_b200 import query as Q
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300_000))
    tables, kinds, links = {}, {}, []
    fact = {"lo_measure": rng.integers(0, 10_000, n).astype(np.int64),
            "lo_a": rng.integers(0, 50, n).astype(np.int64),
            "lo_b": rng.integers(-20, 20, n).astype(np.int64)}
    fkinds = {"lo_measure": 1, "lo_a": 1, "lo_b": 1}
    nd = int(rng.integers(1, 4))
    for d in range(nd):
        rows = int(rng.integers(1, 30_000))
        sparse = rng.random() < 0.4
        pk = (np.sort(rng.choice(5_000_000, rows, replace=False)) if sparse else np.arange(rows)).astype(np.int64)
        rng.shuffle(pk)
        name = f"dim{d}"
        tables[name] = {"pk": pk, "x": rng.integers(0, 7, rows).astype(np.int64),
                        "y": rng.integers(0, 40, rows).astype(np.int64), "z": rng.integers(0, 1000, rows).astype(np.int64)}
        kinds[name] = {"pk": 0, "x": 1, "y": 1, "z": 1}
        fk = rng.choice(pk, n)
        if rng.random() < 0.3:  # dangling keys
            miss = rng.random(n) < 0.05
            fk[miss] = pk.max() + 1 + rng.integers(0, 100, miss.sum())
        fact[f"lo_fk{d}"] = fk
        fkinds[f"lo_fk{d}"] = 0
        links.append((f"lo_fk{d}", name, "pk"))
    tables = {"lineorder": fact, **tables}
    kinds = {"lineorder": fkinds, **kinds}
    joins = [Q.StarLink(*l) for l in links]
    filters, group = [], []
    for j in range(nd):
        r = rng.random()
        if r < 0.3:
            filters.append(Q.FilterSpec(j, "x", Q.Pred.lt(int(rng.integers(1, 7)))))
        elif r < 0.5:
            filters.append(Q.FilterSpec(j, "z", Q.Pred.between(int(rng.integers(0, 500)), int(rng.integers(500, 1000)))))
        elif r < 0.65:
            filters.append(Q.FilterSpec(j, "y", Q.Pred.in_set(rng.choice(40, int(rng.integers(1, 10)), replace=False))))
        if rng.random() < 0.5:
            group.append(Q.GroupRef(j, "x" if rng.random() < 0.6 else "y"))
    r = rng.random()
    if r < 0.3:
        filters.append(Q.FilterSpec(-1, "lo_a", Q.Pred.between(int(rng.integers(0, 25)), int(rng.integers(25, 50)))))
    elif r < 0.45:
        filters.append(Q.FilterSpec(-1, "lo_b", Q.Pred.in_set(rng.choice(np.arange(-20, 20), 5, replace=False))))
    if rng.random() < 0.15:
        group.append(Q.GroupRef(-1, "lo_a"))
    q = Q.QuerySpec(id=f"fuzz{seed}", group=0, joins=joins, filters=filters, measure="lo_measure", group_by=group,
                    order_by=bool(group) and rng.random() < 0.5)
    return tables, kinds, links, q


@pytest.mark.parametrize("seed", range(40))
def test_random_star_queries_match_oracle(gpu_ctx, seed):
    from paper_2306_08367_b200 import star
    tables, kinds, links, q = _random_case(seed)
    ds = star.DeviceStar.from_tables(tables, kinds, links)
    got = ds.run_query(q)
    want = O.run_query(tables, q)
    assert got.shape == want.shape and np.array_equal(got, want), (seed, q)
