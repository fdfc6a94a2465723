"""CPU: pin the numpy restatement (oracle/laq_oracle.py) to the reference.

Golden vectors were produced by the reference's own compiled code
(tests/golden/make_golden.py); the known answers come from the reference's
tests (test_laqops.cpp, test_fusion.cpp, acceptance.cpp).  When the compiled
reference is present (this container), also cross-check it live.
"""
import numpy as np
import pytest

from conftest import fa, ia, load_golden
from oracle import laq_oracle as O

OPS = load_golden("ops.json")
FUS = load_golden("fusion.json")


def test_key_domain_worked_example():
    # test_laqops.cpp:155-162
    d = O.build_key_domain([1, 0, 4, 2, 3], [2, 3, 0, 4, 7])
    assert d.tolist() == [0, 1, 2, 3, 4, 7] == OPS["domain_example"]["out"]
    assert O.position(d, [7]).tolist() == [5]
    with pytest.raises(O.DomainError):
        O.position(d, [6])
    with pytest.raises(O.DomainError):
        O.build_key_domain([-1], [2, 4])
    assert OPS["domain_negative_code"] == 8


def test_key_domains_random_and_update():
    for c in OPS["domains"]:
        d = O.build_key_domain(c["r"], c["s"])
        assert d.tolist() == c["out"]
        assert O.update_key_domain(d, c["new"]).tolist() == c["updated"]


def test_key_matrix_examples():
    g = OPS["key_matrix_example"]
    rp, ci, vv = O.key_matrix(g["keys"], g["domain"], "RowsByDomain")
    assert rp.tolist() == g["rbd"]["row_ptr"] and ci.tolist() == g["rbd"]["col_idx"] == [2, 3, 0, 4, 5]
    rp, ci, vv = O.key_matrix(g["keys"], g["domain"], "DomainByRows")
    assert rp.tolist() == g["dbr"]["row_ptr"] and ci.tolist() == g["dbr"]["col_idx"]
    v = OPS["key_matrix_valued"]
    rp, ci, vv = O.key_matrix(v["keys"], v["domain"], "RowsByDomain", fa(v["values_in"]))
    assert ci.tolist() == v["col_idx"] and np.array_equal(vv, fa(v["values"]))
    with pytest.raises(O.DomainError):
        O.key_matrix([9], g["domain"])


def test_mm_join_golden():
    for c in OPS["mm_join"]:
        r, s = O.mm_join(c["r"], c["s"])
        assert r.tolist() == c["out_r"] and s.tolist() == c["out_s"]


def test_star_join_golden():
    for c in OPS["star_join"]:
        surv, rows = O.multiway_star_join(c["fks"], c["pks"])
        assert surv.tolist() == c["survivors"]
        assert [r.tolist() for r in rows] == c["dim_rows"]
    with pytest.raises(O.DuplicateKeyError):
        O.multiway_star_join([[0, 1]], [[0, 0]])
    assert OPS["star_join_dup_code"] == 9


def test_groupby_golden():
    e = OPS["groupby_single_example"]  # test_laqops.cpp:399-412
    g, s = O.groupby_sum_single(e["kr"], fa(e["vr"]), e["ks"], e["gs"])
    assert g.tolist() == e["groups"] == [0, 1, 2]
    assert s.tolist() == fa(e["sums"]).tolist() == [1000.0, 10010.0, 100.0]
    for c in OPS["groupby_single"]:
        g, s = O.groupby_sum_single(c["kr"], fa(c["vr"]), c["ks"], c["gs"])
        assert g.tolist() == c["groups"]
        assert np.array_equal(s, fa(c["sums"]))
    for c in OPS["groupby_multi"]:
        k, s = O.groupby_sum_multi(c["cols"], fa(c["vals"]))
        assert [x.tolist() for x in k] == c["keys"]
        assert np.array_equal(s, fa(c["sums"]))  # row-order sums: bit-exact


def _star(c):
    dims = [fa(d["data"], (d["rows"], d["cols"])) for d in c["dims"]]
    L = fa(c["L"]["data"], (c["L"]["k"], c["L"]["l"]))
    return dims, c["placements"], L, [ia(i) for i in c["idx"]]


def test_fusion_golden_bit_exact():
    for c in FUS["stars"]:
        dims, pls, L, idx = _star(c)
        parts = O.prefuse_linear(dims, pls, L)
        for p, want in zip(parts, c["partials"]):
            assert np.array_equal(p.ravel(), fa(want))
        if len(idx[0]):
            Y = O.apply_fused_linear(idx, parts)
            assert np.array_equal(Y.ravel(), fa(c["Y"]))
            T = O.materialize(idx, dims, pls, L.shape[0])
            assert np.array_equal(T.ravel(), fa(c["T"]))
            assert np.array_equal(O.predict_linear(T, L).ravel(), fa(c["Y_nonfused"]))
            # fused vs non-fused agree to the reference's own 1e-9 (test_fusion.cpp:133-150)
            yn = fa(c["Y_nonfused"])
            rel = np.abs(Y.ravel() - yn) / np.maximum(np.maximum(np.abs(Y.ravel()), np.abs(yn)), 1e-300)
            assert np.all((Y.ravel() == yn) | (rel <= 1e-9))


def test_matmul_golden_bit_exact():
    for c in FUS["matmul"]:
        a = fa(c["a"], (c["m"], c["k"]))
        b = fa(c["b"], (c["k"], c["n"]))
        assert np.array_equal(O.dense_matmul(a, b).ravel(), fa(c["c"]))


def test_cost_model_golden():
    for c in FUS["cost"]:
        assert O.speedup_ratio_linear(c["i"], c["k"], c["l"], c["dims"]) == float.fromhex(c["linear"])
        assert O.speedup_ratio_tree(c["i"], c["k"], c["l"], c["dims"]) == float.fromhex(c["tree"])
        assert O.decide_fusion(float.fromhex(c["linear"])) == c["fuse"]
    # test_fusion.cpp:350-355 and 421-427
    assert O.speedup_ratio_linear(1_000_000, 128, 2, [100_000]) > 64.0
    assert not O.decide_fusion(1.0) and O.decide_fusion(1.5, 1.2) and not O.decide_fusion(1.2, 1.2)
    with pytest.raises(O.DomainError):
        O.speedup_ratio_linear(0, 8, 2, [100])
    assert FUS["placement_errors"] == {"overlap": 7, "gap": 3, "range": 7}


def test_placement_errors():
    with pytest.raises(O.MappingError):
        O.check_placements([[0, 1], [1, 2]], 3)
    with pytest.raises(O.ShapeError):
        O.check_placements([[0, 1]], 3)


def _tables_from_ref_or_gen(setting, sf, seed):
    from paper_2306_08367_b200 import gen
    try:
        g = gen.gen_star(setting, sf, seed)
    except Exception:
        pytest.skip("native generator not built")
    return g


def test_ssb_queries_golden_s2():
    """run_query restatement == reference results (S2 sf=2, seed 42), checksums equal."""
    from paper_2306_08367_b200 import query as Q
    G = load_golden("ssb_s2_sf2.json")
    g = _tables_from_ref_or_gen(G["setting"], G["sf"], G["seed"])
    for qg in G["queries"]:
        q = Q.spec_with_dial(Q.group_defs(qg["group"])[int(qg["id"][1]) - 1], qg["group"], qg["dial"])
        m = O.run_query(g.tables, q)
        assert m.shape == (qg["rows"], qg["cols"])
        assert np.array_equal(m.ravel(), fa(qg["result"])), qg["id"]
        assert str(O.checksum_rows(m)) == qg["checksum"]
        assert O.measure_selectivity(g.tables, q) == float.fromhex(qg["selectivity"])


def test_gen_queries_restatement_picks_reference_dials():
    """query.gen_queries (benchgen.cpp:413-457 restated) + the oracle's
    measure_selectivity choose exactly the reference's dial constants."""
    from paper_2306_08367_b200 import query as Q
    G = load_golden("ssb_s2_sf2.json")
    g = _tables_from_ref_or_gen(G["setting"], G["sf"], G["seed"])
    for grp in (1, 2, 3, 4):
        qs = Q.gen_queries(lambda q: O.measure_selectivity(g.tables, q), grp)
        want = [x for x in G["queries"] if x["group"] == grp]
        assert [q.filters[-1].pred.lo for q in qs] == [w["dial"] for w in want]
        assert [q.realized_selectivity for q in qs] == [float.fromhex(w["realized"]) for w in want]


@pytest.mark.skipif(not __import__("oracle.ref", fromlist=["available"]).available(),
                    reason="compiled reference (oracle/_ref) not present")
def test_live_reference_agrees_with_restatement():
    from oracle import ref
    rng = np.random.default_rng(5)
    for _ in range(5):
        r = rng.integers(0, 50, 300)
        s = rng.integers(0, 50, 200)
        a, b = ref.mm_join(r, s)
        c, d = O.mm_join(r, s)
        assert np.array_equal(a, c) and np.array_equal(b, d)
        assert np.array_equal(ref.build_key_domain(r, s), O.build_key_domain(r, s))


def test_tree_oracle_matches_reference():
    """The numpy restatement of compile_tree / predict_tree / partition_tree /
    prefuse_tree / apply_fused_tree against the reference compiled from its own
    sources (bench::gen_tree trees): labels and partials bit-identical."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(1)
    for trial in range(12):
        k = int(rng.integers(2, 40))
        leaves = int(rng.integers(2, 60))
        t = ref.gen_tree(k, int(rng.integers(1, k + 1)), leaves, trial)
        X = rng.random((300, k))
        assert np.array_equal(ref.predict_tree(t, X), O.predict_tree(X, O.compile_tree(t, k)))
        perm = rng.permutation(k)
        cut = int(rng.integers(1, k)) if k > 1 else k
        pl = [perm[:cut], perm[cut:]] if cut < k else [perm]
        owner = np.zeros(k, np.int64)
        for j, p in enumerate(pl):
            owner[p] = j
        dims = [rng.random((int(rng.integers(5, 50)), len(p))) for p in pl]
        idx = [rng.integers(0, d.shape[0], 200) for d in dims]
        ya, pa = ref.fused_tree(t, dims, pl, k, owner, idx)
        comp = O.compile_tree(t, k)
        pb = O.prefuse_tree(dims, pl, O.partition_tree(comp, owner, len(dims)))
        assert all(np.array_equal(x, y) for x, y in zip(pa, pb))
        assert np.array_equal(ya, O.apply_fused_tree(idx, pb, comp[3], comp[4]))
