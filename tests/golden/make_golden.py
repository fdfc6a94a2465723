"""Generate the golden vectors in tests/golden/*.json from the REFERENCE itself.

Runs the reference's own C++ implementation (compiled unmodified from
/root/reference/proj/src by oracle/Makefile into oracle/_ref/liblaq_ref.so) on
small seeded inputs and records inputs + outputs.  Floats are stored as
float.hex() strings so comparisons can be bit-exact.  Run in the dev
container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

The GPU box never runs this; it only reads the committed JSON.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2306_08367_b200 import query as Q  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def fx(a):
    return [float(v).hex() for v in np.asarray(a, np.float64).ravel()]


def il(a):
    return [int(v) for v in np.asarray(a).ravel()]


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name)


def err_code(fn):
    try:
        fn()
        return 0
    except ref.RefError as e:
        return e.code


def ops_golden():
    rng = np.random.default_rng(20260101)
    g = {}
    # Worked examples (test_laqops.cpp:155-228, acceptance.cpp:108-144).
    g["domain_example"] = {"r": [1, 0, 4, 2, 3], "s": [2, 3, 0, 4, 7],
                           "out": il(ref.build_key_domain([1, 0, 4, 2, 3], [2, 3, 0, 4, 7]))}
    g["domain_negative_code"] = err_code(lambda: ref.build_key_domain([-1], [2, 4]))
    dom = ref.build_key_domain([1, 0, 4, 2, 3], [2, 3, 0, 4, 7])
    rp, ci, vv = ref.key_matrix([2, 3, 0, 4, 7], dom, "RowsByDomain")
    rp2, ci2, vv2 = ref.key_matrix([2, 3, 0, 4, 7], dom, "DomainByRows")
    g["key_matrix_example"] = {"keys": [2, 3, 0, 4, 7], "domain": il(dom),
                               "rbd": {"row_ptr": il(rp), "col_idx": il(ci), "values": fx(vv)},
                               "dbr": {"row_ptr": il(rp2), "col_idx": il(ci2), "values": fx(vv2)}}
    g["key_matrix_missing_code"] = err_code(lambda: ref.key_matrix([9], dom, "RowsByDomain"))
    d2 = ref.build_key_domain([1, 5], [])
    rp, ci, vv = ref.key_matrix([5, 1], d2, "RowsByDomain", values=[10.0, 20.0])
    g["key_matrix_valued"] = {"keys": [5, 1], "domain": il(d2), "values_in": fx([10.0, 20.0]),
                              "row_ptr": il(rp), "col_idx": il(ci), "values": fx(vv)}
    # Random domains / updates.
    g["domains"] = []
    for _ in range(12):
        a = rng.integers(0, int(rng.integers(1, 5000)), int(rng.integers(0, 300)))
        b = rng.integers(0, 100000, int(rng.integers(0, 300)))
        c = rng.integers(0, 1 << 40, int(rng.integers(1, 50)))
        d = ref.build_key_domain(a, b)
        g["domains"].append({"r": il(a), "s": il(b), "out": il(d), "new": il(c),
                             "updated": il(ref.update_key_domain(d, c))})
    # mm_join (many-to-many with duplicates).
    g["mm_join"] = []
    for _ in range(16):
        uni = int(rng.integers(1, 60))
        r = rng.integers(0, uni, int(rng.integers(0, 200)))
        s = rng.integers(0, uni, int(rng.integers(0, 200)))
        orr, oss = ref.mm_join(r, s)
        g["mm_join"].append({"r": il(r), "s": il(s), "out_r": il(orr), "out_s": il(oss)})
    # Star joins (test_laqops.cpp:264-301 style: iota pks, fks past the key space).
    g["star_join"] = []
    for _ in range(10):
        n = int(rng.integers(0, 600))
        pks, fks = [], []
        for _d in range(3):
            rows = int(rng.integers(1, 60))
            pk = rng.permutation(rows * 3)[:rows] if rng.random() < 0.5 else np.arange(rows)
            pks.append(pk.astype(np.int64))
            fks.append(rng.integers(0, int(pk.max()) + 9, n))
        surv, rows_ = ref.star_join(fks, pks)
        g["star_join"].append({"fks": [il(f) for f in fks], "pks": [il(p) for p in pks],
                               "survivors": il(surv), "dim_rows": [il(x) for x in rows_]})
    g["star_join_dup_code"] = err_code(lambda: ref.star_join([np.array([0, 1])], [np.array([0, 0])]))
    # Aggregation.
    ks = [2, 3, 0, 4, 7]
    gs = [0, 1, 1, 2, 2]
    kr = [1, 0, 4, 2, 3]
    vr = [1.0, 10.0, 100.0, 1000.0, 10000.0]
    og, osm = ref.groupby_sum_single(kr, vr, ks, gs)
    g["groupby_single_example"] = {"kr": kr, "vr": fx(vr), "ks": ks, "gs": gs, "groups": il(og), "sums": fx(osm)}
    g["groupby_single"] = []
    for _ in range(10):
        nr, ns = int(rng.integers(0, 300)), int(rng.integers(1, 200))
        kr = rng.integers(0, 40, nr)
        vr = np.round(rng.normal(size=nr) * 100) / 4  # exactly representable
        ks = rng.integers(0, 40, ns)
        gs = rng.integers(-5, 12, ns)
        og, osm = ref.groupby_sum_single(kr, vr, ks, gs)
        g["groupby_single"].append({"kr": il(kr), "vr": fx(vr), "ks": il(ks), "gs": il(gs),
                                    "groups": il(og), "sums": fx(osm)})
    g["groupby_multi"] = []
    for _ in range(10):
        n = int(rng.integers(1, 400))
        cols = [rng.integers(-3, int(rng.integers(1, 9)), n) for _c in range(int(rng.integers(1, 4)))]
        vals = rng.normal(size=n)
        keys, sums = ref.groupby_sum_multi(cols, vals)
        g["groupby_multi"].append({"cols": [il(c) for c in cols], "vals": fx(vals),
                                   "keys": [il(k) for k in keys], "sums": fx(sums)})
    dump("ops.json", g)


def fusion_golden():
    rng = np.random.default_rng(777)
    g = {"stars": [], "matmul": [], "cost": [], "placement_errors": {}}
    for _ in range(10):
        nd = int(rng.integers(1, 4))
        widths = [int(rng.integers(1, 6)) for _d in range(nd)]
        k = sum(widths)
        l = int(rng.choice([1, 2, 3, 5, 16]))
        dims, pls, idx = [], [], []
        perm = rng.permutation(k)
        off = 0
        m = int(rng.integers(0, 300))
        for w in widths:
            rows = int(rng.integers(5, 65))
            dims.append(rng.random((rows, w)) * 2 - 1)
            pls.append(perm[off: off + w].astype(np.int64))
            off += w
            idx.append(rng.integers(0, rows, m))
        L = rng.random((k, l)) * 2 - 1
        parts = ref.prefuse_linear(dims, pls, L)
        Y = ref.apply_fused_linear(idx, parts) if m else np.zeros((0, l))
        T, Yn = ref.materialize_predict(dims, pls, k, idx, L) if m else (np.zeros((0, k)), np.zeros((0, l)))
        g["stars"].append({"dims": [{"rows": d.shape[0], "cols": d.shape[1], "data": fx(d)} for d in dims],
                           "placements": [il(p) for p in pls], "L": {"k": k, "l": l, "data": fx(L)},
                           "idx": [il(i) for i in idx], "partials": [fx(p) for p in parts], "Y": fx(Y),
                           "T": fx(T), "Y_nonfused": fx(Yn)})
    for _ in range(6):
        m, kk, n = int(rng.integers(1, 70)), int(rng.integers(1, 40)), int(rng.integers(1, 70))
        a = rng.random((m, kk)) * 2 - 1
        a[rng.random((m, kk)) < 0.2] = 0.0
        b = rng.random((kk, n)) * 2 - 1
        g["matmul"].append({"m": m, "k": kk, "n": n, "a": fx(a), "b": fx(b), "c": fx(ref.dense_matmul(a, b))})
    for ke in range(4, 12):
        for le in range(1, 12, 2):
            i = int(rng.integers(1000, 1000000))
            dims = [int(rng.integers(500, 20000)), 2555, int(rng.integers(1000, 6000))]
            g["cost"].append({"i": i, "k": 1 << ke, "l": 1 << le, "dims": dims,
                              "linear": float(ref.speedup_ratio(i, 1 << ke, 1 << le, dims)).hex(),
                              "tree": float(ref.speedup_ratio(i, 1 << ke, 1 << le, dims, tree=True)).hex(),
                              "fuse": ref.decide_fusion(ref.speedup_ratio(i, 1 << ke, 1 << le, dims))})
    d1 = [rng.random((4, 2))]
    g["placement_errors"]["overlap"] = err_code(lambda: ref.prefuse_linear(d1 * 2, [[0, 1], [1, 2]], np.ones((3, 1))))
    g["placement_errors"]["gap"] = err_code(lambda: ref.prefuse_linear(d1, [[0, 1]], np.ones((3, 1))))
    g["placement_errors"]["range"] = err_code(lambda: ref.prefuse_linear(d1, [[0, 5]], np.ones((2, 1))))
    dump("fusion.json", g)


def arr_hash(a) -> str:
    from oracle.laq_oracle import fnv1a
    return "%016x" % fnv1a(np.ascontiguousarray(a).tobytes())


def ssb_golden(setting, sf, seed, name, groups=(1, 2, 3, 4)):
    s = ref.gen_star(setting, sf=sf, seed=seed)
    out = {"setting": setting, "sf": sf, "seed": seed, "tables": {}, "queries": []}
    for t, cols in s.tables.items():
        out["tables"][t] = {c: {"rows": len(a), "fnv": arr_hash(a.astype(np.int64) if a.dtype != np.float64 else a)}
                            for c, a in cols.items()}
    for grp in groups:
        dials, real = ref.gen_queries(s, grp)
        for qi, d in enumerate(Q.group_defs(grp)):
            q = Q.spec_with_dial(d, grp, int(dials[qi]))
            m, secs = ref.run_query(s, q)
            out["queries"].append({"id": d.id, "group": grp, "dial": int(dials[qi]), "realized": float(real[qi]).hex(),
                                   "rows": m.shape[0], "cols": m.shape[1], "result": fx(m),
                                   "checksum": str(ref.checksum_rows(m)), "selectivity": float(
                                       ref.measure_selectivity(s, q)).hex()})
            print(f"  {setting} sf={sf} Q{d.id}: dial={dials[qi]} rows={m.shape[0]} ({secs:.2f}s)")
    dump(name, out)


def cfg1_golden():
    from paper_2306_08367_b200 import gen
    fk, pk, feats, W = gen.cfg1_inputs(n_fact=20000, dim_rows=300, k=16, l=1)
    Y, secs = ref.fused_pipeline([fk], [pk], [feats], W)
    dump("cfg1_small.json", {"n_fact": 20000, "dim_rows": 300, "k": 16, "l": 1, "fk_fnv": arr_hash(fk),
                             "feats_fnv": arr_hash(feats), "W": fx(W), "Y_fnv": arr_hash(Y),
                             "checksum": str(ref.checksum_rows(Y)), "Y_head": fx(Y[:16])})


if __name__ == "__main__":
    what = sys.argv[1:] or ["ops", "fusion", "s2", "cfg1", "ssb1"]
    if "ops" in what:
        ops_golden()
    if "fusion" in what:
        fusion_golden()
    if "cfg1" in what:
        cfg1_golden()
    if "s2" in what:
        ssb_golden("S2", 2, 42, "ssb_s2_sf2.json")
        ssb_golden("Ssb", 1, 7, "ssb_tiny_check.json", groups=(1,)) if False else None
    if "ssb1" in what:
        ssb_golden("Ssb", 1, 42, "ssb_sf1.json")
