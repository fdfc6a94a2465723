"""GPU parity: every C-ABI operator vs the reference's golden vectors and the
pinned oracle.  Bar: bit-exact for keys / indices / integer aggregates, and
bit-exact for the fp64 fused-prediction paths too (same association order),
and for groupby_sum_single's fp64 sums (each group's terms summed in
ascending R-row order, laqops.cpp:404-405)."""
import numpy as np
import pytest

from conftest import fa, ia, load_golden
from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu

OPS = load_golden("ops.json")
FUS = load_golden("fusion.json")


@pytest.fixture(scope="module")
def lib(gpu_ctx):
    from paper_2306_08367_b200 import errors, fusion, ops
    return ops, fusion, errors


def test_key_domain(lib):
    ops, _, errors = lib
    d = ops.build_key_domain(np.array([1, 0, 4, 2, 3]), np.array([2, 3, 0, 4, 7]))
    assert d.sorted_keys.tolist() == [0, 1, 2, 3, 4, 7]
    assert d.position(7) == 5
    with pytest.raises(errors.DomainError):
        d.position(6)
    with pytest.raises(errors.DomainError):
        ops.build_key_domain(np.array([-1]), np.array([2, 4]))
    for c in OPS["domains"]:
        d = ops.build_key_domain(ia(c["r"]), ia(c["s"]))
        assert d.sorted_keys.tolist() == c["out"]
        assert ops.update_key_domain(d, ia(c["new"])).sorted_keys.tolist() == c["updated"]


def test_key_domain_large_and_wide(lib):
    ops, _, _ = lib
    rng = np.random.default_rng(1)
    for hi in (1000, 1 << 26, 1 << 45):  # bitmap path, big bitmap, radix-sort path
        a = rng.integers(0, hi, 500_000)
        b = rng.integers(0, hi, 30_000)
        assert np.array_equal(ops.build_key_domain(a, b).sorted_keys, O.build_key_domain(a, b))


def test_key_encoding_dense_unaligned(lib):
    """The shared-memory bitmap path (a dense key range whose bitmap fits one
    CTA: 1.5M keys, 4M rows) and the vectorised position lookups, on device
    views 8 bytes off a 16-byte boundary (scalar head/tail) and with odd
    lengths; a key outside the domain still raises DomainError."""
    import torch
    ops, _, errors = lib
    rng = np.random.default_rng(5)
    for hi, na, nb in ((1_500_000, 4_000_001, 3), (1000, 70_001, 0), (50_000, 3_333_333, 17)):
        a = rng.integers(0, hi, na)
        b = rng.integers(0, hi, nb)
        da = torch.from_numpy(np.concatenate([[0], a])).cuda()[1:]
        db = torch.from_numpy(np.concatenate([[0], b])).cuda()[1:]
        want = O.build_key_domain(a, b)
        d = ops.build_key_domain(da, db)
        got = d.sorted_keys.cpu().numpy() if hasattr(d.sorted_keys, "cpu") else d.sorted_keys
        assert np.array_equal(got, want), hi
        m = ops.key_matrix(da, ops.KeyDomain(want), "RowsByDomain")
        assert np.array_equal(np.asarray(m.col_idx), np.searchsorted(want, a)), hi
    with pytest.raises(errors.DomainError):
        keys = torch.from_numpy(np.concatenate([[0], np.arange(1000), [5000]])).cuda()[1:]
        ops.key_matrix(keys, ops.KeyDomain(np.arange(1000)), "RowsByDomain")


def test_key_matrix(lib):
    ops, _, errors = lib
    g = OPS["key_matrix_example"]
    d = ops.KeyDomain(ia(g["domain"]))
    m = ops.key_matrix(ia(g["keys"]), d, "RowsByDomain")
    assert m.row_ptr.tolist() == g["rbd"]["row_ptr"] and m.col_idx.tolist() == g["rbd"]["col_idx"]
    m = ops.key_matrix(ia(g["keys"]), d, "DomainByRows")
    assert m.row_ptr.tolist() == g["dbr"]["row_ptr"] and m.col_idx.tolist() == g["dbr"]["col_idx"]
    v = OPS["key_matrix_valued"]
    m = ops.key_matrix(ia(v["keys"]), ops.KeyDomain(ia(v["domain"])), "RowsByDomain", fa(v["values_in"]))
    assert m.col_idx.tolist() == v["col_idx"] and np.array_equal(m.values, fa(v["values"]))
    with pytest.raises(errors.DomainError):
        ops.key_matrix(ia([9]), d, "RowsByDomain")
    rng = np.random.default_rng(2)
    keys = rng.integers(0, 5000, 200_000)
    vals = rng.integers(-2, 3, 200_000).astype(np.float64)
    dom = O.build_key_domain(keys, [])
    rp, ci, vv = O.key_matrix(keys, dom, "DomainByRows", vals)
    m = ops.key_matrix(keys, ops.KeyDomain(dom), "DomainByRows", vals)
    assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci) and np.array_equal(m.values, vv)
    # row pointers both ways: a domain much smaller than the entries (per-position
    # search) and a big domain with long empty runs (one pass over the entries)
    for dom, keys in ((np.arange(64), rng.integers(0, 64, 300_000)),
                      (np.arange(100_000), rng.choice(np.array([5, 50_000, 99_999]), 3_000))):
        rp, ci, _ = O.key_matrix(keys, dom, "DomainByRows")
        m = ops.key_matrix(keys, ops.KeyDomain(dom), "DomainByRows")
        assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci)


def test_mm_join(lib):
    ops, _, errors = lib
    for c in OPS["mm_join"]:
        m = ops.mm_join(ia(c["r"]), ia(c["s"]))
        assert m.row_idx.tolist() == c["out_r"] and m.col_idx.tolist() == c["out_s"]
    rng = np.random.default_rng(3)
    r = rng.integers(0, 3000, 100_000)
    s = rng.integers(0, 3000, 20_000)
    m = ops.mm_join(r, s)
    a, b = O.mm_join(r, s)
    assert np.array_equal(m.row_idx, a) and np.array_equal(m.col_idx, b)
    # cached superset domain gives identical output (test_laqops.cpp:256-262)
    dom = ops.update_key_domain(ops.build_key_domain(r, s), rng.integers(0, 6000, 500))
    m2 = ops.mm_join(r, s, dom)
    assert np.array_equal(m2.row_idx, a) and np.array_equal(m2.col_idx, b)
    assert ops.mm_join(ia([1, 2]), ia([3, 4])).nnz() == 0
    with pytest.raises(errors.DomainError):
        ops.mm_join(ia([-3]), ia([1]))


def test_star_join(lib):
    ops, _, errors = lib
    for c in OPS["star_join"]:
        surv, rows = ops.multiway_star_join([ia(f) for f in c["fks"]], [ia(p) for p in c["pks"]])
        assert surv.tolist() == c["survivors"]
        assert [r.tolist() for r in rows] == c["dim_rows"]
    with pytest.raises(errors.DuplicateKeyError):
        ops.multiway_star_join([ia([0, 1])], [ia([0, 0])])
    # trivial cases (test_laqops.cpp:303-322)
    surv, rows = ops.multiway_star_join([ia([2, 0, 1, 2])], [ia([0, 1, 2])])
    assert surv.tolist() == [0, 1, 2, 3]
    surv, rows = ops.multiway_star_join([ia([2, 0, 1, 2])] * 2, [ia([0, 1, 2]), ia([])])
    assert len(surv) == 0 and all(len(r) == 0 for r in rows)


def test_star_join_large_direct_and_hash(lib):
    ops, _, _ = lib
    rng = np.random.default_rng(4)
    n = 3_000_000
    pks = [np.arange(800_000), rng.permutation(1 << 40)[:0] if False else rng.choice(1 << 40, 20_000, replace=False),
           np.arange(2555) * 7 + 11]
    fks = [rng.integers(0, 900_000, n), np.where(rng.random(n) < 0.8, pks[1][rng.integers(0, 20_000, n)], 5),
           rng.integers(0, 2555 * 7 + 20, n)]
    surv, rows = ops.multiway_star_join(fks, pks)
    ws, wr = O.multiway_star_join(fks, pks)
    assert np.array_equal(surv, ws)
    for a, b in zip(rows, wr):
        assert np.array_equal(a, b)


def test_groupby(lib):
    ops, _, errors = lib
    e = OPS["groupby_single_example"]
    g, s = ops.groupby_sum_single(ia(e["kr"]), fa(e["vr"]), ia(e["ks"]), ia(e["gs"]))
    assert g.tolist() == [0, 1, 2] and s.tolist() == [1000.0, 10010.0, 100.0]
    for c in OPS["groupby_single"]:
        g, s = ops.groupby_sum_single(ia(c["kr"]), fa(c["vr"]), ia(c["ks"]), ia(c["gs"]))
        assert g.tolist() == c["groups"] and np.array_equal(s, fa(c["sums"]))
    for c in OPS["groupby_multi"]:  # row-order segmented sums: bit-exact
        k, s = ops.groupby_sum_multi([ia(x) for x in c["cols"]], fa(c["vals"]))
        assert [x.tolist() for x in k] == c["keys"] and np.array_equal(s, fa(c["sums"]))
    rng = np.random.default_rng(6)
    kr = rng.integers(0, 500, 100_000)
    vr = rng.normal(size=100_000)
    ks = rng.integers(0, 500, 700)
    gs = rng.integers(0, 30, 700)
    g, s = ops.groupby_sum_single(kr, vr, ks, gs)
    wg, ws = O.groupby_sum_single(kr, vr, ks, gs)
    assert np.array_equal(g, wg)
    assert np.array_equal(s, ws)  # R-row-ordered sums: bit-identical, run to run too
    g2, s2 = ops.groupby_sum_single(kr, vr, ks, gs)
    assert np.array_equal(s2, s)


def test_groupby_multi_large_signed_wide(lib):
    """groupby_sum_multi at scale vs the oracle, bit-exact: long fp64 segments
    (thousands of rows, lengths not multiples of 32: the warp fold's partial
    chunks), a negative-valued column (the bitmap distinct path with a negative
    base), a column spanning more than 2^31 (the radix-sort distinct path) and
    a single-column case."""
    ops, _, _ = lib
    rng = np.random.default_rng(9)
    n = 400_003
    a = rng.integers(-3, 4, n)
    b = rng.integers(0, 25, n)
    w = rng.choice(np.array([-(1 << 40), 5, 1 << 41]), n)
    v = rng.normal(size=n) * 1e3
    for cols in ([a, b], [w, a], [b]):
        k, sums = ops.groupby_sum_multi(cols, v)
        wk, ws = O.groupby_sum_multi(cols, v)
        assert all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(k, wk))
        assert np.array_equal(sums, ws)


def _star(c):
    dims = [fa(d["data"], (d["rows"], d["cols"])) for d in c["dims"]]
    L = fa(c["L"]["data"], (c["L"]["k"], c["L"]["l"]))
    return dims, c["placements"], L, [ia(i) for i in c["idx"]]


def test_fusion_bit_exact(lib):
    ops, fusion, errors = lib
    for c in FUS["stars"]:
        dims, pls, L, idx = _star(c)
        f = fusion.prefuse_linear(dims, pls, L)
        for p, want in zip(f.partials, c["partials"]):
            assert np.array_equal(p.ravel(), fa(want))
        if len(idx[0]) == 0:
            continue
        assert np.array_equal(fusion.apply_fused_linear(idx, f).ravel(), fa(c["Y"]))
        T = ops.materialize(idx, dims, pls, L.shape[0])
        assert np.array_equal(T.ravel(), fa(c["T"]))
        assert np.array_equal(fusion.predict_linear(T, L).ravel(), fa(c["Y_nonfused"]))
    for c in FUS["matmul"]:
        a = fa(c["a"], (c["m"], c["k"]))
        b = fa(c["b"], (c["k"], c["n"]))
        assert np.array_equal(fusion.dense_matmul(a, b).ravel(), fa(c["c"]))
    d1 = [np.random.default_rng(0).random((4, 2))]
    with pytest.raises(errors.MappingError):
        fusion.prefuse_linear(d1 * 2, [[0, 1], [1, 2]], np.ones((3, 1)))
    with pytest.raises(errors.ShapeError):
        fusion.prefuse_linear(d1, [[0, 1]], np.ones((3, 1)))


def test_fused_star_predict_cfg1_small(lib):
    _, fusion, _ = lib
    from paper_2306_08367_b200 import gen
    G = load_golden("cfg1_small.json")
    fk, pk, feats, W = gen.cfg1_inputs(G["n_fact"], G["dim_rows"], G["k"], G["l"])
    f = fusion.prefuse_linear([feats], [np.arange(16)], W)
    y, surv = fusion.fused_star_predict([fk], [pk], f.partials)
    assert str(O.checksum_rows(y)) == G["checksum"]
    assert [float(v).hex() for v in y[:16].ravel()] == G["Y_head"]
    assert np.array_equal(surv, np.arange(G["n_fact"]))


@pytest.mark.parametrize("l", [1, 3, 8, 40])
def test_fused_star_predict_multi_dim(lib, l):
    _, fusion, _ = lib
    rng = np.random.default_rng(10 + l)
    n = 1_234_567
    rows = [2000, 517, 2555]
    pks = [np.arange(r) + 3 for r in rows]
    fks = [rng.integers(0, r + 10, n) for r in rows]
    ks = [6, 5, 5]
    dims = [rng.random((r, k)) for r, k in zip(rows, ks)]
    pls = [np.arange(0, 6), np.arange(6, 11), np.arange(11, 16)]
    L = rng.random((16, l)) * 2 - 1
    f = fusion.prefuse_linear(dims, pls, L)
    y, surv = fusion.fused_star_predict(fks, pks, f.partials)
    ws, wr = O.multiway_star_join(fks, pks)
    wy = O.apply_fused_linear(wr, O.prefuse_linear(dims, pls, L))
    assert np.array_equal(surv, ws)
    assert np.array_equal(y, wy)  # bit-exact: same association as fusion.cpp:73-76


def test_predictor_graph_capturable(lib):
    import torch
    _, fusion, _ = lib
    rng = np.random.default_rng(3)
    pk = np.arange(10_000)
    fk = rng.integers(0, 10_000, 1_000_000)
    P = rng.random((10_000, 1))
    pred = fusion.FusedStarPredictor([pk], [P])
    fk_d = torch.from_numpy(fk.astype(np.int32)).cuda()
    out = torch.empty((1_000_000, 1), dtype=torch.float64, device="cuda")
    pred([fk_d], out=out, sync=False)  # warm-up (allocates look-back scratch)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pred.ctx.bind_stream(s)
        with torch.cuda.graph(g, stream=s):
            pred([fk_d], out=out, sync=False)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    pred.ctx.bind_stream()
    assert np.array_equal(out.cpu().numpy()[:, 0], P[fk, 0] + 0.0)
    assert int(pred.nnz_dev.item()) == 1_000_000


def test_predictor_miss_fallback_alternating(lib):
    """Optimistic single pass with device-decided compaction: calls with and
    without missing keys in any order (the miss counter is moved and cleared
    on the device) and graph replays over both kinds stay exact."""
    import torch
    _, fusion, _ = lib
    rng = np.random.default_rng(21)
    pk = np.arange(5_000) + 7
    P = rng.random((5_000, 1))
    pred = fusion.FusedStarPredictor([pk], [P])
    full = rng.integers(7, 5_007, 700_001)
    miss = full.copy()
    miss[rng.random(full.size) < 0.01] = 1  # keys below the domain: dropped (inner join)

    def check(fk, y, nnz):
        keep = (fk >= 7) & (fk < 5_007)
        want = P[fk[keep] - 7, 0] + 0.0
        assert nnz == keep.sum() and np.array_equal(y[:nnz, 0], want)

    for fk in (full, miss, miss, full, miss, full, full):
        fk_d = torch.from_numpy(fk.astype(np.int32)).cuda()
        out = torch.empty((fk.size, 1), dtype=torch.float64, device="cuda")
        pred([fk_d], out=out, sync=False)
        torch.cuda.synchronize()
        check(fk, out.cpu().numpy(), int(pred.nnz_dev.item()))
    # graph with one call, replayed over inputs that change between replays
    fk_d = torch.from_numpy(full.astype(np.int32)).cuda()
    out = torch.empty((full.size, 1), dtype=torch.float64, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pred.ctx.bind_stream(s)
        with torch.cuda.graph(g, stream=s):
            pred([fk_d], out=out, sync=False)
    for fk in (full, miss, full, miss, miss, full):
        fk_d.copy_(torch.from_numpy(fk.astype(np.int32)))
        g.replay()
        torch.cuda.synchronize()
        check(fk, out.cpu().numpy(), int(pred.nnz_dev.item()))
    pred.ctx.bind_stream()


@pytest.mark.parametrize("n,chunk", [(0, 0), (1, 0), (1_000_000, 0), (700_001, 65_536), (300_000, 1_000)])
def test_predictor_host_buffers_pipelined(lib, n, chunk):
    """laq_probe_fused_predict_host: keys in and predictions out in host
    memory, chunked over two copy streams; with and without missing keys (the
    per-chunk survivors are closed up on the host) -- equal to the oracle's
    fused pipeline (bit-exact) and to the device-buffer call."""
    import torch
    _, fusion, _ = lib
    rng = np.random.default_rng(31 + n)
    pk = [np.arange(4_000) + 3, np.arange(900)]
    P = [rng.random((4_000, 2)), rng.random((900, 2))]
    pred = fusion.FusedStarPredictor(pk, P)
    full = [rng.integers(3, 4_003, n), rng.integers(0, 900, n)]
    miss = [full[0].copy(), full[1]]
    miss[0][rng.random(n) < 0.02] = 5_000  # past the domain: dropped (inner join)
    for fks in (full, miss):
        keys = [torch.from_numpy(f.astype(np.int32)).pin_memory() for f in fks]
        y, nnz = pred.predict_host(keys, chunk_rows=chunk)
        ws, wr = O.multiway_star_join(fks, pk)
        want = O.apply_fused_linear(wr, P)
        assert nnz == len(ws) and np.array_equal(y.numpy(), want)
        # pageable numpy keys take the same path
        y2, nnz2 = pred.predict_host([f.astype(np.int32) for f in fks], chunk_rows=chunk)
        assert nnz2 == nnz and np.array_equal(y2.numpy(), want)
        if n:
            yd, nd = pred([torch.from_numpy(f.astype(np.int32)).cuda() for f in fks])
            assert nd == nnz and np.array_equal(yd.cpu().numpy(), want)


def test_dense_matmul_more_row_tiles_than_grid_y(gpu_ctx):
    """dense_matmul (matrix.cpp:158-174) over more than 65,535 row tiles of 64
    (the drop-in's non-fused pipeline at S2 sf=2000 multiplies 6M x 64 by 64 x 4):
    bit-exact vs the sequential oracle."""
    from paper_2306_08367_b200 import fusion
    rng = np.random.default_rng(17)
    m = 64 * 65_536 + 5
    a = rng.random((m, 3))
    a[::7, 1] = 0.0  # zero entries are skipped (matrix.cpp:168)
    b = rng.uniform(-1, 1, (3, 5))
    assert np.array_equal(np.asarray(fusion.dense_matmul(a, b)), O.dense_matmul(a, b))
