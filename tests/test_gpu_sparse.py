"""GPU parity for the matrix / selection API rows of SURVEY §8(a) that round 1
left to the reference's CPU code: spmm (matrix.cpp:81-123), csr_from_coo /
coo_from_csr (matrix.cpp:198-221) with check_canonical's errors,
row_mapping_matrices (laqops.cpp:321-336), build_selection_mask / mask_and /
apply_mask (laqops.cpp:65-121, predicate.hpp:81-103) and sort_rows
(laqops.cpp:457-478) -- each against the reference itself (oracle/_ref,
compiled from /root/reference/proj), bit-exact."""
import numpy as np
import pytest

from oracle import ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="compiled reference (oracle/_ref) not present")]


def _rand_csr(rng, rows, cols, density, ints=False):
    from paper_2306_08367_b200 import ops
    m = rng.random((rows, cols)) < density
    vals = rng.integers(-3, 4, (rows, cols)).astype(np.float64) if ints else rng.normal(size=(rows, cols))
    vals[~m] = 0.0
    rp = np.concatenate([[0], np.cumsum((vals != 0).sum(1))]).astype(np.int64)
    r, c = np.nonzero(vals)
    return ops.Csr(rows, cols, rp, c.astype(np.int64), vals[r, c])


@pytest.mark.parametrize("seed", range(8))
def test_spmm_bit_exact(gpu_ctx, seed):
    from paper_2306_08367_b200 import errors, ops
    rng = np.random.default_rng(seed)
    m, k, n = [int(x) for x in rng.integers(1, 400, 3)]
    a = _rand_csr(rng, m, k, float(rng.uniform(0.001, 0.2)), ints=seed % 2 == 0)
    b = _rand_csr(rng, k, n, float(rng.uniform(0.001, 0.2)), ints=seed % 3 == 0)
    got = ops.spmm(a, b)
    rp, ci, cv = ref.spmm(a, b)
    assert np.array_equal(got.row_ptr, rp) and np.array_equal(got.col_idx, ci)
    assert np.array_equal(got.values.view(np.int64), cv.view(np.int64))  # bit-identical, incl. zero drops
    with pytest.raises(errors.ShapeError):
        ops.spmm(a, _rand_csr(rng, k + 1, 3, 0.5))


def test_spmm_cancellation_and_empty(gpu_ctx):
    from paper_2306_08367_b200 import ops
    a = ops.Csr(2, 2, np.array([0, 2, 2]), np.array([0, 1]), np.array([1.0, -1.0]))
    b = ops.Csr(2, 1, np.array([0, 1, 2]), np.array([0, 0]), np.array([2.0, 2.0]))
    c = ops.spmm(a, b)  # 1*2 + (-1)*2 = 0: exact zero not stored (matrix.cpp:117)
    assert c.row_ptr.tolist() == [0, 0, 0] and len(c.col_idx) == 0
    e = ops.spmm(ops.Csr(3, 2, np.zeros(4, np.int64), np.zeros(0, np.int64), np.zeros(0)), b)
    assert e.row_ptr.tolist() == [0, 0, 0, 0]


def test_csr_coo_round_trip_and_errors(gpu_ctx):
    from paper_2306_08367_b200 import errors, ops
    rng = np.random.default_rng(3)
    a = _rand_csr(rng, 300, 200, 0.05)
    coo = ops.coo_from_csr(a)
    assert np.array_equal(coo.row_idx, ref.coo_from_csr(a))
    back = ops.csr_from_coo(coo)
    assert np.array_equal(back.row_ptr, a.row_ptr) and np.array_equal(back.col_idx, a.col_idx)
    assert np.array_equal(back.row_ptr, ref.csr_from_coo(coo.row_idx, coo.col_idx, coo.values, 300, 200))
    # check_canonical's messages (matrix.cpp:246-254): the first offending entry decides
    for r, c, want in [([0, 0], [1, 1], "coo: entries not sorted or duplicated"),
                       ([1, 0], [0, 0], "coo: entries not sorted or duplicated"),
                       ([0, 5], [0, 0], "coo: entry out of bounds"),
                       ([0, 1, 0], [0, -1, 9], "coo: entry out of bounds")]:
        with pytest.raises(errors.Error, match=want):
            ops.csr_from_coo(ops.Coo(3, 3, np.array(r), np.array(c), np.ones(len(r))))
        with pytest.raises(ref.RefError, match=want):
            ref.csr_from_coo(r, c, np.ones(len(r)), 3, 3)


def test_row_mapping_matrices(gpu_ctx):
    from paper_2306_08367_b200 import errors, ops
    rng = np.random.default_rng(4)
    m = ops.mm_join(rng.integers(0, 40, 500), rng.integers(0, 40, 300))
    ir, js = ops.row_mapping_matrices(m)
    assert np.array_equal(ir.col_idx, m.row_idx) and np.array_equal(js.col_idx, m.col_idx)
    assert np.array_equal(ir.row_ptr, np.arange(m.nnz() + 1)) and ir.cols == 500 and js.cols == 300
    bad = ops.RowMatch(3, 3, np.array([1, 0]), np.array([0, 0]))
    with pytest.raises(errors.Error, match="not sorted"):
        ops.row_mapping_matrices(bad)


def test_selection_masks(gpu_ctx):
    from paper_2306_08367_b200 import errors, ops
    from paper_2306_08367_b200.query import Pred, BETWEEN, EQ, GE, GT, INSET, LE, LT
    rng = np.random.default_rng(5)
    ic = rng.integers(-50, 50, 100_003)
    fc = np.round(rng.normal(size=100_003), 2)
    fc[::97] = -0.0
    fc[::101] = np.nan
    preds_i = [Pred.lt(3), Pred.le(-7), Pred.eq(0), Pred.ge(10), Pred.gt(49), Pred.between(-5, 5),
               Pred.in_set([-50, 3, 7, 7, 42]), Pred.in_set([])]
    preds_f = [Pred.flt(LT, 0.0), Pred.flt(LE, -0.5), Pred.flt(EQ, 0.0), Pred.flt(GE, 1.25), Pred.flt(GT, 0.0),
               Pred.flt(BETWEEN, -0.3, 0.3), Pred.flt(INSET, values=[0.0, -1.5, 0.25, 1.0])]
    for p in preds_i:
        assert np.array_equal(ops.build_selection_mask(ic, p), ref.selection_mask(ic, p)), p
    for p in preds_f:
        assert np.array_equal(ops.build_selection_mask(fc, p), ref.selection_mask(fc, p)), p
    with pytest.raises(errors.TypeError_, match="predicate constant is float, column is integer"):
        ops.build_selection_mask(ic, preds_f[0])
    with pytest.raises(errors.TypeError_, match="predicate constant is integer, column is float"):
        ops.build_selection_mask(fc, preds_i[0])
    assert len(ops.build_selection_mask(np.zeros(0), preds_i[0])) == 0  # no throw on an empty column
    a, b = ops.build_selection_mask(ic, preds_i[0]), ops.build_selection_mask(ic, preds_i[5])
    m = ops.mask_and(a, b)
    assert np.array_equal(m, (a & b))
    t = {"i": ic, "f": fc}
    got = ops.apply_mask(t, m)
    assert np.array_equal(got["i"], ic[m.astype(bool)])
    assert np.array_equal(got["f"].view(np.int64), fc[m.astype(bool)].view(np.int64))
    dm = rng.normal(size=(1000, 3))
    mm = (rng.random(1000) < 0.3).astype(np.uint8)
    assert np.array_equal(ops.apply_mask(dm, mm), dm[mm.astype(bool)])


@pytest.mark.parametrize("seed", range(4))
def test_sort_rows(gpu_ctx, seed):
    from paper_2306_08367_b200 import errors, ops
    rng = np.random.default_rng(seed)
    t = rng.integers(-3, 4, (5000, 4)).astype(np.float64)
    t[::7, 1] = -0.0
    t[:, 3] = np.arange(5000)  # payload: exposes the tie order
    keys = [[0], [1, 0], [2, 0, 1], [1, 2]][seed]
    dirs = [["Asc"], ["Desc", "Asc"], ["Asc", "Desc", "Desc"], ["Desc", "Desc"]][seed]
    got = ops.sort_rows(t, keys, dirs)
    assert np.array_equal(got.view(np.int64), ref.sort_rows(t, keys, dirs).view(np.int64))
    with pytest.raises(errors.IndexError):
        ops.sort_rows(t, [4], ["Asc"])
