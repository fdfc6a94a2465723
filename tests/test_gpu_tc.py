"""GPU parity for the tensor-core contractions (csrc/gemm_tc.cu) of the wide
complexity-sweep shapes (BASELINE configs[4]): prefuse_linear (fusion.cpp:50-62),
apply_fused_linear (fusion.cpp:64-77) and the non-fused materialize +
predict_linear (laqops.cpp:338-374, mlops.cpp:248-250), against the pinned
fp64 oracle.  fp16x2 split with fp32 accumulation and fp32 storage: every element is
checked condition-aware, |Y - Y_ref| <= 1e-5 * (|T| |L|);
both plans must agree with each other to the same bound."""
import numpy as np
import pytest

from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _check(y, ref, bound):
    y = np.asarray(y, np.float64).reshape(ref.shape)
    err = np.abs(y - ref)
    assert np.all(err <= TOL * bound), f"condition-aware error {float(np.max(err / np.maximum(bound, 1e-300))):.3e}"


@pytest.fixture(scope="module")
def tco(gpu_ctx):
    from paper_2306_08367_b200 import errors, tc_ops
    return tc_ops, errors


@pytest.mark.parametrize("widths,l,n", [
    ((16,), 1, 3000),          # l = 1 (BN = 16), one 16-feature step
    ((32, 32), 4, 5000),       # cfg3-like K, small l
    ((5, 40), 64, 2049),       # ragged widths, K blocks with 1 and 2 steps, partial tiles
    ((128,), 300, 1500),       # 4 K blocks, two column tiles (BN 256 + ragged 44)
    ((64, 64), 1024, 700),     # wide output, W panel per column tile
])
def test_fused_and_nonfused_match_oracle(tco, widths, l, n):
    tc, _ = tco
    rng = np.random.default_rng(sum(widths) * 7 + l)
    k = sum(widths)
    dims = [rng.random((int(rng.integers(100, 900)), w)) for w in widths]
    perm = rng.permutation(k)
    pl, o = [], 0
    for w in widths:
        pl.append(perm[o:o + w])
        o += w
    L = rng.uniform(-1, 1, (k, l))
    idx = [rng.integers(0, d.shape[0], n) for d in dims]
    T = O.materialize(idx, dims, pl, k)
    ref = T @ L
    bound = np.abs(T) @ np.abs(L)
    P = tc.prefuse_linear_tc(dims, pl, L)
    for Pj, d, p in zip(P, dims, pl):  # each partial against B_j (M_j L)
        _check(Pj.cpu().numpy(), d @ L[np.asarray(p)], np.abs(d) @ np.abs(L[np.asarray(p)]))
    y_f = tc.apply_fused_linear_tc(idx, P).cpu().numpy()
    _check(y_f, ref, bound)
    y_n = tc.predict_nonfused_tc(idx, dims, pl, L).cpu().numpy()
    _check(y_n, ref, bound)


def test_gemm_errors(tco):
    tc, errors = tco
    rng = np.random.default_rng(0)
    with pytest.raises(errors.MappingError):
        tc.prefuse_linear_tc([rng.random((4, 2)), rng.random((4, 2))], [[0, 1], [1, 2]], rng.random((3, 2)))
    with pytest.raises(errors.ShapeError):
        tc.prefuse_linear_tc([rng.random((4, 2))], [[0, 1]], rng.random((3, 2)))
    f = tc.TCFeatures([rng.random((4, 2))], [[0, 1]], 2)
    with pytest.raises(errors.ShapeError):
        f.gemm(rng.random((3, 5)))
    assert f.gemm(rng.random((2, 5)), row_maps=[np.zeros(0, np.int32)]).shape == (0, 5)


@pytest.mark.parametrize("rows,k,l,n", [(300, 16, 1, 50_000), (40_000, 64, 256, 3_000), (2_000, 32, 8, 20_000)])
def test_planner_driven_predict(tco, rows, k, l, n):
    """tc_ops.predict_star_linear: the cost model picks the plan (device model
    via the C-ABI, or the paper's Eq. 2 + decide_fusion); whichever it picks,
    the answer equals the fp64 oracle condition-aware."""
    from paper_2306_08367_b200 import fusion
    tc, _ = tco
    rng = np.random.default_rng(rows + k + l)
    dims = [rng.random((rows, k // 2)), rng.random((rows // 2 + 1, k - k // 2))]
    pl = [np.arange(k // 2), np.arange(k // 2, k)]
    L = rng.uniform(-1, 1, (k, l))
    idx = [rng.integers(0, d.shape[0], n) for d in dims]
    T = O.materialize(idx, dims, pl, k)
    ref, bound = T @ L, np.abs(T) @ np.abs(L)
    want_dev = fusion.plan_linear_device(n, k, l, [d.shape[0] for d in dims])
    want_paper = fusion.plan_linear(n, k, l, [d.shape[0] for d in dims])
    for planner, want in (("device", want_dev), ("paper", want_paper)):
        y, plan = tc.predict_star_linear(idx, dims, pl, L, planner=planner)
        assert plan == want
        _check(y.cpu().numpy(), ref, bound)
    for forced in ("fused", "nonfused"):
        y, plan = tc.predict_star_linear(idx, dims, pl, L, plan=forced)
        assert plan == forced
        _check(y.cpu().numpy(), ref, bound)
