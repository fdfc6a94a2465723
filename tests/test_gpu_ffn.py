"""GPU parity for the tensor-core FFN over a star join (BASELINE configs[2],
csrc/ffn.cu) against the composed oracle (materialize + predict_linear + ReLU +
predict_linear, oracle.laq_oracle.ffn_predict).

Tolerance: a split 16-bit product with fp32 accumulation cannot
meet a per-element 1e-5 relative bound on cancelling sums, so every element is
checked condition-aware:  |Y_gpu - Y_ref| <= 1e-5 * bound  with
bound = sum_n |W2| (|T| |W1|) + |ReLU(H)| |W2|  (the magnitude of every term the
result is built from).  Survivor order and counts are exact."""
import numpy as np
import pytest

from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _check(y, ref, bound):
    y = np.asarray(y, np.float64).reshape(ref.shape)
    err = np.abs(y - ref)
    worst = float(np.max(err / np.maximum(bound, 1e-300))) if err.size else 0.0
    assert np.all(err <= TOL * bound), f"condition-aware error {worst:.3e} > {TOL}"
    return worst


@pytest.fixture(scope="module")
def mods(gpu_ctx):
    from paper_2306_08367_b200 import errors, ffn
    return ffn, errors


@pytest.mark.parametrize("widths,h,l,n", [
    ((32, 32), 256, 1, 5_000),     # cfg3 shape
    ((16,), 32, 1, 1_000),         # smallest hidden width
    ((5, 11, 3), 64, 3, 3_001),    # ragged dim widths (8-padding), l > 1, partial tile
    ((40, 24), 128, 8, 777),       # two K blocks (K = 64 + 16 padded)
    ((64, 32, 16), 96, 2, 2_500),  # K = 112 in 4 blocks, N = 96
])
def test_ffn_rows_matches_oracle(mods, widths, h, l, n):
    ffn, _ = mods
    rng = np.random.default_rng(sum(widths) + h + l)
    k = sum(widths)
    dims = [rng.random((rng.integers(50, 400), w)) for w in widths]
    # placements: a permutation of [0, k) split across dims (exercises W1 row permutation)
    perm = rng.permutation(k)
    pl, o = [], 0
    for w in widths:
        pl.append(perm[o:o + w])
        o += w
    W1 = rng.uniform(-1, 1, (k, h))
    W2 = rng.uniform(-1, 1, (h, l))
    idx = [rng.integers(0, d.shape[0], n) for d in dims]
    m = ffn.StarFFN(dims, pl, W1, W2)
    y = m.predict_rows(idx).cpu().numpy()
    ref, bound = O.ffn_predict(idx, dims, pl, k, W1, W2, exact_order=n <= 1000)
    _check(y, ref, bound)


def test_ffn_star_probe_all_hit_and_misses(mods):
    ffn, _ = mods
    rng = np.random.default_rng(7)
    r0, r1 = 3000, 700
    dims = [rng.random((r0, 32)), rng.random((r1, 32))]
    pks = [rng.permutation(r0).astype(np.int64) + 5, rng.permutation(r1).astype(np.int64)]
    W1 = rng.uniform(-1, 1, (64, 256))
    W2 = rng.uniform(-1, 1, (256, 1))
    pl = [np.arange(32), np.arange(32, 64)]
    n = 20_000
    fks = [pks[0][rng.integers(0, r0, n)], pks[1][rng.integers(0, r1, n)]]
    m = ffn.StarFFN(dims, pl, W1, W2, dim_pks=pks)
    for case in ("all_hit", "misses"):
        f = [x.copy() for x in fks]
        if case == "misses":
            f[0][rng.integers(0, n, 500)] = 10_000_000  # no such key
            f[1][::7] = r1 + 99
        import torch
        surv = torch.empty(n, dtype=torch.int64, device="cuda")
        y, nnz = m([x.astype(np.int32) for x in f], survivors=surv)
        ws, wrows = O.multiway_star_join(f, pks)
        assert nnz == len(ws)
        assert np.array_equal(surv[:nnz].cpu().numpy(), ws)
        ref, bound = O.ffn_predict(wrows, dims, pl, 64, W1, W2)
        _check(y.cpu().numpy(), ref, bound)


def test_ffn_empty_and_errors(mods):
    ffn, errors = mods
    rng = np.random.default_rng(3)
    dims = [rng.random((10, 8))]
    m = ffn.StarFFN(dims, [np.arange(8)], rng.random((8, 32)), rng.random((32, 1)), dim_pks=[np.arange(10)])
    y = m.predict_rows([np.zeros(0, np.int32)])
    assert y.shape[0] == 0
    y, nnz = m([np.full(5, 99, np.int32)])  # nothing joins
    assert nnz == 0
    with pytest.raises(errors.MappingError):
        ffn.StarFFN([rng.random((4, 2)), rng.random((4, 2))], [[0, 1], [1, 2]], rng.random((3, 32)),
                    rng.random((32, 1)))
    with pytest.raises(errors.ShapeError):
        ffn.StarFFN(dims, [np.arange(8)], rng.random((9, 32)), rng.random((32, 1)))
    with pytest.raises(errors.UnsupportedError):
        ffn.StarFFN(dims, [np.arange(8)], rng.random((8, 48)), rng.random((48, 1)))  # h not multiple of 32
    with pytest.raises(errors.UnsupportedError):  # W1 + two stages exceed shared memory
        big = [rng.random((10, 64)), rng.random((10, 64)), rng.random((10, 64))]
        ffn.StarFFN(big, [np.arange(64), np.arange(64, 128), np.arange(128, 192)], rng.random((192, 256)),
                    rng.random((256, 1)))


def test_ffn_cfg3_ssb_sample(mods):
    """cfg3 on generated SSB data (sf=1 here; the bench runs sf=10): every
    lineorder row joins customer and part; a 200K-row slice is checked."""
    ffn, _ = mods
    from paper_2306_08367_b200 import gen
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    fks, pks, dims, pl, W1, W2 = ffn.cfg3_inputs(g)
    n = 200_000
    m = ffn.StarFFN(dims, pl, W1, W2, dim_pks=pks)
    y, nnz = m([f[:n] for f in fks])
    assert nnz == n
    ws, wrows = O.multiway_star_join([f[:n] for f in fks], pks)
    ref, bound = O.ffn_predict(wrows, dims, pl, 64, W1, W2)
    _check(y.cpu().numpy(), ref, bound)


@pytest.mark.parametrize("widths,h,l,n", [((32, 32), 256, 1, 5000), ((16, 40), 128, 3, 777)])
def test_ffn_cta_pair_variant_matches_oracle(mods, monkeypatch, widths, h, l, n):
    """LAQ_FFN_2CTA=1: M = 256 UMMAs on CTA pairs (cta_group::2, W1 split by
    hidden units across the pair, the peer's stages relayed to the leader) give
    the same condition-aware answer, including a ragged last 256-row tile."""
    monkeypatch.setenv("LAQ_FFN_2CTA", "1")
    test_ffn_rows_matches_oracle(mods, widths, h, l, n)
