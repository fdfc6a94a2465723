"""GPU parity for decision-tree fusion (csrc/tree.cu):
prefuse_tree partials and apply_fused_tree / predict_tree labels are
bit-identical to the reference (oracle/_ref, the reference compiled from its own
sources, when present; else the pinned numpy oracle, itself checked against the
reference in tests/test_oracle_golden.py::test_tree_oracle_matches_reference).
Trees come from the reference's own generator (bench::gen_tree) or, without
oracle/_ref, from a seeded Python builder."""
import numpy as np
import pytest

from oracle import laq_oracle as O

pytestmark = pytest.mark.gpu


def _random_tree(k, leaves, rng):
    nodes = {"is_leaf": [1], "feature": [-1], "threshold": [0.0], "true_child": [-1], "false_child": [-1],
             "label": [0]}
    leaf_ids = [0]
    while len(leaf_ids) < leaves:
        pick = leaf_ids.pop(int(rng.integers(0, len(leaf_ids))))
        t, f = len(nodes["is_leaf"]), len(nodes["is_leaf"]) + 1
        for _ in range(2):
            for key, v in (("is_leaf", 1), ("feature", -1), ("threshold", 0.0), ("true_child", -1),
                           ("false_child", -1), ("label", 0)):
                nodes[key].append(v)
        nodes["is_leaf"][pick] = 0
        nodes["feature"][pick] = int(rng.integers(0, k))
        nodes["threshold"][pick] = float(rng.random())
        nodes["true_child"][pick], nodes["false_child"][pick] = t, f
        leaf_ids += [t, f]
    for i, leaf in enumerate(leaf_ids):
        nodes["label"][leaf] = i
    return {key: np.array(v) for key, v in nodes.items()}


def _tree(k, leaves, seed):
    from oracle import ref
    if ref.available():
        return ref.gen_tree(k, max(1, min(k, leaves)), leaves, seed)
    return _random_tree(k, leaves, np.random.default_rng(seed))


@pytest.fixture(scope="module")
def T(gpu_ctx):
    from paper_2306_08367_b200 import errors, tree
    return tree, errors


@pytest.mark.parametrize("k,leaves,n_dims", [(16, 2, 1), (32, 64, 3), (64, 200, 2), (7, 33, 4)])
def test_fused_tree_bit_exact(T, k, leaves, n_dims):
    tree, _ = T
    rng = np.random.default_rng(k * 100 + leaves)
    t = _tree(k, leaves, k + leaves)
    cuts = np.sort(rng.choice(np.arange(1, k), size=n_dims - 1, replace=False)) if n_dims > 1 else []
    widths = np.diff(np.concatenate([[0], cuts, [k]])).astype(int)
    perm = rng.permutation(k)
    pl, o = [], 0
    for w in widths:
        pl.append(perm[o:o + w])
        o += w
    owner = np.zeros(k, np.int64)
    for j, p in enumerate(pl):
        owner[p] = j
    dims = [rng.random((int(rng.integers(10, 3000)), len(p))) for p in pl]
    idx = [rng.integers(0, d.shape[0], 20_000) for d in dims]
    m = tree.compile_tree(t, k)
    f = tree.prefuse_tree(dims, pl, tree.partition_tree(m, owner, n_dims), m.path_score, m.labels)
    y = tree.apply_fused_tree(idx, f)
    comp = O.compile_tree(t, k)
    want_parts = O.prefuse_tree(dims, pl, O.partition_tree(comp, owner, n_dims))
    want = O.apply_fused_tree(idx, want_parts, comp[3], comp[4])
    for got, w in zip(f.partials, want_parts):
        assert np.array_equal(got.cpu().numpy(), w)
    assert np.array_equal(y, want)
    from oracle import ref
    if ref.available():
        yr, pr = ref.fused_tree(t, dims, pl, k, owner, idx)
        assert np.array_equal(y, yr)
        assert all(np.array_equal(g.cpu().numpy(), r) for g, r in zip(f.partials, pr))
    # non-fused: materialize + predict_tree gives the same labels
    Tm = O.materialize(idx, dims, pl, k)
    assert np.array_equal(tree.predict_tree(Tm, m), want)


def test_tree_model_errors(T):
    tree, errors = T
    f = tree.FusedTree([np.array([[1.0, 1.0], [0.0, 2.0]])], np.array([1.0, 2.0]), np.array([7, 8]))
    assert tree.apply_fused_tree([np.array([1, 1])], f).tolist() == [8, 8]
    with pytest.raises(errors.ModelError, match="row 1 matches several leaves"):
        tree.apply_fused_tree([np.array([0, 1, 0])], tree.FusedTree(
            [np.array([[0.0, 2.0], [1.0, 2.0]])], np.array([1.0, 2.0]), np.array([7, 8])))
    with pytest.raises(errors.ModelError, match="row 2 matches no leaf"):
        tree.apply_fused_tree([np.array([1, 1, 0])], tree.FusedTree(
            [np.array([[5.0, 5.0], [0.0, 2.0]])], np.array([1.0, 2.0]), np.array([7, 8])))
    with pytest.raises(errors.TreeError):
        tree.compile_tree({"is_leaf": np.array([0]), "feature": np.array([0]), "threshold": np.array([0.5]),
                           "true_child": np.array([5]), "false_child": np.array([0]), "label": np.array([0])}, 4)
    with pytest.raises(errors.MappingError):
        m = tree.compile_tree(_random_tree(4, 3, np.random.default_rng(0)), 4)
        tree.partition_tree(m, np.full(4, 5), 1)  # no feature has an owning dim
