"""CPU tests of the host-side logic around the device operators (no GPU):
the compact transfer format (star.pack_columns), the tree model compile /
partition that feeds tree fusion (tree.compile_tree / partition_tree, checked
against the pinned oracle restatement of mlops.cpp:188-243 / fusion.cpp:79-126),
and the FFN / tensor-core input checks that run before any device work."""
import numpy as np
import pytest

from oracle import laq_oracle as O
from paper_2306_08367_b200 import errors, star, tree


def test_pack_columns_round_trip():
    rng = np.random.default_rng(0)
    cols = {"u8": rng.integers(5, 200, 1001), "u16": rng.integers(-3000, 40000, 1001),
            "i32": rng.integers(-10**9, 10**9, 1001), "const": np.full(1001, 7), "empty": np.zeros(0, np.int64),
            "f": rng.random(1001)}
    packed = star.pack_columns(cols)
    assert "f" not in packed  # float columns stay on the host path
    widths = {c: w for c, (_, w, _) in packed.items()}
    assert widths == {"u8": 1, "u16": 2, "i32": 4, "const": 1, "empty": 1}
    for c, (buf, w, off) in packed.items():
        n = len(cols[c])
        assert buf.size == n * w + 16 and not buf[n * w:].any()  # 16 bytes of zero padding
        dt = {1: np.uint8, 2: np.uint16, 4: np.int32}[w]
        assert np.array_equal(buf[: n * w].view(dt).astype(np.int64) + off, cols[c])


def _tree(k, leaves, rng):
    nodes = {"is_leaf": [1], "feature": [-1], "threshold": [0.0], "true_child": [-1], "false_child": [-1],
             "label": [0]}
    leaf_ids = [0]
    while len(leaf_ids) < leaves:
        pick = leaf_ids.pop(int(rng.integers(0, len(leaf_ids))))
        t = len(nodes["is_leaf"])
        for key, v in (("is_leaf", 1), ("feature", -1), ("threshold", 0.0), ("true_child", -1),
                       ("false_child", -1), ("label", 0)):
            nodes[key] += [v, v]
        nodes["is_leaf"][pick] = 0
        nodes["feature"][pick] = int(rng.integers(0, k))
        nodes["threshold"][pick] = float(rng.random())
        nodes["true_child"][pick], nodes["false_child"][pick] = t, t + 1
        leaf_ids += [t, t + 1]
    for i, leaf in enumerate(leaf_ids):
        nodes["label"][leaf] = 100 + i
    return {key: np.array(v) for key, v in nodes.items()}


@pytest.mark.parametrize("k,leaves", [(1, 2), (8, 9), (40, 77)])
def test_compile_and_partition_tree_match_oracle(k, leaves):
    rng = np.random.default_rng(k + leaves)
    t = _tree(k, leaves, rng)
    m = tree.compile_tree(t, k)
    feats, thr, H, score, labels = O.compile_tree(t, k)
    assert np.array_equal(m.node_feature, feats) and np.array_equal(m.thresholds, thr)
    assert np.array_equal(m.paths, H) and np.array_equal(m.path_score, score) and np.array_equal(m.labels, labels)
    owner = rng.integers(0, 3, k)
    parts = tree.partition_tree(m, owner, 3)
    want = O.partition_tree((feats, thr, H, score, labels), owner, 3)
    for p, (ids, nf, nt, ph) in zip(parts, want):
        assert np.array_equal(p.node_ids, ids) and np.array_equal(p.node_feature, nf)
        assert np.array_equal(p.thresholds, nt) and np.array_equal(p.path_rows, ph)


def test_tree_validation_errors():
    bad_child = {"is_leaf": np.array([0, 1]), "feature": np.array([0, -1]), "threshold": np.array([0.5, 0.0]),
                 "true_child": np.array([1, -1]), "false_child": np.array([3, -1]), "label": np.array([0, 1])}
    with pytest.raises(errors.TreeError):
        tree.compile_tree(bad_child, 4)
    t = _tree(6, 5, np.random.default_rng(1))
    with pytest.raises(errors.TreeError):
        tree.compile_tree(t, 2)  # a node tests feature >= input width (mlops.cpp:190-193)
    m = tree.compile_tree(t, 6)
    with pytest.raises(errors.MappingError):
        tree.partition_tree(m, np.zeros(5, np.int64), 1)  # ownership list must cover every feature


def test_bitpack_roundtrip():
    """The bit-packed transfer format: exact round trip, word count contract."""
    import numpy as np
    from paper_2306_08367_b200 import star
    rng = np.random.default_rng(3)
    for bits in (1, 4, 6, 12, 15, 20, 31, 32):
        for n in (0, 1, 31, 32, 127, 128, 129, 10_007):
            v = rng.integers(0, 2 ** bits, n, dtype=np.int64)
            w = star.bitpack_words(v, bits)
            assert w.dtype == np.uint32 and w.size == -(-n // 128) * 4 * bits + 4
            assert np.array_equal(star.bitunpack_words(w, n, bits), v)
    cols = {"a": np.array([5, 7, 6], np.int32), "b": np.array([100, 9999, 4000], np.int32)}
    p = star.bitpack_columns(cols)
    assert p["a"][1:] == (2, 5) and p["b"][1:] == (14, 100)
