"""Decision-tree fusion on the device (mirror of
fusion.hpp:20-55 and mlops.hpp:49-80).

  compile_tree      TreeModel -> TreeLA (F, v, H, h, labels)        mlops.cpp:188-243 (host: model compile)
  partition_tree    TreeLA -> per-dimension node blocks             fusion.cpp:79-126 (host)
  prefuse_tree      P_j = ((B_j M_j F_j) > v_j) H_j                 fusion.cpp:39-47, 128-144 (device)
  apply_fused_tree  labels of ((P_0[i_0] + ...) == h)               fusion.cpp:146-168 (device)
  predict_tree      labels of (((T F) > v) H == h)                  mlops.cpp:254-280 (device)

A tree is a dict of node arrays (TreeNode, mlops.hpp:18-25): is_leaf, feature,
threshold, true_child, false_child, label; node 0 is the root.  Partials and
labels are bit-identical to the reference (sequential node-order sums of the
path rows, exactly as dense_matmul does).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import errors
from .device import context, dev, host, ptrs

f64 = torch.float64


@dataclass
class TreeLA:
    node_feature: np.ndarray  # p: feature tested by node n (F as a column -> row map)
    thresholds: np.ndarray    # p
    paths: np.ndarray         # p x l (H)
    path_score: np.ndarray    # l (h)
    labels: np.ndarray        # l
    input_width: int

    @property
    def leaf_count(self) -> int:
        return int(self.paths.shape[1])


@dataclass
class TreeDimBlock:
    node_ids: np.ndarray
    node_feature: np.ndarray
    thresholds: np.ndarray
    path_rows: np.ndarray


@dataclass
class FusedTree:
    partials: list
    path_score: np.ndarray
    labels: np.ndarray


def validate_tree(tree):
    """mlops.cpp validate_tree: one tree rooted at 0, two valid children per internal node."""
    n = len(tree["is_leaf"])
    if n == 0:
        raise errors.TreeError("tree has no nodes")
    seen = np.zeros(n, bool)
    stack = [0]
    while stack:
        i = stack.pop()
        if seen[i]:
            raise errors.TreeError(f"node {i} reached twice")
        seen[i] = True
        if not tree["is_leaf"][i]:
            for c in (int(tree["true_child"][i]), int(tree["false_child"][i])):
                if c < 0 or c >= n:
                    raise errors.TreeError(f"node {i} has an invalid child {c}")
                stack.append(c)
    if not seen.all():
        raise errors.TreeError("unreachable nodes")


def compile_tree(tree, input_width: int) -> TreeLA:
    """mlops.cpp:188-243: nodes and leaves numbered by a pre-order walk, true branch first."""
    validate_tree(tree)
    is_leaf = np.asarray(tree["is_leaf"])
    for i in np.nonzero(~is_leaf.astype(bool))[0]:
        if tree["feature"][i] >= input_width:
            raise errors.TreeError(f"tree feature {int(tree['feature'][i])} exceeds input width {input_width}")
    feats, thr, paths, score, labels = [], [], [], [], []
    stack = [(0, (), -1, 0.0)]
    while stack:
        nid, path, parent, sign = stack.pop()
        if parent >= 0:
            path = path + ((parent, sign),)
        if is_leaf[nid]:
            paths.append(path)
            score.append(float(sum(1 for _, s in path if s > 0)))
            labels.append(int(tree["label"][nid]))
        else:
            pos = len(feats)
            feats.append(int(tree["feature"][nid]))
            thr.append(float(tree["threshold"][nid]))
            stack.append((int(tree["false_child"][nid]), path, pos, -1.0))
            stack.append((int(tree["true_child"][nid]), path, pos, 1.0))
    H = np.zeros((len(feats), len(labels)))
    for leaf, path in enumerate(paths):
        for node, s in path:
            H[node, leaf] = s
    return TreeLA(np.array(feats, np.int64), np.array(thr), H, np.array(score), np.array(labels, np.int64),
                  input_width)


def partition_tree(m: TreeLA, feature_owner, dim_count: int):
    """fusion.cpp:79-126: nodes split by the dimension owning their feature."""
    owner = np.asarray(feature_owner, np.int64)
    if len(owner) != m.input_width:
        raise errors.MappingError(f"partition_tree: ownership list must cover all {m.input_width} features")
    blocks = [[] for _ in range(dim_count)]
    for node, f in enumerate(m.node_feature):
        o = int(owner[f])
        if o < 0 or o >= dim_count:
            raise errors.MappingError(f"partition_tree: feature {int(f)} has no owning dim")
        blocks[o].append(node)
    return [TreeDimBlock(np.array(b, np.int64), m.node_feature[b], m.thresholds[b], m.paths[b]) for b in blocks]


def _tree_partial(ctx, Bd, node_col, thresholds, path_rows, l):
    rows, cols = int(Bd.shape[0]), int(Bd.shape[1])
    out = torch.empty((rows, l), dtype=f64, device="cuda")
    nc = np.ascontiguousarray(node_col, np.int64)
    th = np.ascontiguousarray(thresholds, np.float64)
    H = np.ascontiguousarray(path_rows, np.float64).reshape(len(nc), l)
    ctx.check(ctx.lib.laq_tree_partial(ctx.h, Bd.data_ptr(), rows, cols, len(nc),
                                       nc.ctypes.data_as(C.POINTER(C.c_int64)), None,
                                       th.ctypes.data_as(C.POINTER(C.c_double)),
                                       H.ctypes.data_as(C.POINTER(C.c_double)), l, out.data_ptr()))
    return out


def prefuse_tree(dims, placements, parts, path_score, labels, k: int | None = None) -> FusedTree:
    """fusion.cpp:128-144 on the device; partials stay resident (fp64)."""
    if len(dims) == 0 or len(dims) != len(placements) or len(dims) != len(parts):
        raise errors.ShapeError("prefuse_tree: input list lengths")
    if len(path_score) != len(labels):
        raise errors.ShapeError("prefuse_tree: score/label lengths")
    k = k if k is not None else int(sum(len(p) for p in placements))
    from .tc_ops import _check_placements
    _check_placements(placements, k)
    ctx = context()
    l = len(labels)
    out = []
    for d, pl, part in zip(dims, placements, parts):
        Bd = dev(d, f64)
        if Bd.shape[1] != len(pl):
            raise errors.ShapeError("fusion: column map does not fit dim table")
        inv = {int(g): c for c, g in enumerate(np.asarray(pl, np.int64))}
        node_col = [inv.get(int(f), -1) for f in part.node_feature]
        out.append(_tree_partial(ctx, Bd, node_col, part.thresholds, part.path_rows, l))
    return FusedTree(out, np.asarray(path_score, np.float64), np.asarray(labels, np.int64))


def _decode(ctx, idx_ptrs, n_parts, rows, partials, path_score, labels, what):
    out = torch.empty(max(rows, 1), dtype=torch.int64, device="cuda")
    hs = np.ascontiguousarray(path_score, np.float64)
    lb = np.ascontiguousarray(labels, np.int64)
    bad_row, several = C.c_int64(), C.c_int32()
    rc = ctx.lib.laq_apply_fused_tree(ctx.h, n_parts, idx_ptrs, rows, ptrs(partials), len(lb),
                                      hs.ctypes.data_as(C.POINTER(C.c_double)),
                                      lb.ctypes.data_as(C.POINTER(C.c_int64)), out.data_ptr(),
                                      C.byref(bad_row), C.byref(several))
    if rc == 11:  # LAQ_ERR_MODEL
        raise errors.ModelError(f"{what}: row {bad_row.value} matches "
                                + ("several leaves" if several.value else "no leaf"))
    ctx.check(rc)
    return out[:rows]


def apply_fused_tree(i_maps, f: FusedTree):
    """fusion.cpp:146-168 over row maps (one source row per target row)."""
    if len(i_maps) == 0 or len(i_maps) != len(f.partials):
        raise errors.ShapeError("apply_fused_tree: map/partial list lengths")
    on = any(isinstance(x, torch.Tensor) and x.is_cuda for x in i_maps)
    ctx = context()
    idx = [dev(i, torch.int64) for i in i_maps]
    P = [dev(p, f64) for p in f.partials]
    y = _decode(ctx, ptrs(idx), len(idx), int(idx[0].numel()), P, f.path_score, f.labels, "apply_fused_tree")
    return y if on else host(y)


def predict_tree(T, m: TreeLA):
    """mlops.cpp:254-280: the one-block case over T (all nodes), then the decode."""
    on = isinstance(T, torch.Tensor) and T.is_cuda
    Td = dev(T, f64)
    if Td.shape[1] != m.input_width:
        raise errors.ShapeError(f"predict_tree: input width {Td.shape[1]} vs model {m.input_width}")
    ctx = context()
    S = _tree_partial(ctx, Td, m.node_feature, m.thresholds, m.paths, m.leaf_count)
    y = _decode(ctx, None, 1, int(Td.shape[0]), [S], m.path_score, m.labels, "predict_tree")
    return y if on else host(y)
