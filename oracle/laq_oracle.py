"""TEST INFRASTRUCTURE ONLY — a numpy restatement of the reference's hot path.

This is the CPU checker the GPU engine is compared against.  Each function
restates one reference function (file:line under /root/reference/proj) and is
itself pinned against golden vectors produced by the reference's own compiled
code (tests/golden/, made by tests/golden/make_golden.py through
oracle/_ref/liblaq_ref.so) and against the known answers in the reference's
tests (tests/test_oracle_golden.py).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import it; the product path never does.

Floating-point functions reproduce the reference's accumulation order
(sequential, separately rounded products), so they are bit-exact with it.
"""
from __future__ import annotations

import numpy as np


class DomainError(Exception):
    pass


class DuplicateKeyError(Exception):
    pass


class MappingError(Exception):
    pass


class TreeError(Exception):
    pass


class ModelError(Exception):
    pass


class ShapeError(Exception):
    pass


# ---------------------------------------------------------------------------
# key domains and key matrices (laqops.cpp:123-220)
# ---------------------------------------------------------------------------

def build_key_domain(keys_r, keys_s) -> np.ndarray:
    """laqops.cpp:142-155: ascending distinct union; DomainError on a negative key."""
    allk = np.concatenate([np.asarray(keys_r, np.int64), np.asarray(keys_s, np.int64)])
    if allk.size and allk.min() < 0:
        raise DomainError(f"negative join key {int(allk.min())}")
    return np.unique(allk)


def update_key_domain(domain, new_keys) -> np.ndarray:
    """laqops.cpp:157-171."""
    nk = np.asarray(new_keys, np.int64)
    if nk.size and nk.min() < 0:
        raise DomainError(f"negative join key {int(nk.min())}")
    return np.unique(np.concatenate([np.asarray(domain, np.int64), nk]))


def position(domain, keys) -> np.ndarray:
    """KeyDomain::position (laqops.cpp:123-127), vectorised; DomainError if absent."""
    d = np.asarray(domain, np.int64)
    k = np.asarray(keys, np.int64)
    p = np.searchsorted(d, k)
    ok = (p < len(d)) & (d[np.minimum(p, max(len(d) - 1, 0))] == k) if len(d) else np.zeros(len(k), bool)
    if not np.all(ok):
        raise DomainError("key not in domain")
    return p.astype(np.int64)


def key_matrix(keys, domain, orientation="RowsByDomain", values=None):
    """laqops.cpp:173-220 -> (row_ptr, col_idx, values)."""
    keys = np.asarray(keys, np.int64)
    n, d = len(keys), len(domain)
    pos = position(domain, keys)
    vals = np.ones(n) if values is None else np.asarray(values, np.float64)
    keep = vals != 0.0
    if orientation == "RowsByDomain":
        row_ptr = np.concatenate([[0], np.cumsum(keep)]).astype(np.int64)
        return row_ptr, pos[keep], vals[keep]
    idx = np.nonzero(keep)[0]
    order = np.argsort(pos[idx], kind="stable")
    col = idx[order].astype(np.int64)
    counts = np.bincount(pos[idx], minlength=d) if d else np.zeros(0, np.int64)
    row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return row_ptr, col, vals[col]


# ---------------------------------------------------------------------------
# joins (laqops.cpp:222-319)
# ---------------------------------------------------------------------------

def mm_join(keys_r, keys_s):
    """laqops.cpp:222-231: all (r, s) with equal keys, sorted (r asc, s asc)."""
    r = np.asarray(keys_r, np.int64)
    s = np.asarray(keys_s, np.int64)
    build_key_domain(r, s)  # DomainError on negatives
    order = np.argsort(s, kind="stable")
    ss = s[order]
    lo = np.searchsorted(ss, r, "left")
    hi = np.searchsorted(ss, r, "right")
    cnt = hi - lo
    rr = np.repeat(np.arange(len(r), dtype=np.int64), cnt)
    if len(rr) == 0:
        return rr, np.zeros(0, np.int64)
    starts = np.repeat(lo, cnt)
    within = np.arange(len(rr)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    return rr, order[starts + within].astype(np.int64)


def multiway_star_join(fks, pks):
    """laqops.cpp:233-319: (survivors, [dim row per link]) in ascending fact order.
    Unique pks required (DuplicateKeyError, laqops.cpp:252-254)."""
    n = len(fks[0]) if fks else 0
    alive = np.ones(n, bool)
    rows = []
    for j, (fk, pk) in enumerate(zip(fks, pks)):
        fk = np.asarray(fk, np.int64)
        pk = np.asarray(pk, np.int64)
        if len(np.unique(pk)) != len(pk):
            raise DuplicateKeyError(f"multiway_star_join: duplicate keys in dim {j}")
        live = fk[alive]
        if (live.size and live.min() < 0) or (pk.size and pk.min() < 0):
            raise DomainError("negative join key")
        order = np.argsort(pk, kind="stable")
        sp = pk[order]
        p = np.searchsorted(sp, fk)
        pc = np.minimum(p, max(len(sp) - 1, 0))
        hit = (p < len(sp)) & (sp[pc] == fk) if len(sp) else np.zeros(n, bool)
        r = np.where(hit, order[pc] if len(sp) else 0, -1)
        alive &= hit
        rows.append(r)
    surv = np.nonzero(alive)[0].astype(np.int64)
    return surv, [r[surv].astype(np.int64) for r in rows]


# ---------------------------------------------------------------------------
# dense products and fusion (matrix.cpp:125-174, fusion.cpp:11-77, laqops.cpp:338-374)
# ---------------------------------------------------------------------------

def dense_matmul(a, b) -> np.ndarray:
    """matrix.cpp:158-174: i-k-j, zero a skipped, sequential k, product then add."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape[1] != b.shape[0]:
        raise ShapeError("dense_matmul")
    out = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        col = a[:, k]
        nz = col != 0.0
        if nz.any():
            out[nz] = out[nz] + col[nz, None] * b[k][None, :]
    return out


def check_placements(placements, k):
    """fusion.cpp:11-25 (+ make_map target range, laqops.cpp:33-37)."""
    claimed = np.zeros(k, bool)
    total = 0
    for p in placements:
        for t in p:
            if t < 0 or t >= k:
                raise MappingError(f"column map: target index {t} out of range")
            if claimed[t]:
                raise MappingError(f"fusion: overlapping target column {t}")
            claimed[t] = True
            total += 1
    if total != k:
        raise ShapeError(f"fusion: placements claim {total} of {k} feature columns")


def prefuse_linear(dims, placements, L):
    """fusion.cpp:50-62: P_j = B_j (M_j L)."""
    L = np.asarray(L, np.float64)
    check_placements(placements, L.shape[0])
    return [dense_matmul(np.asarray(B, np.float64), L[np.asarray(p, np.int64)]) for B, p in zip(dims, placements)]


def apply_fused_linear(idx, partials):
    """fusion.cpp:64-77: ((P_0[i_0] + P_1[i_1]) + ...)."""
    out = 0.0 + np.asarray(partials[0])[np.asarray(idx[0], np.int64)]  # spmm_dense: 0 + 1*x
    for i, p in zip(idx[1:], partials[1:]):
        out = out + np.asarray(p)[np.asarray(i, np.int64)]
    return out


def materialize(idx, dims, placements, k):
    """laqops.cpp:338-374."""
    rows = len(idx[0])
    T = np.zeros((rows, k))
    for i, B, p in zip(idx, dims, placements):
        T[:, np.asarray(p, np.int64)] = 0.0 + np.asarray(B)[np.asarray(i, np.int64)]
    return T


def predict_linear(T, W):
    """mlops.cpp:248-250."""
    return dense_matmul(T, W)


def ffn_predict(idx, dims, placements, k, W1, W2, exact_order=False):
    """cfg3: the reference has no FFN; it is the composition
    Y = predict_linear(ReLU(predict_linear(materialize(...), W1)), W2) of pinned
    functions (laqops.cpp:338-374, mlops.cpp:248-250) with an elementwise ReLU.
    Returns (Y, bound) where bound[m, c] is the condition-aware error scale
        sum_n |W2[n,c]| * sum_k |T[m,k] W1[k,n]|  +  sum_n |ReLU(H[m,n]) W2[n,c]|
    used for the 1e-5 tolerance.  exact_order=True uses
    dense_matmul's sequential-k order (small cases); otherwise BLAS (the
    association difference, ~1e-16 relative, is far below the tolerance)."""
    T = materialize(idx, dims, placements, k)
    W1 = np.asarray(W1, np.float64)
    W2 = np.asarray(W2, np.float64)
    mm = dense_matmul if exact_order else (lambda a, b: a @ b)
    H = mm(T, W1)
    R = np.maximum(H, 0.0)
    Y = mm(R, W2)
    bound = (np.abs(T) @ np.abs(W1)) @ np.abs(W2) + R @ np.abs(W2)
    return Y, bound


# ---------------------------------------------------------------------------
# decision trees (mlops.cpp:188-280, fusion.cpp:39-168)
# A tree is a dict of node arrays (TreeNode, mlops.hpp:18-25): is_leaf,
# feature, threshold, true_child, false_child, label; root = node 0.
# ---------------------------------------------------------------------------

def compile_tree(tree, input_width):
    """mlops.cpp:188-243: pre-order walk, true branch first.  Returns
    (node_feature[p], thresholds[p], paths p x l, path_score[l], labels[l])."""
    is_leaf = np.asarray(tree["is_leaf"])
    for i in range(len(is_leaf)):
        if not is_leaf[i] and tree["feature"][i] >= input_width:
            raise TreeError(f"tree feature {tree['feature'][i]} exceeds input width {input_width}")
    feats, thr, cols, score, labels = [], [], [], [], []
    stack = [(0, [], -1, 0.0)]
    while stack:
        nid, path, parent, sign = stack.pop()
        path = path + ([(parent, sign)] if parent >= 0 else [])
        if is_leaf[nid]:
            cols.append(path)
            score.append(float(sum(1 for _, sg in path if sg > 0)))
            labels.append(int(tree["label"][nid]))
        else:
            pos = len(feats)
            feats.append(int(tree["feature"][nid]))
            thr.append(float(tree["threshold"][nid]))
            stack.append((int(tree["false_child"][nid]), path, pos, -1.0))
            stack.append((int(tree["true_child"][nid]), path, pos, 1.0))
    H = np.zeros((len(feats), len(labels)))
    for leaf, path in enumerate(cols):
        for node, sg in path:
            H[node, leaf] = sg
    return (np.array(feats, np.int64), np.array(thr), H, np.array(score), np.array(labels, np.int64))


def _scores_to_labels(scores, path_score, labels, what):
    """mlops.cpp:269-280 / fusion.cpp:154-167: the unique leaf with score == h."""
    eq = scores == np.asarray(path_score)[None, :]
    cnt = eq.sum(axis=1)
    bad = np.nonzero(cnt != 1)[0]
    if len(bad):
        i = int(bad[0])
        raise ModelError(f"{what}: row {i} matches " + ("several leaves" if cnt[i] > 1 else "no leaf"))
    return np.asarray(labels)[np.argmax(eq, axis=1)]


def _node_scores(X, node_col, thr, H):
    """dense_matmul((X F > v), H) with dense_matmul's sequential node order and
    zero skipping (matrix.cpp:158-174): exact for any H."""
    bits = np.stack([(X[:, c] if c >= 0 else np.zeros(len(X))) > t for c, t in zip(node_col, thr)], axis=1) \
        if len(node_col) else np.zeros((len(X), 0), bool)
    out = np.zeros((len(X), H.shape[1]))
    for n in range(H.shape[0]):
        b = bits[:, n]
        if b.any():
            out[b] = out[b] + 1.0 * H[n][None, :]
    return out


def predict_tree(T, compiled):
    """mlops.cpp:254-280."""
    feats, thr, H, score, labels = compiled
    T = np.asarray(T, np.float64)
    return _scores_to_labels(_node_scores(T, feats, thr, H), score, labels, "predict_tree")


def partition_tree(compiled, feature_owner, dim_count):
    """fusion.cpp:79-126 -> per dim (node_ids, node_feature, thresholds, path_rows)."""
    feats, thr, H, _, _ = compiled
    blocks = [[] for _ in range(dim_count)]
    for node, f in enumerate(feats):
        o = int(feature_owner[f])
        if o < 0 or o >= dim_count:
            raise MappingError(f"partition_tree: feature {f} has no owning dim")
        blocks[o].append(node)
    return [(np.array(b, np.int64), feats[b], thr[b], H[b]) for b in blocks]


def prefuse_tree(dims, placements, parts):
    """fusion.cpp:39-47, 128-144: P_j = ((B_j M_j F_j) > v_j) H_j."""
    out = []
    for B, pl, (_, nf, nt, H) in zip(dims, placements, parts):
        inv = {int(g): c for c, g in enumerate(pl)}
        cols = [inv.get(int(f), -1) for f in nf]
        out.append(_node_scores(np.asarray(B, np.float64), cols, nt, H))
    return out


def apply_fused_tree(idx, partials, path_score, labels):
    """fusion.cpp:146-168."""
    return _scores_to_labels(apply_fused_linear(idx, partials), path_score, labels, "apply_fused_tree")


# ---------------------------------------------------------------------------
# aggregation (laqops.cpp:376-478)
# ---------------------------------------------------------------------------

def groupby_sum_single(keys_r, vals_r, keys_s, group_s):
    """laqops.cpp:376-413: groups = distinct group_s asc (zero groups kept);
    sums[g] += v_r * multiplicity(key_r, g), rows in order."""
    kr = np.asarray(keys_r, np.int64)
    vr = np.asarray(vals_r, np.float64)
    ks = np.asarray(keys_s, np.int64)
    gs = np.asarray(group_s, np.int64)
    build_key_domain(kr, ks)
    groups = np.unique(gs)
    sums = [0.0] * len(groups)
    gpos = {int(g): i for i, g in enumerate(groups)}
    mult: dict[int, dict[int, float]] = {}
    for k, g in zip(ks.tolist(), gs.tolist()):
        mult.setdefault(k, {}).setdefault(gpos[g], 0.0)
        mult[k][gpos[g]] += 1.0
    for k, v in zip(kr.tolist(), vr.tolist()):
        if v == 0.0 or k not in mult:
            continue
        for g in sorted(mult[k]):
            sums[g] += v * mult[k][g]
    return groups, np.asarray(sums, np.float64)


def groupby_sum_multi(cols, vals):
    """laqops.cpp:415-455: present tuples ascending; sum in row order."""
    cols = [np.asarray(c, np.int64) for c in cols]
    vals = np.asarray(vals, np.float64)
    n = len(vals)
    if n == 0:
        return np.zeros((len(cols), 0), np.int64), np.zeros(0)
    order = np.lexsort(tuple([np.arange(n)] + cols[::-1]))
    keys = np.stack([c[order] for c in cols])
    brk = np.ones(n, bool)
    brk[1:] = np.any(keys[:, 1:] != keys[:, :-1], axis=0)
    starts = np.nonzero(brk)[0]
    ends = np.append(starts[1:], n)
    sums = []
    for s, e in zip(starts, ends):
        acc = 0.0
        for r in order[s:e].tolist():
            acc += float(vals[r])
        sums.append(acc)
    return keys[:, starts], np.asarray(sums)


def sort_rows(t, key_cols, asc=True):
    """laqops.cpp:457-478 (stable, ascending)."""
    t = np.asarray(t)
    order = np.lexsort(tuple(t[:, c] for c in reversed(key_cols)))
    return t[order]


# ---------------------------------------------------------------------------
# cost model (fusion.cpp:259-302)
# ---------------------------------------------------------------------------

def speedup_ratio_linear(i, k, l, dims):
    if i <= 0 or k <= 0 or l <= 0 or not dims or any(r <= 0 for r in dims):
        raise DomainError("cost model: all inputs must be positive")
    s = float(sum(float(r) for r in dims))
    i, k, l = float(i), float(k), float(l)
    return ((i * k + k * k / 3.0) * s + i * k * l) / (i * l * s)


def speedup_ratio_tree(i, k, l, dims, p=None):
    if i <= 0 or k <= 0 or l <= 0 or (p is not None and p <= 0) or not dims or any(r <= 0 for r in dims):
        raise DomainError("cost model: all inputs must be positive")
    s = float(sum(float(r) for r in dims))
    i, k, l = float(i), float(k), float(l)
    return k / l + k * k / (3.0 * i * l) + k * k / (l * s) + k / s + k / (l * s) + 1.0 / s


def decide_fusion(ratio, threshold=1.0):
    if not np.isfinite(ratio):
        raise DomainError("decide_fusion: ratio not finite")
    return ratio > threshold


# ---------------------------------------------------------------------------
# query driver (cli.cpp:33-138) and measure_selectivity (benchgen.cpp:366-411)
# ---------------------------------------------------------------------------

def _pred(p, v):
    from paper_2306_08367_b200.query import Pred  # the workload's own predicate type
    assert isinstance(p, Pred)
    return p.matches(v)


def _link_pass(tables, q):
    """Per link: dim row of each fact row (or -1) after the dim filters."""
    fact = tables["lineorder"]
    alive = np.ones(len(next(iter(fact.values()))), bool)
    for f in q.filters:
        if f.target == -1:
            alive &= _pred(f.pred, np.asarray(fact[f.column]))
    rows = []
    for j, l in enumerate(q.joins):
        dim = tables[l.dim_name]
        pk = np.asarray(dim[l.dim_pk], np.int64)
        keep = np.ones(len(pk), bool)
        for f in q.filters:
            if f.target == j:
                keep &= _pred(f.pred, np.asarray(dim[f.column]))
        lut = np.full(int(pk.max()) + 1 if len(pk) else 1, -1, np.int64)
        kp = np.nonzero(keep)[0]
        lut[pk[kp]] = kp
        fk = np.asarray(fact[l.fact_fk], np.int64)
        inr = (fk >= 0) & (fk < len(lut))
        r = np.where(inr, lut[np.clip(fk, 0, len(lut) - 1)], -1)
        alive &= r >= 0
        rows.append(r)
    return alive, rows


def run_query(tables, q) -> np.ndarray:
    """run_query_laq (cli.cpp:73-138) semantics with exact int64 sums."""
    fact = tables["lineorder"]
    alive, rows = _link_pass(tables, q)
    vals = np.asarray(fact[q.measure], np.int64)[alive]
    if not q.group_by:
        return np.array([[float(vals.sum())]])
    gcols = []
    for g in q.group_by:
        if g.target == -1:
            gcols.append(np.asarray(fact[g.column], np.int64)[alive])
        else:
            dim = tables[q.joins[g.target].dim_name]
            gcols.append(np.asarray(dim[g.column], np.int64)[rows[g.target][alive]])
    if len(vals) == 0:
        return np.zeros((0, len(gcols) + 1))
    order = np.lexsort(tuple(gcols[::-1]))
    keys = np.stack([c[order] for c in gcols])
    v = vals[order]
    brk = np.ones(len(v), bool)
    brk[1:] = np.any(keys[:, 1:] != keys[:, :-1], axis=0)
    starts = np.nonzero(brk)[0]
    sums = np.add.reduceat(v, starts)  # int64: exact in any order
    out = np.zeros((len(starts), len(gcols) + 1))
    out[:, :-1] = keys[:, starts].T
    out[:, -1] = sums
    return out


def measure_selectivity(tables, q) -> float:
    """benchgen.cpp:366-411."""
    alive, _ = _link_pass(tables, q)
    n = len(alive)
    return 0.0 if n == 0 else float(np.count_nonzero(alive)) / float(n)


# ---------------------------------------------------------------------------
# report helpers (report.cpp:90-119) and rng (rng.hpp:41-51)
# ---------------------------------------------------------------------------

def fnv1a(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for c in data:
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def checksum_rows(m) -> int:
    """report.cpp:102-110: order-independent sum of per-row fnv hashes of '%.9g' values."""
    m = np.asarray(m, np.float64)
    if m.ndim == 1:
        m = m[:, None]
    total = (fnv1a(b"rows") + m.shape[1]) & 0xFFFFFFFFFFFFFFFF
    for row in m:
        h = 0xCBF29CE484222325
        for v in row:
            s = ("%.9g" % v).encode()
            h = ((fnv1a(s, h) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF) ^ 0x2C
        total = (total + h) & 0xFFFFFFFFFFFFFFFF
    return total
