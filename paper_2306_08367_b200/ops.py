"""laq::ops on the device (mirror of proj/include/laq/laqops.hpp).

Each function takes numpy arrays (host, like the reference's std::vector
arguments; results come back as numpy) or CUDA tensors (device-resident;
results stay on the device).  All compute runs in liblaq_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import errors
from .device import context, dev, host, ptrs

i64 = torch.int64


def _is_dev(*xs) -> bool:
    return any(isinstance(x, torch.Tensor) and x.is_cuda for x in xs)


def _out(t: torch.Tensor, on_dev: bool):
    return t if on_dev else host(t)


@dataclass
class KeyDomain:
    """laqops.hpp:54-65: sorted distinct keys; position = index."""
    sorted_keys: np.ndarray | torch.Tensor

    def size(self) -> int:
        return int(self.sorted_keys.shape[0])

    def position(self, key: int) -> int:
        k = host(self.sorted_keys) if isinstance(self.sorted_keys, torch.Tensor) else self.sorted_keys
        i = int(np.searchsorted(k, key))
        if i >= len(k) or k[i] != key:
            raise errors.DomainError(f"key {key} not in domain")
        return i

    def contains(self, key: int) -> bool:
        try:
            self.position(key)
            return True
        except errors.DomainError:
            return False


def build_key_domain(keys_r, keys_s, sorted: bool = True) -> KeyDomain:  # noqa: A002
    """laqops.cpp:142-155 (K1 domain_build)."""
    on = _is_dev(keys_r, keys_s)
    ctx = context()
    r, s = dev(keys_r, i64), dev(keys_s, i64)
    out = torch.empty(max(1, r.numel() + s.numel()), dtype=i64, device=r.device)
    n = C.c_int64()
    ctx.check(ctx.lib.laq_build_key_domain(ctx.h, r.data_ptr(), r.numel(), s.data_ptr(), s.numel(),
                                           out.data_ptr(), C.byref(n)))
    return KeyDomain(_out(out[: n.value], on))


def update_key_domain(d: KeyDomain, new_keys) -> KeyDomain:
    """laqops.cpp:157-171."""
    on = _is_dev(d.sorted_keys, new_keys)
    ctx = context()
    a, b = dev(d.sorted_keys, i64), dev(new_keys, i64)
    out = torch.empty(max(1, a.numel() + b.numel()), dtype=i64, device=a.device)
    n = C.c_int64()
    ctx.check(ctx.lib.laq_update_key_domain(ctx.h, a.data_ptr(), a.numel(), b.data_ptr(), b.numel(),
                                            out.data_ptr(), C.byref(n)))
    return KeyDomain(_out(out[: n.value], on))


@dataclass
class Csr:
    """SparseCsr (matrix.hpp:42-58)."""
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray


def key_matrix(keys, domain: KeyDomain, orientation: str = "RowsByDomain", values=None) -> Csr:
    """laqops.cpp:173-220."""
    ctx = context()
    k = dev(keys, i64)
    d = dev(domain.sorted_keys, i64)
    n, nd = k.numel(), d.numel()
    if values is not None and len(values) != n:
        raise errors.ShapeError("key_matrix: values length mismatch")
    v = dev(values, torch.float64) if values is not None else None
    if orientation == "RowsByDomain":
        pos = torch.empty(max(n, 1), dtype=i64, device=k.device)
        ctx.check(ctx.lib.laq_key_positions(ctx.h, k.data_ptr(), n, d.data_ptr(), nd, pos.data_ptr()))
        pos = host(pos[:n])
        vals = np.ones(n) if v is None else host(v)
        keep = vals != 0.0  # laqops.cpp:188-190
        row_ptr = np.concatenate([[0], np.cumsum(keep)]).astype(np.int64)
        return Csr(n, nd, row_ptr, pos[keep], vals[keep])
    row_ptr = torch.empty(nd + 1, dtype=i64, device=k.device)
    col = torch.empty(max(n, 1), dtype=i64, device=k.device)
    ov = torch.empty(max(n, 1), dtype=torch.float64, device=k.device)
    nnz = C.c_int64()
    ctx.check(ctx.lib.laq_key_matrix_dbr(ctx.h, k.data_ptr(), n, d.data_ptr(), nd,
                                         v.data_ptr() if v is not None else None, row_ptr.data_ptr(),
                                         col.data_ptr(), ov.data_ptr(), C.byref(nnz)))
    m = nnz.value
    return Csr(nd, n, host(row_ptr), host(col[:m]), host(ov[:m]))


@dataclass
class RowMatch:
    """RowMatch (laqops.hpp:85-89): canonical COO of matched (r, s) pairs."""
    rows: int
    cols: int
    row_idx: np.ndarray | torch.Tensor
    col_idx: np.ndarray | torch.Tensor

    def nnz(self) -> int:
        return int(self.col_idx.shape[0])


def mm_join(keys_r, keys_s, domain: KeyDomain | None = None) -> RowMatch:
    """laqops.cpp:222-231 (many-to-many, (r asc, s asc)).  A cached superset
    domain only validates: the result is identical (test_laqops.cpp:256-262)."""
    on = _is_dev(keys_r, keys_s)
    ctx = context()
    r, s = dev(keys_r, i64), dev(keys_s, i64)
    if domain is not None:  # every key must be in the domain (KeyDomain::position)
        pos = torch.empty(max(1, r.numel() + s.numel()), dtype=i64, device=r.device)
        dd = dev(domain.sorted_keys, i64)
        for t in (r, s):
            ctx.check(ctx.lib.laq_key_positions(ctx.h, t.data_ptr(), t.numel(), dd.data_ptr(), dd.numel(),
                                                pos.data_ptr()))
    cap = max(1, r.numel())
    while True:
        orr = torch.empty(cap, dtype=i64, device=r.device)
        oss = torch.empty(cap, dtype=i64, device=r.device)
        nnz = C.c_int64()
        rc = ctx.lib.laq_mm_join(ctx.h, r.data_ptr(), r.numel(), s.data_ptr(), s.numel(), orr.data_ptr(),
                                 oss.data_ptr(), cap, C.byref(nnz))
        if rc == 13 and nnz.value > cap:
            cap = nnz.value
            continue
        ctx.check(rc)
        m = nnz.value
        return RowMatch(r.numel(), s.numel(), _out(orr[:m], on), _out(oss[:m], on))


def multiway_star_join(fact_fks, dim_pks):
    """laqops.cpp:233-319: (survivors, [dim rows per link]) in ascending fact order.
    fact_fks[j] are the fact's fk columns, dim_pks[j] the dims' pk columns."""
    on = _is_dev(*fact_fks, *dim_pks)
    ctx = context()
    fks = [dev(f, i64) for f in fact_fks]
    pks = [dev(p, i64) for p in dim_pks]
    n = fks[0].numel() if fks else 0
    surv = torch.empty(max(n, 1), dtype=i64, device="cuda")
    outs = [torch.empty(max(n, 1), dtype=i64, device="cuda") for _ in fks]
    nnz = C.c_int64()
    prow = (C.c_int64 * max(1, len(pks)))(*[p.numel() for p in pks])
    ctx.check(ctx.lib.laq_star_join(ctx.h, len(fks), ptrs(fks), n, ptrs(pks), prow, surv.data_ptr(),
                                    ptrs(outs), C.byref(nnz)))
    m = nnz.value
    return _out(surv[:m], on), [_out(o[:m], on) for o in outs]


def materialize(i_maps, dims, placements, k: int):
    """laqops.cpp:338-374: T = sum_j I_j B_j M_j (one-hot gathers)."""
    on = _is_dev(*i_maps, *dims)
    ctx = context()
    idx = [dev(i, i64) for i in i_maps]
    B = [dev(d, torch.float64) for d in dims]
    rows = idx[0].numel() if idx else 0
    for i in idx:
        if i.numel() != rows:
            raise errors.ShapeError("materialize: row mapping row counts differ")
    pl = [np.ascontiguousarray(p, np.int64) for p in placements]
    plp = (C.POINTER(C.c_int64) * len(pl))(*[p.ctypes.data_as(C.POINTER(C.c_int64)) for p in pl])
    out = torch.empty((rows, k), dtype=torch.float64, device="cuda")
    drows = (C.c_int64 * len(B))(*[b.shape[0] for b in B])
    dcols = (C.c_int64 * len(B))(*[b.shape[1] for b in B])
    ctx.check(ctx.lib.laq_materialize(ctx.h, len(idx), ptrs(idx), rows, ptrs(B), drows, dcols,
                                      C.cast(plp, C.c_void_p), k, out.data_ptr()))
    return _out(out, on)


def groupby_sum_single(keys_r, vals_r, keys_s, group_s):
    """laqops.cpp:376-413 -> (groups ascending, sums) incl. zero-sum groups."""
    if len(keys_r) != len(vals_r):
        raise errors.ShapeError("groupby_sum_single: R lengths")
    if len(keys_s) != len(group_s):
        raise errors.ShapeError("groupby_sum_single: S lengths")
    on = _is_dev(keys_r, vals_r, keys_s, group_s)
    ctx = context()
    kr, vr = dev(keys_r, i64), dev(vals_r, torch.float64)
    ks, gs = dev(keys_s, i64), dev(group_s, i64)
    og = torch.empty(max(1, ks.numel()), dtype=i64, device="cuda")
    osm = torch.empty(max(1, ks.numel()), dtype=torch.float64, device="cuda")
    n = C.c_int64()
    ctx.check(ctx.lib.laq_groupby_sum_single(ctx.h, kr.data_ptr(), vr.data_ptr(), kr.numel(), ks.data_ptr(),
                                             gs.data_ptr(), ks.numel(), og.data_ptr(), osm.data_ptr(), C.byref(n)))
    return _out(og[: n.value], on), _out(osm[: n.value], on)


def groupby_sum_multi(group_cols, vals):
    """laqops.cpp:415-455 -> (keys [n_cols x G], sums [G]), present tuples ascending."""
    if len(group_cols) == 0:
        raise errors.ShapeError("groupby_sum_multi: no group columns")
    for c in group_cols:
        if len(c) != len(vals):
            raise errors.ShapeError("groupby_sum_multi: column length mismatch")
    on = _is_dev(*group_cols, vals)
    ctx = context()
    cols = [dev(c, i64) for c in group_cols]
    v = dev(vals, torch.float64)
    n = v.numel()
    cap = max(n, 1)
    keys = torch.empty((len(cols), cap), dtype=i64, device="cuda")
    sums = torch.empty(cap, dtype=torch.float64, device="cuda")
    ng = C.c_int64()
    ctx.check(ctx.lib.laq_groupby_sum_multi(ctx.h, len(cols), ptrs(cols), v.data_ptr(), n, keys.data_ptr(),
                                            sums.data_ptr(), cap, C.byref(ng)))
    g = ng.value
    return _out(keys[:, :g], on), _out(sums[:g], on)


def sort_rows(t: np.ndarray, key_cols, directions):
    """laqops.cpp:457-478 (host; ORDER BY over <= a few hundred result rows)."""
    if len(key_cols) != len(directions):
        raise errors.ShapeError("sort_rows: key/direction counts")
    t = np.asarray(t)
    for c in key_cols:
        if c < 0 or c >= t.shape[1]:
            raise errors.IndexError(f"sort_rows: key column {c}")
    order = np.arange(t.shape[0])
    for c, d in reversed(list(zip(key_cols, directions))):  # stable LSD passes
        col = t[order, c]
        o = np.argsort(-col if d == "Desc" else col, kind="stable")
        order = order[o]
    return t[order]
