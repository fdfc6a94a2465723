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


def sort_rows(t, key_cols, directions):
    """laqops.cpp:457-478 on the device (laq_sort_rows): stable lexicographic,
    directions "Asc" / "Desc"."""
    if len(key_cols) != len(directions):
        raise errors.ShapeError("sort_rows: key/direction counts")
    on = _is_dev(t)
    ctx = context()
    d = dev(t, torch.float64)
    if d.dim() != 2:
        raise errors.ShapeError("sort_rows: matrix expected")
    rows, cols = d.shape
    out = torch.empty((max(rows, 1), max(cols, 1)), dtype=torch.float64, device="cuda")[:rows, :cols].contiguous()
    kc = (C.c_int64 * max(1, len(key_cols)))(*[int(c) for c in key_cols])
    kd = (C.c_int32 * max(1, len(key_cols)))(*[1 if x == "Desc" else 0 for x in directions])
    ctx.check(ctx.lib.laq_sort_rows(ctx.h, d.data_ptr(), rows, cols, kc, kd, len(key_cols), out.data_ptr()))
    return _out(out, on)


# ---------------------------------------------------------------------------
# sparse formats and SpGEMM (matrix.hpp:44-100)
# ---------------------------------------------------------------------------

@dataclass
class Coo:
    """SparseCoo (matrix.hpp:60-71)."""
    rows: int
    cols: int
    row_idx: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(len(self.col_idx))


def _chk_coo(c):
    if c.rows < 0 or c.cols < 0:
        raise errors.Error("coo: negative dimension")
    if len(c.row_idx) != len(c.col_idx) or len(c.values) != len(c.col_idx):
        raise errors.Error("coo: index/value length mismatch")


def csr_from_coo(c: Coo) -> Csr:
    """matrix.cpp:210-221 (check_canonical first, matrix.cpp:243-255)."""
    _chk_coo(c)
    ctx = context()
    r, ci = dev(c.row_idx, i64), dev(c.col_idx, i64)
    rp = torch.empty(c.rows + 1, dtype=i64, device="cuda")
    ctx.check(ctx.lib.laq_csr_from_coo(ctx.h, r.data_ptr(), ci.data_ptr(), len(c.col_idx), c.rows, c.cols,
                                       rp.data_ptr()))
    return Csr(c.rows, c.cols, host(rp), np.asarray(c.col_idx, np.int64).copy(), np.asarray(c.values, np.float64).copy())


def coo_from_csr(m: Csr) -> Coo:
    """matrix.cpp:198-208."""
    ctx = context()
    rp = dev(m.row_ptr, i64)
    nnz = len(m.col_idx)
    out = torch.empty(max(nnz, 1), dtype=i64, device="cuda")
    ctx.check(ctx.lib.laq_coo_from_csr(ctx.h, rp.data_ptr(), m.rows, nnz, out.data_ptr()))
    return Coo(m.rows, m.cols, host(out[:nnz]), np.asarray(m.col_idx, np.int64).copy(),
               np.asarray(m.values, np.float64).copy())


def spmm(a: Csr, b: Csr) -> Csr:
    """matrix.cpp:81-123: Gustavson SpGEMM, bit-identical (laq_spmm)."""
    if a.cols != b.rows:
        raise errors.ShapeError(f"spmm: {a.rows}x{a.cols} x {b.rows}x{b.cols}")
    ctx = context()
    ar, ac, av = dev(a.row_ptr, i64), dev(a.col_idx, i64), dev(a.values, torch.float64)
    br, bc, bv = dev(b.row_ptr, i64), dev(b.col_idx, i64), dev(b.values, torch.float64)
    rp = torch.empty(a.rows + 1, dtype=i64, device="cuda")
    cap = max(1, len(a.col_idx), len(b.col_idx))
    while True:
        ci = torch.empty(cap, dtype=i64, device="cuda")
        cv = torch.empty(cap, dtype=torch.float64, device="cuda")
        nnz = C.c_int64()
        rc = ctx.lib.laq_spmm(ctx.h, ar.data_ptr(), ac.data_ptr(), av.data_ptr(), a.rows, a.cols, br.data_ptr(),
                              bc.data_ptr(), bv.data_ptr(), b.rows, b.cols, rp.data_ptr(), ci.data_ptr(),
                              cv.data_ptr(), cap, C.byref(nnz))
        if rc == 13 and nnz.value > cap:
            cap = nnz.value
            continue
        ctx.check(rc)
        m = nnz.value
        return Csr(a.rows, b.cols, host(rp), host(ci[:m]), host(cv[:m]))


def row_mapping_matrices(match: RowMatch):
    """laqops.cpp:321-336: (I_R, I_S) one-hot CSR from a canonical RowMatch
    (validated on the device, check_canonical)."""
    ctx = context()
    r, s = dev(match.row_idx, i64), dev(match.col_idx, i64)
    ctx.check(ctx.lib.laq_coo_check(ctx.h, r.data_ptr(), s.data_ptr(), r.numel(), match.rows, match.cols))
    n = r.numel()
    rp = np.arange(n + 1, dtype=np.int64)
    return (Csr(n, match.rows, rp, host(r), np.ones(n)), Csr(n, match.cols, rp.copy(), host(s), np.ones(n)))


# ---------------------------------------------------------------------------
# selection (laqops.cpp:65-121, predicate.hpp:81-103)
# ---------------------------------------------------------------------------

def _pred_desc(p):
    from . import _abi
    keep = []
    d = _abi.PredDesc()
    d.kind, d.is_float = p.kind, 1 if p.is_float else 0
    if p.is_float:
        d.flo, d.fhi = float(p.lo), float(p.hi)
        fs = np.ascontiguousarray(np.asarray(p.values, np.float64))
        keep.append(fs)
        d.fset = fs.ctypes.data_as(_abi.f64p) if len(fs) else _abi.f64p()
        d.set_len = len(fs)
    else:
        d.ilo, d.ihi = int(p.lo), int(p.hi)
        si = np.ascontiguousarray(np.asarray(p.values, np.int64))
        keep.append(si)
        d.iset = si.ctypes.data_as(_abi.i64p) if len(si) else _abi.i64p()
        d.set_len = len(si)
    return d, keep


def build_selection_mask(col, pred):
    """laqops.cpp:65-79: uint8 mask of pred.matches(col[i]) (TypeError on a
    typed mismatch over a non-empty column)."""
    on = _is_dev(col)
    ctx = context()
    is_float = (col.dtype == torch.float64) if isinstance(col, torch.Tensor) else np.asarray(col).dtype.kind == "f"
    c = dev(col, torch.float64 if is_float else i64)
    n = c.numel()
    m = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
    d, keep = _pred_desc(pred)
    ctx.check(ctx.lib.laq_selection_mask(ctx.h, c.data_ptr(), 1 if is_float else 0, n, C.byref(d), m.data_ptr(), 0))
    return _out(m[:n], on)


def mask_and(a, b):
    """laqops.cpp:87-93."""
    if len(a) != len(b):
        raise errors.ShapeError("mask_and: length mismatch")
    on = _is_dev(a, b)
    ctx = context()
    x, y = dev(a, torch.uint8), dev(b, torch.uint8)
    out = torch.empty(max(x.numel(), 1), dtype=torch.uint8, device="cuda")
    ctx.check(ctx.lib.laq_mask_and(ctx.h, x.data_ptr(), y.data_ptr(), x.numel(), out.data_ptr()))
    return _out(out[: x.numel()], on)


def mask_indices(mask):
    on = _is_dev(mask)
    ctx = context()
    m = dev(mask, torch.uint8)
    out = torch.empty(max(m.numel(), 1), dtype=i64, device="cuda")
    n = C.c_int64()
    ctx.check(ctx.lib.laq_mask_indices(ctx.h, m.data_ptr(), m.numel(), out.data_ptr(), C.byref(n)))
    return _out(out[: n.value], on)


def apply_mask(table, mask):
    """laqops.cpp:95-121: rows whose mask is set, in order.  table: a 2-D
    matrix (DenseMat) or a {column: array} dict (Table)."""
    on = _is_dev(mask)
    ctx = context()
    idx = mask_indices(dev(mask, torch.uint8))
    n = idx.numel()

    def gather(a, row_elems, a_dev):
        src = dev(a)
        kind = {torch.int32: 0, torch.int64: 1, torch.float64: 2}[src.dtype]
        out = torch.empty((max(n, 1), row_elems) if row_elems > 1 else (max(n, 1),),
                          dtype=torch.float64 if kind == 2 else i64, device="cuda")
        ctx.check(ctx.lib.laq_gather(ctx.h, src.data_ptr(), kind, row_elems, idx.data_ptr(), n, out.data_ptr(),
                                     2 if kind == 2 else 1))
        return _out(out[:n], on or a_dev)

    if isinstance(table, dict):
        for c, a in table.items():
            if len(a) != len(mask):
                raise errors.ShapeError("apply_mask: mask length mismatch")
        return {c: gather(a, 1, isinstance(a, torch.Tensor)) for c, a in table.items()}
    t = dev(table, torch.float64)
    if t.shape[0] != len(mask):
        raise errors.ShapeError("apply_mask: mask length mismatch")
    return gather(t, t.shape[1], isinstance(table, torch.Tensor))
