"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/_ref/liblaq_ref.so.

oracle/_ref/liblaq_ref.so is the reference's own C++ implementation
(/root/reference/proj/src, compiled unmodified by oracle/Makefile) plus our
C-ABI wrapper oracle/ref_capi.cpp.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import this module; it is the checker and the CPU
baseline, never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "liblaq_ref.so")

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen_star.restype = C.c_void_p
        L.ref_gen_star.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.c_double, C.c_int64]
        L.ref_star_from_columns.restype = C.c_void_p
        L.ref_star_free.argtypes = [C.c_void_p]
        for n in ("ref_star_n_tables",):
            getattr(L, n).argtypes = [C.c_void_p]
        L.ref_star_table_name.restype = C.c_char_p
        L.ref_star_table_name.argtypes = [C.c_void_p, C.c_int]
        L.ref_star_table_rows.restype = C.c_int64
        L.ref_star_table_rows.argtypes = [C.c_void_p, C.c_int]
        L.ref_star_table_ncols.argtypes = [C.c_void_p, C.c_int]
        L.ref_star_col_name.restype = C.c_char_p
        L.ref_star_col_name.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_star_col_kind.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_star_col_data.restype = C.c_void_p
        L.ref_star_col_data.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_checksum_rows.restype = C.c_uint64
        L.ref_write_dataset.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.c_double, C.c_char_p]
        L.ref_load_csv.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_void_p),
                                   C.POINTER(C.c_int64)]
        L.ref_checksum_rows.argtypes = [f64p, C.c_int64, C.c_int64]
        L.ref_star_make_shards.argtypes = [C.c_void_p, C.c_int]
        vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
        sigs = {
            "ref_run_query": [vp, vp, i32, vp, i64, vp, vp, vp],
            "ref_run_query_sharded": [vp, vp, i32, vp, i64, vp, vp, vp],
            "ref_measure_selectivity": [vp, vp, vp],
            "ref_gen_queries": [vp, i32, vp, i32, vp, vp],
            "ref_build_key_domain": [vp, i64, vp, i64, vp, vp],
            "ref_update_key_domain": [vp, i64, vp, i64, vp, vp],
            "ref_key_matrix": [vp, i64, vp, i64, i32, vp, vp, vp, vp, vp, vp],
            "ref_mm_join": [vp, i64, vp, i64, vp, vp, i64, vp],
            "ref_star_join": [i32, vp, i64, vp, vp, vp, vp, vp, vp],
            "ref_oracle_star_join": [i32, vp, i64, vp, vp, vp, vp, i64, vp],
            "ref_groupby_sum_single": [vp, vp, i64, vp, vp, i64, vp, vp, vp],
            "ref_groupby_sum_multi": [i32, vp, vp, i64, vp, vp, i64, vp],
            "ref_prefuse_linear": [i32, vp, vp, vp, vp, vp, i64, i64, vp],
            "ref_apply_fused_linear": [i32, vp, i64, vp, vp, i64, vp],
            "ref_materialize_predict": [i32, vp, vp, vp, vp, i64, vp, i64, vp, i64, vp, vp],
            "ref_dense_matmul": [vp, i64, i64, vp, i64, vp],
            "ref_fused_pipeline": [i32, vp, i64, vp, vp, vp, vp, vp, i64, vp, vp, vp],
            "ref_speedup_ratio": [i32, i64, i64, i64, i64, vp, i32, vp],
            "ref_decide_fusion": [dbl, dbl, vp],
            "ref_gen_tree": [i64, i64, i64, C.c_uint64, i64, vp, vp, vp, vp, vp, vp, vp],
            "ref_predict_tree": [i32, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp],
            "ref_fused_tree": [i32, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, i64, vp, vp, i64, vp, vp],
        }
        for name, args in sigs.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p64(a: np.ndarray):
    return a.ctypes.data_as(i64p)


def _pf(a: np.ndarray):
    return a.ctypes.data_as(f64p)


def _ptr_array(arrs, ctype):
    arr = (C.POINTER(ctype) * len(arrs))()
    for i, a in enumerate(arrs):
        arr[i] = a.ctypes.data_as(C.POINTER(ctype)) if a is not None else C.POINTER(ctype)()
    return arr


# ---------------------------------------------------------------------------
# star schemas from the reference generator (benchgen.cpp:103-199)
# ---------------------------------------------------------------------------

SETTINGS = {"S1": 0, "S2": 1, "Ssb": 2}


class RefStar:
    """A reference StarSchema; tables exposed as dicts of numpy views."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        L = lib()
        self.tables: dict[str, dict[str, np.ndarray]] = {}
        self.kinds: dict[str, dict[str, int]] = {}
        for t in range(L.ref_star_n_tables(self.h)):
            name = L.ref_star_table_name(self.h, t).decode()
            rows = L.ref_star_table_rows(self.h, t)
            cols, kinds = {}, {}
            for c in range(L.ref_star_table_ncols(self.h, t)):
                cname = L.ref_star_col_name(self.h, t, c).decode()
                kind = L.ref_star_col_kind(self.h, t, c)
                ptr = L.ref_star_col_data(self.h, t, c)
                ct = C.c_double if kind == 2 else C.c_int64
                if rows:
                    buf = (ct * rows).from_address(ptr)
                    cols[cname] = np.frombuffer(buf, dtype=np.float64 if kind == 2 else np.int64)
                else:
                    cols[cname] = np.zeros(0, dtype=np.float64 if kind == 2 else np.int64)
                kinds[cname] = kind
            self.tables[name] = cols
            self.kinds[name] = kinds

    def __del__(self):
        try:
            lib().ref_star_free(self.h)
        except Exception:
            pass

    @property
    def fact(self):
        return self.tables["lineorder"]


def gen_star(setting="Ssb", sf=1, seed=42, feature_width=0, dangling=0.0, max_bytes=0) -> RefStar:
    L = lib()
    h = L.ref_gen_star(SETTINGS[setting], sf, seed, feature_width, dangling, max_bytes)
    if not h:
        raise RefError(-1, L.ref_last_error().decode())
    return RefStar(h)


def star_from_tables(tables: list[tuple[str, dict]], links: list[tuple[str, str, str]]) -> RefStar:
    """tables: [(name, {col: array})], first is the fact table. int64 arrays
    are Key columns when the name is a pk/fk in `links`, else Int; float64 → Float."""
    keycols = {l[0] for l in links} | {l[2] for l in links}
    L = lib()
    n = len(tables)
    names = (C.c_char_p * n)(*[t[0].encode() for t in tables])
    rows = (C.c_int64 * n)(*[len(next(iter(t[1].values()))) if t[1] else 0 for t in tables])
    ncols = (C.c_int * n)(*[len(t[1]) for t in tables])
    keep = []
    colnames = (C.POINTER(C.c_char_p) * n)()
    kinds = (C.POINTER(C.c_int) * n)()
    colptrs = (C.POINTER(C.c_void_p) * n)()
    for i, (_, cols) in enumerate(tables):
        cn = (C.c_char_p * len(cols))(*[c.encode() for c in cols])
        kd = (C.c_int * len(cols))()
        cp = (C.c_void_p * len(cols))()
        for j, (c, a) in enumerate(cols.items()):
            if a.dtype == np.float64:
                kd[j] = 2
            else:
                a = np.ascontiguousarray(a, dtype=np.int64)
                kd[j] = 0 if c in keycols else 1
            a = np.ascontiguousarray(a)
            keep.append(a)
            cp[j] = a.ctypes.data
        keep += [cn, kd, cp]
        colnames[i] = C.cast(cn, C.POINTER(C.c_char_p))
        kinds[i] = C.cast(kd, C.POINTER(C.c_int))
        colptrs[i] = C.cast(cp, C.POINTER(C.c_void_p))
    from paper_2306_08367_b200._abi import LinkDesc
    ls = (LinkDesc * len(links))(*[LinkDesc(a.encode(), b.encode(), c.encode()) for a, b, c in links])
    L.ref_star_from_columns.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    h = L.ref_star_from_columns(n, names, rows, ncols, colnames, kinds, colptrs, len(links), ls)
    if not h:
        raise RefError(-1, L.ref_last_error().decode())
    return RefStar(h)


# ---------------------------------------------------------------------------
# query driver (cli.cpp:73-232) and workload tuning (benchgen.cpp:366-457)
# ---------------------------------------------------------------------------

def run_query(star: RefStar, q, engine="laq", sharded=False):
    """Returns (result rows as float64 2-D array, seconds)."""
    from paper_2306_08367_b200.query import QueryDescHolder
    holder = QueryDescHolder(q)
    cap = 1 << 22
    out = np.zeros(cap, dtype=np.float64)
    rows, cols, secs = C.c_int64(), C.c_int64(), C.c_double()
    fn = lib().ref_run_query_sharded if sharded else lib().ref_run_query
    _check(fn(star.h, C.byref(holder.desc), 0 if engine == "laq" else 1, _pf(out), C.c_int64(cap),
              C.byref(rows), C.byref(cols), C.byref(secs)))
    return out[: rows.value * cols.value].reshape(rows.value, cols.value).copy(), secs.value


def make_shards(star: RefStar, n: int):
    _check(lib().ref_star_make_shards(star.h, n))


def measure_selectivity(star: RefStar, q) -> float:
    from paper_2306_08367_b200.query import QueryDescHolder
    holder = QueryDescHolder(q)
    out = C.c_double()
    _check(lib().ref_measure_selectivity(star.h, C.byref(holder.desc), C.byref(out)))
    return out.value


def gen_queries(star: RefStar, group: int, targets=()):
    t = np.asarray(targets if targets else [], dtype=np.float64)
    dials = np.zeros(3, dtype=np.int64)
    real = np.zeros(3, dtype=np.float64)
    tp = _pf(t) if len(t) else f64p()
    _check(lib().ref_gen_queries(star.h, group, tp, len(t), _p64(dials), _pf(real)))
    return dials, real


def _csr_args(m):
    rp = np.ascontiguousarray(m.row_ptr, np.int64)
    ci = np.ascontiguousarray(m.col_idx, np.int64)
    v = np.ascontiguousarray(m.values, np.float64)
    return (rp, ci, v), (rp.ctypes.data, ci.ctypes.data, v.ctypes.data, m.rows, m.cols)


def spmm(a, b):
    """matrix.cpp:81-123 -> (row_ptr, col_idx, values)."""
    ka, aa = _csr_args(a)
    kb, bb = _csr_args(b)
    cap = max(1, len(ka[1]) * max(1, b.cols))
    cap = min(cap, max(1, len(ka[1])) * max(1, int(np.diff(kb[0]).max()) if b.rows else 1))
    rp = np.zeros(a.rows + 1, np.int64)
    ci = np.zeros(cap, np.int64)
    cv = np.zeros(cap, np.float64)
    nnz = C.c_int64()
    L = lib()
    L.ref_spmm.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 2 + [C.c_void_p] * 3 + [C.c_int64] * 3 + \
        [C.c_void_p] * 3 + [C.c_void_p]
    _check(L.ref_spmm(*aa, *bb, cap, rp.ctypes.data, ci.ctypes.data, cv.ctypes.data, C.byref(nnz)))
    return rp, ci[: nnz.value].copy(), cv[: nnz.value].copy()


def csr_from_coo(row_idx, col_idx, values, rows, cols):
    r = np.ascontiguousarray(row_idx, np.int64)
    c = np.ascontiguousarray(col_idx, np.int64)
    v = np.ascontiguousarray(values, np.float64)
    rp = np.zeros(rows + 1 if rows >= 0 else 1, np.int64)
    L = lib()
    L.ref_csr_from_coo.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 3 + [C.c_void_p]
    _check(L.ref_csr_from_coo(r.ctypes.data, c.ctypes.data, v.ctypes.data, len(c), rows, cols, rp.ctypes.data))
    return rp


def coo_from_csr(m):
    k, a = _csr_args(m)
    out = np.zeros(max(1, len(k[1])), np.int64)
    L = lib()
    L.ref_coo_from_csr.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 2 + [C.c_void_p]
    _check(L.ref_coo_from_csr(*a[:3], m.rows, m.cols, out.ctypes.data))
    return out[: len(k[1])]


def sort_rows(t, key_cols, directions):
    t = np.ascontiguousarray(t, np.float64)
    out = np.zeros_like(t)
    k = np.ascontiguousarray(key_cols, np.int64)
    d = np.ascontiguousarray([1 if x == "Desc" else 0 for x in directions], np.int32)
    L = lib()
    L.ref_sort_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    _check(L.ref_sort_rows(t.ctypes.data, t.shape[0], t.shape[1], k.ctypes.data, d.ctypes.data, len(k),
                           out.ctypes.data))
    return out


def selection_mask(col, pred):
    """build_selection_mask (laqops.cpp:65-79) with a query.Pred."""
    col = np.asarray(col)
    is_float = col.dtype.kind == "f"
    col = np.ascontiguousarray(col, np.float64 if is_float else np.int64)
    out = np.zeros(max(1, len(col)), np.uint8)
    iset = np.ascontiguousarray(np.asarray(pred.values if not pred.is_float else [], np.int64))
    fset = np.ascontiguousarray(np.asarray(pred.values if pred.is_float else [], np.float64))
    L = lib()
    L.ref_selection_mask.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                     C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    _check(L.ref_selection_mask(col.ctypes.data, 1 if is_float else 0, len(col), pred.kind,
                                1 if pred.is_float else 0, int(pred.lo) if not pred.is_float else 0,
                                int(pred.hi) if not pred.is_float else 0,
                                float(pred.lo) if pred.is_float else 0.0, float(pred.hi) if pred.is_float else 0.0,
                                iset.ctypes.data, fset.ctypes.data, len(pred.values), out.ctypes.data))
    return out[: len(col)]


def cfg1_inputs(n_fact=1_000_000, dim_rows=10_000, k=16, l=1, seed=42):
    """cfg1 inputs from the reference's own Rng / gen_linear (ref_cfg1_inputs)."""
    fk = np.zeros(n_fact, np.int64)
    pk = np.zeros(dim_rows, np.int64)
    feats = np.zeros((dim_rows, k), np.float64)
    W = np.zeros((k, l), np.float64)
    L = lib()
    L.ref_cfg1_inputs.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]
    _check(L.ref_cfg1_inputs(n_fact, dim_rows, k, l, seed, fk.ctypes.data, pk.ctypes.data, feats.ctypes.data,
                             W.ctypes.data))
    return fk, pk, feats, W


def checksum_rows(m: np.ndarray) -> int:
    m = np.ascontiguousarray(m, dtype=np.float64)
    return int(lib().ref_checksum_rows(_pf(m), m.shape[0], m.shape[1] if m.ndim == 2 else 1))


# ---------------------------------------------------------------------------
# operators (laqops.cpp, fusion.cpp, matrix.cpp)
# ---------------------------------------------------------------------------

def build_key_domain(r, s):
    r = np.ascontiguousarray(r, np.int64); s = np.ascontiguousarray(s, np.int64)
    out = np.zeros(len(r) + len(s), np.int64); n = C.c_int64()
    _check(lib().ref_build_key_domain(_p64(r), len(r), _p64(s), len(s), _p64(out), C.byref(n)))
    return out[: n.value].copy()


def update_key_domain(dom, new):
    dom = np.ascontiguousarray(dom, np.int64); new = np.ascontiguousarray(new, np.int64)
    out = np.zeros(len(dom) + len(new), np.int64); n = C.c_int64()
    _check(lib().ref_update_key_domain(_p64(dom), len(dom), _p64(new), len(new), _p64(out), C.byref(n)))
    return out[: n.value].copy()


def key_matrix(keys, domain, orientation="RowsByDomain", values=None):
    keys = np.ascontiguousarray(keys, np.int64); domain = np.ascontiguousarray(domain, np.int64)
    n, d = len(keys), len(domain)
    rp = np.zeros(max(n, d) + 2, np.int64)
    ci = np.zeros(max(n, 1), np.int64)
    vv = np.zeros(max(n, 1), np.float64)
    nnz, rows = C.c_int64(), C.c_int64()
    vals = np.ascontiguousarray(values, np.float64) if values is not None else None
    _check(lib().ref_key_matrix(_p64(keys), n, _p64(domain), d, 0 if orientation == "RowsByDomain" else 1,
                                _pf(vals) if vals is not None else f64p(), _p64(rp), _p64(ci), _pf(vv),
                                C.byref(nnz), C.byref(rows)))
    return rp[: rows.value + 1].copy(), ci[: nnz.value].copy(), vv[: nnz.value].copy()


def mm_join(r, s):
    r = np.ascontiguousarray(r, np.int64); s = np.ascontiguousarray(s, np.int64)
    cap = max(1, len(r) * 4)
    while True:
        orr = np.zeros(cap, np.int64); oss = np.zeros(cap, np.int64); nnz = C.c_int64()
        rc = lib().ref_mm_join(_p64(r), len(r), _p64(s), len(s), _p64(orr), _p64(oss), cap, C.byref(nnz))
        if rc == 13 and nnz.value > cap:
            cap = nnz.value
            continue
        _check(rc)
        return orr[: nnz.value].copy(), oss[: nnz.value].copy()


def star_join(fks, pks):
    fks = [np.ascontiguousarray(f, np.int64) for f in fks]
    pks = [np.ascontiguousarray(p, np.int64) for p in pks]
    n = len(fks[0]) if fks else 0
    surv = np.zeros(max(n, 1), np.int64)
    outs = [np.zeros(max(n, 1), np.int64) for _ in fks]
    nnz = C.c_int64(); secs = C.c_double()
    prow = (C.c_int64 * len(pks))(*[len(p) for p in pks])
    _check(lib().ref_star_join(len(fks), _ptr_array(fks, C.c_int64), n, _ptr_array(pks, C.c_int64), prow,
                               _p64(surv), _ptr_array(outs, C.c_int64), C.byref(nnz), C.byref(secs)))
    m = nnz.value
    return surv[:m].copy(), [o[:m].copy() for o in outs]


def oracle_star_join(fks, pks):
    fks = [np.ascontiguousarray(f, np.int64) for f in fks]
    pks = [np.ascontiguousarray(p, np.int64) for p in pks]
    n = len(fks[0])
    cap = max(1, n * 4)
    while True:
        fr = np.zeros(cap, np.int64); outs = [np.zeros(cap, np.int64) for _ in fks]; nnz = C.c_int64()
        prow = (C.c_int64 * len(pks))(*[len(p) for p in pks])
        rc = lib().ref_oracle_star_join(len(fks), _ptr_array(fks, C.c_int64), n, _ptr_array(pks, C.c_int64),
                                        prow, _p64(fr), _ptr_array(outs, C.c_int64), cap, C.byref(nnz))
        if rc == 13 and nnz.value > cap:
            cap = nnz.value
            continue
        _check(rc)
        m = nnz.value
        return fr[:m].copy(), [o[:m].copy() for o in outs]


def groupby_sum_single(kr, vr, ks, gs):
    kr = np.ascontiguousarray(kr, np.int64); vr = np.ascontiguousarray(vr, np.float64)
    ks = np.ascontiguousarray(ks, np.int64); gs = np.ascontiguousarray(gs, np.int64)
    og = np.zeros(max(len(ks), 1), np.int64); osm = np.zeros(max(len(ks), 1), np.float64); n = C.c_int64()
    _check(lib().ref_groupby_sum_single(_p64(kr), _pf(vr), len(kr), _p64(ks), _p64(gs), len(ks),
                                        _p64(og), _pf(osm), C.byref(n)))
    return og[: n.value].copy(), osm[: n.value].copy()


def groupby_sum_multi(cols, vals):
    cols = [np.ascontiguousarray(c, np.int64) for c in cols]
    vals = np.ascontiguousarray(vals, np.float64)
    n = len(vals); cap = max(n, 1)
    keys = np.zeros(len(cols) * cap, np.int64); sums = np.zeros(cap, np.float64); ng = C.c_int64()
    _check(lib().ref_groupby_sum_multi(len(cols), _ptr_array(cols, C.c_int64), _pf(vals), n, _p64(keys),
                                       _pf(sums), cap, C.byref(ng)))
    g = ng.value
    return np.stack([keys[c * cap: c * cap + g] for c in range(len(cols))]) if cols else None, sums[:g].copy()


def _dims_args(dims, placements):
    dims = [np.ascontiguousarray(d, np.float64) for d in dims]
    pls = [np.ascontiguousarray(p, np.int64) for p in placements]
    rows = (C.c_int64 * len(dims))(*[d.shape[0] for d in dims])
    cols = (C.c_int64 * len(dims))(*[d.shape[1] for d in dims])
    return dims, pls, rows, cols


def prefuse_linear(dims, placements, L):
    dims, pls, rows, cols = _dims_args(dims, placements)
    L = np.ascontiguousarray(L, np.float64)
    k, l = L.shape
    parts = [np.zeros((d.shape[0], l), np.float64) for d in dims]
    _check(lib().ref_prefuse_linear(len(dims), _ptr_array(dims, C.c_double), rows, cols,
                                    _ptr_array(pls, C.c_int64), _pf(L), k, l, _ptr_array(parts, C.c_double)))
    return parts


def apply_fused_linear(idx, partials):
    idx = [np.ascontiguousarray(i, np.int64) for i in idx]
    partials = [np.ascontiguousarray(p, np.float64) for p in partials]
    m = len(idx[0]); l = partials[0].shape[1]
    out = np.zeros((m, l), np.float64)
    prow = (C.c_int64 * len(partials))(*[p.shape[0] for p in partials])
    _check(lib().ref_apply_fused_linear(len(idx), _ptr_array(idx, C.c_int64), m,
                                        _ptr_array(partials, C.c_double), prow, l, _pf(out)))
    return out


def materialize_predict(dims, placements, k, idx, L=None):
    dims, pls, rows, cols = _dims_args(dims, placements)
    idx = [np.ascontiguousarray(i, np.int64) for i in idx]
    m = len(idx[0])
    T = np.zeros((m, k), np.float64)
    if L is not None:
        L = np.ascontiguousarray(L, np.float64)
        Y = np.zeros((m, L.shape[1]), np.float64)
    _check(lib().ref_materialize_predict(len(dims), _ptr_array(dims, C.c_double), rows, cols,
                                         _ptr_array(pls, C.c_int64), k, _ptr_array(idx, C.c_int64), m,
                                         _pf(L) if L is not None else f64p(), L.shape[1] if L is not None else 0,
                                         _pf(T), _pf(Y) if L is not None else f64p()))
    return (T, Y) if L is not None else T


def dense_matmul(a, b):
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    c = np.zeros((a.shape[0], b.shape[1]), np.float64)
    _check(lib().ref_dense_matmul(_pf(a), a.shape[0], a.shape[1], _pf(b), b.shape[1], _pf(c)))
    return c


def fused_pipeline(fks, pks, feats, L):
    """cfg1 path through the reference API; returns (Y, [join, csr, prefuse, apply] seconds)."""
    fks = [np.ascontiguousarray(f, np.int64) for f in fks]
    pks = [np.ascontiguousarray(p, np.int64) for p in pks]
    feats = [np.ascontiguousarray(f, np.float64) for f in feats]
    L = np.ascontiguousarray(L, np.float64)
    n = len(fks[0]); l = L.shape[1]
    y = np.zeros((n, l), np.float64); nnz = C.c_int64(); secs = np.zeros(4, np.float64)
    prow = (C.c_int64 * len(pks))(*[len(p) for p in pks])
    kj = (C.c_int64 * len(feats))(*[f.shape[1] for f in feats])
    _check(lib().ref_fused_pipeline(len(fks), _ptr_array(fks, C.c_int64), n, _ptr_array(pks, C.c_int64), prow,
                                    _ptr_array(feats, C.c_double), kj, _pf(L), l, _pf(y), C.byref(nnz), _pf(secs)))
    return y[: nnz.value], secs


def speedup_ratio(i, k, l, dims, tree=False, p=None):
    d = np.ascontiguousarray(dims, np.int64)
    out = C.c_double()
    _check(lib().ref_speedup_ratio(1 if tree else 0, i, k, l, p if p is not None else k,
                                   _p64(d) if len(d) else i64p(), len(d), C.byref(out)))
    return out.value


def decide_fusion(ratio, threshold=1.0):
    out = C.c_int()
    _check(lib().ref_decide_fusion(C.c_double(ratio), C.c_double(threshold), C.byref(out)))
    return bool(out.value)


# ---- decision trees -------------------------------------------------------------
# A tree is a dict of node arrays: is_leaf (int32), feature, threshold, true_child,
# false_child, label (TreeNode, mlops.hpp:18-25; root = node 0).

def _tree_args(t):
    a = [np.ascontiguousarray(t["is_leaf"], np.int32), np.ascontiguousarray(t["feature"], np.int64),
         np.ascontiguousarray(t["threshold"], np.float64), np.ascontiguousarray(t["true_child"], np.int64),
         np.ascontiguousarray(t["false_child"], np.int64), np.ascontiguousarray(t["label"], np.int64)]
    return a, [x.ctypes.data for x in a]


def gen_tree(k, p, leaves, seed):
    """bench::gen_tree (benchgen.cpp:463-...)."""
    cap = 2 * leaves + 1
    t = {"is_leaf": np.zeros(cap, np.int32), "feature": np.zeros(cap, np.int64), "threshold": np.zeros(cap),
         "true_child": np.zeros(cap, np.int64), "false_child": np.zeros(cap, np.int64),
         "label": np.zeros(cap, np.int64)}
    n = C.c_int64()
    _check(lib().ref_gen_tree(k, p, leaves, seed, cap, *[t[x].ctypes.data for x in
                                                          ("is_leaf", "feature", "threshold", "true_child",
                                                           "false_child", "label")], C.byref(n)))
    return {x: v[:n.value].copy() for x, v in t.items()}


def predict_tree(tree, T):
    keep, ptrs = _tree_args(tree)
    T = np.ascontiguousarray(T, np.float64)
    out = np.zeros(T.shape[0], np.int64)
    _check(lib().ref_predict_tree(len(keep[0]), *ptrs, _pf(T), T.shape[0], T.shape[1], _p64(out)))
    return out


def fused_tree(tree, dims, placements, k, feature_owner, idx=None):
    """Returns (labels or None, partials) through prefuse_tree / apply_fused_tree."""
    keep, ptrs = _tree_args(tree)
    dims_, pls, rows, cols = _dims_args(dims, placements)
    owner = np.ascontiguousarray(feature_owner, np.int64)
    leaves = int(np.sum(keep[0] != 0))
    parts = [np.zeros((d.shape[0], leaves)) for d in dims_]
    if idx is not None:
        idx = [np.ascontiguousarray(i, np.int64) for i in idx]
        m = len(idx[0])
        out = np.zeros(m, np.int64)
        ip = _ptr_array(idx, C.c_int64)
    else:
        m, out, ip = 0, None, None
    _check(lib().ref_fused_tree(len(keep[0]), *ptrs, len(dims_), _ptr_array(dims_, C.c_double), rows, cols,
                                _ptr_array(pls, C.c_int64), k, _p64(owner), ip, m,
                                _p64(out) if out is not None else None, _ptr_array(parts, C.c_double)))
    return out, parts


# ---- dataset files (cli.cpp:430-481, storage.cpp:112-150) ---------------------

SETTINGS = {"S1": 0, "S2": 1, "Ssb": 2}


def write_dataset(directory, setting="S2", sf=1, seed=42, features=0, dangling=0.0):
    """The reference's write_dataset (CSV tables + manifest.json) for gen_star(cfg)."""
    L = lib()
    rc = L.ref_write_dataset(SETTINGS[setting], sf, seed, features, dangling, str(directory).encode())
    if rc:
        raise RefError(rc, L.ref_last_error().decode())


def load_csv(path, kinds, cap):
    """The reference's load_csv -> (columns list, rows) or RefError(code, message)."""
    L = lib()
    cols = [np.zeros(max(cap, 1), np.float64 if k == 2 else np.int64) for k in kinds]
    kd = (C.c_int32 * len(kinds))(*kinds)
    ptrs = (C.c_void_p * len(kinds))(*[c.ctypes.data for c in cols])
    rows = C.c_int64()
    rc = L.ref_load_csv(str(path).encode(), len(kinds), kd, cap, ptrs, C.byref(rows))
    if rc:
        raise RefError(rc, L.ref_last_error().decode())
    return [c[:rows.value] for c in cols], rows.value
