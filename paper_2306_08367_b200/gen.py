"""Host-side synthetic star schemas (bit-exact restatement of the reference
generator, benchgen.cpp:13-199 / rng.hpp) via _native/liblaq_gen.so.

gen_star(...) returns a GenStar whose .tables map table name -> {column: numpy
array} (int64, or int32 when narrow=True; float64 features).  Arrays are views
into native memory owned by the GenStar object.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors
from ._abi import GEN_LIB_PATH

SETTINGS = {"S1": 0, "S2": 1, "Ssb": 2}
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(GEN_LIB_PATH):
            raise errors.Error(f"{GEN_LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(GEN_LIB_PATH)
        L.laqgen_last_error.restype = C.c_char_p
        L.laqgen_star_create.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.c_double, C.c_int64,
                                         C.c_int, C.POINTER(C.c_void_p)]
        L.laqgen_star_create_tagged.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.c_double, C.c_int64,
                                                C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]
        L.laqgen_star_create_shard.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.c_double, C.c_int64,
                                               C.c_int, C.c_char_p, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]
        L.laqgen_star_destroy.argtypes = [C.c_void_p]
        L.laqgen_n_tables.argtypes = [C.c_void_p]
        L.laqgen_table_name.restype = C.c_char_p
        L.laqgen_table_name.argtypes = [C.c_void_p, C.c_int]
        L.laqgen_table_rows.restype = C.c_int64
        L.laqgen_table_rows.argtypes = [C.c_void_p, C.c_int]
        L.laqgen_table_ncols.argtypes = [C.c_void_p, C.c_int]
        L.laqgen_col_name.restype = C.c_char_p
        L.laqgen_col_name.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.laqgen_col_kind.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.laqgen_col_width.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.laqgen_col_data.restype = C.c_void_p
        L.laqgen_col_data.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.laqgen_gen_linear.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]
        L.laqgen_range.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.laqgen_unit_matrix.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_int64, C.c_void_p]
        L.laqgen_fastmod.restype = C.c_uint64
        L.laqgen_fastmod.argtypes = [C.c_uint64, C.c_uint64]
        _lib = L
    return _lib


class GenStar:
    def __init__(self, handle, narrow):
        self.h = C.c_void_p(handle)
        self.narrow = narrow
        L = lib()
        self.tables: dict[str, dict[str, np.ndarray]] = {}
        self.kinds: dict[str, dict[str, int]] = {}
        for t in range(L.laqgen_n_tables(self.h)):
            name = L.laqgen_table_name(self.h, t).decode()
            rows = L.laqgen_table_rows(self.h, t)
            cols, kinds = {}, {}
            for c in range(L.laqgen_table_ncols(self.h, t)):
                cn = L.laqgen_col_name(self.h, t, c).decode()
                kind = L.laqgen_col_kind(self.h, t, c)
                width = L.laqgen_col_width(self.h, t, c)
                dt = np.float64 if kind == 2 else (np.int32 if width == 4 else np.int64)
                ptr = L.laqgen_col_data(self.h, t, c)
                if rows:
                    buf = (C.c_char * (rows * width)).from_address(ptr)
                    cols[cn] = np.frombuffer(buf, dtype=dt)
                else:
                    cols[cn] = np.zeros(0, dtype=dt)
                kinds[cn] = kind
            self.tables[name] = cols
            self.kinds[name] = kinds

    def __del__(self):
        try:
            lib().laqgen_star_destroy(self.h)
        except Exception:
            pass

    @property
    def fact(self):
        return self.tables["lineorder"]

    def links(self):
        """StarSchema links (benchgen.cpp:154-158)."""
        ls = [("lo_part", "part", "p_key"), ("lo_supplier", "supplier", "s_key"),
              ("lo_orderdate", "date", "d_key"), ("lo_commitdate", "date", "d_key")]
        if "customer" in self.tables:
            ls.append(("lo_customer", "customer", "c_key"))
        return ls


def gen_star(setting="Ssb", sf=1, seed=42, feature_width=0, dangling=0.0, max_bytes=0, narrow=False,
             fact_tag=None, row_range=None) -> GenStar:
    """gen_star (benchgen.cpp:190-193).  fact_tag: draw the fact table from an
    independent stream over the same dimensions.  row_range=(lo, hi): keep only
    lineorder rows [lo, hi) of the canonical table (a row shard: the full
    stream is drawn, only the shard is stored)."""
    h = C.c_void_p()
    lo, hi = row_range if row_range is not None else (0, -1)
    rc = lib().laqgen_star_create_shard(SETTINGS[setting], sf, seed, feature_width, dangling, max_bytes,
                                        1 if narrow else 0, fact_tag.encode() if fact_tag else None, lo, hi,
                                        C.byref(h))
    errors.raise_for(rc, lib().laqgen_last_error().decode())
    return GenStar(h.value, narrow)


def gen_linear(k: int, l: int, seed: int) -> np.ndarray:
    """benchgen.cpp:512-518."""
    out = np.zeros((k, l), np.float64)
    rc = lib().laqgen_gen_linear(k, l, seed, out.ctypes.data)
    errors.raise_for(rc, lib().laqgen_last_error().decode())
    return out


def rng_range(seed: int, tag, n: int, lo: int, hi: int, dtype=np.int64) -> np.ndarray:
    out = np.zeros(n, dtype)
    p64 = out.ctypes.data if dtype == np.int64 else None
    p32 = out.ctypes.data if dtype == np.int32 else None
    lib().laqgen_range(seed, tag.encode() if tag else None, n, lo, hi, p64, p32)
    return out


def unit_matrix(seed: int, tag, rows: int, cols: int) -> np.ndarray:
    out = np.zeros((rows, cols), np.float64)
    lib().laqgen_unit_matrix(seed, tag.encode() if tag else None, rows, cols, out.ctypes.data)
    return out


def cfg1_inputs(n_fact=1_000_000, dim_rows=10_000, k=16, l=1, seed=42):
    """cfg1: fk = Rng(derive_seed(42,"lineorder")).range(0, dim_rows) x n_fact;
    pk = iota(dim_rows); k unit() feature columns drawn column by column from
    derive_seed(42,"dim"); W = gen_linear(k, l, 7)."""
    fk = rng_range(seed, "lineorder", n_fact, 0, dim_rows)
    pk = np.arange(dim_rows, dtype=np.int64)
    feats = unit_matrix(seed, "dim", dim_rows, k)
    W = gen_linear(k, l, 7)
    return fk, pk, feats, W
