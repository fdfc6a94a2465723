"""TEST INFRASTRUCTURE ONLY -- the full-size query checker (never the product).

run_query(tables, q) has the contract of laq_oracle.run_query (the numpy
restatement of run_query_laq, cli.cpp:73-138) and computes the same result the
way the reference's scalar oracle does (run_query_oracle, cli.cpp:140-225:
scalar filters, hash star join over unique dimension keys, SUM(measure) per
group, groups ascending), with the fact-row loop in multi-threaded C
(oracle/ssb_oracle.c -> oracle/_bin/libssb_oracle.so).  It is what lets the
SF=100 configuration (600M lineorder rows) be checked in seconds.

partial(...) returns the raw per-group (count, sum) arrays of a row range so
row shards checked on different ranks can be merged exactly (int64 sums).
Queries outside its fast form (fact-side group columns, float measures or
fact predicates, InSet fact filters, duplicate / very sparse dimension keys)
fall back to laq_oracle.run_query.

Pinned against the reference's goldens in tests/test_oracle_fast.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import laq_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_bin", "libssb_oracle.so")
_lib = None


class _Col(C.Structure):
    _fields_ = [("p", C.c_void_p), ("width", C.c_int32)]


def build():
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    src = os.path.join(HERE, "ssb_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread", src, "-o", LIB_PATH],
                       check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.oc_star_query.restype = C.c_int
        _lib = L
    return _lib


class Unsupported(Exception):
    pass


def _col(a):
    a = np.asarray(a)
    if a.dtype == np.int32:
        return _Col(a.ctypes.data, 4), a
    if a.dtype == np.int64:
        return _Col(a.ctypes.data, 8), a
    raise Unsupported(f"column dtype {a.dtype}")


def _interval(p):
    from paper_2306_08367_b200.query import BETWEEN, EQ, GE, GT, LE, LT
    big = np.iinfo(np.int64)
    if p.is_float:
        raise Unsupported("float fact predicate")
    k = p.kind
    if k == LT: return big.min, p.lo - 1
    if k == LE: return big.min, p.lo
    if k == EQ: return p.lo, p.lo
    if k == GE: return p.lo, big.max
    if k == GT: return p.lo + 1, big.max
    if k == BETWEEN: return p.lo, p.hi
    raise Unsupported("InSet fact predicate")


class Prepared:
    """The dimension side of one query (hash tables composed with the dim
    filters and group columns); reusable across row ranges."""

    def __init__(self, tables, q):
        fact = tables["lineorder"]
        self.q = q
        self.fact = fact
        if any(g.target == -1 for g in q.group_by):
            raise Unsupported("fact-side group column")
        m = np.asarray(fact[q.measure])
        if m.dtype.kind != "i":
            raise Unsupported("float measure")
        # group columns: sorted distinct values -> mixed radix, first column most significant
        self.distinct = []
        for g in q.group_by:
            col = np.asarray(tables[q.joins[g.target].dim_name][g.column])
            if col.dtype.kind != "i":
                raise Unsupported("float group column")
            self.distinct.append(np.unique(col.astype(np.int64)))
        self.stride = [1] * len(self.distinct)
        s = 1
        for i in range(len(self.distinct) - 1, -1, -1):
            self.stride[i] = s
            s *= max(1, len(self.distinct[i]))
        self.G = max(1, s)
        if self.G > 1 << 26:
            raise Unsupported("group space")
        self.base, self.span, self.tabs = [], [], []
        for j, l in enumerate(q.joins):
            dim = tables[l.dim_name]
            pk = np.asarray(dim[l.dim_pk], np.int64)
            n = len(pk)
            lo = int(pk.min()) if n else 0
            span = (int(pk.max()) - lo + 1) if n else 1
            if span > 4 * n + (1 << 22):
                raise Unsupported("sparse dimension keys")
            keep = np.ones(n, bool)
            for f in q.filters:
                if f.target == j:
                    keep &= O._pred(f.pred, np.asarray(dim[f.column]))
            code = np.zeros(n, np.int64)
            for gi, g in enumerate(q.group_by):
                if g.target == j:
                    v = np.asarray(dim[g.column], np.int64)
                    code += np.searchsorted(self.distinct[gi], v) * self.stride[gi]
            tab = np.full(span, -1, np.int64)
            slot = pk - lo
            if n and len(np.unique(slot)) != n:
                raise Unsupported("duplicate dimension keys")
            tab[slot[keep]] = code[keep]
            self.base.append(lo)
            self.span.append(span)
            self.tabs.append(tab)
        self.ff = [(f.column, *_interval(f.pred)) for f in q.filters if f.target == -1]

    def partial(self, row0=0, rows=None, threads=None):
        """int64 (count, sum) per group code over fact rows [row0, row0 + rows)."""
        q, fact = self.q, self.fact
        n_all = len(np.asarray(fact[q.measure]))
        rows = n_all - row0 if rows is None else rows
        threads = threads or min(64, os.cpu_count() or 1)
        keep = []
        fk = (_Col * max(1, len(q.joins)))()
        for j, l in enumerate(q.joins):
            fk[j], a = _col(fact[l.fact_fk])
            keep.append(a)
        ff = (_Col * max(1, len(self.ff)))()
        lo = np.array([x[1] for x in self.ff] or [0], np.int64)
        hi = np.array([x[2] for x in self.ff] or [0], np.int64)
        for i, (c, _, _) in enumerate(self.ff):
            ff[i], a = _col(fact[c])
            keep.append(a)
        meas, a = _col(fact[q.measure])
        keep.append(a)
        base = np.array(self.base or [0], np.int64)
        span = np.array(self.span or [1], np.int64)
        tabs = (C.c_void_p * max(1, len(self.tabs)))(*[t.ctypes.data for t in self.tabs])
        cnt = np.zeros(self.G, np.int64)
        s = np.zeros(self.G, np.int64)
        rc = lib().oc_star_query(C.c_int64(row0), C.c_int64(rows), C.c_int32(len(q.joins)), fk,
                                 base.ctypes.data_as(C.c_void_p), span.ctypes.data_as(C.c_void_p), tabs,
                                 C.c_int32(len(self.ff)), ff, lo.ctypes.data_as(C.c_void_p),
                                 hi.ctypes.data_as(C.c_void_p), C.byref(meas), C.c_int64(self.G),
                                 cnt.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p), C.c_int32(threads))
        if rc != 0:
            raise RuntimeError("oc_star_query failed")
        return cnt, s

    def emit(self, cnt, s) -> np.ndarray:
        """DenseMat [group cols..., sum]: present groups ascending (cli.cpp:124-136);
        1x1 plain sum without group-by."""
        if not self.q.group_by:
            return np.array([[float(s[0])]])
        present = np.nonzero(cnt > 0)[0]
        out = np.zeros((len(present), len(self.distinct) + 1))
        for i, d in enumerate(self.distinct):
            out[:, i] = d[(present // self.stride[i]) % len(d)]
        out[:, -1] = s[present].astype(np.float64)
        return out


def run_query(tables, q, row_range=None, threads=None) -> np.ndarray:
    """laq_oracle.run_query over fact rows [lo, hi) (default all)."""
    try:
        p = Prepared(tables, q)
    except Unsupported:
        if row_range is not None:
            lo, hi = row_range
            t = dict(tables)
            t["lineorder"] = {c: a[lo:hi] for c, a in tables["lineorder"].items()}
            return O.run_query(t, q)
        return O.run_query(tables, q)
    lo, hi = row_range if row_range is not None else (0, None)
    cnt, s = p.partial(lo, None if hi is None else hi - lo, threads)
    return p.emit(cnt, s)
