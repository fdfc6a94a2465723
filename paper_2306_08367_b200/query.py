"""Query descriptions (mirror of laq::bench::QuerySpec, benchgen.hpp:296-326) and
the SSB-style workload definitions (benchgen.cpp:207-362).

The workload definitions are restated here so the engine can tune the dial
constants on the device (measure_selectivity, benchgen.cpp:366-411) instead of
the reference's ~10 full CPU scans per query; gen_queries below follows
benchgen.cpp:413-457 step for step, so the constants it picks are identical.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi

LT, LE, EQ, GE, GT, BETWEEN, INSET = range(7)  # predicate.hpp:15-28 / laq_pred_kind


@dataclass(frozen=True)
class Pred:
    """Integer Predicate (predicate.hpp:15-103). Between is inclusive."""
    kind: int
    lo: int = 0
    hi: int = 0
    values: tuple = ()
    is_float: bool = False

    @staticmethod
    def lt(v): return Pred(LT, int(v))
    @staticmethod
    def le(v): return Pred(LE, int(v))
    @staticmethod
    def eq(v): return Pred(EQ, int(v))
    @staticmethod
    def ge(v): return Pred(GE, int(v))
    @staticmethod
    def gt(v): return Pred(GT, int(v))
    @staticmethod
    def between(lo, hi): return Pred(BETWEEN, int(lo), int(hi))
    @staticmethod
    def in_set(vals): return Pred(INSET, values=tuple(sorted(int(v) for v in vals)))

    @staticmethod
    def flt(kind, lo=0.0, hi=0.0, values=()):
        """A float-typed Predicate (predicate.hpp:25-33): matches float columns only."""
        return Pred(kind, float(lo), float(hi), tuple(sorted(float(v) for v in values)), True)

    def matches(self, v: np.ndarray) -> np.ndarray:
        k = self.kind
        if k == LT: return v < self.lo
        if k == LE: return v <= self.lo
        if k == EQ: return v == self.lo
        if k == GE: return v >= self.lo
        if k == GT: return v > self.lo
        if k == BETWEEN: return (v >= self.lo) & (v <= self.hi)
        return np.isin(v, np.asarray(self.values, dtype=np.int64))


@dataclass(frozen=True)
class StarLink:
    """storage.hpp:75-81."""
    fact_fk: str
    dim_name: str
    dim_pk: str


@dataclass(frozen=True)
class FilterSpec:
    """benchgen.hpp:302-309; target -1 = fact, else index into joins."""
    target: int
    column: str
    pred: Pred


@dataclass(frozen=True)
class GroupRef:
    """benchgen.hpp:311-314."""
    target: int
    column: str


@dataclass
class QuerySpec:
    """benchgen.hpp:316-326."""
    id: str
    group: int
    joins: list
    filters: list
    measure: str = "lo_revenue"
    group_by: list = field(default_factory=list)
    order_by: bool = False
    target_selectivity: float = 0.0
    realized_selectivity: float = 0.0


class QueryDescHolder:
    """Builds the C struct laq_query_desc (include/laq_b200.h) and keeps every
    buffer it points to alive."""

    def __init__(self, q: QuerySpec):
        self._keep = []
        joins = (_abi.LinkDesc * max(1, len(q.joins)))()
        for i, l in enumerate(q.joins):
            joins[i] = _abi.LinkDesc(l.fact_fk.encode(), l.dim_name.encode(), l.dim_pk.encode())
        filts = (_abi.FilterDesc * max(1, len(q.filters)))()
        for i, f in enumerate(q.filters):
            p = f.pred
            sv = np.ascontiguousarray(np.asarray(p.values, dtype=np.int64))
            self._keep.append(sv)
            filts[i] = _abi.FilterDesc(f.target, f.column.encode(), p.kind, 1 if p.is_float else 0, p.lo, p.hi,
                                       sv.ctypes.data_as(_abi.i64p) if len(sv) else _abi.i64p(), len(sv))
        groups = (_abi.GroupDesc * max(1, len(q.group_by)))()
        for i, g in enumerate(q.group_by):
            groups[i] = _abi.GroupDesc(g.target, g.column.encode())
        self._keep += [joins, filts, groups]
        self.desc = _abi.QueryDesc(len(q.joins), joins, len(q.filters), filts, q.measure.encode(),
                                   len(q.group_by), groups, 1 if q.order_by else 0)


def build_query_desc_links(q: QuerySpec):  # convenience for tests
    return QueryDescHolder(q)


# ---------------------------------------------------------------------------
# SSB-style workload (benchgen.cpp:207-362)
# ---------------------------------------------------------------------------

PART = StarLink("lo_part", "part", "p_key")
SUPPLIER = StarLink("lo_supplier", "supplier", "s_key")
ORDERDATE = StarLink("lo_orderdate", "date", "d_key")
COMMITDATE = StarLink("lo_commitdate", "date", "d_key")

K_DAY_RANGE, K_SIZE_RANGE, K_RANK_RANGE = 365, 1000, 1000  # benchgen.cpp:17-25


@dataclass(frozen=True)
class QueryDef:
    """benchgen.cpp:214-223."""
    id: str
    joins: tuple
    fixed: tuple
    dial_target: int
    dial_column: str
    dial_range: int
    group_by: tuple
    order_by: bool


def group_defs(group: int) -> list:
    """benchgen.cpp:225-339."""
    if group == 1:
        return [
            QueryDef("11", (ORDERDATE,), (FilterSpec(-1, "lo_discount", Pred.between(1, 3)),
                                          FilterSpec(-1, "lo_quantity", Pred.lt(25))),
                     0, "d_dayofyear", K_DAY_RANGE, (), False),
            QueryDef("12", (ORDERDATE,), (FilterSpec(-1, "lo_discount", Pred.between(4, 6)),
                                          FilterSpec(-1, "lo_quantity", Pred.between(26, 35))),
                     0, "d_dayofyear", K_DAY_RANGE, (), False),
            QueryDef("13", (ORDERDATE,), (FilterSpec(-1, "lo_discount", Pred.between(5, 7)),
                                          FilterSpec(-1, "lo_quantity", Pred.between(36, 40))),
                     0, "d_dayofyear", K_DAY_RANGE, (), False),
        ]
    three = (PART, SUPPLIER, ORDERDATE)
    if group == 2:
        gb = (GroupRef(2, "d_year"), GroupRef(0, "p_brand"))
        return [
            QueryDef("21", three, (FilterSpec(1, "s_region", Pred.eq(0)),), 0, "p_size", K_SIZE_RANGE, gb, True),
            QueryDef("22", three, (FilterSpec(1, "s_region", Pred.eq(1)),), 0, "p_size", K_SIZE_RANGE, gb, True),
            QueryDef("23", three, (FilterSpec(1, "s_region", Pred.eq(2)), FilterSpec(2, "d_year", Pred.eq(1994))),
                     0, "p_size", K_SIZE_RANGE, gb, True),
        ]
    if group == 3:
        gb = (GroupRef(1, "s_nation"), GroupRef(2, "d_year"))
        return [
            QueryDef("31", three, (FilterSpec(2, "d_year", Pred.between(1992, 1997)),), 1, "s_rank", K_RANK_RANGE,
                     gb, True),
            QueryDef("32", three, (FilterSpec(2, "d_year", Pred.between(1994, 1996)),), 1, "s_rank", K_RANK_RANGE,
                     gb, True),
            QueryDef("33", three, (FilterSpec(2, "d_year", Pred.in_set([1992, 1997])),), 1, "s_rank", K_RANK_RANGE,
                     gb, True),
        ]
    if group == 4:
        four = (PART, SUPPLIER, ORDERDATE, COMMITDATE)
        gb = (GroupRef(2, "d_year"), GroupRef(1, "s_nation"))
        return [
            QueryDef("41", four, (FilterSpec(1, "s_region", Pred.eq(0)),), 0, "p_size", K_SIZE_RANGE, gb, True),
            QueryDef("42", four, (FilterSpec(1, "s_region", Pred.eq(1)), FilterSpec(2, "d_month", Pred.between(1, 6))),
                     0, "p_size", K_SIZE_RANGE, gb, True),
            QueryDef("43", four, (FilterSpec(1, "s_region", Pred.eq(2)), FilterSpec(3, "d_year", Pred.eq(1995))),
                     0, "p_size", K_SIZE_RANGE, gb, True),
        ]
    from .errors import GenError
    raise GenError("unknown query group")


DEFAULT_TARGETS = {1: (0.08, 0.03, 0.01), 2: (0.10, 0.04, 0.015), 3: (0.09, 0.033, 0.0125),
                   4: (0.05, 0.02, 0.008)}  # benchgen.cpp:341-349


def spec_with_dial(d: QueryDef, group: int, dial: int) -> QuerySpec:
    """benchgen.cpp:351-362."""
    return QuerySpec(id=d.id, group=group, joins=list(d.joins),
                     filters=list(d.fixed) + [FilterSpec(d.dial_target, d.dial_column, Pred.lt(dial))],
                     measure="lo_revenue", group_by=list(d.group_by), order_by=d.order_by)


def gen_queries(measure, group: int, targets: Sequence[float] = ()) -> list:
    """gen_queries (benchgen.cpp:413-457) with a caller-supplied
    measure_selectivity(QuerySpec) -> float (the device one in production)."""
    from .errors import GenError
    defs = group_defs(group)
    tg = list(DEFAULT_TARGETS[group])
    for i, t in enumerate(targets[: len(tg)]):
        tg[i] = t
    out = []
    for d, target in zip(defs, tg):
        if target <= 0.0 or target >= 1.0:
            raise GenError("selectivity target must be in (0,1)")
        lo, hi = 0, d.dial_range
        while lo < hi:
            mid = lo + (hi - lo) // 2
            if measure(spec_with_dial(d, group, mid)) < target:
                lo = mid + 1
            else:
                hi = mid
        best_sel = measure(spec_with_dial(d, group, lo))
        best = lo
        if lo > 0:
            below = measure(spec_with_dial(d, group, lo - 1))
            if abs(below - target) < abs(best_sel - target):
                best, best_sel = lo - 1, below
        if abs(best_sel - target) > 0.2 * target:
            raise GenError(f"query {d.id}: cannot reach selectivity {target} (closest {best_sel})")
        q = spec_with_dial(d, group, best)
        q.target_selectivity = target
        q.realized_selectivity = best_sel
        out.append(q)
    return out
