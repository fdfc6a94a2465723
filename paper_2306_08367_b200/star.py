"""A StarSchema resident in HBM and the query plan driver on it.

  DeviceStar.run_query(q)          run_query_laq          cli.cpp:73-138
  DeviceStar.measure_selectivity   measure_selectivity    benchgen.cpp:366-411
  DeviceStar.gen_queries(group)    gen_queries            benchgen.cpp:413-457 (device-tuned dials)
  DeviceStar.prepare(q) -> Plan    prepared form: execute() enqueues the fused
                                   scan into an int64 accumulator (no host sync,
                                   CUDA-graph capturable, all-reduce friendly);
                                   emit() turns the accumulator into result rows.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi, errors, query
from .device import context


class Plan:
    def __init__(self, star: "DeviceStar", q: query.QuerySpec):
        self.star = star
        self.q = q
        self.ctx = star.ctx
        self._holder = query.QueryDescHolder(q)
        h = C.c_void_p()
        g = C.c_int64()
        self.ctx.check(self.ctx.lib.laq_query_prepare(self.ctx.h, star.h, C.byref(self._holder.desc), C.byref(h),
                                                      C.byref(g)))
        self.h = h
        self.n_groups = g.value
        self.acc = torch.zeros(2 * self.n_groups, dtype=torch.int64, device="cuda")

    def execute(self, acc: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
        acc = self.acc if acc is None else acc
        self.ctx.bind_stream()
        self.ctx.check(self.ctx.lib.laq_plan_execute(self.ctx.h, self.h, acc.data_ptr(), 1 if accumulate else 0))
        return acc

    def build_codes(self):
        self.ctx.check(self.ctx.lib.laq_plan_build_codes(self.ctx.h, self.h))

    def scan(self, acc: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
        acc = self.acc if acc is None else acc
        self.ctx.check(self.ctx.lib.laq_plan_scan(self.ctx.h, self.h, acc.data_ptr(), 1 if accumulate else 0))
        return acc

    def scan_range(self, row0: int, rows: int, acc: torch.Tensor | None = None, accumulate: bool = False):
        """Scan fact rows [row0, row0 + rows) with the current code tables."""
        acc = self.acc if acc is None else acc
        self.ctx.check(self.ctx.lib.laq_plan_scan_range(self.ctx.h, self.h, row0, rows, acc.data_ptr(),
                                                        1 if accumulate else 0))
        return acc

    @property
    def bytes_per_row(self) -> int:
        return int(self.ctx.lib.laq_plan_bytes_per_row(self.h))

    @property
    def scanned_links(self) -> int:
        return int(self.ctx.lib.laq_plan_scanned_links(self.h))

    def emit(self, acc_host: np.ndarray) -> np.ndarray:
        acc_host = np.ascontiguousarray(acc_host, np.int64)
        cap = max(1, 2 * self.n_groups) * (len(self.q.group_by) + 1)
        out = np.zeros(cap, np.float64)
        rows, cols = C.c_int64(), C.c_int64()
        rc = self.ctx.lib.laq_plan_emit(self.h, acc_host.ctypes.data_as(_abi.i64p),
                                        out.ctypes.data_as(_abi.f64p), cap, C.byref(rows), C.byref(cols))
        errors.raise_for(rc, "laq_plan_emit failed")
        return out[: rows.value * cols.value].reshape(rows.value, cols.value).copy()

    def run(self) -> np.ndarray:
        acc = self.execute()
        return self.emit(acc.cpu().numpy())

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.laq_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceStar:
    """laq_star: tables uploaded once (int32 device layout), probes cached per link."""

    def __init__(self, ctx=None):
        self.ctx = ctx or context()
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.laq_star_create(self.ctx.h, C.byref(h)))
        self.h = h
        self._keep = []
        self.rows = {}

    @classmethod
    def from_tables(cls, tables: dict, kinds: dict, links, fact="lineorder", row_range=None, ctx=None):
        """tables: {name: {col: np.ndarray}} (int64/int32 ints, float64 floats);
        kinds: {name: {col: 0 key | 1 int | 2 float}}; row_range=(b, e) uploads
        only that slice of the fact table (row sharding)."""
        s = cls(ctx)
        order = [fact] + [t for t in tables if t != fact]
        for name in order:
            cols = tables[name]
            if name == fact and row_range is not None:
                b, e = row_range
                cols = {c: a[b:e] for c, a in cols.items()}
            s.add_table(name, cols, kinds[name], is_fact=(name == fact))
        for l in links:
            s.add_link(*l)
        return s

    def add_table(self, name, cols: dict, kinds: dict, is_fact=False):
        names = list(cols)
        rows = len(cols[names[0]]) if names else 0
        width = 8
        arrays = []
        for c in names:
            a = cols[c]
            if kinds[c] == 2:
                a = np.ascontiguousarray(a, np.float64)
            elif a.dtype == np.int32:
                width = 4
            arrays.append(a)
        conv = []
        for c, a in zip(names, arrays):
            if kinds[c] != 2:
                a = np.ascontiguousarray(a, np.int32 if width == 4 else np.int64)
            conv.append(a)
        self._keep.append(conv)
        cn = (C.c_char_p * len(names))(*[c.encode() for c in names])
        kd = (C.c_int32 * len(names))(*[kinds[c] for c in names])
        ptrs = (C.c_void_p * len(names))(*[a.ctypes.data for a in conv])
        self.ctx.check(self.ctx.lib.laq_star_add_table(self.star_h, name.encode(), 1 if is_fact else 0, rows,
                                                       len(names), cn, kd, width, ptrs))
        self._keep.pop()  # host columns were copied to the device
        self.rows[name] = rows

    def add_table_device64(self, name, cols: dict, kinds: dict, is_fact=False):
        """int64 (key/int) / float64 CUDA tensors as the device CSV loader
        produces them; integer columns are narrowed to int32 on the device
        (range-checked), float columns are not kept (no float device path)."""
        names = list(cols)
        rows = cols[names[0]].numel() if names else 0
        cn = (C.c_char_p * len(names))(*[c.encode() for c in names])
        kd = (C.c_int32 * len(names))(*[kinds[c] for c in names])
        ptrs = (C.c_void_p * len(names))(*[cols[c].data_ptr() for c in names])
        self.ctx.check(self.ctx.lib.laq_star_add_table(self.star_h, name.encode(), 1 if is_fact else 0, rows,
                                                       len(names), cn, kd, 8, ptrs))
        self.rows[name] = rows

    def add_table_device(self, name, cols: dict, kinds: dict, is_fact=False):
        """int32 CUDA tensors, used in place (caller keeps them alive)."""
        names = list(cols)
        rows = cols[names[0]].numel()
        self._keep.append(cols)
        cn = (C.c_char_p * len(names))(*[c.encode() for c in names])
        kd = (C.c_int32 * len(names))(*[kinds[c] for c in names])
        ptrs = _abi.ptr_array([cols[c].data_ptr() for c in names])
        self.ctx.check(self.ctx.lib.laq_star_add_table_device(self.star_h, name.encode(), 1 if is_fact else 0, rows,
                                                              len(names), cn, kd, ptrs))
        self.rows[name] = rows

    def add_table_device_packed(self, name, cols: dict, kinds: dict, is_fact=False):
        """Byte-packed CUDA tensors {column: (tensor, width, offset)} used in place
        (value = stored + offset; uint8 / int16-bits / int32 storage, see
        pack_columns).  Each tensor needs >= 16 bytes of padding past the rows."""
        names = list(cols)
        rows = self._packed_rows(cols)
        self._keep.append(cols)
        cn = (C.c_char_p * len(names))(*[c.encode() for c in names])
        kd = (C.c_int32 * len(names))(*[kinds[c] for c in names])
        ptrs = _abi.ptr_array([cols[c][0].data_ptr() for c in names])
        w = (C.c_int32 * len(names))(*[int(cols[c][1]) for c in names])
        off = (C.c_int32 * len(names))(*[int(cols[c][2]) for c in names])
        self.ctx.check(self.ctx.lib.laq_star_add_table_device_packed(
            self.star_h, name.encode(), 1 if is_fact else 0, rows, len(names), cn, kd, ptrs, w, off))
        self.rows[name] = rows

    def add_table_device_bitpacked(self, name, cols: dict, kinds: dict, rows: int, is_fact=False):
        """Bit-packed CUDA tensors {column: (uint32 tensor, bits, offset)} used in
        place (the bit-packed transfer format, see bitpack_columns)."""
        names = list(cols)
        self._keep.append(cols)
        cn = (C.c_char_p * len(names))(*[c.encode() for c in names])
        kd = (C.c_int32 * len(names))(*[kinds[c] for c in names])
        ptrs = _abi.ptr_array([cols[c][0].data_ptr() for c in names])
        b = (C.c_int32 * len(names))(*[int(cols[c][1]) for c in names])
        off = (C.c_int32 * len(names))(*[int(cols[c][2]) for c in names])
        self.ctx.check(self.ctx.lib.laq_star_add_table_device_bitpacked(
            self.star_h, name.encode(), 1 if is_fact else 0, rows, len(names), cn, kd, ptrs, b, off))
        self.rows[name] = rows

    @staticmethod
    def _packed_rows(cols):
        t, w, _ = next(iter(cols.values()))[:3]
        return (t.numel() * t.element_size() - 16) // int(w)

    @property
    def star_h(self):
        return self.h

    def add_link(self, fact_fk, dim_name, dim_pk):
        self.ctx.check(self.ctx.lib.laq_star_add_link(self.h, fact_fk.encode(), dim_name.encode(), dim_pk.encode()))

    def prepare(self, q: query.QuerySpec) -> Plan:
        return Plan(self, q)

    def run_query(self, q: query.QuerySpec) -> np.ndarray:
        holder = query.QueryDescHolder(q)
        cap = 1 << 20
        out = np.zeros(cap, np.float64)
        rows, cols = C.c_int64(), C.c_int64()
        rc = self.ctx.lib.laq_run_query(self.ctx.h, self.h, C.byref(holder.desc), out.ctypes.data_as(_abi.f64p),
                                        cap, C.byref(rows), C.byref(cols))
        self.ctx.check(rc)
        return out[: rows.value * cols.value].reshape(rows.value, cols.value).copy()

    def measure_selectivity(self, q: query.QuerySpec) -> float:
        holder = query.QueryDescHolder(q)
        out = C.c_double()
        self.ctx.check(self.ctx.lib.laq_measure_selectivity(self.ctx.h, self.h, C.byref(holder.desc), C.byref(out)))
        return out.value

    def gen_queries(self, group: int, targets=()):
        return query.gen_queries(self.measure_selectivity, group, targets)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.laq_star_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_codes_batch(plans) -> None:
    """Code tables of several plans (one step of queries) in one launch
    (laq_plans_build_codes)."""
    if not plans:
        return
    ctx = plans[0].ctx
    arr = (C.c_void_p * len(plans))(*[p.h.value if hasattr(p.h, "value") else p.h for p in plans])
    ctx.check(ctx.lib.laq_plans_build_codes(ctx.h, len(plans), arr))


def scan_shared(plans, accs, accumulate=False) -> bool:
    """One pass over the fact table for a batch of 2-3 plans reading the same
    columns (laq_plans_scan_shared); returns whether the batch was shared."""
    ctx = plans[0].ctx
    hp = (C.c_void_p * len(plans))(*[p.h.value for p in plans])
    ha = (C.c_void_p * len(plans))(*[a.data_ptr() for a in accs])
    shared = C.c_int32()
    ctx.check(ctx.lib.laq_plans_scan_shared(ctx.h, len(plans), hp, ha, 1 if accumulate else 0, C.byref(shared)))
    return bool(shared.value)


class Batch:
    """A batch of 1..4 plans over the same fact table scanned in ONE pass with
    one probe per link for the whole batch (laq_batch_*, csrc/ssb_batch.cuh).
    build() = every plan's code tables + the link dictionaries; scan(accs)
    fills each plan's own accumulator, exactly as plan.scan would.  Batches the
    fused pass cannot take are scanned plan by plan (`fused` False, `why`)."""

    def __init__(self, plans):
        self.plans = list(plans)
        self.ctx = self.plans[0].ctx
        hp = (C.c_void_p * len(self.plans))(*[p.h.value for p in self.plans])
        h = C.c_void_p()
        fused = C.c_int32()
        self.ctx.check(self.ctx.lib.laq_batch_prepare(self.ctx.h, len(self.plans), hp, C.byref(h), C.byref(fused)))
        self.h = h
        f, bpr, nl = C.c_int32(), C.c_int64(), C.c_int32()
        why = C.create_string_buffer(256)
        self.ctx.lib.laq_batch_info(self.h, C.byref(f), C.byref(bpr), C.byref(nl), why, 256)
        self.fused = bool(f.value)
        self.bytes_per_row = int(bpr.value)
        self.n_links = int(nl.value)
        self.why = why.value.decode()

    def build(self):
        self.ctx.check(self.ctx.lib.laq_batch_build(self.ctx.h, self.h))

    def scan(self, accs=None, accumulate=False):
        accs = [p.acc for p in self.plans] if accs is None else list(accs)
        ha = (C.c_void_p * len(accs))(*[a.data_ptr() for a in accs])
        self.ctx.check(self.ctx.lib.laq_batch_scan(self.ctx.h, self.h, ha, 1 if accumulate else 0))
        return accs

    def run(self):
        """Build + scan + emit every plan's result rows."""
        self.ctx.bind_stream()
        self.build()
        accs = self.scan()
        return [p.emit(a.cpu().numpy()) for p, a in zip(self.plans, accs)]

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.laq_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def upload_gen_star(g, ctx=None, row_range=None) -> DeviceStar:
    """Upload a gen.GenStar (or oracle RefStar-like object with .tables/.kinds/.links())."""
    links = g.links() if callable(getattr(g, "links", None)) else g.links
    return DeviceStar.from_tables(g.tables, g.kinds, links, row_range=row_range, ctx=ctx)


def pack_columns(cols: dict) -> dict:
    """Host-side compact transfer format for integer columns: value - min stored
    as uint8 when the range fits 8 bits, uint16 when it fits 16, else int32
    (offset 0); each array carries 16 bytes of zero padding.  Returns
    {column: (numpy array, width, offset)}."""
    out = {}
    for c, a in cols.items():
        a = np.asarray(a)
        if a.dtype.kind == "f":
            continue
        mn, mx = (int(a.min()), int(a.max())) if a.size else (0, 0)
        rng = mx - mn
        if rng < 256:
            w, dt, off = 1, np.uint8, mn
        elif rng < 65536:
            w, dt, off = 2, np.uint16, mn
        else:
            w, dt, off = 4, np.int32, 0
        buf = np.zeros(a.size * w + 16, np.uint8)
        buf[: a.size * w].view(dt)[:] = (a.astype(np.int64) - off).astype(dt)
        out[c] = (buf, w, off)
    return out


def bitpack_words(v: np.ndarray, bits: int) -> np.ndarray:
    """Little-endian bitstream of `bits` bits per value (v >= 0, < 2^bits):
    value i occupies bits [i*bits, (i+1)*bits), so a group of 32 values is
    `bits` consecutive uint32 words.  Sized to whole 128-row blocks + 16 bytes
    (the laq_star_add_table_device_bitpacked contract).  The fields are
    disjoint, so OR == ADD and two weighted bincounts build every word exactly
    (each word's sum < 2^32 is exact in float64)."""
    n = v.size
    nwords = -(-n // 128) * 4 * bits + 4
    if n == 0:
        return np.zeros(nwords, np.uint32)
    v = v.astype(np.uint64)
    s = np.arange(n, dtype=np.uint64) * np.uint64(bits)
    w0 = (s >> np.uint64(5)).astype(np.int64)
    sh = s & np.uint64(31)
    lo = (v << sh) & np.uint64(0xFFFFFFFF)
    hi = v >> (np.uint64(32) - sh)  # sh == 0: v >> 32 == 0 for v < 2^32
    words = np.bincount(w0, weights=lo.astype(np.float64), minlength=nwords)
    words += np.bincount(w0 + 1, weights=hi.astype(np.float64), minlength=nwords)[:nwords]
    return words[:nwords].astype(np.uint64).astype(np.uint32)


def bitunpack_words(words: np.ndarray, n: int, bits: int) -> np.ndarray:
    """Inverse of bitpack_words (host check for tests)."""
    w = np.concatenate([words.astype(np.uint64), np.zeros(2, np.uint64)])
    s = np.arange(n, dtype=np.uint64) * np.uint64(bits)
    i = (s >> np.uint64(5)).astype(np.int64)
    sh = s & np.uint64(31)
    both = w[i] | (w[i + 1] << np.uint64(32))
    return ((both >> sh) & np.uint64((1 << bits) - 1)).astype(np.int64)


def bitpack_columns(cols: dict) -> dict:
    """Host-side bit-packed transfer format for integer columns: value - min in
    the fewest bits its range needs (SF=10 lineorder scan columns: 71 bits per
    row instead of 96 in the byte-packed format).  Returns
    {column: (uint32 words, bits, offset)}."""
    out = {}
    for c, a in cols.items():
        a = np.asarray(a)
        if a.dtype.kind == "f":
            continue
        mn, mx = (int(a.min()), int(a.max())) if a.size else (0, 0)
        bits = max(1, (mx - mn).bit_length())
        if bits > 32:
            raise ValueError(f"column {c}: range needs {bits} bits")
        out[c] = (bitpack_words(a.astype(np.int64) - mn, bits), bits, mn)
    return out
