"""Ingest: the reference's on-disk dataset (CSV tables + manifest.json) loaded
into HBM, parsed on the device.

Mirrors the reference's host API:
  * ``load_csv(path, schema)``      -- storage.cpp:112-150 (laq::load_csv);
  * ``load_dataset(dir)``           -- cli.cpp:483-513 (laq::cli::load_dataset);
  * ``schema_from_json`` / kinds    -- cli.cpp:397-410, storage.cpp:9-23.

The file bytes are read on the host (I/O) and copied to the device once; line
indexing and number parsing run in csv.cu (``laq_csv_open`` /
``laq_csv_parse``), with the reference's parse semantics and error messages.

Binary columnar cache: after the first parse each table's
columns are written next to the CSV as raw little-endian arrays
(``.laq_cache/<table>/<column>.bin``, int64 / float64, plus a ``meta.json``
keyed on the CSV's size and mtime); later loads copy those bytes straight to
the device and skip the text entirely.  The cache is a pure performance
device: results are identical either way (tests/test_gpu_ingest.py).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np
import torch

from . import errors
from .device import context

KIND_BY_NAME = {"key": 0, "int": 1, "float": 2}  # storage.hpp:14 / storage.cpp:18-23
NAME_BY_KIND = {v: k for k, v in KIND_BY_NAME.items()}


def col_kind_from_name(name: str) -> int:
    """storage.cpp:18-23 (FormatError on an unknown kind)."""
    if name not in KIND_BY_NAME:
        raise errors.FormatError(f"unknown column kind: {name}")
    return KIND_BY_NAME[name]


def schema_from_json(j) -> list:
    """cli.cpp:404-410: [[name, kind], ...] -> [(name, kind code)]."""
    return [(c[0], col_kind_from_name(c[1])) for c in j]


def _validate(schema):
    """Schema::validate (storage.hpp:19-33): non-empty, unique names."""
    if not schema:
        raise errors.FormatError("schema has no columns")
    seen = set()
    for n, _ in schema:
        if n in seen:
            raise errors.FormatError(f"duplicate column name: {n}")
        seen.add(n)


def _parse_pinned(host: torch.Tensor, n: int, schema, ctx) -> dict:
    """host: pinned uint8 tensor holding n text bytes + 16 zero bytes."""
    _validate(schema)
    dev = host.to(f"cuda:{ctx.device}", non_blocking=True)
    ctx.bind_stream()
    h = C.c_void_p()
    lines = C.c_int64()
    ctx.check(ctx.lib.laq_csv_open(ctx.h, dev.data_ptr(), n, C.byref(h), C.byref(lines)))
    try:
        rows = lines.value
        cols = {}
        for name, kind in schema:
            dt = torch.float64 if kind == 2 else torch.int64
            cols[name] = torch.empty(max(rows, 1), dtype=dt, device=dev.device)
        kinds = (C.c_int32 * len(schema))(*[k for _, k in schema])
        ptrs = (C.c_void_p * len(schema))(*[cols[nm].data_ptr() for nm, _ in schema])
        ctx.check(ctx.lib.laq_csv_parse(ctx.h, h, len(schema), kinds, ptrs))
        torch.cuda.current_stream(ctx.device).synchronize()
        return {k: v[:rows] for k, v in cols.items()}
    finally:
        ctx.lib.laq_csv_close(h)


def parse_csv_bytes(data: bytes, schema, ctx=None) -> dict:
    """Parse CSV text (host bytes) on the device -> {column: CUDA tensor}
    (int64 for key/int columns, float64 for float columns)."""
    ctx = ctx or context()
    n = len(data)
    # 16 bytes of zero padding: the line indexer reads 16-byte vectors.
    host = torch.zeros(n + 16, dtype=torch.uint8, pin_memory=True)
    if n:
        host[:n] = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    return _parse_pinned(host, n, schema, ctx)


def load_csv(path, schema, ctx=None) -> dict:
    """laq::load_csv (storage.cpp:112-150): FormatError 'cannot open <path>'.
    The file is read straight into pinned memory (one host copy), then parsed
    on the device."""
    ctx = ctx or context()
    try:
        n = os.path.getsize(path)
        host = torch.empty(n + 16, dtype=torch.uint8, pin_memory=True)
        host[n:] = 0
        with open(path, "rb") as f:
            got = f.readinto(memoryview(host.numpy())[:n]) if n else 0
    except OSError:
        raise errors.FormatError(f"cannot open {path}") from None
    if got != n:
        raise errors.FormatError(f"cannot open {path}")
    return _parse_pinned(host, n, schema, ctx)


# ---- binary columnar cache ------------------------------------------------------

def _cache_dir(directory, table):
    return os.path.join(directory, ".laq_cache", table)


def _stamp(path):
    st = os.stat(path)
    return {"size": st.st_size, "mtime_ns": st.st_mtime_ns}


def _cache_load(directory, table, csv_path, schema, device):
    d = _cache_dir(directory, table)
    meta_p = os.path.join(d, "meta.json")
    if not os.path.exists(meta_p):
        return None
    try:
        meta = json.load(open(meta_p))
    except (OSError, ValueError):
        return None
    if meta.get("stamp") != _stamp(csv_path) or meta.get("schema") != [[n, k] for n, k in schema]:
        return None
    rows = int(meta["rows"])
    out = {}
    for name, kind in schema:
        dt = np.float64 if kind == 2 else np.int64
        a = np.fromfile(os.path.join(d, f"{name}.bin"), dtype=dt)
        if a.size != rows:
            return None
        out[name] = torch.from_numpy(a).pin_memory().to(device, non_blocking=True)
    return out


def _cache_store(directory, table, csv_path, schema, cols):
    d = _cache_dir(directory, table)
    try:
        os.makedirs(d, exist_ok=True)
        rows = 0
        for name, _ in schema:
            a = cols[name].cpu().numpy()
            rows = a.size
            a.tofile(os.path.join(d, f"{name}.bin"))
        json.dump({"stamp": _stamp(csv_path), "schema": [[n, k] for n, k in schema], "rows": rows},
                  open(os.path.join(d, "meta.json"), "w"))
    except OSError:
        pass  # read-only dataset directory: no cache


def load_table(directory, tj, ctx=None, cache=True) -> dict:
    """One manifest table entry -> device columns (cache first, else parse)."""
    ctx = ctx or context()
    schema = schema_from_json(tj["schema"])
    path = os.path.join(directory, tj["file"])
    device = f"cuda:{ctx.device}"
    if cache and os.path.exists(path):
        hit = _cache_load(directory, tj["name"], path, schema, device)
        if hit is not None:
            return hit
    cols = load_csv(path, schema, ctx)
    if cache:
        _cache_store(directory, tj["name"], path, schema, cols)
    return cols


def load_dataset(directory, ctx=None, cache=True):
    """laq::cli::load_dataset (cli.cpp:483-513) -> (DeviceStar, generator config,
    models [(kind, path)], {table: {column: CUDA tensor}})."""
    from .star import DeviceStar
    ctx = ctx or context()
    mp = os.path.join(directory, "manifest.json")
    try:
        manifest = json.load(open(mp))
    except OSError:
        raise errors.FormatError(f"cannot open {mp}") from None
    g = manifest["generator"]
    cfg = {"setting": g["setting"], "sf": int(g["sf"]), "seed": int(g["seed"]), "features": int(g["features"]),
           "dangling": float(g["dangling"]), "max_bytes": int(g["max_bytes"])}
    ds = DeviceStar(ctx)
    tables = {}
    fact_entries = [t for t in manifest["tables"] if t["role"] == "fact"]
    dim_entries = [t for t in manifest["tables"] if t["role"] != "fact"]
    for tj in fact_entries + dim_entries:
        cols = load_table(directory, tj, ctx, cache)
        kinds = {n: k for n, k in schema_from_json(tj["schema"])}
        ds.add_table_device64(tj["name"], cols, kinds, is_fact=tj["role"] == "fact")
        tables[tj["name"]] = cols
    for fk, dim, pk in manifest["links"]:
        ds.add_link(fk, dim, pk)
    models = [(m["kind"], os.path.join(directory, m["file"])) for m in manifest.get("models", [])]
    return ds, cfg, models, tables
