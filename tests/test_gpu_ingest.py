"""GPU: the device CSV loader (csv.cu, ingest.py) against the reference's own
load_csv / write_dataset (oracle/_ref, storage.cpp:112-150, cli.cpp:430-513):
values bit-exact (ints and correctly rounded floats), the same first-error
line and message, and a dataset written by the reference loaded into HBM and
queried with the same results as the oracle on the generator's arrays."""
import os

import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu


def _device_parse(data: bytes, kinds):
    from paper_2306_08367_b200 import ingest
    schema = [(f"c{i}", k) for i, k in enumerate(kinds)]
    cols = ingest.parse_csv_bytes(data, schema)
    return [cols[f"c{i}"].cpu().numpy() for i in range(len(kinds))]


def _ref_parse(tmp_path, data: bytes, kinds):
    p = tmp_path / "t.csv"
    p.write_bytes(data)
    return R.load_csv(p, kinds, cap=data.count(b"\n") + 2)


def _same(a, b):
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.int64), b.view(np.int64))  # bit-exact (signed zero, nan payload aside)
    return np.array_equal(a, b)


def _check(tmp_path, data: bytes, kinds):
    """Device and reference agree: same values, or the same error and message."""
    from paper_2306_08367_b200 import errors
    try:
        want, rows = _ref_parse(tmp_path, data, kinds)
        ref_err = None
    except R.RefError as e:
        ref_err = (e.code, str(e).split("] ", 1)[1])
    try:
        got = _device_parse(data, kinds)
        dev_err = None
    except errors.Error as e:
        dev_err = (type(e).__name__, str(e))
    if ref_err is not None:
        assert dev_err is not None, (data, ref_err)
        assert dev_err[0] == "FormatError" and ref_err[0] == 4, (data, ref_err, dev_err)
        assert dev_err[1] == ref_err[1], (data, ref_err, dev_err)
        return None
    assert dev_err is None, (data, dev_err)
    for g, w in zip(got, want):
        assert len(g) == rows
        nan = np.isnan(w) if w.dtype == np.float64 else np.zeros(len(w), bool)
        assert _same(g[~nan], w[~nan]), data
        if nan.any():
            assert np.isnan(g[nan]).all()
    return got


CASES = [
    (b"1,2.5\n3,4\n", [1, 2]),
    (b"1,2.5\r\n3,4\r\n", [1, 2]),            # CRLF
    (b"1,2.5\n3,4", [1, 2]),                  # no final newline
    (b"", [1, 2]),                            # empty file: no rows
    (b"\n", [1]),                             # lone empty line, one column: missing value
    (b"5\n\n6\n", [1]),
    (b"1,2\n\n3,4\n", [1, 1]),                # empty line, two columns: expected 2 fields
    (b"1,2,3\n", [1, 1]),                     # too many fields
    (b"1\n", [1, 1]),                         # too few
    (b"1,\n", [1, 1]),                        # trailing empty field
    (b",1\n", [1, 1]),
    (b"+5\n", [1]), (b"-\n", [1]), (b"1.0\n", [1]), (b" 1\n", [1]), (b"1 \n", [1]), (b"007\n-0\n", [1]),
    (b"9223372036854775807\n-9223372036854775808\n", [1]),
    (b"9223372036854775808\n", [1]), (b"-9223372036854775809\n", [1]),
    (b"inf\n-INF\ninfinity\nnan\nNaN\nnan(123)\n-nan\n", [2]),
    (b"nan(\n", [2]), (b"in\n", [2]), (b"infin\n", [2]), (b"+1\n", [2]), (b".\n", [2]), (b"e5\n", [2]),
    (b".5\n5.\n-.5e3\n1E5\n1e+5\n1e-5\n-0\n0e-999\n0.000\n", [2]),
    (b"1e\n", [2]), (b"1e+\n", [2]), (b"0x10\n", [2]),
    (b"1e-400\n", [2]), (b"2e-324\n", [2]), (b"3e-324\n", [2]), (b"5e-324\n", [2]), (b"1e400\n", [2]),
    (b"1.7976931348623157e308\n1.7976931348623158e308\n", [2]), (b"1.7976931348623159e308\n", [2]),
    (b"2.4703282292062328e-324\n", [2]), (b"2.4703282292062327e-324\n", [2]),
    (b"2.2250738585072011e-308\n2.2250738585072014e-308\n4.9406564584124654e-324\n", [2]),
    (b"9007199254740993\n9007199254740992.5\n123456789012345678\n0.1\n0.30000000000000004\n", [2]),
    (b"1,2\n3,x\n4,y\n", [1, 1]),             # first bad line wins
    (b"1,2\n3,4\n5,6.5\n", [1, 1]),
    (b"7,1.5,9\n8,2e3,10\n", [0, 2, 1]),
]


@pytest.mark.parametrize("data,kinds", CASES)
def test_csv_cases_match_reference(gpu_ctx, tmp_path, data, kinds):
    _check(tmp_path, data, kinds)


def test_float_fuzz_bit_exact(gpu_ctx, tmp_path):
    """200K floats: shortest round-trip reprs (what the reference's writer emits),
    random 1-19-digit significands over the whole exponent range, halfway
    cases and subnormals -- bit-exact vs std::from_chars."""
    rng = np.random.default_rng(7)
    lines = []
    bits = rng.integers(0, 2**63 - 1, 60_000, dtype=np.int64)
    vals = bits.view(np.float64)
    vals = vals[np.isfinite(vals)]
    lines += [repr(float(v)) for v in vals]
    lines += [repr(float(v)) for v in rng.random(40_000)]
    lines += [format(float(v), ".17g") for v in rng.random(20_000) * 10.0 ** rng.integers(-30, 30, 20_000)]
    for _ in range(60_000):
        nd = int(rng.integers(1, 20))
        digits = "".join(str(int(d)) for d in rng.integers(0, 10, nd))
        e = int(rng.integers(-340, 300))
        lines.append(f"{'-' if rng.random() < 0.3 else ''}{digits}e{e}")
    # exact halfway points between adjacent doubles (ties to even): integers in
    # [2^53, 2^63) where the spacing is 2^(k-52), midpoints need <= 19 digits
    for _ in range(10_000):
        k = int(rng.integers(53, 63))
        m = int(rng.integers(2**52, 2**53))
        lines.append(str(m * 2 ** (k - 52) + 2 ** (k - 53)))
        lines.append(f"{m * 2 ** (k - 52) + 2 ** (k - 53)}e-{int(rng.integers(1, 30))}")
    # subnormals
    lines += [repr(float(v)) for v in rng.random(5_000) * 2.2250738585072014e-308]
    data = ("\n".join(lines) + "\n").encode()
    # keep only lines the reference accepts (out-of-range ones are separate cases)
    p = tmp_path / "f.csv"
    ok = []
    for chunk in [lines]:
        for ln in chunk:
            try:
                float(ln)
            except ValueError:
                continue
            f = float(ln)
            if f == 0.0 and any(c in "123456789" for c in ln.split("e")[0]):
                continue  # underflow to zero: from_chars rejects
            if f in (float("inf"), float("-inf")):
                continue
            ok.append(ln)
    data = ("\n".join(ok) + "\n").encode()
    got = _check(tmp_path, data, [2])
    assert got is not None and len(got[0]) == len(ok)
    # and Python's correctly rounded float() agrees too
    want = np.array([float(x) for x in ok])
    assert np.array_equal(got[0].view(np.int64), want.view(np.int64))


def test_dataset_roundtrip_and_query(gpu_ctx, tmp_path):
    """write_dataset (reference) -> load_dataset (device) == gen_star columns;
    a query over the loaded star equals the oracle; the binary cache reloads
    identical columns."""
    from oracle import laq_oracle as O
    from paper_2306_08367_b200 import ingest, query as Q
    d = tmp_path / "ds"
    R.write_dataset(d, "S2", 2, 42, features=4)
    ds, cfg, models, tables = ingest.load_dataset(str(d))
    assert cfg["setting"] == "2" and cfg["sf"] == 2 and cfg["seed"] == 42
    h = R.lib().ref_gen_star(1, 2, 42, 4, 0.0, 0)
    L = R.lib()
    try:
        for t in range(L.ref_star_n_tables(h)):
            name = L.ref_star_table_name(h, t).decode()
            rows = L.ref_star_table_rows(h, t)
            for c in range(L.ref_star_table_ncols(h, t)):
                cn = L.ref_star_col_name(h, t, c).decode()
                kind = L.ref_star_col_kind(h, t, c)
                ptr = L.ref_star_col_data(h, t, c)
                import ctypes as C
                buf = (C.c_char * (rows * 8)).from_address(ptr)
                want = np.frombuffer(buf, dtype=np.float64 if kind == 2 else np.int64).copy()
                got = tables[name][cn].cpu().numpy()
                assert _same(got, want), (name, cn)
    finally:
        L.ref_star_free(h)
    host = {t: {c: v.cpu().numpy() for c, v in cols.items()} for t, cols in tables.items()}
    for gi, dial in ((1, 100), (2, 498)):
        q = Q.spec_with_dial(Q.group_defs(gi)[0], gi, dial)
        assert np.array_equal(ds.run_query(q), O.run_query(host, q))
    # second load hits the binary cache and returns identical columns
    assert os.path.exists(d / ".laq_cache" / "lineorder" / "meta.json")
    _, _, _, tables2 = ingest.load_dataset(str(d))
    for name in tables:
        for cn in tables[name]:
            assert _same(tables2[name][cn].cpu().numpy(), tables[name][cn].cpu().numpy())
