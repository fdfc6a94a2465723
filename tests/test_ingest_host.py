"""CPU: ingest host logic (schema kinds, manifest errors) and the reference's
own load_csv messages that the device loader reproduces (oracle/_ref)."""
import pytest

from oracle import ref as R


def test_schema_kinds():
    from paper_2306_08367_b200 import errors, ingest
    assert ingest.schema_from_json([["a", "key"], ["b", "int"], ["c", "float"]]) == [("a", 0), ("b", 1), ("c", 2)]
    with pytest.raises(errors.FormatError, match="unknown column kind: dbl"):
        ingest.col_kind_from_name("dbl")
    with pytest.raises(errors.FormatError, match="duplicate column name: a"):
        ingest._validate([("a", 1), ("a", 2)])
    with pytest.raises(errors.FormatError, match="schema has no columns"):
        ingest._validate([])


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("data,kinds,msg", [
    (b"1,2\n3\n", [1, 1], "line 2: expected 2 fields"),
    (b"\n", [1], "line 1: missing value"),
    (b"1,,\n", [1, 1, 1], "line 1: missing value"),
    (b"+5\n", [1], "line 1: bad integer '+5'"),
    (b"1e400\n", [2], "line 1: bad float '1e400'"),
    (b"1e-400\n", [2], "line 1: bad float '1e-400'"),
    (b"1e\n", [2], "line 1: bad float '1e'"),
])
def test_reference_load_csv_messages(tmp_path, data, kinds, msg):
    """Pins the messages the device loader must rebuild (storage.cpp:82-96, 130-143)."""
    p = tmp_path / "t.csv"
    p.write_bytes(data)
    with pytest.raises(R.RefError) as e:
        R.load_csv(p, kinds, cap=8)
    assert e.value.code == 4 and str(e.value).endswith(msg)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_reference_accepts_special_floats(tmp_path):
    p = tmp_path / "t.csv"
    p.write_bytes(b"inf\nnan\n5e-324\n-0\n")
    (c,), rows = R.load_csv(p, [2], cap=8)
    assert rows == 4 and c[0] == float("inf") and c[1] != c[1] and c[2] == 5e-324
