"""Columnar CSV ingest (ingest.load_relation) against the
reference's load_relation (relation.py:186-257): every fixture of
tests/golden/ingest.json.gz (made by make_ingest_golden.py from the
reference) must give the same schema, eids and values, or the same error
class and message -- through the native tokenizer and through the
csv.reader fallback."""

import base64
import gzip
import json
import os

import numpy as np
import pytest

from paper_2410_04349_b200 import errors, ingest
from paper_2410_04349_b200.relation import is_missing

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ingest.json.gz")


def _cases():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)["cases"]


def _outcome(path, kw):
    try:
        r = ingest.load_relation(path, **kw)
    except Exception as e:  # noqa: BLE001 -- compared with the reference's own error
        return {"error": type(e).__name__, "message": str(e).replace(str(path), "<path>")}
    rows = [[rec.eid, [None if is_missing(v) else (["f", repr(v)] if isinstance(v, float) else v) for v in rec.values]]
            for rec in r.tuples]
    return {"schema": [[n, k.value] for n, k in r.schema.attributes], "eid_attr": r.schema.eid_attr, "rows": rows}


@pytest.mark.parametrize("via", ["native", "csv_reader"])
def test_ingest_matches_reference(tmp_path, via, monkeypatch):
    if via == "csv_reader":  # force the fallback path for every file
        monkeypatch.setattr(ingest, "_OK", 12345)
    cases = _cases()
    assert len(cases) > 300
    for k, case in enumerate(cases):
        p = tmp_path / f"c{k}.csv"
        p.write_bytes(base64.b64decode(case["csv"]))
        exp = case["expected"]
        got = _outcome(p, case["kwargs"])
        assert got == exp, (k, got, exp)


def test_native_path_is_used(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text('eid,name,price\ne1,"a, b",$1\ne2,-,2\n')
    called = []
    orig = ingest._load_python
    try:
        ingest._load_python = lambda *a, **k: called.append(1) or orig(*a, **k)
        r = ingest.load_relation(p)
    finally:
        ingest._load_python = orig
    assert not called and len(r) == 2
    assert r.tuples[0].values == ("e1", "a, b", 1.0) and is_missing(r.tuples[1].values[1])
    col = r.text_column("name")
    assert col.all_ascii() and col.missing.tolist() == [0, 1]
    vals, miss = r.numeric_column("price")
    assert np.array_equal(vals, [1.0, 2.0])


def test_errors(tmp_path):
    with pytest.raises(errors.DataParseError, match="unsupported format"):
        ingest.load_relation(tmp_path / "x.csv", fmt="tsv")
    with pytest.raises(errors.DataParseError, match="no such file"):
        ingest.load_relation(tmp_path / "missing.csv")
    p = tmp_path / "e.csv"
    p.write_bytes(b"")
    with pytest.raises(errors.DataParseError, match="empty file"):
        ingest.load_relation(p)


@pytest.mark.parametrize("name", ["citation", "random_007", "edge_unicode", "edge_cross_attr", "grouped"])
def test_columnar_encoding_matches_row_encoding(tmp_path, name):
    """A relation written to CSV and read back by the columnar ingest encodes
    to exactly the same device columns as the row relation (native encoders
    fed straight from the CSV buffers)."""
    import csv

    import goldens
    from paper_2410_04349_b200.encode import RelationEncoding

    rel, path, _ = goldens.load(name)
    p = tmp_path / "r.csv"
    with open(p, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(rel.schema.names)
        for rec in rel.tuples:
            w.writerow(["<<MISSING>>" if is_missing(v) else (repr(v) if isinstance(v, float) else v)
                        for v in rec.values])
    hints = {n: k.value for n, k in rel.schema.attributes}
    col = ingest.load_relation(p, schema_hints=hints, missing_markers=("<<MISSING>>",), eid_attr=None)
    assert [r.values for r in col.tuples] == [r.values for r in rel.tuples]
    a = RelationEncoding(rel).prepare(path.predicate_table)
    b = RelationEncoding(col).prepare(path.predicate_table)
    assert a.index == b.index
    for ca, cb in zip(a.columns, b.columns):
        assert ca.kind == cb.kind
        for fa, fb in ((ca.data, cb.data), (ca.offsets, cb.offsets), (ca.missing, cb.missing)):
            assert (fa is None) == (fb is None)
            if fa is not None:
                assert np.array_equal(fa, fb)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["citation", "products"])
def test_csv_to_candidates_on_gpu(tmp_path, name):
    """End to end: the golden relation written to CSV, read by the columnar
    ingest, evaluated on the device through the drop-in run_partition --
    the reference's own rows."""
    import csv

    import goldens
    from paper_2410_04349_b200 import DataPartition, EngineConfig, run_partition

    rel, path, cases = goldens.load(name)
    p = tmp_path / "r.csv"
    with open(p, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(rel.schema.names)
        for rec in rel.tuples:
            w.writerow(["<<MISSING>>" if is_missing(v) else (repr(v) if isinstance(v, float) else v)
                        for v in rec.values])
    hints = {n: k.value for n, k in rel.schema.attributes}
    col = ingest.load_relation(p, schema_hints=hints, missing_markers=("<<MISSING>>",), eid_attr=None)
    for case in cases:
        if case["left"] is not None:
            continue
        refs = tuple(range(len(col))) if case["refs"] is None else tuple(case["refs"])
        cfg = EngineConfig(symmetric_mode=case["symmetric"], enumerate_witnesses=case["enumerate"])
        cs = run_partition(DataPartition(0, refs), col, path, cfg)
        assert sorted(cs.pairs) == goldens.expected_rows(case), case["name"]
