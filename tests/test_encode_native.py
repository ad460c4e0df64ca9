"""The native ASCII encoder (include/rbencode.h) is byte-identical to the
Python encoder that restates the reference (CPython str semantics)."""

import random
import string

import numpy as np
import pytest

from paper_2410_04349_b200.encode import RelationEncoding
from paper_2410_04349_b200.relation import MISSING, relation_from_rows

ALPHABET = string.ascii_letters + string.digits + string.punctuation + " \t\n\v\f\r\x1c\x1d\x1e\x1f"


def _rows(seed, n=400):
    rng = random.Random(seed)
    rows = []
    for _ in range(n):
        row = []
        for _ in range(3):
            if rng.random() < 0.08:
                row.append(MISSING)
            elif rng.random() < 0.1:
                row.append(rng.choice(["", "  ", "\x1c", "A", "a", "Foo  Bar", "foo bar"]))
            else:
                row.append("".join(rng.choice(ALPHABET) for _ in range(rng.randint(0, 30))))
        rows.append(row)
    return rows


def _encode_all(rel, monkeypatch, native):
    monkeypatch.setenv("RB_NATIVE_ENCODE", "1" if native else "0")
    enc = RelationEncoding(rel)
    out = {}
    for key in [("codes", "a"), ("codes", "b"), ("tokens", "a"), ("tokens", "c"), ("chars", "b"), ("chars", "c"),
                ("xtokens", "a", "c", 0), ("xtokens", "a", "c", 1)]:
        col = enc.columns[enc.get(key)]
        out[key] = (col.data.copy(), None if col.offsets is None else col.offsets.copy(),
                    None if col.missing is None else col.missing.copy())
    return out


@pytest.mark.parametrize("seed", range(8))
def test_native_equals_python(seed, monkeypatch):
    rel = relation_from_rows(["a", "b", "c"], ["short_text"] * 3, _rows(seed))
    nat = _encode_all(rel, monkeypatch, True)
    py = _encode_all(rel, monkeypatch, False)
    for key in nat:
        for x, y in zip(nat[key], py[key]):
            if x is None:
                assert y is None
            else:
                assert x.dtype == y.dtype and np.array_equal(x, y), key


def test_non_ascii_column_uses_python_semantics(monkeypatch):
    rel = relation_from_rows(["a", "b", "c"], ["short_text"] * 3,
                             [["Straße", "ÉCOLE", "x"], ["STRASSE", "école", "y"], ["a b", " x", "z"]])
    monkeypatch.setenv("RB_NATIVE_ENCODE", "1")
    enc = RelationEncoding(rel)
    ch = enc.columns[enc.get(("chars", "a"))]
    assert ch.data.dtype == np.uint32  # non-ASCII column -> utf-32 codepoints, Python casefold
    toks = enc.columns[enc.get(("tokens", "a"))]
    assert list(np.diff(toks.offsets)) == [1, 1, 2]
