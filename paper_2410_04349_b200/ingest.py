"""Columnar CSV ingest: ``load_relation`` of the reference
(pkg/src/ruleblock/relation.py:186-257), same signature, errors and result,
without one Python object per cell on the way.

The reference reads every row with ``csv.reader``, substitutes missing
markers, infers each column's kind (``_infer_kind``, relation.py:167-183),
parses numeric columns with ``parse_number`` and builds a ``TupleRecord``
per row -- about 13 us per tuple in Python.  Here the native tokenizer
(``rb_csv_parse``, csrc/rb_csv.cpp: csv.reader's state machine over the
raw bytes) hands back one byte buffer + offsets per column; markers,
``parse_number`` and the token counts of ``_infer_kind`` run column-wise
(native for ASCII cells, ``parse_number`` itself for the rest), and the
result is a ``ColumnarRelation``: the reference's relation interface whose
rows are materialised only when something asks for them.  Its text columns
feed the native encoders (``rb_encode_*``) straight from the CSV buffers.

Inputs the native tokenizer hands back (invalid UTF-8, NUL bytes, oversize
fields, a record with the wrong field count) are read by ``csv.reader``
itself, so errors carry the reference's exact messages.
"""

from __future__ import annotations

import csv
import ctypes
from pathlib import Path
from typing import Iterable, Mapping, Optional, Union

import numpy as np

from .errors import DataParseError, SchemaError
from .relation import MISSING, Kind, Schema, TupleRecord, parse_number

DEFAULT_MISSING_MARKERS = ("", "-", "NULL")
LONG_TEXT_TOKEN_THRESHOLD = 8

_OK, _FIELD_COUNT, _NEEDS_PYTHON, _EMPTY = 0, -1, -2, -3


def _lib():
    from . import _lib as lb

    L = lb.lib()
    return L, lb


class TextColumn:
    """One column's cells: UTF-8 bytes back to back with int64 offsets, and
    the missing mask."""

    def __init__(self, buf: np.ndarray, offsets: np.ndarray, missing: np.ndarray):
        self.buf = buf
        self.offsets = offsets
        self.missing = missing
        self._ascii = None

    def __len__(self) -> int:
        return len(self.offsets) - 1

    def cell(self, i: int) -> str:
        return self.buf[self.offsets[i]:self.offsets[i + 1]].tobytes().decode("utf-8")

    def texts(self) -> list:
        raw = self.buf.tobytes()
        o = self.offsets.tolist()
        return [raw[o[i]:o[i + 1]].decode("utf-8") for i in range(len(o) - 1)]

    def all_ascii(self) -> bool:
        if self._ascii is None:
            self._ascii = bool(len(self.buf) == 0 or int(self.buf.max()) < 0x80)
        return self._ascii


class ColumnarRelation:
    """The reference relation interface (``schema``, ``tuples``, ``len``)
    over columnar storage.  ``tuples`` is built on first use; the encoders
    read the columns directly (``text_column`` / ``numeric_column``)."""

    def __init__(self, schema: Schema, n: int, text: dict, numeric: dict, eids: Optional["TextColumn"]):
        self.schema = schema
        self.n = n
        self._text = text  # attr -> TextColumn (non-numeric kinds)
        self._numeric = numeric  # attr -> (values float64, missing uint8)
        self._eids = eids
        self._tuples = None

    def __len__(self) -> int:
        return self.n

    def text_column(self, attr: str) -> Optional[TextColumn]:
        return self._text.get(attr)

    def numeric_column(self, attr: str):
        return self._numeric.get(attr)

    def column(self, attr: str) -> list:
        if attr in self._numeric:
            vals, miss = self._numeric[attr]
            return [MISSING if m else v for v, m in zip(vals.tolist(), miss.tolist())]
        col = self._text[attr]
        return [MISSING if m else t for t, m in zip(col.texts(), col.missing.tolist())]

    @property
    def tuples(self) -> tuple:
        if self._tuples is None:
            cols = [self.column(name) for name in self.schema.names]
            e = self._eids
            eids = [None] * self.n if e is None else [None if m else t for t, m in zip(e.texts(), e.missing.tolist())]
            self._tuples = tuple(TupleRecord(tid=i, eid=eids[i], values=tuple(c[i] for c in cols))
                                 for i in range(self.n))
        return self._tuples


def _missing_mask(col_buf: np.ndarray, offs: np.ndarray, markers: set) -> np.ndarray:
    """cell in markers, column-wise: cells of a marker's byte length are
    compared with it byte by byte (vectorised gather)."""
    lens = np.diff(offs)
    miss = np.zeros(len(lens), dtype=np.uint8)
    for m in markers:
        mb = np.frombuffer(m.encode("utf-8"), dtype=np.uint8)
        idx = np.nonzero(lens == len(mb))[0]
        if not len(idx):
            continue
        if len(mb) == 0:
            miss[idx] = 1
            continue
        cells = col_buf[offs[idx][:, None] + np.arange(len(mb))[None, :]]
        miss[idx[(cells == mb[None, :]).all(axis=1)]] = 1
    return miss


def load_relation(path: Union[str, Path], fmt: str = "csv_with_header",
                  schema_hints: Optional[Mapping[str, Union[Kind, str]]] = None,
                  missing_markers: Iterable[str] = DEFAULT_MISSING_MARKERS,
                  eid_attr: Optional[str] = "eid") -> ColumnarRelation:
    """relation.py:186-257: header-ed CSV -> relation (columnar)."""
    if fmt != "csv_with_header":
        raise DataParseError(f"unsupported format {fmt!r}")
    path = Path(path)
    if not path.exists():
        raise DataParseError(f"no such file: {path}")
    markers = set(missing_markers)
    hints = dict(schema_hints or {})
    data = path.read_bytes()

    L, lb = _lib()
    h = lb.c_vp()
    err = ctypes.c_int64(0)
    rc = L.rb_csv_parse(data, len(data), ctypes.byref(h), ctypes.byref(err))
    if rc == _EMPTY:
        raise DataParseError(f"{path}: empty file, header row required")
    if rc != _OK:  # the exact csv.reader behaviour and messages
        return _load_python(path, markers, hints, eid_attr)
    try:
        rows = ctypes.c_int64(0)
        ncols = ctypes.c_int32(0)
        L.rb_csv_shape(h, ctypes.byref(rows), ctypes.byref(ncols))
        n, k = rows.value, ncols.value
        header, cols = [], []
        for c in range(k):
            p = ctypes.c_void_p()
            nb = ctypes.c_int64(0)
            L.rb_csv_header(h, c, ctypes.byref(p), ctypes.byref(nb))
            header.append(ctypes.string_at(p.value, nb.value).decode("utf-8") if nb.value else "")
            po = ctypes.POINTER(ctypes.c_int64)()
            L.rb_csv_column(h, c, ctypes.byref(p), ctypes.byref(nb), ctypes.byref(po))
            raw = ctypes.string_at(p.value, nb.value) if nb.value else b""
            buf = np.frombuffer(raw, dtype=np.uint8).copy()
            offs = np.ctypeslib.as_array(po, shape=(n + 1,)).copy()
            cols.append((buf, offs))
    finally:
        L.rb_csv_free(h)
    return _build(path, header, cols, n, markers, hints, eid_attr)


def _build(path, header, cols, n, markers, hints, eid_attr) -> ColumnarRelation:
    if len(set(header)) != len(header):
        dupes = sorted({x for x in header if header.count(x) > 1})
        raise SchemaError(f"{path}: duplicate header names {dupes}")
    L, lb = _lib()
    kinds, text, numeric, first_bad = [], {}, {}, []
    for (buf, offs), name in zip(cols, header):
        miss = _missing_mask(buf, offs, markers)
        vals = np.zeros(n, dtype=np.float64)
        status = np.zeros(n, dtype=np.uint8)
        if n:
            L.rb_parse_numbers(buf.ctypes.data, lb.ptr(offs), n, lb.ptr(vals), lb.ptr(status))
        col = TextColumn(buf, offs, miss)
        slow = np.nonzero(status == 2)[0]  # non-ASCII cells: parse_number itself
        for i in slow.tolist():
            x = parse_number(col.cell(i))
            status[i], vals[i] = (0, 0.0) if x is None else (1, x)
        present = miss == 0
        if name in hints:
            kind = Kind(hints[name])
        elif present.any() and bool((status[present] == 1).all()):
            kind = Kind.NUMERIC
        else:
            counts = np.zeros(n, dtype=np.int32)
            if n:
                L.rb_token_counts(buf.ctypes.data, lb.ptr(offs), n, lb.ptr(counts))
            for i in np.nonzero(counts < 0)[0].tolist():
                counts[i] = len(col.cell(i).split())
            pc = np.sort(counts[present])
            kind = Kind.SHORT_TEXT
            if len(pc):
                mid = len(pc) // 2
                median = float(pc[mid]) if len(pc) % 2 else (int(pc[mid - 1]) + int(pc[mid])) / 2.0
                if median > LONG_TEXT_TOKEN_THRESHOLD:
                    kind = Kind.LONG_TEXT
        kinds.append(kind)
        if kind is Kind.NUMERIC:
            bad = np.nonzero(present & (status != 1))[0]
            if len(bad):  # (row, column) order of the reference's row-major value loop
                first_bad.append((int(bad[0]), len(kinds) - 1, col.cell(int(bad[0]))))
            numeric[name] = (vals, miss)
        else:
            text[name] = col
    if first_bad:
        tid, _, cell = min(first_bad)
        raise DataParseError(f"{path}: row {tid}: non-numeric cell {cell!r} in numeric column")
    schema = Schema(attributes=tuple(zip(header, kinds)), eid_attr=eid_attr if eid_attr in header else None)
    eids = None  # the eid column's cells, decoded when rows are materialised
    if eid_attr in header:
        c = header.index(eid_attr)
        buf, offs = cols[c]
        eids = TextColumn(buf, offs, _missing_mask(buf, offs, markers))
    return ColumnarRelation(schema, n, text, numeric, eids)


def _load_python(path, markers, hints, eid_attr) -> ColumnarRelation:
    """csv.reader path (relation.py:208-218): exact reader behaviour and
    errors; the rows are then stored column-wise like the native path."""
    with path.open(newline="", encoding="utf-8") as fh:
        reader = csv.reader(fh)
        try:
            header = next(reader)
        except StopIteration:
            raise DataParseError(f"{path}: empty file, header row required") from None
        if len(set(header)) != len(header):
            dupes = sorted({h for h in header if header.count(h) > 1})
            raise SchemaError(f"{path}: duplicate header names {dupes}")
        raw_rows = []
        for lineno, row in enumerate(reader, start=2):
            if len(row) != len(header):
                raise DataParseError(f"{path}: line {lineno}: expected {len(header)} fields, found {len(row)}")
            raw_rows.append(row)
    cols = []
    for c in range(len(header)):
        enc = [row[c].encode("utf-8") for row in raw_rows]
        offs = np.zeros(len(enc) + 1, dtype=np.int64)
        np.cumsum([len(x) for x in enc], out=offs[1:])
        cols.append((np.frombuffer(b"".join(enc), dtype=np.uint8).copy(), offs))
    return _build(path, header, cols, len(raw_rows), markers, hints, eid_attr)
