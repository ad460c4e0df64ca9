"""Input types of the rule-evaluation path: schema, tuples, relation, partition.

These are the value types the reference engine consumes
(pkg/src/ruleblock/relation.py:30-164).  They are restated here so the
package runs where the reference is not installed (the GPU box).  The
engine itself is duck-typed: it accepts the reference's own ``Relation`` /
``DataPartition`` objects as well, because it only reads ``schema.kind_of``,
``schema.index_of``, ``tuples[i].values`` and ``tuple_refs``.

CSV ingest (relation.py:186-257) is out of scope for this path.
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from enum import Enum
from typing import Optional, Union

from .errors import SchemaError


class Kind(str, Enum):
    """Attribute kinds (relation.py:30-34).  A ``str`` enum so that the
    reference's ``Kind`` members compare equal to ours by value."""

    CATEGORICAL = "categorical"
    NUMERIC = "numeric"
    SHORT_TEXT = "short_text"
    LONG_TEXT = "long_text"


class Missing:
    """The absent-cell marker (relation.py:37-51).  Falsy singleton."""

    _one: Optional["Missing"] = None

    def __new__(cls) -> "Missing":
        if cls._one is None:
            cls._one = super().__new__(cls)
        return cls._one

    def __repr__(self) -> str:
        return "Missing"

    def __bool__(self) -> bool:
        return False


MISSING = Missing()

AttrValue = Union[Missing, str, float]


def is_missing(value) -> bool:
    """True for our marker, the reference's marker (any class named
    ``Missing``) and ``None``."""
    return value is None or value is MISSING or type(value).__name__ == "Missing"


_CURRENCY = re.compile(r"^[\s$€£¥]+|[\s]+$")
_THOUSANDS = re.compile(r",(?=\d{3}(\D|$))")


def parse_number(text: str) -> Optional[float]:
    """Finite decimal parse tolerant of currency glyphs and thousands
    separators; None when the text is not a number (relation.py:64-77)."""
    body = _THOUSANDS.sub("", _CURRENCY.sub("", text.strip()))
    if not body:
        return None
    try:
        x = float(body)
    except ValueError:
        return None
    if x != x or x in (float("inf"), float("-inf")):
        return None
    return x


def is_numeric_kind(kind) -> bool:
    return kind == Kind.NUMERIC or kind == "numeric"


@dataclass(frozen=True)
class Schema:
    attributes: tuple[tuple[str, Kind], ...]
    eid_attr: Optional[str] = None

    def __post_init__(self) -> None:
        names = [n for n, _ in self.attributes]
        if len(set(names)) != len(names):
            raise SchemaError(f"duplicate attribute names: {sorted({n for n in names if names.count(n) > 1})}")
        if self.eid_attr is not None and self.eid_attr not in names:
            raise SchemaError(f"eid attribute {self.eid_attr!r} not in schema")

    @property
    def names(self) -> tuple[str, ...]:
        return tuple(n for n, _ in self.attributes)

    def index_of(self, attr: str) -> int:
        for i, (n, _) in enumerate(self.attributes):
            if n == attr:
                return i
        raise SchemaError(f"unknown attribute {attr!r}")

    def kind_of(self, attr: str) -> Kind:
        return self.attributes[self.index_of(attr)][1]

    @property
    def arity(self) -> int:
        return len(self.attributes)


@dataclass(frozen=True)
class TupleRecord:
    tid: int
    eid: Optional[str]
    values: tuple


@dataclass(frozen=True)
class Relation:
    schema: Schema
    tuples: tuple[TupleRecord, ...]

    def __post_init__(self) -> None:
        for pos, rec in enumerate(self.tuples):
            if rec.tid != pos:
                raise SchemaError(f"tuple ids must be dense 0..n-1, found {rec.tid} at {pos}")
            if len(rec.values) != self.schema.arity:
                raise SchemaError(f"tuple {rec.tid} has {len(rec.values)} values, schema arity is {self.schema.arity}")

    def __len__(self) -> int:
        return len(self.tuples)

    def column(self, attr: str) -> list:
        k = self.schema.index_of(attr)
        return [rec.values[k] for rec in self.tuples]


@dataclass
class DataPartition:
    """Ordered tuple ids of one partition (relation.py:143-164).  Refs must
    be non-empty and duplicate-free; their ORDER matters: in symmetric mode
    the lower position plays ``t``."""

    pid: int
    tuple_refs: tuple[int, ...]
    branch_id: Optional[int] = None
    key_group: Optional[str] = None
    sibling_group: Optional[int] = None

    def __post_init__(self) -> None:
        if not self.tuple_refs:
            raise SchemaError(f"partition {self.pid} is empty")
        if len(set(self.tuple_refs)) != len(self.tuple_refs):
            raise SchemaError(f"partition {self.pid} has duplicate tuple refs")

    def __len__(self) -> int:
        return len(self.tuple_refs)


def relation_from_rows(names, kinds, rows) -> Relation:
    """Build a relation from already-typed rows (str / float / MISSING)."""
    schema = Schema(attributes=tuple((n, Kind(k)) for n, k in zip(names, kinds)))
    recs = tuple(
        TupleRecord(tid=i, eid=None, values=tuple(MISSING if is_missing(v) else v for v in row))
        for i, row in enumerate(rows)
    )
    return Relation(schema=schema, tuples=recs)
