"""Columnar encodings, exact integer threshold tables and the device program.

This is the host half of the boundary.  It turns a ``Relation`` plus an
``ExecutionPath`` into the plain arrays the C ABI takes
(include/rbgpu.h): relation-wide feature columns and a flat program.

Column semantics restate ``EncodedRelation`` (pkg/src/ruleblock/encode.py:58-175):

* codes  -- int32 dictionary codes over canonical keys, -1 = missing
            (encode.py:33-38, 77-89); cross-attribute equality shares one
            dictionary over both columns (encode.py:91-111).
* mask   -- uint8 per tuple, ``t.attr = const`` (encode.py:113-124).
* tokens -- CSR of sorted unique int32 token ids interned per attribute in
            first-appearance order (encode.py:126-138), plus a missing flag.
* chars  -- CSR of folded codepoints, uint8 when the column is all ASCII,
            else uint32 (encode.py:140-154), plus a missing flag.

Slot semantics restate ``compile_slot`` (encode.py:191-324).  The float64
threshold tests of the reference are replaced by integer tables computed
here in float64 with the very same expressions, so the device compares
integers only and still agrees bit-for-bit (SURVEY §8a "Exact-threshold
tables"):

* EDIT, prefilter form (encode.py:236-238):
    maxgap[L] = max{g : not (g > (1.0-d)*L)},  maxd[L] = max{k : 1.0 - k/L >= d}
    accept <=> L == 0  or  (|la-lb| <= maxgap[L] and lev <= maxd[L])
* JACCARD, prefilter form (encode.py:256-259):
    minsmall[b] = min{s : not (s < d*b)},  mink[t] = min{k : k/(t-k) >= d}
    accept <=> not both empty and min(n,m) >= minsmall[max(n,m)] and inter >= mink[n+m]

The "fallback" slots of the reference (cross-attribute jaccard / exact_token,
edit over columns of different char widths, equality across numeric/text
columns; encode.py:281-324) are not evaluated on the CPU here: they are
encoded into the same integer slot kinds with the scorer's semantics
(measures.py:45-70, 145-174) -- no length prefilter, shared vocabularies.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import ConfigError
from .plan import is_checkpoint
from .relation import is_missing, is_numeric_kind, parse_number
from .rules import BUILTIN_MEASURES
from .text import eval_equality, fold_text, tokenize, value_text

# column kinds (rb_column_kind in include/rbgpu.h)
COL_CODES, COL_MASK, COL_TOKENS, COL_CHARS = 0, 1, 2, 3
# slot kinds (rb_slot_kind)
SLOT_EQ_CODE, SLOT_EQ_CONST, SLOT_JACCARD, SLOT_EXACT, SLOT_EDIT = 0, 1, 2, 3, 4
SLOT_FLAG_PREFILTER = 1
# instruction ops
OP_EVAL, OP_CHECKPOINT = 0, 1
# program limits of the device interpreter (reuse/value bits are one u64 each)
MAX_SLOTS = 64
MAX_CHECKPOINTS = 64
NEVER = 1 << 30  # table value that no count reaches


BUILTIN_SCORERS = {"edit": "edit_score", "jaccard": "jaccard_score", "exact_token": "exact_token_score"}


def _require_builtin_scorer(reg, p) -> None:
    """Where the reference scores a predicate through the registry
    (_fallback_slot -> eval_predicate, encode.py:281-288, measures.py:145-174)
    the device evaluates the built-in measure.  A registry that maps the
    measure to anything else (a custom scorer, fold=False) would change
    results, so it is refused instead of silently replaced."""
    if reg is None or not hasattr(reg, "get"):
        return
    m = reg.get(p.measure)
    scorer = getattr(m, "scorer", None)
    name = getattr(scorer, "__name__", None)
    module = getattr(scorer, "__module__", "") or ""
    if name != BUILTIN_SCORERS.get(p.measure) or not module.endswith("measures") or not getattr(m, "fold", True):
        raise ConfigError(f"measure {p.measure!r} is registered with a custom scorer ({module}.{name}, "
                          f"fold={getattr(m, 'fold', True)}); {p.describe()} is scored through the registry by the "
                          f"reference and has no device kernel for a custom scorer")


@dataclass
class Column:
    kind: int
    data: np.ndarray  # codes int32[n] | mask uint8[n] | ids int32[nnz] | chars uint8/uint32[nnz]
    offsets: Optional[np.ndarray] = None  # int64[n+1] for tokens / chars
    missing: Optional[np.ndarray] = None  # uint8[n] for tokens / chars

    @property
    def width(self) -> int:
        return int(self.data.dtype.itemsize) if self.kind == COL_CHARS else 0

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.offsets)

    def max_row_length(self) -> int:
        """Longest row (computed once per column: compile_program asks per slot)."""
        cached = self.__dict__.get("_max_len")
        if cached is None or cached[0] is not self.offsets:
            cached = (self.offsets, int(self.row_lengths().max(initial=0)))
            self.__dict__["_max_len"] = cached
        return cached[1]


def ragged(rows: list, dtype) -> tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    flat = np.concatenate([np.asarray(r, dtype=dtype) for r in rows]) if rows and offsets[-1] else np.empty(0, dtype)
    return offsets, flat.astype(dtype, copy=False)


# ---------------------------------------------------------------------------
# Exact threshold tables


def edit_tables(delta: float, lmax: int, prefilter: bool) -> tuple[np.ndarray, np.ndarray]:
    maxgap = np.zeros(lmax + 1, dtype=np.int32)
    maxd = np.zeros(lmax + 1, dtype=np.int32)
    for L in range(1, lmax + 1):
        if prefilter:
            g = min(L, math.floor((1.0 - delta) * L))
            while g + 1 <= L and not (g + 1 > (1.0 - delta) * L):
                g += 1
            while g >= 0 and g > (1.0 - delta) * L:
                g -= 1
            maxgap[L] = g
        else:
            maxgap[L] = L
        k = min(L, max(0, math.floor((1.0 - delta) * L) + 2))
        while k >= 0 and not (1.0 - k / L >= delta):
            k -= 1
        while k + 1 <= L and 1.0 - (k + 1) / L >= delta:
            k += 1
        maxd[L] = k
    return maxgap, maxd


def jaccard_tables(delta: float, nmax: int, prefilter: bool) -> tuple[np.ndarray, np.ndarray]:
    minsmall = np.zeros(nmax + 1, dtype=np.int32)
    if prefilter:
        for big in range(nmax + 1):
            s = max(0, math.ceil(delta * big) - 1)
            while s < delta * big:
                s += 1
            minsmall[big] = s
    mink = np.full(2 * nmax + 1, NEVER, dtype=np.int32)
    for t in range(1, 2 * nmax + 1):
        k = max(0, math.floor(delta * t / (1.0 + delta)) - 2)
        while k <= t // 2:
            if k / (t - k) >= delta:
                mink[t] = k
                break
            k += 1
    return minsmall, mink


# ---------------------------------------------------------------------------
# Relation-wide encodings


def _canonical_key(value, numeric: bool):
    # encode.py:33-38
    if is_missing(value):
        return None
    if numeric:
        return float(value) if isinstance(value, float) else value
    return str(value).strip()


class Encoded:
    """Relation-wide feature columns keyed by what they encode.  One
    ``Encoded`` is uploaded to a device once (``rb_relation``) and shared by
    every program and partition over that relation."""

    def __init__(self, n: int):
        self.n = int(n)
        self.columns: list[Column] = []
        self.index: dict = {}
        self.relation = None

    def add(self, key, col: Column) -> int:
        if key in self.index:
            return self.index[key]
        self.columns.append(col)
        self.index[key] = len(self.columns) - 1
        return self.index[key]

    def get(self, key) -> int:
        if key in self.index:
            return self.index[key]
        built = self._build(key)
        if built is None:
            raise ConfigError(f"no encoded column for {key!r}")
        if isinstance(built, tuple):  # a shared-dictionary pair
            a, b = built
            self.add(key[:-1] + (0,), a)
            self.add(key[:-1] + (1,), b)
            return self.index[key]
        return self.add(key, built)

    def _build(self, key):  # overridden by RelationEncoding
        return None

    # -- predicate -> slot ------------------------------------------------

    def slot_for(self, p, reg=None) -> tuple[int, int, int, int]:
        """(kind, lhs column, rhs column, flags) for one predicate; restates
        ``compile_slot`` (encode.py:291-324)."""
        if p.comparator == "eq":
            if p.rhs_attr is None:
                c = self.get(("mask", p.lhs_attr, _const_key(p.const)))
                return SLOT_EQ_CONST, c, c, 0
            if p.is_cross_attr:
                a = self.get(("xcodes", p.lhs_attr, p.rhs_attr, 0))
                b = self.get(("xcodes", p.lhs_attr, p.rhs_attr, 1))
                return SLOT_EQ_CODE, a, b, 0
            c = self.get(("codes", p.lhs_attr))
            return SLOT_EQ_CODE, c, c, 0
        if p.measure is None:
            raise ConfigError(f"similarity predicate without measure: {p.describe()}")
        if p.measure not in BUILTIN_MEASURES:
            raise ConfigError(f"measure {p.measure!r} has no device kernel (built-ins: {BUILTIN_MEASURES})")
        if reg is not None and hasattr(reg, "get"):
            reg.get(p.measure)  # the reference raises ConfigError for unregistered measures
        rhs = p.rhs_attr or p.lhs_attr
        if p.measure == "edit":
            a = self.get(("chars", p.lhs_attr))
            b = self.get(("chars", rhs))
            same_width = self.columns[a].width == self.columns[b].width
            if not same_width:  # the reference's _fallback_slot: scored by the registry (encode.py:307-308)
                _require_builtin_scorer(reg, p)
            return SLOT_EDIT, a, b, SLOT_FLAG_PREFILTER if same_width else 0
        kind = SLOT_JACCARD if p.measure == "jaccard" else SLOT_EXACT
        if p.is_cross_attr:
            _require_builtin_scorer(reg, p)  # _fallback_slot (encode.py:310-317)
            a = self.get(("xtokens", p.lhs_attr, rhs, 0))
            b = self.get(("xtokens", p.lhs_attr, rhs, 1))
            return kind, a, b, 0
        c = self.get(("tokens", p.lhs_attr))
        return kind, c, c, SLOT_FLAG_PREFILTER if kind == SLOT_JACCARD else 0


def _const_key(const):
    return ("num", float(const)) if isinstance(const, (int, float)) and not isinstance(const, bool) else ("str", const)


def _is_columnar(relation) -> bool:
    return hasattr(relation, "text_column") and hasattr(relation, "numeric_column")


def _ascii_column(cols: list):
    """(bytes, offsets int64, missing uint8) of the concatenated str columns
    when every present value is an ASCII ``str``; None otherwise (the
    Python encoder then keeps CPython's full Unicode semantics)."""
    import os

    if os.environ.get("RB_NATIVE_ENCODE", "1") == "0":
        return None
    vals, miss = [], []
    for col in cols:
        for v in col:
            if is_missing(v):
                vals.append("")
                miss.append(1)
            elif type(v) is str:
                vals.append(v)
                miss.append(0)
            else:
                return None
    text = "".join(vals)
    if not text.isascii():
        return None
    lens = np.fromiter(map(len, vals), dtype=np.int64, count=len(vals))
    offsets = np.zeros(len(vals) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    return text.encode("ascii"), offsets, np.array(miss, dtype=np.uint8)


def _native():
    from . import _lib

    return _lib.lib(), _lib


class RelationEncoding(Encoded):
    """Lazily encodes the columns a path touches, from a ``Relation``
    (ours or the reference's)."""

    def __init__(self, relation):
        super().__init__(len(relation))
        self.relation = relation
        self.schema = relation.schema
        self._cols: dict = {}

    def _column(self, attr: str) -> list:
        if attr not in self._cols:
            if _is_columnar(self.relation):  # one column's values, no row objects
                self._cols[attr] = self.relation.column(attr)
            else:
                k = self.schema.index_of(attr)
                self._cols[attr] = [rec.values[k] for rec in self.relation.tuples]
        return self._cols[attr]

    def _ascii_raw(self, attrs: list):
        """(bytes, offsets, missing) of text columns straight from a
        columnar relation's CSV buffers when all of them are ASCII, else the
        generic path over the column values."""
        import os

        rel = self.relation
        if _is_columnar(rel) and os.environ.get("RB_NATIVE_ENCODE", "1") != "0":
            cols = [rel.text_column(a) for a in attrs]
            if all(c is not None and c.all_ascii() for c in cols):
                if len(cols) == 1:
                    c = cols[0]
                    return c.buf.tobytes(), c.offsets, c.missing
                bufs = [c.buf for c in cols]
                offs = [cols[0].offsets]
                base = int(cols[0].offsets[-1])
                for c in cols[1:]:
                    offs.append(c.offsets[1:] + base)
                    base += int(c.offsets[-1])
                return (np.concatenate(bufs).tobytes(), np.concatenate(offs),
                        np.concatenate([c.missing for c in cols]))
        return _ascii_column([self._column(a) for a in attrs])

    def _numeric_codes(self, attr: str):
        """First-appearance dictionary codes of a columnar numeric column
        (_canonical_key on floats), vectorised; None if not columnar."""
        rel = self.relation
        got = rel.numeric_column(attr) if _is_columnar(rel) else None
        if got is None:
            return None
        vals, miss = got
        out = np.full(self.n, -1, dtype=np.int32)
        idx = np.nonzero(miss == 0)[0]
        if len(idx):
            u, first, inv = np.unique(vals[idx], return_index=True, return_inverse=True)
            rank = np.empty(len(u), dtype=np.int32)
            rank[np.argsort(first, kind="stable")] = np.arange(len(u), dtype=np.int32)
            out[idx] = rank[inv]
        return out

    def _numeric(self, attr: str) -> bool:
        return is_numeric_kind(self.schema.kind_of(attr))

    def prepare(self, predicates) -> "RelationEncoding":
        for p in predicates:
            self.slot_for(p)
        return self

    def _build(self, key):
        tag = key[0]
        if tag == "codes" and self._numeric(key[1]):
            codes = self._numeric_codes(key[1])
            if codes is not None:
                return Column(COL_CODES, codes)
        if tag == "codes" and not self._numeric(key[1]):
            nat = self._ascii_raw([key[1]])
            if nat is not None:  # rb_encode_eq_codes: strip + first-appearance dictionary
                buf, offs, miss = nat
                L, lb = _native()
                out = np.empty(self.n, dtype=np.int32)
                L.rb_encode_eq_codes(buf, lb.ptr(offs), lb.ptr(miss), self.n, lb.ptr(out))
                return Column(COL_CODES, out)
        if tag == "codes":
            numeric = self._numeric(key[1])
            mapping: dict = {}
            out = np.empty(self.n, dtype=np.int32)
            for i, v in enumerate(self._column(key[1])):
                k = _canonical_key(v, numeric)
                out[i] = -1 if k is None else mapping.setdefault(k, len(mapping))
            return Column(COL_CODES, out)
        if tag == "xcodes":
            return self._cross_codes(key[1], key[2])
        if tag == "mask":
            attr, (ctype, cval) = key[1], key[2]
            numeric = self._numeric(attr)
            m = np.fromiter(
                (not is_missing(v) and eval_equality(v, cval, numeric_kind=numeric) for v in self._column(attr)),
                dtype=np.uint8,
                count=self.n,
            )
            return Column(COL_MASK, m)
        if tag == "tokens":
            return self._tokens([key[1]], {})[0]
        if tag == "xtokens":
            vocab: dict = {}
            a, b = self._tokens([key[1], key[2]], vocab)
            return a, b
        if tag == "chars":
            nat = self._ascii_raw([key[1]])
            if nat is not None:  # rb_encode_chars: strip + casefold, uint8 (all ASCII)
                buf, offs, miss = nat
                L, lb = _native()
                out_off = np.empty(self.n + 1, dtype=np.int64)
                out = np.empty(max(1, len(buf)), dtype=np.uint8)
                m = L.rb_encode_chars(buf, lb.ptr(offs), lb.ptr(miss), self.n, lb.ptr(out_off), lb.ptr(out))
                return Column(COL_CHARS, out[:m].copy(), out_off, miss)
            col = self._column(key[1])
            missing = np.fromiter((is_missing(v) for v in col), dtype=np.uint8, count=self.n)
            texts = ["" if is_missing(v) else fold_text(value_text(v)) for v in col]
            if all(t.isascii() for t in texts):
                rows = [np.frombuffer(t.encode("ascii"), dtype=np.uint8) for t in texts]
                offsets, flat = ragged(rows, np.uint8)
            else:
                rows = [np.frombuffer(t.encode("utf-32-le"), dtype=np.uint32) for t in texts]
                offsets, flat = ragged(rows, np.uint32)
            return Column(COL_CHARS, flat, offsets, missing)
        return None

    def _tokens(self, attrs: list, vocab: dict) -> list:
        nat = self._ascii_raw(attrs)
        cols = [self._column(a) for a in attrs] if nat is None else attrs
        if nat is not None:  # rb_encode_tokens over the columns back to back (one shared vocabulary)
            buf, offs, miss = nat
            L, lb = _native()
            total = len(offs) - 1
            out_off = np.empty(total + 1, dtype=np.int64)
            ids = np.empty(max(1, len(buf)), dtype=np.int32)
            vs = lb.ctypes.c_int32(0)
            nnz = L.rb_encode_tokens(buf, lb.ptr(offs), lb.ptr(miss), total, lb.ptr(out_off), lb.ptr(ids),
                                     lb.ctypes.byref(vs))
            ids = ids[:nnz]
            res = []
            for k in range(len(cols)):
                a, b = k * self.n, (k + 1) * self.n
                o = out_off[a:b + 1] - out_off[a]
                res.append(Column(COL_TOKENS, ids[out_off[a]:out_off[b]].copy(), o, miss[a:b].copy()))
            return res
        out = []
        for col in cols:
            rows = []
            missing = np.zeros(self.n, dtype=np.uint8)
            for i, v in enumerate(col):
                if is_missing(v):
                    missing[i] = 1
                    rows.append(())
                    continue
                rows.append(sorted({vocab.setdefault(t, len(vocab)) for t in tokenize(value_text(v))}))
            offsets, flat = ragged(rows, np.int32)
            out.append(Column(COL_TOKENS, flat, offsets, missing))
        return out

    def _cross_codes(self, lhs: str, rhs: str):
        ln, rn = self._numeric(lhs), self._numeric(rhs)
        lcol, rcol = self._column(lhs), self._column(rhs)
        if ln == rn:
            # encode.py:98-110: one dictionary over canonical keys
            def key_of(v):
                return _canonical_key(v, ln)
        else:
            # encode.py:98-99 routes this to eval_predicate, where
            # numeric = False and eval_equality compares numerically as soon
            # as one side is a float (measures.py:129-141).  Encodable as one
            # key space when every pair has a float side.
            def all_float(col):
                return all(isinstance(v, float) for v in col if not is_missing(v))

            def any_float(col):
                return any(isinstance(v, float) for v in col if not is_missing(v))

            if all_float(lcol) or all_float(rcol):
                def key_of(v):
                    if is_missing(v):
                        return None
                    x = v if isinstance(v, float) else parse_number(str(v))
                    return ("unparseable",) if x is None else x
            elif not any_float(lcol) and not any_float(rcol):
                def key_of(v):
                    return None if is_missing(v) else str(v).strip()
            else:
                raise ConfigError(f"equality t.{lhs} = s.{rhs} mixes float and text cells on both sides")
        mapping: dict = {}

        def encode(col):
            out = np.empty(self.n, dtype=np.int32)
            for i, v in enumerate(col):
                k = key_of(v)
                if k is None:
                    out[i] = -1
                elif k == ("unparseable",):
                    out[i] = -2  # matches nothing, not even itself
                else:
                    out[i] = mapping.setdefault(k, len(mapping))
            return Column(COL_CODES, out)

        return encode(lcol), encode(rcol)


# ---------------------------------------------------------------------------
# Program


# numpy mirror of struct rb_slot (include/rbgpu.h)
SLOT_DTYPE = np.dtype(
    [
        ("kind", np.int32),
        ("lhs", np.int32),
        ("rhs", np.int32),
        ("flags", np.int32),
        ("tab0", np.int64),
        ("tab1", np.int64),
        ("len0", np.int32),
        ("len1", np.int32),
        ("delta", np.float64),
    ]
)


@dataclass
class Program:
    """Flat device program: instruction arrays, slot descriptors, tables."""

    ins_op: np.ndarray
    ins_slot: np.ndarray
    ins_fail: np.ndarray
    ins_rule: np.ndarray
    slots: np.ndarray  # SLOT_DTYPE
    tables: np.ndarray  # int32
    rule_ids: list
    n_slots: int
    extra: dict = field(default_factory=dict)


def compile_program(path, enc: Encoded, reg=None) -> Program:
    """ExecutionPath (+ encodings) -> flat program.  Instruction semantics
    follow ``evaluate_pair`` (pkg/src/ruleblock/engine.py:93-132)."""
    n_ins = len(path.instructions)
    rule_index = {rid: k for k, rid in enumerate(path.rule_ids)}
    op = np.zeros(n_ins, dtype=np.int32)
    slot = np.full(n_ins, -1, dtype=np.int32)
    fail = np.full(n_ins, -1, dtype=np.int32)
    rule = np.full(n_ins, -1, dtype=np.int32)
    n_cp = 0
    for k, ins in enumerate(path.instructions):
        if is_checkpoint(ins):
            if ins.rule_id not in rule_index:
                raise ConfigError(f"checkpoint names unknown rule {ins.rule_id!r}")
            op[k], rule[k] = OP_CHECKPOINT, rule_index[ins.rule_id]
            n_cp += 1
        else:
            if not 0 <= ins.slot < len(path.predicate_table):
                raise ConfigError(f"instruction {k}: slot {ins.slot} out of range")
            if not k < ins.fail_jump <= n_ins:
                raise ConfigError(f"instruction {k}: fail_jump {ins.fail_jump} out of range")
            op[k], slot[k], fail[k] = OP_EVAL, ins.slot, ins.fail_jump
    n_slots = len(path.predicate_table)
    if n_slots > MAX_SLOTS:
        raise ConfigError(f"path has {n_slots} predicate slots; the device interpreter supports {MAX_SLOTS}")
    if n_cp > MAX_CHECKPOINTS:
        raise ConfigError(f"path has {n_cp} checkpoints; the device interpreter supports {MAX_CHECKPOINTS}")

    slots = np.zeros(n_slots, dtype=SLOT_DTYPE)
    tables: list[np.ndarray] = []
    at = 0

    def put(arr: np.ndarray) -> int:
        nonlocal at
        off = at
        tables.append(arr.astype(np.int32))
        at += len(arr)
        return off

    for s, p in enumerate(path.predicate_table):
        kind, a, b, flags = enc.slot_for(p, reg)
        row = slots[s]
        row["kind"], row["lhs"], row["rhs"], row["flags"] = kind, a, b, flags
        row["delta"] = float(p.threshold) if p.threshold is not None else 0.0
        if kind == SLOT_EDIT:
            lmax = max(enc.columns[a].max_row_length(), enc.columns[b].max_row_length())
            g, d = edit_tables(float(p.threshold), lmax, bool(flags & SLOT_FLAG_PREFILTER))
            row["tab0"], row["len0"] = put(g), len(g)
            row["tab1"], row["len1"] = put(d), len(d)
        elif kind == SLOT_JACCARD:
            nmax = max(enc.columns[a].max_row_length(), enc.columns[b].max_row_length())
            ms, mk = jaccard_tables(float(p.threshold), nmax, bool(flags & SLOT_FLAG_PREFILTER))
            row["tab0"], row["len0"] = put(ms), len(ms)
            row["tab1"], row["len1"] = put(mk), len(mk)
    flat = np.concatenate(tables) if tables else np.zeros(1, dtype=np.int32)
    return Program(op, slot, fail, rule, slots, flat, list(path.rule_ids), n_slots)
