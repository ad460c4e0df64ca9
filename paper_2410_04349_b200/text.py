"""Host-side cell semantics that fix what the device compares.

Every function restates one rule of the reference's measure layer
(pkg/src/ruleblock/measures.py) on the host; the device only ever sees the
integers these produce (dictionary codes, token ids, folded codepoints), so
text semantics stay byte-identical to CPython's ``str`` methods.
"""

from __future__ import annotations

import string

from .relation import is_missing, parse_number

_DROP_PUNCT = str.maketrans("", "", string.punctuation)


def fold_text(text: str) -> str:
    """measures.py:25-26 -- strip, then casefold (edit-distance operand)."""
    return text.strip().casefold()


def tokenize(text: str) -> list[str]:
    """measures.py:29-34 -- casefold, drop ASCII punctuation, split on
    Unicode whitespace."""
    return text.casefold().translate(_DROP_PUNCT).split()


def value_text(value) -> str:
    """measures.py:112-117 -- integral floats print without '.0'."""
    if isinstance(value, float):
        return str(int(value)) if value == int(value) else repr(value)
    return str(value)


def eval_equality(a, b, numeric_kind: bool = False) -> bool:
    """measures.py:120-142 -- missing never matches; numeric kinds compare
    parsed decimals; mixed float/text compares numerically when both parse;
    otherwise trimmed text compares byte-exact."""
    if is_missing(a) or is_missing(b):
        return False
    if numeric_kind or isinstance(a, float) or isinstance(b, float):
        na = a if isinstance(a, float) else parse_number(str(a))
        nb = b if isinstance(b, float) else parse_number(str(b))
        return na is not None and nb is not None and na == nb
    return str(a).strip() == str(b).strip()
