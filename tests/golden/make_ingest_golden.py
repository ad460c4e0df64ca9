"""Golden fixtures for the columnar CSV ingest, from the REFERENCE's
``load_relation`` (pkg/src/ruleblock/relation.py:186-257).

    python tests/golden/make_ingest_golden.py   # writes tests/golden/ingest.json.gz

Each case is a CSV byte string (seeded generator: quotes, embedded and bare
\\r / \\n line ends, empty lines, ragged rows, missing markers, currency /
thousands / underscore numbers, non-ASCII text, invalid UTF-8, NUL bytes),
optional schema hints / missing markers, and the reference's outcome: the
schema, eid attribute and every row's values, or the exception class and
message.  The bundled pkg/data/products.csv is included as is.
"""

from __future__ import annotations

import base64
import gzip
import json
import os
import random
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("RB_REFERENCE", "/root/reference/pkg")
sys.path.insert(0, os.path.join(REF, "src"))

from ruleblock.relation import is_missing, load_relation  # noqa: E402

PIECES = ["a", "b", "x y", " ", ",", '"', '""', "\n", "\r\n", "\r", "1", "23", "4.5", "-", "NULL", "$", "1,000",
          "12_3", "_1", "1e3", "E-2", ".", "€", "é", "ß", "\t", "inf", "nan", "+", "0x1", "१", "\x1c", "eid",
          "1,0000", ",000", "lorem ipsum dolor sit amet consectetur adipiscing elit sed do"]
NUMS = ["1", "2.5", "-3", "$4", " 5 ", "6e2", "7_0", "1,234", "$ 1,234.5", "", "-", "NULL", ".5", "5.", "1__0", "x",
        "1e400", "-0", "+.5e-3", "0001", "1_000_000", "12,345,678.9"]


def _cell(rng):
    return "".join(rng.choice(PIECES) for _ in range(rng.randint(0, 4)))


def _make(rng, ragged: float) -> bytes:
    names = [rng.choice(["eid", "a", "b", "c", "d", "e", "f"]) for _ in range(rng.randint(1, 5))]
    if rng.random() < 0.9:
        names = list(dict.fromkeys(names))
    lines = [",".join(names)]
    for _ in range(rng.randint(0, 10)):
        if rng.random() < ragged:
            lines.append("".join(_cell(rng) for _ in range(rng.randint(0, 6))))
            continue
        row = [rng.choice(NUMS) if rng.random() < 0.5 else _cell(rng) for _ in names]
        row = ['"' + c.replace('"', '""') + '"' if any(x in c for x in ',"\r\n') and rng.random() < 0.9 else c
               for c in row]
        lines.append(",".join(row))
    term = rng.choice(["\n", "\r\n", "\r"])
    data = (term.join(lines) + (term if rng.random() < 0.7 else "")).encode("utf-8")
    if rng.random() < 0.03:
        data += b"\xff"
    if rng.random() < 0.02:
        data = data.replace(b"a", b"\x00", 1)
    return data


def _outcome(path, kw):
    try:
        r = load_relation(path, **kw)
    except Exception as e:  # noqa: BLE001 -- the reference's own error is the expected outcome
        return {"error": type(e).__name__, "message": str(e).replace(str(path), "<path>")}
    rows = [[rec.eid, [None if is_missing(v) else (["f", repr(v)] if isinstance(v, float) else v) for v in rec.values]]
            for rec in r.tuples]
    return {"schema": [[n, k.value] for n, k in r.schema.attributes], "eid_attr": r.schema.eid_attr, "rows": rows}


def main():
    rng = random.Random(20240)
    cases = []
    srcs = [(open(os.path.join(REF, "data", "products.csv"), "rb").read(), {})]
    for k in range(400):
        kw = {}
        if rng.random() < 0.3:
            kw["schema_hints"] = {rng.choice(["a", "b", "c"]): rng.choice(["numeric", "short_text", "long_text",
                                                                           "categorical"])}
        if rng.random() < 0.2:
            kw["missing_markers"] = rng.choice([[], ["x"], ["", "NA"], ["-"]])
        srcs.append((_make(rng, 0.5 if k < 150 else 0.03), kw))
    with tempfile.TemporaryDirectory() as d:
        for k, (data, kw) in enumerate(srcs):
            p = os.path.join(d, "case.csv")
            open(p, "wb").write(data)
            cases.append({"csv": base64.b64encode(data).decode(), "kwargs": kw, "expected": _outcome(p, kw)})
    with gzip.open(os.path.join(HERE, "ingest.json.gz"), "wt") as fh:
        json.dump({"cases": cases}, fh)
    print(len(cases), "ingest cases")


if __name__ == "__main__":
    main()
