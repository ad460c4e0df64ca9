"""One COMPLETE oracle run of BASELINE config 2 (citation3, 1M tuples, seed
2024, one symmetric partition: 499,999,500,000 pairs) -- test infrastructure.

Runs oracle/rb_oracle.c over the whole triangle in outer-row slices
(resumable: finished slices are kept under --state), then writes
tests/golden/citation3_full.json: the row count, per-rule counts and the
sha256 of the sorted (t, s, rule) rows as little-endian int32 triples.
tests/test_full_golden.py (GPU) checks the GPU engine's complete output
against it.  Takes a few CPU-hours once:

    nice python tools/full_oracle_citation3.py --threads 6
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--threads", type=int, default=6)
    ap.add_argument("--slices", type=int, default=400)
    ap.add_argument("--state", default="/tmp/citation3_full_state")
    args = ap.parse_args()
    from oracle import oracle
    from paper_2410_04349_b200 import synth
    from paper_2410_04349_b200.encode import compile_program
    from paper_2410_04349_b200.engine import split_rows_by_pairs

    os.makedirs(args.state, exist_ok=True)
    w = synth.citation3(args.n, seed=args.seed)
    prog = compile_program(w.path, w.enc)
    cuts = split_rows_by_pairs(w.n, args.slices)
    t0 = time.time()
    pairs = 0
    for k, (lo, hi) in enumerate(cuts):
        f = os.path.join(args.state, f"slice{k:04d}.npz")
        if os.path.exists(f):
            pairs += int(np.load(f)["pairs"])
            continue
        rows, cmp, _ = oracle.run(w.enc, prog, None, w.n, row_lo=lo, row_hi=hi, flags=1, nthreads=args.threads)
        np.savez(f + ".tmp.npz", rows=rows.astype(np.int32), pairs=np.int64(cmp))
        os.replace(f + ".tmp.npz", f)
        pairs += cmp
        el = time.time() - t0
        print(f"slice {k + 1}/{len(cuts)} rows {len(rows)} pairs {pairs:.4e} elapsed {el:.0f}s", flush=True)
    rows = np.concatenate([np.load(os.path.join(args.state, f"slice{k:04d}.npz"))["rows"]
                           for k in range(len(cuts))])
    order = np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))
    rows = np.ascontiguousarray(rows[order].astype("<i4"))
    doc = {
        "workload": f"synth.citation3(n={args.n}, seed={args.seed}), one symmetric partition, identity refs",
        "pairs": int(pairs),
        "rows": int(len(rows)),
        "rows_per_rule": {w.path.rule_ids[r]: int((rows[:, 2] == r).sum()) for r in range(len(w.path.rule_ids))},
        "sha256_sorted_t_s_rule_int32le": hashlib.sha256(rows.tobytes()).hexdigest(),
        "generator": "tools/full_oracle_citation3.py (oracle/rb_oracle.c over every pair)",
        "path_rule_ids": list(w.path.rule_ids),
    }
    out = os.path.join(ROOT, "tests", "golden", "citation3_full.json")
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
