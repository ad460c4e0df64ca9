"""Random relations and rule sets that stress the device program's shapes:
many equality / token / string features (beyond the filtered maxima), more
than 32 rules (64-bit masks), cross-attribute slots, constants, missing and
empty cells, non-ASCII text."""

from __future__ import annotations

import json
import random

from paper_2410_04349_b200.plan import plan_from_stats
from paper_2410_04349_b200.relation import MISSING, relation_from_rows
from paper_2410_04349_b200.rules import parse_ruleset, predicate_universe

WORDS = ["alpha", "beta", "gamma", "delta", "eps", "zeta", "eta", "theta", "iota", "kappa", "lambda", "mu",
         "Nu", "XI", "omicron", "pi", "rho", "σίγμα", "tau", "ÜPSILON"]


def make(seed: int, n: int = 220):
    rng = random.Random(seed)
    n_cat, n_txt = rng.randint(2, 8), rng.randint(2, 5)
    names = [f"c{k}" for k in range(n_cat)] + [f"t{k}" for k in range(n_txt)] + ["num"]
    kinds = ["short_text"] * n_cat + ["long_text"] * n_txt + ["numeric"]
    alph = [rng.randint(2, 9) for _ in range(n_cat)]
    base = []
    for _ in range(max(3, n // 6)):
        row = [f"v{rng.randrange(alph[k])}" for k in range(n_cat)]
        row += [" ".join(rng.choices(WORDS, k=rng.randint(1, 9))) for _ in range(n_txt)]
        row.append(float(rng.randint(0, 6)))
        base.append(row)
    rows = []
    for _ in range(n):
        r = list(rng.choice(base))
        for k in range(len(r)):
            x = rng.random()
            if x < 0.07:
                r[k] = MISSING
            elif x < 0.12 and kinds[k] != "numeric":
                r[k] = "" if rng.random() < 0.5 else "  "
            elif x < 0.35 and kinds[k] == "long_text":
                w = r[k].split() if isinstance(r[k], str) else []
                if w:
                    w[rng.randrange(len(w))] = rng.choice(WORDS)
                r[k] = " ".join(w)
        rows.append(r)
    rel = relation_from_rows(names, kinds, rows)

    def pred():
        kind = rng.random()
        if kind < 0.35:
            a = rng.choice(names[:n_cat] + ["num"])
            b = a if rng.random() < 0.8 else rng.choice(names[:n_cat] + ["num"])
            return {"t_attr": a, "op": "eq", "s_attr": b}
        if kind < 0.45:
            a = rng.randrange(n_cat)
            return {"t_attr": names[a], "op": "eq", "const": f"v{rng.randrange(alph[a])}"}
        a = rng.choice(names[n_cat:n_cat + n_txt])
        b = a if rng.random() < 0.8 else rng.choice(names[n_cat:n_cat + n_txt])
        m = rng.choice(["jaccard", "jaccard", "edit", "exact_token"])
        th = {"jaccard": rng.choice([0.2, 0.34, 0.5, 0.75]), "edit": rng.choice([0.4, 0.6, 0.8, 0.95]),
              "exact_token": 1.0}[m]
        return {"t_attr": a, "op": "sim", "s_attr": b, "measure": m, "threshold": th}

    n_rules = rng.choice([1, 3, 6, 12, 40])
    doc = []
    for r in range(n_rules):
        preds, seen = [], set()
        for _ in range(rng.randint(1, 4)):
            p = pred()
            key = json.dumps(p, sort_keys=True)
            if key not in seen:
                seen.add(key)
                preds.append(p)
        doc.append({"id": f"r{r}", "when": preds})
    rules = parse_ruleset(json.dumps(doc))
    uni = predicate_universe(rules)
    if len(uni) > 64:
        return make(seed + 100_000, n)
    costs = {p: rng.choice([0.1, 0.3, 1.0]) for p in uni}
    sps = {p: rng.choice([0.05, 0.3, 0.7]) for p in uni}
    return rel, rules, plan_from_stats(rules, costs, sps)
