"""Seeded synthetic relations of the benchmark shapes, generated column-wise.

The reference generates citation-style workloads row by row in Python
(``citation_benchmark``, pkg/src/ruleblock/datasets.py:332-398) and encodes
them with ``EncodedRelation`` at ~14 us/tuple.  At 1M-10M tuples that is
minutes of host time, so the benchmark relations here are produced directly
in the encoded columnar form the C ABI takes (codes / token CSR / char CSR),
with the same value domains and the same duplicate-injection scheme, and
a data-aware plan is derived from sampled selectivities (SURVEY §8d,
config 2).  Text is generated already folded (lower-case ASCII, single
spaces inside names), so the column values equal their folded forms.
"""

from __future__ import annotations

from dataclasses import dataclass

import json

import numpy as np

from .encode import COL_CHARS, COL_CODES, COL_TOKENS, Column, Encoded
from .plan import plan_from_stats
from .rules import parse_ruleset, predicate_universe

TITLE_VOCAB = 800  # datasets.py:320-323: 20 stems x 40 suffixes
FIRST = ["alice", "bob", "carol", "david", "erin", "frank", "grace", "henry", "irene", "jack",
         "karen", "liam", "maria", "nolan", "olivia", "peter", "quinn", "rachel", "simon", "tara"]
LAST = ["anders", "brown", "chen", "davis", "evans", "fischer", "garcia", "hansen", "ito", "jones",
        "kumar", "larsen", "meyer", "novak", "olsen", "patel", "quirk", "rossi", "schmidt", "tanaka"]

CITATION3_RULES = [
    {"id": "R1", "when": [
        {"t_attr": "year", "op": "eq", "s_attr": "year"},
        {"t_attr": "title", "op": "sim", "s_attr": "title", "measure": "jaccard", "threshold": 0.75}]},
    {"id": "R2", "when": [
        {"t_attr": "authors", "op": "sim", "s_attr": "authors", "measure": "edit", "threshold": 0.8},
        {"t_attr": "title", "op": "sim", "s_attr": "title", "measure": "jaccard", "threshold": 0.5}]},
    {"id": "R3", "when": [
        {"t_attr": "venue", "op": "eq", "s_attr": "venue"},
        {"t_attr": "cat", "op": "eq", "s_attr": "cat"},
        {"t_attr": "title", "op": "sim", "s_attr": "title", "measure": "exact_token", "threshold": 1.0}]},
]

KIND_COST = {"eq": 0.1, "exact_token": 0.3, "jaccard": 0.6, "edit": 1.0}


@dataclass
class Workload:
    name: str
    enc: Encoded
    rules: object
    path: object
    n: int
    blocks: object = None  # [(refs int32, split)]: cross blocks / partitions instead of one partition
    injected: object = None  # (a, b) int arrays: the generator's duplicate pairs (recall checks)
    block_attr: object = None  # blocks keyed on this attribute's value (its equality holds inside every block)

    def pairs(self, symmetric: bool = True) -> int:
        if self.blocks is None:
            return self.n * (self.n - 1) // 2 if symmetric else self.n * (self.n - 1)
        total = 0
        for refs, split in self.blocks:
            k = len(refs)
            total += split * (k - split) if split >= 0 else (k * (k - 1) // 2 if symmetric else k * (k - 1))
        return total


def _distinct_rows(rng, n: int, width: int, domain: int) -> np.ndarray:
    """n rows of `width` distinct ints in [0, domain), rejection-sampled."""
    out = rng.integers(0, domain, size=(n, width), dtype=np.int32)
    while True:
        s = np.sort(out, axis=1)
        bad = np.nonzero((s[:, 1:] == s[:, :-1]).any(axis=1))[0]
        if len(bad) == 0:
            return out
        out[bad] = rng.integers(0, domain, size=(len(bad), width), dtype=np.int32)


def _csr_from_padded(vals: np.ndarray, lens: np.ndarray, sort_rows: bool) -> tuple[np.ndarray, np.ndarray]:
    n, w = vals.shape
    if sort_rows:
        big = np.where(np.arange(w)[None, :] < lens[:, None], vals, np.iinfo(vals.dtype).max)
        vals = np.sort(big, axis=1)
    mask = np.arange(w)[None, :] < lens[:, None]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    return offsets, vals[mask]


def citation3(n: int = 1_000_000, seed: int = 2024, plan_sample: int = 200_000) -> Workload:
    """BASELINE config 2: citation-style relation, 3 rules mixing eq,
    jaccard and edit predicates."""
    rng = np.random.default_rng(seed)
    n_pairs = n // 4  # half of the tuples belong to an injected duplicate pair
    # ---- base records (one per entity): duplicates copy and perturb
    title_k = rng.integers(6, 11, size=n, dtype=np.int64)
    title = _distinct_rows(rng, n, 10, TITLE_VOCAB)
    n_auth = rng.integers(1, 4, size=n)
    auth_first = rng.integers(0, len(FIRST), size=(n, 3))
    auth_last = rng.integers(0, len(LAST), size=(n, 3))
    year = rng.integers(0, 16, size=n, dtype=np.int32)
    venue = rng.integers(0, 10, size=n, dtype=np.int32)
    zipf_p = 1.0 / np.arange(1, 1001) ** 1.1
    cat = rng.choice(1000, size=n, p=zipf_p / zipf_p.sum()).astype(np.int32)
    # ---- duplicates: tuple 2k+1 describes the same paper as 2k (k < n_pairs)
    a = np.arange(0, 2 * n_pairs, 2)
    b = a + 1
    title[b] = title[a]
    roll = rng.random(n_pairs)
    drop1 = (roll >= 0.55) & (roll < 0.90) & (title_k[a] > 6)
    drop2 = (roll >= 0.90) & (title_k[a] > 7)
    title_k[b] = title_k[a] - drop1 - 2 * drop2
    n_auth[b], auth_first[b], auth_last[b] = n_auth[a], auth_first[a], auth_last[a]
    year[b] = np.where(rng.random(n_pairs) < 0.96, year[a], (year[a] + 1) % 16)
    venue[b] = np.where(rng.random(n_pairs) < 0.8, venue[a], rng.integers(0, 10, size=n_pairs))
    cat[b] = np.where(rng.random(n_pairs) < 0.9, cat[a], cat[b])
    auth_edit = np.zeros(n, dtype=np.int8)  # 1: double the first space, 2: drop the last char
    r = rng.random(n_pairs)
    auth_edit[b] = np.where(r < 0.35, np.where(rng.random(n_pairs) < 0.5, 1, 2), 0)

    # ---- encode: token CSR (ids = vocabulary index), author chars
    t_off, t_ids = _csr_from_padded(title, title_k, sort_rows=True)
    names = [f"{f} {l}".encode() for f in FIRST for l in LAST]
    name_idx = auth_first * len(LAST) + auth_last
    strs = []
    for k in range(n):
        s = b", ".join(names[name_idx[k, j]] for j in range(n_auth[k]))
        e = auth_edit[k]
        if e == 1:
            s = s.replace(b" ", b"  ", 1)
        elif e == 2 and len(s) > 1:
            s = s[:-1]
        strs.append(s)
    a_len = np.fromiter((len(s) for s in strs), dtype=np.int64, count=n)
    a_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(a_len, out=a_off[1:])
    a_chars = np.frombuffer(b"".join(strs), dtype=np.uint8).copy()

    enc = Encoded(n)
    enc.add(("codes", "year"), Column(COL_CODES, year))
    enc.add(("codes", "venue"), Column(COL_CODES, venue))
    enc.add(("codes", "cat"), Column(COL_CODES, cat))
    enc.add(("tokens", "title"), Column(COL_TOKENS, t_ids.astype(np.int32), t_off, np.zeros(n, np.uint8)))
    enc.add(("chars", "authors"), Column(COL_CHARS, a_chars, a_off, np.zeros(n, np.uint8)))
    import json

    rules = parse_ruleset(json.dumps(CITATION3_RULES))
    path = data_aware_plan(enc, rules, sample=plan_sample, seed=seed)
    return Workload("citation3", enc, rules, path, n, injected=(a, b))


def sampled_selectivity(enc: Encoded, predicates, sample: int, seed: int) -> dict:
    """Pass rate of each predicate over `sample` random pairs, measured with
    the reference's exact slot semantics (host numpy, no device)."""
    from .encode import compile_program  # noqa: F401  (semantics live in the tables)

    rng = np.random.default_rng(seed + 17)
    i = rng.integers(0, enc.n, size=sample)
    j = rng.integers(0, enc.n, size=sample)
    keep = i != j
    i, j = i[keep], j[keep]
    out = {}
    for p in predicates:
        kind, lc, rc, _ = enc.slot_for(p)
        L, R = enc.columns[lc], enc.columns[rc]
        if p.comparator == "eq" and p.rhs_attr is not None:
            hit = (L.data[i] >= 0) & (L.data[i] == R.data[j])
        elif p.comparator == "eq":
            hit = L.data[i] != 0
        elif p.measure in ("jaccard", "exact_token"):
            hit = np.zeros(len(i), dtype=bool)
            m = min(len(i), 20000)
            for k in range(m):
                x = L.data[L.offsets[i[k]]:L.offsets[i[k] + 1]]
                y = R.data[R.offsets[j[k]]:R.offsets[j[k] + 1]]
                if p.measure == "exact_token":
                    hit[k] = len(x) > 0 and np.array_equal(x, y)
                else:
                    inter = len(np.intersect1d(x, y, assume_unique=True))
                    u = len(x) + len(y) - inter
                    hit[k] = u > 0 and inter / u >= p.threshold
            hit = hit[:m]
        else:
            la = np.diff(L.offsets)[i]
            lb = np.diff(R.offsets)[j]
            longest = np.maximum(la, lb)
            hit = (longest - np.minimum(la, lb)) <= (1.0 - p.threshold) * longest  # length part only
        out[p] = float(np.clip(hit.mean(), 1e-6, 1 - 1e-6))
    return out


def data_aware_plan(enc: Encoded, rules, sample: int = 200_000, seed: int = 0):
    """Cost-effectiveness order (1 - sp) / cost from sampled selectivities
    and per-kind cost constants, then the reference's tree + compile
    (planner/plan.py:28-76, 147-300)."""
    uni = predicate_universe(rules)
    sps = sampled_selectivity(enc, uni, sample, seed)
    costs = {p: KIND_COST["eq" if p.comparator == "eq" else p.measure] for p in uni}
    return plan_from_stats(rules, costs, sps)


EDIT_HEAVY_RULES = [
    {"id": "R1", "when": [
        {"t_attr": "text", "op": "sim", "s_attr": "text", "measure": "edit", "threshold": 0.98}]},
    {"id": "R2", "when": [
        {"t_attr": "name", "op": "sim", "s_attr": "name", "measure": "edit", "threshold": 0.97},
        {"t_attr": "zip", "op": "eq", "s_attr": "zip"}]},
]

ALPHA = b"abcdefghijklmnopqrstuvwxyz "


def _perturb(rng, base: bytes, k: int) -> bytes:
    """k random single-character substitutions / insertions / deletions
    (rng: random.Random)."""
    b = bytearray(base)
    for _ in range(k):
        op = rng.randrange(3)
        p = rng.randrange(len(b))
        c = ALPHA[rng.randrange(27)]
        if op == 0:
            b[p] = c
        elif op == 1:
            b.insert(p, c)
        elif len(b) > 1:
            del b[p]
    return bytes(b)


def _chars_column(strs: list) -> Column:
    lens = np.fromiter(map(len, strs), dtype=np.int64, count=len(strs))
    off = np.zeros(len(strs) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    data = np.frombuffer(b"".join(strs), dtype=np.uint8).copy()
    return Column(COL_CHARS, data, off, np.zeros(len(strs), np.uint8))


def edit_heavy(n: int = 1_000_000, seed: int = 11, plan_sample: int = 200_000) -> Workload:
    """BASELINE config 3: long-string edit distance with thresholds whose
    maxd[L] is 2-3: 64-256-char texts in groups of 2-50
    near-duplicates (0-3 random substitutions / indels), a short name with
    the same group structure and a Zipf zip code."""
    import random

    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    zipf_p = 1.0 / np.arange(1, 100_001) ** 1.1
    zip_draws = nrng.choice(100_000, size=2 * n, p=zipf_p / zipf_p.sum()).astype(np.int32).tolist()
    zd = 0
    texts, names, zips, gid = [], [], [], []
    while len(texts) < n:
        g = rng.randint(2, 50)
        base = bytes(ALPHA[rng.randrange(27)] for _ in range(rng.randint(64, 256)))
        nb = f"{rng.choice(FIRST)} {rng.choice(LAST)}".encode()
        z = zip_draws[zd]
        zd += 1
        g_id = len(texts)  # the group's first position: a unique group id
        for _ in range(min(g, n - len(texts))):
            gid.append(g_id)
            texts.append(_perturb(rng, base, rng.randint(0, 3)))
            names.append(nb if rng.random() < 0.8 else _perturb(rng, nb, 1))
            if rng.random() < 0.9:
                zips.append(z)
            else:
                zips.append(zip_draws[zd])
                zd += 1
    order = nrng.permutation(n)
    gid = np.asarray(gid, dtype=np.int64)
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    same = np.flatnonzero(gid[1:] == gid[:-1])  # consecutive members of one near-duplicate group
    injected = (inv[same], inv[same + 1])
    texts = [texts[k] for k in order]
    names = [names[k] for k in order]
    zips = np.asarray(zips, dtype=np.int32)[order]
    enc = Encoded(n)
    enc.add(("chars", "text"), _chars_column(texts))
    enc.add(("chars", "name"), _chars_column(names))
    enc.add(("codes", "zip"), Column(COL_CODES, zips))
    import json

    rules = parse_ruleset(json.dumps(EDIT_HEAVY_RULES))
    path = data_aware_plan(enc, rules, sample=plan_sample, seed=seed)
    return Workload("edit_heavy", enc, rules, path, n, injected=injected)


SYL = ["ka", "ri", "mo", "ta", "le", "sa", "no", "vi", "de", "ru", "mi", "ko", "na", "el", "an", "to", "be", "ga",
       "lu", "si", "ha", "jo", "pe", "ze", "ul", "or", "in", "ma", "ne", "bo", "ch", "st", "fr", "gr", "th", "ph",
       "wi", "ya", "qu", "ex", "ol", "ar", "en", "is", "um", "ad", "ed", "ik", "ov", "ey"]

LINKAGE_RULES = [
    {"id": "name", "when": [
        {"t_attr": "block", "op": "eq", "s_attr": "block"},
        {"t_attr": "name", "op": "sim", "s_attr": "name", "measure": "edit", "threshold": 0.85}]},
    {"id": "addr", "when": [
        {"t_attr": "block", "op": "eq", "s_attr": "block"},
        {"t_attr": "addr", "op": "sim", "s_attr": "addr", "measure": "jaccard", "threshold": 0.6}]},
]


def linkage(n: int = 1_000_000, seed: int = 5, zipf_s: float = 1.3, n_blocks: int = 200_000,
            plan_sample: int = 100_000) -> Workload:
    """BASELINE config 5: two-table record linkage.  One relation holds both
    sources (n/2 tuples each, a ``src`` split); a Zipf(1.3) block key makes a
    few blocks very large and most tiny.  Every block is one cross run
    (left = source A of the block, right = source B), i.e. run_cross per
    block.  30% of B tuples are perturbed copies of
    an A tuple of the same block."""
    rng = np.random.default_rng(seed)
    half = n // 2
    p = 1.0 / np.arange(1, n_blocks + 1) ** zipf_s
    p /= p.sum()
    block = rng.choice(n_blocks, size=n, p=p).astype(np.int32)
    # person names from syllables: ~2.5k first x ~125k last names
    first = rng.integers(0, len(SYL) ** 2, size=n)
    last = rng.integers(0, len(SYL) ** 3, size=n)
    n_tok = rng.integers(8, 15, size=n)
    addr = _distinct_rows(rng, n, 14, 5000)
    # duplicates: B tuple j copies A tuple dup_of[j] (same block), lightly perturbed
    dup = np.nonzero(rng.random(n - half) < 0.3)[0] + half
    src = rng.integers(0, half, size=len(dup))
    block[dup] = block[src]
    first[dup], last[dup] = first[src], last[src]
    addr[dup] = addr[src]
    n_tok[dup] = n_tok[src]
    drop = rng.random(len(dup)) < 0.3
    n_tok[dup[drop]] = np.maximum(8, n_tok[dup[drop]] - 1)
    import random as _random

    prng = _random.Random(seed)
    S = len(SYL)
    names = [(SYL[a // S] + SYL[a % S] + " " + SYL[b // (S * S)] + SYL[(b // S) % S] + SYL[b % S]).encode()
             for a, b in zip(first.tolist(), last.tolist())]
    for j in dup[rng.random(len(dup)) < 0.5]:
        names[j] = _perturb(prng, names[j], 1)
    t_off, t_ids = _csr_from_padded(addr, n_tok, sort_rows=True)
    enc = Encoded(n)
    enc.add(("codes", "block"), Column(COL_CODES, block))
    enc.add(("chars", "name"), _chars_column(names))
    enc.add(("tokens", "addr"), Column(COL_TOKENS, t_ids.astype(np.int32), t_off, np.zeros(n, np.uint8)))
    # blocks: group tuple ids by block key and source
    order = np.lexsort((np.arange(n) >= half, block))
    bk = block[order]
    starts = np.flatnonzero(np.r_[True, bk[1:] != bk[:-1]])
    ends = np.r_[starts[1:], n]
    blocks = []
    for a, b in zip(starts, ends):
        ids = order[a:b].astype(np.int32)
        nl = int((ids < half).sum())  # lexsort put the A side first: left = ids[:nl]
        if nl and nl < len(ids):
            blocks.append((ids, nl))
    import json

    rules = parse_ruleset(json.dumps(LINKAGE_RULES))
    path = data_aware_plan(enc, rules, sample=plan_sample, seed=seed)
    return Workload("linkage", enc, rules, path, n, blocks=blocks, injected=(src, dup), block_attr="block")


PERSON5_RULES = [
    {"id": "R1", "when": [
        {"t_attr": "last", "op": "eq", "s_attr": "last"},
        {"t_attr": "dob", "op": "eq", "s_attr": "dob"},
        {"t_attr": "first", "op": "sim", "s_attr": "first", "measure": "edit", "threshold": 0.8}]},
    {"id": "R2", "when": [
        {"t_attr": "zip", "op": "eq", "s_attr": "zip"},
        {"t_attr": "address", "op": "sim", "s_attr": "address", "measure": "jaccard", "threshold": 0.7}]},
    {"id": "R3", "when": [
        {"t_attr": "phone", "op": "eq", "s_attr": "phone"}]},
    {"id": "R4", "when": [
        {"t_attr": "first", "op": "eq", "s_attr": "first"},
        {"t_attr": "zip", "op": "eq", "s_attr": "zip"},
        {"t_attr": "last", "op": "sim", "s_attr": "last", "measure": "edit", "threshold": 0.85}]},
    {"id": "R5", "when": [
        {"t_attr": "dob", "op": "eq", "s_attr": "dob"},
        {"t_attr": "address", "op": "sim", "s_attr": "address", "measure": "jaccard", "threshold": 0.6},
        {"t_attr": "first", "op": "sim", "s_attr": "first", "measure": "edit", "threshold": 0.7}]},
]


def person5(n: int = 10_000_000, seed: int = 4, plan_sample: int = 100_000) -> Workload:
    """BASELINE config 4: a person-style relation -- zip (100k, Zipf), last
    name (50k, Zipf), first name (5k), date of birth, phone (90% unique),
    address (8-14 tokens) -- with five rules mixing equality roots with edit
    and Jaccard tails, planned data-aware from sampled selectivities
    (SURVEY §8d config 4).  20% of tuples are perturbed duplicates."""
    rng = np.random.default_rng(seed)

    def zipf(k, size, a=1.1):
        p = 1.0 / np.arange(1, k + 1) ** a
        return rng.choice(k, size=size, p=p / p.sum()).astype(np.int32)

    zipc = zipf(100_000, n)
    last_id = zipf(50_000, n)
    first_id = rng.integers(0, 5_000, size=n)
    dob = rng.integers(0, 30_000, size=n).astype(np.int32)
    phone = rng.integers(0, 1 << 30, size=n).astype(np.int32)
    shared = rng.random(n) < 0.1  # 10% of phones come from a small shared pool
    phone[shared] = rng.integers(0, 1000, size=int(shared.sum()), dtype=np.int32)
    n_tok = rng.integers(8, 15, size=n)
    addr = _distinct_rows(rng, n, 14, 200_000)
    dup = np.flatnonzero(rng.random(n) < 0.2)
    src = rng.integers(0, n, size=len(dup))
    for arr in (zipc, last_id, first_id, dob, phone, n_tok):
        arr[dup] = arr[src]
    addr[dup] = addr[src]
    import random as _random

    prng = _random.Random(seed)
    S = len(SYL)

    def name_of(k, parts):
        out = []
        for _ in range(parts):
            out.append(SYL[k % S])
            k //= S
        return "".join(out).encode()

    # names from per-id tables (each distinct id spelled once), then the
    # perturbed first names; codes = rank among the sorted distinct strings
    # (np.unique's inverse), computed per table entry
    def spelled(ids, parts, mul=1, add=0):
        uniq, inv = np.unique(ids, return_inverse=True)
        table = np.array([name_of(int(k) * mul + add, parts) for k in uniq], dtype=object)
        return table, inv

    f_table, f_inv = spelled(first_id, 3)
    l_table, l_inv = spelled(last_id, 4, 7919, 13)
    firsts = f_table[f_inv].tolist()
    lasts = l_table[l_inv].tolist()
    pert = dup[rng.random(len(dup)) < 0.5]
    for j in pert:
        firsts[j] = _perturb(prng, firsts[j], 1)

    def codes_of(table, inv, extra_idx, strs):
        distinct = sorted(set(table.tolist()) | {strs[j] for j in extra_idx})
        rank = {x: i for i, x in enumerate(distinct)}
        codes = np.array([rank[x] for x in table.tolist()], dtype=np.int32)[inv]
        for j in extra_idx:
            codes[j] = rank[strs[j]]
        return codes

    first_codes = codes_of(f_table, f_inv, pert, firsts)
    last_codes = codes_of(l_table, l_inv, [], lasts)
    t_off, t_ids = _csr_from_padded(addr, n_tok, sort_rows=True)
    enc = Encoded(n)
    enc.add(("codes", "zip"), Column(COL_CODES, zipc))
    enc.add(("codes", "last"), Column(COL_CODES, last_codes))
    enc.add(("codes", "first"), Column(COL_CODES, first_codes))
    enc.add(("codes", "dob"), Column(COL_CODES, dob))
    enc.add(("codes", "phone"), Column(COL_CODES, phone))
    enc.add(("chars", "first"), _chars_column(firsts))
    enc.add(("chars", "last"), _chars_column(lasts))
    enc.add(("tokens", "address"), Column(COL_TOKENS, t_ids.astype(np.int32), t_off, np.zeros(n, np.uint8)))
    import json

    rules = parse_ruleset(json.dumps(PERSON5_RULES))
    path = data_aware_plan(enc, rules, sample=plan_sample, seed=seed)
    return Workload("person5", enc, rules, path, n, injected=(src, dup))


def citation3_parts(n: int = 1_000_000, seed: int = 2024, part: int = 512) -> Workload:
    """Config 2's relation cut into the reference pipeline's default
    partition size (max_partition_size = 512, pipeline.py:74): many small
    partitions evaluated in one batched launch."""
    w = citation3(n, seed)
    perm = np.random.default_rng(seed + 1).permutation(n).astype(np.int32)
    w.blocks = [(perm[a:a + part], -1) for a in range(0, n, part)]
    w.name = "citation3_parts"
    return w


def plan_partitions(enc: Encoded, path, max_partition_size: int = 65536, slots: list = None) -> list:
    """The reference pipeline's partitions and sibling pulls for a plan whose
    root edges are all same-attribute equalities (iter_partitions,
    partitioning.py:93-131; sibling_pull_pairs, 144-157), from the encoded
    code columns: one branch per root edge, one partition per distinct key
    (tids ascending; missing values form their own key group, as the
    reference's MISSING_KEY), a group above ``max_partition_size`` dealt
    round-robin into ceil(|g| / max) siblings, and every sibling pair pulled
    as a cross block.  Returns [(refs int32, split)] with split = -1 for a
    partition and |left| for a pull; single-tuple partitions (no pairs) are
    dropped as pipeline_run drops them in symmetric mode.  ``slots``: when
    given a list, receives each block's root slot (the equality its key
    implies for all its pairs; -1 for the missing-value group)."""
    from .pipeline import root_predicates

    blocks = []
    for b, pred in enumerate(root_predicates(path)):
        if pred.comparator != "eq" or pred.is_cross_attr:
            raise ValueError(f"plan_partitions handles equality roots only, not {pred.describe()}")
        codes = enc.columns[enc.get(("codes", pred.lhs_attr))].data
        order = np.argsort(codes, kind="stable").astype(np.int32)  # tids ascending inside each key
        sc = codes[order]
        starts = np.flatnonzero(np.r_[True, sc[1:] != sc[:-1]])
        sizes = np.diff(np.r_[starts, len(sc)])
        for a, m in zip(starts[sizes > 1].tolist(), sizes[sizes > 1].tolist()):  # single tuples: no pairs
            g = order[a:a + m]
            n_before = len(blocks)
            if len(g) <= max_partition_size:
                blocks.append((g, -1))
            else:
                k = -(-len(g) // max_partition_size)
                subs = [g[i::k] for i in range(k)]
                blocks += [(x, -1) for x in subs if len(x) > 1]
                blocks += [(np.concatenate([subs[i], subs[j]]), len(subs[i])) for i in range(k) for j in range(i + 1, k)]
            if slots is not None:
                slot = -1 if sc[a] < 0 else int(path.root_slots[b])
                slots += [slot] * (len(blocks) - n_before)
    return blocks


def person5_parts(n: int = 1_000_000, seed: int = 4, max_partition_size: int = 65536) -> Workload:
    """BASELINE config 4 (i): person5's relation and frozen plan, evaluated
    over the reference pipeline's plan-derived partitions (one branch per
    equality root, max_partition_size = 65536) plus sibling pulls, in one
    batched launch."""
    w = person5(n, seed)
    slots: list = []
    w.blocks = plan_partitions(w.enc, w.path, max_partition_size, slots)
    w.block_implied = [0 if s < 0 else 1 << s for s in slots]  # each block's branch root holds for its pairs
    w.name = "person5_parts"
    return w


def citation_small(n: int = 0, seed: int = 2024) -> Workload:
    """BASELINE config 1: the reference's own small benchmark relation --
    ``citation_benchmark(seed=2024)`` (datasets.py:332-398, 4,591 tuples)
    with its frozen plan, as recorded from the reference in
    tests/golden/citation.json.gz -- one symmetric partition (1.05e7 pairs).
    ``n`` and ``seed`` are fixed by the fixture."""
    import gzip
    import os

    from .encode import RelationEncoding
    from .plan import path_from_dict
    from .relation import relation_from_rows

    here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        "citation.json.gz")
    with gzip.open(here, "rt") as fh:
        doc = json.load(fh)
    r = doc["relation"]
    rel = relation_from_rows(r["names"], r["kinds"], r["rows"])
    path = path_from_dict(doc["path"])
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    return Workload("citation_small", enc, None, path, len(rel))


WORKLOADS = {"citation3": citation3, "edit_heavy": edit_heavy, "linkage": linkage, "person5": person5,
             "citation3_parts": citation3_parts, "citation_small": citation_small,
             "person5_parts": person5_parts}
