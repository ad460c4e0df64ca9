"""List the backward-branch loops of a SASS dump with instruction counts
and an opcode histogram:  python tools/sass_loops.py FILE.sass [min_len]"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 20
funcs, ins = [], None
for l in lines:
    f = re.match(r"\s*Function : (\S+)", l)
    if f:
        ins = []
        funcs.append((f.group(1), ins))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and ins is not None:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
only = sys.argv[3] if len(sys.argv) > 3 else ""
for fname, ins in funcs:
  if only not in fname:
    continue
  addr_idx = {a: k for k, (a, _) in enumerate(ins)}
  for k, (a, txt) in enumerate(ins):
      m = re.search(r"\bBRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", txt)
      if not m:
          continue
      tgt = int(m.group(1), 16)
      if tgt >= a or tgt not in addr_idx:
          continue
      body = ins[addr_idx[tgt]: k + 1]
      if len(body) < minlen:
          continue
      hist = collections.Counter()
      for _, t in body:
          op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
          hist[op.split(".")[0]] += 1
      print(f"{fname[:24]} loop 0x{tgt:x}-0x{a:x}: {len(body)} instrs  " + " ".join(f"{o}:{c}" for o, c in hist.most_common()))
