"""Instruction mix of one kernel launch from an ncu source-page CSV
(`ncu -i rep --page source --csv --print-source sass`): warp-level executed
instructions per opcode, plus the top instructions by execution count.
    python tools/ncu_opcount.py x.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


seen = set()
ops = Counter()
tot = 0.0
uniq = []
for d in data:
    if d["Address"] in seen:
        continue
    seen.add(d["Address"])
    n = f(d["Instructions Executed"])
    src = d["Source"].strip()
    toks = src.split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    ops[op.split(".")[0]] += n
    tot += n
    uniq.append((n, d["Address"], src))
print(f"total warp instructions {tot:.0f}")
for k, v in ops.most_common(25):
    print(f"  {k:12s} {v:12.0f} {100 * v / tot:5.1f}%")
for n, a, s in sorted(uniq, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 0]:
    print(f"{n:10.0f} {a} {s[:70]}")
