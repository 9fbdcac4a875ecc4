"""Summarise an ncu '--page source --print-source sass --csv' dump: top
instructions by warp-stall samples and the stall-reason totals.
    ncu -i rep --page source --csv --print-source sass > x.csv; python ncu_sass_hot.py x.csv [N]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot = Counter()


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for d in data:
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            tot[k] += f(d[k])
S = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
print("total samples", S)
for k, v in tot.most_common(12):
    print(f"  {k:28s} {v:10.0f} {100*v/max(S,1):5.1f}%")
top = sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for d in top:
    s = f(d["Warp Stall Sampling (All Samples)"])
    reasons = sorted(((f(d[k]), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
    print(f"{d['Address']:>6} {100*s/max(S,1):5.1f}% {d['Source'][:60]:60s} " + " ".join(f"{k}={v:.0f}" for v, k in reasons if v))
