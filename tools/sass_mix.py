"""Executed-instruction mix of an ncu source page (csv from profile_shrink.sh):
    python tools/sass_mix.py gpurun_out/X_sass.csv [units]   (units: divide counts, e.g. stages)"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], encoding="latin-1")))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ops, samp, tot = collections.Counter(), collections.Counter(), 0
stall_cols = [c for c in h if c.startswith("stall_")] if any(c.startswith("stall_") for c in h) else []
for r in rows[2:]:
    if len(r) < len(h) - 5:
        continue
    src = r[idx["Source"]].strip().split()
    if not src:
        continue
    op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
    n = int(r[idx["Instructions Executed"]] or 0)
    ops[op] += n
    tot += n
    samp[op] += int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
print(f"total warp instructions {tot}  per unit {tot / units:.1f}")
for op, n in ops.most_common(22):
    print(f"{op:10s} {n / units:9.1f}  samples {samp[op]}")
