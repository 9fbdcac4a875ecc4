"""Opcode histogram of the hottest loop of one kernel in a cubin/so/binary.
    python tools/sass_loop.py <binary> <function-substring> [loop-index]
Loops are backward branches; the body is [target, branch].  Lists loops by size."""
import re
import subprocess
import sys
from collections import Counter

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
pat = sys.argv[2]
body = None
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat in name:
        body = f
        print("function", name)
        break
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a:
            j = next(k for k, (b, _) in enumerate(ins) if b == tgt)
            loops.append((i - j + 1, j, i))
loops.sort(reverse=True)
for n, j, i in loops[:6]:
    print(f"loop {ins[j][0]:#x}-{ins[i][0]:#x}: {n} instructions")
sel = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n, j, i = loops[sel]
c = Counter()
for _, t in ins[j:i + 1]:
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    c[t.split()[0]] += 1
for k, v in c.most_common(40):
    print(f"{v:6d} {k}")
