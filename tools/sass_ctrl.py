"""Decode SASS control bits (stall, write/read scoreboard, wait mask) for a
kernel's instructions in an address range.
    python tools/sass_ctrl.py <binary> <function-substring> <start_hex> <end_hex>"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
body = next(f for f in funcs[1:] if sys.argv[2] in f.split("\n", 1)[0])
lines = body.split("\n")
lo_a, hi_a = int(sys.argv[3], 16), int(sys.argv[4], 16)
i = 0
while i < len(lines):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", lines[i])
    if m:
        addr = int(m.group(1), 16)
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        hi = int(m2.group(1), 16)
        ctrl = hi >> 41
        stall = ctrl & 0xF
        yld = (ctrl >> 4) & 1
        wr = (ctrl >> 5) & 7
        rd = (ctrl >> 8) & 7
        wait = (ctrl >> 11) & 0x3F
        if lo_a <= addr <= hi_a:
            w = "".join(str(b) for b in range(6) if wait >> b & 1)
            print(f"{addr:06x} s{stall:2d} {'Y' if yld else ' '} wr{wr if wr != 7 else '-'} rd{rd if rd != 7 else '-'} wait[{w:6s}] {m.group(2)[:80]}")
        i += 2
        continue
    i += 1
