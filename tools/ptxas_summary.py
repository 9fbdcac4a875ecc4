"""Registers and spills per kernel from ptxas -v output (build.py writes
paper_2505_16210_b200/ptxas_info.txt).  python tools/ptxas_summary.py [file] [filter]"""
import re
import sys

txt = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2505_16210_b200/ptxas_info.txt").read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
info = {}
for line in txt.splitlines():
    m = re.search(r"(?:Compiling entry function|Function properties for) '?([_A-Za-z0-9]+)", line)
    if m:
        cur = m.group(1)
        info.setdefault(cur, {})
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        info[cur]["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        info[cur]["regs"] = int(m.group(1))
for k, v in info.items():
    if flt in k:
        d = re.sub(r"_ZN4nqkv\d+", "", k)
        d = re.sub(r"EEEvNS_\w+", "", d)
        print(f"{d[:70]:70s} regs={v.get('regs')} spill={v.get('spill')}")
