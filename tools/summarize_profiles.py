"""Summarise a round's ncu artefacts (gpurun_out/<round>_*) into profiles/.

    python tools/summarize_profiles.py r1 [workload-name]
"""
import csv
import json
import os
import statistics
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r1"
WL = sys.argv[2] if len(sys.argv) > 2 else "c2-opt1.3b"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)


def launches():
    path = os.path.join(G, f"{R}_launches.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    d = defaultdict(list)
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        d[name].append(float(r[idx["Metric Value"]]) / 1000.0)
    total = sum(sum(v) for v in d.values())
    out = [f"# ncu launch list ({R}): python bench.py --steps 4 --warmup 3 --no-cpu-baseline",
           "# --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)",
           f"{'kernel':45s} {'launches':>8s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:45s} {len(v):8d} {statistics.mean(v):9.2f} {sum(v):10.1f} {100*sum(v)/total:5.1f}%")
    txt = "\n".join(out) + "\n"
    open(os.path.join(P, f"{R}_launches_summary.txt"), "w").write(txt)
    print(txt)


KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "SM Active Cycles", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "Registers Per Thread", "Achieved Occupancy", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Mem Busy", "Max Bandwidth")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed.sum",
       "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active")


def page(tag, name, args):
    """An ncu page as csv text: from the report if it is here, else from the
    csv that tools/profile_shrink.sh wrote on the GPU box."""
    rep = os.path.join(G, f"{R}_{tag}.ncu-rep")
    if os.path.exists(rep):
        return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
    return open(os.path.join(G, f"{R}_{tag}_{name}.csv"), encoding="latin-1").read()


def ncu_report(tag):
    det = page(tag, "details", ["--page", "details", "--csv"])
    rows = list(csv.reader(det.splitlines()))
    hdr = rows[0]
    lines = [f"# ncu --set full ({R}, {tag}): " + rows[1][hdr.index("Kernel Name")][:90]]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            lines.append(f"{d['Section Name'][:34]:34s} {d['Metric Name']:34s} {d['Metric Value']:>14s} {d['Metric Unit']}")
    raw = page(tag, "raw", ["--page", "raw", "--csv"])
    rr = list(csv.reader(raw.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]
    vals = {}
    for name, unit, val in zip(h, u, v):
        if name in RAW:
            lines.append(f"{'raw':34s} {name:70s} {val:>14s} {unit}")
            vals[name] = (val, unit)
    src = page(tag, "sass", ["--page", "source", "--csv", "--print-source", "sass"])
    tmp = os.path.join(G, f"{R}_{tag}_sass.csv")
    open(tmp, "w", encoding="latin-1").write(src)
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass_hot.py"), tmp, "12"],
                         capture_output=True, text=True).stdout
    txt = "\n".join(lines) + "\n\n# warp-stall sampling (top SASS)\n" + hot
    open(os.path.join(P, f"{R}_{tag}_ncu.txt"), "w").write(txt)
    print(txt[:3000])
    return vals


launches()
dv = ncu_report("decode")
qv = ncu_report("quantize")
if os.path.exists(os.path.join(G, f"{R}_prefill_details.csv")) or os.path.exists(os.path.join(G, f"{R}_prefill.ncu-rep")):
    ncu_report("prefill")


def to_bytes(val, unit):
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


tr = {}
tp = os.path.join(P, "traffic.json")
if os.path.exists(tp):
    tr = json.load(open(tp))
rd = to_bytes(*dv["dram__bytes_read.sum"])
wr = to_bytes(*dv["dram__bytes_write.sum"])
tr[WL] = {"decode_dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "source": f"profiles/{R}_decode_ncu.txt"}
if "dram__bytes_read.sum" in qv:
    tr[WL]["quantize_dram_bytes_per_launch"] = to_bytes(*qv["dram__bytes_read.sum"]) + to_bytes(*qv["dram__bytes_write.sum"])
    tr[WL]["quantize_source"] = f"profiles/{R}_quantize_ncu.txt"
json.dump(tr, open(tp, "w"), indent=1)
print(tr)
