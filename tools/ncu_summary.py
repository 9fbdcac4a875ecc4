"""Print the key sections of an ncu report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
keep = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Launch Statistics",
        "Warp State Statistics", "Compute Workload Analysis", "Scheduler Statistics")
skip = ("Cluster", "Block Limit", "TPC", "Green", "Stack", "Function Cache", "Driver Shared")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Section Name") in keep and d.get("Metric Name") and not any(k in d["Metric Name"] for k in skip):
        print(f"{d['Kernel Name'][:28]:28s} | {d['Section Name'][:18]:18s} | {d['Metric Name']:40s} | {d['Metric Value']} {d['Metric Unit']}")
