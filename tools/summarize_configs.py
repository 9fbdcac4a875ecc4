"""Summarise tools/profile_configs.sh captures into profiles/<round>_configs_ncu.txt:
per config and kernel, duration, DRAM bytes and throughput, L1 data-pipe and
issue utilisation.   python tools/summarize_configs.py r1f"""
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r1f"
G = os.path.join(ROOT, "gpurun_out")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active"]
lines = [f"# ncu --set full ({R}): one launch per kernel and config (tools/profile_configs.sh);"
         " cold L2, serialised"]
lines.append(f"{'config':7s} {'kernel':16s} {'us':>8s} {'DRAM rd MB':>11s} {'DRAM wr MB':>11s} "
             f"{'GB/s':>7s} {'rd%pk':>6s} {'L1pipe%':>8s} {'issue%':>7s} {'elig/sched':>10s}")
for c in ("c3", "c4", "c5"):
    for k, name in (("attend", "decode_kernel"), ("quantize", "quantize_kernel")):
        rep = os.path.join(G, f"{R}_{c}_{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        hdr, units, val = rows[0], rows[1], rows[-1]
        d = {}
        for key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                v = float(val[i].replace(",", ""))
                u = units[i]
                if u == "nsecond":
                    v /= 1e3
                elif u == "usecond":
                    pass
                elif u == "msecond":
                    v *= 1e3
                elif u == "Kbyte":
                    v /= 1e3
                elif u == "Gbyte":
                    v *= 1e3
                elif u == "byte":
                    v /= 1e6
                d[key] = v
        us = d.get("gpu__time_duration.sum", float("nan"))
        rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        lines.append(f"{c:7s} {name:16s} {us:8.1f} {rd:11.1f} {wr:11.1f} {(rd + wr) / us * 1e3:7.0f} "
                     f"{d.get(KEYS[3], 0):6.1f} {d.get(KEYS[4], 0):8.1f} {d.get(KEYS[5], 0):7.1f} "
                     f"{d.get(KEYS[6], 0):10.2f}")
open(os.path.join(ROOT, "profiles", f"{R}_configs_ncu.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
