"""Development: build decode-kernel tuning variants (compile-time defines) and
time each with tools/latency_probe.py in a fresh process.
    python tools/sweep_variants.py "NQKV_DECODE_WARPS=16" "NQKV_DECODE_WARPS=12,NQKV_TPS=2" ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_16210_b200 import build as bld  # noqa: E402

cases = os.environ.get("CASES", "8 32 64 2049;1 148 128 4096;32 32 128 1537").split(";")
for spec in sys.argv[1:]:
    defs = dict(kv.split("=") for kv in spec.split(",")) if spec else {}
    out = "/tmp/libnqkv_" + "_".join(f"{k}{v}" for k, v in defs.items()) + ".so"
    bld.build_variant(out, defs)
    env = dict(os.environ, NQKV_LIB=out)
    for c in cases:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "latency_probe.py")] + c.split(),
                           capture_output=True, text=True, env=env, timeout=120)
        print(f"{spec:40s} {r.stdout.strip()} {r.stderr.strip()[-200:] if r.returncode else ''}", flush=True)
