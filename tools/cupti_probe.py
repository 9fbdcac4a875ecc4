"""Probe: DRAM bytes of one kernel launch measured in-process through the
CUPTI range profiler that torch.profiler exposes (no ncu)."""
import json
import torch
from torch.profiler import profile, ProfilerActivity, _ExperimentalConfig

x = torch.randn(64 << 20, device="cuda")
y = torch.empty_like(x)
torch.cuda.synchronize()
cfg = _ExperimentalConfig(profiler_metrics=["dram__bytes_read.sum", "dram__bytes_write.sum"],
                          profiler_measure_per_kernel=True)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], experimental_config=cfg) as prof:
    y.add_(x)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tr.json")
t = json.load(open("/tmp/tr.json"))
for ev in t.get("traceEvents", []):
    s = json.dumps(ev)
    if "dram" in s or "kernel" in ev.get("cat", ""):
        print(s[:600])
