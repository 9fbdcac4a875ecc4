"""Cost of the fused all-gather epilogue on one GPU (one NCCL rank): c2 decode
steps through DecodeRunner(fused_gather=True) -- gather launches, epoch bump,
flag wait -- against the plain fused runtime, both as replayed step graphs.
    python tools/gather_overhead.py [steps]"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2505_16210_b200.runtime import DecodeRunner  # noqa: E402
from synth import workloads as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
s_ = socket.socket()
s_.bind(("127.0.0.1", 0))
port = s_.getsockname()[1]
s_.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
w = W.CONFIGS["c2"]
runs = {}
for name, fg in (("plain", False), ("fused_gather", True)):
    r = DecodeRunner(w, range(w.heads), "cuda", group=dist.group.WORLD, world=1, fused_gather=fg)
    r.prefill()
    r.capture(timing_slots=())
    runs[name] = r
for rep in range(2):
    for name, r in runs.items():
        for i in range(5):
            r.replay(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            r.replay(i)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:13s} {e0.elapsed_time(e1) / steps * 1e3:8.1f} us per step "
              f"({r.L} layers)", flush=True)
dist.destroy_process_group()
