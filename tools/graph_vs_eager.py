"""Per-layer time of the bench's c5 step: CUDA-graph replay vs eager launches
(both PDL-attributed; tests whether the graph keeps the programmatic edges).
    python tools/graph_vs_eager.py [layers]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_16210_b200.runtime import DecodeRunner  # noqa: E402
from synth import workloads as W  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
w = W.CONFIGS["c5"]
r = DecodeRunner(w, range(12), "cuda", layers=L)
r.prefill()
r.step(0)
r.capture(timing_slots=())
torch.cuda.synchronize()


def timed(fn, n=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3 / L


print(f"graph replay: {timed(lambda: r.replay(0)):.1f} us/layer")
print(f"eager step:   {timed(lambda: r.step(0)):.1f} us/layer")
