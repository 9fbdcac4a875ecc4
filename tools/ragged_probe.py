"""Decode launch time at the c3 shape with ragged (U[1024, 2048], the
BASELINE config) vs equal lengths (1536 = the ragged mean): per-step CUDA
graphs of DecodeRunner, fused (append + attend) or unfused, planned or not.
Development tool."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from synth import workloads as W  # noqa: E402

__graft_entry__.build()
from paper_2505_16210_b200.runtime import DecodeRunner  # noqa: E402

dev = torch.device("cuda", 0)
base = W.CONFIGS["c3"]
works = (("ragged", base), ("equal-1536", dataclasses.replace(base, seq_len=1536, ragged_min=None)))
for fused, planned in ((True, True), (False, True), (False, False)):
    for name, w in works:
        r = DecodeRunner(w, range(w.heads), dev, layers=8, fused=fused, planned=planned)
        r.prefill()
        r.capture(timing_slots=())
        for i in range(5):
            r.replay(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20):
            r.replay(i)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 / r.L * 1e3
        print(f"fused={fused:d} planned={planned:d} {name:11s} {us:7.2f} us/layer ({r.decode_bytes(0) / 1e6:.1f} MB)")
        del r
        torch.cuda.empty_cache()
