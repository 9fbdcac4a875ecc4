"""Prefill attention timing (development tool): c3/c4-shaped prompts, FLOP
roofline (algorithmic causal FLOPs, 2*hd*len*(len+1) per (b, h): the hi/lo
splits' extra tensor work is not counted) against MEASURED_PEAKS bf16."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N  # noqa: E402
from synth import workloads as W  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
for name, H in (("c3", 32), ("c4", 40)):
    w = W.CONFIGS[name]
    lens = W.seq_lens(w)
    B, hd, T = w.batch, w.head_dim, int(lens.max())
    Tc = W.capacity(T)
    cache = N.KVCache(B, H, hd, Tc, w.blk, "cuda")
    K, V = W.layer_kv(w, 0, heads=range(H), tokens=T, device="cuda")
    cache.append(K, V, torch.zeros(B, dtype=torch.int32, device="cuda"))
    del K, V
    q = torch.randn(B, T, H, hd, device="cuda").half()
    L = lens.to("cuda")
    out = torch.empty(B, T, H, hd, device="cuda")
    for _ in range(3):
        N.nqkv_prefill_attention(q, cache.k_codes, cache.k_scales, cache.v_codes, cache.v_scales, L, w.blk, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 5
    for _ in range(n):
        N.nqkv_prefill_attention(q, cache.k_codes, cache.k_scales, cache.v_codes, cache.v_scales, L, w.blk, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    flop = sum(2.0 * hd * int(x) * (int(x) + 1) for x in lens.tolist()) * H
    tf = flop / (ms * 1e-3) / 1e12
    print(json.dumps({"config": name, "B": B, "H": H, "T": T, "ms": ms, "tflops": tf,
                      "frac_of_bf16_peak": tf / peak, "peak_tflops": peak}), flush=True)
    del cache, q, out
    torch.cuda.empty_cache()
