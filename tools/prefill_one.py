import os, sys, torch
sys.path.insert(0, "/root/repo")
import __graft_entry__
__graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N
from synth import workloads as W
w = W.CONFIGS["c4"]; H = 40
lens = W.seq_lens(w); B, hd, T = w.batch, w.head_dim, int(lens.max()); Tc = W.capacity(T)
cache = N.KVCache(B, H, hd, Tc, w.blk, "cuda")
K, V = W.layer_kv(w, 0, heads=range(H), tokens=T, device="cuda")
cache.append(K, V, torch.zeros(B, dtype=torch.int32, device="cuda")); del K, V
q = torch.randn(B, T, H, hd, device="cuda").half(); L = lens.to("cuda")
for _ in range(2):
    N.nqkv_prefill_attention(q, cache.k_codes, cache.k_scales, cache.v_codes, cache.v_scales, L, w.blk)
torch.cuda.synchronize()
