"""Per-launch time of nqkv_decode_attention for tiny and c1-sized problems:
back-to-back launches (no flush) vs. single launches after a GPU sleep.
Development tool: separates fixed launch/prologue cost from streaming."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N  # noqa: E402

dev = "cuda"
CASES = [(1, 1, 64, 64), (1, 12, 64, 513), (8, 32, 64, 2049), (1, 148, 128, 4096)]
if len(sys.argv) > 4:
    CASES = [tuple(int(x) for x in sys.argv[1:5])]
for (B, H, hd, T) in CASES:
    Tc = -(-T // 64) * 64
    cache = N.KVCache(B, H, hd, Tc, 64, dev)
    cache.k_codes.random_(0, 256)
    cache.v_codes.random_(0, 256)
    cache.k_scales.uniform_(0.5, 2)
    cache.v_scales.uniform_(0.5, 2)
    q = torch.randn(B, H, hd, device=dev).half()
    L = torch.full((B,), T, dtype=torch.int32, device=dev)
    ws = N.make_workspace(B, H, hd, Tc, dev)
    out = torch.empty(B, H, hd, device=dev)
    for _ in range(5):
        cache.attend(q, L, ws, out=out)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    n = 200
    torch.cuda._sleep(1000000)
    a.record()
    for _ in range(n):
        cache.attend(q, L, ws, out=out)
    b.record()
    torch.cuda.synchronize()
    loop = a.elapsed_time(b) / n * 1e3
    ts = []
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(20):
        flush.sum()                 # read-only L2 sweep: the single launch streams from HBM
        torch.cuda._sleep(200000)
        a.record()
        cache.attend(q, L, ws, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    mb = cache.nbytes() / 1e6
    print(f"B={B} H={H} hd={hd} T={T} ({mb:.1f} MB): back-to-back {loop:7.2f} us/launch, "
          f"single {ts[len(ts) // 2]:7.2f} us", flush=True)
