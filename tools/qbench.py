"""Development: bulk-quantize timing (L2 flushed) for a few shapes, one
line per shape.  NQKV_LIB selects a library variant."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("NQKV_LIB"):
    import __graft_entry__
    __graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for (B, T, H, hd) in [(8, 2048, 32, 64), (32, 1988, 32, 128), (4, 8192, 40, 128), (64, 4096, 12, 128)]:
    x = torch.randn(B, T, H, hd, device="cuda").half()
    Tc = -(-(T + 1) // 64) * 64
    codes = torch.zeros(B, H, Tc, hd // 2, dtype=torch.uint8, device="cuda")
    scales = torch.zeros(B, H, Tc, hd // 64, dtype=torch.float32, device="cuda")
    z = torch.zeros(B, dtype=torch.int32, device="cuda")
    ts = []
    for i in range(12):
        flush.sum()                 # read-only L2 sweep: evicts without leaving dirty lines
        torch.cuda._sleep(100000)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        N.nqkv_quantize(x, z, codes, scales, 64)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    t = ts[len(ts) // 2]
    nb = x.numel() * (2 + 0.5 + 4 / 64)
    print(f"B={B} T={T} H={H} hd={hd}: {t * 1e3:8.1f} us {nb / t / 1e6:7.0f} GB/s", flush=True)
    if hasattr(N, "nqkv_quantize_pair"):        # K and V in one launch
        y = torch.randn_like(x)
        codes2, scales2 = torch.zeros_like(codes), torch.zeros_like(scales)
        ts = []
        for i in range(12):
            flush.sum()
            torch.cuda._sleep(100000)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            N.nqkv_quantize_pair(x, y, z, codes, scales, codes2, scales2, 64)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        t = ts[len(ts) // 2]
        print(f"   pair (K+V): {t * 1e3:8.1f} us {2 * nb / t / 1e6:7.0f} GB/s", flush=True)
        del y, codes2, scales2
    del x, codes, scales
