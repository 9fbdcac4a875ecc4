"""Debug: a few decode launches on one synthetic layer (random codes/scales),
for ncu captures of the steady state.  python tools/long_case.py B H hd T [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2505_16210_b200 import nqkv as N  # noqa: E402

B, H, hd, T = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
Tc = -(-T // 64) * 64
cache = N.KVCache(B, H, hd, Tc, 64, "cuda")
cache.k_codes.random_(0, 256)
cache.v_codes.random_(0, 256)
cache.k_scales.uniform_(0.5, 2)
cache.v_scales.uniform_(0.5, 2)
q = torch.randn(B, H, hd, device="cuda").half()
L = torch.full((B,), T, dtype=torch.int32, device="cuda")
ws = N.make_workspace(B, H, hd, Tc, "cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(reps):
    flush.sum()
    cache.attend(q, L, ws)
torch.cuda.synchronize()
print("ok")
