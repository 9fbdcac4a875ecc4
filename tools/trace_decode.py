"""Debug: per-warp globaltimer trace of the decode kernel (NQKV_TRACE build)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
tr = torch.zeros(148 * 32 * 8, dtype=torch.int64, device="cuda")
os.environ["NQKV_TRACE_PTR"] = str(tr.data_ptr())
from paper_2505_16210_b200 import nqkv as N  # noqa: E402

w = W.CONFIGS[cfg]
H = 12 if cfg == "c5" else w.heads
lens = W.seq_lens(w)
T = int(lens.max())
Tc = W.capacity(T + 1)
K, V = W.layer_kv(w, 0, heads=range(H), tokens=T, device="cuda")
cache = N.KVCache(w.batch, H, w.head_dim, Tc, w.blk, "cuda")
z = torch.zeros(w.batch, dtype=torch.int32, device="cuda")
cache.append(K, V, z)
_, _, q = W.step_inputs(w, 0, 0, heads=range(H), device="cuda")
L = (lens + 1).to("cuda")
ws = N.make_workspace(w.batch, H, w.head_dim, Tc, "cuda")
for _ in range(3):
    tr.zero_()
    cache.attend(q, L, ws)
    torch.cuda.synchronize()
t = tr.view(-1, 8).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0).double() / 1000.0
names = ["entry", "lut+sync", "pdl_wait", "prefix", "primed", "1st stage", "exit"]
for k, n in enumerate(names):
    col = rel[:, k]
    col = col[t[:, k] > 0]
    if len(col):
        print(f"{n:10s} min {col.min():8.2f} med {col.median():8.2f} max {col.max():8.2f} us (n={len(col)})")
