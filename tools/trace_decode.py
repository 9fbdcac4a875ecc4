"""Debug: per-warp globaltimer trace of the decode kernel.  Builds an
NQKV_TRACE variant of the library to /tmp and loads it via NQKV_LIB.
    python tools/trace_decode.py [B H hd T]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_16210_b200 import build as bld  # noqa: E402

defs = {"NQKV_TRACE": 1}
for kv in os.environ.get("DEFS", "").split(","):
    if kv:
        k, v = kv.split("=")
        defs[k] = v
lib = bld.build_variant("/tmp/libnqkv_trace.so", defs)
os.environ["NQKV_LIB"] = lib
import torch  # noqa: E402

NW = 16
tr = torch.zeros(148 * NW * 16, dtype=torch.int64, device="cuda")
os.environ["NQKV_TRACE_PTR"] = str(tr.data_ptr())
from paper_2505_16210_b200 import nqkv as N  # noqa: E402

B, H, hd, T = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 32, 64, 2049)
Tc = -(-T // 64) * 64
cache = N.KVCache(B, H, hd, Tc, 64, "cuda")
cache.k_codes.random_(0, 256)
cache.v_codes.random_(0, 256)
cache.k_scales.uniform_(0.5, 2)
cache.v_scales.uniform_(0.5, 2)
q = torch.randn(B, H, hd, device="cuda").half()
L = torch.full((B,), T, dtype=torch.int32, device="cuda")
if os.environ.get("RAGGED"):           # lengths uniform in [T // 2, T] (BASELINE c3's recipe at T = 2049)
    L = torch.randint(T // 2, T + 1, (B,), generator=torch.Generator().manual_seed(0),
                      dtype=torch.int64).to(torch.int32).cuda()
ws = N.make_workspace(B, H, hd, Tc, "cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
warm = os.environ.get("WARM") == "1"    # trace the 2nd of two back-to-back launches (no flush between)
planned = os.environ.get("PLAN") == "1"
plan = N.make_plan("cuda")
fused = os.environ.get("FUSED") == "1"   # fused append + attend (the runtime's step), planned
N.nqkv_decode_plan(L, H, Tc, fused, plan, hd=hd)
if fused:
    kn = torch.randn(B, H, hd, device="cuda").half()
    vn = torch.randn(B, H, hd, device="cuda").half()
    cache.attend = lambda q_, L_, ws_: cache.step_planned(kn, vn, q_, L_, ws_, plan)
elif planned:
    cache.attend = lambda q_, L_, ws_: cache.attend_planned(q_, L_, ws_, plan)
for _ in range(5):
    flush.sum()                         # read-only L2 sweep (no dirty lines): HBM-honest timing
    torch.cuda._sleep(100000)
    if warm:
        cache.attend(q, L, ws)
    torch.cuda.synchronize()
    tr.zero_()
    torch.cuda._sleep(20000)
    cache.attend(q, L, ws)
    torch.cuda.synchronize()
t = tr.view(148, NW, 16).cpu()
t0 = t[:, :, 0][t[:, :, 0] > 0].min()
names = ["entry", "pdl_wait", "prefix", "prod: start", "loads issued", "V LUT", "table0", "sync", "full0", "loop end", "exit", "prod: last done", "last odd step", "g0/g1", ""]
# producer phase sums (ns) in slots 4, 5, 13, 15 of the producer warp
pw = t[:, NW - 1, :].double()
for k, n in ((4, "waits on consumers"), (5, "merges"), (13, "table builds"), (15, "appended tokens")):
    col = pw[:, k] / 1000.0
    print(f"producer sum {n:20s} med {col.median():7.2f} max {col.max():7.2f} us")
for role, sl in (("consumer", slice(0, NW - 1)), ("producer", slice(NW - 1, NW))):
    x = t[:, sl, :].reshape(-1, 16)
    x = x[x[:, 0] > 0]
    for k, n in enumerate(names):
        if not n or (role == "producer" and k in (4, 5, 13, 15)):
            continue
        col = x[:, k]
        col = col[col > 0]
        if len(col):
            r = (col - t0).double() / 1000.0
            print(f"{role:9s} {n:11s} min {r.min():8.2f} med {r.median():8.2f} max {r.max():8.2f} us (n={len(col)})")
w = t[:, :NW - 1, 15]
w = w[w > 0].double() / 1000.0
print(f"consumer wait on full barriers: med {w.median():.2f} max {w.max():.2f} us per warp")

# per-CTA: slowest consumer loop end vs number of pieces in the CTA's range
import numpy as np  # noqa: E402
lens_h = L.cpu().tolist()
N = B * H * T
C = min(148, max(1, -(-N // 512)))
pref = np.cumsum([0] + [H * n for n in lens_h])
ends = (t[:, :NW - 1, 9].double() - t0.double()) / 1000.0
rows = []
for c in range(C):
    g0, g1 = c * N // C, (c + 1) * N // C
    starts = [int(pref[b] + h * lens_h[b]) for b in range(B) for h in range(H)]
    inner = sum(1 for s0 in starts if g0 < s0 < g1)
    e = ends[c][ends[c] > 0]
    rows.append((inner + 1, float(e.max()) if len(e) else 0.0, float(e.min()) if len(e) else 0.0))
for npc in sorted(set(r[0] for r in rows)):
    sel = [r for r in rows if r[0] == npc]
    print(f"pieces={npc}: CTAs {len(sel)} loop-end max med {np.median([r[1] for r in sel]):.2f} "
          f"min-warp med {np.median([r[2] for r in sel]):.2f} us")
order = sorted(rows, key=lambda r: r[1])
print("fastest CTAs", [(r[0], round(r[1], 1)) for r in order[:5]], "slowest", [(r[0], round(r[1], 1)) for r in order[-5:]])

# per-CTA streaming time vs SM id (stamp 14 of warp 0 = smid + 1)
sm = t[:, 0, 14].long() - 1
f0 = (t[:, :NW - 1, 8].double() - t0.double()) / 1000.0
dur = [float(ends[c][ends[c] > 0].max() - f0[c][f0[c] > 0].min()) for c in range(C)]
rows2 = sorted(((int(sm[c]), dur[c], rows[c][0]) for c in range(C)), key=lambda r: r[0])
print("smid:dur(us):pieces  " + " ".join(f"{a}:{b:.1f}:{c}" for a, b, c in rows2))
tpc = {}
for a, b, c in rows2:
    tpc.setdefault(a // 2, []).append(b)
import statistics as st_  # noqa: E402
print("slowest SMs", sorted(rows2, key=lambda r: -r[1])[:12])
print("fastest SMs", sorted(rows2, key=lambda r: r[1])[:12])
# per-warp-index medians of (loop end - full0): SM sub-partition (warp % 4) balance
le = (t[:, :NW - 1, 9].double() - t0.double()) / 1000.0
f0w = (t[:, :NW - 1, 8].double() - t0.double()) / 1000.0
dd = le - f0w
print("warp: median stream time (us) " + " ".join(f"{w}:{float(dd[:, w].median()):.2f}" for w in range(NW - 1)))
