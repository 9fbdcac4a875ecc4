"""Debug: globaltimer trace of L back-to-back fused decode steps (one per
layer, PDL-chained, planned, as the runtime issues them) to see where a
layer's time goes: launch gap, prologue, streaming, tail.
    python tools/trace_chain.py [B H hd T L]      (env DEFS=K=V,... as trace_decode.py)"""
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
if os.environ.get("NOTRACE") != "1":      # NOTRACE=1: time the in-tree build (no stamps)
    os.environ["NQKV_LIB"] = bld.build_variant("/tmp/libnqkv_trace.so", defs)
import torch  # noqa: E402
from paper_2505_16210_b200 import nqkv as N  # noqa: E402

NW = 16
EARLY = os.environ.get("EARLY", "1") == "1"
B, H, hd, T, L = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (8, 32, 64, 2048, 8)
Tc = -(-(T + 16) // 64) * 64
caches = []
for _ in range(L):
    c = N.KVCache(B, H, hd, Tc, int(os.environ.get("BLK", "64")), "cuda")
    c.k_codes.random_(0, 256)
    c.v_codes.random_(0, 256)
    c.k_scales.uniform_(0.5, 2)
    c.v_scales.uniform_(0.5, 2)
    caches.append(c)
q = torch.randn(L, B, H, hd, device="cuda").half()
kn = torch.randn(L, B, H, hd, device="cuda").half()
vn = torch.randn(L, B, H, hd, device="cuda").half()
out = torch.empty(L, B, H, hd, device="cuda", dtype=torch.float32)
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
ws = N.make_workspace(B, H, hd, Tc, "cuda")
plan = N.make_plan("cuda")
tr = torch.zeros(L, 148 * NW * 16, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def chain(traced):
    N.nqkv_decode_plan(lens, H, Tc, True, plan, hd=hd)
    for i in range(L):
        os.environ["NQKV_TRACE_PTR"] = str(tr[i].data_ptr() if traced else 0)
        kw = {"flags": N.EARLY_START if i > 0 and EARLY else 0} if hasattr(N, "EARLY_START") else {}
        caches[i].step_planned(kn[i], vn[i], q[i], lens, ws, plan, out=out[i], **kw)


for it in range(0 if os.environ.get("NOTRACE") == "1" else 4):
    flush.sum()
    torch.cuda.synchronize()
    tr.zero_()
    torch.cuda._sleep(2000000)          # queue the whole chain behind a sleep
    chain(it > 0)
    torch.cuda.synchronize()
if os.environ.get("GRAPH") == "1":           # the same chain captured in a CUDA graph (as bench.py)
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    with torch.cuda.stream(s_):
        with torch.cuda.graph(g, stream=s_):
            chain(False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.sum()
        torch.cuda._sleep(200000)
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        g.replay()
        b_.record()
        torch.cuda.synchronize()
        ts.append(a_.elapsed_time(b_))
    ts.sort()
    print(f"graph chain: {ts[len(ts) // 2] * 1e3 / L:.2f} us per layer (incl. plan), min {ts[0] * 1e3 / L:.2f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
flush.sum()
torch.cuda._sleep(2000000)
e0.record()
chain(False)
e1.record()
torch.cuda.synchronize()
print(f"untraced chain: {e0.elapsed_time(e1) * 1e3 / L:.2f} us per layer (incl. plan)")

if os.environ.get("NOTRACE") == "1":
    sys.exit(0)
t = tr.view(L, 148, NW, 16).cpu().double()
t0 = t[0, :, :, 0][t[0, :, :, 0] > 0].min()
t = torch.where(t > 0, (t - t0) / 1000.0, torch.full_like(t, float("nan")))
prev_exit = None
print("layer  first-entry  med-entry  med-wait  med-full0  med-loopend  max-loopend  med-exit  last-exit  gap")
for i in range(L):
    x = t[i]
    cons = x[:, :NW - 1, :]

    def st(v, f):
        v = v[~torch.isnan(v)]
        return float(f(v)) if len(v) else float("nan")
    fe = st(x[:, :, 0], torch.min)
    row = [fe, st(x[:, :, 0], torch.median), st(x[:, :, 1], torch.median), st(cons[:, :, 8], torch.median),
           st(cons[:, :, 9], torch.median), st(cons[:, :, 9], torch.max), st(x[:, :, 10], torch.median),
           st(x[:, :, 10], torch.max)]
    gap = fe - prev_exit if prev_exit is not None else float("nan")
    prev_exit = row[-1]
    print(f"{i:5d} " + " ".join(f"{v:10.2f}" for v in row) + f" {gap:6.2f}")

# detail for one steady-state layer: per-role medians of every stamp, and the slowest CTA
names = ["entry", "pdl_wait", "prefix", "walk", "loads issued", "V LUT", "table0", "sync", "full0",
         "loop end", "exit", "prod: last done", "last odd step|merge in", "g0/g1", "smid|merge comb"]
i = min(3, L - 1)
x = t[i] - t[i, :, :, 0][~torch.isnan(t[i, :, :, 0])].min()
for role, sl in (("consumer", slice(0, NW - 1)), ("producer", slice(NW - 1, NW))):
    for k, n in enumerate(names):
        v = x[:, sl, k].reshape(-1)
        v = v[~torch.isnan(v)]
        if len(v):
            print(f"L{i} {role:9s} {n:15s} min {v.min():7.2f} med {v.median():7.2f} max {v.max():7.2f}")
ex = x[:, :, 10]
ex = torch.where(torch.isnan(ex), torch.full_like(ex, -1), ex)
cta = int(ex.max(dim=1).values.argmax())
print("slowest CTA", cta)
for w in (0, 7, NW - 2, NW - 1):
    print(f" warp {w:2d}: " + " ".join(f"{n}={x[cta, w, k]:.2f}" for k, n in enumerate(names)
                                    if not torch.isnan(x[cta, w, k])))
le = x[:, :NW - 1, 9]
print("per-CTA max loop end sorted (last 8):", [round(float(v), 2) for v in le.max(dim=1).values.sort().values[-8:]])
print("per-CTA min loop end sorted (first 8):", [round(float(v), 2) for v in le.max(dim=1).values.sort().values[:8]])
