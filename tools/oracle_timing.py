"""Oracle (CPU) timings for BASELINE.md section 4: c1 in full; c2-c5 on a
sample (one layer, one head, the first sequences) scaled linearly to the
full layer (labelled extrapolated).  Host cores / CPU model reported.
    python tools/oracle_timing.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import nqkv_oracle as O  # noqa: E402
from synth import workloads as W  # noqa: E402

import bench  # noqa: E402  (host_cores / cpu model helpers only)


def time_one(w, heads, batch):
    lens = W.seq_lens(w)[:batch].tolist()
    T = int(W.seq_lens(w).max())
    K, V = W.layer_kv(w, 0, heads=range(heads), tokens=T)
    K, V = K[:batch].numpy(), V[:batch].numpy()
    Tc = W.capacity(T + 1)
    kc, ks = O.empty_cache(batch, heads, Tc, w.head_dim, w.blk)
    vc, vs = O.empty_cache(batch, heads, Tc, w.head_dim, w.blk)
    t0 = time.perf_counter()
    O.quantize_append(K, [0] * batch, w.blk, kc, ks)
    tq = time.perf_counter() - t0
    O.quantize_append(V, [0] * batch, w.blk, vc, vs)
    k1, v1, q = W.step_inputs(w, 0, 0, heads=range(heads))
    t0 = time.perf_counter()
    O.quantize_append(k1[:batch].numpy(), lens, w.blk, kc, ks)
    O.quantize_append(v1[:batch].numpy(), lens, w.blk, vc, vs)
    O.decode_attention(q[:batch].numpy(), kc, ks, vc, vs, [n + 1 for n in lens], w.blk)
    td = time.perf_counter() - t0
    elems = K.size
    toks = sum(n + 1 for n in lens)
    return elems / tq, toks / td, elems, toks


rows = {}
for name in ("c1", "c2", "c3", "c4", "c5"):
    w = W.CONFIGS[name]
    if name == "c1":
        heads, batch, how = w.heads, w.batch, "full layer"
    else:
        heads, batch = 1, max(1, min(w.batch, (1 << 22) // ((w.seq_len + 1) * w.head_dim)))
        how = f"1 of {w.heads} heads, {batch} of {w.batch} sequences, one layer; extrapolated"
    qe, dt, _, _ = time_one(w, heads, batch)
    # per-second rates scale linearly: a KV token of the full model = all heads
    rows[name] = {"quantize_elem_per_s": qe, "decode_kv_tokens_per_s_full_heads": dt * heads / w.heads,
                  "sample": how}
    print(json.dumps({name: rows[name]}), flush=True)
print(json.dumps({"host": bench.host_cores()}))
