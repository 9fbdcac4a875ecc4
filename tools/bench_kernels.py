"""Per-kernel micro-benchmark: decode attention / fused step / bulk quantize
on one layer of each BASELINE config (synthetic, L2 flushed before every
launch).  Prints achieved algorithmic GB/s.  Development tool, not the bench."""
import argparse
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N  # noqa: E402
from synth import workloads as W  # noqa: E402


def timeit(fn, flush, reps=10):
    ts = []
    for _ in range(reps):
        flush.sum()                 # read-only L2 sweep: evicts without leaving dirty lines
        torch.cuda._sleep(200000)       # keep the GPU busy while the host enqueues
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--heads5", type=int, default=12)
    ap.add_argument("--only", default="", help="attend|step|quantize: run just that once (for ncu)")
    ap.add_argument("--scale16", action="store_true", help="fp16 block scales (NQKV_SCALE_F16)")
    ap.add_argument("--blk", type=int, default=0, help="override the config's block size (e.g. 256)")
    args = ap.parse_args()
    dev = "cuda"
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for name in args.configs.split(","):
        w = W.CONFIGS[name]
        if args.blk:
            w = dataclasses.replace(w, blk=args.blk)
        H = args.heads5 if name == "c5" else w.heads
        lens = W.seq_lens(w)
        T = int(lens.max())
        Tc = W.capacity(T + 1)
        K, V = W.layer_kv(w, 0, heads=range(H), tokens=T, device=dev)
        cache = N.KVCache(w.batch, H, w.head_dim, Tc, w.blk, dev,
                          scale_dtype=torch.float16 if args.scale16 else torch.float32)
        z = torch.zeros(w.batch, dtype=torch.int32, device=dev)
        if args.only == "quantize":
            N.nqkv_quantize(K, z, cache.k_codes, cache.k_scales, w.blk)
            torch.cuda.synchronize()
            continue
        qt = timeit(lambda: N.nqkv_quantize(K, z, cache.k_codes, cache.k_scales, w.blk), flush)
        N.nqkv_quantize(V, z, cache.v_codes, cache.v_scales, w.blk)
        elems = K.numel()
        sb = 2 if args.scale16 else 4
        qbytes = elems * (2 + 0.5 + sb / w.blk)
        k1, v1, q = W.step_inputs(w, 0, 0, heads=range(H), device=dev)
        L = (lens + 1).to(dev)
        ws = N.make_workspace(w.batch, H, w.head_dim, Tc, dev)
        out = torch.empty((w.batch, H, w.head_dim), dtype=torch.float32, device=dev)
        if args.only in ("attend", "step"):
            for _ in range(3):
                if args.only == "attend":
                    cache.attend(q, L, ws, out=out)
                else:
                    cache.step(k1[:, 0], v1[:, 0], q, L, ws, out=out)
            torch.cuda.synchronize()
            continue
        at = timeit(lambda: cache.attend(q, L, ws, out=out), flush)
        st = timeit(lambda: cache.step(k1[:, 0], v1[:, 0], q, L, ws, out=out), flush)
        toks = int(L.sum())
        dbytes = toks * H * w.head_dim * 2 * (0.5 + sb / w.blk) + w.batch * H * w.head_dim * 6
        print(f"{name}: H={H} T={T} quantize {qt*1e3:8.1f} us {qbytes/qt/1e6:7.0f} GB/s | "
              f"attend {at*1e3:8.1f} us {dbytes/at/1e6:7.0f} GB/s | step {st*1e3:8.1f} us "
              f"{dbytes/st/1e6:7.0f} GB/s | cache {dbytes/1e6:.1f} MB", flush=True)
        del K, V, cache
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
