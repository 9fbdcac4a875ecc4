#!/usr/bin/env python
"""NQKV decode benchmark (BASELINE.json metric: decode-attn KV tokens/s over
the 4-bit cache; HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2]

A step = one decode step of the whole hot path over every layer of the
workload: 1-token NF4 quantize-append of K and V (nqkv_quantize) and fused
dequant decode attention (nqkv_decode_attention), per layer, in layer order.
Default workload: configs[1] (c2, OPT-1.3B-shaped: 24 layers, B=8, 32 heads,
head_dim 64, 2048 prompt tokens, 16 decode-step slots replayed cyclically).
Inputs are synthetic (synth/workloads.py) and resident in HBM; one step
touches 24 layers x ~38 MB = ~0.9 GB of packed cache, more than the 126 MB L2.

N > 1 (torchrun): weak scaling over heads -- every rank owns a 32-head shard
of a 32*N-head model and the per-layer outputs are all-gathered over NCCL.

--impl reference: the CPU oracle (oracle/) on rank 0, timed on a bounded
sample of the same workload (one layer, a few heads); other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn KV tokens/s over 4-bit cache; HBM GB/s vs peak at 1/2/4/8 GPU"
UNIT = "KV tokens/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """Polls NVML during the timed region (SM clock, throttle reasons)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report it
            self.err = str(e)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            pass

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            if not self.samples:
                self.sample()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ cpu baseline --
class OracleSample:
    """The CPU oracle on a bounded sample of the workload: one layer's decode
    step (1-token append of K and V + attention over the dequantised cache)
    for `heads` heads of all B sequences.  Prefill is untimed, as on the GPU."""

    def __init__(self, w, heads: int):
        from oracle import nqkv_oracle as O
        from synth import workloads as W
        self.O, self.w, self.h = O, w, heads
        hr = range(heads)
        self.lens = W.seq_lens(w).tolist()
        T = max(self.lens)
        Tc = W.capacity(T + 1)
        K, V = W.layer_kv(w, 0, heads=hr, tokens=T)
        k1, v1, q = W.step_inputs(w, 0, 0, heads=hr)
        self.kc, self.ks = O.empty_cache(w.batch, heads, Tc, w.head_dim, w.blk)
        self.vc, self.vs = O.empty_cache(w.batch, heads, Tc, w.head_dim, w.blk)
        O.quantize_append(K.numpy(), [0] * w.batch, w.blk, self.kc, self.ks)
        O.quantize_append(V.numpy(), [0] * w.batch, w.blk, self.vc, self.vs)
        self.k1, self.v1, self.q = k1.numpy(), v1.numpy(), q.numpy()
        # KV tokens of the full-H model represented by one sampled step
        self.tokens = sum(n + 1 for n in self.lens) * heads / w.heads

    def step(self):
        O, w = self.O, self.w
        O.quantize_append(self.k1, self.lens, w.blk, self.kc, self.ks)
        O.quantize_append(self.v1, self.lens, w.blk, self.vc, self.vs)
        O.decode_attention(self.q, self.kc, self.ks, self.vc, self.vs,
                           [n + 1 for n in self.lens], w.blk)

    def describe(self, reps):
        w = self.w
        return (f"1 of {w.layers} layers, {self.h} of {w.heads} heads, all {w.batch} sequences "
                f"({max(self.lens)} tokens), 1-token append + attention, {reps} reps; "
                f"value scaled to {w.heads}-head KV tokens")


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return 1


def cpu_baseline(w, seconds=10.0, heads=2):
    smp = OracleSample(w, heads)
    smp.step()
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or not times:
        t0 = time.perf_counter()
        smp.step()
        times.append(time.perf_counter() - t0)
    per = statistics.median(times)
    return {"value": smp.tokens / per, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
            "sample": smp.describe(len(times)) + f"; host cores available {len(os.sched_getaffinity(0))}"}


def run_reference(args, w, rank, world):
    """Base-contract reference arm = the oracle, timed as it stands."""
    if rank != 0:
        return 0
    smp = OracleSample(w, 1)
    for _ in range(args.warmup):
        smp.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        smp.step()
    el = time.perf_counter() - t0
    val = smp.tokens * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "oracle": "numpy float64 oracle/nqkv_oracle.py",
                       "step": smp.describe(args.steps)},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
                             "sample": smp.describe(args.steps)},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- ours --
def run_ours(args, w, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_2505_16210_b200 import sharding
    from paper_2505_16210_b200.runtime import DecodeRunner

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    group = dist.group.WORLD if world > 1 else None
    heads = sharding.weak_head_range(rank, w.heads, max(w.blk // w.head_dim, 1))
    runner = DecodeRunner(w, heads, dev, group=group, world=world)
    peak, peak_src = load_peaks()

    # prefill (bulk quantize) with L2 flushed before each launch: quantize roofline
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    q_ms = runner.prefill(flush=flush)
    T = int(runner.lens0.max())
    elems = w.batch * T * runner.Hl * w.head_dim
    q_bytes = elems * (2 + 0.5 + 4.0 / w.blk)
    q_gbs = [q_bytes / (t * 1e-3) / 1e9 for t in q_ms]
    del flush
    torch.cuda.synchronize()

    # warm-up (eager, initialises kernel attributes) then capture graphs
    runner.step(0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    runner.capture(timing_slots=(0,))
    for i in range(args.warmup):
        runner.replay(i)
    torch.cuda.synchronize()

    # ---------------------------------------------------------- timed region
    sampler = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" in os.environ
                           else local_rank)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        e0.record()
        for i in range(args.steps):
            runner.replay(args.warmup + i)
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    dec_ms = runner.decode_kernel_ms()          # slot 0's last replay (inside the region)
    tokens = sum(runner.tokens_per_step(args.warmup + i) for i in range(args.steps))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tok = torch.tensor([tokens], dtype=torch.float64, device=dev)
        dist.all_reduce(tok, op=dist.ReduceOp.SUM)
        tokens = float(tok.item())
    value = tokens / (ms * 1e-3)

    # ------------------------------------------------------------- e2e (host)
    host_in = torch.empty(runner.inputs.shape, dtype=runner.inputs.dtype, pin_memory=True)
    host_in.copy_(runner.inputs.cpu())
    host_out = torch.empty(runner.out.shape, dtype=runner.out.dtype, pin_memory=True)
    h2d = host_in[0].numel() * host_in.element_size()
    d2h = host_out.numel() * host_out.element_size()
    # Pipelined: step i+1's inputs go host->device on a copy stream while step
    # i computes, and step i's outputs come back device->host on it right after
    # step i (outputs are double-buffered by slot parity, so step i+1 never
    # waits for that read).  Every step still moves its own inputs in and its
    # own outputs out inside the timed region.
    main = torch.cuda.current_stream()
    cs = torch.cuda.Stream()
    h2d_ev = [torch.cuda.Event() for _ in range(runner.S)]
    d2h_ev = [torch.cuda.Event() for _ in range(2)]
    comp_ev = torch.cuda.Event()

    def e2e_run(first, n):
        with torch.cuda.stream(cs):
            s0 = first % runner.S
            runner.inputs[s0].copy_(host_in[s0], non_blocking=True)
            h2d_ev[s0].record(cs)
        for i in range(first, first + n):
            s, s1 = i % runner.S, (i + 1) % runner.S
            main.wait_event(h2d_ev[s])
            main.wait_event(d2h_ev[s % 2])       # this slot's output buffer was read back
            runner.replay(s)
            comp_ev.record(main)
            with torch.cuda.stream(cs):
                if i + 1 < first + n:
                    runner.inputs[s1].copy_(host_in[s1], non_blocking=True)
                    h2d_ev[s1].record(cs)
                cs.wait_event(comp_ev)
                host_out.copy_(runner.out_of(s), non_blocking=True)
                d2h_ev[s % 2].record(cs)
        main.wait_stream(cs)

    e2e_run(0, min(args.warmup, 4))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record()
    e2e_run(args.warmup, args.steps)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = tokens / (e2e_ms * 1e-3)

    if rank != 0:
        return 0
    # roofline for the dominant kernel (decode attention): algorithmic bytes
    # per launch / average launch duration.  The launches of a step are
    # PDL-chained (each one's prologue overlaps its predecessor's tail), so the
    # average duration is the device-timed step time over the decode launches
    # of a step -- conservative: the per-step plan kernel is charged to them.
    # The isolated duration (CUDA events around each launch, which break the
    # chaining) is reported beside it.
    bytes_per_launch = runner.decode_bytes(0)
    dec_mean_ms = statistics.mean(dec_ms) if dec_ms else float("nan")
    chained_ms = (ms / args.steps) / w.layers
    achieved = bytes_per_launch / (chained_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(w.name, {}).get("decode_dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)
    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {
            "workload": f"{w.name}: {w.layers} layers, B={w.batch}, {w.heads} heads/GPU x "
                        f"{world} GPU, head_dim {w.head_dim}, prompt {T} + {runner.S} decode-step "
                        f"slots replayed cyclically, NF4 blk {w.blk}, fp32 scales",
            "storage": "nf4 codes (u4) + fp32 block scales; fp32 arithmetic",
            "l2": f"inputs larger than L2: one step reads {w.layers} layers x "
                  f"{runner.caches[0].nbytes() / 1e6:.1f} MB of packed cache (L2 "
                  f"{l2 / 1e6:.0f} MB)",
            "execution": "per-step CUDA graph; one fused nqkv_decode_step launch per layer (append + attend, PDL-chained)",
            "parallelism": f"head-sharded x{world} (weak)" + (", NCCL all-gather of outputs"
                                                              if world > 1 else ""),
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "decode_kernel (nqkv_decode_attention)",
                     "bytes_per_launch": bytes_per_launch, "mean_launch_us": chained_ms * 1e3,
                     "launches_timed": args.steps * w.layers, "peak_source": peak_src,
                     "timing": "device-timed step (CUDA events around the timed region) / decode "
                               "launches per step; launches PDL-chained inside the step graph; the "
                               "per-step plan kernel is charged to them",
                     "isolated_launch_us": dec_mean_ms * 1e3,
                     "isolated_timing": "CUDA events around every layer's launch in step slot "
                                        "0's graph (its last replay inside the timed region; "
                                        "the events break the PDL chaining)"},
        "quantize_roofline": {"bound": "hbm", "achieved": statistics.median(q_gbs), "peak": peak,
                              "unit": "GB/s", "frac": statistics.median(q_gbs) / peak,
                              "kernel": "quantize_kernel (nqkv_quantize, bulk prefill, L2 flushed)",
                              "bytes_per_launch": q_bytes, "launches": len(q_ms)},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "how": "pinned H2D of every layer's new k/v/q, graph replay, D2H of every "
                       "layer's output; the next step's H2D and this step's D2H run on a "
                       "copy stream beside the step's kernels (outputs double-buffered)"},
        "gpu_launches": runner.launches_per_step() * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from synth import workloads as W
    w = W.CONFIGS[args.workload]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, w, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        # bound NCCL's SM use to the 2 SMs the decode grid leaves free (runtime.py)
        os.environ.setdefault("NCCL_MAX_NCHANNELS", "2")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, w, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
