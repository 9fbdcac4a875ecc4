#!/usr/bin/env python
"""NQKV decode benchmark (BASELINE.json metric: decode-attn KV tokens/s over
the 4-bit cache; HBM GB/s vs peak at 1/2/4/8 GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5] [--scaling weak|strong] [--no-configs]

A step = one decode step of the whole hot path over every layer of the
workload: per layer, the 1-token NF4 quantize-append of K and V fused with the
dequant-in-registers decode attention (nqkv_decode_step_planned), captured as
one CUDA graph per step.  Inputs are synthetic (synth/workloads.py) and
resident in HBM.

Default workload: BASELINE.json configs[4] (c5, OPT-175B-shaped: 96 layers,
B = 64, head_dim 128, 4096 cached tokens, blk 64) as the 8-GPU weak shard of
12 heads per GPU (43.5 GB of 4-bit cache per GPU), the configuration
BASELINE.json times at 1/2/4/8 GPUs.  --scaling strong splits the fixed
96 heads over the GPUs instead (at 1 GPU the layer count is cut to what fits).

At N = 1 the same JSON line also carries a "configs" block: c2, c3 (blk
32/64/128), c4 and c5 with all 96 heads on one GPU, each with its decode and
quantize rooflines (--no-configs skips it).

N > 1 (torchrun): every rank owns its head shard; the per-layer outputs are
all-gathered over NCCL on a side stream.

--impl reference: the CPU oracle (oracle/) on rank 0, timed on a bounded
sample of the same workload; other ranks exit 0.
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
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> dict:
    return {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "cpu_model": cpu_model(), "blas_threads": blas_threads()}


class OracleSample:
    """The CPU oracle on a bounded sample of the workload: one layer's decode
    step (1-token append of K and V + attention over the dequantised cache)
    for `heads` heads of the first `batch` sequences.  Prefill is untimed, as
    on the GPU.  `scale` converts the sample's KV tokens to the full step's
    (all heads of the shard, all sequences, all layers are the same work)."""

    def __init__(self, w, heads: int, batch: int | None = None, shard_heads: int | None = None):
        from oracle import nqkv_oracle as O
        from synth import workloads as W
        self.O, self.w, self.h = O, w, heads
        self.b = w.batch if batch is None else min(batch, w.batch)
        self.shard = w.heads if shard_heads is None else shard_heads
        hr = range(heads)
        lens = W.seq_lens(w)
        T = int(lens.max())
        self.lens = lens[:self.b].tolist()
        Tc = W.capacity(T + 1)
        K, V = W.layer_kv(w, 0, heads=hr, tokens=T)
        k1, v1, q = W.step_inputs(w, 0, 0, heads=hr)
        b = self.b
        self.kc, self.ks = O.empty_cache(b, heads, Tc, w.head_dim, w.blk)
        self.vc, self.vs = O.empty_cache(b, heads, Tc, w.head_dim, w.blk)
        O.quantize_append(K[:b].numpy(), [0] * b, w.blk, self.kc, self.ks)
        O.quantize_append(V[:b].numpy(), [0] * b, w.blk, self.vc, self.vs)
        self.k1, self.v1, self.q = k1[:b].numpy(), v1[:b].numpy(), q[:b].numpy()
        # KV tokens (a token = all heads of the shard) represented by one sampled step
        self.tokens = sum(n + 1 for n in self.lens) * heads / self.shard

    def step(self):
        O, w = self.O, self.w
        O.quantize_append(self.k1, self.lens, w.blk, self.kc, self.ks)
        O.quantize_append(self.v1, self.lens, w.blk, self.vc, self.vs)
        O.decode_attention(self.q, self.kc, self.ks, self.vc, self.vs,
                           [n + 1 for n in self.lens], w.blk)

    def describe(self, reps):
        w = self.w
        return (f"{w.name}: 1 of {w.layers} layers, {self.h} of the {self.shard}-head shard, "
                f"{self.b} of {w.batch} sequences ({max(self.lens)} tokens), 1-token append + "
                f"attention, {reps} reps; value scaled to KV tokens of the full shard (a token = "
                f"all {self.shard} heads); extrapolated linearly in heads and sequences")


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return 1


def sample_for(w, shard_heads):
    """Bounded oracle sample (~10-30 s of CPU work per timed loop)."""
    per_seq = (int(w.seq_len) + 1) * w.head_dim
    batch = max(1, min(w.batch, (1 << 22) // per_seq))      # ~4 M cached elements per head
    return OracleSample(w, 1, batch=batch, shard_heads=shard_heads)


def cpu_baseline(w, shard_heads, seconds=10.0):
    smp = sample_for(w, shard_heads)
    smp.step()
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or not times:
        t0 = time.perf_counter()
        smp.step()
        times.append(time.perf_counter() - t0)
    per = statistics.median(times)
    hc = host_cores()
    return {"value": smp.tokens / per, "unit": UNIT, "cores": hc["blas_threads"], "kind": "oracle",
            "sample": smp.describe(len(times)), "host": hc}


def run_reference(args, w, rank, world):
    """Base-contract reference arm = the oracle, timed as it stands."""
    if rank != 0:
        return 0
    shard = shard_heads(w, args.scaling, world)
    smp = sample_for(w, shard)
    for _ in range(args.warmup):
        smp.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        smp.step()
    el = time.perf_counter() - t0
    val = smp.tokens * args.steps / el          # KV tokens of the sampled layer-steps / time
    hc = host_cores()
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(w, shard, world, args.scaling),
                       "oracle": "numpy float64 oracle/nqkv_oracle.py", "step": smp.describe(args.steps)},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": hc["blas_threads"], "kind": "oracle",
                             "sample": smp.describe(args.steps), "host": hc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- ours --
WEAK_SHARD = {"c1": 12, "c2": 32, "c3": 32, "c4": 5, "c5": 12}    # heads per GPU (c4/c5: the 8-GPU shard)


def shard_heads(w, scaling, world):
    key = w.name.split("-")[0]
    if scaling == "strong":
        return w.heads // world
    return WEAK_SHARD.get(key, w.heads)


def workload_name(w, shard, world, scaling):
    return (f"{w.name} (BASELINE configs[{int(w.name[1]) - 1}]): {w.layers} layers, B={w.batch}, "
            f"{shard} heads/GPU x {world} GPU ({scaling}), head_dim {w.head_dim}, "
            f"{'lengths U[%d, %d]' % (w.ragged_min, w.seq_len) if w.ragged_min else '%d cached tokens' % w.seq_len}"
            f" + 1 appended per step, NF4 blk {w.blk}, fp32 scales")


def layers_that_fit(w, heads, dev, reserve=0.80):
    """Largest layer count whose cache fits in `reserve` of free memory
    (BASELINE.json c5: "scaling the layer count to fit a single GPU")."""
    import torch
    from synth import workloads as W
    T = int(W.seq_lens(w).max())
    Tc = W.capacity(T + w.decode_steps)
    per = 2 * w.batch * heads * Tc * (w.head_dim // 2 + 4 * w.head_dim // w.blk)
    gen = 3 * w.batch * T * heads * w.head_dim * 2          # prefill generation buffers
    free = torch.cuda.mem_get_info(dev)[0]
    return max(1, min(w.layers, int((reserve * free - gen) // per)))


def measure(args, w, heads, dev, world, group, layers=None, steps=None, warmup=None, e2e=False,
            isolated=True):
    """Prefill (bulk quantize, L2 flushed per launch), capture the step
    graphs, time `steps` replays on the device.  Returns a result dict (and the
    runner when e2e is requested)."""
    import torch
    import torch.distributed as dist
    from paper_2505_16210_b200.runtime import DecodeRunner

    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    runner = DecodeRunner(w, heads, dev, group=group, world=world, layers=layers,
                          gather_mode=getattr(args, "gather", "overlap"))
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    q_ms = runner.prefill(flush=flush)
    T = int(runner.lens0.max())
    elems = w.batch * T * runner.Hl * w.head_dim
    q_bytes = 2 * elems * (2 + 0.5 + 4.0 / w.blk)      # K and V: one nqkv_quantize_pair launch
    q_gbs = [q_bytes / (t * 1e-3) / 1e9 for t in q_ms]
    del flush
    torch.cuda.synchronize()
    runner.step(0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the timed graphs carry no event nodes (events around a launch break the
    # PDL chaining between layers; with one step slot, as at c5, an
    # instrumented slot would be every step)
    runner.capture(timing_slots=())
    for i in range(warmup):
        runner.replay(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" in os.environ
                           else dev.index or 0)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        e0.record()
        for i in range(steps):
            runner.replay(warmup + i)
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    dec_ms = []
    if isolated:
        # isolated launch durations: one replay of an instrumented capture of
        # slot 0, after the timed region
        if world > 1:
            dist.barrier()
        runner.capture(timing_slots=(0,))
        runner.replay(0)
        torch.cuda.synchronize()
        dec_ms = runner.decode_kernel_ms()
        runner.capture(timing_slots=())
    tokens = sum(runner.tokens_per_step(warmup + i) for i in range(steps))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tok = torch.tensor([tokens], dtype=torch.float64, device=dev)
        dist.all_reduce(tok, op=dist.ReduceOp.SUM)
        tokens = float(tok.item())
    L = runner.L
    bytes_per_launch = runner.decode_bytes(0)
    chained_ms = (ms / steps) / L
    res = {"value": tokens / (ms * 1e-3), "ms_per_step": ms / steps, "layers": L,
           "heads": runner.Hl, "bytes_per_launch": bytes_per_launch, "chained_launch_us": chained_ms * 1e3,
           "decode_gbs": bytes_per_launch / (chained_ms * 1e-3) / 1e9,
           "isolated_launch_us": statistics.mean(dec_ms) * 1e3 if dec_ms else None,
           "quantize_gbs": statistics.median(q_gbs), "quantize_bytes_per_launch": q_bytes,
           "quantize_launches": len(q_ms), "clocks": sampler.summary(),
           "gpu_launches": runner.launches_per_step() * steps, "steps": steps}
    if e2e:
        return res, runner
    del runner
    torch.cuda.empty_cache()
    return res, None


def e2e_measure(args, runner, world, dev):
    """Same metric through the public API with host buffers: every step's new
    k/v/q go host->device (pinned) and every layer's output device->host,
    inside the timed region (pipelined on a copy stream)."""
    import torch
    import torch.distributed as dist
    host_in = torch.empty(runner.inputs.shape, dtype=runner.inputs.dtype, pin_memory=True)
    host_in.copy_(runner.inputs.cpu())
    host_out = torch.empty(runner.out.shape, dtype=runner.out.dtype, pin_memory=True)
    h2d = host_in[0].numel() * host_in.element_size()
    d2h = host_out.numel() * host_out.element_size()
    main = torch.cuda.current_stream()
    cs = torch.cuda.Stream()
    n_slots = len(runner.graphs)
    # H2D lands in one of two device staging buffers on the copy stream (the
    # next step's inputs while this step computes); the step then takes them
    # with one device-to-device copy into its input slot (stream-ordered)
    stage = torch.empty((2,) + tuple(runner.inputs.shape[1:]), dtype=runner.inputs.dtype,
                        device=runner.inputs.device)
    h2d_ev = [torch.cuda.Event() for _ in range(2)]
    used_ev = [torch.cuda.Event() for _ in range(2)]
    d2h_ev = [torch.cuda.Event() for _ in range(2)]
    comp_ev = torch.cuda.Event()

    def e2e_run(first, n):
        with torch.cuda.stream(cs):
            stage[first % 2].copy_(host_in[first % runner.S], non_blocking=True)
            h2d_ev[first % 2].record(cs)
        for i in range(first, first + n):
            p, s = i % 2, i % runner.S
            main.wait_event(h2d_ev[p])
            main.wait_event(d2h_ev[p])           # this parity's output buffer was read back
            runner.inputs[s].copy_(stage[p])
            used_ev[p].record(main)
            runner.replay(i % n_slots)
            comp_ev.record(main)
            with torch.cuda.stream(cs):
                if i + 1 < first + n:
                    cs.wait_event(used_ev[1 - p])    # staging buffer free again
                    stage[1 - p].copy_(host_in[(i + 1) % runner.S], non_blocking=True)
                    h2d_ev[1 - p].record(cs)
                cs.wait_event(comp_ev)
                host_out.copy_(runner.out_of(i % n_slots), non_blocking=True)
                d2h_ev[p].record(cs)
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
    tokens = sum(runner.tokens_per_step(args.warmup + i) for i in range(args.steps))
    if world > 1:
        tok = torch.tensor([tokens], dtype=torch.float64, device=dev)
        dist.all_reduce(tok, op=dist.ReduceOp.SUM)
        tokens = float(tok.item())
    return {"value": tokens / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "how": "pinned H2D of every layer's new k/v/q into a device staging buffer, a D2D copy "
                   "into the step's input slot, graph replay, D2H of every layer's output; the next "
                   "step's H2D and this step's D2H run on a copy stream beside the step's kernels "
                   "(staging and outputs double-buffered)"}


def load_traffic(name):
    """DRAM bytes per decode launch from the committed ncu capture of the same
    launch configuration (profiles/traffic.json; in-process DRAM counters are
    not available to this process)."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(tp)).get(name, {})
        src = d.get("source")
        if src and d.get("quantize_source"):
            src = f"ncu --set full of this launch configuration: decode {src}, quantize {d['quantize_source']}"
        return d.get("decode_dram_bytes_per_launch"), d.get("quantize_dram_bytes_per_launch"), src
    except Exception:
        return None, None, None


def extra_configs(args, dev, peak):
    """Per-config rooflines at N = 1 (BASELINE configs[1..4]); fewer steps,
    the sweep variants with fewer layers (per-launch numbers do not depend on
    the layer count once a step reads more than L2)."""
    import dataclasses
    from synth import workloads as W
    out = {}
    plan = [("c2", W.CONFIGS["c2"], 32, None), ("c3", W.CONFIGS["c3"], 32, None),
            ("c3-blk32", dataclasses.replace(W.CONFIGS["c3"], blk=32), 32, 8),
            ("c3-blk128", dataclasses.replace(W.CONFIGS["c3"], blk=128), 32, 8),
            ("c4", W.CONFIGS["c4"], 40, None), ("c5-96heads", W.CONFIGS["c5"], 96, -1)]
    for key, w, heads, layers in plan:
        if layers == -1:
            layers = layers_that_fit(w, heads, dev)
        try:
            r, _ = measure(args, w, range(heads), dev, 1, None, layers=layers, steps=10, warmup=3,
                           isolated=False)
        except Exception as e:  # noqa: BLE001 -- report, keep the headline
            out[key] = {"error": str(e)[:200]}
            continue
        out[key] = {"workload": workload_name(w, heads, 1, "strong" if key.startswith("c5") else "weak"),
                    "layers_timed": r["layers"], "value": r["value"], "unit": UNIT,
                    "ms_per_step": r["ms_per_step"],
                    "decode_roofline": {"achieved": r["decode_gbs"], "peak": peak, "unit": "GB/s",
                                        "frac": r["decode_gbs"] / peak,
                                        "bytes_per_launch": r["bytes_per_launch"],
                                        "mean_launch_us": r["chained_launch_us"]},
                    "quantize_roofline": {"achieved": r["quantize_gbs"], "peak": peak, "unit": "GB/s",
                                          "frac": r["quantize_gbs"] / peak,
                                          "bytes_per_launch": r["quantize_bytes_per_launch"]},
                    "clocks": r["clocks"]}
    return out


def prefill_config(dev, peak_tflops, name="c4", heads=40):
    """§8(f) row 4: causal prefill attention over the 4-bit cache
    (nqkv_prefill_attention, tcgen05) at the config's prompt length; FLOP
    roofline with algorithmic causal FLOPs 2*hd*len*(len+1) per (b, h)."""
    import torch
    from paper_2505_16210_b200 import nqkv as N
    from synth import workloads as W
    w = W.CONFIGS[name]
    lens = W.seq_lens(w)
    B, hd, T = w.batch, w.head_dim, int(lens.max())
    Tc = W.capacity(T)
    cache = N.KVCache(B, heads, hd, Tc, w.blk, dev)
    K, V = W.layer_kv(w, 0, heads=range(heads), tokens=T, device=dev)
    cache.append(K, V, torch.zeros(B, dtype=torch.int32, device=dev))
    del K, V
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(B, T, heads, hd, generator=g, device=dev).half()
    L = lens.to(dev)
    out = torch.empty(B, T, heads, hd, device=dev)
    call = lambda: N.nqkv_prefill_attention(q, cache.k_codes, cache.k_scales, cache.v_codes,
                                            cache.v_scales, L, w.blk, out=out)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        call()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    flop = sum(2.0 * hd * int(x) * (int(x) + 1) for x in lens.tolist()) * heads
    tf = flop / (ms * 1e-3) / 1e12
    del cache, q, out
    torch.cuda.empty_cache()
    return {"workload": f"{w.name} prompt: B={B}, {heads} heads, hd {hd}, {T} tokens (causal)",
            "ms_per_layer": ms,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": tf / peak_tflops,
                         "flops_per_launch": flop,
                         "peak_source": "measured (MEASURED_PEAKS.json bf16_tflops; fp16 dense = bf16)",
                         "note": "algorithmic causal FLOPs; the fp16 hi/lo operand splits do ~2.5x that on the tensor cores"}}


def layouts_config(dev, peak):
    """§8(f) row 4 KV layouts at the c5 shard's shape (64 x 12 heads x 4097
    tokens, hd 128, blk 64): decode attention launches (unplanned, back to
    back; one layer's cache is 3.4x L2) over the contiguous cache, the same
    rows in a paged cache of 256-token pages in shuffled order, and
    grouped-query (48 query heads over the 12 KV heads; the group-native
    kernel, decode_gqa.cuh).  Algorithmic bytes count the cache once (+ q/out
    of every query head)."""
    import numpy as np
    import torch
    from paper_2505_16210_b200 import nqkv as N
    B, Hkv, hd, blk, T, P = 64, 12, 128, 64, 4097, 256
    maxp = -(-T // P)
    n_pages = B * maxp
    Tc = maxp * P
    g = torch.Generator(device=dev).manual_seed(0)
    perm = np.random.default_rng(0).permutation(n_pages).reshape(B, maxp)
    bt = torch.tensor(perm, dtype=torch.int32, device=dev)
    ck = torch.zeros(B, Hkv, Tc, hd // 2, dtype=torch.uint8, device=dev)
    cs = torch.zeros(B, Hkv, Tc, hd // blk, dtype=torch.float32, device=dev)
    cv, cvs = torch.zeros_like(ck), torch.zeros_like(cs)
    pk = torch.zeros(n_pages, Hkv, P, hd // 2, dtype=torch.uint8, device=dev)
    ps = torch.zeros(n_pages, Hkv, P, hd // blk, dtype=torch.float32, device=dev)
    pv, pvs = torch.zeros_like(pk), torch.zeros_like(ps)
    lay = N.kv_layout(0, bt, P, n_pages)
    z = torch.zeros(B, dtype=torch.int32, device=dev)
    for codes, scales, pc, pcs in ((ck, cs, pk, ps), (cv, cvs, pv, pvs)):
        x = torch.randn(B, T, Hkv, hd, generator=g, device=dev).half()
        N.nqkv_quantize(x, z, codes, scales, blk)
        N.nqkv_quantize_kv(x, z, pc, pcs, blk, lay, Tc)
        del x
    L = torch.full((B,), T, dtype=torch.int32, device=dev)
    res = {}
    cases = [("contiguous", Hkv, lambda q, ws, o: N.nqkv_decode_attention(q, ck, cs, cv, cvs, L, blk, ws, out=o)),
             ("paged-256", Hkv, lambda q, ws, o: N.nqkv_decode_attention_kv(q, pk, ps, pv, pvs, L, blk, lay, Tc, ws, out=o)),
             ("gqa-4", 4 * Hkv, lambda q, ws, o: N.nqkv_decode_attention_kv(q, ck, cs, cv, cvs, L, blk,
                                                                            N.kv_layout(Hkv), Tc, ws, out=o))]
    for name, H, call in cases:
        q = torch.randn(B, H, hd, generator=g, device=dev).half()
        ws = N.make_workspace(B, H, hd, Tc, dev)
        o = torch.empty(B, H, hd, device=dev)
        for _ in range(3):
            call(q, ws, o)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        a.record()
        for _ in range(n):
            call(q, ws, o)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / n * 1e3
        nbytes = B * T * Hkv * hd * 2 * (0.5 + 4 / blk) + B * H * hd * (2 + 4)
        res[name] = {"query_heads": H, "kv_heads": Hkv, "us_per_launch": us,
                     "bytes_per_launch": nbytes,
                     "decode_roofline": {"achieved": nbytes / (us * 1e-6) / 1e9, "peak": peak,
                                         "unit": "GB/s", "frac": nbytes / (us * 1e-6) / 1e9 / peak}}
        del q, ws, o
    del ck, cs, cv, cvs, pk, ps, pv, pvs
    torch.cuda.empty_cache()
    res["workload"] = (f"c5 shard shape: B={B}, {Hkv} KV heads, hd {hd}, {T} tokens, blk {blk}; "
                       f"paged: {P}-token pages, shuffled block table; gqa-4: 4 query heads per KV head "
                       f"(group-native kernel: each KV head streamed once for its 4 query heads; "
                       f"KV bytes counted once)")
    res["timing"] = "back-to-back unplanned nqkv_decode_attention(_kv) launches, CUDA events, mean of 20"
    return res


def run_ours(args, w, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_2505_16210_b200 import sharding

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    group = dist.group.WORLD if world > 1 else None
    shard = shard_heads(w, args.scaling, world)
    grp = max(w.blk // w.head_dim, 1)
    if args.scaling == "strong":
        heads = sharding.head_range(rank, world, w.heads, grp)
        layers = layers_that_fit(w, shard, dev)
        if world > 1:
            t = torch.tensor([layers], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            layers = int(t.item())
    else:
        heads = sharding.weak_head_range(rank, shard, grp)
        layers = None
    peak, peak_src = load_peaks()
    r, runner = measure(args, w, heads, dev, world, group, layers=layers, e2e=True)
    e2e = e2e_measure(args, runner, world, dev)
    L = runner.L
    del runner
    torch.cuda.empty_cache()
    if rank != 0:
        return 0
    traffic, q_traffic, t_src = load_traffic(w.name)
    cpu = None
    configs = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, shard)
    if world == 1 and not args.no_configs:
        configs = extra_configs(args, dev, peak)
        try:
            tfp = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        except Exception:
            tfp = 1590.0
        try:
            configs["prefill-c4"] = prefill_config(dev, tfp)
        except Exception as e:  # noqa: BLE001
            configs["prefill-c4"] = {"error": str(e)[:200]}
        try:
            configs["kv-layouts"] = layouts_config(dev, peak)
        except Exception as e:  # noqa: BLE001
            configs["kv-layouts"] = {"error": str(e)[:200]}
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {
            "workload": workload_name(w, shard, world, args.scaling) +
                        (f"; {L} of {w.layers} layers (fit one GPU)" if L != w.layers else ""),
            "storage": "nf4 codes (u4) + fp32 block scales; fp32 arithmetic",
            "l2": f"inputs larger than L2: one step reads {L} layers x "
                  f"{r['bytes_per_launch'] / 1e6:.1f} MB of packed cache (L2 "
                  f"{torch.cuda.get_device_properties(dev).L2_cache_size / 1e6:.0f} MB)",
            "execution": "per-step CUDA graph; per-step plan kernel + one fused nqkv_decode_step "
                         "launch per layer (append + attend, PDL-chained)",
            "parallelism": f"head-sharded x{world} ({args.scaling})" +
                           ({"overlap": ", NCCL all-gather of each layer's outputs on a side stream",
                             "serialized": ", NCCL all-gather of each layer's outputs, serialized",
                             "per_step": ", one NCCL all-gather of all layers' outputs per step"}
                            [args.gather] if world > 1 else ""),
        },
        "roofline": {"bound": "hbm", "achieved": r["decode_gbs"], "peak": peak, "unit": "GB/s",
                     "frac": r["decode_gbs"] / peak, "traffic": traffic,
                     "traffic_source": t_src or "none",
                     "kernel": "decode_kernel (nqkv_decode_step_planned)",
                     "bytes_per_launch": r["bytes_per_launch"], "mean_launch_us": r["chained_launch_us"],
                     "launches_timed": args.steps * L, "peak_source": peak_src,
                     "timing": "device-timed step (CUDA events around the timed region) / decode "
                               "launches per step; launches PDL-chained inside the step graph; the "
                               "per-step plan kernel is charged to them",
                     "isolated_launch_us": r["isolated_launch_us"],
                     "isolated_timing": "CUDA events around every layer's launch in one replay "
                                        "of an instrumented capture of step slot 0, after the "
                                        "timed region (the events break the PDL chaining; the "
                                        "timed graphs carry none)"},
        "quantize_roofline": {"bound": "hbm", "achieved": r["quantize_gbs"], "peak": peak,
                              "unit": "GB/s", "frac": r["quantize_gbs"] / peak, "traffic": q_traffic,
                              "kernel": "quantize_kernel (nqkv_quantize_pair: a layer's K and V per launch, bulk prefill, L2 flushed)",
                              "bytes_per_launch": r["quantize_bytes_per_launch"],
                              "launches": r["quantize_launches"]},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": r["gpu_launches"],
        "clocks": r["clocks"],
    }
    if configs is not None:
        line["configs"] = configs
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--gather", default="overlap", choices=["overlap", "serialized", "per_step"],
                    help="N > 1: per-layer all-gather overlapped on a side stream (default), "
                         "serialized on the compute stream, or one per step (SURVEY 8(e))")
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
