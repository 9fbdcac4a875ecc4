"""Decode-step runtime over a multi-layer NF4 KV cache.

One decode step for every layer l, in order -- fused
(default, one launch per layer, nqkv_decode_step):
    quantize k_new, v_new -> append at row len_b   (I <- Concat(I, I_t))
    attention over len_b + 1 tokens                 (append-before-attend)
or unfused (three launches: nqkv_quantize x2 + nqkv_decode_attention).
    [world > 1] all-gather of the per-head outputs on a side stream (overlapped
    with the next layer; the synthetic q does not depend on the previous layer)

The per-step launch sequence is captured once per step slot into a CUDA graph
(the library's calls are stream-ordered and allocation-free, so they capture
as-is); replays cost only GPU-side kernel boundaries.  All compute is in
libnqkv.so; this module only owns buffers, streams and graphs.
"""
from __future__ import annotations

import os

import torch

from synth import workloads as W

from . import nqkv as N
from . import sharding

_EARLY = os.environ.get("NQKV_EARLY_START", "1") != "0"   # A/B switch for measurements


class DecodeRunner:
    def __init__(self, w: W.Workload, heads: range, device, group=None, world: int = 1,
                 step_slots: int | None = None, layers: int | None = None, fused: bool = True,
                 gen_device=None, planned: bool = True, fused_gather: bool | None = None,
                 nccl_gather: bool | None = None, gather_mode: str = "overlap"):
        self.w = w
        self.fused = fused
        if fused_gather is None:
            fused_gather = os.environ.get("NQKV_FUSED_GATHER", "0") == "1"
        # the all-gather fused into the decode epilogue (nqkv_decode_step_gather)
        # over symmetric-memory buffers instead of NCCL on a side stream
        self.fused_gather = fused_gather and fused and planned
        if world > 1:
            # the all-gather kernels on the side stream need SMs of their own (a
            # decode CTA fills an SM): leave 2 free (read once by libnqkv)
            sms = torch.cuda.get_device_properties(torch.device(device)).multi_processor_count
            os.environ.setdefault("NQKV_DECODE_CTAS", str(max(1, sms - 2)))
        # one nqkv_decode_plan per step, shared by every layer's decode launch
        self.planned = planned
        self.heads = heads
        self.dev = torch.device(device)
        # where the seeded synthetic inputs are drawn (CPU and CUDA generators
        # give different streams; parity tests draw on the CPU)
        self.gen_dev = self.dev if gen_device is None else torch.device(gen_device)
        self.group, self.world = group, world
        self.L = w.layers if layers is None else layers
        self.S = max(1, w.decode_steps if step_slots is None else step_slots)
        self.B, self.Hl, self.hd, self.blk = w.batch, len(heads), w.head_dim, w.blk
        lens0 = W.seq_lens(w)
        self.lens0 = lens0
        self.Tc = W.capacity(int(lens0.max()) + self.S)
        self.caches = [N.KVCache(self.B, self.Hl, self.hd, self.Tc, self.blk, self.dev)
                       for _ in range(self.L)]
        self.ws = N.make_workspace(self.B, self.Hl, self.hd, self.Tc, self.dev)
        self.plan = N.make_plan(self.dev)
        # outputs double-buffered by slot parity, so a step's device->host
        # read can overlap the next step's kernels (bench.py e2e)
        self.outs = torch.zeros((2, self.L, self.B, self.Hl, self.hd), dtype=torch.float32,
                                device=self.dev)
        self._last = 0
        steps = torch.arange(self.S, dtype=torch.int32)[:, None]
        self.pos = (lens0[None, :] + steps).to(torch.int32).to(self.dev)          # [S, B]
        self.attn_lens = (self.pos + 1).contiguous()                               # [S, B]
        self.inputs = torch.empty((self.S, self.L, 3, self.B, self.Hl, self.hd),
                                  dtype=torch.float16, device=self.dev)
        for s in range(self.S):
            for l in range(self.L):
                k, v, q = W.step_inputs(w, l, s, heads=heads, device=self.gen_dev)
                self.inputs[s, l, 0] = k[:, 0]
                self.inputs[s, l, 1] = v[:, 0]
                self.inputs[s, l, 2] = q
        self.gathered = None
        # NCCL all-gather of each layer's outputs on a side stream: always at
        # world > 1; selectable at world 1 (tests run it under graph capture)
        self.nccl_gather = (world > 1 if nccl_gather is None else nccl_gather) and not self.fused_gather
        # "overlap" -- per layer on a side stream beside the next
        # layer's attention (default); "serialized" -- per layer on the compute
        # stream (the honest, unoverlapped number); "per_step" -- one
        # all-gather of every layer's outputs at the end of the step
        if gather_mode not in ("overlap", "serialized", "per_step"):
            raise ValueError(f"gather_mode {gather_mode!r}")
        self.gather_mode = gather_mode
        if self.fused_gather:
            self._setup_fused_gather(group, world)
        elif self.nccl_gather and gather_mode == "per_step":
            # rank-major [world, L, B, Hl, hd]: gathered_layer(l) assembles a layer
            self.gathered = torch.empty((world, self.L, self.B, self.Hl, self.hd),
                                        dtype=torch.float32, device=self.dev)
        elif self.nccl_gather:
            self.gathered = torch.empty((self.L, world * self.B, self.Hl, self.hd),
                                        dtype=torch.float32, device=self.dev)
            self.comm = torch.cuda.Stream(device=self.dev)
        self.graphs: list[torch.cuda.CUDAGraph] = []
        self.events: list[list[tuple[torch.cuda.Event, torch.cuda.Event]]] = []

    def _setup_fused_gather(self, group, world):
        """Gathered outputs [2, L, B, world*Hl, hd] and per-layer flag arrays
        [2, L, world] in symmetric memory, double-buffered by step parity;
        every rank's kernels store into every rank's buffer through the peer
        pointers (sharding: rank r owns heads [r*Hl, (r+1)*Hl)).

        Read contract: a consumer of step n's gathered buffer (parity n % 2)
        must be stream-ordered before this rank's step n + 1 gather launches
        (which publish epoch n + 1).  A peer can then overwrite parity n % 2
        (its step n + 2) only after waiting for epoch n + 1 from every rank,
        i.e. after those reads.  Graph slots alternate parity, so the number
        of captured step graphs is even (doubled when step_slots is odd)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        grp = group if group is not None else dist.group.WORLD
        G, L, B, Hl, hd = world, self.L, self.B, self.Hl, self.hd
        self.g_rank = dist.get_rank(grp)
        self.g_world = G
        per = B * G * Hl * hd
        self.g_out = symm_mem.empty(2 * L * per, dtype=torch.float32, device=self.dev)
        self.g_flags = symm_mem.empty(2 * L * G, dtype=torch.int32, device=self.dev)
        self.g_flags.zero_()
        h_out = symm_mem.rendezvous(self.g_out, grp)
        h_flg = symm_mem.rendezvous(self.g_flags, grp)
        self.g_out_ptrs = torch.tensor(
            [[[h_out.buffer_ptrs[r] + ((p * L + l) * per) * 4 for r in range(G)] for l in range(L)]
             for p in range(2)], dtype=torch.int64, device=self.dev)
        self.g_flag_ptrs = torch.tensor(
            [[[h_flg.buffer_ptrs[r] + ((p * L + l) * G) * 4 for r in range(G)] for l in range(L)]
             for p in range(2)], dtype=torch.int64, device=self.dev)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.gathered = self.g_out.view(2, L, B, G * Hl, hd)
        torch.cuda.synchronize()
        dist.barrier(grp)

    def _graph_slots(self) -> int:
        """Captured step graphs: one per step slot; the fused gather alternates
        buffer parity, so it needs an even count."""
        return self.S * 2 if (self.fused_gather and self.S % 2) else self.S

    # ------------------------------------------------------------ prefill --
    def prefill(self, flush: torch.Tensor | None = None) -> list[float]:
        """Quantize every layer's prompt K/V (bulk nqkv_quantize, n_new =
        prompt length).  Returns per-launch kernel times in ms (L2 flushed
        before each launch when a flush buffer is given)."""
        T = int(self.lens0.max())
        zero = torch.zeros(self.B, dtype=torch.int32, device=self.dev)
        times = []
        for l, c in enumerate(self.caches):
            K, V = W.layer_kv(self.w, l, heads=self.heads, tokens=T, device=self.gen_dev)
            K, V = K.to(self.dev), V.to(self.dev)
            if flush is not None:
                flush.sum()             # read-only L2 sweep: evicts without dirty write-backs
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            c.append(K, V, zero)        # K and V of the layer: one nqkv_quantize_pair launch
            e1.record()
            times.append((e0, e1))
            del K, V
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in times]

    # --------------------------------------------------------------- step --
    @property
    def out(self) -> torch.Tensor:
        """Outputs [L, B, H, hd] of the most recent step (replay); the
        gathered [L, B, world*H, hd] outputs with the fused gather."""
        return self.out_of(self._last)

    def gathered_layer(self, l: int) -> torch.Tensor:
        """Layer l's gathered outputs [world*B, Hl, hd] (rank-major, as
        sharding.assemble takes them) in any NCCL gather mode."""
        if self.gather_mode == "per_step":
            return sharding.step_gather_layer(self.gathered, l)
        return self.gathered[l]

    def out_of(self, s: int) -> torch.Tensor:
        """Output buffer written by step (graph) slot s."""
        if self.fused_gather:
            return self.gathered[s % 2]
        return self.outs[(s % self.S) % 2]

    def step(self, s: int, events=None) -> None:
        """One decode step with the inputs of step slot s % S (graph slot s)."""
        self._last = s
        out = self.outs[s % 2]
        x = self.inputs[s % self.S]
        pos, lens = self.pos[s % self.S], self.attn_lens[s % self.S]
        cur = torch.cuda.current_stream()
        if self.fused_gather:
            self._step_fused_gather(x, lens, s % 2, events)
            return
        if self.planned:
            N.nqkv_decode_plan(lens, self.Hl, self.Tc, self.fused, self.plan, hd=self.hd)
        for l, c in enumerate(self.caches):
            if not self.fused:
                c.append(x[l, 0].unsqueeze(1), x[l, 1].unsqueeze(1), pos)   # [B, 1, H, hd] views
            if events is not None:
                events[l][0].record()
            # layers 1.. of a fused step: the kernel just before is the previous
            # layer's decode, which writes neither the plan nor this cache
            early = N.EARLY_START if (self.fused and l > 0 and _EARLY) else 0
            if self.fused and self.planned:
                c.step_planned(x[l, 0], x[l, 1], x[l, 2], lens, self.ws, self.plan, out=out[l],
                               flags=early)
            elif self.fused:
                c.step(x[l, 0], x[l, 1], x[l, 2], lens, self.ws, out=out[l])
            elif self.planned:
                c.attend_planned(x[l, 2], lens, self.ws, self.plan, out=out[l])
            else:
                c.attend(x[l, 2], lens, self.ws, out=out[l])
            if events is not None:
                events[l][1].record()
            if self.nccl_gather and self.gather_mode == "overlap":
                self.comm.wait_stream(cur)
                with torch.cuda.stream(self.comm):
                    sharding.all_gather_heads(out[l], self.gathered[l], self.group)
            elif self.nccl_gather and self.gather_mode == "serialized":
                sharding.all_gather_heads(out[l], self.gathered[l], self.group)
        if self.nccl_gather and self.gather_mode == "overlap":
            cur.wait_stream(self.comm)
        elif self.nccl_gather and self.gather_mode == "per_step":
            sharding.all_gather_heads(out, self.gathered.view(self.world * self.L, self.B, self.Hl, self.hd),
                                      self.group)

    def _step_fused_gather(self, x, lens, parity, events=None) -> None:
        N.nqkv_gather_epoch_bump(self.epoch)
        N.nqkv_decode_plan(lens, self.Hl, self.Tc, True, self.plan, hd=self.hd)
        for l, c in enumerate(self.caches):
            if events is not None:
                events[l][0].record()
            early = N.EARLY_START if (l > 0 and _EARLY) else 0
            N.nqkv_decode_step_gather(x[l, 0], x[l, 1], x[l, 2], c.k_codes, c.k_scales, c.v_codes,
                                      c.v_scales, lens, self.blk, self.ws, self.plan,
                                      self.g_out_ptrs[parity, l], self.g_flag_ptrs[parity, l],
                                      self.g_world, self.g_rank, epoch_ptr=self.epoch, flags=early)
            if events is not None:
                events[l][1].record()
        # every rank's rows of every layer have landed in this rank's buffer
        L, G = self.L, self.g_world
        N.nqkv_gather_wait(self.g_flags[parity * L * G:(parity + 1) * L * G], self.epoch)

    def capture(self, timing_slots=(0,)) -> None:
        """One CUDA graph per step slot (pointers differ per slot).  Slots in
        `timing_slots` also record an event pair around every decode launch
        (event nodes break the PDL overlap between layers, so only a few slots
        carry them)."""
        torch.cuda.synchronize()
        self.graphs, self.events = [], []
        for s in range(self._graph_slots()):
            ev = None
            if s in timing_slots:
                ev = [(torch.cuda.Event(enable_timing=True, external=True),
                       torch.cuda.Event(enable_timing=True, external=True)) for _ in range(self.L)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.step(s, ev)
            self.graphs.append(g)
            self.events.append(ev)
        torch.cuda.synchronize()

    def replay(self, i: int) -> None:
        n = len(self.graphs)
        self._last = i % n
        self.graphs[i % n].replay()

    def decode_kernel_ms(self) -> list[float]:
        """Durations of the decode-attention launches of the most recent replay
        of every step slot (events recorded inside the graphs)."""
        out = []
        for ev in self.events:
            if ev is None:
                continue
            out.extend(a.elapsed_time(b) for a, b in ev)
        return out

    # ------------------------------------------------------------ metrics --
    def tokens_per_step(self, s: int) -> int:
        """KV tokens attended in one step over all layers (a token = all of
        this rank's heads)."""
        return int(self.attn_lens[s % self.S].sum().item()) * self.L

    def decode_bytes(self, s: int) -> int:
        """Algorithmic HBM bytes of ONE decode launch at slot s: codes + scales
        of K and V for the attended tokens, q in, out; fused steps also read
        the new k, v (fp16) -- the new row's codes are written, not re-read."""
        toks = int(self.attn_lens[s % self.S].sum().item())
        per_tok = self.Hl * self.hd * 2 * (0.5 + 4.0 / self.blk)
        extra = self.B * self.Hl * self.hd * 2 * 2 if self.fused else 0
        return int(toks * per_tok + self.B * self.Hl * self.hd * (2 + 4) + extra)

    def launches_per_step(self) -> int:
        """Kernels this library launches per step: per layer one decode kernel
        (split partials merge in-kernel), plus two quantize launches when the
        append is not fused; plus one plan kernel per step when planned."""
        per_layer = 1 + (0 if self.fused else 2)
        return per_layer * self.L + (1 if self.planned else 0)
