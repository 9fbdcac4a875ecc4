"""Seeded synthetic inputs shaped like the paper's OPT workloads.

This module is shared by the oracle side (tests, cpu baseline) and the CUDA
side (tests, bench).  It holds NO arithmetic of the NQKV method: it only draws
random fp16 K/V/q tensors and sequence lengths.  The recipe (DESIGN.md
"Input recipe") follows BASELINE.json configs and SURVEY.md 8(d):

  K[b,t,h,j] = fp16(sigma_K[l,h,j] * z),  V likewise with an independent sigma_V,
  z ~ N(0,1),  sigma = exp(0.5 * N(0,1))  (LogNormal(0, 0.5) per channel),
  K-only outlier channels get sigma x 10 (c2-c4: 2 of every 64 channels of a
  head; c5: each channel with probability 0.03),
  q ~ N(0,1) in fp16.

Each (layer, head) slab draws from its own torch.Generator seeded from
(seed, layer, head, purpose), so any head shard regenerates exactly its own
heads and the data do not depend on the GPU count.  CPU and CUDA generators
give different streams; parity tests generate on the CPU.
"""
from __future__ import annotations

import dataclasses
import hashlib

import torch


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    layers: int
    batch: int
    heads: int
    head_dim: int
    seq_len: int                 # cached tokens before decoding (max when ragged)
    blk: int = 64
    decode_steps: int = 1
    ragged_min: int | None = None  # lengths ~ U[ragged_min, seq_len] when set
    outliers: str = "none"       # "none" | "2of64" | "p0.03"
    seed: int = 0

    @property
    def hidden(self) -> int:
        return self.heads * self.head_dim


# BASELINE.json "configs" (indices 0..4)
CONFIGS = {
    "c1": Workload("c1-single-layer", 1, 1, 12, 64, 512, 64, 1, None, "none"),
    "c2": Workload("c2-opt1.3b", 24, 8, 32, 64, 2048, 64, 16, None, "2of64"),
    "c3": Workload("c3-opt6.7b", 32, 32, 32, 128, 2048, 64, 1, 1024, "2of64"),
    "c4": Workload("c4-opt13b-long", 40, 4, 40, 128, 8192, 64, 1, None, "2of64"),
    "c5": Workload("c5-opt175b", 96, 64, 96, 128, 4096, 64, 1, None, "p0.03"),
}


def _seed(*parts) -> int:
    h = hashlib.sha256(("/".join(str(p) for p in parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def _gen(device, *parts) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(_seed(*parts))
    return g


def seq_lens(w: Workload) -> torch.Tensor:
    """Cached lengths per sequence (int32, CPU).  Ragged configs draw integers
    uniform in [ragged_min, seq_len] from seed w.seed (BASELINE.json c3)."""
    if w.ragged_min is None:
        return torch.full((w.batch,), w.seq_len, dtype=torch.int32)
    g = _gen("cpu", w.seed, "lens")
    return torch.randint(w.ragged_min, w.seq_len + 1, (w.batch,), generator=g,
                         dtype=torch.int64).to(torch.int32)


def channel_sigma(w: Workload, layer: int, head: int, which: str, device="cpu") -> torch.Tensor:
    """Per-channel std of one (layer, head) for 'k' or 'v' (fp32 [hd])."""
    g = _gen(device, w.seed, layer, head, "sigma", which)
    sig = torch.exp(0.5 * torch.randn(w.head_dim, generator=g, device=device))
    if which == "k" and w.outliers != "none":
        if w.outliers == "2of64":
            mask = torch.zeros(w.head_dim, dtype=torch.bool, device=device)
            for g0 in range(0, w.head_dim, 64):
                width = min(64, w.head_dim - g0)
                pick = torch.randperm(width, generator=g, device=device)[:2] + g0
                mask[pick] = True
        elif w.outliers == "p0.03":
            mask = torch.rand(w.head_dim, generator=g, device=device) < 0.03
        else:
            raise ValueError(w.outliers)
        sig = torch.where(mask, sig * 10.0, sig)
    return sig


def layer_kv(w: Workload, layer: int, heads: range | None = None, tokens: int | None = None,
             device="cpu") -> tuple[torch.Tensor, torch.Tensor]:
    """Prompt K, V of one layer: fp16 [B, T, H_local, hd] (token-major)."""
    heads = range(w.heads) if heads is None else heads
    T = w.seq_len if tokens is None else tokens
    K = torch.empty((w.batch, T, len(heads), w.head_dim), dtype=torch.float16, device=device)
    V = torch.empty_like(K)
    for i, h in enumerate(heads):
        for which, dst in (("k", K), ("v", V)):
            sig = channel_sigma(w, layer, h, which, device)
            g = _gen(device, w.seed, layer, h, "cache", which)
            z = torch.randn((w.batch, T, w.head_dim), generator=g, device=device)
            dst[:, :, i, :] = (z * sig).to(torch.float16)
    return K, V


def step_inputs(w: Workload, layer: int, step: int, heads: range | None = None,
                device="cpu") -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Decode-step inputs of one layer: new k, v fp16 [B, 1, H_local, hd] and
    q fp16 [B, H_local, hd]."""
    heads = range(w.heads) if heads is None else heads
    k = torch.empty((w.batch, 1, len(heads), w.head_dim), dtype=torch.float16, device=device)
    v = torch.empty_like(k)
    q = torch.empty((w.batch, len(heads), w.head_dim), dtype=torch.float16, device=device)
    for i, h in enumerate(heads):
        for which, dst in (("k", k), ("v", v)):
            sig = channel_sigma(w, layer, h, which, device)
            g = _gen(device, w.seed, layer, h, "tok", step, which)
            z = torch.randn((w.batch, w.head_dim), generator=g, device=device)
            dst[:, 0, i, :] = (z * sig).to(torch.float16)
        g = _gen(device, w.seed, layer, h, "q", step)
        q[:, i, :] = torch.randn((w.batch, w.head_dim), generator=g, device=device).to(torch.float16)
    return k, v, q


def capacity(tokens: int, align: int = 64) -> int:
    """Cache capacity Tc: tokens rounded up to the library's 64-row alignment."""
    return max(align, -(-tokens // align) * align)
