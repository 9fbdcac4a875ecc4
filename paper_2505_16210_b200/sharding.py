"""Head sharding across the GPUs of one node (BASELINE.json
north_star (c)).

Heads are independent in decode attention (PAPER.md:232-235 is per head once
X_K', X_V' are split), so rank r owns a contiguous head range of every layer:
its own codes, scales, q and out.  Quantize and attention need no
communication; the single exchange step is an all-gather of the per-head
outputs [B, H_local, hd] -> [B, H, hd].
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(rank: int, world: int, heads: int, group: int = 1) -> range:
    """Strong scaling: split a fixed head count evenly (heads % world == 0).
    group = heads per quantisation block (blk / hd when blk > hd, the paper's
    blk 256): a shard must hold whole head groups, or a block would straddle
    two ranks."""
    if heads % world:
        raise ValueError(f"{heads} heads do not shard evenly over {world} ranks")
    per = heads // world
    if per % group:
        raise ValueError(f"a {per}-head shard splits {group}-head quantisation blocks")
    return range(rank * per, (rank + 1) * per)


def weak_head_range(rank: int, heads_per_rank: int, group: int = 1) -> range:
    """Weak scaling: every rank owns a fixed shard; the job has world x shard heads."""
    if heads_per_rank % group:
        raise ValueError(f"a {heads_per_rank}-head shard splits {group}-head quantisation blocks")
    return range(rank * heads_per_rank, (rank + 1) * heads_per_rank)


def gather_buffer(out_local: torch.Tensor, world: int) -> torch.Tensor:
    """Receive buffer for all_gather_into_tensor: the rank-major concatenation
    [G*B, H_local, hd] (the layout both NCCL and gloo accept)."""
    B = out_local.shape[0]
    return torch.empty((world * B,) + tuple(out_local.shape[1:]), dtype=out_local.dtype,
                       device=out_local.device)


def all_gather_heads(out_local: torch.Tensor, gathered: torch.Tensor,
                     group=None, async_op: bool = False):
    """all-gather of per-head outputs: out_local [B, H_local, hd] from every
    rank into gathered [G*B, H_local, hd] (rank-major)."""
    return dist.all_gather_into_tensor(gathered, out_local.contiguous(), group=group,
                                       async_op=async_op)


def assemble(gathered: torch.Tensor, world: int) -> torch.Tensor:
    """[G*B, H_local, hd] (rank-major) -> [B, G*H_local, hd] in global head order."""
    GB, Hl, hd = gathered.shape
    B = GB // world
    return gathered.view(world, B, Hl, hd).permute(1, 0, 2, 3).reshape(B, world * Hl, hd)


def step_gather_layer(gathered: torch.Tensor, layer: int) -> torch.Tensor:
    """Per-step gather (one all-gather of every layer's [L, B, H_local, hd]
    outputs, rank-major [G, L, B, H_local, hd]) -> layer `layer`'s
    [G*B, H_local, hd] (rank-major, as assemble takes it)."""
    G, L, B, Hl, hd = gathered.shape
    return gathered[:, layer].reshape(G * B, Hl, hd)
