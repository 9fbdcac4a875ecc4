"""Multi-process (world_size 2, gloo, CPU) check of the head-sharding path
(SURVEY.md 8(e)): every rank regenerates ONLY its own heads from the seeded
generator, computes their decode attention (oracle stands in for the CUDA
kernel, which needs a GPU), and the per-head outputs are all-gathered and
assembled -- the result must equal the unsharded computation exactly."""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import nqkv_oracle as O
from paper_2505_16210_b200 import sharding
from synth import workloads as W

WORK = W.Workload("dist", 1, 2, 8, 64, 96, 64, 1, None, "2of64")
# the paper's blk 256 (reading R2b): 4-head groups at hd 64, one group per rank
WORK256 = dataclasses.replace(WORK, blk=256)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _heads_output(heads, w=WORK):
    K, V = W.layer_kv(w, 0, heads=heads)
    _, _, q = W.step_inputs(w, 0, 0, heads=heads)
    B, T, H, hd = K.shape
    kc, ks = O.empty_cache(B, H, 128, hd, w.blk)
    vc, vs = O.empty_cache(B, H, 128, hd, w.blk)
    O.quantize_append(K.numpy(), [0] * B, w.blk, kc, ks)
    O.quantize_append(V.numpy(), [0] * B, w.blk, vc, vs)
    return O.decode_attention(q.numpy(), kc, ks, vc, vs, [T] * B, w.blk).astype(np.float32)


def _worker(rank, world, port, mode, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = WORK256 if mode == "strong256" else WORK
        group = max(w.blk // w.head_dim, 1)
        if mode in ("strong", "strong256"):
            heads = sharding.head_range(rank, world, w.heads, group)
        else:
            heads = sharding.weak_head_range(rank, w.heads // world, group)
        local = torch.from_numpy(_heads_output(heads, w))
        if mode == "per_step":
            # one all-gather of two "layers" of outputs ([L, B, H_local, hd]),
            # split back per layer (the runtime's per-step gather mode)
            layers = torch.stack([local, 2.0 * local])
            gathered = torch.empty((world * 2,) + tuple(local.shape), dtype=local.dtype)
            sharding.all_gather_heads(layers, gathered)
            g5 = gathered.view((world, 2) + tuple(local.shape))
            full = torch.stack([sharding.assemble(sharding.step_gather_layer(g5, l), world)
                                for l in range(2)])
        else:
            gathered = sharding.gather_buffer(local, world)
            sharding.all_gather_heads(local, gathered)
            full = sharding.assemble(gathered, world)
        if rank == 0:
            torch.save(full, out_path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["strong", "weak", "strong256", "per_step"])
def test_head_sharded_all_gather_matches_unsharded(tmp_path, mode):
    world = 2
    out = str(tmp_path / "full.pt")
    mp.spawn(_worker, args=(world, _free_port(), mode, out), nprocs=world, join=True)
    full = torch.load(out).numpy()
    w = WORK256 if mode == "strong256" else WORK
    ref = _heads_output(range(w.heads), w)
    if mode == "per_step":
        ref = np.stack([ref, 2.0 * ref])
    assert full.shape == ref.shape
    assert np.array_equal(full, ref)


def test_head_range_validation():
    assert list(sharding.head_range(1, 4, 40)) == list(range(10, 20))
    # blk 256 at hd 128 groups heads in pairs: a 10-head shard is fine, 5 is not
    assert list(sharding.head_range(1, 4, 40, group=2)) == list(range(10, 20))
    with pytest.raises(ValueError):
        sharding.head_range(0, 8, 40, group=2)
    with pytest.raises(ValueError):
        sharding.weak_head_range(0, 5, group=4)
    with pytest.raises(ValueError):
        sharding.head_range(0, 3, 40)
    g = torch.arange(2 * 3 * 4 * 5, dtype=torch.float32).reshape(2, 3, 4, 5)
    a = sharding.assemble(g.reshape(6, 4, 5), 2)
    assert a.shape == (3, 8, 5) and torch.equal(a[:, 4:], g[1])
