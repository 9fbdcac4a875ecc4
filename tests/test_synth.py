"""Seeded synthetic inputs: deterministic, shard-invariant, shaped like the
BASELINE.json configs (CPU only)."""
import torch

from synth import workloads as W


def test_shapes_and_determinism():
    w = W.CONFIGS["c1"]
    k1, v1 = W.layer_kv(w, 0)
    k2, v2 = W.layer_kv(w, 0)
    assert k1.shape == (1, 512, 12, 64) and k1.dtype == torch.float16
    assert torch.equal(k1, k2) and torch.equal(v1, v2)
    assert not torch.equal(k1, v1)


def test_head_shard_regenerates_same_data():
    w = W.Workload("t", 2, 2, 8, 64, 32, 64, 1, None, "2of64")
    kf, vf = W.layer_kv(w, 1)
    ks, vs = W.layer_kv(w, 1, heads=range(4, 8))
    assert torch.equal(kf[:, :, 4:8], ks) and torch.equal(vf[:, :, 4:8], vs)
    a = W.step_inputs(w, 1, 3)
    b = W.step_inputs(w, 1, 3, heads=range(2, 6))
    for x, y in zip(a[:2], b[:2]):
        assert torch.equal(x[:, :, 2:6], y)
    assert torch.equal(a[2][:, 2:6], b[2])


def test_outlier_channels():
    w = W.CONFIGS["c2"]
    sk = W.channel_sigma(w, 0, 0, "k")
    sv = W.channel_sigma(w, 0, 0, "v")
    base = W.channel_sigma(W.Workload("x", 24, 8, 32, 64, 2048), 0, 0, "k")
    assert int((sk / base > 5).sum()) == 2          # 2 of every 64 K channels x10
    assert int((sv > 20).sum()) <= 1                 # V: plain LogNormal(0, .5)


def test_ragged_lengths():
    w = W.CONFIGS["c3"]
    L = W.seq_lens(w)
    assert L.shape == (32,) and int(L.min()) >= 1024 and int(L.max()) <= 2048
    assert torch.equal(L, W.seq_lens(w))
    assert W.capacity(2049) == 2112 and W.capacity(0) == 64
