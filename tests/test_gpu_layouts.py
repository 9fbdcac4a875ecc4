"""KV layouts on the GPU (readings R16, R17):
grouped-query head mapping and the paged cache, through the C ABI's *_kv
calls.  Bars as everywhere: codes and scales bit-exact against the oracle,
attention within 2e-3 of the float64 oracle; and, because a layout only
changes which row is read, the paged kernels must give BIT-IDENTICAL
results to the contiguous ones on the same data (the schedule depends on
(B, H, seq_lens, grid) only)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import nqkv_oracle as O

pytestmark = pytest.mark.gpu
ATOL = 2e-3
DEV = "cuda"


@pytest.fixture(scope="module")
def N():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2505_16210_b200 import nqkv
    assert torch.cuda.is_available()
    return nqkv


def _kv(B, T, H, hd, seed):
    g = torch.Generator().manual_seed(seed)
    sig = torch.exp(0.5 * torch.randn(H, hd, generator=g))
    sig[:, ::29] *= 10                                  # K-style outlier channels
    return (torch.randn(B, T, H, hd, generator=g) * sig).to(torch.float16)


def _contig(N, x, blk, Tc):
    B, T, H, hd = x.shape
    codes = torch.zeros(B, H, Tc, hd // 2, dtype=torch.uint8, device=DEV)
    scales = torch.zeros(N.scales_shape(B, H, Tc, hd, blk), dtype=torch.float32, device=DEV)
    N.nqkv_quantize(x.to(DEV), torch.zeros(B, dtype=torch.int32, device=DEV), codes, scales, blk)
    return codes, scales


def _paged(N, x, blk, P, n_pages, bt, lens_alloc):
    """quantize x into a paged cache via nqkv_quantize_kv (prompt appended in
    two pieces to exercise pos offsets across page boundaries)"""
    B, T, H, hd = x.shape
    hpb = blk // hd if blk > hd else 1
    codes = torch.zeros(n_pages, H, P, hd // 2, dtype=torch.uint8, device=DEV)
    scales = torch.zeros(n_pages, H // hpb, P, max(hd // blk, 1), dtype=torch.float32, device=DEV)
    lay = N.kv_layout(0, bt, P, n_pages)
    Tc = bt.shape[1] * P
    cut = T // 3 + 5
    N.nqkv_quantize_kv(x[:, :cut].contiguous().to(DEV), torch.zeros(B, dtype=torch.int32, device=DEV),
                       codes, scales, blk, lay, Tc)
    N.nqkv_quantize_kv(x[:, cut:].contiguous().to(DEV), torch.full((B,), cut, dtype=torch.int32, device=DEV),
                       codes, scales, blk, lay, Tc)
    return codes, scales


GEOMS = [(64, 32), (64, 64), (64, 256), (128, 32), (128, 64), (128, 128), (128, 256)]


@pytest.mark.parametrize("hd,blk", GEOMS)
@pytest.mark.parametrize("group", [2, 4, 8])
def test_gqa_decode_matches_oracle(N, hd, blk, group):
    hpb = blk // hd if blk > hd else 1
    Hkv = 2 * hpb
    H = Hkv * group
    lens = [0, 1, 700, 1500]
    B, T = len(lens), max(lens)
    Tc = -(-T // 64) * 64
    k, v = _kv(B, T, Hkv, hd, hd + blk), _kv(B, T, Hkv, hd, hd + blk + 1)
    kc, ks = _contig(N, k, blk, Tc)
    vc, vs = _contig(N, v, blk, Tc)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(group)).half()
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    out = N.nqkv_decode_attention_kv(q.to(DEV), kc, ks, vc, vs, L, blk, N.kv_layout(Hkv), Tc, ws)
    torch.cuda.synchronize()
    okc, oks = O.empty_cache(B, Hkv, Tc, hd, blk)
    O.quantize_append(k.numpy(), [0] * B, blk, okc, oks)
    ovc, ovs = O.empty_cache(B, Hkv, Tc, hd, blk)
    O.quantize_append(v.numpy(), [0] * B, blk, ovc, ovs)
    assert np.array_equal(kc.cpu().numpy(), okc) and np.array_equal(vs.cpu().numpy(), ovs)
    ref = O.decode_attention(q.numpy(), okc, oks, ovc, ovs, lens, blk)
    err = np.max(np.abs(out.cpu().numpy().astype(np.float64) - ref))
    assert err <= ATOL, err
    assert not ws.any()                                          # workspace left zero


@pytest.mark.parametrize("hd,blk", [(64, 64), (128, 64), (128, 256)])
def test_gqa_prefill_matches_oracle(N, hd, blk):
    hpb = blk // hd if blk > hd else 1
    Hkv, group = 2 * hpb, 4
    H = Hkv * group
    lens = [0, 1, 65, 300]
    B, T = len(lens), max(lens)
    Tc = 320
    k, v = _kv(B, T, Hkv, hd, 7), _kv(B, T, Hkv, hd, 8)
    kc, ks = _contig(N, k, blk, Tc)
    vc, vs = _contig(N, v, blk, Tc)
    q = torch.randn(B, T, H, hd, generator=torch.Generator().manual_seed(9)).half()
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    out = N.nqkv_prefill_attention_kv(q.to(DEV), kc, ks, vc, vs, L, blk, N.kv_layout(Hkv), Tc)
    torch.cuda.synchronize()
    ref = O.prefill_attention(q.numpy(), kc.cpu().numpy(), ks.cpu().numpy(), vc.cpu().numpy(),
                              vs.cpu().numpy(), lens, blk)
    assert np.max(np.abs(out.cpu().numpy().astype(np.float64) - ref)) <= ATOL


def _table(B, maxp, n_pages, seed):
    rng = np.random.default_rng(seed)
    return torch.tensor(rng.permutation(n_pages)[:B * maxp].reshape(B, maxp), dtype=torch.int32,
                        device=DEV)


@pytest.mark.parametrize("hd,blk", GEOMS)
@pytest.mark.parametrize("P", [64, 256])
def test_paged_quantize_bit_exact(N, hd, blk, P):
    hpb = blk // hd if blk > hd else 1
    H = 2 * hpb
    B, T = 3, 700
    maxp = -(-T // P)
    n_pages = B * maxp + 3                                       # 3 pages nobody uses
    bt = _table(B, maxp, n_pages, P + hd)
    x = _kv(B, T, H, hd, blk)
    codes, scales = _paged(N, x, blk, P, n_pages, bt, T)
    torch.cuda.synchronize()
    Tc = maxp * P
    oc, os_ = O.empty_cache(B, H, Tc, hd, blk)
    O.quantize_append(x.numpy(), [0] * B, blk, oc, os_)
    btn = bt.cpu().numpy()
    assert np.array_equal(codes.cpu().numpy(), O.contiguous_to_paged(oc, btn, P, n_pages))
    assert np.array_equal(scales.cpu().numpy(), O.contiguous_to_paged(os_, btn, P, n_pages))


@pytest.mark.parametrize("hd,blk", GEOMS)
@pytest.mark.parametrize("P", [64, 128])
@pytest.mark.parametrize("group", [1, 4])
def test_paged_decode_equals_contiguous_and_oracle(N, hd, blk, P, group):
    """Paged decode == contiguous decode bit for bit (same rows, same
    schedule), and within 2e-3 of the oracle; ragged lengths crossing pages,
    an empty sequence, GQA on top."""
    hpb = blk // hd if blk > hd else 1
    Hkv = 2 * hpb
    H = Hkv * group
    lens = [0, 1, 63, 64, 65, 700]
    B, T = len(lens), max(lens)
    maxp = -(-T // P)
    n_pages = B * maxp + 1
    bt = _table(B, maxp, n_pages, hd * blk + P)
    Tc = maxp * P
    k, v = _kv(B, T, Hkv, hd, 3 * hd + blk), _kv(B, T, Hkv, hd, 5 * hd + blk)
    pkc, pks = _paged(N, k, blk, P, n_pages, bt, T)
    pvc, pvs = _paged(N, v, blk, P, n_pages, bt, T)
    ckc, cks = _contig(N, k, blk, Tc)
    cvc, cvs = _contig(N, v, blk, Tc)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(P)).half().to(DEV)
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    outp = N.nqkv_decode_attention_kv(q, pkc, pks, pvc, pvs, L, blk,
                                      N.kv_layout(Hkv, bt, P, n_pages), Tc, ws)
    outc = N.nqkv_decode_attention_kv(q, ckc, cks, cvc, cvs, L, blk, N.kv_layout(Hkv), Tc, ws)
    torch.cuda.synchronize()
    assert torch.equal(outp, outc)
    assert not ws.any()
    ref = O.decode_attention(q.cpu().numpy(), ckc.cpu().numpy(), cks.cpu().numpy(), cvc.cpu().numpy(),
                             cvs.cpu().numpy(), lens, blk)
    assert np.max(np.abs(outp.cpu().numpy().astype(np.float64) - ref)) <= ATOL


@pytest.mark.parametrize("hd,blk", [(64, 64), (128, 32), (128, 256)])
def test_paged_prefill_equals_contiguous_and_oracle(N, hd, blk):
    hpb = blk // hd if blk > hd else 1
    Hkv, group = 2 * hpb, 2
    H = Hkv * group
    P = 128
    lens = [0, 1, 129, 300]
    B, T = len(lens), max(lens)
    maxp = -(-T // P)
    n_pages = B * maxp + 2
    bt = _table(B, maxp, n_pages, 11)
    Tc = maxp * P
    k, v = _kv(B, T, Hkv, hd, 21), _kv(B, T, Hkv, hd, 22)
    pkc, pks = _paged(N, k, blk, P, n_pages, bt, T)
    pvc, pvs = _paged(N, v, blk, P, n_pages, bt, T)
    ckc, cks = _contig(N, k, blk, Tc)
    cvc, cvs = _contig(N, v, blk, Tc)
    q = torch.randn(B, T, H, hd, generator=torch.Generator().manual_seed(4)).half().to(DEV)
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    outp = N.nqkv_prefill_attention_kv(q, pkc, pks, pvc, pvs, L, blk, N.kv_layout(Hkv, bt, P, n_pages), Tc)
    outc = N.nqkv_prefill_attention_kv(q, ckc, cks, cvc, cvs, L, blk, N.kv_layout(Hkv), Tc)
    torch.cuda.synchronize()
    assert torch.equal(outp, outc)
    ref = O.prefill_attention(q.cpu().numpy(), ckc.cpu().numpy(), cks.cpu().numpy(), cvc.cpu().numpy(),
                              cvs.cpu().numpy(), lens, blk)
    assert np.max(np.abs(outp.cpu().numpy().astype(np.float64) - ref)) <= ATOL


def test_paged_decode_c5_shape_sampled(N):
    """The c5 shard's shape (64 x 12 heads x 4097 tokens, hd 128, blk 64) on
    a paged cache of 256-token pages in shuffled order: bit-identical to the
    contiguous cache, sampled rows against the oracle."""
    B, H, hd, blk, T, P = 64, 12, 128, 64, 4097, 256
    maxp = -(-T // P)
    n_pages = B * maxp
    bt = _table(B, maxp, n_pages, 5)
    Tc = maxp * P
    g = torch.Generator(device=DEV).manual_seed(3)
    k = torch.randn(B, T, H, hd, generator=g, device=DEV).half()
    v = torch.randn(B, T, H, hd, generator=g, device=DEV).half()
    pkc, pks = _paged(N, k, blk, P, n_pages, bt, T)
    pvc, pvs = _paged(N, v, blk, P, n_pages, bt, T)
    ckc, cks = _contig(N, k, blk, Tc)
    cvc, cvs = _contig(N, v, blk, Tc)
    del k, v
    q = torch.randn(B, H, hd, generator=g, device=DEV).half()
    L = torch.full((B,), T, dtype=torch.int32, device=DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    outp = N.nqkv_decode_attention_kv(q, pkc, pks, pvc, pvs, L, blk, N.kv_layout(0, bt, P, n_pages), Tc, ws)
    outc = N.nqkv_decode_attention(q, ckc, cks, cvc, cvs, L, blk, ws)
    torch.cuda.synchronize()
    assert torch.equal(outp, outc)
    for b in (0, 37, 63):
        ref = O.decode_attention(q[b:b + 1].cpu().numpy(), ckc[b:b + 1].cpu().numpy(), cks[b:b + 1].cpu().numpy(),
                                 cvc[b:b + 1].cpu().numpy(), cvs[b:b + 1].cpu().numpy(), [T], blk)
        assert np.max(np.abs(outp[b:b + 1].cpu().numpy() - ref)) <= ATOL


def test_gqa_decode_c5_shape_sampled(N):
    """The bench's gqa-4 case at full size (64 x 48 query heads over 12 KV
    heads x 4097 tokens, hd 128, blk 64; 3072 CTAs, several chunks per
    group merged across CTAs): the group-native kernel against the oracle
    on sampled sequences (every query head of each), ragged lengths, the
    workspace left zero, and the paged cache bit-identical."""
    B, Hkv, grp, hd, blk, P = 64, 12, 4, 128, 64, 256
    H = Hkv * grp
    rng = np.random.default_rng(11)
    lens = [4097] * B
    lens[5], lens[17], lens[40] = 1, 0, 2500
    T = max(lens)
    maxp = -(-T // P)
    n_pages = B * maxp
    bt = _table(B, maxp, n_pages, 7)
    Tc = maxp * P
    g = torch.Generator(device=DEV).manual_seed(4)
    k = torch.randn(B, T, Hkv, hd, generator=g, device=DEV).half()
    v = torch.randn(B, T, Hkv, hd, generator=g, device=DEV).half()
    ckc, cks = _contig(N, k, blk, Tc)
    cvc, cvs = _contig(N, v, blk, Tc)
    pkc, pks = _paged(N, k, blk, P, n_pages, bt, T)
    pvc, pvs = _paged(N, v, blk, P, n_pages, bt, T)
    del k, v
    q = torch.randn(B, H, hd, generator=g, device=DEV).half()
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    outc = N.nqkv_decode_attention_kv(q, ckc, cks, cvc, cvs, L, blk, N.kv_layout(Hkv), Tc, ws)
    outp = N.nqkv_decode_attention_kv(q, pkc, pks, pvc, pvs, L, blk,
                                      N.kv_layout(Hkv, bt, P, n_pages), Tc, ws)
    torch.cuda.synchronize()
    assert not ws.any()
    assert torch.equal(outp, outc)
    for b in (0, 5, 17, 40, int(rng.integers(0, B)), 63):
        ref = O.decode_attention(q[b:b + 1].cpu().numpy(), ckc[b:b + 1].cpu().numpy(), cks[b:b + 1].cpu().numpy(),
                                 cvc[b:b + 1].cpu().numpy(), cvs[b:b + 1].cpu().numpy(), [lens[b]], blk)
        assert np.max(np.abs(outc[b:b + 1].cpu().numpy() - ref)) <= ATOL


@pytest.mark.parametrize("env", [{"NQKV_GQA_TC": "0"}, {"NQKV_GQA_NATIVE": "0"}])
def test_gqa_alternative_paths_match_oracle(N, env):
    """The non-default grouped-query paths (read once per process from the
    environment, so run in a child process): the group-native kernel with
    FFMA2 scores (NQKV_GQA_TC=0) and the per-query-head MHA kernel
    (NQKV_GQA_NATIVE=0), groups 2/4/8 at hd 64 and 128, within 2e-3 of the
    oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import numpy as np, torch, sys
sys.path.insert(0, %r)
from paper_2505_16210_b200 import nqkv as N
from oracle import nqkv_oracle as O
for hd, blk, group in ((64, 64, 2), (128, 64, 4), (128, 32, 8), (64, 32, 4)):
    Hkv, B, lens = 2, 3, [0, 9, 1300]
    H, T = Hkv * group, max(lens)
    Tc = -(-T // 64) * 64
    g = torch.Generator().manual_seed(hd + blk + group)
    k = torch.randn(B, T, Hkv, hd, generator=g).half()
    v = torch.randn(B, T, Hkv, hd, generator=g).half()
    q = torch.randn(B, H, hd, generator=g).half()
    kc = torch.zeros(B, Hkv, Tc, hd // 2, dtype=torch.uint8, device="cuda")
    ks = torch.zeros(B, Hkv, Tc, hd // blk, device="cuda")
    vc, vs = torch.zeros_like(kc), torch.zeros_like(ks)
    z = torch.zeros(B, dtype=torch.int32, device="cuda")
    N.nqkv_quantize(k.cuda(), z, kc, ks, blk)
    N.nqkv_quantize(v.cuda(), z, vc, vs, blk)
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    ws = N.make_workspace(B, H, hd, Tc, "cuda")
    out = N.nqkv_decode_attention_kv(q.cuda(), kc, ks, vc, vs, L, blk, N.kv_layout(Hkv), Tc, ws)
    torch.cuda.synchronize()
    ref = O.decode_attention(q.numpy(), kc.cpu().numpy(), ks.cpu().numpy(), vc.cpu().numpy(),
                             vs.cpu().numpy(), lens, blk)
    err = float(np.max(np.abs(out.cpu().numpy().astype(np.float64) - ref)))
    assert err <= 2e-3, (hd, blk, group, err)
    assert not ws.any()
print("ok")
''' % root
    r = subprocess.run([sys.executable, "-c", script], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("hd,blk", [(64, 64), (128, 32), (128, 128)])
def test_gqa_decode_fp16_scales_equals_fp32(N, hd, blk):
    """Grouped-query decode over a cache with fp16 block scales (lossless for
    fp16 inputs) is BIT-IDENTICAL to the fp32-scale cache's (the same
    group-native kernel reads the same scale values), within 2e-3 of the
    oracle, the workspace left zero."""
    Hkv, group = 2, 4
    H = Hkv * group
    lens = [0, 1, 333, 1200]
    B, T = len(lens), max(lens)
    Tc = -(-T // 64) * 64
    k, v = _kv(B, T, Hkv, hd, 21), _kv(B, T, Hkv, hd, 22)
    kc, ks = _contig(N, k, blk, Tc)
    vc, vs = _contig(N, v, blk, Tc)
    ks16, vs16 = ks.half(), vs.half()             # exact: every scale is an fp16 absmax
    assert torch.equal(ks16.float(), ks) and torch.equal(vs16.float(), vs)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(23)).half().to(DEV)
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    o16 = N.nqkv_decode_attention_kv(q, kc, ks16, vc, vs16, L, blk, N.kv_layout(Hkv), Tc, ws)
    o32 = N.nqkv_decode_attention_kv(q, kc, ks, vc, vs, L, blk, N.kv_layout(Hkv), Tc, ws)
    torch.cuda.synchronize()
    assert not ws.any()
    ref = O.decode_attention(q.cpu().numpy(), kc.cpu().numpy(), ks.cpu().numpy(), vc.cpu().numpy(),
                             vs.cpu().numpy(), lens, blk)
    assert torch.equal(o16, o32)
    assert np.max(np.abs(o32.cpu().numpy().astype(np.float64) - ref)) <= ATOL
