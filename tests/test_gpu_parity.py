"""GPU-vs-oracle parity through the C ABI (needs a B200).

Bars (BASELINE.json north_star): codes, scales and dequantised values
bit-exact; attention max-abs error <= 2e-3 against the oracle's float64
attention over the same dequantised cache."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest
import torch

from oracle import nqkv_oracle as O
from synth import workloads as W

pytestmark = pytest.mark.gpu
ATOL = 2e-3
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def N():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2505_16210_b200 import nqkv
    assert torch.cuda.is_available()
    return nqkv


DEV = "cuda"


def _rand_kv(B, T, H, hd, seed, outlier=True):
    g = torch.Generator().manual_seed(seed)
    sig = torch.exp(0.5 * torch.randn(H, hd, generator=g))
    if outlier:
        sig[:, ::37] *= 10
    x = (torch.randn(B, T, H, hd, generator=g) * sig).to(torch.float16)
    return x


def _hpb(hd, blk):
    """heads per block: blk > hd spans blk/hd adjacent heads (paper's blk 256)"""
    return blk // hd if blk > hd else 1


def _oracle_cache(x, pos, blk, Tc, codes=None, scales=None):
    B, n, H, hd = x.shape
    if codes is None:
        codes, scales = O.empty_cache(B, H, Tc, hd, blk)
    O.quantize_append(x.numpy(), pos, blk, codes, scales)
    return codes, scales


# ------------------------------------------------------------ code function
def test_encode_normalized_matches_oracle(N):
    cand = []
    for t in list(O.thresholds_f32()) + [np.float32((k - 16.5) / 16) for k in range(34)]:
        v = np.float32(t)
        for _ in range(64):
            v = np.nextafter(v, np.float32(-2))
        for _ in range(128):
            cand.append(v)
            v = np.nextafter(v, np.float32(2))
    rng = np.random.default_rng(0)
    n = np.concatenate([np.clip(np.array(cand, np.float32), -1, 1),
                        rng.uniform(-1, 1, 1 << 20).astype(np.float32),
                        np.array([-1.0, 1.0, 0.0, -0.0], np.float32)])
    got = N.nqkv_encode_normalized(torch.from_numpy(n).to(DEV)).cpu().numpy()
    assert np.array_equal(got, O.nearest_level_codes(n))


# ----------------------------------------------------------------- quantize
@pytest.mark.parametrize("hd,blk", [(64, 32), (64, 64), (128, 32), (128, 64), (128, 128),
                                    (64, 128), (64, 256), (128, 256)])
def test_quantize_bit_exact(N, hd, blk):
    B, T = 3, 200
    H = 5 if blk <= hd else 3 * _hpb(hd, blk)
    Tc = 256
    x = _rand_kv(B, T, H, hd, seed=hd + blk)
    sshape = N.scales_shape(B, H, Tc, hd, blk)
    codes = torch.full((B, H, Tc, hd // 2), 0xAB, dtype=torch.uint8, device=DEV)
    scales = torch.full(sshape, -7.0, dtype=torch.float32, device=DEV)
    pos = torch.tensor([0, 17, 56], dtype=torch.int32)
    N.nqkv_quantize(x.to(DEV), pos.to(DEV), codes, scales, blk)
    oc = np.full((B, H, Tc, hd // 2), 0xAB, np.uint8)
    os_ = np.full(sshape, -7.0, np.float32)
    _oracle_cache(x, pos.tolist(), blk, Tc, oc, os_)
    assert np.array_equal(codes.cpu().numpy(), oc)            # incl. untouched bytes
    assert np.array_equal(scales.cpu().numpy(), os_)


def test_quantize_strided_input_and_zero_blocks(N):
    B, T, H, hd, blk, Tc = 2, 33, 4, 128, 64, 64
    big = _rand_kv(B, T, H + 3, hd + 64, seed=5)             # padded buffer -> strided view
    x = big[:, :, 1:H + 1, 32:32 + hd]
    x[:, 3, 2, :64] = 0                                       # an all-zero block
    x[:, 4, 1, :] = -0.0
    codes = torch.zeros((B, H, Tc, hd // 2), dtype=torch.uint8, device=DEV)
    scales = torch.zeros((B, H, Tc, hd // blk), dtype=torch.float32, device=DEV)
    xd = big.to(DEV)[:, :, 1:H + 1, 32:32 + hd]
    N.nqkv_quantize(xd, torch.zeros(B, dtype=torch.int32, device=DEV), codes, scales, blk)
    oc, os_ = _oracle_cache(x.contiguous(), [0, 0], blk, Tc)
    c = codes.cpu().numpy()
    assert np.array_equal(c, oc) and np.array_equal(scales.cpu().numpy(), os_)
    assert np.all(c[:, 2, 3, :32] == 0x77) and np.all(scales.cpu().numpy()[:, 2, 3, 0] == 0)


@pytest.mark.parametrize("hd", [64, 128])
def test_quantize_strided_head_groups(N, hd):
    # blk 256 over a strided view (heads not adjacent in memory): the block is
    # still the token's slice of 256/hd logical heads
    B, T, H, blk, Tc = 2, 37, 8, 256, 64
    big = _rand_kv(B, T, H + 2, hd + 32, seed=7 + hd)
    x = big[:, :, 1:H + 1, 16:16 + hd]
    codes = torch.zeros((B, H, Tc, hd // 2), dtype=torch.uint8, device=DEV)
    scales = torch.zeros(N.scales_shape(B, H, Tc, hd, blk), dtype=torch.float32, device=DEV)
    xd = big.to(DEV)[:, :, 1:H + 1, 16:16 + hd]
    N.nqkv_quantize(xd, torch.tensor([0, 20], dtype=torch.int32, device=DEV), codes, scales, blk)
    oc, os_ = _oracle_cache(x.contiguous(), [0, 20], blk, Tc)
    assert np.array_equal(codes.cpu().numpy(), oc) and np.array_equal(scales.cpu().numpy(), os_)


def test_quantize_streaming_equivalence(N):
    # bulk prefill == prefix + one-token appends, byte for byte
    B, T, H, hd, blk, Tc = 2, 48, 3, 64, 64, 64
    x = _rand_kv(B, T, H, hd, seed=9).to(DEV)
    a_c = torch.zeros((B, H, Tc, hd // 2), dtype=torch.uint8, device=DEV)
    a_s = torch.zeros((B, H, Tc, 1), dtype=torch.float32, device=DEV)
    N.nqkv_quantize(x, torch.zeros(B, dtype=torch.int32, device=DEV), a_c, a_s, blk)
    b_c, b_s = torch.zeros_like(a_c), torch.zeros_like(a_s)
    N.nqkv_quantize(x[:, :20], torch.zeros(B, dtype=torch.int32, device=DEV), b_c, b_s, blk)
    for t in range(20, T):
        N.nqkv_quantize(x[:, t:t + 1], torch.full((B,), t, dtype=torch.int32, device=DEV), b_c, b_s, blk)
    assert torch.equal(a_c, b_c) and torch.equal(a_s, b_s)


def test_near_threshold_golden_pairs(N):
    rows = [l.split() for l in open(os.path.join(HERE, "golden", "near_threshold_pairs.txt"))
            if not l.startswith("#")]
    xs = np.array([int(r[0], 16) for r in rows], np.uint16).view(np.float16)
    ss = np.array([int(r[1], 16) for r in rows], np.uint16).view(np.float16)
    want = np.array([int(r[2]) for r in rows], np.uint8)
    blocks = np.zeros((len(rows), 64), np.float16)
    blocks[:, 0] = ss
    blocks[:, 1] = xs
    x = torch.from_numpy(blocks).reshape(1, len(rows), 1, 64).to(DEV)
    Tc = -(-len(rows) // 64) * 64
    codes = torch.zeros((1, 1, Tc, 32), dtype=torch.uint8, device=DEV)
    scales = torch.zeros((1, 1, Tc, 1), dtype=torch.float32, device=DEV)
    N.nqkv_quantize(x, torch.zeros(1, dtype=torch.int32, device=DEV), codes, scales, 64)
    got = (codes.cpu().numpy()[0, 0, :len(rows), 0] >> 4)
    assert np.array_equal(got, want)
    assert len(rows) == 178


def _sweep(N, s_bits):
    """All fp16 x with |x| <= s for each scale s: block {s, x_1..x_63}; GPU
    codes vs the oracle's threshold code of RN32(x/s)."""
    allx = np.arange(0, 0x10000, dtype=np.uint32).astype(np.uint16).view(np.float16)
    allx = allx[np.isfinite(allx)]
    order = np.argsort(np.abs(allx.astype(np.float32)), kind="stable")
    ax, xs_all = np.abs(allx.astype(np.float32))[order], allx[order]
    L = O.nf_levels_f32()
    blocks, want = [], []
    for sb in s_bits:
        s = np.array([sb], np.uint16).view(np.float16)[0]
        xs = xs_all[:np.searchsorted(ax, np.float32(s), side="right")]
        pad = (-len(xs)) % 63
        xs = np.concatenate([xs, np.zeros(pad, np.float16)]).reshape(-1, 63)
        blk = np.concatenate([np.full((len(xs), 1), s, np.float16), xs], axis=1)
        blocks.append(blk)
        n = (blk.astype(np.float32) / np.float32(s)).astype(np.float32)
        want.append(O.codes_by_threshold(n, L))
    blocks = np.concatenate(blocks)
    want = np.concatenate(want)
    total = len(blocks)
    Tc = -(-total // 64) * 64
    x = torch.from_numpy(blocks).reshape(1, total, 1, 64).to(DEV)
    codes = torch.zeros((1, 1, Tc, 32), dtype=torch.uint8, device=DEV)
    scales = torch.zeros((1, 1, Tc, 1), dtype=torch.float32, device=DEV)
    N.nqkv_quantize(x, torch.zeros(1, dtype=torch.int32, device=DEV), codes, scales, 64)
    c = codes.cpu().numpy()[0, 0, :total]
    got = np.empty((total, 64), np.uint8)
    got[:, 0::2] = c & 0xF
    got[:, 1::2] = c >> 4
    mism = int(np.count_nonzero(got != want))
    assert mism == 0, f"{mism} code mismatches"
    return total * 63


def test_fp16_pair_sweep_sampled(N):
    # every 97th positive finite fp16 scale (incl. subnormals) + edge scales,
    # each against EVERY fp16 x with |x| <= s
    s_bits = sorted(set(list(range(1, 0x7C00, 97)) + [1, 0x3C00, 0x7BFF, 0x0400, 0x03FF]))
    _sweep(N, s_bits)


def test_fp16_pair_sweep_exhaustive(N):
    # every positive finite fp16 scale against every |x| <= s: ~1.0e9 pairs
    done = 0
    for lo in range(1, 0x7C00, 1024):
        done += _sweep(N, range(lo, min(lo + 1024, 0x7C00)))
    assert done >= 1007713278


# --------------------------------------------------------------- dequantize
@pytest.mark.parametrize("hd,blk", [(64, 64), (128, 32), (128, 128), (64, 256), (128, 256)])
def test_dequantize_bit_exact(N, hd, blk):
    B, T, Tc = 2, 130, 192
    H = 3 if blk <= hd else 2 * _hpb(hd, blk)
    x = _rand_kv(B, T, H, hd, seed=3)
    oc, os_ = _oracle_cache(x, [0, 0], blk, Tc)
    c, s = torch.from_numpy(oc).to(DEV), torch.from_numpy(os_).to(DEV)
    for dt, ndt in ((torch.float32, np.float32), (torch.float16, np.float16)):
        got = N.nqkv_dequantize(c, s, blk, T, out_dtype=dt).cpu().numpy()
        want = O.dequantize(oc, os_, blk, T, out_dtype=ndt)
        assert got.dtype == want.dtype and np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_dequantize_fp16_every_scale_code_pair(N):
    """All 31,743 positive finite fp16 scales x 16 codes (507,888 pairs, plus
    s = 0) through nqkv_dequantize with fp16 output: RN16(RN32(s * L[c])),
    bit for bit (57 of these pairs differ from RN16(s * L))."""
    s = np.arange(1, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32)
    s = np.concatenate([s, np.zeros(1, np.float32)])
    Tc = -(-s.size // 64) * 64
    scales = np.zeros((1, 1, Tc, 2), np.float32)            # hd 64, blk 32: two blocks per row
    scales[0, 0, :s.size, 0] = s
    scales[0, 0, :s.size, 1] = s
    codes = np.arange(64, dtype=np.uint8) % 16              # every code in both blocks
    packed = O.pack_nibbles(np.broadcast_to(codes, (1, 1, Tc, 64)).copy())
    got = N.nqkv_dequantize(torch.from_numpy(packed).to(DEV), torch.from_numpy(scales).to(DEV), 32,
                            s.size, out_dtype=torch.float16).cpu().numpy()
    want = O.dequantize(packed, scales, 32, s.size, out_dtype=np.float16)
    assert np.array_equal(got.view(np.uint16), want.view(np.uint16))
    # the double-rounding cases are really in the sweep
    exact16 = (s[:, None].astype(np.float64) * O.nf_levels_f32()[None, :].astype(np.float64)).astype(np.float16)
    assert np.count_nonzero(want[0, 0, :, :16].view(np.uint16) != exact16.view(np.uint16)) > 0


# ---------------------------------------------------------------- attention
def _attn_case(N, B, H, hd, blk, lens, Tc, seed, outlier=True, dev_ws=None):
    T = max(max(lens), 1)
    k = _rand_kv(B, T, H, hd, seed, outlier)
    v = _rand_kv(B, T, H, hd, seed + 1, False)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(seed + 2)).to(torch.float16)
    kc, ks = _oracle_cache(k, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(v, [0] * B, blk, Tc)
    ref = O.decode_attention(q.numpy(), kc, ks, vc, vs, lens, blk)
    t = lambda a: torch.from_numpy(a).to(DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    out = N.nqkv_decode_attention(q.to(DEV), t(kc), t(ks), t(vc), t(vs),
                                  torch.tensor(lens, dtype=torch.int32, device=DEV), blk, ws)
    torch.cuda.synchronize()
    assert torch.count_nonzero(ws) == 0       # counters and partial records reset
    return out.cpu().numpy(), ref, (q, kc, ks, vc, vs)


@pytest.mark.parametrize("hd,blk", [(64, 32), (64, 64), (128, 32), (128, 64), (128, 128),
                                    (64, 128), (64, 256), (128, 256)])
def test_attention_ragged_lengths(N, hd, blk):
    lens = [0, 1, 63, 64, 65, 127, 128, 129, 300, 511, 512]
    H = 3 if blk <= hd else 2 * _hpb(hd, blk)
    out, ref, _ = _attn_case(N, len(lens), H, hd, blk, lens, 512, seed=hd * 7 + blk)
    err = np.max(np.abs(out.astype(np.float64) - ref))
    assert err <= ATOL, err
    assert np.all(out[0] == 0)                                # empty sequence


def test_attention_c1_full(N):
    w = W.CONFIGS["c1"]
    K, V = W.layer_kv(w, 0)
    _, _, q = W.step_inputs(w, 0, 0)
    Tc = 512
    kc, ks = _oracle_cache(K, [0], w.blk, Tc)
    vc, vs = _oracle_cache(V, [0], w.blk, Tc)
    cache = N.KVCache(1, w.heads, w.head_dim, Tc, w.blk, DEV)
    cache.append(K.to(DEV), V.to(DEV), torch.zeros(1, dtype=torch.int32, device=DEV))
    assert np.array_equal(cache.k_codes.cpu().numpy(), kc)
    assert np.array_equal(cache.v_scales.cpu().numpy(), vs)
    ws = N.make_workspace(1, w.heads, w.head_dim, Tc, DEV)
    out = cache.attend(q.to(DEV), torch.tensor([512], dtype=torch.int32, device=DEV), ws)
    ref = O.decode_attention(q.numpy(), kc, ks, vc, vs, [512], w.blk)
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= ATOL


def test_attention_closed_forms(N):
    # identical keys -> mean of dequantised values; single token -> that value
    B, H, hd, blk, Tc, T = 1, 2, 128, 64, 256, 200
    k = _rand_kv(1, 1, H, hd, 11).repeat(1, T, 1, 1)
    v = _rand_kv(1, T, H, hd, 12)
    q = torch.randn(B, H, hd).to(torch.float16)
    kc, ks = _oracle_cache(k, [0], blk, Tc)
    vc, vs = _oracle_cache(v, [0], blk, Tc)
    t = lambda a: torch.from_numpy(a).to(DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    for L in (1, T):
        out = N.nqkv_decode_attention(q.to(DEV), t(kc), t(ks), t(vc), t(vs),
                                      torch.tensor([L], dtype=torch.int32, device=DEV), blk, ws)
        mean = O.dequantize(vc, vs, blk, L).astype(np.float64).mean(axis=2)
        assert np.max(np.abs(out.cpu().numpy() - mean)) < 1e-5


def test_attention_invariances_bit_exact(N):
    # bit-identical across Tc and across repeated calls; a head shard of the
    # same data is split over CTAs differently, so it may differ by fp32
    # reassociation only (reading R7)
    B, H, hd, blk = 4, 6, 128, 64
    lens = [700, 64, 1000, 1]
    out1, ref, (q, kc, ks, vc, vs) = _attn_case(N, B, H, hd, blk, lens, 1024, seed=21)
    assert np.max(np.abs(out1 - ref)) <= ATOL
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    L = torch.tensor(lens, dtype=torch.int32, device=DEV)
    # larger capacity, same content
    pad = lambda a: np.concatenate([a, np.zeros(a.shape[:2] + (1024,) + a.shape[3:], a.dtype)], 2)
    ws2 = N.make_workspace(B, H, hd, 2048, DEV)
    out2 = N.nqkv_decode_attention(q.to(DEV), t(pad(kc)), t(pad(ks)), t(pad(vc)), t(pad(vs)), L, blk, ws2)
    assert np.array_equal(out1, out2.cpu().numpy())
    # head shard [2:5) alone
    ws3 = N.make_workspace(B, 3, hd, 1024, DEV)
    out3 = N.nqkv_decode_attention(q[:, 2:5].contiguous().to(DEV), t(kc[:, 2:5]), t(ks[:, 2:5]),
                                   t(vc[:, 2:5]), t(vs[:, 2:5]), L, blk, ws3)
    assert np.max(np.abs(out1[:, 2:5] - out3.cpu().numpy())) <= 1e-6
    for _ in range(3):
        again = N.nqkv_decode_attention(q.to(DEV), t(kc), t(ks), t(vc), t(vs), L, blk,
                                        N.make_workspace(B, H, hd, 1024, DEV))
        assert np.array_equal(out1, again.cpu().numpy())


@pytest.mark.parametrize("hd", [64, 128])
def test_head_group_shard_matches_unsharded(N, hd):
    # blk 256 (R2b): a head shard holding whole head groups sees its groups'
    # scale rows; its output equals the unsharded run's heads (fp32
    # reassociation only, reading R7) and both match the oracle
    blk, B = 256, 3
    hpb = blk // hd
    H = 3 * hpb
    lens = [900, 1, 333]
    out1, ref, (q, kc, ks, vc, vs) = _attn_case(N, B, H, hd, blk, lens, 1024, seed=61 + hd)
    assert np.max(np.abs(out1 - ref)) <= ATOL
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    h0, h1 = hpb, 3 * hpb                                     # groups 1 and 2
    g0, g1 = 1, 3
    out2 = N.nqkv_decode_attention(q[:, h0:h1].contiguous().to(DEV), t(kc[:, h0:h1]), t(ks[:, g0:g1]),
                                   t(vc[:, h0:h1]), t(vs[:, g0:g1]),
                                   torch.tensor(lens, dtype=torch.int32, device=DEV), blk,
                                   N.make_workspace(B, h1 - h0, hd, 1024, DEV))
    # different CTA splits sum in a different order: a few fp32 ulps of |out|
    assert np.allclose(out1[:, h0:h1], out2.cpu().numpy(), rtol=1e-5, atol=1e-6)


def test_attention_max_capacity_long(N):
    # c4-like long row (8192 tokens, 128 splits) on a few heads
    B, H, hd, blk, Tc = 1, 2, 128, 64, 8192
    out, ref, _ = _attn_case(N, B, H, hd, blk, [8192], Tc, seed=31)
    assert np.max(np.abs(out - ref)) <= ATOL


# --------------------------------------------- full-size configs, sampled
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_full_size_layer_sampled(N, cfg):
    """One layer at the config's full size, generated and quantised on the GPU
    in the bench's launch configuration; the oracle checks sampled (b, h)
    slabs: codes/scales bit-exact and the decode output."""
    w = W.CONFIGS[cfg]
    B, H, hd, blk = w.batch, w.heads, w.head_dim, w.blk
    lens = W.seq_lens(w)
    T = int(lens.max())
    Tc = W.capacity(T + 1)
    if cfg == "c5":
        H = 12                       # one 8-GPU head shard of OPT-175B (all 64 x 4096 tokens)
    free = torch.cuda.mem_get_info()[0]
    need = 2 * B * T * H * hd * 2 * 2 + 2 * B * H * Tc * (hd // 2 + 4 * hd // blk)
    if need > 0.8 * free:
        pytest.skip("not enough device memory")
    heads = range(H)
    K, V = W.layer_kv(w, 0, heads=heads, tokens=T, device=DEV)
    k1, v1, q = W.step_inputs(w, 0, 0, heads=heads, device=DEV)
    cache = N.KVCache(B, H, hd, Tc, blk, DEV)
    cache.append(K, V, torch.zeros(B, dtype=torch.int32, device=DEV))
    cache.append(k1, v1, lens.to(DEV))                     # new token at row len_b
    L = (lens + 1).to(DEV)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    out = cache.attend(q, L, ws).cpu().numpy()
    rng = np.random.default_rng(0)
    for b, h in {(0, 0), (B - 1, H - 1)} | {(int(rng.integers(B)), int(rng.integers(H))) for _ in range(2)}:
        n = int(lens[b])
        kx = torch.cat([K[b:b + 1, :n, h:h + 1], k1[b:b + 1, :, h:h + 1]], 1).cpu()
        vx = torch.cat([V[b:b + 1, :n, h:h + 1], v1[b:b + 1, :, h:h + 1]], 1).cpu()
        kc, ks = _oracle_cache(kx, [0], blk, Tc)
        vc, vs = _oracle_cache(vx, [0], blk, Tc)
        assert np.array_equal(cache.k_codes[b, h, :n + 1].cpu().numpy(), kc[0, 0, :n + 1])
        assert np.array_equal(cache.v_scales[b, h, :n + 1].cpu().numpy(), vs[0, 0, :n + 1])
        ref = O.decode_attention(q[b:b + 1, h:h + 1].cpu().numpy(), kc, ks, vc, vs, [n + 1], blk)
        assert np.max(np.abs(out[b, h] - ref[0, 0])) <= ATOL
    del K, V, cache
    torch.cuda.empty_cache()


# ------------------------------------------------- fused append + attention
@pytest.mark.parametrize("hd,blk", [(64, 64), (64, 32), (128, 64), (128, 128), (64, 256), (128, 256)])
def test_decode_step_fused_matches_separate_calls(N, hd, blk):
    """nqkv_decode_step == nqkv_quantize(n_new=1) + nqkv_decode_attention:
    identical cache bytes, output within 2e-3 of the oracle, and equal to the
    unfused attention on the updated cache up to fp32 reassociation (the fused
    kernel folds the appended token into the merge; reading R7)."""
    B, Tc = 5, 512
    H = 3 if blk <= hd else 2 * _hpb(hd, blk)
    lens0 = [0, 1, 127, 128, 300]           # cached tokens before the step
    T = max(lens0)
    x = _rand_kv(B, max(T, 1), H, hd, seed=41)
    y = _rand_kv(B, max(T, 1), H, hd, seed=42, outlier=False)
    kn = _rand_kv(B, 1, H, hd, seed=43)[:, 0]
    vn = _rand_kv(B, 1, H, hd, seed=44, outlier=False)[:, 0]
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(45)).to(torch.float16)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    # stale data beyond len must not leak: rows >= len hold the prompt's later tokens
    t = lambda a: torch.from_numpy(a.copy()).to(DEV)
    lens = torch.tensor([n + 1 for n in lens0], dtype=torch.int32, device=DEV)
    fk, fks, fv, fvs = t(kc), t(ks), t(vc), t(vs)
    ws = N.make_workspace(B, H, hd, Tc, DEV)
    out_f = N.nqkv_decode_step(kn.to(DEV), vn.to(DEV), q.to(DEV), fk, fks, fv, fvs, lens, blk, ws)
    # separate calls
    sk, sks, sv, svs = t(kc), t(ks), t(vc), t(vs)
    pos = torch.tensor(lens0, dtype=torch.int32, device=DEV)
    N.nqkv_quantize(kn.to(DEV).unsqueeze(1), pos, sk, sks, blk)
    N.nqkv_quantize(vn.to(DEV).unsqueeze(1), pos, sv, svs, blk)
    out_s = N.nqkv_decode_attention(q.to(DEV), sk, sks, sv, svs, lens, blk, N.make_workspace(B, H, hd, Tc, DEV))
    torch.cuda.synchronize()
    assert torch.equal(fk, sk) and torch.equal(fks, sks) and torch.equal(fv, sv) and torch.equal(fvs, svs)
    assert torch.allclose(out_f, out_s, rtol=1e-5, atol=1e-6)
    O.quantize_append(kn.unsqueeze(1).numpy(), lens0, blk, kc, ks)
    O.quantize_append(vn.unsqueeze(1).numpy(), lens0, blk, vc, vs)
    assert np.array_equal(fk.cpu().numpy(), kc) and np.array_equal(fvs.cpu().numpy(), vs)
    ref = O.decode_attention(q.numpy(), kc, ks, vc, vs, [n + 1 for n in lens0], blk)
    assert np.max(np.abs(out_f.cpu().numpy() - ref)) <= ATOL
    assert torch.count_nonzero(ws) == 0


def test_decode_runner_graph_matches_oracle(N):
    """The bench's runtime (CUDA-graph replay of fused steps over layers)
    reproduces the oracle on a reduced c2-shaped model."""
    from paper_2505_16210_b200.runtime import DecodeRunner
    w = W.Workload("t", 3, 2, 4, 64, 200, 64, 3, None, "2of64")
    run = DecodeRunner(w, range(w.heads), DEV, gen_device="cpu")
    run.prefill()
    run.step(0)
    run.capture(timing_slots=(1,))
    for s in range(1, 3):
        run.replay(s)
    torch.cuda.synchronize()
    lens = W.seq_lens(w).tolist()
    for l in range(w.layers):
        K, V = W.layer_kv(w, l)
        Tc = run.Tc
        kc, ks = _oracle_cache(K, [0] * w.batch, w.blk, Tc)
        vc, vs = _oracle_cache(V, [0] * w.batch, w.blk, Tc)
        for s in range(3):
            k1, v1, q = W.step_inputs(w, l, s)
            O.quantize_append(k1.numpy(), [n + s for n in lens], w.blk, kc, ks)
            O.quantize_append(v1.numpy(), [n + s for n in lens], w.blk, vc, vs)
        assert np.array_equal(run.caches[l].k_codes.cpu().numpy(), kc)
        assert np.array_equal(run.caches[l].v_scales.cpu().numpy(), vs)
        ref = O.decode_attention(q.numpy(), kc, ks, vc, vs, [n + 3 for n in lens], w.blk)
        assert np.max(np.abs(run.out[l].cpu().numpy() - ref)) <= ATOL
    assert all(t > 0 for t in run.decode_kernel_ms())


@pytest.mark.parametrize("cfg", ["c2", "c5"])
def test_bench_path_full_size(N, cfg):
    """The exact path bench.py times -- DecodeRunner with the per-step plan,
    fused append + attention, NQKV_EARLY_START on layers 1.. and CUDA-graph
    replay -- at the config's full per-launch size (c5: the 12-head shard,
    B 64, 4096 tokens), inputs generated on the GPU as in the bench.  Every
    cache byte of the checked (layer, b, h) slabs and their outputs against
    the oracle; all step slots replayed in order."""
    from paper_2505_16210_b200.runtime import DecodeRunner
    w = W.CONFIGS[cfg]
    layers = 3 if cfg == "c5" else w.layers
    heads = range(12) if cfg == "c5" else range(w.heads)
    free = torch.cuda.mem_get_info()[0]
    T = int(W.seq_lens(w).max())
    per_layer = 2 * w.batch * len(heads) * W.capacity(T + w.decode_steps) * (w.head_dim // 2 + 4 * w.head_dim // w.blk)
    if layers * per_layer + 3 * w.batch * T * len(heads) * w.head_dim * 2 > 0.8 * free:
        pytest.skip("not enough device memory")
    run = DecodeRunner(w, heads, DEV, layers=layers)
    run.prefill()
    run.step(0)                         # eager warm-up (slot 0)
    run.capture(timing_slots=())
    for s in range(run.S):              # graph replays of every slot, in order
        run.replay(s)
    torch.cuda.synchronize()
    assert torch.count_nonzero(run.ws) == 0
    lens = W.seq_lens(w).tolist()
    S = run.S
    rng = np.random.default_rng(7)
    H = len(heads)
    picks = {(0, 0, 0), (layers - 1, w.batch - 1, H - 1)}
    picks |= {(int(rng.integers(layers)), int(rng.integers(w.batch)), int(rng.integers(H))) for _ in range(6)}
    for l, b, h in sorted(picks):
        n = lens[b]
        K, V = W.layer_kv(w, l, heads=range(heads[h], heads[h] + 1), tokens=T, device=DEV)
        kx, vx = [K[b:b + 1, :n].cpu()], [V[b:b + 1, :n].cpu()]
        for s in range(S):
            k1, v1, q = W.step_inputs(w, l, s, heads=range(heads[h], heads[h] + 1), device=DEV)
            kx.append(k1[b:b + 1].cpu())
            vx.append(v1[b:b + 1].cpu())
        kc, ks = _oracle_cache(torch.cat(kx, 1), [0], w.blk, run.Tc)
        vc, vs = _oracle_cache(torch.cat(vx, 1), [0], w.blk, run.Tc)
        c = run.caches[l]
        m = n + S
        assert np.array_equal(c.k_codes[b, h, :m].cpu().numpy(), kc[0, 0, :m])
        assert np.array_equal(c.v_codes[b, h, :m].cpu().numpy(), vc[0, 0, :m])
        assert np.array_equal(c.k_scales[b, h, :m].cpu().numpy(), ks[0, 0, :m])
        assert np.array_equal(c.v_scales[b, h, :m].cpu().numpy(), vs[0, 0, :m])
        ref = O.decode_attention(q[b:b + 1].cpu().numpy(), kc, ks, vc, vs, [m], w.blk)
        got = run.out_of(S - 1)[l, b, h].cpu().numpy()
        assert np.max(np.abs(got - ref[0, 0])) <= ATOL
    del run
    torch.cuda.empty_cache()


# ------------------------------------------------------ per-step plan API
@pytest.mark.parametrize("hd,blk", [(64, 64), (128, 64), (128, 32), (128, 256)])
def test_planned_calls_match_unplanned_bit_exact(N, hd, blk):
    """nqkv_decode_plan + *_planned calls give bit-identical results to the
    unplanned calls (same schedule), for plain and fused steps, with empty,
    single-token and ragged sequences."""
    B, Tc = 6, 1024
    H = 5 if blk <= hd else 3 * _hpb(hd, blk)
    lens0 = [0, 1, 63, 300, 777, 1000]
    T = max(lens0)
    x = _rand_kv(B, T, H, hd, seed=51)
    y = _rand_kv(B, T, H, hd, seed=52, outlier=False)
    kn = _rand_kv(B, 1, H, hd, seed=53)[:, 0].to(DEV)
    vn = _rand_kv(B, 1, H, hd, seed=54, outlier=False)[:, 0].to(DEV)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(55)).to(torch.float16).to(DEV)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(a.copy()).to(DEV)
    L = torch.tensor(lens0, dtype=torch.int32, device=DEV)
    plan = N.make_plan(DEV)
    # plain attention
    N.nqkv_decode_plan(L, H, Tc, False, plan, hd=hd)
    o1 = N.nqkv_decode_attention(q, t(kc), t(ks), t(vc), t(vs), L, blk, N.make_workspace(B, H, hd, Tc, DEV))
    o2 = N.nqkv_decode_attention_planned(q, t(kc), t(ks), t(vc), t(vs), L, blk,
                                         N.make_workspace(B, H, hd, Tc, DEV), plan)
    # plan and first cache loads before the PDL wait (the kernel just before
    # writes neither: it is torch's workspace fill)
    o3 = N.nqkv_decode_attention_planned(q, t(kc), t(ks), t(vc), t(vs), L, blk,
                                         N.make_workspace(B, H, hd, Tc, DEV), plan,
                                         flags=N.EARLY_START)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(o1, o3)
    # fused step (lens after the append)
    L1 = L + 1
    N.nqkv_decode_plan(L1, H, Tc, True, plan, hd=hd)
    a = [t(z) for z in (kc, ks, vc, vs)]
    b = [t(z) for z in (kc, ks, vc, vs)]
    f1 = N.nqkv_decode_step(kn, vn, q, *a, L1, blk, N.make_workspace(B, H, hd, Tc, DEV))
    c = [t(z) for z in (kc, ks, vc, vs)]
    f2 = N.nqkv_decode_step_planned(kn, vn, q, *b, L1, blk, N.make_workspace(B, H, hd, Tc, DEV), plan)
    f3 = N.nqkv_decode_step_planned(kn, vn, q, *c, L1, blk, N.make_workspace(B, H, hd, Tc, DEV), plan,
                                    flags=N.EARLY_START)
    torch.cuda.synchronize()
    assert torch.equal(f1, f2) and torch.equal(f1, f3)
    assert all(torch.equal(u, v) and torch.equal(u, w) for u, v, w in zip(a, b, c))
    O.quantize_append(kn.unsqueeze(1).cpu().numpy(), lens0, blk, kc, ks)
    O.quantize_append(vn.unsqueeze(1).cpu().numpy(), lens0, blk, vc, vs)
    ref = O.decode_attention(q.cpu().numpy(), kc, ks, vc, vs, [n + 1 for n in lens0], blk)
    assert np.max(np.abs(f2.cpu().numpy() - ref)) <= ATOL


@pytest.mark.parametrize("hd", [64, 128])
@pytest.mark.parametrize("blk", [64, 256])
def test_planned_many_pieces_deferred_order(N, hd, blk):
    """CTAs holding more pieces than prebuilt q-table slots process a split
    first piece last (WalkState "defer"): planned == unplanned bit for bit,
    and both match the oracle (also with head-group blocks, blk 256)."""
    lens0 = [(37 * i) % 190 + 3 for i in range(40)]
    B, H, T = len(lens0), 6 if blk <= hd else 4, max(lens0)
    Tc = -(-T // 64) * 64
    x = _rand_kv(B, T, H, hd, seed=61)
    y = _rand_kv(B, T, H, hd, seed=62, outlier=False)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(63)).to(torch.float16).to(DEV)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(a.copy()).to(DEV)
    L = torch.tensor(lens0, dtype=torch.int32, device=DEV)
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L, H, Tc, False, plan, hd=hd)
    o1 = N.nqkv_decode_attention(q, t(kc), t(ks), t(vc), t(vs), L, blk, N.make_workspace(B, H, hd, Tc, DEV))
    o2 = N.nqkv_decode_attention_planned(q, t(kc), t(ks), t(vc), t(vs), L, blk,
                                         N.make_workspace(B, H, hd, Tc, DEV), plan)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    ref = O.decode_attention(q.cpu().numpy(), kc, ks, vc, vs, lens0, blk)
    assert np.max(np.abs(o2.cpu().numpy() - ref)) <= ATOL


def test_planned_large_batch_arrays(N):
    """B > 512: the per-batch arrays take two entries per thread in the
    planned prologue (and pref[B] comes from the plan header)."""
    blk, hd, H = 64, 64, 2
    B = 700
    lens0 = [(i * 7919) % 97 for i in range(B)]          # includes empty sequences
    T = max(lens0)
    Tc = -(-T // 64) * 64
    x = _rand_kv(B, T, H, hd, seed=71)
    y = _rand_kv(B, T, H, hd, seed=72, outlier=False)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(73)).to(torch.float16).to(DEV)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(a.copy()).to(DEV)
    L = torch.tensor(lens0, dtype=torch.int32, device=DEV)
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L, H, Tc, False, plan, hd=hd)
    o1 = N.nqkv_decode_attention(q, t(kc), t(ks), t(vc), t(vs), L, blk, N.make_workspace(B, H, hd, Tc, DEV))
    o2 = N.nqkv_decode_attention_planned(q, t(kc), t(ks), t(vc), t(vs), L, blk,
                                         N.make_workspace(B, H, hd, Tc, DEV), plan,
                                         flags=N.EARLY_START)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    rng = np.random.default_rng(1)
    for b in sorted(set(rng.integers(0, B, 24).tolist()) | {0, B - 1}):
        ref = O.decode_attention(q[b:b + 1].cpu().numpy(), kc[b:b + 1], ks[b:b + 1], vc[b:b + 1],
                                 vs[b:b + 1], [lens0[b]], blk)
        assert np.max(np.abs(o2[b:b + 1].cpu().numpy() - ref)) <= ATOL


@pytest.mark.parametrize("seed", range(10))
def test_random_geometries_planned_fused(N, seed):
    """Random (B, H, hd, blk, lengths incl. 0, 1 and Tc): unplanned ==
    planned (with and without early start) bit for bit, and the fused step
    matches the oracle on sampled (b, h) rows."""
    rng = np.random.default_rng(1000 + seed)
    hd = int(rng.choice([64, 128]))
    blk = int(rng.choice([32, 64] if hd == 64 else [32, 64, 128]))
    B = int(rng.integers(1, 48))
    H = int(rng.integers(1, 9))
    if seed >= 6:                       # head-spanning blocks (blk > hd)
        blk = int(rng.choice([128, 256] if hd == 64 else [256]))
        H = _hpb(hd, blk) * int(rng.integers(1, 4))
    Tc = 64 * int(rng.integers(1, 12))
    lens0 = rng.integers(0, Tc, B)                              # existing rows (< Tc: one is appended)
    lens0[rng.integers(0, B)] = 0
    lens0 = [int(x) for x in lens0]
    T = max(max(lens0), 1)
    x = _rand_kv(B, T, H, hd, seed=seed * 7 + 1)
    y = _rand_kv(B, T, H, hd, seed=seed * 7 + 2, outlier=False)
    kn = _rand_kv(B, 1, H, hd, seed=seed * 7 + 3)[:, 0].to(DEV)
    vn = _rand_kv(B, 1, H, hd, seed=seed * 7 + 4, outlier=False)[:, 0].to(DEV)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(seed * 7 + 5)).to(torch.float16).to(DEV)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(a.copy()).to(DEV)
    L1 = torch.tensor([n + 1 for n in lens0], dtype=torch.int32, device=DEV)
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L1, H, Tc, True, plan, hd=hd)
    caches = [[t(z) for z in (kc, ks, vc, vs)] for _ in range(3)]
    f0 = N.nqkv_decode_step(kn, vn, q, *caches[0], L1, blk, N.make_workspace(B, H, hd, Tc, DEV))
    f1 = N.nqkv_decode_step_planned(kn, vn, q, *caches[1], L1, blk, N.make_workspace(B, H, hd, Tc, DEV), plan)
    f2 = N.nqkv_decode_step_planned(kn, vn, q, *caches[2], L1, blk, N.make_workspace(B, H, hd, Tc, DEV), plan,
                                    flags=N.EARLY_START)
    torch.cuda.synchronize()
    assert torch.equal(f0, f1) and torch.equal(f0, f2)
    for c in caches[1:]:
        assert all(torch.equal(u, v) for u, v in zip(caches[0], c))
    O.quantize_append(kn.unsqueeze(1).cpu().numpy(), lens0, blk, kc, ks)
    O.quantize_append(vn.unsqueeze(1).cpu().numpy(), lens0, blk, vc, vs)
    assert np.array_equal(caches[0][0].cpu().numpy(), kc) and np.array_equal(caches[0][3].cpu().numpy(), vs)
    for b in sorted({0, B - 1} | set(rng.integers(0, B, 4).tolist())):
        ref = O.decode_attention(q[b:b + 1].cpu().numpy(), kc[b:b + 1], ks[b:b + 1], vc[b:b + 1],
                                 vs[b:b + 1], [lens0[b] + 1], blk)
        assert np.max(np.abs(f0[b:b + 1].cpu().numpy() - ref)) <= ATOL


@pytest.mark.parametrize("hd,blk", [(64, 32), (64, 64), (128, 64), (128, 128), (64, 256), (128, 256)])
def test_fp16_scales_lossless(N, hd, blk):
    """NQKV_SCALE_F16: a block scale is the absmax of fp16
    inputs, itself an fp16 value, so storing it as fp16 changes nothing --
    codes, dequantised values, attention (plain, fused, planned) are bit-for-
    bit those of the fp32-scale layout, and the scales equal the oracle's."""
    B = 5
    H = 3 if blk <= hd else 2 * _hpb(hd, blk)
    lens0 = [0, 1, 70, 333, 511]
    T, Tc = max(lens0), 576
    x = _rand_kv(B, T, H, hd, seed=81)
    y = _rand_kv(B, T, H, hd, seed=82, outlier=False)
    kn = _rand_kv(B, 1, H, hd, seed=83)[:, 0].to(DEV)
    vn = _rand_kv(B, 1, H, hd, seed=84, outlier=False)[:, 0].to(DEV)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(85)).to(torch.float16).to(DEV)
    c32 = N.KVCache(B, H, hd, Tc, blk, DEV)
    c16 = N.KVCache(B, H, hd, Tc, blk, DEV, scale_dtype=torch.float16)
    z = torch.zeros(B, dtype=torch.int32, device=DEV)
    for c in (c32, c16):
        c.append(x.to(DEV), y.to(DEV), z)
    torch.cuda.synchronize()
    assert torch.equal(c32.k_codes, c16.k_codes) and torch.equal(c32.v_codes, c16.v_codes)
    assert torch.equal(c32.k_scales, c16.k_scales.float()) and torch.equal(c32.v_scales, c16.v_scales.float())
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    assert np.array_equal(c16.k_scales.float().cpu().numpy(), ks)
    assert torch.equal(N.nqkv_dequantize(c32.k_codes, c32.k_scales, blk),
                       N.nqkv_dequantize(c16.k_codes, c16.k_scales, blk))
    L = torch.tensor(lens0, dtype=torch.int32, device=DEV)
    ws = lambda: N.make_workspace(B, H, hd, Tc, DEV)
    a32, a16 = c32.attend(q, L, ws()), c16.attend(q, L, ws())
    L1 = L + 1
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L1, H, Tc, True, plan, hd=hd)
    f32 = c32.step(kn, vn, q, L1, ws())
    d16 = N.KVCache(B, H, hd, Tc, blk, DEV, scale_dtype=torch.float16)
    d16.k_codes.copy_(c16.k_codes); d16.v_codes.copy_(c16.v_codes)
    d16.k_scales.copy_(c16.k_scales); d16.v_scales.copy_(c16.v_scales)
    f16 = c16.step(kn, vn, q, L1, ws())
    p16 = d16.step_planned(kn, vn, q, L1, ws(), plan, flags=N.EARLY_START)
    torch.cuda.synchronize()
    assert torch.equal(a32, a16)
    assert torch.equal(f32, f16) and torch.equal(f32, p16)
    assert torch.equal(c32.k_codes, c16.k_codes) and torch.equal(c32.v_scales, c16.v_scales.float())
    assert torch.equal(c16.k_scales, d16.k_scales) and torch.equal(c16.v_codes, d16.v_codes)


@pytest.mark.parametrize("hd", [64, 128])
def test_uniform_small_batch_one_cta_per_sequence(N, hd):
    """Uniform lengths, few sequences: one CTA per sequence (no cross-CTA
    merge); planned == unplanned bit for bit, matches the oracle, and the
    workspace stays zero."""
    blk, B, H, T = 64, 2, 5, 600
    Tc = 640
    x = _rand_kv(B, T, H, hd, seed=91)
    y = _rand_kv(B, T, H, hd, seed=92, outlier=False)
    q = torch.randn(B, H, hd, generator=torch.Generator().manual_seed(93)).to(torch.float16).to(DEV)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(a.copy()).to(DEV)
    L = torch.full((B,), T, dtype=torch.int32, device=DEV)
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L, H, Tc, False, plan, hd=hd)
    ws1, ws2 = N.make_workspace(B, H, hd, Tc, DEV), N.make_workspace(B, H, hd, Tc, DEV)
    o1 = N.nqkv_decode_attention(q, t(kc), t(ks), t(vc), t(vs), L, blk, ws1)
    o2 = N.nqkv_decode_attention_planned(q, t(kc), t(ks), t(vc), t(vs), L, blk, ws2, plan)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    assert torch.count_nonzero(ws1) == 0 and torch.count_nonzero(ws2) == 0
    assert int(plan[4:8].view(torch.int32)[0]) == B * H          # header: C = #sequences
    ref = O.decode_attention(q.cpu().numpy(), kc, ks, vc, vs, [T] * B, blk)
    assert np.max(np.abs(o1.cpu().numpy() - ref)) <= ATOL


@pytest.mark.parametrize("hd,blk,G", [(64, 64, 2), (128, 64, 3), (128, 256, 2)])
def test_fused_gather_simulated_ranks(N, hd, blk, G):
    """nqkv_decode_step_gather (all-gather fused into the epilogue, SURVEY
    8(f) row 3) with G ranks simulated on one GPU: the peers' buffers are
    local, and each rank's launch completes before the next starts (no launch
    waits on another).  Every rank's buffer must hold every shard's rows,
    bit-identical to nqkv_decode_step_planned on that shard; each flag holds
    the epoch; the caches equal the unfused step's; the workspace is zero."""
    hpb = _hpb(hd, blk)
    B, Hl, Tc = 4, 2 * hpb, 1024
    Ht = G * Hl
    lens0 = [0, 1, 300, 700]
    x = _rand_kv(B, max(lens0), Ht, hd, seed=71)
    y = _rand_kv(B, max(lens0), Ht, hd, seed=72, outlier=False)
    kn = _rand_kv(B, 1, Ht, hd, seed=73)[:, 0].to(DEV)
    vn = _rand_kv(B, 1, Ht, hd, seed=74, outlier=False)[:, 0].to(DEV)
    q = torch.randn(B, Ht, hd, generator=torch.Generator().manual_seed(75)).to(torch.float16).to(DEV)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    L1 = torch.tensor([n + 1 for n in lens0], dtype=torch.int32, device=DEV)
    bufs = [torch.full((B, Ht, hd), float("nan"), device=DEV) for _ in range(G)]
    flags = [torch.zeros(G, dtype=torch.int32, device=DEV) for _ in range(G)]
    out_ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    flag_ptrs = torch.tensor([f.data_ptr() for f in flags], dtype=torch.int64, device=DEV)
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L1, Hl, Tc, True, plan, hd=hd)
    refs = []
    for r in range(G):
        hs, gs = slice(r * Hl, (r + 1) * Hl), slice(r * Hl // hpb, (r + 1) * Hl // hpb)
        shard = lambda c, s_: [t(c[:, hs]), t(s_[:, gs])]
        a = shard(kc, ks) + shard(vc, vs)
        b = shard(kc, ks) + shard(vc, vs)
        ws = N.make_workspace(B, Hl, hd, Tc, DEV)
        N.nqkv_decode_step_gather(kn[:, hs], vn[:, hs], q[:, hs].contiguous(), a[0], a[1], a[2], a[3], L1,
                                  blk, ws, plan, out_ptrs, flag_ptrs, G, r, epoch=7)
        o = N.nqkv_decode_step_planned(kn[:, hs], vn[:, hs], q[:, hs].contiguous(), b[0], b[1], b[2], b[3],
                                       L1, blk, N.make_workspace(B, Hl, hd, Tc, DEV), plan)
        torch.cuda.synchronize()
        assert all(torch.equal(u, v) for u, v in zip(a, b))
        assert torch.count_nonzero(ws) == 0
        refs.append(o)
    full = torch.cat(refs, dim=1)
    for r in range(G):
        assert torch.equal(bufs[r], full)
        assert flags[r].tolist() == [7] * G
    O.quantize_append(kn.unsqueeze(1).cpu().numpy(), lens0, blk, kc, ks)
    O.quantize_append(vn.unsqueeze(1).cpu().numpy(), lens0, blk, vc, vs)
    ref = O.decode_attention(q.cpu().numpy(), kc, ks, vc, vs, [n + 1 for n in lens0], blk)
    assert np.max(np.abs(bufs[0].cpu().numpy() - ref)) <= ATOL


@pytest.mark.parametrize("hd,blk,G", [(64, 64, 2), (128, 64, 4)])
def test_fused_gather_ranks_in_flight(N, hd, blk, G):
    """The fused gather with G simulated ranks launched on G streams with no
    host synchronisation between them, two back-to-back epochs each into
    parity-double-buffered outputs and flags (the runtime's protocol): the
    ranks' kernels overlap (a later rank starts as earlier CTAs retire),
    their peer stores, fences, completion counters and flag releases
    interleave.  No kernel waits on another (the profiling recipe forbids
    that pattern on one GPU): the flags are checked after a device sync.
    Every buffer holds every shard's rows bit for bit; flags hold the epoch."""
    B, Hl, Tc = 4, 2, 1024
    Ht = G * Hl
    lens0 = [5, 1, 300, 700]
    x = _rand_kv(B, max(lens0), Ht, hd, seed=81)
    y = _rand_kv(B, max(lens0), Ht, hd, seed=82, outlier=False)
    kc, ks = _oracle_cache(x, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(y, [0] * B, blk, Tc)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    L1 = torch.tensor([n + 1 for n in lens0], dtype=torch.int32, device=DEV)
    plan = N.make_plan(DEV)
    N.nqkv_decode_plan(L1, Hl, Tc, True, plan, hd=hd)
    bufs = [[torch.full((B, Ht, hd), float("nan"), device=DEV) for _ in range(G)] for _ in range(2)]
    flags = [[torch.zeros(G, dtype=torch.int32, device=DEV) for _ in range(G)] for _ in range(2)]
    optr = [torch.tensor([b.data_ptr() for b in bufs[par]], dtype=torch.int64, device=DEV) for par in range(2)]
    fptr = [torch.tensor([f.data_ptr() for f in flags[par]], dtype=torch.int64, device=DEV) for par in range(2)]
    caches, wss, steps = [], [], {}
    for r in range(G):
        hs = slice(r * Hl, (r + 1) * Hl)
        caches.append([t(kc[:, hs]), t(ks[:, hs]), t(vc[:, hs]), t(vs[:, hs])])
        wss.append(N.make_workspace(B, Hl, hd, Tc, DEV))
    ref_caches = [[c.clone() for c in cc] for cc in caches]
    for e in (8, 9):
        kn = _rand_kv(B, 1, Ht, hd, seed=83 + e)[:, 0].to(DEV)
        vn = _rand_kv(B, 1, Ht, hd, seed=85 + e, outlier=False)[:, 0].to(DEV)
        q = torch.randn(B, Ht, hd, generator=torch.Generator().manual_seed(87 + e)).to(torch.float16).to(DEV)
        steps[e] = (kn, vn, q)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(G)]
    for e in (8, 9):                              # launch everything, no host sync
        kn, vn, q = steps[e]
        for r in range(G):
            hs = slice(r * Hl, (r + 1) * Hl)
            with torch.cuda.stream(streams[r]):
                c = caches[r]
                N.nqkv_decode_step_gather(kn[:, hs], vn[:, hs], q[:, hs].contiguous(), c[0], c[1], c[2], c[3],
                                          L1, blk, wss[r], plan, optr[e & 1], fptr[e & 1], G, r, epoch=e)
    torch.cuda.synchronize()
    for e in (8, 9):                              # the same steps, one rank at a time, unfused gather
        kn, vn, q = steps[e]
        outs = []
        for r in range(G):
            hs = slice(r * Hl, (r + 1) * Hl)
            c = ref_caches[r]
            outs.append(N.nqkv_decode_step_planned(kn[:, hs], vn[:, hs], q[:, hs].contiguous(), c[0], c[1], c[2],
                                                   c[3], L1, blk, N.make_workspace(B, Hl, hd, Tc, DEV), plan))
        full = torch.cat(outs, dim=1)
        for r in range(G):
            assert torch.equal(bufs[e & 1][r], full), (e, r)
            assert flags[e & 1][r].tolist() == [e] * G
    for r in range(G):
        assert all(torch.equal(a, b) for a, b in zip(caches[r], ref_caches[r]))
        assert torch.count_nonzero(wss[r]) == 0


def test_runtime_fused_gather_single_rank(N):
    """DecodeRunner with the all-gather fused into the epilogue over
    symmetric memory (one rank: the plumbing -- peer pointers, device epoch
    bumped per step and graph replay, flag wait): the gathered outputs equal
    the plain fused runtime's, eagerly and under CUDA-graph replay."""
    import socket
    import torch.distributed as dist
    from paper_2505_16210_b200.runtime import DecodeRunner
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device(DEV, 0))
    try:
        w = W.CONFIGS["c1"]
        a = DecodeRunner(w, range(w.heads), DEV, group=dist.group.WORLD, world=1, step_slots=2, layers=2,
                         fused_gather=True)
        b = DecodeRunner(w, range(w.heads), DEV, step_slots=2, layers=2, fused_gather=False)
        a.prefill()
        b.prefill()
        for s in range(2):
            a.step(s)
            b.step(s)
            torch.cuda.synchronize()
            assert torch.equal(a.out_of(s), b.out_of(s))
            assert a.out is a.out_of(s) or torch.equal(a.out, a.out_of(s))
        assert a.g_flags.tolist() == [1, 1, 2, 2]          # [parity][layer][rank]: epochs 1, 2
        ev = [[(torch.cuda.Event(enable_timing=True, external=True),
                torch.cuda.Event(enable_timing=True, external=True)) for _ in range(2)]]
        a.capture(timing_slots=(0,))
        b.capture()
        for s in (0, 1):
            a.replay(s)
            b.replay(s)
        torch.cuda.synchronize()
        assert torch.equal(a.out_of(1), b.out_of(1)) and torch.equal(a.out_of(0), b.out_of(0))
        assert a.g_flags.tolist() == [3, 3, 4, 4] and int(a.epoch.item()) == 4
        assert all(t > 0 for t in a.decode_kernel_ms())   # events recorded around the gather launches
        del ev
        # odd step-slot count: graphs are doubled so buffer parity alternates
        c = DecodeRunner(w, range(w.heads), DEV, group=dist.group.WORLD, world=1, step_slots=1, layers=2,
                         fused_gather=True)
        c.prefill()
        c.capture(timing_slots=())
        assert len(c.graphs) == 2
        for i in range(3):
            c.replay(i)
        torch.cuda.synchronize()
        assert c.g_flags.tolist() == [3, 3, 2, 2]
    finally:
        dist.destroy_process_group()


def test_runtime_nccl_side_stream_gather_world1(N):
    """The runtime's NCCL all-gather of per-head outputs on a side stream
    (the multi-GPU exchange step), forced on at world size 1
    and run eagerly and under CUDA-graph capture/replay: the gathered buffer
    equals the rank's own outputs bit for bit."""
    import socket
    import torch.distributed as dist
    from paper_2505_16210_b200.runtime import DecodeRunner
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device(DEV, 0))
    try:
        w = W.CONFIGS["c1"]
        r = DecodeRunner(w, range(w.heads), DEV, group=dist.group.WORLD, world=1, step_slots=2, layers=3,
                         nccl_gather=True)
        assert r.nccl_gather
        r.prefill()
        r.step(0)
        torch.cuda.synchronize()
        assert torch.equal(r.gathered, r.out_of(0))
        r.capture(timing_slots=())
        r.gathered.zero_()
        r.replay(1)
        torch.cuda.synchronize()
        assert torch.equal(r.gathered, r.out_of(1))
        assert r.launches_per_step() == 3 + 1
        # the other gather modes: serialized per layer, one per step
        for mode in ("serialized", "per_step"):
            r2 = DecodeRunner(w, range(w.heads), DEV, group=dist.group.WORLD, world=1, step_slots=2,
                              layers=3, nccl_gather=True, gather_mode=mode)
            r2.prefill()
            r2.step(0)
            torch.cuda.synchronize()
            for l in range(3):
                assert torch.equal(r2.gathered_layer(l), r2.out_of(0)[l])
            r2.capture(timing_slots=())
            r2.gathered.zero_()
            r2.replay(1)
            torch.cuda.synchronize()
            for l in range(3):
                assert torch.equal(r2.gathered_layer(l), r2.out_of(1)[l])
    finally:
        dist.destroy_process_group()


# ---------------------------------------------- prefill attention (8(f) row 4)
def _prefill_case(N, B, T, H, hd, blk, lens, Tc, seed, f16s=False):
    k = _rand_kv(B, T, H, hd, seed)
    v = _rand_kv(B, T, H, hd, seed + 1, False)
    q = torch.randn(B, T, H, hd, generator=torch.Generator().manual_seed(seed + 2)).to(torch.float16)
    kc, ks = _oracle_cache(k, [0] * B, blk, Tc)
    vc, vs = _oracle_cache(v, [0] * B, blk, Tc)
    ref = O.prefill_attention(q.numpy(), kc, ks, vc, vs, lens, blk)
    t = lambda a: torch.from_numpy(a).to(DEV)
    sk, sv = t(ks), t(vs)
    if f16s:
        sk, sv = sk.half(), sv.half()
    out = N.nqkv_prefill_attention(q.to(DEV), t(kc), sk, t(vc), sv,
                                   torch.tensor(lens, dtype=torch.int32, device=DEV), blk)
    torch.cuda.synchronize()
    return out.cpu().numpy(), ref


@pytest.mark.parametrize("hd,blk", [(64, 64), (64, 32), (128, 64), (128, 32), (128, 128), (64, 256), (128, 256)])
def test_prefill_attention_matches_oracle(N, hd, blk):
    """Causal prefill attention over the dequantised cache (PAPER.md:213-221,
    SPEC.md:236-244) within 2e-3 of the float64 oracle: ragged prompt lengths
    spanning several 64-query / 64-key tiles and a ragged tail, an empty and a
    one-token prompt, K outlier channels."""
    H = 2 if blk <= hd else 2 * _hpb(hd, blk)
    lens = [0, 1, 63, 64, 65, 200]
    out, ref = _prefill_case(N, len(lens), 200, H, hd, blk, lens, 256, seed=hd + blk)
    err = np.max(np.abs(out.astype(np.float64) - ref))
    assert err <= ATOL, err
    assert np.all(out[0] == 0) and np.all(out[2, 63:] == 0)          # rows >= len are zero


def test_prefill_attention_fp16_scales_and_long(N):
    out, ref = _prefill_case(N, 2, 700, 3, 128, 64, [700, 513], 704, seed=77, f16s=True)
    assert np.max(np.abs(out.astype(np.float64) - ref)) <= ATOL


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_prefill_attention_config_prompt_sampled(N, cfg):
    """The config's prompt length (c3: U[1024, 2048], c4: 8192) on the GPU for
    a few heads; the oracle checks sampled query rows of sampled sequences
    (each row equals the oracle's decode attention of q_i over i + 1 tokens,
    which is cheap to evaluate one row at a time)."""
    w = W.CONFIGS[cfg]
    H = 2
    lens = W.seq_lens(w)
    B = min(w.batch, 3)
    lens = lens[:B]
    T = int(lens.max())
    Tc = W.capacity(T)
    K, V = W.layer_kv(w, 0, heads=range(H), tokens=T, device=DEV)
    K, V = K[:B].contiguous(), V[:B].contiguous()
    q = torch.randn(B, T, H, w.head_dim, generator=torch.Generator(device=DEV).manual_seed(5), device=DEV).half()
    cache = N.KVCache(B, H, w.head_dim, Tc, w.blk, DEV)
    cache.append(K, V, torch.zeros(B, dtype=torch.int32, device=DEV))
    L = lens.to(DEV)
    out = N.nqkv_prefill_attention(q, cache.k_codes, cache.k_scales, cache.v_codes, cache.v_scales, L, w.blk)
    torch.cuda.synchronize()
    kc, ks = cache.k_codes.cpu().numpy(), cache.k_scales.cpu().numpy()
    vc, vs = cache.v_codes.cpu().numpy(), cache.v_scales.cpu().numpy()
    qn = q.cpu().numpy()
    on = out.cpu().numpy()
    rng = np.random.default_rng(1)
    for b in range(B):
        n = int(lens[b])
        for i in sorted({0, 63, 64, n - 1} | {int(rng.integers(n)) for _ in range(4)}):
            ref = O.decode_attention(qn[b:b + 1, i], kc[b:b + 1], ks[b:b + 1], vc[b:b + 1], vs[b:b + 1], [i + 1], w.blk)
            assert np.max(np.abs(on[b, i] - ref[0])) <= ATOL, (b, i)
        assert np.all(on[b, n:] == 0)


@pytest.mark.parametrize("hd,blk", [(64, 32), (64, 256), (128, 64), (128, 128)])
def test_quantize_pair_equals_two_calls_and_oracle(N, hd, blk):
    """nqkv_quantize_pair (K and V in one launch) writes exactly what two
    nqkv_quantize calls write, bit for bit, and what the oracle writes;
    strided inputs, a row count that is not a multiple of the 64-chunk unit."""
    hpb = _hpb(hd, blk)
    B, T, H = 3, 37, 2 * hpb
    Tc = 64
    kv = _rand_kv(B, T, 2 * H, hd, seed=hd * blk)         # K and V interleaved by head: strided views
    k, v = kv[:, :, :H], kv[:, :, H:]
    pos = torch.tensor([0, 5, 27], dtype=torch.int32, device=DEV)
    shape = N.scales_shape(B, H, Tc, hd, blk)
    outs = []
    for pair in (True, False):
        kc = torch.zeros(B, H, Tc, hd // 2, dtype=torch.uint8, device=DEV)
        vc = torch.zeros_like(kc)
        ks = torch.zeros(shape, dtype=torch.float32, device=DEV)
        vs = torch.zeros_like(ks)
        kd, vd = kv.to(DEV)[:, :, :H], kv.to(DEV)[:, :, H:]
        if pair:
            N.nqkv_quantize_pair(kd, vd, pos, kc, ks, vc, vs, blk)
        else:
            N.nqkv_quantize(kd, pos, kc, ks, blk)
            N.nqkv_quantize(vd, pos, vc, vs, blk)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (kc, ks, vc, vs)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    okc, oks = _oracle_cache(k.contiguous(), pos.tolist(), blk, Tc)
    ovc, ovs = _oracle_cache(v.contiguous(), pos.tolist(), blk, Tc)
    for a, b in zip(outs[0], (okc, oks, ovc, ovs)):
        assert np.array_equal(a, b)
