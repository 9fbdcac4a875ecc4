"""Pins for the CPU oracle: each test ties an oracle function to something
other than itself -- an independent 50-digit quantile evaluation, a closed
form, brute force in exact rational arithmetic, a bound, or a value the paper
prints.  CPU only (no GPU marker)."""
from __future__ import annotations

import math
import statistics
import struct
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from oracle import nqkv_oracle as O

L32 = O.nf_levels_f32()


# ---------------------------------------------------------------- levels ----
def _mp_levels(bits=4, dps=50):
    """Independent evaluation: Phi^-1(p) = sqrt(2) erfinv(2p-1) at 50 digits on
    the SPEC.md:58 probability grid, computed in exact rationals."""
    mpmath.mp.dps = dps
    n = 1 << bits
    delta = 1 - Fraction(1, 2) * (Fraction(1, 2 * n) + Fraction(1, 2 * (n - 1)))
    half = n // 2

    def ppf(p):
        return mpmath.sqrt(2) * mpmath.erfinv(2 * mpmath.mpf(p.numerator) / p.denominator - 1)

    negs = [-ppf(delta + k * (Fraction(1, 2) - delta) / (half - 1)) for k in range(half - 1)]
    poss = [ppf(Fraction(1, 2) + k * (delta - Fraction(1, 2)) / half) for k in range(1, half + 1)]
    d = ppf(delta)
    vals = sorted([v / d for v in negs] + [mpmath.mpf(0)] + [v / d for v in poss])
    return vals, delta, d


def _f32_bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_levels_structure():
    # 16 values, strictly increasing, -1 / exact 0 / +1
    assert L32.shape == (16,) and L32.dtype == np.float32
    assert np.all(np.diff(L32) > 0)
    assert L32[0] == -1.0 and L32[15] == 1.0
    assert L32.view(np.uint32)[7] == 0          # +0.0 exactly
    assert np.count_nonzero(L32 == 0) == 1
    assert np.count_nonzero(L32 < 0) == 7 and np.count_nonzero(L32 > 0) == 8


def test_levels_match_50_digit_quantiles_bit_exact():
    vals, delta, d = _mp_levels()
    # RN to fp32 of a 50-digit value: round via Python float (53 bits) is safe
    # because every level sits >= 0.02 fp32-ulp from a rounding boundary; we
    # check that margin explicitly so a double-rounding hazard would fail here.
    for i, v in enumerate(vals):
        f = float(v)
        r32 = np.float32(f)
        ulp = float(np.spacing(np.float32(abs(r32)))) if r32 != 0 else 1.0
        lo = float(r32) - ulp / 2
        hi = float(r32) + ulp / 2
        if v != 0:
            margin = min(abs(v - mpmath.mpf(lo)), abs(mpmath.mpf(hi) - v)) / ulp
            assert margin > 0.01, (i, margin)
        assert _f32_bits(float(r32)) == int(L32.view(np.uint32)[i]), i
    assert abs(float(delta) - O.nf_offset()) < 4e-16   # double evaluation, <= 2 ulp
    assert abs(float(delta) - 0.96770833333333333) < 1e-15


def test_levels_match_statistics_normaldist():
    # a third, unrelated Phi^-1 (Python's statistics module, Wichura AS241)
    nd = statistics.NormalDist()
    delta = O.nf_offset()
    neg = [-nd.inv_cdf(p) for p in np.linspace(delta, 0.5, 8)[:-1]]
    pos = [nd.inv_cdf(p) for p in np.linspace(0.5, delta, 9)[1:]]
    d = nd.inv_cdf(delta)
    vals = np.float32(np.array(sorted([v / d for v in neg] + [0.0] + [v / d for v in pos])))
    assert np.array_equal(vals.view(np.uint32), L32.view(np.uint32))


def test_normal_quantile_examples():
    from scipy.special import ndtri
    assert abs(ndtri(0.975) - 1.959964) < 1e-5
    assert abs(ndtri(0.025) + 1.959964) < 1e-5
    assert ndtri(0.5) == 0.0
    assert abs(ndtri(O.nf_offset()) - 1.8481314207079737) < 1e-13


def test_bits2_codebook():
    # 4 codepoints, strictly increasing, containing -1, 0, 1
    c = O.nf_levels_f64(2)
    assert c.shape == (4,) and np.all(np.diff(c) > 0)
    assert c[0] == -1.0 and c[-1] == 1.0 and 0.0 in c


def test_max_gap():
    g = np.max(np.diff(L32.astype(np.float64)))
    assert abs(g - 0.30380720) < 1e-7
    assert np.argmax(np.diff(L32)) == 0


# ---------------------------------------------------------- code function --
def _rn32_div(x: float, s: float) -> float:
    """RN32(x/s) for fp32 x, s: exact rational quotient rounded to nearest-even
    fp32 (independent of numpy's division)."""
    q = Fraction(x) / Fraction(s)
    return _rn32(q)


def _rn32(q: Fraction) -> float:
    if q == 0:
        return 0.0
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = math.floor(math.log2(a.numerator) - math.log2(a.denominator))
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    ulp = Fraction(2) ** (max(e, -126) - 23)
    m = a / ulp
    fl = math.floor(m)
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * float(fl * ulp)


def _brute_code(n: float) -> int:
    """Nearest level in exact rationals; strict '<' keeps the lower index on ties."""
    best, bestd = 0, None
    for i, lv in enumerate(L32.tolist()):
        d = abs(Fraction(n) - Fraction(lv))
        if bestd is None or d < bestd:
            best, bestd = i, d
    return best


def test_brute_force_256_normals():
    # 256 seeded normals vs a brute-force nearest-codepoint search
    rng = np.random.default_rng(0)
    x = rng.standard_normal(256).astype(np.float16)
    s, c = O.quantize_blocks(x.reshape(4, 64))
    for blk in range(4):
        xs = x.reshape(4, 64)[blk].astype(np.float32)
        sc = max(abs(float(v)) for v in xs)
        assert s[blk] == np.float32(sc)
        for j in range(64):
            n = _rn32_div(float(xs[j]), sc)
            assert c[blk, j] == _brute_code(n)


def test_fp32_division_is_ieee_rn():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(2000).astype(np.float16).astype(np.float32)
    s = np.float32(np.max(np.abs(x)))
    n = (x / s).astype(np.float32)
    for i in range(0, 2000, 7):
        assert float(n[i]) == _rn32_div(float(x[i]), float(s))


def test_tie_rule_lower_index():
    # midpoints exactly representable in fp32 -> n == midpoint -> lower code
    lv = L32.astype(np.float64)
    exact = []
    for i in range(15):
        mid = (lv[i] + lv[i + 1]) / 2
        if float(np.float32(mid)) == mid:
            exact.append(i)
            n = np.float32(mid)
            assert O.nearest_level_codes(np.array([n]))[0] == i
            assert O.codes_by_threshold(np.array([n]))[0] == i
            assert _brute_code(float(n)) == i
            up = np.nextafter(n, np.float32(2))
            assert O.nearest_level_codes(np.array([up]))[0] == i + 1
    assert exact == [2, 6, 7, 14]


def test_threshold_form_equals_brute_force_near_every_boundary():
    t = O.thresholds_f32()
    cand = []
    for ti in t:
        v = ti
        for _ in range(40):
            v = np.nextafter(v, np.float32(-2))
        for _ in range(80):
            cand.append(v)
            v = np.nextafter(v, np.float32(2))
    rng = np.random.default_rng(2)
    cand = np.concatenate([np.array(cand, np.float32),
                           rng.uniform(-1, 1, 200000).astype(np.float32),
                           np.array([-1, 1, 0, -0.0], np.float32)])
    a = O.nearest_level_codes(cand)
    b = O.codes_by_threshold(cand)
    assert np.array_equal(a, b)
    # exact-rational brute force on the near-boundary slice
    for v in cand[:15 * 80:3]:
        assert a[list(cand).index(v)] == _brute_code(float(v))


def test_threshold_values_are_rounded_down_midpoints():
    lv = L32.astype(np.float64)
    t = O.thresholds_f32()
    for i in range(15):
        mid = Fraction(float(lv[i])) / 2 + Fraction(float(lv[i + 1])) / 2
        assert Fraction(float(t[i])) <= mid
        assert Fraction(float(np.nextafter(t[i], np.float32(2)))) > mid


# ---------------------------------------------------------------- quantize --
def test_grid_fixed_point():
    # SPEC.md:70 adapted to fp16 input: block {fp16(s*L_c)} -> codes c
    for s in [1.0, 0.5, 3.0, 17.25, 1e-3, 6.0e4]:
        x = (np.float32(s) * L32).astype(np.float16)
        sc, c = O.quantize_blocks(x.reshape(1, 16))
        assert sc[0] == np.float32(np.float16(s))
        assert np.array_equal(c[0], np.arange(16))


def test_zero_block():
    # SPEC.md:71, 79
    sc, c = O.quantize_blocks(np.zeros((3, 64), np.float16))
    assert np.all(sc == 0) and np.all(c == O.ZERO_CODE)
    codes, scales = O.empty_cache(1, 1, 64, 64, 64)
    O.quantize_append(np.zeros((1, 1, 1, 64), np.float16), [0], 64, codes, scales)
    assert np.all(O.dequantize(codes, scales, 64, 1) == 0)


def test_nonfinite_rejected():
    with pytest.raises(ValueError):
        O.quantize_blocks(np.array([[1.0, np.inf]], np.float16))


def test_monotone_in_x():
    # for fixed scale the code is nondecreasing in x
    s = np.float16(2.5)
    xs = np.sort(np.unique(np.linspace(-2.5, 2.5, 4001).astype(np.float16)))
    blocks = np.stack([np.array([s, x], np.float16) for x in xs])
    _, c = O.quantize_blocks(blocks)
    assert np.all(np.diff(c[:, 1].astype(int)) >= 0)


def test_idempotence():
    # quantize(fp16(dequant(quantize(x)))) == quantize(x)
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((500, 64)) * rng.lognormal(0, 0.5, 64)).astype(np.float16)
    s, c = O.quantize_blocks(x)
    deq = (s[:, None] * L32[c]).astype(np.float32).astype(np.float16)
    s2, c2 = O.quantize_blocks(deq)
    assert np.array_equal(c, c2) and np.array_equal(s, s2)


def test_round_trip_bound_10000_blocks():
    # |x - deq| <= scale * g/2, g = largest adjacent gap
    rng = np.random.default_rng(4)
    x = rng.standard_normal((10000, 64)).astype(np.float16)
    s, c = O.quantize_blocks(x)
    deq = (s[:, None] * L32[c]).astype(np.float32)
    g = float(np.max(np.diff(L32.astype(np.float64))))
    err = np.abs(x.astype(np.float64) - deq.astype(np.float64))
    assert np.all(err <= s[:, None].astype(np.float64) * g / 2 * (1 + 1e-6))


def test_nf4_beats_uniform_on_normal_blocks():
    # SPEC.md:105 / acceptance 3: NF4 MSE strictly below a uniform 16-level
    # absmax grid on >= 10,000 normal blocks of 256
    rng = np.random.default_rng(5)
    x = rng.standard_normal((10000, 256)).astype(np.float16)
    s, c = O.quantize_blocks(x)
    nf = (s[:, None] * L32[c]).astype(np.float64)
    uni = np.linspace(-1, 1, 16)
    xf = x.astype(np.float64)
    n = xf / s[:, None]
    uq = uni[np.argmin(np.abs(n[..., None] - uni), axis=-1)] * s[:, None]
    mse_nf = np.mean((xf - nf) ** 2)
    mse_u = np.mean((xf - uq) ** 2)
    assert mse_nf < mse_u
    rel = math.sqrt(mse_nf) / math.sqrt(np.mean(xf ** 2))
    assert 0.09 < rel < 0.105       # 0.0986 at blk 256


def test_fig5_geometry():
    # PAPER.md:193 (Fig. 5 caption): hidden 24, 1024 tokens, block 6 ->
    # 4 blocks per token, 1024 x 4 blocks; 4096 scales
    rng = np.random.default_rng(6)
    x = rng.standard_normal((1, 1024, 1, 24)).astype(np.float16)
    codes, scales = O.empty_cache(1, 1, 1024, 24, 6)
    O.quantize_append(x, [0], 6, codes, scales)
    assert scales.shape[-1] == 4 and scales[0, 0].size == 4096
    assert codes[0, 0].shape == (1024, 12)


def test_fig2_block256_geometry():
    # PAPER.md:141 (Fig. 2 caption): OPT-6.7B hidden size 4096, block size 256
    # -> 16 blocks per token (here 32 heads x 128 channels, 8 tokens)
    rng = np.random.default_rng(16)
    x = rng.standard_normal((1, 8, 32, 128)).astype(np.float16)
    codes, scales = O.empty_cache(1, 32, 64, 128, 256)
    O.quantize_append(x, [0], 256, codes, scales)
    assert scales.shape == (1, 16, 64, 1)
    assert np.count_nonzero(scales[0, :, :8]) == 16 * 8      # 16 blocks per token
    # closed form: a block scale is max |x| over its 256 hidden channels
    hid = x.reshape(1, 8, 4096).astype(np.float32)
    for t in range(8):
        for g in range(16):
            assert scales[0, g, t, 0] == np.abs(hid[0, t, 256 * g:256 * (g + 1)]).max()


@pytest.mark.parametrize("hd,blk", [(64, 128), (64, 256), (128, 256)])
def test_head_spanning_block_reduces_to_per_head(hd, blk):
    # a group whose other heads are zero has the absmax of the remaining head:
    # codes and scale equal the blk = hd quantisation of that head, and the
    # zero heads get the zero code
    hpb = blk // hd
    rng = np.random.default_rng(17 + blk)
    H = 2 * hpb
    x = np.zeros((1, 3, H, hd), np.float16)
    live = [1, hpb + hpb - 1]                        # one head in each group
    for h in live:
        x[0, :, h] = (rng.standard_normal((3, hd)) * 2).astype(np.float16)
    c, sc = O.empty_cache(1, H, 64, hd, blk)
    O.quantize_append(x, [0], blk, c, sc)
    for gi, h in enumerate(live):
        sh, ch = O.quantize_blocks(x[0, :, h])
        assert np.array_equal(sc[0, gi, :3, 0], sh)
        assert np.array_equal(O.unpack_nibbles(c[0, h, :3]), ch)
        for h2 in range(gi * hpb, (gi + 1) * hpb):
            if h2 != h:
                assert np.all(O.unpack_nibbles(c[0, h2, :3]) == O.ZERO_CODE)
    # dequant: every head of group g uses the group's scale, RN32(s * L)
    dq = O.dequantize(c, sc, blk, 3)
    for h in range(H):
        ref = (sc[0, h // hpb, :3, :] * L32[O.unpack_nibbles(c[0, h, :3])]).astype(np.float32)
        assert np.array_equal(dq[0, h], ref)


def test_head_spanning_grid_fixed_point():
    # SPEC.md:70 across heads: the 16 values fp16(s * L_c) spread over the 4
    # heads of a 256-block (hd 64) come back as codes c, scale s
    s = 3.0
    grid = (np.float32(s) * L32).astype(np.float16)                 # 16 values
    x = np.zeros((1, 1, 4, 64), np.float16)
    flat = x.reshape(256)
    idx = np.arange(16) * 16 + 5                                     # 4 per head
    flat[idx] = grid
    c, sc = O.empty_cache(1, 4, 64, 64, 256)
    O.quantize_append(flat.reshape(1, 1, 4, 64), [0], 256, c, sc)
    assert sc[0, 0, 0, 0] == np.float32(s)
    codes = O.unpack_nibbles(c[0, :, 0]).reshape(256)
    assert np.array_equal(codes[idx], np.arange(16))
    mask = np.ones(256, bool)
    mask[idx] = False
    assert np.all(codes[mask] == O.ZERO_CODE)


def test_head_spanning_blocks_stream_and_reject_straddle():
    rng = np.random.default_rng(18)
    x = (rng.standard_normal((2, 5, 4, 128)) * 3).astype(np.float16)
    c1, s1 = O.empty_cache(2, 4, 64, 128, 256)
    O.quantize_append(x, [0, 7], 256, c1, s1)
    c2, s2 = O.empty_cache(2, 4, 64, 128, 256)
    for t in range(5):
        O.quantize_append(x[:, t:t + 1], [t, 7 + t], 256, c2, s2)
    assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
    with pytest.raises(ValueError):
        O.empty_cache(1, 3, 64, 128, 256)                            # 3 heads: 1.5 blocks


def test_pack_layout_golden_row():
    # element 2i low nibble, 2i+1 high nibble
    c = np.arange(16, dtype=np.uint8)
    p = O.pack_nibbles(c)
    assert p.tolist() == [0x10, 0x32, 0x54, 0x76, 0x98, 0xBA, 0xDC, 0xFE]
    assert np.array_equal(O.unpack_nibbles(p), c)
    rng = np.random.default_rng(7)
    r = rng.integers(0, 16, (100, 64)).astype(np.uint8)
    assert np.array_equal(O.unpack_nibbles(O.pack_nibbles(r)), r)


def test_streaming_equivalence_and_append_only():
    # SPEC.md:164, 194-195
    rng = np.random.default_rng(8)
    B, T, H, hd, blk = 2, 16, 3, 64, 32
    x = (rng.standard_normal((B, T, H, hd)) * 3).astype(np.float16)
    c1, s1 = O.empty_cache(B, H, 64, hd, blk)
    O.quantize_append(x, [0, 0], blk, c1, s1)
    for j in (0, 5, 15):
        c2, s2 = O.empty_cache(B, H, 64, hd, blk)
        if j:
            O.quantize_append(x[:, :j], [0, 0], blk, c2, s2)
        for t in range(j, T):
            before_c, before_s = c2.copy(), s2.copy()
            O.quantize_append(x[:, t:t + 1], [t, t], blk, c2, s2)
            mask = np.ones(64, bool)
            mask[t] = False
            assert np.array_equal(before_c[:, :, mask], c2[:, :, mask])
            assert np.array_equal(before_s[:, :, mask], s2[:, :, mask])
        assert np.array_equal(c1, c2) and np.array_equal(s1, s2)


def test_ragged_positions():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((2, 3, 1, 64)).astype(np.float16)
    c, s = O.empty_cache(2, 1, 64, 64, 64)
    O.quantize_append(x, [5, 40], 64, c, s)
    ref_c, ref_s = O.empty_cache(1, 1, 64, 64, 64)
    O.quantize_append(x[1:2], [40], 64, ref_c, ref_s)
    assert np.array_equal(c[1], ref_c[0]) and np.all(c[0, :, 40:43] == 0)
    assert np.all(s[0, :, :5] == 0) and np.all(s[0, :, 5:8] > 0)


# ------------------------------------------------------------- dequantize --
def test_dequant_examples():
    # SPEC.md:79-80
    codes = np.full((1, 1, 1, 1), 0xF0, np.uint8)     # elem0 code 0 (-1), elem1 code 15 (+1)
    scales = np.full((1, 1, 1, 1), 2.0, np.float32)
    v = O.dequantize(codes, scales, 2)
    assert v.ravel().tolist() == [-2.0, 2.0]
    assert np.all(O.dequantize(codes, np.zeros_like(scales), 2) == 0)


def test_dequant_fp16_is_rn16_of_rn32():
    # fp16 output = RN16(RN32(s * L))
    rng = np.random.default_rng(10)
    s = rng.uniform(0.01, 60000, 4096).astype(np.float16).astype(np.float32)
    c = rng.integers(0, 16, 4096)
    v32 = np.array([_rn32(Fraction(float(a)) * Fraction(float(L32[k]))) for a, k in zip(s, c)],
                   np.float32)
    codes = O.pack_nibbles(np.stack([c, c], -1).astype(np.uint8)).reshape(1, 1, 4096, 1)
    out32 = O.dequantize(codes, s.reshape(1, 1, 4096, 1), 2)[..., 0].ravel()
    assert np.array_equal(out32, v32)
    out16 = O.dequantize(codes, s.reshape(1, 1, 4096, 1), 2, out_dtype=np.float16)[..., 0].ravel()
    assert np.array_equal(out16, v32.astype(np.float16))


# -------------------------------------------------------------- attention --
def _cache_from(x, blk, Tc=64):
    B, T, H, hd = x.shape
    c, s = O.empty_cache(B, H, Tc, hd, blk)
    O.quantize_append(x, [0] * B, blk, c, s)
    return c, s


def test_single_token_attention_returns_value():
    # one cached token -> weight 1 -> t_O = dequantised v
    rng = np.random.default_rng(11)
    k = rng.standard_normal((2, 1, 3, 64)).astype(np.float16)
    v = rng.standard_normal((2, 1, 3, 64)).astype(np.float16)
    q = rng.standard_normal((2, 3, 64)).astype(np.float16)
    kc, ks = _cache_from(k, 64)
    vc, vs = _cache_from(v, 64)
    out = O.decode_attention(q, kc, ks, vc, vs, [1, 1], 64)
    assert np.array_equal(out, O.dequantize(vc, vs, 64, 1)[:, :, 0, :].astype(np.float64))


def test_identical_keys_average_values():
    # identical keys -> uniform weights -> mean of the V rows
    rng = np.random.default_rng(12)
    k = np.repeat(rng.standard_normal((1, 1, 2, 64)).astype(np.float16), 37, axis=1)
    v = rng.standard_normal((1, 37, 2, 64)).astype(np.float16)
    q = rng.standard_normal((1, 2, 64)).astype(np.float16)
    kc, ks = _cache_from(k, 32)
    vc, vs = _cache_from(v, 32)
    out = O.decode_attention(q, kc, ks, vc, vs, [37], 32)
    mean = O.dequantize(vc, vs, 32, 37).astype(np.float64).mean(axis=2)
    assert np.max(np.abs(out - mean)) < 1e-12


def test_empty_sequence_and_masking():
    rng = np.random.default_rng(13)
    k = rng.standard_normal((2, 20, 1, 64)).astype(np.float16)
    v = rng.standard_normal((2, 20, 1, 64)).astype(np.float16)
    q = rng.standard_normal((2, 1, 64)).astype(np.float16)
    kc, ks = _cache_from(k, 64)
    vc, vs = _cache_from(v, 64)
    out = O.decode_attention(q, kc, ks, vc, vs, [0, 7], 64)
    assert np.all(out[0] == 0)
    # tokens >= seq_len must not matter: scribble over them
    kc2, vc2 = kc.copy(), vc.copy()
    kc2[:, :, 7:] = 0x5A
    vc2[:, :, 7:] = 0xA5
    out2 = O.decode_attention(q, kc2, ks, vc2, vs, [0, 7], 64)
    assert np.array_equal(out[1], out2[1])


def test_softmax_weights_and_dominant_key():
    rng = np.random.default_rng(14)
    K = rng.standard_normal((50, 64))
    q = rng.standard_normal(64)
    p = O.attention_weights(q, K, 0.125)
    assert np.all(p >= 0) and abs(p.sum() - 1) < 1e-12
    # a key aligned with q and huge norm dominates -> output -> its value row
    x = np.zeros((1, 8, 1, 64), np.float16)
    x[0, 3, 0, :] = np.sign(rng.standard_normal(64)).astype(np.float16) * 60
    qq = (x[0, 3, 0, :] / 60).astype(np.float16).reshape(1, 1, 64)
    v = rng.standard_normal((1, 8, 1, 64)).astype(np.float16)
    kc, ks = _cache_from(x, 64)
    vc, vs = _cache_from(v, 64)
    out = O.decode_attention(qq, kc, ks, vc, vs, [8], 64)
    vrow = O.dequantize(vc, vs, 64, 8)[0, 0, 3].astype(np.float64)
    assert np.max(np.abs(out[0, 0] - vrow)) < 1e-9


def test_token_permutation_invariance():
    rng = np.random.default_rng(15)
    k = rng.standard_normal((1, 30, 2, 64)).astype(np.float16)
    v = rng.standard_normal((1, 30, 2, 64)).astype(np.float16)
    q = rng.standard_normal((1, 2, 64)).astype(np.float16)
    perm = rng.permutation(30)
    a = O.decode_attention(q, *_cache_from(k, 64), *_cache_from(v, 64), [30], 64)
    b = O.decode_attention(q, *_cache_from(k[:, perm], 64), *_cache_from(v[:, perm], 64), [30], 64)
    assert np.max(np.abs(a - b)) < 1e-12


# ------------------------------------------------------------- byte model --
def test_byte_model_spec_examples():
    # SPEC.md:190-191
    assert O.cache_bytes(1, 256, 256, 4) == 264
    assert (O.cache_bytes(1000, 256, 256, 4) * 8) / (2 * 1000 * 256) == 4.125


def test_paper_memory_arithmetic():
    # OPT-175B (96 layers, d 12288), batch 64, seq 8192:
    # KV cache "2.3TB", "seven times the size of the model's own parameters"
    kv = O.fp16_kv_bytes(96, 64, 8192, 12288)
    assert round(kv / 2 ** 40, 1) == 2.3 or round(kv / 1e12, 1) == 2.5
    assert round(kv / 2 ** 40, 2) == 2.25
    assert round(kv / (175e9 * 2)) == 7


# ------------------------------------------------- softmax temperature pin --
def _grid_rows(codes: np.ndarray) -> np.ndarray:
    """fp16 rows whose block absmax is exactly 1.0 (code 15 present) and whose
    elements are fp16(L[c]): the grid fixed point maps them back to codes c,
    so the dequantised row is exactly L32[c] (scale 1.0)."""
    return L32[codes].astype(np.float16)


@pytest.mark.parametrize("hd", [64, 128])
def test_softmax_temperature_two_token_closed_form(hd):
    """Two cached tokens with grid-exact keys: p1/p0 = exp(q.(k1 - k0)/sqrt(hd))
    (PAPER.md:233 writes Softmax(t_Q X_K'^T); the 1/sqrt(d) factor is DESIGN.md
    reading R6).  The expected output is evaluated at 50 digits
    from exact rationals, independently of the oracle's arithmetic.  The same
    closed form with no temperature, 1/hd, or base 2 misses the oracle by far,
    so a plausible temperature mistake in the oracle fails here."""
    rng = np.random.default_rng(2025 + hd)
    kc = rng.integers(0, 16, size=(2, hd))
    vc = rng.integers(0, 16, size=(2, hd))
    kc[:, 0] = 15                      # absmax 1.0 in every block (blk = hd)
    vc[:, 0] = 15
    # q with a moderate q.(k1 - k0): keep the ratio away from 0 and infinity
    for _ in range(100):
        q = (rng.standard_normal(hd) * 0.35).astype(np.float16)
        d = sum(Fraction(float(a)) * (Fraction(float(L32[c1])) - Fraction(float(L32[c0])))
                for a, c0, c1 in zip(q, kc[0], kc[1]))
        if 2.0 < abs(float(d)) < 12.0:
            break
    kx = _grid_rows(kc).reshape(1, 2, 1, hd)
    vx = _grid_rows(vc).reshape(1, 2, 1, hd)
    kcache, ks = _cache_from(kx, hd)
    vcache, vs = _cache_from(vx, hd)
    assert np.all(ks[0, 0, :2] == 1.0) and np.all(vs[0, 0, :2] == 1.0)
    kd = O.dequantize(kcache, ks, hd, 2)[0, 0]
    assert np.array_equal(kd, L32[kc])                     # keys exactly on the grid
    out = O.decode_attention(q.reshape(1, 1, hd), kcache, ks, vcache, vs, [2], hd)[0, 0]

    mpmath.mp.dps = 50
    v0 = [mpmath.mpf(float(L32[c])) for c in vc[0]]
    v1 = [mpmath.mpf(float(L32[c])) for c in vc[1]]
    dm = mpmath.mpf(d.numerator) / d.denominator

    def expect(ratio):
        return np.array([float((a + ratio * b) / (1 + ratio)) for a, b in zip(v0, v1)])

    right = expect(mpmath.exp(dm / mpmath.sqrt(hd)))
    assert np.max(np.abs(out - right)) < 1e-12
    # mutation sensitivity: the wrong temperatures are far from the oracle
    for wrong in (mpmath.exp(dm), mpmath.exp(dm / hd), mpmath.power(2, dm / mpmath.sqrt(hd))):
        assert np.max(np.abs(out - expect(wrong))) > 1e-3


# ------------------------------------------------------ prefill attention --
def test_prefill_single_token_returns_value():
    # l = 1 -> the output row is the dequantised value row
    rng = np.random.default_rng(21)
    k = rng.standard_normal((2, 1, 3, 64)).astype(np.float16)
    v = rng.standard_normal((2, 1, 3, 64)).astype(np.float16)
    q = rng.standard_normal((2, 1, 3, 64)).astype(np.float16)
    kc, ks = _cache_from(k, 64)
    vc, vs = _cache_from(v, 64)
    out = O.prefill_attention(q, kc, ks, vc, vs, [1, 1], 64)
    assert np.array_equal(out[:, 0], O.dequantize(vc, vs, 64, 1)[:, :, 0, :].astype(np.float64))


def test_prefill_identical_keys_causal_mean():
    # identical keys -> uniform weights over j <= i -> the running mean of V
    rng = np.random.default_rng(22)
    k = np.repeat(rng.standard_normal((1, 1, 2, 64)).astype(np.float16), 9, axis=1)
    v = rng.standard_normal((1, 9, 2, 64)).astype(np.float16)
    q = rng.standard_normal((1, 9, 2, 64)).astype(np.float16)
    kc, ks = _cache_from(k, 32)
    vc, vs = _cache_from(v, 32)
    out = O.prefill_attention(q, kc, ks, vc, vs, [9], 32)
    vd = O.dequantize(vc, vs, 32, 9)[0].astype(np.float64)            # [H, 9, hd]
    run = np.cumsum(vd, axis=1) / np.arange(1, 10)[None, :, None]
    assert np.max(np.abs(out[0].transpose(1, 0, 2) - run)) < 1e-12


def test_prefill_causality_and_padding_rows():
    # row i does not depend on tokens > i; rows >= seq_len are zero
    rng = np.random.default_rng(23)
    k = rng.standard_normal((1, 12, 2, 64)).astype(np.float16)
    v = rng.standard_normal((1, 12, 2, 64)).astype(np.float16)
    q = rng.standard_normal((1, 12, 2, 64)).astype(np.float16)
    a = O.prefill_attention(q, *_cache_from(k, 64), *_cache_from(v, 64), [12], 64)
    k2, v2 = k.copy(), v.copy()
    k2[:, 7:] = rng.standard_normal(k2[:, 7:].shape).astype(np.float16)
    v2[:, 7:] = rng.standard_normal(v2[:, 7:].shape).astype(np.float16)
    b = O.prefill_attention(q, *_cache_from(k2, 64), *_cache_from(v2, 64), [12], 64)
    assert np.array_equal(a[:, :7], b[:, :7]) and not np.array_equal(a[:, 7:], b[:, 7:])
    c = O.prefill_attention(q, *_cache_from(k, 64), *_cache_from(v, 64), [5], 64)
    assert np.all(c[:, 5:] == 0) and np.max(np.abs(c[:, :5] - a[:, :5])) < 1e-12


@pytest.mark.parametrize("hd", [64, 128])
def test_prefill_two_token_row_closed_form(hd):
    """Row 1 of a 2-token prompt with grid-exact keys: p1/p0 = exp(q1.(k1 - k0)
    / sqrt(hd)), evaluated at 50 digits from exact rationals (as the decode
    temperature pin); row 0 is v0."""
    rng = np.random.default_rng(3030 + hd)
    kc_ = rng.integers(0, 16, size=(2, hd))
    vc_ = rng.integers(0, 16, size=(2, hd))
    kc_[:, 0] = 15
    vc_[:, 0] = 15
    for _ in range(100):
        q1 = (rng.standard_normal(hd) * 0.35).astype(np.float16)
        d = sum(Fraction(float(a)) * (Fraction(float(L32[c1])) - Fraction(float(L32[c0])))
                for a, c0, c1 in zip(q1, kc_[0], kc_[1]))
        if 2.0 < abs(float(d)) < 12.0:
            break
    q = np.stack([rng.standard_normal(hd).astype(np.float16), q1]).reshape(1, 2, 1, hd)
    kx = _grid_rows(kc_).reshape(1, 2, 1, hd)
    vx = _grid_rows(vc_).reshape(1, 2, 1, hd)
    out = O.prefill_attention(q, *_cache_from(kx, hd), *_cache_from(vx, hd), [2], hd)[0, :, 0]
    mpmath.mp.dps = 50
    r = mpmath.exp((mpmath.mpf(d.numerator) / d.denominator) / mpmath.sqrt(hd))
    want1 = np.array([float((mpmath.mpf(float(L32[a])) + r * mpmath.mpf(float(L32[b]))) / (1 + r))
                      for a, b in zip(vc_[0], vc_[1])])
    assert np.array_equal(out[0], L32[vc_[0]].astype(np.float64))
    assert np.max(np.abs(out[1] - want1)) < 1e-12


def test_prefill_rows_equal_decode_steps():
    # row i of prefill == the (separately pinned) decode attention of q_i over i + 1 tokens
    rng = np.random.default_rng(24)
    k = rng.standard_normal((2, 10, 3, 128)).astype(np.float16) * 3
    v = rng.standard_normal((2, 10, 3, 128)).astype(np.float16)
    q = rng.standard_normal((2, 10, 3, 128)).astype(np.float16)
    kc, ks = _cache_from(k, 64)
    vc, vs = _cache_from(v, 64)
    out = O.prefill_attention(q, kc, ks, vc, vs, [10, 6], 64)
    for i in range(10):
        lens = [min(i + 1, 10), min(i + 1, 6)]
        dec = O.decode_attention(q[:, i], kc, ks, vc, vs, lens, 64)
        for b, L in enumerate([10, 6]):
            if i < L:
                assert np.max(np.abs(out[b, i] - dec[b])) < 1e-12


# ------------------------------------------- KV layouts --
def test_gqa_is_mha_over_repeated_kv_heads():
    # reading R16: query head h reads KV head h // g.  Pinned to
    # the (separately pinned) MHA oracle on a cache whose heads are repeated
    # g times -- a mapping h % H_kv or a wrong group size fails this.
    rng = np.random.default_rng(31)
    B, Hkv, g, hd, T = 2, 2, 4, 64, 9
    k = rng.standard_normal((B, T, Hkv, hd)).astype(np.float16)
    v = rng.standard_normal((B, T, Hkv, hd)).astype(np.float16)
    kc, ks = _cache_from(k, 64)
    vc, vs = _cache_from(v, 64)
    rep = lambda a: np.repeat(a, g, axis=1)      # noqa: E731  kv head j -> query heads j*g .. j*g+g-1
    q = rng.standard_normal((B, Hkv * g, hd)).astype(np.float16)
    a = O.decode_attention(q, kc, ks, vc, vs, [T, 5], 64)
    b = O.decode_attention(q, rep(kc), rep(ks), rep(vc), rep(vs), [T, 5], 64)
    assert np.array_equal(a, b)
    qp = rng.standard_normal((B, T, Hkv * g, hd)).astype(np.float16)
    a = O.prefill_attention(qp, kc, ks, vc, vs, [T, 5], 64)
    b = O.prefill_attention(qp, rep(kc), rep(ks), rep(vc), rep(vs), [T, 5], 64)
    assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        O.decode_attention(q[:, :7], kc, ks, vc, vs, [T, 5], 64)


def test_gqa_single_token_closed_form():
    # SPEC.md:251 per group: one cached token -> every query head of the group
    # returns that KV head's dequantised value
    rng = np.random.default_rng(32)
    k = rng.standard_normal((1, 1, 2, 64)).astype(np.float16)
    v = rng.standard_normal((1, 1, 2, 64)).astype(np.float16)
    kc, ks = _cache_from(k, 64)
    vc, vs = _cache_from(v, 64)
    q = rng.standard_normal((1, 6, 64)).astype(np.float16)
    out = O.decode_attention(q, kc, ks, vc, vs, [1], 64)
    vhat = O.dequantize(vc, vs, 64, 1)[0, :, 0]        # [2][hd]
    for h in range(6):
        assert np.array_equal(out[0, h], vhat[h // 3].astype(np.float64))


def test_paged_layout_identity_table_is_a_reshape():
    # reading R17: with block_table[b][j] = b * maxp + j the paged cache is the
    # contiguous one cut into pages: a numpy reshape/transpose, independent of
    # the oracle's per-token gather
    rng = np.random.default_rng(33)
    B, H, P, maxp, w = 3, 2, 64, 4, 32
    cont = rng.integers(0, 256, (B, H, P * maxp, w), dtype=np.uint8)
    bt = np.arange(B * maxp, dtype=np.int32).reshape(B, maxp)
    pages = cont.reshape(B, H, maxp, P, w).transpose(0, 2, 1, 3, 4).reshape(B * maxp, H, P, w)
    assert np.array_equal(O.paged_to_contiguous(pages, bt, P, P * maxp), cont)
    assert np.array_equal(O.contiguous_to_paged(cont, bt, P, B * maxp), pages)


def test_paged_layout_permuted_pages_round_trip():
    # any injective page assignment: contiguous -> paged -> contiguous is the
    # identity on covered rows, and every used page holds exactly its rows
    rng = np.random.default_rng(34)
    B, H, P, maxp, w = 2, 3, 64, 3, 8
    n_pages = 9
    cont = rng.integers(0, 256, (B, H, P * maxp, w), dtype=np.uint8)
    bt = rng.permutation(n_pages)[:B * maxp].reshape(B, maxp).astype(np.int32)
    pages = O.contiguous_to_paged(cont, bt, P, n_pages)
    assert np.array_equal(O.paged_to_contiguous(pages, bt, P, P * maxp), cont)
    for b in range(B):
        for j in range(maxp):
            assert np.array_equal(pages[bt[b, j]], cont[b, :, j * P:(j + 1) * P])
    unused = sorted(set(range(n_pages)) - set(bt.ravel().tolist()))
    assert all(not pages[u].any() for u in unused)
