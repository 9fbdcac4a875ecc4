"""NQKV CPU oracle -- TEST INFRASTRUCTURE ONLY.

This module is the plain, slow, obviously-correct reference for the NQKV hot
path (arXiv 2505.16210).  It is NOT part of the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The CUDA path
(``paper_2505_16210_b200``) never imports it and shares no code with it.

Every function follows the paper or the CPU spec written from it
 step by step; line numbers refer to /root/reference/PAPER.md and
/root/reference/SPEC.md.  Floating point is float64 except where the method
fixes fp32 (the level table is rounded to fp32, x/s is an IEEE fp32 division,
dequantisation is one fp32 multiply) -- see DESIGN.md "Readings".

Pins (tests/test_oracle_pins.py) tie each function to something other than
itself: 50-digit mpmath quantiles, closed forms (grid fixed point, zero block,
single-token / identical-key attention), brute force, the round-trip bound,
and the paper's worked geometry (Fig. 5 caption).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import ndtri  # float64 inverse standard-normal CDF

NBITS = 4
NLEVELS = 1 << NBITS
ZERO_CODE = 7  # index of the exact 0.0 level (7 negative levels below it)


# --------------------------------------------------------------------------
# a0. NF4 level table
# --------------------------------------------------------------------------
def nf_offset(bits: int = NBITS) -> float:
    """delta = 1 - 1/2 (1/(2*2^k) + 1/(2*(2^k - 1)))."""
    n = 1 << bits
    return 1.0 - 0.5 * (1.0 / (2.0 * n) + 1.0 / (2.0 * (n - 1)))


def nf_levels_f64(bits: int = NBITS) -> np.ndarray:
    """NormalFloat codebook in float64 (PAPER.md:72, 82, 201 cite QLoRA's NF4;
    the explicit quantile recipe is SPEC.md:55-63).

    Negative side: 2^(k-1) quantiles for probabilities from delta down to 0.5;
    positive side: 2^(k-1)+1 quantiles from 0.5 up to delta; merge the shared
    0.5 point (exact zero); divide by the largest magnitude Phi^-1(delta).
    """
    if not 2 <= bits <= 8:
        raise ValueError("bits must be in [2, 8]")
    delta = nf_offset(bits)
    half = 1 << (bits - 1)
    # SPEC.md:58 evaluates 2^(k-1) quantiles on the negative side *including*
    # the 0.5 point and 2^(k-1)+1 on the positive side including 0.5; after
    # merging the shared zero this leaves 2^(k-1)-1 negatives, one zero and
    # 2^(k-1) positives = 2^k values (7 / 1 / 8 for NF4).
    neg = -ndtri(np.linspace(delta, 0.5, half)[:-1])
    pos = ndtri(np.linspace(0.5, delta, half + 1)[1:])
    vals = np.concatenate([neg, [0.0], pos])
    vals = vals / ndtri(delta)
    return np.sort(vals)


def nf_levels_f32(bits: int = NBITS) -> np.ndarray:
    """The level table the method stores and computes with: RN-to-fp32 of the
    float64 values (reading R1)."""
    return nf_levels_f64(bits).astype(np.float32)


# --------------------------------------------------------------------------
# a1-a2. per-block absmax + nearest level (brute force, ties -> lower index)
# --------------------------------------------------------------------------
def quantize_blocks(x_blocks: np.ndarray, levels32: np.ndarray | None = None):
    """Block-wise NF4 quantisation.

    x_blocks: float16 array [..., blk] -- each trailing row is one block.
    Returns (scales float32 [...], codes uint8 [..., blk]).

    scale  = max |x| over the block, computed in fp32 (exact: it is an fp16 value)
    n      = fp32(x) / fp32(scale)   -- IEEE round-to-nearest fp32 division
    code   = argmin_i |n - L_i| evaluated in float64, first minimum wins
             (ties -> lower index)
    scale == 0  ->  all codes = index of the zero level
    """
    if levels32 is None:
        levels32 = nf_levels_f32()
    x = np.asarray(x_blocks)
    if x.dtype != np.float16:
        raise TypeError("quantize_blocks expects float16 input")
    xf = x.astype(np.float32)
    if not np.all(np.isfinite(xf)):
        raise ValueError("non-finite input (SPEC.md:68)")
    scales = np.max(np.abs(xf), axis=-1)
    safe = np.where(scales > 0, scales, np.float32(1.0)).astype(np.float32)
    n = (xf / safe[..., None]).astype(np.float32)
    codes = nearest_level_codes(n, levels32)
    codes[scales == 0] = ZERO_CODE
    return scales.astype(np.float32), codes


def nearest_level_codes(n32: np.ndarray, levels32: np.ndarray | None = None) -> np.ndarray:
    """Brute force over the 16 levels: argmin_i |n - L_i| in float64 (exact for
    fp32 n and fp32 L), first minimum wins -> ties go to the lower index
    (SPEC.md:67, 72, 111)."""
    if levels32 is None:
        levels32 = nf_levels_f32()
    lv = np.asarray(levels32, dtype=np.float32).astype(np.float64)
    n = np.asarray(n32, dtype=np.float32)
    codes = np.empty(n.shape, dtype=np.uint8)
    flat_n = n.reshape(-1)
    flat_c = codes.reshape(-1)
    step = 1 << 20
    for i in range(0, flat_n.size, step):
        d = np.abs(flat_n[i:i + step].astype(np.float64)[:, None] - lv[None, :])
        flat_c[i:i + step] = np.argmin(d, axis=1)  # first minimum = lower index
    return codes


def thresholds_f32(levels32: np.ndarray | None = None) -> np.ndarray:
    """Decision thresholds equivalent to the brute-force argmin on fp32 n:
    T_i = RD32((L_i + L_{i+1}) / 2), the exact midpoint rounded toward -inf.
    code(n) = #{i : n > T_i}.  Used only to vectorise the exhaustive sweep;
    pinned against quantize_blocks' brute force in the tests."""
    if levels32 is None:
        levels32 = nf_levels_f32()
    lv = levels32.astype(np.float64)
    mid = (lv[:-1] + lv[1:]) / 2.0                 # exact in float64
    t = mid.astype(np.float32)
    over = t.astype(np.float64) > mid
    t[over] = np.nextafter(t[over], np.float32(-np.inf))
    return t


def codes_by_threshold(n32: np.ndarray, levels32: np.ndarray | None = None) -> np.ndarray:
    """code = #{i : n > T_i} for fp32 n (same result as the brute force)."""
    t = thresholds_f32(levels32)
    return np.searchsorted(t, np.asarray(n32, dtype=np.float32), side="left").astype(np.uint8)


# --------------------------------------------------------------------------
# a3. pack + append into the cache layout
# --------------------------------------------------------------------------
def pack_nibbles(codes: np.ndarray) -> np.ndarray:
    """Element 2i -> low nibble, 2i+1 -> high nibble of byte i."""
    c = np.asarray(codes, dtype=np.uint8)
    assert c.shape[-1] % 2 == 0
    return (c[..., 0::2] | (c[..., 1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed: np.ndarray) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.shape[:-1] + (p.shape[-1] * 2,), dtype=np.uint8)
    out[..., 0::2] = p & 0xF
    out[..., 1::2] = p >> 4
    return out


def heads_per_block(hd: int, blk: int) -> int:
    """blk <= hd: a block is blk channels of one head (1).  blk > hd: a block
    is the hidden-state slice of blk / hd adjacent heads of one token -- the
    paper's own setting, blk 256 over OPT's hidden dimension (PAPER.md:141,
    302; reading R2b)."""
    if blk <= hd:
        if hd % blk:
            raise ValueError("blk must divide hd")
        return 1
    if blk % hd:
        raise ValueError("hd must divide blk")
    return blk // hd


def empty_cache(B: int, H: int, Tc: int, hd: int, blk: int):
    """codes uint8 [B][H][Tc][hd/2]; scales float32 [B][H][Tc][hd/blk], or
    [B][H*hd/blk][Tc][1] when a block spans blk/hd heads."""
    hpb = heads_per_block(hd, blk)
    if H % hpb:
        raise ValueError("a block may not straddle the last head")
    return (np.zeros((B, H, Tc, hd // 2), np.uint8),
            np.zeros((B, H // hpb, Tc, max(hd // blk, 1)), np.float32))


def quantize_append(x: np.ndarray, pos, blk: int, codes: np.ndarray, scales: np.ndarray,
                    levels32: np.ndarray | None = None) -> None:
    """I <- Concat(I, quantize_NF4(x)).

    x: float16 [B][n_new][H][hd] (token-major, as a QKV projection emits it).
    Rows pos[b] .. pos[b]+n_new-1 of codes/scales are written; every other
    byte is left untouched (append-only).  A block is blk
    consecutive channels of one (token, head) -- DESIGN.md reading R2.
    With blk > hd a block is the slice of blk/hd adjacent heads of one token's
    hidden state (the paper's blk 256 over d): scales then
    hold one value per (token, head group).
    """
    x = np.asarray(x)
    B, n_new, H, hd = x.shape
    hpb = heads_per_block(hd, blk)
    nb = max(hd // blk, 1)
    # [H, hd] -> [H/hpb groups, nb blocks per group, blk]: hd is contiguous and
    # heads are adjacent in a token's hidden state
    blocks = x.reshape(B, n_new, H // hpb, nb, blk)
    s, c = quantize_blocks(blocks, levels32)              # [B,n,Hs,nb], [B,n,Hs,nb,blk]
    packed = pack_nibbles(c.reshape(B, n_new, H, hd))     # [B,n,H,hd/2]
    for b in range(B):
        p0 = int(pos[b])
        codes[b, :, p0:p0 + n_new, :] = packed[b].transpose(1, 0, 2)
        scales[b, :, p0:p0 + n_new, :] = s[b].transpose(1, 0, 2)


# --------------------------------------------------------------------------
# a4. dequantisation by table lookup
# --------------------------------------------------------------------------
def dequantize(codes: np.ndarray, scales: np.ndarray, blk: int, n_tokens: int | None = None,
               out_dtype=np.float32, levels32: np.ndarray | None = None) -> np.ndarray:
    """X' = dequantize_NF4(I): v = RN32(scale * L[code])  (
    SPEC.md:73-81).  fp16 output is RN16 of that fp32 value.

    codes [B][H][Tc][hd/2], scales [B][H][Tc][hd/blk] (blk > hd:
    [B][H*hd/blk][Tc][1]) -> [B][H][n_tokens][hd].
    """
    if levels32 is None:
        levels32 = nf_levels_f32()
    B, H, Tc, hb = codes.shape
    hd = hb * 2
    hpb = heads_per_block(hd, blk)
    if n_tokens is None:
        n_tokens = Tc
    c = unpack_nibbles(codes[:, :, :n_tokens, :])                 # [B,H,n,hd]
    lv = levels32[c]                                              # fp32 lookup
    s = scales[:, :, :n_tokens, :]
    if hpb > 1:                      # head group g -> heads g*hpb .. g*hpb+hpb-1
        s = np.repeat(s, hpb, axis=1)
    s = np.repeat(s, min(blk, hd), axis=-1)                       # [B,H,n,hd]
    v = (s.astype(np.float32) * lv.astype(np.float32)).astype(np.float32)
    return v.astype(out_dtype)


# --------------------------------------------------------------------------
# KV layouts orthogonal to the method
# --------------------------------------------------------------------------
def kv_group(h_q: int, h_kv: int) -> int:
    """Query heads per cache head (grouped-query attention, reading R16)."""
    if h_kv <= 0 or h_q % h_kv:
        raise ValueError("the number of query heads must be a multiple of the KV heads")
    return h_q // h_kv


def paged_to_contiguous(pages: np.ndarray, block_table, page_size: int, n_tokens: int) -> np.ndarray:
    """A paged cache, the layout of PagedAttention that PAPER.md:62, 103
    calls orthogonal to NQKV (reading R17), as the contiguous one: token t
    of sequence b lives in row t % P of page block_table[b][t // P];
    pages: [n_pages][H][P][w] -> [B][H][n_tokens][w] (rows the table does not
    cover are zero).  A plain gather: it does no arithmetic of the method."""
    bt = np.asarray(block_table)
    B = bt.shape[0]
    n_pages, H, P, w = pages.shape
    if P != page_size:
        raise ValueError("page size mismatch")
    out = np.zeros((B, H, n_tokens, w), pages.dtype)
    for b in range(B):
        for t in range(n_tokens):
            if t // P < bt.shape[1]:
                out[b, :, t, :] = pages[int(bt[b, t // P]), :, t % P, :]
    return out


def contiguous_to_paged(cache: np.ndarray, block_table, page_size: int, n_pages: int) -> np.ndarray:
    """Inverse of paged_to_contiguous for the rows the table covers:
    [B][H][Tc][w] -> [n_pages][H][P][w] (pages no sequence uses are zero)."""
    bt = np.asarray(block_table)
    B, H, Tc, w = cache.shape
    out = np.zeros((n_pages, H, page_size, w), cache.dtype)
    for b in range(B):
        for t in range(min(Tc, bt.shape[1] * page_size)):
            out[int(bt[b, t // page_size]), :, t % page_size, :] = cache[b, :, t, :]
    return out


# --------------------------------------------------------------------------
# a5-a7. decode attention over the dequantised cache (float64)
# --------------------------------------------------------------------------
def decode_attention(q: np.ndarray, k_codes, k_scales, v_codes, v_scales, seq_lens, blk: int,
                     softmax_scale: float | None = None, levels32=None) -> np.ndarray:
    """t_O = Softmax(t_Q X_K'^T / sqrt(hd)) X_V'  per (b, h)  (
    the 1/sqrt(hd) factor is reading R6).

    q: float16 [B][H][hd]; seq_lens[b] counts the cached tokens including the
    token appended this step (append-before-attend).  Positions
    >= seq_lens[b] are not part of the sequence.  seq_lens[b] == 0 -> zeros
    (reading R12).  Computed in float64 over the fp32 dequantised values.

    Grouped-query layout (reading R16): the cache may hold fewer
    heads than q (H_kv | H); query head h reads cache head h // (H / H_kv),
    consecutive query heads sharing one KV head (the multi-query / grouped
    attention the paper names as orthogonal to NQKV).
    """
    B, H, hd = q.shape
    g = kv_group(H, k_codes.shape[1])
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    out = np.zeros((B, H, hd), np.float64)
    for b in range(B):
        L = int(seq_lens[b])
        if L == 0:
            continue
        K = dequantize(k_codes[b:b + 1], k_scales[b:b + 1], blk, L, np.float32, levels32)[0]
        V = dequantize(v_codes[b:b + 1], v_scales[b:b + 1], blk, L, np.float32, levels32)[0]
        for h in range(H):
            qh = q[b, h].astype(np.float64)
            s = (K[h // g].astype(np.float64) @ qh) * float(softmax_scale)
            s = s - s.max()
            p = np.exp(s)
            p = p / p.sum()
            out[b, h] = p @ V[h // g].astype(np.float64)
    return out


def prefill_attention(q: np.ndarray, k_codes, k_scales, v_codes, v_scales, seq_lens, blk: int,
                      softmax_scale: float | None = None, levels32=None) -> np.ndarray:
    """Causal attention of the prompt's own queries over the DEQUANTISED
    prompt cache (PAPER.md:213-221 prefill phase: I_K = quantize_NF4(X_K), the
    cache holds indices; causal multi-head scaled dot-product
    attention over the dequantised K, V, so prefill and decode see the same
    quantised world).  The 1/sqrt(hd) factor is reading R6.

    q: float16 [B][T][H][hd] (token-major, as the projections produce it);
    row i of sequence b attends to cached tokens j <= i, j < seq_lens[b].
    Returns float64 [B][T][H][hd]; rows i >= seq_lens[b] are 0.
    """
    B, T, H, hd = q.shape
    g = kv_group(H, k_codes.shape[1])
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    out = np.zeros((B, T, H, hd), np.float64)
    for b in range(B):
        L = min(int(seq_lens[b]), T)
        if L == 0:
            continue
        K = dequantize(k_codes[b:b + 1], k_scales[b:b + 1], blk, L, np.float32, levels32)[0]
        V = dequantize(v_codes[b:b + 1], v_scales[b:b + 1], blk, L, np.float32, levels32)[0]
        for h in range(H):
            Q = q[b, :L, h].astype(np.float64)                        # [L, hd]
            S = (Q @ K[h // g].astype(np.float64).T) * float(softmax_scale)  # [L, L]
            S[np.triu_indices(L, 1)] = -np.inf                         # causal: j <= i
            S = S - S.max(axis=1, keepdims=True)
            P = np.exp(S)
            P = P / P.sum(axis=1, keepdims=True)
            out[b, :L, h] = P @ V[h // g].astype(np.float64)
    return out


def attention_weights(q_h: np.ndarray, K_h: np.ndarray, softmax_scale: float) -> np.ndarray:
    """Softmax row for one head (diagnostic)."""
    s = (K_h.astype(np.float64) @ q_h.astype(np.float64)) * softmax_scale
    s = s - s.max()
    p = np.exp(s)
    return p / p.sum()


# --------------------------------------------------------------------------
# Byte model -- used by the harness
# --------------------------------------------------------------------------
def cache_bytes(tokens: int, d: int, blk: int, scale_bytes: int = 4, layers: int = 1) -> int:
    """Stored bytes of K and V: 2 x tokens x (ceil(d/2) + ceil(d/blk) x scale_bytes)."""
    return layers * 2 * tokens * ((d + 1) // 2 + -(-d // blk) * scale_bytes)


def fp16_kv_bytes(layers: int, batch: int, seq: int, d: int) -> int:
    """Unquantised fp16 KV cache bytes: 2 (K,V) x layers x b x s x d x 2 B."""
    return 2 * layers * batch * seq * d * 2
