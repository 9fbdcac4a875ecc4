// a4-a7: fused dequant-in-registers decode attention (+ optional fused
// 1-token append) and the split-K combine kernel.
//
// X' = dequantize_NF4(I); A = Softmax(t_Q X_K'^T); t_O = A X_V'
// (the 1/sqrt(hd) factor is DESIGN.md reading R6).  The dequantised cache is
// never written anywhere: codes stream from HBM into registers and are turned
// into fp32 levels by shared-memory table lookups.
//
// Work decomposition.  A work item is (b, h, 128-token segment); the
// segmentation depends on seq_len only and partials are merged in segment
// order, so results are independent of B, H, the grid and the GPU.  Items are
// assigned statically (strided) to the warps of a persistent grid; each
// WARP streams its items as one continuous sequence of stages:
//   - a stage = kTPS tokens per lane (ST = G*kTPS tokens per warp);
//   - stages live in a kRing-deep register ring, loads run kRing-1 stages
//     ahead and cross item boundaries, so the next item's first stages are in
//     flight while the current item is finished;
//   - per-item q (and, when fusing the append, the new token's raw k/v) are
//     prefetched into per-warp shared memory with cp.async when the load side
//     enters the item; item descriptors travel through a 4-entry smem queue.
// Each lane owns 16 consecutive head dims (8 packed bytes): LPT = hd/16
// lanes cover a token row, G = 32/LPT token groups per warp.
//
// Dequantisation.  A packed byte (two 4-bit codes) becomes the pair
// (L[lo], L[hi]) through ONE shared-memory load from a 256-entry fp32-pair
// table replicated per lane (64 KB, conflict-free: lane l reads bank pair 2l),
// addressed by one PRMT that splices the code byte above lane*8; the pair feeds
// one FFMA2.  Scores use fp32 levels with the block scale applied once per
// 16 dims; values accumulate w*L with w = p * scale (online softmax per stage).
#pragma once
#include "common.cuh"

namespace nqkv {

constexpr int kSeg = 128;
constexpr int kTPS = 4;          // tokens per lane per stage
constexpr int kLutBytes = 256 * 32 * 8;
constexpr int kMaxBatch = 4096;
#ifndef NQKV_DECODE_WARPS
#define NQKV_DECODE_WARPS 12
#endif
#ifndef NQKV_RING
#define NQKV_RING 3
#endif
constexpr int kDecodeWarps = NQKV_DECODE_WARPS;
constexpr int kRing = NQKV_RING;   // stage ring depth: loads run kRing-1 stages ahead
constexpr int kQueue = 4;

struct DecodeParams {
  const __half* q;
  const uint8_t* kc;
  const float* ks;
  const uint8_t* vc;
  const float* vs;
  const int32_t* seq_lens;
  const __half* k_new;      // fused append (nullptr: attention only)
  const __half* v_new;
  long long new_sb, new_sh; // element strides of k_new / v_new ([B][H][hd])
  float* out;
  float* ws_o;              // [B*H*max_segs][hd]  split partials
  float2* ws_ml;            // [B*H*max_segs]      (max, sum) per partial
  int* sched;               // [2]: item counter, exited-warp counter
  int B, H, Tc, blk_shift, max_segs;
  float scale_log2;         // softmax_scale * log2(e)
  Levels lv;
  BucketTab tab;
};

constexpr int kLaneDims = 16;      // head dims owned by one lane

template <int HD>
struct DecodeShape {
  static constexpr int LPT = HD / kLaneDims;
  static constexpr int G = 32 / LPT;
  static constexpr int ST = G * kTPS;
  // per-warp shared memory block
  static constexpr int kRed = 0;                                  // 32 lanes x 16 floats = 2 KB
  static constexpr int kQ = 2048;                                 // kQueue x hd fp16
  static constexpr int kNew = kQ + kQueue * HD * 2;               // kQueue x {k, v} x hd fp16
  static constexpr int kDesc = kNew + kQueue * 2 * HD * 2;        // kQueue x 8 ints
  static constexpr int kWarpBytes = kDesc + kQueue * 8 * 4;
};

// Shared-memory layout.  The pair LUT must start on a 64 KB boundary of the
// shared window so that ONE PRMT can produce a complete LDS address
// (byte 0 = lane*8, byte 1 = code byte, bytes 2-3 = LUT base >> 16): the
// dynamic window starts at 0x400 (1 KB driver reserve), so the LUT goes at
// dynamic offset kLutOff = 0xFC00 and the warp blocks fill the space before
// it when they fit (checked on device; a mismatch traps).
constexpr int kLutOff = 0xFC00;
template <int HD, int NW>
struct SmemLayout {
  static constexpr int kWarps = NW * DecodeShape<HD>::kWarpBytes;
  static constexpr int kSmall = 512;                                  // bucket tab + levels
  static constexpr bool kBefore = kWarps + kSmall <= kLutOff;
  static constexpr int kWarpOff = kBefore ? 0 : kLutOff + kLutBytes;
  static constexpr int kSmallOff = kWarpOff + kWarps;
  static constexpr int kTailOff = kBefore ? kLutOff + kLutBytes : kSmallOff + kSmall;   // prefix + lens
  static constexpr size_t bytes(int B) {
    return static_cast<size_t>(kTailOff) + static_cast<size_t>(2 * B + 1) * sizeof(int);
  }
};

struct Stage {
  uint2 k[kTPS], v[kTPS];     // 8 packed bytes = 16 codes per lane per token
  float ks[kTPS], vs[kTPS];
};

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait(int newer) {   // groups allowed to stay pending
  if (newer <= 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
  else if (newer == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
  else if (newer == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
  else asm volatile("cp.async.wait_group 3;" ::: "memory");
}

// Quantize this lane's 16 dims of the appended token (fp16, from shared
// memory) exactly as nqkv_quantize would: block absmax across the blk/16
// adjacent lanes of the block, then the code of every element.  Kept out of
// line: it runs once per (b, h) and would otherwise be inlined per ring slot.
struct NewTok {
  uint2 k, v;
  float ks, vs;
};

__device__ __forceinline__ uint2 quantize_lane16(const __half* src, int blk_lanes, uint32_t tab,
                                                 float& scale) {
  const uint4 r0 = reinterpret_cast<const uint4*>(src)[0];
  const uint4 r1 = reinterpret_cast<const uint4*>(src)[1];
  float s = fmaxf(absmax8(r0), absmax8(r1));
  for (int o = 1; o < blk_lanes; o <<= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
  const float r = block_rcp(s);
  scale = s;
  return make_uint2(encode8(r0, r, tab), encode8(r1, r, tab));
}

__device__ __noinline__ NewTok quantize_new_token(const __half* nb, int sub, int hd, int blk_lanes,
                                                  uint32_t tab) {
  NewTok t;
  t.k = quantize_lane16(nb + sub * kLaneDims, blk_lanes, tab, t.ks);
  t.v = quantize_lane16(nb + hd + sub * kLaneDims, blk_lanes, tab, t.vs);
  return t;
}

// lane_sel: byte 0 = lane*8 (this lane's replica inside a 256-B LUT entry),
// bytes 2-3 = the LUT's 64 KB-aligned shared address >> 16.  One PRMT splices
// the code byte k of `word` in as byte 1 -> the full LDS address.
__device__ __forceinline__ uint64_t lut_pair(uint32_t word, int k, uint32_t lane_sel) {
  return lds64(__byte_perm(word, lane_sel, 0x7604 | (k << 4)));
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// One stage: kTPS tokens per lane.  The online softmax runs per token GROUP
// (the G groups of a warp see disjoint tokens; the LPT lanes of a group hold
// identical scores), so no cross-lane max is needed per stage; groups are
// merged once per item in close_item().
template <int HD>
__device__ __forceinline__ void compute_stage(const Stage& S, int tok0, int end, int g,
                                              const uint64_t (&q2)[8], uint64_t (&o2)[8],
                                              float& m, float& l, uint32_t lane_sel,
                                              float scale_log2) {
  using Sh = DecodeShape<HD>;
  constexpr int LPT = Sh::LPT;
  float sc[kTPS];
#pragma unroll
  for (int i = 0; i < kTPS; ++i) {
    // two independent fp32x2 chains over the lane's 8 packed bytes
    uint64_t a0 = 0, a1 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a0 = ffma2(q2[k], lut_pair(S.k[i].x, k, lane_sel), a0);
      a1 = ffma2(q2[4 + k], lut_pair(S.k[i].y, k, lane_sel), a1);
    }
    const float2 a = unpack2(fadd2(a0, a1));
    sc[i] = (a.x + a.y) * S.ks[i];
  }
#pragma unroll
  for (int o = 1; o < LPT; o <<= 1) {
#pragma unroll
    for (int i = 0; i < kTPS; ++i) sc[i] += __shfl_xor_sync(0xffffffffu, sc[i], o);
  }
  float mt = m;
#pragma unroll
  for (int i = 0; i < kTPS; ++i) {
    sc[i] = (tok0 + i * Sh::G + g < end) ? sc[i] * scale_log2 : -INFINITY;
    mt = fmaxf(mt, sc[i]);
  }
  // rescale unconditionally (corr = 1 when the group max did not move).  A
  // group that has seen only masked tokens keeps m = -inf; subtracting the
  // finite ms keeps every exponent -inf or finite (ex2(-inf) = 0, no NaN).
  const float ms = fmaxf(mt, -3.0e38f);
  const float corr = fast_exp2(m - ms);
  m = mt;
  l *= corr;
  const uint64_t c2 = pack2(corr, corr);
#pragma unroll
  for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], c2);
#pragma unroll
  for (int i = 0; i < kTPS; ++i) {
    const float pr = fast_exp2(sc[i] - ms);
    l += pr;
    const float w = pr * S.vs[i];
    const uint64_t w2 = pack2(w, w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o2[k] = ffma2(lut_pair(S.v[i].x, k, lane_sel), w2, o2[k]);
      o2[4 + k] = ffma2(lut_pair(S.v[i].y, k, lane_sel), w2, o2[4 + k]);
    }
  }
}

// Load side: walks items/stages two stages ahead of the compute side.
struct LoadCursor {
  int active;            // 1 while items remain
  int next;              // prefetched item id (atomic result, lane-0 value broadcast)
  int q;                 // queue position of the item being loaded
  int st, nst, start, end;
  long long row0;
};

template <int HD, int NW>
__global__ void __launch_bounds__(NW * 32, 1) decode_kernel(const DecodeParams p) {
  using Sh = DecodeShape<HD>;
  constexpr int LPT = Sh::LPT, G = Sh::G, ST = Sh::ST;
  constexpr int DPL = HD / 32;   // output dims per lane after the group reduction
  extern __shared__ __align__(16) unsigned char smem[];
  using Lay = SmemLayout<HD, NW>;
  unsigned char* wbase_all = smem + Lay::kWarpOff;
  unsigned char* gbase = smem + Lay::kSmallOff;
  float2* s_tab = reinterpret_cast<float2*>(gbase);
  float* s_lv = reinterpret_cast<float*>(gbase + 384);
  int* s_pref = reinterpret_cast<int*>(smem + Lay::kTailOff);          // [B+1]
  int* s_len = s_pref + p.B + 1;                                     // [B]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wb = wbase_all + warp * Sh::kWarpBytes;
  float* red = reinterpret_cast<float*>(wb + Sh::kRed);
  __half* qbuf = reinterpret_cast<__half*>(wb + Sh::kQ);
  __half* nbuf = reinterpret_cast<__half*>(wb + Sh::kNew);
  int* desc = reinterpret_cast<int*>(wb + Sh::kDesc);

  // ---- prologue independent of the previous kernel: tables + pair LUT
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) s_lv[k] = p.lv.v[k];
  }
  for (int i = threadIdx.x; i < kNumBuckets; i += blockDim.x) s_tab[i] = p.tab.e[i];
  __syncthreads();
  {
    float4* lut4 = reinterpret_cast<float4*>(smem + kLutOff);
    for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
      const int e = i >> 4;
      const float lo = s_lv[e & 15], hi = s_lv[e >> 4];
      lut4[i] = make_float4(lo, hi, lo, hi);
    }
  }
  pdl_trigger();
  pdl_wait();
  // ---- per-batch lengths and item prefix: items(b) = H * max(1, ceil(len/kSeg))
  if (warp == 0) {
    int carry = 0;
    if (lane == 0) s_pref[0] = 0;
    for (int b0 = 0; b0 < p.B; b0 += 32) {
      const int b = b0 + lane;
      int n = 0;
      if (b < p.B) {
        const int len = min(max(p.seq_lens[b], 0), p.Tc);
        s_len[b] = len;
        n = p.H * max(1, (len + kSeg - 1) / kSeg);
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, n, o);
        if (lane >= o) n += v;
      }
      if (b < p.B) s_pref[b + 1] = carry + n;
      carry += __shfl_sync(0xffffffffu, n, 31);
    }
  }
  __syncthreads();
  const int total = s_pref[p.B];
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(smem + kLutOff));
  if (lut & 0xFFFFu) __trap();        // the single-PRMT address needs a 64 KB-aligned LUT
  const uint32_t lane_sel = (lut & 0xFFFF0000u) | (lane * 8u);
  const uint32_t tab = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
  const int g = lane / LPT, sub = lane % LPT;
  const int nblk = HD >> p.blk_shift;
  const int sidx = (sub * kLaneDims) >> p.blk_shift;
  const bool fused = p.k_new != nullptr;
  const int blk_lanes = (1 << p.blk_shift) / kLaneDims;

  // Static strided schedule: warp w takes items w, w + W, w + 2W, ... (items
  // are near-uniform in cost; a global atomic queue was measured to serialise
  // ~2k warps on one address at kernel start).
  const int gwarp = static_cast<int>(blockIdx.x) * NW + warp;
  const int nwarps = static_cast<int>(gridDim.x) * NW;
  int sched_next = gwarp;
  auto fetch = [&]() -> int {
    const int v = sched_next;
    sched_next += nwarps;
    return v;
  };

  // Load side: enter the next scheduled item that has tokens -- decode it,
  // publish its descriptor in the queue and prefetch q (and, for the item
  // holding the appended token, the raw new k/v) with cp.async.  Empty
  // sequences are finished right here (out = 0, reading R12).
  // Returns false when the scheduler is exhausted.
  LoadCursor L;
  L.q = 0;
  auto enter_next = [&]() -> bool {
    for (;;) {
      const int item = __shfl_sync(0xffffffffu, L.next, 0);
      if (item >= total) return false;
      L.next = fetch();
      int lo = 0, hi = p.B;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid] <= item) lo = mid; else hi = mid;
      }
      const int b = lo;
      const int len = s_len[b];
      const int nseg = max(1, (len + kSeg - 1) / kSeg);
      const int r = item - s_pref[b];
      const int h = r / nseg, seg = r - h * nseg;
      const int bh = b * p.H + h;
      if (len == 0) {
        for (int d = lane; d < HD; d += 32) p.out[static_cast<long long>(bh) * HD + d] = 0.0f;
        continue;
      }
      const int start = seg * kSeg;
      const int end = min(len, start + kSeg);
      const int row_new = (fused && len - 1 >= start && len - 1 < end) ? len - 1 : -1;
      const int slot = L.q & (kQueue - 1);
      if (lane == 0) {
        int* d = desc + slot * 8;
        d[0] = bh; d[1] = start; d[2] = end; d[3] = nseg; d[4] = seg; d[5] = row_new;
      }
      constexpr int CH = HD * 2 / 16;       // 16-byte chunks per fp16 row (8 or 16)
      const uint32_t qs = static_cast<uint32_t>(__cvta_generic_to_shared(qbuf + slot * HD));
      if (lane < CH) cp_async16(qs + lane * 16, p.q + static_cast<long long>(bh) * HD + lane * 8);
      if (row_new >= 0) {
        const uint32_t ns = static_cast<uint32_t>(__cvta_generic_to_shared(nbuf + slot * 2 * HD));
        const long long off = static_cast<long long>(b) * p.new_sb + static_cast<long long>(h) * p.new_sh;
        if (lane < CH) cp_async16(ns + lane * 16, p.k_new + off + lane * 8);
        else if (lane < 2 * CH) cp_async16(ns + HD * 2 + (lane - CH) * 16, p.v_new + off + (lane - CH) * 8);
      }
      cp_async_commit();
      L.st = 0;
      L.nst = (end - start + ST - 1) / ST;
      L.start = start;
      L.end = end;
      L.row0 = static_cast<long long>(bh) * p.Tc;
      ++L.q;
      return true;
    }
  };
  auto advance = [&]() {
    if (++L.st >= L.nst) L.active = enter_next();
  };

  auto issue = [&](Stage& S) {
    const int tok0 = L.start + L.st * ST;
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      const int t = min(tok0 + i * G + g, L.end - 1);
      const long long row = L.row0 + t;
#ifdef NQKV_DBG_NOLOAD
      S.k[i] = make_uint2(row, row * 3); S.v[i] = make_uint2(row * 5, row * 7);
      S.ks[i] = 1.0f; S.vs[i] = 1.0f;
      continue;
#endif
      S.k[i] = ldg_stream_64(p.kc + row * (HD / 2) + sub * (kLaneDims / 2));
      S.v[i] = ldg_stream_64(p.vc + row * (HD / 2) + sub * (kLaneDims / 2));
      S.ks[i] = ldg_f32(p.ks + row * nblk + sidx);
      S.vs[i] = ldg_f32(p.vs + row * nblk + sidx);
    }
  };

  // ---- compute-side state
  int cq = 0, cst = 0, cnst = 0, cstart = 0, cend = 0, cbh = 0, cnseg = 1, cseg = 0, crow_new = -1;
  bool copen = false;
  uint64_t q2[8], o2[8];
  float m = -INFINITY, l = 0.0f;

  auto open_item = [&]() {
    __syncwarp();
    const int slot = cq & (kQueue - 1);
    const int* d = desc + slot * 8;
    cbh = d[0]; cstart = d[1]; cend = d[2]; cnseg = d[3]; cseg = d[4]; crow_new = d[5];
    cnst = (cend - cstart + ST - 1) / ST;
    cst = 0;
    cp_async_wait(L.q - cq - 1);      // this item's prefetch group has landed
    __syncwarp();
    const uint4* qp = reinterpret_cast<const uint4*>(qbuf + slot * HD + sub * kLaneDims);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint4 rq = qp[j];
      const uint32_t w4[4] = {rq.x, rq.y, rq.z, rq.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __half2 h2;
        memcpy(&h2, &w4[k], 4);
        const float2 f = __half22float2(h2);
        q2[j * 4 + k] = pack2(f.x, f.y);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) o2[j] = 0;
    m = -INFINITY;
    l = 0.0f;
    copen = true;
  };

  auto close_item = [&]() {
    // merge the G per-group softmax states: common max M, rescale, sum l
    float M = m;
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float f = fast_exp2(m - M);          // 0 for a group that saw no token
    l *= f;
    const uint64_t f2 = pack2(f, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], f2);
    m = M;
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    {
      // lane -> smem: 4 16-byte chunks per lane, xor-swizzled
      float4* r4 = reinterpret_cast<float4*>(red);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float2 a = unpack2(o2[2 * c]), bb = unpack2(o2[2 * c + 1]);
        r4[lane * 4 + (c ^ (lane & 3))] = make_float4(a.x, a.y, bb.x, bb.y);
      }
    }
    __syncwarp();
    float res[DPL];
#pragma unroll
    for (int d = 0; d < DPL; ++d) res[d] = 0.0f;
    {
      const int dim0 = lane * DPL;
      const int src_sub = dim0 / kLaneDims, c = (dim0 % kLaneDims) / 4, off = dim0 % 4;
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const int sl = gg * LPT + src_sub;
        const float* src = red + (sl * 4 + (c ^ (sl & 3))) * 4 + off;
#pragma unroll
        for (int d = 0; d < DPL; ++d) res[d] += src[d];
      }
    }
    __syncwarp();
    float* dst;
    if (cnseg == 1) {
      const float inv = 1.0f / l;
#pragma unroll
      for (int d = 0; d < DPL; ++d) res[d] *= inv;
      dst = p.out + static_cast<long long>(cbh) * HD + lane * DPL;
    } else {
      const long long slot = static_cast<long long>(cbh) * p.max_segs + cseg;
      dst = p.ws_o + slot * HD + lane * DPL;
      if (lane == 0) p.ws_ml[slot] = make_float2(m, l);
    }
    if constexpr (DPL == 4) *reinterpret_cast<float4*>(dst) = make_float4(res[0], res[1], res[2], res[3]);
    else *reinterpret_cast<float2*>(dst) = make_float2(res[0], res[1]);
    ++cq;
    copen = false;
  };

  // Compute one stage at the compute cursor (the fused append is done here).
  auto consume = [&](Stage& S) {
    const int tok0 = cstart + cst * ST;
    if (crow_new >= tok0 && crow_new < tok0 + ST) {   // warp-uniform: stage holds the new token
      const int d = crow_new - tok0;
      const int i_new = d / G, g_new = d % G;
      const __half* nb = nbuf + (cq & (kQueue - 1)) * 2 * HD;
      const NewTok nt = quantize_new_token(nb, sub, HD, blk_lanes, tab);
      const uint2 nk = nt.k, nv = nt.v;
      const float nks = nt.ks, nvs = nt.vs;
      if (g == g_new) {
        const long long row = static_cast<long long>(cbh) * p.Tc + crow_new;
        *reinterpret_cast<uint2*>(const_cast<uint8_t*>(p.kc) + row * (HD / 2) + sub * (kLaneDims / 2)) = nk;
        *reinterpret_cast<uint2*>(const_cast<uint8_t*>(p.vc) + row * (HD / 2) + sub * (kLaneDims / 2)) = nv;
        if (((sub * kLaneDims) & ((1 << p.blk_shift) - 1)) == 0) {
          const_cast<float*>(p.ks)[row * nblk + sidx] = nks;
          const_cast<float*>(p.vs)[row * nblk + sidx] = nvs;
        }
#pragma unroll
        for (int i = 0; i < kTPS; ++i) {
          if (i == i_new) { S.k[i] = nk; S.v[i] = nv; S.ks[i] = nks; S.vs[i] = nvs; }
        }
      }
    }
#ifdef NQKV_DBG_NOCOMPUTE
    {
      uint32_t x = 0;
#pragma unroll
      for (int i = 0; i < kTPS; ++i) x ^= S.k[i].x ^ S.k[i].y ^ S.v[i].x ^ S.v[i].y ^ __float_as_uint(S.ks[i] + S.vs[i]);
      o2[0] += x;
      l = 1.0f;
    }
#else
    compute_stage<HD>(S, tok0, cend, g, q2, o2, m, l, lane_sel, p.scale_log2);
#endif
    if (++cst == cnst) close_item();
  };

  // ---- prime the pipeline: kRing-1 stages in flight
  L.next = fetch();
  L.active = enter_next();
  Stage S[kRing];
  int pending = 0;
#pragma unroll
  for (int r = 0; r < kRing - 1; ++r) {
    if (L.active) { issue(S[r]); advance(); ++pending; }
  }
  // steady state: issue the stage kRing-1 ahead, then consume the current one
  for (;;) {
#pragma unroll
    for (int r = 0; r < kRing; ++r) {
      if (pending == 0) goto drained;
      if (L.active) { issue(S[(r + kRing - 1) % kRing]); advance(); ++pending; }
      if (!copen) open_item();
      consume(S[r]);
      --pending;
    }
  }
drained:
  return;
}

// ------------------------------------------------------- a7: split combine
// out = sum_i e^(m_i - M) o_i / sum_i e^(m_i - M) l_i over the segments of
// one (b, h), in segment order.  One warp per (b, h) with nseg > 1.
struct CombineParams {
  const int32_t* seq_lens;
  const float* ws_o;
  const float2* ws_ml;
  float* out;
  int B, H, Tc, max_segs;
};

template <int HD>
__global__ void __launch_bounds__(256) combine_kernel(const CombineParams p) {
  constexpr int DPL = HD / 32;
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long bh = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (bh >= static_cast<long long>(p.B) * p.H) return;
  const int b = static_cast<int>(bh / p.H);
  const int len = min(max(p.seq_lens[b], 0), p.Tc);
  const int nseg = (len + kSeg - 1) / kSeg;
  if (nseg <= 1) return;
  const long long base = bh * p.max_segs;
  float M = -INFINITY;
  for (int i = lane; i < nseg; i += 32) M = fmaxf(M, p.ws_ml[base + i].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float den = 0.0f;
  float acc[DPL];
#pragma unroll
  for (int d = 0; d < DPL; ++d) acc[d] = 0.0f;
  for (int i0 = 0; i0 < nseg; i0 += 32) {
    float f = 0.0f;
    if (i0 + lane < nseg) {
      const float2 ml = p.ws_ml[base + i0 + lane];
      f = fast_exp2(ml.x - M);
      den += f * ml.y;
    }
    const int cnt = min(32, nseg - i0);
#pragma unroll 8
    for (int i = 0; i < cnt; ++i) {
      const float fi = __shfl_sync(0xffffffffu, f, i);
      const float* src = p.ws_o + (base + i0 + i) * HD + lane * DPL;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[d] += fi * src[d];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  const float inv = 1.0f / den;
  float* out = p.out + bh * HD + lane * DPL;
#pragma unroll
  for (int d = 0; d < DPL; ++d) out[d] = acc[d] * inv;
}

}  // namespace nqkv
