// a4-a7: fused dequant-in-registers decode attention (+ optional fused
// 1-token append) and the split-K combine kernel.
//
// X' = dequantize_NF4(I); A = Softmax(t_Q X_K'^T); t_O = A X_V'
// (the 1/sqrt(hd) factor is DESIGN.md reading R6).  The dequantised cache is
// never written anywhere: packed codes stream from HBM into shared memory and
// are turned into fp32 levels by shared-memory table lookups in registers.
//
// Work decomposition.  A work item is (b, h, 128-token segment); the
// segmentation depends on seq_len only and partials are merged in segment
// order, so results are independent of B, H, the grid and the GPU.  Items are
// assigned statically (strided) to the warps of a persistent grid; each WARP
// streams its items as one continuous sequence of stages (ST tokens of one
// (b, h)):
//   - lane 0 of the warp is the producer: it issues TMA bulk copies
//     (cp.async.bulk, completion on an mbarrier) of a stage's K codes, V codes,
//     K scales and V scales into a kStages-deep per-warp shared-memory ring,
//     kStages-1 stages ahead of the consumer and across item boundaries;
//   - all 32 lanes consume: each lane owns 16 consecutive head dims (8 packed
//     bytes): LPT = hd/16 lanes cover a token row, G = 32/LPT token groups,
//     kTPS = 4 tokens per lane per stage (ST = G*kTPS);
//   - per-item q is prefetched with cp.async into a per-warp queue slot when the
//     producer enters the item; item descriptors travel through the same queue.
//
// Dequantisation.  A packed byte (two 4-bit codes) becomes the pair
// (L[lo], L[hi]) through ONE shared-memory load from a 256-entry fp32-pair
// table replicated per lane (64 KB, conflict-free: lane l reads bank pair 2l)
// whose address is built by one PRMT (the table sits on a 64 KB boundary of
// the shared window); the pair feeds one FFMA2.  Scores use fp32 levels with
// the block scale applied once per 16 dims; values accumulate w*L with
// w = p * scale.  The online softmax runs per token group (no cross-lane max
// per stage); groups merge once per item.
#pragma once
#include "common.cuh"

namespace nqkv {

constexpr int kSeg = 128;
constexpr int kLutBytes = 256 * 32 * 8;
constexpr int kMaxBatch = 1024;
#ifndef NQKV_DECODE_WARPS
#define NQKV_DECODE_WARPS 16
#endif
#ifndef NQKV_STAGES
#define NQKV_STAGES 3
#endif
constexpr int kDecodeWarps = NQKV_DECODE_WARPS;
constexpr int kStages = NQKV_STAGES;  // smem ring depth: TMA runs kStages-1 stages ahead
constexpr int kQueue = 4;
constexpr int kLaneDims = 16;         // head dims owned by one lane
constexpr int kTPS = 4;               // tokens per lane per stage

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
  int* grid_bar;            // [2] arrive / depart counters (zero between launches)
  int B, H, Tc, blk_shift, max_segs;
  float scale_log2;         // softmax_scale * log2(e)
  Levels lv;
  BucketTab tab;
  unsigned long long* trace;   // debug builds (NQKV_TRACE): per-warp timestamps
};

#ifdef NQKV_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(k) do { if (p.trace && lane == 0) p.trace[(blockIdx.x * NW + warp) * 8 + (k)] = gtimer(); } while (0)
#else
#define TRACE(k) do { } while (0)
#endif

template <int HD>
struct DecodeShape {
  static constexpr int LPT = HD / kLaneDims;
  static constexpr int G = 32 / LPT;
  static constexpr int ST = G * kTPS;                     // tokens per stage (32 or 16)
  static constexpr int kCodeBytes = ST * HD / 2;          // 1 KB per tensor per stage
  static constexpr int kScaleBytes = ST * (HD / 32) * 4;  // room for blk = 32 (256 B)
  static constexpr int kSlotBytes = 2 * kCodeBytes + 2 * kScaleBytes;
  // per-warp block: ring | q queue (kQueue x hd fp16) | descriptors | mbarriers
  static constexpr int kRingOff = 0;
  static constexpr int kQOff = kStages * kSlotBytes;
  static constexpr int kDescOff = kQOff + kQueue * HD * 2;
  static constexpr int kMbarOff = kDescOff + kQueue * 8 * 4;
  static constexpr int kWarpBytes = (kMbarOff + kStages * 8 + 15) / 16 * 16;
};

// Shared-memory layout.  The pair LUT must start on a 64 KB boundary of the
// shared window so that ONE PRMT can produce a complete LDS address
// (byte 0 = lane*8, byte 1 = code byte, bytes 2-3 = LUT base >> 16): the
// dynamic window starts at 0x400 (1 KB driver reserve), so the LUT goes at
// dynamic offset kLutOff = 0xFC00 (checked on device; a mismatch traps).  Warp
// blocks fill the space before the LUT first, the rest follow it.
constexpr int kLutOff = 0xFC00;
template <int HD, int NW>
struct SmemLayout {
  static constexpr int kWB = DecodeShape<HD>::kWarpBytes;
  static constexpr int kSmall = 512;                                 // bucket tab + levels
  static constexpr int kPre = (kLutOff - kSmall) / kWB;              // warp blocks before the LUT
  static constexpr int kBefore = kPre < NW ? kPre : NW;
  static constexpr int kAfterOff = kLutOff + kLutBytes;
  static constexpr int kTailOff = kAfterOff + (NW - kBefore) * kWB;   // prefix [B+1] + lens [B]
  __host__ __device__ static constexpr int warp_off(int w) {
    return w < kBefore ? kSmall + w * kWB : kAfterOff + (w - kBefore) * kWB;
  }
  __host__ __device__ static constexpr size_t bytes(int B) {
    return static_cast<size_t>(kTailOff) + static_cast<size_t>(2 * B + 1) * sizeof(int);
  }
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
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" :: "r"(mbar), "r"(phase) : "memory");
}
// 1-D TMA bulk copy global -> shared, completion signalled on mbar.
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

// Quantize this lane's 16 dims of the appended token (fp16) exactly as
// nqkv_quantize would: block absmax across the blk/16 adjacent lanes of the
// block, then the code of every element.  Out of line: runs once per (b, h).
struct NewTok {
  uint2 k, v;
  float ks, vs;
};

__device__ __forceinline__ uint2 quantize_lane16(const __half* src, int blk_lanes, uint32_t tab,
                                                 float& scale) {
  const uint4 r0 = __ldg(reinterpret_cast<const uint4*>(src));
  const uint4 r1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
  float s = fmaxf(absmax8(r0), absmax8(r1));
  for (int o = 1; o < blk_lanes; o <<= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
  const float r = block_rcp(s);
  scale = s;
  return make_uint2(encode8c(r0, r, tab - 0x5A000000u), encode8c(r1, r, tab - 0x5A000000u));
}

__device__ __noinline__ NewTok quantize_new_token(const __half* kp, const __half* vp, int blk_lanes,
                                                  uint32_t tab) {
  NewTok t;
  t.k = quantize_lane16(kp, blk_lanes, tab, t.ks);
  t.v = quantize_lane16(vp, blk_lanes, tab, t.vs);
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
__device__ __forceinline__ uint2 lds_u2(const uint8_t* p) { return *reinterpret_cast<const uint2*>(p); }

// One stage from a shared-memory slot: kTPS tokens per lane.  The online
// softmax runs per token GROUP (the G groups see disjoint tokens; the LPT lanes
// of a group hold identical scores), so no cross-lane max is needed here.
template <int HD>
__device__ __forceinline__ void compute_stage(const uint8_t* slot, int tok0, int end, int g, int sub,
                                              int nblk, int sidx, const uint64_t (&q2)[8],
                                              uint64_t (&o2)[8], float& m, float& l,
                                              uint32_t lane_sel, float scale_log2) {
  using Sh = DecodeShape<HD>;
  constexpr int LPT = Sh::LPT, G = Sh::G;
  const uint8_t* kb = slot;
  const uint8_t* vb = slot + Sh::kCodeBytes;
  const float* ksb = reinterpret_cast<const float*>(slot + 2 * Sh::kCodeBytes);
  const float* vsb = reinterpret_cast<const float*>(slot + 2 * Sh::kCodeBytes + Sh::kScaleBytes);
  float sc[kTPS];
#pragma unroll
  for (int i = 0; i < kTPS; ++i) {
    const int r = i * G + g;
    const uint2 kw = lds_u2(kb + r * (HD / 2) + sub * (kLaneDims / 2));
    uint64_t a0 = 0, a1 = 0;   // two independent fp32x2 chains over 8 packed bytes
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a0 = ffma2(q2[k], lut_pair(kw.x, k, lane_sel), a0);
      a1 = ffma2(q2[4 + k], lut_pair(kw.y, k, lane_sel), a1);
    }
    const float2 a = unpack2(fadd2(a0, a1));
    sc[i] = (a.x + a.y) * ksb[r * nblk + sidx];
  }
#pragma unroll
  for (int o = 1; o < LPT; o <<= 1) {
#pragma unroll
    for (int i = 0; i < kTPS; ++i) sc[i] += __shfl_xor_sync(0xffffffffu, sc[i], o);
  }
  float mt = m;
#pragma unroll
  for (int i = 0; i < kTPS; ++i) {
    sc[i] = (tok0 + i * G + g < end) ? sc[i] * scale_log2 : -INFINITY;
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
    const int r = i * G + g;
    const uint2 vw = lds_u2(vb + r * (HD / 2) + sub * (kLaneDims / 2));
    const float pr = fast_exp2(sc[i] - ms);
    l += pr;
    const float w = pr * vsb[r * nblk + sidx];
    const uint64_t w2 = pack2(w, w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o2[k] = ffma2(lut_pair(vw.x, k, lane_sel), w2, o2[k]);
      o2[4 + k] = ffma2(lut_pair(vw.y, k, lane_sel), w2, o2[4 + k]);
    }
  }
}

// Producer-side cursor (warp-uniform): walks items/stages kStages-1 ahead.
struct LoadCursor {
  int active;            // 1 while items remain
  int q;                 // items entered so far (queue position of the next one)
  int st, nst, start, end;
  long long row0;
};

template <int HD, int NW>
__global__ void __launch_bounds__(NW * 32, 1) decode_kernel(const DecodeParams p) {
  using Sh = DecodeShape<HD>;
  using Lay = SmemLayout<HD, NW>;
  constexpr int LPT = Sh::LPT, G = Sh::G, ST = Sh::ST;
  extern __shared__ __align__(16) unsigned char smem[];
  float2* s_tab = reinterpret_cast<float2*>(smem);
  float* s_lv = reinterpret_cast<float*>(smem + 384);
  int* s_pref = reinterpret_cast<int*>(smem + Lay::kTailOff);           // [B+1]
  int* s_len = s_pref + p.B + 1;                                        // [B]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TRACE(0);
  unsigned char* wb = smem + Lay::warp_off(warp);
  __half* qbuf = reinterpret_cast<__half*>(wb + Sh::kQOff);
  int* desc = reinterpret_cast<int*>(wb + Sh::kDescOff);
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(wb + Sh::kRingOff));
  const uint32_t mbar0 = static_cast<uint32_t>(__cvta_generic_to_shared(wb + Sh::kMbarOff));

  // ---- prologue independent of the previous kernel: tables, pair LUT, barriers
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) s_lv[k] = p.lv.v[k];
  }
  for (int i = threadIdx.x; i < kNumBuckets; i += blockDim.x) s_tab[i] = p.tab.e[i];
  if (lane < kStages) mbar_init(mbar0 + lane * 8, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  {
    float4* lut4 = reinterpret_cast<float4*>(smem + kLutOff);
    for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
      const int e = i >> 4;
      const float lo = s_lv[e & 15], hi = s_lv[e >> 4];
      lut4[i] = make_float4(lo, hi, lo, hi);
    }
  }
  TRACE(1);
  pdl_trigger();
  pdl_wait();
  TRACE(2);
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
  TRACE(3);
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(smem + kLutOff));
  if (lut & 0xFFFFu) __trap();        // the single-PRMT address needs a 64 KB-aligned LUT
  const uint32_t lane_sel = (lut & 0xFFFF0000u) | (lane * 8u);
  const uint32_t tab = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
  const int g = lane / LPT, sub = lane % LPT;
  const int nblk = HD >> p.blk_shift;
  const int sidx = (sub * kLaneDims) >> p.blk_shift;
  const bool fused = p.k_new != nullptr;
  const int blk_lanes = (1 << p.blk_shift) / kLaneDims;

  // Static strided schedule: warp w takes items w, w + W, w + 2W, ...
  const int gwarp = static_cast<int>(blockIdx.x) * NW + warp;
  const int nwarps = static_cast<int>(gridDim.x) * NW;
  int next_item = gwarp;

  // ---- producer: enter the next scheduled item that has tokens (decode it,
  // publish its descriptor, prefetch q).  Empty sequences are finished here
  // (out = 0, reading R12).  Returns false when exhausted.
  LoadCursor L;
  L.q = 0;
  auto enter_next = [&]() -> bool {
    for (;;) {
      const int item = next_item;
      if (item >= total) return false;
      next_item += nwarps;
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
        d[0] = bh; d[1] = start; d[2] = end; d[3] = nseg; d[4] = seg; d[5] = row_new; d[6] = b; d[7] = h;
      }
      constexpr int CH = HD * 2 / 16;       // 16-byte chunks per fp16 row (8 or 16)
      const uint32_t qs = static_cast<uint32_t>(__cvta_generic_to_shared(qbuf + slot * HD));
      if (lane < CH) cp_async16(qs + lane * 16, p.q + static_cast<long long>(bh) * HD + lane * 8);
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
  // TMA one stage (ST rows of one (b, h), clipped at Tc) into ring slot `pos % kStages`.
  auto issue = [&](int pos) {
    if (lane == 0) {
      const int s = pos % kStages;
      const uint32_t dst = ring + s * Sh::kSlotBytes;
      const uint32_t mb = mbar0 + s * 8;
      const int tok0 = L.start + L.st * ST;
      const int rows = min(ST, p.Tc - tok0);
      const long long row = L.row0 + tok0;
      const uint32_t cb = rows * (HD / 2), sb = rows * nblk * 4;
      mbar_expect_tx(mb, 2 * cb + 2 * sb);
      tma_load_1d(dst, p.kc + row * (HD / 2), cb, mb);
      tma_load_1d(dst + Sh::kCodeBytes, p.vc + row * (HD / 2), cb, mb);
      tma_load_1d(dst + 2 * Sh::kCodeBytes, p.ks + row * nblk, sb, mb);
      tma_load_1d(dst + 2 * Sh::kCodeBytes + Sh::kScaleBytes, p.vs + row * nblk, sb, mb);
    }
  };

  // ---- consumer state
  int cq = 0, cst = 0, cnst = 0, cstart = 0, cend = 0, cbh = 0, cnseg = 1, cseg = 0, crow_new = -1;
  int cb_ = 0, ch_ = 0;
  bool copen = false;
  uint64_t q2[8], o2[8];
  float m = -INFINITY, l = 0.0f;

  auto open_item = [&]() {
    __syncwarp();
    const int slot = cq & (kQueue - 1);
    const int* d = desc + slot * 8;
    cbh = d[0]; cstart = d[1]; cend = d[2]; cnseg = d[3]; cseg = d[4]; crow_new = d[5];
    cb_ = d[6]; ch_ = d[7];
    cnst = (cend - cstart + ST - 1) / ST;
    cst = 0;
    cp_async_wait(L.q - cq - 1);      // this item's q prefetch has landed
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
    // merge the G per-group softmax states: common max M, rescale, sum
    float M = m;
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float f = fast_exp2(m - M);          // 0 for a group that saw no token
    l *= f;
    const uint64_t f2 = pack2(f, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], f2);
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2 a = unpack2(o2[j]);
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
        o2[j] = pack2(a.x, a.y);
      }
    }
    // every group now holds the full sums for its sub's 16 dims; group g
    // writes dims [sub*16 + g*(16/G), +16/G)
    constexpr int PER = kLaneDims / G;          // 2 (hd 64) or 4 (hd 128)
    float res[PER];
#pragma unroll
    for (int d = 0; d < PER; ++d) {
      const int idx = g * PER + d;              // 0..15 within the lane's 16 dims
      float v = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 a = unpack2(o2[j]);
        if (idx == 2 * j) v = a.x;
        if (idx == 2 * j + 1) v = a.y;
      }
      res[d] = v;
    }
    float* dst;
    if (cnseg == 1) {
      const float inv = 1.0f / l;
#pragma unroll
      for (int d = 0; d < PER; ++d) res[d] *= inv;
      dst = p.out + static_cast<long long>(cbh) * HD + sub * kLaneDims + g * PER;
    } else {
      const long long slot = static_cast<long long>(cbh) * p.max_segs + cseg;
      dst = p.ws_o + slot * HD + sub * kLaneDims + g * PER;
      if (lane == 0) p.ws_ml[slot] = make_float2(M, l);
    }
    if constexpr (PER == 4) *reinterpret_cast<float4*>(dst) = make_float4(res[0], res[1], res[2], res[3]);
    else *reinterpret_cast<float2*>(dst) = make_float2(res[0], res[1]);
    ++cq;
    copen = false;
  };

  // Consume stage position `pos` (slot pos % kStages, parity (pos / kStages) & 1).
  auto consume = [&](int pos) {
    const int s = pos % kStages;
    mbar_wait(mbar0 + s * 8, (pos / kStages) & 1);
    uint8_t* slot = wb + Sh::kRingOff + s * Sh::kSlotBytes;
    const int tok0 = cstart + cst * ST;
    if (crow_new >= tok0 && crow_new < tok0 + ST) {   // warp-uniform: the stage holds the new token
      const int r_new = crow_new - tok0;               // row inside the slot
      const long long off = static_cast<long long>(cb_) * p.new_sb + static_cast<long long>(ch_) * p.new_sh +
                            sub * kLaneDims;
      const NewTok nt = quantize_new_token(p.k_new + off, p.v_new + off, blk_lanes, tab);
      if (g == r_new % G) {
        const long long row = static_cast<long long>(cbh) * p.Tc + crow_new;
        const int cofs = sub * (kLaneDims / 2);
        *reinterpret_cast<uint2*>(const_cast<uint8_t*>(p.kc) + row * (HD / 2) + cofs) = nt.k;
        *reinterpret_cast<uint2*>(const_cast<uint8_t*>(p.vc) + row * (HD / 2) + cofs) = nt.v;
        *reinterpret_cast<uint2*>(slot + r_new * (HD / 2) + cofs) = nt.k;
        *reinterpret_cast<uint2*>(slot + Sh::kCodeBytes + r_new * (HD / 2) + cofs) = nt.v;
        if (((sub * kLaneDims) & ((1 << p.blk_shift) - 1)) == 0) {
          const_cast<float*>(p.ks)[row * nblk + sidx] = nt.ks;
          const_cast<float*>(p.vs)[row * nblk + sidx] = nt.vs;
          reinterpret_cast<float*>(slot + 2 * Sh::kCodeBytes)[r_new * nblk + sidx] = nt.ks;
          reinterpret_cast<float*>(slot + 2 * Sh::kCodeBytes + Sh::kScaleBytes)[r_new * nblk + sidx] = nt.vs;
        }
      }
      __syncwarp();
    }
    compute_stage<HD>(slot, tok0, cend, g, sub, nblk, sidx, q2, o2, m, l, lane_sel, p.scale_log2);
    __syncwarp();                                      // slot reads done before it is refilled
    if (++cst == cnst) close_item();
  };

  // ---- prime the pipeline: kStages-1 stages in flight
  L.active = enter_next();
  int issued = 0, consumed = 0;
  for (int r = 0; r < kStages - 1 && L.active; ++r) {
    issue(issued++);
    advance();
  }
  TRACE(4);
  // steady state: refill the slot consumed last, then consume the next stage
  while (consumed < issued) {
    if (L.active) {
      issue(issued++);
      advance();
    }
    if (!copen) open_item();
    consume(consumed++);
    if (consumed == 1) TRACE(5);
  }
  TRACE(6);

  // ---- a7: merge the split partials in-kernel after one grid-wide barrier
  // (cooperative launch: every CTA is resident).  One release/acquire pair per
  // CTA instead of one per work item.
  if (p.max_segs > 1) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      atomicAdd(p.grid_bar, 1);
      int seen = 0;
      do {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(p.grid_bar) : "memory");
      } while (seen < static_cast<int>(gridDim.x));
    }
    __syncthreads();
    TRACE(7);
    constexpr int DPL = HD / 32;        // output dims per lane
    for (int r = gwarp; r < p.B * p.H; r += nwarps) {
      const int len = s_len[r / p.H];
      const int nseg = max(1, (len + kSeg - 1) / kSeg);
      if (nseg <= 1) continue;
      const long long base = static_cast<long long>(r) * p.max_segs;
      float Mx = -INFINITY;
      for (int i = lane; i < nseg; i += 32) Mx = fmaxf(Mx, __ldcg(&p.ws_ml[base + i].x));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
      float den = 0.0f, acc[DPL];
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[d] = 0.0f;
      for (int i0 = 0; i0 < nseg; i0 += 32) {
        float f = 0.0f;
        if (i0 + lane < nseg) {
          const float2 ml = __ldcg(&p.ws_ml[base + i0 + lane]);
          f = fast_exp2(ml.x - Mx);
          den += f * ml.y;
        }
        const int cnt = min(32, nseg - i0);
#pragma unroll 8
        for (int i = 0; i < cnt; ++i) {
          const float fi = __shfl_sync(0xffffffffu, f, i);
          const float* src = p.ws_o + (base + i0 + i) * HD + lane * DPL;
          if constexpr (DPL == 4) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(src));
            acc[0] += fi * v.x; acc[1] += fi * v.y; acc[2] += fi * v.z; acc[3] += fi * v.w;
          } else {
            const float2 v = __ldcg(reinterpret_cast<const float2*>(src));
            acc[0] += fi * v.x; acc[1] += fi * v.y;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
      const float inv = 1.0f / den;
      float* outp = p.out + static_cast<long long>(r) * HD + lane * DPL;
      if constexpr (DPL == 4)
        *reinterpret_cast<float4*>(outp) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      else
        *reinterpret_cast<float2*>(outp) = make_float2(acc[0] * inv, acc[1] * inv);
    }
    // leave the barrier counters zero for the next launch: the last CTA out resets
    if (threadIdx.x == 0) {
      const int d = atomicAdd(p.grid_bar + 1, 1);
      if (d == static_cast<int>(gridDim.x) - 1) {
        p.grid_bar[0] = 0;
        p.grid_bar[1] = 0;
      }
    }
  }
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

// One thread per (b, h, dim): independent loads over the segments, the
// segment (max, sum) pairs are broadcast loads shared by the warp.
template <int HD>
__global__ void __launch_bounds__(256) combine_kernel(const CombineParams p) {
  pdl_trigger();
  pdl_wait();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long bh = t / HD;
  const int d = static_cast<int>(t % HD);
  if (bh >= static_cast<long long>(p.B) * p.H) return;
  const int b = static_cast<int>(bh / p.H);
  const int len = min(max(p.seq_lens[b], 0), p.Tc);
  const int nseg = (len + kSeg - 1) / kSeg;
  if (nseg <= 1) return;
  const long long base = bh * p.max_segs;
  float M = -INFINITY;
#pragma unroll 8
  for (int i = 0; i < nseg; ++i) M = fmaxf(M, p.ws_ml[base + i].x);
  float den = 0.0f, acc = 0.0f;
#pragma unroll 8
  for (int i = 0; i < nseg; ++i) {
    const float2 ml = p.ws_ml[base + i];
    const float f = fast_exp2(ml.x - M);
    den += f * ml.y;
    acc += f * p.ws_o[(base + i) * HD + d];
  }
  p.out[bh * HD + d] = acc / den;
}

}  // namespace nqkv
