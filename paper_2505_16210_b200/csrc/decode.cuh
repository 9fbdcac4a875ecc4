// a4-a7: fused dequant-in-registers decode attention (+ optional fused
// 1-token append).
//
// X' = dequantize_NF4(I); A = Softmax(t_Q X_K'^T); t_O = A X_V'
// (the 1/sqrt(hd) factor is DESIGN.md reading R6).  The dequantised cache is
// never materialised: packed codes go from HBM straight into registers and
// are turned into products by shared-memory table lookups.
//
// Dequantisation by lookup:
//  * K side -- a per-(b, h) q-table.  For head-dim pair j and code byte e
//    (two 4-bit codes), T[e][j] = c * (q[2j] L[e & 15] + q[2j+1] L[e >> 4]),
//    c = softmax_scale * log2(e), built in fp32 once per (b, h) piece.  A
//    token's score is then sum_blocks s_blk * sum_{j in blk} T[byte_j][j]:
//    ONE 4-byte shared load + one add per packed byte.  Row e of the table is
//    256 B; a lane's 8 pairs are visited in a lane-rotated order so that the 32
//    lanes of a warp always hit 32 distinct banks.
//  * V side -- a constant fp32 pair table P[e] = (L[e & 15], L[e >> 4]),
//    replicated per lane (lane l's copy in banks 2l, 2l+1): one 8-byte shared
//    load + one fp32x2 FMA (weight p * s_blk) per packed byte.
//  Both tables are addressed by ONE PRMT per byte (the code byte becomes
//  address byte 1, i.e. row * 256; the lane/pair offset sits in byte 0) plus the
//  load's immediate offset -- the dynamic shared window starts at 0x400
//  (checked on device).
//
// Work decomposition.  The (b, h, t) token list of the launch (N tokens) is
// cut into C equal contiguous ranges, one per CTA (C = min(grid, N /
// min_tokens)); a range splits into "pieces" at (b, h) boundaries.
// Warp specialisation inside the CTA:
//  * NC consumer warps stream: stage s (ST tokens) of a piece goes to consumer
//    s % NC.  Lane (g, sub) owns 16 head dims (8 packed bytes) of token g of
//    each of the kTPS slots of a stage; loads run one stage ahead, across piece
//    boundaries.  The online softmax keeps a warp-uniform running max.  At a
//    piece end a consumer sums its token groups and publishes (m, l, o[hd]).
//  * one producer warp builds the q-table of piece k into ring slot k % R
//    (R = 4 for hd 64, 2 for hd 128) once every consumer has left piece k - R,
//    and merges the consumers' states of each finished piece into the output.
// Consumers therefore never wait on each other -- only on the producer's
// "full" barrier of the next table, which is normally long complete.
// A piece that does not cover a whole sequence (only a CTA's first and last
// pieces can be partial) is written as an unnormalised partial (m, l, o);
// the last of the sequence's CTAs to arrive (per-(b, h) counter) merges the
// partials in CTA order.  Results depend on (B, H, seq_lens, grid) only: the
// same call is bit-reproducible; a different head shard of the same data can
// differ by fp32 reassociation (reading R7).
#pragma once
#include "common.cuh"

namespace nqkv {

constexpr int kMaxBatch = 1024;
constexpr int kMaxGrid = 1024;         // partial slots in the workspace (>= CTAs per launch)
constexpr int kMinTokensPerCta = 512;  // below this a CTA's table build would dominate
#ifndef NQKV_DECODE_WARPS
#define NQKV_DECODE_WARPS 16     // 15 consumers + 1 producer
#endif
#ifndef NQKV_TPS
#define NQKV_TPS 4
#endif
#ifndef NQKV_PF
#define NQKV_PF 0                // L2 prefetch distance in a warp's own stages (0: off; measured no gain)
#endif
constexpr int kDecodeWarps = NQKV_DECODE_WARPS;
constexpr int kLaneDims = 16;          // head dims owned by one lane
constexpr int kTPS = NQKV_TPS;         // token slots per lane per stage
constexpr uint32_t kSmemWindow = 0x400;  // shared address of dynamic smem offset 0

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
  int* cnt;                 // [B*H] partial-arrival counters (zero between launches)
  float* part;              // [kMaxGrid][2][hd + 2] partial (o[hd], m, l)
  int B, H, Tc, blk_shift, min_tokens;
  float scale_log2;         // softmax_scale * log2(e)
  Levels lv;
  BucketTab tab;
  unsigned long long* trace;   // NQKV_TRACE builds: per-warp globaltimer stamps [grid][NW][8]
};

#ifdef NQKV_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(k) do { if (p.trace && lane == 0) p.trace[(blockIdx.x * NW + warp) * 8 + (k)] = gtimer(); } while (0)
#else
#define TRACE(k) do { } while (0)
#endif

template <int HD>
struct Geo {
  static constexpr int LPT = HD / kLaneDims;  // lanes per token row (4 / 8)
  static constexpr int G = 32 / LPT;          // token groups per warp (8 / 4)
  static constexpr int ST = G * kTPS;         // tokens per warp stage
  static constexpr int R = HD == 64 ? 4 : 2;  // q-table ring depth
  static constexpr int PPL = HD / 64;         // table pairs per producer lane (1 / 2)
};

// Dynamic shared memory (offsets from the window start, shared address 0x400):
//   [0, 64K)             V pair LUT: row e (256 B) = 32 lane copies of (L[lo], L[hi])
//   [64K, 192K)          K q-table ring: row e of a table is 128 B (hd 64; two
//                        tables share a 64 KB block of 256-B rows) or 256 B (hd 128)
//   misc                 levels, bucket table, mbarriers, consumer states, lens/prefix
template <int HD, int NW>
struct Smem {
  static constexpr int NC = NW - 1;
  static constexpr int R = Geo<HD>::R;
  static constexpr uint32_t kV = 0;
  static constexpr uint32_t kK = 0x10000;
  static constexpr uint32_t kLv = kK + 0x20000;           // float[16]
  static constexpr uint32_t kTab = kLv + 64;              // float2[kNumBuckets]
  static constexpr uint32_t kMbar = kTab + 272;           // u64 full[R], done[R]
  static constexpr uint32_t kMl = kMbar + 16 * R;         // float2 [R][NC]
  static constexpr uint32_t kPc = (kMl + R * NC * 8 + 15) / 16 * 16;   // Piece [R] (producer)
  static constexpr uint32_t kO = kPc + R * 32;            // float [R][NC][HD]
  static constexpr uint32_t kPref = kO + R * NC * HD * 4; // int [kMaxBatch + 1]
  static constexpr uint32_t kLen = kPref + (kMaxBatch + 1) * 4 + 12;  // int [kMaxBatch]
  static constexpr uint32_t kBytes = kLen + kMaxBatch * 4;
  static_assert(kBytes <= 227 * 1024, "decode smem over budget");
  static_assert((kTab % 16) == 0 && (kMbar % 8) == 0 && (kO % 16) == 0, "alignment");
};

// ------------------------------------------------------------ primitives
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
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
// K table entry (row/pair offset from one PRMT) -- immediate = table base
__device__ __forceinline__ float lds_k(uint32_t off) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+0x10400];" : "=f"(v) : "r"(off));
  return v;
}
// V pair LUT entry
__device__ __forceinline__ uint64_t lds_v(uint32_t off) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1+0x400];" : "=l"(v) : "r"(off));
  return v;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int o) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v), o);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), o);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}
// TMA bulk prefetch of [p, p + bytes) into L2 (no registers, no completion)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t a0 = a & ~static_cast<uintptr_t>(15);
  const uint32_t n = static_cast<uint32_t>((a + bytes - a0 + 15) & ~static_cast<uintptr_t>(15));
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a0), "r"(n) : "memory");
}
__device__ __forceinline__ float ldg_nc_f32(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
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

// One CTA-contiguous run of tokens of one (b, h): tokens [t0, t1) of a
// sequence of length len.  Walked identically by every warp.
struct __align__(16) Piece {
  long long gs;   // global (b, h, t) index of t0
  int b, h, len, t0, t1, pad;
};

// Registers of one stage: kTPS token slots of this lane.
struct StageRegs {
  uint2 k[kTPS], v[kTPS];
  float ks[kTPS], vs[kTPS];
};

template <int HD, int NW>
__global__ void __launch_bounds__(NW * 32, 1) decode_kernel(const DecodeParams p) {
  using Ge = Geo<HD>;
  using Sm = Smem<HD, NW>;
  constexpr int LPT = Ge::LPT, G = Ge::G, ST = Ge::ST, R = Ge::R;
  constexpr int NT = NW * 32, NC = NW - 1;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TRACE(0);
  if (static_cast<uint32_t>(__cvta_generic_to_shared(smem)) != kSmemWindow) __trap();
  float* s_lv = reinterpret_cast<float*>(smem + Sm::kLv);
  float2* s_tab = reinterpret_cast<float2*>(smem + Sm::kTab);
  const uint32_t mb_full = kSmemWindow + Sm::kMbar;          // full[R]  (count 1: producer)
  const uint32_t mb_done = kSmemWindow + Sm::kMbar + 8 * R;  // done[R]  (count NC)
  float* s_o = reinterpret_cast<float*>(smem + Sm::kO);
  float2* s_ml = reinterpret_cast<float2*>(smem + Sm::kMl);
  Piece* s_pc = reinterpret_cast<Piece*>(smem + Sm::kPc);
  int* s_pref = reinterpret_cast<int*>(smem + Sm::kPref);
  int* s_len = reinterpret_cast<int*>(smem + Sm::kLen);

  // ---- prologue independent of the previous kernel: levels, V LUT, barriers
  if (tid < 16) s_lv[tid] = p.lv.v[tid];
  if (tid < kNumBuckets) s_tab[tid] = p.tab.e[tid];
  if (tid == 0) {
    for (int r = 0; r < R; ++r) {
      mbar_init(mb_full + 8 * r, 1);
      mbar_init(mb_done + 8 * r, NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  pdl_wait();
  TRACE(1);
  // seq_lens (warp 0) in flight while the V LUT is written
  int lens_r[kMaxBatch / 32];
  if (warp == 0) {
#pragma unroll
    for (int u = 0; u < kMaxBatch / 32; ++u) {
      const int b = u * 32 + lane;
      lens_r[u] = (u * 32 < p.B && b < p.B) ? p.seq_lens[b] : 0;
    }
  }
  __syncthreads();
  for (int i = tid; i < 256 * 16; i += NT) {     // 16 B = two lane copies per store
    const int e = i >> 4;
    const float lo = s_lv[e & 15], hi = s_lv[e >> 4];
    *reinterpret_cast<float4*>(smem + Sm::kV + e * 256 + (i & 15) * 16) = make_float4(lo, hi, lo, hi);
  }
  // ---- per-batch lengths and token prefix: tokens(b) = H * len_b
  if (warp == 0) {
    int carry = 0;
    if (lane == 0) s_pref[0] = 0;
#pragma unroll
    for (int u = 0; u < kMaxBatch / 32; ++u) {
      if (u * 32 >= p.B) break;
      const int b = u * 32 + lane;
      int n = 0;
      if (b < p.B) {
        const int len = min(max(lens_r[u], 0), p.Tc);
        s_len[b] = len;
        n = p.H * len;
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
  TRACE(2);
  const long long N = s_pref[p.B];
  // empty sequences: out = 0 (reading R12); strided over the grid
  for (long long i = static_cast<long long>(blockIdx.x) * NT + tid; i < static_cast<long long>(p.B) * p.H * HD;
       i += static_cast<long long>(gridDim.x) * NT) {
    if (s_len[i / (static_cast<long long>(p.H) * HD)] == 0) p.out[i] = 0.0f;
  }
  if (N == 0) return;
  const int C = static_cast<int>(min(static_cast<long long>(gridDim.x),
                                     max(1ll, (N + p.min_tokens - 1) / p.min_tokens)));
  if (static_cast<int>(blockIdx.x) >= C) return;
  const int cta = blockIdx.x;
  const long long g0 = static_cast<long long>(cta) * N / C;
  const long long g1 = static_cast<long long>(cta + 1) * N / C;

  // ---- piece walking (identical in every warp)
  auto locate = [&](long long g, Piece& pc) {
    int lo = 0, hi = p.B;                 // largest b with pref[b] <= g (pref[B] > g)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pref[mid] <= g) lo = mid; else hi = mid;
    }
    pc.b = lo;
    pc.len = s_len[lo];
    const long long off = g - s_pref[lo];
    pc.h = static_cast<int>(off / pc.len);
    pc.t0 = static_cast<int>(off - static_cast<long long>(pc.h) * pc.len);
    pc.gs = g;
    pc.t1 = static_cast<int>(min(static_cast<long long>(pc.len), pc.t0 + (g1 - g)));
  };
  auto next_piece = [&](Piece& pc) -> bool {
    const long long g = pc.gs + (pc.t1 - pc.t0);
    if (g >= g1) return false;
    if (pc.h + 1 < p.H) {
      ++pc.h;
    } else {
      do { ++pc.b; } while (s_len[pc.b] == 0);
      pc.h = 0;
      pc.len = s_len[pc.b];
    }
    pc.t0 = 0;
    pc.gs = g;
    pc.t1 = static_cast<int>(min(static_cast<long long>(pc.len), g1 - g));
    return true;
  };

  // L2 prefetch of rows [r0, r1) of (b, h) -- codes and scales of K and V
  const int nblk_ = HD >> p.blk_shift;
  auto prefetch_rows = [&](long long bh, int r0, int r1) {
    if (r1 <= r0) return;
    const long long row = bh * p.Tc + r0;
    const uint32_t n = static_cast<uint32_t>(r1 - r0);
    prefetch_l2(p.kc + row * (HD / 2), n * (HD / 2));
    prefetch_l2(p.vc + row * (HD / 2), n * (HD / 2));
    prefetch_l2(p.ks + row * nblk_, n * nblk_ * 4);
    prefetch_l2(p.vs + row * nblk_, n * nblk_ * 4);
  };

  // ---- table of piece 0, built by all threads (thread: pair quad tid % Q)
  {
    Piece p0;
    locate(g0, p0);
    constexpr int Q = HD / 8;
    const long long bh = static_cast<long long>(p0.b) * p.H + p0.h;
    const uint4 qraw = __ldg(reinterpret_cast<const uint4*>(p.q + bh * HD) + (tid % Q));
    __half2 h2[4];
    memcpy(h2, &qraw, 16);
    float qa[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(h2[k]);
      qa[2 * k] = f.x * p.scale_log2;
      qa[2 * k + 1] = f.y * p.scale_log2;
    }
    for (int e = tid / Q; e < 256; e += NT / Q) {
      const float lo = s_lv[e & 15], hi = s_lv[e >> 4];
      *reinterpret_cast<float4*>(smem + Sm::kK + e * 256 + (tid % Q) * 16) =
          make_float4(fmaf(qa[1], hi, qa[0] * lo), fmaf(qa[3], hi, qa[2] * lo),
                      fmaf(qa[5], hi, qa[4] * lo), fmaf(qa[7], hi, qa[6] * lo));
    }
  }
  __syncthreads();

  if (warp == NC) {
    // ================================================================ producer
    // q-table slot r: hd 64 -> block r >> 1, half r & 1; hd 128 -> block r
    auto build = [&](int slot, const float (&qa)[2 * Ge::PPL]) {
#pragma unroll
      for (int u = 0; u < Ge::PPL; ++u) {
        const int j = lane + 32 * u;
        const uint32_t base = Sm::kK + (HD == 64 ? (slot >> 1) * 0x10000 + (slot & 1) * 128
                                                 : slot * 0x10000) + j * 4;
        float A[16], Bv[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          A[c] = qa[2 * u] * s_lv[c];
          Bv[c] = qa[2 * u + 1] * s_lv[c];
        }
        float* t = reinterpret_cast<float*>(smem + base);
#pragma unroll
        for (int e = 0; e < 256; ++e) t[e * 64] = A[e & 15] + Bv[e >> 4];
      }
    };
    auto load_q = [&](const Piece& pc, float (&qa)[2 * Ge::PPL]) {
      const long long bh = static_cast<long long>(pc.b) * p.H + pc.h;
#pragma unroll
      for (int u = 0; u < Ge::PPL; ++u) {
        const __half2 h2 = __ldg(reinterpret_cast<const __half2*>(p.q + bh * HD) + lane + 32 * u);
        const float2 f = __half22float2(h2);
        qa[2 * u] = f.x * p.scale_log2;
        qa[2 * u + 1] = f.y * p.scale_log2;
      }
    };
    constexpr int DL = HD / 32;
    // merge piece k's NC consumer states (ring slot k % R): output or partial
    auto merge = [&](int k) {
      const int slot = k % R;
      const Piece pc = s_pc[slot];
      float M = -INFINITY;
      for (int w = 0; w < NC; ++w) M = fmaxf(M, s_ml[slot * NC + w].x);
      float den = 0.0f, acc[DL];
#pragma unroll
      for (int d = 0; d < DL; ++d) acc[d] = 0.0f;
      for (int w = 0; w < NC; ++w) {
        const float2 ml = s_ml[slot * NC + w];
        if (ml.x == -INFINITY) continue;                 // consumer saw no token
        const float f = fast_exp2(ml.x - M);
        den += f * ml.y;
        const float* o = s_o + (slot * NC + w) * HD + lane * DL;
#pragma unroll
        for (int d = 0; d < DL; ++d) acc[d] = fmaf(f, o[d], acc[d]);
      }
      const long long bh = static_cast<long long>(pc.b) * p.H + pc.h;
      if (pc.t0 == 0 && pc.t1 == pc.len) {
        const float inv = 1.0f / den;
#pragma unroll
        for (int d = 0; d < DL; ++d) p.out[bh * HD + lane * DL + d] = acc[d] * inv;
        return;
      }
      // partial piece: slot 0 = this CTA's first piece, 1 = its last
      float* part = p.part + (static_cast<long long>(cta) * 2 + (k == 0 ? 0 : 1)) * (HD + 2);
#pragma unroll
      for (int d = 0; d < DL; ++d) part[lane * DL + d] = acc[d];
      if (lane == 0) {
        part[HD] = M;
        part[HD + 1] = den;
      }
      __threadfence();
      __syncwarp();
      const long long st = pc.gs - pc.t0;                           // global index of token 0
      const int ca = static_cast<int>(((st + 1) * C - 1) / N);
      const int cb = static_cast<int>(((st + pc.len) * C - 1) / N);
      int last = 0;
      if (lane == 0) last = atomicAdd(p.cnt + bh, 1) == cb - ca;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (!last) return;
      __threadfence();
      float Mx = -INFINITY;
      for (int c = ca; c <= cb; ++c) {
        const int sl = (c == ca && static_cast<long long>(c) * N / C != st) ? 1 : 0;
        Mx = fmaxf(Mx, __ldcg(p.part + (static_cast<long long>(c) * 2 + sl) * (HD + 2) + HD));
      }
      float dsum = 0.0f, o[DL];
#pragma unroll
      for (int d = 0; d < DL; ++d) o[d] = 0.0f;
      for (int c = ca; c <= cb; ++c) {
        const int sl = (c == ca && static_cast<long long>(c) * N / C != st) ? 1 : 0;
        const float* pp = p.part + (static_cast<long long>(c) * 2 + sl) * (HD + 2);
        const float fc = fast_exp2(__ldcg(pp + HD) - Mx);
        dsum += fc * __ldcg(pp + HD + 1);
#pragma unroll
        for (int d = 0; d < DL; ++d) o[d] = fmaf(fc, __ldcg(pp + lane * DL + d), o[d]);
      }
      const float inv = 1.0f / dsum;
#pragma unroll
      for (int d = 0; d < DL; ++d) p.out[bh * HD + lane * DL + d] = o[d] * inv;
      if (lane == 0) p.cnt[bh] = 0;
    };

    Piece pc;
    locate(g0, pc);
    float qa[2 * Ge::PPL], qn[2 * Ge::PPL];
#pragma unroll
    for (int u = 0; u < 2 * Ge::PPL; ++u) qa[u] = 0.0f;
    Piece nx = pc;
    bool more = next_piece(nx);
    if (more) load_q(nx, qn);
    int k = 0;
    for (;;) {
      if (k >= R) {
        mbar_wait(mb_done + 8 * ((k - R) % R), ((k - R) / R) & 1);
        merge(k - R);
      }
      if (lane == 0) s_pc[k % R] = pc;
      if (k > 0) {
        build(k % R, qa);
        // the first stage of every consumer in this piece: L2 prefetch
        if (lane == 0)
          prefetch_rows(static_cast<long long>(pc.b) * p.H + pc.h, pc.t0, min(pc.t1, pc.t0 + NC * ST));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(mb_full + 8 * (k % R));
      if (k == 0) TRACE(3);
      if (!more) break;
      pc = nx;
      ++k;
#pragma unroll
      for (int u = 0; u < 2 * Ge::PPL; ++u) qa[u] = qn[u];
      more = next_piece(nx);
      if (more) load_q(nx, qn);
    }
    TRACE(5);
    for (int j = max(0, k + 1 - R); j <= k; ++j) {
      mbar_wait(mb_done + 8 * (j % R), (j / R) & 1);
      merge(j);
    }
    TRACE(6);
    return;
  }

  // ================================================================ consumers
  const int g = lane / LPT, sub = lane % LPT;
  const int nblk = HD >> p.blk_shift;
  const int sidx = (sub * kLaneDims) >> p.blk_shift;
  const int blk_lanes = (1 << p.blk_shift) / kLaneDims;
  const int rho = (g + (HD == 128 ? 4 * (sub >> 2) : 0)) & 7;     // bank rotation
  uint32_t rotA = 0, rotB = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    rotA |= static_cast<uint32_t>((i + rho) & 7) << (4 * i);
    rotB |= static_cast<uint32_t>((i + 4 + rho) & 7) << (4 * i);
  }
  const uint32_t vsel = static_cast<uint32_t>(lane) * 8u;
  const bool fused = p.k_new != nullptr;
  const uint32_t tab = kSmemWindow + Sm::kTab;
  auto nstages = [&](const Piece& pc) { return (pc.t1 - pc.t0 + ST - 1) / ST; };

  uint32_t jsel[8];
  auto set_jsel = [&](int slot) {
    const uint32_t add = HD == 64 ? (static_cast<uint32_t>(slot >> 1) << 16) | ((slot & 1) * 128u)
                                  : static_cast<uint32_t>(slot) << 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) jsel[k] = static_cast<uint32_t>(sub * 8 + ((k + rho) & 7)) * 4u + add;
  };

  uint64_t o2[8];
  float m = -INFINITY, l = 0.0f;
  bool any = false;            // this warp consumed a stage of the current piece
  auto reset_state = [&]() {
#pragma unroll
    for (int j = 0; j < 8; ++j) o2[j] = 0;
    m = -INFINITY;
    l = 0.0f;
    any = false;
  };

  auto load_stage = [&](StageRegs& Rg, const Piece& pc, int s) {
    const long long bh = static_cast<long long>(pc.b) * p.H + pc.h;
    const int tok0 = pc.t0 + s * ST;
    if (NQKV_PF > 0 && lane == 0) {   // L2 prefetch NQKV_PF of this warp's stages ahead
      const int first = s == warp ? 1 : NQKV_PF;
      for (int d = first; d <= NQKV_PF; ++d) {
        const int r0 = tok0 + d * NC * ST;
        if (r0 >= pc.t1) break;
        prefetch_rows(bh, r0, min(pc.t1, r0 + ST));
      }
    }
#ifdef NQKV_EXP_NOLOAD
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      Rg.k[i] = make_uint2(0x12345678u * (i + 1) + tok0, 0x9abcdef0u + lane);
      Rg.v[i] = make_uint2(0x31415926u * (i + 3) + tok0, 0x27182818u + lane);
      Rg.ks[i] = 1.0f;
      Rg.vs[i] = 0.5f;
    }
    return;
#endif
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      const int row = min(tok0 + i * G + g, pc.t1 - 1);     // clamp: masked rows read valid data
      const long long r = bh * p.Tc + row;
      Rg.k[i] = ldg_stream_64(p.kc + r * (HD / 2) + sub * 8);
      Rg.v[i] = ldg_stream_64(p.vc + r * (HD / 2) + sub * 8);
      Rg.ks[i] = ldg_nc_f32(p.ks + r * nblk + sidx);
      Rg.vs[i] = ldg_nc_f32(p.vs + r * nblk + sidx);
    }
  };

  auto consume = [&](StageRegs& Rg, const Piece& pc, int s) {
    const int tok0 = pc.t0 + s * ST;
    any = true;
    if (fused) {
      const int row_new = pc.len - 1;
      if (row_new >= tok0 && row_new < tok0 + ST && row_new < pc.t1) {   // warp-uniform
        const int rn = row_new - tok0, i_new = rn / G, g_new = rn % G;
        const long long off = static_cast<long long>(pc.b) * p.new_sb +
                              static_cast<long long>(pc.h) * p.new_sh + sub * kLaneDims;
        const NewTok nt = quantize_new_token(p.k_new + off, p.v_new + off, blk_lanes, tab);
        if (g == g_new) {
#pragma unroll
          for (int i = 0; i < kTPS; ++i) {
            if (i == i_new) {
              Rg.k[i] = nt.k; Rg.v[i] = nt.v; Rg.ks[i] = nt.ks; Rg.vs[i] = nt.vs;
            }
          }
          const long long r = (static_cast<long long>(pc.b) * p.H + pc.h) * p.Tc + row_new;
          *reinterpret_cast<uint2*>(const_cast<uint8_t*>(p.kc) + r * (HD / 2) + sub * 8) = nt.k;
          *reinterpret_cast<uint2*>(const_cast<uint8_t*>(p.vc) + r * (HD / 2) + sub * 8) = nt.v;
          if (((sub * kLaneDims) & ((1 << p.blk_shift) - 1)) == 0) {
            const_cast<float*>(p.ks)[r * nblk + sidx] = nt.ks;
            const_cast<float*>(p.vs)[r * nblk + sidx] = nt.vs;
          }
        }
      }
    }
#ifdef NQKV_EXP_NOCOMPUTE
    {
      uint32_t x = 0;
#pragma unroll
      for (int i = 0; i < kTPS; ++i)
        x ^= Rg.k[i].x ^ Rg.k[i].y ^ Rg.v[i].x ^ Rg.v[i].y ^ __float_as_uint(Rg.ks[i]) ^ __float_as_uint(Rg.vs[i]);
      o2[0] ^= x;
      l += 1.0f;
      m = 0.0f;
      return;
    }
#endif
    // scores (log2 domain): this lane's 16 dims via the q-table
    float sc[kTPS];
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      const uint32_t r0 = prmt(Rg.k[i].x, Rg.k[i].y, rotA);
      const uint32_t r1 = prmt(Rg.k[i].x, Rg.k[i].y, rotB);
      float a0 = lds_k(prmt(r0, jsel[0], 0x7604));
      float a1 = lds_k(prmt(r0, jsel[1], 0x7614));
      a0 += lds_k(prmt(r0, jsel[2], 0x7624));
      a1 += lds_k(prmt(r0, jsel[3], 0x7634));
      a0 += lds_k(prmt(r1, jsel[4], 0x7604));
      a1 += lds_k(prmt(r1, jsel[5], 0x7614));
      a0 += lds_k(prmt(r1, jsel[6], 0x7624));
      a1 += lds_k(prmt(r1, jsel[7], 0x7634));
      sc[i] = (a0 + a1) * Rg.ks[i];
    }
#pragma unroll
    for (int o = 1; o < LPT; o <<= 1) {
#pragma unroll
      for (int i = 0; i < kTPS; ++i) sc[i] += __shfl_xor_sync(0xffffffffu, sc[i], o);
    }
    float mt = -INFINITY;
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      sc[i] = (tok0 + i * G + g < pc.t1) ? sc[i] : -INFINITY;
      mt = fmaxf(mt, sc[i]);
    }
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
    if (mt > m) {                     // warp-uniform; the stage has >= 1 valid token
      const float corr = fast_exp2(m - mt);     // m = -inf -> 0
      m = mt;
      l *= corr;
      const uint64_t c2 = pack2(corr, corr);
#pragma unroll
      for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], c2);
    }
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      const float pr = fast_exp2(sc[i] - m);     // masked: exp2(-inf) = 0
      l += pr;
      const float w = pr * Rg.vs[i];
      const uint64_t w2 = pack2(w, w);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        o2[k] = ffma2(lds_v(prmt(Rg.v[i].x, vsel, 0x7604 | (k << 4))), w2, o2[k]);
        o2[4 + k] = ffma2(lds_v(prmt(Rg.v[i].y, vsel, 0x7604 | (k << 4))), w2, o2[4 + k]);
      }
    }
  };

  // end of piece k: sum the G token groups (common max), publish, arrive
  auto end_piece = [&](int k) {
    const int slot = k % R;
    if (any) {
#pragma unroll
      for (int o = LPT; o < 32; o <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
        for (int j = 0; j < 8; ++j) o2[j] = fadd2(o2[j], shfl_xor64(o2[j], o));
      }
      if (g == 0) {
        float* dst = s_o + (slot * NC + warp) * HD + sub * kLaneDims;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 a = unpack2(o2[2 * j]), b2 = unpack2(o2[2 * j + 1]);
          *reinterpret_cast<float4*>(dst + 4 * j) = make_float4(a.x, a.y, b2.x, b2.y);
        }
      }
    }
    if (lane == 0) s_ml[slot * NC + warp] = make_float2(any ? m : -INFINITY, l);
    __syncwarp();
    if (lane == 0) mbar_arrive(mb_done + 8 * slot);
  };

  // load cursor: (lp, ls) = next stage of this warp in piece order (index lpi)
  Piece cp;
  locate(g0, cp);
  Piece lp = cp;
  int ls = warp, lpi = 0;
  bool lvalid = true;
  while (ls >= nstages(lp)) {
    if (!next_piece(lp)) { lvalid = false; break; }
    ls = warp;
    ++lpi;
  }
  StageRegs RA, RB;
  if (lvalid) load_stage(RA, lp, ls);
  int cpi = 0;
  auto open_piece = [&]() {
    set_jsel(cpi % R);
    mbar_wait(mb_full + 8 * (cpi % R), (cpi / R) & 1);
    reset_state();
  };
  open_piece();
  TRACE(3);
  auto step = [&](StageRegs& cur, StageRegs& nxt) -> bool {
    // cur holds stage (lp, ls) of piece index lpi: advance the load cursor and
    // issue the next stage's loads, then catch consumption up to cur's piece
    const int cur_s = ls, cur_pi = lpi;
    ls += NC;
    while (ls >= nstages(lp)) {
      if (!next_piece(lp)) { lvalid = false; break; }
      ls = warp;
      ++lpi;
    }
    if (lvalid) load_stage(nxt, lp, ls);
    while (cpi < cur_pi) {
      end_piece(cpi);
      next_piece(cp);
      ++cpi;
      open_piece();
    }
    consume(cur, cp, cur_s);
    return lvalid;
  };
  if (lvalid) {
    for (;;) {
      if (!step(RA, RB)) break;
      TRACE(4);
      if (!step(RB, RA)) break;
    }
  }
  TRACE(5);
  // close the current piece and any remaining ones (no stages of this warp)
  for (;;) {
    end_piece(cpi);
    if (!next_piece(cp)) break;
    ++cpi;
    open_piece();
  }
  TRACE(6);
}

}  // namespace nqkv
