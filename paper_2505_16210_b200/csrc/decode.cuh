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
//    (s + o) % NC, o continuing the round robin of the CTA's previous pieces.  Lane (g, sub) owns 16 head dims (8 packed bytes) of token g of
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
#include <climits>
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
#ifndef NQKV_DEPTH
#define NQKV_DEPTH 2             // register ring depth: stages in flight per consumer warp
#endif
#ifndef NQKV_PEEK
#define NQKV_PEEK -1             // early last-arriver role for the last piece: 1 on, 0 off, -1 hd 128 only (measured)
#endif
#ifndef NQKV_QPF
#define NQKV_QPF 1               // early start: L2-prefetch the first pieces' q rows before the wait
#endif
#ifndef NQKV_SPLIT
#define NQKV_SPLIT -1            // split K/V ring: 1 on, 0 off, -1 hd 64 only (measured)
#endif
#ifndef NQKV_V16
#define NQKV_V16 0               // V levels as 16-bit fixed point in a 4-byte pair LUT (see lds_v16)
#endif
#ifndef NQKV_R64
#define NQKV_R64 4               // q-table ring depth at hd 64 (two tables per 64 KB block)
#endif
#ifndef NQKV_LATE_APPEND
#define NQKV_LATE_APPEND 1       // producer: release a piece's consumers before its appended token
#endif
#ifndef NQKV_PF
#define NQKV_PF 0                // bulk L2 prefetch distance in a warp's own stages (0: off; measured: no gain)
#endif
constexpr int kDecodeWarps = NQKV_DECODE_WARPS;
constexpr int kLaneDims = 16;          // head dims owned by one lane
constexpr int kTPS = NQKV_TPS;         // token slots per lane per stage
constexpr uint32_t kSmemWindow = 0x400;  // shared address of dynamic smem offset 0

struct DecodeParams {
  const __half* q;
  const uint8_t* kc;
  const void* ks;            // block scales, fp32 or fp16 (kernel template F16S)
  const uint8_t* vc;
  const void* vs;
  const int32_t* seq_lens;
  const __half* k_new;      // fused append (nullptr: attention only)
  const __half* v_new;
  long long new_sb, new_sh; // element strides of k_new / v_new ([B][H][hd])
  float* out;
  int* cnt;                 // [B*H] partial-arrival counters (zero between launches)
  unsigned long long* part; // [kMaxGrid][2][hd + 2] tagged partial words (o[hd], m, l);
                            // zero (= no partial) between launches
  int B, H, Tc, blk_shift, min_tokens;
  float scale_log2;         // softmax_scale * log2(e)
  Levels lv;
  BucketTab tab;
  const int* plan;             // optional per-step schedule (nqkv_decode_plan); nullptr: computed here
  int early;                   // NQKV_EARLY_START: plan and cache readable before the PDL wait
  int hpb_shift;               // blk > hd: scale rows [B][H >> hpb_shift][Tc] (blk_shift = log2 hd)
  // KV layouts (readings R16, R17):
  int kv_shift;                // grouped-query: query head h reads cache head h >> kv_shift
  const int32_t* bt;           // paged cache (kernel template PAGED): block table [B][bt_stride];
  int bt_stride, page_shift;   // token t of sequence b: page bt[b][t >> page_shift], row t & (P - 1)
  unsigned long long* trace;   // NQKV_TRACE builds: per-warp globaltimer stamps [grid][NW][16]
  // fused all-gather epilogue (kernel template GATHER):
  // every output row goes straight to all gather_g ranks' buffers
  // [B][h_total][hd] (peer pointers over NVLink P2P), at head offset
  // gather_rank * H; the last CTA then release-stores `epoch` into slot
  // gather_rank of every rank's flag array
  float* const* peer_out;
  unsigned* const* peer_flags;
  unsigned* gctr;              // CTA completion counter (zero between launches)
  int gather_g, gather_rank, h_total;
  unsigned epoch;
  const unsigned* epoch_ptr;   // non-null: the epoch is read here (graph replays bump it)
};

// one output float2 of row (b, h), dims d, d+1: local, or to every rank's
// gathered buffer (GATHER)
template <bool GATHER, int HD>
__device__ __forceinline__ void store_out2(const DecodeParams& p, long long bh, int b, int h, int d,
                                           float2 v) {
  if constexpr (GATHER) {
    const long long row = static_cast<long long>(b) * p.h_total + p.gather_rank * p.H + h;
    for (int r = 0; r < p.gather_g; ++r)
      *reinterpret_cast<float2*>(p.peer_out[r] + row * HD + d) = v;
  } else {
    (void)b; (void)h;
    *reinterpret_cast<float2*>(p.out + bh * HD + d) = v;
  }
}

// GATHER: this CTA's output stores are complete.  System-scope fence, then
// count; the last CTA of the launch resets the counter and publishes the
// epoch to every rank (release, system scope).
#ifndef NQKV_GFENCE
#define NQKV_GFENCE 1           // 0: none (timing only), 1: fence.sc.sys, 2: fence.acq_rel.sys,
#endif                          // 3: gpu-scope per CTA, system scope by the last CTA only
#if NQKV_GFENCE == 0 && !defined(NQKV_TIMING_ONLY)
#error "NQKV_GFENCE=0 builds a racy gather (no fences): timing experiments only, define NQKV_TIMING_ONLY"
#endif
#if NQKV_GFENCE == 3 && !defined(NQKV_GFENCE3_UNVERIFIED)
// gpu-scope fences per CTA rely on fence cumulativity to carry other CTAs' NVLink peer
// stores; only serialized simulated ranks on one GPU have run it
#error "NQKV_GFENCE=3 is unverified across GPUs: define NQKV_GFENCE3_UNVERIFIED to build it"
#endif
__device__ __forceinline__ void gather_fence(bool last) {
#if NQKV_GFENCE == 1
  __threadfence_system();
#elif NQKV_GFENCE == 2
  asm volatile("fence.acq_rel.sys;" ::: "memory");
#elif NQKV_GFENCE == 3
  if (last) __threadfence_system();
  else __threadfence();
#endif
  (void)last;
}
__device__ __forceinline__ void gather_cta_done(const DecodeParams& p) {
  gather_fence(false);
  const unsigned old = atomicAdd(p.gctr, 1u);
  if (old == gridDim.x - 1) {
    *p.gctr = 0u;
    gather_fence(true);
    const unsigned e = p.epoch_ptr ? *p.epoch_ptr : p.epoch;
    for (int r = 0; r < p.gather_g; ++r) {
      unsigned* f = p.peer_flags[r] + p.gather_rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(f), "r"(e) : "memory");
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef NQKV_TRACE
#define TRACE(k) do { if (p.trace && lane == 0) p.trace[(blockIdx.x * NW + warp) * 16 + (k)] = gtimer(); } while (0)
// producer phase durations (trace builds): accumulated, stored in slots
// 4 (mb_done waits), 5 (merges), 13 (table builds), 15 (appended tokens)
#define PT_START(t) const unsigned long long t = gtimer()
#define PT_ACC(acc, t) acc += gtimer() - t
#else
#define TRACE(k) do { } while (0)
#define PT_START(t) do { } while (0)
#define PT_ACC(acc, t) do { } while (0)
#endif

template <int HD>
struct Geo {
  static constexpr int LPT = HD / kLaneDims;  // lanes per token row (4 / 8)
  static constexpr int G = 32 / LPT;          // token groups per warp (8 / 4)
  static constexpr int ST = G * kTPS;         // tokens per warp stage
  static constexpr int R = HD == 64 ? NQKV_R64 : 2;  // q-table ring depth
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
  static constexpr uint32_t kLv = kK + (HD == 64 ? (R + 1) / 2 : R) * 0x10000u;   // float[16]
  static constexpr uint32_t kTab = kLv + 64;              // float2[kNumBuckets]
  static constexpr uint32_t kMbar = kTab + 272;           // u64 full[R], done[R]
  static constexpr uint32_t kMl = kMbar + 16 * R;         // float2 [R][NC]
  static constexpr uint32_t kPc = (kMl + R * NC * 8 + 15) / 16 * 16;   // Piece [R] (producer)
  static constexpr uint32_t kO = kPc + R * 32;            // float [R][NC][HD]
  static constexpr uint32_t kNew = kO + R * NC * HD * 4;  // float [R][HD + 4] appended-token state
  static constexpr uint32_t kPref = kNew + R * (HD + 4) * 4;  // int [kMaxBatch + 1]
  static constexpr uint32_t kLen = kPref + (kMaxBatch + 1) * 4 + 12;  // int [kMaxBatch]
  static constexpr uint32_t kOne = kLen + kMaxBatch * 4;  // u32 [kMaxBatch / 32]: fused, len == 1
  static constexpr uint32_t kWalk = kOne + kMaxBatch / 8;  // WalkState (80 B)
  // + int4 next pieces at kWalk + 80; int "prefetched partials" flag at
  // kWalk + 96; float [kPreRecs][HD + 2] prefetched partner records
  static constexpr uint32_t kPreFlag = kWalk + 96;
  static constexpr uint32_t kPre = kWalk + 112;
  static constexpr int kPreRecs = 4;
  static constexpr uint32_t kCur = (kPre + kPreRecs * (HD + 2) * 4 + 15) / 16 * 16;   // per-warp cursor (48 B)
  static constexpr uint32_t kBytes = kCur + NW * 48;
  static_assert(kBytes <= 227 * 1024, "decode smem over budget");
  static_assert(kMaxBatch <= 2 * NW * 32, "per-batch arrays: two entries per thread");
  static_assert((kTab % 16) == 0 && (kMbar % 8) == 0 && (kO % 16) == 0 && (kWalk % 16) == 0,
                "alignment");
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
// the same with a suspend-time hint: a waiter that is expected to wait long
// (the producer, for a whole piece) sleeps instead of re-polling, leaving the
// issue slots of its scheduler to the consumer warps
__device__ __forceinline__ void mbar_wait_sleep(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
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
// V pair LUT entry, 16-bit fixed point (NQKV_V16): (u[lo] | u[hi] << 16),
// u = RN(L * 32767) + 32768.  Returned as the fp32 pair (u[lo], u[hi]) * 2^-149:
// the payload IS the bit pattern of a subnormal float, so the value is exact
// and linear in u (no offset to cancel); weights carry a 2^100 factor so the
// products are normal.
__device__ __forceinline__ uint64_t lds_v16(uint32_t off) {
  uint64_t v;
  asm volatile("{.reg .b32 e, a, b;\n ld.shared.b32 e, [%1+0x400];\n and.b32 a, e, 65535;\n"
               " shr.u32 b, e, 16;\n mov.b64 %0, {a, b};}" : "=l"(v) : "r"(off));
  return v;
}
constexpr float kV16WScale = 0x1p100f;                      // weight factor
constexpr float kV16Out = 0x1p49f / 32767.0f;               // o * 2^49 / 32767 ...
constexpr float kV16Bias = 32768.0f / 32767.0f;             // ... - W * 32768 / 32767
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
// L2 prefetch of the cache rows [r0, r1) of one stage (r = (b*H + h)*Tc + t):
// one instruction per warp; lanes 0-8 / 9-17 take the K / V code lines,
// 18-19 / 20-21 the K / V scale lines (only lines holding bytes of the rows,
// so every address is inside the cache tensors).  A prefetch is a hint: it
// never changes what a load returns, so it may run before the PDL wait.
// The scale rows of the same tokens start at s0 (differs from r0 when a
// block spans several heads).
template <int HD, int NBLK, int SB, typename P>
__device__ __forceinline__ void prefetch_rows_l2(const P& p, int lane, long long r0, long long r1,
                                                 long long s0) {
  const bool sc = lane >= 18;
  const bool isv = sc ? lane >= 20 : lane >= 9;
  const int li = lane - (sc ? (isv ? 20 : 18) : (isv ? 9 : 0));
  const long long w = sc ? NBLK * SB : HD / 2;
  const long long a0 = sc ? s0 : r0, a1 = a0 + (r1 - r0);
  const long long f = (a0 * w) >> 7, l = (a1 * w - 1) >> 7;
  const unsigned char* base = sc ? reinterpret_cast<const unsigned char*>(isv ? p.vs : p.ks)
                                 : (isv ? p.vc : p.kc);
  if (lane < 22 && f + li <= l) asm volatile("prefetch.global.L2 [%0];" :: "l"(base + ((f + li) << 7)));
}
// 64-bit address = base + a * b (one IMAD.WIDE.U32)
__device__ __forceinline__ const void* addr_wide(const void* base, uint32_t a, uint32_t b) {
  unsigned long long r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(reinterpret_cast<unsigned long long>(base)));
  return reinterpret_cast<const void*>(r);
}
__device__ __forceinline__ float ldg_nc_f32(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
// block scale at byte offset `off` of a scale tensor: fp32, or fp16 (F16S;
// exact -- a block absmax of fp16 inputs is an fp16 value)
template <bool F16S>
__device__ __forceinline__ float ld_scale(const void* base, uint32_t off) {
  if constexpr (F16S) {
    unsigned short h;
    asm volatile("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(h)
                 : "l"(reinterpret_cast<const uint8_t*>(base) + off));
    return __half2float(__ushort_as_half(h));
  } else {
    return ldg_nc_f32(reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(base) + off));
  }
}

// One CTA-contiguous run of tokens of one (b, h): tokens [t0, t1) of a
// sequence whose streamed length is len.  Walked identically by every warp.
// All indices fit in 32 bits (the host enforces B*H*Tc < 2^31).
struct Piece {
  int gs;         // global (b, h, t) index of t0
  int b, h, len, t0, t1;
};

// Registers of one stage: kTPS token slots of this lane.
// RS (reduce-scatter, BLK = 16*kTPS): one K and one V scale per lane -- the
// scale of token slot sub % kTPS of its block -- instead of one per slot.
template <bool RS>
struct StageRegsT {
  uint2 k[kTPS], v[kTPS];
  float ks[RS ? 1 : kTPS], vs[RS ? 1 : kTPS];
};

// Launch-wide scheduling constants: C CTAs own equal contiguous ranges of
// the N-token (b, h, t) list; range c = [bnd(c), bnd(c + 1)).
struct Sched {
  int N, C, q, r;        // N = q*C + r
  __device__ __forceinline__ int bnd(int c) const { return c * q + (c * r) / C; }   // floor(c*N/C)
  __device__ int cta_of(int g) const {                                             // bnd(c) <= g < bnd(c+1)
    int lo = 0, hi = C;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (bnd(mid) <= g) lo = mid; else hi = mid;
    }
    return lo;
  }
};

// q-table slot offset (bytes from Smem::kK): hd 64 -> 64 KB block r >> 1,
// 128-B half r & 1 of each 256-B row; hd 128 -> block r
template <int HD>
__device__ __forceinline__ uint32_t slot_off(int r) {
  return HD == 64 ? static_cast<uint32_t>(r >> 1) * 0x10000u + static_cast<uint32_t>(r & 1) * 128u
                  : static_cast<uint32_t>(r) * 0x10000u;
}

// ------------------------------------------------------------------- plan
// A decode step's schedule depends only on (B, H, Tc, seq_lens, fused, grid),
// which every layer of the step shares: nqkv_decode_plan computes it once
// (decode_plan_kernel) and each layer's decode kernel reads its CTA's entry
// instead of rebuilding it on its own serial prologue path.
// Layout (int32): header [0, 8) = {N, C, q, r, B, H, fused, Tc};
// per-CTA entries [8, 8 + 28 kMaxGrid) = {first piece (6), last piece (6),
// order flags, limit, g0, g1, b*H + h of pieces 1..3 in processing order (-1:
// none), min(4, #pieces), first middle piece (6), 0, 0} (WalkState); then
// len'[kMaxBatch], prefix[kMaxBatch + 1] and the fused single-token
// mask[kMaxBatch / 32].
constexpr int kPlanHdr = 8;
constexpr int kPlanEntry = 28;
constexpr int kPlanLen = kPlanHdr + kPlanEntry * kMaxGrid;
constexpr int kPlanPref = kPlanLen + kMaxBatch;
constexpr int kPlanOne = kPlanPref + kMaxBatch + 1;
constexpr int kPlanInts = kPlanOne + kMaxBatch / 32;

// The piece of the range [g, g1) that starts at global token g.
__device__ __forceinline__ void locate_piece(const int* pref, const int* len, int B, int H, int g, int g1,
                                             Piece& pc) {
  int lo = 0, hi = B;                   // largest b with pref[b] <= g (pref[B] > g)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pref[mid] <= g) lo = mid; else hi = mid;
  }
  pc.b = lo;
  pc.len = len[lo];
  const int off = g - pref[lo];
  pc.h = off / pc.len;
  pc.t0 = off - pc.h * pc.len;
  pc.gs = g;
  pc.t1 = min(pc.len, pc.t0 + (g1 - g));
}

// Processing order of a CTA's pieces (range [g0, g1)):
//   [pl if split with the next CTA ("reorder": its partial is published
//   early)], then either pf, pf+1, ... or -- "defer", when pf continues the
//   previous CTA's sequence, a middle piece exists and the CTA has more
//   pieces than prebuilt q-table slots R -- pm = pf+1, ..., the last middle,
//   and pf last, so that no short split piece precedes a producer-built table.
struct WalkState {
  Piece pf, pl, pm;
  int flags;                 // bit 0: reorder, bit 1: defer
  int limit;                 // end of the sequential run (pl.gs if reorder, else g1)
};

// piece after pc in token order, if it starts below lim (len: per-batch streamed lengths)
__device__ __forceinline__ bool next_in_order(const int* len, int H, int g1, int lim, Piece& pc) {
  const int g = pc.gs + (pc.t1 - pc.t0);
  if (g >= lim) return false;
  if (pc.h + 1 < H) {
    ++pc.h;
  } else {
    do { ++pc.b; } while (len[pc.b] == 0);
    pc.h = 0;
    pc.len = len[pc.b];
  }
  pc.t0 = 0;
  pc.gs = g;
  pc.t1 = min(pc.len, g1 - g);
  return true;
}
__device__ __forceinline__ Piece walk_first_ws(const WalkState& w) {
  return (w.flags & 1) ? w.pl : (w.flags & 2) ? w.pm : w.pf;
}
// pc = piece k of the order -> piece k + 1 (false: none)
__device__ __forceinline__ bool walk_next_ws(const WalkState& w, const int* len, int H, int g1, Piece& pc,
                                             int k) {
  const bool defer = (w.flags & 2) != 0;
  if ((w.flags & 1) && k == 0) {
    pc = defer ? w.pm : w.pf;
    return true;
  }
  if (defer && pc.gs == w.pf.gs) return false;      // the deferred first piece was last
  if (next_in_order(len, H, g1, w.limit, pc)) return true;
  if (defer) {
    pc = w.pf;
    return true;
  }
  return false;
}

__device__ __forceinline__ void cta_walk(const int* pref, const int* len, int B, int H, int g0, int g1,
                                         int R, WalkState& w) {
  locate_piece(pref, len, B, H, g0, g1, w.pf);
  locate_piece(pref, len, B, H, g1 - 1, g1, w.pl);
  locate_piece(pref, len, B, H, max(g0, g1 - 1 - w.pl.t0), g1, w.pl);
  const bool reorder = w.pl.gs != w.pf.gs && w.pl.t1 < w.pl.len;
  w.limit = reorder ? w.pl.gs : g1;
  w.pm = w.pf;
  const bool middle = next_in_order(len, H, g1, w.limit, w.pm);
  bool defer = false;
  if (middle && w.pf.t0 > 0) {              // count pieces (up to R + 1)
    int n = 1 + (reorder ? 1 : 0);
    Piece x = w.pf;
    while (n <= R && next_in_order(len, H, g1, w.limit, x)) ++n;
    defer = n > R;
  }
  w.flags = (reorder ? 1 : 0) | (defer ? 2 : 0);
}

// b*H + h of pieces 1..3 in processing order (-1: none) and min(4, #pieces).
__device__ __forceinline__ int4 next_pieces(const WalkState& w, const int* len, int H, int g1) {
  int bh[3] = {-1, -1, -1};
  Piece x = walk_first_ws(w);
  int n = 1;
  for (int k = 1; k < 4; ++k) {
    if (!walk_next_ws(w, len, H, g1, x, k - 1)) break;
    bh[k - 1] = x.b * H + x.h;
    ++n;
  }
  return make_int4(bh[0], bh[1], bh[2], n);
}

// CTAs for an N-token launch: ~min_tokens per CTA, at most G.  When every
// non-empty sequence has the same streamed length and that count would give
// between nseq and 2*nseq - 1 CTAs, use exactly nseq: each CTA then holds one
// whole sequence and no cross-CTA merge is needed (small batches, e.g. c1).
__device__ __forceinline__ int cta_count(int N, int G, int min_tokens, int nseq, bool uniform) {
  int C = min(G, max(1, (N + min_tokens - 1) / min_tokens));
  if (uniform && nseq >= 1 && nseq <= G && C >= nseq && C < 2 * nseq) C = nseq;
  return C;
}

__global__ void __launch_bounds__(1024) decode_plan_kernel(const int32_t* seq_lens, int B, int H, int Tc,
                                                           int fused, int G, int min_tokens, int R,
                                                           int* plan) {
  __shared__ int s_len[kMaxBatch], s_pref[kMaxBatch + 1], s_wsum[32];
  pdl_enter();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int raw = tid < B ? min(max(seq_lens[tid], 0), Tc) : 0;
  const unsigned one = __ballot_sync(0xffffffffu, fused && raw == 1);
  if (lane == 0 && warp * 32 < B) plan[kPlanOne + warp] = static_cast<int>(one);
  const int len = fused ? max(raw - 1, 0) : raw;
  int n = H * len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, n, o);
    if (lane >= o) n += v;
  }
  if (lane == 31) s_wsum[warp] = n;
  __syncthreads();
  if (warp == 0) {
    int w = s_wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    s_wsum[lane] = w;                    // inclusive prefix of the warp totals
  }
  __syncthreads();
  if (tid < B) {
    const int incl = n + (warp ? s_wsum[warp - 1] : 0);
    s_len[tid] = len;
    s_pref[tid + 1] = incl;
    plan[kPlanLen + tid] = len;
    plan[kPlanPref + tid + 1] = incl;
  }
  if (tid == 0) {
    s_pref[0] = 0;
    plan[kPlanPref] = 0;
  }
  __shared__ int s_lmin, s_lmax;
  if (tid == 0) {
    s_lmin = INT_MAX;
    s_lmax = 0;
  }
  __syncthreads();
  if (tid < B && len > 0) {
    atomicMin(&s_lmin, len);
    atomicMax(&s_lmax, len);
  }
  const int nb = __syncthreads_count(tid < B && len > 0);
  Sched sc;
  sc.N = s_pref[B];
  sc.C = cta_count(sc.N, G, min_tokens, nb * H, nb > 0 && s_lmin == s_lmax);
  sc.q = sc.N / sc.C;
  sc.r = sc.N - sc.q * sc.C;
  if (tid == 0) {
    plan[0] = sc.N; plan[1] = sc.C; plan[2] = sc.q; plan[3] = sc.r;
    plan[4] = B; plan[5] = H; plan[6] = fused; plan[7] = Tc;
  }
  if (sc.N > 0 && tid < sc.C) {
    const int g0 = sc.bnd(tid), g1 = sc.bnd(tid + 1);
    WalkState w;
    cta_walk(s_pref, s_len, B, H, g0, g1, R, w);
    int* e = plan + kPlanHdr + tid * kPlanEntry;
    const Piece& pf = w.pf;
    const Piece& pl = w.pl;
    const Piece& pm = w.pm;
    e[0] = pf.gs; e[1] = pf.b; e[2] = pf.h; e[3] = pf.len; e[4] = pf.t0; e[5] = pf.t1;
    e[6] = pl.gs; e[7] = pl.b; e[8] = pl.h; e[9] = pl.len; e[10] = pl.t0; e[11] = pl.t1;
    e[12] = w.flags; e[13] = w.limit; e[14] = g0; e[15] = g1;
    const int4 nx = next_pieces(w, s_len, H, g1);
    e[16] = nx.x; e[17] = nx.y; e[18] = nx.z; e[19] = nx.w;
    e[20] = pm.gs; e[21] = pm.b; e[22] = pm.h; e[23] = pm.len; e[24] = pm.t0; e[25] = pm.t1;
    e[26] = e[27] = 0;
  }
}

// ---------------------------------------------------------------- producer
// Out of line (run once per piece by one warp): keeps the kernel's hot code
// compact in the instruction cache.

// blk > hd: this lane's max |k_new|, max |v_new| over the other (at most 3)
// heads of head h's group; all loads issued at once (one round trip)
template <int HD>
__device__ __forceinline__ float2 group_absmax(const DecodeParams& p, int b, int h) {
  constexpr int PPL = Geo<HD>::PPL;
  const int lane = threadIdx.x & 31;
  const int n = 1 << p.hpb_shift, h0 = h & -n;
  uint32_t rk[3][PPL], rv[3][PPL];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int hh = h0 + i + (h0 + i >= h ? 1 : 0);        // the group's heads other than h
    const long long so = static_cast<long long>(b) * p.new_sb + static_cast<long long>(hh) * p.new_sh;
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      rk[i][u] = rv[i][u] = 0u;
      if (i < n - 1) {
        rk[i][u] = __ldg(reinterpret_cast<const unsigned int*>(p.k_new + so) + lane + 32 * u);
        rv[i][u] = __ldg(reinterpret_cast<const unsigned int*>(p.v_new + so) + lane + 32 * u);
      }
    }
  }
  float mk = 0.0f, mv = 0.0f;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      __half2 hk, hv;
      memcpy(&hk, &rk[i][u], 4);
      memcpy(&hv, &rv[i][u], 4);
      const float2 fk = __half22float2(__habs2(hk)), fv = __half22float2(__habs2(hv));
      mk = fmaxf(mk, fmaxf(fk.x, fk.y));
      mv = fmaxf(mv, fmaxf(fv.x, fv.y));
    }
  }
  return make_float2(mk, mv);
}

// The appended token of a fused step, warp-wide: lane owns pairs j = lane +
// 32u (dims 2j, 2j+1).  Quantised exactly as quantize_kernel does, written to
// the cache row `row` of (b, h); vh gets its dequantised values and the return
// value is its score (log2 domain) from the q-table in `slot` (slot < 0: 0).
template <int HD, int NW, bool F16S, bool GRP>
#ifndef NQKV_NEWTOK_INLINE
#define NQKV_NEWTOK_INLINE 1          // inlined: c3 -2.7 % (a fused step calls it once per piece)
#endif
#if NQKV_NEWTOK_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
float new_token_fn(const DecodeParams& p, unsigned char* smem, int b, int h,
                                           int row, int slot, float* vh) {
  using Sm = Smem<HD, NW>;
  constexpr int PPL = Geo<HD>::PPL;
  const int lane = threadIdx.x & 31;
  const float* s_lv = reinterpret_cast<const float*>(smem + Sm::kLv);
  const uint32_t tabc = kSmemWindow + Sm::kTab - 0x5A000000u;
  const int nblk = HD >> p.blk_shift;
  const long long bh = static_cast<long long>(b) * p.H + h;
  const long long src = static_cast<long long>(b) * p.new_sb + static_cast<long long>(h) * p.new_sh;
  const long long r = bh * p.Tc + row;
  const int bp = 1 << (p.blk_shift - 1);                         // pairs per block
  float xk[2 * PPL], xv[2 * PPL], sk[PPL], sv[PPL];
#pragma unroll
  for (int u = 0; u < PPL; ++u) {
    const int j = lane + 32 * u;
    const float2 fk = __half22float2(__ldg(reinterpret_cast<const __half2*>(p.k_new + src) + j));
    const float2 fv = __half22float2(__ldg(reinterpret_cast<const __half2*>(p.v_new + src) + j));
    xk[2 * u] = fk.x; xk[2 * u + 1] = fk.y;
    xv[2 * u] = fv.x; xv[2 * u + 1] = fv.y;
    sk[u] = fmaxf(fabsf(fk.x), fabsf(fk.y));
    sv[u] = fmaxf(fabsf(fv.x), fabsf(fv.y));
  }
  if constexpr (GRP) {                 // blk > hd: the block is the token's slice of the
    const float2 m = group_absmax<HD>(p, b, h);   // head group: fold in the other heads
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      sk[u] = fmaxf(sk[u], m.x);
      sv[u] = fmaxf(sv[u], m.y);
    }
  }
  if (bp > 32) {                       // one block spans both halves (hd 128, blk 128)
    sk[0] = sk[PPL - 1] = fmaxf(sk[0], sk[PPL - 1]);
    sv[0] = sv[PPL - 1] = fmaxf(sv[0], sv[PPL - 1]);
  }
  const int span = min(bp, 32);
#pragma unroll
  for (int u = 0; u < PPL; ++u) {
    for (int o = 1; o < span; o <<= 1) {
      sk[u] = fmaxf(sk[u], __shfl_xor_sync(0xffffffffu, sk[u], o));
      sv[u] = fmaxf(sv[u], __shfl_xor_sync(0xffffffffu, sv[u], o));
    }
  }
  float part = 0.0f;
#pragma unroll
  for (int u = 0; u < PPL; ++u) {
    const int j = lane + 32 * u;
    const float rk = block_rcp(sk[u]), rv = block_rcp(sv[u]);
    const uint32_t ck = nf4_code_c(__fmul_rn(xk[2 * u], rk), tabc) |
                        (nf4_code_c(__fmul_rn(xk[2 * u + 1], rk), tabc) << 4);
    const uint32_t cvl = nf4_code_c(__fmul_rn(xv[2 * u], rv), tabc);
    const uint32_t cvh = nf4_code_c(__fmul_rn(xv[2 * u + 1], rv), tabc);
    const_cast<uint8_t*>(p.kc)[r * (HD / 2) + j] = static_cast<uint8_t>(ck);
    const_cast<uint8_t*>(p.vc)[r * (HD / 2) + j] = static_cast<uint8_t>(cvl | (cvh << 4));
    // scale writer: first lane of each block (blk > hd: of the group's first head)
    if (((2 * j) & ((1 << p.blk_shift) - 1)) == 0 && (!GRP || (h & ((1 << p.hpb_shift) - 1)) == 0)) {
      const long long si = GRP ? (bh >> p.hpb_shift) * p.Tc + row
                                       : r * nblk + ((2 * j) >> p.blk_shift);
      if constexpr (F16S) {                   // exact: an absmax of fp16 values
        reinterpret_cast<__half*>(const_cast<void*>(p.ks))[si] = __float2half_rn(sk[u]);
        reinterpret_cast<__half*>(const_cast<void*>(p.vs))[si] = __float2half_rn(sv[u]);
      } else {
        reinterpret_cast<float*>(const_cast<void*>(p.ks))[si] = sk[u];
        reinterpret_cast<float*>(const_cast<void*>(p.vs))[si] = sv[u];
      }
    }
    vh[2 * u] = __fmul_rn(sv[u], s_lv[cvl]);
    vh[2 * u + 1] = __fmul_rn(sv[u], s_lv[cvh]);
    if (slot >= 0)
      part += reinterpret_cast<const float*>(smem + Sm::kK + slot_off<HD>(slot) + ck * 256)[j] * sk[u];
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  return part;
}

// q-table of one piece into ring slot `slot`: lane owns pair quad qd = lane %
// Q for rows whose high nibble is lane / Q (mod 32 / Q).  T[e][j] =
// RN(c q_{2j} L[e & 15]) + RN(c q_{2j+1} L[e >> 4]) (the same formula as the
// cooperative table-0 build).
template <int HD, int NW>
#ifndef NQKV_BUILD_INLINE
#define NQKV_BUILD_INLINE 0
#endif
#if NQKV_BUILD_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void build_fn(unsigned char* smem, int slot, uint4 qraw, float scale_log2) {
  using Sm = Smem<HD, NW>;
  constexpr int Q = HD / 8;
  const int lane = threadIdx.x & 31;
  const float* s_lv = reinterpret_cast<const float*>(smem + Sm::kLv);
  __half2 h2[4];
  memcpy(h2, &qraw, 16);
  float a[4], b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __half22float2(h2[k]);
    a[k] = f.x * scale_log2;
    b[k] = f.y * scale_log2;
  }
  const int qd = lane % Q;
  uint64_t A01[16], A23[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const float L = s_lv[c];
    A01[c] = pack2(a[0] * L, a[1] * L);
    A23[c] = pack2(a[2] * L, a[3] * L);
  }
  unsigned char* base = smem + Sm::kK + slot_off<HD>(slot) + qd * 16;
#pragma unroll 1
  for (int hi = lane / Q; hi < 16; hi += 32 / Q) {
    const float L = s_lv[hi];
    const uint64_t B01 = pack2(b[0] * L, b[1] * L), B23 = pack2(b[2] * L, b[3] * L);
    unsigned char* row = base + hi * 16 * 256;
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) {
      const float2 t01 = unpack2(fadd2(A01[lo], B01)), t23 = unpack2(fadd2(A23[lo], B23));
      *reinterpret_cast<float4*>(row + lo * 256) = make_float4(t01.x, t01.y, t23.x, t23.y);
    }
  }
}

__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Before waiting for the consumers to finish the CTA's last piece k: if it is
// split across CTAs and every other CTA of its sequence has already arrived
// (counter = #others), this CTA will be the last arriver -- it takes that role
// without its own atomic.  If the others' records are already complete (one
// read, no spinning) it pulls them into shared memory, clears them and flags
// piece k; merge_fn then needs no global round trip at the end of the
// kernel.  Otherwise merge_fn runs the normal protocol.
template <int HD, int NW>
#ifndef NQKV_PEEK_INLINE
#define NQKV_PEEK_INLINE 0
#endif
#if NQKV_PEEK_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void peek_fn(const DecodeParams& p, unsigned char* smem, int k, Sched sc, int cta) {
  using Sm = Smem<HD, NW>;
  constexpr int PPL = Geo<HD>::PPL, R = Geo<HD>::R;
  const int lane = threadIdx.x & 31;
  const Piece pc = reinterpret_cast<const Piece*>(smem + Sm::kPc)[k % R];
  if (pc.t0 == 0 && pc.t1 == pc.len) return;
  const int st0 = pc.gs - pc.t0;
  const int ca = sc.cta_of(st0), cb = sc.cta_of(st0 + pc.len - 1);
  if (cb - ca > Sm::kPreRecs) return;
  const long long bh = static_cast<long long>(pc.b) * p.H + pc.h;
  int arrived = 0;
  if (lane == 0) arrived = ld_relaxed_s32(p.cnt + bh);
  arrived = __shfl_sync(0xffffffffu, arrived, 0);
  if (arrived != cb - ca) return;
  float* pre = reinterpret_cast<float*>(smem + Sm::kPre);
  auto dim = [&](int u) { return 2 * (lane + 32 * u); };
  auto rec_of = [&](int c) {
    return p.part + (static_cast<long long>(c) * 2 + ((c == ca && sc.bnd(c) != st0) ? 1 : 0)) * (HD + 2);
  };
  // one read of every record (no spinning: a record not yet complete makes
  // the final merge take the normal path); all complete -> keep and clear
  bool ok = true;
  for (int c = ca; c <= cb; ++c) {
    if (c == cta) continue;
    const unsigned long long* r = rec_of(c);
    const unsigned long long wm = ld_relaxed_u64(r + HD), wl = ld_relaxed_u64(r + HD + 1);
    bool good = (wm >> 32) && (wl >> 32);
    float* dst = pre + (c - ca - (c > cta ? 1 : 0)) * (HD + 2);
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      const unsigned long long w0 = ld_relaxed_u64(r + dim(u)), w1 = ld_relaxed_u64(r + dim(u) + 1);
      good = good && (w0 >> 32) && (w1 >> 32);
      dst[dim(u)] = __uint_as_float(static_cast<uint32_t>(w0));
      dst[dim(u) + 1] = __uint_as_float(static_cast<uint32_t>(w1));
    }
    if (lane == 0) {
      dst[HD] = __uint_as_float(static_cast<uint32_t>(wm));
      dst[HD + 1] = __uint_as_float(static_cast<uint32_t>(wl));
    }
    ok = ok && __all_sync(0xffffffffu, good);
  }
  if (!ok) return;
  for (int c = ca; c <= cb; ++c) {
    if (c == cta) continue;
    unsigned long long* r = rec_of(c);
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      st_relaxed_u64(r + dim(u), 0ull);
      st_relaxed_u64(r + dim(u) + 1, 0ull);
    }
    if (lane == 0) {
      st_relaxed_u64(r + HD, 0ull);
      st_relaxed_u64(r + HD + 1, 0ull);
    }
  }
  __syncwarp();
  if (lane == 0) *reinterpret_cast<int*>(smem + Sm::kPreFlag) = k + 1;
}

// Merge piece k's NC consumer states (ring slot k % R) and, in a fused step,
// the appended token's state: write the output, or a partial (+ the
// last-arriver merge of the sequence's partials across CTAs).
template <int HD, int NW, bool GATHER>
#ifndef NQKV_MERGE_INLINE
#define NQKV_MERGE_INLINE 1          // inlined: a call to cold code at the kernel's end costs ~1 %
#endif
#if NQKV_MERGE_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void merge_fn(const DecodeParams& p, unsigned char* smem, int k, Sched sc,
                                      int cta, int g0) {
  using Sm = Smem<HD, NW>;
  constexpr int PPL = Geo<HD>::PPL, R = Geo<HD>::R, NC = NW - 1;
  const int lane = threadIdx.x & 31;
  const int slot = k % R;
  const Piece pc = reinterpret_cast<const Piece*>(smem + Sm::kPc)[slot];
  const float* st = reinterpret_cast<const float*>(smem + Sm::kNew) + slot * (HD + 4);
  const float2* s_ml = reinterpret_cast<const float2*>(smem + Sm::kMl) + slot * NC;
  const float* s_o = reinterpret_cast<const float*>(smem + Sm::kO) + slot * NC * HD;
  auto dim = [&](int u) { return 2 * (lane + 32 * u); };
#ifdef NQKV_TRACE
  const int warp = threadIdx.x >> 5;
  if (p.trace && lane == 0) p.trace[(blockIdx.x * NW + warp) * 16 + 12] = gtimer();   // merge entry
#endif
  const float snew = st[HD];
  float mw[NC];
  float M = snew;
#pragma unroll
  for (int w = 0; w < NC; ++w) {
    mw[w] = s_ml[w].x;
    M = fmaxf(M, mw[w]);
  }
  float den = 0.0f, acc[2 * PPL];
#pragma unroll
  for (int d = 0; d < 2 * PPL; ++d) acc[d] = 0.0f;
#pragma unroll
  for (int w = 0; w < NC; ++w) {
    const float f = fast_exp2(mw[w] - M);           // consumer without tokens: -inf -> 0
    den = fmaf(f, s_ml[w].y, den);
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      const float2 x = *reinterpret_cast<const float2*>(s_o + w * HD + dim(u));
      acc[2 * u] = fmaf(f, x.x, acc[2 * u]);
      acc[2 * u + 1] = fmaf(f, x.y, acc[2 * u + 1]);
    }
  }
  if (snew != -INFINITY) {
    const float f = fast_exp2(snew - M);
    den += f;
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      const float2 x = *reinterpret_cast<const float2*>(st + dim(u));
      acc[2 * u] = fmaf(f, x.x, acc[2 * u]);
      acc[2 * u + 1] = fmaf(f, x.y, acc[2 * u + 1]);
    }
  }
  const long long bh = static_cast<long long>(pc.b) * p.H + pc.h;
#ifdef NQKV_TRACE
  if (p.trace && lane == 0) p.trace[(blockIdx.x * NW + warp) * 16 + 14] = gtimer();   // combined
#endif
  if (pc.t0 == 0 && pc.t1 == pc.len) {
    const float inv = 1.0f / den;
#pragma unroll
    for (int u = 0; u < PPL; ++u)
      store_out2<GATHER, HD>(p, bh, pc.b, pc.h, dim(u), make_float2(acc[2 * u] * inv, acc[2 * u + 1] * inv));
    return;
  }
  // Partial piece.  Record slot 0 = this CTA's first piece (starts at g0),
  // 1 = its last.  Arrive first (relaxed counter): a CTA that is not the
  // last arriver publishes its partial as tagged words and leaves; the last
  // one polls the others' records -- every one of them was, or is about to
  // be, stored by a CTA that has already arrived and never waits on anyone,
  // so the poll terminates -- merges all of them in CTA order, and clears
  // the records and the counter for the next launch.  Two L2 round trips on
  // the critical path (atomic, poll), no fence.
  const int st0 = pc.gs - pc.t0;                                // global index of token 0
  const int ca = sc.cta_of(st0), cb = sc.cta_of(st0 + pc.len - 1);
  // prefetched by peek_fn: this CTA is the last arriver, the others' records
  // are in shared memory (already cleared in global memory)
  const bool pre = *reinterpret_cast<const int*>(smem + Sm::kPreFlag) == k + 1;
  int last = 1;
  if (!pre) {
    if (lane == 0) last = atom_add_relaxed(p.cnt + bh, 1) == cb - ca;
    last = __shfl_sync(0xffffffffu, last, 0);
  }
  auto rec = [&](int c, int sl) { return p.part + (static_cast<long long>(c) * 2 + sl) * (HD + 2); };
  auto tag = [](float v) {
    return static_cast<unsigned long long>(__float_as_uint(v)) | (1ull << 32);
  };
  if (!last) {
    unsigned long long* r = rec(cta, pc.gs == g0 ? 0 : 1);
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      st_relaxed_u64(r + dim(u), tag(acc[2 * u]));
      st_relaxed_u64(r + dim(u) + 1, tag(acc[2 * u + 1]));
    }
    if (lane == 0) {
      st_relaxed_u64(r + HD, tag(M));
      st_relaxed_u64(r + HD + 1, tag(den));
    }
    return;
  }
  constexpr int MAXC = 4;                     // records merged per pass (registers)
  float Mx = -INFINITY, dsum = 0.0f, o[2 * PPL];
#pragma unroll
  for (int d = 0; d < 2 * PPL; ++d) o[d] = 0.0f;
  for (int c0 = ca; c0 <= cb; c0 += MAXC) {
    float rm[MAXC], rl[MAXC], ro[MAXC][2 * PPL];
    const int nc = min(MAXC, cb - c0 + 1);
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      if (i >= nc) break;
      const int c = c0 + i;
      if (c == cta) {
        rm[i] = M; rl[i] = den;
#pragma unroll
        for (int d = 0; d < 2 * PPL; ++d) ro[i][d] = acc[d];
        continue;
      }
      if (pre) {
        const float* src = reinterpret_cast<const float*>(smem + Sm::kPre) + (c - ca - (c > cta ? 1 : 0)) * (HD + 2);
        rm[i] = src[HD];
        rl[i] = src[HD + 1];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          ro[i][2 * u] = src[dim(u)];
          ro[i][2 * u + 1] = src[dim(u) + 1];
        }
        continue;
      }
      const unsigned long long* r = rec(c, (c == ca && sc.bnd(c) != st0) ? 1 : 0);
      unsigned long long wm, wl, wo[2 * PPL];
      for (;;) {
        wm = ld_relaxed_u64(r + HD);
        wl = ld_relaxed_u64(r + HD + 1);
        bool ok = (wm >> 32) && (wl >> 32);
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          wo[2 * u] = ld_relaxed_u64(r + dim(u));
          wo[2 * u + 1] = ld_relaxed_u64(r + dim(u) + 1);
          ok = ok && (wo[2 * u] >> 32) && (wo[2 * u + 1] >> 32);
        }
        if (__all_sync(0xffffffffu, ok)) break;
      }
      rm[i] = __uint_as_float(static_cast<uint32_t>(wm));
      rl[i] = __uint_as_float(static_cast<uint32_t>(wl));
#pragma unroll
      for (int d = 0; d < 2 * PPL; ++d) ro[i][d] = __uint_as_float(static_cast<uint32_t>(wo[d]));
      unsigned long long* rw = const_cast<unsigned long long*>(r);  // clear for the next launch
#pragma unroll
      for (int u = 0; u < PPL; ++u) {
        st_relaxed_u64(rw + dim(u), 0ull);
        st_relaxed_u64(rw + dim(u) + 1, 0ull);
      }
      if (lane == 0) {
        st_relaxed_u64(rw + HD, 0ull);
        st_relaxed_u64(rw + HD + 1, 0ull);
      }
    }
    // merge in CTA order: batch max first, the running sum rescaled only
    // when a batch raises it (one batch -- the usual case -- is a plain
    // two-pass softmax merge)
    float Mn = Mx;
#pragma unroll
    for (int i = 0; i < MAXC; ++i)
      if (i < nc) Mn = fmaxf(Mn, rm[i]);
    const float fa = fast_exp2(Mx - Mn);      // Mx = -inf on the first batch: 0
    dsum *= fa;
#pragma unroll
    for (int d = 0; d < 2 * PPL; ++d) o[d] *= fa;
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      if (i >= nc) break;
      const float fc = fast_exp2(rm[i] - Mn);
      dsum = fmaf(fc, rl[i], dsum);
#pragma unroll
      for (int d = 0; d < 2 * PPL; ++d) o[d] = fmaf(fc, ro[i][d], o[d]);
    }
    Mx = Mn;
  }
  const float inv = 1.0f / dsum;
#pragma unroll
  for (int u = 0; u < PPL; ++u)
    store_out2<GATHER, HD>(p, bh, pc.b, pc.h, dim(u), make_float2(o[2 * u] * inv, o[2 * u + 1] * inv));
  if (lane == 0) p.cnt[bh] = 0;
}

// GRP: blk > hd (a block spans 2^hpb_shift heads; instantiated with BLK = HD)
template <int HD, int BLK, int NW, bool F16S, bool GRP, bool GATHER, bool PAGED = false>
__global__ void __launch_bounds__(NW * 32, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int SB = F16S ? 2 : 4;   // bytes per stored block scale
  using Ge = Geo<HD>;
  using Sm = Smem<HD, NW>;
  constexpr int LPT = Ge::LPT, G = Ge::G, ST = Ge::ST, R = Ge::R, PPL = Ge::PPL;
  constexpr int NT = NW * 32, NC = NW - 1;
  constexpr int Q = HD / 8;          // 4-pair quads per q-table row
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TRACE(0);
#ifdef NQKV_TRACE
  if (p.trace && lane == 0 && warp == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[(blockIdx.x * NW + warp) * 16 + 14] = smid + 1;
  }
#endif
  if (static_cast<uint32_t>(__cvta_generic_to_shared(smem)) != kSmemWindow) __trap();
  float* s_lv = reinterpret_cast<float*>(smem + Sm::kLv);
  float2* s_tab = reinterpret_cast<float2*>(smem + Sm::kTab);
  const uint32_t mb_full = kSmemWindow + Sm::kMbar;          // full[R]  (count 1: producer)
  const uint32_t mb_done = kSmemWindow + Sm::kMbar + 8 * R;  // done[R]  (count NC)
  float* s_o = reinterpret_cast<float*>(smem + Sm::kO);
  float2* s_ml = reinterpret_cast<float2*>(smem + Sm::kMl);
  Piece* s_pc = reinterpret_cast<Piece*>(smem + Sm::kPc);
  float* s_new = reinterpret_cast<float*>(smem + Sm::kNew);
  int* s_pref = reinterpret_cast<int*>(smem + Sm::kPref);
  int* s_len = reinterpret_cast<int*>(smem + Sm::kLen);
  const bool fused = p.k_new != nullptr;
  const int nblk = HD >> p.blk_shift;

  // ---- prologue independent of the previous kernel.  Warm the constant
  // cache: one lane per 64-byte line of the parameter block, all in parallel
  // (otherwise each first use of a parameter line on the serial prologue path
  // is a separate cold miss).
  if (warp == 1 && lane * 16 < static_cast<int>(sizeof(DecodeParams) / 4)) {
    const uint32_t w = reinterpret_cast<const uint32_t*>(&p)[lane * 16];
    if (w == 0x9E3779B9u && lane == 31) s_tab[0].x = 0.0f;   // keeps the load; never true in practice
  }
  if (tid < 16) s_lv[tid] = p.lv.v[tid];
  if (tid < kNumBuckets) s_tab[tid] = p.tab.e[tid];
  if (tid == 0) {
    *reinterpret_cast<int*>(smem + Sm::kPreFlag) = 0;
    for (int r = 0; r < R; ++r) {
      mbar_init(mb_full + 8 * r, 1);
      mbar_init(mb_done + 8 * r, NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // V LUT (independent of the previous kernel); levels via shared memory
  // (a divergent constant-bank index would serialise)
  __syncthreads();
#if NQKV_V16
  for (int i = tid; i < 256 * 8; i += NT) {      // 16 B = four lane copies per store
    const int e = i >> 3;
    const uint32_t u = static_cast<uint32_t>(__float2int_rn(s_lv[e & 15] * 32767.0f) + 32768) |
                       (static_cast<uint32_t>(__float2int_rn(s_lv[e >> 4] * 32767.0f) + 32768) << 16);
    *reinterpret_cast<uint4*>(smem + Sm::kV + e * 256 + (i & 7) * 16) = make_uint4(u, u, u, u);
  }
#else
  for (int i = tid; i < 256 * 16; i += NT) {     // 16 B = two lane copies per store
    const int e = i >> 4;
    const float lo = s_lv[e & 15], hi = s_lv[e >> 4];
    *reinterpret_cast<float4*>(smem + Sm::kV + e * 256 + (i & 15) * 16) = make_float4(lo, hi, lo, hi);
  }
#endif
  const uint32_t* s_one = reinterpret_cast<const uint32_t*>(smem + Sm::kOne);
  WalkState* s_ws = reinterpret_cast<WalkState*>(smem + Sm::kWalk);
  static_assert(sizeof(WalkState) == 80, "walk state layout");
  const int cta = blockIdx.x;
  Sched sc;
  int g0 = 0, g1 = 0;
  // pieces 0..R0-1 (processing order) get their q-tables built by the whole
  // CTA before the consumers start (plan mode: up to R; else piece 0 only),
  // so short leading pieces never leave consumers waiting on the producer
  int R0 = 1;
  int4 pbh = make_int4(-1, -1, -1, 1);     // b*H + h of pieces 1..3, #pieces (<= 4)
  Piece p0;                    // first piece in processing order
  // per-batch arrays into shared memory: from the plan, or computed here
  auto copy_plan_arrays = [&]() {
    for (int i = tid; i < p.B; i += NT) s_len[i] = __ldcg(p.plan + kPlanLen + i);
    for (int i = tid; i <= p.B; i += NT) s_pref[i] = __ldcg(p.plan + kPlanPref + i);
    for (int i = tid; i < (p.B + 31) / 32; i += NT)
      reinterpret_cast<uint32_t*>(smem + Sm::kOne)[i] = __ldcg(p.plan + kPlanOne + i);
  };
  auto read_plan = [&]() {
    const int4* e4 = reinterpret_cast<const int4*>(p.plan + kPlanHdr + cta * kPlanEntry);
    const int4 hdr = __ldcg(reinterpret_cast<const int4*>(p.plan));
    sc.N = hdr.x; sc.C = hdr.y; sc.q = hdr.z; sc.r = hdr.w;
    if (sc.N == 0 || cta >= sc.C) {
      if (sc.N == 0) copy_plan_arrays();
      __syncthreads();
    } else {
      const int4 a = __ldcg(e4), b = __ldcg(e4 + 1), c = __ldcg(e4 + 2), d = __ldcg(e4 + 3);
      pbh = __ldcg(e4 + 4);
      const int4 f = __ldcg(e4 + 5), h2 = __ldcg(e4 + 6);
      R0 = min(R, pbh.w);
      WalkState w;
      w.pf.gs = a.x; w.pf.b = a.y; w.pf.h = a.z; w.pf.len = a.w; w.pf.t0 = b.x; w.pf.t1 = b.y;
      w.pl.gs = b.z; w.pl.b = b.w; w.pl.h = c.x; w.pl.len = c.y; w.pl.t0 = c.z; w.pl.t1 = c.w;
      w.pm.gs = f.x; w.pm.b = f.y; w.pm.h = f.z; w.pm.len = f.w; w.pm.t0 = h2.x; w.pm.t1 = h2.y;
      w.flags = d.x;
      w.limit = d.y;
      g0 = d.z;
      g1 = d.w;
      p0 = walk_first_ws(w);
      if (tid == 0) *s_ws = w;
    }
  };
  // NQKV_EARLY_START (planned calls): neither the plan nor the cache is
  // written by the kernel launched just before this one, and every kernel of
  // the library triggers its successor only after its own wait, so both are
  // complete: read the plan and issue the first cache loads before the PDL
  // wait; everything else (q, k_new / v_new, out, workspace) after it.
  const bool pre = p.plan != nullptr && p.early != 0;
  if (!pre) {
    pdl_enter();
    TRACE(1);
  }
  if (p.plan) {
    read_plan();
  } else {
    // ---- per-batch streamed lengths and token prefix: tokens(b) = H * len'_b.
    // Fused step: the appended row (len - 1) is not streamed; the producer
    // quantises it and folds it into the piece merge (s_len holds len').
    if (warp == 0) {
      int carry = 0, lmin = INT_MAX, lmax = 0, nb = 0;
      if (lane == 0) s_pref[0] = 0;
      for (int b0 = 0; b0 < p.B; b0 += 32) {
        const int b = b0 + lane;
        const int raw = b < p.B ? min(max(p.seq_lens[b], 0), p.Tc) : 0;
        const unsigned one = __ballot_sync(0xffffffffu, fused && raw == 1);
        if (lane == 0) reinterpret_cast<uint32_t*>(smem + Sm::kOne)[b0 >> 5] = one;
        int n = 0;
        if (b < p.B) {
          const int len = fused ? max(raw - 1, 0) : raw;
          s_len[b] = len;
          n = p.H * len;
          if (len > 0) {
            lmin = min(lmin, len);
            lmax = max(lmax, len);
            ++nb;
          }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, n, o);
          if (lane >= o) n += v;
        }
        if (b < p.B) s_pref[b + 1] = carry + n;
        carry += __shfl_sync(0xffffffffu, n, 31);
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
      }
      if (lane == 0) {
        reinterpret_cast<int*>(smem + Sm::kPreFlag)[1] = nb;
        reinterpret_cast<int*>(smem + Sm::kPreFlag)[2] = nb > 0 && lmin == lmax;
      }
    }
    __syncthreads();
    sc.N = s_pref[p.B];
    if (sc.N > 0) {
      const int nb = reinterpret_cast<const int*>(smem + Sm::kPreFlag)[1];
      sc.C = cta_count(sc.N, static_cast<int>(gridDim.x), p.min_tokens, nb * p.H,
                       reinterpret_cast<const int*>(smem + Sm::kPreFlag)[2] != 0);
      sc.q = sc.N / sc.C;
      sc.r = sc.N - sc.q * sc.C;
      if (cta < sc.C) {
        g0 = sc.bnd(cta);
        g1 = sc.bnd(cta + 1);
        // Processing order.  If the range's last piece is split with the next
        // CTA it is processed FIRST, so that both cross-CTA partials of this CTA
        // are published early (WalkState: full order).  Kept in shared memory:
        // the walkers run rarely.
        if (tid == 0) {
          WalkState w;
          cta_walk(s_pref, s_len, p.B, p.H, g0, g1, R, w);
          *s_ws = w;
          *reinterpret_cast<int4*>(smem + Sm::kWalk + 80) = next_pieces(w, s_len, p.H, g1);
        }
      }
    }
    __syncthreads();
    if (sc.N > 0 && cta < sc.C) {
      p0 = walk_first_ws(*s_ws);
      pbh = *reinterpret_cast<const int4*>(smem + Sm::kWalk + 80);
      R0 = min(R, pbh.w);
    }
  }
  TRACE(2);

  // ---- empty sequences (out = 0, reading R12) and, in a fused step,
  // sequences whose only token is the appended one (out = its value).  Off
  // the critical path: done by the producer warps after table 0 (or here by
  // every CTA when there is no token to stream at all).
  auto empties = [&](int wid, int nwarps) {
    for (int i = wid * 32 + lane; i < p.B * p.H * HD; i += nwarps * 32) {
      const int b = i / (p.H * HD);
      if (s_len[b] == 0 && !((s_one[b >> 5] >> (b & 31)) & 1u)) {
        if constexpr (GATHER) {
          const int bh = i / HD, h = bh - b * p.H;
          const long long row = static_cast<long long>(b) * p.h_total + p.gather_rank * p.H + h;
          for (int r = 0; r < p.gather_g; ++r) p.peer_out[r][row * HD + (i - bh * HD)] = 0.0f;
        } else {
          p.out[i] = 0.0f;
        }
      }
    }
    if (!fused) return;
    for (int bh = wid; bh < p.B * p.H; bh += nwarps) {
      const int b = bh / p.H, h = bh - b * p.H;
      if (!((s_one[b >> 5] >> (b & 31)) & 1u)) continue;
      float vh[2 * PPL];
      new_token_fn<HD, NW, F16S, GRP>(p, smem, b, h, 0, -1, vh);
#pragma unroll
      for (int u = 0; u < PPL; ++u)
        store_out2<GATHER, HD>(p, static_cast<long long>(bh), b, h, 2 * (lane + 32 * u),
                               make_float2(vh[2 * u], vh[2 * u + 1]));
    }
  };
  if (sc.N == 0 || cta >= sc.C) {
    if (pre) pdl_enter();                     // empties read k_new / write out
    if (sc.N == 0) empties(blockIdx.x * NW + warp, gridDim.x * NW);
    if constexpr (GATHER) {
      __syncthreads();
      if (tid == 0) gather_cta_done(p);
    }
    return;
  }
  TRACE(13);

  // ---- piece walking (identical in every warp; needs s_len / s_pref)
  auto walk_first = [&](Piece& pc) { pc = walk_first_ws(*s_ws); };
  auto walk_next = [&](Piece& pc, int k) -> bool {   // k = index of pc in processing order
    return walk_next_ws(*s_ws, s_len, p.H, g1, pc, k);
  };
  auto nstages = [&](const Piece& pc) { return (pc.t1 - pc.t0 + ST - 1) / ST; };
  // cache rows of a piece: its KV head (query head h >> kv_shift, R16)
  auto kvhead = [&](const Piece& pc) { return pc.b * (p.H >> p.kv_shift) + (pc.h >> p.kv_shift); };
  auto rowbase = [&](const Piece& pc) { return kvhead(pc) * p.Tc; };
  // scale row base: the head group's row when a block spans heads (blk > hd)
  auto srowbase = [&](const Piece& pc) {
    if constexpr (GRP) return (kvhead(pc) >> p.hpb_shift) * p.Tc;
    else return rowbase(pc);
  };
  auto load_quad = [&](const Piece& pc, int qd) -> uint4 {
    const long long bh = static_cast<long long>(pc.b) * p.H + pc.h;
    return __ldg(reinterpret_cast<const uint4*>(p.q + bh * HD) + qd);
  };

  // ---- q of piece 0 first (its table is the first thing the consumers
  // need), then the consumers' first stage loads
  uint4 q0, qx[R > 1 ? R - 1 : 1];          // q quads of the prebuilt pieces (loaded below)
  const int g = lane / LPT, sub = lane % LPT;
  constexpr int NBLK = HD / BLK;
  const int sidx = (sub * kLaneDims) / BLK;
  // Reduce-scatter layout (BLK >= 16 * kTPS, i.e. blk 64 or 128): the kTPS lanes of a
  // block each own one token slot j = sub % kTPS of the stage: they load its
  // K / V scale, finish its score, exponentiate it, and hand its weight
  // p_j * vs_j to the other lanes of the block.  1 scale load, 1 exp2 per lane
  // and stage instead of kTPS.
  // (blk 128 at hd 128: the two 4-lane halves of the block share one scale,
  // so the same per-half reduce-scatter applies)
  constexpr bool RS = BLK >= kLaneDims * kTPS && kTPS == 4;
  const uint32_t soff_rs = RS ? static_cast<uint32_t>((sub & 3) * G * NBLK * SB) : 0u;
  // ---- load cursor: this lane's bytes of the next stage this warp loads.
  // Stage ls of piece lp (ST tokens from lp.t0 + ls * ST) belongs to
  // consumer (ls + lro) mod NC, where lro (the warp of the piece's first
  // stage) continues the previous piece's round robin: over a CTA's whole
  // range the warps' stage counts differ by at most one.  Fast path (the next
  // stage is in the same piece): pointer increments only; the piece walk runs
  // at piece boundaries.  (The host guarantees each codes tensor is < 4 GB,
  // so row offsets fit 32 bits.)
  using StageRegs = StageRegsT<RS>;
  // Registers hold only the fast path: this lane's K-code pointer (V codes at
  // a fixed distance), its scale byte offset, the rows left in the piece from
  // its slot-0 row, the warp's stages left in the piece, and the piece index.
  // The walk state (piece, first/last stage, round-robin origin) lives in a
  // per-warp shared-memory slot, read only at piece boundaries.
  struct WCur {
    Piece lp;
    int ls_last, lro, lns, pad[3];
  };
  static_assert(sizeof(WCur) == 48, "cursor slot");
  WCur* s_cur = reinterpret_cast<WCur*>(smem + Sm::kCur) + warp;
  const uint8_t* kcp = p.kc;
  const long long vdelta = p.vc - p.kc;
  uint32_t soff = 0;
  int nvl = 0, left = 0, lpi = 0;
  int ptok = 0;                  // PAGED: first token of the cursor's stage
  int npa = -1;                  // PAGED: page id of the cursor's stage, read one stage early (-1: not read)
  bool lvalid = warp < NC;
  constexpr int KSTEP = NC * ST * (HD / 2), SSTEP = NC * ST * NBLK * SB;
  auto set_cursor = [&](const Piece& lp, int ls, int lro, int lns) {
    const int ltok = lp.t0 + ls * ST;
    if constexpr (PAGED) {
      // paged cache (R17): the cursor keeps the token, the sequence's
      // block-table row (in kcp) and the KV head (in soff); rows are found
      // per stage in load_stage
      ptok = ltok;
      npa = -1;
      kcp = reinterpret_cast<const uint8_t*>(p.bt + static_cast<long long>(lp.b) * p.bt_stride);
      soff = static_cast<uint32_t>(lp.h >> p.kv_shift);
      // the piece's page ids into L1 now: the per-stage lookups then hit L1
      // instead of adding an L2 round trip before each stage's loads
      if (lane < 2) {
        const int32_t* pp = reinterpret_cast<const int32_t*>(kcp) + (ltok >> p.page_shift) + 32 * lane;
        asm volatile("prefetch.global.L1 [%0];" :: "l"(pp));
      }
    } else {
      const uint32_t r = static_cast<uint32_t>(rowbase(lp) + ltok + g);
      const uint32_t rs = GRP ? static_cast<uint32_t>(srowbase(lp) + ltok + g) : r;
      kcp = p.kc + (r * (HD / 2) + sub * 8);
      soff = (rs * NBLK + sidx) * SB + soff_rs;
    }
    nvl = lp.t1 - ltok - g;                 // slot i of this lane holds a row iff i*G < nvl
    left = (lns - 1 - ls) / NC;             // this warp's further stages in the piece
    if (lane == 0) {
      WCur c;
      c.lp = lp;
      c.ls_last = ls + NC * left;
      c.lro = lro;
      c.lns = lns;
      *s_cur = c;
    }
    __syncwarp();
  };
  // cursor at this warp's first stage at or after (lp, ls): walks pieces
  auto seek = [&](Piece lp, int ls, int lro, int lns) -> bool {
    while (ls >= lns) {
      lro = (lro + lns) % NC;
      if (!walk_next(lp, lpi)) { lvalid = false; return false; }
      ++lpi;
      lns = nstages(lp);
      ls = warp >= lro ? warp - lro : warp + NC - lro;
    }
    set_cursor(lp, ls, lro, lns);
    return true;
  };
  // this warp's next stage
  auto advance = [&]() -> bool {
    if (!lvalid) return false;
    if (left > 0) {
      --left;
      if constexpr (PAGED) {
        ptok += NC * ST;
      } else {
        kcp += KSTEP;
        soff += SSTEP;
      }
      nvl -= NC * ST;
      return true;
    }
    const WCur c = *s_cur;
    return seek(c.lp, c.ls_last + NC, c.lro, c.lns);
  };
  // loads of the cursor's stage; rows >= t1 are not loaded (a partial stage
  // -- only a piece's last -- keeps earlier finite data in those slots, and
  // consume masks them)
  auto load_stage = [&](StageRegs& Rg, int& nv, int& pi, int dep) {
    nv = nvl;
    pi = lpi;
#ifdef NQKV_EXP_NOLOAD
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      Rg.k[i] = make_uint2(0x12345678u * (i + 1) + nv, 0x9abcdef0u + lane);
      Rg.v[i] = make_uint2(0x31415926u * (i + 3) + nv, 0x27182818u + lane);
    }
    return;
#endif
    // The loads are predicated on rows < t1, and the predicate carries `dep`
    // (always 0, but computed from the previous stage's first code word):
    // ptxas puts every global load of this loop on one scoreboard, so the
    // next stage's loads must not issue before the wait for the current
    // stage's data -- otherwise that wait would also wait for them.
    if constexpr (PAGED) {
      // The stage's ST tokens span at most two pages (P >= 64 > ST): their
      // ids are read (L1) after the wait, then each slot's row is
      // (page * H_kv + kv head) * P + t % P in [n_pages][H_kv][P] storage.
      const int32_t* btp = reinterpret_cast<const int32_t*>(kcp);
      const int ps = p.page_shift, pm = (1 << ps) - 1;
      const int hkv = p.H >> p.kv_shift;
      const int tend = ptok + min(ST, nvl + g) - 1;      // last row of the stage in the piece
      // page id of this stage: read by the previous stage's load_stage (its
      // load completed with that stage's data), else now (after the wait)
      const int pa = npa >= 0 ? npa : __ldg(btp + (ptok >> ps) + dep);
      // ... and the next stage's (same piece: `left` stages to go), issued
      // after this stage's code loads below
      auto look_ahead = [&]() {
        npa = left > 0 ? __ldg(btp + ((ptok + NC * ST) >> ps)) : -1;
      };
      if ((ptok & pm) + ST <= pm + 1) {
        // common case: the whole stage lies in one page -- slot rows are
        // consecutive there, as in the contiguous layout
        const uint32_t r0 = static_cast<uint32_t>((pa * hkv + static_cast<int>(soff)) << ps) +
                            static_cast<uint32_t>((ptok & pm) + g);
        uint32_t s0 = r0;
        if constexpr (GRP)
          s0 = static_cast<uint32_t>((pa * (hkv >> p.hpb_shift) + (static_cast<int>(soff) >> p.hpb_shift)) << ps) +
               static_cast<uint32_t>((ptok & pm) + g);
        const uint8_t* kp = p.kc + (r0 * (HD / 2) + sub * 8);
        const uint8_t* vp = p.vc + (r0 * (HD / 2) + sub * 8);
        const uint32_t so = (s0 * NBLK + sidx) * SB;
#pragma unroll
        for (int i = 0; i < kTPS; ++i) {
          if (i * G < nvl) {
            Rg.k[i] = ldg_stream_64(kp + i * G * (HD / 2));
            Rg.v[i] = ldg_stream_64(vp + i * G * (HD / 2));
            if constexpr (!RS) {
              Rg.ks[i] = ld_scale<F16S>(p.ks, so + i * G * NBLK * SB);
              Rg.vs[i] = ld_scale<F16S>(p.vs, so + i * G * NBLK * SB);
            }
          }
        }
        if constexpr (RS) {
          if ((sub & 3) * G < nvl) {
            Rg.ks[0] = ld_scale<F16S>(p.ks, so + soff_rs);
            Rg.vs[0] = ld_scale<F16S>(p.vs, so + soff_rs);
          }
        }
        look_ahead();
        return;
      }
      const int pb = __ldg(btp + (max(tend, ptok) >> ps) + dep);
      auto row_of = [&](int t) -> uint32_t {
        const int pg = ((t >> ps) == (ptok >> ps)) ? pa : pb;
        return static_cast<uint32_t>((pg * hkv + static_cast<int>(soff)) << ps) + static_cast<uint32_t>(t & pm);
      };
      auto srow_of = [&](int t) -> uint32_t {
        if constexpr (GRP) {
          const int pg = ((t >> ps) == (ptok >> ps)) ? pa : pb;
          return static_cast<uint32_t>((pg * (hkv >> p.hpb_shift) + (static_cast<int>(soff) >> p.hpb_shift)) << ps) +
                 static_cast<uint32_t>(t & pm);
        } else {
          return row_of(t);
        }
      };
#pragma unroll
      for (int i = 0; i < kTPS; ++i) {
        if (i * G < nvl) {
          const uint32_t r = row_of(ptok + g + i * G);
          Rg.k[i] = ldg_stream_64(p.kc + (r * (HD / 2) + sub * 8));
          Rg.v[i] = ldg_stream_64(p.vc + (r * (HD / 2) + sub * 8));
          if constexpr (!RS) {
            const uint32_t so = (srow_of(ptok + g + i * G) * NBLK + sidx) * SB;
            Rg.ks[i] = ld_scale<F16S>(p.ks, so);
            Rg.vs[i] = ld_scale<F16S>(p.vs, so);
          }
        }
      }
      if constexpr (RS) {
        if ((sub & 3) * G < nvl) {
          const uint32_t so = (srow_of(ptok + g + (sub & 3) * G) * NBLK + sidx) * SB;
          Rg.ks[0] = ld_scale<F16S>(p.ks, so);
          Rg.vs[0] = ld_scale<F16S>(p.vs, so);
        }
      }
      look_ahead();
      return;
    }
    const uint8_t* vcp = kcp + vdelta;
    const uint8_t* ksp = static_cast<const uint8_t*>(p.ks) + soff;
    const uint8_t* vsp = static_cast<const uint8_t*>(p.vs) + soff;
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      if (i * G + dep < nvl) {
        Rg.k[i] = ldg_stream_64(kcp + i * G * (HD / 2));
        Rg.v[i] = ldg_stream_64(vcp + i * G * (HD / 2));
        if constexpr (!RS) {
          Rg.ks[i] = ld_scale<F16S>(ksp, i * G * NBLK * SB);
          Rg.vs[i] = ld_scale<F16S>(vsp, i * G * NBLK * SB);
        }
      }
    }
    if constexpr (RS) {
      if ((sub & 3) * G + dep < nvl) {
        Rg.ks[0] = ld_scale<F16S>(ksp, 0);
        Rg.vs[0] = ld_scale<F16S>(vsp, 0);
      }
    }
#if NQKV_PF > 0
    // bulk L2 prefetch of this warp's stage NQKV_PF ahead in the piece (lane
    // 0's cursor is the stage's first row; K and V rows are contiguous)
    if (lane == 0 && left >= NQKV_PF) {
      const uint8_t* a = kcp + NQKV_PF * KSTEP;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a), "r"(ST * (HD / 2)) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a + vdelta), "r"(ST * (HD / 2)) : "memory");
    }
#endif
  };
  // two-stage register ring, unrolled as buffers A and B
  StageRegs RA, RB;
#pragma unroll
  for (int i = 0; i < kTPS; ++i) {
    RA.k[i] = RA.v[i] = RB.k[i] = RB.v[i] = make_uint2(0, 0);
    RA.ks[RS ? 0 : i] = RA.vs[RS ? 0 : i] = RB.ks[RS ? 0 : i] = RB.vs[RS ? 0 : i] = 0.0f;
  }
  int nva = 0, pia = 0, nvb = 0, pib = 0;
  bool ha = false, hb = false;
  auto fill_first = [&]() {
    if (lvalid && seek(p0, warp, 0, nstages(p0))) {
      load_stage(RA, nva, pia, 0);
      ha = true;
    }
  };
  // first stage now if it needs no walking (and the arrays are present)
  const bool early = !p.plan || warp < nstages(p0);
  if (early) fill_first();
  // per-batch arrays (plan mode): loaded now, stored to shared memory after
  // the table build, so their latency overlaps the q loads' instead of
  // stalling the builders (they are first read after the barrier below)
  int pa_len[2], pa_pref[2], pa_one = 0;
  if (p.plan) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int b = tid + i * NT;
      pa_len[i] = b < p.B ? __ldcg(p.plan + kPlanLen + b) : 0;
      pa_pref[i] = b < p.B ? __ldcg(p.plan + kPlanPref + b) : 0;   // pref[B] = N (header)
    }
    if (tid < (p.B + 31) / 32) pa_one = __ldcg(p.plan + kPlanOne + tid);
  }
  if (pre) {
#if NQKV_QPF
    // L2 prefetch of the prebuilt pieces' q rows (a hint, coherent: the
    // loads below still read after the wait; in a model the predecessor has
    // just written q, so it is L2-resident anyway)
    if (warp == 0 && lane < R0) {
      const int bh = lane == 0 ? p0.b * p.H + p0.h : lane == 1 ? pbh.x : lane == 2 ? pbh.y : pbh.z;
      asm volatile("prefetch.global.L2 [%0];" :: "l"(p.q + static_cast<long long>(bh) * HD));
      if (HD == 128)
        asm volatile("prefetch.global.L2 [%0];" :: "l"(p.q + static_cast<long long>(bh) * HD + 64));
    }
#endif
    pdl_enter();
    TRACE(1);
  }
  q0 = load_quad(p0, tid % Q);
#pragma unroll
  for (int k = 1; k < R; ++k)
    if (k < R0)
      qx[k - 1] = __ldg(reinterpret_cast<const uint4*>(p.q + static_cast<long long>(k == 1 ? pbh.x : k == 2 ? pbh.y : pbh.z) * HD) + tid % Q);
  TRACE(4);
  // ---- the table of piece 0, built by all threads (thread: pair quad
  // tid % Q); T[e][j] = RN(c q_{2j} L[e & 15]) + RN(c q_{2j+1} L[e >> 4])
  TRACE(5);
  // T[e][j] = RN(RN(c q_{2j} L[e & 15]) + RN(c q_{2j+1} L[e >> 4])), exactly
  // as build_fn rounds it (thread: pair quad tid % Q of rows e = tid / Q + ...)
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (k >= R0) break;
    __half2 h2[4];
    memcpy(h2, k == 0 ? &q0 : &qx[k > 0 ? k - 1 : 0], 16);
    float a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(h2[i]);
      a[i] = f.x * p.scale_log2;
      b[i] = f.y * p.scale_log2;
    }
    unsigned char* base = smem + Sm::kK + slot_off<HD>(k) + (tid % Q) * 16;
    for (int e = tid / Q; e < 256; e += NT / Q) {
      const float lo = s_lv[e & 15], hi = s_lv[e >> 4];
      *reinterpret_cast<float4*>(base + e * 256) =
          make_float4(__fadd_rn(__fmul_rn(a[0], lo), __fmul_rn(b[0], hi)),
                      __fadd_rn(__fmul_rn(a[1], lo), __fmul_rn(b[1], hi)),
                      __fadd_rn(__fmul_rn(a[2], lo), __fmul_rn(b[2], hi)),
                      __fadd_rn(__fmul_rn(a[3], lo), __fmul_rn(b[3], hi)));
    }
  }
  if (p.plan) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int b = tid + i * NT;
      if (b < p.B) {
        s_len[b] = pa_len[i];
        s_pref[b] = pa_pref[i];
      }
    }
    if (tid == 0) s_pref[p.B] = sc.N;
    if (tid < (p.B + 31) / 32) reinterpret_cast<uint32_t*>(smem + Sm::kOne)[tid] = pa_one;
  }
  TRACE(6);
  __syncthreads();
  TRACE(7);
  if (!early) fill_first();

  if (warp == NC) {
    // ================================================================ producer
    // appended-token state of piece k (fused step, the sequence's last piece)
    auto new_state = [&](int k, const Piece& pc) {
      float* st = s_new + (k % R) * (HD + 4);
      if (fused && pc.t1 == pc.len) {
        float vh[2 * PPL];
        const float sco = new_token_fn<HD, NW, F16S, GRP>(p, smem, pc.b, pc.h, min(pc.len, p.Tc - 1), k % R, vh);
#pragma unroll
        for (int u = 0; u < PPL; ++u)
          *reinterpret_cast<float2*>(st + 2 * (lane + 32 * u)) = make_float2(vh[2 * u], vh[2 * u + 1]);
        if (lane == 0) st[HD] = sco;
      } else if (lane == 0) {
        st[HD] = -INFINITY;
      }
    };
    Piece pc = p0;
    TRACE(3);
    if (lane == 0) s_pc[0] = pc;
#if NQKV_LATE_APPEND
    // consumers need only the table; the appended-token state is read by the
    // piece's merge (this warp, later): release them first
    __syncwarp();
    if (lane == 0) mbar_arrive(mb_full);
    new_state(0, pc);
    __syncwarp();
#else
    new_state(0, pc);
    __syncwarp();
    if (lane == 0) mbar_arrive(mb_full);
#endif
    TRACE(8);
    empties(cta, sc.C);
    Piece nx = pc;
    bool more = walk_next(nx, 0);
    uint4 qn = more ? load_quad(nx, lane % Q) : make_uint4(0, 0, 0, 0);
    int k = 0;
#ifdef NQKV_TRACE
    unsigned long long acc_w = 0, acc_m = 0, acc_b = 0, acc_n = 0;
#endif
    while (more) {
      pc = nx;
      ++k;
      const uint4 qc = qn;
      more = walk_next(nx, k);
      if (more) qn = load_quad(nx, lane % Q);
      if (k >= R) {
        {
          PT_START(t0w);
          mbar_wait_sleep(mb_done + 8 * ((k - R) % R), ((k - R) / R) & 1);
          PT_ACC(acc_w, t0w);
        }
        PT_START(t0m);
        merge_fn<HD, NW, GATHER>(p, smem, k - R, sc, cta, g0);
        PT_ACC(acc_m, t0m);
      }
      {
        PT_START(t0b);
        if (k >= R0) build_fn<HD, NW>(smem, k % R, qc, p.scale_log2);
        __syncwarp();
        PT_ACC(acc_b, t0b);
      }
      if (lane == 0) s_pc[k % R] = pc;
#if NQKV_LATE_APPEND
      __syncwarp();
      if (lane == 0) mbar_arrive(mb_full + 8 * (k % R));
#endif
      {
        PT_START(t0n);
        new_state(k, pc);
        __syncwarp();
        PT_ACC(acc_n, t0n);
      }
#if !NQKV_LATE_APPEND
      if (lane == 0) mbar_arrive(mb_full + 8 * (k % R));
#endif
    }
#ifdef NQKV_TRACE
    if (p.trace && lane == 0) {
      unsigned long long* tw = p.trace + (blockIdx.x * NW + warp) * 16;
      tw[4] = acc_w; tw[5] = acc_m; tw[13] = acc_b; tw[15] = acc_n;
    }
#endif
    TRACE(9);
    for (int j = max(0, k + 1 - R); j <= k; ++j) {
      // the last piece: try to take the last-arriver role early (after the
      // previous pieces' merges, so the partners have had time to arrive)
      if (j == k && (NQKV_PEEK > 0 || (NQKV_PEEK < 0 && HD == 128)))
        peek_fn<HD, NW>(p, smem, k, sc, cta);
      mbar_wait_sleep(mb_done + 8 * (j % R), (j / R) & 1);
      if (j == k) TRACE(11);
      merge_fn<HD, NW, GATHER>(p, smem, j, sc, cta, g0);
    }
    if constexpr (GATHER) {    // every output of this CTA was stored by this warp
      __syncwarp();
      if (lane == 0) gather_cta_done(p);
    }
    TRACE(10);
    return;
  }

  // ================================================================ consumers
  const int rho = (g + (HD == 128 ? 4 * (sub >> 2) : 0)) & 7;     // bank rotation
  uint32_t rotA = 0, rotB = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    rotA |= static_cast<uint32_t>((i + rho) & 7) << (4 * i);
    rotB |= static_cast<uint32_t>((i + 4 + rho) & 7) << (4 * i);
  }
  const uint32_t vsel = static_cast<uint32_t>(lane) * (NQKV_V16 ? 4u : 8u);

  uint32_t jsel[8];
  auto set_jsel = [&](int slot) {
    const uint32_t add = slot_off<HD>(slot);
#pragma unroll
    for (int k = 0; k < 8; ++k) jsel[k] = static_cast<uint32_t>(sub * 8 + ((k + rho) & 7)) * 4u + add;
  };

  uint64_t o2[8];
  float m = -INFINITY, l = 0.0f;
#if NQKV_V16
  float wsum = 0.0f;           // sum of this lane's V weights (the fixed-point offset)
#endif
  bool any = false;            // this warp consumed a stage of the current piece
  auto reset_state = [&]() {
#pragma unroll
    for (int j = 0; j < 8; ++j) o2[j] = 0;
    m = -INFINITY;
    l = 0.0f;
#if NQKV_V16
    wsum = 0.0f;
#endif
    any = false;
  };

  // scores, online-softmax update and the V weights of one stage ...
  auto consume_s = [&](const StageRegs& Rg, int nv, float (&wv)[kTPS]) {
    any = true;
#ifdef NQKV_EXP_NOCOMPUTE
    {
      uint32_t x = 0;
#pragma unroll
      for (int i = 0; i < kTPS; ++i)
        x ^= Rg.k[i].x ^ Rg.k[i].y ^ Rg.v[i].x ^ Rg.v[i].y ^ __float_as_uint(Rg.ks[RS ? 0 : i]) ^
             __float_as_uint(Rg.vs[RS ? 0 : i]);
      o2[0] ^= x;
      l += 1.0f;
      m = 0.0f;
#pragma unroll
      for (int i = 0; i < kTPS; ++i) wv[i] = 0.0f;
      return;
    }
#endif
    // scores (log2 domain): this lane's 16 dims via the q-table
    float s[kTPS];
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      const uint32_t r0 = prmt(Rg.k[i].x, Rg.k[i].y, rotA);
      const uint32_t r1 = prmt(Rg.k[i].x, Rg.k[i].y, rotB);
      // pairs of lookups accumulate as fp32x2
      uint64_t a = pack2(lds_k(prmt(r0, jsel[0], 0x7604)), lds_k(prmt(r0, jsel[1], 0x7614)));
      a = fadd2(a, pack2(lds_k(prmt(r0, jsel[2], 0x7624)), lds_k(prmt(r0, jsel[3], 0x7634))));
      const uint64_t b = pack2(lds_k(prmt(r1, jsel[4], 0x7604)), lds_k(prmt(r1, jsel[5], 0x7614)));
      a = fadd2(a, fadd2(b, pack2(lds_k(prmt(r1, jsel[6], 0x7624)), lds_k(prmt(r1, jsel[7], 0x7634)))));
      const float2 af = unpack2(a);
      s[i] = RS ? af.x + af.y : (af.x + af.y) * Rg.ks[i];
    }
    if constexpr (RS) {
      // reduce-scatter over the 4 lanes of the block: lane j = sub % 4 ends
      // with the block sum of slot j (xor 2 keeps the pair holding j, xor 1
      // the element), scales it, then (hd 128) adds the other block's half
      const bool b1 = (lane >> 1) & 1, b0 = lane & 1;
      const float x0 = __shfl_xor_sync(0xffffffffu, b1 ? s[0] : s[2], 2);
      const float x1 = __shfl_xor_sync(0xffffffffu, b1 ? s[1] : s[3], 2);
      const float k0 = (b1 ? s[2] : s[0]) + x0, k1 = (b1 ? s[3] : s[1]) + x1;
      float sj = (b0 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, b0 ? k0 : k1, 1);
      sj *= Rg.ks[0];
      if (LPT == 8) sj += __shfl_xor_sync(0xffffffffu, sj, 4);
      if (nv + g < ST)                // warp-uniform: only a piece's last stage is partial
        sj = ((sub & 3) * G < nv) ? sj : -INFINITY;
      // running max per token row group g (its 4 / 8 lanes share the V
      // weights, so they must share the max): 2 shuffle rounds, not 4-5;
      // groups are brought to a common max once per piece in end_piece
      float mt = sj;
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
      const bool up = mt > m;         // uniform within the group
      if (__any_sync(0xffffffffu, up)) {
        const float corr = up ? fast_exp2(m - mt) : 1.0f;   // m = -inf -> 0
        m = up ? mt : m;
        l *= corr;
#if NQKV_V16
        wsum *= corr;
#endif
        const uint64_t c2 = pack2(corr, corr);
#pragma unroll
        for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], c2);
      }
      // masked: exp2(-inf) = 0 (a group that has seen only masked slots keeps
      // m = -inf: subtract 0 there, not -inf)
      const float pr = fast_exp2(sj - (m == -INFINITY ? 0.0f : m));
      l += pr;                        // this lane's slot only (reduced in end_piece)
      const float w = pr * Rg.vs[0];
#if NQKV_V16
      wsum += w;                      // this lane's slot only (reduced in end_piece, like l)
      const float ws = w * kV16WScale;
#else
      const float ws = w;
#endif
#pragma unroll
      for (int i = 0; i < kTPS; ++i) wv[i] = __shfl_sync(0xffffffffu, ws, (lane & ~3) | i);
    } else {
#pragma unroll
      for (int o = 1; o < LPT; o <<= 1) {
#pragma unroll
        for (int i = 0; i < kTPS; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
      }
      if (nv + g < ST) {              // warp-uniform: only a piece's last stage is partial
#pragma unroll
        for (int i = 0; i < kTPS; ++i) s[i] = (i * G < nv) ? s[i] : -INFINITY;
      }
      float mt = s[0];
#pragma unroll
      for (int i = 1; i < kTPS; ++i) mt = fmaxf(mt, s[i]);
#pragma unroll
      for (int o = LPT; o < 32; o <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
      if (mt > m) {                   // warp-uniform; the stage has >= 1 valid token
        const float corr = fast_exp2(m - mt);   // m = -inf -> 0
        m = mt;
        l *= corr;
#if NQKV_V16
        wsum *= corr;
#endif
        const uint64_t c2 = pack2(corr, corr);
#pragma unroll
        for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], c2);
      }
#pragma unroll
      for (int i = 0; i < kTPS; ++i) {
        const float pr = fast_exp2(s[i] - m);   // masked: exp2(-inf) = 0
        l += pr;
        wv[i] = pr * Rg.vs[i];
#if NQKV_V16
        wsum += wv[i];
        wv[i] *= kV16WScale;
#endif
      }
    }
  };
  // ... and its P.V accumulation
  auto consume_v = [&](const StageRegs& Rg, const float (&wv)[kTPS]) {
#ifdef NQKV_EXP_NOCOMPUTE
    return;
#endif
#pragma unroll
    for (int i = 0; i < kTPS; ++i) {
      const uint64_t w2 = pack2(wv[i], wv[i]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#if NQKV_V16
        o2[k] = ffma2(lds_v16(prmt(Rg.v[i].x, vsel, 0x7604 | (k << 4))), w2, o2[k]);
        o2[4 + k] = ffma2(lds_v16(prmt(Rg.v[i].y, vsel, 0x7604 | (k << 4))), w2, o2[4 + k]);
#else
        o2[k] = ffma2(lds_v(prmt(Rg.v[i].x, vsel, 0x7604 | (k << 4))), w2, o2[k]);
        o2[4 + k] = ffma2(lds_v(prmt(Rg.v[i].y, vsel, 0x7604 | (k << 4))), w2, o2[4 + k]);
#endif
      }
    }
  };

  // end of piece k: sum the G token groups (common max), publish, arrive.
  // A warp that saw no token publishes zeros and m = -inf.
  auto end_piece = [&](int k) {
    const int slot = k % R;
    if (any) {
      if constexpr (RS) {             // l: one slot per lane (hd 128: lanes sub, sub ^ 4 alike)
#pragma unroll
        for (int o = 1; o < LPT; o <<= 1)
          if (o != 4) {
            l += __shfl_xor_sync(0xffffffffu, l, o);
#if NQKV_V16
            wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
#endif
          }
        // bring the row groups to the warp max (a group that saw no token has
        // m = -inf, l = 0, o = 0: its factor is 0)
        float M = m;
#pragma unroll
        for (int o = LPT; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float f = m == -INFINITY ? 0.0f : fast_exp2(m - M);
        l *= f;
#if NQKV_V16
        wsum *= f;
#endif
        const uint64_t f2 = pack2(f, f);
#pragma unroll
        for (int j = 0; j < 8; ++j) o2[j] = fmul2(o2[j], f2);
        m = M;
      }
#pragma unroll
      for (int o = LPT; o < 32; o <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
#if NQKV_V16
        wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
#endif
#pragma unroll
        for (int j = 0; j < 8; ++j) o2[j] = fadd2(o2[j], shfl_xor64(o2[j], o));
      }
#if NQKV_V16
      // sum_t w_t L = (sum_t w_t u_t - 32768 W) / 32767, o = 2^-49 sum_t w_t u_t
      const uint64_t sc2 = pack2(kV16Out, kV16Out), b2 = pack2(-wsum * kV16Bias, -wsum * kV16Bias);
#pragma unroll
      for (int j = 0; j < 8; ++j) o2[j] = ffma2(o2[j], sc2, b2);
#endif
    }
    if (g == 0) {
      float* dst = s_o + (slot * NC + warp) * HD + sub * kLaneDims;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = unpack2(o2[2 * j]), b2 = unpack2(o2[2 * j + 1]);
        *reinterpret_cast<float4*>(dst + 4 * j) = make_float4(a.x, a.y, b2.x, b2.y);
      }
    }
    if (lane == 0) s_ml[slot * NC + warp] = make_float2(any ? m : -INFINITY, l);
    if (k < R0) mbar_wait(mb_full + 8 * k, 0);   // phase 0 of a prebuilt slot (see open_piece)
    __syncwarp();
    if (lane == 0) mbar_arrive(mb_done + 8 * slot);
  };

  int cpi = 0;
#ifdef NQKV_TRACE
  unsigned long long waited = 0;
#endif
  auto open_piece = [&]() {
    set_jsel(cpi % R);
#ifdef NQKV_TRACE
    const unsigned long long w0 = gtimer();
#endif
    // Tables 0..R0-1 were built by the whole CTA before the __syncthreads, so
    // those pieces need no wait (the producer's arrivals can lag by ~1 us);
    // their phase 0 is consumed in end_piece(k), before this warp's done(k)
    // arrival -- phase 1 cannot complete before that (the producer waits for
    // done(k) before refilling slot k), so the parity wait is unambiguous.
    if (cpi >= R0) mbar_wait(mb_full + 8 * (cpi % R), (cpi / R) & 1);
#ifdef NQKV_TRACE
    waited += gtimer() - w0;
#endif
    reset_state();
  };
  open_piece();
  TRACE(8);
  // Buffers A and B alternate: once a stage's data has arrived (the first
  // use of its first word waits for it), the next stage's loads are issued
  // into the other buffer and stay in flight while this stage is computed.
  uint32_t zero;
#if !defined(NQKV_DEPZERO) || NQKV_DEPZERO
  zero = static_cast<uint32_t>(p.early) >> 1;   // always 0, but not a constant ptxas can fold
#else
  asm volatile("mov.u32 %0, 0;" : "=r"(zero));
#endif
  auto close_to = [&](int pi) {
    while (cpi < pi) {
      end_piece(cpi);
      ++cpi;
      open_piece();
    }
  };
  while (ha) {
    {
      const int dep = static_cast<int>(RA.k[0].x & zero);
      hb = advance();
      load_stage(RB, nvb, pib, dep);         // no next stage: re-reads the last one (unused)
      close_to(pia);
      float wv[kTPS];
      consume_s(RA, nva, wv);
      consume_v(RA, wv);
    }
    if (!hb) break;
    {
      const int dep = static_cast<int>(RB.k[0].x & zero);
      ha = advance();
      load_stage(RA, nva, pia, dep);
      close_to(pib);
      float wv[kTPS];
      consume_s(RB, nvb, wv);
      consume_v(RB, wv);
    }
    TRACE(12);
  }
  TRACE(9);
  // close the current piece and any remaining ones (no stages of this warp);
  // the number of pieces is the same for every warp
  {
    Piece cp;
    walk_first(cp);
    for (int k = 0; k < cpi; ++k) walk_next(cp, k);
    for (;;) {
      end_piece(cpi);
      if (!walk_next(cp, cpi)) break;
      ++cpi;
      open_piece();
    }
  }
  TRACE(10);
#ifdef NQKV_TRACE
  if (p.trace && lane == 0) p.trace[(blockIdx.x * NW + warp) * 16 + 15] = waited + 1;
#endif
}

// ----------------------------------------------- fused all-gather helpers
// epoch += 1 (one thread; stream-ordered before the step's gather launches)
__global__ void gather_epoch_bump_kernel(unsigned* epoch) {
  pdl_enter();
  *epoch += 1u;
}
// wait until flags[0..n) all reached *epoch (acquire, system scope): the
// gathered buffer this rank reads is then complete.  Wrap-safe: a flag that
// a faster peer has already advanced past the epoch also satisfies the wait
// (epochs compare as a 32-bit serial number).
__global__ void gather_wait_kernel(const unsigned* flags, int n, const unsigned* epoch) {
  pdl_enter();
  const unsigned e = *epoch;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
    } while (static_cast<int>(v - e) < 0);
  }
  __syncthreads();
}
// a rank with nothing to compute (B == 0 or H == 0) still publishes its epoch
// to every rank, so no peer waits for it forever
__global__ void gather_publish_kernel(unsigned* const* peer_flags, int G, int rank, unsigned epoch,
                                      const unsigned* epoch_ptr) {
  pdl_enter();
  const unsigned e = epoch_ptr ? *epoch_ptr : epoch;
  for (int r = threadIdx.x; r < G; r += blockDim.x) {
    unsigned* f = peer_flags[r] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(f), "r"(e) : "memory");
  }
}

}  // namespace nqkv
