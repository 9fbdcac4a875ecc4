// Prefill attention over the 4-bit cache on the 5th-generation tensor cores
// (tcgen05 + TMEM).  Same operation and exactness
// scheme as prefill.cuh: causal
// softmax(q . k^ / sqrt(hd)) . v^ with k^, v^ = RN32(s * L[code]) split into
// fp16 hi + lo parts, P split the same way, fp32 accumulation.
//
// CTA = 256 queries of one (b, h) in two sets of 128 rows (one tcgen05
// M = 128 accumulator each), warp-specialised (FlashAttention-4 style):
//   - the softmax threads (one query row each) first write their q row into
//     TMEM: Q is the TMEM A operand of S = Q K^T, so the MMAs read only K
//     from shared memory (the shared-memory port is the scarce resource:
//     an SS-mode M = 128, N = 64 MMA needs 192 B/clk of operand reads);
//   - dequantisation warps fill a 3-stage ring of K and V tiles (64 keys) in
//     shared memory: fp16 hi and lo, no-swizzle canonical core-matrix
//     layout (8 keys x 8 dims per 128-byte core matrix).  K is the K-major
//     B operand of S = Q K^T, V the MN-major B operand of P V;
//   - one thread issues the MMAs, the two row sets ping-ponging:
//     P.V_0(t), S_0(t+1), P.V_1(t), S_1(t+1), ... with
//     S_s = Q_s K_hi^T + Q_s K_lo^T and O_s += P_hi V_hi + P_lo V_hi + P_hi V_lo,
//     so the tensor cores work on one set while the other set's softmax runs;
//   - 8 softmax warps (4 per set), one query row per thread (= TMEM lane,
//     tcgen05.ld 32x32b): causal mask, online softmax with a lazy reference
//     max (O is rescaled in TMEM only when the row max grows by more than
//     2^8), P = exp2(s - m) split into hi / lo fp16 and written over the
//     row's S columns (tcgen05.st) as the TMEM A operand of P V.
// TMEM (512 columns): O_s at s * HD, S/P_s at 2 HD + 64 s, Q_s after them.
// S_s(t) is issued after P.V_s(t - 1) and MMAs complete in issue order, so
// "S_s(t) complete" also means O_s is stable and P_s(t - 1) consumed.
// Hand-offs are mbarriers (K/V full/empty, S full, P full, all done).  The
// output rows are read from TMEM, normalised and stored (fp32).
#pragma once
#include "prefill.cuh"

namespace nqkv {
#ifndef NQKV_PF_WARP_ISSUE
#define NQKV_PF_WARP_ISSUE 0       // 1: whole-warp MMA issue with elect.sync (measured: see DESIGN 6.4)
#endif
#ifndef NQKV_PF_MMAW
#define NQKV_PF_MMAW 1             // MMA-issuing warps: 1 (both row sets) or 2 (one per row set; measured slower)
#endif
#ifdef NQKV_PF_TRACE
__device__ unsigned* g_pf_trace;     // development builds: see PF_TR below
#endif

constexpr int kTcQ = 256;        // queries per CTA (2 x M = 128)
constexpr int kTcK = 64;         // keys per tile
constexpr int kTcSoftW = 8;      // softmax warps (4 per row set)
constexpr int kTcStages = 3;     // K/V ring depth
#ifndef NQKV_PF_DQW
#define NQKV_PF_DQW (8 - NQKV_PF_MMAW)
#endif
constexpr int kTcDqW = NQKV_PF_DQW;   // dequantisation warps
constexpr int kTcMmaW = NQKV_PF_MMAW;
constexpr int kTcThreads = (kTcSoftW + kTcDqW + kTcMmaW) * 32;   // + the MMA warp(s)

template <int HD>
constexpr size_t prefill_tc_smem_bytes() {
  // 3 stages x (K hi/lo + V hi/lo) (64 x HD fp16 each) + alignment slack
  return static_cast<size_t>(kTcStages) * 4 * kTcK * HD * 2 + 1024;
}

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // no-swizzle canonical layout, version 1 (sm_100): start, LBO, SBO in 16-byte units
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46);
}
// start-address field += v (16-byte units); opaque to the compiler so the
// descriptor stays one register pair advanced by one add per k-step
__device__ __forceinline__ uint64_t desc_add(uint64_t d, uint32_t v) {
  uint64_t r;
  asm volatile("add.u64 %0, %1, %2;" : "=l"(r) : "l"(d), "l"(static_cast<uint64_t>(v)));
  return r;
}
// kind::f16 instruction descriptor: fp16 A/B, fp32 D, A K-major, B K- or MN-major
__host__ __device__ constexpr uint32_t umma_idesc_f16(int m, int n, bool b_mn) {
  return (1u << 4) | (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// A operand in TMEM (row m at lane m, two fp16 per 32-bit column, even element low)
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
      :: "r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
}
// Warp-wide issue (NQKV_PF_WARP_ISSUE): the whole MMA warp runs the issue
// loop with warp-uniform operands and ONE elected lane issues each
// instruction.  Issued from a single thread (lane == 0), the compiler wraps
// every tcgen05.mma in an elect / R2UR / BRA.U.ANY loop (its operands live
// in uniform registers), ~8 instructions per MMA.
__device__ __forceinline__ void umma_f16_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
      :: "r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_w(uint32_t mbar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
               :: "r"(mbar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait_tc(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
      :: "r"(mbar), "r"(phase) : "memory");
}
// the same with a suspend-time hint: a waiting warp sleeps instead of
// spinning (its retries would take issue slots from the other roles)
__device__ __forceinline__ void mbar_wait_tc_sleep(uint32_t mbar, uint32_t phase) {
#ifdef NQKV_PF_TRACE
  for (;;) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(mbar), "r"(phase) : "memory");
    if (ok) return;
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0 && g_pf_trace) {
      uint64_t st;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(st) : "r"(mbar));
      *reinterpret_cast<volatile unsigned*>(g_pf_trace + (threadIdx.x >> 5) * 4 + 3) = static_cast<unsigned>(st >> 32);
      *reinterpret_cast<volatile unsigned*>(g_pf_trace + 64 + (threadIdx.x >> 5) * 2) = static_cast<unsigned>(st);
      *reinterpret_cast<volatile unsigned*>(g_pf_trace + 65 + (threadIdx.x >> 5) * 2) = mbar;
    }
  }
#endif
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n@!p bra W_%=;\n}\n"
      :: "r"(mbar), "r"(phase) : "memory");
}
// (hi, lo) fp16 split of an fp32 pair: hi = RN16(x), lo = RN16(x - hi), with
// x - hi (exact in fp32) from the mixed-precision FMA hi * -1 + x
__device__ __forceinline__ void split2_tc(uint64_t xy, uint32_t& hi, uint32_t& lo) {
  asm("{\n.reg .b16 h0, h1, m1;\n.reg .f32 x, y, r0, r1;\n"
      "mov.b64 {x, y}, %2;\n"
      "cvt.rn.f16x2.f32 %0, y, x;\n"
      "mov.b32 {h0, h1}, %0;\n"
      "mov.b16 m1, 0xBC00;\n"
      "fma.rn.f32.f16 r0, h0, m1, x;\n"
      "fma.rn.f32.f16 r1, h1, m1, y;\n"
      "cvt.rn.f16x2.f32 %1, r1, r0;\n}"
      : "=r"(hi), "=r"(lo) : "l"(xy));
}
__device__ __forceinline__ uint64_t fadd2_tc(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void mbar_arrive_tc(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
}

#ifdef NQKV_PF_TRACE
// development: progress of CTA (0, 0, 0)'s warps in mapped host memory, readable while it runs
#define PF_TR(slot, val)                                                                 \
  do {                                                                                   \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0 && g_pf_trace) { \
      *reinterpret_cast<volatile unsigned*>(g_pf_trace + (threadIdx.x >> 5) * 4 + (slot)) = (val); \
      __threadfence_system();                                                            \
    }                                                                                    \
  } while (0)
#else
#define PF_TR(slot, val) do { } while (0)
#endif

template <int HD, bool F16S, bool GRP>
__global__ void __launch_bounds__(kTcThreads, 1) prefill_tc_kernel(const __grid_constant__ PrefillParams p) {
  constexpr int DG = HD / 8;                       // 8-dim groups
  constexpr uint32_t kTileBytes = kTcK * HD * 2, kStageBytes = 4 * kTileBytes;   // K hi, K lo, V hi, V lo
  constexpr uint32_t kCols = 512;
  constexpr uint32_t kSP = 2 * HD;                 // TMEM: O_s at s * HD, S/P_s at kSP + 64 s, Q_s at kQc + HD/2 s
  constexpr uint32_t kQc = kSP + 2 * kTcK;
  static_assert(kQc + HD <= kCols, "TMEM columns");
  extern __shared__ __align__(1024) unsigned char tc_smem[];
  const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(tc_smem)) + 1023u) & ~1023u;
  unsigned char* gbase = tc_smem + (sbase - static_cast<uint32_t>(__cvta_generic_to_shared(tc_smem)));
  __shared__ float s_lv[16];                       // the levels: 16 words in 16 banks (no conflicts)
  __shared__ uint32_t s_tmem;
  // [0,3) K full, [3,6) K empty, [6,9) V full, [9,12) V empty, 12-13 S full, 14-15 P full, 16 all MMAs done
  constexpr int kBars = 17;
  __shared__ __align__(8) uint64_t s_bar[kBars];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qt = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);   // longest causal rows first
  const int h = blockIdx.y, b = blockIdx.z;
  if (tid < 16) s_lv[tid] = p.lv.v[tid];
  pdl_enter();
  const int len = min(max(p.seq_lens[b], 0), p.T);
  const int q0 = qt * kTcQ;
  const long long rstride = static_cast<long long>(p.H) * HD;
  float* outb = p.out + (static_cast<long long>(b) * p.T) * rstride + static_cast<long long>(h) * HD;
  if (q0 >= len) {
    for (int i = tid; i < kTcQ * HD; i += kTcThreads) {
      const int r = q0 + i / HD;
      if (r < p.T) outb[r * rstride + (i % HD)] = 0.0f;
    }
    return;
  }
  const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar[0]));
  auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
                     "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem))), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < kBars; ++i) {
      const bool dq = i < 3 || (i >= 6 && i < 9);      // arrivals of every dequantisation thread
      const bool sm = i == 14 || i == 15;                // of the 128 threads of a row set
      // K/V-empty (3-5, 9-11) and all-done (16): one commit per MMA warp
      const bool mw = (i >= 3 && i < 6) || (i >= 9 && i < 12) || i == 16;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar(i)),
                   "r"(dq ? kTcDqW * 32 : sm ? 128 : mw ? kTcMmaW : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const int last_key = min(q0 + kTcQ, len);
  const int ntiles = (last_key + kTcK - 1) / kTcK;
  if (warp < kTcSoftW) {
    // ================= softmax: one query row per thread
    const int set = warp >> 2, quad = warp & 3;       // row set, TMEM lane quadrant
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int row = q0 + set * 128 + quad * 32 + lane;
    const uint32_t tO = tmem + set * HD + lane_off;
    const uint32_t tS = tmem + kSP + set * kTcK + lane_off;
    // ---- the q row (fp16, exact) into TMEM: the A operand of S (two fp16 per column)
    {
      const __half* qr = p.q + (static_cast<long long>(b) * p.T + min(row, p.T - 1)) * rstride +
                         static_cast<long long>(h) * HD;
      const uint32_t tQ = tmem + kQc + set * (HD / 2) + lane_off;
#pragma unroll
      for (int c = 0; c < HD / 2; c += 16) {
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          uint4 w = make_uint4(0u, 0u, 0u, 0u);
          if (row < len) w = *reinterpret_cast<const uint4*>(qr + 2 * (c + i));
          v[i] = w.x; v[i + 1] = w.y; v[i + 2] = w.z; v[i + 3] = w.w;
        }
        tmem_st16(tQ + c, v);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_tc(bar(14 + set));                 // P-full phase 0 doubles as "Q written"
    }
    const bool pos_scale = p.scale_log2 >= 0.0f;
    float m_ref = -INFINITY;
    uint64_t lsum = pack2(0.0f, 0.0f);               // two partial sums
    for (int t = 0; t < ntiles; ++t) {
      const int k0 = t * kTcK;
      PF_TR(0, (0x1u << 12) | (set << 8) | t);
      mbar_wait_tc_sleep(bar(12 + set), t & 1);      // S_s(t) done: also P.V_s(t - 1) (issue order)
      PF_TR(1, (0x1u << 12) | (set << 8) | t);
      tc_fence_after();
      float sv[kTcK];
      {
        uint32_t v[32];
        tmem_ld32(tS, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(v[c]);
        tmem_ld32(tS + 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[32 + c] = __uint_as_float(v[c]);
      }
      // masked max of the raw scores (scale_log2 >= 0; a negative scale takes the min)
      const bool interior = k0 + kTcK <= q0 + 1 && k0 + kTcK <= len;   // every key valid for every row
      if (!interior) {
#pragma unroll
        for (int c = 0; c < kTcK; ++c) {
          const int key = k0 + c;
          if (!(key <= row && key < len)) sv[c] = pos_scale ? -INFINITY : INFINITY;
        }
      }
      float mx = pos_scale ? -INFINITY : INFINITY;
      if (pos_scale) {
#pragma unroll
        for (int c = 0; c < kTcK; ++c) mx = fmaxf(mx, sv[c]);
      } else {
#pragma unroll
        for (int c = 0; c < kTcK; ++c) mx = fminf(mx, sv[c]);
      }
      mx = fabsf(mx) == INFINITY ? -INFINITY : mx * p.scale_log2;
      // lazy reference max: rescale only when the max grows by more than 2^8
      const bool grow = mx > m_ref + 8.0f;
      float corr = 1.0f;
      if (grow) {
        corr = m_ref == -INFINITY ? 0.0f : fast_exp2(m_ref - mx);
        m_ref = mx;
        lsum = fmul2(lsum, pack2(corr, corr));
      }
      if (t > 0 && __any_sync(0xffffffffu, grow && corr != 1.0f)) {   // O_s is stable: see above
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t v[32];
          tmem_ld32(tO + c, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
          tmem_st32(tO + c, v);
        }
      }
      const float moff = m_ref == -INFINITY ? 0.0f : m_ref;
      const uint64_t sc2 = pack2(p.scale_log2, p.scale_log2), mo2 = pack2(-moff, -moff);
      // P over the row's S columns: hi at [0, 32), lo at [32, 64) (key 2c, 2c+1 in column c)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t hh[16], ll[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = unpack2(ffma2(pack2(sv[hf * 32 + 2 * e], sv[hf * 32 + 2 * e + 1]), sc2, mo2));
          const uint64_t pp = pack2(fast_exp2(x.x), fast_exp2(x.y));
          lsum = fadd2_tc(lsum, pp);
          split2_tc(pp, hh[e], ll[e]);
        }
        tmem_st16(tS + hf * 16, hh);
        tmem_st16(tS + 32 + hf * 16, ll);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_tc(bar(14 + set));                 // P-full phase t + 1
      PF_TR(2, (0x3u << 12) | (set << 8) | t);
    }
    PF_TR(0, (0x4u << 12) | (set << 8));
    mbar_wait_tc_sleep(bar(16), 0);                  // every MMA done (completes once)
    PF_TR(1, (0x4u << 12) | (set << 8));
    tc_fence_after();
    // ---- epilogue: O / l for rows < len (0 beyond)
    const float2 l2 = unpack2(lsum);
    const float lsum1 = l2.x + l2.y;
    const float inv = lsum1 > 0.0f ? 1.0f / lsum1 : 0.0f;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t v[32];
      tmem_ld32(tO + c, v);
      tmem_wait_ld();
      if (row < p.T) {
        float* o = outb + row * rstride + c;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(o + i) =
              row < len ? make_float4(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv,
                                      __uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv)
                        : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    }
  } else if (warp < kTcSoftW + kTcDqW) {
    // ================= dequantisation: K(t), V(t) into ring stage t % 3
    const int dt = tid - kTcSoftW * 32;
    const int hkv = p.H >> p.kv_shift, kvh = h >> p.kv_shift;
    const long long row_base = (static_cast<long long>(b) * hkv + kvh) * p.Tc;
    const long long srow_base = GRP ? ((static_cast<long long>(b) * hkv + kvh) >> p.hpb_shift) * p.Tc : row_base;
    const int nblk = GRP ? 1 : HD >> p.blk_shift;
    // Item = 32 dims (16 code bytes, one scale: blk >= 32) of one key; the
    // key's row within the core matrix varies fastest across lanes, so a warp
    // loads 512 contiguous bytes of codes and each 16-byte store instruction
    // writes 4 whole core matrices.  K(t) and V(t) codes load together.
    constexpr int kQuads = HD / 32;
    constexpr int kItems = kTcK * kQuads;
    constexpr int kPer = (kItems + kTcDqW * 32 - 1) / (kTcDqW * 32);   // 2 (hd 128) / 1 (hd 64) at 4 warps
    int key[kPer], soff[kPer];
    uint32_t coff[kPer], doff[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int it = dt + u * kTcDqW * 32;
      const int j = it & 7, q = (it >> 3) % kQuads, kg = (it >> 3) / kQuads;
      key[u] = it < kItems ? kg * 8 + j : (1 << 29);     // no such item: never loaded or stored
      coff[u] = static_cast<uint32_t>(key[u] * (HD / 2) + q * 16);
      doff[u] = static_cast<uint32_t>((kg * DG + 4 * q) * 128 + j * 16);
      soff[u] = GRP ? key[u] : key[u] * nblk + ((q * 32) >> p.blk_shift);
    }
    struct Raw {
      uint4 w[kPer];
      float s[kPer];
    };
    auto load = [&](const uint8_t* codes, const void* scales, int k0, Raw& r, int dep) {
      long long rb = row_base + k0, srb = srow_base + k0;
      if (p.bt && k0 < len) {     // paged (R17): a 64-key tile lies in one page (P >= 64)
        const long long pg = __ldg(p.bt + static_cast<long long>(b) * p.bt_stride + (k0 >> p.page_shift));
        const int within = k0 & ((1 << p.page_shift) - 1);
        rb = ((pg * hkv + kvh) << p.page_shift) + within;
        srb = GRP ? ((pg * (hkv >> p.hpb_shift) + (kvh >> p.hpb_shift)) << p.page_shift) + within : rb;
      }
      const uint8_t* cb = codes + rb * (HD / 2);
      const long long sb = GRP ? srb : rb * nblk;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        r.w[u] = make_uint4(0u, 0u, 0u, 0u);
        r.s[u] = 0.0f;
        if (k0 + key[u] + dep < len) {
          r.w[u] = *reinterpret_cast<const uint4*>(cb + coff[u]);
          r.s[u] = F16S ? __half2float(reinterpret_cast<const __half*>(scales)[sb + soff[u]])
                        : reinterpret_cast<const float*>(scales)[sb + soff[u]];
        }
      }
    };
    auto convert = [&](const Raw& r, unsigned char* dhi) {
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        if (kItems % (kTcDqW * 32) != 0 && key[u] >= kTcK) continue;
        const uint64_t s2 = pack2(r.s[u], r.s[u]);
        const uint32_t ww[4] = {r.w[u].x, r.w[u].y, r.w[u].z, r.w[u].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {                  // dim group 4q + i
          uint32_t hh[4], ll[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)                  // RN32(s * L[code]) for dims 8i + 2e, + 1
            split2_tc(fmul2(s2, pack2(s_lv[(ww[i] >> (8 * e)) & 15u], s_lv[(ww[i] >> (8 * e + 4)) & 15u])),
                      hh[e], ll[e]);
          *reinterpret_cast<uint4*>(dhi + doff[u] + i * 128) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
          *reinterpret_cast<uint4*>(dhi + kTileBytes + doff[u] + i * 128) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    };
    // Tile t + 1's loads are issued once tile t's data has arrived (their
    // predicate carries `dep`, 0 computed from tile t's first code word):
    // ptxas keeps all these loads on one scoreboard, so loads issued earlier
    // would make the wait for tile t's data also wait for them.
    uint32_t zero;
#if !defined(NQKV_PDEPZERO) || NQKV_PDEPZERO
    zero = static_cast<uint32_t>(p.hpb_shift) >> 8;   // always 0, but not a constant ptxas can fold
#else
    asm volatile("mov.u32 %0, 0;" : "=r"(zero));
#endif
    Raw rk, rv;
    load(p.kc, p.ks, 0, rk, 0);
    load(p.vc, p.vs, 0, rv, 0);
    for (int t = 0; t < ntiles; ++t) {
      const int st = t % kTcStages;
      const uint32_t ph = ((t / kTcStages) & 1) ^ 1;   // a fresh barrier passes parity 1
      const int dep = static_cast<int>(rk.w[0].x & zero);
      Raw nk, nv;
      const int kn = t + 1 < ntiles ? (t + 1) * kTcK : len;   // past the end: no loads
      load(p.kc, p.ks, kn, nk, dep);
      load(p.vc, p.vs, kn, nv, dep);
      unsigned char* stg = gbase + st * kStageBytes;
      PF_TR(0, (0x5u << 12) | t);
      mbar_wait_tc_sleep(bar(3 + st), ph);
      convert(rk, stg);
      mbar_arrive_tc(bar(0 + st));
      PF_TR(0, (0x6u << 12) | t);
      mbar_wait_tc_sleep(bar(9 + st), ph);
      convert(rv, stg + 2 * kTileBytes);
      mbar_arrive_tc(bar(6 + st));
      PF_TR(1, (0x7u << 12) | t);
      rk = nk;
      rv = nv;
    }
#if NQKV_PF_WARP_ISSUE
  } else {
    // ================= MMA issue (the whole warp; one elected lane per instruction)
#define umma_f16_ts umma_f16_ts_w
#define umma_commit umma_commit_w
    // One CTA per SM allocating all 512 columns: the allocation starts at
    // column 0.  A compile-time base keeps every MMA operand warp-uniform
    // (uniform registers, no per-instruction elect loop).
    if (tmem != 0u) __trap();
    constexpr uint32_t tmem_u = 0u;
#define tmem tmem_u
#else
  } else if (lane == 0) {
    // ================= MMA issue (one thread)
#endif
    constexpr uint32_t idS = umma_idesc_f16(128, kTcK, false);
    constexpr uint32_t idO = umma_idesc_f16(128, HD, true);
    auto issue_s = [&](int s, int t) {  // S_s(t) = Q_s K_hi^T + Q_s K_lo^T
      const uint32_t kh = sbase + (t % kTcStages) * kStageBytes, kl = kh + kTileBytes;
      const uint32_t d = tmem + kSP + s * kTcK, a = tmem + kQc + s * (HD / 2);
      // descriptors built once per tile; a k-step advances the start address
      // field (bits 0-13, 16-byte units; smem addresses < 2^18 never carry out)
      const uint64_t dh = umma_sdesc(kh, 128, DG * 128), dl = umma_sdesc(kl, 128, DG * 128);
      uint64_t dhk = dh, dlk = dl;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        umma_f16_ts(d, a + kk * 8, dhk, idS, kk > 0);
        umma_f16_ts(d, a + kk * 8, dlk, idS, 1u);
        dhk = desc_add(dhk, 16u);
        dlk = desc_add(dlk, 16u);
      }
      umma_commit(bar(12 + s));
    };
    auto issue_pv = [&](int s, int t) { // O_s += P_hi V_hi + P_lo V_hi + P_hi V_lo
      const uint32_t vh = sbase + (t % kTcStages) * kStageBytes + 2 * kTileBytes, vl = vh + kTileBytes;
      const uint32_t ph = tmem + kSP + s * kTcK, pl = ph + 32, d = tmem + s * HD;
      const uint64_t bh0 = umma_sdesc(vh, DG * 128, 128), bl0 = umma_sdesc(vl, DG * 128, 128);
#pragma unroll
      for (int kk = 0; kk < kTcK / 16; ++kk) {
        const uint64_t bh = kk ? desc_add(bh0, static_cast<uint32_t>(kk * 2 * DG * 8)) : bh0;   // + kk * 2 * DG * 128 B
        const uint64_t bl = kk ? desc_add(bl0, static_cast<uint32_t>(kk * 2 * DG * 8)) : bl0;
        umma_f16_ts(d, ph + kk * 8, bh, idO, (t > 0 || kk > 0) ? 1u : 0u);
        umma_f16_ts(d, pl + kk * 8, bh, idO, 1u);
        umma_f16_ts(d, ph + kk * 8, bl, idO, 1u);
      }
    };
    auto wait_k = [&](int t) {
      PF_TR(0, (0x8u << 12) | t);
      mbar_wait_tc(bar(0 + t % kTcStages), (t / kTcStages) & 1);
      tc_fence_after();
    };
#if NQKV_PF_MMAW == 2
    // one MMA warp per row set: the two sets' MMAs are issued concurrently
    // (per-thread commits track only the issuing thread's MMAs; a K/V stage
    // is free once BOTH warps committed it: count-2 barriers)
    const int s = warp - (kTcSoftW + kTcDqW);
    mbar_wait_tc(bar(14 + s), 0);        // Q_s rows written (P-full phase 0)
    wait_k(0);
    issue_s(s, 0);
    umma_commit(bar(3 + 0));
    for (int t = 0; t < ntiles; ++t) {
      mbar_wait_tc(bar(6 + t % kTcStages), (t / kTcStages) & 1);      // V(t)
      const bool more = t + 1 < ntiles;
      mbar_wait_tc(bar(14 + s), (t + 1) & 1);    // P_s(t): phase t + 1 (phase 0 = Q)
      tc_fence_after();
      issue_pv(s, t);
      if (more) {
        wait_k(t + 1);
        issue_s(s, t + 1);
      }
      umma_commit(bar(9 + t % kTcStages));        // V stage free (this warp's share)
      if (more) umma_commit(bar(3 + (t + 1) % kTcStages));   // K stage free (this warp's share)
    }
    umma_commit(bar(16));
#else
    // Q rows written (P-full phase 0 of both sets)
    mbar_wait_tc(bar(14), 0);
    mbar_wait_tc(bar(15), 0);
    wait_k(0);
    issue_s(0, 0);
    issue_s(1, 0);
    umma_commit(bar(3 + 0));             // K stage 0 free once both S are done
    for (int t = 0; t < ntiles; ++t) {
      PF_TR(0, (0x9u << 12) | t);
      mbar_wait_tc(bar(6 + t % kTcStages), (t / kTcStages) & 1);      // V(t)
      const bool more = t + 1 < ntiles;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        PF_TR(0, (0xAu << 12) | (s << 8) | t);
        mbar_wait_tc(bar(14 + s), (t + 1) & 1);    // P_s(t): phase t + 1 (phase 0 = Q)
        PF_TR(1, (0xAu << 12) | (s << 8) | t);
        tc_fence_after();
        issue_pv(s, t);
        if (more) {
          if (s == 0) wait_k(t + 1);
          issue_s(s, t + 1);
        }
      }
      umma_commit(bar(9 + t % kTcStages));        // V stage free
      if (more) umma_commit(bar(3 + (t + 1) % kTcStages));   // K stage free
    }
    umma_commit(bar(16));
#endif
  }
#if NQKV_PF_WARP_ISSUE
#undef umma_f16_ts
#undef umma_commit
#undef tmem
#endif
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(kCols));
}

}  // namespace nqkv
