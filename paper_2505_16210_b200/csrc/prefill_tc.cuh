// Prefill attention over the 4-bit cache on the 5th-generation tensor cores
// (tcgen05 + TMEM).  Same operation and exactness
// scheme as prefill.cuh: causal
// softmax(q . k^ / sqrt(hd)) . v^ with k^, v^ = RN32(s * L[code]) split into
// fp16 hi + lo parts, P split the same way, fp32 accumulation.
//
// CTA = 8 warps, 256 queries of one (b, h) in two sets of 128 (one tcgen05
// M = 128 accumulator each).  Per 64-key tile:
//   1. all threads dequantise the K and V tiles into shared memory (fp16 hi
//      and lo, no-swizzle canonical core-matrix layout: 8 keys x 8 dims per
//      128-byte core matrix, rows = keys) -- K serves as the K-major B operand
//      of S = Q K^T, V as the MN-major B operand of O += P V;
//   2. one thread issues S_s = Q_s K_hi^T + Q_s K_lo^T (S in TMEM, 64 columns
//      per set) and commits to an mbarrier;
//   3. every thread owns one query row = one TMEM lane (tcgen05.ld 32x32b):
//      causal mask, online softmax with a lazy reference max (O is rescaled
//      in TMEM only when the row max grows by more than 2^8), P = exp2(s - m)
//      split into hi / lo fp16 and written to shared memory (K-major A);
//   4. one thread issues O_s += P_hi V_hi + P_lo V_hi + P_hi V_lo (O in TMEM,
//      hd columns per set).
// The output rows are read from TMEM, normalised and stored (fp32).
#pragma once
#include "prefill.cuh"

namespace nqkv {

constexpr int kTcQ = 256;        // queries per CTA (2 x M = 128)
constexpr int kTcK = 64;         // keys per tile
constexpr int kTcThreads = 256;

template <int HD>
constexpr size_t prefill_tc_smem_bytes() {
  // Q (256 x HD) + K hi/lo + 2 x V hi/lo (64 x HD each) + P hi/lo (2 x 128 x 64 each) + slack
  return static_cast<size_t>(kTcQ) * HD * 2 + 6 * static_cast<size_t>(kTcK) * HD * 2 +
         2 * 2 * 128 * kTcK * 2 + 1024;
}

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // no-swizzle canonical layout, version 1 (sm_100): start, LBO, SBO in 16-byte units
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46);
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
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
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
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait_tc(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
      :: "r"(mbar), "r"(phase) : "memory");
}

template <int HD, bool F16S, bool GRP>
__global__ void __launch_bounds__(kTcThreads, 1) prefill_tc_kernel(const __grid_constant__ PrefillParams p) {
  constexpr int DG = HD / 8;                       // 8-dim groups
  constexpr uint32_t kQBytes = kTcQ * HD * 2, kTileBytes = kTcK * HD * 2, kPBytes = 128 * kTcK * 2;
  constexpr uint32_t kCols = HD == 128 ? 512 : 256;  // S: 2 x 64, O: 2 x HD (power of two)
  extern __shared__ __align__(1024) unsigned char tc_smem[];
  const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(tc_smem)) + 1023u) & ~1023u;
  unsigned char* gbase = tc_smem + (sbase - static_cast<uint32_t>(__cvta_generic_to_shared(tc_smem)));
  // layout: Q | K hi | K lo | V hi (x2) | V lo (x2) | P hi (2 sets) | P lo (2 sets)
  const uint32_t sQ = sbase, sKh = sQ + kQBytes, sKl = sKh + kTileBytes, sVh = sKl + kTileBytes,
                 sVl = sVh + 2 * kTileBytes, sPh = sVl + 2 * kTileBytes, sPl = sPh + 2 * kPBytes;
  unsigned char* gQ = gbase;
  unsigned char* gK[2] = {gbase + kQBytes, gbase + kQBytes + kTileBytes};
  unsigned char* gV[2] = {gbase + kQBytes + 2 * kTileBytes, gbase + kQBytes + 4 * kTileBytes};   // hi, lo (+ buffer)
  unsigned char* gP[2] = {gbase + kQBytes + 6 * kTileBytes, gbase + kQBytes + 6 * kTileBytes + 2 * kPBytes};
  __shared__ float s_lv[16];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar[2];      // S ready, O ready
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int set = warp >> 2, quad = warp & 3;       // accumulator set, TMEM lane quadrant
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
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
  const uint32_t mb_s = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar[0]));
  const uint32_t mb_o = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar[1]));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
                     "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem))), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb_s));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb_o));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- Q (fp16, exact) into the K-major A layout: core (row group, dim group)
  const __half* qb = p.q + (static_cast<long long>(b) * p.T) * rstride + static_cast<long long>(h) * HD;
  for (int it = tid; it < kTcQ * DG; it += kTcThreads) {     // (row group, dim group, row): row fastest
    const int j = it & 7, dg = (it >> 3) % DG, rg = (it >> 3) / DG;
    const int row = q0 + rg * 8 + j;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < len) v = *reinterpret_cast<const uint4*>(qb + row * rstride + dg * 8);
    *reinterpret_cast<uint4*>(gQ + (rg * DG + dg) * 128 + j * 16) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tS = tmem + set * kTcK;                     // this thread's set: S columns
  const uint32_t tO = tmem + 2 * kTcK + set * HD;            //                    O columns
  const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
  const int rloc = quad * 32 + lane;                          // row within the set
  const int row = q0 + set * 128 + rloc;                      // query row in the sequence
  const long long row_base = (static_cast<long long>(b) * p.H + h) * p.Tc;
  const long long srow_base = GRP ? ((static_cast<long long>(b) * p.H + h) >> p.hpb_shift) * p.Tc : row_base;
  const int nblk = GRP ? 1 : HD >> p.blk_shift;
  const int last_key = min(q0 + kTcQ, len);
  float m_ref = -INFINITY, lsum = 0.0f;
  constexpr uint32_t idS = umma_idesc_f16(128, kTcK, false);
  constexpr uint32_t idO = umma_idesc_f16(128, HD, true);
  // dequantise the K tile and V tile `buf` for keys [k0, k0 + 64).  Item =
  // one key row of one 8-dim group (16 B hi + 16 B lo); the row index within
  // the core matrix varies fastest across lanes, so a warp stores 4 whole core
  // matrices (512 contiguous bytes: no bank conflicts); each thread's items
  // load first, then convert.
  constexpr int kItems = 2 * kTcK * DG;               // (tensor, key, dim group)
  constexpr int kPer = kItems / kTcThreads;            // 8 (hd 128) / 4 (hd 64)
  auto dequant = [&](int k0, int buf) {
    uint32_t w[kPer];
    float sc[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int it = tid + u * kTcThreads;
      const int j = it & 7, dg = (it >> 3) % DG, kg = (it >> 3) / DG % (kTcK / 8), isv = it >= kItems / 2;
      const int tok = k0 + kg * 8 + j;
      w[u] = 0u;
      sc[u] = 0.0f;
      if (tok < len) {
        const uint8_t* codes = isv ? p.vc : p.kc;
        const void* scales = isv ? p.vs : p.ks;
        w[u] = *reinterpret_cast<const uint32_t*>(codes + (row_base + tok) * (HD / 2) + dg * 4);
        const long long si = GRP ? srow_base + tok : (row_base + tok) * nblk + ((dg * 8) >> p.blk_shift);
        sc[u] = F16S ? __half2float(reinterpret_cast<const __half*>(scales)[si])
                     : reinterpret_cast<const float*>(scales)[si];
      }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int it = tid + u * kTcThreads;
      const int j = it & 7, dg = (it >> 3) % DG, kg = (it >> 3) / DG % (kTcK / 8), isv = it >= kItems / 2;
      uint32_t hh[4], ll[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x0 = __fmul_rn(sc[u], s_lv[(w[u] >> (8 * e)) & 15u]);        // RN32(s * L[code])
        const float x1 = __fmul_rn(sc[u], s_lv[(w[u] >> (8 * e + 4)) & 15u]);
        split2(x0, x1, hh[e], ll[e]);
      }
      const uint32_t off = (kg * DG + dg) * 128 + j * 16;
      *reinterpret_cast<uint4*>((isv ? gV[0] + buf * kTileBytes : gK[0]) + off) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
      *reinterpret_cast<uint4*>((isv ? gV[1] + buf * kTileBytes : gK[1]) + off) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
  };
  auto issue_s = [&]() {       // S_s = Q_s K_hi^T + Q_s K_lo^T
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t a = umma_sdesc(sQ + s * (kQBytes / 2) + kk * 256, 128, DG * 128);
          umma_f16(tmem + s * kTcK, a, umma_sdesc(sKh + kk * 256, 128, DG * 128), idS, kk > 0);
          umma_f16(tmem + s * kTcK, a, umma_sdesc(sKl + kk * 256, 128, DG * 128), idS, 1u);
        }
      }
      umma_commit(mb_s);
    }
  };
  // Pipeline per tile t: softmax(t) -> issue P.V(t) -> dequantise tile t + 1
  // (K single-buffered: S(t) is complete; V double-buffered: P.V(t) reads
  // V(t) meanwhile) -> issue S(t + 1).  P and the O rescale wait for P.V(t-1).
  const int ntiles = (last_key + kTcK - 1) / kTcK;
  dequant(0, 0);
  issue_s();
  for (int tile = 0; tile < ntiles; ++tile) {
    const int k0 = tile * kTcK;
    mbar_wait_tc(mb_s, tile & 1);
    tc_fence_after();
    float sv[kTcK];
    {
      uint32_t v[32];
      tmem_ld32(tS + lane_off, v);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(v[c]);
      tmem_ld32(tS + lane_off + 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 32; ++c) sv[32 + c] = __uint_as_float(v[c]);
    }
    float mx = -INFINITY;
    if (k0 + kTcK <= q0 + 1 && k0 + kTcK <= len) {       // interior tile: every key valid for every row
#pragma unroll
      for (int c = 0; c < kTcK; ++c) {
        sv[c] *= p.scale_log2;
        mx = fmaxf(mx, sv[c]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < kTcK; ++c) {
        const int key = k0 + c;
        sv[c] = (key <= row && key < len) ? sv[c] * p.scale_log2 : -INFINITY;
        mx = fmaxf(mx, sv[c]);
      }
    }
    // lazy reference max: rescale only when the max grows by more than 2^8
    const bool grow = mx > m_ref + 8.0f;
    float corr = 1.0f;
    if (grow) {
      corr = m_ref == -INFINITY ? 0.0f : fast_exp2(m_ref - mx);
      m_ref = mx;
      lsum *= corr;
    }
    if (tile > 0) {
      mbar_wait_tc(mb_o, (tile - 1) & 1);       // P.V(t - 1) done: O stable, P free
      tc_fence_after();
    }
    if (tile > 0 && __any_sync(0xffffffffu, grow && corr != 1.0f)) {
#pragma unroll
      for (int c = 0; c < HD; c += 32) {
        uint32_t v[32];
        tmem_ld32(tO + lane_off + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * corr);
        tmem_st32(tO + lane_off + c, v);
      }
      tmem_wait_st();
    }
    const float moff = m_ref == -INFINITY ? 0.0f : m_ref;
    unsigned char* ph = gP[0] + set * kPBytes;
    unsigned char* pl = gP[1] + set * kPBytes;
#pragma unroll
    for (int kg = 0; kg < kTcK / 8; ++kg) {
      uint32_t hh[4], ll[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p0 = fast_exp2(sv[kg * 8 + 2 * e] - moff);
        const float p1 = fast_exp2(sv[kg * 8 + 2 * e + 1] - moff);
        lsum += p0 + p1;
        split2(p0, p1, hh[e], ll[e]);
      }
      const uint32_t off = ((rloc >> 3) * (kTcK / 8) + kg) * 128 + (rloc & 7) * 16;
      *reinterpret_cast<uint4*>(ph + off) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
      *reinterpret_cast<uint4*>(pl + off) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    // O_s += P_hi V_hi + P_lo V_hi + P_hi V_lo  (V buffer tile & 1)
    if (tid == 0) {
      tc_fence_after();
      const uint32_t vb = (tile & 1) * kTileBytes;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int kk = 0; kk < kTcK / 16; ++kk) {
          const uint64_t ah = umma_sdesc(sPh + s * kPBytes + kk * 256, 128, (kTcK / 8) * 128);
          const uint64_t al = umma_sdesc(sPl + s * kPBytes + kk * 256, 128, (kTcK / 8) * 128);
          const uint64_t bh = umma_sdesc(sVh + vb + kk * 2 * DG * 128, DG * 128, 128);
          const uint64_t bl = umma_sdesc(sVl + vb + kk * 2 * DG * 128, DG * 128, 128);
          const uint32_t d = tmem + 2 * kTcK + s * HD;
          umma_f16(d, ah, bh, idO, (tile > 0 || kk > 0) ? 1u : 0u);
          umma_f16(d, al, bh, idO, 1u);
          umma_f16(d, ah, bl, idO, 1u);
        }
      }
      umma_commit(mb_o);
    }
    if (tile + 1 < ntiles) {
      dequant(k0 + kTcK, (tile + 1) & 1);        // overlaps P.V(t)
      issue_s();
    }
  }
  mbar_wait_tc(mb_o, (ntiles - 1) & 1);
  tc_fence_after();
  // ---- epilogue: O / l for rows < len (0 beyond)
  const float inv = lsum > 0.0f ? 1.0f / lsum : 0.0f;
#pragma unroll
  for (int c = 0; c < HD; c += 32) {
    uint32_t v[32];
    tmem_ld32(tO + lane_off + c, v);
    tmem_wait_ld();
    if (row < p.T) {
      float* o = outb + row * rstride + c;
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(o + j) =
            row < len ? make_float4(__uint_as_float(v[j]) * inv, __uint_as_float(v[j + 1]) * inv,
                                    __uint_as_float(v[j + 2]) * inv, __uint_as_float(v[j + 3]) * inv)
                      : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(kCols));
}

}  // namespace nqkv
