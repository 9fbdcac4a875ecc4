// Grouped-query decode attention (reading R16):
// one CTA streams a chunk of ONE KV head's cache once for GN (2 or 4) query
// heads of its group, instead of once per query head.
//
// Paper: PAPER.md:229-235 (dequantise the cached indices, Softmax(t_Q X_K'^T),
// A X_V'), per query head; grouped-query attention only changes which cache
// head a query head reads (R16).  The arithmetic is the MHA kernel's: k^ and
// v^ are s * L[code] with fp32 levels, scores (q . k^) / sqrt(hd) in fp32,
// online softmax, fp32 P.V; only the summation order differs.
//
// Why a separate kernel: the MHA kernel (decode.cuh) folds q into a per-(b, h)
// byte table (one 4-byte lookup per code byte) -- a table per QUERY head, so
// a GQA group would need g tables (g x 64 KB at hd 128).  Here the lookup is
// query-independent: a lane-replicated fp32 pair LUT P[byte] = (L[lo], L[hi])
// (one 8-byte lookup per code byte) feeds GN packed FMAs, one per query head,
// for K (q pairs held in registers) and for V (the GN softmax weights).  Per
// code byte: PRMT + LDS.64 + GN x FFMA2 on each of K and V, shared by GN
// query heads.
//
// Work: item = (b, kv head, query sub-group, chunk c of nc); the chunk is
// [len*c/nc, len*(c+1)/nc) of the sequence's tokens.  Lane (sl, r) owns dims
// [8 sl, 8 sl + 8) (one 32-bit code word) of token row r; a stage is S slots
// x 32/(hd/8) consecutive tokens, stages go round-robin to the CTA's warps.
// Warps merge in shared memory; chunks merge in the last-arriving CTA (per
// group arrival counter), in chunk order -- results depend on (B, H, seq_lens,
// nc) only.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace nqkv {

#ifndef NQKV_GQA_WARPS
#define NQKV_GQA_WARPS 4
#endif
#ifndef NQKV_GQA_CTAS
#define NQKV_GQA_CTAS 3
#endif
constexpr int kGqaWarps = NQKV_GQA_WARPS;      // per CTA (4 x 3 CTAs per SM: 170 registers per thread)
constexpr int kGqaCtasPerSm = NQKV_GQA_CTAS;
constexpr int kGqaSlots = 4;        // token slots per lane per stage
constexpr int kGqaMaxChunkCap = 64;          // chunks per (b, kv head, sub-group)
constexpr long long kGqaMaxRecords = 16384;  // partial records (hd + 2 floats) in the workspace
constexpr uint32_t kGqaLut = 256 * 32 * 8;   // pair LUT bytes (32 lane copies)

template <int HD, int GN>
constexpr size_t gqa_smem_bytes() {
  return kGqaLut + static_cast<size_t>(kGqaWarps) * GN * (2 + HD) * 4 + 16;
}

struct GqaParams {
  const __half* q;           // [B][H][hd]
  const uint8_t* kc;         // [B][Hkv][Tc][hd/2]
  const void* ks;            // [B][Hkv][Tc][hd/blk] fp32, or fp16 (gqa_tc_kernel template F16S)
  const uint8_t* vc;
  const void* vs;
  const int32_t* seq_lens;   // [B]
  float* out;                // [B][H][hd]
  int* cnt;                  // [B*H] arrival counters (zero between launches)
  float* part;               // [records][hd + 2] chunk partials (o[hd], m, l)
  int B, H, Hkv, Tc, nsg, nc, kv_shift, blk_shift;
  const int32_t* bt;         // paged cache (template PAGED): block table [B][bt_stride]
  int bt_stride, page_shift; // token t of sequence b: page bt[b][t >> page_shift], row t & (P - 1)
  float scale_log2;          // softmax_scale * log2(e)
  int zero;                  // always 0: the load-order dependency (a parameter, not foldable)
  Levels lv;
};

__device__ __forceinline__ uint64_t gqa_lds_pair(uint32_t off) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1+0x400];" : "=l"(v) : "r"(off));   // LUT at dynamic smem 0
  return v;
}
__device__ __forceinline__ uint32_t gqa_prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
// predicated 32-bit streaming load (0 when off: no branch)
__device__ __forceinline__ uint32_t gqa_ld32p(const void* p, bool on) {
  uint32_t r;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b32 %0, 0;\n"
               " @q ld.global.nc.L1::no_allocate.u32 %0, [%1];\n}"
               : "=r"(r) : "l"(p), "r"(static_cast<int>(on)));
  return r;
}
__device__ __forceinline__ float gqa_exp2_or_zero(float m, float M) {   // 2^(m - M), 0 for m = -inf
  return m == -INFINITY ? 0.0f : fast_exp2(m - M);
}

// CTA merge of the warps' states (s_m/s_l [NW][GN], s_o [NW][GN][HD], fixed
// order), then either the output (nc = 1) or the chunk partial; the last
// CTA of the group to arrive merges the nc partials in chunk order, writes
// the output, and zeroes the partials and the counter.
template <int HD, int GN, int NW>
__device__ __forceinline__ void gqa_epilogue(const GqaParams& p, const float* s_m, const float* s_l,
                                             const float* s_o, int& s_last, int grp, int c, int b,
                                             int h0) {
  const int tid = threadIdx.x;
  const int nthr = NW * 32;
  float* part_grp = p.part + static_cast<size_t>(grp) * p.nc * GN * (HD + 2);
  for (int x = tid; x < GN * HD; x += nthr) {
    const int qi = x / HD, d = x - qi * HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w * GN + qi]);
    float O = 0.0f, L = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float f = gqa_exp2_or_zero(s_m[w * GN + qi], M);
      O += f * s_o[(w * GN + qi) * HD + d];
      L += f * s_l[w * GN + qi];
    }
    if (p.nc == 1) {
      p.out[(static_cast<size_t>(b) * p.H + h0 + qi) * HD + d] = L > 0.0f ? O / L : 0.0f;
    } else {
      float* rec = part_grp + (static_cast<size_t>(c) * GN + qi) * (HD + 2);
      rec[d] = O;
      if (d == 0) {
        rec[HD] = M;
        rec[HD + 1] = L;
      }
    }
  }
  if (p.nc == 1) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int prev = atomicAdd(p.cnt + grp, 1);
    s_last = prev == p.nc - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int x = tid; x < GN * HD; x += nthr) {
    const int qi = x / HD, d = x - qi * HD;
    float M = -INFINITY;
    for (int cc = 0; cc < p.nc; ++cc)
      M = fmaxf(M, __ldcg(part_grp + (static_cast<size_t>(cc) * GN + qi) * (HD + 2) + HD));
    float O = 0.0f, L = 0.0f;
    for (int cc = 0; cc < p.nc; ++cc) {
      const float* rec = part_grp + (static_cast<size_t>(cc) * GN + qi) * (HD + 2);
      const float f = gqa_exp2_or_zero(__ldcg(rec + HD), M);
      O += f * __ldcg(rec + d);
      L += f * __ldcg(rec + HD + 1);
    }
    p.out[(static_cast<size_t>(b) * p.H + h0 + qi) * HD + d] = L > 0.0f ? O / L : 0.0f;
  }
  // leave the workspace zero (the library's workspace contract)
  __syncthreads();
  const int nrec = p.nc * GN * (HD + 2);
  for (int x = tid; x < nrec; x += nthr) part_grp[x] = 0.0f;
  if (tid == 0) p.cnt[grp] = 0;
}

__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

template <int HD, int GN, bool PAGED>
__global__ void __launch_bounds__(kGqaWarps * 32, kGqaCtasPerSm)
gqa_decode_kernel(const __grid_constant__ GqaParams p) {
  constexpr int LPT = HD / 8;                 // lanes per token row
  constexpr int R = ilog2c(LPT);
  constexpr int TPR = 32 / LPT;               // token rows per warp
  constexpr int S = kGqaSlots;
  constexpr int ST = S * TPR;                 // tokens per stage
  constexpr int NV = GN * S;                  // score values of one token row: n = qi * S + i
  constexpr int LOGS = ilog2c(S);
  // after the reduce-scatter a lane holds NVH values: n = NVH * sl + k (NV >= LPT)
  // or n = sl >> DSH (NV < LPT; 2^DSH lanes hold the same value)
  constexpr int NVH = NV >= LPT ? NV / LPT : 1;
  constexpr int DSH = NV >= LPT ? 0 : R - ilog2c(NV);
  constexpr int IL = NV >= LPT ? 0 : DSH;                  // lowest lane bit of the slot index
  constexpr int NIB = NV >= LPT ? ilog2c(S / NVH) : LOGS;  // lane bits of the slot index
  constexpr int NW = kGqaWarps;
  static_assert(NVH <= S && S % NVH == 0, "held values share one query head");

  extern __shared__ __align__(16) unsigned char smem[];
  float* s_m = reinterpret_cast<float*>(smem + kGqaLut);        // [NW][GN]
  float* s_l = s_m + NW * GN;                                   // [NW][GN]
  float* s_o = s_l + NW * GN;                                   // [NW][GN][HD]
  int& s_last = *reinterpret_cast<int*>(s_o + NW * GN * HD);    // (no static smem: the LUT's
                                                                //  immediate offset assumes it)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sl = lane & (LPT - 1), r = lane >> R;

  // pair LUT (independent of the previous kernel: built before the PDL wait)
  {
    float2* lut = reinterpret_cast<float2*>(smem);
    for (int i = tid; i < 256 * 32; i += NW * 32) {
      const int e = i >> 5;
      lut[i] = make_float2(p.lv.v[e & 15], p.lv.v[e >> 4]);
    }
  }
  __syncthreads();
  pdl_enter();

  const int item = blockIdx.x;
  const int c = item % p.nc;
  const int grp = item / p.nc;                // (b * Hkv + kvh) * nsg + sg
  const int sg = grp % p.nsg;
  const int bk = grp / p.nsg;                 // b * Hkv + kvh
  const int b = bk / p.Hkv;
  const int kvh = bk - b * p.Hkv;
  const int h0 = (kvh << p.kv_shift) + sg * GN;   // first query head of the sub-group
  const int len = __ldg(p.seq_lens + b);
  const int t0 = static_cast<int>(static_cast<long long>(len) * c / p.nc);
  const int t1 = static_cast<int>(static_cast<long long>(len) * (c + 1) / p.nc);
  const int nst = (t1 - t0 + ST - 1) / ST;

  // q pairs of this lane's 8 dims, scaled by log2(e)/sqrt(hd)
  uint64_t qp[GN][4];
#pragma unroll
  for (int qi = 0; qi < GN; ++qi) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(
        p.q + (static_cast<size_t>(b) * p.H + h0 + qi) * HD + sl * 8));
    const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[j]));
      qp[qi][j] = pack2(f.x * p.scale_log2, f.y * p.scale_log2);
    }
  }

  const int nblk = HD >> p.blk_shift;
  // contiguous: row of token t = bk * Tc + t; paged: (page * Hkv + kvh) * P + (t & (P - 1))
  const size_t row0 = PAGED ? static_cast<size_t>(kvh) << p.page_shift : static_cast<size_t>(bk) * p.Tc;
  const uint8_t* kbase = p.kc + sl * 4;
  const uint8_t* vbase = p.vc + sl * 4;
  const int sblk = (sl * 8) >> p.blk_shift;
  const float* ksbase = static_cast<const float*>(p.ks) + sblk;
  const float* vsbase = static_cast<const float*>(p.vs) + sblk;
  const int32_t* btrow = PAGED ? p.bt + static_cast<size_t>(b) * p.bt_stride : nullptr;
  const size_t page_rows = PAGED ? static_cast<size_t>(p.Hkv) << p.page_shift : 0;   // rows per page
  const int pmask = PAGED ? (1 << p.page_shift) - 1 : 0;
  const int slot_sstride = TPR * nblk;        // scale floats between a row's slots
  const uint32_t vsel = static_cast<uint32_t>(lane) * 8u;

  struct Buf {
    uint32_t k[S], v[S];
    float ks[S], vs[S];
  };
  // one stage's loads; rows past the chunk's end are predicated off (their
  // scores are masked), so no branches
  auto load = [&](Buf& bf, int st, int dep) {
    const int tb = t0 + st * ST + r + dep;
    const int nv = t1 - tb;                   // this row's slot i is valid iff i * TPR < nv
    if constexpr (PAGED) {
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const int t = tb + i * TPR;
        const bool ok = i * TPR < nv;
        const int pg = ok ? __ldg(btrow + (t >> p.page_shift)) : 0;
        const size_t row = static_cast<size_t>(pg) * page_rows + row0 + (t & pmask);
        bf.k[i] = gqa_ld32p(kbase + row * (HD / 2), ok);
        bf.v[i] = gqa_ld32p(vbase + row * (HD / 2), ok);
        bf.ks[i] = __uint_as_float(gqa_ld32p(ksbase + row * nblk, ok));
        bf.vs[i] = __uint_as_float(gqa_ld32p(vsbase + row * nblk, ok));
      }
    } else {
      const size_t row = row0 + static_cast<size_t>(tb);
      const uint8_t* ck = kbase + row * (HD / 2);
      const uint8_t* cv = vbase + row * (HD / 2);
      const float* sk = ksbase + row * nblk;
      const float* sv = vsbase + row * nblk;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const bool ok = i * TPR < nv;
        bf.k[i] = gqa_ld32p(ck + i * TPR * (HD / 2), ok);
        bf.v[i] = gqa_ld32p(cv + i * TPR * (HD / 2), ok);
        bf.ks[i] = __uint_as_float(gqa_ld32p(sk, ok));
        bf.vs[i] = __uint_as_float(gqa_ld32p(sv, ok));
        sk += slot_sstride;
        sv += slot_sstride;
      }
    }
  };

  uint64_t o[GN][4];
  float m[GN];
#pragma unroll
  for (int qi = 0; qi < GN; ++qi) {
    m[qi] = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[qi][j] = 0;
  }
  float lown = 0.0f;                          // sum of this lane's weights (its query head)
  const int n0 = NV >= LPT ? NVH * sl : (sl >> DSH);
  const int qmine = n0 >> LOGS;

  auto consume = [&](const Buf& bf, int st) {
    // ---- scores: v[n], n = qi * S + i, partial over this lane's 8 dims
    float v[NV];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      uint64_t acc[GN];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t pr = gqa_lds_pair(gqa_prmt(bf.k[i], vsel, 0x7604u | (j << 4)));
#pragma unroll
        for (int qi = 0; qi < GN; ++qi) acc[qi] = j ? ffma2(pr, qp[qi][j], acc[qi]) : fmul2(pr, qp[qi][0]);
      }
#pragma unroll
      for (int qi = 0; qi < GN; ++qi) {
        const float2 a = unpack2(acc[qi]);
        v[qi * S + i] = (a.x + a.y) * bf.ks[i];
      }
    }
    // ---- reduce over the LPT lanes of a token row: reduce-scatter, then butterfly
#pragma unroll
    for (int rd = 0; rd < R; ++rd) {
      const int off = LPT >> (rd + 1);
      const int cntv = NV >> rd;
      if (cntv >= 2) {
        const int half = cntv >> 1;
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int k = 0; k < half; ++k) {
          const float send = up ? v[k] : v[k + half];
          const float keep = up ? v[k + half] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
      }
    }
    // ---- mask the rows past the chunk's end (only a chunk's last stage is partial)
    const int nvalid = t1 - (t0 + st * ST);
    if (nvalid < ST) {
#pragma unroll
      for (int k = 0; k < NVH; ++k) {
        const int i = (n0 + k) & (S - 1);
        if (i * TPR + r >= nvalid) v[k] = -INFINITY;
      }
    }
    // ---- stage max per query head, broadcast to every lane
    float mt = v[0];
#pragma unroll
    for (int k = 1; k < NVH; ++k) mt = fmaxf(mt, v[k]);
#pragma unroll
    for (int bb = 0; bb < NIB; ++bb) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1 << (IL + bb)));
#pragma unroll
    for (int off = LPT; off < 32; off <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
    float mcur = m[0];
#pragma unroll
    for (int qi = 0; qi < GN; ++qi) {
      const int src = NV >= LPT ? (qi * S) / NVH : ((qi * S) << DSH);
      const float mq = __shfl_sync(0xffffffffu, mt, src);
      if (mq > m[qi]) {                       // warp-uniform
        const float corr = fast_exp2(m[qi] - mq);   // m = -inf -> 0
        m[qi] = mq;
        const uint64_t c2 = pack2(corr, corr);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[qi][j] = fmul2(o[qi][j], c2);
        if (qmine == qi) lown *= corr;
      }
      if (qmine == qi) mcur = m[qi];
    }
    // ---- weights of the held values
    float pv[NVH];
#pragma unroll
    for (int k = 0; k < NVH; ++k) {
      pv[k] = fast_exp2(v[k] - mcur);         // masked: 0
      lown += pv[k];
    }
    // ---- P.V: gather the row's GN x S weights, scale by the lane's V block scale
#pragma unroll
    for (int i = 0; i < S; ++i) {
      float w[GN];
#pragma unroll
      for (int qi = 0; qi < GN; ++qi) {
        const int n = qi * S + i;
        const int srcsl = NV >= LPT ? n / NVH : (n << DSH);
        const int kk = NV >= LPT ? n % NVH : 0;
        w[qi] = __shfl_sync(0xffffffffu, pv[kk], srcsl, LPT) * bf.vs[i];   // within the row's lanes
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t pr = gqa_lds_pair(gqa_prmt(bf.v[i], vsel, 0x7604u | (j << 4)));
#pragma unroll
        for (int qi = 0; qi < GN; ++qi) o[qi][j] = ffma2(pr, pack2(w[qi], w[qi]), o[qi][j]);
      }
    }
  };

  // ---- stream this warp's stages: buffers A/B; the next stage's loads are
  // issued once the current stage's data has arrived (all
  // global loads share one scoreboard)
  {
    Buf A, Bf;
    int st = warp;
    if (st < nst) load(A, st, 0);
    while (st < nst) {
      int dep = static_cast<int>(A.k[0] & static_cast<uint32_t>(p.zero));
      if (st + NW < nst) load(Bf, st + NW, dep);
      consume(A, st);
      st += NW;
      if (st >= nst) break;
      dep = static_cast<int>(Bf.k[0] & static_cast<uint32_t>(p.zero));
      if (st + NW < nst) load(A, st + NW, dep);
      consume(Bf, st);
      st += NW;
    }
  }

  // ---- warp state -> shared memory: o summed over token rows, l per query head
#pragma unroll
  for (int off = LPT; off < 32; off <<= 1) {
#pragma unroll
    for (int qi = 0; qi < GN; ++qi)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = unpack2(o[qi][j]);
        o[qi][j] = pack2(a.x + __shfl_xor_sync(0xffffffffu, a.x, off),
                         a.y + __shfl_xor_sync(0xffffffffu, a.y, off));
      }
  }
  const float lcnt = (NV >= LPT || (sl & ((1 << DSH) - 1)) == 0) ? lown : 0.0f;  // one copy per value
#pragma unroll
  for (int qi = 0; qi < GN; ++qi) {
    float lq = qmine == qi ? lcnt : 0.0f;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) lq += __shfl_xor_sync(0xffffffffu, lq, off);
    if (lane == 0) {
      s_m[warp * GN + qi] = m[qi];
      s_l[warp * GN + qi] = lq;
    }
    if (r == 0) {
      float* dst = s_o + (warp * GN + qi) * HD + sl * 8;
#pragma unroll
      for (int j = 0; j < 4; ++j) reinterpret_cast<float2*>(dst)[j] = unpack2(o[qi][j]);
    }
  }
  __syncthreads();

  gqa_epilogue<HD, GN, NW>(p, s_m, s_l, s_o, s_last, grp, c, b, h0);
}

// ---------------------------------------------------------------------------
// Tensor-core variant (NQKV_GQA_TC): the group's K scores on mma.sync
// m16n8k16 (fp16 x fp16 -> fp32).  A = 16 keys x 16 dims of LEVELS L[code]
// as exact-ish fp16 hi/lo pairs (two MMAs: L = hi + lo to ~2^-22), B = the
// group's unscaled fp16 queries (exact; columns >= GN zero), one fp32
// accumulator per 32-dim segment, so the block scale (blk >= 32) and
// log2(e)/sqrt(hd) multiply the accumulators afterwards.  The dims inside a
// segment are permuted consistently in A and B (lane c of a quad supplies
// 32-bit word c of each 16-byte quarter row, each byte one A register), so
// every MMA stays inside one scale block.  V as in gqa_decode_kernel: fp32
// pair LUT + one FFMA2 per query head, with the weights handed over through
// shared memory.
//   K LUT entry (8 B): {half2(hi(L[lo]), hi(L[hi])), half2(lo(L[lo]), lo(L[hi]))}
//   V LUT entry (8 B): {L[lo], L[hi]} fp32
//   row e of the 64 KB table: 16 K copies, then 16 V copies (2 wavefronts
//   per warp LDS.64 either way: lanes l and l + 16 share a copy)
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
               "{%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// predicated loads that leave the register UNDEFINED when off (no zeroing
// move): only for values whose rows are masked afterwards -- K words and K
// scales (the row's scores become -inf) and V words (their weight is 0; the
// V scale, which multiplies the weight, is loaded zeroing)
__device__ __forceinline__ uint32_t gqa_ld32c(const void* p, bool on) {   // L1-allocating
  uint32_t r;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
               " @q ld.global.nc.u32 %0, [%1];\n}"
               : "=r"(r) : "l"(p), "r"(static_cast<int>(on)));
  return r;
}
// 16-bit (fp16 block scale) forms: zeroing and undefined-when-off
__device__ __forceinline__ float gqa_ldh(const void* p, bool on, bool zeroing) {
  unsigned short r;
  if (zeroing)
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b16 %0, 0;\n"
                 " @q ld.global.nc.L1::no_allocate.u16 %0, [%1];\n}"
                 : "=h"(r) : "l"(p), "r"(static_cast<int>(on)));
  else
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
                 " @q ld.global.nc.L1::no_allocate.u16 %0, [%1];\n}"
                 : "=h"(r) : "l"(p), "r"(static_cast<int>(on)));
  return __half2float(__ushort_as_half(r));
}
__device__ __forceinline__ uint32_t gqa_ld32u(const void* p, bool on) {   // streaming
  uint32_t r;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
               " @q ld.global.nc.L1::no_allocate.u32 %0, [%1];\n}"
               : "=r"(r) : "l"(p), "r"(static_cast<int>(on)));
  return r;
}

template <int HD, int GN>
constexpr size_t gqa_tc_smem_bytes() {
  return kGqaLut + static_cast<size_t>(kGqaWarps) * GN * (2 + HD) * 4 +
         static_cast<size_t>(kGqaWarps) * 16 * GN * 4 + 16;
}

template <int HD, int GN, bool PAGED, bool F16S>
__global__ void __launch_bounds__(kGqaWarps * 32, kGqaCtasPerSm)
gqa_tc_kernel(const __grid_constant__ GqaParams p) {
  constexpr int NSEG = HD / 32;              // 32-dim segments = 16-byte quarter rows
  constexpr int LPT = HD / 8;                // V: lanes per token row (8 dims each)
  constexpr int R = ilog2c(LPT);
  constexpr int TPR = 32 / LPT;
  constexpr int SV = 16 / TPR;               // V slots per 16-token stage
  constexpr int NW = kGqaWarps;
  static_assert(GN == 2 || GN == 4, "queries per CTA");

  extern __shared__ __align__(16) unsigned char smem[];
  float* s_m = reinterpret_cast<float*>(smem + kGqaLut);
  float* s_l = s_m + NW * GN;
  float* s_o = s_l + NW * GN;
  float* s_w = s_o + NW * GN * HD;           // [NW][16][GN] stage weights
  int& s_last = *reinterpret_cast<int*>(s_w + NW * 16 * GN);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;     // MMA fragment coordinates
  const int sl = lane & (LPT - 1), r = lane >> R;   // V lane coordinates

  {
    uint2* lut = reinterpret_cast<uint2*>(smem);
    for (int i = tid; i < 256 * 32; i += NW * 32) {
      const int e = i >> 5, cp = i & 31;
      const float l0 = p.lv.v[e & 15], l1 = p.lv.v[e >> 4];
      uint2 v;
      if (cp < 16) {
        const __half h0 = __float2half_rn(l0), h1 = __float2half_rn(l1);
        const __half r0 = __float2half_rn(l0 - __half2float(h0));
        const __half r1 = __float2half_rn(l1 - __half2float(h1));
        const __half2 hi = __halves2half2(h0, h1), lo = __halves2half2(r0, r1);
        v.x = *reinterpret_cast<const uint32_t*>(&hi);
        v.y = *reinterpret_cast<const uint32_t*>(&lo);
      } else {
        v.x = __float_as_uint(l0);
        v.y = __float_as_uint(l1);
      }
      lut[i] = v;
    }
  }
  __syncthreads();
  pdl_enter();

  const int item = blockIdx.x;
  const int cix = item % p.nc;
  const int grp = item / p.nc;
  const int sg = grp % p.nsg;
  const int bk = grp / p.nsg;
  const int b = bk / p.Hkv;
  const int kvh = bk - b * p.Hkv;
  const int h0 = (kvh << p.kv_shift) + sg * GN;
  const int len = __ldg(p.seq_lens + b);
  const int t0 = static_cast<int>(static_cast<long long>(len) * cix / p.nc);
  const int t1 = static_cast<int>(static_cast<long long>(len) * (cix + 1) / p.nc);
  const int nst = (t1 - t0 + 15) / 16;

  // B fragments: query n = g (zero for g >= GN); chunk (seg i, half h):
  // b0 = dims 32i + 8c + 4h + {0,1}, b1 = dims 32i + 8c + 4h + {2,3}
  uint32_t qb[NSEG][2][2];
  {
    const __half* qrow = p.q + (static_cast<size_t>(b) * p.H + h0 + (g < GN ? g : 0)) * HD;
#pragma unroll
    for (int i = 0; i < NSEG; ++i) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(qrow + 32 * i + 8 * c));
      const uint2 w2 = __ldg(reinterpret_cast<const uint2*>(qrow + 32 * i + 8 * c + 4));
      qb[i][0][0] = g < GN ? w.x : 0u;
      qb[i][0][1] = g < GN ? w.y : 0u;
      qb[i][1][0] = g < GN ? w2.x : 0u;
      qb[i][1][1] = g < GN ? w2.y : 0u;
    }
  }

  const int nblk = HD >> p.blk_shift;
  const size_t row0 = PAGED ? static_cast<size_t>(kvh) << p.page_shift : static_cast<size_t>(bk) * p.Tc;
  const int32_t* btrow = PAGED ? p.bt + static_cast<size_t>(b) * p.bt_stride : nullptr;
  const size_t page_rows = PAGED ? static_cast<size_t>(p.Hkv) << p.page_shift : 0;
  const int pmask = PAGED ? (1 << p.page_shift) - 1 : 0;
  auto row_of = [&](int t) -> size_t {
    if constexpr (PAGED)
      return static_cast<size_t>(__ldg(btrow + (t >> p.page_shift))) * page_rows + row0 + (t & pmask);
    else
      return row0 + static_cast<size_t>(t);
  };
  const uint32_t ksel = static_cast<uint32_t>(lane & 15) * 8u;
  const uint32_t vsel = ksel + 128u;
  const int vblk = (sl * 8) >> p.blk_shift;

  struct Buf {
    uint32_t k[2][NSEG];
    float ks[2][NSEG];
    uint32_t v[SV];
    float vs[SV];
  };
  // per-segment scale offsets (blk >= 32: segment i lies in block (32 i) / blk)
  int soff[NSEG];
#pragma unroll
  for (int i = 0; i < NSEG; ++i) soff[i] = (32 * i) >> p.blk_shift;
  const int vsstride = TPR * nblk;            // V scale elements between a lane's slots
  using SE = typename std::conditional<F16S, __half, float>::type;   // scale element
  const SE* ksp = static_cast<const SE*>(p.ks);
  const SE* vsp = static_cast<const SE*>(p.vs);
  // zeroing: the V scale (it multiplies a masked row's zero weight); K scales
  // of masked rows may stay undefined (their scores become -inf)
  auto lds = [&](const SE* ptr, bool ok, bool zeroing) -> float {
    if constexpr (F16S) return gqa_ldh(ptr, ok, zeroing);
    else return __uint_as_float(zeroing ? gqa_ld32p(ptr, ok) : gqa_ld32u(ptr, ok));
  };
  auto load = [&](Buf& bf, int st, int dep) {
    const int tb = t0 + st * 16 + dep;
    if constexpr (PAGED) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int t = tb + g + 8 * hr;
        const bool ok = t < t1;
        const size_t row = row_of(ok ? t : t0);
        const uint8_t* kr = p.kc + row * (HD / 2) + 4 * c;
        const SE* sr = ksp + row * nblk;
#pragma unroll
        for (int i = 0; i < NSEG; ++i) {
          bf.k[hr][i] = gqa_ld32c(kr + 16 * i, ok);
          bf.ks[hr][i] = lds(sr + soff[i], ok, true);
        }
      }
#pragma unroll
      for (int i = 0; i < SV; ++i) {
        const int t = tb + i * TPR + r;
        const bool ok = t < t1;
        const size_t row = row_of(ok ? t : t0);
        bf.v[i] = gqa_ld32p(p.vc + row * (HD / 2) + 4 * sl, ok);
        bf.vs[i] = lds(vsp + row * nblk + vblk, ok, true);
      }
    } else {
      // one base pointer per stream and stage; slots / rows / segments are offsets
      const size_t rk = row0 + static_cast<size_t>(tb + g);
      const uint8_t* kr = p.kc + rk * (HD / 2) + 4 * c;
      const SE* sr = ksp + rk * nblk;
      const int nk = t1 - tb - g;             // row g valid iff 0 < nk, row g + 8 iff 8 < nk
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const bool ok = 8 * hr < nk;
#pragma unroll
        for (int i = 0; i < NSEG; ++i) {
          bf.k[hr][i] = gqa_ld32c(kr + hr * 8 * (HD / 2) + 16 * i, ok);
          bf.ks[hr][i] = lds(sr + soff[i], ok, false);
        }
        sr += 8 * nblk;
      }
      const size_t rv = row0 + static_cast<size_t>(tb + r);
      const uint8_t* vr = p.vc + rv * (HD / 2) + 4 * sl;
      const SE* vsr = vsp + rv * nblk + vblk;
      const int nv = t1 - tb - r;
#pragma unroll
      for (int i = 0; i < SV; ++i) {
        const bool ok = i * TPR < nv;
        bf.v[i] = gqa_ld32u(vr + i * TPR * (HD / 2), ok);
        bf.vs[i] = lds(vsr, ok, true);
        vsr += vsstride;
      }
    }
  };

  uint64_t o[GN][4];
  float m2[2] = {-INFINITY, -INFINITY};       // running max of queries 2c, 2c + 1
  float l2[2] = {0.0f, 0.0f};                 // this lane's rows' weight sums
#pragma unroll
  for (int qi = 0; qi < GN; ++qi)
#pragma unroll
    for (int j = 0; j < 4; ++j) o[qi][j] = 0;
  float* ws = s_w + warp * 16 * GN;

  auto consume = [&](const Buf& bf, int st) {
    // ---- K: S(row, query) per segment on the tensor cores
    float acc[NSEG][4];
#pragma unroll
    for (int i = 0; i < NSEG; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][e] = 0.0f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t a0 = gqa_lds_pair(gqa_prmt(bf.k[0][i], ksel, 0x7604u | ((2 * h) << 4)));
        const uint64_t a1 = gqa_lds_pair(gqa_prmt(bf.k[1][i], ksel, 0x7604u | ((2 * h) << 4)));
        const uint64_t a2 = gqa_lds_pair(gqa_prmt(bf.k[0][i], ksel, 0x7604u | ((2 * h + 1) << 4)));
        const uint64_t a3 = gqa_lds_pair(gqa_prmt(bf.k[1][i], ksel, 0x7604u | ((2 * h + 1) << 4)));
        mma_16816(acc[i], static_cast<uint32_t>(a0), static_cast<uint32_t>(a1), static_cast<uint32_t>(a2),
                  static_cast<uint32_t>(a3), qb[i][h][0], qb[i][h][1]);
        mma_16816(acc[i], static_cast<uint32_t>(a0 >> 32), static_cast<uint32_t>(a1 >> 32),
                  static_cast<uint32_t>(a2 >> 32), static_cast<uint32_t>(a3 >> 32), qb[i][h][0],
                  qb[i][h][1]);
      }
    }
    // scores in log2 units: rows g (e = 0, 1) and g + 8 (e = 2, 3), queries 2c + (e & 1)
    float sc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int hr = e >> 1;
      float x = acc[0][e] * bf.ks[hr][0];
#pragma unroll
      for (int i = 1; i < NSEG; ++i) x = fmaf(acc[i][e], bf.ks[hr][i], x);
      sc[e] = x * p.scale_log2;
    }
    const int nvalid = t1 - (t0 + st * 16);
    if (nvalid < 16) {
      if (g >= nvalid) sc[0] = sc[1] = -INFINITY;
      if (g + 8 >= nvalid) sc[2] = sc[3] = -INFINITY;
    }
    // ---- online softmax per query (lanes with equal c share queries)
    float pw[4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float mt = fmaxf(sc[j], sc[2 + j]);
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 4));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 8));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 16));
      const float mn = fmaxf(m2[j], mt);
      const float corr = fast_exp2(m2[j] - mn);   // m = -inf -> 0
      m2[j] = mn;
      pw[j] = fast_exp2(sc[j] - mn);
      pw[2 + j] = fast_exp2(sc[2 + j] - mn);
      l2[j] = l2[j] * corr + pw[j] + pw[2 + j];
      sc[j] = corr;                             // (reuse: the correction factor)
    }
    // weights -> shared memory [16 rows][GN]
    __syncwarp();
    if (2 * c < GN) {
      reinterpret_cast<float2*>(ws + g * GN)[c] = make_float2(pw[0], pw[1]);
      reinterpret_cast<float2*>(ws + (g + 8) * GN)[c] = make_float2(pw[2], pw[3]);
    }
    // rescale o by the per-query corrections (held by lanes c = qi / 2)
#pragma unroll
    for (int qi = 0; qi < GN; ++qi) {
      const float corr = __shfl_sync(0xffffffffu, sc[qi & 1], qi >> 1);
      if (corr != 1.0f) {                       // warp-uniform
        const uint64_t c2 = pack2(corr, corr);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[qi][j] = fmul2(o[qi][j], c2);
      }
    }
    __syncwarp();
    // ---- V: P.V with the pair LUT, one FFMA2 per query head
#pragma unroll
    for (int i = 0; i < SV; ++i) {
      const int t = i * TPR + r;
      float w[GN];
      if constexpr (GN == 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(ws + t * 4);
        w[0] = w4.x * bf.vs[i]; w[1] = w4.y * bf.vs[i]; w[2] = w4.z * bf.vs[i]; w[3] = w4.w * bf.vs[i];
      } else {
        const float2 w2 = *reinterpret_cast<const float2*>(ws + t * 2);
        w[0] = w2.x * bf.vs[i]; w[1] = w2.y * bf.vs[i];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t pr = gqa_lds_pair(gqa_prmt(bf.v[i], vsel, 0x7604u | (j << 4)));
#pragma unroll
        for (int qi = 0; qi < GN; ++qi) o[qi][j] = ffma2(pr, pack2(w[qi], w[qi]), o[qi][j]);
      }
    }
  };

  {
    Buf A, Bf;
    int st = warp;
    if (st < nst) load(A, st, 0);
    while (st < nst) {
      int dep = static_cast<int>(A.k[0][0] & static_cast<uint32_t>(p.zero));
      if (st + NW < nst) load(Bf, st + NW, dep);
      consume(A, st);
      st += NW;
      if (st >= nst) break;
      dep = static_cast<int>(Bf.k[0][0] & static_cast<uint32_t>(p.zero));
      if (st + NW < nst) load(A, st + NW, dep);
      consume(Bf, st);
      st += NW;
    }
  }

  // ---- warp state -> shared memory
#pragma unroll
  for (int off = LPT; off < 32; off <<= 1) {
#pragma unroll
    for (int qi = 0; qi < GN; ++qi)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = unpack2(o[qi][j]);
        o[qi][j] = pack2(a.x + __shfl_xor_sync(0xffffffffu, a.x, off),
                         a.y + __shfl_xor_sync(0xffffffffu, a.y, off));
      }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    l2[j] += __shfl_xor_sync(0xffffffffu, l2[j], 4);
    l2[j] += __shfl_xor_sync(0xffffffffu, l2[j], 8);
    l2[j] += __shfl_xor_sync(0xffffffffu, l2[j], 16);
  }
  if (g == 0 && 2 * c < GN) {
    s_m[warp * GN + 2 * c] = m2[0];
    s_m[warp * GN + 2 * c + 1] = m2[1];
    s_l[warp * GN + 2 * c] = l2[0];
    s_l[warp * GN + 2 * c + 1] = l2[1];
  }
  if (r == 0) {
#pragma unroll
    for (int qi = 0; qi < GN; ++qi) {
      float* dst = s_o + (warp * GN + qi) * HD + sl * 8;
#pragma unroll
      for (int j = 0; j < 4; ++j) reinterpret_cast<float2*>(dst)[j] = unpack2(o[qi][j]);
    }
  }
  __syncthreads();
  gqa_epilogue<HD, GN, NW>(p, s_m, s_l, s_o, s_last, grp, cix, b, h0);
}

}  // namespace nqkv
