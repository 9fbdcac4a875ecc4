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
#include "common.cuh"

namespace nqkv {

constexpr int kGqaWarps = 4;        // per CTA (3 CTAs per SM: 170 registers per thread)
constexpr int kGqaCtasPerSm = 3;
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
  const float* ks;           // [B][Hkv][Tc][hd/blk]
  const uint8_t* vc;
  const float* vs;
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
  const float* ksbase = p.ks + sblk;
  const float* vsbase = p.vs + sblk;
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

  // ---- CTA merge of the warps (fixed order), then the chunk merge
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

}  // namespace nqkv
