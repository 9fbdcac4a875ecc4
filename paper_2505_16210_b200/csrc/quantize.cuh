// Quantize/append (a1-a3), standalone dequantize (a4) and the code-function
// test hook.  The code function itself is in common.cuh.
#pragma once
#include "common.cuh"

namespace nqkv {

// ------------------------------------------------ a1-a3: quantize + append
struct QuantParams {
  const __half* x;
  long long sb, st, sh;          // element strides
  const int32_t* pos;
  uint8_t* codes;
  void* scales;                  // fp32, or fp16 (template F16S; exact for fp16 inputs)
  int B, n_new, H, Tc, blk_shift;
  int hpb_shift;                 // blk > hd: a block spans 2^hpb_shift heads
  uint32_t total;                // 16-element chunks: B * n_new * H * hd / 16 (x2 two tensors)
  // fused K + V call (nqkv_quantize_pair): chunks [total1, total) are the
  // second tensor's (x2 -> codes2 / scales2, same strides and geometry)
  uint32_t total1;
  const __half* x2;
  uint8_t* codes2;
  void* scales2;
  int v256;                      // bit 0: x and strides 32-byte aligned (256-bit loads);
                                 // bit 1: x contiguous [B][n_new][H][hd]
  FastDiv cpr;                   // chunks per token row (b, t): H * hd / 16
  FastDiv nnew;                  // n_new
  BucketTab tab;
  // paged cache (reading R17): row pos of sequence b is row
  // pos & (P - 1) of page bt[b][pos >> page_shift] in [n_pages][H][P] storage
  const int32_t* bt;             // nullptr: contiguous [B][H][Tc]
  int bt_stride, page_shift;
};

// Bucket table replicated per lane: entry e for lane l at shared address
// 0x400 + e*256 + l*8 (conflict-free lookups).  The dynamic shared window of
// this kernel starts at 0x400 (1 KB driver reserve, no static smem -- checked on
// device), so idx = RN(16 n + 16) taken from the low byte of the fma result
// with +4 folded into the magic constant gives the full address with ONE PRMT:
// byte 0 = lane*8, byte 1 = idx + 4, bytes 2-3 = 0.
constexpr int kRepEntryBytes = 256;
constexpr size_t kQuantSmem = static_cast<size_t>(kNumBuckets) * kRepEntryBytes;
constexpr float kBucketMagic = 12582932.0f;   // 1.5*2^23 + 16 + 4 (bits 0x4B400014)
#ifndef NQKV_Q_PAIRS
#define NQKV_Q_PAIRS 1             // fp32x2 pair arithmetic in the quantize kernel
#endif

__device__ __forceinline__ uint32_t nf4_code_rep(float n, uint32_t lane8) {
  const float y = __fmaf_rn(n, 16.0f, kBucketMagic);
  const float2 e = unpack2(lds64(__byte_perm(__float_as_uint(y), lane8, 0x5504)));
  // lo + (n > thr): the sign bit of thr - n (thr = +inf -> never; equal -> +0)
  return __float_as_uint(e.y) + (__float_as_uint(__fsub_rn(e.x, n)) >> 31);
}

// Codes of 8 fp16 values (one uint4) with reciprocal scale r -> 8 nibbles,
// element 2i in the low nibble of byte i.
__device__ __forceinline__ uint32_t encode8_rep(const uint4 raw, float r, uint32_t lane8) {
  __half2 hv[4];
  memcpy(hv, &raw, 16);
  uint32_t b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 xf = __half22float2(hv[k]);
    const uint32_t lo = nf4_code_rep(__fmul_rn(xf.x, r), lane8);
    const uint32_t hi = nf4_code_rep(__fmul_rn(xf.y, r), lane8);
    b[k] = hi * 16u + lo;
  }
  return __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
}

// Codes of 8 fp16 values, element pairs in fp32x2 arithmetic: n = RN32(x * r)
// and y = RN32(16 n + magic) are the same per-element roundings as
// nf4_code_rep's (fma.rn.f32x2 / mul.rn.f32x2 round each lane exactly like
// the scalar forms), so the codes are identical; the pair conversion, one
// FMUL2 and one FFMA2 per two elements, and a set-and-subtract compare save
// ~3 instructions per element.
__device__ __forceinline__ uint32_t encode8_rep2(const uint4 raw, uint64_t r2, uint32_t lane8) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
  uint32_t b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint64_t x2;
    asm("{.reg .f16 a, b;\n .reg .f32 fa, fb;\n mov.b32 {a, b}, %1;\n cvt.f32.f16 fa, a;\n"
        " cvt.f32.f16 fb, b;\n mov.b64 %0, {fa, fb};}" : "=l"(x2) : "r"(w[k]));
    uint64_t n2, y2;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(n2) : "l"(x2), "l"(r2));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y2)
        : "l"(n2), "l"(0x4180000041800000ull), "l"(0x4B4000144B400014ull));   // 16, kBucketMagic
    const float2 n = unpack2(n2), y = unpack2(y2);
    const float2 e0 = unpack2(lds64(__byte_perm(__float_as_uint(y.x), lane8, 0x5504)));
    const float2 e1 = unpack2(lds64(__byte_perm(__float_as_uint(y.y), lane8, 0x5504)));
    // lo + (n > thr): the sign bit of thr - n (thr = +inf -> never; equal -> +0)
    const uint32_t lo = __float_as_uint(e0.y) + (__float_as_uint(__fsub_rn(e0.x, n.x)) >> 31);
    const uint32_t hi = __float_as_uint(e1.y) + (__float_as_uint(__fsub_rn(e1.x, n.y)) >> 31);
    b[k] = hi * 16u + lo;
  }
  return __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
}

// 32 contiguous bytes per lane in ONE 256-bit load (a warp reads 1 KB)
__device__ __forceinline__ void ldg_stream_256(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

__device__ __forceinline__ float absmax16(const uint4 a, const uint4 b) {
  __half2 ha[4], hb[4];
  memcpy(ha, &a, 16);
  memcpy(hb, &b, 16);
  const __half2 m = __hmax2(__hmax2(__hmax2(__habs2(ha[0]), __habs2(ha[1])), __hmax2(__habs2(ha[2]), __habs2(ha[3]))),
                            __hmax2(__hmax2(__habs2(hb[0]), __habs2(hb[1])), __hmax2(__habs2(hb[2]), __habs2(hb[3]))));
  return fmaxf(__low2float(m), __high2float(m));
}

// Work unit = 64 consecutive 16-element chunks of the flattened (b, t, h,
// chunk) order; lane l owns chunks 2l and 2l+1 of the unit (32 contiguous
// elements: a block of blk elements spans blk/32 lanes, or half a lane when
// blk = 32).  Units are strided over the warps of the grid; the next unit's
// loads are issued before the current one is encoded (ping-pong registers).
// When x is contiguous ([B][n_new][H][hd] packed), chunk c starts at x + 16c.
// LAYOUT: 0 one tensor, contiguous cache; 1 K and V pair (nqkv_quantize_pair);
// 2 one tensor into a paged cache (nqkv_quantize_kv; R17).  Separate
// instantiations: the plain kernel carries no layout code.
template <int HD, int BLK, bool F16S, int LAYOUT = 0>
__global__ void __launch_bounds__(256, 4) quantize_kernel(const __grid_constant__ QuantParams p) {
  constexpr int CPT = HD / 16;                 // chunks per (token, head)
  constexpr int LOG_CPT = CPT == 4 ? 2 : 3;
  constexpr int GL = BLK >= 32 ? BLK / 32 : 1; // lanes per block (>= 1)
  extern __shared__ __align__(16) unsigned char qsmem[];
  for (int i = threadIdx.x; i < kNumBuckets * 32; i += blockDim.x)
    reinterpret_cast<float2*>(qsmem)[i] = p.tab.e[i >> 5];
  if (static_cast<uint32_t>(__cvta_generic_to_shared(qsmem)) != 0x400u) __trap();
  __syncthreads();
  pdl_enter();                       // wait, then trigger: see common.cuh
  const int lane = threadIdx.x & 31;
  const uint32_t lane8 = lane * 8u;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const int nblk = HD >> p.blk_shift;
  const bool contig = p.v256 > 1;
  // chunk c of the call -> (tensor, chunk within it); a lane's two chunks
  // and a block never straddle the tensors (total1 is a multiple of a row)
  auto src_of = [&](const __half* x, uint32_t c) -> const __half* {
    if (contig) return x + static_cast<unsigned long long>(c) * 16u;
    const uint32_t row = fdiv(c, p.cpr), within = c - row * p.cpr.d;
    const uint32_t b = fdiv(row, p.nnew), t = row - b * p.nnew.d;
    return x + b * p.sb + t * p.st + (within >> LOG_CPT) * p.sh + (within & (CPT - 1)) * 16;
  };
  struct Buf { uint4 v[4]; };
  auto load = [&](uint32_t unit, Buf& B, uint32_t dep) {
    uint32_t c = unit * 64u + 2u * lane + dep;
    if (c < p.total) {
      const bool sec = LAYOUT == 1 && c >= p.total1;
      const __half* x = sec ? p.x2 : p.x;
      if (sec) c -= p.total1;
      const __half* s0 = src_of(x, c);
      const __half* s1 = contig ? s0 + 16 : src_of(x, c + 1);
      if (p.v256 & 1) {
        ldg_stream_256(s0, B.v[0], B.v[1]);
        ldg_stream_256(s1, B.v[2], B.v[3]);
      } else {
        B.v[0] = ldg_stream_128(s0);
        B.v[1] = ldg_stream_128(s0 + 8);
        B.v[2] = ldg_stream_128(s1);
        B.v[3] = ldg_stream_128(s1 + 8);
      }
    }
  };
  // chunks c and c + 1 of a lane (c even; CPT even) lie in the same (b, t, h)
  // row: one 16-byte store of both code words, and the block scale (both
  // chunks share a block: blk >= 32) by the block's first lane
  auto store_pair = [&](uint32_t c, uint4 words, float s, bool scale_writer) {
    const bool sec = LAYOUT == 1 && c >= p.total1;
    uint8_t* const codes = sec ? p.codes2 : p.codes;
    void* const scales = sec ? p.scales2 : p.scales;
    if (sec) c -= p.total1;
    const uint32_t row = fdiv(c, p.cpr), within = c - row * p.cpr.d;
    const uint32_t bb = fdiv(row, p.nnew), t = row - bb * p.nnew.d;
    const int pos = __ldg(p.pos + bb) + static_cast<int>(t);
    if (pos < 0 || pos >= p.Tc) return;
    const uint32_t h = within >> LOG_CPT, cr = within & (CPT - 1);
    // row of (b, h, pos): contiguous, or in its page (R17)
    long long base = static_cast<long long>(bb), rowin = pos, rows = p.Tc;
    if (LAYOUT == 2) {
      base = __ldg(p.bt + static_cast<long long>(bb) * p.bt_stride + (pos >> p.page_shift));
      rowin = pos & ((1 << p.page_shift) - 1);
      rows = 1ll << p.page_shift;
    }
    const long long rr = (base * p.H + h) * rows + rowin;
    *reinterpret_cast<uint4*>(codes + rr * (HD / 2) + cr * 8) = words;
    if (scale_writer) {
      // blk > hd: one scale per (token, head group): [B][H >> hpb_shift][Tc]
      const long long si = BLK > HD ? ((base * p.H + h) >> p.hpb_shift) * rows + rowin
                                    : rr * nblk + ((cr * 16) >> p.blk_shift);
      if constexpr (F16S)
        reinterpret_cast<__half*>(scales)[si] = __float2half_rn(s);   // exact: s is an fp16 value
      else
        reinterpret_cast<float*>(scales)[si] = s;
    }
  };
  auto encode = [&](uint32_t unit, const Buf& B) {
    const uint32_t c = unit * 64u + 2u * lane;
    const bool valid = c < p.total;
    float s0 = valid ? absmax16(B.v[0], B.v[1]) : 0.0f;
    float s1 = valid ? absmax16(B.v[2], B.v[3]) : 0.0f;
    if (BLK > 16) s0 = s1 = fmaxf(s0, s1);     // both chunks in one block (blk >= 32)
#pragma unroll
    for (int o = 1; o < GL; o <<= 1) {
      s0 = fmaxf(s0, __shfl_xor_sync(0xffffffffu, s0, o));
      if (BLK <= 16) s1 = fmaxf(s1, __shfl_xor_sync(0xffffffffu, s1, o));
    }
    if (BLK > 16) s1 = s0;
    const float r0 = block_rcp(s0), r1 = BLK > 16 ? r0 : block_rcp(s1);
#if NQKV_Q_PAIRS
    const uint64_t r0p = pack2(r0, r0), r1p = pack2(r1, r1);
    const uint2 w0 = make_uint2(encode8_rep2(B.v[0], r0p, lane8), encode8_rep2(B.v[1], r0p, lane8));
    const uint2 w1 = make_uint2(encode8_rep2(B.v[2], r1p, lane8), encode8_rep2(B.v[3], r1p, lane8));
#else
    const uint2 w0 = make_uint2(encode8_rep(B.v[0], r0, lane8), encode8_rep(B.v[1], r0, lane8));
    const uint2 w1 = make_uint2(encode8_rep(B.v[2], r1, lane8), encode8_rep(B.v[3], r1, lane8));
#endif
#ifdef NQKV_EXP_QNOSTORE
    if (w0.x == 0x12345678u && w1.y == 0x9abcdef0u && s0 == 1.5f) reinterpret_cast<float*>(p.scales)[0] = s0;
    return;
#endif
    if (!valid) return;
    // scale writer: the first lane of each block (blk 32: every lane)
    const bool first = ((2 * lane * 16) & ((1 << p.blk_shift) - 1)) == 0;
    static_assert(BLK > 16, "both chunks of a lane share one block");
    store_pair(c, make_uint4(w0.x, w0.y, w1.x, w1.y), s0, first);
  };
  // Two units in flight per warp.  ptxas puts every global load on one
  // scoreboard, so a unit's loads are issued only after the previous unit's
  // data has arrived (`dep`, always 0, is computed from its first word):
  // otherwise the wait for a unit would also wait for the loads just issued.
  uint32_t zero;
#if !defined(NQKV_QDEPZERO) || NQKV_QDEPZERO
  zero = static_cast<uint32_t>(p.v256) >> 2;   // always 0, but not a constant ptxas can fold
#else
  asm volatile("mov.u32 %0, 0;" : "=r"(zero));
#endif
  uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  Buf A{}, Bb{};
  load(u, A, 0u);
  while (u * 64u < p.total) {
    load(u + nw, Bb, A.v[0].x & zero);
    encode(u, A);
    u += nw;
    if (u * 64u >= p.total) break;
    load(u + nw, A, Bb.v[0].x & zero);
    encode(u, Bb);
    u += nw;
  }
}

// ------------------------------------------------- a4 standalone: dequant
struct DequantParams {
  const uint8_t* codes;
  const void* scales;       // fp32, or fp16 (template F16S)
  void* out;
  long long total_chunks;   // B*H*n_tokens*hd/8
  int Tc, hd, n_tokens, blk_shift, chunks_per_row;
  int hpb_shift;            // blk > hd: scales [B][H >> hpb_shift][Tc] (blk_shift = log2 hd)
  Levels lv;
};

template <bool F16, bool F16S>
__global__ void __launch_bounds__(256) dequant_kernel(const DequantParams p) {
  __shared__ float s_lv[16];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) s_lv[k] = p.lv.v[k];
  }
  __syncthreads();
  pdl_enter();                       // wait, then trigger: see common.cuh
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       c < p.total_chunks; c += stride) {
    const int cr = static_cast<int>(c % p.chunks_per_row);
    const long long tok = c / p.chunks_per_row;               // (b*H + h)*n_tokens + t
    const long long bh = tok / p.n_tokens;
    const int t = static_cast<int>(tok % p.n_tokens);
    const long long rowid = bh * p.Tc + t;
    const uint32_t w = reinterpret_cast<const uint32_t*>(p.codes + rowid * (p.hd / 2))[cr];
    const long long si = p.hpb_shift ? (bh >> p.hpb_shift) * p.Tc + t
                                     : rowid * (p.hd >> p.blk_shift) + ((cr * 8) >> p.blk_shift);
    const float s = F16S ? __half2float(reinterpret_cast<const __half*>(p.scales)[si])
                         : reinterpret_cast<const float*>(p.scales)[si];
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __fmul_rn(s, s_lv[(w >> (4 * k)) & 15u]);
    if (F16) {
      __half2 h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = __floats2half2_rn(v[2 * k], v[2 * k + 1]);
      reinterpret_cast<uint4*>(p.out)[c] = *reinterpret_cast<uint4*>(h);
    } else {
      float4* o = reinterpret_cast<float4*>(p.out) + 2 * c;
      o[0] = make_float4(v[0], v[1], v[2], v[3]);
      o[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// --------------------------------------------------- test hook: code(n)
__global__ void encode_normalized_kernel(const float* n, long long count, uint8_t* codes,
                                         const BucketTab tab) {
  __shared__ float2 s_tab[kNumBuckets];
  for (int i = threadIdx.x; i < kNumBuckets; i += blockDim.x) s_tab[i] = tab.e[i];
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float v = fminf(fmaxf(n[i], -1.0f), 1.0f);
    codes[i] = static_cast<uint8_t>(nf4_code(v, base));
  }
}

}  // namespace nqkv
