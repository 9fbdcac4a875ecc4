// NQKV hot path for B200 (sm_100a): NF4 quantize/pack/append, standalone
// dequantize, and fused dequant-in-registers split-K decode attention.
// The C ABI (include/nqkv.h) is implemented at the bottom of this file.
//
// Paper: PAPER.md:193 (block-wise quantile quantisation, index table lookup),
// :205 (prefill quantisation, 4-bit index storage), :219-235 (decode:
// quantize new token, Concat, dequantize, Softmax(t_Q X_K'^T), A X_V').
// The paper's own GPU design (materialise an fp16 copy of the whole cache,
// pad to 16 tokens, Cutlass BMM) is NOT followed: the
// decode kernel streams the packed nibbles from HBM and dequantises them in
// registers, so the only HBM traffic is the 4-bit codes + scales.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/nqkv.h"
#include "nqkv_internal.h"

namespace nqkv {

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ uint4 ldg_stream_128(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float ldg_f32(const float* p) {
  float r;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint64_t pack2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 unpack2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// d = a * b + c on a pair of fp32 lanes (SASS FFMA2, sm_100)
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float fast_exp2(float x) {  // ex2.approx(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------- a2: code function
// n in [-1, 1] (n = RN32(x/s), |x| <= s).  idx = RN(16 n + 16) is produced
// exactly by one fma against the magic constant 1.5*2^23 + 16 (unit ulp);
// bucket idx covers [(idx-16.5)/16, (idx-15.5)/16] and holds at most one
// decision threshold (host-checked), so code = lo[idx] + (n > thr[idx]) is
// exactly #{i : n > T_i} = argmin_i |n - L_i| with ties to the lower index.
__device__ __forceinline__ uint32_t nf4_code(float n, uint32_t tab_base) {
  const float y = __fmaf_rn(n, 16.0f, 12582928.0f);
  const uint32_t off = __float_as_uint(y) * 8u - 0x5A000000u;  // (bits - 0x4B400000) * 8
  const float2 e = unpack2(lds64(tab_base + off));
  return __float_as_uint(e.y) + (n > e.x ? 1u : 0u);
}

struct BucketTab {
  float2 e[kNumBuckets];   // {thr, lo (uint bits)}
};

__device__ __forceinline__ uint32_t load_bucket_table(const BucketTab& t, float2* smem) {
  for (int i = threadIdx.x; i < kNumBuckets; i += blockDim.x) smem[i] = t.e[i];
  return static_cast<uint32_t>(__cvta_generic_to_shared(smem));
}

// ------------------------------------------------ a1-a3: quantize + append
struct QuantParams {
  const __half* x;
  long long sb, st, sh;          // element strides
  const int32_t* pos;
  uint8_t* codes;
  float* scales;
  long long total_chunks;        // B * n_new * H * hd/8
  int H, hd, n_new, Tc, blk_shift, chunks_per_row;
  BucketTab tab;
};

// One thread = one 8-element chunk (16 B of fp16); blk/8 consecutive lanes
// form a block and reduce the absmax with xor-shuffles.
template <int GS>   // lanes per block = blk / 8
__global__ void __launch_bounds__(256) quantize_kernel(const QuantParams p) {
  __shared__ float2 s_tab[kNumBuckets];
  const uint32_t tab = load_bucket_table(p.tab, s_tab);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long warp0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x - lane);
  const long long wstride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long base = warp0; base < p.total_chunks; base += wstride) {
    const long long c = base + lane;
    const bool valid = c < p.total_chunks;
    long long r = valid ? c : 0;
    const int cr = static_cast<int>(r % p.chunks_per_row);   // chunk within the head row
    r /= p.chunks_per_row;
    const int h = static_cast<int>(r % p.H);
    r /= p.H;
    const int t = static_cast<int>(r % p.n_new);
    const int b = static_cast<int>(r / p.n_new);
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (valid) raw = ldg_stream_128(p.x + b * p.sb + t * p.st + h * p.sh + cr * 8);
    __half2 hv[4];
    memcpy(hv, &raw, 16);
    __half2 am = __hmax2(__hmax2(__habs2(hv[0]), __habs2(hv[1])),
                         __hmax2(__habs2(hv[2]), __habs2(hv[3])));
    float s = fmaxf(__low2float(am), __high2float(am));
#pragma unroll
    for (int o = 1; o < GS; o <<= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
    // correctly rounded reciprocal once per block, Markstein correction per
    // element: n = RN32(x/s) exactly (no fast-math anywhere in this file)
    const float rcp = s > 0.0f ? __frcp_rn(s) : 0.0f;
    uint32_t word = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 xf = __half22float2(hv[k]);
      const float q0 = __fmul_rn(xf.x, rcp), q1 = __fmul_rn(xf.y, rcp);
      const float e0 = __fmaf_rn(-q0, s, xf.x), e1 = __fmaf_rn(-q1, s, xf.y);
      const float n0 = __fmaf_rn(e0, rcp, q0), n1 = __fmaf_rn(e1, rcp, q1);
      word |= nf4_code(n0, tab) << (8 * k);
      word |= nf4_code(n1, tab) << (8 * k + 4);
    }
    if (valid) {
      const int row = p.pos[b] + t;
      if (row >= 0 && row < p.Tc) {
        const long long rowid = (static_cast<long long>(b) * p.H + h) * p.Tc + row;
        reinterpret_cast<uint32_t*>(p.codes + rowid * (p.hd / 2))[cr] = word;
        if ((cr & (GS - 1)) == 0) p.scales[rowid * (p.hd >> p.blk_shift) + cr / GS] = s;
      }
    }
  }
}

// ------------------------------------------------- a4 standalone: dequant
struct DequantParams {
  const uint8_t* codes;
  const float* scales;
  void* out;
  long long total_chunks;   // B*H*n_tokens*hd/8
  int Tc, hd, n_tokens, blk_shift, chunks_per_row;
  float levels[16];
};

template <bool F16>
__global__ void __launch_bounds__(256) dequant_kernel(const DequantParams p) {
  __shared__ float s_lv[16];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) s_lv[k] = p.levels[k];
  }
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       c < p.total_chunks; c += stride) {
    const int cr = static_cast<int>(c % p.chunks_per_row);
    const long long tok = c / p.chunks_per_row;               // (b*H + h)*n_tokens + t
    const long long bh = tok / p.n_tokens;
    const int t = static_cast<int>(tok % p.n_tokens);
    const long long rowid = bh * p.Tc + t;
    const uint32_t w = reinterpret_cast<const uint32_t*>(p.codes + rowid * (p.hd / 2))[cr];
    const float s = p.scales[rowid * (p.hd >> p.blk_shift) + ((cr * 8) >> p.blk_shift)];
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
  const uint32_t base = load_bucket_table(tab, s_tab);
  __syncthreads();
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float v = fminf(fmaxf(n[i], -1.0f), 1.0f);
    codes[i] = static_cast<uint8_t>(nf4_code(v, base));
  }
}

// ------------------------------------------ a4-a7: fused decode attention
// Work item = (b, h, 64-token chunk), processed by ONE warp.  Each lane owns
// 32 consecutive head dims (16 packed bytes): LPT = hd/32 lanes cover a
// token row, G = 32/LPT token groups per warp, NT = 64/G tokens per lane.
//
// Dequantisation never leaves the SM: a packed byte (two 4-bit codes) is
// turned into the pair (L[lo], L[hi]) by ONE shared-memory load from a
// 256-entry fp32-pair table replicated per lane (64 KB, conflict-free: lane l
// reads bank pair 2l), addressed by one PRMT that splices the code byte above
// lane*8; the pair then feeds one FFMA2 (fp32x2 fma).  Scores use the fp32
// level (block scale applied once per 32 dims); values accumulate w*L with
// w = p * scale.  Softmax is exact within the chunk (single max); chunks merge
// with the usual (m, l, o) rescaling in fixed chunk order.
constexpr int kChunk = 64;
constexpr int kLutBytes = 256 * 32 * 8;

struct DecodeParams {
  const __half* q;
  const uint8_t* kc;
  const float* ks;
  const uint8_t* vc;
  const float* vs;
  const int32_t* seq_lens;
  float* out;
  float* ws_o;       // [B*H*max_splits][hd]
  float2* ws_ml;     // [B*H*max_splits]
  int* counters;     // [B*H]
  long long items;   // B*H*max_splits
  int H, Tc, blk_shift, max_splits;
  float scale_log2;  // softmax_scale * log2(e)
  float levels[16];
};

template <int HD>
struct DecodeShape {
  static constexpr int LPT = HD / 32;
  static constexpr int G = 32 / LPT;
  static constexpr int NT = kChunk / G;
};

template <int HD, int NW>
__global__ void __launch_bounds__(NW * 32, 1) decode_kernel(const DecodeParams p) {
  using S = DecodeShape<HD>;
  constexpr int LPT = S::LPT, G = S::G, NT = S::NT;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // pair LUT: entry e (a packed byte), replica r -> (L[e & 15], L[e >> 4])
  {
    float4* lut4 = reinterpret_cast<float4*>(smem);
    for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
      const int e = i >> 4;
      const float lo = p.levels[e & 15], hi = p.levels[e >> 4];
      lut4[i] = make_float4(lo, hi, lo, hi);
    }
  }
  float* red = reinterpret_cast<float*>(smem + kLutBytes) + warp * 1024;
  __syncthreads();
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const uint32_t lane8 = lane * 8u;   // replica of this lane inside a 256-B LUT entry
  const int g = lane / LPT, sub = lane % LPT;
  const int nblk = HD >> p.blk_shift;
  const int sidx = (sub * 32) >> p.blk_shift;

  for (long long it = static_cast<long long>(blockIdx.x) * NW + warp; it < p.items;
       it += static_cast<long long>(gridDim.x) * NW) {
    const int split = static_cast<int>(it % p.max_splits);
    const long long bh = it / p.max_splits;
    const int b = static_cast<int>(bh / p.H);
    const int len = min(p.seq_lens[b], p.Tc);
    const int nsplit = len > 0 ? (len + kChunk - 1) / kChunk : 1;
    if (split >= nsplit) continue;
    if (len <= 0) {   // empty sequence -> zeros (reading R12)
      for (int d = lane; d < HD; d += 32) p.out[bh * HD + d] = 0.0f;
      continue;
    }
    const int start = split * kChunk;
    const int end = min(len, start + kChunk);
    const long long row0 = bh * p.Tc;

    // issue every load of the chunk first (codes: 16 B per lane per token)
    uint4 kw[NT], vw[NT];
    float ksc[NT], vsc[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const int t = min(start + i * G + g, end - 1);
      const long long row = row0 + t;
      kw[i] = ldg_stream_128(p.kc + row * (HD / 2) + sub * 16);
      vw[i] = ldg_stream_128(p.vc + row * (HD / 2) + sub * 16);
      ksc[i] = ldg_f32(p.ks + row * nblk + sidx);
      vsc[i] = ldg_f32(p.vs + row * nblk + sidx);
    }
    // q for this lane's 32 dims as 16 fp32 pairs
    uint64_t q2[16];
    {
      const uint4* qp = reinterpret_cast<const uint4*>(p.q + bh * HD + sub * 32);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 r = __ldg(qp + j);
        const uint32_t w4[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          __half2 h2;
          memcpy(&h2, &w4[k], 4);
          const float2 f = __half22float2(h2);
          q2[j * 4 + k] = pack2(f.x, f.y);
        }
      }
    }
    // a5: scores
    float sc[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const uint32_t w4[4] = {kw[i].x, kw[i].y, kw[i].z, kw[i].w};
      uint64_t acc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          acc = ffma2(q2[j * 4 + k], lds64(__byte_perm(w4[j], lane8, 0x5504 | (k << 4)) + lut), acc);
      const float2 a = unpack2(acc);
      float part = (a.x + a.y) * ksc[i];
#pragma unroll
      for (int o = 1; o < LPT; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      sc[i] = (start + i * G + g < end) ? part * p.scale_log2 : -INFINITY;
    }
    float m = sc[0];
#pragma unroll
    for (int i = 1; i < NT; ++i) m = fmaxf(m, sc[i]);
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    // a6: P.V with w = p * scale
    uint64_t o2[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) o2[j] = 0;
    float l = 0.0f;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const float pr = fast_exp2(sc[i] - m);
      l += pr;
      const float w = pr * vsc[i];
      const uint64_t w2 = pack2(w, w);
      const uint32_t w4[4] = {vw[i].x, vw[i].y, vw[i].z, vw[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          o2[j * 4 + k] = ffma2(lds64(__byte_perm(w4[j], lane8, 0x5504 | (k << 4)) + lut), w2, o2[j * 4 + k]);
    }
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    // sum the G token groups: lane -> smem (16-byte chunks xor-swizzled)
    {
      float4* r4 = reinterpret_cast<float4*>(red);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float2 a = unpack2(o2[2 * c]), bb = unpack2(o2[2 * c + 1]);
        r4[lane * 8 + (c ^ (lane & 7))] = make_float4(a.x, a.y, bb.x, bb.y);
      }
    }
    __syncwarp();
    constexpr int DPL = HD / 32;   // output dims per lane
    float res[DPL];
#pragma unroll
    for (int d = 0; d < DPL; ++d) res[d] = 0.0f;
    {
      const int dim0 = lane * DPL;            // first dim this lane reduces
      const int src_sub = dim0 / 32, c = (dim0 % 32) / 4, off = dim0 % 4;
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const int sl = gg * LPT + src_sub;
        const float* src = red + (sl * 8 + (c ^ (sl & 7))) * 4 + off;
#pragma unroll
        for (int d = 0; d < DPL; ++d) res[d] += src[d];
      }
    }
    __syncwarp();
    float* dst;
    if (nsplit == 1) {
      const float inv = 1.0f / l;
      dst = p.out + bh * HD + lane * DPL;
#pragma unroll
      for (int d = 0; d < DPL; ++d) dst[d] = res[d] * inv;
      continue;
    }
    dst = p.ws_o + it * HD + lane * DPL;
#pragma unroll
    for (int d = 0; d < DPL; ++d) dst[d] = res[d];
    if (lane == 0) p.ws_ml[it] = make_float2(m, l);
    __threadfence();
    int prev = 0;
    if (lane == 0) prev = atomicAdd(p.counters + bh, 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != nsplit - 1) continue;
    // a7: last chunk to finish merges all partials in chunk order
    __threadfence();
    const long long base = bh * p.max_splits;
    float M = -INFINITY;
    for (int i = 0; i < nsplit; ++i) M = fmaxf(M, __ldcg(&p.ws_ml[base + i].x));
    float den = 0.0f;
    float acc[DPL];
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[d] = 0.0f;
    for (int i = 0; i < nsplit; ++i) {
      const float2 ml = __ldcg(&p.ws_ml[base + i]);
      const float f = fast_exp2(ml.x - M);
      den += f * ml.y;
      const float* src = p.ws_o + (base + i) * HD + lane * DPL;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[d] += f * __ldcg(src + d);
    }
    const float inv = 1.0f / den;
    dst = p.out + bh * HD + lane * DPL;
#pragma unroll
    for (int d = 0; d < DPL; ++d) dst[d] = acc[d] * inv;
    if (lane == 0) p.counters[bh] = 0;
  }
}

constexpr int kDecodeWarps = 8;
template <int HD>
constexpr size_t decode_smem() { return kLutBytes + kDecodeWarps * 1024 * sizeof(float); }

// ------------------------------------------------------------ host side
thread_local char g_err[256] = "";

int cuda_fail(cudaError_t e) {
  std::snprintf(g_err, sizeof(g_err), "%s", cudaGetErrorString(e));
  return NQKV_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int blk_shift_of(int blk) { return blk == 32 ? 5 : blk == 64 ? 6 : blk == 128 ? 7 : -1; }

int check_geometry(int hd, int blk) {
  if (hd != 64 && hd != 128) return NQKV_ERR_UNSUPPORTED;
  if (blk_shift_of(blk) < 0 || blk > hd) return NQKV_ERR_UNSUPPORTED;
  return NQKV_OK;
}

BucketTab make_bucket_tab() {
  BucketTab t;
  const BucketEntry* e = bucket_table();
  for (int i = 0; i < kNumBuckets; ++i) {
    float lo;
    std::memcpy(&lo, &e[i].lo, sizeof(lo));
    t.e[i] = make_float2(e[i].thr, lo);
  }
  return t;
}

int device_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return sms > 0 ? sms : 148;
}

long long grid_for(long long work, int threads, int per_sm) {
  long long blocks = (work + threads - 1) / threads;
  const long long cap = static_cast<long long>(device_sms()) * per_sm;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : blocks;
}

template <int HD>
int launch_decode(const DecodeParams& p, cudaStream_t st) {
  auto kern = decode_kernel<HD, kDecodeWarps>;
  constexpr size_t smem = decode_smem<HD>();
  static int blocks_per_sm = -1;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (blocks_per_sm < 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return cuda_fail(e);
      int n = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kDecodeWarps * 32, smem);
      if (e != cudaSuccess) return cuda_fail(e);
      blocks_per_sm = n > 0 ? n : 1;
    }
  }
  long long blocks = (p.items + kDecodeWarps - 1) / kDecodeWarps;
  const long long cap = static_cast<long long>(device_sms()) * blocks_per_sm;
  if (blocks > cap) blocks = cap;
  kern<<<static_cast<unsigned>(blocks), kDecodeWarps * 32, smem, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct WsLayout {
  size_t counters, ml, o, total;
};

WsLayout ws_layout(long long B, long long H, int hd, int Tc) {
  const long long ms = (Tc + kChunk - 1) / kChunk;
  WsLayout w;
  w.counters = 0;
  w.ml = align_up(static_cast<size_t>(B * H) * sizeof(int), 256);
  w.o = align_up(w.ml + static_cast<size_t>(B * H * ms) * sizeof(float2), 256);
  w.total = align_up(w.o + static_cast<size_t>(B * H * ms) * hd * sizeof(float), 256);
  return w;
}

}  // namespace nqkv

// ====================================================================== ABI
using namespace nqkv;

extern "C" {

int nqkv_abi_version(void) { return NQKV_ABI_VERSION; }

const char* nqkv_status_string(int status) {
  switch (status) {
    case NQKV_OK: return "ok";
    case NQKV_ERR_NULL: return "null pointer";
    case NQKV_ERR_SHAPE: return "invalid shape";
    case NQKV_ERR_UNSUPPORTED: return "unsupported head_dim/block size";
    case NQKV_ERR_ALIGN: return "misaligned pointer or stride";
    case NQKV_ERR_WORKSPACE: return "workspace too small";
    case NQKV_ERR_CUDA: return "CUDA error";
    case NQKV_ERR_INTERNAL: return "level table invariant violated";
    default: return "unknown status";
  }
}

const char* nqkv_last_error(void) { return g_err; }

int nqkv_levels(float levels[16]) {
  if (!levels) return NQKV_ERR_NULL;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  std::memcpy(levels, level_table(), 16 * sizeof(float));
  return NQKV_OK;
}

int nqkv_thresholds(float thresholds[15]) {
  if (!thresholds) return NQKV_ERR_NULL;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  std::memcpy(thresholds, threshold_table(), 15 * sizeof(float));
  return NQKV_OK;
}

int nqkv_quantize(const void* x, int64_t stride_b, int64_t stride_t, int64_t stride_h, int B,
                  int H, int hd, int n_new, int blk, const int32_t* d_pos, int Tc,
                  uint8_t* codes, float* scales, void* stream) {
  if (!x || !d_pos || !codes || !scales) return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  if (B < 0 || H < 0 || n_new < 0 || Tc <= 0 || Tc % 64) return NQKV_ERR_SHAPE;
  if (!aligned16(x) || !aligned16(codes) || (reinterpret_cast<uintptr_t>(scales) & 3u) ||
      (stride_b % 8) || (stride_t % 8) || (stride_h % 8))
    return NQKV_ERR_ALIGN;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  const long long total = static_cast<long long>(B) * n_new * H * (hd / 8);
  if (total == 0) return NQKV_OK;
  QuantParams p;
  p.x = static_cast<const __half*>(x);
  p.sb = stride_b; p.st = stride_t; p.sh = stride_h;
  p.pos = d_pos; p.codes = codes; p.scales = scales;
  p.total_chunks = total;
  p.H = H; p.hd = hd; p.n_new = n_new; p.Tc = Tc;
  p.blk_shift = blk_shift_of(blk);
  p.chunks_per_row = hd / 8;
  p.tab = make_bucket_tab();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>(grid_for(total, 256, 8));
  switch (blk) {
    case 32: quantize_kernel<4><<<grid, 256, 0, st>>>(p); break;
    case 64: quantize_kernel<8><<<grid, 256, 0, st>>>(p); break;
    default: quantize_kernel<16><<<grid, 256, 0, st>>>(p); break;
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

int nqkv_dequantize(const uint8_t* codes, const float* scales, int B, int H, int Tc, int hd,
                    int blk, int n_tokens, int out_dtype, void* out, void* stream) {
  if (!codes || !scales || !out) return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  if (B < 0 || H < 0 || Tc <= 0 || Tc % 64 || n_tokens < 0 || n_tokens > Tc)
    return NQKV_ERR_SHAPE;
  if (out_dtype != 0 && out_dtype != 1) return NQKV_ERR_UNSUPPORTED;
  if (!aligned16(codes) || !aligned16(out) || (reinterpret_cast<uintptr_t>(scales) & 3u))
    return NQKV_ERR_ALIGN;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  const long long total = static_cast<long long>(B) * H * n_tokens * (hd / 8);
  if (total == 0) return NQKV_OK;
  DequantParams p;
  p.codes = codes; p.scales = scales; p.out = out;
  p.total_chunks = total;
  p.Tc = Tc; p.hd = hd; p.n_tokens = n_tokens;
  p.blk_shift = blk_shift_of(blk);
  p.chunks_per_row = hd / 8;
  std::memcpy(p.levels, level_table(), sizeof(p.levels));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>(grid_for(total, 256, 8));
  if (out_dtype == 1) dequant_kernel<true><<<grid, 256, 0, st>>>(p);
  else dequant_kernel<false><<<grid, 256, 0, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

size_t nqkv_decode_workspace_bytes(int B, int H, int hd, int Tc) {
  if (B < 0 || H < 0 || Tc <= 0) return 0;
  return ws_layout(B, H, hd, Tc).total;
}

int nqkv_decode_attention(const void* q, const uint8_t* k_codes, const float* k_scales,
                          const uint8_t* v_codes, const float* v_scales,
                          const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                          float softmax_scale, float* out, void* workspace, size_t ws_bytes,
                          void* stream) {
  if (!q || !k_codes || !k_scales || !v_codes || !v_scales || !d_seq_lens || !out)
    return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  if (B < 0 || H < 0 || Tc <= 0 || Tc % 64) return NQKV_ERR_SHAPE;
  if (!aligned16(q) || !aligned16(k_codes) || !aligned16(v_codes) || !aligned16(out) ||
      (reinterpret_cast<uintptr_t>(k_scales) & 3u) || (reinterpret_cast<uintptr_t>(v_scales) & 3u))
    return NQKV_ERR_ALIGN;
  if (B == 0 || H == 0) return NQKV_OK;
  const WsLayout w = ws_layout(B, H, hd, Tc);
  if (!workspace) return NQKV_ERR_NULL;
  if (!aligned16(workspace)) return NQKV_ERR_ALIGN;
  if (ws_bytes < w.total) return NQKV_ERR_WORKSPACE;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  DecodeParams p;
  p.q = static_cast<const __half*>(q);
  p.kc = k_codes; p.ks = k_scales; p.vc = v_codes; p.vs = v_scales;
  p.seq_lens = d_seq_lens; p.out = out;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  p.counters = reinterpret_cast<int*>(ws + w.counters);
  p.ws_ml = reinterpret_cast<float2*>(ws + w.ml);
  p.ws_o = reinterpret_cast<float*>(ws + w.o);
  p.max_splits = (Tc + kChunk - 1) / kChunk;
  p.items = static_cast<long long>(B) * H * p.max_splits;
  p.H = H; p.Tc = Tc;
  p.blk_shift = blk_shift_of(blk);
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  std::memcpy(p.levels, level_table(), sizeof(p.levels));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return hd == 64 ? launch_decode<64>(p, st) : launch_decode<128>(p, st);
}

int nqkv_encode_normalized(const float* d_n, int64_t count, uint8_t* d_codes, void* stream) {
  if (!d_n || !d_codes) return NQKV_ERR_NULL;
  if (count < 0) return NQKV_ERR_SHAPE;
  if (count == 0) return NQKV_OK;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>(grid_for(count, 256, 8));
  encode_normalized_kernel<<<grid, 256, 0, st>>>(d_n, count, d_codes, make_bucket_tab());
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

}  // extern "C"
