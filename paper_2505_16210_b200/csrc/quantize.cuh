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
  float* scales;
  int B, n_new, H, Tc, blk_shift;
  BucketTab tab;
};

// Quantize one 16-byte chunk (8 fp16 values) against the block absmax shared
// by the GS lanes of its block; returns the 8 packed nibbles.
template <int GS>
__device__ __forceinline__ uint32_t quantize_chunk(const uint4 raw, uint32_t tabc, float& s) {
  s = absmax8(raw);
#pragma unroll
  for (int o = 1; o < GS; o <<= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
  return encode8c(raw, block_rcp(s), tabc);
}

// A warp owns one token row (b, t) at a time: the row's (b, t) decode, the
// append position and base pointers are computed once per row; the lanes then
// sweep the row's H * hd/8 chunks, two per lane per step (both loads issued
// before either is used).  blk/8 consecutive lanes form a block and reduce its
// absmax with xor-shuffles (a 32-chunk step always holds whole heads).
template <int HD, int GS>   // GS = lanes per block = blk / 8
__global__ void __launch_bounds__(256) quantize_kernel(const QuantParams p) {
  constexpr int CPR = HD / 8;                  // chunks per (token, head)
  constexpr int LOG_CPR = CPR == 8 ? 3 : 4;
  __shared__ float2 s_tab[kNumBuckets];
  for (int i = threadIdx.x; i < kNumBuckets; i += blockDim.x) s_tab[i] = p.tab.e[i];
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  const uint32_t tabc = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab)) - 0x5A000000u;
  const int lane = threadIdx.x & 31;
  const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  const int rows = p.B * p.n_new;
  const int chunks = p.H * CPR;
  const int nblk = HD >> p.blk_shift;
  for (int row = gw; row < rows; row += nw) {
    const int b = row / p.n_new, t = row - b * p.n_new;
    const int pos = __ldg(p.pos + b) + t;
    const bool in_range = pos >= 0 && pos < p.Tc;
    const __half* xrow = p.x + b * p.sb + t * p.st;
    const long long orow = static_cast<long long>(b) * p.H * p.Tc + pos;   // + h*Tc
    for (int c0 = 0; c0 < chunks; c0 += 64) {
      const int ca = c0 + lane, cb = c0 + 32 + lane;
      const bool va = ca < chunks, vb = cb < chunks;
      uint4 ra = make_uint4(0, 0, 0, 0), rb = ra;
      if (va) ra = ldg_stream_128(xrow + (ca >> LOG_CPR) * p.sh + (ca & (CPR - 1)) * 8);
      if (vb) rb = ldg_stream_128(xrow + (cb >> LOG_CPR) * p.sh + (cb & (CPR - 1)) * 8);
      float sa, sb;
      const uint32_t wa = quantize_chunk<GS>(ra, tabc, sa);
      if (c0 + 32 < chunks) {                // warp-uniform
        const uint32_t wb = quantize_chunk<GS>(rb, tabc, sb);
        if (vb && in_range) {
          const long long r = orow + static_cast<long long>(cb >> LOG_CPR) * p.Tc;
          reinterpret_cast<uint32_t*>(p.codes + r * (HD / 2))[cb & (CPR - 1)] = wb;
          if ((cb & (GS - 1)) == 0) p.scales[r * nblk + ((cb & (CPR - 1)) / GS)] = sb;
        }
      }
      if (va && in_range) {
        const long long r = orow + static_cast<long long>(ca >> LOG_CPR) * p.Tc;
        reinterpret_cast<uint32_t*>(p.codes + r * (HD / 2))[ca & (CPR - 1)] = wa;
        if ((ca & (GS - 1)) == 0) p.scales[r * nblk + ((ca & (CPR - 1)) / GS)] = sa;
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
  Levels lv;
};

template <bool F16>
__global__ void __launch_bounds__(256) dequant_kernel(const DequantParams p) {
  __shared__ float s_lv[16];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) s_lv[k] = p.lv.v[k];
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();
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
