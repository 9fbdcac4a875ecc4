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
  uint32_t rows;                 // B * n_new * H
  FastDiv divH, divN;
  int H, n_new, Tc, blk_shift;
  BucketTab tab;
};

// One thread = one 8-element chunk (16 B of fp16); blk/8 consecutive lanes
// form a block and reduce the absmax with xor-shuffles.  A warp covers
// 32/(HD/8) consecutive (b, t, h) rows per iteration.
template <int HD, int GS>   // GS = lanes per block = blk / 8
__global__ void __launch_bounds__(256) quantize_kernel(const QuantParams p) {
  constexpr int CPR = HD / 8, RPW = 32 / CPR;
  __shared__ float2 s_tab[kNumBuckets];
  for (int i = threadIdx.x; i < kNumBuckets; i += blockDim.x) s_tab[i] = p.tab.e[i];
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  const uint32_t tab = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
  const int lane = threadIdx.x & 31;
  const int cr = lane % CPR;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r0 = gwarp * RPW; r0 < p.rows; r0 += nwarp * RPW) {
    const uint32_t r = r0 + lane / CPR;
    const bool valid = r < p.rows;
    const uint32_t rr = valid ? r : 0;
    const uint32_t bt = fdiv(rr, p.divH);
    const int h = static_cast<int>(rr - bt * p.H);
    const uint32_t b = fdiv(bt, p.divN);
    const int t = static_cast<int>(bt - b * p.n_new);
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (valid) raw = ldg_stream_128(p.x + b * p.sb + t * p.st + h * p.sh + cr * 8);
    float s = absmax8(raw);
#pragma unroll
    for (int o = 1; o < GS; o <<= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
    const uint32_t word = encode8(raw, block_rcp(s), tab);
    if (valid) {
      const int row = p.pos[b] + t;
      if (row >= 0 && row < p.Tc) {
        const long long rowid = (static_cast<long long>(b) * p.H + h) * p.Tc + row;
        reinterpret_cast<uint32_t*>(p.codes + rowid * (HD / 2))[cr] = word;
        if ((cr & (GS - 1)) == 0) p.scales[rowid * (HD >> p.blk_shift) + cr / GS] = s;
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
