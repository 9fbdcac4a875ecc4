// Prefill attention over the 4-bit cache.
//
// in the prefill phase the prompt's keys and values are
// quantised into the cache (I_K = quantize_NF4(X_K), I_V = quantize_NF4(X_V));
// the prompt's causal attention runs over the DEQUANTISED
// K, V so that prefill and decode see the same quantised values.  For query
// row i of sequence b: out_i = softmax_j<=i(q_i . k^_j / sqrt(hd)) . v^_j.
//
// A block of 64 queries against 64-token key tiles makes this a dense
// contraction, so it runs on the tensor cores (mma.sync m16n8k16, fp16 x fp16
// -> fp32; FlashAttention-2 structure: online softmax, P reused from the S
// accumulators as the A operand of P.V).  Exactness: the dequantised values
// k^ = RN32(s * L[code]) (as the oracle) are split into fp16 hi + lo parts
// (hi = RN16(k^), lo = RN16(k^ - hi): ~22 significant bits), q is fp16 (exact),
// products are exact in fp32 and accumulate in fp32; P is split the same way
// for P.V (P_hi V_hi + P_lo V_hi + P_hi V_lo).  The dequantised tiles live in
// shared memory only (never written to HBM).
//
// Layout: q fp16 [B][T][H][hd] (token-major, like the projections' output),
// out fp32 [B][T][H][hd]; rows i >= seq_lens[b] are written as 0.
#pragma once
#include "common.cuh"

namespace nqkv {

struct PrefillParams {
  const __half* q;
  const uint8_t* kc;
  const void* ks;
  const uint8_t* vc;
  const void* vs;
  const int32_t* seq_lens;
  float* out;
  int B, H, T, Tc, blk_shift, hpb_shift;
  float scale_log2;          // softmax_scale * log2(e)
  Levels lv;
  // KV layouts (tcgen05 kernel; readings R16, R17): query head h
  // reads cache head h >> kv_shift; paged cache: key t of sequence b is row
  // t & (P - 1) of page bt[b][t >> page_shift] in [n_pages][H_kv][P] storage
  int kv_shift;
  const int32_t* bt;         // nullptr: contiguous [B][H_kv][Tc]
  int bt_stride, page_shift;
};

constexpr int kPfW = 8;      // warps per CTA
constexpr int kPfQ = 16 * kPfW;   // queries per CTA (16 rows per warp): each dequantised tile serves them all
constexpr int kPfK = 64;     // keys per tile

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// (hi, lo) fp16 split of two fp32 values, packed as half2 pairs
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x - hf.x, y - hf.y);
  memcpy(&hi, &h, 4);
  memcpy(&lo, &l, 4);
}

template <int HD>
constexpr size_t prefill_smem_bytes() {
  return 4 * static_cast<size_t>(kPfK) * (HD + 8) * 2 + 64;
}
// B fragments (k = 16 keys, n = 8 dims) of P.V from V stored [key][dim]
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t& b0, uint32_t& b1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
               : "=r"(b0), "=r"(b1) : "r"(addr));
}

template <int HD, bool F16S, bool GRP>
__global__ void __launch_bounds__(kPfW * 32) prefill_kernel(const __grid_constant__ PrefillParams p) {
  constexpr int KS = HD + 8;          // K tile row stride (halves): conflict-free B-fragment loads
  constexpr int VS = HD + 8;          // V tile row stride (halves): conflict-free ldmatrix rows
  constexpr int NT = kPfW * 32;
  constexpr int NKT = kPfK / 8;       // n-tiles of S per warp
  constexpr int NDT = HD / 8;         // n-tiles of O per warp
  extern __shared__ __align__(16) unsigned char pf_smem[];
  __half* sKh = reinterpret_cast<__half*>(pf_smem);
  __half* sKl = sKh + kPfK * KS;
  __half* sVh = sKl + kPfK * KS;
  __half* sVl = sVh + kPfK * VS;
  float* s_lv = reinterpret_cast<float*>(sVl + kPfK * VS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  if (tid < 16) s_lv[tid] = p.lv.v[tid];
  pdl_enter();
  const int len = min(max(p.seq_lens[b], 0), p.T);
  const int q0 = qt * kPfQ;
  const long long rstride = static_cast<long long>(p.H) * HD;      // elements between tokens
  float* outb = p.out + (static_cast<long long>(b) * p.T) * rstride + static_cast<long long>(h) * HD;
  if (q0 >= len) {                    // rows beyond the prompt: zeros
    for (int i = tid; i < kPfQ * HD; i += NT) {
      const int r = q0 + i / HD;
      if (r < p.T) outb[r * rstride + (i % HD)] = 0.0f;
    }
    return;
  }
  // Q fragments of this warp's 16 rows (fp16, exact): A operand per 16-dim k-step
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
  const __half* qb = p.q + (static_cast<long long>(b) * p.T) * rstride + static_cast<long long>(h) * HD;
  uint32_t qa[HD / 16][4];
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) {
    const int d0 = ks * 16 + 2 * t;
    qa[ks][0] = r0 < len ? *reinterpret_cast<const uint32_t*>(qb + r0 * rstride + d0) : 0u;
    qa[ks][1] = r1 < len ? *reinterpret_cast<const uint32_t*>(qb + r1 * rstride + d0) : 0u;
    qa[ks][2] = r0 < len ? *reinterpret_cast<const uint32_t*>(qb + r0 * rstride + d0 + 8) : 0u;
    qa[ks][3] = r1 < len ? *reinterpret_cast<const uint32_t*>(qb + r1 * rstride + d0 + 8) : 0u;
  }
  float o[NDT][4];
#pragma unroll
  for (int j = 0; j < NDT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;   // rows r0, r1 (quad-partial sums)
  const long long row_base = (static_cast<long long>(b) * p.H + h) * p.Tc;
  const long long srow_base = GRP ? ((static_cast<long long>(b) * p.H + h) >> p.hpb_shift) * p.Tc : row_base;
  constexpr int NBLK_MAX = HD / 32;
  const int nblk = GRP ? 1 : HD >> p.blk_shift;
  const int last_key = min(q0 + kPfQ, len);                        // keys [0, last_key)
  for (int k0 = 0; k0 < last_key; k0 += kPfK) {
    __syncthreads();                  // previous tile fully consumed
    // ---- dequantise the K and V tiles: thread -> (token, 16 dims) x 2 passes
    for (int it = tid; it < kPfK * (HD / 16); it += NT) {
      const int tk = it / (HD / 16), c = it % (HD / 16);     // token in tile, 16-dim chunk
      const int tok = k0 + tk;
      float kv[16], vv[16];
      if (tok < len) {
        const uint2 kw = *reinterpret_cast<const uint2*>(p.kc + (row_base + tok) * (HD / 2) + c * 8);
        const uint2 vw = *reinterpret_cast<const uint2*>(p.vc + (row_base + tok) * (HD / 2) + c * 8);
        const long long si = GRP ? srow_base + tok : (row_base + tok) * nblk + ((c * 16) >> p.blk_shift);
        float sk, sv;
        if constexpr (F16S) {
          sk = __half2float(reinterpret_cast<const __half*>(p.ks)[si]);
          sv = __half2float(reinterpret_cast<const __half*>(p.vs)[si]);
        } else {
          sk = reinterpret_cast<const float*>(p.ks)[si];
          sv = reinterpret_cast<const float*>(p.vs)[si];
        }
        const uint32_t kw2[2] = {kw.x, kw.y}, vw2[2] = {vw.x, vw.y};
#pragma unroll
        for (int e = 0; e < 16; ++e) {       // element 2i low nibble of byte i
          const uint32_t kcd = (kw2[e >> 3] >> (4 * (e & 7))) & 15u;
          const uint32_t vcd = (vw2[e >> 3] >> (4 * (e & 7))) & 15u;
          kv[e] = __fmul_rn(sk, s_lv[kcd]);  // RN32(s * L[code]), as the oracle
          vv[e] = __fmul_rn(sv, s_lv[vcd]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) kv[e] = vv[e] = 0.0f;
      }
      uint32_t khi[8], klo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) split2(kv[2 * e], kv[2 * e + 1], khi[e], klo[e]);
      *reinterpret_cast<uint4*>(sKh + tk * KS + c * 16) = make_uint4(khi[0], khi[1], khi[2], khi[3]);
      *reinterpret_cast<uint4*>(sKh + tk * KS + c * 16 + 8) = make_uint4(khi[4], khi[5], khi[6], khi[7]);
      *reinterpret_cast<uint4*>(sKl + tk * KS + c * 16) = make_uint4(klo[0], klo[1], klo[2], klo[3]);
      *reinterpret_cast<uint4*>(sKl + tk * KS + c * 16 + 8) = make_uint4(klo[4], klo[5], klo[6], klo[7]);
      uint32_t vhi[8], vlo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) split2(vv[2 * e], vv[2 * e + 1], vhi[e], vlo[e]);
      *reinterpret_cast<uint4*>(sVh + tk * VS + c * 16) = make_uint4(vhi[0], vhi[1], vhi[2], vhi[3]);
      *reinterpret_cast<uint4*>(sVh + tk * VS + c * 16 + 8) = make_uint4(vhi[4], vhi[5], vhi[6], vhi[7]);
      *reinterpret_cast<uint4*>(sVl + tk * VS + c * 16) = make_uint4(vlo[0], vlo[1], vlo[2], vlo[3]);
      *reinterpret_cast<uint4*>(sVl + tk * VS + c * 16 + 8) = make_uint4(vlo[4], vlo[5], vlo[6], vlo[7]);
    }
    (void)NBLK_MAX;
    __syncthreads();
    // ---- S = Q K^T (16 rows x 64 keys per warp), log2 domain, causal mask
    float sacc[NKT][4];
#pragma unroll
    for (int n = 0; n < NKT; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
      for (int n = 0; n < NKT; ++n) {
        const __half* kr = sKh + (n * 8 + g) * KS + ks * 16 + 2 * t;
        const __half* kl = sKl + (n * 8 + g) * KS + ks * 16 + 2 * t;
        mma16816(sacc[n], qa[ks], *reinterpret_cast<const uint32_t*>(kr), *reinterpret_cast<const uint32_t*>(kr + 8));
        mma16816(sacc[n], qa[ks], *reinterpret_cast<const uint32_t*>(kl), *reinterpret_cast<const uint32_t*>(kl + 8));
      }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < NKT; ++n) {
      const int j0 = k0 + n * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = j0 + (e & 1), r = (e & 2) ? r1 : r0;
        const bool ok = j <= r && j < len;
        sacc[n][e] = ok ? sacc[n][e] * p.scale_log2 : -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(sacc[n][0], sacc[n][1]));
      mx1 = fmaxf(mx1, fmaxf(sacc[n][2], sacc[n][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    // rows with no valid key yet keep m = -inf: subtract 0 there
    const float c0 = mn0 == -INFINITY ? 1.0f : fast_exp2(m0 - mn0);
    const float c1 = mn1 == -INFINITY ? 1.0f : fast_exp2(m1 - mn1);
    const float b0 = mn0 == -INFINITY ? 0.0f : mn0, b1 = mn1 == -INFINITY ? 0.0f : mn1;
    m0 = mn0;
    m1 = mn1;
    l0 *= c0;
    l1 *= c1;
#pragma unroll
    for (int j = 0; j < NDT; ++j) {
      o[j][0] *= c0;
      o[j][1] *= c0;
      o[j][2] *= c1;
      o[j][3] *= c1;
    }
#pragma unroll
    for (int n = 0; n < NKT; ++n) {
      sacc[n][0] = fast_exp2(sacc[n][0] - b0);
      sacc[n][1] = fast_exp2(sacc[n][1] - b0);
      sacc[n][2] = fast_exp2(sacc[n][2] - b1);
      sacc[n][3] = fast_exp2(sacc[n][3] - b1);
      l0 += sacc[n][0] + sacc[n][1];
      l1 += sacc[n][2] + sacc[n][3];
    }
    // ---- O += P V: P from the S accumulators (two n8 tiles = one k16 A fragment)
#pragma unroll
    for (int kk = 0; kk < kPfK / 16; ++kk) {
      uint32_t ph[4], pl[4];
      split2(sacc[2 * kk][0], sacc[2 * kk][1], ph[0], pl[0]);
      split2(sacc[2 * kk][2], sacc[2 * kk][3], ph[1], pl[1]);
      split2(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1], ph[2], pl[2]);
      split2(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3], ph[3], pl[3]);
      // ldmatrix.trans row addresses: lanes 0-15 -> keys kk*16 + (lane & 15)
      const uint32_t vrow = static_cast<uint32_t>(((kk * 16 + (lane & 15)) * VS) * 2);
      const uint32_t vh_base = static_cast<uint32_t>(__cvta_generic_to_shared(sVh)) + vrow;
      const uint32_t vl_base = static_cast<uint32_t>(__cvta_generic_to_shared(sVl)) + vrow;
#pragma unroll
      for (int j = 0; j < NDT; ++j) {
        uint32_t vh0, vh1, vl0, vl1;
        ldsm_x2_trans(vh_base + j * 16, vh0, vh1);
        ldsm_x2_trans(vl_base + j * 16, vl0, vl1);
        mma16816(o[j], ph, vh0, vh1);
        mma16816(o[j], pl, vh0, vh1);
        mma16816(o[j], ph, vl0, vl1);
      }
    }
  }
  // ---- normalise and store (rows < len)
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.0f / l0, i1 = 1.0f / l1;
#pragma unroll
  for (int j = 0; j < NDT; ++j) {
    const int d = j * 8 + 2 * t;
    if (r0 < p.T)
      *reinterpret_cast<float2*>(outb + r0 * rstride + d) =
          r0 < len ? make_float2(o[j][0] * i0, o[j][1] * i0) : make_float2(0.0f, 0.0f);
    if (r1 < p.T)
      *reinterpret_cast<float2*>(outb + r1 * rstride + d) =
          r1 < len ? make_float2(o[j][2] * i1, o[j][3] * i1) : make_float2(0.0f, 0.0f);
  }
}

}  // namespace nqkv
