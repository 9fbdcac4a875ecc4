// Device helpers shared by the NQKV kernels: vector loads, fp32x2 math,
// PDL control, the exact NF4 code function and block encoding.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "nqkv_internal.h"

namespace nqkv {

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ uint4 ldg_stream_128(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream_64(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
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
// fp32x2 fma / mul (SASS FFMA2 / FMUL2, sm_100)
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
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
// Programmatic dependent launch: wait for the previous kernel before touching
// its outputs, then let the next kernel in the stream start its prologue.
// Every kernel here triggers only AFTER its own wait, so a kernel that runs
// knows that all kernels before its immediate predecessor have completed.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
__device__ __forceinline__ int atom_add_relaxed(int* p, int v) {
  int r;
  asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
// Tagged 64-bit words (value bits | tag << 32): an aligned 64-bit relaxed
// access is single-copy atomic, so a reader that sees the tag also sees the
// value written with it -- no fence or acquire needed.
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Fast unsigned division by a runtime constant (n < 2^31).
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d > 1) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.s = s;
    f.m = static_cast<uint32_t>(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  }
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return static_cast<uint32_t>((static_cast<uint64_t>(__umulhi(n, f.m)) + n) >> f.s);
}

// ------------------------------------------------------- a2: code function
// n in [-1, 1].  idx = RN(16 n + 16) is produced exactly by one fma against
// the magic constant 1.5*2^23 + 16 (unit ulp); bucket idx covers
// [(idx-16.5)/16, (idx-15.5)/16] and holds at most one decision threshold
// (host-checked), so code = lo[idx] + (n > thr[idx]) is exactly
// #{i : n > T_i} = argmin_i |n - L_i| with ties to the lower index.
__device__ __forceinline__ uint32_t nf4_code(float n, uint32_t tab_base) {
  const float y = __fmaf_rn(n, 16.0f, 12582928.0f);
  // (bits - 0x4B400000) * 8 + tab_base as a single IMAD
  const float2 e = unpack2(lds64(__float_as_uint(y) * 8u + (tab_base - 0x5A000000u)));
  return __float_as_uint(e.y) + (n > e.x ? 1u : 0u);
}

// Same code function with the table base pre-folded: tabc = tab_base - 0x5A000000,
// so the entry address is ONE integer multiply-add of the fma result's bits;
// the comparison is a set.gt mask subtracted from lo (no predicate/select).
__device__ __forceinline__ uint32_t nf4_code_c(float n, uint32_t tabc) {
  const float y = __fmaf_rn(n, 16.0f, 12582928.0f);
  uint32_t addr;
  asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(addr) : "r"(__float_as_uint(y)), "r"(tabc));
  const float2 e = unpack2(lds64(addr));
  uint32_t gt;
  asm("set.gt.u32.f32 %0, %1, %2;" : "=r"(gt) : "f"(n), "f"(e.x));
  return __float_as_uint(e.y) - gt;       // gt = 0xFFFFFFFF (true) or 0
}

// Normalisation n' = RN32(x * RN32(1/s)).  For every fp16 pair with |x| <= s
// this yields the same code as n = RN32(x / s) (exhaustive proof:
// tests/test_exactness_cpu.py; GPU sweep: tests/test_gpu_parity.py).
__device__ __forceinline__ float block_rcp(float s) { return s > 0.0f ? __frcp_rn(s) : 0.0f; }

// Quantize 8 fp16 values (one uint4) with reciprocal scale r -> 8 nibbles.
__device__ __forceinline__ uint32_t encode8(const uint4 raw, float r, uint32_t tab) {
  __half2 hv[4];
  memcpy(hv, &raw, 16);
  uint32_t word = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 xf = __half22float2(hv[k]);
    word |= nf4_code(__fmul_rn(xf.x, r), tab) << (8 * k);
    word |= nf4_code(__fmul_rn(xf.y, r), tab) << (8 * k + 4);
  }
  return word;
}
// encode8 with the pre-folded table constant (see nf4_code_c); nibble pairs are
// combined with one multiply-add each.
__device__ __forceinline__ uint32_t encode8c(const uint4 raw, float r, uint32_t tabc) {
  __half2 hv[4];
  memcpy(hv, &raw, 16);
  uint32_t b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 xf = __half22float2(hv[k]);
    const uint32_t lo = nf4_code_c(__fmul_rn(xf.x, r), tabc);
    const uint32_t hi = nf4_code_c(__fmul_rn(xf.y, r), tabc);
    b[k] = hi * 16u + lo;
  }
  return __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
}
__device__ __forceinline__ float absmax8(const uint4 raw) {
  __half2 hv[4];
  memcpy(hv, &raw, 16);
  const __half2 am = __hmax2(__hmax2(__habs2(hv[0]), __habs2(hv[1])),
                             __hmax2(__habs2(hv[2]), __habs2(hv[3])));
  return fmaxf(__low2float(am), __high2float(am));
}

struct BucketTab {
  float2 e[kNumBuckets];   // {thr, lo (uint bits)}
};
struct Levels {
  float v[16];
};

}  // namespace nqkv
