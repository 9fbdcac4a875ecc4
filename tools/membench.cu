// Development microbenchmark (not part of the library): HBM read bandwidth of
// the decode kernel's access pattern vs a plain streaming read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench tools/membench.cu
//   /tmp/membench [MB]
// A: grid-stride 16-byte loads over one buffer.
// B: decode-like: codes [rows][64 B] x2 (K, V) + scales [rows][8 B] x2; one CTA
//    per SM owns a contiguous row range; warp w takes 16-row stages w, w+NC,...;
//    lane (g, sub) loads 8 B of rows g + 4i (i < 4) -- D stages kept in flight
//    in registers.
// C: as B, but each warp streams its stages with TMA bulk copies into a
//    per-warp shared-memory ring of depth D (mbarrier completion).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void stream_read(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint2 ld64(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld32(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

template <int D>
__global__ void __launch_bounds__(512, 1) decode_like(const uint8_t* kc, const uint8_t* vc, const float* ks,
                                                      const float* vs, int rows, unsigned* out) {
  constexpr int NC = 16, ST = 16;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / 8, sub = lane % 8;
  const long long r0 = (long long)blockIdx.x * rows / gridDim.x, r1 = (long long)(blockIdx.x + 1) * rows / gridDim.x;
  const int nst = (int)((r1 - r0) / ST);
  uint2 K[D][4], V[D][4];
  float S[D][4], T[D][4];
  unsigned acc = 0;
  auto load = [&](int d, int s) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long r = r0 + (long long)s * ST + i * 4 + g;
      K[d][i] = ld64(kc + r * 64 + sub * 8);
      V[d][i] = ld64(vc + r * 64 + sub * 8);
      S[d][i] = ld32(ks + r * 2 + (sub >> 2));
      T[d][i] = ld32(vs + r * 2 + (sub >> 2));
    }
  };
  int s = warp;
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (s + d * NC < nst) load(d, s + d * NC);
  for (; s < nst; s += D * NC) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (s + d * NC >= nst) break;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        acc ^= K[d][i].x ^ K[d][i].y ^ V[d][i].x ^ V[d][i].y ^ __float_as_uint(S[d][i]) ^ __float_as_uint(T[d][i]);
      if (s + (d + D) * NC < nst) load(d, s + (d + D) * NC);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_tx(uint32_t a, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(a), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(dst), "l"(src), "r"(bytes), "r"(mb) : "memory");
}

template <int D>
__global__ void __launch_bounds__(512, 1) decode_like_tma(const uint8_t* kc, const uint8_t* vc, const float* ks,
                                                          const float* vs, int rows, unsigned* out) {
  constexpr int NC = 16, ST = 16, SLOT = ST * 64 * 2 + ST * 8 * 2;
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / 8, sub = lane % 8;
  unsigned char* ring = sm + warp * (D * SLOT + 64);
  const uint32_t rs = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t mb = rs + D * SLOT;
  if (lane < D) mbar_init(mb + 8 * lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long r0 = (long long)blockIdx.x * rows / gridDim.x, r1 = (long long)(blockIdx.x + 1) * rows / gridDim.x;
  const int nst = (int)((r1 - r0) / ST);
  auto issue = [&](int d, int s) {
    if (lane == 0) {
      const long long r = r0 + (long long)s * ST;
      const uint32_t dst = rs + d * SLOT, m = mb + 8 * d;
      mbar_tx(m, SLOT);
      tma1d(dst, kc + r * 64, ST * 64, m);
      tma1d(dst + ST * 64, vc + r * 64, ST * 64, m);
      tma1d(dst + ST * 128, ks + r * 2, ST * 8, m);
      tma1d(dst + ST * 136, vs + r * 2, ST * 8, m);
    }
  };
  unsigned acc = 0;
  int s = warp, it = 0;
  for (int d = 0; d < D; ++d)
    if (s + d * NC < nst) issue(d, s + d * NC);
  for (; s < nst; s += NC, ++it) {
    const int d = it % D;
    mbar_wait(mb + 8 * d, (it / D) & 1);
    const unsigned char* sl = ring + d * SLOT;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = i * 4 + g;
      const uint2 k = *reinterpret_cast<const uint2*>(sl + r * 64 + sub * 8);
      const uint2 v = *reinterpret_cast<const uint2*>(sl + ST * 64 + r * 64 + sub * 8);
      const float a = reinterpret_cast<const float*>(sl + ST * 128)[r * 2 + (sub >> 2)];
      const float b = reinterpret_cast<const float*>(sl + ST * 136)[r * 2 + (sub >> 2)];
      acc ^= k.x ^ k.y ^ v.x ^ v.y ^ __float_as_uint(a) ^ __float_as_uint(b);
    }
    __syncwarp();
    if (s + D * NC < nst) issue(d, s + D * NC);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  std::vector<float> ts;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

#include <algorithm>
int main(int argc, char** argv) {
  const size_t MB = argc > 1 ? atoi(argv[1]) : 1024;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  CK(cudaMalloc(&out, 4));
  // A
  const size_t nbytes = MB << 20;
  uint4* buf;
  CK(cudaMalloc(&buf, nbytes));
  cudaMemset(buf, 1, nbytes);
  for (int tpb : {256, 512, 1024}) {
    for (int per : {1, 2, 4}) {
      float ms = timeit([&] { stream_read<<<sms * per, tpb>>>(buf, nbytes / 16, out); });
      printf("A stream_read  grid %4d x %4d: %7.1f GB/s\n", sms * per, tpb, nbytes / ms / 1e6);
    }
  }
  CK(cudaFree(buf));
  // B/C: rows such that the four tensors total ~MB
  const int rows = (int)((nbytes / 144) / (sms * 256)) * sms * 256;
  uint8_t *kc, *vc;
  float *ks, *vs;
  CK(cudaMalloc(&kc, (size_t)rows * 64));
  CK(cudaMalloc(&vc, (size_t)rows * 64));
  CK(cudaMalloc(&ks, (size_t)rows * 8));
  CK(cudaMalloc(&vs, (size_t)rows * 8));
  cudaMemset(kc, 3, (size_t)rows * 64);
  cudaMemset(vc, 5, (size_t)rows * 64);
  cudaMemset(ks, 0, (size_t)rows * 8);
  cudaMemset(vs, 0, (size_t)rows * 8);
  const double tot = (double)rows * 144;
  float ms;
  ms = timeit([&] { decode_like<1><<<sms, 512>>>(kc, vc, ks, vs, rows, out); });
  printf("B regs D=1: %7.1f GB/s\n", tot / ms / 1e6);
  ms = timeit([&] { decode_like<2><<<sms, 512>>>(kc, vc, ks, vs, rows, out); });
  printf("B regs D=2: %7.1f GB/s\n", tot / ms / 1e6);
  ms = timeit([&] { decode_like<3><<<sms, 512>>>(kc, vc, ks, vs, rows, out); });
  printf("B regs D=3: %7.1f GB/s\n", tot / ms / 1e6);
  CK(cudaGetLastError());
  for (int D : {2, 4, 6}) {
    const int SLOT = 16 * 64 * 2 + 16 * 8 * 2;
    const size_t smem = 16 * (D * SLOT + 64);
    if (D == 2) { CK(cudaFuncSetAttribute(decode_like_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); ms = timeit([&] { decode_like_tma<2><<<sms, 512, smem>>>(kc, vc, ks, vs, rows, out); }); }
    if (D == 4) { CK(cudaFuncSetAttribute(decode_like_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); ms = timeit([&] { decode_like_tma<4><<<sms, 512, smem>>>(kc, vc, ks, vs, rows, out); }); }
    if (D == 6) { CK(cudaFuncSetAttribute(decode_like_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); ms = timeit([&] { decode_like_tma<6><<<sms, 512, smem>>>(kc, vc, ks, vs, rows, out); }); }
    CK(cudaGetLastError());
    printf("C tma  D=%d (%zu KB smem): %7.1f GB/s\n", D, smem >> 10, tot / ms / 1e6);
  }
  return 0;
}
