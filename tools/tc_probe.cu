// Development probe (not part of the library): one CTA computes
// D[128 x N] = A[128 x K] . B[N x K]^T with tcgen05.mma (kind::f16, fp32
// accumulate in TMEM), operands K-major in shared memory in the no-swizzle
// canonical layout (8-row x 16-byte core matrices), and reads D back with
// tcgen05.ld.32x32b -- to validate the descriptor encodings used by the
// prefill kernel.  Also the MN-major B variant (B stored [K][N]).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tcp.bin tools/tc_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int M = 128;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;     // version 1 (sm100)
  return d;                                // base offset 0, lbo mode 0, SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n, bool b_mn) {
  return (1u << 4) | (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// K-major canonical: element (r, k) of an R x K operand at
// ((r/8) * (K/8) + k/8) * 128 + (r%8) * 16 + (k%8) * 2 bytes
__device__ __forceinline__ uint32_t kmaj_off(int r, int k, int K) {
  return static_cast<uint32_t>(((r >> 3) * (K >> 3) + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
// MN-major canonical (B stored with N contiguous): element (n, k) at
// ((k/8) * (N/8) + n/8) * 128 + (k%8) * 16 + (n%8) * 2 bytes
__device__ __forceinline__ uint32_t mnmaj_off(int n, int k, int N) {
  return static_cast<uint32_t>(((k >> 3) * (N >> 3) + (n >> 3)) * 128 + (k & 7) * 16 + (n & 7) * 2);
}

template <int N, int K, bool BMN>
__global__ void __launch_bounds__(128) probe(const __half* A, const __half* B, float* D, uint32_t lbo_b,
                                           uint32_t sbo_b) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sA = sm;
  unsigned char* sB = sm + M * K * 2;
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += 128) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sA + kmaj_off(r, k, K)) = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + (BMN ? mnmaj_off(n, k, N) : kmaj_off(n, k, K))) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
                     "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem))), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar))));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
  if (tid == 0) {
    const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sA));
    const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sB));
    constexpr uint32_t id = idesc_f16(M, N, BMN);
#pragma unroll
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t ad = sdesc(a0 + s * 256, 128, (K / 8) * 128);
      const uint64_t bd = BMN ? sdesc(b0 + s * 2 * (N / 8) * 128, lbo_b, sbo_b)
                              : sdesc(b0 + s * 256, 128, (K / 8) * 128);
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
          :: "r"(tmem), "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
      :: "r"(mbar) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // row = tid: TMEM lane tid, columns 0..N-1
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(128));
}


// A in TMEM: row r of A at TMEM lane r, K elements packed two fp16 per 32-bit
// column (element 2c in the low half).  B K-major in shared memory.
template <int N, int K>
__global__ void __launch_bounds__(128) probe_ta(const __half* A, const __half* B, float* D, int swap_halves) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sB = sm;
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + kmaj_off(n, k, K)) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
                     "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem))), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar))));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const uint32_t ta = tmem + 128;            // A columns [128, 128 + K/2)
  // row tid -> lane tid
  for (int c = 0; c < K / 2; ++c) {
    __half lo = A[tid * K + 2 * c], hi = A[tid * K + 2 * c + 1];
    if (swap_halves) { __half t = lo; lo = hi; hi = t; }
    const uint32_t w = static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(ta + (static_cast<uint32_t>(warp * 32) << 16) + c), "r"(w) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
  if (tid == 0) {
    const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sB));
    constexpr uint32_t id = idesc_f16(M, N, false);
#pragma unroll
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t bd = sdesc(b0 + s * 256, 128, (K / 8) * 128);
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
          :: "r"(tmem), "r"(ta + s * 8), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
      :: "r"(mbar) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(256));
}

template <int N, int K, bool BMN>
bool run(const char* name, uint32_t lbo_b = 0, uint32_t sbo_b = 0) {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  for (int i = 0; i < M * K; ++i) { Af[i] = static_cast<float>((i * 7 + 3) % 11 - 5); A[i] = __float2half(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = static_cast<float>((i * 5 + 1) % 9 - 4); B[i] = __float2half(Bf[i]); }
  __half *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, M * K * 2));
  CK(cudaMalloc(&dB, N * K * 2));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, M * N * 4));
  const int smem = (M + N) * K * 2;
  CK(cudaFuncSetAttribute(probe<N, K, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<N, K, BMN><<<1, 128, smem>>>(dA, dB, dD, lbo_b, sbo_b);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> D(M * N);
  CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < K; ++k) ref += Af[r * K + k] * Bf[n * K + k];
      if (D[r * N + n] != ref) {
        if (bad < 5) printf("  mismatch r=%d n=%d got %f want %f\n", r, n, D[r * N + n], ref);
        ++bad;
      }
    }
  printf("%-40s %s (%d bad)\n", name, bad ? "FAIL" : "ok", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}


template <int N, int K>
bool run_ta(const char* name, int swap) {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  for (int i = 0; i < M * K; ++i) { Af[i] = static_cast<float>((i * 7 + 3) % 11 - 5); A[i] = __float2half(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = static_cast<float>((i * 5 + 1) % 9 - 4); B[i] = __float2half(Bf[i]); }
  __half *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, M * K * 2));
  CK(cudaMalloc(&dB, N * K * 2));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, M * N * 4));
  const int smem = N * K * 2;
  CK(cudaFuncSetAttribute(probe_ta<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_ta<N, K><<<1, 128, smem>>>(dA, dB, dD, swap);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> D(M * N);
  CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < K; ++k) ref += Af[r * K + k] * Bf[n * K + k];
      if (D[r * N + n] != ref) {
        if (bad < 3) printf("  mismatch r=%d n=%d got %f want %f\n", r, n, D[r * N + n], ref);
        ++bad;
      }
    }
  printf("%-40s %s (%d bad)\n", name, bad ? "FAIL" : "ok", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  if (argc > 1 && argv[1][0] == 't') {   // A in TMEM
    run_ta<64, 64>("A in TMEM, N=64, K=64, even elem low", 0);
    run_ta<64, 64>("A in TMEM, N=64, K=64, even elem high", 1);
    run_ta<128, 64>("A in TMEM, N=128, K=64, even elem low", 0);
    return 0;
  }
  if (argc > 1) {       // MN-major only, the layout the prefill kernel uses
    return run<128, 64, true>("MN-major B, N=128, K=64, lbo=K-grp sbo=N-grp", (128 / 8) * 128, 128) &&
           run<64, 64, true>("MN-major B, N=64, K=64, lbo=K-grp sbo=N-grp", (64 / 8) * 128, 128) ? 0 : 1;
  }
  run<64, 16, false>("K-major B, N=64, K=16");
  run<64, 128, false>("K-major B, N=64, K=128");
  run<128, 64, false>("K-major B, N=128, K=64");
  // MN-major B (N contiguous): LBO = byte stride of K groups, SBO = of N groups
  // (the swapped assignment faults: the unit reads outside the operand)
  run<128, 64, true>("MN-major B, N=128, K=64", (128 / 8) * 128, 128);
  run<64, 64, true>("MN-major B, N=64, K=64", (64 / 8) * 128, 128);
  return 0;
}
