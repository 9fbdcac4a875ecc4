// NQKV hot path for B200 (sm_100a): NF4 quantize/pack/append, standalone
// dequantize, and fused dequant-in-registers split-K decode attention (with
// an optional fused 1-token append).  The C ABI (include/nqkv.h) is at the
// bottom of this file.
//
// Paper: PAPER.md:193 (block-wise quantile quantisation, index-table lookup),
// :205 (prefill quantisation, 4-bit index storage), :219-235 (decode:
// quantize the new token, Concat, dequantize, Softmax(t_Q X_K'^T), A X_V').
// The paper's own GPU design (materialise an fp16 copy of the whole cache,
// pad to 16 tokens, Cutlass BMM) is NOT followed: decode
// streams the packed nibbles from HBM and dequantises them in registers, so
// the only HBM traffic is the 4-bit codes + scales (+ q in, out).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>

#include "../../include/nqkv.h"
#include "common.cuh"
#include "decode.cuh"
#include "decode_gqa.cuh"
#include "nqkv_internal.h"
#include "quantize.cuh"
#include "prefill.cuh"
#include "prefill_tc.cuh"

namespace nqkv {

// ------------------------------------------------------------ host side
thread_local char g_err[256] = "";

int cuda_fail(cudaError_t e) {
  std::snprintf(g_err, sizeof(g_err), "%s", cudaGetErrorString(e));
  return NQKV_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int blk_shift_of(int blk) {
  return blk == 32 ? 5 : blk == 64 ? 6 : blk == 128 ? 7 : blk == 256 ? 8 : -1;
}

int check_geometry(int hd, int blk) {
  if (hd != 64 && hd != 128) return NQKV_ERR_UNSUPPORTED;
  if (blk & ~(0x1ff | NQKV_SCALE_F16)) return NQKV_ERR_UNSUPPORTED;
  blk &= 0x1ff;
  if (blk_shift_of(blk) < 0) return NQKV_ERR_UNSUPPORTED;   // powers of 2: blk | hd or hd | blk
  return NQKV_OK;
}
// blk argument -> (block size, scales stored as fp16)
int blk_of(int blk) { return blk & 0x1ff; }
// blk > hd: a block spans 2^hpb_shift adjacent heads (one scale per head group)
int hpb_shift_of(int hd, int blk) { return blk > hd ? blk_shift_of(blk) - blk_shift_of(hd) : 0; }
bool heads_fit(int H, int hd, int blk) { return H % (1 << hpb_shift_of(hd, blk_of(blk))) == 0; }
bool f16s_of(int blk) { return (blk & NQKV_SCALE_F16) != 0; }
bool scale_aligned(const void* p, bool f16s) {
  return (reinterpret_cast<uintptr_t>(p) & (f16s ? 1u : 3u)) == 0;
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

Levels make_levels() {
  Levels l;
  std::memcpy(l.v, level_table(), sizeof(l.v));
  return l;
}

int device_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return sms > 0 ? sms : 148;
}

// One decode CTA per SM (a CTA fills an SM's registers and shared memory),
// or fewer when NQKV_DECODE_CTAS asks for it: with a collective running on a
// side stream (multi-GPU runtime), its kernel needs SMs of its own, because it
// cannot share an SM with a decode CTA.  Read once per process.
int decode_grid() {
  static int cached = 0;
  if (cached <= 0) {
    const int sms = device_sms();
    int g = sms > kMaxGrid ? kMaxGrid : sms;
    if (const char* e = std::getenv("NQKV_DECODE_CTAS")) {
      const int v = std::atoi(e);
      if (v > 0 && v < g) g = v;
    }
    cached = g;
  }
  return cached;
}

long long grid_for(long long work, int threads, int per_sm) {
  long long blocks = (work + threads - 1) / threads;
  const long long cap = static_cast<long long>(device_sms()) * per_sm;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : blocks;
}

// Launch with programmatic stream serialization (PDL) so the kernel's
// prologue overlaps the previous kernel's tail; device code waits with
// griddepcontrol.wait before reading anything the previous kernel wrote.
template <typename... Args, typename... Actual>
cudaError_t launch_pdl_n(void (*kern)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                         Actual... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename P>
cudaError_t launch_pdl(void (*kern)(P), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       const P& prm) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, prm);
}

template <int HD, int BLK, bool F16S, bool GRP, bool GATHER, bool PAGED = false>
int launch_decode_blk(const DecodeParams& p, cudaStream_t st) {
  auto kern = decode_kernel<HD, BLK, kDecodeWarps, F16S, GRP, GATHER, PAGED>;
  const size_t smem = Smem<HD, kDecodeWarps>::kBytes;
  static bool attr_set = false;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!attr_set) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
      if (e != cudaSuccess) return cuda_fail(e);
      attr_set = true;
    }
  }
  // one CTA per SM (the kernel needs ~150-225 KB of shared memory); CTAs
  // beyond what the token count needs exit after the prologue
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(decode_grid())),
                                   dim3(kDecodeWarps * 32), smem, st, p);
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

template <int HD, bool F16S, bool GATHER>
int launch_decode_g(const DecodeParams& p, cudaStream_t st) {
  if (p.hpb_shift) return launch_decode_blk<HD, HD, F16S, true, GATHER>(p, st);   // blk > hd
  switch (p.blk_shift) {
    case 5: return launch_decode_blk<HD, 32, F16S, false, GATHER>(p, st);
    case 6: return launch_decode_blk<HD, 64, F16S, false, GATHER>(p, st);
    default:
      if constexpr (HD == 128) return launch_decode_blk<HD, 128, F16S, false, GATHER>(p, st);
      else return NQKV_ERR_UNSUPPORTED;    // blk 128 at hd 64 is a head-group block (GRP)
  }
}

// paged cache (reading R17): fp32 scales, no fused gather
template <int HD>
int launch_decode_paged(const DecodeParams& p, cudaStream_t st) {
  if (p.hpb_shift) return launch_decode_blk<HD, HD, false, true, false, true>(p, st);
  switch (p.blk_shift) {
    case 5: return launch_decode_blk<HD, 32, false, false, false, true>(p, st);
    case 6: return launch_decode_blk<HD, 64, false, false, false, true>(p, st);
    default:
      if constexpr (HD == 128) return launch_decode_blk<HD, 128, false, false, false, true>(p, st);
      else return NQKV_ERR_UNSUPPORTED;
  }
}

template <int HD, bool F16S>
int launch_decode(const DecodeParams& p, cudaStream_t st) {
  if (p.bt) {
    if constexpr (F16S) return NQKV_ERR_UNSUPPORTED;
    else return launch_decode_paged<HD>(p, st);
  }
  return p.peer_out ? launch_decode_g<HD, F16S, true>(p, st) : launch_decode_g<HD, F16S, false>(p, st);
}

// KV layout of a call (nqkv_kv_layout, validated): grouped-query head
// mapping (R16) and the paged cache (R17)
struct KvLayout {
  int kv_shift = 0;
  const int32_t* bt = nullptr;
  int bt_stride = 0, page_shift = 0;
  long long n_pages = 0;
};

int log2_exact(long long v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int s = 0;
  while ((1ll << s) < v) ++s;
  return s;
}

// H query heads over a cache described by `kv` (may be null: MHA, contiguous)
int kv_layout_of(const nqkv_kv_layout* kv, int H, int hd, int blk, int Tc, KvLayout& out, int& H_kv) {
  out = KvLayout();
  H_kv = H;
  if (!kv) return NQKV_OK;
  H_kv = kv->kv_heads ? kv->kv_heads : H;
  if (H_kv < 0 || (H_kv > 0 && H % H_kv)) return NQKV_ERR_SHAPE;
  if (H_kv > 0) {
    out.kv_shift = log2_exact(H / H_kv);
    if (out.kv_shift < 0) return NQKV_ERR_UNSUPPORTED;        // group size: a power of two
  }
  if (kv->block_table) {
    const int ps = log2_exact(kv->page_size);
    if (ps < 6) return NQKV_ERR_UNSUPPORTED;                    // P: power of two >= 64
    if (kv->n_pages <= 0 || kv->pages_per_seq <= 0) return NQKV_ERR_SHAPE;
    if (static_cast<long long>(kv->pages_per_seq) * kv->page_size < Tc) return NQKV_ERR_SHAPE;
    if (static_cast<long long>(kv->n_pages) * H_kv * kv->page_size * (hd / 2) >= (1ll << 32))
      return NQKV_ERR_SHAPE;                                    // 32-bit row offsets
    if (reinterpret_cast<uintptr_t>(kv->block_table) & 3u) return NQKV_ERR_ALIGN;
    out.bt = kv->block_table;
    out.bt_stride = kv->pages_per_seq;
    out.page_shift = ps;
    out.n_pages = kv->n_pages;
  }
  (void)blk;
  return NQKV_OK;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// workspace: [B*H] int arrival counters (zero between launches) | partials
// [kMaxGrid][2][hd + 2] fp32
struct WsLayout {
  size_t cnt, part, gctr, gqa, total;
  long long gqa_records;
};

// grouped-query kernel (decode_gqa.cuh): chunk partials of (hd + 2) floats
long long gqa_records_of(long long B, long long H) {
  const long long r = B * H * kGqaMaxChunkCap;
  return r < kGqaMaxRecords ? r : kGqaMaxRecords;
}

WsLayout ws_layout(long long B, long long H, int hd) {
  WsLayout w;
  w.cnt = 0;
  w.part = align_up(static_cast<size_t>(B * H) * sizeof(int), 256);
  w.gctr = align_up(w.part + static_cast<size_t>(kMaxGrid) * 2 * (hd + 2) * sizeof(unsigned long long), 256);
  w.gqa = w.gctr + 256;         // gctr[0]: gather CTA-completion counter (zero between calls)
  w.gqa_records = gqa_records_of(B, H);
  w.total = align_up(w.gqa + static_cast<size_t>(w.gqa_records) * (hd + 2) * sizeof(float), 256);
  return w;
}

bool gqa_native_enabled() {     // NQKV_GQA_NATIVE=0: GQA through the per-query-head MHA kernel
  static const bool on = [] {
    const char* e = std::getenv("NQKV_GQA_NATIVE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool gqa_tc_enabled() {         // NQKV_GQA_TC=0: K scores with FFMA2 instead of mma.sync
  static const bool on = [] {
    const char* e = std::getenv("NQKV_GQA_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int HD, int GN, bool PAGED, bool F16S>
int launch_gqa_t(const GqaParams& p, long long items, cudaStream_t st) {
  // fp16 scales: tensor-core kernel only (the dispatch guarantees it)
  const bool tc = F16S || gqa_tc_enabled();
  auto kern = tc ? gqa_tc_kernel<HD, GN, PAGED, F16S> : gqa_decode_kernel<HD, GN, PAGED>;
  const size_t smem = tc ? gqa_tc_smem_bytes<HD, GN>() : gqa_smem_bytes<HD, GN>();
  static bool attr_set = false;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!attr_set) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
      if (e != cudaSuccess) return cuda_fail(e);
      attr_set = true;
    }
  }
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(items)), dim3(kGqaWarps * 32),
                                   smem, st, p);
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

// chunks per (b, kv head, sub-group): the count whose CTA waves fill the last
// wave best (3 CTAs per SM), chunks of >= 256 tokens of capacity, within the
// workspace's partial records
int gqa_chunks(long long groups, long long B, long long H, int Tc) {
  const long long slots = static_cast<long long>(device_sms()) * kGqaCtasPerSm;
  long long ncmax = gqa_records_of(B, H) / (B * H);
  if (ncmax > kGqaMaxChunkCap) ncmax = kGqaMaxChunkCap;
  int best = 1;
  double best_eff = -1.0;
  for (int n = 1; n <= ncmax; ++n) {
    if (n > 1 && Tc / n < 256) break;
    const double waves = static_cast<double>(groups * n) / static_cast<double>(slots);
    const double eff = waves / std::ceil(waves);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = n;
    }
  }
  return best;
}

template <bool PAGED, bool F16S>
int launch_gqa_p(const GqaParams& p, int hd, int GN, long long items, cudaStream_t st) {
  if (hd == 64)
    return GN == 4 ? launch_gqa_t<64, 4, PAGED, F16S>(p, items, st) : launch_gqa_t<64, 2, PAGED, F16S>(p, items, st);
  return GN == 4 ? launch_gqa_t<128, 4, PAGED, F16S>(p, items, st)
                 : launch_gqa_t<128, 2, PAGED, F16S>(p, items, st);
}

int launch_gqa(const DecodeParams& dp, int H_kv, int hd, int blk, bool f16s, float* part,
               long long records, cudaStream_t st) {
  const int g = 1 << dp.kv_shift;
  const int GN = g >= 4 ? 4 : g;
  GqaParams p;
  p.q = dp.q;
  p.kc = dp.kc; p.ks = dp.ks;
  p.vc = dp.vc; p.vs = dp.vs;
  p.seq_lens = dp.seq_lens;
  p.out = dp.out;
  p.cnt = dp.cnt;
  p.part = part;
  p.B = dp.B; p.H = dp.H; p.Hkv = H_kv; p.Tc = dp.Tc;
  p.nsg = g / GN;
  p.kv_shift = dp.kv_shift;
  p.blk_shift = blk_shift_of(blk);
  p.bt = dp.bt;
  p.bt_stride = dp.bt_stride;
  p.page_shift = dp.page_shift;
  p.scale_log2 = dp.scale_log2;
  p.zero = 0;
  p.lv = dp.lv;
  const long long groups = static_cast<long long>(dp.B) * H_kv * p.nsg;
  p.nc = gqa_chunks(groups, dp.B, dp.H, dp.Tc);
  if (p.nc > 1 && groups * p.nc * GN > records) return NQKV_ERR_WORKSPACE;
  const long long items = groups * p.nc;
  if (items >= (1ll << 31)) return NQKV_ERR_SHAPE;
  if (f16s) return launch_gqa_p<false, true>(p, hd, GN, items, st);   // contiguous only (dispatch)
  return p.bt ? launch_gqa_p<true, false>(p, hd, GN, items, st) : launch_gqa_p<false, false>(p, hd, GN, items, st);
}

// fused all-gather epilogue arguments (nqkv_decode_step_gather)
struct GatherArgs {
  float* const* peer_out;
  unsigned* const* peer_flags;
  int G, rank, H_total;
  unsigned epoch;
  const unsigned* epoch_ptr;
};

int decode_common(const void* q, const uint8_t* k_codes, const void* k_scales,
                  const uint8_t* v_codes, const void* v_scales, const int32_t* d_seq_lens,
                  const void* k_new, const void* v_new, int64_t new_sb, int64_t new_sh, int B,
                  int H, int hd, int blk, int Tc, float softmax_scale, float* out, void* workspace,
                  size_t ws_bytes, const void* plan, int flags, cudaStream_t st,
                  const GatherArgs* ga = nullptr, const nqkv_kv_layout* kv = nullptr) {
  if (!q || !k_codes || !k_scales || !v_codes || !v_scales || !d_seq_lens || (!out && !ga))
    return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  if (B < 0 || H < 0 || Tc <= 0 || Tc % 64 || B > kMaxBatch) return NQKV_ERR_SHAPE;
  KvLayout lay;
  int H_kv = H;
  if (int s = kv_layout_of(kv, H, hd, blk_of(blk), Tc, lay, H_kv)) return s;
  if (kv && (k_new || plan || ga)) return NQKV_ERR_UNSUPPORTED;   // layouts: attention-only calls
  if (lay.bt && f16s_of(blk)) return NQKV_ERR_UNSUPPORTED;
  if (!heads_fit(H_kv, hd, blk_of(blk))) return NQKV_ERR_SHAPE;
  if (static_cast<long long>(B) * H * Tc >= (1ll << 31)) return NQKV_ERR_SHAPE;
  if (!lay.bt && static_cast<long long>(B) * H_kv * Tc * (hd / 2) >= (1ll << 32))
    return NQKV_ERR_SHAPE;  // 32-bit offsets
  const bool f16s = f16s_of(blk);
  blk = blk_of(blk);
  if (!aligned16(q) || !aligned16(k_codes) || !aligned16(v_codes) || (out && !aligned16(out)) ||
      !aligned16(k_scales) || !aligned16(v_scales))
    return NQKV_ERR_ALIGN;
  if (k_new && (!aligned16(k_new) || !aligned16(v_new) || (new_sb % 8) || (new_sh % 8)))
    return NQKV_ERR_ALIGN;
  if (B == 0 || H == 0) {
    if (!ga) return NQKV_OK;
    const cudaError_t e = launch_pdl_n(gather_publish_kernel, dim3(1), dim3(64), 0, st, ga->peer_flags,
                                       ga->G, ga->rank, ga->epoch, ga->epoch_ptr);
    return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
  }
  const WsLayout w = ws_layout(B, H, hd);
  if (!workspace) return NQKV_ERR_NULL;
  if (!aligned16(workspace)) return NQKV_ERR_ALIGN;
  if (ws_bytes < w.total) return NQKV_ERR_WORKSPACE;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  DecodeParams p;
  p.q = static_cast<const __half*>(q);
  p.kc = k_codes; p.ks = k_scales; p.vc = v_codes; p.vs = v_scales;
  p.seq_lens = d_seq_lens; p.out = out;
  p.k_new = static_cast<const __half*>(k_new);
  p.v_new = static_cast<const __half*>(v_new);
  p.new_sb = new_sb; p.new_sh = new_sh;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  p.cnt = reinterpret_cast<int*>(ws + w.cnt);
  p.part = reinterpret_cast<unsigned long long*>(ws + w.part);
  p.B = B; p.H = H; p.Tc = Tc;
  // blk > hd: attention sees one scale per (token, head) row, as at blk = hd,
  // read from the head group's scale row
  p.blk_shift = blk_shift_of(blk > hd ? hd : blk);
  p.hpb_shift = hpb_shift_of(hd, blk);
  p.kv_shift = lay.kv_shift;
  p.bt = lay.bt;
  p.bt_stride = lay.bt_stride;
  p.page_shift = lay.page_shift;
  p.min_tokens = kMinTokensPerCta;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.lv = make_levels();
  p.tab = make_bucket_tab();
  p.plan = static_cast<const int*>(plan);
  p.early = plan && (flags & NQKV_EARLY_START) ? 1 : 0;
  p.trace = nullptr;
  p.peer_out = ga ? ga->peer_out : nullptr;
  p.peer_flags = ga ? ga->peer_flags : nullptr;
  p.gctr = reinterpret_cast<unsigned*>(ws + w.gctr);
  p.gather_g = ga ? ga->G : 1;
  p.gather_rank = ga ? ga->rank : 0;
  p.h_total = ga ? ga->H_total : H;
  p.epoch = ga ? ga->epoch : 0u;
  p.epoch_ptr = ga ? ga->epoch_ptr : nullptr;
  // grouped-query attention over an fp32-scale cache (contiguous or paged)
  // with blk <= hd: the group-native kernel (each KV head streamed once per
  // <= 4 query heads)
  if (lay.kv_shift > 0 && blk <= hd && !plan && !k_new && !ga && gqa_native_enabled() &&
      (!f16s || (gqa_tc_enabled() && !lay.bt)))
    return launch_gqa(p, H_kv, hd, blk, f16s, reinterpret_cast<float*>(ws + w.gqa), w.gqa_records, st);
#ifdef NQKV_TRACE
  if (const char* t = std::getenv("NQKV_TRACE_PTR"))
    p.trace = reinterpret_cast<unsigned long long*>(std::strtoull(t, nullptr, 0));
#endif
  if (f16s) return hd == 64 ? launch_decode<64, true>(p, st) : launch_decode<128, true>(p, st);
  return hd == 64 ? launch_decode<64, false>(p, st) : launch_decode<128, false>(p, st);
}

}  // namespace nqkv

// ====================================================================== ABI
using namespace nqkv;

extern "C" {

int nqkv_abi_version(void) { return NQKV_ABI_VERSION; }

#ifndef NQKV_BUILD_ID
#define NQKV_BUILD_ID "unknown"
#endif
// "NQKV_BUILD_ID=<id>" is also found by build.py in the file itself (no dlopen)
__attribute__((used)) static const char kBuildIdTag[] = "NQKV_BUILD_ID=" NQKV_BUILD_ID;
const char* nqkv_build_id(void) { return kBuildIdTag + 14; }

#ifdef NQKV_PF_TRACE
// development builds only: mapped host buffer the prefill kernel writes its progress to
unsigned* nqkv_pf_trace_host(void) {
  static unsigned* h = nullptr;
  if (!h) {
    if (cudaHostAlloc(&h, 4096, cudaHostAllocMapped) != cudaSuccess) return nullptr;
    memset(h, 0, 4096);
    unsigned* d = nullptr;
    cudaHostGetDevicePointer(&d, h, 0);
    cudaMemcpyToSymbol(g_pf_trace, &d, sizeof(d));
  }
  return h;
}
#endif

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

static int quantize_common(const void* x, int64_t stride_b, int64_t stride_t, int64_t stride_h,
                           int B, int H, int hd, int n_new, int blk, const int32_t* d_pos, int Tc,
                           uint8_t* codes, void* scales, void* stream, const nqkv_kv_layout* kv,
                           const void* x2 = nullptr, uint8_t* codes2 = nullptr,
                           void* scales2 = nullptr) {
  if (!x || !d_pos || !codes || !scales) return NQKV_ERR_NULL;
  const bool pair = x2 != nullptr;
  if (pair && (!codes2 || !scales2)) return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  const bool f16s = f16s_of(blk);
  blk = blk_of(blk);
  if (B < 0 || H < 0 || n_new < 0 || Tc <= 0 || Tc % 64) return NQKV_ERR_SHAPE;
  if (!heads_fit(H, hd, blk)) return NQKV_ERR_SHAPE;
  KvLayout lay;
  int H_kv = H;
  if (int s = kv_layout_of(kv, H, hd, blk, Tc, lay, H_kv)) return s;
  if (H_kv != H) return NQKV_ERR_SHAPE;      // x holds the cache's (KV) heads
  if (!aligned16(x) || !aligned16(codes) || !scale_aligned(scales, f16s) ||
      (stride_b % 8) || (stride_t % 8) || (stride_h % 8))
    return NQKV_ERR_ALIGN;
  if (pair && (!aligned16(x2) || !aligned16(codes2) || !scale_aligned(scales2, f16s) ||
               ((reinterpret_cast<uintptr_t>(x) ^ reinterpret_cast<uintptr_t>(x2)) & 31u)))
    return NQKV_ERR_ALIGN;                   // both tensors take the same load width
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  const long long rows = static_cast<long long>(B) * n_new;   // token rows (b, t)
  if (rows == 0 || H == 0) return NQKV_OK;
  const long long chunks1 = rows * H * (hd / 16);              // 16-element chunks per tensor
  const long long chunks = pair ? 2 * chunks1 : chunks1;
  if (chunks >= (1ll << 31)) return NQKV_ERR_SHAPE;
  QuantParams p;
  p.x = static_cast<const __half*>(x);
  p.sb = stride_b; p.st = stride_t; p.sh = stride_h;
  p.pos = d_pos; p.codes = codes; p.scales = scales;
  p.B = B; p.n_new = n_new; p.H = H; p.Tc = Tc;
  p.blk_shift = blk_shift_of(blk);
  p.hpb_shift = hpb_shift_of(hd, blk);
  p.total = static_cast<uint32_t>(chunks);
  p.total1 = static_cast<uint32_t>(chunks1);
  p.x2 = static_cast<const __half*>(x2);
  p.codes2 = codes2;
  p.scales2 = scales2;
  p.v256 = ((reinterpret_cast<uintptr_t>(x) & 31u) == 0 && stride_b % 16 == 0 && stride_t % 16 == 0 &&
            stride_h % 16 == 0) ? 1 : 0;
  if (stride_h == hd && stride_t == static_cast<int64_t>(H) * hd &&
      (B == 1 || stride_b == static_cast<int64_t>(n_new) * H * hd))
    p.v256 |= 2;
  p.cpr = make_fastdiv(static_cast<uint32_t>(H * (hd / 16)));
  p.nnew = make_fastdiv(static_cast<uint32_t>(n_new));
  p.tab = make_bucket_tab();
  p.bt = lay.bt;
  p.bt_stride = lay.bt_stride;
  p.page_shift = lay.page_shift;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // one warp per 64-chunk unit, grid-strided over one wave of resident CTAs
#ifndef NQKV_Q_CTAS_PER_SM
#define NQKV_Q_CTAS_PER_SM 4            // = resident CTAs (64 regs x 256 threads): one wave
#endif
  const dim3 grid(static_cast<unsigned>(grid_for((chunks + 1) / 2, 256, NQKV_Q_CTAS_PER_SM)));
  cudaError_t e;
  const size_t sm = kQuantSmem;
  auto launch_l = [&](auto f16s_tag, auto lay_tag) {
    constexpr bool F = decltype(f16s_tag)::value;
    constexpr int Y = decltype(lay_tag)::value;
    if (hd == 64)
      return blk == 32    ? launch_pdl(quantize_kernel<64, 32, F, Y>, grid, dim3(256), sm, st, p)
             : blk == 64  ? launch_pdl(quantize_kernel<64, 64, F, Y>, grid, dim3(256), sm, st, p)
             : blk == 128 ? launch_pdl(quantize_kernel<64, 128, F, Y>, grid, dim3(256), sm, st, p)
                          : launch_pdl(quantize_kernel<64, 256, F, Y>, grid, dim3(256), sm, st, p);
    return blk == 32    ? launch_pdl(quantize_kernel<128, 32, F, Y>, grid, dim3(256), sm, st, p)
           : blk == 64  ? launch_pdl(quantize_kernel<128, 64, F, Y>, grid, dim3(256), sm, st, p)
           : blk == 128 ? launch_pdl(quantize_kernel<128, 128, F, Y>, grid, dim3(256), sm, st, p)
                        : launch_pdl(quantize_kernel<128, 256, F, Y>, grid, dim3(256), sm, st, p);
  };
  auto launch = [&](auto f16s_tag) {
    if (pair) return launch_l(f16s_tag, std::integral_constant<int, 1>{});
    if (lay.bt) return launch_l(f16s_tag, std::integral_constant<int, 2>{});
    return launch_l(f16s_tag, std::integral_constant<int, 0>{});
  };
  e = f16s ? launch(std::true_type{}) : launch(std::false_type{});
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

int nqkv_quantize(const void* x, int64_t stride_b, int64_t stride_t, int64_t stride_h, int B,
                  int H, int hd, int n_new, int blk, const int32_t* d_pos, int Tc,
                  uint8_t* codes, void* scales, void* stream) {
  return quantize_common(x, stride_b, stride_t, stride_h, B, H, hd, n_new, blk, d_pos, Tc, codes,
                         scales, stream, nullptr);
}

int nqkv_quantize_pair(const void* x_k, const void* x_v, int64_t stride_b, int64_t stride_t,
                       int64_t stride_h, int B, int H, int hd, int n_new, int blk,
                       const int32_t* d_pos, int Tc, uint8_t* k_codes, void* k_scales,
                       uint8_t* v_codes, void* v_scales, void* stream) {
  if (!x_v) return NQKV_ERR_NULL;
  return quantize_common(x_k, stride_b, stride_t, stride_h, B, H, hd, n_new, blk, d_pos, Tc, k_codes,
                         k_scales, stream, nullptr, x_v, v_codes, v_scales);
}

int nqkv_quantize_kv(const void* x, int64_t stride_b, int64_t stride_t, int64_t stride_h, int B,
                     int H, int hd, int n_new, int blk, const int32_t* d_pos, int Tc,
                     const nqkv_kv_layout* kv, uint8_t* codes, void* scales, void* stream) {
  if (!kv) return NQKV_ERR_NULL;
  return quantize_common(x, stride_b, stride_t, stride_h, B, H, hd, n_new, blk, d_pos, Tc, codes,
                         scales, stream, kv);
}

int nqkv_dequantize(const uint8_t* codes, const void* scales, int B, int H, int Tc, int hd,
                    int blk, int n_tokens, int out_dtype, void* out, void* stream) {
  if (!codes || !scales || !out) return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  const bool f16s = f16s_of(blk);
  blk = blk_of(blk);
  if (B < 0 || H < 0 || Tc <= 0 || Tc % 64 || n_tokens < 0 || n_tokens > Tc)
    return NQKV_ERR_SHAPE;
  if (!heads_fit(H, hd, blk)) return NQKV_ERR_SHAPE;
  if (out_dtype != 0 && out_dtype != 1) return NQKV_ERR_UNSUPPORTED;
  if (!aligned16(codes) || !aligned16(out) || !scale_aligned(scales, f16s))
    return NQKV_ERR_ALIGN;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  const long long total = static_cast<long long>(B) * H * n_tokens * (hd / 8);
  if (total == 0) return NQKV_OK;
  DequantParams p;
  p.codes = codes; p.scales = scales; p.out = out;
  p.total_chunks = total;
  p.Tc = Tc; p.hd = hd; p.n_tokens = n_tokens;
  p.blk_shift = blk_shift_of(blk > hd ? hd : blk);
  p.hpb_shift = hpb_shift_of(hd, blk);
  p.chunks_per_row = hd / 8;
  p.lv = make_levels();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(static_cast<unsigned>(grid_for(total, 256, 8)));
  const cudaError_t e =
      out_dtype == 1 ? (f16s ? launch_pdl(dequant_kernel<true, true>, grid, dim3(256), 0, st, p)
                             : launch_pdl(dequant_kernel<true, false>, grid, dim3(256), 0, st, p))
                     : (f16s ? launch_pdl(dequant_kernel<false, true>, grid, dim3(256), 0, st, p)
                             : launch_pdl(dequant_kernel<false, false>, grid, dim3(256), 0, st, p));
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

size_t nqkv_decode_workspace_bytes(int B, int H, int hd, int Tc) {
  if (B < 0 || H < 0 || Tc <= 0 || (hd != 64 && hd != 128)) return 0;
  return ws_layout(B, H, hd).total;
}

size_t nqkv_decode_counter_bytes(int B, int H) {
  if (B < 0 || H < 0) return 0;
  return static_cast<size_t>(B) * H * sizeof(int);
}

int nqkv_decode_attention(const void* q, const uint8_t* k_codes, const void* k_scales,
                          const uint8_t* v_codes, const void* v_scales,
                          const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                          float softmax_scale, float* out, void* workspace, size_t ws_bytes,
                          void* stream) {
  return decode_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, nullptr, nullptr, 0,
                       0, B, H, hd, blk, Tc, softmax_scale, out, workspace, ws_bytes, nullptr, 0,
                       static_cast<cudaStream_t>(stream));
}

int nqkv_decode_attention_kv(const void* q, const uint8_t* k_codes, const void* k_scales,
                             const uint8_t* v_codes, const void* v_scales,
                             const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                             const nqkv_kv_layout* kv, float softmax_scale, float* out,
                             void* workspace, size_t ws_bytes, void* stream) {
  if (!kv) return NQKV_ERR_NULL;
  return decode_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, nullptr, nullptr, 0,
                       0, B, H, hd, blk, Tc, softmax_scale, out, workspace, ws_bytes, nullptr, 0,
                       static_cast<cudaStream_t>(stream), nullptr, kv);
}

size_t nqkv_decode_plan_bytes(void) { return static_cast<size_t>(kPlanInts) * sizeof(int); }

int nqkv_decode_plan(const int32_t* d_seq_lens, int B, int H, int hd, int Tc, int fused, void* plan,
                     size_t plan_bytes, void* stream) {
  if (!d_seq_lens || !plan) return NQKV_ERR_NULL;
  if (hd != 64 && hd != 128) return NQKV_ERR_UNSUPPORTED;
  if (B < 0 || H <= 0 || Tc <= 0 || Tc % 64 || B > kMaxBatch) return NQKV_ERR_SHAPE;
  if (static_cast<long long>(B) * H * Tc >= (1ll << 31)) return NQKV_ERR_SHAPE;
  if (!aligned16(plan)) return NQKV_ERR_ALIGN;
  if (plan_bytes < nqkv_decode_plan_bytes()) return NQKV_ERR_WORKSPACE;
  const cudaError_t e = launch_pdl_n(decode_plan_kernel, dim3(1), dim3(1024), 0,
                                   static_cast<cudaStream_t>(stream), d_seq_lens, B, H, Tc,
                                   fused ? 1 : 0, decode_grid(), kMinTokensPerCta,
                                   hd == 64 ? Geo<64>::R : Geo<128>::R, static_cast<int*>(plan));
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

int nqkv_decode_attention_planned(const void* q, const uint8_t* k_codes, const void* k_scales,
                                  const uint8_t* v_codes, const void* v_scales,
                                  const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                                  float softmax_scale, float* out, void* workspace,
                                  size_t ws_bytes, const void* plan, int flags, void* stream) {
  if (!plan) return NQKV_ERR_NULL;
  return decode_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, nullptr, nullptr, 0,
                       0, B, H, hd, blk, Tc, softmax_scale, out, workspace, ws_bytes, plan,
                       flags, static_cast<cudaStream_t>(stream));
}

int nqkv_decode_step(const void* k_new, const void* v_new, int64_t new_stride_b,
                     int64_t new_stride_h, const void* q, uint8_t* k_codes, void* k_scales,
                     uint8_t* v_codes, void* v_scales, const int32_t* d_seq_lens, int B, int H,
                     int hd, int blk, int Tc, float softmax_scale, float* out, void* workspace,
                     size_t ws_bytes, void* stream) {
  if (!k_new || !v_new) return NQKV_ERR_NULL;
  return decode_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, k_new, v_new,
                       new_stride_b, new_stride_h, B, H, hd, blk, Tc, softmax_scale, out,
                       workspace, ws_bytes, nullptr, 0, static_cast<cudaStream_t>(stream));
}

int nqkv_decode_step_planned(const void* k_new, const void* v_new, int64_t new_stride_b,
                             int64_t new_stride_h, const void* q, uint8_t* k_codes,
                             void* k_scales, uint8_t* v_codes, void* v_scales,
                             const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                             float softmax_scale, float* out, void* workspace, size_t ws_bytes,
                             const void* plan, int flags, void* stream) {
  if (!k_new || !v_new || !plan) return NQKV_ERR_NULL;
  return decode_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, k_new, v_new,
                       new_stride_b, new_stride_h, B, H, hd, blk, Tc, softmax_scale, out,
                       workspace, ws_bytes, plan, flags, static_cast<cudaStream_t>(stream));
}

int nqkv_decode_step_gather(const void* k_new, const void* v_new, int64_t new_stride_b,
                            int64_t new_stride_h, const void* q, uint8_t* k_codes, void* k_scales,
                            uint8_t* v_codes, void* v_scales, const int32_t* d_seq_lens, int B,
                            int H, int hd, int blk, int Tc, float softmax_scale,
                            float* const* d_peer_out, unsigned* const* d_peer_flags, int G, int rank,
                            int H_total, unsigned epoch, const unsigned* d_epoch, void* workspace,
                            size_t ws_bytes, const void* plan, int flags, void* stream) {
  if (!k_new || !v_new || !plan || !d_peer_out || !d_peer_flags) return NQKV_ERR_NULL;
  if (G < 1 || G > 64 || rank < 0 || rank >= G || (epoch == 0u && !d_epoch)) return NQKV_ERR_SHAPE;
  if (H_total != static_cast<long long>(G) * H) return NQKV_ERR_SHAPE;
  GatherArgs ga{d_peer_out, d_peer_flags, G, rank, H_total, epoch, d_epoch};
  return decode_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, k_new, v_new,
                       new_stride_b, new_stride_h, B, H, hd, blk, Tc, softmax_scale, nullptr,
                       workspace, ws_bytes, plan, flags, static_cast<cudaStream_t>(stream), &ga);
}

int nqkv_gather_epoch_bump(unsigned* d_epoch, void* stream) {
  if (!d_epoch) return NQKV_ERR_NULL;
  const cudaError_t e = launch_pdl_n(gather_epoch_bump_kernel, dim3(1), dim3(1), 0,
                                   static_cast<cudaStream_t>(stream), d_epoch);
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

int nqkv_gather_wait(const unsigned* d_flags, int n, const unsigned* d_epoch, void* stream) {
  if (!d_flags || !d_epoch) return NQKV_ERR_NULL;
  if (n < 0) return NQKV_ERR_SHAPE;
  if (n == 0) return NQKV_OK;
  const cudaError_t e = launch_pdl_n(gather_wait_kernel, dim3(1), dim3(256), 0,
                                   static_cast<cudaStream_t>(stream), d_flags, n, d_epoch);
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

static int prefill_common(const void* q, const uint8_t* k_codes, const void* k_scales,
                          const uint8_t* v_codes, const void* v_scales, const int32_t* d_seq_lens,
                          int B, int H, int hd, int blk, int Tc, int T, float softmax_scale,
                          float* out, void* stream, const nqkv_kv_layout* kv) {
  if (!q || !k_codes || !k_scales || !v_codes || !v_scales || !d_seq_lens || !out) return NQKV_ERR_NULL;
  if (int s = check_geometry(hd, blk)) return s;
  const bool f16s = f16s_of(blk);
  blk = blk_of(blk);
  if (B < 0 || H < 0 || T < 0 || Tc <= 0 || Tc % 64 || T > Tc) return NQKV_ERR_SHAPE;
  KvLayout lay;
  int H_kv = H;
  if (int s = kv_layout_of(kv, H, hd, blk, Tc, lay, H_kv)) return s;
#if NQKV_PREFILL_MMA_SYNC
  if (kv) return NQKV_ERR_UNSUPPORTED;       // the comparison build has no KV layouts
#endif
  if (!heads_fit(H_kv, hd, blk)) return NQKV_ERR_SHAPE;
  if (static_cast<long long>(B) * H * Tc >= (1ll << 31) || B > 65535 || H > 65535) return NQKV_ERR_SHAPE;
  if (!aligned16(q) || !aligned16(k_codes) || !aligned16(v_codes) || !aligned16(out) ||
      !scale_aligned(k_scales, f16s) || !scale_aligned(v_scales, f16s))
    return NQKV_ERR_ALIGN;
  if (tables_status() != 0) return NQKV_ERR_INTERNAL;
  if (B == 0 || H == 0 || T == 0) return NQKV_OK;
  PrefillParams p;
  p.q = static_cast<const __half*>(q);
  p.kc = k_codes; p.ks = k_scales; p.vc = v_codes; p.vs = v_scales;
  p.seq_lens = d_seq_lens; p.out = out;
  p.B = B; p.H = H; p.T = T; p.Tc = Tc;
  p.blk_shift = blk_shift_of(blk > hd ? hd : blk);
  p.hpb_shift = hpb_shift_of(hd, blk);
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.lv = make_levels();
  p.kv_shift = lay.kv_shift;
  p.bt = lay.bt;
  p.bt_stride = lay.bt_stride;
  p.page_shift = lay.page_shift;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool grp = blk > hd;
  cudaError_t e;
#if NQKV_PREFILL_MMA_SYNC
  // legacy tensor-core path (mma.sync m16n8k16), kept for comparison builds
  const dim3 grid(static_cast<unsigned>((T + kPfQ - 1) / kPfQ), static_cast<unsigned>(H), static_cast<unsigned>(B));
  auto go = [&](auto kern, size_t sm) {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e2 != cudaSuccess) return e2;
    return launch_pdl(kern, grid, dim3(kPfW * 32), sm, st, p);
  };
  if (hd == 64) {
    constexpr size_t sm = prefill_smem_bytes<64>();
    e = f16s ? (grp ? go(prefill_kernel<64, true, true>, sm) : go(prefill_kernel<64, true, false>, sm))
             : (grp ? go(prefill_kernel<64, false, true>, sm) : go(prefill_kernel<64, false, false>, sm));
  } else {
    constexpr size_t sm = prefill_smem_bytes<128>();
    e = f16s ? (grp ? go(prefill_kernel<128, true, true>, sm) : go(prefill_kernel<128, true, false>, sm))
             : (grp ? go(prefill_kernel<128, false, true>, sm) : go(prefill_kernel<128, false, false>, sm));
  }
#else
  // tcgen05 / TMEM path: 256 queries per CTA
  const dim3 grid(static_cast<unsigned>((T + kTcQ - 1) / kTcQ), static_cast<unsigned>(H), static_cast<unsigned>(B));
  auto go = [&](auto kern, size_t sm) {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e2 != cudaSuccess) return e2;
    return launch_pdl(kern, grid, dim3(kTcThreads), sm, st, p);
  };
  if (hd == 64) {
    constexpr size_t sm = prefill_tc_smem_bytes<64>();
    e = f16s ? (grp ? go(prefill_tc_kernel<64, true, true>, sm) : go(prefill_tc_kernel<64, true, false>, sm))
             : (grp ? go(prefill_tc_kernel<64, false, true>, sm) : go(prefill_tc_kernel<64, false, false>, sm));
  } else {
    constexpr size_t sm = prefill_tc_smem_bytes<128>();
    e = f16s ? (grp ? go(prefill_tc_kernel<128, true, true>, sm) : go(prefill_tc_kernel<128, true, false>, sm))
             : (grp ? go(prefill_tc_kernel<128, false, true>, sm) : go(prefill_tc_kernel<128, false, false>, sm));
  }
#endif
  return e == cudaSuccess ? NQKV_OK : cuda_fail(e);
}

int nqkv_prefill_attention(const void* q, const uint8_t* k_codes, const void* k_scales,
                           const uint8_t* v_codes, const void* v_scales, const int32_t* d_seq_lens,
                           int B, int H, int hd, int blk, int Tc, int T, float softmax_scale,
                           float* out, void* stream) {
  return prefill_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, B, H, hd, blk, Tc, T,
                        softmax_scale, out, stream, nullptr);
}

int nqkv_prefill_attention_kv(const void* q, const uint8_t* k_codes, const void* k_scales,
                              const uint8_t* v_codes, const void* v_scales,
                              const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                              int T, const nqkv_kv_layout* kv, float softmax_scale, float* out,
                              void* stream) {
  if (!kv) return NQKV_ERR_NULL;
  return prefill_common(q, k_codes, k_scales, v_codes, v_scales, d_seq_lens, B, H, hd, blk, Tc, T,
                        softmax_scale, out, stream, kv);
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
