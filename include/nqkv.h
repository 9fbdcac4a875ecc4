/*
 * nqkv.h -- C ABI of the B200-native NQKV hot path (arXiv 2505.16210).
 *
 * NQKV stores the K/V cache as 4-bit NormalFloat (NF4) indices plus one
 * absmax scale per block and dequantises by table lookup at decode time
 * (PAPER.md:193, 201, 205, 213-235).  This library implements the four
 * operations of the paper's problem statement:
 *
 *   nqkv_levels            the NF4 level table
 *   nqkv_quantize          I <- Concat(I, quantize_NF4(X))
 *   nqkv_dequantize        X' = dequantize_NF4(I)
 *   nqkv_decode_attention  t_O = Softmax(t_Q X_K'^T/sqrt(d)) X_V'  with the
 *                          dequantisation fused in registers
 *
 * plus the decode step with the append fused in (nqkv_decode_step), planned
 * variants of both (nqkv_decode_plan, *_planned) and the step with the
 * head-sharded all-gather fused into its epilogue (nqkv_decode_step_gather,
 * nqkv_gather_epoch_bump, nqkv_gather_wait).
 *
 * Conventions (all entry points)
 *  - The caller owns every buffer.  The library never allocates, frees or
 *    synchronises; device work is enqueued on `stream` (a cudaStream_t passed
 *    as void*, NULL = legacy default stream) and returns immediately.
 *  - "device" pointers must be device-accessible (cudaMalloc / torch CUDA
 *    tensors); "host" pointers are ordinary host memory.
 *  - Host-checkable argument errors return a negative nqkv_status and launch
 *    nothing.  A failed launch returns NQKV_ERR_CUDA; nqkv_last_error()
 *    returns the CUDA error string (thread-local).
 *  - Values that live on the device (positions, sequence lengths, input
 *    values) are not checked: out-of-range positions are skipped, a
 *    non-finite input value produces unspecified codes (the CPU oracle
 *    rejects non-finite input).
 *  - Cache layout (one tensor each for K and V; fixed):
 *        codes  uint8   [B][H][Tc][hd/2]   element 2i in the low nibble of byte i,
 *                                          2i+1 in the high nibble
 *        scales float32 [B][H][Tc][hd/blk] absmax of each block of blk
 *                                          consecutive channels of one (token, head)
 *    With blk > hd a block is the hidden-state slice of hpb = blk/hd adjacent
 *    heads of one token (the paper's blk 256 over d):
 *        scales float32 [B][H/hpb][Tc]     one scale per (token, head group);
 *                                          head h uses group h/hpb
 *    H must then be a multiple of hpb (a head shard must hold whole groups).
 *  - Supported geometry: hd in {64, 128}; blk in {32, 64, 128, 256} with
 *    blk | hd or hd | blk; Tc a positive multiple of 64.  Anything else ->
 *    NQKV_ERR_UNSUPPORTED / NQKV_ERR_SHAPE.
 *  - Calls are thread-safe and reentrant.  The only global state is the level
 *    table, computed once on the host (std::call_once) and passed to kernels
 *    by value.
 */
#ifndef NQKV_H_
#define NQKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NQKV_ABI_VERSION 4   /* 2: blk 256 / head-group scales; NQKV_SCALE_F16 moved to 0x10000;
                                3: nqkv_prefill_attention, nqkv_build_id;
                                4: struct nqkv_kv_layout for grouped-query / paged caches, the *_kv calls */

typedef enum {
  NQKV_OK = 0,
  NQKV_ERR_NULL = -1,        /* a required pointer is NULL */
  NQKV_ERR_SHAPE = -2,       /* negative size, Tc % 64 != 0, ... */
  NQKV_ERR_UNSUPPORTED = -3, /* hd / blk combination not built */
  NQKV_ERR_ALIGN = -4,       /* pointer or stride not 16-byte aligned */
  NQKV_ERR_WORKSPACE = -5,   /* workspace smaller than nqkv_decode_workspace_bytes */
  NQKV_ERR_CUDA = -6,        /* kernel launch / device query failed */
  NQKV_ERR_INTERNAL = -7     /* level-table construction invariant violated */
} nqkv_status;

int nqkv_abi_version(void);
/* Hash of the sources the library was built from (build.py passes it in):
 * lets a caller detect a stale build.  Host only. */
const char* nqkv_build_id(void);
const char* nqkv_status_string(int status);
const char* nqkv_last_error(void);

/* a0. NF4 levels.
 * levels: host float[16], written ascending.  delta = 1 - (1/32 + 1/30)/2;
 * negatives -Phi^-1(delta + k(0.5-delta)/7), k=0..6; zero; positives
 * Phi^-1(0.5 + k(delta-0.5)/8), k=1..8; all divided by Phi^-1(delta),
 * evaluated in double (Phi^-1 by Halley-refined erfc) and rounded to fp32.
 * L[0] = -1, L[7] = +0, L[15] = +1.  Host only; no device needed. */
int nqkv_levels(float levels[16]);

/* Decision thresholds used by the kernels: T[i] = RD32((L[i]+L[i+1])/2),
 * code(n) = #{i : n > T[i]} == argmin_i |n - L[i]| with ties to the lower
 * index.  Host only. */
int nqkv_thresholds(float thresholds[15]);

/* Block-scale storage: every call that takes `blk`
 * accepts blk | NQKV_SCALE_F16, meaning the scales tensor holds fp16 instead
 * of fp32 values.  This is lossless: a block's scale is the absmax of fp16
 * inputs, itself an fp16 value, so codes, dequantised values and attention
 * are identical to the fp32-scale layout; scale bytes halve (-5.6 % of the
 * cache at blk 64).  Scales: 2-byte aligned instead of 4. */
#define NQKV_SCALE_F16 0x10000

/* a1-a3. Quantize + pack + append.
 * x      device fp16, logical [B][n_new][H][hd] with element strides
 *        stride_b, stride_t, stride_h (hd contiguous); 16-byte aligned, all
 *        strides multiples of 8 elements.
 * d_pos  device int32[B]: token row where batch b's first new token goes;
 *        rows d_pos[b] .. d_pos[b]+n_new-1 are written, all other bytes of
 *        codes/scales are left untouched (append-only).  Rows
 *        outside [0, Tc) are skipped.
 * codes  device uint8  [B][H][Tc][hd/2]    (16-byte aligned)
 * scales device float  [B][H][Tc][hd/blk], or [B][H/hpb][Tc] for blk > hd
 *        (4-byte aligned; fp16 with NQKV_SCALE_F16, 2-byte aligned)
 * Per block: s = max|x| (fp32, exact); code = nearest level to n = RN32(x/s),
 * ties lower; s == 0 -> code 7 (the zero level).  The kernel normalises with
 * n' = RN32(x * RN32(1/s)), which gives the identical code for every fp16
 * pair |x| <= s (exhaustive: tests/test_exactness_cpu.py). */
int nqkv_quantize(const void* x, int64_t stride_b, int64_t stride_t, int64_t stride_h,
                  int B, int H, int hd, int n_new, int blk,
                  const int32_t* d_pos, int Tc, uint8_t* codes, void* scales,
                  void* stream);

/* a4 (standalone). Dequantize rows [0, n_tokens) of every (b, h)
 * (no padding).
 * out: device, [B][H][n_tokens][hd], out_dtype 0 = fp32 (RN32(s*L[code])),
 * 1 = fp16 (RN16 of that fp32 value); 16-byte aligned.  n_tokens <= Tc. */
int nqkv_dequantize(const uint8_t* codes, const void* scales, int B, int H, int Tc, int hd,
                    int blk, int n_tokens, int out_dtype, void* out, void* stream);

/* Bytes of workspace nqkv_decode_attention / nqkv_decode_step need for this
 * geometry (0 for an unsupported hd).  Layout: [0, nqkv_decode_counter_bytes)
 * int32 per-(b, h) arrival counters, then per-CTA split-partial records of
 * tagged 64-bit words (value | valid << 32), then the grouped-query kernel's
 * chunk partials (min(B*H*64, 16384) records of hd + 2 floats; H = query
 * heads).  The WHOLE workspace must be ZERO before the first call; every
 * completed call leaves it zero again. */
size_t nqkv_decode_workspace_bytes(int B, int H, int hd, int Tc);
size_t nqkv_decode_counter_bytes(int B, int H);

/* a4-a7. Fused decode attention over the 4-bit cache.
 * For every (b, h): out = softmax(softmax_scale * q . k_t) . v_t over
 * t < seq_lens[b], with k_t, v_t dequantised in registers (never written to
 * memory).  Long sequences are split across CTAs (flash-decoding split-K)
 * and their partial (max, sum, o) merged in-kernel (see below).
 * q          device fp16 [B][H][hd], 16-byte aligned
 * k_codes,…  the cache tensors described above
 * d_seq_lens device int32[B], 0..Tc, counting the token appended this step
 *            (append-before-attend); 0 -> out[b] = 0
 * out        device fp32 [B][H][hd], 16-byte aligned
 * workspace  device, >= nqkv_decode_workspace_bytes(B,H,hd,Tc) bytes,
 *            16-byte aligned, ALL ZERO before the first use; every
 *            completed call leaves it zero again.  Do not share one workspace between calls
 *            that may run concurrently (calls ordered on one stream may).
 * One launch of one CTA per SM (or NQKV_DECODE_CTAS from the environment,
 * read once, if smaller: leaves SMs free for a collective running beside it)
 * with programmatic dependent launch (PDL).  The
 * (b, h, t) token list is cut into equal contiguous per-CTA ranges; a
 * sequence split across CTAs is merged by the last of its CTAs to arrive
 * (per-(b, h) relaxed counter; the others publish tagged partial records
 * that the last one polls), in CTA order.  Results are bit-reproducible for a
 * given (B, H, seq_lens, GPU); a different head shard of the same data may
 * differ by fp32 reassociation only (reading R7).  B <= 1024 and
 * B*H*Tc < 2^31. */
int nqkv_decode_attention(const void* q, const uint8_t* k_codes, const void* k_scales,
                          const uint8_t* v_codes, const void* v_scales,
                          const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                          float softmax_scale, float* out, void* workspace, size_t ws_bytes,
                          void* stream);

/* NEXT f1: one fused decode step = nqkv_quantize of the
 * new token (n_new = 1, at row seq_lens[b]-1) for K and V followed by
 * nqkv_decode_attention over seq_lens[b] tokens, in ONE launch
 * (quantize t_K, t_V; Concat; dequantize; attend).
 * k_new, v_new  device fp16 [B][H][hd] with element strides new_stride_b,
 *               new_stride_h (hd contiguous; 16-byte aligned; strides % 8 == 0)
 * d_seq_lens    device int32[B] AFTER the append (>= 1 to append; 0 -> out = 0,
 *               nothing written).  The codes/scales written are byte-identical
 *               to nqkv_quantize's; the attention result equals
 *               nqkv_decode_attention's on the updated cache.
 * Other arguments as nqkv_decode_attention. */
int nqkv_decode_step(const void* k_new, const void* v_new, int64_t new_stride_b,
                     int64_t new_stride_h, const void* q, uint8_t* k_codes, void* k_scales,
                     uint8_t* v_codes, void* v_scales, const int32_t* d_seq_lens, int B, int H,
                     int hd, int blk, int Tc, float softmax_scale, float* out, void* workspace,
                     size_t ws_bytes, void* stream);

/* Per-step schedule (optional).  Every layer of a decode step shares
 * (B, H, Tc, seq_lens): nqkv_decode_plan computes the launch's work
 * partition once -- streamed lengths, token prefix, CTA count and each CTA's
 * piece order -- into `plan` (device, >= nqkv_decode_plan_bytes() bytes,
 * 16-byte aligned, caller-owned), so that each layer's decode kernel starts
 * streaming without rebuilding it.  hd (64 or 128, else
 * NQKV_ERR_UNSUPPORTED) is the head_dim of the calls that will use the plan
 * (the piece order depends on it).  fused = 1 for nqkv_decode_step_planned
 * (the appended row is not streamed), 0 for nqkv_decode_attention_planned.
 * The plan must be recomputed whenever seq_lens, B, H, hd, Tc or fused
 * change; results are bit-identical to the unplanned calls.
 *
 * flags (the *_planned calls): 0, or NQKV_EARLY_START when neither the plan
 * nor the cache tensors passed to the call are written by the kernel
 * launched immediately before it on the same stream -- e.g. layers 1.. of a
 * decode step whose plan was computed before layer 0.  Every kernel of this
 * library waits for its predecessor (programmatic dependent launch) before
 * it lets its successor start, so -- provided the kernels launched between
 * the writer and this call are this library's or launched without
 * programmatic dependent launch -- such a plan and cache are complete when
 * the call starts, and the kernel reads the plan and issues its first cache
 * loads before that wait, overlapping the predecessor's tail.  q, k_new,
 * v_new, seq_lens, out and the workspace are always accessed after the wait.
 * Results do not depend on flags. */
#define NQKV_EARLY_START 1
size_t nqkv_decode_plan_bytes(void);
int nqkv_decode_plan(const int32_t* d_seq_lens, int B, int H, int hd, int Tc, int fused, void* plan,
                     size_t plan_bytes, void* stream);
int nqkv_decode_attention_planned(const void* q, const uint8_t* k_codes, const void* k_scales,
                                  const uint8_t* v_codes, const void* v_scales,
                                  const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                                  float softmax_scale, float* out, void* workspace,
                                  size_t ws_bytes, const void* plan, int flags, void* stream);
int nqkv_decode_step_planned(const void* k_new, const void* v_new, int64_t new_stride_b,
                             int64_t new_stride_h, const void* q, uint8_t* k_codes,
                             void* k_scales, uint8_t* v_codes, void* v_scales,
                             const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                             float softmax_scale, float* out, void* workspace, size_t ws_bytes,
                             const void* plan, int flags, void* stream);

/* a8 fused into the step: nqkv_decode_step_planned
 * whose output rows go straight to the all-gathered output of every rank, so
 * no separate collective runs.  Rank `rank` of G owns heads
 * [rank*H, (rank+1)*H) of an H_total = G*H head layer (heads
 * are independent); every output row (b, h) is stored to
 * d_peer_out[r][(b*H_total + rank*H + h)*hd ..] for r = 0..G-1.
 * d_peer_out   device array [G] of device pointers: each rank's gathered
 *              output float [B][H_total][hd] (peer pointers over NVLink P2P /
 *              symmetric memory; the caller maps them).
 * d_peer_flags device array [G] of device pointers: each rank's uint32[G]
 *              flag array.  After all of this launch's output stores
 *              (system-scope fence), the launch release-stores `epoch`
 *              (!= 0; or *d_epoch when d_epoch is not NULL) into
 *              d_peer_flags[r][rank] for every r.  A consumer on
 *              rank r may read its gathered buffer once flags[0..G-1] all
 *              equal the epoch (acquire, system scope).  Flags are
 *              caller-owned; epochs must differ between uses of a buffer.
 * The workspace's completion counter is zero between calls (reset by the
 * launch).  G in [1, 64], 0 <= rank < G, H_total == G*H, else NQKV_ERR_SHAPE;
 * NULL pointers -> NQKV_ERR_NULL.  Other arguments as nqkv_decode_step_planned.
 * Results are bit-identical to nqkv_decode_step_planned on the same shard. */
int nqkv_decode_step_gather(const void* k_new, const void* v_new, int64_t new_stride_b,
                            int64_t new_stride_h, const void* q, uint8_t* k_codes, void* k_scales,
                            uint8_t* v_codes, void* v_scales, const int32_t* d_seq_lens, int B,
                            int H, int hd, int blk, int Tc, float softmax_scale,
                            float* const* d_peer_out, unsigned* const* d_peer_flags, int G, int rank,
                            int H_total, unsigned epoch, const unsigned* d_epoch, void* workspace,
                            size_t ws_bytes, const void* plan, int flags, void* stream);

/* Helpers for the fused gather under CUDA-graph replay, where a launch's
 * `epoch` argument is frozen: pass d_epoch (device uint32, read at the end
 * of the launch instead of `epoch`) and bump it once per step.
 * nqkv_gather_epoch_bump: *d_epoch += 1 (stream-ordered).
 * nqkv_gather_wait: stream-ordered wait until d_flags[0..n) (this rank's
 *   flag arrays, device) all equal *d_epoch, with system-scope acquire loads;
 *   kernels after it on the stream may read the gathered buffers.  It spins
 *   on the device: every rank must issue its gather launches for the epoch. */
int nqkv_gather_epoch_bump(unsigned* d_epoch, void* stream);
int nqkv_gather_wait(const unsigned* d_flags, int n, const unsigned* d_epoch, void* stream);

/* NEXT f4: prefill attention over the 4-bit cache.
 * PAPER.md:213-221 (prefill phase: the prompt's K/V are quantised into the
 * cache, I_K = quantize_NF4(X_K)); SPEC.md:236-244 (causal multi-head scaled
 * dot-product attention of the prompt over the DEQUANTISED K, V).  For query
 * row i of sequence b and head h:
 *   out[b][i][h] = sum_{j <= i, j < seq_lens[b]} softmax_j(softmax_scale * q_i . k^_j) v^_j
 * with k^, v^ = RN32(s * L[code]) dequantised in shared memory (never
 * written to memory).  Runs on the tensor cores (fp16 hi/lo split of k^, v^
 * and the probabilities: ~22-bit operands, fp32 accumulation).
 * q          device fp16 [B][T][H][hd] (token-major, contiguous), 16-byte aligned
 * k_codes,…  the cache tensors (rows 0 .. seq_lens[b]-1 hold the prompt)
 * d_seq_lens device int32[B], prompt lengths (clamped to [0, T])
 * T          query rows per sequence, T <= Tc
 * out        device fp32 [B][T][H][hd], 16-byte aligned; rows i >= seq_lens[b]
 *            are written as 0.
 * No workspace; B, H < 65536. */
int nqkv_prefill_attention(const void* q, const uint8_t* k_codes, const void* k_scales,
                           const uint8_t* v_codes, const void* v_scales, const int32_t* d_seq_lens,
                           int B, int H, int hd, int blk, int Tc, int T, float softmax_scale,
                           float* out, void* stream);

/* K and V of a layer in ONE launch (the fused K+V variant SURVEY.md 8(b)
 * allows): exactly nqkv_quantize(x_k -> k_codes/k_scales) followed by
 * nqkv_quantize(x_v -> v_codes/v_scales), same strides, geometry and d_pos
 * for both, with half the launches (one ramp-up and tail per layer).  Errors
 * as nqkv_quantize; x_k and x_v must agree modulo 32 bytes. */
int nqkv_quantize_pair(const void* x_k, const void* x_v, int64_t stride_b, int64_t stride_t,
                       int64_t stride_h, int B, int H, int hd, int n_new, int blk,
                       const int32_t* d_pos, int Tc, uint8_t* k_codes, void* k_scales,
                       uint8_t* v_codes, void* v_scales, void* stream);

/* KV layouts.  The paper calls both orthogonal to
 * NQKV (multi-query / grouped attention reduce the number of
 * KV heads; PagedAttention's paged KV memory); neither
 * changes an encoded byte or the attention arithmetic, only which cache row
 * a (sequence, head, token) reads (readings R16, R17).
 *   kv_heads       cache heads H_kv (0: = H).  Grouped-query attention: H is
 *                  a multiple of H_kv and H / H_kv a power of two; query head
 *                  h reads cache head h / (H / H_kv).  With blk > hd a block
 *                  spans adjacent CACHE heads.
 *   block_table    NULL: contiguous cache [B][H_kv][Tc][...] (as the plain
 *                  calls).  Else paged: device int32 [B][pages_per_seq] (4-byte
 *                  aligned, caller-owned); codes [n_pages][H_kv][page_size][hd/2],
 *                  scales [n_pages][H_kv][page_size][hd/blk] fp32
 *                  ([n_pages][H_kv*hd/blk][page_size][1] when blk > hd);
 *                  token t of sequence b is row t % page_size of page
 *                  block_table[b][t / page_size].  Page ids out of [0, n_pages)
 *                  are undefined behaviour (not checked on the device).
 *   pages_per_seq  row stride of block_table; pages_per_seq * page_size >= Tc
 *                  (Tc = the per-sequence token capacity, seq_lens <= Tc)
 *   page_size      tokens per page: a power of two >= 64
 *   n_pages        pages in the cache tensors; n_pages * H_kv * page_size * hd/2
 *                  < 2^32
 * Errors: NQKV_ERR_SHAPE (H % H_kv, capacity, sizes), NQKV_ERR_UNSUPPORTED
 * (group or page size not a power of two, page_size < 64, fp16 scales with a
 * paged decode), NQKV_ERR_ALIGN (block_table). */
typedef struct nqkv_kv_layout {
  int kv_heads;
  const int32_t* block_table;
  int pages_per_seq;
  int page_size;
  int n_pages;
} nqkv_kv_layout;

/* nqkv_decode_attention over a KV layout (attention only: append with
 * nqkv_quantize_kv).  Same semantics, workspace (sized with the QUERY head
 * count H) and errors as nqkv_decode_attention; q/out are [B][H][hd].
 * Grouped-query calls (H > H_kv) with blk <= hd (fp32 scales; fp16 scales on
 * a contiguous cache) run a group-native kernel: one CTA streams a chunk of ONE cache head once for up
 * to 4 query heads of its group (groups of 8: two sub-groups), chunks
 * [len*c/nc, len*(c+1)/nc) merged by the last-arriving CTA in chunk order
 * (nc from B, H, H_kv, Tc and the SM count, so the result is reproducible
 * call to call; it equals the MHA kernel's up to fp32 reassociation).  Other
 * grouped-query calls (blk > hd, fp16 scales with NQKV_GQA_TC=0, or
 * NQKV_GQA_NATIVE=0 in the environment, read once) stream each cache head
 * once per query head. */
int nqkv_decode_attention_kv(const void* q, const uint8_t* k_codes, const void* k_scales,
                             const uint8_t* v_codes, const void* v_scales,
                             const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                             const nqkv_kv_layout* kv, float softmax_scale, float* out,
                             void* workspace, size_t ws_bytes, void* stream);
/* nqkv_prefill_attention over a KV layout; q/out [B][T][H][hd]. */
int nqkv_prefill_attention_kv(const void* q, const uint8_t* k_codes, const void* k_scales,
                              const uint8_t* v_codes, const void* v_scales,
                              const int32_t* d_seq_lens, int B, int H, int hd, int blk, int Tc,
                              int T, const nqkv_kv_layout* kv, float softmax_scale, float* out,
                              void* stream);
/* nqkv_quantize into a paged cache (kv->block_table non-NULL) or the
 * contiguous one.  x holds the CACHE heads: kv_heads must be 0 or H.  Rows
 * d_pos[b] .. d_pos[b]+n_new-1 (< Tc) are written; the pages holding them
 * must be in block_table. */
int nqkv_quantize_kv(const void* x, int64_t stride_b, int64_t stride_t, int64_t stride_h, int B,
                     int H, int hd, int n_new, int blk, const int32_t* d_pos, int Tc,
                     const nqkv_kv_layout* kv, uint8_t* codes, void* scales, void* stream);

/* Test hook: the kernels' code function on fp32 inputs already normalised
 * to [-1, 1] (values outside are clamped).  d_n device float[count],
 * d_codes device uint8[count]. */
int nqkv_encode_normalized(const float* d_n, int64_t count, uint8_t* d_codes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NQKV_H_ */
