/*
 * mea.h — memory-efficient exact attention on NVIDIA B200 (sm_100a).
 *
 * C ABI of libmea.so. Implements the hot path of Rabe & Staats, "Self-attention
 * Does Not Need O(n^2) Memory" (arXiv 2112.05682): exact softmax attention
 *     s_i = dot(q, k_i) * scale,  out = sum_i v_i e^{s_i} / sum_j e^{s_j}
 * (Eq. (1) at PAPER.md:50-53), evaluated key tile by key tile with
 * the running value sum v*, weight sum s* and running max m* of PAPER.md:85-90,
 * so the n_q x n_k score matrix is never stored. The backward pass recomputes each
 * tile of scores from per-row statistics (checkpointing).
 *
 * Conventions (all entry points):
 *  - Every data pointer is a DEVICE pointer owned by the caller. The library never
 *    allocates, frees or synchronises; scratch is the caller-provided workspace,
 *    whose size the *_workspace_size queries return. Outputs are fully overwritten.
 *    Outputs must not alias inputs.
 *  - Layouts are dense row-major: q/out/dout/dq [B, n_q, H, d]; k/v/dk/dv
 *    [B, n_k, H, d]; lse [B, H, n_q] (float32, natural log); single-query q/out
 *    [B, H, d]. Base pointers must be 16-byte aligned.
 *  - ``scale`` multiplies every score. Figure 1 uses 1/sqrt(d); the
 *    paper's Secs. 1-3 use 1. Must be finite.
 *  - ``stream`` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    stream-ordered and asynchronous: a MEA_OK return means the work was enqueued.
 *  - Errors are detected before any launch and returned as mea_status_t; nothing is
 *    launched on error. No exception or abort crosses the ABI.
 *      n_q == 0 (or B*H == 0 work)    -> MEA_OK, nothing launched
 *      n_k == 0                       -> MEA_ERR_EMPTY_KEYS (an explicit error, not NaN)
 *      B, H, d < 1, chunk < 0, bad dtype, non-finite scale -> MEA_ERR_INVALID_VALUE
 *      shape/dtype not implemented    -> MEA_ERR_UNSUPPORTED
 *      pointer not 16-byte aligned    -> MEA_ERR_MISALIGNED
 *      workspace smaller than needed  -> MEA_ERR_WORKSPACE_TOO_SMALL
 *      CUDA launch/encode failure     -> MEA_ERR_CUDA (detail in mea_last_error_detail)
 *  - Non-finite input values are not checked; they propagate.
 *  - Supported: bf16 inputs with d = 64 or d = 128 on every entry point (tcgen05 tensor-core
 *    kernels; single query: streaming SIMT kernels); f32 inputs with 1 <= d <= 128 (exact-f32 SIMT kernels, forward and
 *    single query).
 */
#ifndef MEA_H_
#define MEA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MEA_API __attribute__((visibility("default")))
#else
#define MEA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/*
 * MEA_F32_SPLIT (mea_attention_fwd's in_dtype only): float32 tensors computed on the bf16 tensor
 * cores by split precision (q, k, v and P each in three bf16 parts, 24 bits; S and O as 6
 * products each down to 2^-16 of the leading term, every key tile's P.V summed into a fresh TMEM
 * tile and added to v* in fp32 registers; d == 64, float32 output, no key chunks, not causal).
 * Scores, lse and outputs meet the strict fp32 bar (1e-5 absolute) at any finite scale
 * (tests/test_gpu_forward.py::test_f32_split_precision_tensor_core_path). MEA_F32 is exact fp32
 * FFMA arithmetic (any d <= 128), the default fp32 path.
 */
typedef enum { MEA_F32 = 0, MEA_BF16 = 1, MEA_F32_SPLIT = 2 } mea_dtype_t;

/* k_chunk value selecting the paper's sqrt(n) key chunk, ceil(sqrt(n_k)) keys (PAPER.md:179:
 * "Assuming a chunk size of sqrt(n) for the keys and values ... O(sqrt(n)) memory"). */
#define MEA_CHUNK_SQRT_N (-1)

typedef enum {
  MEA_OK = 0,
  MEA_ERR_INVALID_VALUE = 1,
  MEA_ERR_EMPTY_KEYS = 2,
  MEA_ERR_UNSUPPORTED = 3,
  MEA_ERR_MISALIGNED = 4,
  MEA_ERR_WORKSPACE_TOO_SMALL = 5,
  MEA_ERR_CUDA = 6
} mea_status_t;

/* Library version, e.g. "mea 0.1 sm_100a". Static string. */
MEA_API const char* mea_version(void);
/* Static description of a status code. */
MEA_API const char* mea_status_string(mea_status_t status);
/* Thread-local detail of the last error on this thread (e.g. which check failed). */
MEA_API const char* mea_last_error_detail(void);

/*
 * Self-/cross-attention forward (PAPER.md:21-25 with PAPER.md:85-90; Figure 1,
 * PAPER.md:107-163, gives the chunked schedule).
 *   q [B,n_q,H,d], k,v [B,n_k,H,d] of in_dtype; out [B,n_q,H,d] of out_dtype.
 *   lse [B,H,n_q] float32, nullable: lse_i = log sum_j e^{s_ij}, the per-row residual
 *     the backward pass consumes.
 *   q_chunk, k_chunk: the paper's query_chunk_size / key_chunk_size;
 *     k_chunk = MEA_CHUNK_SQRT_N picks ceil(sqrt(n_k)).
 *     0 = default schedule: every work item streams all keys with an on-chip running
 *     (v*, s*, m*), zero workspace. k_chunk in (0, n_k) selects the paper's key-chunk
 *     summaries: each chunk's (m*, s*, v*) goes to the workspace
 *     and a merge pass combines them (bf16 path; rounded up to a multiple of 128
 *     keys). With a key split, q_chunk > 0 processes the query rows in chunks of
 *     q_chunk rows (rounded up to 256), one after another, as Figure 1's outer map over
 *     query chunks does, so only one chunk's summaries are alive:
 *     workspace = splits * B * H * min(n_q, q_chunk') * (d + 2) * 4 bytes (at d = 64 with at
 *     most 16 splits rounded up to 16 bytes, + 4 bytes per (b, h, 256-row query block of a
 *     chunk): the arrival counters of the merge, which the last key-chunk CTA of each query
 *     block then performs in the same launch). Without a key split q_chunk has no effect. Results do not depend on q_chunk.
 *   in_dtype MEA_BF16 requires d in {64, 128} and out_dtype in {BF16, F32};
 *   in_dtype MEA_F32 requires d <= 128, out_dtype F32 and k_chunk == 0.
 */
MEA_API mea_status_t mea_attention_fwd(const void* q, const void* k, const void* v, void* out,
                               int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                               mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                               float* lse, int64_t q_chunk, int64_t k_chunk,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes mea_attention_fwd needs for these arguments (0 unless 0 < k_chunk < n_k;
 * k_chunk = MEA_CHUNK_SQRT_N selects ceil(sqrt(n_k)) in both calls). */
MEA_API mea_status_t mea_attention_fwd_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k,
                                              int64_t d, mea_dtype_t in_dtype, int64_t q_chunk,
                                              int64_t k_chunk, size_t* bytes);

/*
 * The paper's chunked forward with multi-stage (tree) summarisation ("A multi-stage
 * summarization approach could achieve O(log n) but would complicate the implementation";
 * SURVEY.md §8(f) item 1). For each query chunk of q_chunk rows (0 = all rows; rounded up to the
 * CTA's 256 rows, 128 at d = 128), processed one after another, the key chunks
 * of k_chunk keys (MEA_CHUNK_SQRT_N or 0 = ceil(sqrt(n_k)); rounded up to a multiple of 128) are
 * summarised one after another (Figure 1 lines 12-19) and merged like a binary
 * counter with Figure 1's rescale for two summaries: level l holds the
 * summary of 2^l consecutive chunks, a new summary carries upward while its level is occupied,
 * and the occupied levels are merged and normalised at the end (out = v* / s*).
 * At most floor(log2(chunks)) + 2 summaries per query row are alive:
 *   workspace = (floor(log2(chunks)) + 2) * B * H * q_rows * (d + 2) * 4 bytes
 * (mea_attention_fwd_tree_workspace_size) instead of Figure 1's chunks * (...). Same arguments,
 * layouts and results (within rounding) as mea_attention_fwd; bf16 inputs with d in {64, 128}
 * (MEA_ERR_UNSUPPORTED otherwise). One kernel launch per (query chunk, key chunk): a schedule
 * for memory fidelity, not speed (the default online schedule needs no workspace at all).
 */
MEA_API mea_status_t mea_attention_fwd_tree(const void* q, const void* k, const void* v, void* out,
                                    int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                    mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                                    float* lse, int64_t q_chunk, int64_t k_chunk,
                                    void* workspace, size_t workspace_bytes, void* stream);
MEA_API mea_status_t mea_attention_fwd_tree_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k,
                                                   int64_t d, mea_dtype_t in_dtype, int64_t q_chunk,
                                                   int64_t k_chunk, size_t* bytes);

/*
 * Causal self-attention forward (not in the paper, which disabled
 * packing to avoid masking; reimplementations added it): query i
 * attends keys j <= i only. q, k, v, out [B,n,H,d] (n_q == n_k == n, top-left aligned), lse as
 * for mea_attention_fwd. bf16 inputs with d in {64, 128} (MEA_ERR_UNSUPPORTED otherwise); online
 * schedule (no key chunks), no workspace. Key tiles past a query tile's diagonal are skipped.
 */
MEA_API mea_status_t mea_attention_fwd_causal(const void* q, const void* k, const void* v, void* out,
                                      int64_t B, int64_t H, int64_t n, int64_t d,
                                      mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                                      float* lse, void* stream);

/*
 * Key padding (masking needed to drop the library into a Transformer over
 * a padded batch; the paper disabled packing to avoid it): batch element b attends
 * only keys j < kv_lens[b] (clamped to [0, n_k]); the masked keys get probability 0 (scores
 * -inf in the definition). kv_lens [B] int32 is a DEVICE array (read by the
 * kernels, never by the host; 4-byte aligned; MEA_ERR_INVALID_VALUE if NULL). A row with no
 * keys (kv_lens[b] = 0) yields out = 0 and lse = -inf. Otherwise as mea_attention_fwd on the
 * online schedule (no key chunks, no causal mask); bf16 inputs with d in {64, 128}
 * (MEA_ERR_UNSUPPORTED otherwise). Padded query rows need no mask: rows are independent.
 */
MEA_API mea_status_t mea_attention_fwd_padded(const void* q, const void* k, const void* v, void* out,
                                      int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                      mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                                      float* lse, const int* kv_lens, void* stream);

/*
 * Single-query attention per (b,h) — the paper's O(1)-memory algorithm (PAPER.md:59-63,
 * stabilised as in PAPER.md:85-90). q,out [B,H,d]; k,v [B,n_k,H,d]. Keys are split into
 * ranges processed in parallel (split-K); each range yields a triple (m*, s*, v*) in the
 * workspace and the last CTA of each (b, head block) merges them with Figure 1's
 * global-max rescale in the same launch. Workspace (>= 8-byte aligned,
 * mea_single_query_workspace_size bytes) is independent of n_k (bounded by the split count);
 * its contents need no initialisation (counters left by a call are reset by that call;
 * uninitialised ones are recognised and restarted). Calls sharing one workspace must be
 * stream-ordered.
 */
MEA_API mea_status_t mea_single_query_fwd(const void* q, const void* k, const void* v, void* out,
                                  int64_t B, int64_t H, int64_t n_k, int64_t d,
                                  mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                                  void* workspace, size_t workspace_bytes, void* stream);

MEA_API mea_status_t mea_single_query_workspace_size(int64_t B, int64_t H, int64_t n_k, int64_t d,
                                             mea_dtype_t in_dtype, size_t* bytes);

/*
 * Multi-GPU building blocks for attention sharded over key ranges (MNNFast-style KV
 * sharding; merge = PAPER.md:140-147).
 * mea_single_query_partial writes, per (b,h), the stream state over this call's keys:
 *   m [B*H]      : reference max (natural-log units of the scaled score), an observed
 *                  score, so m <= the true max; the lazily updated reference of the
 *                  tensor-core kernels may lag it by up to 64*ln2 (every term e^{s_j - m}
 *                  is certified < 2^64, reading 9; the single-query kernel
 *                  keeps the exact blocked max). All terms are relative to m,
 *   s [B*H]      : s* = sum_j e^{s_j - m}  (so 1 <= s* < n_k * 2^64 for n_k >= 1),
 *   vstar [B*H*d]: v* = sum_j v_j e^{s_j - m}   (all float32).
 * n_k == 0 is allowed here and yields the empty triple (-inf, 0, 0).
 * mea_merge_partials combines P stacked triples m [P,B*H], s [P,B*H], vstar [P,B*H,d]
 * into out [B,H,d] (out_dtype); for self-attention rows pass H := n_q * H (out [B,n_q,H,d]). Empty triples contribute nothing; all-empty rows are
 * MEA_ERR_EMPTY_KEYS only if detectable on the host (P == 0), else they yield NaN.
 */
/*
 * Self-attention over one key range, as a stream state per query row (multi-GPU building block:
 * key-range sharding of long-context self-attention; the merge is
 * mea_merge_partials with H := n_q * H).
 *   q [B,n_q,H,d], k,v [B,n_k,H,d] bf16, d in {64, 128} (MEA_ERR_UNSUPPORTED otherwise).
 *   m [B,n_q,H], s [B,n_q,H], vstar [B,n_q,H,d] float32 outputs, same meaning as for
 *   mea_single_query_partial (m in natural-log units of the scaled score).
 *   n_k == 0 yields the empty triple (-inf, 0, 0) for every row; n_q == 0 is a no-op.
 * No workspace. Errors as mea_attention_fwd.
 */
MEA_API mea_status_t mea_attention_partial_fwd(const void* q, const void* k, const void* v, float* m,
                                       float* s, float* vstar, int64_t B, int64_t H, int64_t n_q,
                                       int64_t n_k, int64_t d, mea_dtype_t in_dtype, float scale,
                                       void* stream);

MEA_API mea_status_t mea_single_query_partial(const void* q, const void* k, const void* v, float* m,
                                      float* s, float* vstar, int64_t B, int64_t H, int64_t n_k,
                                      int64_t d, mea_dtype_t in_dtype, float scale,
                                      void* workspace, size_t workspace_bytes, void* stream);

MEA_API mea_status_t mea_merge_partials(const float* m, const float* s, const float* vstar, int64_t P,
                                int64_t B, int64_t H, int64_t d, void* out, mea_dtype_t out_dtype,
                                void* stream);

/*
 * Packed triples, for a collective that moves one buffer (torch all_gather_into_tensor):
 * record r = { v*[0..d), m, s, 0-pad, 0-pad }: MEA_TRIPLE_FLOATS(d) = d + 4 floats (16-byte
 * aligned rows), same meanings as above (m natural log). The partial calls write
 * [B*H] (single query) or [B*n_q*H] (self-attention, row (b, i, h)) records; the pad floats
 * are not written. mea_merge_triples merges P stacked record arrays [P][rows] into out
 * [rows, d] (out_dtype): the layout an all-gather of every rank's records produces.
 * triples must be 16-byte aligned. Errors as the unpacked calls.
 */
#define MEA_TRIPLE_FLOATS(d) ((d) + 4)
MEA_API mea_status_t mea_single_query_partial_packed(const void* q, const void* k, const void* v, float* triples,
                                             int64_t B, int64_t H, int64_t n_k, int64_t d,
                                             mea_dtype_t in_dtype, float scale, void* workspace,
                                             size_t workspace_bytes, void* stream);
MEA_API mea_status_t mea_attention_partial_fwd_packed(const void* q, const void* k, const void* v, float* triples,
                                              int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                              mea_dtype_t in_dtype, float scale, void* stream);
MEA_API mea_status_t mea_merge_triples(const float* triples, int64_t P, int64_t rows, int64_t d, void* out,
                               mea_dtype_t out_dtype, void* stream);

/*
 * Backward of out = attention(q, k, v) (the VJP the paper obtains with jax.grad through
 * jax.checkpoint): given dout, writes dq, dk, dv (same dtype/layout as
 * q, k, v). Scores and probabilities are recomputed tile by tile from lse (PAPER.md:256:
 * "recomputed during backpropagation"); no n_q x n_k buffer exists. lse is the forward's
 * residual; NULL makes the call recompute it first (one extra statistics pass).
 * The max carries no gradient (stop_gradient).
 * Workspace: delta [B,H,n_q] f32 + dq accumulator [B,n_q,H,d] f32 (+ lse if NULL).
 * bf16 with d in {64, 128}: one fused kernel per call at either d (dq reduced across key tiles
 * in the f32 accumulator, so dq is reproducible only to rounding order; use
 * mea_attention_bwd_deterministic for bitwise results); d = 64 with scale == 0 runs the
 * two-kernel path of mea_attention_bwd_deterministic (the workspace asked for here covers it).
 */
MEA_API mea_status_t mea_attention_bwd(const void* q, const void* k, const void* v, const void* out,
                               const void* dout, void* dq, void* dk, void* dv, int64_t B,
                               int64_t H, int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t dtype,
                               float scale, const float* lse, void* workspace,
                               size_t workspace_bytes, void* stream);

/*
 * Backward of mea_attention_fwd_padded: as mea_attention_bwd (same workspace,
 * mea_attention_bwd_workspace_size), with keys j >= kv_lens[b] masked (kv_lens as for the
 * forward); their dk, dv rows are written as 0. lse NULL recomputes it with the same padding.
 */
MEA_API mea_status_t mea_attention_bwd_padded(const void* q, const void* k, const void* v, const void* out,
                                      const void* dout, void* dq, void* dk, void* dv, int64_t B,
                                      int64_t H, int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t dtype,
                                      float scale, const float* lse, const int* kv_lens,
                                      void* workspace, size_t workspace_bytes, void* stream);

/*
 * Deterministic backward: same contract and results as mea_attention_bwd (within tolerance), but
 * dK/dV and dQ come from two kernels with no cross-CTA reduction, so the result is bitwise
 * reproducible run to run and the workspace is only delta and lse (B*H*n_q*8 bytes, + lse and a
 * forward-output scratch if lse is NULL) instead of the fp32 dQ accumulator. Costs two extra
 * recomputed GEMMs per tile (slower than mea_attention_bwd).
 */
MEA_API mea_status_t mea_attention_bwd_deterministic(const void* q, const void* k, const void* v,
                                                     const void* out, const void* dout, void* dq, void* dk,
                                                     void* dv, int64_t B, int64_t H, int64_t n_q,
                                                     int64_t n_k, int64_t d, mea_dtype_t dtype, float scale,
                                                     const float* lse, void* workspace,
                                                     size_t workspace_bytes, void* stream);

MEA_API mea_status_t mea_attention_bwd_deterministic_workspace_size(int64_t B, int64_t H, int64_t n_q,
                                                                    int64_t n_k, int64_t d,
                                                                    mea_dtype_t dtype, int lse_given,
                                                                    size_t* bytes);

MEA_API mea_status_t mea_attention_bwd_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k,
                                              int64_t d, mea_dtype_t dtype, int lse_given,
                                              size_t* bytes);

/*
 * Backward of mea_attention_fwd_causal: arguments as mea_attention_bwd with n_q == n_k == n;
 * lse (nullable) must come from the causal forward. Workspace: mea_attention_bwd_workspace_size
 * (B, H, n, n, d, dtype, lse_given). scale == 0 is MEA_ERR_UNSUPPORTED here. Each key tile
 * loops over the query tiles from its diagonal on.
 */
MEA_API mea_status_t mea_attention_bwd_causal(const void* q, const void* k, const void* v,
                                      const void* out, const void* dout, void* dq, void* dk,
                                      void* dv, int64_t B, int64_t H, int64_t n, int64_t d,
                                      mea_dtype_t dtype, float scale, const float* lse,
                                      void* workspace, size_t workspace_bytes, void* stream);

/*
 * Synthetic input generator (not part of the method; used by tests and the bench so
 * large configs never cross PCIe). Fills dst[i] = value(seed, tensor_id, offset + i),
 * i < numel, with the counter-based Irwin-Hall(12) generator documented in
 * synth/gen.py, rounded to dtype (RNE). Bit-identical to the host generator.
 */
MEA_API mea_status_t mea_fill_synthetic(void* dst, int64_t numel, mea_dtype_t dtype, uint64_t seed,
                                uint32_t tensor_id, int64_t offset, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MEA_H_ */
