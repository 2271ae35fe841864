// internal.h — launcher interfaces between the C-ABI layer (mea_api.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>

namespace mea {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is per
// device, and one process may drive several GPUs (a plain function-local static would set it on
// the first device only).
template <auto Kernel>
inline cudaError_t ensure_smem_attr(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

constexpr int kHeadDim = 64;      // tensor-core path head dimension
constexpr int kTileM = 128;       // query rows per softmax warpgroup (UMMA M)
constexpr int kTileN = 128;       // keys per tile (UMMA N of QK^T, K of PV)
constexpr int kRowsPerCta = 256;  // two query tiles per CTA share each K/V tile

constexpr int kFusedMergeMax = 16;  // key splits the in-kernel merge handles (more: merge_rows)

struct FwdParams {
  int B, H, n_q, n_k;
  float scale_log2;        // scale * log2(e): exponent base change folded into one FFMA
  float scale;
  void* out;               // [B,n_q,H,64], bf16 or f32 (unused in split mode)
  int out_f32;
  float* lse;              // [B,H,n_q] natural log, nullable
  int q_begin, q_count;    // query-row window of this launch (paper's query chunk)
  int num_q_blocks;        // ceil(q_count / 256)
  int num_splits;          // key splits (1 = online over all keys)
  int tiles_per_split;     // key tiles of 128 per split
  int split_base;          // key chunk of blockIdx split 0 (tree schedule: one chunk per launch)
  float* part_o;           // [splits][B*H][q_count][d] unnormalised v* (split / tree mode; non-null
                           // selects the summary epilogue)
  float* part_ml;          // [splits][B*H][q_count][2]  (m* in log2 units, s*) (split mode)
  float* tri_m;            // partial mode (mea_attention_partial_fwd): [B,n_q,H] m* (natural log)
  float* tri_s;            //   [B,n_q,H] s*
  float* tri_v;            //   [B,n_q,H,64] v* (unnormalised)
  int tri_vs, tri_ms;      //   floats between rows of tri_v (d) and of tri_m / tri_s (1); packed
                           //   records {v*[d], m, s, pad, pad}: both d + 4
  int causal;              // query i sees keys j <= i (n_q == n_k, one window, no key split)
  int d;                   // head dimension (64: fwd_bf16, 128: fwd128_bf16); merge_rows reads it
  unsigned* merge_cnt;     // d = 64 key split: [B*H][num_q_blocks] arrival counters (zeroed, self-
                           // resetting); the last split CTA of a query block merges its rows
  int pdl;                 // programmatic dependent launch (key-split windows after the first): the
                           // kernel may start while the previous window's merge drains; it waits
                           // (griddepcontrol.wait) only before its first global write
  const int* kv_lens;      // [B] keys per batch element (key padding: keys >= kv_lens[b] masked);
                           // nullable; online schedule only (no causal mask, no key split)
  int stats_only;          // B0 (fwd_db, d = 64): row statistics only — lse written, no V, no out
};

struct BwdParams {
  int B, H, n_q, n_k;
  int d;                   // head dimension: 64 or 128
  float scale, scale_log2;
  const float* lse2;       // [B*H][nq_pad]: lse * log2(e), +inf in the padding
  const float* delta;      // [B*H][nq_pad]: dO_i . O_i, 0 in the padding
  const uint8_t* aug;      // fused kernel: per (b,h, 128-query tile) 8 KiB = the bf16 K-extension
                           // tiles [lse/scale hi, lo] and [delta hi, lo] (see bwd_preprocess)
  void* dk;                // [B,n_k,H,64] bf16
  void* dv;                // [B,n_k,H,64] bf16
  void* dq;                // [B,n_q,H,64] bf16 (deterministic path writes it directly)
  float* dq_acc;           // [B,n_q,H,64] f32 reduction target (fused path)
  int num_k_blocks;        // ceil(n_k / 128)
  int causal;              // query i sees keys j <= i (n_q == n_k): query tiles from the diagonal on
  const int* kv_lens;      // [B] key padding (keys >= kv_lens[b] get P = 0 and zero dK, dV); nullable
};

// keys batch element b attends: min(n_k, max(0, kv_lens[b])) with key padding, else n_k
__device__ __forceinline__ int keys_of(const int* kv_lens, int b, int n_k) {
  return kv_lens ? min(n_k, max(0, __ldg(kv_lens + b))) : n_k;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_fn();

// 4-D tensor map over a [B, n, H, d] tensor (d innermost), box {64, 1, box_rows, 1},
// 128-byte swizzle. elem = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 or FLOAT32.
cudaError_t make_bnhd_map(CUtensorMap* map, const void* base, CUtensorMapDataType elem, int elem_bytes,
                          int64_t B, int64_t n, int64_t H, int64_t d, int box_inner, int box_rows,
                          CUtensorMapSwizzle swz, const char** why);

cudaError_t launch_fwd_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                            const CUtensorMap& mv, cudaStream_t s);
cudaError_t launch_merge_rows(const FwdParams& p, cudaStream_t s);
// dst <- dst (+) src for `rows` summaries (v* [rows][d], (m* log2, s*) [rows]): the pairwise merge
// of the tree schedule (PAPER.md:140-147 applied to two summaries).
cudaError_t launch_merge_pair(float* dst_o, float2* dst_ml, const float* src_o, const float2* src_ml, int64_t rows,
                              int d, cudaStream_t s);
// d = 64 forward with double-buffered 96-key score tiles (fwd_db_sm100a.cu): online over all
// keys (causal or not), no key split, no triple output; K/V maps with fwd_db_key_tile() rows.
int fwd_db_key_tile();
cudaError_t launch_fwd_db_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                               const CUtensorMap& mv, cudaStream_t s);
cudaError_t launch_fwd128_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                               const CUtensorMap& mv, cudaStream_t s);
cudaError_t launch_split_f32(const float* x, void* const* parts, int nparts, int64_t n, cudaStream_t s);
cudaError_t launch_fwd_f32tc(const FwdParams& p, const CUtensorMap (&maps)[9], cudaStream_t s);
cudaError_t launch_empty_triples(float* m, float* s, float* vstar, int64_t ms, int64_t vs, int64_t rows, int d,
                                 cudaStream_t st);
cudaError_t launch_fwd_f32(const float* q, const float* k, const float* v, float* out, float* lse, int B,
                           int H, int n_q, int n_k, int d, float scale, cudaStream_t s);

// single query (single_query.cu): one kernel per call, the last CTA of each group merges
struct SqParams {
  const void *q, *k, *v;   // q [B,H,d]; k, v [B,n_k,H,d]
  int B, H, n_k, d;
  float c;                 // scale * log2(e)
  int splits;              // key ranges per (b, head block)
  float* rec;              // workspace: partial records [B*H][splits][d+2], then the tickets
  unsigned long long* tickets;  // [groups] arrival tickets (single_query.cu counter_take)
  unsigned long long* claims;   // [groups] dynamic-pool claim counters (same tagged scheme)
  int static_keys;         // keys of each split's static range (pool mode: split * static_keys ...)
  int chunk_keys;          // keys per pool chunk (one CTA step)
  int pool_begin;          // first key of the dynamic pool (= splits * static_keys)
  int pool_chunks;         // chunks in the pool (0: static ranges only)
  int mode;                // 0: out = attention; 1: the merged triple (m natural log, s, v*)
  void* out;               // mode 0: [B,H,d] bf16 or f32
  int out_f32;
  float *tri_m, *tri_s, *tri_v;  // mode 1: row bh at tri_m[bh*ms], tri_s[bh*ms], tri_v[bh*vs + f]
  int64_t tri_ms_stride, tri_v_stride;
};
struct SqPlan {
  int hc, splits;
  int static_keys, chunk_keys, pool_begin, pool_chunks;
  int64_t groups;
  size_t rec_bytes, bytes;
};
SqPlan sq_plan(int64_t B, int64_t H, int64_t n_k, int64_t d, int bf16);
cudaError_t launch_sq(SqParams p, const SqPlan& pl, int bf16, cudaStream_t s);
extern int g_sq_heads_per_cta, g_sq_ctas_per_sm, g_sq_l2_256, g_sq_static_pct;
// m at m[(i*rows + r)*ms], s likewise, v* at vstar[(i*rows + r)*vs + f]
cudaError_t launch_merge_partials(const float* m, const float* s, const float* vstar, int64_t ms, int64_t vs, int P,
                                  int64_t rows, int d, void* out, int out_f32, cudaStream_t st);
cudaError_t launch_read_probe(const void* p, size_t bytes, int ctas, float* sink, cudaStream_t s);

// backward
// dq_acc nullable: zeroed when given (fused path)
cudaError_t launch_bwd_preprocess(const void* out, const void* dout, const float* lse, float* delta, float* lse2,
                                  float* dq_acc, uint8_t* aug, float scale, int B, int H, int n_q, int d,
                                  cudaStream_t s);
constexpr int kAugTileBytes = 4096;   // 128 rows x 16 bf16, no-swizzle K-major core matrices
cudaError_t launch_bwd_bf16(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                            const CUtensorMap& mdo, const CUtensorMap& mdq, cudaStream_t s);
cudaError_t launch_dq_convert(const float* dq_acc, void* dq, int64_t numel, float scale, cudaStream_t s);
// d = 128 fused backward (bwd128_sm100a.cu): mq / mdo boxes of 64 rows, mdq {32, 1, 64, 1} f32
cudaError_t launch_bwd128(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                          const CUtensorMap& mdo, const CUtensorMap& mdq, cudaStream_t s);
cudaError_t launch_bwd_dkdv(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                            const CUtensorMap& mdo, cudaStream_t s);
cudaError_t launch_bwd_dq(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                          const CUtensorMap& mdo, cudaStream_t s);

// generator
cudaError_t launch_fill_synthetic(void* dst, int64_t numel, int bf16, uint64_t seed, uint32_t tid,
                                  int64_t offset, cudaStream_t s);

// debug probe
cudaError_t launch_debug_umma_tile(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mv,
                                   float* s_out, float* o_out, cudaStream_t s);

}  // namespace mea
