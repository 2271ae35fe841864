// mea_api.cu — the C ABI of libmea.so (include/mea.h): argument validation, TMA descriptor
// encoding, work decomposition and launches. No allocation, no host synchronisation.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <map>
#include <cstdio>

#include "internal.h"
#include "mea.h"
#include "mea_debug.h"

namespace {

thread_local std::string g_detail;

mea_status_t fail(mea_status_t s, const std::string& why) {
  g_detail = why;
  return s;
}
mea_status_t cuda_fail(cudaError_t e, const char* where) {
  g_detail = std::string(where) + ": " + cudaGetErrorString(e);
  return MEA_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool valid_dtype(mea_dtype_t t) { return t == MEA_F32 || t == MEA_BF16; }

constexpr int64_t kMaxInt = 2147483647;

// ------------------------------------------------------------------ launch profiling
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;

// Brackets one launch with events on `st` when profiling is enabled.
struct ProfScope {
  cudaEvent_t a = nullptr, b = nullptr;
  const char* name;
  cudaStream_t st;
  ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (!g_prof_on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back({name, a, b});
  }
};

}  // namespace

#ifndef MEA_FWD_DB
#define MEA_FWD_DB 1
#endif

namespace mea {

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

cudaError_t make_bnhd_map(CUtensorMap* map, const void* base, CUtensorMapDataType elem, int elem_bytes, int64_t B,
                          int64_t n, int64_t H, int64_t d, int box_inner, int box_rows, CUtensorMapSwizzle swz,
                          const char** why) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) {
    *why = "cuTensorMapEncodeTiled unavailable";
    return cudaErrorNotSupported;
  }
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)n, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)(d * elem_bytes), (cuuint64_t)(H * d * elem_bytes),
                           (cuuint64_t)(n * H * d * elem_bytes)};
  cuuint32_t box[4] = {(cuuint32_t)box_inner, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, elem, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *why = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

}  // namespace mea

using namespace mea;

namespace {

struct FwdPlan {
  int splits = 1, tiles_per_split = 0;
  int64_t q_window = 0;  // query rows per launch (split mode): the paper's query chunk
  size_t ws = 0;
  size_t cnt_off = 0;    // d = 64: byte offset of the fused merge's arrival counters
};

// Key split (k_chunk < n_k): Figure 1's summaries of key chunks of k_chunk keys (rounded up to
// whole 128-key tiles), merged per row afterwards. With q_chunk > 0 the query
// rows are processed in windows of q_chunk rows (rounded up to the 256-row CTA), one after the
// other, as Figure 1's outer map over query chunks does, so the summaries of
// only one query chunk are alive at a time: workspace = splits * B * H * q_window * (d + 2) f32.
// k_chunk == MEA_CHUNK_SQRT_N (-1): the paper's sqrt(n) key chunk, ceil(sqrt(n_k)).
int64_t resolve_k_chunk(int64_t k_chunk, int64_t n_k) {
  if (k_chunk != MEA_CHUNK_SQRT_N) return k_chunk;
  int64_t r = (int64_t)std::ceil(std::sqrt((double)n_k));
  while (r > 1 && (r - 1) * (r - 1) >= n_k) --r;
  while (r * r < n_k) ++r;
  return std::max<int64_t>(r, 1);
}

FwdPlan plan_fwd(int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t q_chunk, int64_t k_chunk, int64_t d) {
  k_chunk = resolve_k_chunk(k_chunk, n_k);
  FwdPlan pl;
  const int64_t n_tiles = (n_k + kTileN - 1) / kTileN;
  pl.tiles_per_split = (int)n_tiles;
  pl.q_window = n_q;
  if (k_chunk > 0 && k_chunk < n_k) {
    const int64_t tps = (k_chunk + kTileN - 1) / kTileN;
    const int64_t splits = (n_tiles + tps - 1) / tps;
    if (splits > 1) {
      pl.splits = (int)splits;
      pl.tiles_per_split = (int)tps;
      if (q_chunk > 0) pl.q_window = std::min(n_q, (q_chunk + kRowsPerCta - 1) / kRowsPerCta * kRowsPerCta);
      pl.ws = (size_t)splits * B * H * pl.q_window * (d + 2) * sizeof(float);
      if (d == kHeadDim && splits <= kFusedMergeMax) {  // + one arrival counter per (b, h, 256-row block)
        pl.cnt_off = (pl.ws + 15) / 16 * 16;
        pl.ws = pl.cnt_off + (size_t)B * H * ((pl.q_window + kRowsPerCta - 1) / kRowsPerCta) * sizeof(unsigned);
      }
    }
  }
  return pl;
}

// f32 inputs at d = 64: three bf16 parts of q, k and v: 6 + 6 + 6 bytes per element
size_t f32tc_workspace(int64_t B, int64_t H, int64_t n_q, int64_t n_k) {
  return (size_t)B * H * kHeadDim * (6 * n_q + 12 * n_k);
}

mea_status_t check_common(int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d, float scale) {
  if (B < 1 || H < 1 || d < 1 || n_q < 0 || n_k < 0) return fail(MEA_ERR_INVALID_VALUE, "B, H, d must be >= 1; n >= 0");
  if (!std::isfinite(scale)) return fail(MEA_ERR_INVALID_VALUE, "scale must be finite");
  if (n_q > kMaxInt || n_k > kMaxInt || B > 65535 || H > 65535)
    return fail(MEA_ERR_UNSUPPORTED, "size beyond the 32-bit grid/coordinate limits");
  return MEA_OK;
}

}  // namespace

extern "C" {

const char* mea_version(void) { return "mea 0.1 sm_100a"; }

const char* mea_status_string(mea_status_t s) {
  switch (s) {
    case MEA_OK: return "MEA_OK";
    case MEA_ERR_INVALID_VALUE: return "MEA_ERR_INVALID_VALUE";
    case MEA_ERR_EMPTY_KEYS: return "MEA_ERR_EMPTY_KEYS";
    case MEA_ERR_UNSUPPORTED: return "MEA_ERR_UNSUPPORTED";
    case MEA_ERR_MISALIGNED: return "MEA_ERR_MISALIGNED";
    case MEA_ERR_WORKSPACE_TOO_SMALL: return "MEA_ERR_WORKSPACE_TOO_SMALL";
    case MEA_ERR_CUDA: return "MEA_ERR_CUDA";
  }
  return "MEA_ERR_UNKNOWN";
}

const char* mea_last_error_detail(void) { return g_detail.c_str(); }

mea_status_t mea_attention_fwd_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                              mea_dtype_t in_dtype, int64_t q_chunk, int64_t k_chunk, size_t* bytes) {
  if (!bytes) return fail(MEA_ERR_INVALID_VALUE, "bytes is NULL");
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, 1.f)) return s;
  if (q_chunk < 0 || (k_chunk < 0 && k_chunk != MEA_CHUNK_SQRT_N)) return fail(MEA_ERR_INVALID_VALUE, "negative chunk size");
  if (!valid_dtype(in_dtype) && in_dtype != MEA_F32_SPLIT) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  k_chunk = resolve_k_chunk(k_chunk, n_k);
  if (in_dtype == MEA_F32_SPLIT)
    *bytes = (d == kHeadDim) ? f32tc_workspace(B, H, n_q, n_k) : 0;
  else if (in_dtype == MEA_F32)
    *bytes = 0;
  else
    *bytes = (d == kHeadDim || d == 128) ? plan_fwd(B, H, n_q, n_k, q_chunk, k_chunk, d).ws : 0;
  return MEA_OK;
}

}  // extern "C"

static mea_status_t fwd_impl(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                             int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t in_dtype, mea_dtype_t out_dtype,
                             float scale, float* lse, int64_t q_chunk, int64_t k_chunk, void* workspace,
                             size_t workspace_bytes, void* stream, bool causal, const int* kv_lens = nullptr,
                             bool stats_only = false) {
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, scale)) return s;
  if (causal && n_q != n_k) return fail(MEA_ERR_UNSUPPORTED, "causal attention needs n_q == n_k");
  if (causal && in_dtype != MEA_BF16) return fail(MEA_ERR_UNSUPPORTED, "causal attention: bf16 path only");
  if (causal) q_chunk = k_chunk = 0;  // causal runs the online schedule (no key split)
  if (q_chunk < 0 || (k_chunk < 0 && k_chunk != MEA_CHUNK_SQRT_N)) return fail(MEA_ERR_INVALID_VALUE, "negative chunk size");
  k_chunk = resolve_k_chunk(k_chunk, n_k);
  if ((!valid_dtype(in_dtype) && in_dtype != MEA_F32_SPLIT) || !valid_dtype(out_dtype))
    return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  if (in_dtype == MEA_F32_SPLIT && (d != kHeadDim || out_dtype != MEA_F32 || causal || (k_chunk > 0 && k_chunk < n_k)))
    return fail(MEA_ERR_UNSUPPORTED, "MEA_F32_SPLIT: d == 64, float32 output, no key chunks, not causal");
  if (n_q == 0) return MEA_OK;
  if (n_k == 0) return fail(MEA_ERR_EMPTY_KEYS, "attention over an empty key list");
  // B0 (backward statistics pass): lse only, no output (d = 64 online schedule)
  if (stats_only && (d != kHeadDim || in_dtype != MEA_BF16 || !lse || (k_chunk > 0 && k_chunk < n_k) || !MEA_FWD_DB))
    return fail(MEA_ERR_UNSUPPORTED, "statistics pass: bf16, d = 64, online schedule, lse required");
  if (!q || !k || !v || (!out && !stats_only)) return fail(MEA_ERR_INVALID_VALUE, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out))
    return fail(MEA_ERR_MISALIGNED, "q, k, v, out must be 16-byte aligned");
  if (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)) return fail(MEA_ERR_MISALIGNED, "lse must be 4-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  if (in_dtype == MEA_F32 || in_dtype == MEA_F32_SPLIT) {
    if (d > 128) return fail(MEA_ERR_UNSUPPORTED, "f32 path supports d <= 128");
    if (out_dtype != MEA_F32) return fail(MEA_ERR_UNSUPPORTED, "f32 inputs need f32 output");
    if (k_chunk > 0 && k_chunk < n_k) return fail(MEA_ERR_UNSUPPORTED, "key chunking is a bf16-path schedule");
    if (in_dtype == MEA_F32_SPLIT) {
      // split-precision tensor-core path (fwd_f32tc_sm100a.cu): q, k, v -> three bf16 parts in the workspace
      const size_t need = f32tc_workspace(B, H, n_q, n_k);
      if (!workspace || workspace_bytes < need) return fail(MEA_ERR_WORKSPACE_TOO_SMALL, "f32 split workspace");
      if (!aligned16(workspace)) return fail(MEA_ERR_MISALIGNED, "workspace must be 16-byte aligned");
      uint8_t* w = static_cast<uint8_t*>(workspace);
      const size_t nq_el = (size_t)B * n_q * H * d, nk_el = (size_t)B * n_k * H * d;
      // q, k, v: three bf16 parts each
      void* qp[3] = {w, w + nq_el * 2, w + nq_el * 4};
      uint8_t* wk = w + nq_el * 6;
      void* kp[3] = {wk, wk + nk_el * 2, wk + nk_el * 4};
      uint8_t* wv = wk + nk_el * 6;
      void* vp[3] = {wv, wv + nk_el * 2, wv + nk_el * 4};
      cudaError_t e;
      {
        ProfScope ps("split_f32", st);
        if ((e = launch_split_f32(static_cast<const float*>(q), qp, 3, (int64_t)nq_el, st)) != cudaSuccess ||
            (e = launch_split_f32(static_cast<const float*>(k), kp, 3, (int64_t)nk_el, st)) != cudaSuccess ||
            (e = launch_split_f32(static_cast<const float*>(v), vp, 3, (int64_t)nk_el, st)) != cudaSuccess)
          return cuda_fail(e, "split_f32 launch");
      }
      CUtensorMap maps[9];
      const char* why = "";
      const void* bases[9] = {qp[0], qp[1], qp[2], kp[0], kp[1], kp[2], vp[0], vp[1], vp[2]};
      for (int i = 0; i < 9; ++i)
        if ((e = make_bnhd_map(&maps[i], bases[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, i < 3 ? n_q : n_k, H, d,
                               64, 128, CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess)
          return cuda_fail(e, why);
      FwdParams p{};
      p.B = (int)B;
      p.H = (int)H;
      p.n_q = (int)n_q;
      p.n_k = (int)n_k;
      p.scale = scale;
      p.scale_log2 = scale * 1.4426950408889634f;
      p.out = out;
      p.out_f32 = 1;
      p.lse = lse;
      ProfScope ps("fwd_f32tc", st);
      if ((e = launch_fwd_f32tc(p, maps, st)) != cudaSuccess) return cuda_fail(e, "fwd_f32tc launch");
      return MEA_OK;
    }
    ProfScope ps("fwd_f32", st);
    cudaError_t e = launch_fwd_f32(static_cast<const float*>(q), static_cast<const float*>(k),
                                   static_cast<const float*>(v), static_cast<float*>(out), lse, (int)B, (int)H,
                                   (int)n_q, (int)n_k, (int)d, scale, st);
    return e == cudaSuccess ? MEA_OK : cuda_fail(e, "fwd_f32 launch");
  }

  if (d != kHeadDim && d != 128) return fail(MEA_ERR_UNSUPPORTED, "bf16 tensor-core path supports d in {64, 128}");
  const FwdPlan pl = plan_fwd(B, H, n_q, n_k, q_chunk, k_chunk, d);
  const int rows_per_cta = d == 128 ? 128 : kRowsPerCta;  // fwd128: one query tile per CTA
  if (pl.ws > 0) {
    if (workspace_bytes < pl.ws || !workspace) return fail(MEA_ERR_WORKSPACE_TOO_SMALL, "key-chunk summaries need workspace");
    if (!aligned16(workspace)) return fail(MEA_ERR_MISALIGNED, "workspace must be 16-byte aligned");
  }
  const int64_t nqb = (n_q + rows_per_cta - 1) / rows_per_cta;
  if (nqb * pl.splits > kMaxInt) return fail(MEA_ERR_UNSUPPORTED, "grid too large");
  if (causal && nqb * B * H > kMaxInt) return fail(MEA_ERR_UNSUPPORTED, "causal grid (blocks x B x H) too large");

  // the plain d = 64 forward (online over all keys, no mask) runs the double-buffered kernel
  const bool use_db = MEA_FWD_DB && d == kHeadDim && pl.splits == 1;
  // key padding is implemented by fwd_db (d = 64) and fwd128 only: never silently drop the mask
  if (kv_lens && d == kHeadDim && !use_db)
    return fail(MEA_ERR_UNSUPPORTED, "key padding needs the online d = 64 forward (no key split; MEA_FWD_DB build)");
  const int key_box = use_db ? fwd_db_key_tile() : kTileN;
  CUtensorMap mq, mk, mv;
  const char* why = "";
  cudaError_t e;
  if ((e = make_bnhd_map(&mq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, kTileM,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, key_box,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, key_box,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess)
    return cuda_fail(e, why);

  FwdParams p{};
  p.B = (int)B;
  p.H = (int)H;
  p.n_q = (int)n_q;
  p.n_k = (int)n_k;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.out_f32 = out_dtype == MEA_F32;
  p.lse = lse;
  p.causal = causal ? 1 : 0;
  p.kv_lens = kv_lens;
  p.stats_only = stats_only ? 1 : 0;
  p.d = (int)d;
  p.num_splits = pl.splits;
  p.tiles_per_split = pl.tiles_per_split;
  if (pl.splits > 1) {
    const size_t rows = (size_t)pl.splits * B * H * pl.q_window;
    p.part_o = static_cast<float*>(workspace);
    p.part_ml = p.part_o + rows * d;
    if (pl.cnt_off > 0) {  // fused merge (last split CTA per query block); counters start at 0
      p.merge_cnt = reinterpret_cast<unsigned*>(static_cast<uint8_t*>(workspace) + pl.cnt_off);
      if ((e = cudaMemsetAsync(p.merge_cnt, 0, pl.ws - pl.cnt_off, st)) != cudaSuccess)
        return cuda_fail(e, "merge counter reset");
    }
  }
  // one window (all rows) unless the key-split schedule runs query chunk by query chunk
  for (int64_t w0 = 0; w0 < n_q; w0 += pl.q_window) {
    p.q_begin = (int)w0;
    p.q_count = (int)std::min<int64_t>(pl.q_window, n_q - w0);
    p.num_q_blocks = (p.q_count + rows_per_cta - 1) / rows_per_cta;
    // windows after the first follow our own forward (its fused merge does not touch q, k, v):
    // the d = 64 split forward may start on the SMs its last wave leaves idle (PDL) and waits for
    // it only before writing summaries
    p.pdl = (w0 > 0 && p.merge_cnt) ? 1 : 0;
    if (d == 128) {
      ProfScope ps("fwd128_bf16", st);
      if ((e = launch_fwd128_bf16(p, mq, mk, mv, st)) != cudaSuccess) return cuda_fail(e, "fwd128_bf16 launch");
    } else if (use_db) {
      ProfScope ps(stats_only ? "bwd_stats" : "fwd_bf16", st);
      if ((e = launch_fwd_db_bf16(p, mq, mk, mv, st)) != cudaSuccess) return cuda_fail(e, "fwd_db_bf16 launch");
    } else {
      ProfScope ps("fwd_bf16", st);
      if ((e = launch_fwd_bf16(p, mq, mk, mv, st)) != cudaSuccess) return cuda_fail(e, "fwd_bf16 launch");
    }
    if (pl.splits > 1 && !p.merge_cnt) {
      ProfScope ps("merge_rows", st);
      if ((e = launch_merge_rows(p, st)) != cudaSuccess) return cuda_fail(e, "merge_rows launch");
    }
  }
  return MEA_OK;
}

// ---------------------------------------------------------------------------------------------
// Multi-stage (tree) summarisation — PAPER.md:183: "A multi-stage summarization approach could
// achieve O(log n)". Per query chunk, the key chunks are summarised one after another (one launch
// of the split-mode forward kernel per chunk, split_base = chunk) and combined like a binary
// counter: level l holds the summary of 2^l consecutive chunks; a new chunk summary merges upward
// (merge_pair, Figure 1's rescale for two summaries) while its level is occupied. At most
// floor(log2(chunks)) + 1 levels are occupied, plus the incoming summary, so the workspace holds
// floor(log2(chunks)) + 2 summaries per query row instead of Figure 1's `chunks`. The remaining
// levels are merged at the end and normalised (merge_rows over one summary: out = v*/s*, lse).
struct TreePlan {
  int64_t kc = 0;          // keys per chunk (a multiple of the 128-key tile)
  int tiles_per_chunk = 0;
  int chunks = 0;
  int slots = 0;           // summaries alive at once
  int64_t q_window = 0;    // query rows per pass
  size_t ws = 0;
};

TreePlan plan_tree(int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t q_chunk, int64_t k_chunk, int64_t d) {
  TreePlan t;
  const int64_t kc = resolve_k_chunk(k_chunk <= 0 ? MEA_CHUNK_SQRT_N : k_chunk, n_k);
  const int64_t n_tiles = (n_k + kTileN - 1) / kTileN;
  t.tiles_per_chunk = (int)std::min<int64_t>(n_tiles, (kc + kTileN - 1) / kTileN);
  t.kc = (int64_t)t.tiles_per_chunk * kTileN;
  t.chunks = (int)((n_tiles + t.tiles_per_chunk - 1) / t.tiles_per_chunk);
  int lg = 0;
  while ((2 << lg) <= t.chunks) ++lg;  // floor(log2(chunks))
  t.slots = lg + 2;
  const int rows_per_cta = d == 128 ? 128 : kRowsPerCta;
  t.q_window = q_chunk > 0 ? std::min(n_q, (q_chunk + rows_per_cta - 1) / rows_per_cta * rows_per_cta) : n_q;
  t.ws = (size_t)t.slots * B * H * t.q_window * (d + 2) * sizeof(float);
  return t;
}

static mea_status_t fwd_tree_impl(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                                  int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t in_dtype, mea_dtype_t out_dtype,
                                  float scale, float* lse, int64_t q_chunk, int64_t k_chunk, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, scale)) return s;
  if (q_chunk < 0 || (k_chunk < 0 && k_chunk != MEA_CHUNK_SQRT_N)) return fail(MEA_ERR_INVALID_VALUE, "negative chunk size");
  if (in_dtype != MEA_BF16 || !valid_dtype(out_dtype))
    return fail(in_dtype == MEA_F32 || in_dtype == MEA_F32_SPLIT ? MEA_ERR_UNSUPPORTED : MEA_ERR_INVALID_VALUE,
                "tree schedule: bf16 inputs, bf16 or f32 output");
  if (d != kHeadDim && d != 128) return fail(MEA_ERR_UNSUPPORTED, "tree schedule supports d in {64, 128}");
  if (n_q == 0) return MEA_OK;
  if (n_k == 0) return fail(MEA_ERR_EMPTY_KEYS, "attention over an empty key list");
  if (!q || !k || !v || !out) return fail(MEA_ERR_INVALID_VALUE, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out))
    return fail(MEA_ERR_MISALIGNED, "q, k, v, out must be 16-byte aligned");
  if (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)) return fail(MEA_ERR_MISALIGNED, "lse must be 4-byte aligned");
  const TreePlan tp = plan_tree(B, H, n_q, n_k, q_chunk, k_chunk, d);
  if (!workspace || workspace_bytes < tp.ws) return fail(MEA_ERR_WORKSPACE_TOO_SMALL, "tree schedule needs workspace");
  if (!aligned16(workspace)) return fail(MEA_ERR_MISALIGNED, "workspace must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rows_per_cta = d == 128 ? 128 : kRowsPerCta;

  CUtensorMap mq, mk, mv;
  const char* why = "";
  cudaError_t e;
  if ((e = make_bnhd_map(&mq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, kTileM,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, kTileN,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, kTileN,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess)
    return cuda_fail(e, why);

  FwdParams p{};
  p.B = (int)B;
  p.H = (int)H;
  p.n_q = (int)n_q;
  p.n_k = (int)n_k;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.out_f32 = out_dtype == MEA_F32;
  p.lse = lse;
  p.d = (int)d;
  p.num_splits = 1;  // one chunk per launch
  p.tiles_per_split = tp.tiles_per_chunk;
  const size_t slot_rows = (size_t)B * H * tp.q_window;
  float* base_o = static_cast<float*>(workspace);
  float2* base_ml = reinterpret_cast<float2*>(base_o + (size_t)tp.slots * slot_rows * d);
  for (int64_t w0 = 0; w0 < n_q; w0 += tp.q_window) {
    p.q_begin = (int)w0;
    p.q_count = (int)std::min<int64_t>(tp.q_window, n_q - w0);
    p.num_q_blocks = (p.q_count + rows_per_cta - 1) / rows_per_cta;
    const int64_t rows = (int64_t)B * H * p.q_count;  // summaries of this pass, [B*H][q_count]
    auto slot_o = [&](int sl) { return base_o + (size_t)sl * rows * d; };
    auto slot_ml = [&](int sl) { return base_ml + (size_t)sl * rows; };
    std::vector<int> free_slots, level_slot(tp.slots, -1);
    for (int sl = tp.slots - 1; sl >= 0; --sl) free_slots.push_back(sl);
    for (int c = 0; c < tp.chunks; ++c) {
      int cur = free_slots.back();
      free_slots.pop_back();
      p.split_base = c;
      p.part_o = slot_o(cur);
      p.part_ml = reinterpret_cast<float*>(slot_ml(cur));
      {
        ProfScope ps(d == 128 ? "fwd128_bf16" : "fwd_bf16", st);
        e = d == 128 ? launch_fwd128_bf16(p, mq, mk, mv, st) : launch_fwd_bf16(p, mq, mk, mv, st);
        if (e != cudaSuccess) return cuda_fail(e, "tree chunk launch");
      }
      for (int l = 0;; ++l) {  // binary-counter carry
        if (level_slot[l] < 0) {
          level_slot[l] = cur;
          break;
        }
        ProfScope ps("merge_pair", st);
        if ((e = launch_merge_pair(slot_o(level_slot[l]), slot_ml(level_slot[l]), slot_o(cur), slot_ml(cur), rows,
                                   (int)d, st)) != cudaSuccess)
          return cuda_fail(e, "merge_pair launch");
        free_slots.push_back(cur);
        cur = level_slot[l];
        level_slot[l] = -1;
      }
    }
    // fold the occupied levels (low to high) into the highest one, then normalise
    int acc = -1;
    for (int l = 0; l < tp.slots; ++l) {
      if (level_slot[l] < 0) continue;
      if (acc >= 0) {
        ProfScope ps("merge_pair", st);
        if ((e = launch_merge_pair(slot_o(level_slot[l]), slot_ml(level_slot[l]), slot_o(acc), slot_ml(acc), rows,
                                   (int)d, st)) != cudaSuccess)
          return cuda_fail(e, "merge_pair launch");
      }
      acc = level_slot[l];
    }
    FwdParams pm = p;
    pm.num_splits = 1;
    pm.part_o = slot_o(acc);
    pm.part_ml = reinterpret_cast<float*>(slot_ml(acc));
    ProfScope ps("merge_rows", st);
    if ((e = launch_merge_rows(pm, st)) != cudaSuccess) return cuda_fail(e, "merge_rows launch");
  }
  return MEA_OK;
}

extern "C" {

mea_status_t mea_attention_fwd_tree(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                                    int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t in_dtype, mea_dtype_t out_dtype,
                                    float scale, float* lse, int64_t q_chunk, int64_t k_chunk, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  return fwd_tree_impl(q, k, v, out, B, H, n_q, n_k, d, in_dtype, out_dtype, scale, lse, q_chunk, k_chunk, workspace,
                       workspace_bytes, stream);
}

mea_status_t mea_attention_fwd_tree_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                                   mea_dtype_t in_dtype, int64_t q_chunk, int64_t k_chunk,
                                                   size_t* bytes) {
  if (!bytes) return fail(MEA_ERR_INVALID_VALUE, "bytes is NULL");
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, 1.f)) return s;
  if (q_chunk < 0 || (k_chunk < 0 && k_chunk != MEA_CHUNK_SQRT_N)) return fail(MEA_ERR_INVALID_VALUE, "negative chunk size");
  if (in_dtype != MEA_BF16) return fail(MEA_ERR_UNSUPPORTED, "tree schedule: bf16 inputs");
  if (d != kHeadDim && d != 128) return fail(MEA_ERR_UNSUPPORTED, "tree schedule supports d in {64, 128}");
  *bytes = (n_q == 0 || n_k == 0) ? 0 : plan_tree(B, H, n_q, n_k, q_chunk, k_chunk, d).ws;
  return MEA_OK;
}

mea_status_t mea_attention_fwd(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                               int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t in_dtype, mea_dtype_t out_dtype,
                               float scale, float* lse, int64_t q_chunk, int64_t k_chunk, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return fwd_impl(q, k, v, out, B, H, n_q, n_k, d, in_dtype, out_dtype, scale, lse, q_chunk, k_chunk, workspace,
                  workspace_bytes, stream, false);
}

mea_status_t mea_attention_fwd_causal(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                                      int64_t n, int64_t d, mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                                      float* lse, void* stream) {
  return fwd_impl(q, k, v, out, B, H, n, n, d, in_dtype, out_dtype, scale, lse, 0, 0, nullptr, 0, stream, true);
}

// ------------------------------------------------------------------ partial self-attention
static mea_status_t partial_fwd_impl(const void* q, const void* k, const void* v, float* m, float* s, float* vstar,
                                     int64_t ms, int64_t vs, int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                     mea_dtype_t in_dtype, float scale, void* stream) {
  if (mea_status_t r = check_common(B, H, n_q, n_k, d, scale)) return r;
  if (!valid_dtype(in_dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  if (in_dtype != MEA_BF16 || (d != kHeadDim && d != 128))
    return fail(MEA_ERR_UNSUPPORTED, "partial forward: bf16, d in {64, 128}");
  if (n_q == 0) return MEA_OK;
  if (!m || !s || !vstar || !q) return fail(MEA_ERR_INVALID_VALUE, "NULL pointer");
  if (!aligned16(q) || !aligned16(vstar) || (reinterpret_cast<uintptr_t>(m) & 3u) ||
      (reinterpret_cast<uintptr_t>(s) & 3u))
    return fail(MEA_ERR_MISALIGNED, "q, vstar must be 16-byte aligned; m, s 4-byte");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (n_k == 0) {  // empty key range: the initial stream state
    ProfScope ps("empty_triples", st);
    e = launch_empty_triples(m, s, vstar, ms, vs, B * n_q * H, (int)d, st);
    return e == cudaSuccess ? MEA_OK : cuda_fail(e, "empty_triples launch");
  }
  if (!k || !v) return fail(MEA_ERR_INVALID_VALUE, "NULL tensor pointer");
  if (!aligned16(k) || !aligned16(v)) return fail(MEA_ERR_MISALIGNED, "k, v must be 16-byte aligned");
  CUtensorMap mq, mk, mv;
  const char* why = "";
  if ((e = make_bnhd_map(&mq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, kTileM,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, kTileN,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, kTileN,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess)
    return cuda_fail(e, why);
  FwdParams p{};
  p.B = (int)B;
  p.H = (int)H;
  p.n_q = (int)n_q;
  p.n_k = (int)n_k;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.num_splits = 1;
  p.tiles_per_split = (int)((n_k + kTileN - 1) / kTileN);
  p.q_begin = 0;
  p.q_count = (int)n_q;
  p.num_q_blocks = (int)((n_q + (d == 128 ? 128 : kRowsPerCta) - 1) / (d == 128 ? 128 : kRowsPerCta));
  p.d = (int)d;
  p.tri_m = m;
  p.tri_s = s;
  p.tri_v = vstar;
  p.tri_vs = (int)vs;
  p.tri_ms = (int)ms;
  if (d == 128) {
    ProfScope ps("fwd128_bf16", st);
    if ((e = launch_fwd128_bf16(p, mq, mk, mv, st)) != cudaSuccess) return cuda_fail(e, "fwd128_bf16 launch");
    return MEA_OK;
  }
  ProfScope ps("fwd_bf16", st);
  if ((e = launch_fwd_bf16(p, mq, mk, mv, st)) != cudaSuccess) return cuda_fail(e, "fwd_bf16 launch");
  return MEA_OK;
}

mea_status_t mea_attention_partial_fwd(const void* q, const void* k, const void* v, float* m, float* s, float* vstar,
                                       int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                       mea_dtype_t in_dtype, float scale, void* stream) {
  return partial_fwd_impl(q, k, v, m, s, vstar, 1, d, B, H, n_q, n_k, d, in_dtype, scale, stream);
}

mea_status_t mea_attention_partial_fwd_packed(const void* q, const void* k, const void* v, float* triples, int64_t B,
                                              int64_t H, int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t in_dtype,
                                              float scale, void* stream) {
  if (!triples && n_q > 0) return fail(MEA_ERR_INVALID_VALUE, "NULL triples");
  return partial_fwd_impl(q, k, v, triples + d, triples + d + 1, triples, d + 4, d + 4, B, H, n_q, n_k, d, in_dtype,
                          scale, stream);
}

// ------------------------------------------------------------------ single query
mea_status_t mea_single_query_workspace_size(int64_t B, int64_t H, int64_t n_k, int64_t d, mea_dtype_t in_dtype,
                                             size_t* bytes) {
  if (!bytes) return fail(MEA_ERR_INVALID_VALUE, "bytes is NULL");
  if (mea_status_t s = check_common(B, H, 1, n_k, d, 1.f)) return s;
  if (!valid_dtype(in_dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  *bytes = sq_plan(B, H, n_k, d, in_dtype == MEA_BF16).bytes;
  return MEA_OK;
}

static mea_status_t sq_common(const void* q, const void* k, const void* v, int64_t B, int64_t H, int64_t n_k,
                              int64_t d, mea_dtype_t in_dtype, float scale, void* workspace, size_t workspace_bytes,
                              SqPlan* plan) {
  if (mea_status_t s = check_common(B, H, 1, n_k, d, scale)) return s;
  if (!valid_dtype(in_dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  if (in_dtype == MEA_BF16 && d != kHeadDim && d != 128)
    return fail(MEA_ERR_UNSUPPORTED, "bf16 single query supports d in {64, 128}");
  if (in_dtype == MEA_F32 && d > 128) return fail(MEA_ERR_UNSUPPORTED, "f32 single query supports d <= 128");
  if (B * H > 65535) return fail(MEA_ERR_UNSUPPORTED, "B*H > 65535");
  if (!q || (n_k > 0 && (!k || !v))) return fail(MEA_ERR_INVALID_VALUE, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v)) return fail(MEA_ERR_MISALIGNED, "q, k, v must be 16-byte aligned");
  *plan = sq_plan(B, H, n_k, d, in_dtype == MEA_BF16);
  if (!workspace || workspace_bytes < plan->bytes)
    return fail(MEA_ERR_WORKSPACE_TOO_SMALL, "single query needs mea_single_query_workspace_size bytes");
  if (reinterpret_cast<uintptr_t>(workspace) & 7u) return fail(MEA_ERR_MISALIGNED, "workspace must be 8-byte aligned");
  return MEA_OK;
}

static SqParams sq_params(const void* q, const void* k, const void* v, int64_t B, int64_t H, int64_t n_k, int64_t d,
                          float scale, void* workspace) {
  SqParams p{};
  p.q = q;
  p.k = k;
  p.v = v;
  p.B = (int)B;
  p.H = (int)H;
  p.n_k = (int)n_k;
  p.d = (int)d;
  p.c = scale * 1.4426950408889634f;
  p.rec = static_cast<float*>(workspace);
  return p;
}

mea_status_t mea_single_query_fwd(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                                  int64_t n_k, int64_t d, mea_dtype_t in_dtype, mea_dtype_t out_dtype, float scale,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  if (n_k == 0 && B >= 1 && H >= 1 && d >= 1) return fail(MEA_ERR_EMPTY_KEYS, "attention over an empty key list");
  if (!valid_dtype(out_dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  SqPlan pl{};
  if (mea_status_t s = sq_common(q, k, v, B, H, n_k, d, in_dtype, scale, workspace, workspace_bytes, &pl)) return s;
  if (!out || !aligned16(out)) return fail(out ? MEA_ERR_MISALIGNED : MEA_ERR_INVALID_VALUE, "bad out pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SqParams p = sq_params(q, k, v, B, H, n_k, d, scale, workspace);
  p.mode = 0;
  p.out = out;
  p.out_f32 = out_dtype == MEA_F32;
  ProfScope ps("sq_fused", st);
  const cudaError_t e = launch_sq(p, pl, in_dtype == MEA_BF16, st);
  return e == cudaSuccess ? MEA_OK : cuda_fail(e, "single query launch");
}

static mea_status_t sq_partial_impl(const void* q, const void* k, const void* v, float* m, float* s, float* vstar,
                                    int64_t ms, int64_t vs, int64_t B, int64_t H, int64_t n_k, int64_t d,
                                    mea_dtype_t in_dtype, float scale, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  SqPlan pl{};
  if (mea_status_t r = sq_common(q, k, v, B, H, n_k, d, in_dtype, scale, workspace, workspace_bytes, &pl)) return r;
  if (!m || !s || !vstar) return fail(MEA_ERR_INVALID_VALUE, "NULL triple pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SqParams p = sq_params(q, k, v, B, H, n_k, d, scale, workspace);
  p.mode = 1;
  p.tri_m = m;
  p.tri_s = s;
  p.tri_v = vstar;
  p.tri_ms_stride = ms;
  p.tri_v_stride = vs;
  ProfScope ps("sq_fused_triple", st);
  const cudaError_t e = launch_sq(p, pl, in_dtype == MEA_BF16, st);
  return e == cudaSuccess ? MEA_OK : cuda_fail(e, "single query launch");
}

mea_status_t mea_single_query_partial(const void* q, const void* k, const void* v, float* m, float* s, float* vstar,
                                      int64_t B, int64_t H, int64_t n_k, int64_t d, mea_dtype_t in_dtype, float scale,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  return sq_partial_impl(q, k, v, m, s, vstar, 1, d, B, H, n_k, d, in_dtype, scale, workspace, workspace_bytes, stream);
}

mea_status_t mea_single_query_partial_packed(const void* q, const void* k, const void* v, float* triples, int64_t B,
                                             int64_t H, int64_t n_k, int64_t d, mea_dtype_t in_dtype, float scale,
                                             void* workspace, size_t workspace_bytes, void* stream) {
  if (!triples) return fail(MEA_ERR_INVALID_VALUE, "NULL triples");
  if (!aligned16(triples)) return fail(MEA_ERR_MISALIGNED, "triples must be 16-byte aligned");
  return sq_partial_impl(q, k, v, triples + d, triples + d + 1, triples, d + 4, d + 4, B, H, n_k, d, in_dtype, scale,
                         workspace, workspace_bytes, stream);
}

static mea_status_t merge_impl(const float* m, const float* s, const float* vstar, int64_t ms, int64_t vs, int64_t P,
                               int64_t rows, int64_t d, void* out, mea_dtype_t out_dtype, void* stream) {
  if (P < 0 || rows < 1 || d < 1) return fail(MEA_ERR_INVALID_VALUE, "bad sizes");
  if (P == 0) return fail(MEA_ERR_EMPTY_KEYS, "no partials to merge");
  if (d > 128) return fail(MEA_ERR_UNSUPPORTED, "d <= 128");
  if (P > kMaxInt) return fail(MEA_ERR_UNSUPPORTED, "P too large");
  if (!valid_dtype(out_dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  if (!m || !s || !vstar || !out) return fail(MEA_ERR_INVALID_VALUE, "NULL pointer");
  if ((rows + 7) / 8 > kMaxInt) return fail(MEA_ERR_UNSUPPORTED, "too many rows");
  ProfScope ps("merge_partials", static_cast<cudaStream_t>(stream));
  cudaError_t e = launch_merge_partials(m, s, vstar, ms, vs, (int)P, rows, (int)d, out, out_dtype == MEA_F32,
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MEA_OK : cuda_fail(e, "merge_partials launch");
}

mea_status_t mea_merge_partials(const float* m, const float* s, const float* vstar, int64_t P, int64_t B, int64_t H,
                                int64_t d, void* out, mea_dtype_t out_dtype, void* stream) {
  if (B < 1 || H < 1) return fail(MEA_ERR_INVALID_VALUE, "bad sizes");
  return merge_impl(m, s, vstar, 1, d, P, B * H, d, out, out_dtype, stream);
}

mea_status_t mea_merge_triples(const float* triples, int64_t P, int64_t rows, int64_t d, void* out,
                               mea_dtype_t out_dtype, void* stream) {
  if (!triples) return fail(MEA_ERR_INVALID_VALUE, "NULL triples");
  return merge_impl(triples + d, triples + d + 1, triples, d + 4, d + 4, P, rows, d, out, out_dtype, stream);
}

// ------------------------------------------------------------------ backward
namespace {
struct BwdLayout {
  size_t delta, lse2, dq_acc, aug, lse_tmp, out_tmp, total;
};
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
BwdLayout bwd_layout(int64_t B, int64_t H, int64_t n_q, int64_t d, bool lse_given, bool fused) {
  const size_t nq_pad = (size_t)((n_q + kTileM - 1) / kTileM) * kTileM;
  const size_t rows_pad = (size_t)B * H * nq_pad;
  BwdLayout L{};
  size_t off = 0;
  L.delta = off;  off = align256(off + rows_pad * sizeof(float));
  L.lse2 = off;   off = align256(off + rows_pad * sizeof(float));
  if (fused) {  // the fused kernel's dQ reduction target (+ at d = 64 its score K-extension tiles)
    L.dq_acc = off; off = align256(off + (size_t)B * n_q * H * d * sizeof(float));
    if (d == kHeadDim) {
      L.aug = off;  off = align256(off + rows_pad / kTileM * 2 * kAugTileBytes);
    }
  }
  if (!lse_given) {  // B0: lse recomputed (d = 64: statistics pass, no output; d = 128: full forward)
    L.lse_tmp = off; off = align256(off + (size_t)B * H * n_q * sizeof(float));
    if (d != kHeadDim) {
      L.out_tmp = off; off = align256(off + (size_t)B * n_q * H * d * 2);
    }
  }
  L.total = off;
  return L;
}
}  // namespace

mea_status_t mea_attention_bwd_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                                              mea_dtype_t dtype, int lse_given, size_t* bytes) {
  if (!bytes) return fail(MEA_ERR_INVALID_VALUE, "bytes is NULL");
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, 1.f)) return s;
  if (!valid_dtype(dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  *bytes = bwd_layout(B, H, n_q, d, lse_given != 0, true).total;  // the fused path (d = 64 and 128)
  return MEA_OK;
}

}  // extern "C"

static mea_status_t bwd_impl(const void* q, const void* k, const void* v, const void* out, const void* dout, void* dq,
                             void* dk, void* dv, int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                             mea_dtype_t dtype, float scale, const float* lse, void* workspace,
                             size_t workspace_bytes, void* stream, bool fused, bool causal = false,
                             const int* kv_lens = nullptr) {
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, scale)) return s;
  if (causal && n_q != n_k) return fail(MEA_ERR_UNSUPPORTED, "causal attention needs n_q == n_k");
  if (causal && scale == 0.f) return fail(MEA_ERR_UNSUPPORTED, "causal backward needs scale != 0");
  if (!valid_dtype(dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  if (n_k == 0) return fail(MEA_ERR_EMPTY_KEYS, "attention over an empty key list");
  if (dtype != MEA_BF16 || (d != kHeadDim && d != 128)) return fail(MEA_ERR_UNSUPPORTED, "backward: bf16, d in {64, 128}");
  if (!k || !v || !dk || !dv) return fail(MEA_ERR_INVALID_VALUE, "NULL tensor pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (n_q == 0) {  // no queries: the gradients of k and v are zero
    if (!aligned16(dk) || !aligned16(dv)) return fail(MEA_ERR_MISALIGNED, "dk, dv must be 16-byte aligned");
    const size_t nb = (size_t)B * n_k * H * d * 2;
    if ((e = cudaMemsetAsync(dk, 0, nb, st)) != cudaSuccess || (e = cudaMemsetAsync(dv, 0, nb, st)) != cudaSuccess)
      return cuda_fail(e, "memset");
    return MEA_OK;
  }
  if (!q || !out || !dout || !dq) return fail(MEA_ERR_INVALID_VALUE, "NULL tensor pointer");
  // The d = 64 fused kernel folds lse/scale into its score MMA; scale == 0 (all scores 0, P
  // uniform) takes the two-kernel path, whose workspace is a prefix-sized subset of the fused one.
  // The d = 128 fused kernel (bwd128_sm100a.cu) reads lse per column and takes any scale.
  if (fused && scale == 0.f && d == kHeadDim) fused = false;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out) || !aligned16(dout) || !aligned16(dq) ||
      !aligned16(dk) || !aligned16(dv))
    return fail(MEA_ERR_MISALIGNED, "tensors must be 16-byte aligned");
  // causal grids are 1-D over (key or query blocks) x B x H
  if (causal && ((std::max(n_q, n_k) + 63) / 64) * B * H > kMaxInt)
    return fail(MEA_ERR_UNSUPPORTED, "causal grid (blocks x B x H) too large");
  const BwdLayout L = bwd_layout(B, H, n_q, d, lse != nullptr, fused);
  if (!workspace || workspace_bytes < L.total) return fail(MEA_ERR_WORKSPACE_TOO_SMALL, "backward workspace");
  if (!aligned16(workspace)) return fail(MEA_ERR_MISALIGNED, "workspace must be 16-byte aligned");
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  float* delta = reinterpret_cast<float*>(ws + L.delta);
  float* lse2 = reinterpret_cast<float*>(ws + L.lse2);
  float* dq_acc = fused ? reinterpret_cast<float*>(ws + L.dq_acc) : nullptr;
  uint8_t* aug = fused && d == kHeadDim ? ws + L.aug : nullptr;

  CUtensorMap mq, mk, mv, mdo, mdq;
  const char* why = "";
  if ((e = make_bnhd_map(&mq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, kTileM,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mdo, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, kTileM,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, kTileN,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, kTileN,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (fused && (e = make_bnhd_map(&mdq, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, n_q, H, d, 32,
                                   d == kHeadDim ? kTileM : 64, CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess))
    return cuda_fail(e, why);

  if (!lse) {
    // B0: the statistics pass. d = 64: Q K^T and the exponential row sums
    // only (fwd_db_kernel<true>: no V, no P V, no output); d = 128: the forward rerun with its
    // output in scratch.
    float* lse_tmp = reinterpret_cast<float*>(ws + L.lse_tmp);
    const bool stats = d == kHeadDim;
    mea_status_t r = fwd_impl(q, k, v, stats ? nullptr : ws + L.out_tmp, B, H, n_q, n_k, d, MEA_BF16, MEA_BF16, scale,
                              lse_tmp, 0, 0, nullptr, 0, stream, causal, kv_lens, stats);
    if (r != MEA_OK) return r;
    lse = lse_tmp;
  }
  {
    ProfScope ps("bwd_preprocess", st);
    if ((e = launch_bwd_preprocess(out, dout, lse, delta, lse2, dq_acc, aug, scale, (int)B, (int)H, (int)n_q, (int)d,
                                   st)) != cudaSuccess)
      return cuda_fail(e, "bwd_preprocess launch");
  }
  BwdParams p{};
  p.B = (int)B;
  p.H = (int)H;
  p.n_q = (int)n_q;
  p.n_k = (int)n_k;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.lse2 = lse2;
  p.delta = delta;
  p.dk = dk;
  p.dv = dv;
  p.dq_acc = dq_acc;
  p.aug = aug;
  p.dq = dq;
  p.dq_acc = dq_acc;
  p.num_k_blocks = (int)((n_k + kTileN - 1) / kTileN);
  p.causal = causal ? 1 : 0;
  p.kv_lens = kv_lens;
  p.d = (int)d;
  if (fused && d == 128) {
    // 64-query tiles (TMEM holds dV and dK at 128 columns each): Q / dO boxes of 64 rows
    CUtensorMap mq_t, mdo_t;
    if ((e = make_bnhd_map(&mq_t, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, 64,
                           CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
        (e = make_bnhd_map(&mdo_t, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, 64,
                           CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess)
      return cuda_fail(e, why);
    {
      ProfScope ps("bwd128", st);
      if ((e = launch_bwd128(p, mq_t, mk, mv, mdo_t, mdq, st)) != cudaSuccess) return cuda_fail(e, "bwd128 launch");
    }
    ProfScope ps("dq_convert", st);
    if ((e = launch_dq_convert(dq_acc, dq, B * n_q * H * d, scale, st)) != cudaSuccess)
      return cuda_fail(e, "dq_convert launch");
  } else if (fused) {
    {
      ProfScope ps("bwd_bf16", st);
      if ((e = launch_bwd_bf16(p, mq, mk, mv, mdo, mdq, st)) != cudaSuccess) return cuda_fail(e, "bwd_bf16 launch");
    }
    ProfScope ps("dq_convert", st);
    if ((e = launch_dq_convert(dq_acc, dq, B * n_q * H * d, scale, st)) != cudaSuccess)
      return cuda_fail(e, "dq_convert launch");
  } else {
    {
      // d = 128: the dK/dV kernel takes 64-query tiles (TMEM), so its Q / dO boxes are 64 rows
      CUtensorMap mq_t = mq, mdo_t = mdo;
      if (d == 128 &&
          ((e = make_bnhd_map(&mq_t, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, 64,
                              CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
           (e = make_bnhd_map(&mdo_t, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_q, H, d, 64, 64,
                              CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess))
        return cuda_fail(e, why);
      ProfScope ps("bwd_dkdv", st);
      if ((e = launch_bwd_dkdv(p, mq_t, mk, mv, mdo_t, st)) != cudaSuccess) return cuda_fail(e, "bwd_dkdv launch");
    }
    // d = 128: the dQ kernel takes 64-key tiles (a 4-stage K/V ring next to resident Q, dO)
    CUtensorMap mk_t = mk, mv_t = mv;
    if (d == 128 &&
        ((e = make_bnhd_map(&mk_t, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, 64,
                            CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
         (e = make_bnhd_map(&mv_t, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, n_k, H, d, 64, 64,
                            CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess))
      return cuda_fail(e, why);
    ProfScope ps("bwd_dq", st);
    if ((e = launch_bwd_dq(p, mq, mk_t, mv_t, mdo, st)) != cudaSuccess) return cuda_fail(e, "bwd_dq launch");
  }
  return MEA_OK;
}

extern "C" {

mea_status_t mea_attention_bwd(const void* q, const void* k, const void* v, const void* out, const void* dout, void* dq,
                               void* dk, void* dv, int64_t B, int64_t H, int64_t n_q, int64_t n_k, int64_t d,
                               mea_dtype_t dtype, float scale, const float* lse, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return bwd_impl(q, k, v, out, dout, dq, dk, dv, B, H, n_q, n_k, d, dtype, scale, lse, workspace, workspace_bytes,
                  stream, true);
}

mea_status_t mea_attention_bwd_causal(const void* q, const void* k, const void* v, const void* out,
                                      const void* dout, void* dq, void* dk, void* dv, int64_t B, int64_t H, int64_t n,
                                      int64_t d, mea_dtype_t dtype, float scale, const float* lse, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  return bwd_impl(q, k, v, out, dout, dq, dk, dv, B, H, n, n, d, dtype, scale, lse, workspace, workspace_bytes,
                  stream, true, true);
}

// Key padding: per batch element, keys >= kv_lens[b] are masked.
static mea_status_t check_kv_lens(const int* kv_lens, mea_dtype_t dtype) {
  if (!kv_lens) return fail(MEA_ERR_INVALID_VALUE, "kv_lens is NULL");
  if (reinterpret_cast<uintptr_t>(kv_lens) & 3u) return fail(MEA_ERR_MISALIGNED, "kv_lens must be 4-byte aligned");
  if (dtype != MEA_BF16) return fail(valid_dtype(dtype) ? MEA_ERR_UNSUPPORTED : MEA_ERR_INVALID_VALUE,
                                     "key padding: bf16 path only");
  return MEA_OK;
}

mea_status_t mea_attention_bwd_padded(const void* q, const void* k, const void* v, const void* out, const void* dout,
                                      void* dq, void* dk, void* dv, int64_t B, int64_t H, int64_t n_q, int64_t n_k,
                                      int64_t d, mea_dtype_t dtype, float scale, const float* lse,
                                      const int* kv_lens, void* workspace, size_t workspace_bytes, void* stream) {
  if (mea_status_t s = check_kv_lens(kv_lens, dtype)) return s;
  return bwd_impl(q, k, v, out, dout, dq, dk, dv, B, H, n_q, n_k, d, dtype, scale, lse, workspace, workspace_bytes,
                  stream, true, false, kv_lens);
}

mea_status_t mea_attention_fwd_padded(const void* q, const void* k, const void* v, void* out, int64_t B, int64_t H,
                                      int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t in_dtype,
                                      mea_dtype_t out_dtype, float scale, float* lse, const int* kv_lens,
                                      void* stream) {
  if (mea_status_t s = check_kv_lens(kv_lens, in_dtype)) return s;
  return fwd_impl(q, k, v, out, B, H, n_q, n_k, d, in_dtype, out_dtype, scale, lse, 0, 0, nullptr, 0, stream, false,
                  kv_lens);
}

mea_status_t mea_attention_bwd_deterministic_workspace_size(int64_t B, int64_t H, int64_t n_q, int64_t n_k,
                                                            int64_t d, mea_dtype_t dtype, int lse_given,
                                                            size_t* bytes) {
  if (!bytes) return fail(MEA_ERR_INVALID_VALUE, "bytes is NULL");
  if (mea_status_t s = check_common(B, H, n_q, n_k, d, 1.f)) return s;
  if (!valid_dtype(dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad dtype");
  *bytes = bwd_layout(B, H, n_q, d, lse_given != 0, false).total;
  return MEA_OK;
}

mea_status_t mea_attention_bwd_deterministic(const void* q, const void* k, const void* v, const void* out,
                                             const void* dout, void* dq, void* dk, void* dv, int64_t B, int64_t H,
                                             int64_t n_q, int64_t n_k, int64_t d, mea_dtype_t dtype, float scale,
                                             const float* lse, void* workspace, size_t workspace_bytes,
                                             void* stream) {
  return bwd_impl(q, k, v, out, dout, dq, dk, dv, B, H, n_q, n_k, d, dtype, scale, lse, workspace, workspace_bytes,
                  stream, false);
}

// ------------------------------------------------------------------ generator / debug
mea_status_t mea_fill_synthetic(void* dst, int64_t numel, mea_dtype_t dtype, uint64_t seed, uint32_t tensor_id,
                                int64_t offset, void* stream) {
  if (numel < 0 || offset < 0 || !valid_dtype(dtype)) return fail(MEA_ERR_INVALID_VALUE, "bad arguments");
  if (numel == 0) return MEA_OK;
  if (!dst) return fail(MEA_ERR_INVALID_VALUE, "NULL dst");
  ProfScope ps("fill_synthetic", static_cast<cudaStream_t>(stream));
  cudaError_t e = launch_fill_synthetic(dst, numel, dtype == MEA_BF16, seed, tensor_id, offset,
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MEA_OK : cuda_fail(e, "fill launch");
}

void mea_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
}

mea_status_t mea_profile_read(char* buf, size_t cap) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    recs.swap(g_prof);
  }
  std::map<std::string, std::pair<int, double>> agg;
  cudaError_t err = cudaSuccess;
  for (auto& r : recs) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess) err = e;
    auto& x = agg[r.name];
    x.first += 1;
    x.second += ms;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  std::string out;
  char line[160];
  for (auto& kv : agg) {
    snprintf(line, sizeof line, "%s %d %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
    out += line;
  }
  if (buf && cap) {
    size_t n = out.size() < cap - 1 ? out.size() : cap - 1;
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return err == cudaSuccess ? MEA_OK : cuda_fail(err, "profile events");
}

mea_status_t mea_debug_set_option(const char* name, int value) {
  if (!name) return fail(MEA_ERR_INVALID_VALUE, "NULL name");
  const std::string n(name);
  if (n == "sq_heads_per_cta") mea::g_sq_heads_per_cta = value;
  else if (n == "sq_ctas_per_sm") mea::g_sq_ctas_per_sm = value;
  else if (n == "sq_l2_256") mea::g_sq_l2_256 = value;
  else if (n == "sq_static_pct") mea::g_sq_static_pct = value;
  else return fail(MEA_ERR_INVALID_VALUE, "unknown option");
  return MEA_OK;
}

mea_status_t mea_debug_read_probe(const void* p, size_t bytes, int ctas, float* sink, void* stream) {
  if (!p || !sink || !aligned16(p) || (bytes & 15u)) return fail(MEA_ERR_INVALID_VALUE, "bad read probe arguments");
  const cudaError_t e = mea::launch_read_probe(p, bytes, ctas, sink, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MEA_OK : cuda_fail(e, "read probe launch");
}

mea_status_t mea_debug_umma_tile(const void* a, const void* b, const void* v, float* s_out, float* o_out,
                                 void* stream) {
  if (!a || !b || !v || !s_out || !o_out) return fail(MEA_ERR_INVALID_VALUE, "NULL pointer");
  CUtensorMap ma, mb, mv;
  const char* why = "";
  cudaError_t e;
  if ((e = make_bnhd_map(&ma, a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 1, 128, 1, 64, 64, 128,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mb, b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 1, 128, 1, 64, 64, 128,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess ||
      (e = make_bnhd_map(&mv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 1, 128, 1, 64, 64, 128,
                         CU_TENSOR_MAP_SWIZZLE_128B, &why)) != cudaSuccess)
    return cuda_fail(e, why);
  e = launch_debug_umma_tile(ma, mb, mv, s_out, o_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MEA_OK : cuda_fail(e, "debug launch");
}

}  // extern "C"
