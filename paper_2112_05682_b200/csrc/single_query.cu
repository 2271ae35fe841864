// single_query.cu — the paper's O(1)-memory single-query attention (made
// stable by the running max of PAPER.md:85-90), split over key ranges (split-K), plus the
// merge of the per-range states with Figure 1's global-max rescale.
//
// HBM-bound: every key costs 4*d bytes (k and v rows, bf16) and 4*d flops, 1 flop/byte.
// bf16 d=64 kernel: a warp reads 16 keys per step; 8 lanes share one 128-byte key row
// (16 B = 8 bf16 each, coalesced 128-bit loads), the dot product finishes with 3 xor-shuffles
// inside the 8-lane group, and each group runs its own stream state (m*, s*, v*[8 dims per
// lane]) with one rescale per 4 keys (block max first). Groups, warps and CTAs are then
// merged with the same rescale rule. Two steps are unrolled so 8 K and 8 V loads (256 B)
// per lane are in flight.
//
// Partial layout (workspace, float32): part[(bh * splits + split) * (d + 2) + {0: m*, 1: s*,
// 2..: v*}], with m* in log2 units of the scaled score (p = 2^(s*c - m*), c = scale*log2 e).
#include <cuda_bf16.h>

#include <cmath>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

#ifndef MEA_SQ_THREADS
#define MEA_SQ_THREADS 512
#endif
#ifndef MEA_SQ_UNROLL
#define MEA_SQ_UNROLL 2
#endif
#ifndef MEA_SQ_CTAS
#define MEA_SQ_CTAS 148
#endif
constexpr int kSqThreads = MEA_SQ_THREADS;  // one CTA per SM: 16 warps x 256 B x 2 steps in flight
constexpr int kSqWarps = kSqThreads / 32;
// D = 64: 8 lanes per 128-byte key row, 4 key groups per warp; D = 128: 16 lanes per 256-byte
// row, 2 groups. Every lane holds 8 dims of its group's state.
template <int D> struct SqCfg {
  static constexpr int LPR = D / 8;                  // lanes per key row
  static constexpr int G = 32 / LPR;                 // key groups per warp
  static constexpr int kKeysPerWarpStep = 4 * G;     // 4 keys per group per step
};
constexpr int kUnroll = MEA_SQ_UNROLL;  // warp steps in flight

struct State {
  float m, l, a[8];
};

// Merge state o into s (both relative to their own reference max).
__device__ __forceinline__ void merge_state(State& s, const State& o) {
  const float M = fmaxf(s.m, o.m);
  if (M == -INFINITY) return;
  const float ws = ex2_approx(s.m - M), wo = ex2_approx(o.m - M);
  s.l = s.l * ws + o.l * wo;
#pragma unroll
  for (int i = 0; i < 8; ++i) s.a[i] = s.a[i] * ws + o.a[i] * wo;
  s.m = M;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int D>
__global__ void __launch_bounds__(kSqThreads) sq_partial_bf16_kernel(const __nv_bfloat16* __restrict__ q,
                                                                     const __nv_bfloat16* __restrict__ k,
                                                                     const __nv_bfloat16* __restrict__ v, int H,
                                                                     int n_k, float scale_log2, int splits,
                                                                     float* __restrict__ part) {
  asm volatile("griddepcontrol.launch_dependents;");
  using C = SqCfg<D>;
  constexpr int LPR = C::LPR, kKeysPerWarpStep = C::kKeysPerWarpStep;
  const int split = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, cidx = lane % LPR;  // key group in the warp, 16-byte chunk of the row
  const int per = (n_k + splits - 1) / splits;
  const int k_lo = split * per, k_hi = min(n_k, k_lo + per);
  const size_t row_stride = (size_t)H * D;  // elements between consecutive keys
  const __nv_bfloat16* kb = k + ((size_t)b * n_k * H + h) * D + cidx * 8;
  const __nv_bfloat16* vb = v + ((size_t)b * n_k * H + h) * D + cidx * 8;

  float qf[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(q + (size_t)bh * D + cidx * 8), qf);
#pragma unroll
  for (int i = 0; i < 8; ++i) qf[i] *= scale_log2;

  State st;
  st.m = -INFINITY;
  st.l = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) st.a[i] = 0.f;

  constexpr int kStep = kSqWarps * kKeysPerWarpStep;  // keys per CTA step
  for (int base = k_lo + warp * kKeysPerWarpStep; base < k_hi; base += kStep * kUnroll) {
    uint4 kr[kUnroll][4], vr[kUnroll][4];
#pragma unroll
    for (int s = 0; s < kUnroll; ++s)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int key = base + s * kStep + u * C::G + g;
        if (key < k_hi) {
          kr[s][u] = ld_stream(kb + (size_t)key * row_stride);
          vr[s][u] = ld_stream(vb + (size_t)key * row_stride);
        } else {
          kr[s][u] = make_uint4(0, 0, 0, 0);
          vr[s][u] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
    for (int s = 0; s < kUnroll; ++s) {
      float sc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float kf[8];
        bf16x8_to_f32(kr[s][u], kf);
        float dot = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) dot = fmaf(qf[i], kf[i], dot);
#pragma unroll
        for (int o = 1; o < LPR; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const int key = base + s * kStep + u * C::G + g;
        sc[u] = key < k_hi ? dot : -INFINITY;
      }
      const float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
      const float m_new = fmaxf(st.m, mx);
      if (m_new == -INFINITY) continue;  // nothing valid yet for this group
      const float alpha = ex2_approx(st.m - m_new);
      st.l *= alpha;
#pragma unroll
      for (int i = 0; i < 8; ++i) st.a[i] *= alpha;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float pu = ex2_approx(sc[u] - m_new);
        st.l += pu;
        float vf[8];
        bf16x8_to_f32(vr[s][u], vf);
#pragma unroll
        for (int i = 0; i < 8; ++i) st.a[i] = fmaf(pu, vf[i], st.a[i]);
      }
      st.m = m_new;
    }
  }
  // merge the key groups of the warp (lanes with equal cidx hold the same 8 dims)
#pragma unroll
  for (int off = LPR; off <= 16; off <<= 1) {
    State o;
    o.m = __shfl_xor_sync(0xffffffffu, st.m, off);
    o.l = __shfl_xor_sync(0xffffffffu, st.l, off);
#pragma unroll
    for (int i = 0; i < 8; ++i) o.a[i] = __shfl_xor_sync(0xffffffffu, st.a[i], off);
    merge_state(st, o);
  }
  __shared__ float sm_m[kSqWarps], sm_l[kSqWarps], sm_a[kSqWarps][D];
  if (lane < LPR) {
    if (lane == 0) {
      sm_m[warp] = st.m;
      sm_l[warp] = st.l;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sm_a[warp][cidx * 8 + i] = st.a[i];
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const int f = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < kSqWarps; ++w) M = fmaxf(M, sm_m[w]);
    float l = 0.f, a = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < kSqWarps; ++w) {
        const float wt = ex2_approx(sm_m[w] - M);
        l += wt * sm_l[w];
        a += wt * sm_a[w][f];
      }
    }
    float* dst = part + ((size_t)bh * splits + split) * (D + 2);
    if (f == 0) {
      dst[0] = M;
      dst[1] = l;
    }
    dst[2 + f] = a;
  }
}

// f32 inputs, any d <= 128: one warp per key, lanes own dims {lane, lane+32, lane+64, lane+96}.
__global__ void __launch_bounds__(128) sq_partial_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                            const float* __restrict__ v, int H, int n_k, int d,
                                                            float scale_log2, int splits, float* __restrict__ part) {
  const int split = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = (n_k + splits - 1) / splits;
  const int k_lo = split * per, k_hi = min(n_k, k_lo + per);
  float qf[4], a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) qf[i] = (lane + 32 * i < d) ? q[(size_t)bh * d + lane + 32 * i] : 0.f;
  float m = -INFINITY, l = 0.f;
  for (int key = k_lo + warp; key < k_hi; key += 4) {
    const size_t off = (((size_t)b * n_k + key) * H + h) * d;
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < d) dot = fmaf(qf[i], k[off + lane + 32 * i], dot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const float s = dot * scale_log2;
    const float m_new = fmaxf(m, s);
    const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
    const float p = exp2f(s - m_new);
    l = l * alpha + p;
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = a[i] * alpha + ((lane + 32 * i < d) ? p * v[off + lane + 32 * i] : 0.f);
    m = m_new;
  }
  __shared__ float sm_m[4], sm_l[4], sm_a[4][128];
  if (lane == 0) {
    sm_m[warp] = m;
    sm_l[warp] = l;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) sm_a[warp][lane + 32 * i] = a[i];
  __syncthreads();
  if (threadIdx.x < d) {
    const int f = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w]);
    float ls = 0.f, as = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < 4; ++w) {
        const float wt = exp2f(sm_m[w] - M);
        ls += wt * sm_l[w];
        as += wt * sm_a[w][f];
      }
    float* dst = part + ((size_t)bh * splits + split) * (d + 2);
    if (f == 0) {
      dst[0] = M;
      dst[1] = ls;
    }
    dst[2 + f] = as;
  }
}

// Merge `splits` partial states per (b,h) (Figure 1 lines 33-40):
//   M = max m_s;  out = sum_s 2^(m_s - M) v*_s / sum_s 2^(m_s - M) s*_s.
// One CTA of 8 warps per (b,h): the max by a block reduction, then warp w folds splits
// w, w+8, ... (lanes own dims lane + 32 i, 4 independent loads in flight per lane), then
// the 8 warp results are combined. mode 0: out (dtype); mode 1: the merged triple with m in
// natural-log units (m_nat = m ln 2) for the cross-GPU merge.
constexpr int kMergeWarps = 8;
__global__ void __launch_bounds__(kMergeWarps * 32) sq_merge_kernel(const float* __restrict__ part, int splits,
                                                                    int d, int mode, void* out, int out_f32,
                                                                    float* m_out, float* s_out, float* v_out) {
  // PDL: everything above this point may overlap the tail of the partial kernel.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int bh = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* base = part + (size_t)bh * splits * (d + 2);
  __shared__ float sm_red[kMergeWarps], sm_l[kMergeWarps], sm_a[kMergeWarps][128];
  float M = -INFINITY;
  for (int s = threadIdx.x; s < splits; s += blockDim.x) M = fmaxf(M, base[(size_t)s * (d + 2)]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  if (lane == 0) sm_red[warp] = M;
  __syncthreads();
  M = sm_red[0];
#pragma unroll
  for (int w = 1; w < kMergeWarps; ++w) M = fmaxf(M, sm_red[w]);
  float l = 0.f, a[4] = {0.f, 0.f, 0.f, 0.f};
  if (M != -INFINITY) {
    // 16 splits per warp per round, all loads issued before any use (latency-bound otherwise)
    for (int s0 = warp; s0 < splits; s0 += 16 * kMergeWarps) {
      float mw[16], lw[16], vw[16][4];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int s = s0 + u * kMergeWarps;
        const bool ok = s < splits;
        const float* ps = base + (size_t)(ok ? s : 0) * (d + 2);
        mw[u] = ok ? ps[0] : -INFINITY;
        lw[u] = ok ? ps[1] : 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) vw[u][i] = (ok && lane + 32 * i < d) ? ps[2 + lane + 32 * i] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float w = exp2f(mw[u] - M);
        l = fmaf(w, lw[u], l);
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = fmaf(w, vw[u][i], a[i]);
      }
    }
  }
  if (lane == 0) sm_l[warp] = l;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (lane + 32 * i < d) sm_a[warp][lane + 32 * i] = a[i];
  __syncthreads();
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < kMergeWarps; ++w) {
      L += sm_l[w];
      A += sm_a[w][f];
    }
    if (mode == 0) {
      const float r = A / L;
      if (out_f32) static_cast<float*>(out)[(size_t)bh * d + f] = r;
      else static_cast<__nv_bfloat16*>(out)[(size_t)bh * d + f] = __float2bfloat16_rn(r);
    } else {
      if (f == 0) {
        m_out[bh] = M * 0.6931471805599453f;
        s_out[bh] = L;
      }
      v_out[(size_t)bh * d + f] = A;
    }
  }
}

// Cross-rank merge: P triples with natural-log m. One warp per row (a (b,h)
// of a single query, or a (b, query, h) row of self-attention), lanes over the d features.
__global__ void merge_partials_kernel(const float* __restrict__ m, const float* __restrict__ s,
                                      const float* __restrict__ vstar, int P, int64_t rows, int d, void* out,
                                      int out_f32) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float M = -INFINITY;
  for (int i = 0; i < P; ++i) M = fmaxf(M, m[(size_t)i * rows + r]);
  float L = 0.f, A[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < P; ++i) {
    const float mi = m[(size_t)i * rows + r];
    const float w = (mi == -INFINITY) ? 0.f : expf(mi - M);
    L += w * s[(size_t)i * rows + r];
    const float* vi = vstar + ((size_t)i * rows + r) * d;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (lane + 32 * j < d) A[j] += w * vi[lane + 32 * j];
  }
  const float inv = 1.f / L;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int f = lane + 32 * j;
    if (f >= d) break;
    if (out_f32) static_cast<float*>(out)[(size_t)r * d + f] = A[j] * inv;
    else static_cast<__nv_bfloat16*>(out)[(size_t)r * d + f] = __float2bfloat16_rn(A[j] * inv);
  }
}

}  // namespace

// Splits: one 512-thread CTA per SM streaming (HBM needs ~35 KB in flight per SM; a CTA has
// 256 KB in flight), at least ~1024 keys per split, so the merge stays small.
int sq_num_splits(int64_t BH, int64_t n_k) {
  const int64_t target_ctas = MEA_SQ_CTAS;
  int64_t splits = (target_ctas + BH - 1) / BH;
  const int64_t max_by_keys = (n_k + 1023) / 1024;
  if (splits > max_by_keys) splits = max_by_keys;
  if (splits < 1) splits = 1;
  if (splits > 4096) splits = 4096;
  return (int)splits;
}

cudaError_t launch_sq_partial(const void* q, const void* k, const void* v, int bf16, int B, int H, int n_k, int d,
                              float scale, int splits, float* ws, cudaStream_t s) {
  const float c = scale * 1.4426950408889634f;
  dim3 grid(splits, B * H);
  if (bf16 && d == 128) {
    sq_partial_bf16_kernel<128><<<grid, kSqThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(q),
                                                           static_cast<const __nv_bfloat16*>(k),
                                                           static_cast<const __nv_bfloat16*>(v), H, n_k, c, splits, ws);
  } else if (bf16) {
    sq_partial_bf16_kernel<64><<<grid, kSqThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(q),
                                                          static_cast<const __nv_bfloat16*>(k),
                                                          static_cast<const __nv_bfloat16*>(v), H, n_k, c, splits, ws);
  } else {
    sq_partial_f32_kernel<<<grid, 128, 0, s>>>(static_cast<const float*>(q), static_cast<const float*>(k),
                                               static_cast<const float*>(v), H, n_k, d, c, splits, ws);
  }
  return cudaGetLastError();
}

cudaError_t launch_sq_merge(const float* ws, int splits, int BH, int d, int mode, void* out, int out_f32, float* m,
                            float* sum, float* vstar, cudaStream_t s) {
  // Programmatic dependent launch: the merge grid is scheduled while the partial kernel
  // drains and waits (griddepcontrol.wait) for its results, hiding the launch gap.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(BH);
  cfg.blockDim = dim3(kMergeWarps * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sq_merge_kernel, ws, splits, d, mode, out, out_f32, m, sum, vstar);
}

cudaError_t launch_merge_partials(const float* m, const float* s, const float* vstar, int P, int64_t rows, int d,
                                  void* out, int out_f32, cudaStream_t st) {
  merge_partials_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(m, s, vstar, P, rows, d, out, out_f32);
  return cudaGetLastError();
}

}  // namespace mea
