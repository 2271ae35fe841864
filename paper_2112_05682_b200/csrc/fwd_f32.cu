// fwd_f32.cu — exact-fp32 forward on the CUDA cores (configuration 1, f32 parity).
//
// tf32 tensor-core MMA (10-bit mantissa) cannot meet a 1e-5 absolute bound, so the f32 path
// is plain FFMA. One thread = one query row running the paper's stable stream
// over key tiles of 32 staged in shared memory; within a tile the max is
// taken first and v*, s* are rescaled once (the blocked form of the same update).
#include <cmath>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

constexpr int kF32Rows = 128;  // query rows (threads) per CTA
constexpr int kF32Keys = 32;   // keys per shared-memory tile

template <int DP>  // head dim padded to DP (d <= DP); padding is zero so it changes nothing
__global__ void __launch_bounds__(kF32Rows) fwd_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                          const float* __restrict__ v, float* __restrict__ out,
                                                          float* __restrict__ lse, int B, int H, int n_q, int n_k,
                                                          int d, float scale_log2) {
  __shared__ float ks[kF32Keys][DP];
  __shared__ float vs[kF32Keys][DP];
  __shared__ float ss[kF32Keys][kF32Rows];  // this thread's scores of the tile
  const int h = blockIdx.y, b = blockIdx.z;
  const int row = blockIdx.x * kF32Rows + threadIdx.x;
  const bool live = row < n_q;
  float qr[DP], acc[DP];
#pragma unroll
  for (int f = 0; f < DP; ++f) {
    qr[f] = (live && f < d) ? q[(((size_t)b * n_q + row) * H + h) * d + f] : 0.f;
    acc[f] = 0.f;
  }
  float m = -INFINITY, l = 0.f;  // m* (log2 units of the scaled score), s*
  for (int j0 = 0; j0 < n_k; j0 += kF32Keys) {
    __syncthreads();
    for (int e = threadIdx.x; e < kF32Keys * DP; e += kF32Rows) {
      const int j = e / DP, f = e % DP;
      const bool ok = (j0 + j < n_k) && f < d;
      const size_t off = (((size_t)b * n_k + j0 + j) * H + h) * d + f;
      ks[j][f] = ok ? k[off] : 0.f;
      vs[j][f] = ok ? v[off] : 0.f;
    }
    __syncthreads();
    const int valid = min(kF32Keys, n_k - j0);
    float mx = -INFINITY;
#pragma unroll 1
    for (int j = 0; j < valid; ++j) {
      float dot = 0.f;
#pragma unroll
      for (int f = 0; f < DP; ++f) dot = fmaf(qr[f], ks[j][f], dot);
      const float sj = dot * scale_log2;
      ss[j][threadIdx.x] = sj;
      mx = fmaxf(mx, sj);
    }
    const float m_new = fmaxf(m, mx);
    const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
    l *= alpha;
#pragma unroll
    for (int f = 0; f < DP; ++f) acc[f] *= alpha;
#pragma unroll 1
    for (int j = 0; j < valid; ++j) {
      const float p = exp2f(ss[j][threadIdx.x] - m_new);
      l += p;
#pragma unroll
      for (int f = 0; f < DP; ++f) acc[f] = fmaf(p, vs[j][f], acc[f]);
    }
    m = m_new;
  }
  if (!live) return;
  const float inv = 1.f / l;
  for (int f = 0; f < d && f < DP; ++f) out[(((size_t)b * n_q + row) * H + h) * d + f] = acc[f] * inv;
  if (lse) lse[((size_t)b * H + h) * n_q + row] = (m + log2f(l)) * 0.6931471805599453f;
}

template <int DP>
cudaError_t launch_dp(const float* q, const float* k, const float* v, float* out, float* lse, int B, int H, int n_q,
                      int n_k, int d, float scale_log2, cudaStream_t s) {
  dim3 grid((n_q + kF32Rows - 1) / kF32Rows, H, B);
  fwd_f32_kernel<DP><<<grid, kF32Rows, 0, s>>>(q, k, v, out, lse, B, H, n_q, n_k, d, scale_log2);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fwd_f32(const float* q, const float* k, const float* v, float* out, float* lse, int B, int H,
                           int n_q, int n_k, int d, float scale, cudaStream_t s) {
  const float c = scale * 1.4426950408889634f;
  if (d <= 16) return launch_dp<16>(q, k, v, out, lse, B, H, n_q, n_k, d, c, s);
  if (d <= 32) return launch_dp<32>(q, k, v, out, lse, B, H, n_q, n_k, d, c, s);
  if (d <= 64) return launch_dp<64>(q, k, v, out, lse, B, H, n_q, n_k, d, c, s);
  return launch_dp<128>(q, k, v, out, lse, B, H, n_q, n_k, d, c, s);
}

}  // namespace mea
