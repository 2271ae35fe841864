// fwd_f32tc_sm100a.cu — float32 self-attention forward on the bf16 tensor cores by split precision
// ("fp32 at tensor-core speed"). fp32 inputs are split into bf16 parts:
// q, k, v and P into three, x = h + m + l (h = bf16(x), m = bf16(x - h), l = bf16(x - h - m): 24
// significant bits, the fp32 precision), and each product keeps the terms down to 2^-16 of the
// leading one (the dropped ones are ~2^-24):
//   S = Qm Km^T + Ql Kh^T + Qh Kl^T + Qm Kh^T + Qh Km^T + Qh Kh^T   (relative error ~2^-24)
//   O += Pm Vm + Pl Vh + Ph Vl + Pm Vh + Ph Vm + Ph Vh              (relative error ~2^-24)
// S must be fp32-exact because the log-sum-exp residual (and every weight) depends on it to the
// absolute 1e-5 of the fp32 bar; with three-part P and v the output meets the same bar at any
// scale (round 1 kept two parts of P and v: 3 * 2^-18 * max|v|, which broke 1e-5 when a large
// scale made the weights peaked). Selected by in_dtype MEA_F32_SPLIT; MEA_F32 stays exact SIMT
// FFMA (fwd_f32.cu).
// Accumulation is fp32 in TMEM, the row statistics are fp32 in registers. The method is the paper's stream as in
// fwd_sm100a.cu; every tile takes the exact row maximum (no overflow certificate shortcut), with
// the lazy rescale of P:86. The relative error of a product is ~2^-16 in the worst case and
// averages out over the sums; the parity bar is the fp32 one (1e-5 absolute, BASELINE.json).
//
// Layout as fwd128_sm100a.cu: one 128-row query tile per CTA, S double-buffered in TMEM.
// TMEM (512): S0 [0,128) S1 [128,256) O [256,320) Ph [320,384) Pm [384,448) Pl [448,512).
// Shared memory (192 KB): Qh, Qm, Ql resident; a 2-stage ring of (Kh, Km, Kl) and ONE stage of
// (Vh, Vm, Vl): V_{t+1} loads while QK_{t+2} runs (the issue order is PV_t, QK_{t+2}, PV_{t+1}).
// Warps: 0 K producer (and Q once), 1 MMA issuer, 2 TMEM allocator, 3 V producer, 4-11 softmax
// (thread = one row half).
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

constexpr int kStagesTc = 2;
constexpr int kTileB = 128 * 64 * 2;  // 16 KiB bf16 tile (one SW128 atom)
constexpr int kThreadsTc = 384;
constexpr uint32_t kColO = 256, kColPh = 320, kColPm = 384, kColPl = 448;
constexpr float kLazyTc = 8.0f;
constexpr uint32_t kIdQK = idesc_bf16_f32(128, 128, false, false);
constexpr uint32_t kIdPV = idesc_bf16_f32(128, 64, false, true);

struct TcSmem {
  uint8_t qh[kTileB], qm[kTileB], ql[kTileB];
  uint8_t kh[kStagesTc][kTileB], km[kStagesTc][kTileB], kl[kStagesTc][kTileB];
  uint8_t vh[kTileB], vm[kTileB], vl[kTileB];
  uint64_t q_full, kv_full[kStagesTc], kv_empty[kStagesTc], v_full, v_empty;
  uint64_t s_full[2], s_loaded[2], p_full, pv_done, o_done;
  uint32_t tmem_base;
};
constexpr size_t kTcSmemBytes = sizeof(TcSmem) + 1024;

__device__ __forceinline__ uint8_t* align1024_tc(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

struct SplitMaps {
  CUtensorMap qh, qm, ql, kh, km, kl, vh, vm, vl;
};

__global__ void __launch_bounds__(kThreadsTc, 1)
    fwd_f32tc_kernel(const __grid_constant__ SplitMaps m, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>(align1024_tc(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * 128;
  const int T = (p.n_k + kTileN - 1) / kTileN;

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStagesTc; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    mbar_init(&sm.v_full, 1);
    mbar_init(&sm.v_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_loaded[i], 256);
    }
    mbar_init(&sm.p_full, 256);
    mbar_init(&sm.pv_done, 1);
    mbar_init(&sm.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
    if (elect_one()) {
      mbar_arrive_expect_tx(&sm.q_full, 3 * kTileB);
      tma_load_4d(sm.qh, &m.qh, &sm.q_full, 0, h, q0, b, stream);
      tma_load_4d(sm.qm, &m.qm, &sm.q_full, 0, h, q0, b, stream);
      tma_load_4d(sm.ql, &m.ql, &sm.q_full, 0, h, q0, b, stream);
    }
    __syncwarp();
    for (int t = 0; t < T; ++t) {
      const int st = t % kStagesTc, n = t / kStagesTc;
      if (t >= kStagesTc) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
      const int krow = t * kTileN;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.kv_full[st], 3 * kTileB);
        tma_load_4d(sm.kh[st], &m.kh, &sm.kv_full[st], 0, h, krow, b, keep);
        tma_load_4d(sm.km[st], &m.km, &sm.kv_full[st], 0, h, krow, b, keep);
        tma_load_4d(sm.kl[st], &m.kl, &sm.kv_full[st], 0, h, krow, b, keep);
      }
      __syncwarp();
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- V producer (one stage)
    const uint64_t keep = policy_evict_last();
    for (int t = 0; t < T; ++t) {
      if (t > 0) mbar_wait(&sm.v_empty, (t - 1) & 1);  // PV_{t-1} has read the stage
      const int krow = t * kTileN;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.v_full, 3 * kTileB);
        tma_load_4d(sm.vh, &m.vh, &sm.v_full, 0, h, krow, b, keep);
        tma_load_4d(sm.vm, &m.vm, &sm.v_full, 0, h, krow, b, keep);
        tma_load_4d(sm.vl, &m.vl, &sm.v_full, 0, h, krow, b, keep);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint64_t dqh = shfl0_u64(sdesc_sw128(smem_u32(sm.qh), 16, 1024));
    const uint64_t dqm = shfl0_u64(sdesc_sw128(smem_u32(sm.qm), 16, 1024));
    const uint64_t dql = shfl0_u64(sdesc_sw128(smem_u32(sm.ql), 16, 1024));
    const uint64_t dkh = shfl0_u64(sdesc_sw128(smem_u32(sm.kh[0]), 16, 1024));
    const uint64_t dkm = shfl0_u64(sdesc_sw128(smem_u32(sm.km[0]), 16, 1024));
    const uint64_t dkl = shfl0_u64(sdesc_sw128(smem_u32(sm.kl[0]), 16, 1024));
    const uint64_t dvh = shfl0_u64(sdesc_sw128(smem_u32(sm.vh), 16, 1024));
    const uint64_t dvm = shfl0_u64(sdesc_sw128(smem_u32(sm.vm), 16, 1024));
    const uint64_t dvl = shfl0_u64(sdesc_sw128(smem_u32(sm.vl), 16, 1024));
    constexpr uint64_t kStep = kTileB >> 4;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    auto qk = [&](int st, int buf) {  // S = mm + lh + hl + mh + hm + hh (smallest terms first)
      const uint32_t d = tm + buf * 128;
      const uint64_t kh = dkh + st * kStep, km = dkm + st * kStep, kl = dkl + st * kStep;
      const uint64_t qa[6] = {dqm, dql, dqh, dqm, dqh, dqh}, ka[6] = {km, kh, kl, kh, km, kh};
#pragma unroll
      for (int t6 = 0; t6 < 6; ++t6)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_ss(d, qa[t6] + kk * 2, ka[t6] + kk * 2, kIdQK, (t6 > 0 || kk > 0));
    };
    auto pv = [&]() {  // O_t = Pm Vm + Pl Vh + Ph Vl + Pm Vh + Ph Vm + Ph Vh (smallest first), fresh per tile
      const uint32_t pa[6] = {kColPm, kColPl, kColPh, kColPm, kColPh, kColPh};
      const uint64_t vb[6] = {dvm, dvh, dvl, dvh, dvm, dvh};
#pragma unroll
      for (int t6 = 0; t6 < 6; ++t6)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tm + kColO, tm + pa[t6] + kk * 8, vb[t6] + kk * 128, kIdPV, (t6 > 0 || kk > 0));
    };
    mbar_wait(&sm.q_full, 0);
    for (int t = 0; t < 2 && t < T; ++t) {
      mbar_wait(&sm.kv_full[t], 0);
      tc_fence_after();
      if (elect_one()) {
        qk(t, t);
        umma_commit(&sm.s_full[t]);
        umma_commit(&sm.kv_empty[t]);   // the K stage is free once QK_t is done
      }
      __syncwarp();
    }
    for (int t = 0; t < T; ++t) {
      const int st = t % kStagesTc;
      mbar_wait(&sm.p_full, t & 1);
      mbar_wait(&sm.v_full, t & 1);
      tc_fence_after();
      if (elect_one()) {
        pv();
        umma_commit(&sm.pv_done);
        umma_commit(&sm.v_empty);
        if (t + 1 == T) umma_commit(&sm.o_done);
      }
      __syncwarp();
      if (t + 2 < T) {
        const int s2 = (t + 2) % kStagesTc;
        mbar_wait(&sm.kv_full[s2], ((t + 2) / kStagesTc) & 1);
        mbar_wait(&sm.s_loaded[t & 1], (t >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          qk(s2, t & 1);
          umma_commit(&sm.s_full[t & 1]);
          umma_commit(&sm.kv_empty[s2]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax (8 warps)
    const int sw = warp - 4;
    const int sub = sw >> 2;
    const int quarter = warp & 3;
    const int half = lane >> 4;
    const int rloc = quarter * 32 + sub * 16 + (lane & 15);
    const int row = q0 + rloc;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32 + sub * 16) << 16);
    const float c = p.scale_log2;
    float m_ref = -INFINITY;
    float l = 0.f;
    // v* in registers (this thread's 32 output columns): the tensor cores sum one key tile into a
    // fresh TMEM tile (48 MMA steps, fp32) and the tiles are added here in fp32 round-to-nearest
    // (accumulating every tile in TMEM measured up to 1.5e-5 absolute error at scale 0.5)
    float vacc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) vacc[i] = 0.f;
    for (int t = 0; t < T; ++t) {
      const int buf = t & 1;
      const uint32_t colS = buf * 128;
      mbar_wait(&sm.s_full[buf], (t >> 1) & 1);
      tc_fence_after();
      uint32_t sr[64];
      tmem_ld32_split<64>(lane_base + colS + 0, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tmem_ld32_split<64>(lane_base + colS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&sm.s_loaded[buf]);
      const int valid = p.n_k - t * kTileN - half * 64;  // keys of my half in range (may be <= 0)
      // exact row extremum (max for c >= 0, min for c < 0) over both halves
      float e0 = c >= 0.f ? -INFINITY : INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (i < valid) e0 = c >= 0.f ? fmaxf(e0, __uint_as_float(sr[i])) : fminf(e0, __uint_as_float(sr[i]));
      const float eo = __shfl_xor_sync(0xffffffffu, e0, 16);
      e0 = c >= 0.f ? fmaxf(e0, eo) : fminf(e0, eo);
      const float m_cand = e0 * c;
      const bool need = m_cand > m_ref + kLazyTc;  // always on the first tile
      float alpha = 1.f;
      if (need) {
        alpha = ex2_approx(m_ref - m_cand);
        m_ref = m_cand;
        l *= alpha;
      }
      // P = 2^(s c - m*) in f32 (in place of the scores), then three bf16 parts h, m, l
      const float neg_m = -m_ref;
      float rs = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float pi = (i < valid) ? ex2_approx(fmaf(__uint_as_float(sr[i]), c, neg_m)) : 0.f;
        rs += pi;
        sr[i] = __float_as_uint(pi);
      }
      l += rs;
      if (t > 0) mbar_wait(&sm.pv_done, (t - 1) & 1);  // PV_{t-1} has consumed Ph, Pm, Pl
      tc_fence_after();
#pragma unroll
      for (int part = 0; part < 3; ++part) {
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {   // pairs [16 q2, 16 q2 + 16): columns +16 q2 of each half
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int e = 2 * (16 * q2 + i);
            const float p0 = __uint_as_float(sr[e]), p1 = __uint_as_float(sr[e + 1]);
            const __nv_bfloat16 h0 = __float2bfloat16_rn(p0), h1 = __float2bfloat16_rn(p1);
            pk[i] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
            sr[e] = __float_as_uint(p0 - __bfloat162float(h0));       // exact residual
            sr[e + 1] = __float_as_uint(p1 - __bfloat162float(h1));
          }
          tmem_st16_split<32>(lane_base + (part == 0 ? kColPh : part == 1 ? kColPm : kColPl) + 16 * q2, pk);
          tmem_st_wait();   // pk is reused
        }
      }
      if (t > 0) {
        // fold PV_{t-1}'s tile sum (complete: pv_done above) into v* with an fp32 round-to-nearest
        // add, then apply this tile's rescale to the whole v*; PV_t overwrites the tile after p_full
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          uint32_t o[16];
          tmem_ld16_split<32>(lane_base + kColO + part * 16, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) vacc[part * 16 + i] = (vacc[part * 16 + i] + __uint_as_float(o[i])) * alpha;
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.p_full);
    }
    // ---------------------------------------------------------------- epilogue: out = v*/s*
    const float lrow = l + __shfl_xor_sync(0xffffffffu, l, 16);
    mbar_wait(&sm.o_done, 0);
    tc_fence_after();
    uint32_t o[32];
    tmem_ld32_split<32>(lane_base + kColO, o);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(vacc[i] + __uint_as_float(o[i]));
    if (row < p.n_q) {
      const float inv = 1.f / lrow;
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) +
                                              (((size_t)b * p.n_q + row) * p.H + h) * kHeadDim + half * 32);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        dst[i] = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                             __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
      if (p.lse && half == 0) p.lse[((size_t)b * p.H + h) * p.n_q + row] = (m_ref + __log2f(lrow)) * 0.6931471805599453f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// x (f32) -> parts[0] = bf16(x), parts[1] = bf16(x - parts[0]), parts[2] = bf16(x - parts[0] - parts[1])
// (the first `nparts`), 4 elements per thread
__global__ void split_f32_kernel(const float4* __restrict__ x, uint2* __restrict__ p0, uint2* __restrict__ p1,
                                 uint2* __restrict__ p2, int nparts, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float r[4];
    const float4 v = x[i];
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
    uint2* outs[3] = {p0, p1, p2};
    for (int part = 0; part < nparts; ++part) {
      uint32_t w[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const __nv_bfloat16 a = __float2bfloat16_rn(r[2 * j]), c = __float2bfloat16_rn(r[2 * j + 1]);
        w[j] = (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(c) << 16);
        r[2 * j] -= __bfloat162float(a);
        r[2 * j + 1] -= __bfloat162float(c);
      }
      outs[part][i] = make_uint2(w[0], w[1]);
    }
  }
}

}  // namespace

cudaError_t launch_split_f32(const float* x, void* const* parts, int nparts, int64_t n, cudaStream_t s) {
  const int64_t n4 = n / 4;
  const int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 16);
  split_f32_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(x), static_cast<uint2*>(parts[0]),
                                           static_cast<uint2*>(parts[1]),
                                           static_cast<uint2*>(nparts > 2 ? parts[2] : nullptr), nparts, n4);
  return cudaGetLastError();
}

cudaError_t launch_fwd_f32tc(const FwdParams& p, const CUtensorMap (&maps)[9], cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr<fwd_f32tc_kernel>((int)kTcSmemBytes);
  if (attr != cudaSuccess) return attr;
  SplitMaps m{maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], maps[7], maps[8]};
  dim3 grid((p.n_q + 127) / 128, p.H, p.B);
  fwd_f32tc_kernel<<<grid, kThreadsTc, kTcSmemBytes, s>>>(m, p);
  return cudaGetLastError();
}

}  // namespace mea
