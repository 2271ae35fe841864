// fwd128_sm100a.cu — self-attention forward for head dimension d = 128 ("d=64
// first; d=128 NEXT"), bf16 in, fp32 accumulate. Same method as fwd_sm100a.cu (the paper's
// per-query stream, evaluated one 128-key tile at a time with a lazily
// rescaled reference max), re-laid out for d = 128:
//   * the O accumulator of a 128-row query tile is 128 TMEM columns, so a CTA holds ONE query
//     tile and spends the freed columns on a second S buffer: S_{t+1} and S_{t+2} are computed
//     into alternating buffers while the softmax works on S_t;
//   * Q, K and V tiles are two 128B-swizzle atoms wide (d 0-63, 64-127): QK^T takes 8 K steps
//     (4 per atom), PV is one N = 128 MMA per 16 keys with B = V MN-major across both atoms
//     (LBO = 16 KiB between them).
// Per key tile: tensor work 2 x 128·128·128 MACs (1024 cycles at the dense rate) against 16384
// exponentials (1024 cycles of MUFU at 16/clk/SM): the ratio is twice d = 64's, so the tensor
// pipe and the exponential unit are balanced here.
//
// Warps: 0 TMA producer (Q once, 3-stage K/V ring), 1 MMA issuer, 2 TMEM allocator, 3 idle,
// 4-11 softmax (thread = one row-half, 16x32bx2 TMEM shape as in fwd_sm100a.cu).
// TMEM (512): S0 [0,128) S1 [128,256) O [256,384) P [384,448).
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

// MMA-issuer waits: up to 32 unrolled polls, then suspend (-2.5 % against suspending at once;
// the fused backward (+1 to +6 %) and the key-split forward (+0.6 %) keep plain try_wait)
#ifdef MEA_ISSUER_SUSPEND
#define IWAIT mbar_wait
#else
#define IWAIT mbar_poll_wait<32>
#endif

constexpr int kD = 128;
constexpr int kStages128 = 3;
constexpr int kAtomBytes = 128 * 128;           // 128 rows x 64 bf16 (one SW128 atom column)
constexpr int kTile128Bytes = 2 * kAtomBytes;   // 128 rows x 128 bf16
constexpr int kThreads128 = 384;
constexpr uint32_t kColS0 = 0, kColO = 256, kColP = 384;
constexpr float kLazy = 8.0f;
constexpr float kSafe = 18446744073709551616.0f;  // 2^64, see fwd_sm100a.cu
constexpr uint32_t kIdQK = idesc_bf16_f32(128, 128, false, false);  // A=Q K-major, B=K K-major
constexpr uint32_t kIdPV = idesc_bf16_f32(128, 128, false, true);   // A=P (TMEM), B=V MN-major

struct Fwd128Smem {
  uint8_t q[kTile128Bytes];
  uint8_t k[kStages128][kTile128Bytes];
  uint8_t v[kStages128][kTile128Bytes];
  uint64_t q_full, kv_full[kStages128], kv_empty[kStages128];
  uint64_t s_full[2], s_loaded[2], p_full, pv_done, o_done;
  uint32_t tmem_base;
};
constexpr size_t kFwd128SmemBytes = sizeof(Fwd128Smem) + 1024;

__device__ __forceinline__ uint8_t* align1024_128(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

__global__ void __launch_bounds__(kThreads128, 1)
    fwd128_bf16_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                       const __grid_constant__ CUtensorMap mv, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  Fwd128Smem& sm = *reinterpret_cast<Fwd128Smem*>(align1024_128(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;  // causal: 1-D grid, heaviest first
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  // causal (n_q == n_k): query tile qb needs key tiles [0, qb] (the last one is its diagonal);
  // the blocks with the most key tiles are scheduled first
  // key split (the paper's key chunks): blockIdx.x = split * num_q_blocks + query block; the
  // query blocks cover this launch's window [q_begin, q_begin + q_count)
  const int qb = p.causal ? p.num_q_blocks - 1 - (int)(blockIdx.x / (p.H * p.B)) : (int)(blockIdx.x % p.num_q_blocks);
  const int split = p.causal ? 0 : blockIdx.x / p.num_q_blocks;
  const int q0 = p.q_begin + qb * 128;
  const int q_end = min(p.n_q, p.q_begin + p.q_count);
  // key padding (kv_lens, online schedule only): keys [0, nk), at least one tile (all masked if nk = 0)
  const int nk = keys_of(p.kv_lens, b, p.n_k);
  const int n_tiles = p.kv_lens ? max(1, (nk + kTileN - 1) / kTileN) : (p.n_k + kTileN - 1) / kTileN;
  const int t_begin = (p.split_base + split) * p.tiles_per_split;  // split_base: tree schedule, one chunk per launch
  const int t_end = p.causal ? min(n_tiles, qb + 1) : min(n_tiles, t_begin + p.tiles_per_split);
  const int T = t_end - t_begin;
  const int diag = p.causal ? qb : -1;
  const int key_end = min(nk, t_end * kTileN);

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages128; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_loaded[i], 256);
    }
    mbar_init(&sm.p_full, 256);
    mbar_init(&sm.pv_done, 1);
    mbar_init(&sm.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mk);
    tma_prefetch_desc(&mv);
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
      mbar_arrive_expect_tx(&sm.q_full, kTile128Bytes);
      tma_load_4d(sm.q, &mq, &sm.q_full, 0, h, q0, b, stream);
      tma_load_4d(sm.q + kAtomBytes, &mq, &sm.q_full, 64, h, q0, b, stream);
    }
    __syncwarp();
    for (int t = 0; t < T; ++t) {
      const int st = t % kStages128, n = t / kStages128;
      if (t >= kStages128) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
      const int krow = (t_begin + t) * kTileN;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.kv_full[st], 2 * kTile128Bytes);
        tma_load_4d(sm.k[st], &mk, &sm.kv_full[st], 0, h, krow, b, keep);
        tma_load_4d(sm.k[st] + kAtomBytes, &mk, &sm.kv_full[st], 64, h, krow, b, keep);
        tma_load_4d(sm.v[st], &mv, &sm.kv_full[st], 0, h, krow, b, keep);
        tma_load_4d(sm.v[st] + kAtomBytes, &mv, &sm.kv_full[st], 64, h, krow, b, keep);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint64_t dq = shfl0_u64(sdesc_sw128(smem_u32(sm.q), 16, 1024));
    const uint64_t dk0 = shfl0_u64(sdesc_sw128(smem_u32(sm.k[0]), 16, 1024));
    // V as the MN-major B operand of PV: N = d over two 64-column atoms 16 KiB apart (LBO)
    const uint64_t dv0 = shfl0_u64(sdesc_sw128(smem_u32(sm.v[0]), kAtomBytes, 1024));
    constexpr uint64_t kStageStep = kTile128Bytes >> 4, kAtomStep = kAtomBytes >> 4;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    auto qk = [&](int st, int buf) {  // S[buf] = Q K^T, K = 128 in 8 steps (4 per atom)
      const uint64_t dk = dk0 + st * kStageStep;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t off = (kk >> 2) * kAtomStep + (kk & 3) * 2;
        umma_ss(tm + kColS0 + buf * 128, dq + off, dk + off, kIdQK, kk > 0);
      }
    };
    auto pv = [&](int st, bool acc) {  // O (+)= P V, K = 128 keys in steps of 16
      const uint64_t dv = dv0 + st * kStageStep;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) umma_ts(tm + kColO, tm + kColP + kk * 8, dv + kk * 128, kIdPV, (acc || kk > 0));
    };
    mbar_wait(&sm.q_full, 0);
    for (int t = 0; t < 2 && t < T; ++t) {
      mbar_wait(&sm.kv_full[t], 0);
      tc_fence_after();
      if (elect_one()) {
        qk(t, t);
        umma_commit(&sm.s_full[t]);
      }
      __syncwarp();
    }
    for (int t = 0; t < T; ++t) {
      const int st = t % kStages128;
      IWAIT(&sm.p_full, t & 1);
      tc_fence_after();
      if (elect_one()) {
        pv(st, t > 0);
        umma_commit(&sm.pv_done);
        umma_commit(&sm.kv_empty[st]);
        if (t + 1 == T) umma_commit(&sm.o_done);
      }
      __syncwarp();
      if (t + 2 < T) {  // S_{t+2} into the buffer S_t occupied (read at s_loaded, before p_full)
        const int s2 = (t + 2) % kStages128;
        IWAIT(&sm.kv_full[s2], ((t + 2) / kStages128) & 1);
        IWAIT(&sm.s_loaded[t & 1], (t >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          qk(s2, t & 1);
          umma_commit(&sm.s_full[t & 1]);
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
    for (int t = 0; t < T; ++t) {
      const int buf = t & 1;
      const uint32_t colS = kColS0 + buf * 128;
      mbar_wait(&sm.s_full[buf], (t >> 1) & 1);
      tc_fence_after();
      uint32_t sr[64];
      const int tile_valid = (p.causal ? min(key_end, row + 1) : key_end) - (t_begin + t) * kTileN;  // keys <= row if causal
      const int valid = tile_valid - half * 64;
      uint32_t pk[32];
      bool fast = (t > 0) && (t != diag) && (key_end - (t_begin + t) * kTileN >= kTileN) && (c >= 0.f);
      tmem_ld32_split<64>(lane_base + colS + 0, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      if (fast) {
        tmem_ld_wait();
        tmem_ld32_split<64>(lane_base + colS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        const float2 c2 = make_float2(c, c), nm2 = make_float2(-m_ref, -m_ref);
        float2 rs = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i == 16) {
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sm.s_loaded[buf]);
          }
          const float2 s2 = make_float2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1]));
          const float2 x = __ffma2_rn(s2, c2, nm2);
          const float2 e = (i == 9 || i == 25) ? exp2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
          rs = __fadd2_rn(rs, e);
          pk[i] = pack_bf16x2(e.x, e.y);
        }
        const float rsum = rs.x + rs.y;
        const bool need = !(rsum <= kSafe);
        if (__any_sync(0xffffffffu, need)) {
          fast = false;
        } else {
          l += rsum;
        }
      } else {
        tmem_ld32_split<64>(lane_base + colS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&sm.s_loaded[buf]);
      }
      if (!fast) {
        // exact row extremum of the raw scores (max for c >= 0, min for c < 0), both halves
        float e0;
        if (c >= 0.f) {
          e0 = -INFINITY;
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i < valid) e0 = fmaxf(e0, __uint_as_float(sr[i]));
          e0 = fmaxf(e0, __shfl_xor_sync(0xffffffffu, e0, 16));
        } else {
          e0 = INFINITY;
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i < valid) e0 = fminf(e0, __uint_as_float(sr[i]));
          e0 = fminf(e0, __shfl_xor_sync(0xffffffffu, e0, 16));
        }
        const float m_cand = e0 * c;
        const bool need = m_cand > m_ref + kLazy;
        float alpha = 1.f;
        if (need) {
          alpha = ex2_approx(m_ref - m_cand);
          m_ref = m_cand;
          l *= alpha;
        }
        if (t > 0 && __any_sync(0xffffffffu, need)) {
          // v* <- v* alpha once PV_{t-1} is done: lanes 0-15 O columns [0,64), 16-31 [64,128)
          mbar_wait(&sm.pv_done, (t - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int part = 0; part < 4; ++part) {
            uint32_t o[16];
            tmem_ld16_split<64>(lane_base + kColO + part * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16_split<64>(lane_base + kColO + part * 16, o);
          }
        }
        const float neg_m = -m_ref;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float p0 = (2 * i < valid) ? ex2_approx(fmaf(__uint_as_float(sr[2 * i]), c, neg_m)) : 0.f;
          const float p1 = (2 * i + 1 < valid) ? ex2_approx(fmaf(__uint_as_float(sr[2 * i + 1]), c, neg_m)) : 0.f;
          rs0 += p0;
          rs1 += p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        l += rs0 + rs1;
      }
      if (t > 0) mbar_wait(&sm.pv_done, (t - 1) & 1);  // PV_{t-1} has consumed P_{t-1}
      tc_fence_after();
      tmem_st32_split<32>(lane_base + kColP, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
    }
    // ---------------------------------------------------------------- epilogue: out = v*/s*
    const float lrow = l + __shfl_xor_sync(0xffffffffu, l, 16);
    mbar_wait(&sm.o_done, 0);
    tc_fence_after();
    uint32_t o[64];
    tmem_ld32_split<64>(lane_base + kColO, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
    tmem_ld32_split<64>(lane_base + kColO + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
    tmem_ld_wait();
    if (row < q_end && p.tri_v) {
      // this call's (m*, s*, v*) per row, for a merge across key ranges
      const size_t idx = ((size_t)b * p.n_q + row) * p.H + h;
      float4* dst = reinterpret_cast<float4*>(p.tri_v + idx * p.tri_vs + half * 64);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        dst[i] = make_float4(__uint_as_float(o[4 * i]), __uint_as_float(o[4 * i + 1]), __uint_as_float(o[4 * i + 2]),
                             __uint_as_float(o[4 * i + 3]));
      if (half == 0) {
        p.tri_m[idx * p.tri_ms] = m_ref * 0.6931471805599453f;
        p.tri_s[idx * p.tri_ms] = lrow;
      }
    } else if (row < q_end && p.part_o) {  // key-split / tree summaries
      const size_t prow = ((size_t)split * p.B * p.H + (size_t)b * p.H + h) * p.q_count + (row - p.q_begin);
      float4* dst = reinterpret_cast<float4*>(p.part_o + prow * kD + half * 64);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        dst[i] = make_float4(__uint_as_float(o[4 * i]), __uint_as_float(o[4 * i + 1]), __uint_as_float(o[4 * i + 2]),
                             __uint_as_float(o[4 * i + 3]));
      if (half == 0) reinterpret_cast<float2*>(p.part_ml)[prow] = make_float2(m_ref, lrow);
    } else if (row < q_end) {
      const size_t bh = (size_t)b * p.H + h;
      const float inv = lrow > 0.f ? 1.f / lrow : 0.f;  // a row with no keys (padding): out = 0, lse = -inf
      const size_t off = (((size_t)b * p.n_q + row) * p.H + h) * kD + half * 64;
      if (p.out_f32) {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          dst[i] = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                               __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
      } else {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv);
          dst[i] = w;
        }
      }
      if (p.lse && half == 0) p.lse[bh * p.n_q + row] = (m_ref + __log2f(lrow)) * 0.6931471805599453f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

cudaError_t launch_fwd128_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                               const CUtensorMap& mv, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr<fwd128_bf16_kernel>((int)kFwd128SmemBytes);
  if (attr != cudaSuccess) return attr;
  const dim3 grid = p.causal ? dim3(p.num_q_blocks * p.H * p.B) : dim3(p.num_q_blocks * p.num_splits, p.H, p.B);
  fwd128_bf16_kernel<<<grid, kThreads128, kFwd128SmemBytes, s>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace mea
