// fwd_kp_sm100a.cu — d = 64 self-attention forward (bf16 in, fp32 accumulate) as FOUR independent
// key streams per CTA: two 128-row query tiles x {even, odd} 64-key tiles, each stream with its
// own running (m*, s*, v*) (Figure 1 lines 12-19 = PAPER.md:118-126), merged per
// query row at the end by Figure 1's global-max rescale of chunk summaries:
// the even and odd key tiles are the paper's key chunks, summarised on chip.
//
// Why streams: in fwd_db the two softmax warps of a query tile on an SM sub-partition are
// released by the same barrier and compete for the exponential unit at the same moments, then
// sit in their per-tile waits together. Here every sub-partition holds ONE softmax warp per
// stream (thread = query row, 64 keys per step, 32x32b TMEM shape, no shuffles), the four
// streams' barriers are independent, and one MMA issuer per stream runs its Q K^T -> P V chain.
//
//   TMEM (512 columns): S[s] = columns [64 s, 64 s + 64) (P_t written over its first 32),
//                       O[s] = [256 + 64 s, 320 + 64 s);  stream s = 2 * query tile + parity.
// Warps: 0 TMA producer (Q0, Q1 once; kStages-deep ring of 64-row K/V tiles, each tile read by
// the two streams of its parity), 1-4 MMA issuers (stream w - 1), 5 TMEM allocator, 6-7 idle,
// 8-23 softmax (stream (w - 8) / 4, TMEM lane quadrant w % 4).
//
// kStats = true is the backward's statistics pass B0: Q K^T and the row sums
// only (no V, P, P V or output), the two parities' (m*, s*) merged into lse.
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

constexpr int kN = 64;                                // keys per tile
#ifndef MEA_KP_STAGES
#define MEA_KP_STAGES 8
#endif
constexpr int kStages = MEA_KP_STAGES;
constexpr int kQTileBytes = kTileM * kHeadDim * 2;    // 16 KiB
constexpr int kKVTileBytes = kN * kHeadDim * 2;       // 8 KiB
constexpr int kThreads = 768;
constexpr int kSoftmaxRegs = 104;                     // per lane slot: 80 x 6 warps = 480
constexpr int kIssuerRegs = 40;
constexpr int kControlRegs = 24;
constexpr float kLazyThreshold = 8.0f;
constexpr float kSafeSum = 18446744073709551616.0f;   // 2^64
__host__ __device__ constexpr uint32_t col_s(int s) { return (uint32_t)(64 * s); }
__host__ __device__ constexpr uint32_t col_o(int s) { return (uint32_t)(256 + 64 * s); }

constexpr uint32_t kIdescQK = idesc_bf16_f32(128, kN, false, false);   // A = Q, B = K, both K-major
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 64, false, true);    // A = P (TMEM), B = V MN-major

#ifndef MEA_KP_POLY_MASK
#define MEA_KP_POLY_MASK 0x00010001u  // pairs 0 and 16 of the 32 pairs of a row on the FMA pipe
#endif
#ifndef MEA_KP_POLY_MASK_STATS
#define MEA_KP_POLY_MASK_STATS 0x49249249u
#endif
template <bool kStats>
__device__ __forceinline__ constexpr bool poly_pair(int i) {
  return (((kStats ? MEA_KP_POLY_MASK_STATS : MEA_KP_POLY_MASK)) >> i) & 1u;
}

struct KpSmem {
  uint8_t q[2][kQTileBytes];
  uint8_t k[kStages][kKVTileBytes];
  uint8_t v[kStages][kKVTileBytes];
  float2 ml[2][kTileM];   // [query tile][row]: the odd stream's (m*, s*) for the final merge
  uint64_t q_full;
  uint64_t kv_full[kStages];
  uint64_t kv_empty[kStages];
  uint64_t s_full[4];     // [stream]: Q K_t^T done
  uint64_t p_full[4];     // [stream]: P_t stored (stats: S_t read) by the stream's 128 threads
  uint64_t pv_done[4];
  uint64_t o_done[4];
  uint64_t odd_done[2];   // [query tile]: the odd stream's (m*, s*) in ml, its O final
  uint32_t tmem_base;
};
constexpr size_t kKpSmemBytes = sizeof(KpSmem) + 1024;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

template <bool kStats>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_kp_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  KpSmem& sm = *reinterpret_cast<KpSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: a 1-D grid ordered heaviest block (last rows) first across all (b, h)
  const int qblk = p.causal ? p.num_q_blocks - 1 - (int)(blockIdx.x / (p.H * p.B)) : (int)blockIdx.x;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int q0 = p.q_begin + qblk * kRowsPerCta;
  const int q_end = min(p.n_q, p.q_begin + p.q_count);
  // key padding: this batch element's keys [0, nk); at least one tile runs (all masked if nk = 0)
  const int nk = keys_of(p.kv_lens, b, p.n_k);
  // key tiles query tile qt needs (causal, n_q == n_k: keys below its last row + 1); the
  // producer streams the union (query tile 1's)
  auto tiles_for = [&](int qt) {
    return max(1, ((p.causal ? min(nk, q0 + (qt + 1) * kTileM) : nk) + kN - 1) / kN);
  };
  const int T = tiles_for(1);

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 2);  // the two streams of the tile's parity
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.p_full[s], 128);
      mbar_init(&sm.pv_done[s], 1);
      mbar_init(&sm.o_done[s], 1);
    }
    mbar_init(&sm.odd_done[0], 128);
    mbar_init(&sm.odd_done[1], 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mk);
    tma_prefetch_desc(&mv);
  }
  if (warp == 5) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 8) {
    // issuers 40 registers, the producer and the idle warps 24: 40 + 24 + 4 x 104 = 480
    if (warp == 0) {
      setmaxnreg_dec<kControlRegs>();
      // ---------------------------------------------------------- TMA producer
      const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.q_full, 2 * kQTileBytes);
        tma_load_4d(sm.q[0], &mq, &sm.q_full, 0, h, q0, b, stream);
        tma_load_4d(sm.q[1], &mq, &sm.q_full, 0, h, q0 + kTileM, b, stream);
      }
      __syncwarp();
      for (int t = 0; t < T; ++t) {
        const int st = t % kStages;
        if (t >= kStages) mbar_wait(&sm.kv_empty[st], ((t / kStages) - 1) & 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm.kv_full[st], (kStats ? 1 : 2) * kKVTileBytes);
          tma_load_4d(sm.k[st], &mk, &sm.kv_full[st], 0, h, t * kN, b, keep);
          if (!kStats) tma_load_4d(sm.v[st], &mv, &sm.kv_full[st], 0, h, t * kN, b, keep);
        }
        __syncwarp();
      }
    } else if (warp <= 4) {
      setmaxnreg_dec<kIssuerRegs>();
      // ---------------------------------------------------------- MMA issuer of stream s
      const int s = warp - 1, qt = s >> 1, par = s & 1;
      const int Tq = tiles_for(qt);
      const uint64_t dq = shfl0_u64(sdesc_sw128(smem_u32(sm.q[qt]), 16, 1024));
      const uint64_t dk0 = shfl0_u64(sdesc_sw128(smem_u32(sm.k[0]), 16, 1024));
      const uint64_t dv0 = shfl0_u64(sdesc_sw128(smem_u32(sm.v[0]), 16, 1024));
      constexpr uint64_t kStageStep = kKVTileBytes >> 4;
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t ts = tmem_u + col_s(s), to = tmem_u + col_o(s);
      auto qk = [&](int t) {  // S[s] = Q K_t^T
        const uint64_t dk = dk0 + (t % kStages) * kStageStep;
#pragma unroll
        for (int kk = 0; kk < kHeadDim / 16; ++kk) umma_ss(ts, dq + kk * 2, dk + kk * 2, kIdescQK, kk > 0);
        umma_commit(&sm.s_full[s]);
      };
      auto pv = [&](int t, bool first) {  // O[s] += P_t V_t, P_t over the first 32 columns of S[s]
        const uint64_t dv = dv0 + (t % kStages) * kStageStep;
#pragma unroll
        for (int kk = 0; kk < kN / 16; ++kk)
          umma_ts(to, ts + kk * 8, dv + kk * 128, kIdescPV, (!first || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&sm.q_full, 0);
      if (par < Tq) {
        mbar_wait(&sm.kv_full[par % kStages], (par / kStages) & 1);
        tc_fence_after();
        if (elect_one()) qk(par);
        __syncwarp();
      }
      int j = 0;
      for (int t = par; t < Tq; t += 2, ++j) {
        mbar_poll_wait<32>(&sm.p_full[s], j & 1);
        tc_fence_after();
        if (elect_one()) {
          if (!kStats) {
            pv(t, j == 0);
            umma_commit(&sm.pv_done[s]);
            if (t + 2 >= Tq) umma_commit(&sm.o_done[s]);
          }
          umma_commit(&sm.kv_empty[t % kStages]);
        }
        __syncwarp();
        if (t + 2 < Tq) {
          // S_{t+2} into the buffer P_t occupies: wait until P_t V_t has read it
          mbar_poll_wait<32>(&sm.kv_full[(t + 2) % kStages], ((t + 2) / kStages) & 1);
#ifndef MEA_KP_NO_PV_WAIT
          if (!kStats) mbar_poll_wait<32>(&sm.pv_done[s], j & 1);
#endif
          tc_fence_after();
          if (elect_one()) qk(t + 2);
          __syncwarp();
        }
      }
      // key tiles of this parity past this query tile's last row (causal): release unused
      for (int t = (Tq > par ? par + 2 * ((Tq - par + 1) / 2) : par); t < T; t += 2) {
        mbar_wait(&sm.kv_full[t % kStages], (t / kStages) & 1);
        if (elect_one()) umma_commit(&sm.kv_empty[t % kStages]);
        __syncwarp();
      }
    } else {
      setmaxnreg_dec<kControlRegs>();  // allocator / idle
    }
  } else {
    setmaxnreg_inc<kSoftmaxRegs>();
    // ------------------------------------------------------------ softmax warps (thread = row)
    const int s = (warp - 8) >> 2, qt = s >> 1, par = s & 1;
    const int quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const int r0 = q0 + qt * kTileM;  // first row of this query tile
    const int row = r0 + rloc;
    const int Tq = tiles_for(qt);
    const int key_lim = p.causal ? min(nk, row + 1) : nk;  // keys this row sees: [0, key_lim)
    // tiles [0, full) are complete for every row of the query tile (fast-path candidates)
    const int full = (p.causal ? min(nk, r0 + 1) : nk) / kN;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    float m_ref = -INFINITY;  // reference max m* (log2 units of the scaled score)
    float l = 0.f;            // s* of this stream
    int j = 0;
    // one half of S_t (32 keys) into registers
    auto load_half = [&](int half, uint32_t (&r)[32]) {
      tmem_ld32(lane_base + col_s(s) + half * 32, r);
      tmem_ld_wait();
    };
    for (int t = par; t < Tq; t += 2, ++j) {
      mbar_wait(&sm.s_full[s], j & 1);
      tc_fence_after();
      const int valid = key_lim - t * kN;  // keys of this tile the row sees (may be <= 0)
      uint32_t pk[32];
      // fast path: m* set, and every row of the query tile sees every key of this tile; S is
      // read half by half (32 registers), each half exponentiated as soon as it lands
      bool fast = (j > 0) && (t < full) && (c >= 0.f);
      if (fast) {
        const float2 c2 = make_float2(c, c), nm2 = make_float2(-m_ref, -m_ref);
        float2 rs = make_float2(0.f, 0.f);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t sr[32];
          load_half(half, sr);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 s2 = make_float2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1]));
            const float2 x = __ffma2_rn(s2, c2, nm2);  // s*c - m*
            const float2 e = poly_pair<kStats>(half * 16 + i) ? exp2_poly2(x)
                                                              : make_float2(ex2_approx(x.x), ex2_approx(x.y));
            rs = __fadd2_rn(rs, e);
            pk[half * 16 + i] = pack_bf16x2(e.x, e.y);
          }
        }
        // a finite row sum below 2^64 certifies every 2^(s c - m*) term (fwd_sm100a.cu)
        const float rsum = rs.x + rs.y;
        const bool need = !(rsum <= kSafeSum);
        if (__any_sync(0xffffffffu, need)) fast = false;
        else l += rsum;
      }
      if (!fast) {
        // exact max over the row's valid keys (two half loads), then the exponentials (two more)
        float ext = c >= 0.f ? -INFINITY : INFINITY;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t sr[32];
          load_half(half, sr);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (half * 32 + i < valid)
              ext = c >= 0.f ? fmaxf(ext, __uint_as_float(sr[i])) : fminf(ext, __uint_as_float(sr[i]));
        }
        const float m_cand = ext * c;
        const bool need = m_cand > m_ref + kLazyThreshold;  // always true on the stream's first tile
        float alpha = 1.f;
        if (need) {
          alpha = ex2_approx(m_ref - m_cand);  // 0 when m_ref = -inf
          m_ref = m_cand;
          l *= alpha;
        }
        if (!kStats && j > 0 && __any_sync(0xffffffffu, need)) {
          // v* <- v* alpha: P_{t-2} V_{t-2} has completed (its commit precedes Q K_t^T's, whose
          // s_full this thread has observed)
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            uint32_t o[32];
            tmem_ld32(lane_base + col_o(s) + part * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(lane_base + col_o(s) + part * 32, o);
          }
        }
        const float neg_m = -m_ref;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t sr[32];
          load_half(half, sr);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int k0 = half * 32 + 2 * i;
            const float p0 = (k0 < valid) ? ex2_approx(fmaf(__uint_as_float(sr[2 * i]), c, neg_m)) : 0.f;
            const float p1 = (k0 + 1 < valid) ? ex2_approx(fmaf(__uint_as_float(sr[2 * i + 1]), c, neg_m)) : 0.f;
            rs0 += p0;
            rs1 += p1;
            pk[half * 16 + i] = pack_bf16x2(p0, p1);
          }
        }
        l += rs0 + rs1;
      }
      tc_fence_before();
      if (!kStats) {  // P_t over the first 32 columns of S[s]
        tmem_st32(lane_base + col_s(s), pk);
        tmem_st_wait();
        tc_fence_before();
      }
      mbar_arrive(&sm.p_full[s]);  // stats: S_t has been read and may be refilled
    }
    // ------------------------------------------------------------ merge the two parities
    const bool odd_ran = Tq > 1;  // the odd stream had key tiles (the even one always does)
    if (par == 1) {
      if (!kStats && odd_ran) {
        mbar_wait(&sm.o_done[s], 0);
        tc_fence_after();
      }
      sm.ml[qt][rloc] = make_float2(m_ref, l);
      tc_fence_before();
      mbar_arrive(&sm.odd_done[qt]);
    } else {
      mbar_wait(&sm.odd_done[qt], 0);
      tc_fence_after();
      const float2 mo = sm.ml[qt][rloc];
      const float M = fmaxf(m_ref, mo.x);
      const float we = M == -INFINITY ? 0.f : ex2_approx(m_ref - M);
      const float wo = M == -INFINITY ? 0.f : ex2_approx(mo.x - M);
      const float L = l * we + mo.y * wo;  // s* of the row (Figure 1's global rescale)
      const size_t bh = (size_t)b * p.H + h;
      if (kStats) {
        if (row < q_end) p.lse[bh * p.n_q + row] = (M + __log2f(L)) * 0.6931471805599453f;
      } else {
        mbar_wait(&sm.o_done[s], 0);
        tc_fence_after();
        const float inv = L > 0.f ? 1.f / L : 0.f;  // a row with no keys (padding): out = 0, lse = -inf
        const float ce = we * inv, co = odd_ran ? wo * inv : 0.f;
        const size_t off = (((size_t)b * p.n_q + row) * p.H + h) * kHeadDim;
#pragma unroll
        for (int part = 0; part < 4; ++part) {  // 16 columns of O per part
          uint32_t oe[16], oo[16];
          tmem_ld16(lane_base + col_o(s) + part * 16, oe);
          if (odd_ran) tmem_ld16(lane_base + col_o(s + 1) + part * 16, oo);
          tmem_ld_wait();
          float r[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            r[i] = __uint_as_float(oe[i]) * ce + (odd_ran ? __uint_as_float(oo[i]) * co : 0.f);
          if (row < q_end) {
            if (p.out_f32) {
              float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off + part * 16);
#pragma unroll
              for (int i = 0; i < 4; ++i) dst[i] = make_float4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off + part * 16);
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                uint4 w;
                w.x = pack_bf16x2(r[8 * i + 0], r[8 * i + 1]);
                w.y = pack_bf16x2(r[8 * i + 2], r[8 * i + 3]);
                w.z = pack_bf16x2(r[8 * i + 4], r[8 * i + 5]);
                w.w = pack_bf16x2(r[8 * i + 6], r[8 * i + 7]);
                dst[i] = w;
              }
            }
          }
        }
        if (row < q_end && p.lse) p.lse[bh * p.n_q + row] = (M + __log2f(L)) * 0.6931471805599453f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int fwd_kp_key_tile() { return kN; }

cudaError_t launch_fwd_kp_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                               const CUtensorMap& mv, cudaStream_t s) {
  const dim3 grid = p.causal ? dim3(p.num_q_blocks * p.H * p.B) : dim3(p.num_q_blocks, p.H, p.B);
  if (p.stats_only) {
    const cudaError_t attr = ensure_smem_attr<fwd_kp_kernel<true>>((int)kKpSmemBytes);
    if (attr != cudaSuccess) return attr;
    fwd_kp_kernel<true><<<grid, kThreads, kKpSmemBytes, s>>>(mq, mk, mv, p);
  } else {
    const cudaError_t attr = ensure_smem_attr<fwd_kp_kernel<false>>((int)kKpSmemBytes);
    if (attr != cudaSuccess) return attr;
    fwd_kp_kernel<false><<<grid, kThreads, kKpSmemBytes, s>>>(mq, mk, mv, p);
  }
  return cudaGetLastError();
}

}  // namespace mea
