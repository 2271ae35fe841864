// fwd_db_sm100a.cu — d = 64 self-attention forward with double-buffered scores (bf16 in, fp32
// accumulate): the d = 64 forward online over all keys, with or without the causal mask (the
// key-split schedule and the triple output run fwd_sm100a.cu).
//
// Same method as fwd_sm100a.cu (the paper's per-query stream, key chunk by
// key chunk, Figure 1 lines 12-19 = PAPER.md:118-126; lazy rescale "as needed"), same
// CTA shape (two 128-row query tiles of one (b, h), 16 softmax warps of 16 rows each; here a
// quad of threads shares two rows, see the softmax section), but the key tile is 96 wide so that
// each query tile gets TWO score buffers:
//
//   TMEM (512 columns): S[qt][0] S[qt][1] = 4 x 96 columns at 0, 96, 192, 288;
//                       O0 [384,448), O1 [448,512).
//   P_t (bf16 pairs, 48 columns) is written over the first half of the buffer S_t came from.
//
// With one buffer (fwd_sm100a.cu) S_{t+1} could only be computed after the softmax had read
// S_t, and it queued behind the PV products of both tiles on the tensor pipe: the softmax
// waited for scores ~150 cycles and for PV_{t-1} ~300 cycles per tile, and the two query tiles
// drifted into phase, leaving the exponential unit (the binding unit at d = 64: 2 exps per
// 128 MMA flops) idle ~22 % of the time. Here QK_{t+2} is issued as soon as PV_t has consumed
// P_t, a whole softmax step ahead, so the scores of the next tile are always waiting; the
// softmax prefetches them (tcgen05.ld) before storing P_t, hiding the TMEM latency, and never
// waits on PV except before a (rare) O rescale.
//
// Warp roles: 0 TMA producer (Q0, Q1 once; kStages-deep K/V ring of 96-row tiles), 1 / 3 MMA
// issuers for query tile 0 / 1, 2 TMEM allocator, 4-19 softmax (as fwd_sm100a.cu).
//
// kStats = true is the backward's statistics pass B0 (the forward's
// statistics recomputed when they were not saved): the same row max / row sum of exponentials
// over Q K^T, but no V stream, no P store, no P V product and no output: only lse is written.
// Without P V the issuer refills a score buffer as soon as the softmax has read it.
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

constexpr int kN = 96;                                // keys per tile
#ifndef MEA_DB_STAGES
#define MEA_DB_STAGES 6
#endif
constexpr int kStages = MEA_DB_STAGES;                // K/V ring depth
constexpr int kQTileBytes = kTileM * kHeadDim * 2;    // 16 KiB
constexpr int kKVTileBytes = kN * kHeadDim * 2;       // 12 KiB (a multiple of the 1 KiB swizzle atom)
constexpr int kThreads = 640;
constexpr int kSoftmaxRegs = 112;                     // 32 + 4 x 112 = 480 per lane slot
constexpr int kControlRegs = 32;
constexpr float kLazyThreshold = 8.0f;
constexpr float kSafeSum = 18446744073709551616.0f;   // 2^64
__host__ __device__ constexpr uint32_t col_s(int qt, int b) { return (uint32_t)((qt * 2 + b) * kN); }
__host__ __device__ constexpr uint32_t col_o(int qt) { return qt ? 448u : 384u; }

constexpr uint32_t kIdescQK = idesc_bf16_f32(128, kN, false, false);   // A = Q, B = K, both K-major
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 64, false, true);    // A = P (TMEM), B = V MN-major

#ifndef MEA_DB_POLY_MASK
#define MEA_DB_POLY_MASK 0x00000080u  // 1 of the 24 pairs on the FMA pipe (0: +1.4 %, 2: +1.6 %, 3: +2.3 %, 4: +1.6 % measured)
#endif
// the statistics pass (no P pack, no P store) has issue slots to spare for more of them
#ifndef MEA_DB_POLY_MASK_STATS
#define MEA_DB_POLY_MASK_STATS 0x00249249u  // every third pair: 8 of 24 (2: +4.9 %, 4: +2.4 %, 6: +0.6 %, 10: +0.5 %, 12: +1.9 % measured)
#endif
template <bool kStats>
__device__ __forceinline__ constexpr bool poly_pair(int i) {
  return (((kStats ? MEA_DB_POLY_MASK_STATS : MEA_DB_POLY_MASK)) >> i) & 1u;
}

struct DbSmem {
  uint8_t q[2][kQTileBytes];
  uint8_t k[kStages][kKVTileBytes];
  uint8_t v[kStages][kKVTileBytes];
  uint64_t q_full;
  uint64_t kv_full[kStages];
  uint64_t kv_empty[kStages];
  uint64_t s_full[2][2];  // [query tile][buffer]
  uint64_t p_full[2][2];  // [query tile][tile parity]: an arrival for tile t+1 never lands in tile t's phase
  uint64_t pv_done[2];
  uint64_t o_done[2];
  uint32_t tmem_base;
};
constexpr size_t kDbSmemBytes = sizeof(DbSmem) + 1024;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

template <bool kStats>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_db_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  DbSmem& sm = *reinterpret_cast<DbSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: a 1-D grid ordered heaviest block (last rows) first across all (b, h)
  const int qblk = p.causal ? p.num_q_blocks - 1 - (int)(blockIdx.x / (p.H * p.B)) : (int)blockIdx.x;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int q0 = p.q_begin + qblk * kRowsPerCta;
  const int q_end = min(p.n_q, p.q_begin + p.q_count);
  // key tiles query tile qt needs (causal, n_q == n_k: keys below its last row + 1); the
  // producer streams the union (query tile 1's)
  // key padding: this batch element's keys [0, nk); at least one tile runs (all masked if nk = 0)
  const int nk = keys_of(p.kv_lens, b, p.n_k);
  auto tiles_for = [&](int qt) {
    return max(1, ((p.causal ? min(nk, q0 + (qt + 1) * kTileM) : nk) + kN - 1) / kN);
  };
  const int T = tiles_for(1);

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 2);  // one commit per query tile
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i][0], 1);
      mbar_init(&sm.s_full[i][1], 1);
      mbar_init(&sm.p_full[i][0], 256);
      mbar_init(&sm.p_full[i][1], 256);
      mbar_init(&sm.pv_done[i], 1);
      mbar_init(&sm.o_done[i], 1);
    }
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

  if (warp < 4) {
    setmaxnreg_dec<kControlRegs>();
    if (warp == 0) {
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
    } else if (warp == 1 || warp == 3) {
      // ---------------------------------------------------------- MMA issuers
      const int qt = warp >> 1;
      const int Tq = tiles_for(qt);
      const uint64_t dq = shfl0_u64(sdesc_sw128(smem_u32(sm.q[qt]), 16, 1024));
      const uint64_t dk0 = shfl0_u64(sdesc_sw128(smem_u32(sm.k[0]), 16, 1024));
      const uint64_t dv0 = shfl0_u64(sdesc_sw128(smem_u32(sm.v[0]), 16, 1024));
      constexpr uint64_t kStageStep = kKVTileBytes >> 4;
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t to = tmem_u + col_o(qt);
      auto qk = [&](int t) {  // S[qt][t & 1] = Q K_t^T
        const uint64_t dk = dk0 + (t % kStages) * kStageStep;
        const uint32_t ts = tmem_u + col_s(qt, t & 1);
#pragma unroll
        for (int kk = 0; kk < kHeadDim / 16; ++kk) umma_ss(ts, dq + kk * 2, dk + kk * 2, kIdescQK, kk > 0);
        umma_commit(&sm.s_full[qt][t & 1]);
      };
      auto pv = [&](int t) {  // O += P_t V_t, P_t over the first 48 columns of S[qt][t & 1]
        const uint64_t dv = dv0 + (t % kStages) * kStageStep;
        const uint32_t tp = tmem_u + col_s(qt, t & 1);
#pragma unroll
        for (int kk = 0; kk < kN / 16; ++kk)
          umma_ts(to, tp + kk * 8, dv + kk * 128, kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&sm.q_full, 0);
      for (int t = 0; t < 2 && t < Tq; ++t) {
        mbar_wait(&sm.kv_full[t], 0);
        tc_fence_after();
        if (elect_one()) qk(t);
        __syncwarp();
      }
#ifdef MEA_EXP_TIMING
#define IPROBE(k) if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 && t >= 8 && t < 24) \
    reinterpret_cast<unsigned long long*>(p.lse)[512 + (qt * 16 + (t - 8)) * 8 + (k)] = clock64();
#else
#define IPROBE(k)
#endif
      // The issuer's waits poll (mbarrier.test_wait) up to 32 times before suspending: it resumes
      // as soon as the last softmax warp has stored P_t, without burning issue slots and power on
      // long waits (vs try_wait: -2 % at full clocks; vs pure polling: -0.7 % at full clocks and
      // -1 % under the sustained power cap, measured).
      if (kStats) {
        // scores only: K_t is released when QK_t completes; S_{t+2} refills S_t's buffer as soon
        // as the softmax has read S_t into registers (p_full)
        for (int t = 0; t < Tq; ++t) {
          if (elect_one()) umma_commit(&sm.kv_empty[t % kStages]);   // tracks QK_t (issued above)
          __syncwarp();
          mbar_poll_wait<32>(&sm.p_full[qt][t & 1], (t >> 1) & 1);
          if (t + 2 < Tq) {
            mbar_poll_wait<32>(&sm.kv_full[(t + 2) % kStages], ((t + 2) / kStages) & 1);
            tc_fence_after();
            if (elect_one()) qk(t + 2);
            __syncwarp();
          }
        }
      }
      for (int t = 0; t < (kStats ? 0 : Tq); ++t) {
        mbar_poll_wait<32>(&sm.p_full[qt][t & 1], (t >> 1) & 1);
        IPROBE(0)
        tc_fence_after();
        if (elect_one()) {
          pv(t);
          umma_commit(&sm.kv_empty[t % kStages]);
          umma_commit(&sm.pv_done[qt]);
          if (t + 1 == Tq) umma_commit(&sm.o_done[qt]);
        }
        __syncwarp();
        IPROBE(1)
        if (t + 2 < Tq) {
          // S_{t+2} goes into the buffer P_t occupies: wait until PV_t has read it
          mbar_poll_wait<32>(&sm.kv_full[(t + 2) % kStages], ((t + 2) / kStages) & 1);
#ifndef MEA_DB_NO_PV_WAIT
          mbar_poll_wait<32>(&sm.pv_done[qt], t & 1);
#endif
          IPROBE(2)
          tc_fence_after();
          if (elect_one()) qk(t + 2);
          __syncwarp();
          IPROBE(3)
        }
      }
      // key tiles past this query tile's last row (causal): release their ring stages unused
      for (int t = Tq; t < T; ++t) {
        mbar_wait(&sm.kv_full[t % kStages], (t / kStages) & 1);
        if (elect_one()) umma_commit(&sm.kv_empty[t % kStages]);
        __syncwarp();
      }
    }
  } else {
    setmaxnreg_inc<kSoftmaxRegs>();
    // ------------------------------------------------------------ softmax warps
    // warp (qt, sub, quarter) owns TMEM lanes L0 = quarter*32 + sub*16 + [0,16) of query tile qt.
    // Scores are read with the .16x256b shape and P written with .16x128b (ptx.cuh): thread t
    // (q = t % 4) holds rows a = L0 + t/4 and b = L0 + 8 + t/4, score columns 8r + 2q, 8r + 2q + 1
    // of both (r = 0..11) — exactly the keys of P column 4r + q, which .16x128b stores from the
    // same thread. A row is spread over the 4 threads of a quad (max / sum: two xor-shuffles).
    // These shapes cost the exponential unit far less per byte than .16x32bx2 (tools/micro/mio_mix.cu:
    // the forward's per-tile traffic 18.2 -> 16.3 cycles per exponential pair per SMSP).
    const int sw = warp - 4;
    const int qt = sw >> 3;
    const int sub = (sw >> 2) & 1;
    const int quarter = warp & 3;
    const int q = lane & 3;
    const int ra = lane >> 2;              // row a = L0 + ra, row b = L0 + 8 + ra
    const int L0 = quarter * 32 + sub * 16;
    const int r0 = q0 + qt * kTileM;       // first row of this query tile
    const int row_a = r0 + L0 + ra, row_b = row_a + 8;
    const int Tq = tiles_for(qt);
    const int lim_a = p.causal ? min(nk, row_a + 1) : nk;  // keys these rows see: [0, lim)
    const int lim_b = p.causal ? min(nk, row_b + 1) : nk;
    // tiles [0, full) are complete for every row of the query tile (fast-path candidates)
    const int full = (p.causal ? min(nk, r0 + 1) : nk) / kN;
    const uint32_t lane_base = tmem + ((uint32_t)L0 << 16);
    const uint32_t colO = col_o(qt);
    const float c = p.scale_log2;
    float m_a = -INFINITY, m_b = -INFINITY;  // reference max m* per row (log2 units of the scaled score)
    float l_a = 0.f, l_b = 0.f;              // this thread's part of s* per row
#ifdef MEA_EXP_TIMING
    unsigned long long* tdbg = reinterpret_cast<unsigned long long*>(p.lse);
    const bool probe = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && quarter == 0 && sub == 0 && lane == 0;
#define TPROBE(k) if (probe && t >= 8 && t < 24) tdbg[(qt * 16 + (t - 8)) * 8 + (k)] = clock64();
#else
#define TPROBE(k)
#endif
    uint32_t sr[48];
    auto load_s = [&](int t) {
      const uint32_t a = lane_base + col_s(qt, t & 1);
      tmem_ld_16x256b_x8(a, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tmem_ld_16x256b_x4(a + 64, *reinterpret_cast<uint32_t(*)[16]>(&sr[32]));
    };
    auto quad_max = [](float x) {
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1));
      return fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 2));
    };
    auto quad_min = [](float x) {
      x = fminf(x, __shfl_xor_sync(0xffffffffu, x, 1));
      return fminf(x, __shfl_xor_sync(0xffffffffu, x, 2));
    };
    if (Tq > 0) {
      mbar_wait(&sm.s_full[qt][0], 0);
      tc_fence_after();
      load_s(0);
    }
    for (int t = 0; t < Tq; ++t) {
      TPROBE(0)
      tmem_ld_wait();
      TPROBE(1)
      if (kStats) {  // S_t is in registers: its buffer may be refilled
        tc_fence_before();
        mbar_arrive(&sm.p_full[qt][t & 1]);
      }
      const int valid_a = lim_a - t * kN, valid_b = lim_b - t * kN;  // keys of this tile each row sees
      uint32_t pk[24];
      // fast path: m* set, and every row of the query tile sees every key of this tile
      bool fast = (t > 0) && (t < full) && (c >= 0.f);
      if (fast) {
        const float2 c2 = make_float2(c, c), na2 = make_float2(-m_a, -m_a), nb2 = make_float2(-m_b, -m_b);
        float2 rsa = make_float2(0.f, 0.f), rsb = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 12; ++r) {
          const float2 sa = make_float2(__uint_as_float(sr[4 * r]), __uint_as_float(sr[4 * r + 1]));
          const float2 sb = make_float2(__uint_as_float(sr[4 * r + 2]), __uint_as_float(sr[4 * r + 3]));
          const float2 xa = __ffma2_rn(sa, c2, na2), xb = __ffma2_rn(sb, c2, nb2);  // s*c - m*
#ifdef MEA_EXP_NOEXP
          const float2 ea = __fmul2_rn(xa, make_float2(1e-30f, 1e-30f)), eb = __fmul2_rn(xb, make_float2(1e-30f, 1e-30f));
#else
          const float2 ea = poly_pair<kStats>(2 * r) ? exp2_poly2(xa) : make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
          const float2 eb = poly_pair<kStats>(2 * r + 1) ? exp2_poly2(xb) : make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
#endif
          rsa = __fadd2_rn(rsa, ea);
          rsb = __fadd2_rn(rsb, eb);
          pk[2 * r] = pack_bf16x2(ea.x, ea.y);      // P row a, column 4r + q
          pk[2 * r + 1] = pack_bf16x2(eb.x, eb.y);  // P row b, column 4r + q
        }
        // finite per-thread row sums below 2^64 certify every 2^(s c - m*) term (fwd_sm100a.cu)
        const float suma = rsa.x + rsa.y, sumb = rsb.x + rsb.y;
        const bool need = !(suma <= kSafeSum) || !(sumb <= kSafeSum);
        if (__any_sync(0xffffffffu, need)) fast = false;
        else {
          l_a += suma;
          l_b += sumb;
        }
      }
      if (!fast) {
        // exact extreme of each row's visible scores (this thread's 24, then the quad)
        float ea = c >= 0.f ? -INFINITY : INFINITY, eb = ea;
#pragma unroll
        for (int r = 0; r < 12; ++r)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int k = 8 * r + 2 * q + j;
            const float sa = __uint_as_float(sr[4 * r + j]), sb = __uint_as_float(sr[4 * r + 2 + j]);
            if (c >= 0.f) {
              if (k < valid_a) ea = fmaxf(ea, sa);
              if (k < valid_b) eb = fmaxf(eb, sb);
            } else {
              if (k < valid_a) ea = fminf(ea, sa);
              if (k < valid_b) eb = fminf(eb, sb);
            }
          }
        if (c >= 0.f) {
          ea = quad_max(ea);
          eb = quad_max(eb);
        } else {
          ea = quad_min(ea);
          eb = quad_min(eb);
        }
        const float mca = ea * c, mcb = eb * c;
        const bool need_a = mca > m_a + kLazyThreshold, need_b = mcb > m_b + kLazyThreshold;  // always on the first tile
        float alpha_a = 1.f, alpha_b = 1.f;
        if (need_a) {
          alpha_a = ex2_approx(m_a - mca);  // 0 when m* = -inf
          m_a = mca;
          l_a *= alpha_a;
        }
        if (need_b) {
          alpha_b = ex2_approx(m_b - mcb);
          m_b = mcb;
          l_b *= alpha_b;
        }
        if (!kStats && t > 0 && __any_sync(0xffffffffu, need_a || need_b)) {
          // v* <- v* alpha once PV_{t-1} has finished: O (64 columns) in the same .16x256b layout
          mbar_wait(&sm.pv_done[qt], (t - 1) & 1);
          tc_fence_after();
          uint32_t o[32];
          tmem_ld_16x256b_x8(lane_base + colO, o);
          tmem_ld_wait();
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            o[4 * r] = __float_as_uint(__uint_as_float(o[4 * r]) * alpha_a);
            o[4 * r + 1] = __float_as_uint(__uint_as_float(o[4 * r + 1]) * alpha_a);
            o[4 * r + 2] = __float_as_uint(__uint_as_float(o[4 * r + 2]) * alpha_b);
            o[4 * r + 3] = __float_as_uint(__uint_as_float(o[4 * r + 3]) * alpha_b);
          }
          tmem_st_16x256b_x8(lane_base + colO, o);
        }
        float sa0 = 0.f, sa1 = 0.f, sb0 = 0.f, sb1 = 0.f;
#pragma unroll
        for (int r = 0; r < 12; ++r) {
          const int k = 8 * r + 2 * q;
          const float pa0 = k < valid_a ? ex2_approx(fmaf(__uint_as_float(sr[4 * r]), c, -m_a)) : 0.f;
          const float pa1 = k + 1 < valid_a ? ex2_approx(fmaf(__uint_as_float(sr[4 * r + 1]), c, -m_a)) : 0.f;
          const float pb0 = k < valid_b ? ex2_approx(fmaf(__uint_as_float(sr[4 * r + 2]), c, -m_b)) : 0.f;
          const float pb1 = k + 1 < valid_b ? ex2_approx(fmaf(__uint_as_float(sr[4 * r + 3]), c, -m_b)) : 0.f;
          sa0 += pa0;
          sa1 += pa1;
          sb0 += pb0;
          sb1 += pb1;
          pk[2 * r] = pack_bf16x2(pa0, pa1);
          pk[2 * r + 1] = pack_bf16x2(pb0, pb1);
        }
        l_a += sa0 + sa1;
        l_b += sb0 + sb1;
      }
      TPROBE(4)
      // store P_t over the first half of S_t's buffer and prefetch S_{t+1} (already computed: it
      // sits in the other buffer); then wait for the store and hand P_t to the issuer
      if (!kStats) {
        const uint32_t pa = lane_base + col_s(qt, t & 1);
        tmem_st_16x128b_x8(pa, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
        tmem_st_16x128b_x4(pa + 32, *reinterpret_cast<uint32_t(*)[8]>(&pk[16]));
      }
      // (store issued before the load: waiting for it does not also wait for the load; -1.0 %,
      // -1.3 % causal vs load first, profiles/r02_fwd_ab_store_order.txt)
      if (t + 1 < Tq) {
        mbar_wait(&sm.s_full[qt][(t + 1) & 1], ((t + 1) >> 1) & 1);
        tc_fence_after();
        load_s(t + 1);
      }
      TPROBE(2)
      if (!kStats) {
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&sm.p_full[qt][t & 1]);
      }
      TPROBE(5)
    }
    // ------------------------------------------------------------ epilogue: out = v*/s*
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    const size_t bh = (size_t)b * p.H + h;
    if (kStats) {
      if (q == 0) {
        if (row_a < q_end) p.lse[bh * p.n_q + row_a] = (m_a + __log2f(l_a)) * 0.6931471805599453f;
        if (row_b < q_end) p.lse[bh * p.n_q + row_b] = (m_b + __log2f(l_b)) * 0.6931471805599453f;
      }
    } else {
    mbar_wait(&sm.o_done[qt], 0);
    tc_fence_after();
    uint32_t o[32];
    tmem_ld_16x256b_x8(lane_base + colO, o);
    tmem_ld_wait();
    const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f;  // a row with no keys (padding): out = 0, lse = -inf
    const float inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int row = hb ? row_b : row_a;
      const float inv = hb ? inv_b : inv_a;
      if (row < q_end) {
        const size_t off = (((size_t)b * p.n_q + row) * p.H + h) * kHeadDim + 2 * q;
        if (p.out_f32) {
          float* dst = static_cast<float*>(p.out) + off;
#pragma unroll
          for (int r = 0; r < 8; ++r)
            *reinterpret_cast<float2*>(dst + 8 * r) = make_float2(__uint_as_float(o[4 * r + 2 * hb]) * inv,
                                                                  __uint_as_float(o[4 * r + 2 * hb + 1]) * inv);
        } else {
          uint32_t* dst = reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(p.out) + off);
#pragma unroll
          for (int r = 0; r < 8; ++r)
            dst[4 * r] = pack_bf16x2(__uint_as_float(o[4 * r + 2 * hb]) * inv, __uint_as_float(o[4 * r + 2 * hb + 1]) * inv);
        }
#ifndef MEA_EXP_TIMING
        if (p.lse && q == 0) p.lse[bh * p.n_q + row] = ((hb ? m_b : m_a) + __log2f(hb ? l_b : l_a)) * 0.6931471805599453f;
#endif
      }
    }
    }  // !kStats
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int fwd_db_key_tile() { return kN; }

cudaError_t launch_fwd_db_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                               const CUtensorMap& mv, cudaStream_t s) {
  const dim3 grid = p.causal ? dim3(p.num_q_blocks * p.H * p.B) : dim3(p.num_q_blocks, p.H, p.B);
  if (p.stats_only) {
    const cudaError_t attr = ensure_smem_attr<fwd_db_kernel<true>>((int)kDbSmemBytes);
    if (attr != cudaSuccess) return attr;
    fwd_db_kernel<true><<<grid, kThreads, kDbSmemBytes, s>>>(mq, mk, mv, p);
  } else {
    const cudaError_t attr = ensure_smem_attr<fwd_db_kernel<false>>((int)kDbSmemBytes);
    if (attr != cudaSuccess) return attr;
    fwd_db_kernel<false><<<grid, kThreads, kDbSmemBytes, s>>>(mq, mk, mv, p);
  }
  return cudaGetLastError();
}

}  // namespace mea
