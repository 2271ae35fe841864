// fwd_sm100a.cu — self-attention forward on tcgen05 tensor cores (bf16 in, fp32 accumulate).
//
// The paper's per-query stream run for 128 query rows at a time: one
// softmax thread owns one query row and keeps its running max m* and weight sum s* in
// registers; the running value sum v* (the O accumulator) lives in TMEM. Keys arrive in
// tiles of 128 (a "key chunk", Figure 1 lines 12-19 = PAPER.md:118-126):
//   S  = Q K^T                 tcgen05.mma SS  -> TMEM         (einsum qhd,khd->qhk)
//   m  = max(m*, rowmax S)     registers
//   P  = 2^(S*c - m), c = scale*log2 e                        (scale P:116)
//   s* = s* alpha + rowsum P,  v* = v* alpha + P V            (PV = tcgen05.mma TS)
// and out = v*/s* at the end. The rescale by alpha = 2^(m_old - m_new) is
// applied lazily ("renormalize ... as needed"): only when the row max grows by more
// than 2^8, so v* and s* are kept relative to a reference max that may lag the true max by
// at most 8 (in log2 units). All terms share the reference, so the result is unchanged.
//
// CTA = 2 query tiles (256 rows) of one (b, h) sharing every K/V tile:
//   warp 0      TMA producer: Q0,Q1 once, then a 4-stage K/V ring (mbarrier full/empty)
//   warps 1, 3  MMA issuers for query tile 0 / 1 (one elected lane each): S = Q K^T,
//               O += P V; commits -> mbarriers
//   warp 2      TMEM allocator
//   warps 4-11  softmax for query tile 0: warps 4-7 take score columns 0-63 of each key tile,
//               warps 8-11 columns 64-127 (a thread = one row-half = one TMEM lane)
//   warps 12-19 softmax for query tile 1, same split
// Splitting each row over two threads gives 4 softmax warps per SM sub-partition: enough
// independent instruction streams to keep the exponential units busy (one warp per SMSP
// reached only ~0.5 IPC on its dependency chains). The halves exchange their partial row
// max through shared memory once per tile.
// Per query tile, the issuer writes S_{t+1} = Q K_{t+1}^T as soon as the softmax warps have read
// S_t out of TMEM ("s_loaded"), so scores are computed while the softmax runs; O += P_t V_t
// follows once P_t is stored ("p_full"). The softmax waits "pv_done" of tile t-1 before it
// overwrites P or rescales O (rare).
//
// TMEM columns (512 allocated): S0 [0,128) S1 [128,256) O0 [256,320) O1 [320,384)
//                                P0 [384,448) P1 [448,512)  (P = bf16 pairs, 2 per column)
//
// Key split (the paper's key chunks): with num_splits > 1 each CTA covers a
// contiguous key range and stores its unnormalised (m*, s*, v*) instead of out; merge_rows()
// then applies Figure 1's global-max rescale (lines 33-40).
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

#ifndef MEA_FSTAGES
#define MEA_FSTAGES 4
#endif
constexpr int kStages = MEA_FSTAGES;  // K/V ring depth
constexpr int kTileBytes = kTileN * kHeadDim * 2;  // 16 KiB: 128 rows x 128 B
constexpr int kThreads = 640;  // 4 producer/MMA/alloc warps + 4 softmax warpgroups
// setmaxnreg.inc can only redistribute the registers the CTA was launched with (640 x 96:
// 480 per lane slot of an SM sub-partition, which holds 1 control + 4 softmax warps); a larger
// total blocks forever (measured).
// 112 / 32 (32 + 4 * 112 = 480): the softmax's scores, P pairs and the redo copy spilled at 104
// (76 bytes per thread, ~4 % of the kernel time); the producer / MMA-issuer warps fit in 32.
#ifndef MEA_FREG_SOFT
#define MEA_FREG_SOFT 112
#define MEA_FREG_CTRL 32
#endif
constexpr int kSoftmaxRegs = MEA_FREG_SOFT;
constexpr int kControlRegs = MEA_FREG_CTRL;
__host__ __device__ constexpr uint32_t col_s(int wg) { return wg ? 128u : 0u; }
__host__ __device__ constexpr uint32_t col_o(int wg) { return wg ? 320u : 256u; }
__host__ __device__ constexpr uint32_t col_p(int wg) { return wg ? 448u : 384u; }
constexpr float kLazyThreshold = 8.0f;
constexpr float kSafeSum = 18446744073709551616.0f;  // 2^64: bound on a tile's half-row sum of terms

constexpr uint32_t kIdescQK = idesc_bf16_f32(128, 128, false, false);  // A=Q K-major, B=K K-major
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 64, false, true);    // A=P (TMEM), B=V MN-major

struct FwdSmem {
  uint8_t q[2][kTileBytes];
  uint8_t k[kStages][kTileBytes];
  uint8_t v[kStages][kTileBytes];
  uint64_t q_full;
  uint64_t kv_full[kStages];
  uint64_t kv_empty[kStages];
  uint64_t s_full[2];
  uint64_t s_loaded[2];  // the softmax warps of a query tile have read S_t (S_{t+1} may be written)
  uint64_t pv_done[2];   // PV_t finished: P buffer free again, O quiescent
  uint64_t p_full[2];
  uint64_t o_done[2];
  uint32_t tmem_base;
  uint32_t merge_last;  // fused merge: this CTA is the last split of its query block
};
constexpr size_t kFwdSmemBytes = sizeof(FwdSmem) + 1024;

// 1024-byte alignment (128B-swizzle atoms) by pointer arithmetic on the __shared__ array, so
// the compiler keeps the shared address space (LDS/STS instead of generic LD/ST).
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// S[tmem d_col] = Qtile . Ktile^T  (M=128 queries, N=128 keys, K=64 in 4 steps of 16)
__device__ __forceinline__ void issue_qk(uint32_t d_tmem, const uint8_t* qt, const uint8_t* kt) {
  const uint32_t qa = smem_u32(qt), ka = smem_u32(kt);
#pragma unroll
  for (int kk = 0; kk < kHeadDim / 16; ++kk) {
    // K-major SW128: 16 bf16 = 32 B per K step inside the 128-B swizzle row.
    umma_ss(d_tmem, sdesc_sw128(qa + kk * 32, 16, 1024), sdesc_sw128(ka + kk * 32, 16, 1024), kIdescQK,
            kk > 0);
  }
}
// O[tmem d_col] (+)= P[tmem p_col] . Vtile  (M=128, N=64, K=128 keys in 8 steps of 16)
__device__ __forceinline__ void issue_pv(uint32_t d_tmem, uint32_t p_tmem, const uint8_t* vt, bool acc) {
  const uint32_t va = smem_u32(vt);
#pragma unroll
  for (int kk = 0; kk < kTileN / 16; ++kk) {
    // MN-major SW128 B operand: 16 keys = 2 groups of 8 rows of 128 B; SBO = 1024 B.
    umma_ts(d_tmem, p_tmem + kk * 8, sdesc_sw128(va + kk * 2048, 16, 1024), kIdescPV, (acc || kk > 0) ? 1u : 0u);
  }
}

// Which of the 32 exponential pairs of a half row go to the FMA pipe (bit i = pair i). Measured
// at configs[2] with interleaved timing (tools/fwd_experiments.py): pairs {9, 25} 6 % faster than
// {15, 31}; {7, 23} and every 8th pair no better than {15, 31}; every 24th slower. The placement
// matters because it decides what the scheduler can overlap with the MUFU queue.
#ifndef MEA_POLY_MASK
#define MEA_POLY_MASK 0x02000200u
#endif
__device__ __forceinline__ constexpr bool poly_pair(int i) { return ((MEA_POLY_MASK) >> i) & 1u; }

__global__ void __launch_bounds__(kThreads, 1)
    fwd_bf16_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                    const __grid_constant__ CUtensorMap mv, const FwdParams p) {
  // PDL: the next kernel in the stream (the window's merge) may be scheduled now; it waits for
  // this grid's results itself (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ uint8_t smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: the blocks with the most key tiles (the last rows) are scheduled first
  // causal: a 1-D grid ordered heaviest block first across all (b, h) (the block scheduler then
  // runs a longest-job-first schedule); otherwise x = split * num_q_blocks + block, y = h, z = b
  const int cidx = blockIdx.x / (p.H * p.B);
  const int qblk = p.causal ? p.num_q_blocks - 1 - cidx : blockIdx.x % p.num_q_blocks;
  const int split = p.causal ? 0 : blockIdx.x / p.num_q_blocks;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int q0 = p.q_begin + qblk * kRowsPerCta;
  const int q_end = min(p.n_q, p.q_begin + p.q_count);
  const int n_tiles = (p.n_k + kTileN - 1) / kTileN;
  const int t_begin = (p.split_base + split) * p.tiles_per_split;  // split_base: tree schedule, one chunk per launch
  // causal (n_q == n_k, no split): query tile qt of this block needs key tiles [0, 2 qblk + qt]
  // (the last one is its diagonal tile); the producer streams the union.
  const int t_end = p.causal ? min(n_tiles, 2 * qblk + 2) : min(n_tiles, t_begin + p.tiles_per_split);
  const int T = t_end - t_begin;
  const int key_end = min(p.n_k, t_end * kTileN);

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 2);  // one commit per query tile
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.p_full[i], 256);  // both halves of every row
      mbar_init(&sm.s_loaded[i], 256);
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

  // Register hand-off (inside each role branch so ptxas sees the budget per region):
  // warpgroup 0 (producer / MMA / allocator) needs few registers; the softmax warpgroups
  // hold a 128-score row each.
  if (warp < 4) {
    setmaxnreg_dec<kControlRegs>();
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
    if (elect_one()) {
      mbar_arrive_expect_tx(&sm.q_full, 2 * kTileBytes);
      tma_load_4d(sm.q[0], &mq, &sm.q_full, 0, h, q0, b, stream);
      tma_load_4d(sm.q[1], &mq, &sm.q_full, 0, h, q0 + kTileM, b, stream);
    }
    __syncwarp();
    for (int t = 0; t < T; ++t) {
      const int st = t % kStages, n = t / kStages;
      if (t >= kStages) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
      const int krow = (t_begin + t) * kTileN;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.kv_full[st], 2 * kTileBytes);
        tma_load_4d(sm.k[st], &mk, &sm.kv_full[st], 0, h, krow, b, keep);
        tma_load_4d(sm.v[st], &mv, &sm.kv_full[st], 0, h, krow, b, keep);
      }
      __syncwarp();
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers
    // One issuer warp per query tile (warp 1: tile 0, warp 3: tile 1), so the two tiles'
    // softmax pipelines are not forced into lockstep by a single program order. The whole
    // warp walks the schedule (waits are warp-wide); one elected lane issues. Descriptors are
    // precomputed: a K step or a ring stage is a plain add to the start-address field.
    const int qt = __shfl_sync(0xffffffffu, warp >> 1, 0);
    const int Tq = p.causal ? min(T, 2 * qblk + qt + 1) : T;  // key tiles this query tile uses
    const uint64_t dq = shfl0_u64(sdesc_sw128(smem_u32(sm.q[qt]), 16, 1024));
    const uint64_t dk0 = shfl0_u64(sdesc_sw128(smem_u32(sm.k[0]), 16, 1024));
    const uint64_t dv0 = shfl0_u64(sdesc_sw128(smem_u32(sm.v[0]), 16, 1024));
    constexpr uint64_t kStageStep = kTileBytes >> 4;
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t ts = tmem_u + col_s(qt), to = tmem_u + col_o(qt), tp = tmem_u + col_p(qt);
    auto qk = [&](int st) {
      const uint64_t dk = dk0 + st * kStageStep;
#pragma unroll
      for (int kk = 0; kk < kHeadDim / 16; ++kk) umma_ss(ts, dq + kk * 2, dk + kk * 2, kIdescQK, kk > 0);
    };
    auto pv = [&](int st, bool acc) {
      const uint64_t dv = dv0 + st * kStageStep;
#pragma unroll
      for (int kk = 0; kk < kTileN / 16; ++kk) umma_ts(to, tp + kk * 8, dv + kk * 128, kIdescPV, (acc || kk > 0) ? 1u : 0u);
    };
    mbar_wait(&sm.q_full, 0);
    mbar_wait(&sm.kv_full[0], 0);
    tc_fence_after();
    if (elect_one()) {
      qk(0);
      umma_commit(&sm.s_full[qt]);
    }
    __syncwarp();
#ifdef MEA_EXP_TIMING
#define IPROBE(k) if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 && t >= 8 && t < 24) \
    reinterpret_cast<unsigned long long*>(p.lse)[512 + (qt * 16 + (t - 8)) * 8 + (k)] = clock64();
#else
#define IPROBE(k)
#endif
    for (int t = 0; t < Tq; ++t) {
      IPROBE(0)
      const int st = t % kStages;
      const int nx = (t + 1) % kStages;
      const bool more = (t + 1) < Tq;
      // S_{t+1} = Q K_{t+1}^T as soon as the softmax warps have read S_t out of TMEM, so the
      // next scores are computed while the current softmax runs.
      if (more) {
        mbar_wait(&sm.kv_full[nx], ((t + 1) / kStages) & 1);
        IPROBE(1)
        mbar_wait(&sm.s_loaded[qt], t & 1);
        IPROBE(2)
        tc_fence_after();
        if (elect_one()) {
          qk(nx);
          umma_commit(&sm.s_full[qt]);
        }
        __syncwarp();
        IPROBE(3)
      }
      // O += P_t V_t once P_t is in TMEM
      mbar_wait(&sm.p_full[qt], t & 1);
      IPROBE(4)
      tc_fence_after();
      if (elect_one()) {
        pv(st, t > 0);
        umma_commit(&sm.pv_done[qt]);
        umma_commit(&sm.kv_empty[st]);  // this tile is done with K_t, V_t (2 arrivals free it)
        if (!more) umma_commit(&sm.o_done[qt]);
      }
      __syncwarp();
      IPROBE(5)
    }
    // key tiles past this query tile's diagonal (causal): release their ring stage without
    // using it (a commit keeps the arrival ordered after this warp's earlier MMAs)
    for (int t = Tq; t < T; ++t) {
      mbar_wait(&sm.kv_full[t % kStages], (t / kStages) & 1);
      if (elect_one()) umma_commit(&sm.kv_empty[t % kStages]);
      __syncwarp();
    }
  }
  } else {
    setmaxnreg_inc<kSoftmaxRegs>();
    // ------------------------------------------------------------ softmax warps
    // 16 warps; warp (qt, sub, quarter) owns query tile qt, TMEM lanes L0 = quarter*32 + sub*16
    // + [0,16). S is read as .16x256b and P written as .16x128b (ptx.cuh, as fwd_db): thread t
    // (q = t % 4) holds rows a = L0 + t/4 and b = a + 8, score columns 8r + 2q, 8r + 2q + 1
    // (r = 0..15) of both — the keys of P column 4r + q it stores; a row is spread over a quad
    // (max / sum: two xor-shuffles). Every thread keeps both rows' reference max m* (identical
    // across the quad) and its part of their s*.
    const int sw = warp - 4;
    const int qt = sw >> 3;
    const int sub = (sw >> 2) & 1;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int q = lane & 3, ra = lane >> 2;
    const int L0 = quarter * 32 + sub * 16;
    const int row_a = q0 + qt * kTileM + L0 + ra, row_b = row_a + 8;
    const uint32_t lane_base = tmem + ((uint32_t)L0 << 16);
    const uint32_t colS = col_s(qt), colO = col_o(qt), colP = col_p(qt);
    const float c = p.scale_log2;
    float m_a = -INFINITY, m_b = -INFINITY;  // reference max m*, log2 units of the scaled score
    float l_a = 0.f, l_b = 0.f;              // this thread's part of s*
#ifdef MEA_EXP_TIMING
    unsigned long long* tdbg = reinterpret_cast<unsigned long long*>(p.lse);
    const bool probe = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && quarter == 0 && sub == 0 && lane == 0;
#define TPROBE(k) if (probe && t >= 8 && t < 24) tdbg[(qt * 16 + (t - 8)) * 8 + (k)] = clock64();
#else
#define TPROBE(k)
#endif
    const int Tq = p.causal ? min(T, 2 * qblk + qt + 1) : T;
    const int diag = p.causal ? 2 * qblk + qt : -1;  // the causal diagonal key tile of this query tile
    for (int t = 0; t < Tq; ++t) {
      TPROBE(0)
      mbar_wait(&sm.s_full[qt], t & 1);
      TPROBE(1)
      tc_fence_after();
      uint32_t sr[64];
      // keys of this tile in range per row (causal: keys <= row)
      const int kb = (t_begin + t) * kTileN;
      const int valid_a = (p.causal ? min(key_end, row_a + 1) : key_end) - kb;
      const int valid_b = (p.causal ? min(key_end, row_b + 1) : key_end) - kb;
      uint32_t pk[32];  // P in bf16 pairs: [2r] row a, [2r + 1] row b, column 4r + q
      // Fast path (full tile, m* already set): exponentiate against the current reference max.
      // The second 64 score columns load while the first 64 are exponentiated.
      bool fast = (t > 0) && (t != diag) && (key_end - kb >= kTileN) && (c >= 0.f);
      tmem_ld_16x256b_x8(lane_base + colS + 0, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      if (fast) {
        tmem_ld_wait();
        tmem_ld_16x256b_x8(lane_base + colS + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        const float2 c2 = make_float2(c, c), na2 = make_float2(-m_a, -m_a), nb2 = make_float2(-m_b, -m_b);
        float2 rsa = make_float2(0.f, 0.f), rsb = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (r == 8) {  // second half of the scores has landed; S_t may now be overwritten
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sm.s_loaded[qt]);
          }
          const float2 sa = make_float2(__uint_as_float(sr[4 * r]), __uint_as_float(sr[4 * r + 1]));
          const float2 sb = make_float2(__uint_as_float(sr[4 * r + 2]), __uint_as_float(sr[4 * r + 3]));
          const float2 xa = __ffma2_rn(sa, c2, na2), xb = __ffma2_rn(sb, c2, nb2);  // s*c - m*
          const float2 ea = poly_pair(2 * r) ? exp2_poly2(xa) : make_float2(ex2_approx(xa.x), ex2_approx(xa.y));
          const float2 eb = poly_pair(2 * r + 1) ? exp2_poly2(xb) : make_float2(ex2_approx(xb.x), ex2_approx(xb.y));
          rsa = __fadd2_rn(rsa, ea);
          rsb = __fadd2_rn(rsb, eb);
          pk[2 * r] = pack_bf16x2(ea.x, ea.y);
          pk[2 * r + 1] = pack_bf16x2(eb.x, eb.y);
        }
        // No row max here: the max only guards overflow, and every term is
        // bounded by the row sum, so a finite row sum below 2^64 certifies that all
        // 2^(s c - m*) terms (and hence P in bf16 and the fp32 sums) are safe. Otherwise redo
        // the tile with the exact max (rare: the max must grow by > 2^64).
        const float suma = rsa.x + rsa.y, sumb = rsb.x + rsb.y;
        const bool need = !(suma <= kSafeSum) || !(sumb <= kSafeSum);  // also catches inf / NaN
        if (__any_sync(0xffffffffu, need)) {  // warp-uniform: covers every quad of these rows
          fast = false;  // redo from the raw scores (still in registers)
        } else {
          l_a += suma;
          l_b += sumb;
        }
      } else {
        tmem_ld_16x256b_x8(lane_base + colS + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&sm.s_loaded[qt]);  // S_t is in registers: the MMA may overwrite it
      }
      if (!fast) {
        // row extremum of the raw score over valid keys: max if c >= 0, min if c < 0 (thread, quad)
        float ea = c >= 0.f ? -INFINITY : INFINITY, eb = ea;
#pragma unroll
        for (int r = 0; r < 16; ++r)
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
          ea = fmaxf(ea, __shfl_xor_sync(0xffffffffu, ea, 1));
          ea = fmaxf(ea, __shfl_xor_sync(0xffffffffu, ea, 2));
          eb = fmaxf(eb, __shfl_xor_sync(0xffffffffu, eb, 1));
          eb = fmaxf(eb, __shfl_xor_sync(0xffffffffu, eb, 2));
        } else {
          ea = fminf(ea, __shfl_xor_sync(0xffffffffu, ea, 1));
          ea = fminf(ea, __shfl_xor_sync(0xffffffffu, ea, 2));
          eb = fminf(eb, __shfl_xor_sync(0xffffffffu, eb, 1));
          eb = fminf(eb, __shfl_xor_sync(0xffffffffu, eb, 2));
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
        if (t > 0 && __any_sync(0xffffffffu, need_a || need_b)) {
          // v* <- v* alpha once PV_{t-1} has finished (O in the same .16x256b layout)
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
        // P = 2^(s c - m*) in bf16 pairs; s* += rowsum P
        float sa0 = 0.f, sa1 = 0.f, sb0 = 0.f, sb1 = 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
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
      if (t > 0) mbar_wait(&sm.pv_done[qt], (t - 1) & 1);  // PV_{t-1} has consumed P_{t-1}
      tc_fence_after();
      tmem_st_16x128b_x16(lane_base + colP, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full[qt]);
      TPROBE(5)
    }
    // ------------------------------------------------------------ epilogue: out = v*/s*
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);  // s* of the whole rows
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    mbar_wait(&sm.o_done[qt], 0);
    tc_fence_after();
    uint32_t o[32];  // rows a, b; O columns 8r + 2q, 8r + 2q + 1 (r = 0..7)
    tmem_ld_16x256b_x8(lane_base + colO, o);
    tmem_ld_wait();
    // PDL: the previous kernel (the last window's merge) reads the summaries this epilogue
    // overwrites; everything above (all of Q/K/V's streaming) overlapped its drain
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int row = hb ? row_b : row_a;
      if (row >= q_end) continue;
      const float lrow = hb ? l_b : l_a, mrow = hb ? m_b : m_a;
      const size_t bh = (size_t)b * p.H + h;
      auto put_f32 = [&](float* dst, float sc) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
          *reinterpret_cast<float2*>(dst + 8 * r) =
              make_float2(__uint_as_float(o[4 * r + 2 * hb]) * sc, __uint_as_float(o[4 * r + 2 * hb + 1]) * sc);
      };
      if (p.tri_v) {
        // this call's (m*, s*, v*) per row, for a merge across key ranges
        const size_t idx = ((size_t)b * p.n_q + row) * p.H + h;
        put_f32(p.tri_v + idx * p.tri_vs + 2 * q, 1.f);
        if (q == 0) {
          p.tri_m[idx * p.tri_ms] = mrow * 0.6931471805599453f;
          p.tri_s[idx * p.tri_ms] = lrow;
        }
      } else if (p.part_o) {  // key-split / tree summaries
        const size_t prow = ((size_t)split * p.B * p.H + bh) * p.q_count + (row - p.q_begin);
        put_f32(p.part_o + prow * kHeadDim + 2 * q, 1.f);
        if (q == 0) reinterpret_cast<float2*>(p.part_ml)[prow] = make_float2(mrow, lrow);
      } else {
        const float inv = 1.f / lrow;
        const size_t off = (((size_t)b * p.n_q + row) * p.H + h) * kHeadDim + 2 * q;
        if (p.out_f32) {
          put_f32(static_cast<float*>(p.out) + off, inv);
        } else {
          uint32_t* dst = reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(p.out) + off);
#pragma unroll
          for (int r = 0; r < 8; ++r)
            dst[4 * r] = pack_bf16x2(__uint_as_float(o[4 * r + 2 * hb]) * inv, __uint_as_float(o[4 * r + 2 * hb + 1]) * inv);
        }
#ifndef MEA_EXP_TIMING
        if (p.lse && q == 0) p.lse[bh * p.n_q + row] = (mrow + __log2f(lrow)) * 0.6931471805599453f;
#endif
      }
    }
    if (p.merge_cnt) {
      // Fused merge of the key-split summaries (Figure 1 lines 33-40): the last
      // of the num_splits CTAs of this query block to finish merges its 256 rows, so no separate
      // merge launch sits between two query windows (threadfence-reduction pattern).
      __threadfence();
      named_bar_sync(1, 512);  // the 16 softmax warps have written this CTA's summaries
      if (sw == 0 && lane == 0) {
        const size_t ci = ((size_t)b * p.H + h) * p.num_q_blocks + qblk;
        const unsigned prev = atomicAdd(p.merge_cnt + ci, 1u);
        sm.merge_last = prev == (unsigned)(p.num_splits - 1);
        if (sm.merge_last) p.merge_cnt[ci] = 0u;  // every split has arrived: reset for the next window
      }
      named_bar_sync(1, 512);
      if (sm.merge_last) {
        __threadfence();
        const size_t bh = (size_t)b * p.H + h, stride = (size_t)p.B * p.H * p.q_count;
        const float2* ml = reinterpret_cast<const float2*>(p.part_ml);
        for (int rr = sw; rr < kRowsPerCta; rr += 16) {  // warp sw: rows sw, sw + 16, ... of the block
          const int grow = q0 + rr;
          if (grow >= q_end) break;
          const size_t r = bh * p.q_count + (grow - p.q_begin);
          // two passes over the splits, 4 summaries in flight per step (few registers: this code
          // shares the softmax warps' register budget)
          float M = -INFINITY;
          for (int s0 = 0; s0 < p.num_splits; s0 += 4) {
            float mm[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) mm[u] = s0 + u < p.num_splits ? __ldcg(&ml[(s0 + u) * stride + r]).x : -INFINITY;
            M = fmaxf(M, fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])));
          }
          float den = 0.f;
          float2 acc = make_float2(0.f, 0.f);
          for (int s0 = 0; s0 < p.num_splits; s0 += 4) {
            float2 t[4], ov[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const bool ok = s0 + u < p.num_splits;
              const size_t sr = (size_t)(ok ? s0 + u : 0) * stride + r;
              t[u] = ok ? __ldcg(&ml[sr]) : make_float2(-INFINITY, 0.f);
              ov[u] = ok ? __ldcg(reinterpret_cast<const float2*>(p.part_o + sr * kHeadDim) + lane) : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float w = ex2_approx(t[u].x - M);
              den += w * t[u].y;
              acc.x += w * ov[u].x;
              acc.y += w * ov[u].y;
            }
          }
          const float inv = 1.f / den;
          const size_t off = (((size_t)b * p.n_q + grow) * p.H + h) * kHeadDim + 2 * lane;
          if (p.out_f32) reinterpret_cast<float2*>(static_cast<float*>(p.out) + off)[0] = make_float2(acc.x * inv, acc.y * inv);
          else reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(p.out) + off)[0] = pack_bf16x2(acc.x * inv, acc.y * inv);
          if (p.lse && lane == 0) p.lse[bh * p.n_q + grow] = (M + __log2f(den)) * 0.6931471805599453f;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Figure 1 lines 33-40 over the key-split partials of each query row:
// M = max_c m_c; out = sum_c 2^(m_c - M) v*_c / sum_c 2^(m_c - M) s*_c. One warp per row.
__global__ void merge_rows_kernel(const FwdParams p) {
  // PDL trigger first: the grid is small enough to be resident at once, so the next window's
  // forward may start on the SMs the current forward's last wave leaves idle (it waits for this
  // merge itself before overwriting the summaries); then wait for this window's summaries
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t rows = (int64_t)p.B * p.H * p.q_count;  // rows of this query window
  const int lane = threadIdx.x & 31;
  const int64_t stride = rows;  // rows per split
  const int d = p.d, per = d / 32;  // 2 (d = 64) or 4 (d = 128) features per lane
  const float2* ml = reinterpret_cast<const float2*>(p.part_ml);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows;
       r += (int64_t)gridDim.x * (blockDim.x / 32)) {
    float M = -INFINITY;
    for (int s = 0; s < p.num_splits; ++s) M = fmaxf(M, ml[s * stride + r].x);
    float den = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < p.num_splits; ++s) {
      const float2 t = ml[s * stride + r];
      const float w = ex2_approx(t.x - M);
      den += w * t.y;
      const float* o = p.part_o + (s * stride + r) * d + per * lane;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < per) acc[i] += w * o[i];
    }
    const int64_t bh = r / p.q_count, row = p.q_begin + r % p.q_count;
    if (row >= p.n_q) continue;
    const int64_t b = bh / p.H, h = bh % p.H;
    const size_t off = (((size_t)b * p.n_q + row) * p.H + h) * d + per * lane;
    const float inv = 1.f / den;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i >= per) break;
      if (p.out_f32) static_cast<float*>(p.out)[off + i] = acc[i] * inv;
      else static_cast<__nv_bfloat16*>(p.out)[off + i] = __float2bfloat16_rn(acc[i] * inv);
    }
    if (p.lse && lane == 0) p.lse[bh * p.n_q + row] = (M + __log2f(den)) * 0.6931471805599453f;
  }
}

// ---------------------------------------------------------------------------- debug probe
struct DbgSmem {
  uint8_t a[kTileBytes];
  uint8_t b[kTileBytes];
  uint8_t v[kTileBytes];
  uint64_t full, s_done, o_done;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 1)
    debug_umma_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                      const __grid_constant__ CUtensorMap mv, float* s_out, float* o_out) {
  extern __shared__ uint8_t smem_raw[];
  DbgSmem& sm = *reinterpret_cast<DbgSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&sm.full, 1);
    mbar_init(&sm.s_done, 1);
    mbar_init(&sm.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sm.full, 3 * kTileBytes);
    tma_load_4d(sm.a, &ma, &sm.full, 0, 0, 0, 0, policy_evict_first());
    tma_load_4d(sm.b, &mb, &sm.full, 0, 0, 0, 0, policy_evict_first());
    tma_load_4d(sm.v, &mv, &sm.full, 0, 0, 0, 0, policy_evict_first());
    mbar_wait(&sm.full, 0);
    tc_fence_after();
    issue_qk(tmem + col_s(0), sm.a, sm.b);
    umma_commit(&sm.s_done);
  }
  __syncwarp();
  mbar_wait(&sm.s_done, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  uint32_t sr[128];
  for (int c = 0; c < 4; ++c) tmem_ld32(lane_base + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
  tmem_ld_wait();
  for (int i = 0; i < 128; ++i) s_out[row * 128 + i] = __uint_as_float(sr[i]);
  uint32_t pk[64];
  for (int i = 0; i < 64; ++i) pk[i] = pack_bf16x2(__uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1]));
  tmem_st32(lane_base + col_p(0), *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
  tmem_st32(lane_base + col_p(0) + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    issue_pv(tmem + col_o(0), tmem + col_p(0), sm.v, false);
    umma_commit(&sm.o_done);
  }
  __syncwarp();
  mbar_wait(&sm.o_done, 0);
  tc_fence_after();
  uint32_t o[64];
  tmem_ld32(lane_base + col_o(0), *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
  tmem_ld32(lane_base + col_o(0) + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
  tmem_ld_wait();
  for (int i = 0; i < 64; ++i) o_out[row * 64 + i] = __uint_as_float(o[i]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

cudaError_t launch_fwd_bf16(const FwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                            const CUtensorMap& mv, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr<fwd_bf16_kernel>((int)kFwdSmemBytes);
  if (attr != cudaSuccess) return attr;
  const dim3 grid = p.causal ? dim3(p.num_q_blocks * p.H * p.B) : dim3(p.num_q_blocks * p.num_splits, p.H, p.B);
  if (!p.pdl) {
    fwd_bf16_kernel<<<grid, kThreads, kFwdSmemBytes, s>>>(mq, mk, mv, p);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kFwdSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fwd_bf16_kernel, mq, mk, mv, p);
}

// The triple of an empty key range: (m*, s*, v*) = (-inf, 0, 0) (PAPER.md:89's initial state).
__global__ void empty_triples_kernel(float* m, float* s, float* vstar, int64_t ms, int64_t vs, int64_t rows, int d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) {
    m[i * ms] = -INFINITY;
    s[i * ms] = 0.f;
  }
  if (i < rows * d) vstar[(i / d) * vs + i % d] = 0.f;
}

cudaError_t launch_empty_triples(float* m, float* s, float* vstar, int64_t ms, int64_t vs, int64_t rows, int d,
                                 cudaStream_t st) {
  const int64_t n = rows * d;
  empty_triples_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(m, s, vstar, ms, vs, rows, d);
  return cudaGetLastError();
}

cudaError_t launch_merge_rows(const FwdParams& p, cudaStream_t s) {
  const int64_t rows = (int64_t)p.B * p.H * p.q_count;
  const int warps = 8;
  // PDL: scheduled while the forward grid drains; waits for its summaries (griddepcontrol.wait)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::min<int64_t>((rows + warps - 1) / warps, 148 * 4));  // resident at once
  cfg.blockDim = dim3(warps * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, merge_rows_kernel, p);
}

// Two summaries of the same query rows over disjoint key ranges -> one (Figure 1 lines 33-36,
// PAPER.md:140-144, for two chunks): M = max(m_a, m_b), w = 2^(m - M), s = s_a w_a + s_b w_b,
// v* = v*_a w_a + v*_b w_b. Empty summaries (m = -inf) contribute nothing. Warp per row.
__global__ void merge_pair_kernel(float* dst_o, float2* dst_ml, const float* src_o, const float2* src_ml,
                                  int64_t rows, int d) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float2 a = dst_ml[r], b = src_ml[r];
  const float M = fmaxf(a.x, b.x);
  const float wa = M == -INFINITY ? 0.f : ex2_approx(a.x - M);
  const float wb = M == -INFINITY ? 0.f : ex2_approx(b.x - M);
  for (int i = lane; i < d; i += 32) dst_o[r * d + i] = dst_o[r * d + i] * wa + src_o[r * d + i] * wb;
  __syncwarp();
  if (lane == 0) dst_ml[r] = make_float2(M, a.y * wa + b.y * wb);
}

cudaError_t launch_merge_pair(float* dst_o, float2* dst_ml, const float* src_o, const float2* src_ml, int64_t rows,
                              int d, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int warps = 8;
  merge_pair_kernel<<<(unsigned)((rows + warps - 1) / warps), warps * 32, 0, s>>>(dst_o, dst_ml, src_o, src_ml,
                                                                               rows, d);
  return cudaGetLastError();
}

cudaError_t launch_debug_umma_tile(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mv,
                                   float* s_out, float* o_out, cudaStream_t s) {
  const size_t smem = sizeof(DbgSmem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(debug_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  debug_umma_kernel<<<1, 128, smem, s>>>(ma, mb, mv, s_out, o_out);
  return cudaGetLastError();
}

}  // namespace mea
