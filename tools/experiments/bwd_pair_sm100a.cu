// bwd_pair_sm100a.cu — the fused backward of bwd_sm100a.cu with the two score MMAs of each
// tile (S^T = K Q^T and dP^T = V dO^T, with their K-extension) issued as CTA-pair MMAs
// (tcgen05.mma.cta_group::2, a cluster of two CTAs = 256 keys of one (b, h)): the leader issues
// M = 256 rows (its 128 keys and its peer's), and each CTA supplies half of the B operand (64 of
// the 128 queries of the Q / dO tile), so the B reads of those MMAs halve. dV, dK and dQ stay
// per-CTA (cta_group::1) MMAs on the pair-allocated TMEM (tools/micro/mma_pair.cu: exact).
// The follower CTA stores its Q / dO tiles with the two 64-query halves swapped (its half for
// the pair MMA sits where the leader keeps queries 0-63), so it keeps every query-indexed operand
// of its own MMAs in that rotated order: P^T columns, the dS^T halves, and the dQ rows.
// Cross-CTA signals: the follower's K/V and Q/dO stages are forwarded to the leader (warp 3),
// and its softmax warps arrive on the leader's s_loaded (one remote arrive per warp).
// Same method, numerics and results as bwd_sm100a.cu.
// Non-causal, no key padding, d = 64 (the launcher falls back to bwd_sm100a.cu otherwise).
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared-memory offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(rank));
#ifdef MEA_PAIR_RELAXED
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
#else
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
#endif
}
__device__ __forceinline__ void alloc2(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void dealloc2(uint32_t t, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(cols));
}
__device__ __forceinline__ void umma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// commit the issuing thread's MMAs to the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3));
}

#ifndef MEA_BSTAGES
#define MEA_BSTAGES 3
#endif
#ifndef MEA_DQBUFS
#define MEA_DQBUFS 1
#endif
constexpr int kBStages = MEA_BSTAGES;       // Q/dO ring
constexpr int kDqBufs = MEA_DQBUFS;         // dQ staging buffers
constexpr int kTile = 128;
constexpr int kTileBytes = kTile * kHeadDim * 2;  // 16 KiB bf16 tile
constexpr int kBThreads = 768;
// setmaxnreg budgets. Measured on B200: setmaxnreg.inc only redistributes the registers the
// CTA was launched with (768 threads x 80 = 480 per lane slot of each SM sub-partition, which
// holds one control, four softmax and one dQ warp); a larger total blocks forever.
// 64 + 4*88 + 56 = 472 <= 480.
#ifndef MEA_BR0
#define MEA_BR0 64
#define MEA_BR1 88
#define MEA_BR2 56
#endif
constexpr int kBCtrlRegs = MEA_BR0, kBSoftRegs = MEA_BR1, kBDqRegs = MEA_BR2;
constexpr uint32_t kColST = 0, kColDPT = 128, kColP = 256, kColDV = 320, kColDK = 384, kColDQ = 448;
constexpr uint32_t kBarDq = 1;              // named barrier of the 4 dQ drain warps

constexpr uint32_t kIdSS = idesc_bf16_f32(256, 128, false, false);   // ST, dPT: pair, M = 256 keys
constexpr uint32_t kIdDV = idesc_bf16_f32(128, 64, false, true);     // A=PT (TMEM), B=dO MN-major
constexpr uint32_t kIdDK = idesc_bf16_f32(128, 64, false, true);     // A=dST K-major, B=Q MN-major
constexpr uint32_t kIdDQ = idesc_bf16_f32(128, 64, true, true);      // A=dS MN-major, B=K MN-major

struct BwdSmem {
  uint8_t k[kTileBytes];
  uint8_t v[kTileBytes];
  uint8_t q[kBStages][kTileBytes];
  uint8_t dout[kBStages][kTileBytes];
  uint8_t ds[2][kTileBytes];          // [query half][128 keys][64 queries] bf16, SW128
  float dq_stage[kDqBufs][2][kTile * 32];  // [buffer][column half][128 rows x 32 f32], SW128
  // K-extension of the score MMAs (one extra K = 16 step each): with A = [-1, -1, 0...] per key
  // and B = [hi, lo, 0...] per query, ST' = K Q^T - lse/scale and dPT' = V dO^T - delta, so the
  // softmax needs no per-query loads: PT = 2^(c ST'), dST = PT o dPT'.
  uint8_t aug_c[kAugTileBytes];              // A: -1 in K columns 0, 1 for all 128 rows
  uint8_t aug[kBStages][2 * kAugTileBytes];  // B: [lse tile][delta tile] of the query tile
  uint64_t kv_full, qdo_full[kBStages], qdo_empty[kBStages];
  uint64_t peer_kv, peer_qdo[kBStages];  // leader: the follower's K/V and Q/dO stages have landed
  uint64_t s_full, s_loaded, p_full, p_free, dq_full, dq_empty, dkv_done;
  uint32_t tmem_base;
};
constexpr size_t kBwdSmemBytes = sizeof(BwdSmem) + 1024;
constexpr uint32_t kAugHalfBytes = kAugTileBytes / 2;  // 64 queries of a K-extension tile

// 1024-byte alignment (128B-swizzle atoms) by pointer arithmetic on the __shared__ array, so
// the compiler keeps the shared address space (LDS/STS instead of generic LD/ST).
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// 1-D bulk copy global -> shared, completion on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// kPad: key padding (p.kv_lens); a separate instantiation keeps the unpadded kernel's register
// allocation untouched (+2 % measured when the padded key limit was folded into the one kernel)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kBThreads, 1)
    bwd_pair_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                    const __grid_constant__ CUtensorMap mdq, const __grid_constant__ CUtensorMap mq64,
                    const __grid_constant__ CUtensorMap mdo64, const BwdParams p) {
  constexpr bool kPad = false;
  extern __shared__ uint8_t smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();  // 0: leader (issues the pair MMAs), 1: follower
  // causal: 1-D grid, key block 0 (the most query tiles) first across all (b, h)
  const int kblk = p.causal ? (int)(blockIdx.x / (p.H * p.B)) : (int)blockIdx.x;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int k0 = kblk * kTile;
  const int NQ = (p.n_q + kTile - 1) / kTile;
  // causal (n_q == n_k): queries before this key tile see none of its keys; iteration i
  // (stages, barrier phases) handles query tile i0 + i
  const int i0 = p.causal ? kblk : 0;
  const int NT = NQ - i0;
  const size_t bh = (size_t)b * p.H + h;

  if (threadIdx.x == 0) {
    mbar_init(&sm.kv_full, 1);
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&sm.qdo_full[i], 1);
      mbar_init(&sm.qdo_empty[i], 2);  // the pair score MMAs (leader's commit) + this CTA's dV/dK
      mbar_init(&sm.peer_qdo[i], 1);
    }
    mbar_init(&sm.peer_kv, 1);
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_loaded, 512 + 16);  // leader: its 16 softmax warps' threads + one per peer warp
    mbar_init(&sm.p_full, 512);
    mbar_init(&sm.p_free, 1);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_empty, 128);
    mbar_init(&sm.dkv_done, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mk);
    tma_prefetch_desc(&mv);
    tma_prefetch_desc(&mdo);
    tma_prefetch_desc(&mdq);
  }
  if (warp == 2) alloc2(&sm.tmem_base, 512);  // pair allocation: 512 columns in both CTAs
  // A side of the K-extension: row r = [-1, -1, 0 ... 0] (bf16), core matrix (r/8, 0) at
  // (r/8)*256 + (r%8)*16, core matrix (r/8, 1) at +128 all zero
  if (threadIdx.x < 256) {
    const int r = threadIdx.x >> 1, kc = threadIdx.x & 1;
    *reinterpret_cast<uint4*>(sm.aug_c + (r >> 3) * 256 + kc * 128 + (r & 7) * 16) =
        make_uint4(kc == 0 ? 0xBF80BF80u : 0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    setmaxnreg_dec<kBCtrlRegs>();
    if (warp == 0) {
      // ---------------------------------------------------------------- TMA producer
      const uint64_t keep = policy_evict_last();
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.kv_full, 2 * kTileBytes);
        tma_load_4d(sm.k, &mk, &sm.kv_full, 0, h, k0, b, keep);
        tma_load_4d(sm.v, &mv, &sm.kv_full, 0, h, k0, b, keep);
      }
      __syncwarp();
      for (int i = 0; i < NT; ++i) {
        const int st = i % kBStages, n = i / kBStages;
        if (i >= kBStages) mbar_wait(&sm.qdo_empty[st], (n - 1) & 1);
        if (elect_one()) {
          const int qrow = (i0 + i) * kTile;
          mbar_arrive_expect_tx(&sm.qdo_full[st], 2 * kTileBytes + kAugTileBytes);
          if (rank == 0) {
            tma_load_4d(sm.q[st], &mq, &sm.qdo_full[st], 0, h, qrow, b, keep);
            tma_load_4d(sm.dout[st], &mdo, &sm.qdo_full[st], 0, h, qrow, b, keep);
          } else {  // follower: queries 64-127 first, then 0-63 (its half of the pair MMAs' B)
            tma_load_4d(sm.q[st], &mq64, &sm.qdo_full[st], 0, h, qrow + 64, b, keep);
            tma_load_4d(sm.q[st] + kTileBytes / 2, &mq64, &sm.qdo_full[st], 0, h, qrow, b, keep);
            tma_load_4d(sm.dout[st], &mdo64, &sm.qdo_full[st], 0, h, qrow + 64, b, keep);
            tma_load_4d(sm.dout[st] + kTileBytes / 2, &mdo64, &sm.qdo_full[st], 0, h, qrow, b, keep);
          }
          // K-extension B halves: this CTA's 64 queries of the lse tile, then of the delta tile
          const uint8_t* ag = p.aug + (bh * NQ + i0 + i) * (2 * kAugTileBytes) + rank * kAugHalfBytes;
          bulk_load(sm.aug[st], ag, kAugHalfBytes, &sm.qdo_full[st]);
          bulk_load(sm.aug[st] + kAugHalfBytes, ag + kAugTileBytes, kAugHalfBytes, &sm.qdo_full[st]);
        }
        __syncwarp();
      }
    } else if (warp == 3) {
      // ---------------------------------------------------------------- follower -> leader
      // the follower's K/V and Q/dO stages have landed: tell the leader (its pair MMAs read them)
      if (rank == 1) {
        mbar_wait(&sm.kv_full, 0);
        if (lane == 0) mbar_arrive_remote(&sm.peer_kv, 0);
        for (int i = 0; i < NT; ++i) {
          mbar_wait(&sm.qdo_full[i % kBStages], (i / kBStages) & 1);
          if (lane == 0) mbar_arrive_remote(&sm.peer_qdo[i % kBStages], 0);
          __syncwarp();
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------------- MMA issuer
      const uint64_t dK = shfl0_u64(sdesc_sw128(smem_u32(sm.k), 16, 1024));
      const uint64_t dV = shfl0_u64(sdesc_sw128(smem_u32(sm.v), 16, 1024));
      const uint64_t dQ0 = shfl0_u64(sdesc_sw128(smem_u32(sm.q[0]), 16, 1024));
      const uint64_t dO0 = shfl0_u64(sdesc_sw128(smem_u32(sm.dout[0]), 16, 1024));
      // dS buffer viewed as K-major dS^T (for dK) and as MN-major dS (for dQ, LBO = the
      // 16 KiB stride between the two 64-query halves)
      const uint64_t dSk = shfl0_u64(sdesc_sw128(smem_u32(sm.ds[0]), 16, 1024));
      const uint64_t dSm = shfl0_u64(sdesc_sw128(smem_u32(sm.ds[0]), kTileBytes, 1024));
      constexpr uint64_t kStep = kTileBytes >> 4;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      // K-extension operands: no-swizzle K-major, core matrices 8 rows x 16 B, K stride 128 B,
      // 8-row stride 256 B
      const uint64_t dC = shfl0_u64(sdesc_noswz(smem_u32(sm.aug_c), 128, 256));
      const uint64_t dA0 = shfl0_u64(sdesc_noswz(smem_u32(sm.aug[0]), 128, 256));
      constexpr uint64_t kAugStep = (2 * kAugTileBytes) >> 4, kAugHalf = kAugHalfBytes >> 4;
      auto scores = [&](int st) {  // ST' = K Q^T - lse/scale ; dPT' = V dO^T - delta
        const uint64_t q = dQ0 + st * kStep, o = dO0 + st * kStep, a = dA0 + st * kAugStep;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma2_ss(tm + kColST, dK + kk * 2, q + kk * 2, kIdSS, kk > 0);
        umma2_ss(tm + kColST, dC, a, kIdSS, 1u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma2_ss(tm + kColDPT, dV + kk * 2, o + kk * 2, kIdSS, kk > 0);
        umma2_ss(tm + kColDPT, dC, a + kAugHalf, kIdSS, 1u);
        commit2_mc(&sm.s_full);         // both CTAs' softmax
        commit2_mc(&sm.qdo_empty[st]);  // the pair's reads of this stage are done (1 of 2 arrivals)
      };
      mbar_wait(&sm.kv_full, 0);
      if (rank == 0) {
        mbar_wait(&sm.peer_kv, 0);
        mbar_wait(&sm.qdo_full[0], 0);
        mbar_wait(&sm.peer_qdo[0], 0);
        tc_fence_after();
        if (elect_one()) scores(0);
        __syncwarp();
      }
#ifdef MEA_EXP_TIMING
      unsigned long long* mdbg = reinterpret_cast<unsigned long long*>(p.dv) + 512;
      const bool mprobe = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0;
#define MPROBE(k) if (mprobe && i >= 8 && i < 24) mdbg[(i - 8) * 8 + (k)] = clock64();
#else
#define MPROBE(k)
#endif
      for (int i = 0; i < NT; ++i) {
        const int st = i % kBStages;
        const bool more = i + 1 < NT;
        MPROBE(0)
        // the next tile's scores as soon as the softmax warps have read ST_i / dPT_i, so they
        // are computed while softmax i runs
        if (more && rank == 0) {
          mbar_wait(&sm.qdo_full[(i + 1) % kBStages], ((i + 1) / kBStages) & 1);
          mbar_wait(&sm.peer_qdo[(i + 1) % kBStages], ((i + 1) / kBStages) & 1);
          MPROBE(1)
          mbar_wait(&sm.s_loaded, i & 1);  // both CTAs' softmax warps have read ST_i / dPT_i
          MPROBE(2)
          tc_fence_after();
          if (elect_one()) scores((i + 1) % kBStages);
          __syncwarp();
        }
        if (rank == 1) mbar_wait(&sm.qdo_full[st], (i / kBStages) & 1);  // its own dV / dK operands
        mbar_wait(&sm.p_full, i & 1);
        MPROBE(3)
        tc_fence_after();
        const uint64_t q = dQ0 + st * kStep, o = dO0 + st * kStep;
        if (elect_one()) {
          // dV += PT dO : K = 128 queries in steps of 16 (PT: 8 columns per step; dO: 16 rows)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) umma_ts(tm + kColDV, tm + kColP + kk * 8, o + kk * 128, kIdDV, (i > 0 || kk > 0));
          // dK += dST Q : A K-major (16 queries = 32 B inside a 64-query half), B = Q MN-major
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_ss(tm + kColDK, dSk + (kk >> 2) * kStep + (kk & 3) * 2, q + kk * 128, kIdDK, (i > 0 || kk > 0));
        }
        __syncwarp();
        if (i > 0) mbar_wait(&sm.dq_empty, (i - 1) & 1);  // dQ of tile i-1 drained from TMEM
        MPROBE(4)
        tc_fence_after();
        if (elect_one()) {
          // dQ = dS K : K = 128 keys in steps of 16 (16 key rows = 2048 B in both operands)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) umma_ss(tm + kColDQ, dSm + kk * 128, dK + kk * 128, kIdDQ, kk > 0);
          umma_commit(&sm.dq_full);
          umma_commit(&sm.p_free);
          umma_commit(&sm.qdo_empty[st]);
          if (!more) umma_commit(&sm.dkv_done);
        }
        __syncwarp();
      }
    }
  } else if (warp < 20) {
    setmaxnreg_inc<kBSoftRegs>();
    // ------------------------------------------------------------------ softmax warpgroups
    const int g = (warp - 4) >> 2;           // query columns [32g, 32g+32)
    const int quarter = warp & 3;
    const int j = quarter * 32 + lane;       // key row within the tile (TMEM lane)
    const bool key_ok = k0 + j < (kPad ? keys_of(p.kv_lens, b, p.n_k) : p.n_k);  // padding: P = 0 -> dK = dV = 0
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    // dST row j, queries [32g, 32g+32) -> half g/2, 16-byte chunks (32g%64)/8 .. +3, swizzled
    // the follower keeps query-indexed operands with the 64-query halves swapped (see header)
    const int gq = rank ? (g ^ 2) : g;
    uint8_t* ds_row = sm.ds[gq >> 1] + j * 128;
    const int chunk0 = ((g & 1) * 32) / 8;
#ifdef MEA_EXP_TIMING
    unsigned long long* tdbg = reinterpret_cast<unsigned long long*>(p.dv);
    const bool probe = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && quarter == 0 && lane == 0;
#define TPROBE(k) if (probe && i >= 8 && i < 24) tdbg[(g * 16 + (i - 8)) * 8 + (k)] = clock64();
#else
#define TPROBE(k)
#endif
    for (int i = 0; i < NT; ++i) {
      const int st = i % kBStages;
      TPROBE(0)
      mbar_wait(&sm.s_full, i & 1);
      TPROBE(1)
      tc_fence_after();
      uint32_t sr[32], dr[32];
      tmem_ld32(lane_base + kColST + g * 32, sr);
      tmem_ld32(lane_base + kColDPT + g * 32, dr);
      tmem_ld_wait();
      tc_fence_before();
      if (rank == 0) {
        mbar_arrive(&sm.s_loaded);  // ST_i / dPT_i are in registers: the next scores may overwrite
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&sm.s_loaded, 0);  // the leader issues the next scores
      }
      const bool diag = p.causal && i == 0;
      uint32_t pk[16], dk[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float2 s2 = make_float2(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
        const float2 d2 = make_float2(__uint_as_float(dr[2 * u]), __uint_as_float(dr[2 * u + 1]));
        const float2 x = __fmul2_rn(s2, c2);  // c (s - lse/scale) = s c - lse log2 e
        // P (padded query rows: lse/scale = +-inf -> 0). MUFU for every pair: moving some pairs
        // to the FMA-pipe polynomial measured +-1 % here (MUFU is not what bounds this kernel).
        float2 pr = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        if (!key_ok) pr = make_float2(0.f, 0.f);
        if (diag) {  // causal diagonal tile: key j > query (32 g + 2 u + {0, 1}) is masked
          if (j > 32 * g + 2 * u) pr.x = 0.f;
          if (j > 32 * g + 2 * u + 1) pr.y = 0.f;
        }
        const float2 ds = __fmul2_rn(pr, d2);  // P (dP - delta)
        pk[u] = pack_bf16x2(pr.x, pr.y);
        dk[u] = pack_bf16x2(ds.x, ds.y);
      }
      TPROBE(2)
      if (i > 0) mbar_wait(&sm.p_free, (i - 1) & 1);  // tile i-1's MMAs no longer read P / dS
      TPROBE(3)
      tmem_st16(lane_base + kColP + gq * 16, pk);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int phys = (chunk0 + cc) ^ (j & 7);
        *reinterpret_cast<uint4*>(ds_row + phys * 16) = make_uint4(dk[4 * cc], dk[4 * cc + 1], dk[4 * cc + 2], dk[4 * cc + 3]);
      }
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
      TPROBE(4)
    }
    // ------------------------------------------------------------------ dV, dK epilogue
    if (g < 2) {
      mbar_wait(&sm.dkv_done, 0);
      tc_fence_after();
      uint32_t r[64];
      const uint32_t col = (g == 0) ? kColDV : kColDK;
      tmem_ld32(lane_base + col, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld32(lane_base + col + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld_wait();
#ifdef MEA_EXP_TIMING
      if (false) {
#else
      if (k0 + j < p.n_k) {
#endif
        const float sc = (g == 0) ? 1.f : p.scale;
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g == 0 ? p.dv : p.dk) +
                             (((size_t)b * p.n_k + k0 + j) * p.H + h) * kHeadDim;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(r[8 * u + 0]) * sc, __uint_as_float(r[8 * u + 1]) * sc);
          w.y = pack_bf16x2(__uint_as_float(r[8 * u + 2]) * sc, __uint_as_float(r[8 * u + 3]) * sc);
          w.z = pack_bf16x2(__uint_as_float(r[8 * u + 4]) * sc, __uint_as_float(r[8 * u + 5]) * sc);
          w.w = pack_bf16x2(__uint_as_float(r[8 * u + 6]) * sc, __uint_as_float(r[8 * u + 7]) * sc);
          reinterpret_cast<uint4*>(dst)[u] = w;
        }
      }
    }
  } else {
    setmaxnreg_dec<kBDqRegs>();
    // ------------------------------------------------------------------ dQ drain
    const int quarter = warp & 3;
    const int rq = (quarter * 32 + lane) ^ (rank ? 64 : 0);  // query row of this TMEM lane
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int i = 0; i < NT; ++i) {
      const int buf = i % kDqBufs;
      mbar_wait(&sm.dq_full, i & 1);
      // the TMA reduce that last read this staging buffer (tile i - kDqBufs) must be done reading
      if (warp == 20 && lane == 0) bulk_wait_group_read<kDqBufs - 1>();
      named_bar_sync(kBarDq, 128);
      tc_fence_after();
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        uint32_t r[32];
        tmem_ld32(lane_base + kColDQ + hc * 32, r);
        tmem_ld_wait();
        if (hc == 1) {
          tc_fence_before();
          mbar_arrive(&sm.dq_empty);  // dQ TMEM may be overwritten by the next tile's MMA
        }
        uint8_t* row = reinterpret_cast<uint8_t*>(sm.dq_stage[buf][hc]) + rq * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const int phys = cc ^ (rq & 7);
          *reinterpret_cast<uint4*>(row + phys * 16) = make_uint4(r[4 * cc], r[4 * cc + 1], r[4 * cc + 2], r[4 * cc + 3]);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(kBarDq, 128);
      if (warp == 20 && lane == 0) {
        tma_reduce_add_4d(&mdq, sm.dq_stage[buf][0], 0, h, (i0 + i) * kTile, b);
        tma_reduce_add_4d(&mdq, sm.dq_stage[buf][1], 32, h, (i0 + i) * kTile, b);
        bulk_commit_group();
      }
    }
    if (warp == 20 && lane == 0) bulk_wait_group0();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer is done with every pair MMA / remote arrive before the TMEM goes
  if (warp == 2) {
    tc_fence_after();
    dealloc2(tmem, 512);
  }
}

}  // namespace

cudaError_t launch_bwd_pair(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                            const CUtensorMap& mdo, const CUtensorMap& mdq, const CUtensorMap& mq64,
                            const CUtensorMap& mdo64, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr<bwd_pair_kernel>((int)kBwdSmemBytes);
  if (attr != cudaSuccess) return attr;
  const dim3 grid((p.num_k_blocks + 1) / 2 * 2, p.H, p.B);  // whole CTA pairs
  bwd_pair_kernel<<<grid, kBThreads, kBwdSmemBytes, s>>>(mq, mk, mv, mdo, mdq, mq64, mdo64, p);
  return cudaGetLastError();
}

}  // namespace mea
