// bwd_sm100a.cu — backward of exact attention on tcgen05 tensor cores, recomputing every tile of
// scores from the saved per-row log-sum-exp instead of storing them (the paper's checkpointed
// differentiation: "recomputed during backpropagation"). The max carries no
// gradient (stop_gradient): with lse fixed the derivative is the plain softmax
// VJP:
//   P = exp(scale q k^T - lse),  dV = P^T dO,  dP = dO V^T,  delta_i = dO_i . O_i,
//   dS = P o (dP - delta),  dQ = scale dS K,  dK = scale dS^T Q.
//
// One CTA owns one tile of 128 keys of one (b, h) and loops over all query tiles of 128:
//   ST  = K Q^T        (SS MMA, M=128 keys, N=128 queries)            TMEM [0,128)
//   dPT = V dO^T       (SS MMA)                                       TMEM [128,256)
//   softmax warps: PT = 2^(ST*c - lse2), dST = PT o (dPT - delta)  (c = scale log2 e,
//                  lse2 = lse log2 e); PT -> TMEM (bf16) for dV; dST -> shared memory (bf16,
//                  128B-swizzled [query half][key][64 queries]) which is at once the K-major
//                  A operand dS^T (for dK) and the MN-major A operand dS (for dQ)
//   dV += PT dO        (TS MMA, A = PT from TMEM, B = dO MN-major)     TMEM [320,384)
//   dK += dST Q        (SS MMA, A = dST K-major, B = Q MN-major)       TMEM [384,448)
//   dQ  = dS K         (SS MMA, A = dS MN-major, B = K MN-major)       TMEM [448,512)
//   dQ drain warps: TMEM -> registers -> swizzled smem -> TMA reduce-add (f32) into dq_acc.
// MMA issue order: ST_{i+1}, dPT_{i+1} as soon as the softmax warps have read ST_i, dPT_i
// ("s_loaded"), then dV_i, dK_i, dQ_i once P_i and dS_i are stored ("p_full"). The scores of
// the next tile are computed under softmax i and the gradients of tile i under softmax i+1;
// the softmax stores of tile i+1 wait on "p_free" (all MMAs of tile i done).
//
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4-19 softmax (4 warpgroups,
// warpgroup g owns query columns [32g, 32g+32) of each tile; thread = key row), 20-23 dQ drain.
#include <cuda_bf16.h>

#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

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

constexpr uint32_t kIdSS = idesc_bf16_f32(128, 128, false, false);   // ST, dPT
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
  uint64_t s_full, s_loaded, p_full, p_free, dq_full, dq_empty, dkv_done;
  uint32_t tmem_base;
};
constexpr size_t kBwdSmemBytes = sizeof(BwdSmem) + 1024;

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
template <bool kPad>
__global__ void __launch_bounds__(kBThreads, 1)
    bwd_bf16_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                    const __grid_constant__ CUtensorMap mdq, const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
      mbar_init(&sm.qdo_empty[i], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_loaded, 512);
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
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
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
          mbar_arrive_expect_tx(&sm.qdo_full[st], 2 * kTileBytes + 2 * kAugTileBytes);
          tma_load_4d(sm.q[st], &mq, &sm.qdo_full[st], 0, h, (i0 + i) * kTile, b, keep);
          tma_load_4d(sm.dout[st], &mdo, &sm.qdo_full[st], 0, h, (i0 + i) * kTile, b, keep);
          bulk_load(sm.aug[st], p.aug + (bh * NQ + i0 + i) * (2 * kAugTileBytes), 2 * kAugTileBytes,
                    &sm.qdo_full[st]);
        }
        __syncwarp();
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
      constexpr uint64_t kAugStep = (2 * kAugTileBytes) >> 4, kAugHalf = kAugTileBytes >> 4;
      auto scores = [&](int st) {  // ST' = K Q^T - lse/scale ; dPT' = V dO^T - delta
        const uint64_t q = dQ0 + st * kStep, o = dO0 + st * kStep, a = dA0 + st * kAugStep;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_ss(tm + kColST, dK + kk * 2, q + kk * 2, kIdSS, kk > 0);
        umma_ss(tm + kColST, dC, a, kIdSS, 1u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_ss(tm + kColDPT, dV + kk * 2, o + kk * 2, kIdSS, kk > 0);
        umma_ss(tm + kColDPT, dC, a + kAugHalf, kIdSS, 1u);
      };
      mbar_wait(&sm.kv_full, 0);
      mbar_wait(&sm.qdo_full[0], 0);
      tc_fence_after();
      if (elect_one()) {
        scores(0);
        umma_commit(&sm.s_full);
      }
      __syncwarp();
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
        if (more) {
          mbar_wait(&sm.qdo_full[(i + 1) % kBStages], ((i + 1) / kBStages) & 1);
          MPROBE(1)
          mbar_wait(&sm.s_loaded, i & 1);
          MPROBE(2)
          tc_fence_after();
          if (elect_one()) {
            scores((i + 1) % kBStages);
            umma_commit(&sm.s_full);
          }
          __syncwarp();
        }
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
    const bool keys_all_ok = __all_sync(0xffffffffu, key_ok);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    // dST row j, queries [32g, 32g+32) -> half g/2, 16-byte chunks (32g%64)/8 .. +3, swizzled
    uint8_t* ds_row = sm.ds[g >> 1] + j * 128;
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
      mbar_arrive(&sm.s_loaded);  // ST_i / dPT_i are in registers: the next scores may overwrite
      const bool diag = p.causal && i == 0;
      uint32_t pk[16], dk[16];
      auto tile = [&](auto masked) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float2 s2 = make_float2(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
          const float2 d2 = make_float2(__uint_as_float(dr[2 * u]), __uint_as_float(dr[2 * u + 1]));
          const float2 x = __fmul2_rn(s2, c2);  // c (s - lse/scale) = s c - lse log2 e
          // P (padded query rows: lse/scale = +-inf -> 0). MUFU for every pair: moving 2 or 4 of
          // the 16 pairs to the FMA-pipe polynomial measured +2.5 to +3.7 % (the longer
          // instruction stream costs more than the MUFU queue; profiles/r02_bwd_ab_poly.txt).
          float2 pr = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          if constexpr (decltype(masked)::value) {
            if (!key_ok) pr = make_float2(0.f, 0.f);
            if (diag) {  // causal diagonal tile: key j > query (32 g + 2 u + {0, 1}) is masked
              if (j > 32 * g + 2 * u) pr.x = 0.f;
              if (j > 32 * g + 2 * u + 1) pr.y = 0.f;
            }
          }
          const float2 ds = __fmul2_rn(pr, d2);  // P (dP - delta)
          pk[u] = pack_bf16x2(pr.x, pr.y);
          dk[u] = pack_bf16x2(ds.x, ds.y);
        }
      };
      // no per-element selects unless this warp's tile has padded keys or is a causal diagonal
      if (diag || !keys_all_ok) tile(std::true_type{});
      else tile(std::false_type{});
      TPROBE(2)
      if (i > 0) mbar_wait(&sm.p_free, (i - 1) & 1);  // tile i-1's MMAs no longer read P / dS
      TPROBE(3)
      tmem_st16(lane_base + kColP + g * 16, pk);
      TPROBE(5)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int phys = (chunk0 + cc) ^ (j & 7);
        *reinterpret_cast<uint4*>(ds_row + phys * 16) = make_uint4(dk[4 * cc], dk[4 * cc + 1], dk[4 * cc + 2], dk[4 * cc + 3]);
      }
      TPROBE(6)
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      TPROBE(7)
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
    const int rq = quarter * 32 + lane;  // query row within the tile (TMEM lane)
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
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// delta_i = dO_i . O_i, lse2 = lse log2 e, both padded to a multiple of 128 rows
// per (b,h) (pads: delta 0, lse2 +inf so padded query rows get P = 0); dq_acc = 0 when given.
// With aug (fused kernel): the B side of the score MMAs' K-extension, per (b,h, query tile) an
// 8 KiB block [lse tile][delta tile], each 128 rows x 16 bf16 in no-swizzle K-major core matrices
// (row r, K column k at (r/8)*256 + (k/8)*128 + (r%8)*16 + (k%8)*2): row = [hi, lo, 0 ...] with
// hi + lo = lse/scale (resp. delta) to ~2^-16 relative; padded rows: lse/scale = +-inf (so that
// c ST' = -inf, P = 0) and delta = 0. 8 threads per row, 16-byte loads.
__device__ __forceinline__ uint32_t bf16_hi_lo(float x) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(x);
  const float rest = isinf(x) ? 0.f : x - __bfloat162float(hi);
  const __nv_bfloat16 lo = __float2bfloat16_rn(rest);
  return (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(lo) << 16);
}

__global__ void bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ dout,
                                      const float* __restrict__ lse, float* __restrict__ delta,
                                      float* __restrict__ lse2, float* __restrict__ dq_acc, uint8_t* __restrict__ aug,
                                      float scale, int B, int H, int n_q, int nq_pad, int d) {
  const int64_t rows = (int64_t)B * H * nq_pad;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int part = threadIdx.x & 7;
  if (r >= rows) return;
  const int64_t bh = r / nq_pad;
  const int q = (int)(r % nq_pad);
  const int64_t b = bh / H, h = bh % H;
  float acc = 0.f;
  if (q < n_q) {
    for (int c = 0; c < d; c += 64) {  // d = 64 or 128: 8 (16) elements per thread
      const size_t off = (((size_t)b * n_q + q) * H + h) * d + c + part * 8;
      const uint4 o = *reinterpret_cast<const uint4*>(out + off);
      const uint4 dd = *reinterpret_cast<const uint4*>(dout + off);
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w}, dw[4] = {dd.x, dd.y, dd.z, dd.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc = fmaf(__uint_as_float(ow[u] << 16), __uint_as_float(dw[u] << 16), acc);
        acc = fmaf(__uint_as_float(ow[u] & 0xFFFF0000u), __uint_as_float(dw[u] & 0xFFFF0000u), acc);
      }
      if (dq_acc) {
        float4* z = reinterpret_cast<float4*>(dq_acc + off);
        z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  const float l = (q < n_q) ? lse[bh * n_q + q] : INFINITY;
  if (part == 0) {
    delta[r] = acc;
    lse2[r] = l * 1.4426950408889634f;
  }
  if (aug && part < 4) {  // parts 0,1: lse tile (K core 0, 1); parts 2,3: delta tile
    const int tile = q / kTile, rr = q % kTile;
    uint8_t* blk = aug + (bh * (nq_pad / kTile) + tile) * (2 * kAugTileBytes) + (part >> 1) * kAugTileBytes;
    const int kc = part & 1;
    uint32_t w0 = 0u;
    if (kc == 0) {
      const float x = (part < 2) ? ((q < n_q) ? l / scale : (scale > 0.f ? INFINITY : -INFINITY)) : acc;
      w0 = bf16_hi_lo(x);
    }
    *reinterpret_cast<uint4*>(blk + (rr >> 3) * 256 + kc * 128 + (rr & 7) * 16) = make_uint4(w0, 0u, 0u, 0u);
  }
}

// dq = bf16(scale * dq_acc)
__global__ void dq_convert_kernel(const float4* __restrict__ acc, uint2* __restrict__ dq, int64_t n4, float scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = acc[i];
    dq[i] = make_uint2(pack_bf16x2(a.x * scale, a.y * scale), pack_bf16x2(a.z * scale, a.w * scale));
  }
}

}  // namespace

cudaError_t launch_bwd_preprocess(const void* out, const void* dout, const float* lse, float* delta, float* lse2,
                                  float* dq_acc, uint8_t* aug, float scale, int B, int H, int n_q, int d,
                                  cudaStream_t s) {
  const int nq_pad = (n_q + kTile - 1) / kTile * kTile;
  const int64_t threads = (int64_t)B * H * nq_pad * 8;
  bwd_preprocess_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), lse, delta, lse2, dq_acc, aug,
      scale, B, H, n_q, nq_pad, d);
  return cudaGetLastError();
}

cudaError_t launch_bwd_bf16(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                            const CUtensorMap& mdo, const CUtensorMap& mdq, cudaStream_t s) {
  const cudaError_t attr = p.kv_lens ? ensure_smem_attr<bwd_bf16_kernel<true>>((int)kBwdSmemBytes)
                                     : ensure_smem_attr<bwd_bf16_kernel<false>>((int)kBwdSmemBytes);
  if (attr != cudaSuccess) return attr;
  const dim3 grid = p.causal ? dim3(p.num_k_blocks * p.H * p.B) : dim3(p.num_k_blocks, p.H, p.B);
  if (p.kv_lens)
    bwd_bf16_kernel<true><<<grid, kBThreads, kBwdSmemBytes, s>>>(mq, mk, mv, mdo, mdq, p);
  else
    bwd_bf16_kernel<false><<<grid, kBThreads, kBwdSmemBytes, s>>>(mq, mk, mv, mdo, mdq, p);
  return cudaGetLastError();
}

#ifdef MEA_DEBUG_HANG
extern "C" __attribute__((visibility("default"))) int mea_debug_hang_read(unsigned int* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_mea_hang, n * sizeof(unsigned int));
}
extern "C" __attribute__((visibility("default"))) int mea_debug_smem_offsets(size_t* out) {
  out[0] = offsetof(BwdSmem, kv_full);
  out[1] = offsetof(BwdSmem, s_full);
  out[2] = sizeof(BwdSmem);
  return 0;
}
#endif

cudaError_t launch_dq_convert(const float* dq_acc, void* dq, int64_t numel, float scale, cudaStream_t s) {
  const int64_t n4 = numel / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  dq_convert_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(dq_acc),
                                                    reinterpret_cast<uint2*>(dq), n4, scale);
  return cudaGetLastError();
}

}  // namespace mea
