// bwd128_sm100a.cu — fused backward at head dimension d = 128, the
// same recomputation as the d = 64 fused kernel (bwd_sm100a.cu, the plain
// softmax VJP of SPEC.md:122 with lse fixed):
//   P = exp(scale q k^T - lse),  dV = P^T dO,  dP = dO V^T,  delta_i = dO_i . O_i,
//   dS = P o (dP - delta),  dQ = scale dS K,  dK = scale dS^T Q,
// in ONE kernel: dQ is reduced across key tiles in an f32 accumulator (TMA reduce-add), so the
// two recomputed GEMMs of the deterministic two-kernel path (S and dP again for dQ) are gone.
//
// One CTA owns 128 keys of one (b, h) and loops over query tiles of 64 rows (at d = 128 the
// accumulators dV, dK take 128 TMEM columns each). TMEM (512 columns, lanes = keys unless noted):
//   ST  [0, 64)      = K Q^T          SS, M = 128 keys, N = 64 queries, K = 128
//   dPT [64, 128)    = V dO^T         SS
//   P   [128, 160)   bf16 pairs       written by the softmax warps
//   dS  [160, 192)   bf16 pairs       written by the softmax warps (A of dK)
//   dV  [192, 320)  += P^T dO         TS (B = dO MN-major, N = 128 over two SW128 atoms)
//   dK  [320, 448)  += dS^T Q         TS
//   dQT [448, 512)   = K^T dS^T       SS, lanes = d (M = 128), N = 64 queries, K = 128 keys:
//                    A = the K tile read MN-major (d contiguous, two atoms LBO apart), B = dS in
//                    shared memory ([key][64 queries] bf16, SW128) read MN-major.
// dS^T goes to TMEM (for dK, no shared-memory operand read) and once to shared memory (for dQ).
// dQ drain warps (lane = d): TMEM -> registers -> swizzled [query][32 d] f32 staging boxes ->
// TMA reduce-add into dq_acc; dq_convert applies the scale and rounds to bf16.
// lse2 and delta come per query column from shared memory (bulk-loaded with Q / dO).
// Schedule as bwd_sm100a.cu: ST_{i+1}, dPT_{i+1} once the softmax warps have read tile i
// ("s_loaded"); dV_i, dK_i, dQT_i once P_i, dS_i are stored ("p_full"); the stores of tile i+1
// wait on "p_free" (all MMAs of tile i done).
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4-11 softmax (two column
// halves x four lane quarters; thread = key row, 32 query columns), 12-15 dQ drain.
#include <cuda_bf16.h>

#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

constexpr int D = 128;
constexpr int QT = 64;                  // queries per tile
constexpr int KT = 128;                 // keys per CTA
constexpr int kStages = 3;              // Q / dO ring
constexpr int kThreads = 512;
constexpr int kKAtom = KT * 128;        // one SW128 atom of the K / V tile: 128 rows x 64 d
constexpr int kQAtom = QT * 128;        // one atom of a Q / dO tile: 64 rows x 64 d
constexpr int kKTileBytes = 2 * kKAtom, kQTileBytes = 2 * kQAtom;
constexpr int kDsBytes = KT * QT * 2;   // [128 keys][64 queries] bf16
constexpr int kStageBox = QT * 128;     // one dQ staging box: 64 queries x 32 d f32
constexpr uint32_t kColST = 0, kColDPT = 64, kColP = 128, kColDS = 160, kColDV = 192, kColDK = 320, kColDQ = 448;
constexpr uint32_t kBarDq = 1;

constexpr uint32_t kIdSS = idesc_bf16_f32(128, QT, false, false);  // ST, dPT
constexpr uint32_t kIdTS = idesc_bf16_f32(128, D, false, true);    // dV, dK: A TMEM, B MN-major
constexpr uint32_t kIdDQ = idesc_bf16_f32(128, QT, true, true);    // dQT: A = K MN-major, B = dS MN-major

struct Smem {
  uint8_t k[kKTileBytes];
  uint8_t v[kKTileBytes];
  uint8_t q[kStages][kQTileBytes];
  uint8_t dout[kStages][kQTileBytes];
  uint8_t ds[kDsBytes];
  uint8_t dq_stage[4][kStageBox];
  float lse2[kStages][QT];
  float delta[kStages][QT];
  uint64_t kv_full, qdo_full[kStages], qdo_empty[kStages];
  uint64_t s_full, s_loaded, p_full, p_free, dq_full, dq_empty, dkv_done;
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <bool kPad>
__global__ void __launch_bounds__(kThreads, 1)
    bwd128_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                  const __grid_constant__ CUtensorMap mdq, const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblk = p.causal ? (int)(blockIdx.x / (p.H * p.B)) : (int)blockIdx.x;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int k0 = kblk * KT;
  const int NQ = (p.n_q + QT - 1) / QT;
  // causal (n_q == n_k): query tiles before k0 see none of this CTA's keys
  const int i0 = p.causal ? k0 / QT : 0;
  const int NT = NQ - i0;
  const int nq_pad = (p.n_q + kTileM - 1) / kTileM * kTileM;  // bwd_preprocess's row padding
  const size_t bh = (size_t)b * p.H + h;

  if (threadIdx.x == 0) {
    mbar_init(&sm.kv_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.qdo_full[i], 1);
      mbar_init(&sm.qdo_empty[i], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_loaded, 256);
    mbar_init(&sm.p_full, 256);
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    const uint64_t keep = policy_evict_last();
    if (elect_one()) {
      mbar_arrive_expect_tx(&sm.kv_full, 2 * kKTileBytes);
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        tma_load_4d(sm.k + a * kKAtom, &mk, &sm.kv_full, 64 * a, h, k0, b, keep);
        tma_load_4d(sm.v + a * kKAtom, &mv, &sm.kv_full, 64 * a, h, k0, b, keep);
      }
    }
    __syncwarp();
    for (int i = 0; i < NT; ++i) {
      const int st = i % kStages, n = i / kStages;
      if (i >= kStages) mbar_wait(&sm.qdo_empty[st], (n - 1) & 1);
      if (elect_one()) {
        const int qrow = (i0 + i) * QT;
        mbar_arrive_expect_tx(&sm.qdo_full[st], 2 * kQTileBytes + 2 * QT * 4);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          tma_load_4d(sm.q[st] + a * kQAtom, &mq, &sm.qdo_full[st], 64 * a, h, qrow, b, keep);
          tma_load_4d(sm.dout[st] + a * kQAtom, &mdo, &sm.qdo_full[st], 64 * a, h, qrow, b, keep);
        }
        bulk_load(sm.lse2[st], p.lse2 + bh * nq_pad + qrow, QT * 4, &sm.qdo_full[st]);
        bulk_load(sm.delta[st], p.delta + bh * nq_pad + qrow, QT * 4, &sm.qdo_full[st]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const uint64_t dK = shfl0_u64(sdesc_sw128(smem_u32(sm.k), 16, 1024));          // K-major A of ST
    const uint64_t dV = shfl0_u64(sdesc_sw128(smem_u32(sm.v), 16, 1024));
    const uint64_t dKm = shfl0_u64(sdesc_sw128(smem_u32(sm.k), kKAtom, 1024));     // MN-major A of dQT
    const uint64_t dQ0 = shfl0_u64(sdesc_sw128(smem_u32(sm.q[0]), 16, 1024));
    const uint64_t dO0 = shfl0_u64(sdesc_sw128(smem_u32(sm.dout[0]), 16, 1024));
    const uint64_t dQm0 = shfl0_u64(sdesc_sw128(smem_u32(sm.q[0]), kQAtom, 1024));   // MN-major B of dK
    const uint64_t dOm0 = shfl0_u64(sdesc_sw128(smem_u32(sm.dout[0]), kQAtom, 1024));
    const uint64_t dSm = shfl0_u64(sdesc_sw128(smem_u32(sm.ds), 16, 1024));         // MN-major B of dQT
    constexpr uint64_t kStep = kQTileBytes >> 4, kKAt = kKAtom >> 4, kQAt = kQAtom >> 4;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    auto scores = [&](int st) {  // ST = K Q^T ; dPT = V dO^T  (K = 128 = two atoms of 4 steps)
      const uint64_t q = dQ0 + st * kStep, o = dO0 + st * kStep;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_ss(tm + kColST, dK + (kk >> 2) * kKAt + (kk & 3) * 2, q + (kk >> 2) * kQAt + (kk & 3) * 2, kIdSS, kk > 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_ss(tm + kColDPT, dV + (kk >> 2) * kKAt + (kk & 3) * 2, o + (kk >> 2) * kQAt + (kk & 3) * 2, kIdSS, kk > 0);
    };
    mbar_wait(&sm.kv_full, 0);
    mbar_wait(&sm.qdo_full[0], 0);
    tc_fence_after();
    if (elect_one()) {
      scores(0);
      umma_commit(&sm.s_full);
    }
    __syncwarp();
    for (int i = 0; i < NT; ++i) {
      const int st = i % kStages;
      const bool more = i + 1 < NT;
      if (more) {
        mbar_wait(&sm.qdo_full[(i + 1) % kStages], ((i + 1) / kStages) & 1);
        mbar_wait(&sm.s_loaded, i & 1);
        tc_fence_after();
        if (elect_one()) {
          scores((i + 1) % kStages);
          umma_commit(&sm.s_full);
        }
        __syncwarp();
      }
      mbar_wait(&sm.p_full, i & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t q = dQm0 + st * kStep, o = dOm0 + st * kStep;
        // dV += P^T dO ; dK += dS^T Q : K = 64 queries in steps of 16 (A: 8 TMEM columns per
        // step; B: 16 rows of 128 B, MN-major over two atoms)
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)
          umma_ts(tm + kColDV, tm + kColP + kk * 8, o + kk * 128, kIdTS, (i > 0 || kk > 0));
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)
          umma_ts(tm + kColDK, tm + kColDS + kk * 8, q + kk * 128, kIdTS, (i > 0 || kk > 0));
      }
      __syncwarp();
      if (i > 0) mbar_wait(&sm.dq_empty, (i - 1) & 1);  // dQT of tile i-1 drained from TMEM
      tc_fence_after();
      if (elect_one()) {
        // dQT = K^T dS^T : K = 128 keys in steps of 16 (16 key rows = 2048 B in both operands)
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk) umma_ss(tm + kColDQ, dKm + kk * 128, dSm + kk * 128, kIdDQ, kk > 0);
        umma_commit(&sm.dq_full);
        umma_commit(&sm.p_free);
        umma_commit(&sm.qdo_empty[st]);
        if (!more) umma_commit(&sm.dkv_done);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------------ softmax warps
    const int g = (warp - 4) >> 2;           // query columns [32 g, 32 g + 32)
    const int quarter = warp & 3;
    const int j = quarter * 32 + lane;       // key row within the tile (TMEM lane)
    const bool key_ok = k0 + j < (kPad ? keys_of(p.kv_lens, b, p.n_k) : p.n_k);
    const bool keys_all_ok = __all_sync(0xffffffffu, key_ok);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    uint8_t* ds_row = sm.ds + j * 128;       // dS row j: 64 queries, 16-byte chunks 4 g .. 4 g + 3
    for (int i = 0; i < NT; ++i) {
      const int st = i % kStages;
      mbar_wait(&sm.s_full, i & 1);
      tc_fence_after();
      uint32_t sr[32], dr[32];
      tmem_ld32(lane_base + kColST + g * 32, sr);
      tmem_ld32(lane_base + kColDPT + g * 32, dr);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&sm.s_loaded);  // ST_i / dPT_i are in registers: the next scores may overwrite
      const float* l2 = sm.lse2[st] + g * 32;
      const float* dl = sm.delta[st] + g * 32;
      const int qbase = (i0 + i) * QT + 32 * g;                     // this thread's first query column
      const bool overlap = p.causal && (i0 + i) * QT < k0 + KT;     // tile crosses the diagonal
      uint32_t pk[16], dk[16];
      auto tile = [&](auto masked) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float2 s2 = make_float2(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
          const float2 d2 = make_float2(__uint_as_float(dr[2 * u]), __uint_as_float(dr[2 * u + 1]));
          const float2 lq = *reinterpret_cast<const float2*>(l2 + 2 * u);
          const float2 de = *reinterpret_cast<const float2*>(dl + 2 * u);
          const float2 x = __ffma2_rn(s2, c2, make_float2(-lq.x, -lq.y));  // s c - lse2
          float2 pr = make_float2(ex2_approx(x.x), ex2_approx(x.y));        // P (padded rows: lse2 = +inf -> 0)
          if constexpr (decltype(masked)::value) {
            if (!key_ok) pr = make_float2(0.f, 0.f);
            if (overlap) {  // causal: key k0 + j > query qbase + 2u (+1) is masked
              if (k0 + j > qbase + 2 * u) pr.x = 0.f;
              if (k0 + j > qbase + 2 * u + 1) pr.y = 0.f;
            }
          }
          const float2 ds = __fmul2_rn(pr, __fadd2_rn(d2, make_float2(-de.x, -de.y)));  // P (dP - delta)
          pk[u] = pack_bf16x2(pr.x, pr.y);
          dk[u] = pack_bf16x2(ds.x, ds.y);
        }
      };
      // no per-element selects unless this warp has padded keys or the tile crosses the diagonal
      if (overlap || !keys_all_ok) tile(std::true_type{});
      else tile(std::false_type{});
      if (i > 0) mbar_wait(&sm.p_free, (i - 1) & 1);  // tile i-1's MMAs no longer read P / dS
      tc_fence_after();
      tmem_st16(lane_base + kColP + g * 16, pk);
      tmem_st16(lane_base + kColDS + g * 16, dk);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int phys = (4 * g + cc) ^ (j & 7);
        *reinterpret_cast<uint4*>(ds_row + phys * 16) = make_uint4(dk[4 * cc], dk[4 * cc + 1], dk[4 * cc + 2], dk[4 * cc + 3]);
      }
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
    }
    // ------------------------------------------------------------------ dV (g = 0), dK (g = 1)
    mbar_wait(&sm.dkv_done, 0);
    tc_fence_after();
    const uint32_t col = g == 0 ? kColDV : kColDK;
    const float sc = g == 0 ? 1.f : p.scale;
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g == 0 ? p.dv : p.dk) + (((size_t)b * p.n_k + k0 + j) * p.H + h) * D;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t r[64];
      tmem_ld32(lane_base + col + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld32(lane_base + col + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld_wait();
      if (k0 + j < p.n_k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(r[8 * u + 0]) * sc, __uint_as_float(r[8 * u + 1]) * sc);
          w.y = pack_bf16x2(__uint_as_float(r[8 * u + 2]) * sc, __uint_as_float(r[8 * u + 3]) * sc);
          w.z = pack_bf16x2(__uint_as_float(r[8 * u + 4]) * sc, __uint_as_float(r[8 * u + 5]) * sc);
          w.w = pack_bf16x2(__uint_as_float(r[8 * u + 6]) * sc, __uint_as_float(r[8 * u + 7]) * sc);
          reinterpret_cast<uint4*>(dst + half * 64)[u] = w;
        }
      }
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------------ dQ drain (lane = d)
    const int quarter = warp & 3;            // = the staging box: d in [32 quarter, 32 quarter + 32)
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    uint8_t* box = sm.dq_stage[quarter];
    for (int i = 0; i < NT; ++i) {
      mbar_wait(&sm.dq_full, i & 1);
      tc_fence_after();
      uint32_t r[64];
      tmem_ld32(lane_base + kColDQ, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld32(lane_base + kColDQ + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&sm.dq_empty);  // the next tile's dQT MMA may overwrite the columns
      // the TMA reduce of tile i-1 must have finished reading the staging boxes
      if (warp == 12 && lane == 0) bulk_wait_group_read<0>();
      named_bar_sync(kBarDq, 128);
      // box row = query (128 B = 32 f32 of d), 16-byte chunk (lane / 4) swizzled by the row
#pragma unroll
      for (int qq = 0; qq < QT; ++qq)
        *reinterpret_cast<uint32_t*>(box + qq * 128 + ((((lane >> 2) ^ (qq & 7))) << 4) + (lane & 3) * 4) = r[qq];
      fence_proxy_async_smem();
      named_bar_sync(kBarDq, 128);
      if (warp == 12 && lane == 0) {
#pragma unroll
        for (int bx = 0; bx < 4; ++bx) tma_reduce_add_4d(&mdq, sm.dq_stage[bx], 32 * bx, h, (i0 + i) * QT, b);
        bulk_commit_group();
      }
    }
    if (warp == 12 && lane == 0) bulk_wait_group0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

size_t bwd128_smem_bytes() { return kSmemBytes; }

// mq / mdo: boxes {64, 1, 64, 1} bf16; mk / mv: {64, 1, 128, 1} bf16; mdq: {32, 1, 64, 1} f32.
cudaError_t launch_bwd128(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                          const CUtensorMap& mdo, const CUtensorMap& mdq, cudaStream_t s) {
  const dim3 grid = p.causal ? dim3(p.num_k_blocks * p.H * p.B) : dim3(p.num_k_blocks, p.H, p.B);
  if (p.kv_lens) {
    const cudaError_t attr = ensure_smem_attr<bwd128_kernel<true>>((int)kSmemBytes);
    if (attr != cudaSuccess) return attr;
    bwd128_kernel<true><<<grid, kThreads, kSmemBytes, s>>>(mq, mk, mv, mdo, mdq, p);
  } else {
    const cudaError_t attr = ensure_smem_attr<bwd128_kernel<false>>((int)kSmemBytes);
    if (attr != cudaSuccess) return attr;
    bwd128_kernel<false><<<grid, kThreads, kSmemBytes, s>>>(mq, mk, mv, mdo, mdq, p);
  }
  return cudaGetLastError();
}

}  // namespace mea
