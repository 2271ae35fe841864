// bwd_det_sm100a.cu — dK and dV for the deterministic backward (mea_attention_bwd_deterministic),
// recomputing every tile of scores from the saved per-row log-sum-exp instead of storing them
// (the paper's checkpointed differentiation: "recomputed during
// backpropagation"). The max carries no gradient (stop_gradient): with lse fixed
// the derivative is the plain softmax VJP:
//   P = exp(scale q k^T - lse),  dV = P^T dO,  dP = dO V^T,  delta_i = dO_i . O_i,
//   dS = P o (dP - delta),  dK = scale dS^T Q     (dQ = scale dS K: bwd_dq_sm100a.cu).
//
// One CTA owns one tile of 128 keys of one (b, h) and loops over all query tiles of 128:
//   ST  = K Q^T      (SS MMA, M=128 keys, N=128 queries)        TMEM [0,128)
//   dPT = V dO^T     (SS MMA)                                   TMEM [128,256)
//   softmax warps: PT = 2^(ST*c - lse2), dST = PT o (dPT - delta)  (c = scale log2 e,
//                  lse2 = lse log2 e, both per query column) -> bf16 pairs into TMEM
//   dV += PT dO      (TS MMA: A = PT from TMEM [256,320), B = dO MN-major)  TMEM [384,448)
//   dK += dST Q      (TS MMA: A = dST from TMEM [320,384), B = Q MN-major)  TMEM [448,512)
// Every MMA reads at most one 16 KiB operand tile from shared memory per 256 cycles. With dQ in
// its own kernel (bwd_dq_sm100a.cu: 2 extra recomputed GEMMs) there is no cross-CTA dQ
// reduction: the result is bitwise reproducible and the workspace is only delta and lse
// (~2 MiB at configs[3] instead of the fused path's 66 MiB). Measured at configs[3]: 1.80 ms
// here + 1.73 ms for dQ, against 3.09 ms for the fused (SMEM-bandwidth-bound) kernel.
// Schedule: ST_{i+1}, dPT_{i+1} issue once the softmax warps have read tile i out of TMEM
// ("s_loaded"); dV_i, dK_i once PT_i, dST_i are stored ("p_full"); the softmax stores of tile
// i+1 wait on "p_free" (dV_i, dK_i done).
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4-19 softmax (4 warpgroups,
// warpgroup g owns query columns [32g, 32g+32) of each tile; thread = key row).
#include <cuda_bf16.h>

#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

constexpr int kBStages = 3;  // Q/dO ring
constexpr int kTile = 128;     // keys per CTA
constexpr int kBThreads = 640;
// D = 64 (kHeadDim) or 128. Query tiles are QT = 128 rows at D = 64 and 64 rows at D = 128 (so
// that Sᵀ, dPᵀ, Pᵀ, dSᵀ, dV and dK fit the 512 TMEM columns: 2 QT + QT + 2 D <= 512). A tile of
// R rows and D columns is D/64 SW128 atoms of R x 128 B.
template <int D> struct DkvCfg {
  static constexpr int QT = D == 64 ? 128 : 64;
  static constexpr int kAtoms = D / 64;
  static constexpr int kKTileBytes = 128 * D * 2, kQTileBytes = QT * D * 2;
  static constexpr int kKAtom = 128 * 128, kQAtom = QT * 128;
  static constexpr uint32_t kColST = 0, kColDPT = QT, kColP = 2 * QT, kColDS = 2 * QT + QT / 2,
                            kColDV = 3 * QT, kColDK = 3 * QT + D;
  // D = 128: the K tile also sits in TMEM (bf16 pairs, D/2 columns) as the A operand of a TS
  // Sᵀ MMA, so Sᵀ = K Qᵀ reads only Q from shared memory (SS at N = 64 is SMEM-bound, 65 %)
  static constexpr bool kKInTmem = D == 128;
  static constexpr uint32_t kColKA = 3 * QT + 2 * D;
};
// setmaxnreg budgets. Measured on B200: setmaxnreg.inc only redistributes the registers the
// CTA was launched with (640 threads x 96 = 480 per lane slot of each SM sub-partition, which
// holds one control and four softmax warps); a larger total blocks forever. 64 + 4*104 = 480.
constexpr int kBCtrlRegs = 64, kBSoftRegs = 104;
template <int D>
struct BwdSmem {
  using C = DkvCfg<D>;
  uint8_t k[C::kKTileBytes];
  uint8_t v[C::kKTileBytes];
  uint8_t q[kBStages][C::kQTileBytes];
  uint8_t dout[kBStages][C::kQTileBytes];
  float lse2[kBStages][C::QT];
  float delta[kBStages][C::QT];
  uint64_t kv_full, qdo_full[kBStages], qdo_empty[kBStages];
  uint64_t s_full, s_loaded, p_full, p_free, dkv_done, ka_full;
  uint32_t tmem_base;
};
template <int D> constexpr size_t dkv_smem_bytes() { return sizeof(BwdSmem<D>) + 1024; }

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

template <int D>
__global__ void __launch_bounds__(kBThreads, 1)
    bwd_dkdv_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                    const BwdParams p) {
  using C = DkvCfg<D>;
  constexpr int QT = C::QT, kAtoms = C::kAtoms;
  constexpr uint32_t kColST = C::kColST, kColDPT = C::kColDPT, kColP = C::kColP, kColDS = C::kColDS,
                     kColDV = C::kColDV, kColDK = C::kColDK;
  constexpr uint32_t kIdSS = idesc_bf16_f32(128, QT, false, false);  // ST, dPT: N = QT queries
  constexpr uint32_t kIdTS = idesc_bf16_f32(128, D, false, true);    // dV, dK: A from TMEM, B MN-major
  constexpr int NC = QT / 4;                                          // query columns per softmax thread
  extern __shared__ uint8_t smem_raw[];
  BwdSmem<D>& sm = *reinterpret_cast<BwdSmem<D>*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: 1-D grid, key block 0 (the most query tiles) first across all (b, h)
  const int kblk = p.causal ? (int)(blockIdx.x / (p.H * p.B)) : (int)blockIdx.x;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int k0 = kblk * kTile;
  const int NQ = (p.n_q + QT - 1) / QT;
  // causal (n_q == n_k): query tiles before this key tile see none of its keys; iteration i
  // (stages, barrier phases) handles query tile i0 + i
  const int i0 = p.causal ? k0 / QT : 0;
  const int NT = NQ - i0;
  const int nq_pad = (p.n_q + kTileM - 1) / kTileM * kTileM;  // bwd_preprocess's row padding
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
    mbar_init(&sm.dkv_done, 1);
    mbar_init(&sm.ka_full, 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mk);
    tma_prefetch_desc(&mv);
    tma_prefetch_desc(&mdo);
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
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
        mbar_arrive_expect_tx(&sm.kv_full, 2 * C::kKTileBytes);
#pragma unroll
        for (int a = 0; a < kAtoms; ++a) {
          tma_load_4d(sm.k + a * C::kKAtom, &mk, &sm.kv_full, 64 * a, h, k0, b, keep);
          tma_load_4d(sm.v + a * C::kKAtom, &mv, &sm.kv_full, 64 * a, h, k0, b, keep);
        }
      }
      __syncwarp();
      for (int i = 0; i < NT; ++i) {
        const int st = i % kBStages, n = i / kBStages;
        if (i >= kBStages) mbar_wait(&sm.qdo_empty[st], (n - 1) & 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm.qdo_full[st], 2 * C::kQTileBytes + 2 * QT * 4);
#pragma unroll
          for (int a = 0; a < kAtoms; ++a) {
            tma_load_4d(sm.q[st] + a * C::kQAtom, &mq, &sm.qdo_full[st], 64 * a, h, (i0 + i) * QT, b, keep);
            tma_load_4d(sm.dout[st] + a * C::kQAtom, &mdo, &sm.qdo_full[st], 64 * a, h, (i0 + i) * QT, b, keep);
          }
          bulk_load(sm.lse2[st], p.lse2 + bh * nq_pad + (i0 + i) * QT, QT * 4, &sm.qdo_full[st]);
          bulk_load(sm.delta[st], p.delta + bh * nq_pad + (i0 + i) * QT, QT * 4, &sm.qdo_full[st]);
        }
        __syncwarp();
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------------- MMA issuer
      const uint64_t dK = shfl0_u64(sdesc_sw128(smem_u32(sm.k), 16, 1024));
      const uint64_t dV = shfl0_u64(sdesc_sw128(smem_u32(sm.v), 16, 1024));
      const uint64_t dQ0 = shfl0_u64(sdesc_sw128(smem_u32(sm.q[0]), 16, 1024));
      const uint64_t dO0 = shfl0_u64(sdesc_sw128(smem_u32(sm.dout[0]), 16, 1024));
      // Q / dO as the MN-major B of dV, dK: N = D over kAtoms atoms C::kQAtom bytes apart (LBO)
      const uint64_t dQm0 = shfl0_u64(sdesc_sw128(smem_u32(sm.q[0]), C::kQAtom, 1024));
      const uint64_t dOm0 = shfl0_u64(sdesc_sw128(smem_u32(sm.dout[0]), C::kQAtom, 1024));
      constexpr uint64_t kStep = C::kQTileBytes >> 4, kKAt = C::kKAtom >> 4, kQAt = C::kQAtom >> 4;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      auto scores = [&](int st) {  // ST = K Q^T ; dPT = V dO^T  (K = D in steps of 16)
        const uint64_t q = dQ0 + st * kStep, o = dO0 + st * kStep;
#pragma unroll
        for (int kk = 0; kk < 4 * kAtoms; ++kk) {
          if constexpr (C::kKInTmem)
            umma_ts(tm + kColST, tm + C::kColKA + kk * 8, q + (kk >> 2) * kQAt + (kk & 3) * 2, kIdSS, kk > 0);
          else
            umma_ss(tm + kColST, dK + (kk >> 2) * kKAt + (kk & 3) * 2, q + (kk >> 2) * kQAt + (kk & 3) * 2, kIdSS, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 4 * kAtoms; ++kk)
          umma_ss(tm + kColDPT, dV + (kk >> 2) * kKAt + (kk & 3) * 2, o + (kk >> 2) * kQAt + (kk & 3) * 2, kIdSS, kk > 0);
      };
      mbar_wait(&sm.kv_full, 0);
      if constexpr (C::kKInTmem) mbar_wait(&sm.ka_full, 0);
      mbar_wait(&sm.qdo_full[0], 0);
      tc_fence_after();
      if (elect_one()) {
        scores(0);
        umma_commit(&sm.s_full);
      }
      __syncwarp();
      for (int i = 0; i < NT; ++i) {
        const int st = i % kBStages;
        const bool more = i + 1 < NT;
        if (more) {
          mbar_wait(&sm.qdo_full[(i + 1) % kBStages], ((i + 1) / kBStages) & 1);
          mbar_wait(&sm.s_loaded, i & 1);
          tc_fence_after();
          if (elect_one()) {
            scores((i + 1) % kBStages);
            umma_commit(&sm.s_full);
          }
          __syncwarp();
        }
        mbar_wait(&sm.p_full, i & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t q = dQm0 + st * kStep, o = dOm0 + st * kStep;
          // dV += PT dO ; dK += dST Q : K = QT queries in steps of 16 (A: 8 TMEM columns per
          // step; B: 16 rows of 128 B, MN-major)
#pragma unroll
          for (int kk = 0; kk < QT / 16; ++kk) umma_ts(tm + kColDV, tm + kColP + kk * 8, o + kk * 128, kIdTS, (i > 0 || kk > 0));
#pragma unroll
          for (int kk = 0; kk < QT / 16; ++kk) umma_ts(tm + kColDK, tm + kColDS + kk * 8, q + kk * 128, kIdTS, (i > 0 || kk > 0));
          umma_commit(&sm.p_free);
          umma_commit(&sm.qdo_empty[st]);
          if (!more) umma_commit(&sm.dkv_done);
        }
        __syncwarp();
      }
    }
  } else {
    setmaxnreg_inc<kBSoftRegs>();
    // ------------------------------------------------------------------ softmax warpgroups
    const int g = (warp - 4) >> 2;           // query columns [NC g, NC g + NC)
    const int quarter = warp & 3;
    const int j = quarter * 32 + lane;       // key row within the tile (TMEM lane)
    const bool key_ok = k0 + j < keys_of(p.kv_lens, b, p.n_k);  // key padding: P = 0 -> dK = dV = 0
    const bool keys_all_ok = __all_sync(0xffffffffu, key_ok);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    if constexpr (C::kKInTmem) {
      if (g == 0) {  // K row j (SW128 smem, D/64 atoms) -> TMEM lane j, columns kColKA + [0, D/2)
        mbar_wait(&sm.kv_full, 0);
#pragma unroll
        for (int a = 0; a < kAtoms; ++a) {
          uint32_t r[32];
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const uint4 w = *reinterpret_cast<const uint4*>(sm.k + a * C::kKAtom + j * 128 + ((cc ^ (j & 7)) * 16));
            r[4 * cc] = w.x; r[4 * cc + 1] = w.y; r[4 * cc + 2] = w.z; r[4 * cc + 3] = w.w;
          }
          tmem_st32(lane_base + C::kColKA + a * 32, r);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&sm.ka_full);
      }
    }
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
      uint32_t sr[NC], dr[NC];
      if constexpr (NC == 32) {
        tmem_ld32(lane_base + kColST + g * NC, sr);
        tmem_ld32(lane_base + kColDPT + g * NC, dr);
      } else {
        tmem_ld16(lane_base + kColST + g * NC, sr);
        tmem_ld16(lane_base + kColDPT + g * NC, dr);
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&sm.s_loaded);  // ST_i / dPT_i are in registers: the next scores may overwrite
      const float* l2 = sm.lse2[st] + g * NC;
      const float* dl = sm.delta[st] + g * NC;
      const int qbase = (i0 + i) * QT + NC * g;                     // first query column of this thread
      const bool overlap = p.causal && (i0 + i) * QT < k0 + kTile;  // tile crosses the diagonal
      uint32_t pk[NC / 2], dk[NC / 2];
      auto tile = [&](auto masked) {
#pragma unroll
        for (int u = 0; u < NC / 2; ++u) {
          const float2 s2 = make_float2(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
          const float2 d2 = make_float2(__uint_as_float(dr[2 * u]), __uint_as_float(dr[2 * u + 1]));
          const float2 lq = *reinterpret_cast<const float2*>(l2 + 2 * u);
          const float2 de = *reinterpret_cast<const float2*>(dl + 2 * u);
          const float2 x = __ffma2_rn(s2, c2, make_float2(-lq.x, -lq.y));  // s c - lse2
          float2 pr = make_float2(ex2_approx(x.x), ex2_approx(x.y));        // P (lse2 = +inf pads -> 0)
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
      TPROBE(2)
      if (i > 0) mbar_wait(&sm.p_free, (i - 1) & 1);  // dV_{i-1}, dK_{i-1} no longer read PT / dST
      TPROBE(3)
      tc_fence_after();
      if constexpr (NC == 32) {
        tmem_st16(lane_base + kColP + g * 16, pk);
        tmem_st16(lane_base + kColDS + g * 16, dk);
      } else {
        tmem_st8(lane_base + kColP + g * 8, pk);
        tmem_st8(lane_base + kColDS + g * 8, dk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
      TPROBE(4)
    }
    // ------------------------------------------------------------------ dV, dK epilogue
    // warpgroup g writes 64 columns: D = 64: g 0 dV, g 1 dK; D = 128: g 0, 1 dV, g 2, 3 dK
    if (g < 2 * kAtoms) {
      mbar_wait(&sm.dkv_done, 0);
      tc_fence_after();
      uint32_t r[64];
      const bool is_dv = g < kAtoms;
      const int cpart = g % kAtoms;
      const uint32_t col = (is_dv ? kColDV : kColDK) + cpart * 64;
      tmem_ld32(lane_base + col, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld32(lane_base + col + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld_wait();
#ifdef MEA_EXP_TIMING
      if (false) {
#else
      if (k0 + j < p.n_k) {
#endif
        const float sc = is_dv ? 1.f : p.scale;
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(is_dv ? p.dv : p.dk) +
                             (((size_t)b * p.n_k + k0 + j) * p.H + h) * D + cpart * 64;
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

template <int D>
static cudaError_t launch_bwd_dkdv_d(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                                     const CUtensorMap& mv, const CUtensorMap& mdo, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr<bwd_dkdv_kernel<D>>((int)dkv_smem_bytes<D>());
  if (attr != cudaSuccess) return attr;
  const dim3 grid = p.causal ? dim3(p.num_k_blocks * p.H * p.B) : dim3(p.num_k_blocks, p.H, p.B);
  bwd_dkdv_kernel<D><<<grid, kBThreads, dkv_smem_bytes<D>(), s>>>(mq, mk, mv, mdo, p);
  return cudaGetLastError();
}

// mq / mdo: boxes of DkvCfg<D>::QT rows (128 at D = 64, 64 at D = 128)
cudaError_t launch_bwd_dkdv(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                            const CUtensorMap& mdo, cudaStream_t s) {
  return p.d == 128 ? launch_bwd_dkdv_d<128>(p, mq, mk, mv, mdo, s) : launch_bwd_dkdv_d<64>(p, mq, mk, mv, mdo, s);
}

}  // namespace mea
