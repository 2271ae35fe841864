// bwd_dq_sm100a.cu — dQ of exact attention on tcgen05 tensor cores (second backward kernel).
//
// dQ = scale * dS K with dS = P o (dP - delta), P = exp(scale q k^T - lse), dP = dO V^T
// (the softmax VJP; the paper differentiates with jax.grad through jax.checkpoint,
// PAPER.md:254-261, and recomputes every tile of scores). One CTA owns 128 query
// rows of one (b, h) and loops over all key tiles of 128, so dQ accumulates in TMEM and is
// written once, in bf16: deterministic, no fp32 accumulator, no atomics.
//   S  = Q K^T    (SS MMA, M=128 queries, N=128 keys)     TMEM [0,128)
//   dP = dO V^T   (SS MMA)                                TMEM [128,256)
//   softmax warps: P = 2^(S c - lse2_row), dS = P o (dP - delta_row) -> bf16 -> TMEM
//                  [320,384) / [384,448) alternately (double buffer)
//   dQ += dS K    (TS MMA: A = dS from TMEM, B = K MN-major, N=64)  TMEM [256,320)
// Per query row lse and delta are scalars (no per-element loads). Padded key rows (K, V zero-
// filled by TMA) give dS * 0 = 0 in dQ, so ragged key tiles need no mask.
// Schedule: S_{t+1}, dP_{t+1} are issued once the softmax warps have read S_t, dP_t out of TMEM
// ("s_loaded"); dQ_t once dS_t is stored ("p_full"); with two dS buffers the softmax only waits
// for dQ_{t-2} ("ds_free") before overwriting one.
// Warps: 0 TMA producer (Q, dO once; 4-stage K/V ring), 1 MMA issuer, 2 TMEM allocator,
// 4-19 softmax: warp (colhalf, sub, quarter) owns rows quarter*32 + sub*16 + [0,16) and key
// columns colhalf*64 + [0,64) (.16x256b: a quad of threads holds two rows, see the softmax section).
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace mea {
namespace {

// D = 64 (kHeadDim) or 128. A tile of R rows is D/64 SW128 atoms (R rows x 128 B) wide. Key
// tiles are KT = 128 keys at D = 64 and 64 keys at D = 128, so that a 4-stage K/V ring fits
// next to the resident Q and dO (a 2-stage ring of 128-key tiles left the MMA waiting on loads).
template <int D> struct DqCfg {
  static constexpr int kAtoms = D / 64;
  static constexpr int KT = D == 64 ? 128 : 64;
  static constexpr int kQTileBytes = 128 * D * 2, kKTileBytes = KT * D * 2;
  static constexpr int kQAtom = 128 * 128, kKAtom = KT * 128;
  static constexpr int kStages = 4;  // K/V ring
  static constexpr uint32_t kColS = 0, kColDP = KT, kColDQ = 2 * KT;  // + dS double buffer after dQ
};
constexpr int kTile = 128;  // query rows per CTA
constexpr int kQThreads = 640;
constexpr int kQCtrlRegs = 64, kQSoftRegs = 104;  // 64 + 4*104 = 480 = launch budget per lane slot
template <int D>
struct DqSmem {
  using C = DqCfg<D>;
  static constexpr int kQStages = C::kStages;
  uint8_t q[C::kQTileBytes];
  uint8_t dout[C::kQTileBytes];
  uint8_t k[kQStages][C::kKTileBytes];
  uint8_t v[kQStages][C::kKTileBytes];
  uint64_t q_full, kv_full[kQStages], kv_empty[kQStages];
  uint64_t s_full, s_loaded, p_full, ds_free[2], o_done;
  uint32_t tmem_base;
};
template <int D> constexpr size_t dq_smem_bytes() { return sizeof(DqSmem<D>) + 1024; }

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

template <int D>
__global__ void __launch_bounds__(kQThreads, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                  const BwdParams p) {
  using C = DqCfg<D>;
  constexpr int kAtoms = C::kAtoms, KT = C::KT, kQStages = C::kStages;
  constexpr uint32_t kColS = C::kColS, kColDP = C::kColDP, kColDQ = C::kColDQ;
  auto col_ds = [](int buf) { return kColDQ + D + buf * (KT / 2u); };  // dS double buffer after dQ
  constexpr uint32_t kIdSS = idesc_bf16_f32(128, KT, false, false);  // S, dP: N = KT keys
  // dQ += dS K: N = D; B = K MN-major, N over kAtoms atoms C::kKAtom bytes apart (LBO)
  constexpr uint32_t kIdDQ = idesc_bf16_f32(128, D, false, true);
  extern __shared__ uint8_t smem_raw[];
  DqSmem<D>& sm = *reinterpret_cast<DqSmem<D>*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: 1-D grid, the last query block (the most key tiles) first across all (b, h)
  const int nqb = (p.n_q + kTile - 1) / kTile;
  const int qblk = p.causal ? nqb - 1 - (int)(blockIdx.x / (p.H * p.B)) : (int)blockIdx.x;
  const int h = p.causal ? (int)(blockIdx.x % p.H) : (int)blockIdx.y;
  const int b = p.causal ? (int)((blockIdx.x / p.H) % p.B) : (int)blockIdx.z;
  const int q0 = qblk * kTile;
  // causal (n_q == n_k): keys up to this block's last query row only
  const int T = p.causal ? min((p.n_k + KT - 1) / KT, (q0 + kTile + KT - 1) / KT) : (p.n_k + KT - 1) / KT;
  const int nk = keys_of(p.kv_lens, b, p.n_k);  // key padding
  const int nq_pad = (p.n_q + kTile - 1) / kTile * kTile;
  const size_t bh = (size_t)b * p.H + h;

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_loaded, 512);
    mbar_init(&sm.p_full, 512);
    mbar_init(&sm.ds_free[0], 1);
    mbar_init(&sm.ds_free[1], 1);
    mbar_init(&sm.o_done, 1);
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
    setmaxnreg_dec<kQCtrlRegs>();
    if (warp == 0) {
      // ---------------------------------------------------------------- TMA producer
      const uint64_t keep = policy_evict_last(), once = policy_evict_first();
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm.q_full, 2 * C::kQTileBytes);
#pragma unroll
        for (int a = 0; a < kAtoms; ++a) {
          tma_load_4d(sm.q + a * C::kQAtom, &mq, &sm.q_full, 64 * a, h, q0, b, once);
          tma_load_4d(sm.dout + a * C::kQAtom, &mdo, &sm.q_full, 64 * a, h, q0, b, once);
        }
      }
      __syncwarp();
      for (int t = 0; t < T; ++t) {
        const int st = t % kQStages, n = t / kQStages;
        if (t >= kQStages) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm.kv_full[st], 2 * C::kKTileBytes);
#pragma unroll
          for (int a = 0; a < kAtoms; ++a) {
            tma_load_4d(sm.k[st] + a * C::kKAtom, &mk, &sm.kv_full[st], 64 * a, h, t * KT, b, keep);
            tma_load_4d(sm.v[st] + a * C::kKAtom, &mv, &sm.kv_full[st], 64 * a, h, t * KT, b, keep);
          }
        }
        __syncwarp();
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------------- MMA issuer
      const uint64_t dQd = shfl0_u64(sdesc_sw128(smem_u32(sm.q), 16, 1024));
      const uint64_t dOd = shfl0_u64(sdesc_sw128(smem_u32(sm.dout), 16, 1024));
      const uint64_t dK0 = shfl0_u64(sdesc_sw128(smem_u32(sm.k[0]), 16, 1024));
      const uint64_t dV0 = shfl0_u64(sdesc_sw128(smem_u32(sm.v[0]), 16, 1024));
      const uint64_t dKm0 = shfl0_u64(sdesc_sw128(smem_u32(sm.k[0]), C::kKAtom, 1024));  // MN-major view
      constexpr uint64_t kStep = C::kKTileBytes >> 4, kQAt = C::kQAtom >> 4, kKAt = C::kKAtom >> 4;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      auto scores = [&](int st) {  // S = Q K^T ; dP = dO V^T
        const uint64_t kd = dK0 + st * kStep, vd = dV0 + st * kStep;
#pragma unroll
        for (int kk = 0; kk < 4 * kAtoms; ++kk)
          umma_ss(tm + kColS, dQd + (kk >> 2) * kQAt + (kk & 3) * 2, kd + (kk >> 2) * kKAt + (kk & 3) * 2, kIdSS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4 * kAtoms; ++kk)
          umma_ss(tm + kColDP, dOd + (kk >> 2) * kQAt + (kk & 3) * 2, vd + (kk >> 2) * kKAt + (kk & 3) * 2, kIdSS, kk > 0);
      };
      mbar_wait(&sm.q_full, 0);
      mbar_wait(&sm.kv_full[0], 0);
      tc_fence_after();
      if (elect_one()) {
        scores(0);
        umma_commit(&sm.s_full);
      }
      __syncwarp();
      for (int t = 0; t < T; ++t) {
        const int st = t % kQStages, nx = (t + 1) % kQStages;
        const bool more = t + 1 < T;
        if (more) {
          mbar_wait(&sm.kv_full[nx], ((t + 1) / kQStages) & 1);
          mbar_wait(&sm.s_loaded, t & 1);
          tc_fence_after();
          if (elect_one()) {
            scores(nx);
            umma_commit(&sm.s_full);
          }
          __syncwarp();
        }
        mbar_wait(&sm.p_full, t & 1);
        tc_fence_after();
        if (elect_one()) {
          // dQ += dS K : K = 128 keys in steps of 16 (dS: 8 TMEM columns; K rows: 2048 B)
          const uint64_t kd = dKm0 + st * kStep;
#pragma unroll
          for (int kk = 0; kk < KT / 16; ++kk) umma_ts(tm + kColDQ, tm + col_ds(t & 1) + kk * 8, kd + kk * 128, kIdDQ, (t > 0 || kk > 0));
          umma_commit(&sm.ds_free[t & 1]);
          umma_commit(&sm.kv_empty[st]);
          if (!more) umma_commit(&sm.o_done);
        }
        __syncwarp();
      }
    }
  } else {
    setmaxnreg_inc<kQSoftRegs>();
    // ------------------------------------------------------------------ softmax warps
    // warp (colhalf, sub, quarter): TMEM lanes L0 = quarter*32 + sub*16 + [0,16), key columns
    // colhalf * KT/2 + [0, KT/2). S and dP are read as .16x256b and dS written as .16x128b
    // (ptx.cuh, as fwd_db): thread t (q = t % 4) holds rows a = L0 + t/4, b = a + 8 and key
    // columns colhalf * KT/2 + 8r + 2q, + 1 — the keys of dS column colhalf * KT/4 + 4r + q.
    const int sw = warp - 4;
    const int colhalf = sw >> 3;
    const int sub = (sw >> 2) & 1;
    const int quarter = warp & 3;
    const int q = lane & 3, ra = lane >> 2;
    const int L0 = quarter * 32 + sub * 16;
    const int row_a = q0 + L0 + ra, row_b = row_a + 8;
    const int rloc = quarter * 32 + sub * 16 + (lane & 15);  // the epilogue's row (16x32bx2 layout)
    const int row = q0 + rloc;
    const uint32_t lane_base = tmem + ((uint32_t)L0 << 16);
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    // +inf lse2 on padded rows -> P = 0
    const float lse2_a = p.lse2[bh * nq_pad + q0 + L0 + ra], lse2_b = p.lse2[bh * nq_pad + q0 + L0 + ra + 8];
    const float delta_a = p.delta[bh * nq_pad + q0 + L0 + ra], delta_b = p.delta[bh * nq_pad + q0 + L0 + ra + 8];
    const float2 nla = make_float2(-lse2_a, -lse2_a), nlb = make_float2(-lse2_b, -lse2_b);
    const float2 nda = make_float2(-delta_a, -delta_a), ndb = make_float2(-delta_b, -delta_b);
#ifdef MEA_EXP_TIMING
    unsigned long long* tdbg = reinterpret_cast<unsigned long long*>(p.dq);
    const bool probe = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && quarter == 0 && sub == 0 && lane == 0;
#define TPROBE(k) if (probe && t >= 8 && t < 24) tdbg[(colhalf * 16 + (t - 8)) * 8 + (k)] = clock64();
#else
#define TPROBE(k)
#endif
    constexpr int NR = KT / 16;  // .16x256b repetitions over this warp's KT/2 key columns
    for (int t = 0; t < T; ++t) {
      TPROBE(0)
      mbar_wait(&sm.s_full, t & 1);
      TPROBE(1)
      tc_fence_after();
      uint32_t sr[4 * NR], dr[4 * NR];
      if constexpr (NR == 8) {
        tmem_ld_16x256b_x8(lane_base + kColS + colhalf * (KT / 2), sr);
        tmem_ld_16x256b_x8(lane_base + kColDP + colhalf * (KT / 2), dr);
      } else {
        tmem_ld_16x256b_x4(lane_base + kColS + colhalf * (KT / 2), sr);
        tmem_ld_16x256b_x4(lane_base + kColDP + colhalf * (KT / 2), dr);
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&sm.s_loaded);  // S_t, dP_t are in registers: the next scores may overwrite them
      TPROBE(2)
      uint32_t pk[2 * NR];  // [2r] row a, [2r + 1] row b: dS column colhalf * KT/4 + 4r + q
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const float2 s2 = make_float2(__uint_as_float(sr[4 * r + 2 * hb]), __uint_as_float(sr[4 * r + 2 * hb + 1]));
          const float2 d2 = make_float2(__uint_as_float(dr[4 * r + 2 * hb]), __uint_as_float(dr[4 * r + 2 * hb + 1]));
          const float2 x = __ffma2_rn(s2, c2, hb ? nlb : nla);                   // s c - lse2
          float2 pr = make_float2(ex2_approx(x.x), ex2_approx(x.y));             // P
          const int key = t * KT + colhalf * (KT / 2) + 8 * r + 2 * q;
          if (p.causal) {  // key > query row: masked
            const int rr = hb ? row_b : row_a;
            if (key > rr) pr.x = 0.f;
            if (key + 1 > rr) pr.y = 0.f;
          }
          if (p.kv_lens) {  // key padding: keys >= nk masked
            if (key >= nk) pr.x = 0.f;
            if (key + 1 >= nk) pr.y = 0.f;
          }
          const float2 ds = __fmul2_rn(pr, __fadd2_rn(d2, hb ? ndb : nda));      // P (dP - delta)
          pk[2 * r + hb] = pack_bf16x2(ds.x, ds.y);
        }
      TPROBE(3)
      if (t > 1) mbar_wait(&sm.ds_free[t & 1], ((t >> 1) - 1) & 1);  // dQ_{t-2} has consumed this buffer
      TPROBE(4)
      tc_fence_after();
      if constexpr (NR == 8) {
        tmem_st_16x128b_x8(lane_base + col_ds(t & 1) + colhalf * (KT / 4), pk);
      } else {
        tmem_st_16x128b_x4(lane_base + col_ds(t & 1) + colhalf * (KT / 4), pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
      TPROBE(5)
    }
    // ------------------------------------------------------------------ epilogue: dq = scale dQ
    // thread (colhalf, lane half) writes dQ columns colhalf * D/2 + (lane >> 4) * D/4 + [0, D/4)
    // of row `row` (the 16x32bx2 layout: lanes t and t + 16 share a row)
    const uint32_t lane_base16 = tmem + ((uint32_t)(quarter * 32 + sub * 16) << 16);
    mbar_wait(&sm.o_done, 0);
    tc_fence_after();
    constexpr int kW = D / 4;  // columns per thread
    uint32_t o[kW];
    if constexpr (D == 64) {
      tmem_ld16_split<16>(lane_base16 + kColDQ + colhalf * 32, o);
    } else {
      tmem_ld32_split<32>(lane_base16 + kColDQ + colhalf * 64, o);
    }
    tmem_ld_wait();
#ifdef MEA_EXP_TIMING
    if (false) {
#else
    if (row < p.n_q) {
#endif
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.dq) + (((size_t)b * p.n_q + row) * p.H + h) * D +
                           colhalf * (D / 2) + (lane >> 4) * kW;
      const float sc = p.scale;
#pragma unroll
      for (int i = 0; i < kW / 8; ++i) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(o[8 * i + 0]) * sc, __uint_as_float(o[8 * i + 1]) * sc);
        w.y = pack_bf16x2(__uint_as_float(o[8 * i + 2]) * sc, __uint_as_float(o[8 * i + 3]) * sc);
        w.z = pack_bf16x2(__uint_as_float(o[8 * i + 4]) * sc, __uint_as_float(o[8 * i + 5]) * sc);
        w.w = pack_bf16x2(__uint_as_float(o[8 * i + 6]) * sc, __uint_as_float(o[8 * i + 7]) * sc);
        reinterpret_cast<uint4*>(dst)[i] = w;
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
static cudaError_t launch_bwd_dq_d(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk,
                                   const CUtensorMap& mv, const CUtensorMap& mdo, cudaStream_t s) {
  const cudaError_t attr = ensure_smem_attr<bwd_dq_kernel<D>>((int)dq_smem_bytes<D>());
  if (attr != cudaSuccess) return attr;
  const int nqb = (p.n_q + kTile - 1) / kTile;
  const dim3 grid = p.causal ? dim3(nqb * p.H * p.B) : dim3(nqb, p.H, p.B);
  bwd_dq_kernel<D><<<grid, kQThreads, dq_smem_bytes<D>(), s>>>(mq, mk, mv, mdo, p);
  return cudaGetLastError();
}

cudaError_t launch_bwd_dq(const BwdParams& p, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                          const CUtensorMap& mdo, cudaStream_t s) {
  return p.d == 128 ? launch_bwd_dq_d<128>(p, mq, mk, mv, mdo, s) : launch_bwd_dq_d<64>(p, mq, mk, mv, mdo, s);
}

}  // namespace mea
