// CTA-pair (cta_group::2) tcgen05.mma on B200: correctness of the operand split and TMEM layout,
// whether a cta_group::1 MMA may use TMEM allocated for the pair, and pair throughput.
//   A (M = 256): rows 0-127 from CTA rank 0's smem, 128-255 from rank 1's (same smem offset)
//   B (N): columns [0, N/2) from rank 0's smem, [N/2, N) from rank 1's (expected split)
//   D: each CTA's TMEM holds its 128 rows x N columns
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2112_05682_b200/csrc mma_pair.cu -o mma_pair
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace mea;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void alloc2(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void dealloc2(uint32_t t, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(cols));
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3));
}

// SW128 K-major tile: row r, element k (bf16, K = 64 -> 128 B per row)
__device__ __forceinline__ uint32_t sw_off(int r, int k) {
  return r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2;
}

// MODE 0: correctness (pair MMA M=256 N=128 K=64), then a cta_group::1 MMA on the same TMEM
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    check(const __nv_bfloat16* A, const __nv_bfloat16* Bm, float* D, float* D1, int do_mix) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint8_t* sa = sm;            // 128 x 64 (16 KB)
  uint8_t* sb = sm + 16384;    // N/2 x 64 (B half) ; for the ::1 test: 64 x 64
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar, bar1;
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw_off(r, k)) = A[(rank * 128 + r) * 64 + k];
  }
  for (int i = threadIdx.x; i < (N / 2) * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(sb + sw_off(r, k)) = Bm[(rank * (N / 2) + r) * 64 + k];
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar1, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) alloc2(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (rank == 0 && warp == 1) {
    const uint64_t a = shfl0_u64(sdesc_sw128(smem_u32(sa), 16, 1024));
    const uint64_t b = shfl0_u64(sdesc_sw128(smem_u32(sb), 16, 1024));
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma2_ss(tm, a + kk * 2, b + kk * 2, idesc_bf16_f32(256, N, false, false), kk > 0);
      commit2_mc(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
    const int row = rank * 128 + warp * 32 + lane;
    for (int c = 0; c < N; c += 32) {
      uint32_t r[32];
      tmem_ld32(lb + c, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) D[row * N + c + i] = __uint_as_float(r[i]);
    }
  }
  if (do_mix) {
    // cta_group::1 MMA (M = 128, N = 64, K = 64) in each CTA into columns [128, 192) of the
    // pair-allocated TMEM: A = this CTA's A tile, B = its first 64 B rows
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
      const uint64_t a = shfl0_u64(sdesc_sw128(smem_u32(sa), 16, 1024));
      const uint64_t b = shfl0_u64(sdesc_sw128(smem_u32(sb), 16, 1024));
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_ss(tm + 128, a + kk * 2, b + kk * 2, idesc_bf16_f32(128, 64, false, false), kk > 0);
        umma_commit(&bar1);
      }
      __syncwarp();
    }
    mbar_wait(&bar1, 0);
    tc_fence_after();
    const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
    const int row = rank * 128 + warp * 32 + lane;
    for (int c = 0; c < 64; c += 32) {
      uint32_t r[32];
      tmem_ld32(lb + 128 + c, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) D1[row * 64 + c + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    dealloc2(tm, 256);
  }
}

// throughput: leader issues 8 pair MMAs (M=256, N, K=16) per iteration, one commit at the end
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) tput(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32768; i += 128) sm[i] = 0x3c;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) alloc2(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = tbase;
  unsigned long long t0 = clock64();
  if (rank == 0 && warp == 1) {
    const uint64_t a = shfl0_u64(sdesc_sw128(smem_u32(sm), 16, 1024));
    const uint64_t b = shfl0_u64(sdesc_sw128(smem_u32(sm + 16384), 16, 1024));
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma2_ss(tm, a + (kk & 3) * 2, b + (kk & 3) * 2, idesc_bf16_f32(256, N, false, false), 1);
        if (it == iters - 1) commit2_mc(&bar);
      }
      __syncwarp();
    }
  }
  mbar_wait(&bar, 0);
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / 2] = (t1 - t0) / iters;
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    dealloc2(tm, 256);
  }
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int N>
int run_check(int mix) {
  std::vector<__nv_bfloat16> hA(256 * 64), hB(N * 64);
  std::vector<float> fA(256 * 64), fB(N * 64);
  srand(1);
  for (int i = 0; i < 256 * 64; ++i) { fA[i] = bf((rand() % 17 - 8) / 8.f); hA[i] = __float2bfloat16(fA[i]); }
  for (int i = 0; i < N * 64; ++i) { fB[i] = bf((rand() % 17 - 8) / 8.f); hB[i] = __float2bfloat16(fB[i]); }
  __nv_bfloat16 *dA, *dB; float *dD, *dD1;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dD, 256 * N * 4); cudaMalloc(&dD1, 256 * 64 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, 256 * N * 4); cudaMemset(dD1, 0, 256 * 64 * 4);
  cudaFuncSetAttribute(check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  check<N><<<2, 128, 40 * 1024>>>(dA, dB, dD, dD1, mix);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> D(256 * N), D1(256 * 64);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(D1.data(), dD1, D1.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, err1 = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < 64; ++k) r += (double)fA[m * 64 + k] * fB[n * 64 + k];
      err = fmax(err, fabs(r - D[m * N + n]));
    }
  if (mix)
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < 64; ++n) {  // CTA c: its A rows x its own first 64 B rows (B half of c)
        const int c = m / 128;
        double r = 0;
        for (int k = 0; k < 64; ++k) r += (double)fA[m * 64 + k] * fB[(c * (N / 2) + n) * 64 + k];
        err1 = fmax(err1, fabs(r - D1[m * 64 + n]));
      }
  printf("pair MMA M=256 N=%d: %s, max |err| %.3g (expect 0)", N, cudaGetErrorString(e), err);
  if (mix) printf(" | cta_group::1 MMA on pair TMEM: max |err| %.3g", err1);
  printf("\n");
  return e != cudaSuccess;
}

template <int N>
void run_tput() {
  unsigned long long* d; cudaMalloc(&d, 74 * 8);
  cudaFuncSetAttribute(tput<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  tput<N><<<148, 128, 40 * 1024>>>(400, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double macs_per_sm = 8.0 * 128 * N * 16;  // each SM computes its 128 rows
  printf("pair streaming M=256 N=%-3d: %s %llu clk per 8 MMAs -> %.0f%% of 4096 MAC/clk/SM\n", N, cudaGetErrorString(e),
         h, 100.0 * macs_per_sm / h / 4096);
}

int main() {
  if (run_check<128>(0)) return 1;
  if (run_check<64>(0)) return 1;
  if (run_check<128>(1)) return 1;
  run_tput<128>();
  run_tput<64>();
  run_tput<256>();
  return 0;
}
