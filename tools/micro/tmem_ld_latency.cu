// Microbenchmark: tcgen05.ld latency (issue -> data usable) with and without concurrent MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2112_05682_b200/csrc tmem_ld_latency.cu -o tmem_ld_latency
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mea;

__global__ void __launch_bounds__(256, 1) kern(int mma_on, int iters, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t a[16384];
  __shared__ __align__(1024) uint8_t b[16384];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384; i += 256) { a[i] = 0x3c; b[i] = 0x3c; }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  if (warp == 1) {
    if (mma_on) {
      const uint64_t da = shfl0_u64(sdesc_sw128(smem_u32(a), 16, 1024));
      const uint64_t db = shfl0_u64(sdesc_sw128(smem_u32(b), 16, 1024));
      const uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
      for (int it = 0; it < 4000 && !stop; ++it) {
        if (elect_one()) {
          for (int kk = 0; kk < 4; ++kk) umma_ss(tm + 256, da + kk * 2, db + kk * 2, idesc, kk > 0);
          umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, it & 1);
      }
    }
  } else if (warp >= 4) {
    const uint32_t lb = tm + ((uint32_t)((warp & 3) * 32) << 16);
    unsigned long long tot = 0;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32], r2[32];
      const unsigned long long t0 = clock64();
      tmem_ld32(lb + 0, r);
      tmem_ld32(lb + 32, r2);
      tmem_ld_wait();
      uint32_t x = 0;
#pragma unroll
      for (int u = 0; u < 32; ++u) x ^= r[u] ^ r2[u];
      acc += x;
      const unsigned long long t1 = clock64();
      tot += t1 - t0;
    }
    if (lane == 0) out[warp - 4] = tot / iters;
    if (acc == 12345) out[10] = acc;
    __syncwarp();
    if (warp == 4 && lane == 0) stop = 1;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 8);
  for (int mma = 0; mma < 2; ++mma) {
    kern<<<148, 256>>>(mma, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("mma_on=%d err=%s  ld(64 cols)+use latency per warp: %llu %llu %llu %llu cycles\n", mma, cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  }
  return 0;
}
