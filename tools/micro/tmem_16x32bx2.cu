// Verify the lane/column mapping of tcgen05.ld / tcgen05.st .16x32bx2 (split half-warps).
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mea;

__device__ __forceinline__ void ld_16x32bx2_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16], 64;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__global__ void kern(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  // fill: TMEM lane L, column c  <- L * 1000 + c   (32x32b: thread = lane)
  const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = (warp * 32 + lane) * 1000 + c0 + i;
    tmem_st16(lb + c0, v);
  }
  tmem_st_wait();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  // read back with 16x32bx2 from lane base warp*32 + 16*sub, column 8, split offset 64
  for (int sub = 0; sub < 2; ++sub) {
    uint32_t r[16];
    ld_16x32bx2_x16(tm + ((uint32_t)(warp * 32 + 16 * sub) << 16) + 8, r);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[((warp * 2 + sub) * 32 + lane) * 16 + i] = r[i];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 4 * 2 * 32 * 16 * 4);
  kern<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  static uint32_t h[4 * 2 * 32 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  for (int w = 0; w < 4; w += 3)
    for (int sub = 0; sub < 2; ++sub)
      for (int t : {0, 1, 15, 16, 17, 31}) {
        const uint32_t* r = h + ((w * 2 + sub) * 32 + t) * 16;
        printf("warp %d sub %d thread %2d: r[0]=%u r[1]=%u r[15]=%u  (lane %u col %u)\n", w, sub, t, r[0], r[1], r[15],
               r[0] / 1000, r[0] % 1000);
      }
  return 0;
}
