// Lane/column mapping of tcgen05.ld .16x64b, .16x128b and .16x256b (one repetition each, and the
// register order across repetitions): TMEM lane L, column c is filled with L * 1000 + c, then
// each thread prints which (lane, column) its registers hold.
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mea;

template <int N>
__device__ __forceinline__ void ld_shape(int which, uint32_t taddr, uint32_t (&r)[N]);
__device__ __forceinline__ void ld64x2(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ld128x2(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ld256x1(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}

__global__ void kern(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = (warp * 32 + lane) * 1000 + c0 + i;
    tmem_st16(lb + c0, v);
  }
  tmem_st_wait();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 1) {   // lanes 32..63; start at lane 32 + 0, column 8
    uint32_t r[3][4];
    const uint32_t a = tm + (32u << 16) + 8;
    ld64x2(a, r[0]);
    ld128x2(a, r[1]);
    ld256x1(a, r[2]);
    tmem_ld_wait();
    for (int s = 0; s < 3; ++s)
      for (int i = 0; i < 4; ++i) out[(s * 32 + lane) * 4 + i] = r[s][i];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 3 * 32 * 4 * 4);
  kern<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  static uint32_t h[3 * 32 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s  (values: lane*1000 + column; loads start at lane 32, column 8)\n", cudaGetErrorString(e));
  const char* nm[3] = {"16x64b.x4 ", "16x128b.x2", "16x256b.x1"};
  for (int s = 0; s < 3; ++s)
    for (int t = 0; t < 32; ++t) {
      printf("%s thread %2d:", nm[s], t);
      for (int i = 0; i < 4; ++i) printf(" (%u,%u)", h[(s * 32 + t) * 4 + i] / 1000, h[(s * 32 + t) * 4 + i] % 1000);
      printf("\n");
    }
  return 0;
}
