// Throughput of tcgen05.mma operand forms used by the kernels (bf16 -> f32, cta_group::1, M=128).
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mea;

// form: 0 SS K/K N=128 (QK^T)   1 TS A=tmem, B MN N=64 (PV, dV)   2 SS A K-major, B MN N=64 (dK)
//       3 SS A MN (2 atoms, LBO 16K), B MN N=64 (dQ)             4 SS K/K N=64
template <int FORM, bool STREAM>
__global__ void __launch_bounds__(128, 1) kern(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536; i += 128) sm[i] = 0x3c;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  if (warp == 1) {
    const uint64_t a = shfl0_u64(sdesc_sw128(smem_u32(sm), 16, 1024));
    const uint64_t am = shfl0_u64(sdesc_sw128(smem_u32(sm), 16384, 1024));
    const uint64_t b = shfl0_u64(sdesc_sw128(smem_u32(sm + 32768), 16, 1024));
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (FORM == 0) umma_ss(tm, a + (kk & 3) * 2, b + (kk & 3) * 2, idesc_bf16_f32(128, 128, false, false), 1);
          if (FORM == 1) umma_ts(tm, tm + 256 + kk * 8, b + kk * 128, idesc_bf16_f32(128, 64, false, true), 1);
          if (FORM == 2) umma_ss(tm, a + (kk >> 2) * 1024 + (kk & 3) * 2, b + kk * 128, idesc_bf16_f32(128, 64, false, true), 1);
          if (FORM == 3) umma_ss(tm, am + kk * 128, b + kk * 128, idesc_bf16_f32(128, 64, true, true), 1);
          if (FORM == 4) umma_ss(tm, a + (kk & 3) * 2, b + (kk & 3) * 2, idesc_bf16_f32(128, 64, false, false), 1);
        }
        if (!STREAM || it == iters - 1) umma_commit(&bar);
      }
      __syncwarp();
      if (!STREAM) mbar_wait(&bar, it & 1);
    }
    if (STREAM) mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = (t1 - t0) / iters;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

template <int F, bool S = false>
void run(const char* name, int n) {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(kern<F, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  kern<F, S><<<148, 128, 66 * 1024>>>(200, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 8.0 * 128 * n * 16;
  printf("%-44s err=%s  %llu clk per 8 MMAs  -> %.0f%% of 4096 MAC/clk\n", name, cudaGetErrorString(e), h,
         100.0 * macs / h / 4096);
}

int main() {
  run<0>("SS  A K-major, B K-major, N=128 (QK^T)", 128);
  run<4>("SS  A K-major, B K-major, N=64", 64);
  run<1>("TS  A TMEM,    B MN-major, N=64 (PV, dV)", 64);
  run<2>("SS  A K-major, B MN-major, N=64 (dK)", 64);
  run<3>("SS  A MN-major,B MN-major, N=64 (dQ)", 64);
  printf("streaming (one commit at the end):\n");
  run<0, true>("SS  A K-major, B K-major, N=128 (QK^T)", 128);
  run<4, true>("SS  A K-major, B K-major, N=64", 64);
  run<1, true>("TS  A TMEM,    B MN-major, N=64 (PV, dV)", 64);
  run<2, true>("SS  A K-major, B MN-major, N=64 (dK)", 64);
  run<3, true>("SS  A MN-major,B MN-major, N=64 (dQ)", 64);
  return 0;
}
