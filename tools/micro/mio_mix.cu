// Does the forward softmax's non-MUFU traffic through the MIO queue (tcgen05.ld / st, mbarrier
// ops, vote) slow the exponentials (MUFU is dispatched through the same queue)? 16 softmax-like
// warps per SM (640 threads, one CTA per SM); per iteration each does the forward's per-tile mix:
// 24 pairs (FFMA2, 2 x MUFU.EX2 or the FMA-pipe polynomial, FADD2, F2FP) plus, by mode,
//   bit 0: tcgen05.ld of 48 columns (.16x32bx2 x32 + x16) and tcgen05.st of 24 (x16 + x8)
//   bit 1: two mbarrier ops (test_wait of a completed phase, arrive on a never-waited barrier)
//   bit 2: one __any_sync + one xor-shuffle
//   bit 3: the tcgen05.ld alone, bit 4: the tcgen05.st alone, bit 5: the load in the .32x32b shape
// cycles per exponential pair per SM sub-partition are reported.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <type_traits>
#include "ptx.cuh"
using namespace mea;

template <int MODE, unsigned POLY>
__global__ void __launch_bounds__(640, 1) kern(int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t done_bar, sink_bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&done_bar, 1);
    mbar_init(&sink_bar, (1u << 20) - 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) mbar_arrive(&done_bar);   // phase 0 completes
  __syncthreads();
  const uint32_t tm = tbase;
  if (warp >= 4) {
    const int sw = warp - 4, quarter = warp & 3, sub = (sw >> 2) & 1, qt = sw >> 3;
    const uint32_t lb = tm + ((uint32_t)(quarter * 32 + sub * 16) << 16) + qt * 192;
    float v[48];
#pragma unroll
    for (int i = 0; i < 48; ++i) v[i] = 0.01f * (float)((threadIdx.x * 7 + i) & 15) - 8.f;
    uint32_t acc = 0;
    float l = 0.f;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE & 9) {
        uint32_t r[48];
        if (MODE & 32) {   // same 48 columns x 32 lanes as .32x32b (thread = TMEM lane)
          const uint32_t lq = tm + ((uint32_t)(quarter * 32) << 16) + qt * 192 + sub * 96;
          tmem_ld32(lq, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld16(lq + 32, *reinterpret_cast<uint32_t(*)[16]>(&r[32]));
        } else {
          tmem_ld32_split<48>(lb, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld16_split<48>(lb + 32, *reinterpret_cast<uint32_t(*)[16]>(&r[32]));
        }
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 48; ++i) v[i] += __uint_as_float(r[i]) * 1e-30f;
      }
      if (MODE & 2) {
        if (mbar_test_wait(&done_bar, 0)) acc += 1;
      }
      const float2 c2 = make_float2(0.01f, 0.01f), nm2 = make_float2(-1.f, -1.f);
      float2 rs = make_float2(0.f, 0.f);
      uint32_t pk[24];
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), c2, nm2);
        const float2 e = ((POLY >> i) & 1u) ? exp2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
        rs = __fadd2_rn(rs, e);
        pk[i] = pack_bf16x2(e.x, e.y);
      }
      const float rsum = rs.x + rs.y;
      if (MODE & 4) {
        if (__any_sync(0xffffffffu, !(rsum <= 1e30f))) acc += 7;
        l += __shfl_xor_sync(0xffffffffu, rsum, 16) * 1e-9f;
      }
      l += rsum;
      if (MODE & 17) {
        tmem_st16_split<24>(lb, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
        tmem_st8_split<24>(lb + 16, *reinterpret_cast<uint32_t(*)[8]>(&pk[16]));
        tmem_st_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 24; ++i) acc ^= pk[i];
      }
      if (MODE & 2) {
        tc_fence_before();
        mbar_arrive(&sink_bar);
      }
#pragma unroll
      for (int i = 0; i < 48; ++i) v[i] += 1e-7f;
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + sw] = t1 - t0;
    sink[blockIdx.x * 640 + threadIdx.x] = l + (float)acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

template <int M, unsigned P>
void run(const char* name, unsigned long long* d, float* sink) {
  cudaFuncSetAttribute(kern<M, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int iters = 400;
  for (int rep = 0; rep < 2; ++rep) {
    kern<M, P><<<148, 640, 120 * 1024>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  }
  unsigned long long h[148 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148 * 16; ++i) s += h[i];
  s /= 148 * 16;
  printf("%-58s %6.2f cycles per pair per SMSP\n", name, s / (iters * 24.0) / 4.0);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 148 * 16 * 8);
  float* sink; cudaMalloc(&sink, 148 * 640 * 4);
  run<0, 0x00080080u>("exp loop only (2 poly pairs)", d, sink);
  run<1, 0x00080080u>("+ tcgen05.ld 48 cols / st 24 cols", d, sink);
  run<8, 0x00080080u>("+ tcgen05.ld 48 cols only", d, sink);
  run<16, 0x00080080u>("+ tcgen05.st 24 cols only", d, sink);
  run<8 | 32, 0x00080080u>("+ tcgen05.ld 48 cols only, .32x32b shape", d, sink);
  run<2, 0x00080080u>("+ 2 mbarrier ops", d, sink);
  run<4, 0x00080080u>("+ vote + shuffle", d, sink);
  run<7, 0x00080080u>("+ all of the above (the forward's mix)", d, sink);
  run<7, 0u>("the forward's mix, 0 poly pairs", d, sink);
  run<7, 0x00410041u>("the forward's mix, 4 poly pairs", d, sink);
  run<7, 0x00888888u>("the forward's mix, 6 poly pairs", d, sink);
  run<7, 0x00249249u>("the forward's mix, 8 poly pairs", d, sink);
  return 0;
}
