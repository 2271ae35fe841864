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

__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(taddr));
}
__device__ __forceinline__ void ld_16x256b_x4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
}
__device__ __forceinline__ void ld_16x128b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(taddr));
}
__device__ __forceinline__ void ld_16x128b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
}
__device__ __forceinline__ void ld_16x64b_x32(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(taddr));
}
__device__ __forceinline__ void ld_16x64b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
}
__device__ __forceinline__ void st_16x128b_x8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void st_16x128b_x4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
__device__ __forceinline__ void st_16x256b_x4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void st_16x256b_x2(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}

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
        if (MODE & 64) {          // .16x256b: 16 lanes x 96 columns (the same 6 KB per warp)
          ld_16x256b_x8(lb, &r[0]);
          ld_16x256b_x4(lb + 64, &r[32]);
        } else if (MODE & 128) {  // .16x128b
          ld_16x128b_x16(lb, &r[0]);
          ld_16x128b_x8(lb + 64, &r[32]);
        } else if (MODE & 256) {  // .16x64b
          ld_16x64b_x32(lb, &r[0]);
          ld_16x64b_x16(lb + 64, &r[32]);
        } else if (MODE & 32) {   // same 48 columns x 32 lanes as .32x32b (thread = TMEM lane)
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
        if (MODE & 512) {          // P (24 words per thread) as .16x128b (12 reps x 2 words)
          st_16x128b_x8(lb, &pk[0]);
          st_16x128b_x4(lb + 32, &pk[16]);
        } else if (MODE & 1024) {  // as .16x256b
          st_16x256b_x4(lb, &pk[0]);
          st_16x256b_x2(lb + 32, &pk[16]);
        } else {
          tmem_st16_split<24>(lb, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
          tmem_st8_split<24>(lb + 16, *reinterpret_cast<uint32_t(*)[8]>(&pk[16]));
        }
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
  run<8 | 64, 0x00080080u>("+ tcgen05.ld 6 KB per warp, .16x256b shape", d, sink);
  run<16 | 512, 0x00080080u>("+ tcgen05.st 3 KB per warp, .16x128b shape", d, sink);
  run<16 | 1024, 0x00080080u>("+ tcgen05.st 3 KB per warp, .16x256b shape", d, sink);
  run<8 | 16 | 64 | 512, 0x00080080u>("+ ld .16x256b and st .16x128b", d, sink);
  run<8 | 16 | 64 | 512 | 2 | 4, 0x00080080u>("the forward's mix with ld .16x256b, st .16x128b", d, sink);
  run<8 | 16 | 64 | 512 | 2 | 4, 0x00410041u>("... with 4 poly pairs", d, sink);
  run<8 | 128, 0x00080080u>("+ tcgen05.ld 6 KB per warp, .16x128b shape", d, sink);
  run<8 | 256, 0x00080080u>("+ tcgen05.ld 6 KB per warp, .16x64b shape", d, sink);
  run<2, 0x00080080u>("+ 2 mbarrier ops", d, sink);
  run<4, 0x00080080u>("+ vote + shuffle", d, sink);
  run<7, 0x00080080u>("+ all of the above (the forward's mix)", d, sink);
  run<7, 0u>("the forward's mix, 0 poly pairs", d, sink);
  run<7, 0x00410041u>("the forward's mix, 4 poly pairs", d, sink);
  run<7, 0x00888888u>("the forward's mix, 6 poly pairs", d, sink);
  run<7, 0x00249249u>("the forward's mix, 8 poly pairs", d, sink);
  return 0;
}
