// Does an MMA issuer whose tcgen05.mma instructions back up on a busy tensor pipe slow the other
// warps of its SM sub-partition (SMSP)? 640 threads per CTA (one CTA per SM) as in the d = 64
// forward: warp 1 (SMSP 1) issues MMAs, warps 4-19 (4 per SMSP) run the softmax's exponential
// loop (FFMA2, 2 x MUFU.EX2, FADD2, F2FP per pair) for a fixed amount of work; each softmax warp's
// duration is recorded and averaged per SMSP.
//   mode 0: no MMAs
//   mode 1: warp 1 streams SS M=128 N=96 K=16 MMAs (a commit per 8, never waits): the pipe's
//           queue stays full, so most tcgen05.mma issues block
//   mode 2: warp 1 issues groups of 8 and waits for each group's commit (queue never backs up)
//   mode 3: as 1, but from warp 0 on SMSP 0 — whose softmax warps are then the slow ones?
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mea;

template <unsigned kPoly>
__global__ void __launch_bounds__(640, 1) kern(int mode, int iters, float cin, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar, bar2;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = 0x3c;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); done = 0; }
  if (warp == 2) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  const int issuer = mode == 3 ? 0 : 1;
  if (warp < 4) {
    if (warp == issuer && mode != 0) {
      const uint64_t a = shfl0_u64(sdesc_sw128(smem_u32(sm), 16, 1024));
      const uint64_t b = shfl0_u64(sdesc_sw128(smem_u32(sm + 32768), 16, 1024));
      int it = 0;
      while (!done && it < 200000) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if (mode == 4) umma_ts(tm, tm + 256 + kk * 8, b + kk * 128, idesc_bf16_f32(128, 64, false, true), 1);
            else if (mode == 5) umma_ts(tm, tm + 256 + (kk & 3) * 8, b + (kk & 3) * 2, idesc_bf16_f32(128, 96, false, false), 1);
            else umma_ss(tm, a + (kk & 3) * 2, b + (kk & 3) * 2, idesc_bf16_f32(128, 96, false, false), 1);
          }
          umma_commit(&bar);
        }
        __syncwarp();
        if (mode == 2) mbar_wait(&bar, it & 1);
        ++it;
      }
      if (threadIdx.x % 32 == 0) out[148 * 16 + blockIdx.x] = it;
    }
  } else {
    const int sw = warp - 4;
    float v[48];
#pragma unroll
    for (int i = 0; i < 48; ++i) v[i] = cin * (float)((threadIdx.x * 7 + i) & 15) - 8.f;
    uint32_t acc = 0;
    float l = 0.f;
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const float2 c2 = make_float2(cin, cin), nm2 = make_float2(-1.f, -1.f);
      float2 rs = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), c2, nm2);
        const float2 e = ((kPoly >> i) & 1u) ? exp2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
        rs = __fadd2_rn(rs, e);
        acc ^= pack_bf16x2(e.x, e.y);
      }
      l += rs.x + rs.y;
#pragma unroll
      for (int i = 0; i < 48; ++i) v[i] += 1e-7f;
    }
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + sw] = t1 - t0;
    sink[blockIdx.x * 640 + threadIdx.x] = l + (float)acc;
  }
  // softmax warps done -> stop the issuer
  if (warp >= 4) {
    named_bar_sync(1, blockDim.x - 128);
    if (threadIdx.x == 128) done = 1;
  }
  __syncthreads();
  if (mode != 0) {
    // make sure every issued MMA has completed before dealloc
    if (warp == issuer) {
      if (elect_one()) umma_commit(&bar2);
      __syncwarp();
      mbar_wait(&bar2, 0);
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

template <unsigned P>
void run(int mode, const char* name, unsigned long long* d, float* sink, int nthr = 640) {
  cudaFuncSetAttribute(kern<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 148 * 17 * 8);
    kern<P><<<148, nthr, 120 * 1024>>>(mode, 400, 0.01f, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  }
  unsigned long long h[148 * 17];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double smsp[4] = {0, 0, 0, 0};
  const int nsw = nthr / 32 - 4;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < nsw; ++w) smsp[(w + 4) & 3] += h[b * 16 + w] / (148.0 * nsw / 4);
  double groups = 0;
  for (int b = 0; b < 148; ++b) groups += h[148 * 16 + b] / 148.0;
  const double per_pair = 1.0 / (400.0 * 24.0);
  printf("%2d sw poly %2d/24  %-36s cyc/pair/warp SMSP0..3: %6.2f %6.2f %6.2f %6.2f  MMA cyc/instr %.1f\n", nthr / 32 - 4, __builtin_popcount(P),
         name, smsp[0] * per_pair, smsp[1] * per_pair, smsp[2] * per_pair, smsp[3] * per_pair,
         mode ? (smsp[0] / (groups * 8)) : 0.0);
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 148 * 17 * 8);
  float* sink; cudaMalloc(&sink, 148 * 640 * 4);
  const char* names[] = {"no MMAs", "SS N=96 streaming (warp 1)", "SS N=96 group+wait", "SS N=96 streaming (warp 0)",
                         "TS N=64 streaming", "TS N=96 K-major B streaming"};
  for (int m : {0, 1}) run<0x00080080u>(m, names[m], d, sink, 384);
  for (int m : {0, 1}) run<0x00410041u>(m, names[m], d, sink, 384);
  for (int m : {0, 1}) run<0x00888888u>(m, names[m], d, sink, 384);
  for (int m : {0, 1}) run<0x00080080u>(m, names[m], d, sink, 256);
  const int modes[] = {0, 1, 4, 5};
  for (int m : modes) run<0x00080080u>(m, names[m], d, sink);
  for (int m : {0, 1}) run<0u>(m, names[m], d, sink);
  for (int m : {0, 1}) run<0x00410041u>(m, names[m], d, sink);     // 4
  for (int m : {0, 1}) run<0x00249249u>(m, names[m], d, sink);     // 8 (every third)
  for (int m : {0, 1}) run<0x00924924u>(m, names[m], d, sink);     // 8, other phase
  for (int m : {0, 1}) run<0x00888888u>(m, names[m], d, sink);     // 6
  for (int m : {0, 1}) run<0x00555555u>(m, names[m], d, sink);     // 12
  return 0;
}
