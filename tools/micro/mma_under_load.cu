// tcgen05.mma throughput of the forward's operand forms with and without 16 softmax warps running
// the exponential loop on the same SM (640 threads, one CTA per SM): does softmax traffic (MUFU,
// TMEM loads/stores) slow the tensor pipe? Warp 1 issues G groups of 8 MMAs back to back (one
// commit at the end) and times them; with load, warps 4-19 run the exponential loop until the
// issuer is done (optionally with tcgen05.ld / st traffic of the forward's size per pair).
//   form 0: SS M=128 N=96 K=16 (Q K^T)   1: TS M=128 N=64 (P V)   2: TS M=128 N=96, B K-major (Q in TMEM)
//   load 0: none   1: exp loop   2: exp loop + tcgen05.ld/st of the forward's per-tile volume
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mea;

template <int form, int load>
__global__ void __launch_bounds__(640, 1) kern(int groups, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = 0x3c;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 2) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  if (warp == 1) {
    const uint64_t a = shfl0_u64(sdesc_sw128(smem_u32(sm), 16, 1024));
    const uint64_t b = shfl0_u64(sdesc_sw128(smem_u32(sm + 32768), 16, 1024));
    const unsigned long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (form == 0) umma_ss(tm, a + (kk & 3) * 2, b + (kk & 3) * 2, idesc_bf16_f32(128, 96, false, false), 1);
          else if (form == 1) umma_ts(tm, tm + 256 + (kk & 3) * 8, b + kk * 128, idesc_bf16_f32(128, 64, false, true), 1);
          else umma_ts(tm, tm + 256 + (kk & 3) * 8, b + (kk & 3) * 2, idesc_bf16_f32(128, 96, false, false), 1);
        }
        if (g == groups - 1) umma_commit(&bar);
      }
      __syncwarp();
    }
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && load) {
    float v[48];
#pragma unroll
    for (int i = 0; i < 48; ++i) v[i] = 0.01f * (float)((threadIdx.x * 7 + i) & 15) - 8.f;
    uint32_t acc = 0;
    float l = 0.f;
    const uint32_t lb = tm + ((uint32_t)((warp & 3) * 32 + ((warp >> 2) & 1) * 16) << 16) + 384;
    while (!done) {
      if (load == 2) {  // the forward's TMEM traffic: 48 columns loaded, 24 stored per 24 pairs
        uint32_t r[32];
        tmem_ld32_split<48>(lb, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += __uint_as_float(r[i]) * 1e-30f;
      }
      const float2 c2 = make_float2(0.01f, 0.01f), nm2 = make_float2(-1.f, -1.f);
      float2 rs = make_float2(0.f, 0.f);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), c2, nm2);
        const float2 e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        rs = __fadd2_rn(rs, e);
        const uint32_t pp = pack_bf16x2(e.x, e.y);
        if (i < 16) pk[i] = pp; else acc ^= pp;
      }
      if (load == 2) {
        tmem_st16_split<24>(lb + 64, pk);
        tmem_st_wait();
      }
      l += rs.x + rs.y;
#pragma unroll
      for (int i = 0; i < 48; ++i) v[i] += 1e-7f;
    }
    sink[blockIdx.x * 640 + threadIdx.x] = l + (float)acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  float* sink; cudaMalloc(&sink, 148 * 640 * 4);
  const char* fn[] = {"SS N=96 (QK)", "TS N=64 (PV)", "TS N=96 (QK, Q in TMEM)"};
  const int nn[] = {96, 64, 96};
  const char* ln[] = {"alone", "+16 exp warps", "+16 exp warps + TMEM ld/st"};
  auto run = [&](auto F, auto L) {
      constexpr int f = decltype(F)::value, l = decltype(L)::value;
      const int G = 2000;
      cudaFuncSetAttribute(kern<f, l>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
      for (int rep = 0; rep < 2; ++rep) {
        kern<f, l><<<148, 640, 120 * 1024>>>(G, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
      }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double s = 0;
      for (int b = 0; b < 148; ++b) s += h[b] / 148.0;
      const double per = s / (G * 8.0), ideal = 128.0 * nn[f] * 16 / 4096.0;
      printf("%-26s %-28s %6.1f cycles per MMA (ideal %4.1f: %3.0f%%)\n", fn[f], ln[l], per, ideal, 100 * ideal / per);
  };
  using Z = std::integral_constant<int, 0>; using O = std::integral_constant<int, 1>; using T = std::integral_constant<int, 2>;
  run(Z{}, Z{}); run(Z{}, O{}); run(Z{}, T{});
  run(O{}, Z{}); run(O{}, O{}); run(O{}, T{});
  run(T{}, Z{}); run(T{}, O{}); run(T{}, T{});
  return 0;
}
