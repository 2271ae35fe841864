// tcgen05.mma issue patterns of the d = 64 forward, alone on an SM (one CTA per SM):
//   0: one warp, groups of 8 TS M=128 N=64 MMAs into one accumulator, one commit at the end
//   1: one warp, [4 TS N=64 (A = TMEM "Q", B K-major) -> S, commit] [4 TS N=64 (A = TMEM "P",
//      B MN-major) -> O, commit] repeated: the forward's QK / PV group pattern
//   2: as 1 from two warps (1 and 3) on separate S / O columns: the two query tiles' issuers
//   3: as 2, each warp waiting for its own previous group's commit before issuing the next
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <type_traits>
#include "ptx.cuh"
using namespace mea;

template <int PAT, int LOAD>
__global__ void __launch_bounds__(640, 1) kern(int groups, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar[2][3];
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = 0x3c;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 3; ++j) mbar_init(&bar[i][j], 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 2) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  const bool active = PAT >= 2 ? (warp == 1 || warp == 3) : warp == 1;
  if (active) {
    const int w = warp >> 1;
    const uint64_t bk = shfl0_u64(sdesc_sw128(smem_u32(sm + 16384 * w), 16, 1024));
    const uint64_t bv = shfl0_u64(sdesc_sw128(smem_u32(sm + 32768 + 16384 * w), 16, 1024));
    const uint32_t ds = tm + 128 * w, dO = tm + 320 + 64 * w, aq = tm + 448 + 32 * w, ap = tm + 256 + 32 * w;
    const uint32_t idk = idesc_bf16_f32(128, 64, false, false), idv = idesc_bf16_f32(128, 64, false, true);
    const unsigned long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (PAT == 3 && g > 0) mbar_wait(&bar[w][1], (g - 1) & 1);
      if (elect_one()) {
        if (PAT == 0) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) umma_ts(dO, ap + (kk & 3) * 8, bv + (kk & 3) * 128, idv, 1);
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_ts(ds, aq + kk * 8, bk + kk * 2, idk, kk > 0);
          umma_commit(&bar[w][0]);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_ts(dO, ap + kk * 8, bv + kk * 128, idv, 1);
          umma_commit(&bar[w][1]);
        }
        if (g == groups - 1) umma_commit(&bar[w][2]);
      }
      __syncwarp();
    }
    mbar_wait(&bar[w][2], 0);
    const unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 2 + w] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && LOAD) {
    float v[48];
#pragma unroll
    for (int i = 0; i < 48; ++i) v[i] = 0.01f * (float)((threadIdx.x * 7 + i) & 15) - 8.f;
    uint32_t acc = 0;
    float l = 0.f;
    const uint32_t lb = tm + ((uint32_t)((warp & 3) * 32 + ((warp >> 2) & 1) * 16) << 16);
    const int sel = (warp >> 3) & 1;
    const uint32_t lds = lb + (LOAD == 2 ? 128 * sel : 64 + 128 * sel), sts = lb + (LOAD == 2 ? 256 + 32 * sel : 64 + 128 * sel);
    while (!done) {
      uint32_t r[32];
      tmem_ld32_split<32>(lds, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += __uint_as_float(r[i]) * 1e-30f;
      const float2 c2 = make_float2(0.01f, 0.01f), nm2 = make_float2(-1.f, -1.f);
      float2 rs = make_float2(0.f, 0.f);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), c2, nm2);
        const float2 e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        rs = __fadd2_rn(rs, e);
        pk[i] = pack_bf16x2(e.x, e.y);
      }
      tmem_st16_split<16>(sts, pk);
      tmem_st_wait();
      l += rs.x + rs.y;
      acc ^= pk[3];
    }
    if (l == 12345.f) out[0] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

template <int P, int L>
void run(const char* name, unsigned long long* d) {
  const int G = 2000;
  cudaFuncSetAttribute(kern<P, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 148 * 2 * 8);
    kern<P, L><<<148, 640, 120 * 1024>>>(G, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  }
  unsigned long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; int n = 0;
  for (int i = 0; i < 296; ++i) if (h[i]) { s += h[i]; ++n; }
  s /= n;
  const int warps = P >= 2 ? 2 : 1;
  printf("%-60s %6.1f cycles per MMA per SM (ideal 32)\n", name, s / (G * 8.0 * warps));
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  unsigned long long* d; cudaMalloc(&d, 296 * 8);
  run<0, 0>("8 TS N=64 into one accumulator per group", d);
  run<1, 0>("1 warp: 4 QK (TS, B K-major) commit, 4 PV (TS, B MN) commit", d);
  run<2, 0>("2 warps: the same pattern each", d);
  run<3, 0>("2 warps: each waits for its previous PV group", d);
  printf("with 16 softmax-like warps (TMEM ld 32 cols, 16 pairs of exps, st 16 cols) on other columns:\n");
  run<0, 1>("8 TS N=64 into one accumulator per group", d);
  run<2, 1>("2 warps: the same pattern each", d);
  run<3, 1>("2 warps: each waits for its previous PV group", d);
  printf("... with the softmax loads/stores on the S / P columns the MMAs use:\n");
  run<2, 2>("2 warps: the same pattern each", d);
  return 0;
}
