// Throughput of ex2.approx (MUFU) vs an FMA-pipe polynomial exp2, per SM, vs warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f); x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(f, make_float2(0.05517164f, 0.05517164f), make_float2(0.24261114f, 0.24261114f));
  q = __ffma2_rn(q, f, make_float2(0.69326097f, 0.69326097f));
  q = __ffma2_rn(q, f, make_float2(0.99992806f, 0.99992806f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}

__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t cvt_h2(float2 v) { uint32_t y; asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(y) : "f"(v.x), "f"(v.y)); return y; }

template <int MODE>
__global__ void kern(float* out, int iters) {
  float2 v[8];
  for (int i = 0; i < 8; ++i) v[i] = make_float2(-0.001f * (threadIdx.x + i), -0.002f * i);
  float2 acc = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float2 e;
      if (MODE == 0) e = make_float2(ex2(v[i].x), ex2(v[i].y));
      else if (MODE == 1) e = poly2(v[i]);
      else {  // packed half-precision: 2 exps per instruction (+ the f32 -> f16x2 conversion)
        const uint32_t h = cvt_h2(v[i]);
        const uint32_t r = MODE == 2 ? ex2h2(h) : ex2bf2(h);
        e = make_float2(__uint_as_float(r << 16), __uint_as_float(r & 0xffff0000u));
      }
      acc = __fadd2_rn(acc, e);
      v[i].x -= 1e-7f; v[i].y -= 1e-7f;
    }
  }
  if (acc.x == 123.f) out[0] = acc.y;
}

int main() {
  float* d; cudaMalloc(&d, 4);
  const int iters = 4096;
  const char* names[4] = {"mufu f32  ", "poly      ", "f16x2     ", "bf16x2    "};
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto k = mode == 0 ? kern<0> : mode == 1 ? kern<1> : mode == 2 ? kern<2> : kern<3>;
      k<<<148, warps * 32>>>(d, iters);
      cudaEventRecord(a);
      k<<<148, warps * 32>>>(d, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double exps = 148.0 * warps * 32 * iters * 16;
      printf("%s warps/SM=%2d: %.3f ms  %.1f exp/clk/SM (at 1.9 GHz)\n", names[mode], warps, ms,
             exps / (ms * 1e-3) / 148 / 1.9e9);
    }
  return 0;
}
