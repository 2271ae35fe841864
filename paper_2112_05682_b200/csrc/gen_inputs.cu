// gen_inputs.cu — device-side synthetic input generator (not part of the method).
//
// Independent implementation of the counter-based Irwin-Hall(12) generator specified in
// synth/gen.py (splitmix64 finaliser, twelve 16-bit limbs, x = (sum + 6)/65536 - 6, exact in
// f32; bf16 by round-to-nearest-even). Lets the bench and tests synthesise the paper's
// N(0,1)-like inputs in HBM without a host copy; tests check bit equality.
#include <cuda_bf16.h>

#include "internal.h"

namespace mea {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(void* dst, int64_t numel, int bf16, uint64_t base, int64_t offset) {
  const uint64_t G = 0x9E3779B97F4A7C15ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)(offset + i);
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const uint64_t z = mix64(base + (3ull * idx + (uint64_t)(r + 1)) * G);
      acc += (uint32_t)(z & 0xFFFF) + (uint32_t)((z >> 16) & 0xFFFF) + (uint32_t)((z >> 32) & 0xFFFF) +
             (uint32_t)(z >> 48);
    }
    // exact: acc + 6 < 2^20 fits the f32 mantissa; /65536 and -6 are exact
    const float x = ((float)(acc + 6u)) * (1.0f / 65536.0f) - 6.0f;
    if (bf16) static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(x);
    else static_cast<float*>(dst)[i] = x;
  }
}

}  // namespace

cudaError_t launch_fill_synthetic(void* dst, int64_t numel, int bf16, uint64_t seed, uint32_t tid, int64_t offset,
                                  cudaStream_t s) {
  const uint64_t base = [&] {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + (uint64_t)tid * 0xD1B54A32D192ED03ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }();
  int64_t blocks = (numel + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, numel, bf16, base, offset);
  return cudaGetLastError();
}

}  // namespace mea
