/*
 * mea_example.c — the C ABI of libmea.so (include/mea.h) from plain C99: seeded synthetic
 * inputs, forward with the lse residual, backward from lse, a single-query (decode) call, and
 * one error path. Prints a few output values so a caller can compare them with the Python
 * binding (tests/test_abi.py builds it; tests/test_gpu_probe.py runs it on a B200).
 *
 *   gcc -std=c99 -Wall -I include -I /usr/local/cuda/include examples/mea_example.c \
 *       -L paper_2112_05682_b200 -lmea -L /usr/local/cuda/lib64 -lcudart -o mea_example
 *   LD_LIBRARY_PATH=paper_2112_05682_b200 ./mea_example
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "mea.h"

#define CHECK(call)                                                                              \
  do {                                                                                           \
    mea_status_t st_ = (call);                                                                   \
    if (st_ != MEA_OK) {                                                                         \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, mea_status_string(st_), mea_last_error_detail()); \
      return 1;                                                                                  \
    }                                                                                            \
  } while (0)
#define CUDA(call)                                                                               \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) {                                                                     \
      fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));                         \
      return 1;                                                                                  \
    }                                                                                            \
  } while (0)

static float bf16_to_f32(unsigned short h) {
  union { unsigned int u; float f; } x;
  x.u = (unsigned int)h << 16;
  return x.f;
}

int main(void) {
  const int64_t B = 1, H = 2, n = 1000, d = 64;   /* ragged: not a multiple of any tile */
  const size_t elems = (size_t)(B * n * H * d);
  const float scale = 1.0f / sqrtf((float)d);
  void *q, *k, *v, *out, *dout, *dq, *dk, *dv, *ws = NULL, *sq_out, *sq_ws = NULL;
  float* lse;
  size_t ws_bytes = 0, sq_ws_bytes = 0;
  unsigned short h_out[8], h_dq[8], h_sq[8];
  float h_lse[4];
  int i;

  printf("%s\n", mea_version());
  CUDA(cudaMalloc(&q, elems * 2));
  CUDA(cudaMalloc(&k, elems * 2));
  CUDA(cudaMalloc(&v, elems * 2));
  CUDA(cudaMalloc(&dout, elems * 2));
  CUDA(cudaMalloc(&out, elems * 2));
  CUDA(cudaMalloc(&dq, elems * 2));
  CUDA(cudaMalloc(&dk, elems * 2));
  CUDA(cudaMalloc(&dv, elems * 2));
  CUDA(cudaMalloc((void**)&lse, (size_t)(B * H * n) * sizeof(float)));
  CUDA(cudaMalloc(&sq_out, (size_t)(B * H * d) * 2));

  /* the counter-based generator the tests use (seed 0; tensor ids 1..4 = q, k, v, dO) */
  CHECK(mea_fill_synthetic(q, (int64_t)elems, MEA_BF16, 0, 1, 0, NULL));
  CHECK(mea_fill_synthetic(k, (int64_t)elems, MEA_BF16, 0, 2, 0, NULL));
  CHECK(mea_fill_synthetic(v, (int64_t)elems, MEA_BF16, 0, 3, 0, NULL));
  CHECK(mea_fill_synthetic(dout, (int64_t)elems, MEA_BF16, 0, 4, 0, NULL));

  /* forward, default (online) schedule: no workspace */
  CHECK(mea_attention_fwd(q, k, v, out, B, H, n, n, d, MEA_BF16, MEA_BF16, scale, lse, 0, 0, NULL, 0, NULL));
  /* backward from the saved lse */
  CHECK(mea_attention_bwd_workspace_size(B, H, n, n, d, MEA_BF16, 1, &ws_bytes));
  CUDA(cudaMalloc(&ws, ws_bytes));
  CHECK(mea_attention_bwd(q, k, v, out, dout, dq, dk, dv, B, H, n, n, d, MEA_BF16, scale, lse, ws, ws_bytes, NULL));
  /* decode: the first query row of each head against all n keys (q row 0 of [B, n, H, d] is
     the [B, H, d] block at the start of q) */
  CHECK(mea_single_query_workspace_size(B, H, n, d, MEA_BF16, &sq_ws_bytes));
  CUDA(cudaMalloc(&sq_ws, sq_ws_bytes));
  CHECK(mea_single_query_fwd(q, k, v, sq_out, B, H, n, d, MEA_BF16, MEA_BF16, scale, sq_ws, sq_ws_bytes, NULL));
  /* an error is a status code, nothing launched */
  if (mea_attention_fwd(q, k, v, out, B, H, n, 0, d, MEA_BF16, MEA_BF16, scale, NULL, 0, 0, NULL, 0, NULL) !=
      MEA_ERR_EMPTY_KEYS) {
    fprintf(stderr, "n_k = 0 should be MEA_ERR_EMPTY_KEYS\n");
    return 1;
  }

  CUDA(cudaDeviceSynchronize());
  CUDA(cudaMemcpy(h_out, out, sizeof(h_out), cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(h_dq, dq, sizeof(h_dq), cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(h_sq, sq_out, sizeof(h_sq), cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(h_lse, lse, sizeof(h_lse), cudaMemcpyDeviceToHost));
  printf("out");
  for (i = 0; i < 8; ++i) printf(" %.8e", bf16_to_f32(h_out[i]));
  printf("\nlse");
  for (i = 0; i < 4; ++i) printf(" %.8e", h_lse[i]);
  printf("\ndq");
  for (i = 0; i < 8; ++i) printf(" %.8e", bf16_to_f32(h_dq[i]));
  printf("\nsq");
  for (i = 0; i < 8; ++i) printf(" %.8e", bf16_to_f32(h_sq[i]));
  printf("\n");

  cudaFree(q); cudaFree(k); cudaFree(v); cudaFree(dout); cudaFree(out); cudaFree(dq); cudaFree(dk);
  cudaFree(dv); cudaFree(lse); cudaFree(ws); cudaFree(sq_out); cudaFree(sq_ws);
  return 0;
}
