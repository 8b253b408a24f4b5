/* stack_demo.c -- using the BrainSlug C ABI (include/bs.h) from plain C99, no Python/PyTorch.
 *
 * Plans the ResNet stem stack BN -> ReLU -> MaxPool3x3/s2/p1 on (N, 64, 112, 112) fp32 NCHW,
 * executes it on the default stream with bs_execute and, end to end, with bs_execute_host
 * (pinned host buffers), and prints the output checksum of both (they must agree).
 *
 *   gcc -std=c99 -O2 -Iinclude -I/usr/local/cuda/include examples/stack_demo.c \
 *       -Lpaper_1804_08378_b200 -lbrainslug -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1804_08378_b200 -o /tmp/stack_demo && /tmp/stack_demo 8
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "bs.h"

#define CHECK(x)                                                                      \
  do {                                                                                \
    bs_status st_ = (x);                                                              \
    if (st_ != BS_OK) {                                                               \
      fprintf(stderr, "%s: %s: %s\n", #x, bs_status_string(st_), bs_last_error());    \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 8, C = 64, H = 112, W = 112;
  float gamma[64], beta[64], mean[64], var[64];
  for (int c = 0; c < C; ++c) {   /* any inference BatchNorm parameters */
    gamma[c] = 1.0f + 0.01f * c;
    beta[c] = 0.05f * (c % 7) - 0.1f;
    mean[c] = 0.02f * (c % 5);
    var[c] = 0.5f + 0.01f * c;
  }
  bs_layer_desc layers[3] = {{0}};
  layers[0].kind = BS_OP_BATCHNORM;
  layers[0].eps = 1e-5f;
  layers[0].gamma = gamma;
  layers[0].beta = beta;
  layers[0].running_mean = mean;
  layers[0].running_var = var;
  layers[1].kind = BS_OP_RELU;
  layers[2].kind = BS_OP_MAXPOOL;
  layers[2].kernel_h = layers[2].kernel_w = 3;
  layers[2].stride_h = layers[2].stride_w = 2;
  layers[2].pad_h = layers[2].pad_w = 1;

  bs_plan* plan = NULL;
  bs_shape in_shape = {N, C, H, W};
  CHECK(bs_plan_create(layers, 3, in_shape, NULL, &plan));
  bs_plan_info info;
  CHECK(bs_plan_query(plan, &info));
  const size_t n_in = (size_t)(N * C * H * W), n_out = (size_t)(info.out.n * info.out.c * info.out.h * info.out.w);
  printf("plan: (%lld,%lld,%lld,%lld) -> (%lld,%lld,%lld,%lld), %d launch(es), %.1f MB algorithmic\n",
         (long long)N, (long long)C, (long long)H, (long long)W, (long long)info.out.n, (long long)info.out.c,
         (long long)info.out.h, (long long)info.out.w, info.n_launches,
         (info.alg_bytes_read + info.alg_bytes_written) / 1e6);

  float *h_in, *h_out, *d_in, *d_out;
  if (cudaMallocHost((void**)&h_in, n_in * 4) != cudaSuccess || cudaMallocHost((void**)&h_out, n_out * 4) != cudaSuccess ||
      cudaMalloc((void**)&d_in, n_in * 4) != cudaSuccess || cudaMalloc((void**)&d_out, n_out * 4) != cudaSuccess) {
    fprintf(stderr, "CUDA allocation failed\n");
    return 1;
  }
  for (size_t i = 0; i < n_in; ++i) h_in[i] = (float)((i * 2654435761u) % 2001u) / 1000.0f - 1.0f;

  /* device-resident execution */
  cudaMemcpy(d_in, h_in, n_in * 4, cudaMemcpyHostToDevice);
  CHECK(bs_execute(plan, d_in, d_out, 0));
  cudaMemcpy(h_out, d_out, n_out * 4, cudaMemcpyDeviceToHost);
  double s1 = 0;
  for (size_t i = 0; i < n_out; ++i) s1 += h_out[i];

  /* end to end from host buffers (copies pipelined with the kernels) */
  const float* h_inputs[1] = {h_in};
  float* d_inputs[1] = {d_in};
  CHECK(bs_execute_host(plan, h_inputs, 1, h_out, d_inputs, d_out, 0, 0));
  cudaStreamSynchronize(0);
  double s2 = 0;
  for (size_t i = 0; i < n_out; ++i) s2 += h_out[i];

  printf("checksum device=%.6f host=%.6f %s\n", s1, s2, s1 == s2 ? "OK" : "MISMATCH");
  bs_plan_destroy(plan);
  cudaFree(d_in);
  cudaFree(d_out);
  cudaFreeHost(h_in);
  cudaFreeHost(h_out);
  return s1 == s2 ? 0 : 1;
}
