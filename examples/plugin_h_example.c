/*
 * plugin_h_example.c -- the C ABI of libplugin.so used from plain C (no Python, no torch):
 * reads a float32 sample (raw little-endian file, or the toy data of PAPER.md P:51 when no file
 * is given), runs Algorithm 1 on the GPU, prints h and the intermediates.
 *   build:  gcc -O2 -I include examples/plugin_h_example.c -L paper_1505_02100_b200 -lplugin
 *           -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o plugin_h_example
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "plugin.h"

int main(int argc, char** argv) {
  static const float toy[8] = {0.0f, 1.0f, 1.1f, 1.5f, 1.9f, 2.8f, 2.9f, 3.5f};
  float* x = (float*)toy;
  long long n = 8;
  if (argc > 1) {
    FILE* f = fopen(argv[1], "rb");
    if (!f) { perror(argv[1]); return 2; }
    fseek(f, 0, SEEK_END);
    n = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    x = (float*)malloc(sizeof(float) * (size_t)n);
    if (fread(x, 4, (size_t)n, f) != (size_t)n) { fprintf(stderr, "short read\n"); return 2; }
    fclose(f);
  }
  /* device input and workspace: the caller owns all memory */
  float* d_x = NULL;
  void* d_ws = NULL;
  const size_t ws = plugin_workspace_bytes(n);
  if (cudaMalloc((void**)&d_x, sizeof(float) * (size_t)n) != cudaSuccess || cudaMalloc(&d_ws, ws) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 3;
  }
  cudaMemcpy(d_x, x, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice);
  plugin_result r;
  const plugin_status st = plugin_h_sync(d_x, n, &r, d_ws, ws, NULL);
  if (st == PLUGIN_E_INVALID || st == PLUGIN_E_CUDA) {
    fprintf(stderr, "plugin_h_sync: %d %s\n", (int)st, plugin_last_error());
    return 4;
  }
  printf("{\"n\": %lld, \"status\": %d, \"sigma\": %.17g, \"g1\": %.17g, \"psi6\": %.17g, \"g2\": %.17g, "
         "\"psi4\": %.17g, \"h\": %.17g, \"version\": \"%s\"}\n",
         n, r.status, r.sigma, r.g1, r.psi6, r.g2, r.psi4, r.h, plugin_version());
  cudaFree(d_x);
  cudaFree(d_ws);
  return r.status == PLUGIN_OK ? 0 : 1;
}
