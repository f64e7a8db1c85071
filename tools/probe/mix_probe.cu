// Dev probe: achievable MUFU.EX2 rate when mixed with NF packed FP32x2 ops per 2 MUFU
// (the psi pair2 shape: K6 = 8, K4 = 7, shifted K4 = 6), independent chains.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ float ex2a(float a) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 pk2(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk2(u64 v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
template <int NF, int CH>
__global__ void mix(float* out, int iters, long long* cyc) {
  u64 v[CH];
  for (int k = 0; k < CH; ++k) v[k] = pk2(-0.001f * (threadIdx.x + k), -0.002f * k);
  const u64 A = pk2(0.999f, 0.999f), B = pk2(-0.0001f, -0.0001f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      u64 x = v[k];
#pragma unroll
      for (int f = 0; f < NF - 1; ++f) x = fma2(x, A, B);
      float a0, a1; upk2(x, a0, a1);
      float e0 = ex2a(a0), e1 = ex2a(a1);
      v[k] = fma2(pk2(e0, e1), A, pk2(-1.f, -1.f));
    }
  }
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < CH; ++k) { float a, b; upk2(v[k], a, b); s += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int NF, int CH>
void run(const char* nm, int blocks_per_sm) {
  int sms = 148, iters = 2048, threads = 256;
  int blocks = sms * blocks_per_sm;
  float* o; long long* c; cudaMalloc(&o, 4 * blocks * threads); cudaMalloc(&c, 8 * blocks);
  mix<NF, CH><<<blocks, threads>>>(o, 16, c);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); mix<NF, CH><<<blocks, threads>>>(o, iters, c); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2048]; cudaMemcpy(h, c, 8 * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  double mufu = 2.0 * CH * iters * (double)threads * blocks;
  printf("{\"mix\":\"%s\",\"NF\":%d,\"chains\":%d,\"ctas_per_sm\":%d,\"mufu_per_clk_per_sm\":%.3f,\"frac_of_16\":%.4f,\"ms\":%.3f}\n",
         nm, NF, CH, blocks_per_sm, mufu / sms / mx, mufu / sms / mx / 16.0, ms);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1, 8>("mufu_only", 2);
  run<6, 8>("shifted_K4", 2);
  run<7, 8>("K4", 2);
  run<8, 8>("K6", 2);
  run<7, 8>("K4", 4);
  run<8, 8>("K6", 4);
  run<7, 16>("K4", 2);
  run<8, 16>("K6", 2);
  run<9, 8>("K6+1", 2);
  return 0;
}
