// MUFU.EX2 characterisation on sm_100a.
// (1) accuracy of ex2.approx.ftz.f32 over every fp32 a in [-1,0) (64 segments)
//     and per binade of |a| below 1/64, vs the correctly rounded 2^a and vs
//     the exact 2^a; (2) throughput of MUFU.EX2, FFMA, FFMA2 per clk per SM.
// Dev tool only: not part of the product path.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ float ex2a(float a) {
  float r; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a)); return r;
}

struct Acc { double n, sum_ulp, sum_rel, max_ulp, n_lo, n_hi; };

// bits in [b0, b1): negative floats (sign bit set) with magnitude bits m.
__global__ void acc_kernel(uint32_t m0, uint32_t m1, Acc* out) {
  double s_ulp = 0, s_rel = 0, mx = 0, n = 0, lo = 0, hi = 0;
  for (uint64_t m = m0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < m1;
       m += (uint64_t)gridDim.x * blockDim.x) {
    float a = __uint_as_float(0x80000000u | (uint32_t)m);
    float e = ex2a(a);
    double ex = exp2((double)a);
    float cr = __double2float_rn(ex);
    double du = (double)((int32_t)__float_as_uint(e) - (int32_t)__float_as_uint(cr));
    s_ulp += du; s_rel += (double)e / ex - 1.0; n += 1;
    if (du < 0) lo += 1; if (du > 0) hi += 1;
    mx = fmax(mx, fabs(du));
  }
  // block reduce via atomics (fine for a probe)
  __shared__ double sh[6];
  if (threadIdx.x < 6) sh[threadIdx.x] = 0;
  __syncthreads();
  for (int o = 16; o; o >>= 1) {
    s_ulp += __shfl_xor_sync(~0u, s_ulp, o); s_rel += __shfl_xor_sync(~0u, s_rel, o);
    n += __shfl_xor_sync(~0u, n, o); lo += __shfl_xor_sync(~0u, lo, o);
    hi += __shfl_xor_sync(~0u, hi, o); mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sh[0], n); atomicAdd(&sh[1], s_ulp); atomicAdd(&sh[2], s_rel);
    atomicAdd(&sh[4], lo); atomicAdd(&sh[5], hi);
    unsigned long long* p = (unsigned long long*)&sh[3];
    atomicMax(p, __double_as_longlong(mx));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&out->n, sh[0]); atomicAdd(&out->sum_ulp, sh[1]); atomicAdd(&out->sum_rel, sh[2]);
    atomicAdd(&out->n_lo, sh[4]); atomicAdd(&out->n_hi, sh[5]);
    atomicMax((unsigned long long*)&out->max_ulp, __double_as_longlong(sh[3]));
  }
}

__global__ void tp_mufu(float* out, int iters, long long* cyc) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = 0.1f * (threadIdx.x + k);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = ex2a(-x[k]);
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void tp_ffma(float* out, int iters, float a, float b, long long* cyc) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = 0.1f * (threadIdx.x + k);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void tp_ffma2(float* out, int iters, float a, float b, long long* cyc) {
  unsigned long long x[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av), B = *reinterpret_cast<unsigned long long*>(&bv);
  for (int k = 0; k < 8; ++k) { float2 v = make_float2(0.1f * (threadIdx.x + k), 0.2f * k); x[k] = *reinterpret_cast<unsigned long long*>(&v); }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(A), "l"(B));
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) { float2 v = *reinterpret_cast<float2*>(&x[k]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// mixed: per iteration 1 MUFU + 8 FFMA-pipe ops per chain (the K6 pair recipe shape)
__global__ void tp_mix(float* out, int iters, float s, long long* cyc) {
  float x[8], acc[8];
  for (int k = 0; k < 8; ++k) { x[k] = 0.01f * (threadIdx.x + k); acc[k] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float d = x[k] - s; float u = d * s; float t = u * u; float a = t * -0.72134752f;
      float e = ex2a(a); float p = t - 15.f; p = fmaf(p, t, 45.f); p = fmaf(p, t, -15.f);
      acc[k] = fmaf(p, e, acc[k]); x[k] += 1e-3f;
    }
  long long t1 = clock64();
  float r = 0; for (int k = 0; k < 8; ++k) r += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\"}\n", p.name, sms, p.major, p.minor);
  Acc* d; CK(cudaMalloc(&d, sizeof(Acc) * 200));
  CK(cudaMemset(d, 0, sizeof(Acc) * 200));
  // 64 segments of [-1,0): seg k = a in [-(k+1)/64, -k/64)
  int nseg = 0;
  uint32_t lo_bits[200], hi_bits[200]; const char* lab[200]; char buf[200][48];
  for (int k = 0; k < 64; ++k) {
    float amin = (float)k / 64.f, amax = (float)(k + 1) / 64.f;  // magnitudes
    uint32_t b0 = (k == 0) ? 0u : __builtin_bit_cast(uint32_t, amin);
    uint32_t b1 = __builtin_bit_cast(uint32_t, amax);
    lo_bits[nseg] = b0; hi_bits[nseg] = b1; snprintf(buf[nseg], 48, "seg64_%02d", k); lab[nseg] = buf[nseg]; ++nseg;
  }
  // binades of |a| below 1/64: [2^-(e+1), 2^-e) for e = 6..30
  for (int e = 6; e <= 30; ++e) {
    uint32_t b0 = __builtin_bit_cast(uint32_t, ldexpf(1.f, -(e + 1)));
    uint32_t b1 = __builtin_bit_cast(uint32_t, ldexpf(1.f, -e));
    lo_bits[nseg] = b0; hi_bits[nseg] = b1; snprintf(buf[nseg], 48, "binade_2^-%d", e + 1); lab[nseg] = buf[nseg]; ++nseg;
  }
  // coarse segments for larger |a|: [1,2),[2,4),...,[64,128)
  for (int e = 0; e < 7; ++e) {
    uint32_t b0 = __builtin_bit_cast(uint32_t, ldexpf(1.f, e));
    uint32_t b1 = __builtin_bit_cast(uint32_t, ldexpf(1.f, e + 1));
    lo_bits[nseg] = b0; hi_bits[nseg] = b1; snprintf(buf[nseg], 48, "mag_[2^%d,2^%d)", e, e + 1); lab[nseg] = buf[nseg]; ++nseg;
  }
  for (int s = 0; s < nseg; ++s) acc_kernel<<<sms * 8, 256>>>(lo_bits[s], hi_bits[s], d + s);
  CK(cudaDeviceSynchronize());
  Acc h[200]; CK(cudaMemcpy(h, d, sizeof(Acc) * nseg, cudaMemcpyDeviceToHost));
  for (int s = 0; s < nseg; ++s)
    printf("{\"seg\":\"%s\",\"n\":%.0f,\"mean_ulp_vs_cr\":%.5f,\"frac_low\":%.5f,\"frac_high\":%.5f,\"max_ulp\":%.0f,\"mean_rel_vs_exact\":%.3e}\n",
           lab[s], h[s].n, h[s].sum_ulp / h[s].n, h[s].n_lo / h[s].n, h[s].n_hi / h[s].n, h[s].max_ulp, h[s].sum_rel / h[s].n);
  // throughput
  float* o; long long* cyc; CK(cudaMalloc(&o, sizeof(float) * sms * 64 * 1024)); CK(cudaMalloc(&cyc, 8 * sms * 64));
  int iters = 4096;
  for (int cfg = 0; cfg < 4; ++cfg) {
    int blocks = sms * 4, threads = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (cfg == 0) tp_mufu<<<blocks, threads>>>(o, iters, cyc);
      if (cfg == 1) tp_ffma<<<blocks, threads>>>(o, iters, 0.999f, 0.001f, cyc);
      if (cfg == 2) tp_ffma2<<<blocks, threads>>>(o, iters, 0.999f, 0.001f, cyc);
      if (cfg == 3) tp_mix<<<blocks, threads>>>(o, iters, 0.37f, cyc);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long hc[1024]; CK(cudaMemcpy(hc, cyc, 8 * blocks, cudaMemcpyDeviceToHost));
    long long mx = 0; for (int b = 0; b < blocks; ++b) mx = hc[b] > mx ? hc[b] : mx;
    double ops = (double)blocks * threads * iters * 8 * (cfg == 2 ? 2 : 1);
    // per-SM: 4 blocks per SM resident concurrently (256 thr, low regs)
    double per_clk_sm = ops / sms / (double)mx;
    const char* nm[4] = {"mufu_ex2", "ffma", "ffma2_lanes", "k6_pairs_scalar"};
    printf("{\"tp\":\"%s\",\"ms\":%.4f,\"max_cycles\":%lld,\"per_clk_per_sm\":%.3f,\"implied_mhz\":%.1f}\n",
           nm[cfg], ms, mx, per_clk_sm, (double)mx / (ms * 1e3));
  }
  return 0;
}
