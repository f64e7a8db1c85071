// simd.cuh -- packed f32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2), MUFU.EX2 and an fp32->fp64
// conversion on the integer pipe, shared by the pairwise kernels (psi.cu, kde.cu).
// Product code: nothing here is shared with oracle/.
#pragma once
#include <cstdint>

namespace plg {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(u64 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float ex2(float a) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}

// float -> double on the integer (ALU) pipe.  cvt.f64.f32 (F2F) issues on the XU pipe,
// which MUFU.EX2 saturates; fp32 denormals and zero map to +-0, Inf/NaN are not expected
// (non-finite samples are rejected before the pass).
__device__ __forceinline__ double f32_to_f64_alu(float f) {
  const unsigned int b = __float_as_uint(f);
  const unsigned int mag = b & 0x7fffffffu;
  unsigned int hi = ((mag >> 3) + 0x38000000u) | (b & 0x80000000u);
  unsigned int lo = b << 29;
  const bool tiny = mag < 0x00800000u;
  hi = tiny ? (b & 0x80000000u) : hi;
  lo = tiny ? 0u : lo;
  return __hiloint2double((int)hi, (int)lo);
}

}  // namespace plg
