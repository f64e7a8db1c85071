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
#ifdef PSI_EX2_EXACT  // A/B probe only: the correctly rounded 2^a (fp64), +0 below 2^-126 as ftz
  return a < -126.f ? 0.f : __double2float_rn(exp2((double)a));
#else
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
#endif
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

// 2^a on the FMA pipe for two lanes, a in [-126, 0] (callers clamp): a = n + f with n = rint(a)
// by the magic-number add (1.5 * 2^23), f in [-1/2, 1/2] exact, 2^f by a degree-5 minimax
// polynomial (relative error 7.5e-8; 2.3e-7 with fp32 Horner), 2^n added to the exponent field
// on the integer pipe.  8 FP32 lane-ops per lane (3 + 5 Horner) + 2 integer ops.
__device__ __forceinline__ u64 ex2_fma2(u64 a) {
  const u64 kMagic = 0x4B4000004B400000ull;  // 1.5 * 2^23
  const u64 r = add2(a, kMagic);             // rint(a) in the low mantissa bits
  const u64 f = sub2(a, sub2(r, kMagic));    // a - rint(a), exact
  u64 q = fma2(0x3AAE04733AAE0473ull, f, 0x3C1E86293C1E8629ull);  // c5 f + c4
  q = fma2(q, f, 0x3D635B723D635B72ull);     // + c3
  q = fma2(q, f, 0x3E75FC8C3E75FC8Cull);     // + c2
  q = fma2(q, f, 0x3F3172143F317214ull);     // + c1
  q = fma2(q, f, 0x3F8000013F800001ull);     // + c0
  float r0, r1, q0, q1;
  upk2(r, r0, r1);
  upk2(q, q0, q1);
  return pk2(__uint_as_float(__float_as_uint(q0) + (__float_as_uint(r0) << 23)),
             __uint_as_float(__float_as_uint(q1) + (__float_as_uint(r1) << 23)));
}

}  // namespace plg
