// psi_tile.cuh -- one T x T tile (T = 256 R) of the pair triangle of Steps IV/VI
// (Eq. 5-7), shared by the persistent pass kernel (psi.cu) and the fused
// small-n kernel (fused.cu) so both give bit-identical tile sums.  See psi.cu for the
// arithmetic and DESIGN.md §6 for the numerics.  Product code: nothing here is shared
// with oracle/.
#pragma once
#include "common.cuh"
#include "simd.cuh"

namespace plg {

// fp32 chunk length (j per flush to fp64) and unroll of the j loop; -D overrides are tuning only
#ifndef PSI_CH
#define PSI_CH 64
#endif
#ifndef PSI_UNROLL
#define PSI_UNROLL 16
#endif
#ifndef PSI_CENTER
#define PSI_CENTER 1  // the centred FMA form of u; 0: difference first (A/B only)
#endif
constexpr int kPsiUnroll = PSI_UNROLL;

// packed constants {v, v}
#define PK(v) ((((u64)__float_as_uint(v)) << 32) | (u64)__float_as_uint(v))

// per-row dither: phase p_i in (-2, -1] (exact fp32, 24 random bits) and scale offset k_i
__device__ __forceinline__ unsigned int row_hash(int64_t i) { return (unsigned int)i * 2654435769u; }
__device__ __forceinline__ float row_phase(int64_t i) {
  return -1.0f - (float)(row_hash(i) >> 8) * (1.0f / 16777216.0f);
}
// Antithetic scale dither: s_i = s + k_i ulp(s) with k_i uniform in [-A, A]
// per row pair and k_(2m+1) = -k_(2m), A = scale_dither_amp(n) = min(n / 16, 128).  The dither
// spreads the fp32 rounding of u, t, a and P(t) over 2A + 1 scales, so the repeated differences of
// a discretised sample do not all round the same way; the dilation it applies to each row
// (<= A ulp <= 7.7e-6 relative) cancels to first order between the two rows of a pair (adjacent
// in sorted order: equal or nearly equal values), leaving a second-order effect ~ (A ulp)^2.  The
// cancellation needs neighbouring rows closer than a bandwidth, hence the smaller A at small n.
constexpr int kScaleDither = 128;
__host__ __device__ __forceinline__ int scale_dither_amp(int64_t n) {
  return n >= 16 * kScaleDither ? kScaleDither : (int)(n >> 4);
}
__device__ __forceinline__ int row_scale_offset(int64_t i, int amp) {
  unsigned int h = ((unsigned int)(i >> 1) * 0x85EBCA6Bu) ^ 0x9E3779B9u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 13;
  const int k = (int)(h % (unsigned int)(2 * amp + 1)) - amp;
  return (i & 1) ? -k : k;
}
// s_i = s + k_i ulp(s), exactly (|k_i| << 2^23): symmetric in k_i also when s - |k_i| ulp(s) falls
// below a power of two (adding k_i to the bit pattern would step by ulp(s)/2 there, a one-sided
// dilation: measured -1e-5 on psi at s = 1)
__device__ __forceinline__ float dither_ulp(float s) {
  const unsigned int e = __float_as_uint(s) & 0x7f800000u;
  return e > (23u << 23) ? __uint_as_float(e - (23u << 23)) : 0.f;  // no dither for s < 2^-103
}
__device__ __forceinline__ float dithered_scale(float s, int64_t i, int64_t n) {
  return __fmaf_rn((float)row_scale_offset(i, scale_dither_amp(n)), dither_ulp(s), s);
}

// He_r(u) for even r as a polynomial in t = u^2 by Horner, monic, exact integer coefficients
// (probabilists' Hermite; K^(r)(u) = He_r(u) phi(u), r = 4, 6: the printed polynomials of
// Steps VI/IV).  All coefficients are exact in fp32 (< 2^24).
template <int ORDER>
__device__ __forceinline__ u64 hermite_t(u64 t) {
  u64 p;
  if (ORDER == 2) {
    p = add2(t, 0xBF800000BF800000ull);      // t - 1
  } else if (ORDER == 4) {
    p = add2(t, 0xC0C00000C0C00000ull);      // t - 6
    p = fma2(p, t, 0x4040000040400000ull);   // (t - 6) t + 3
  } else if (ORDER == 6) {
    p = add2(t, 0xC1700000C1700000ull);      // t - 15
    p = fma2(p, t, 0x4234000042340000ull);   // (t - 15) t + 45
    p = fma2(p, t, 0xC1700000C1700000ull);   // ((t - 15) t + 45) t - 15
  } else if (ORDER == 8) {
    p = add2(t, 0xC1E00000C1E00000ull);      // t - 28
    p = fma2(p, t, 0x4352000043520000ull);   // + 210
    p = fma2(p, t, 0xC3D20000C3D20000ull);   // - 420
    p = fma2(p, t, 0x42D2000042D20000ull);   // + 105
  } else if (ORDER == 10) {
    p = add2(t, 0xC2340000C2340000ull);      // t - 45
    p = fma2(p, t, 0x441D8000441D8000ull);   // + 630
    p = fma2(p, t, 0xC544E000C544E000ull);   // - 3150
    p = fma2(p, t, 0x4593A8004593A800ull);   // + 4725
    p = fma2(p, t, 0xC46C4000C46C4000ull);   // - 945
  } else {  // ORDER == 12
    p = add2(t, 0xC2840000C2840000ull);      // t - 66
    p = fma2(p, t, 0x44B9A00044B9A000ull);   // + 1485
    p = fma2(p, t, 0xC6589000C6589000ull);   // - 13860
    p = fma2(p, t, 0x474B0700474B0700ull);   // + 51975
    p = fma2(p, t, 0xC773A200C773A200ull);   // - 62370
    p = fma2(p, t, 0x46226C0046226C00ull);   // + 10395
  }
  return p;
}

// CENTER = false: xj, xi are raw sample values, u = (x_j - x_i) s (difference first).
// CENTER = true (PSI_CENTER): xj = fl(x_j - c) and xi = -fl(fl(x_i - c) s) for a tile centre c
// (psi_tile_centre), u = fma(xj, s, xi): one FP32 op instead of two.
// CLAMP: t = min(t, kTClamp) first.  Far pairs have e = +0 exactly either way, but without
// the clamp He_r(t) overflows fp32 to inf once |u| passes ~1600 (r = 12) ... ~2.6e6 (r = 6),
// and inf * 0 = NaN; with it He_r(t) <= 1024^6 stays finite and the term is exactly 0, so a
// clamped evaluation is bit-identical to an unclamped one wherever the latter is finite.
constexpr float kTClamp = 1024.f;  // a <= -0.7213 * 1024 - 1: ex2 -> +0
// "wide" tiles take the variant psi_tile_sum<..., WIDE = true>: difference first and clamped,
// inner loop rolled.  A tile is wide if its values span more than kClampSpan bandwidths
// (otherwise |u| <= span * s and He_12(1000^2) < 1e37: no overflow), or its row and column blocks
// together span more than kCenterSpan bandwidths (the centred form shifts each row by
// eps * |x_i - c| * s in u: fine for dense blocks, not for one that holds an
// outlier).  Both only occur with outliers or a tiny g; none of the BASELINE configurations has
// such a tile.
constexpr double kClampSpan = 1000.0;
constexpr double kCenterSpan = 64.0;
// rows in [a, b], columns in [p, q] (sorted: a <= b <= p <= q)
__device__ __forceinline__ bool psi_tile_wide(float a, float b, float p, float q, float s) {
  return (((double)b - (double)a) + ((double)q - (double)p)) * (double)s > kCenterSpan ||
         ((double)q - (double)a) * (double)s > kClampSpan;
}

// c rounded toward zero to a multiple of ulp(q), 0 <= c <= q (the grid is clamped to 2^-126: a
// coarser grid keeps every multiple a multiple of ulp(q))
__device__ __forceinline__ float round_to_ulp_of(float c, float q) {
  const int e = __float_as_int(q) & 0x7f800000;
  const float ulp = __int_as_float(e >= (24 << 23) ? e - (23 << 23) : 0x00800000);
  return truncf(__fdiv_rn(c, ulp)) * ulp;  // exact: ulp is a power of two
}

// Tile centre of the centred form.  Row block [a, b], column block [p, q] of the
// sorted sample (a <= b <= p <= q).  The centre c makes EVERY staged value fl(x_j - c) and every
// row value fl(x_i - c) exact, so the only per-value roundings left are the dithered ones of
// fl((x_i - c) s_i) and of the pair arithmetic (an inexact fl(x_j - c) is a fixed shift of a column
// value shared by all rows of the tile: systematic on discretised samples):
//   all values >= 0: c = a, or, if some value exceeds 2a, a rounded toward 0 to a multiple of
//     ulp(q): every x - c is then a multiple of ulp(x) no larger than x (or Sterbenz-exact);
//   all values <= 0: the mirror image, c = q (rounded toward 0 to a multiple of ulp(a));
//   the tile spans 0: c = 0 (x - 0 is exact).
// For every pair (i, j) of the tile |x_i - c| <= |x_j - x_i| + (b - a) + (q - p) (+ ulp(q)), so the
// dithered rounding of fl((x_i - c) s_i) stays within eps (|u| + (b - a + q - p) s) of u: tiles whose
// two blocks span more than kCenterSpan bandwidths together take the difference-first path
// (psi_tile_wide).
__device__ __forceinline__ float psi_tile_centre(float a, float q) {
  if (a >= 0.f) return (q <= 2.f * a) ? a : round_to_ulp_of(a, q);
  if (q <= 0.f) return (a >= 2.f * q) ? q : -round_to_ulp_of(-q, -a);
  return 0.f;
}

template <int ORDER, bool MASK, bool CENTER = false, bool CLAMP = false>
__device__ __forceinline__ void pair2(u64 xj, u64 xi, u64 s2, u64 ph, u64& acc, bool m0 = true, bool m1 = true) {
  const u64 c2 = 0xBF38AA3BBF38AA3Bull;  // {fp32(-log2(e)/2)} x 2 = -0.72134752f
  u64 u = CENTER ? fma2(xj, s2, xi) : mul2(sub2(xj, xi), s2);
  u64 t = mul2(u, u);
  if (CLAMP) {
    float t0, t1;
    upk2(t, t0, t1);
    t = pk2(fminf(t0, kTClamp), fminf(t1, kTClamp));
  }
  u64 a = fma2(t, c2, ph);
  float a0, a1;
  upk2(a, a0, a1);
  float e0 = ex2(a0), e1 = ex2(a1);
  if (MASK) {
    e0 = m0 ? e0 : 0.f;
    e1 = m1 ? e1 : 0.f;
  }
  u64 e = pk2(e0, e1);
  if (ORDER == 0) {  // K = phi: P = He_0 = 1
    acc = add2(acc, e);
    return;
  }
  acc = fma2(hermite_t<ORDER>(t), e, acc);
}

// pair2 with the exp on the FMA pipe (ex2_fma2) instead of MUFU.EX2, for the r = 4 hybrid
// (PSI_HYB4): results below 2^-126 become +0 as MUFU.EX2.ftz flushes them, so all-zero tiles
// stay exactly zero
template <int ORDER, bool CENTER>
__device__ __forceinline__ void pair2_fma(u64 xj, u64 xi, u64 s2, u64 ph, u64& acc) {
  const u64 c2 = 0xBF38AA3BBF38AA3Bull;
  u64 u = CENTER ? fma2(xj, s2, xi) : mul2(sub2(xj, xi), s2);
  u64 t = mul2(u, u);
  u64 a = fma2(t, c2, ph);
  float a0, a1, e0, e1;
  upk2(a, a0, a1);
  upk2(ex2_fma2(pk2(fmaxf(a0, -126.f), fmaxf(a1, -126.f))), e0, e1);
  e0 = (a0 < -126.f) ? 0.f : e0;
  e1 = (a1 < -126.f) ? 0.f : e1;
  acc = fma2(hermite_t<ORDER>(t), pk2(e0, e1), acc);
}

// r = 4 hybrid exp: 1 pair in 8 on the FMA pipe (the LP optimum for 6 FP32 ops + 1 ex2 per
// pair with the centred form: min(16 / (7/8), 128 / (6 + 8/8)) = 18.3 pairs/clk/SM); 0 = off:
// measured 4.24e12 vs 4.48e12 pairs/s (profiles/r01u_*) -- two saturated pipes interleave worse
// than one
#ifndef PSI_HYB4
#define PSI_HYB4 0
#endif
// the same for r = 6: 1 pair in 16 on the FMA pipe (min(16 / (15/16), 128 / (7 + 8/16)) = 17.07)
#ifndef PSI_HYB6
#define PSI_HYB6 0
#endif

__device__ __forceinline__ Fx128 fx_from_double(double x) {
  Fx128 r;
  double fl = floor(x);
  r.hi = (long long)fl;
  double fr = x - fl;  // exact, in [0, 1)
  r.lo = __double2ull_rn(fr * 18446744073709551616.0);
  return r;
}
__device__ __forceinline__ void fx_add(Fx128& a, Fx128 b) {
  unsigned long long lo = a.lo + b.lo;
  a.hi += b.hi + (lo < a.lo ? 1 : 0);
  a.lo = lo;
}

__device__ __forceinline__ void tile_coords(int64_t t, int64_t nb, int64_t& bi, int64_t& bj) {
  // row-major upper triangle incl. diagonal: row b starts at off(b) = b*nb - b(b-1)/2
  double A = 2.0 * (double)nb + 1.0;
  int64_t b = (int64_t)((A - sqrt(A * A - 8.0 * (double)t)) * 0.5);
  if (b < 0) b = 0;
  if (b > nb - 1) b = nb - 1;
  while (b > 0 && b * nb - b * (b - 1) / 2 > t) --b;
  while (b + 1 < nb && (b + 1) * nb - (b + 1) * b / 2 <= t) ++b;
  bi = b;
  bj = b + (t - (b * nb - b * (b - 1) / 2));
}

// The weighted sum (w = 2 off-diagonal, 1 diagonal) of one tile, divided by phi(0).
//   sx    : the tile's j values (jcount of them, then padding up to a multiple of PSI_CH with
//           xpad), 16-byte aligned, visible to all threads (shared memory)
//   xrows : the sorted sample, rows i0 .. i0 + T - 1 (i >= n reads as xpad and is dropped)
//   red   : shared scratch of kPsiThreads / 32 doubles
// Called by all 256 threads; the result is valid in thread 0.  Contains __syncthreads().
// cen: the tile centre when PSI_CENTER (sx then holds fl(x_j - cen)); ignored otherwise
// WIDE (psi_tile_wide): difference first (sx holds raw values, cen unused) and pair2's overflow
// clamp; the inner loop stays rolled there to keep the code small.
// DIAG (R = 1, a diagonal tile, w = 1): row t starts at its own 64-column band b = t / 64 -- the
// band's 64 x 64 diagonal square is evaluated in both orders (weight 1) and the chunks right of it
// once with weight 2 (the mirror image below the diagonal is skipped: K is even); the lanes of a warp
// share b, so the column loop stays uniform.  10 of 16 chunk units of a T = 256 diagonal tile
// instead of 16.
#ifndef PSI_DIAG_BAND
#define PSI_DIAG_BAND 1  // 0: diagonal tiles as full squares (A/B only)
#endif
template <int R, int ORDER, bool LDG, bool WIDE = false, bool DIAG = false>
__device__ __forceinline__ double psi_tile_sum(const float* sx, const float* __restrict__ xrows, int64_t n, int64_t i0,
                                               int jcount, float s, float xpad, double w, double* red,
                                               float cen = 0.f) {
  static_assert(!DIAG || (R == 1 && PSI_CH == 64), "diagonal banding: one row per thread, 64-column chunks");
  constexpr int CH = PSI_CH;  // j per fp32 chunk (CH/2 per packed lane) before the fp64 flush
  constexpr bool CEN = PSI_CENTER != 0 && !WIDE;
  constexpr bool CLAMP = WIDE;
  const int tid = threadIdx.x;
  u64 xi[R], ph[R], s2[R];
  double drow[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int64_t i = i0 + k * kPsiThreads + tid;
    const float v = (i < n) ? (LDG ? __ldg(xrows + i) : xrows[i]) : xpad;
    const float si = dithered_scale(s, i, n);
    const float vi = CEN ? -__fmul_rn(__fsub_rn(v, cen), si) : v;
    xi[k] = pk2(vi, vi);
    const float p = row_phase(i);
    ph[k] = pk2(p, p);
    s2[k] = pk2(si, si);
    drow[k] = 0.0;
  }
  __syncthreads();
  const float4* sx4 = reinterpret_cast<const float4*>(sx);
  const int full = jcount / CH;
  const int band = DIAG ? (tid >> 6) : 0;  // the row's diagonal chunk (DIAG)
  for (int c = band; c < full; ++c) {
    u64 acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0ull;
#pragma unroll(CLAMP ? 1 : kPsiUnroll)
    for (int q = 0; q < CH / 4; ++q) {
      const float4 v = sx4[c * (CH / 4) + q];
      const u64 j01 = pk2(v.x, v.y), j23 = pk2(v.z, v.w);
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (CLAMP) {
          pair2<ORDER, false, CEN, true>(j01, xi[k], s2[k], ph[k], acc[k]);
          pair2<ORDER, false, CEN, true>(j23, xi[k], s2[k], ph[k], acc[k]);
          continue;
        }
        pair2<ORDER, false, CEN>(j01, xi[k], s2[k], ph[k], acc[k]);
        if ((PSI_HYB4 && ORDER == 4 && R == 8 && (k == (q & 7) || k == ((q + 4) & 7))) ||
            (PSI_HYB6 && ORDER == 6 && R == 8 && k == (q & 7)))
          pair2_fma<ORDER, CEN>(j23, xi[k], s2[k], ph[k], acc[k]);
        else
          pair2<ORDER, false, CEN>(j23, xi[k], s2[k], ph[k], acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      float a0, a1;
      upk2(acc[k], a0, a1);
      const double v = f32_to_f64_alu(a0 + a1);
      drow[k] += (DIAG && c > band) ? 2.0 * v : v;
    }
  }
  if (full * CH < jcount && full >= band) {  // ragged last chunk of the last column tile
    u64 acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0ull;
    const int jb = full * CH;
    for (int q = 0; q < CH / 4; ++q) {
      const float4 v = sx4[full * (CH / 4) + q];
      const int j = jb + 4 * q;
      const u64 j01 = pk2(v.x, v.y), j23 = pk2(v.z, v.w);
#pragma unroll
      for (int k = 0; k < R; ++k) {
        pair2<ORDER, true, CEN, CLAMP>(j01, xi[k], s2[k], ph[k], acc[k], j < jcount, j + 1 < jcount);
        pair2<ORDER, true, CEN, CLAMP>(j23, xi[k], s2[k], ph[k], acc[k], j + 2 < jcount, j + 3 < jcount);
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      float a0, a1;
      upk2(acc[k], a0, a1);
      const double v = f32_to_f64_alu(a0 + a1);
      drow[k] += (DIAG && full > band) ? 2.0 * v : v;
    }
  }
  // undo the dither per row, drop padding rows, weight the tile
  double tsum = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int64_t i = i0 + k * kPsiThreads + tid;
    const double comp = exp2(-(double)row_phase(i));
    if (i < n) tsum = fma(drow[k], comp, tsum);
  }
  tsum *= w;
  for (int o = 16; o; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
  if ((tid & 31) == 0) red[tid >> 5] = tsum;
  __syncthreads();
  double tt = 0.0;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < kPsiThreads / 32; ++k) tt += red[k];
  }
  return tt;
}

// Small tiles for small n (R = 0 in psi_rows_per_thread: n <= kFusedMaxN): T = 64 rows x 64
// columns, so a pass has 16x more, 16x smaller tiles than at T = 256 and spreads over the SMs (at
// these sizes the pass is latency-bound).  The unit of work is a CHUNK: one row of a tile against
// the tile's 64 columns, with the pair arithmetic of the big tiles' difference-first path (pair2,
// always with the overflow clamp), the same dither, and one packed fp32 accumulator (even / odd
// columns) -- the 64-term fp32 chunk of PSI_CH.  Each chunk's value (its fp32 sum in fp64, times
// the row's 2^(-p_i) and the tile weight) becomes a 128-bit fixed-point integer on its own, so a
// pass total is the integer sum of its chunks: the same for any assignment of chunks to threads,
// CTAs or clusters (psi_small_kernel of the multi-kernel path and the single-launch cluster kernel
// of fused.cu give the same bits).  No barrier.
constexpr int kPsiSmallT = 64;
#ifndef PSI_CHUNK64_UNROLL
#define PSI_CHUNK64_UNROLL 16  // iterations of 4 columns unrolled in a full chunk (16: all)
#endif
constexpr int kChunk64Unroll = PSI_CHUNK64_UNROLL;

__device__ __forceinline__ double row_comp(int64_t i) { return exp2(-(double)row_phase(i)); }

// one chunk from its row's values: v = x_i, p = row_phase(i), si = dithered_scale(s, i, n),
// comp = row_comp(i); cols: the tile's 64 column values (16-byte aligned; shared or global memory),
// jcount of them real
template <int ORDER, bool LDG>
__device__ __forceinline__ Fx128 psi_chunk64(const float* cols, int jcount, float v, float p, float si, double comp,
                                             double w) {
  const u64 xi = pk2(v, v), ph = pk2(p, p), s2 = pk2(si, si);
  const float4* c4 = reinterpret_cast<const float4*>(cols);
  u64 acc = 0ull;
  if (jcount >= kPsiSmallT) {
#pragma unroll(kChunk64Unroll)
    for (int q = 0; q < kPsiSmallT / 4; ++q) {
      const float4 t = LDG ? __ldg(c4 + q) : c4[q];
      pair2<ORDER, false, false, true>(pk2(t.x, t.y), xi, s2, ph, acc);
      pair2<ORDER, false, false, true>(pk2(t.z, t.w), xi, s2, ph, acc);
    }
  } else {
#pragma unroll 4
    for (int q = 0; q < kPsiSmallT / 4; ++q) {
      const int j = 4 * q;
      float4 t;
      if (LDG) {  // global memory: no loads past the sample's end
        t.x = j < jcount ? __ldg(cols + j) : 0.f;
        t.y = j + 1 < jcount ? __ldg(cols + j + 1) : 0.f;
        t.z = j + 2 < jcount ? __ldg(cols + j + 2) : 0.f;
        t.w = j + 3 < jcount ? __ldg(cols + j + 3) : 0.f;
      } else {
        t = c4[q];
      }
      pair2<ORDER, true, false, true>(pk2(t.x, t.y), xi, s2, ph, acc, j < jcount, j + 1 < jcount);
      pair2<ORDER, true, false, true>(pk2(t.z, t.w), xi, s2, ph, acc, j + 2 < jcount, j + 3 < jcount);
    }
  }
  float a0, a1;
  upk2(acc, a0, a1);
  return fx_from_double((double)(a0 + a1) * comp * w);  // F2F: the XU pipe has room at these sizes
}

// 128-bit fixed-point sums across a warp and a CTA of NT threads (integer: any order, same bits)
__device__ __forceinline__ Fx128 fx_shfl_xor(Fx128 v, int o) {
  Fx128 r;
  r.lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
  r.hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
  return r;
}
__device__ __forceinline__ Fx128 warp_sum_fx(Fx128 v) {
  for (int o = 16; o; o >>= 1) fx_add(v, fx_shfl_xor(v, o));
  return v;
}
// valid in warp 0; red holds NT / 32 entries; contains __syncthreads() (red may be reused after)
template <int NT>
__device__ __forceinline__ Fx128 block_sum_fx(Fx128 v, Fx128* red) {
  v = warp_sum_fx(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  Fx128 t = {0ull, 0ll};
  if (threadIdx.x < 32) {
    t = threadIdx.x < NT / 32 ? red[threadIdx.x] : t;
    t = warp_sum_fx(t);
  }
  __syncthreads();
  return t;
}

}  // namespace plg
