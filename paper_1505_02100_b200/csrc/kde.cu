// kde.cu -- the kernel density estimate that the bandwidth is for: Eq. 1 with the Gaussian
// kernel of Eq. 2,
//     f(x_k, h) = (1/(n h)) sum_i K((x_k - X_i)/h),   k = 0 .. m-1
// (a second pairwise workload, points x samples, 1 exp per term).
//
// Work decomposition.  Points are taken in blocks of GB = 256 * RG (each thread keeps RG
// points in registers); the sample is the sorted copy made by sort.cu.  For a block of
// points, only samples within C = sqrt(126.5 / |k|) (1 + 1e-6) of [min point, max point]
// can give a non-zero fp32 term (k = fp32(-log2(e) / (2 h^2)); beyond it the exponent is
// below -126.5 and ex2.approx.ftz returns +0 exactly), so the block reads the sorted range
// [lower_bound(min - C), upper_bound(max + C)).  That range is split into S equal segments,
// one CTA per (block, segment), so small point sets still fill the 148 SMs.  Per term:
//     d = x_k - X_i (fp32)   a = (d * k) * d   e = ex2.approx(a)   acc += e
// two terms per packed f32x2 instruction: 4 FP32 lane-ops + 1 MUFU.EX2 per term.  MUFU.EX2
// (16/clk/SM) would bind at 16 terms/clk/SM with the FMA pipe half idle, so one term in four
// evaluates its exp2 on the FMA pipe instead (kde_term2_poly: 8 more FP32 lane-ops): both
// pipes then saturate together at 21.3 terms/clk/SM.  fp32
// accumulators hold 64 terms per point, then go to per-point fp64; each CTA writes its fp64
// per-point partials and the last CTA of a block adds the S partials in segment order
// (deterministic) and scales by phi(0) / (n h).
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "simd.cuh"

namespace plg {

#ifndef KDE_CENTER
#define KDE_CENTER 1  // 0: difference-first terms everywhere (A/B builds)
#endif
#ifndef KDE_POLY16
#define KDE_POLY16 4  // centred hybrid: term pairs in 16 with the FMA-pipe exp (<= 8; A/B: 4 best)
#endif

constexpr int kKdeThreads = 256;
constexpr int kKdeRG = 4;                      // points per thread
constexpr int kKdeGB = kKdeThreads * kKdeRG;   // points per block
constexpr int kKdeTX = 2048;                   // samples per shared-memory tile
constexpr int kKdeCH = 64;                     // samples per fp32 chunk
constexpr int64_t kKdeTargetCtas = 8 * 148;    // ~4 waves of 2 CTAs per SM

__device__ __forceinline__ void kde_term2(u64 xj, u64 p, u64 k2, u64& acc) {
  const u64 d = sub2(p, xj);
  const u64 a = mul2(mul2(d, k2), d);
  float a0, a1;
  upk2(a, a0, a1);
  acc = add2(acc, pk2(ex2(a0), ex2(a1)));
}
__device__ __forceinline__ void kde_term2_masked(u64 xj, u64 p, u64 k2, u64& acc, bool m0, bool m1) {
  const u64 d = sub2(p, xj);
  const u64 a = mul2(mul2(d, k2), d);
  float a0, a1;
  upk2(a, a0, a1);
  const float e0 = m0 ? ex2(a0) : 0.f, e1 = m1 ? ex2(a1) : 0.f;
  acc = add2(acc, pk2(e0, e1));
}

// exp2 on the FMA pipe for the hybrid variant: a = n + f, n = rint(a) (magic-number add),
// f in [-1/2, 1/2], 2^f by a degree-5 minimax polynomial (relative error 7.5e-8; 2.3e-7 with
// fp32 evaluation), 2^n by adding n to the exponent field.  a is clamped at -126 (the result
// stays a normal float; MUFU.EX2 would flush such terms to 0: the difference is < 2^-125.5
// per term).
__device__ __forceinline__ void kde_term2_poly(u64 xj, u64 p, u64 k2, u64& acc) {
  const u64 d = sub2(p, xj);
  float a0, a1;
  upk2(mul2(mul2(d, k2), d), a0, a1);
  acc = add2(acc, ex2_fma2(pk2(fmaxf(a0, -126.f), fmaxf(a1, -126.f))));
}

// Centred form: with c a point of the block, the sample is staged as
// x' = fl(X - c) and each point keeps -P = -fl(fl(x_k - c) sk), sk = fp32(sqrt(log2(e)/2)/h):
// u = fma(x', sk, -P) = (X - x_k) sk, t = u^2, e = 2^-t (MUFU.EX2 takes the negation for free):
// 3 FP32 lane-ops per term instead of 4.  Used when the block's points span <= 2.5 / sk (the
// rounding of P is then <= 2.5 eps absolute in u); otherwise the difference-first terms above.
__device__ __forceinline__ void kde_term2_c(u64 xj, u64 nP, u64 sk2, u64& acc) {
  float t0, t1;
  const u64 u = fma2(xj, sk2, nP);
  upk2(mul2(u, u), t0, t1);
  acc = add2(acc, pk2(ex2(-t0), ex2(-t1)));
}
__device__ __forceinline__ void kde_term2_c_poly(u64 xj, u64 nP, u64 sk2, u64& acc) {
  float t0, t1;
  const u64 u = fma2(xj, sk2, nP);
  upk2(mul2(u, u), t0, t1);
  acc = add2(acc, ex2_fma2(pk2(fmaxf(-t0, -126.f), fmaxf(-t1, -126.f))));
}
__device__ __forceinline__ void kde_term2_c_masked(u64 xj, u64 nP, u64 sk2, u64& acc, bool m0, bool m1) {
  float t0, t1;
  const u64 u = fma2(xj, sk2, nP);
  upk2(mul2(u, u), t0, t1);
  acc = add2(acc, pk2(m0 ? ex2(-t0) : 0.f, m1 ? ex2(-t1) : 0.f));
}

// first index i in [0, n) with xs[i] >= v (strict = false) or xs[i] > v (strict = true)
__device__ int64_t bound(const float* xs, int64_t n, double v, bool strict) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const double x = (double)__ldg(xs + mid);
    if (strict ? (x <= v) : (x < v)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// the sample range [jb, je) against this thread's kKdeRG points (per-point fp64 sums in drow)
template <bool HYB, bool CEN>
__device__ __forceinline__ void kde_tiles(const float* __restrict__ xs, int64_t jb, int64_t je, float c,
                                          const u64 (&p2)[kKdeRG], const u64 (&nP2)[kKdeRG], u64 k2, u64 sk2,
                                          float* sx, double (&drow)[kKdeRG]) {
  const int tid = threadIdx.x;
  const float4* sx4 = reinterpret_cast<const float4*>(sx);
  for (int64_t t0 = jb; t0 < je; t0 += kKdeTX) {
    const int cnt = (int)((je - t0) < kKdeTX ? (je - t0) : kKdeTX);
    __syncthreads();  // previous tile fully consumed
    for (int q = tid; q < kKdeTX; q += kKdeThreads)
      sx[q] = (q < cnt) ? (CEN ? __fsub_rn(__ldg(xs + t0 + q), c) : __ldg(xs + t0 + q)) : 0.f;
    __syncthreads();
    const int full = cnt / kKdeCH;
    for (int c = 0; c < full; ++c) {
      u64 acc[kKdeRG];
#pragma unroll
      for (int k = 0; k < kKdeRG; ++k) acc[k] = 0ull;
#pragma unroll
      for (int q = 0; q < kKdeCH / 4; ++q) {
        const float4 v = sx4[c * (kKdeCH / 4) + q];
        const u64 j01 = pk2(v.x, v.y), j23 = pk2(v.z, v.w);
#pragma unroll
        for (int k = 0; k < kKdeRG; ++k) {
          if (CEN) {
            // hybrid: KDE_POLY16 term pairs in 16 take their exp on the FMA pipe (DESIGN.md §10:
            // the LP optimum of 3 + 8 FP32 ops is 5, measured best 4 -- MUFU-bound, FMA slack)
            kde_term2_c(j01, nP2[k], sk2, acc[k]);
            if (HYB && k < KDE_POLY16 / 2 + ((q & 1) ? (KDE_POLY16 & 1) : 0))
              kde_term2_c_poly(j23, nP2[k], sk2, acc[k]);
            else kde_term2_c(j23, nP2[k], sk2, acc[k]);
          } else {
            kde_term2(j01, p2[k], k2, acc[k]);
            // hybrid: one term pair in four takes its exp on the FMA pipe (kHybFrac = 1/4)
            if (HYB && (q & 1)) kde_term2_poly(j23, p2[k], k2, acc[k]);
            else kde_term2(j23, p2[k], k2, acc[k]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kKdeRG; ++k) {
        float a0, a1;
        upk2(acc[k], a0, a1);
        drow[k] += f32_to_f64_alu(a0 + a1);
      }
    }
    if (full * kKdeCH < cnt) {  // ragged last chunk
      u64 acc[kKdeRG];
#pragma unroll
      for (int k = 0; k < kKdeRG; ++k) acc[k] = 0ull;
      for (int q = 0; q < kKdeCH / 4; ++q) {
        const float4 v = sx4[full * (kKdeCH / 4) + q];
        const int j = full * kKdeCH + 4 * q;
        const u64 j01 = pk2(v.x, v.y), j23 = pk2(v.z, v.w);
#pragma unroll
        for (int k = 0; k < kKdeRG; ++k) {
          if (CEN) {
            kde_term2_c_masked(j01, nP2[k], sk2, acc[k], j < cnt, j + 1 < cnt);
            kde_term2_c_masked(j23, nP2[k], sk2, acc[k], j + 2 < cnt, j + 3 < cnt);
          } else {
            kde_term2_masked(j01, p2[k], k2, acc[k], j < cnt, j + 1 < cnt);
            kde_term2_masked(j23, p2[k], k2, acc[k], j + 2 < cnt, j + 3 < cnt);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kKdeRG; ++k) {
        float a0, a1;
        upk2(acc[k], a0, a1);
        drow[k] += f32_to_f64_alu(a0 + a1);
      }
    }
  }

}


// resident CTAs per SM the register budget is sized for (tuning: -DKDE_OCC=3 fits 78 registers)
#ifndef KDE_OCC
#define KDE_OCC 2
#endif

template <bool HYB>
__global__ void __launch_bounds__(kKdeThreads, KDE_OCC)
kde_kernel(const float* __restrict__ xs, int64_t n, const float* __restrict__ pts, int64_t m, float kf, float sk,
           double cut,
           int S, double scale, const Ctrl* ctrl, double* __restrict__ partial, unsigned int* __restrict__ counters,
           double* __restrict__ f) {
  __shared__ __align__(16) float sx[kKdeTX];
  __shared__ float s_min[kKdeThreads / 32], s_max[kKdeThreads / 32];
  __shared__ long long s_lo, s_hi;
  __shared__ float s_bmin, s_bmax;
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x / S;
  const int s = (int)(blockIdx.x % S);
  const int64_t p0 = b * kKdeGB;

  float pv[kKdeRG];
  u64 p2[kKdeRG];
  double drow[kKdeRG];
  float lmin = INFINITY, lmax = -INFINITY;
#pragma unroll
  for (int k = 0; k < kKdeRG; ++k) {
    const int64_t p = p0 + k * kKdeThreads + tid;
    pv[k] = (p < m) ? __ldg(pts + p) : __int_as_float(0x7fc00000);
    p2[k] = pk2(pv[k], pv[k]);
    drow[k] = 0.0;
    lmin = fminf(lmin, pv[k]);  // fminf/fmaxf ignore NaN (padding and NaN points)
    lmax = fmaxf(lmax, pv[k]);
  }
  for (int o = 16; o; o >>= 1) {
    lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
    lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  }
  if ((tid & 31) == 0) { s_min[tid >> 5] = lmin; s_max[tid >> 5] = lmax; }
  __syncthreads();
  if (tid < 2) {
    float v = (tid == 0) ? INFINITY : -INFINITY;
    for (int w = 0; w < kKdeThreads / 32; ++w) v = (tid == 0) ? fminf(v, s_min[w]) : fmaxf(v, s_max[w]);
    // samples outside [min - C, max + C] give exactly zero fp32 terms for every point of the block
    // (no non-NaN point: min = +inf, max = -inf, and the range below is empty)
    if (tid == 0) { s_lo = bound(xs, n, (double)v - cut, false); s_bmin = v; }
    else { s_hi = bound(xs, n, (double)v + cut, true); s_bmax = v; }
  }
  __syncthreads();
  const int64_t lo = s_lo, hi = s_hi > s_lo ? s_hi : s_lo;
  const int64_t len = hi - lo;
  const int64_t jb = lo + len * s / S, je = lo + len * (s + 1) / S;
  const u64 k2 = pk2(kf, kf);
  const u64 sk2 = pk2(sk, sk);
  // centred form when the block's points are close together (uniform across the CTA)
  const float c = s_bmin;
  const bool centred = KDE_CENTER && isfinite(c) && isfinite(s_bmax) && (s_bmax - c) * sk <= 2.5f;
  u64 nP2[kKdeRG];
#pragma unroll
  for (int k = 0; k < kKdeRG; ++k) {
    const float P = -__fmul_rn(__fsub_rn(pv[k], c), sk);
    nP2[k] = pk2(P, P);
  }

  if (centred) kde_tiles<HYB, true>(xs, jb, je, c, p2, nP2, k2, sk2, sx, drow);
  else kde_tiles<HYB, false>(xs, jb, je, c, p2, nP2, k2, sk2, sx, drow);

  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  const bool bad = ctrl->nonfinite != 0;
  if (S == 1) {
#pragma unroll
    for (int k = 0; k < kKdeRG; ++k) {
      const int64_t p = p0 + k * kKdeThreads + tid;
      if (p < m) f[p] = (bad || pv[k] != pv[k]) ? qnan : drow[k] * scale;
    }
    return;
  }
  double* mine = partial + ((int64_t)b * S + s) * kKdeGB;
#pragma unroll
  for (int k = 0; k < kKdeRG; ++k) mine[k * kKdeThreads + tid] = drow[k];
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(counters + b, 1u) == (unsigned int)(S - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* base = partial + (int64_t)b * S * kKdeGB;
#pragma unroll
  for (int k = 0; k < kKdeRG; ++k) {
    const int64_t p = p0 + k * kKdeThreads + tid;
    if (p >= m) continue;
    double sum = 0.0;
    for (int q = 0; q < S; ++q) sum += __ldcg(base + (int64_t)q * kKdeGB + k * kKdeThreads + tid);
    f[p] = (bad || pv[k] != pv[k]) ? qnan : sum * scale;
  }
}

// hybrid MUFU / FMA-pipe exp (default); PLUGIN_KDE_MUFU_ONLY=1 selects the MUFU-only kernel
bool kde_hybrid() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PLUGIN_KDE_MUFU_ONLY");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

int64_t kde_point_blocks(int64_t m) { return (m + kKdeGB - 1) / kKdeGB; }

int kde_segments(int64_t n, int64_t m) {
  const int64_t nb = kde_point_blocks(m);
  if (nb <= 0) return 1;
  int64_t S = (kKdeTargetCtas + nb - 1) / nb;
  const int64_t smax = (n + kKdeTX - 1) / kKdeTX;  // at least ~one tile of samples per segment
  if (S > smax) S = smax;
  if (S < 1) S = 1;
  return (int)S;
}

size_t kde_extra_bytes(int64_t n, int64_t m) {
  const int64_t nb = kde_point_blocks(m);
  const int S = kde_segments(n, m);
  size_t bytes = align_up(sizeof(unsigned int) * (size_t)(nb > 0 ? nb : 1), 256);
  if (S > 1) bytes += align_up(sizeof(double) * (size_t)S * (size_t)nb * kKdeGB, 256);
  return bytes;
}

cudaError_t launch_kde(const float* xs, int64_t n, double h, const float* pts, int64_t m, const Ctrl* ctrl,
                       void* extra, double* f, cudaStream_t st) {
  const int64_t nb = kde_point_blocks(m);
  if (nb <= 0) return cudaSuccess;
  const int S = kde_segments(n, m);
  unsigned int* counters = static_cast<unsigned int*>(extra);
  double* partial = reinterpret_cast<double*>(static_cast<char*>(extra) +
                                              align_up(sizeof(unsigned int) * (size_t)nb, 256));
  cudaError_t e = cudaMemsetAsync(counters, 0, sizeof(unsigned int) * (size_t)nb, st);
  if (e != cudaSuccess) return e;
  const double kd = -1.4426950408889634074 / (2.0 * h * h);  // -log2(e) / (2 h^2)
  const float kf = (float)kd;
  const float sk = (float)(sqrt(1.4426950408889634074 / 2.0) / h);  // sqrt(log2(e)/2) / h
  const double cut = sqrt(126.5 / fabs((double)kf)) * (1.0 + 1e-6);
  const double scale = kInvSqrt2Pi / ((double)n * h);
  if (kde_hybrid())
    kde_kernel<true><<<(unsigned int)(nb * S), kKdeThreads, 0, st>>>(xs, n, pts, m, kf, sk, cut, S, scale, ctrl,
                                                                    partial, counters, f);
  else
    kde_kernel<false><<<(unsigned int)(nb * S), kKdeThreads, 0, st>>>(xs, n, pts, m, kf, sk, cut, S, scale, ctrl,
                                                                     partial, counters, f);
  return cudaGetLastError();
}

}  // namespace plg
