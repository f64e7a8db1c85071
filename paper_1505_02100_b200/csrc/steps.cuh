// steps.cuh -- device code of the O(n) and O(1) steps of Algorithm 1,
// shared by the multi-kernel path (scalar.cu) and the fused small-n kernel (fused.cu) so both
// compute bit-identical results.  Product code: nothing here is shared with oracle/.
#pragma once
#include <cmath>

#include "common.cuh"

namespace plg {

// x^k by repeated multiplication: keeps raw <-> z conversions exact under 2^k scaling.
__device__ __forceinline__ double ipow(double b, int k) {
  double r = 1.0;
  for (int i = 0; i < k; ++i) r *= b;
  return r;
}

// w^(-1/k) for finite w > 0, 1 <= k <= 15: a float seed 2^(-log2(w) / k) (MUFU lg2 / ex2 on the
// mantissa, the exponent split off so the seed cannot leave float range), then three Newton steps
// z <- z + z (1 - w z^k) / k in fp64 -- no division; quadratic convergence from the ~1e-6 seed
// to the fp64 fixed point (within a few ulp of the exact root).  K is a template parameter so the
// power by squaring and the steps unroll into one straight dependency chain (the scalar steps sit
// on the critical path of the single launch); inv_root(w, k) dispatches a runtime k to the same
// code, so both give the same bits.
template <int K>
__device__ __forceinline__ double inv_root_k(double w) {
  int e;
  const double m = frexp(w, &e);  // w = m 2^e, m in [0.5, 1)
  constexpr double kNegInvK = -1.0 / (double)K;
  const double t = ((double)__log2f((float)m) + (double)e) * kNegInvK;
  const double ti = floor(t);
  double z = ldexp((double)exp2f((float)(t - ti)), (int)ti);
  const double rk = 1.0 / (double)K;
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    double zk = 1.0, b = z;  // z^K by squaring
#pragma unroll
    for (int q = K; q; q >>= 1) {
      if (q & 1) zk *= b;
      b *= b;
    }
    z = fma(z * fma(-w, zk, 1.0), rk, z);
  }
  return z;
}
__device__ __forceinline__ double inv_root(double w, int k) {
  switch (k) {
    case 5: return inv_root_k<5>(w);
    case 7: return inv_root_k<7>(w);
    case 9: return inv_root_k<9>(w);
    case 11: return inv_root_k<11>(w);
    case 13: return inv_root_k<13>(w);
    default: return inv_root_k<15>(w);  // k = 15: r = 12, the last stage of PLUGIN_DPI_MAX_STAGES
  }
}

// the bandwidths of Algorithm 1 and of the l-stage family (Steps III and V):
// g = (num / (mu2 Psi n))^(1/k) = (mu2 Psi n / num)^(-1/k), num = -2 K^(r)(0), k = r + 3
// (the data-independent factor mu2 n / num first: one multiply after psi on the critical path)
__device__ __forceinline__ double plugin_bandwidth(double num, double psi, double nd, int k) {
  return inv_root(psi * (kMu2 * nd / num), k);
}
template <int K>
__device__ __forceinline__ double plugin_bandwidth_k(double num, double psi, double nd) {
  return inv_root_k<K>(psi * (kMu2 * nd / num));
}
// Step VII: h_z = (R(K) / (mu2^2 Psi4 n))^(1/5)
__device__ __forceinline__ double plugin_h_z(double psi4_z, double nd) {
  return inv_root_k<5>(psi4_z * (kMu2 * kMu2 * nd / kRK));
}

// Step I, one block's share: V is shift invariant, so it is evaluated on
// d_i = X_i - X_0 (exact in fp64) with the printed one-pass form; this block (index b of
// nblocks, 256 threads) sums d and d^2 over i = b*256 + tid + k*nblocks*256.  Thread 0
// returns the block partials (a = sum d, q = sum d^2) and the non-finite flag.
__device__ __forceinline__ void step1_block(const float* x, int64_t n, double K, int b, int nblocks, double* sh1,
                                            double* sh2, int* sh_bad, double& a, double& q, int& bb) {
  double s1 = 0.0, s2 = 0.0;
  int bad = 0;
  // the tree is that of 256 threads; in larger CTAs (fused.cu: 1024) the others add nothing.  Up to
  // 8 values are loaded before they are added (independent loads in flight; the same additions in
  // the same order)
  const int64_t stride = (int64_t)nblocks * 256;
  for (int64_t i0 = (int64_t)b * 256 + threadIdx.x; threadIdx.x < 256 && i0 < n; i0 += 8 * stride) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (i0 + k * stride < n) ? x[i0 + k * stride] : 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (i0 + k * stride >= n) break;
      bad |= !isfinite(v[k]);
      const double d = (double)v[k] - K;
      s1 += d;
      s2 = fma(d, d, s2);
    }
  }
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0 && w < 8) { sh1[w] = s1; sh2[w] = s2; sh_bad[w] = bad; }
  __syncthreads();
  a = 0.0; q = 0.0; bb = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) { a += sh1[k]; q += sh2[k]; bb |= sh_bad[k]; }
  __syncthreads();  // sh* may be reused
}

// Step I, final: warp 0 adds the nblocks partials {a, q} (stride-2 array, in global memory
// written by other blocks if GLOBAL, else in shared memory) in a fixed order.  Valid in lane 0.
template <bool GLOBAL>
__device__ __forceinline__ void step1_total(const double* partials, int nblocks, double& a, double& q) {
  const int l = threadIdx.x & 31;
  a = 0.0; q = 0.0;
  for (int k = l; k < nblocks; k += 32) {
    a += GLOBAL ? __ldcg(partials + 2 * k) : partials[2 * k];
    q += GLOBAL ? __ldcg(partials + 2 * k + 1) : partials[2 * k + 1];
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
}

// Step I result and Steps II-III from the totals; one thread.
__device__ __forceinline__ void step1_epilogue(double a, double q, int64_t n, double K, bool nonfinite,
                                               plugin_result* out) {
  const double nd = (double)n;
  const double rn = 1.0 / nd, rn1 = 1.0 / (nd - 1.0);  // data-independent: off the critical path
  const double var = (q - a * a * rn) * rn1;
  out->mean = K + a * rn;
  out->var = var;
  if (nonfinite) { out->status = PLUGIN_E_NONFINITE; return; }
  if (!(var > 0.0)) { out->status = PLUGIN_E_DEGENERATE; return; }
  const double sigma = sqrt(var);
  out->sigma = sigma;
  // Step II in z units (sigma_z = 1) and in data units
  const double psi8_z = 105.0 / (32.0 * sqrt(kPi));
  out->psi8_ns = psi8_z / ipow(sigma, 9);
  // Step III
  const double g1_z = plugin_bandwidth_k<9>(-2.0 * kK6at0, psi8_z, nd);
  out->g1_z = g1_z;
  out->g1 = g1_z * sigma;
}

// Psi_r in z units from the pass sum S = sum_i sum_j K^(r)(u_ij) / phi(0) (Eq. 6/7 with the
// symmetry): phi(0) S / (n^2 g_z^(r+1)), the data-independent factor formed first (one multiply
// after S on the critical path); finalize_pass and the DPI stages share it (bit-identical l = 2)
__device__ __forceinline__ double psi_z_from_sum(double S, double nd, double g_z, int r) {
  return S * (kInvSqrt2Pi / (nd * nd * ipow(g_z, r + 1)));
}

__device__ __forceinline__ double fx_to_double(Fx128 v) {
  return (double)v.hi + (double)v.lo * 5.42101086242752217003726400434970855712890625e-20;  // 2^-64
}

// Step IV -> V (what = 0) or Step VI -> VII + Eq. 4 (what = 1) from the full double sum
// S = sum_i sum_j K^(r)(u_ij) / phi(0); one thread.
__device__ __forceinline__ void finalize_pass(int what, double S, int64_t n, plugin_result* out) {
  if (out->status != PLUGIN_OK) return;
  const double nd = (double)n;
  const double sigma = out->sigma;
  if (what == 0) {
    // Step IV (Eq. 6) in z units: u = (z_i - z_j)/g1_z = (X_i - X_j)/g1
    const double g1_z = out->g1_z;
    const double psi6_z = psi_z_from_sum(S, nd, g1_z, 6);
    out->S6 = S;
    out->psi6_z = psi6_z;
    out->psi6 = psi6_z / ipow(sigma, 7);
    if (!(psi6_z < 0.0)) { out->status = PLUGIN_E_DOMAIN; return; }
    // Step V
    const double g2_z = plugin_bandwidth_k<7>(-2.0 * kK4at0, psi6_z, nd);
    out->g2_z = g2_z;
    out->g2 = g2_z * sigma;
  } else {
    // Step VI (Eq. 7)
    const double g2_z = out->g2_z;
    const double psi4_z = psi_z_from_sum(S, nd, g2_z, 4);
    out->S4 = S;
    out->psi4_z = psi4_z;
    out->psi4 = psi4_z / ipow(sigma, 5);
    if (!(psi4_z > 0.0)) { out->status = PLUGIN_E_DOMAIN; return; }
    // Step VII and Eq. 4
    const double h_z = plugin_h_z(psi4_z, nd);
    out->h_z = h_z;
    out->h = h_z * sigma;
  }
}

// A pass's epilogue from its fixed-point total (finalize_kernel, and the last CTA of psi_kernel):
// what = 0 / 1: finalize_pass; 2: Psi_r(g) = phi(0) S / (n^2 g^(r+1)) in data units into *d_psi
// (NaN if the sample had a non-finite value).  One thread.
__device__ __forceinline__ void finalize_total(int what, Fx128 acc, bool nonfinite, plugin_result* out, int64_t n,
                                               double g, int r, double* d_psi) {
  const double S = fx_to_double(acc);  // = sum_i sum_j K^(r)(u_ij) / phi(0)
  const double nd = (double)n;
  if (what == 2) {
    *d_psi = nonfinite ? __longlong_as_double(0x7ff8000000000000LL) : kInvSqrt2Pi * S / (nd * nd * ipow(g, r + 1));
    return;
  }
  finalize_pass(what, S, n, out);
}

__device__ __forceinline__ void init_result(plugin_result* out, int64_t n) {
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  out->status = PLUGIN_OK;
  out->path = 0;
  out->n = n;
  double* f = &out->mean;
  const int nf = (int)((sizeof(plugin_result) - offsetof(plugin_result, mean)) / sizeof(double));
  for (int i = 0; i < nf; ++i) f[i] = qnan;
}

}  // namespace plg
