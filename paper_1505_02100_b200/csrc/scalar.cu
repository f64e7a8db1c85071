// scalar.cu -- Step I reduction and the O(1) scalar steps (II, III, V, VII, Eq. 4)
// of Algorithm 1, all in fp64 on the device so the whole
// PLUGIN run needs no host round trip.
#include <cmath>

#include "common.cuh"

namespace plg {

// x^k by repeated multiplication: keeps raw <-> z conversions exact under 2^k scaling.
__device__ __forceinline__ double ipow(double b, int k) {
  double r = 1.0;
  for (int i = 0; i < k; ++i) r *= b;
  return r;
}

__global__ void init_result_kernel(plugin_result* out, int64_t n) {
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  out->status = PLUGIN_OK;
  out->reserved = 0;
  out->n = n;
  double* f = &out->mean;
  const int nf = (int)((sizeof(plugin_result) - offsetof(plugin_result, mean)) / sizeof(double));
  for (int i = 0; i < nf; ++i) f[i] = qnan;
}

// Step I.  V is shift invariant, so it is evaluated on d_i = X_i - X_0
// (exact in fp64) with the printed one-pass form V = [sum d^2 - (sum d)^2/n]/(n-1);
// the shift removes the cancellation of the raw one-pass form when |mean| >> sigma.
// Fixed grid + fixed reduction order => bit-reproducible.
__global__ void __launch_bounds__(256) step1_kernel(const float* __restrict__ x, int64_t n, Ctrl* ctrl,
                                                    double* __restrict__ partials, plugin_result* out) {
  __shared__ double sh1[8], sh2[8];
  __shared__ int sh_bad[8];
  __shared__ bool last;
  const double K = (double)x[0];
  double s1 = 0.0, s2 = 0.0;
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float v = __ldg(x + i);
    bad |= !isfinite(v);
    double d = (double)v - K;
    s1 += d;
    s2 = fma(d, d, s2);
  }
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh1[w] = s1; sh2[w] = s2; sh_bad[w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    int bb = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += sh1[k]; b += sh2[k]; bb |= sh_bad[k]; }
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = b;
    if (bb) atomicOr(&ctrl->nonfinite, 1);
    __threadfence();
    unsigned int prev = atomicAdd(&ctrl->step1_done, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  // last block, warp 0: fixed-order sum of the per-block partials
  double a = 0.0, b = 0.0;
  for (int k = l; k < (int)gridDim.x; k += 32) {
    a += __ldcg(partials + 2 * k);
    b += __ldcg(partials + 2 * k + 1);
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (l != 0) return;
  const double nd = (double)n;
  const double var = (b - a * a / nd) / (nd - 1.0);
  out->mean = K + a / nd;
  out->var = var;
  if (atomicAdd(&ctrl->nonfinite, 0) != 0) { out->status = PLUGIN_E_NONFINITE; return; }
  if (!(var > 0.0)) { out->status = PLUGIN_E_DEGENERATE; return; }
  const double sigma = sqrt(var);
  out->sigma = sigma;
  // Step II in z units (sigma_z = 1) and in data units
  const double psi8_z = 105.0 / (32.0 * sqrt(kPi));
  out->psi8_ns = psi8_z / ipow(sigma, 9);
  // Step III
  const double g1_z = pow(-2.0 * kK6at0 / (kMu2 * psi8_z * nd), 1.0 / 9.0);
  out->g1_z = g1_z;
  out->g1 = g1_z * sigma;
}

cudaError_t launch_init_result(plugin_result* out, int64_t n, cudaStream_t s) {
  init_result_kernel<<<1, 1, 0, s>>>(out, n);
  return cudaGetLastError();
}

cudaError_t launch_step1(const float* x, int64_t n, Ctrl* ctrl, double* partials, plugin_result* out,
                         cudaStream_t s) {
  int64_t want = (n + 2047) / 2048;
  int blocks = (int)(want < kStep1Blocks ? (want < 1 ? 1 : want) : kStep1Blocks);
  step1_kernel<<<blocks, 256, 0, s>>>(x, n, ctrl, partials, out);
  return cudaGetLastError();
}

// ---- finalize a psi pass ---------------------------------------------------------
__device__ __forceinline__ double fx_to_double(Fx128 v) {
  return (double)v.hi + (double)v.lo * 5.42101086242752217003726400434970855712890625e-20;  // 2^-64
}

__device__ Fx128 limbs_to_fx(const plugin_fx128* t) {
  // carry-propagate four 32-bit limbs (each an int64 sum over ranks)
  long long c = 0;
  unsigned long long w[4];
  for (int k = 0; k < 4; ++k) {
    long long v = t->limb[k] + c;
    w[k] = (unsigned long long)v & 0xffffffffull;
    c = v >> 32;  // arithmetic shift: floor division by 2^32
  }
  Fx128 r;
  r.lo = w[0] | (w[1] << 32);
  r.hi = (long long)(w[2] | (w[3] << 32));
  return r;
}

__global__ void finalize_kernel(int what, Ctrl* ctrl, int slot, const plugin_fx128* total, plugin_result* out,
                                int64_t n, double g_host, int r, double* d_psi, plugin_fx128* d_limbs) {
  Fx128 acc = {0ull, 0ll};
  if (ctrl) {
    acc = ctrl->acc[slot];
    // reset for the next pass on this workspace
    ctrl->acc[slot].lo = 0ull;
    ctrl->acc[slot].hi = 0ll;
    ctrl->tile_counter[slot] = 0u;
  }
  if (total) acc = limbs_to_fx(total);
  if (n <= 0 && out) n = out->n;
  if (what == 3) {  // export this rank's partial as limbs
    d_limbs->limb[0] = (long long)(acc.lo & 0xffffffffull);
    d_limbs->limb[1] = (long long)(acc.lo >> 32);
    d_limbs->limb[2] = (long long)((unsigned long long)acc.hi & 0xffffffffull);
    d_limbs->limb[3] = acc.hi >> 32;
    return;
  }
  const double S = fx_to_double(acc);  // = sum_i sum_j K^(r)(u_ij) / phi(0)
  const double nd = (double)n;
  if (what == 2) {  // Psi_r(g) in data units (Step IV/VI form, g given)
    const double g = g_host;
    *d_psi = (ctrl && ctrl->nonfinite) ? __longlong_as_double(0x7ff8000000000000LL)
                                       : kInvSqrt2Pi * S / (nd * nd * ipow(g, r + 1));
    return;
  }
  if (out->status != PLUGIN_OK) return;
  const double sigma = out->sigma;
  if (what == 0) {
    // Step IV (Eq. 6) in z units: u = (z_i - z_j)/g1_z = (X_i - X_j)/g1
    const double g1_z = out->g1_z;
    const double psi6_z = kInvSqrt2Pi * S / (nd * nd * ipow(g1_z, 7));
    out->S6 = S;
    out->psi6_z = psi6_z;
    out->psi6 = psi6_z / ipow(sigma, 7);
    if (!(psi6_z < 0.0)) { out->status = PLUGIN_E_DOMAIN; return; }
    // Step V
    const double g2_z = pow(-2.0 * kK4at0 / (kMu2 * psi6_z * nd), 1.0 / 7.0);
    out->g2_z = g2_z;
    out->g2 = g2_z * sigma;
  } else {
    // Step VI (Eq. 7)
    const double g2_z = out->g2_z;
    const double psi4_z = kInvSqrt2Pi * S / (nd * nd * ipow(g2_z, 5));
    out->S4 = S;
    out->psi4_z = psi4_z;
    out->psi4 = psi4_z / ipow(sigma, 5);
    if (!(psi4_z > 0.0)) { out->status = PLUGIN_E_DOMAIN; return; }
    // Step VII and Eq. 4
    const double h_z = pow(kRK / (kMu2 * kMu2 * psi4_z * nd), 1.0 / 5.0);
    out->h_z = h_z;
    out->h = h_z * sigma;
  }
}

cudaError_t launch_finalize(int what, Ctrl* ctrl, int slot, const plugin_fx128* total, plugin_result* out,
                            int64_t n, double g_host, int r, double* d_psi, plugin_fx128* d_limbs,
                            cudaStream_t s) {
  finalize_kernel<<<1, 1, 0, s>>>(what, ctrl, slot, total, out, n, g_host, r, d_psi, d_limbs);
  return cudaGetLastError();
}

}  // namespace plg
