// dpi.cu -- the l-stage direct plug-in family that Algorithm 1 is the
// l = 2 member of (the "PLUGIN" of the book the paper follows):
//     Psi_{2l+4} <- Psi^NS_{2l+4}   (Step II is l = 2: Psi^NS_8 = 105 / (32 sqrt(pi) sigma^9))
//     for j = l .. 1:  g_j = (-2 K^(2j+2)(0) / (mu2 Psi_{2j+4} n))^(1/(2j+5))   (Steps III, V)
//                      Psi_{2j+2} <- Psi_hat_{2j+2}(g_j)                         (Steps IV, VI)
//     h = (R(K) / (mu2^2 Psi_4 n))^(1/5)                                         (Step VII)
// in z units (Eq. 3-4), the passes in data units with g = g_z sigma.  The O(1) steps run in
// these one-thread kernels between the psi passes of psi.cu; the expressions for l = 2 are
// written exactly as in steps.cuh, so plugin_dpi(l = 2) is bit-identical to plugin_h.
#include <cmath>

#include "common.cuh"
#include "steps.cuh"

namespace plg {

// K^(r)(0) = He_r(0) phi(0) = (-1)^(r/2) (r-1)!! phi(0); r = 6, 4 as printed
__device__ __forceinline__ double k_at_zero(int r) {
  if (r == 6) return kK6at0;
  if (r == 4) return kK4at0;
  double df = 1.0;
  for (int k = r - 1; k > 0; k -= 2) df *= (double)k;
  return ((r / 2) & 1 ? -df : df) * kInvSqrt2Pi;
}

// Psi^NS_r (sigma = 1) = (-1)^(r/2) (r-1)!! / (2^(r/2+1) sqrt(pi)); r = 8: 105 / (32 sqrt(pi))
__device__ __forceinline__ double psi_ns_z(int r) {
  double df = 1.0;
  for (int k = r - 1; k > 0; k -= 2) df *= (double)k;
  const double v = df / ((double)(1 << (r / 2 + 1)) * sqrt(kPi));
  return ((r / 2) & 1) ? -v : v;
}

// g_j from Psi_{2j+4} (z units); writes g_z / g of stage j, or the data status
__device__ __forceinline__ void dpi_bandwidth(plugin_dpi_result* out, int j, double psi_next, double nd) {
  const int r = 2 * j + 2;
  const double num = -2.0 * k_at_zero(r);
  if (!(num / psi_next > 0.0)) { out->status = PLUGIN_E_DOMAIN; return; }
  const double g_z = plugin_bandwidth(num, psi_next, nd, r + 3);
  out->g_z[j - 1] = g_z;
  out->g[j - 1] = g_z * out->sigma;
}

__device__ __forceinline__ void dpi_h(plugin_dpi_result* out, double psi4_z, double nd) {
  if (!(psi4_z > 0.0)) { out->status = PLUGIN_E_DOMAIN; return; }
  const double h_z = plugin_h_z(psi4_z, nd);
  out->h_z = h_z;
  out->h = h_z * out->sigma;
}

// after Step I (in s1): copy it, Psi^NS_{2l+4}, and the bandwidth of stage l (or h for l = 0)
__global__ void dpi_init_kernel(const plugin_result* s1, int stages, plugin_dpi_result* out) {
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  out->status = s1->status;
  out->stages = stages;
  out->n = s1->n;
  out->mean = s1->mean;
  out->var = s1->var;
  out->sigma = s1->sigma;
  out->psi_ns_z = qnan;
  for (int k = 0; k < kDpiMaxStages; ++k) out->g_z[k] = out->g[k] = out->psi_z[k] = out->psi[k] = qnan;
  out->h_z = out->h = qnan;
  if (out->status != PLUGIN_OK) return;
  const double nd = (double)out->n;
  const double p = psi_ns_z(2 * stages + 4);
  out->psi_ns_z = p;
  if (stages == 0) dpi_h(out, p, nd);
  else dpi_bandwidth(out, stages, p, nd);
}

// after the pass of stage j: Psi_{2j+2} from the fixed-point sum, then g_{j-1} or h
__global__ void dpi_finalize_kernel(Ctrl* ctrl, int slot, int j, plugin_dpi_result* out) {
  const Fx128 acc = ctrl->acc[slot];
  ctrl->acc[slot].lo = 0ull;  // reset for the next pass on this workspace
  ctrl->acc[slot].hi = 0ll;
  ctrl->tile_counter[slot] = 0ull;
  if (ctrl->smq_used[slot]) {  // a quota pass (psi.cu, scheduler mode 2): its per-SM counters
    for (int k = 0; k < kSchedSms; ++k) ctrl->sm_cnt[slot][k] = 0u;
    ctrl->smq_used[slot] = 0u;
  }
  if (out->status != PLUGIN_OK) return;
  const int r = 2 * j + 2;
  const double nd = (double)out->n;
  const double S = fx_to_double(acc);  // sum_i sum_j K^(r)(u_ij) / phi(0)
  const double g_z = out->g_z[j - 1];
  const double psi_z = psi_z_from_sum(S, nd, g_z, r);
  out->psi_z[j - 1] = psi_z;
  out->psi[j - 1] = psi_z / ipow(out->sigma, r + 1);
  if (j > 1) dpi_bandwidth(out, j - 1, psi_z, nd);
  else dpi_h(out, psi_z, nd);
}

cudaError_t launch_dpi_init(const plugin_result* s1, int stages, plugin_dpi_result* out, cudaStream_t s) {
  dpi_init_kernel<<<1, 1, 0, s>>>(s1, stages, out);
  return cudaGetLastError();
}

cudaError_t launch_dpi_finalize(Ctrl* ctrl, int slot, int j, plugin_dpi_result* out, cudaStream_t s) {
  dpi_finalize_kernel<<<1, 1, 0, s>>>(ctrl, slot, j, out);
  return cudaGetLastError();
}

}  // namespace plg
