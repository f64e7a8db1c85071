// scalar.cu -- Step I reduction and the O(1) scalar steps (II, III, V, VII, Eq. 4)
// of Algorithm 1, all in fp64 on the device so the whole
// PLUGIN run needs no host round trip.
#include <cmath>

#include "common.cuh"
#include "steps.cuh"

namespace plg {

// -DSORT_TIMING: step1_kernel's marks (entry, block sums done, counter taken, epilogue done) in
// g_step1_timing (4 words per CTA, tools/sort_phases.py)
#ifdef SORT_TIMING
__device__ unsigned long long g_step1_timing[64 * 4];
#define S1_MARK(k)                                                             \
  do {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 64) {                                 \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      g_step1_timing[blockIdx.x * 4 + (k)] = t_;                               \
    }                                                                          \
  } while (0)
#else
#define S1_MARK(k) do { } while (0)
#endif

// Step I over a fixed grid (bit-reproducible; see steps.cuh), with the result record's
// initialisation and the Steps II-III epilogue in the last block to finish.
__global__ void __launch_bounds__(256) step1_kernel(const float* __restrict__ x, int64_t n, Ctrl* ctrl,
                                                    double* __restrict__ partials, plugin_result* out) {
  __shared__ double sh1[8], sh2[8];
  __shared__ int sh_bad[8];
  __shared__ bool last;
  S1_MARK(0);
  const double K = (double)x[0];
  double a, q;
  int bb;
  step1_block(x, n, K, blockIdx.x, gridDim.x, sh1, sh2, sh_bad, a, q, bb);
  S1_MARK(1);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = q;
    if (bb) atomicOr(&ctrl->nonfinite, 1);
    __threadfence();
    unsigned int prev = atomicAdd(&ctrl->step1_done, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  S1_MARK(2);
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  // last block, warp 0: fixed-order sum of the per-block partials
  step1_total<true>(partials, gridDim.x, a, q);
  if (threadIdx.x != 0) return;
  init_result(out, n);  // NaN-fill the record first (no separate launch): later steps fill it in
  step1_epilogue(a, q, n, K, atomicAdd(&ctrl->nonfinite, 0) != 0, out);
  S1_MARK(3);
}

cudaError_t launch_step1(const float* x, int64_t n, Ctrl* ctrl, double* partials, plugin_result* out,
                         cudaStream_t s) {
  step1_kernel<<<step1_grid(n), 256, 0, s>>>(x, n, ctrl, partials, out);
  return cudaGetLastError();
}

// ---- finalize a psi pass ---------------------------------------------------------
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
    ctrl->tile_counter[slot] = 0ull;
    if (ctrl->smq_used[slot]) {  // a quota pass (psi.cu, scheduler mode 2): its per-SM counters
      for (int k = 0; k < kSchedSms; ++k) ctrl->sm_cnt[slot][k] = 0u;
      ctrl->smq_used[slot] = 0u;
    }
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
  finalize_total(what, acc, ctrl && ctrl->nonfinite, out, n, g_host, r, d_psi);
}

cudaError_t launch_finalize(int what, Ctrl* ctrl, int slot, const plugin_fx128* total, plugin_result* out,
                            int64_t n, double g_host, int r, double* d_psi, plugin_fx128* d_limbs,
                            cudaStream_t s) {
  finalize_kernel<<<1, 1, 0, s>>>(what, ctrl, slot, total, out, n, g_host, r, d_psi, d_limbs);
  return cudaGetLastError();
}

}  // namespace plg

#ifdef SORT_TIMING
extern "C" int plugin_debug_step1_timing(void* host) {
  return (int)cudaMemcpyFromSymbol(host, plg::g_step1_timing, sizeof(unsigned long long) * 64 * 4);
}
#endif
