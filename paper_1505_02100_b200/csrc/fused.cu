// fused.cu -- the whole of Algorithm 1 in ONE cooperative launch for
// small samples (n <= kFusedMaxN = 2048, which covers the paper's own workloads n = 128..1024
// of Tables 2-4 and BASELINE config 1).  At these sizes a pass is ~0.1-4 us of arithmetic, so
// the 20 launches of the multi-kernel path dominate; here they become one launch and two
// grid-wide barriers.
//
// Every CTA loads X into shared memory, sorts it (bitonic sort on the radix keys of sort.cu:
// the same unique ascending array), and computes Step I and Steps II-III redundantly with the
// reduction tree of step1_kernel (steps.cuh), so every CTA holds the same g1 without
// communication.  The psi pass tiles (psi_tile.cuh, T = 256) are dealt round-robin to the
// CTAs; each CTA writes its exact 128-bit fixed-point partial to its own slot, the grid
// synchronises, and every CTA adds the slots (integer addition: order-free) and finalises
// Step V identically; the Step VI pass follows the same way and CTA 0 writes the result.
// Every tile sum, the fixed-point total and the scalar chain are computed by the same device
// code as the multi-kernel path, so the result is bit-identical to it (tested).
#include <cooperative_groups.h>
#include <cstdlib>

#include "blocksort.cuh"
#include "common.cuh"
#include "psi_tile.cuh"
#include "steps.cuh"

namespace cg = cooperative_groups;

namespace plg {

// -DPLUGIN_FUSED_TIMING: CTA 0 records %globaltimer (ns) at the phase boundaries into the
// workspace after the partials (tools/fused_phases.py reads them); off in the product build
#ifdef PLUGIN_FUSED_TIMING
#define FT_MARK(k)                                                                   \
  do {                                                                               \
    if ((blockIdx.x == 0 || (k) >= 7) && threadIdx.x == 0) { /* 7, 8: the last CTA */ \
      unsigned long long t;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                          \
      reinterpret_cast<unsigned long long*>(parts + 2 * kFusedMaxGrid)[k] = t;       \
    }                                                                                \
  } while (0)
#else
#define FT_MARK(k) \
  do {             \
  } while (0)
#endif

__device__ __forceinline__ Fx128 ldcg_fx(const Fx128* p) {
  Fx128 r;
  r.lo = __ldcg(&p->lo);
  r.hi = __ldcg(&p->hi);
  return r;
}

// Every CTA of a single-sample launch (and each CTA of a batch): the sorted sample in shared
// memory (padded to nsx with its largest value) and Steps I-III in res, with the reduction tree
// of step1_kernel.  Contains __syncthreads().
__device__ __forceinline__ void cta_prologue(const float* __restrict__ x, int64_t n, int nsx, float* xsm,
                                             plugin_result* res, double* sh1, double* sh2, int* sh_bad,
                                             double* p1) {
  unsigned int* key = reinterpret_cast<unsigned int*>(xsm);
  const int tid = threadIdx.x;
  // sort (keys of the raw bits: pads are 0xffffffff and sort last): blocksort.cuh, n <= 2048
  {
    unsigned int k[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = 8 * tid + r;
      k[r] = (i < n) ? blocksort_key(__ldg(reinterpret_cast<const unsigned int*>(x) + i)) : 0xffffffffu;
    }
    cta_sort2048(k, key + nsx, key, (int)n);  // runs: the 2048 words after the sample
  }
  for (int i = tid; i < n; i += kPsiThreads) key[i] = key2bits(key[i]);
  __syncthreads();
  const float xpad = xsm[n - 1];
  for (int64_t i = n + tid; i < nsx; i += kPsiThreads) xsm[i] = xpad;
  if (tid == 0) init_result(res, n);
  __syncthreads();

  // Step I (+ II, III) with step1_kernel's reduction tree over step1_grid(n) blocks
  const int nb1 = step1_grid(n);
  const double K = (double)xsm[0];
  int bad = 0;
  for (int b = 0; b < nb1; ++b) {
    double a, q;
    int bb;
    step1_block(xsm, n, K, b, nb1, sh1, sh2, sh_bad, a, q, bb);
    if (tid == 0) { p1[2 * b] = a; p1[2 * b + 1] = q; bad |= bb; }
  }
  __syncthreads();
  if (tid < 32) {
    double a, q;
    step1_total<false>(p1, nb1, a, q);
    if (tid == 0) step1_epilogue(a, q, n, K, bad != 0, res);
  }
  __syncthreads();
}

template <int R>
__global__ void __launch_bounds__(kPsiThreads)
plugin_fused_kernel(const float* __restrict__ x, int64_t n, int nsx, int skip, plugin_result* out, Fx128* parts) {
  extern __shared__ __align__(16) float xsm[];  // nsx floats: the sorted sample, padded; then sort scratch
  __shared__ double sh1[8], sh2[8], red[kPsiThreads / 32];
  __shared__ int sh_bad[8];
  __shared__ double p1[2 * 8];
  __shared__ plugin_result res;
  __shared__ Fx128 fx_red[kPsiThreads / 32];
  static_assert(R == 0, "the fused path uses the small tiles of psi_tile.cuh");
  constexpr int T = kPsiSmallT;
  const int tid = threadIdx.x;

  FT_MARK(0);
  cta_prologue(x, n, nsx, xsm, &res, sh1, sh2, sh_bad, p1);
  FT_MARK(1);
  const float xpad = xsm[n - 1];
  FT_MARK(2);
  // Steps IV/V and VI/VII
  cg::grid_group grid = cg::this_grid();
  const int64_t nb = (n + T - 1) / T, tiles = nb * (nb + 1) / 2;
  // pass 4's arrival counter (after the partials and the timing slots); zeroed by CTA 0 before
  // the grid barrier of pass 6, incremented only after it
  unsigned int* arrive = reinterpret_cast<unsigned int*>(parts + 2 * kFusedMaxGrid) + 32;
  if (blockIdx.x == 0 && tid == 0) *arrive = 0u;
  for (int pass = 0; pass < 2; ++pass) {
    const bool ok = res.status == PLUGIN_OK;  // the same in every CTA
    if (ok) {
      const float s = __double2float_rn(1.0 / (pass == 0 ? res.g1 : res.g2));
      Fx128 acc = {0ull, 0ll};
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t bi, bj;
        tile_coords(t, nb, bi, bj);
        const int64_t i0 = bi * T, j0 = bj * T;
        if (skip && bi != bj &&
            ((double)xsm[j0] - (double)xsm[i0 + T - 1]) * (double)s * (1.0 - 1e-5) > kSkipU)
          continue;  // all terms exactly zero (psi.cu); uniform across the CTA
        const int jcount = (int)((n - j0) < T ? (n - j0) : T);
        const double w = (bi == bj) ? 1.0 : 2.0;
        const double tt = (pass == 0) ? psi_tile_sum_small<6, false>(xsm + j0, xsm, n, i0, jcount, s, xpad, w, red)
                                      : psi_tile_sum_small<4, false>(xsm + j0, xsm, n, i0, jcount, s, xpad, w, red);
        if (tid == 0) fx_add(acc, fx_from_double(tt));
      }
      if (tid == 0) parts[pass * gridDim.x + blockIdx.x] = acc;
    }
    FT_MARK(3 + 3 * pass);
    if (pass == 0) {
      grid.sync();  // every CTA needs g2 from the whole Step IV sum
    } else {
      // Step VI: only the last CTA to arrive reduces and finalises (threadfence pattern): no
      // second grid barrier
      __shared__ bool last;
      if (tid == 0) {
        __threadfence();
        last = (atomicAdd(arrive, 1u) == gridDim.x - 1);
      }
      __syncthreads();
      if (!last) return;
      __threadfence();
    }
    FT_MARK(4 + 3 * pass);
    if (ok) {
      // the partials: in parallel over the threads (independent L2 loads), then a 128-bit
      // shuffle / shared-memory reduction -- integer addition, so any order gives the same total
      Fx128 tot = {0ull, 0ll};
      for (unsigned int b = tid; b < gridDim.x; b += kPsiThreads) fx_add(tot, ldcg_fx(parts + pass * gridDim.x + b));
      for (int o = 16; o; o >>= 1) {
        Fx128 other;
        other.lo = __shfl_xor_sync(0xffffffffu, tot.lo, o);
        other.hi = __shfl_xor_sync(0xffffffffu, tot.hi, o);
        fx_add(tot, other);
      }
      if ((tid & 31) == 0) fx_red[tid >> 5] = tot;
      __syncthreads();
      if (tid == 0) {
        Fx128 all = {0ull, 0ll};
        for (int w = 0; w < kPsiThreads / 32; ++w) fx_add(all, fx_red[w]);
        finalize_pass(pass, fx_to_double(all), n, &res);
      }
      __syncthreads();
    }
    FT_MARK(5 + 3 * pass);
  }
  // the last CTA of pass 4 (every CTA holds the same record up to here)
  if (tid == 0) *out = res;
}

// Many small samples in one launch (plugin_h_batch): CTA b runs the whole algorithm for sample
// b (2 <= n_b <= 2048) on its own -- no grid barrier: the prologue above (the same sort and
// Step I as plugin_h), then each pass over tiles of T = 256 BATCH_R (the centred form of psi.cu;
// at one CTA per sample the T = 64 tiles of the latency path are overhead-bound, and larger
// tiles waste more on the full-square diagonal tiles: T = 256 measured fastest) and the same
// finalize.  The tiles differ
// from plugin_h's, so results agree with it to fp32 evaluation rounding, not bit for bit.
#ifndef BATCH_R
#define BATCH_R 1  // rows per thread of the batch tiles (T = 256 R); A/B: 1 fastest (less full-square waste)
#endif
constexpr int kBatchR = BATCH_R, kBatchT = kPsiThreads * kBatchR;

// the rare wide tiles of the batch kernel (difference first, clamped), not inlined
__device__ __noinline__ double batch_wide_tile(int pass, const float* sx, const float* xsm, int64_t n, int64_t i0,
                                               int jcount, float s, float xpad, double w, double* red) {
  return (pass == 0) ? psi_tile_sum<kBatchR, 6, false, true>(sx, xsm, n, i0, jcount, s, xpad, w, red)
                     : psi_tile_sum<kBatchR, 4, false, true>(sx, xsm, n, i0, jcount, s, xpad, w, red);
}

__global__ void __launch_bounds__(kPsiThreads, 3)
plugin_batch_kernel(const float* __restrict__ x, const int64_t* __restrict__ offsets, int count, int skip,
                    plugin_result* __restrict__ out) {
  extern __shared__ __align__(16) float xsm[];  // 2048 sample + 2048 sort scratch (reused as the j tile)
  __shared__ double sh1[8], sh2[8], red[kPsiThreads / 32];
  __shared__ int sh_bad[8];
  __shared__ double p1[2 * 8];
  __shared__ plugin_result res;
  constexpr int T = kBatchT;
  const int tid = threadIdx.x;
  for (int b = blockIdx.x; b < count; b += gridDim.x) {
    const int64_t o0 = offsets[b], n = offsets[b + 1] - o0;
    if (n < 2 || n > kFusedMaxN) {  // not a sample this path takes: E_INVALID in its result
      if (tid == 0) {
        init_result(&out[b], n);
        out[b].status = PLUGIN_E_INVALID;
      }
      continue;
    }
    const int64_t nb = (n + T - 1) / T, tiles = nb * (nb + 1) / 2;
    __syncthreads();  // the previous sample's shared data is consumed
    cta_prologue(x + o0, n, kBlockSortN, xsm, &res, sh1, sh2, sh_bad, p1);
    const float xpad = xsm[n - 1];
    float* sx = xsm + kBlockSortN;  // the staged (centred) j block of a tile
    for (int pass = 0; pass < 2; ++pass) {
      if (res.status != PLUGIN_OK) break;  // uniform: shared
      const float s = __double2float_rn(1.0 / (pass == 0 ? res.g1 : res.g2));
      Fx128 acc = {0ull, 0ll};
      for (int64_t t = 0; t < tiles; ++t) {
        int64_t bi, bj;
        tile_coords(t, nb, bi, bj);
        const int64_t i0 = bi * T, j0 = bj * T;
        if (skip && bi != bj &&
            ((double)xsm[j0] - (double)xsm[i0 + T - 1]) * (double)s * (1.0 - 1e-5) > kSkipU)
          continue;
        const int jcount = (int)((n - j0) < T ? (n - j0) : T);
        // tile centre as in psi.cu (psi_tile_centre: every staged x_j - c exact)
        const float a = xsm[i0], b = xsm[(i0 + T < n ? i0 + T : n) - 1], p = xsm[j0], q = xsm[j0 + jcount - 1];
        const bool wide = psi_tile_wide(a, b, p, q, s);
        const float cen = (PSI_CENTER && !wide) ? psi_tile_centre(a, q) : 0.f;
        __syncthreads();  // sx of the previous tile consumed
        for (int k = tid; k < T; k += kPsiThreads) sx[k] = __fsub_rn((k < jcount) ? xsm[j0 + k] : xpad, cen);
        const double w = (bi == bj) ? 1.0 : 2.0;
        double tt;
        if (wide)  // see psi_tile_wide; out of line so the common path keeps its code and registers
          tt = batch_wide_tile(pass, sx, xsm, n, i0, jcount, s, xpad, w, red);
        else
          tt = (pass == 0) ? psi_tile_sum<kBatchR, 6, false>(sx, xsm, n, i0, jcount, s, xpad, w, red, cen)
                           : psi_tile_sum<kBatchR, 4, false>(sx, xsm, n, i0, jcount, s, xpad, w, red, cen);
        if (tid == 0) fx_add(acc, fx_from_double(tt));
      }
      if (tid == 0) finalize_pass(pass, fx_to_double(acc), n, &res);
      __syncthreads();
    }
    if (tid == 0) out[b] = res;
  }
}

cudaError_t launch_batch(const float* x, const int64_t* offsets, int count, int skip, plugin_result* out,
                         cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  static DevCache grid_cache;
  const int max_grid = dev_cached(grid_cache, [](int dev) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, plugin_batch_kernel, kPsiThreads,
                                                  sizeof(float) * 2 * kBlockSortN);
    return device_sms(dev) * (occ > 0 ? occ : 1);
  });
  const int grid = count < max_grid ? count : max_grid;
  plugin_batch_kernel<<<grid, kPsiThreads, sizeof(float) * 2 * kBlockSortN, s>>>(x, offsets, count, skip, out);
  return cudaGetLastError();
}

cudaError_t launch_fused(const float* x, int64_t n, int skip, plugin_result* out, Fx128* parts, cudaStream_t s) {
  if (n < 2 || n > kFusedMaxN || psi_rows_per_thread(n, 6) != 0 || psi_rows_per_thread(n, 4) != 0)
    return cudaErrorNotSupported;
  static DevCache grid_cache, sm_cache;
  const int max_grid = dev_cached(grid_cache, [](int dev) {
    int occ = 0, coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, plugin_fused_kernel<0>, kPsiThreads,
                                                  sizeof(float) * 2 * kBlockSortN);
    const int g = coop ? device_sms(dev) * occ : 0;
    return g > kFusedMaxGrid ? kFusedMaxGrid : g;
  });
  if (max_grid <= 0) return cudaErrorNotSupported;
  const int64_t T = kPsiSmallT, nb = (n + T - 1) / T, tiles = nb * (nb + 1) / 2;
  int nsx = (int)(nb * T > kBlockSortN ? nb * T : kBlockSortN);  // cta_sort2048 writes 2048 positions
  // one CTA per SM at most: every CTA sorts its own copy of X, so more CTAs than SMs add no speed
  const int sms = dev_cached(sm_cache, device_sms);
  int grid = (int)(tiles < max_grid ? tiles : max_grid);
  if (grid > sms) grid = sms;
  if (const char* e = getenv("PLUGIN_FUSED_GRID")) {  // A/B only: fewer CTAs (cheaper barriers)
    const int g = atoi(e);
    if (g >= 1 && g < grid) grid = g;
  }
  size_t smem = sizeof(float) * ((size_t)nsx + kBlockSortN);  // sample + sort scratch
  void* args[] = {(void*)&x, (void*)&n, (void*)&nsx, (void*)&skip, (void*)&out, (void*)&parts};
  return cudaLaunchCooperativeKernel((const void*)plugin_fused_kernel<0>, dim3(grid), dim3(kPsiThreads), args, smem,
                                     s);
}

}  // namespace plg
