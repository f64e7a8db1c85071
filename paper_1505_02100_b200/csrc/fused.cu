// fused.cu -- the whole of Algorithm 1 in ONE launch for small samples
// (n <= kFusedMaxN = 2048, which covers the paper's own workloads n = 128..1024 of Tables 2-4 and
// BASELINE config 1), and many small samples in one launch (plugin_h_batch).  At these sizes a
// pass is ~0.1-4 us of arithmetic, so the launches of the multi-kernel path dominate; here they
// become one thread-block cluster that communicates through distributed shared memory.
#include <cooperative_groups.h>
#include <cstdlib>

#include "blocksort.cuh"
#include "common.cuh"
#include "psi_tile.cuh"
#include "steps.cuh"

namespace cg = cooperative_groups;

namespace plg {

// -DPLUGIN_FUSED_TIMING: CTA 0 records %globaltimer (ns) at the phase boundaries into the
// workspace (tools/fused_phases.py reads them); off in the product build
#ifdef PLUGIN_FUSED_TIMING
#define FT_MARK(k)                                                             \
  do {                                                                         \
    if (crank == 0 && threadIdx.x == 0) {                                      \
      unsigned long long t;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                    \
      reinterpret_cast<unsigned long long*>(parts + 2 * kFusedMaxGrid)[k] = t; \
    }                                                                          \
  } while (0)
#else
#define FT_MARK(k) \
  do {             \
  } while (0)
#endif

// Each CTA of a batch (plugin_batch_kernel): the sorted sample in shared
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

// ---- the single launch for small n: one thread-block cluster ------------------------------------
// C = 16 CTAs of 1024 threads (one cluster; 8 if the device refuses 16), distributed shared memory
// instead of global partials and a cooperative grid barrier:
//   sort  every CTA reads the n keys (blocksort_key, the order of sort.cu); CTA c ranks its slice of
//         ceil(n / C) keys against all n (rank = keys below + equal keys at lower index: unique) and
//         writes each value to its rank in a workspace array; after the cluster barrier every CTA
//         reads the whole array back: THE ascending array (the one the radix and block sorts give;
//         4-byte scattered stores to global memory and one coalesced reload are cheaper than
//         scattering into 16 CTAs' shared memory, measured);
//   I-III every CTA, redundantly, with step1_kernel's reduction tree (steps.cuh): the same g1 as the
//         multi-kernel path, no communication;
//   IV/VI the 64 chunks of each T = 64 tile (psi_chunk64: a row against the tile's 64 columns)
//         are spread over the cluster's threads; each chunk is a 128-bit fixed-point integer, a CTA
//         adds its chunks, and the CTA partials go to every CTA's shared memory (pass 6) or to CTA
//         0's (pass 4); cluster barrier; the receivers add them (integer: order-free) and finalise
//         Step V (every CTA, identically) or Step VII (CTA 0, which writes the record).
// The chunks, their integer total and the scalar chain are computed by the same device code as the
// multi-kernel path (psi_small_kernel, step1_kernel, finalize_pass), so the result is bit-identical to
// it (tested).
constexpr int kFusedThreads = 1024;
constexpr int kFusedClusterMax = 16;

// shared memory of the cluster kernel for n samples: per row 2^-p_i (double), the sorted sample
// padded to whole tiles with its largest value, p_i and the scale dither k_i (float); the C sorted
// runs of the sort (uint64, C (m + 1) <= n + 5 C); the tile table (ushort)
constexpr int kFusedSliceMax = (int)(kFusedMaxN / 8) + 4;  // slice length at the smallest cluster (8)
// up to this n the sort counts each key against all n (one exchange); above, C sorted slices are
// merged by binary search (two exchanges, O(n log n)); measured: the counting sort takes 1.4 / 3.6 us
// at n = 128 / 1024 against 3.0 / 4.0 for the merge, 10.2 against 5.0 at n = 2048
constexpr int64_t kFusedCountMaxN = 1024;
// up to this n every CTA ranks all n keys itself and writes its own copy of the ascending array:
// no exchange and no cluster barrier in the sort (n^2 / 1024 compares per thread); measured: the
// local sort takes 0.9 us at n = 128 (against 1.8 us with the exchange: 14.4 -> 12.4 us per call)
// and 2.5 us at n = 256 (against 1.4 us)
constexpr int64_t kFusedLocalSortN = 160;
static_assert(kFusedCountMaxN <= kFusedThreads, "one key per thread in the counting sort");
__host__ __device__ inline int fused_nsx(int64_t n) { return (int)((n + kPsiSmallT - 1) / kPsiSmallT * kPsiSmallT); }
__host__ __device__ inline int fused_tiles(int64_t n) { const int nb = fused_nsx(n) / kPsiSmallT; return nb * (nb + 1) / 2; }
__host__ __device__ inline int fused_runs(int64_t n) { return (int)n + 5 * kFusedClusterMax; }
inline size_t fused_smem(int64_t n) {
  return (size_t)fused_nsx(n) * 20 + (size_t)fused_runs(n) * 8 + (size_t)fused_tiles(n) * 2;
}

__global__ void __launch_bounds__(kFusedThreads, 1)
plugin_cluster_kernel(const float* __restrict__ x, int64_t n, int skip, plugin_result* out, Fx128* parts) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const int nsx = fused_nsx(n), n4 = (int)((n + 3) / 4);
  double* comp = reinterpret_cast<double*>(fsm);
  float* xsm = reinterpret_cast<float*>(fsm + (size_t)nsx * 8);
  float* rph = xsm + nsx;
  float* rsc = rph + nsx;
  unsigned long long* runs = reinterpret_cast<unsigned long long*>(rsc + nsx);  // C sorted runs of composites
  unsigned short* ttab = reinterpret_cast<unsigned short*>(runs + fused_runs(n));
  __shared__ Fx128 fxred[kFusedThreads / 32];
  __shared__ unsigned long long sk[kFusedSliceMax];  // this CTA's slice of composites
  __shared__ Fx128 cparts[2][kFusedClusterMax];  // the CTAs' pass partials, written by their CTAs
  __shared__ double sh1[8], sh2[8], p1[2 * 8];
  __shared__ int sh_bad[8];
  __shared__ plugin_result res;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks(), crank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const bool local_sort = n <= kFusedLocalSortN;
  // before a CTA writes into another's shared memory, every CTA of the cluster must be running: the
  // sort's cluster barriers see to it, and with the local sort an arrive here and a wait before the
  // first exchange do
  if (local_sort) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  FT_MARK(0);

  // ---- sort: C sorted slices, merged by rank ----
  // CTA crank takes the keys [lo, lo + mm) of X as composites (key << 32) | index (unique: equal keys
  // are ordered by index), ranks them within the slice (P = 2^lp lanes per key) and writes the
  // sorted slice, padded with ~0, to run crank of the workspace; after a cluster barrier every CTA
  // loads all C runs, ranks its own keys in each by binary search (rank = sum over the runs) and
  // writes the values to their ranks (srt); after a second barrier every CTA reads the ascending
  // array back (THE ascending array: the one the radix and block sorts give).  Global scratch plus
  // cluster barriers: scattered 4-byte stores into 16 CTAs' shared memory were slower (measured).
  const unsigned int* xb = reinterpret_cast<const unsigned int*>(x);
  const int m = (int)((n + C - 1) / C + 3) & ~3;  // slice length, a multiple of 4 (<= kFusedSliceMax)
  const int lo = crank * m, mm = (int)n - lo < m ? ((int)n - lo > 0 ? (int)n - lo : 0) : m;
  int mp = 1;  // m rounded up to a power of two
  while (mp < m) mp <<= 1;
  int lp = 5;  // P = min(32, 1024 / mp) lanes per key
  while (lp > 0 && (mp << lp) > kFusedThreads) --lp;
  // counting (n <= 1024 = threads): all n composites in runs[], the slice a part of them; else the
  // slice's m composites in sk[].  The load is issued first and stored after the tables below, so
  // its latency overlaps their arithmetic.
  const bool counting = n <= kFusedCountMaxN;
  const int kidx = counting ? tid : lo + tid;
  const bool kreal = counting ? tid < (int)n : tid < mm;
  const unsigned int kraw = kreal ? __ldg(xb + kidx) : 0u;
  if (tid == 0) init_result(&res, n);
  // pass-independent row tables and the tile table (tile t -> block row, block column)
  const int64_t nb = nsx / kPsiSmallT, tiles = nb * (nb + 1) / 2;
  for (int i = tid; i < nsx; i += kFusedThreads) {
    rph[i] = row_phase(i);
    rsc[i] = (float)row_scale_offset(i, scale_dither_amp(n));  // k_i of dithered_scale
    comp[i] = row_comp(i);
  }
  for (int t = tid; t < tiles; t += kFusedThreads) {
    int64_t bi, bj;
    tile_coords(t, nb, bi, bj);
    ttab[t] = (unsigned short)((bi << 8) | bj);
  }
  {
    const unsigned long long comp64 = ((unsigned long long)blocksort_key(kraw) << 32) | (unsigned int)kidx;
    if (counting) {
      if (kreal) runs[tid] = comp64;
    } else if (tid < m) {
      sk[tid] = kreal ? comp64 : ~0ull;
    }
  }
  __syncthreads();
  FT_MARK(1);
  unsigned long long* grun = reinterpret_cast<unsigned long long*>(parts);            // C runs of m
  float* srt = reinterpret_cast<float*>(grun + kFusedMaxN + 4 * kFusedClusterMax);  // the ascending array
  const int ks = tid >> lp, part = tid & ((1 << lp) - 1);
  if (local_sort) {
    // every CTA: all n keys, P = 2^lq lanes per key, straight into its own sample
    int lq = 5;
    while (lq > 0 && ((int)n << lq) > kFusedThreads) --lq;
    const int kk = tid >> lq, pp = tid & ((1 << lq) - 1);
    unsigned int cnt = 0;
    const unsigned long long ki = kk < n ? runs[kk] : ~0ull;
    if (kk < n) {
#pragma unroll 4
      for (int q = pp; q < (int)n; q += 1 << lq) cnt += runs[q] < ki;
    }
    for (int o = 1; o < (1 << lq); o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    FT_MARK(2);
    if (kk < n && pp == 0) xsm[cnt] = __uint_as_float(key2bits((unsigned int)(ki >> 32)));
    __syncthreads();
  } else {
    if (counting) {
      // small n: every CTA holds all n composites and counts those below each of its keys (P lanes
      // per key, over the composites q = part (mod P))
      const unsigned long long* key = runs;
      FT_MARK(2);
      unsigned int cnt = 0;
      const unsigned long long ki = ks < mm ? key[lo + ks] : ~0ull;
      if (ks < mm) {
  #pragma unroll 4
        for (int q = part; q < (int)n; q += 1 << lp) cnt += key[q] < ki;
      }
      for (int o = 1; o < (1 << lp); o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (ks < mm && part == 0) srt[cnt] = __uint_as_float(key2bits((unsigned int)(ki >> 32)));
    } else {
      const bool own = ks < m;
      const unsigned long long ki = own ? sk[ks] : ~0ull;
      {
        unsigned int cnt = 0;
        for (int q = part; q < m; q += 1 << lp) cnt += sk[q] < ki;
        for (int o = 1; o < (1 << lp); o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        // pads (~0, all equal) keep their slots after the mm real keys
        if (own && part == 0) grun[lo + (ks < mm ? (int)cnt : ks)] = ki;
      }
      cluster.sync();  // release / acquire at cluster scope: every run is in the workspace
      // runs at a stride of m + 1 composites in shared memory: the P lanes of a key search P different
      // runs in lockstep, and an even stride would put them all on the same banks
      for (int e = tid; e < C * m; e += kFusedThreads) {
        const int r = e / m;
        runs[e + r] = __ldcg(grun + e);
      }
      __syncthreads();
      FT_MARK(2);
      unsigned int cnt = 0;
      if (ks < mm) {
        for (int r = part; r < C; r += 1 << lp) {  // composites below ki in run r (pads never count)
          const unsigned long long* run = runs + r * (m + 1);
          int pos = 0;
          for (int step = mp; step >= 1; step >>= 1)
            if (pos + step <= m && run[pos + step - 1] < ki) pos += step;
          cnt += (unsigned int)pos;
        }
      }
      for (int o = 1; o < (1 << lp); o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (ks < mm && part == 0) srt[cnt] = __uint_as_float(key2bits((unsigned int)(ki >> 32)));
    }
    cluster.sync();  // every value is at its rank
    for (int q = tid; q < n4; q += kFusedThreads)
      reinterpret_cast<float4*>(xsm)[q] = __ldcg(reinterpret_cast<const float4*>(srt) + q);
    __syncthreads();
  }
  FT_MARK(3);

  // ---- Steps I-III ----
  const float xpad = xsm[n - 1];
  for (int i = (int)n + tid; i < nsx; i += kFusedThreads) xsm[i] = xpad;
  const int nb1 = step1_grid(n);
  const double K = (double)xsm[0];
  int bad = 0;
  for (int b = 0; b < nb1; ++b) {
    double a, q;
    int bb;
    step1_block(xsm, n, K, b, nb1, sh1, sh2, sh_bad, a, q, bb);
    if (tid == 0) { p1[2 * b] = a; p1[2 * b + 1] = q; bad |= bb; }
  }
  FT_MARK(4);
  __syncthreads();
  if (tid < 32) {
    double a, q;
    step1_total<false>(p1, nb1, a, q);
    if (tid == 0) step1_epilogue(a, q, n, K, bad != 0, &res);
  }
  __syncthreads();
  FT_MARK(5);

  // ---- Steps IV/V and VI/VII ----
  // chunk c = 64 t + (row of tile t), dealt to the cluster's warps 32 at a time round-robin over the
  // CTAs (warp w of CTA crank: chunks 32 (C w + crank) + lane, then + 32 C 32, ...)
  const int nchunks = (int)tiles * kPsiSmallT;
  const int cfirst = 32 * (C * (tid >> 5) + crank) + (tid & 31);
  for (int pass = 0; pass < 2; ++pass) {
    Fx128 acc = {0ull, 0ll};
    if (res.status == PLUGIN_OK) {  // the same record in every CTA: uniform
      const float s = __double2float_rn(1.0 / (pass == 0 ? res.g1 : res.g2));
      const float ulp = dither_ulp(s);
      for (int c = cfirst; c < nchunks; c += C * kFusedThreads) {
        const int t = c >> 6;
        const int bi = ttab[t] >> 8, bj = ttab[t] & 255;
        const int i0 = bi * kPsiSmallT, j0 = bj * kPsiSmallT, i = i0 + (c & (kPsiSmallT - 1));
        if (i >= n) continue;  // padding row
        if (skip && bi != bj &&
            ((double)xsm[j0] - (double)xsm[i0 + kPsiSmallT - 1]) * (double)s * (1.0 - 1e-5) > kSkipU)
          continue;  // all terms exactly zero (psi.cu)
        const int jcount = (int)((n - j0) < kPsiSmallT ? (n - j0) : kPsiSmallT);
        const float si = __fmaf_rn(rsc[i], ulp, s);  // = dithered_scale(s, i, n)
        const double w = (bi == bj) ? 1.0 : 2.0;
        fx_add(acc, pass == 0 ? psi_chunk64<6, false>(xsm + j0, jcount, xsm[i], rph[i], si, comp[i], w)
                              : psi_chunk64<4, false>(xsm + j0, jcount, xsm[i], rph[i], si, comp[i], w));
      }
    }
    FT_MARK(6 + 4 * pass);
    const Fx128 cta = block_sum_fx<kFusedThreads>(acc, fxred);  // valid in warp 0
    FT_MARK(7 + 4 * pass);
    if (pass == 0 && local_sort) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    // pass 6: to every CTA (each finalises Step V); pass 4: to CTA 0
    if (tid < (pass == 0 ? C : 1)) cluster.map_shared_rank(&cparts[pass][0], tid)[crank] = cta;
    cluster.sync();
    FT_MARK(8 + 4 * pass);
    if (pass == 1 && crank != 0) return;  // nothing reads this CTA's shared memory any more
    if (tid == 0 && res.status == PLUGIN_OK) {
      Fx128 tot = {0ull, 0ll};
      for (int r = 0; r < C; ++r) fx_add(tot, cparts[pass][r]);
      finalize_pass(pass, fx_to_double(tot), n, &res);
    }
    __syncthreads();
    FT_MARK(9 + 4 * pass);
  }
  if (tid == 0) *out = res;
}

// Many small samples in one launch (plugin_h_batch): CTA b runs the whole algorithm for sample
// b (2 <= n_b <= 2048) on its own -- no grid barrier: the prologue above (the same sort and
// Step I as plugin_h), then each pass over tiles of T = 256 BATCH_R (the centred form of psi.cu;
// at one CTA per sample the T = 64 tiles of the latency path are overhead-bound, and larger
// tiles waste more on the diagonal tiles: T = 256 measured fastest; diagonal tiles evaluate only
// their 64-wide diagonal squares and the chunks right of them, psi_tile_sum<..., DIAG>) and the
// same finalize.  The tiles differ
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
          tt = (PSI_DIAG_BAND && bi == bj) ? ((pass == 0) ? psi_tile_sum<kBatchR, 6, false, false, true>(sx, xsm, n, i0, jcount, s, xpad, w, red, cen)
                                         : psi_tile_sum<kBatchR, 4, false, false, true>(sx, xsm, n, i0, jcount, s, xpad, w, red, cen))
                          : ((pass == 0) ? psi_tile_sum<kBatchR, 6, false>(sx, xsm, n, i0, jcount, s, xpad, w, red, cen)
                                         : psi_tile_sum<kBatchR, 4, false>(sx, xsm, n, i0, jcount, s, xpad, w, red, cen));
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

// cluster size of the single launch on this device: 16 (non-portable) if it can be scheduled, else
// 8, else 0 (path unavailable); PLUGIN_FUSED_CLUSTER=8 forces 8 (A/B)
static int fused_cluster_size(int dev) {
  (void)dev;
  cudaFuncSetAttribute(plugin_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(plugin_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem(kFusedMaxN));
  const char* e = getenv("PLUGIN_FUSED_CLUSTER");
  const int first = (e && atoi(e) == 8) ? 1 : 0;
  const int cand[2] = {16, 8};
  for (int k = first; k < 2; ++k) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cand[k];
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cand[k]);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = fused_smem(kFusedMaxN);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, plugin_cluster_kernel, &cfg) == cudaSuccess && nc > 0) return cand[k];
    (void)cudaGetLastError();
  }
  return 0;
}

cudaError_t launch_fused(const float* x, int64_t n, int skip, plugin_result* out, Fx128* parts, cudaStream_t s) {
  if (n < 2 || n > kFusedMaxN || psi_rows_per_thread(n, 6) != 0 || psi_rows_per_thread(n, 4) != 0)
    return cudaErrorNotSupported;
  static DevCache cl_cache;
  const int C = dev_cached(cl_cache, fused_cluster_size);
  if (C <= 0) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = fused_smem(n);
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, plugin_cluster_kernel, x, n, skip, out, parts);
}

}  // namespace plg
