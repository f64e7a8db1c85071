// sort.cu -- ascending sort of the float32 sample into the workspace.
//
// Not a step of Algorithm 1: Psi_r is a symmetric sum, so the order of X is free.
// Sorting fixes the summation order so that (a) every fp32 chunk the psi pass adds
// holds terms of similar size (no absorption of the small far-tail terms by a large
// running sum) and (b) tiles of the pair triangle map to bands of |u|.
// Sorting values (not key/value pairs) gives a unique output array, so the result
// is deterministic.  LSD radix sort, 4 passes of 8 bits; each pass: per-tile digit
// histograms, one exclusive scan, and a stable scatter (the tile is ordered by the
// digit with 8 stable 1-bit splits in shared memory).
#include <cstdlib>

// -DSORT_TIMING (tools/sort_phases.py; never in the product build): thread 0 of each block-sort
// or merge CTA records %globaltimer at its phase boundaries into g_sort_timing (16 words per CTA)
#ifdef SORT_TIMING
__device__ unsigned long long g_sort_timing[64 * 16];
#define SB_MARK(k)                                                             \
  do {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 64) {                                 \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      g_sort_timing[blockIdx.x * 16 + (k)] = t_;                               \
    }                                                                          \
  } while (0)
#endif
#include "blocksort.cuh"
#include "common.cuh"

namespace plg {

// Order-preserving float -> uint32 key (bits2key/key2bits in common.cuh), on the raw bits
// (loaded as integers: written on floats, nvcc turns `bits | 0x80000000` into an FADD -|x|
// that canonicalises NaN payloads).
template <bool FIRST>
__device__ __forceinline__ unsigned int load_key(const void* src, int64_t i) {
  const unsigned int v = __ldg(reinterpret_cast<const unsigned int*>(src) + i);
  return FIRST ? bits2key(v) : v;
}

// per-tile histogram of digit (key >> shift) & 255, stored digit-major: hist[d * nb + b]
template <bool FIRST, int TILE>
__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const void* src, int64_t n, int shift,
                                                                 unsigned int* hist, int64_t nb) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * TILE;
  for (int q = threadIdx.x; q < TILE; q += kSortThreads) {
    int64_t i = base + q;
    if (i < n) atomicAdd(&h[(load_key<FIRST>(src, i) >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// block-wide exclusive scan of one value per thread (1024 threads max)
template <int NT>
__device__ __forceinline__ unsigned int block_excl_scan(unsigned int v, unsigned int* warp_tot, unsigned int& total) {
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned int inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (l >= o) inc += y;
  }
  if (l == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned int t = (l < NT / 32) ? warp_tot[l] : 0u;
    unsigned int ti = t;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned int y = __shfl_up_sync(0xffffffffu, ti, o);
      if (l >= o) ti += y;
    }
    if (l < NT / 32) warp_tot[l] = ti - t;  // exclusive warp offsets
    if (l == 31) warp_tot[32] = ti;
  }
  __syncthreads();
  unsigned int r = warp_tot[w] + inc - v;
  total = warp_tot[32];
  __syncthreads();
  return r;
}

// exclusive scan of hist (length m = 256 nb) in place, single CTA of 1024 threads, ONE block
// scan: thread t owns the contiguous chunk [t c, t c + c) (c a multiple of 4: uint4 loads, all
// independent), sums it, takes its offset from the block scan of the 1024 sums and rewrites the
// chunk.  (A loop of 1024-wide block scans costs one barrier chain per 1024 counters: 64 of
// them at n = 2^20, ~1 us each.)  hist is 256-byte aligned (workspace layout).
__global__ void __launch_bounds__(1024) sort_scan_kernel(unsigned int* hist, int64_t m) {
  __shared__ unsigned int wt[33];
  const int64_t c = ((m + 1023) / 1024 + 3) & ~int64_t(3);
  const int64_t b = (int64_t)threadIdx.x * c;
  const int64_t e = (b + c < m) ? b + c : m;
  const bool vec = (b + c <= m);
  unsigned int sum = 0;
  if (vec) {
    const uint4* h4 = reinterpret_cast<const uint4*>(hist + b);
#pragma unroll 8
    for (int64_t q = 0; q < c / 4; ++q) {
      const uint4 v = h4[q];
      sum += v.x + v.y + v.z + v.w;
    }
  } else {
    for (int64_t i = b; i < e; ++i) sum += hist[i];
  }
  unsigned int tot;
  unsigned int run = block_excl_scan<1024>(sum, wt, tot);
  if (vec) {
    uint4* h4 = reinterpret_cast<uint4*>(hist + b);
#pragma unroll 4
    for (int64_t q = 0; q < c / 4; ++q) {
      uint4 v = h4[q], o;
      o.x = run; run += v.x;
      o.y = run; run += v.y;
      o.z = run; run += v.z;
      o.w = run; run += v.w;
      h4[q] = o;
    }
  } else {
    for (int64_t i = b; i < e; ++i) {
      const unsigned int v = hist[i];
      hist[i] = run;
      run += v;
    }
  }
}

template <bool FIRST, bool LAST, int TILE>
__global__ void __launch_bounds__(kSortThreads) sort_scatter_kernel(const void* src, int64_t n, int shift,
                                                                    const unsigned int* __restrict__ offs,
                                                                    int64_t nb, void* dst) {
  constexpr int IPT = TILE / kSortThreads;  // keys per thread, blocked arrangement
  __shared__ unsigned int bufA[TILE];
  __shared__ unsigned int bufB[TILE];
  __shared__ unsigned int wt[33];
  __shared__ unsigned int dstart[256];
  __shared__ unsigned int dcount[256];
  const int64_t base = (int64_t)blockIdx.x * TILE;
  const int cnt = (int)((n - base) < TILE ? (n - base) : TILE);
  for (int q = threadIdx.x; q < TILE; q += kSortThreads)
    bufA[q] = (q < cnt) ? load_key<FIRST>(src, base + q) : 0xffffffffu;  // pads sort last
  dcount[threadIdx.x] = 0;
  __syncthreads();
  unsigned int* in = bufA;
  unsigned int* out = bufB;
  for (int bit = 0; bit < 8; ++bit) {
    unsigned int k[IPT];
    unsigned int zeros = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      k[q] = in[threadIdx.x * IPT + q];
      zeros += ((k[q] >> (shift + bit)) & 1u) ^ 1u;
    }
    unsigned int Z;
    unsigned int zpre = block_excl_scan<kSortThreads>(zeros, wt, Z);
    unsigned int opre = threadIdx.x * IPT - zpre;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      unsigned int one = (k[q] >> (shift + bit)) & 1u;
      unsigned int pos = one ? Z + opre : zpre;
      out[pos] = k[q];
      opre += one;
      zpre += one ^ 1u;
    }
    __syncthreads();
    unsigned int* t = in;
    in = out;
    out = t;
  }
  // tile is now ordered by digit (stable); local start of each digit
  for (int q = threadIdx.x; q < cnt; q += kSortThreads) atomicAdd(&dcount[(in[q] >> shift) & 255u], 1u);
  __syncthreads();
  unsigned int tot;
  unsigned int st = block_excl_scan<kSortThreads>(dcount[threadIdx.x], wt, tot);
  dstart[threadIdx.x] = st;
  __syncthreads();
  for (int q = threadIdx.x; q < cnt; q += kSortThreads) {
    unsigned int key = in[q];
    unsigned int d = (key >> shift) & 255u;
    int64_t o = (int64_t)offs[(int64_t)d * nb + blockIdx.x] + (q - (int)dstart[d]);
    reinterpret_cast<unsigned int*>(dst)[o] = LAST ? key2bits(key) : key;
  }
}

// n <= kBlockSortMax: block sort + rank merge (blocksort.cuh) in 1-2 launches instead of the
// 12 of the radix sort (launch-bound at these sizes); the same ascending array.
constexpr int64_t kBlockSortMax = 32768;  // beyond: the radix sort (measured: cfg3 154 vs 175 us)

// block b of 2048 keys sorted in shared memory -> tmp (or straight to xs as floats when the
// whole sample is one block)
__global__ void __launch_bounds__(256) sort_block_kernel(const float* __restrict__ x, int64_t n,
                                                         unsigned int* __restrict__ tmp, float* __restrict__ xs) {
  __shared__ unsigned int runs[kBlockSortN];
  __shared__ unsigned int out[kBlockSortN];
  SB_MARK(0);
  const int64_t base = (int64_t)blockIdx.x * kBlockSortN;
  unsigned int k[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t i = base + 8 * threadIdx.x + r;
    k[r] = (i < n) ? blocksort_key(__ldg(reinterpret_cast<const unsigned int*>(x) + i)) : 0xffffffffu;
  }
  const int cnt = (int)((n - base) < kBlockSortN ? (n - base) : kBlockSortN);
  cta_sort2048(k, runs, out, cnt);
  if (gridDim.x == 1) {
    for (int i = threadIdx.x; i < cnt; i += 256) reinterpret_cast<unsigned int*>(xs)[i] = key2bits(out[i]);
  } else {
    for (int i = threadIdx.x; i < cnt; i += 256) tmp[base + i] = out[i];
  }
  SB_MARK(7);
}

// every key of the sorted blocks to its final position: its index in its block plus, per other
// block, the keys below it (keys of earlier blocks that are equal count too: unique ranks)
__global__ void __launch_bounds__(256) sort_merge_kernel(const unsigned int* __restrict__ tmp, int64_t n, int nblocks,
                                                         float* __restrict__ xs) {
  // all sorted blocks in shared memory (n <= kBlockSortMax: <= 128 KB), then shared-memory searches
  extern __shared__ unsigned int sb[];
  SB_MARK(8);
  {
    // 16-byte loads, up to kMergeLoads in flight per thread before the first store (one L2 round
    // trip for n <= 16384 instead of one per 4 keys: the fill was half the kernel's time in ncu;
    // sort + Step I 28.9 -> 22.8 us at n = 16384, 48.4 -> 37.1 at 32768, profiles/r05_prep_ab.jsonl)
    constexpr int kMergeLoads = 16;
    const int64_t n4 = n >> 2;  // tmp and sb are 16-byte aligned (workspace layout, dynamic smem)
    const uint4* src4 = reinterpret_cast<const uint4*>(tmp);
    uint4* dst4 = reinterpret_cast<uint4*>(sb);
    for (int64_t b = threadIdx.x; b < n4; b += (int64_t)kMergeLoads * blockDim.x) {
      uint4 v[kMergeLoads];
#pragma unroll
      for (int k = 0; k < kMergeLoads; ++k) {
        const int64_t i = b + (int64_t)k * blockDim.x;
        if (i < n4) v[k] = __ldg(src4 + i);
      }
#pragma unroll
      for (int k = 0; k < kMergeLoads; ++k) {
        const int64_t i = b + (int64_t)k * blockDim.x;
        if (i < n4) dst4[i] = v[k];
      }
    }
    for (int64_t i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) sb[i] = __ldg(tmp + i);
  }
  __syncthreads();
  SB_MARK(9);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / kBlockSortN);
    const unsigned int v = sb[i];
    int64_t rank = i - (int64_t)b * kBlockSortN;
    // four blocks searched in lockstep (independent shared-memory loads per step)
#pragma unroll 1
    for (int b0 = 0; b0 < nblocks; b0 += 4) {
      int pos[4], len[4], base[4];
      unsigned int t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int b2 = b0 + q;
        const int64_t rem = n - (int64_t)b2 * kBlockSortN;
        // missing blocks and our own count nothing (len 0); earlier blocks count equal keys too:
        // x < v + 1 (real keys are <= 0xfffffffe)
        len[q] = (b2 < nblocks && b2 != b) ? (int)(rem < kBlockSortN ? rem : kBlockSortN) : 0;
        base[q] = b2 < nblocks ? b2 * kBlockSortN : 0;
        t[q] = (b2 < b) ? v + 1u : v;
        pos[q] = 0;
      }
#pragma unroll
      for (int step = kBlockSortN; step > 0; step >>= 1) {  // counts 0 .. len, branch-free
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = pos[q] + step - 1;
          const unsigned int x = sb[base[q] + (idx < len[q] ? idx : 0)];
          pos[q] += (idx < len[q] && x < t[q]) ? step : 0;
        }
      }
      rank += pos[0] + pos[1] + pos[2] + pos[3];
    }
    reinterpret_cast<unsigned int*>(xs)[rank] = key2bits(v);
  }
  SB_MARK(10);
}

// x (float) -> xs (float, ascending).  tmp: n uint32; hist: 256*nb uint32.
// Passes ping-pong tmp <-> xs (reinterpreted as keys); the last pass writes floats into xs.
// 4 LSD passes of 8 bits; hist holds 256 * ceil(n / TILE) counters (the workspace sizes it for
// the smaller tile)
template <int TILE>
static cudaError_t radix_sort(const float* x, int64_t n, float* xs, unsigned int* tmp, unsigned int* hist,
                              cudaStream_t s) {
  const int64_t nb = (n + TILE - 1) / TILE;
  unsigned int* xk = reinterpret_cast<unsigned int*>(xs);
  const void* src = x;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 8 * pass;
    void* dst = (pass & 1) ? (void*)xk : (void*)tmp;   // 0: x->tmp, 1: tmp->xs, 2: xs->tmp, 3: tmp->xs
    if (pass == 0) sort_hist_kernel<true, TILE><<<(unsigned)nb, kSortThreads, 0, s>>>(src, n, shift, hist, nb);
    else sort_hist_kernel<false, TILE><<<(unsigned)nb, kSortThreads, 0, s>>>(src, n, shift, hist, nb);
    sort_scan_kernel<<<1, 1024, 0, s>>>(hist, 256 * nb);
    if (pass == 0)
      sort_scatter_kernel<true, false, TILE><<<(unsigned)nb, kSortThreads, 0, s>>>(src, n, shift, hist, nb, dst);
    else if (pass == 3)
      sort_scatter_kernel<false, true, TILE><<<(unsigned)nb, kSortThreads, 0, s>>>(src, n, shift, hist, nb, dst);
    else
      sort_scatter_kernel<false, false, TILE><<<(unsigned)nb, kSortThreads, 0, s>>>(src, n, shift, hist, nb, dst);
    src = dst;
  }
  return cudaGetLastError();
}

cudaError_t launch_sort(const float* x, int64_t n, float* xs, unsigned int* tmp, unsigned int* hist,
                        int64_t nb, cudaStream_t s) {
  (void)nb;  // the workspace's counter capacity: 256 * ceil(n / kSortTileSmall) >= what either tile needs
  static int force_radix = -1;  // PLUGIN_SORT_RADIX=1: always the 4-pass radix sort (testing)
  if (force_radix < 0) {
    const char* e = getenv("PLUGIN_SORT_RADIX");
    force_radix = (e && e[0] == '1') ? 1 : 0;
  }
  if (n <= kBlockSortMax && !force_radix) {
    const int nblocks = (int)((n + kBlockSortN - 1) / kBlockSortN);
    sort_block_kernel<<<nblocks, 256, 0, s>>>(x, n, tmp, xs);
    if (nblocks > 1) {
      static DevCache attr_cache;  // the opt-in is a per-device function attribute
      dev_cached(attr_cache, [](int) {
        return (int)cudaFuncSetAttribute(sort_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(unsigned int) * kBlockSortMax));
      });
      static DevCache sm_cache;
      const int64_t want = (n + 255) / 256, sms = dev_cached(sm_cache, device_sms);
      sort_merge_kernel<<<(unsigned)(want < sms ? want : sms), 256, sizeof(unsigned int) * (size_t)n, s>>>(
          tmp, n, nblocks, xs);
    }
    return cudaGetLastError();
  }
  if (sort_tile(n) == kSortTileSmall) return radix_sort<kSortTileSmall>(x, n, xs, tmp, hist, s);
  return radix_sort<kSortTileLarge>(x, n, xs, tmp, hist, s);
}

}  // namespace plg

#ifdef SORT_TIMING
extern "C" int plugin_debug_sort_timing(void* host) {
  return (int)cudaMemcpyFromSymbol(host, g_sort_timing, sizeof(unsigned long long) * 64 * 16);
}
#endif
