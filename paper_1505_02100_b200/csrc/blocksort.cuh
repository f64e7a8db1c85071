// blocksort.cuh -- ascending sort of radix keys (bits2key of the float bits) for small and
// medium n, shared by sort.cu (multi-kernel path) and fused.cu (single launch).
//
//  * warp_sort256: a warp sorts 256 keys held 8 per lane in registers (bitonic network;
//    strides < 8 inside a lane, strides >= 8 across lanes by __shfl_xor_sync) -- no shared
//    memory, no barriers, no branches;
//  * cta_sort2048: 8 warps sort 8 runs of 256, then up to 3 rounds of pairwise merge-path
//    merges in shared memory.  Equal keys are identical bit patterns, so the output is THE
//    ascending array (the same one the radix sort produces);
//  * across CTAs (sort.cu): a rank merge over sorted blocks of 2048 in global memory.
// The routines run once per launch, so the loops stay rolled: fully unrolled they were ~10k
// instructions fetched cold from L2 (measured 26 us for 2048 keys).
#pragma once
#include "common.cuh"

namespace plg {

// phase marks of the block sort (sort.cu defines SB_MARK under -DSORT_TIMING; empty elsewhere)
#ifndef SB_MARK
#define SB_MARK(k) do { } while (0)
#endif

constexpr int kBlockSortN = 2048;  // keys per CTA (256 threads x 8)

__device__ __forceinline__ void cmpx(unsigned int& a, unsigned int& b, bool asc) {
  const unsigned int lo = min(a, b), hi = max(a, b);
  a = asc ? lo : hi;
  b = asc ? hi : lo;
}

// bitonic sort of the 256 keys k[0..7] of the 32 lanes (lane l holds positions 8l .. 8l+7)
__device__ __forceinline__ void warp_sort256(unsigned int (&k)[8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int kk = 2; kk <= 256; kk <<= 1) {
    // strides >= 8: partner lane = lane ^ (j / 8), same register
#pragma unroll 1
    for (int j = kk >> 1; j >= 8; j >>= 1) {
      const int lm = j >> 3;
      const bool lower = (lane & lm) == 0;
      const bool asc = ((lane << 3) & kk) == 0;  // kk >= 16: bit kk of 8 lane + r does not depend on r
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const unsigned int o = __shfl_xor_sync(0xffffffffu, k[r], lm);
        k[r] = (lower == asc) ? min(k[r], o) : max(k[r], o);
      }
    }
    // strides 4, 2, 1 inside the lane (kk = 2, 4 start lower)
    if (kk >= 8) {
#pragma unroll
      for (int r = 0; r < 4; ++r) cmpx(k[r], k[r + 4], (((lane << 3) + r) & kk) == 0);
    }
    if (kk >= 4) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (!(r & 2)) cmpx(k[r], k[r + 2], (((lane << 3) + r) & kk) == 0);
    }
#pragma unroll
    for (int r = 0; r < 8; r += 2) cmpx(k[r], k[r + 1], (((lane << 3) + r) & kk) == 0);
  }
}

// 256 threads: k[8] are this thread's 8 keys (positions 8 * tid ..; pads 0xffffffff, real keys
// <= 0xfffffffe -- see blocksort_key), cnt <= 2048 of them real (positions < cnt).  On return
// out[0 .. cnt) holds the ascending array; a (2048 words of shared memory) is scratch.  After
// the warp sorts, rounds of pairwise merges (runs of 256 -> 512 -> 1024 -> 2048, only as many as
// the cnt keys need) by merge path: each thread finds where its 8 output positions split the
// two runs (one binary search on the diagonal) and merges them sequentially.
// Contains __syncthreads().
__device__ __forceinline__ void cta_sort2048(unsigned int (&k)[8], unsigned int* a, unsigned int* out, int cnt) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  int lgmax = 8;  // runs of 2^lgmax cover the cnt keys
  while ((1 << lgmax) < cnt) ++lgmax;
  const int active = 1 << lgmax;  // positions that take part (the rest are pads)
  SB_MARK(1);
  if ((w << 8) < active) warp_sort256(k);  // runs of pads only are sorted already
  SB_MARK(2);
  unsigned int* src = (lgmax - 8) & 1 ? a : out;  // the last round writes out
  unsigned int* dst = (lgmax - 8) & 1 ? out : a;
#pragma unroll
  for (int r = 0; r < 8; ++r) src[(w << 8) + (lane << 3) + r] = k[r];
  __syncthreads();
  SB_MARK(3);
#pragma unroll 1
  for (int lg = 8; lg < lgmax; ++lg) {  // runs of L = 2^lg merged pairwise (merge path)
    const int L = 1 << lg;
    const int o = tid << 3;  // this thread writes merged positions o .. o + 7
    if (o < active) {
      const int base = (o >> (lg + 1)) << (lg + 1), d = o & (2 * L - 1);
      const unsigned int* A = src + base;
      const unsigned int* B = A + L;
      // split of the diagonal d: i keys from A, d - i from B (ties: A first)
      int lo = d > L ? d - L : 0, hi = d < L ? d : L;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] <= B[d - mid - 1]) lo = mid + 1;
        else hi = mid;
      }
      int i = lo, j = d - lo;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const unsigned int av = i < L ? A[i] : 0xffffffffu, bv = j < L ? B[j] : 0xffffffffu;
        const bool ta = i < L && (j >= L || av <= bv);
        dst[base + d + q] = ta ? av : bv;
        i += ta ? 1 : 0;
        j += ta ? 0 : 1;
      }
    }
    __syncthreads();
    SB_MARK(lg - 4);  // 4, 5, 6 after the rounds of runs 256, 512, 1024
    unsigned int* tmp = src;
    src = dst;
    dst = tmp;
  }
  // lgmax - 8 rounds: the result is in out (src after the last swap)
}

// the sort key of a float's bits, with the NaN 0x7fffffff folded onto 0x7ffffffe (another NaN)
// so that 0xffffffff marks only the pads of cta_sort2048
__device__ __forceinline__ unsigned int blocksort_key(unsigned int bits) {
  return min(bits2key(bits), 0xfffffffeu);
}

}  // namespace plg
