// blocksort.cuh -- ascending sort of radix keys (bits2key of the float bits) for small and
// medium n, shared by sort.cu (multi-kernel path) and fused.cu (single launch).
//
//  * warp_sort256: a warp sorts 256 keys held 8 per lane in registers (bitonic network;
//    strides < 8 inside a lane, strides >= 8 across lanes by __shfl_xor_sync) -- no shared
//    memory, no barriers, no branches;
//  * cta_sort2048: 8 warps sort 8 runs of 256, then every key finds its final position by
//    merging by rank: its index in its own run plus, for every other run, the number of keys
//    below it (branch-free binary searches in shared memory; keys of earlier runs that are equal
//    count too, so ranks are unique).  Equal keys are identical bit patterns, so the output is
//    THE ascending array (the same one the radix sort produces);
//  * across CTAs (sort.cu): the same rank merge over sorted blocks of 2048 in global memory.
// The routines run once per launch, so the stage loops stay rolled: fully unrolled they are
// ~10k instructions fetched cold from L2 (measured 26 us for 2048 keys).
#pragma once
#include "common.cuh"

namespace plg {

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

// 256 threads: k[8] are this thread's 8 keys (positions 8 * tid ..; pads 0xffffffff).  On
// return out[0 .. 2048) holds the ascending array; runs (2048 words of shared memory) is
// scratch.  The 7 searches of a key run in lockstep, branch-free (9 steps each: counts 0..256),
// so their shared-memory loads overlap.  Contains __syncthreads().
__device__ __forceinline__ void cta_sort2048(unsigned int (&k)[8], unsigned int* runs, unsigned int* out) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  warp_sort256(k);
#pragma unroll
  for (int r = 0; r < 8; ++r) runs[(w << 8) + (lane << 3) + r] = k[r];
  __syncthreads();
#pragma unroll 1
  for (int r = 0; r < 8; ++r) {
    const int mine = (lane << 3) + r;
    const unsigned int v = runs[(w << 8) + mine];
    int pos[8];
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) pos[w2] = 0;
    // steps 256 .. 1: counts 0 .. 256 (positions past the run never count)
#pragma unroll
    for (int step = 256; step > 0; step >>= 1) {
#pragma unroll
      for (int w2 = 0; w2 < 8; ++w2) {
        // runs before ours count keys <= v, runs after ours keys < v: unique ranks
        const int idx = pos[w2] + step - 1;
        const bool in = idx < 256;
        const unsigned int x = runs[(w2 << 8) + (in ? idx : 255)];
        const bool below = in && ((w2 < w) ? (x <= v) : (x < v));  // past the run: never below
        pos[w2] += below ? step : 0;
      }
    }
    int rank = mine;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) rank += (w2 == w) ? 0 : pos[w2];
    out[rank] = v;
  }
  __syncthreads();
}

}  // namespace plg
