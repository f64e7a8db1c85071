// psi.cu -- the O(n^2) hot path: Steps IV and VI of Algorithm 1
// evaluated with the symmetry of Eq. 5-7 on sm_100a.
//
// Work unit: a T x T tile (T = 256 R) of the upper block triangle of the sorted sample.
// Off-diagonal tiles count each pair once with weight 2; diagonal tiles are evaluated as
// full squares (both orders plus the exact i = j terms) with weight 1, which is
// 2 sum_{i<j} + n K(0) of Eq. 6/7 without a mask.  Persistent CTAs pull tiles from an
// atomic counter.  Each thread keeps R rows i in registers and streams the tile's j values
// from shared memory (one LDS.128 broadcast per 4 j); two pairs go through each packed
// f32x2 instruction:
//     u = fma(x'_j, s_i, -x'_i s_i)   (x' = x - c, c the tile centre; s = fp32(1/g))
//     t = u*u   a = t*c + p_i   (c = fp32(-log2(e)/2), p_i in (-2, -1] a per-row phase)
//     e = ex2.approx(a)   P6 = ((t - 15) t + 45) t - 15  |  P4 = (t - 6) t + 3  (exact integers)
//     acc += P * e
// i.e. 7 (r=6) / 6 (r=4) FP32 lane-ops and 1 MUFU.EX2 per pair (the small tiles of n <= 2048
// use difference first, one op more).  Numerics:
// the per-row phase p_i = -1 - frac(i * 0.618...) (24 random bits, a Weyl sequence)
// dithers the SFU exp argument so the table-pattern bias of MUFU.EX2 averages to a
// constant, and keeps |a| >= 1 (no input truncation inside MUFU); it is undone by scaling
// each row's fp64 sum by 2^(-p_i) in fp64.  The antithetic per-row scale s_i = s + k_i ulp(s),
// |k_i| <= 128, spreads the fp32 rounding of u, t, a and P(t) of repeated differences
// (discretised samples) over 257 scales; its dilation cancels to first order between the two
// rows of a pair (psi_tile.cuh).
// fp32 accumulators hold 32 terms per lane (64 per row, PSI_CH), then go to per-row fp64; each tile's fp64
// total is added as a 128-bit fixed-point integer, so the result does not depend on
// tile scheduling, grid size or GPU count.
// The tile centre c makes every staged x_j - c exact (psi_tile_centre); the per-row scale is the
// antithetic s + k_i ulp(s) of psi_tile.cuh.  Wide tiles (blocks spanning > 64 bandwidths, or
// values > 1000: outliers, tiny g) run difference first with u^2 clamped so He_r cannot overflow
// (psi_tile_wide).  With a PsiFin, the pass's last CTA runs its epilogue
// (Steps V / VII or Psi_r) instead of a launch.
#include <cstdlib>

#include "common.cuh"
#include "psi_tile.cuh"
#include "steps.cuh"

namespace plg {

// -DPSI_TIMING (tools/psi_phases.py, never in the product build): thread 0 of each CTA records
// %globaltimer (ns) at the phase boundaries of its first tile, its SM and its tile count into
// g_psi_timing (8 words per CTA; plugin_debug_psi_timing copies them out)
#ifdef PSI_TIMING
constexpr int kPsiTimingCtas = 4096;
__device__ unsigned long long g_psi_timing[kPsiTimingCtas * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PT_MARK(k, v) \
  do { if (threadIdx.x == 0 && blockIdx.x < kPsiTimingCtas) g_psi_timing[blockIdx.x * 8 + (k)] = (v); } while (0)
#else
#define PT_MARK(k, v) do { } while (0)
#endif

// a pass CTA's exact partial into the slot; with a PsiFin, the last CTA to finish runs the pass's
// epilogue (threadfence reduction pattern) and resets the slot for a later pass on the same
// workspace.  cta_acc valid in thread 0; called by every thread; last: a shared flag.
__device__ __forceinline__ void psi_cta_done(Fx128 cta_acc, Ctrl* ctrl, int slot, const PsiFin& fin, int64_t n,
                                             bool* last) {
  const int tid = threadIdx.x;
  unsigned long long* g_lo = &ctrl->acc[slot].lo;
  unsigned long long* g_hi = reinterpret_cast<unsigned long long*>(&ctrl->acc[slot].hi);
  if (tid == 0 && (cta_acc.lo != 0ull || cta_acc.hi != 0ll)) {
    unsigned long long old = atomicAdd(g_lo, cta_acc.lo);
    unsigned long long carry = (old + cta_acc.lo < old) ? 1ull : 0ull;
    atomicAdd(g_hi, (unsigned long long)cta_acc.hi + carry);
  }
  if (fin.what < 0) return;
  if (tid == 0) {
    __threadfence();
    *last = (atomicAdd(&ctrl->psi_done[slot], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!*last || tid != 0) return;
  __threadfence();
  Fx128 total;
  total.lo = atomicExch(g_lo, 0ull);
  total.hi = (long long)atomicExch(g_hi, 0ull);
  ctrl->tile_counter[slot] = 0ull;
  ctrl->psi_done[slot] = 0u;
  finalize_total(fin.what, total, atomicAdd(&ctrl->nonfinite, 0) != 0, fin.out, n, fin.g, fin.r, fin.d_psi);
}

// min resident CTAs per SM for the register budget: R=8 -> 2 (<=128 regs), R=4 -> 3 (<=80 regs), R<=2 -> 4 (<=64)
#ifndef PSI_OCC_R12
#define PSI_OCC_R12 4  // R = 1, 2: <= 64 registers, no spills; 1-3% over 3 CTAs/SM at n = 12K..65K (profiles/r02p_ab_occ.jsonl)
#endif
template <int R>
struct PsiOcc { static constexpr int value = (R >= 8) ? 2 : (R <= 2 ? PSI_OCC_R12 : 3); };

template <int R, int ORDER, bool SMQ>
__global__ void __launch_bounds__(kPsiThreads, PsiOcc<R>::value)
psi_kernel(const float* __restrict__ xs, int64_t n, int skip, double g_host, const double* g_dev,
           const int32_t* status_dev, Ctrl* ctrl, int slot, int64_t tile_begin, int64_t tile_end, int64_t head,
           unsigned int quota, PsiFin fin) {
  static_assert(R >= 1, "R = 0 (small tiles) runs psi_small_kernel");
  static_assert(kPsiThreads >= kSchedSms, "the steal scan reads one per-SM counter per thread");
  constexpr int T = kPsiThreads * R;
  __shared__ __align__(16) float sx[T];
  __shared__ double red[kPsiThreads / 32];
  __shared__ long long s_tile;
  __shared__ int s_phase, s_pick;

  // the sample is heavily tied: group.cu's exact pass evaluates this one (and finalises)
  if (ctrl->grouped) return;
  // g: from the device (a bandwidth an earlier kernel of the stream computed; the pass is
  // skipped if that chain already failed) or from the host
  double g = g_host;
  if (g_dev) {
    if (*status_dev != PLUGIN_OK) return;
    g = *g_dev;
  }
  const float s = __double2float_rn(1.0 / g);
  const int64_t nb = (n + T - 1) / T;
  const float xpad = __ldg(xs + n - 1);
  Fx128 cta_acc = {0ull, 0ll};
  const int tid = threadIdx.x;
#ifdef PSI_TIMING
  int ntiles = 0;
  PT_MARK(0, gtimer());
  {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    PT_MARK(6, smid);
  }
#endif

  // Per-SM quota (SMQ: scheduler mode 2, whole-range passes only; its own instantiation, so the
  // other passes' code is untouched): the head's whole tiles are dealt quota = head / kSchedSms to
  // each SM -- a CTA takes tile k kSchedSms + smid while its SM's counter k < quota (phase 0) --,
  // then the remainder's column slices go out by the global counter to whichever CTA is free
  // (phase 1), and a CTA that finds the slices gone takes whole tiles left on other SMs' quotas
  // (phase 2: SMs that host no CTA of this grid, or that run behind).  Every item is claimed exactly
  // once whatever the placement, and the pass's sum is an exact integer, so the result does not
  // depend on who ran what.  Without SMQ: items in order from the global counter.
  int phase = 0;
  for (;;) {
    if constexpr (!SMQ) {
      if (tid == 0) s_tile = tile_begin + (long long)atomicAdd(&ctrl->tile_counter[slot], 1ull);
      __syncthreads();
    } else {
      if (phase < 2) {
        if (tid == 0) {
          long long it = -1;
          int ph = phase;
          if (ph == 0) {
            unsigned int smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            const unsigned int k = smid < (unsigned int)kSchedSms ? atomicAdd(&ctrl->sm_cnt[slot][smid], 1u) : quota;
            if (k < quota) it = (long long)k * kSchedSms + (long long)smid;
            else ph = 1;
          }
          if (ph == 1) {
            const long long f = (long long)atomicAdd(&ctrl->tile_counter[slot], 1ull);
            if (head + f < tile_end) it = head + f;
            else ph = 2;
          }
          s_tile = it;
          s_phase = ph;
        }
        __syncthreads();
        phase = s_phase;
      }
      if (phase == 2) {
        // steal: find an SM whose quota is not used up (one counter per thread), try to take from it
        if (tid == 0) s_pick = -1;
        __syncthreads();
        if (tid < kSchedSms && *reinterpret_cast<volatile unsigned int*>(&ctrl->sm_cnt[slot][tid]) < quota)
          atomicMax(&s_pick, tid);
        __syncthreads();
        const int v = s_pick;
        if (v < 0) break;  // every whole tile is claimed
        if (tid == 0) {
          const unsigned int k = atomicAdd(&ctrl->sm_cnt[slot][v], 1u);
          s_tile = k < quota ? (long long)k * kSchedSms + v : -1;
        }
        __syncthreads();
        if (s_tile < 0) continue;  // someone else took it: scan again (the scan's first barrier orders s_tile)
      }
    }
    const int64_t item = s_tile;
#ifdef PSI_TIMING
    if (ntiles == 0) PT_MARK(1, gtimer());
#endif
    if (item >= tile_end) break;
    // work item -> tile t and its column range [k0, k0 + kw): items < head are whole tiles, the
    // rest are the kTailCols-column slices of the remainder tiles (psi_tail_head)
    int64_t t = item;
    int k0 = 0, kw = T;
    if (item >= head) {
      constexpr int kSplit = T / kTailCols;
      const int64_t qq = item - head;
      t = head + qq / kSplit;
      kw = kTailCols;
      k0 = (int)(qq % kSplit) * kTailCols;
    }
    int64_t bi, bj;
    tile_coords(t, nb, bi, bj);
    const int64_t i0 = bi * T, j0 = bj * T;
    if (skip && bi != bj) {
      // sorted sample: the smallest |x_j - x_i| of an off-diagonal tile is xs[j0] - xs[i0 + T - 1];
      // if even that gives |u| > 13.25 (with a 1e-5 margin for the per-row scale dither and fp32
      // rounding), every exponent a = t c + p_i is below -127 and ex2.approx.ftz returns +0
      // exactly, so the tile adds exactly nothing (bit-identical to evaluating it)
      const double gap = (double)__ldg(xs + j0) - (double)__ldg(xs + i0 + T - 1);
      if (gap * (double)s * (1.0 - 1e-5) > kSkipU) {
        __syncthreads();  // every thread has read s_tile before thread 0 overwrites it
        continue;
      }
    }
    const int jtile = (int)((n - j0) < T ? (n - j0) : T);  // real columns of the tile
    const int jcount = jtile - k0 < kw ? (jtile - k0 > 0 ? jtile - k0 : 0) : kw;  // ... of this item
    if (jcount == 0) {  // a quarter past the sample's end (ragged last column block): no pairs
      __syncthreads();
      continue;
    }
    // tile centre (PSI_CENTER, not wide): psi_tile_centre makes every staged x_j - cen exact;
    // decided on the whole tile, so the quarters of a tile agree
    // sorted: rows in [a, b] = [xs[i0], xs[i0 + T - 1]], columns in [p, q] = [xs[j0], xs[j0 + jtile - 1]]
    const float a = __ldg(xs + i0), b = __ldg(xs + (i0 + T < n ? i0 + T : n) - 1);
    const float p = __ldg(xs + j0), q = __ldg(xs + j0 + jtile - 1);
    const bool wide = psi_tile_wide(a, b, p, q, s);
    const float cen = (PSI_CENTER && !wide) ? psi_tile_centre(a, q) : 0.f;
    const int64_t jb = j0 + k0;  // first staged column
    // stage the item's column values: float4 loads (xs is 256-byte aligned, jb a multiple of 64)
    if (jcount == kw) {
      const float4* src = reinterpret_cast<const float4*>(xs + jb);
      float4* dst = reinterpret_cast<float4*>(sx);
      // kw / 4 float4: one per thread for kw >= 1024, the first kw / 4 threads otherwise
      for (int q = tid; q < kw / 4; q += kPsiThreads) {
        float4 v = __ldg(src + q);
        v.x = __fsub_rn(v.x, cen);
        v.y = __fsub_rn(v.y, cen);
        v.z = __fsub_rn(v.z, cen);
        v.w = __fsub_rn(v.w, cen);
        dst[q] = v;
      }
    } else {
      for (int q = tid; q < kw; q += kPsiThreads) sx[q] = __fsub_rn((q < jcount) ? __ldg(xs + jb + q) : xpad, cen);
    }
    const double w = (bi == bj) ? 1.0 : 2.0;
#ifdef PSI_TIMING
    if (ntiles == 0) PT_MARK(2, gtimer());
#endif
    double tt;
    if (wide) tt = psi_tile_sum<R, ORDER, true, true>(sx, xs, n, i0, jcount, s, xpad, w, red);
    else tt = psi_tile_sum<R, ORDER, true>(sx, xs, n, i0, jcount, s, xpad, w, red, cen);
    if (tid == 0) fx_add(cta_acc, fx_from_double(tt));
#ifdef PSI_TIMING
    if (ntiles == 0) PT_MARK(3, gtimer());
    ++ntiles;
#endif
    // next iteration's first __syncthreads orders the smem reuse
  }
  __shared__ bool last;
#ifdef PSI_TIMING
  PT_MARK(4, gtimer());
  PT_MARK(7, ntiles);
#endif
  psi_cta_done(cta_acc, ctrl, slot, fin, n, &last);
  // quota counters: reset by the pass's last CTA for a later pass on the slot; without a PsiFin the
  // 1-thread kernel that follows and takes the slot's total resets them (smq_used)
  if constexpr (SMQ) {
    if (fin.what >= 0) {
      if (last && tid < kSchedSms) ctrl->sm_cnt[slot][tid] = 0u;
    } else if (tid == 0 && blockIdx.x == 0) {
      ctrl->smq_used[slot] = 1u;
    }
  }
#ifdef PSI_TIMING
  PT_MARK(5, gtimer());
#endif
}

// Small tiles (R = 0: n <= kFusedMaxN): one chunk per thread -- a row of a T = 64 tile against the
// tile's 64 columns (psi_chunk64), the columns read straight from the sorted sample (a few KB:
// L1-resident) -- the 1024 threads' chunk integers summed per CTA and into the slot.  Work items
// [tile_begin, tile_end) are tiles, as for psi_kernel; the same chunks and the same integer sums as
// the single-launch cluster kernel (fused.cu), hence the same bits.
constexpr int kPsiSmallThreads = 1024;

template <int ORDER>
__global__ void __launch_bounds__(kPsiSmallThreads, 1)
psi_small_kernel(const float* __restrict__ xs, int64_t n, int skip, double g_host, const double* g_dev,
                 const int32_t* status_dev, Ctrl* ctrl, int slot, int64_t tile_begin, int64_t tile_end, PsiFin fin) {
  __shared__ Fx128 fxred[kPsiSmallThreads / 32];
  __shared__ bool last;
  if (ctrl->grouped) return;  // (never at these sizes: kGroupMinN) as psi_kernel
  double g = g_host;
  if (g_dev) {
    if (*status_dev != PLUGIN_OK) return;
    g = *g_dev;
  }
  const float s = __double2float_rn(1.0 / g);
  const int64_t nb = (n + kPsiSmallT - 1) / kPsiSmallT;
  Fx128 acc = {0ull, 0ll};
  const int64_t c1 = tile_end * kPsiSmallT;
  for (int64_t c = tile_begin * kPsiSmallT + (int64_t)blockIdx.x * kPsiSmallThreads + threadIdx.x; c < c1;
       c += (int64_t)gridDim.x * kPsiSmallThreads) {
    int64_t bi, bj;
    tile_coords(c / kPsiSmallT, nb, bi, bj);
    const int64_t i0 = bi * kPsiSmallT, j0 = bj * kPsiSmallT, i = i0 + (c & (kPsiSmallT - 1));
    if (i >= n) continue;  // padding row
    // off-diagonal tile whose terms are all exactly zero (psi_kernel's rule; row block bi is full)
    if (skip && bi != bj && ((double)__ldg(xs + j0) - (double)__ldg(xs + i0 + kPsiSmallT - 1)) * (double)s *
                                    (1.0 - 1e-5) > kSkipU)
      continue;
    const int jcount = (int)((n - j0) < kPsiSmallT ? (n - j0) : kPsiSmallT);
    fx_add(acc, psi_chunk64<ORDER, true>(xs + j0, jcount, __ldg(xs + i), row_phase(i), dithered_scale(s, i, n),
                                         row_comp(i), bi == bj ? 1.0 : 2.0));
  }
  const Fx128 cta = block_sum_fx<kPsiSmallThreads>(acc, fxred);
  psi_cta_done(cta, ctrl, slot, fin, n, &last);
}

template <int ORDER>
static cudaError_t launch_small(const float* xs, int64_t n, int skip, double g, const double* g_dev,
                                const int32_t* status_dev, Ctrl* ctrl, int slot, int64_t tb, int64_t te, cudaStream_t s,
                                PsiFin fin) {
  static DevCache cap_cache;
  const int grid_cap = dev_cached(cap_cache, [](int dev) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, psi_small_kernel<ORDER>, kPsiSmallThreads, 0);
    return device_sms(dev) * (occ > 0 ? occ : 1);
  });
  const int64_t want = ((te - tb) * kPsiSmallT + kPsiSmallThreads - 1) / kPsiSmallThreads;
  const int grid = (int)(want < grid_cap ? (want < 1 ? 1 : want) : grid_cap);
  psi_small_kernel<ORDER><<<grid, kPsiSmallThreads, 0, s>>>(xs, n, skip, g, g_dev, status_dev, ctrl, slot, tb, te, fin);
  return cudaGetLastError();
}

// Work items (a function of n and r only -- and of the A/B switch PLUGIN_PSI_TAIL --, so shards and
// any grid give the same items and bits).  Outside kSplitMinTiles ... kSplitMaxTiles tiles every tile
// is whole.  Inside (n ~ 32K-50K and 64.5K-101K: a pass of 3 to 11 waves of resident CTAs, where the
// last wave's whole tiles cost most) the first tiles - tiles mod kSchedSms tiles are whole and the
// remainder tiles are cut column-wise into T / kTailCols items of kTailCols columns, which the
// atomic counter hands to the CTAs that run ahead at the end of the pass, and the whole tiles are
// dealt evenly to the SMs (the per-SM quota of psi_kernel<.., SMQ = true>): mode 2.  Measured as
// CUDA graphs, whole tiles -> mode 2 (profiles/r09_psi_graph_ab.jsonl): plugin_h 324.8 -> 316.5 us
// at n = 32768, 1157 -> 1109 at 65536, 2481 -> 2444 at 100000; with more tiles the quota
// scheduler (its latency-bound 64-column slices) costs more than the shorter tail gains (+0.8% at n = 49152 with
// 4656 tiles of T = 512, +1.4% at 131072, +0.7% at 262144), and at configs 4 and 5 whole tiles
// also keep the multi-GPU shards (equal item counts) equal in work; with fewer tiles the slices
// lose (n = 8192: +3%, 24576: +4%, profiles/r07_smq.jsonl) and the quota alone gains 1% at
// n = 16384.  PLUGIN_PSI_TAIL=0 / 1 / 2 forces whole tiles / slices without the quota / slices
// with it at any size with at least kSchedSms tiles (A/B).  Earlier: slices without the quota lost
// 1-13% at n = 8192-24576 (profiles/r05_ab_tail_slices.jsonl); column quarters of the last
// S + tiles mod S tiles were 7-11% slower at n = 8K-25K (profiles/r02o_ab_tail.jsonl).
constexpr int64_t kSplitMinTiles = 2000, kSplitMaxTiles = 5000;
int psi_sched_mode(int64_t tiles) {
  if (tiles < kSchedSms) return 0;
  const char* e = getenv("PLUGIN_PSI_TAIL");
  if (e && e[0] >= '0' && e[0] <= '2' && e[1] == 0) return e[0] - '0';
  return (tiles >= kSplitMinTiles && tiles <= kSplitMaxTiles) ? 2 : 0;
}

int64_t psi_tail_head(int64_t n, int r) {
  const int64_t tiles = psi_tiles(n, r);
  const int R = psi_rows_per_thread(n, r);
  if (R == 0 || psi_sched_mode(tiles) == 0) return tiles;
  return tiles - tiles % kSchedSms;
}

int64_t psi_work_units(int64_t n, int r) {
  if (n <= 0) return 0;
  const int64_t tiles = psi_tiles(n, r), head = psi_tail_head(n, r);
  return head + (psi_tile_edge(n, r) / kTailCols) * (tiles - head);
}

bool psi_work_item(int64_t n, int r, int64_t item, int64_t* out) {
  if (n <= 0 || item < 0 || item >= psi_work_units(n, r)) return false;
  const int64_t T = psi_tile_edge(n, r), nb = (n + T - 1) / T, head = psi_tail_head(n, r);
  int64_t t = item, k0 = 0, kw = T;
  if (item >= head) {
    const int64_t split = T / kTailCols;
    t = head + (item - head) / split;
    kw = kTailCols;
    k0 = ((item - head) % split) * kw;
  }
  // row-major upper block triangle incl. the diagonal (as tile_coords)
  int64_t b = 0;
  while (b + 1 < nb && (b + 1) * nb - (b + 1) * b / 2 <= t) ++b;
  const int64_t bj = b + (t - (b * nb - b * (b - 1) / 2));
  out[0] = b * T;
  out[1] = (b * T + T < n) ? b * T + T : n;
  out[2] = bj * T + k0;
  out[3] = (bj * T + k0 + kw < n) ? bj * T + k0 + kw : n;
  if (out[3] < out[2]) out[3] = out[2];
  out[4] = (b == bj) ? 1 : 2;
  return true;
}

int psi_rows_per_thread(int64_t n, int r) {
  if (const char* e = getenv("PLUGIN_PSI_R")) {  // tuning override (8, 4, 2, 1; 0 = small tiles)
    int v = atoi(e);
    if (v == 8 || v == 4 || v == 2 || v == 1 || (v == 0 && n <= kFusedMaxN)) return v;
  }
  if (n <= kFusedMaxN) return 0;  // small tiles (T = 64): latency-bound sizes
  // the largest R whose T = 256 R tiles number at least min_tiles[R]: R = 8 needs ~28 tiles per
  // resident CTA (296 on 148 SMs); the smaller R (3-4 CTAs per SM) need fewer -- measured sweep
  // of R = 1, 2, 4 at n = 3000 ... 130000 (profiles/r01ae_tiles_sweep.txt): R = 2 wins from
  // n ~ 16K (32 blocks), R = 4 from n ~ 65K (64 blocks).  Passes of order r >= 6 (7 or more FP32
  // lane-ops per pair: the FMA pipe is busy beside MUFU) stop at R = 4: 24 warps per SM hide the
  // longer Horner chains better than R = 8's 16 (cfg4 psi6: 0.941 vs 0.925 of the MUFU roofline;
  // psi4 prefers R = 8: 0.962 vs 0.957; profiles/r03d_R_sweep.jsonl)
  const int cand[3] = {8, 4, 2};
  const int64_t min_blocks[3] = {128, 64, 32};
  for (int k = (r >= 6 ? 1 : 0); k < 3; ++k) {
    int64_t T = (int64_t)kPsiThreads * cand[k], nb = (n + T - 1) / T;
    if (nb >= min_blocks[k]) return cand[k];
  }
  return 1;
}

template <int R, int ORDER>
static cudaError_t launch_t(const float* xs, int64_t n, int skip, double g, const double* g_dev,
                            const int32_t* status_dev, Ctrl* ctrl, int slot, int64_t tb, int64_t te, cudaStream_t s,
                            PsiFin fin) {
  static DevCache cap_cache;
  const int grid_cap = dev_cached(cap_cache, [](int dev) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, psi_kernel<R, ORDER, false>, kPsiThreads, 0);
    return device_sms(dev) * (occ > 0 ? occ : 1);
  });
  int64_t tiles = te - tb;
  int grid = (int)(tiles < grid_cap ? tiles : grid_cap);
  if (grid < 1) grid = 1;
  // the per-SM quota needs the whole item range in one grid
  const int64_t head = psi_tail_head(n, ORDER);
  const bool smq = psi_sched_mode(psi_tiles(n, ORDER)) == 2 && tb == 0 && te == psi_work_units(n, ORDER) &&
                   head >= kSchedSms && head < te;
  if (smq)
    psi_kernel<R, ORDER, true><<<grid, kPsiThreads, 0, s>>>(xs, n, skip, g, g_dev, status_dev, ctrl, slot, tb, te, head,
                                                           (unsigned int)(head / kSchedSms), fin);
  else
    psi_kernel<R, ORDER, false><<<grid, kPsiThreads, 0, s>>>(xs, n, skip, g, g_dev, status_dev, ctrl, slot, tb, te, head,
                                                            0u, fin);
  return cudaGetLastError();
}

cudaError_t launch_psi(const float* xs, int64_t n, int r, int skip, double g_host, const double* g_dev,
                       const int32_t* status_dev, Ctrl* ctrl, int slot, int64_t tile_begin, int64_t tile_end,
                       cudaStream_t s, PsiFin fin) {
  const int R = psi_rows_per_thread(n, r);
  if (tile_end <= tile_begin)  // no tiles: the epilogue still runs (on a zero total)
    return fin.what >= 0 ? launch_finalize(fin.what, ctrl, slot, nullptr, fin.out, n, fin.g, fin.r, fin.d_psi,
                                           nullptr, s)
                         : cudaSuccess;
  if (R == 0) {
#define PLG_SMALL(OO) \
  if (r == OO) return launch_small<OO>(xs, n, skip, g_host, g_dev, status_dev, ctrl, slot, tile_begin, tile_end, s, fin);
    PLG_SMALL(6) PLG_SMALL(4) PLG_SMALL(0) PLG_SMALL(2) PLG_SMALL(8) PLG_SMALL(10) PLG_SMALL(12)
#undef PLG_SMALL
    return cudaErrorInvalidValue;
  }
#define PLG_ORDER(RR, OO)                                                                                  \
  if (r == OO) return launch_t<RR, OO>(xs, n, skip, g_host, g_dev, status_dev, ctrl, slot, tile_begin, tile_end, s, fin);
#define PLG_CASE(RR)                                                                                       \
  if (R == RR) {                                                                                           \
    PLG_ORDER(RR, 6) PLG_ORDER(RR, 4) PLG_ORDER(RR, 0) PLG_ORDER(RR, 2) PLG_ORDER(RR, 8) PLG_ORDER(RR, 10) \
    PLG_ORDER(RR, 12)                                                                                      \
  }
  PLG_CASE(8)
  PLG_CASE(4)
  PLG_CASE(2)
  PLG_CASE(1)
#undef PLG_CASE
#undef PLG_ORDER
  return cudaErrorInvalidValue;
}

}  // namespace plg

#ifdef PSI_TIMING
extern "C" int plugin_debug_psi_timing(void* host, int ctas) {
  if (ctas > plg::kPsiTimingCtas) ctas = plg::kPsiTimingCtas;
  return (int)cudaMemcpyFromSymbol(host, plg::g_psi_timing, sizeof(unsigned long long) * 8 * (size_t)ctas);
}
#endif
