// group.cu -- Steps IV/VI for heavily tied samples, exactly, in fp64.
//
// The double sum of Eq. 6/7 regrouped by distinct value: with the sorted sample's distinct
// values v_a and multiplicities c_a,
//     sum_i sum_j K^(r)((X_i - X_j)/g) = sum_a sum_b c_a c_b K^(r)((v_a - v_b)/g),
// an identity (each pair (i, j) with X_i = v_a, X_j = v_b is counted c_a c_b times).  When the
// sample has m <= n/4 distinct values (rounded measurements: BASELINE config 4 rounded to 0.01
// has m = 1631 at n = 2^20), the m x m grouped sum has at most 1/16 of the pairs, so every term
// can be evaluated in fp64: d = v_b - v_a (exact), u = d / g, t = u^2, e^(-t/2) (Cody-Waite +
// degree-11 Taylor, relative error < 1e-15), He_r(u) by Horner in t with exact integer
// coefficients, weighted c_a c_b (exact: < 2^62).  On such samples the fp32 pass cannot average
// its rounding over enough distinct differences (cfg4 rounded to 0.01 drifted to
// 1.1e-5); the grouped pass is exact to ~1e-15 and does O(m^2) work instead of O(n^2).
//
// Device-side decision (no host sync, graph-capturable): group_count_kernel counts the distinct
// values of the sorted copy per chunk and, in its last CTA, the total m; it sets ctrl->grouped
// when n >= kGroupMinN and 4 m <= n (the status of Step I must be OK).  group_write_kernel then
// compacts v_a and the run starts into the workspace.  Both kinds of pass are launched: the fp32
// psi_kernel returns at once when ctrl->grouped is set, the grouped one when it is not; the one
// that runs finalises (PsiFin) exactly as the other would.
//
// Layout of the grouped pass: TG x TG tiles (TG = 256, one row per thread) of the upper block
// triangle of the m distinct values; off-diagonal tiles weight 2, diagonal tiles full squares
// (the a = b terms c_a^2 K(0) included); each thread's row sum c_a sum_b c_b K(.) is added as a
// 128-bit fixed-point integer (exact, order-free), so shards and grids give identical bits.
#include "common.cuh"
#include "psi_tile.cuh"
#include "steps.cuh"

namespace plg {

constexpr int kGroupT = kPsiThreads;  // distinct values per tile edge
constexpr int kGroupChunk = 4096;     // sorted values per counting CTA

// e^(-t/2) for t >= 0 in fp64: k = rint(-t/(2 ln 2)) by the 1.5 2^52 shifter, r = -t/2 - k ln 2
// (Cody-Waite, fdlibm's split of ln 2), e^r by its Taylor polynomial of degree 11 (|r| <= 0.347:
// truncation <= 0.347^12 / 12! = 6e-15 relative), 2^k into the exponent field.  Returns 0 for
// t >= 1416 (e^-708 < 1e-307: such terms are below every sum's resolution).
__device__ __forceinline__ double exp_neg_half(double t) {
  const double y = -0.5 * t;
  const double shifter = 6755399441055744.0;  // 1.5 * 2^52
  const double ks = fma(y, 1.4426950408889634074, shifter);
  const double kd = ks - shifter;
  double r = fma(kd, -6.93147180369123816490e-01, y);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = 2.505210838544171877505e-08;  // 1/11!
  p = fma(p, r, 2.755731922398589065256e-07);  // 1/10!
  p = fma(p, r, 2.755731922398589065256e-06);  // 1/9!
  p = fma(p, r, 2.480158730158730158730e-05);  // 1/8!
  p = fma(p, r, 1.984126984126984126984e-04);  // 1/7!
  p = fma(p, r, 1.388888888888888888889e-03);  // 1/6!
  p = fma(p, r, 8.333333333333333333333e-03);  // 1/5!
  p = fma(p, r, 4.166666666666666666667e-02);  // 1/4!
  p = fma(p, r, 1.666666666666666666667e-01);  // 1/3!
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = __double2loint(ks);  // the shifter sum's low word holds k (two's complement)
  return t < 1416.0 ? p * __hiloint2double((k + 1023) << 20, 0) : 0.0;
}

// He_r(u) as a polynomial in t = u^2 (monic, exact integer coefficients): K^(r) = He_r phi
template <int ORDER>
__device__ __forceinline__ double hermite_t64(double t) {
  if (ORDER == 0) return 1.0;
  if (ORDER == 2) return t - 1.0;
  if (ORDER == 4) return fma(t - 6.0, t, 3.0);
  if (ORDER == 6) return fma(fma(t - 15.0, t, 45.0), t, -15.0);
  if (ORDER == 8) return fma(fma(fma(t - 28.0, t, 210.0), t, -420.0), t, 105.0);
  if (ORDER == 10) return fma(fma(fma(fma(t - 45.0, t, 630.0), t, -3150.0), t, 4725.0), t, -945.0);
  return fma(fma(fma(fma(fma(t - 66.0, t, 1485.0), t, -13860.0), t, 51975.0), t, -62370.0), t, 10395.0);
}

// ---- counting: per-chunk number of distinct values, then m and the decision ------------------
__global__ void __launch_bounds__(256) group_count_kernel(const float* __restrict__ xs, int64_t n, Ctrl* ctrl,
                                                          unsigned int* __restrict__ chunk_heads,
                                                          const plugin_result* s1) {
  __shared__ unsigned int warp_sum[8];
  __shared__ bool last;
  const int64_t c0 = (int64_t)blockIdx.x * kGroupChunk;
  unsigned int heads = 0;
  for (int64_t i = c0 + threadIdx.x; i < c0 + kGroupChunk && i < n; i += 256)
    heads += (i == 0 || __ldg(xs + i) != __ldg(xs + i - 1)) ? 1u : 0u;
  for (int o = 16; o; o >>= 1) heads += __shfl_xor_sync(0xffffffffu, heads, o);
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = heads;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int b = 0;
    for (int w = 0; w < 8; ++w) b += warp_sum[w];
    chunk_heads[blockIdx.x] = b;
    __threadfence();
    last = (atomicAdd(&ctrl->group_done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last CTA: exclusive prefix of the chunk counts in place (chunks processed 256 at a time by a
  // block scan), total m, decision
  __shared__ unsigned int scan[256];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0ull;
  __syncthreads();
  const int64_t nchunks = gridDim.x;
  for (int64_t b0 = 0; b0 < nchunks; b0 += 256) {
    const int64_t b = b0 + threadIdx.x;
    const unsigned int v = (b < nchunks) ? __ldcg(chunk_heads + b) : 0u;
    scan[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {  // Hillis-Steele inclusive scan
      const unsigned int add = threadIdx.x >= o ? scan[threadIdx.x - o] : 0u;
      __syncthreads();
      scan[threadIdx.x] += add;
      __syncthreads();
    }
    if (b < nchunks) chunk_heads[b] = (unsigned int)(carry + scan[threadIdx.x] - v);  // exclusive
    __syncthreads();
    if (threadIdx.x == 255) carry += scan[255];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctrl->distinct = (long long)carry;
    ctrl->grouped = (n >= kGroupMinN && 4 * (long long)carry <= n && s1->status == PLUGIN_OK) ? 1 : 0;
    ctrl->group_done = 0u;
  }
}

// ---- compaction: gv[a] = v_a, gs[a] = first index of v_a in the sorted copy, gs[m] = n -----------
__global__ void __launch_bounds__(256) group_write_kernel(const float* __restrict__ xs, int64_t n, const Ctrl* ctrl,
                                                          const unsigned int* __restrict__ chunk_base,
                                                          float* __restrict__ gv, long long* __restrict__ gs) {
  if (!ctrl->grouped) return;
  __shared__ unsigned int warp_sum[8];
  const int64_t c0 = (int64_t)blockIdx.x * kGroupChunk;
  unsigned int base = chunk_base[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t s0 = c0; s0 < c0 + kGroupChunk && s0 < n; s0 += 256) {
    const int64_t i = s0 + threadIdx.x;
    const bool head = i < n && (i == 0 || __ldg(xs + i) != __ldg(xs + i - 1));
    const unsigned int ballot = __ballot_sync(0xffffffffu, head);
    if (lane == 0) warp_sum[warp] = __popc(ballot);
    __syncthreads();
    unsigned int before = base;
    for (int w = 0; w < warp; ++w) before += warp_sum[w];
    before += __popc(ballot & ((1u << lane) - 1u));
    if (head) {
      gv[before] = __ldg(xs + i);
      gs[before] = (long long)i;
    }
    unsigned int step = 0;
    for (int w = 0; w < 8; ++w) step += warp_sum[w];
    __syncthreads();
    base += step;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) gs[ctrl->distinct] = (long long)n;
}

// ---- the grouped pass ----------------------------------------------------------------------------
template <int ORDER>
__global__ void __launch_bounds__(kPsiThreads)
group_psi_kernel(int64_t n, double g_host, const double* g_dev, const int32_t* status_dev, Ctrl* ctrl, int slot,
                 int rank, int world, const float* __restrict__ gv, const long long* __restrict__ gs, PsiFin fin) {
  if (!ctrl->grouped) return;
  double g = g_host;
  if (g_dev) {
    if (*status_dev != PLUGIN_OK) return;
    g = *g_dev;
  }
  __shared__ double sv[kGroupT], sw[kGroupT];
  __shared__ Fx128 fx_red[kPsiThreads / 32];
  __shared__ long long s_tile;
  const int64_t m = ctrl->distinct;
  const int64_t nb = (m + kGroupT - 1) / kGroupT, tiles = nb * (nb + 1) / 2;
  const int64_t tb = tiles * rank / world, te = tiles * (rank + 1) / world;
  const double s = 1.0 / g;
  const int tid = threadIdx.x;
  Fx128 acc = {0ull, 0ll};
  for (;;) {
    __syncthreads();  // s_tile, sv, sw of the previous tile consumed
    if (tid == 0) s_tile = tb + (long long)atomicAdd(&ctrl->tile_counter[slot], 1ull);
    __syncthreads();
    const int64_t t = s_tile;
    if (t >= te) break;
    int64_t bi, bj;
    tile_coords(t, nb, bi, bj);
    const int64_t a0 = bi * kGroupT, b0 = bj * kGroupT;
    const int bcount = (int)((m - b0) < kGroupT ? (m - b0) : kGroupT);
    // distinct values ascending: the smallest |v_b - v_a| of an off-diagonal tile is
    // v[b0] - v[a0 + TG - 1]; beyond |u| = 37.65 every term is exactly 0 (exp_neg_half)
    if (bi != bj && ((double)__ldg(gv + b0) - (double)__ldg(gv + a0 + kGroupT - 1)) * s > 37.65) continue;
    if (tid < bcount) {
      sv[tid] = (double)__ldg(gv + b0 + tid);
      sw[tid] = (double)(__ldg(gs + b0 + tid + 1) - __ldg(gs + b0 + tid));
    }
    __syncthreads();
    const int64_t a = a0 + tid;
    if (a < m) {
      const double va = (double)__ldg(gv + a);
      const double ca = (double)(__ldg(gs + a + 1) - __ldg(gs + a));
      double row = 0.0;
      for (int j = 0; j < bcount; ++j) {
        const double u = (sv[j] - va) * s;
        const double tt = u * u;
        row = fma(hermite_t64<ORDER>(tt) * exp_neg_half(tt), sw[j], row);
      }
      fx_add(acc, fx_from_double(row * ca * (bi == bj ? 1.0 : 2.0)));
    }
  }
  // block reduction of the exact per-thread totals, one pair of atomics, last-CTA epilogue
  for (int o = 16; o; o >>= 1) {
    Fx128 other;
    other.lo = __shfl_xor_sync(0xffffffffu, acc.lo, o);
    other.hi = __shfl_xor_sync(0xffffffffu, acc.hi, o);
    fx_add(acc, other);
  }
  if ((tid & 31) == 0) fx_red[tid >> 5] = acc;
  __syncthreads();
  unsigned long long* g_lo = &ctrl->acc[slot].lo;
  unsigned long long* g_hi = reinterpret_cast<unsigned long long*>(&ctrl->acc[slot].hi);
  if (tid == 0) {
    Fx128 cta = {0ull, 0ll};
    for (int w = 0; w < kPsiThreads / 32; ++w) fx_add(cta, fx_red[w]);
    if (cta.lo != 0ull || cta.hi != 0ll) {
      const unsigned long long old = atomicAdd(g_lo, cta.lo);
      const unsigned long long carry = (old + cta.lo < old) ? 1ull : 0ull;
      atomicAdd(g_hi, (unsigned long long)cta.hi + carry);
    }
  }
  if (fin.what < 0) return;
  __shared__ bool last;
  if (tid == 0) {
    __threadfence();
    last = (atomicAdd(&ctrl->psi_done[slot], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || tid != 0) return;
  __threadfence();
  Fx128 total;
  total.lo = atomicExch(g_lo, 0ull);
  total.hi = (long long)atomicExch(g_hi, 0ull);
  ctrl->tile_counter[slot] = 0ull;
  ctrl->psi_done[slot] = 0u;
  if (fin.out) fin.out->path |= PLUGIN_PATH_GROUPED;
  finalize_total(fin.what, total, atomicAdd(&ctrl->nonfinite, 0) != 0, fin.out, n, fin.g, fin.r, fin.d_psi);
}

cudaError_t launch_group_build(const float* xs, int64_t n, Ctrl* ctrl, unsigned int* chunk_heads, float* gv, long long* gs,
                               const plugin_result* s1, cudaStream_t s) {
  if (n < kGroupMinN) return cudaSuccess;  // never grouped: ctrl->grouped stays 0 (memset)
  const unsigned int chunks = (unsigned int)((n + kGroupChunk - 1) / kGroupChunk);
  group_count_kernel<<<chunks, 256, 0, s>>>(xs, n, ctrl, chunk_heads, s1);
  group_write_kernel<<<chunks, 256, 0, s>>>(xs, n, ctrl, chunk_heads, gv, gs);
  return cudaGetLastError();
}

template <int ORDER>
static cudaError_t launch_g(int64_t n, double g, const double* g_dev, const int32_t* status_dev, Ctrl* ctrl, int slot,
                            int rank, int world, const float* gv, const long long* gs, cudaStream_t s, PsiFin fin) {
  static DevCache cap_cache;
  const int grid = dev_cached(cap_cache, [](int dev) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, group_psi_kernel<ORDER>, kPsiThreads, 0);
    return device_sms(dev) * (occ > 0 ? occ : 1);
  });
  // the tile count is only known on the device: one persistent wave; idle CTAs exit at once
  const int64_t max_tiles = [n] {
    const int64_t mb = (n / 4 + kGroupT) / kGroupT;
    return mb * (mb + 1) / 2;
  }();
  const int gr = (int)(max_tiles < grid ? (max_tiles < 1 ? 1 : max_tiles) : grid);
  group_psi_kernel<ORDER><<<gr, kPsiThreads, 0, s>>>(n, g, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, fin);
  return cudaGetLastError();
}

cudaError_t launch_group_psi(int64_t n, int r, double g_host, const double* g_dev, const int32_t* status_dev,
                             Ctrl* ctrl, int slot, int rank, int world, const float* gv, const long long* gs, cudaStream_t s,
                             PsiFin fin) {
  if (n < kGroupMinN) return cudaSuccess;  // never grouped (ctrl->grouped stays 0)
  switch (r) {
    case 0: return launch_g<0>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
    case 2: return launch_g<2>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
    case 4: return launch_g<4>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
    case 6: return launch_g<6>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
    case 8: return launch_g<8>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
    case 10: return launch_g<10>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
    case 12: return launch_g<12>(n, g_host, g_dev, status_dev, ctrl, slot, rank, world, gv, gs, s, fin);
  }
  return cudaErrorInvalidValue;
}

}  // namespace plg
