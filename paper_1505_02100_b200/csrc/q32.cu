// q32.cu -- the paper's own arithmetic on B200: the pair sums of
// Steps IV/VI in Q32.32 fixed point, with the hoisted
// reciprocal multiply and polynomial exp of the "fast" FPGA loop (Fig. 5, P:397-422;
// P:218-223).  Definitions Q1-Q7 in DESIGN.md §14:
//   mul(a, b) = floor(a b / 2^32) (128-bit product); u = mul(|d|, rg); t = mul(u, u);
//   term = 0 if t > 42, else mul(P_r(t), exp(-(t >> 1))), P_r by Horner with mul;
//   exp(x) = (Taylor_9(w) in Q2.62) >> (30 - k), x = k ln2 + w, k = round(x / ln2).
// Every operation is an integer operation on the IMAD/ALU pipes, so the sum is exact and the
// same in any order: the GPU total equals the oracle's bit for bit (tested).
//
// Layout: T x T tiles (T = 256 R) of the pair matrix of the (sorted) Q32.32 sample; the upper
// block triangle; diagonal tiles as full squares with weight 1, off-diagonal with weight 2,
// so the grid total is sum_i sum_j term (Eq. 5-7 without a mask).  Per thread R rows, j from
// shared memory; per-row int64 sums (|term| <= 15 * 2^32, <= T terms per row per tile), a
// per-CTA 128-bit sum, one 128-bit atomic add per CTA.
#include "common.cuh"
#include "steps.cuh"

namespace plg {

constexpr int kQ32R = 1;  // T = 256: at ~20 128-bit multiplies per pair even small tiles carry ample work,
                             // and n = 16384 still gets 2080 tiles to spread over the SMs
constexpr int kQ32T = kPsiThreads * kQ32R;

__device__ __forceinline__ long long q32_mul(long long a, long long b) {
  return (long long)(((__int128)a * (__int128)b) >> 32);
}
__device__ __forceinline__ long long q62_mul(long long a, long long b) {
  return (long long)(((__int128)a * (__int128)b) >> 62);
}

// Q2: real -> Q32.32, round to nearest, ties away from zero (v 2^32 is exact in fp64)
__device__ __forceinline__ long long q32_encode_scalar(double v) {
  const double s = v * 4294967296.0;
  const double a = floor(fabs(s) + 0.5);
  return (long long)(s < 0.0 ? -a : a);
}

// exp(x) for -21 <= x <= 0 in Q32.32 (Q3)
__device__ __forceinline__ long long q32_exp(long long x) {
  const long long y = q32_mul(x, 6196328019LL);              // x / ln2   (round(2^32 / ln2))
  const long long k = (y + 2147483648LL) >> 32;               // round half up, k <= 0
  const long long w = x - k * 2977044472LL;                   // x - k ln2 (round(2^32 ln2))
  const long long w62 = w * 1073741824LL;                     // Q2.62
  long long p = 12708570377060LL;                             // round(2^62 / 9!)
  p = q62_mul(p, w62) + 114377133393536LL;                    // 8!
  p = q62_mul(p, w62) + 915017067148291LL;                    // 7!
  p = q62_mul(p, w62) + 6405119470038039LL;                   // 6!
  p = q62_mul(p, w62) + 38430716820228233LL;                  // 5!
  p = q62_mul(p, w62) + 192153584101141163LL;                 // 4!
  p = q62_mul(p, w62) + 768614336404564651LL;                 // 3!
  p = q62_mul(p, w62) + 2305843009213693952LL;                // 2!
  p = q62_mul(p, w62) + 4611686018427387904LL;                // 1!
  p = q62_mul(p, w62) + 4611686018427387904LL;                // 0!
  const long long sh = 30 - k;
  return sh >= 63 ? 0 : (p >> sh);
}

// K^(r)(u)/phi(0) in Q32.32 for the pair zi, zj (Q4-Q5): a = |zi - zj| exactly (uint64, no
// overflow for any two int64), u = floor(a rg / 2^32) tested against 7 on the exact 128-bit
// product before it is narrowed (|d| rg can exceed 2^95 for arbitrary psi_r_q32 inputs)
template <int ORDER>
__device__ __forceinline__ long long q32_term(long long zi, long long zj, long long rg) {
  const long long one = 4294967296LL;
  const unsigned long long a = zi >= zj ? (unsigned long long)zi - (unsigned long long)zj
                                        : (unsigned long long)zj - (unsigned long long)zi;
  const unsigned __int128 ue = ((unsigned __int128)a * (unsigned __int128)(unsigned long long)rg) >> 32;
  if (ue > (unsigned __int128)(7 * one)) return 0;  // then t > 42 too; and u*u would leave int64 for u >= 46341
  const long long u = (long long)ue;
  const long long t = q32_mul(u, u);
  if (t > 42 * one) return 0;  // e^{-t/2} below the e^-21 clamp
  const long long e = q32_exp(-(t >> 1));
  long long P;
  if (ORDER == 4) P = q32_mul(t, t) - 6 * t + 3 * one;
  else P = q32_mul(q32_mul(t - 15 * one, t) + 45 * one, t) - 15 * one;
  return q32_mul(P, e);
}

template <int ORDER>
__global__ void __launch_bounds__(kPsiThreads)
psi_q32_kernel(const long long* __restrict__ zq, int64_t n, long long rg_host, const long long* rg_dev,
               const int32_t* status_dev, Ctrl* ctrl, int slot) {
  __shared__ long long sz[kQ32T];
  __shared__ unsigned long long red_lo[kPsiThreads / 32];
  __shared__ long long red_hi[kPsiThreads / 32];
  __shared__ long long s_tile;
  const int tid = threadIdx.x;
  if (status_dev && *status_dev != PLUGIN_OK) return;
  const long long rg = rg_dev ? *rg_dev : rg_host;
  const int64_t nb = (n + kQ32T - 1) / kQ32T, tiles = nb * (nb + 1) / 2;
  Fx128 cta = {0ull, 0ll};
  for (;;) {
    if (tid == 0) s_tile = (long long)atomicAdd(&ctrl->tile_counter[slot], 1ull);
    __syncthreads();
    const int64_t t = s_tile;
    if (t >= tiles) break;
    int64_t bi, bj;
    {  // row-major upper triangle incl. the diagonal (as psi_tile.cuh's tile_coords)
      double A = 2.0 * (double)nb + 1.0;
      int64_t b = (int64_t)((A - sqrt(A * A - 8.0 * (double)t)) * 0.5);
      if (b < 0) b = 0;
      if (b > nb - 1) b = nb - 1;
      while (b > 0 && b * nb - b * (b - 1) / 2 > t) --b;
      while (b + 1 < nb && (b + 1) * nb - (b + 1) * b / 2 <= t) ++b;
      bi = b;
      bj = b + (t - (b * nb - b * (b - 1) / 2));
    }
    const int64_t i0 = bi * kQ32T, j0 = bj * kQ32T;
    const int jcount = (int)((n - j0) < kQ32T ? (n - j0) : kQ32T);
    for (int q = tid; q < jcount; q += kPsiThreads) sz[q] = zq[j0 + q];
    long long zi[kQ32R];
#pragma unroll
    for (int k = 0; k < kQ32R; ++k) {
      const int64_t i = i0 + k * kPsiThreads + tid;
      zi[k] = (i < n) ? zq[i] : 0;
    }
    __syncthreads();
    long long tsum = 0;  // this thread's rows over the tile: <= R T 15 2^32 < 2^63
#pragma unroll
    for (int k = 0; k < kQ32R; ++k) {
      const int64_t i = i0 + k * kPsiThreads + tid;
      if (i >= n) continue;
      long long acc = 0;
      for (int j = 0; j < jcount; ++j) acc += q32_term<ORDER>(zi[k], sz[j], rg);
      tsum += acc;
    }
    // weight: off-diagonal tiles count (i, j) and (j, i)
    __int128 v = (__int128)tsum * ((bi == bj) ? 1 : 2);
    // warp / block reduction of the 128-bit values (exact)
    unsigned long long lo = (unsigned long long)v;
    long long hi = (long long)(v >> 64);
    for (int o = 16; o; o >>= 1) {
      const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
      const long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
      const unsigned long long s = lo + olo;
      hi = hi + ohi + (s < lo ? 1 : 0);
      lo = s;
    }
    if ((tid & 31) == 0) { red_lo[tid >> 5] = lo; red_hi[tid >> 5] = hi; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < kPsiThreads / 32; ++w) {
        const unsigned long long s = cta.lo + red_lo[w];
        cta.hi += red_hi[w] + (s < cta.lo ? 1 : 0);
        cta.lo = s;
      }
    }
    // the next iteration's first __syncthreads orders the reuse of sz / red
  }
  if (tid == 0 && (cta.lo != 0ull || cta.hi != 0ll)) {
    unsigned long long* g_lo = &ctrl->acc[slot].lo;
    unsigned long long* g_hi = reinterpret_cast<unsigned long long*>(&ctrl->acc[slot].hi);
    const unsigned long long old = atomicAdd(g_lo, cta.lo);
    const unsigned long long carry = (old + cta.lo < old) ? 1ull : 0ull;
    atomicAdd(g_hi, (unsigned long long)cta.hi + carry);
  }
}

// total -> out[0] (low 64 bits), out[1] (high 64 bits) if out; resets the slot.  With res:
// finalize the PLUGIN pass `what` (0: Step IV -> V, 1: Step VI -> VII) from S = total / 2^32
// (= sum_i sum_j K^(r)(u_ij) / phi(0)) and, after the first pass, rg2 = encode(1 / g2_z).
__global__ void q32_finalize_kernel(Ctrl* ctrl, int slot, long long* out, int what, plugin_result* res,
                                    long long* rg_next) {
  const Fx128 acc = ctrl->acc[slot];
  ctrl->acc[slot].lo = 0ull;
  ctrl->acc[slot].hi = 0ll;
  ctrl->tile_counter[slot] = 0ull;
  if (out) {
    out[0] = (long long)acc.lo;
    out[1] = acc.hi;
  }
  if (!res || res->status != PLUGIN_OK) return;
  const double S = (double)acc.hi * 4294967296.0 + (double)acc.lo * 2.3283064365386962890625e-10;
  finalize_pass(what, S, res->n, res);
  if (what == 0 && res->status == PLUGIN_OK) *rg_next = q32_encode_scalar(1.0 / res->g2_z);
}

// rg1 = encode(1 / g1_z) after Step I-III
__global__ void q32_rg1_kernel(const plugin_result* res, long long* rg) {
  if (res->status == PLUGIN_OK) *rg = q32_encode_scalar(1.0 / res->g1_z);
}

// Q2 on the device for plugin_h_q32: z_i = (x_i - mean) / sigma in fp64 (Eq. 3), encoded to
// Q32.32 with round-half-away-from-zero; mean/sigma from Step I (status checked)
__global__ void q32_encode_kernel(const float* __restrict__ xs, int64_t n, const plugin_result* s1,
                                  long long* __restrict__ zq) {
  if (s1->status != PLUGIN_OK) return;
  const double mu = s1->mean, sg = s1->sigma;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    zq[i] = q32_encode_scalar(((double)xs[i] - mu) / sg);
  }
}

cudaError_t launch_psi_q32(const long long* zq, int64_t n, long long rg_host, const long long* rg_dev,
                           const int32_t* status_dev, int r, Ctrl* ctrl, int slot, long long* out, int what,
                           plugin_result* res, long long* rg_next, cudaStream_t s) {
  static DevCache cap_cache;
  const int grid_cap = dev_cached(cap_cache, [](int dev) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, psi_q32_kernel<6>, kPsiThreads, 0);
    return device_sms(dev) * (occ > 0 ? occ : 1);
  });
  const int64_t nb = (n + kQ32T - 1) / kQ32T, tiles = nb * (nb + 1) / 2;
  const int grid = (int)(tiles < grid_cap ? (tiles < 1 ? 1 : tiles) : grid_cap);
  if (r == 6) psi_q32_kernel<6><<<grid, kPsiThreads, 0, s>>>(zq, n, rg_host, rg_dev, status_dev, ctrl, slot);
  else psi_q32_kernel<4><<<grid, kPsiThreads, 0, s>>>(zq, n, rg_host, rg_dev, status_dev, ctrl, slot);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  q32_finalize_kernel<<<1, 1, 0, s>>>(ctrl, slot, out, what, res, rg_next);
  return cudaGetLastError();
}

cudaError_t launch_q32_rg1(const plugin_result* res, long long* rg, cudaStream_t s) {
  q32_rg1_kernel<<<1, 1, 0, s>>>(res, rg);
  return cudaGetLastError();
}

cudaError_t launch_q32_encode(const float* xs, int64_t n, const plugin_result* s1, long long* zq, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * 148) blocks = 4 * 148;
  q32_encode_kernel<<<(unsigned)blocks, 256, 0, s>>>(xs, n, s1, zq);
  return cudaGetLastError();
}

}  // namespace plg
