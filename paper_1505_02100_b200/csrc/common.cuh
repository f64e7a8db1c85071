// common.cuh -- shared device/host pieces of libplugin.so (workspace layout,
// fixed-point accumulator, launch declarations).  Product code: nothing here is
// shared with oracle/.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/plugin.h"

namespace plg {

// ---- constants of Algorithm 1, fp64 -----------------------
constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kInvSqrt2Pi = 0.398942280401432677939946059934381868;  // phi(0), Eq. 2
constexpr double kK6at0 = -15.0 * kInvSqrt2Pi;   // Step III  K^6(0) = -15/sqrt(2 pi)
constexpr double kK4at0 = 3.0 * kInvSqrt2Pi;     // Step V  K^4(0) =  3/sqrt(2 pi)
constexpr double kRK = 0.282094791773878143474039725780386293;  // Step VII R(K) = 1/(2 sqrt(pi))
constexpr double kMu2 = 1.0;                                    // mu_2(K) = 1

// ---- tiling --------------------------------------------------------------------
constexpr int kPsiThreads = 256;   // threads per CTA of the psi pass
// keys per CTA in the radix sort: 2048 up to kSortTileSwitch keys (more CTAs for mid-size n),
// 4096 above (fewer, longer scatter CTAs; measured, profiles/r01af_sort_ab.txt)
constexpr int kSortTileSmall = 2048, kSortTileLarge = 4096;
constexpr int64_t kSortTileSwitch = 262144;
inline int sort_tile(int64_t n) { return n <= kSortTileSwitch ? kSortTileSmall : kSortTileLarge; }
constexpr int kSortThreads = 256;
constexpr int kStep1Blocks = 592;  // 4 x 148: fixed grid so Step I is deterministic
// Step I grid for n samples (a function of n only: the reduction tree, hence the result, is fixed)
inline __host__ __device__ int step1_grid(int64_t n) {
  const int64_t want = (n + 2047) / 2048;
  return (int)(want < kStep1Blocks ? (want < 1 ? 1 : want) : kStep1Blocks);
}
// the fused single-launch path (fused.cu) handles n up to this
constexpr int64_t kFusedMaxN = 2048;
// the grouped exact pass (group.cu) is considered from this n on, for samples with at most n / 4
// distinct values; below it the fp32 pass meets 1e-5 on the discretised test samples
// and the extra launches would weigh on the latency
constexpr int64_t kGroupMinN = 32768;

// rows per thread R as a function of n and the order r of the pass (tile edge T = 256 R); see
// DESIGN.md §5
int psi_rows_per_thread(int64_t n, int r);
// R = 0: the small-tile mode of psi_tile.cuh (T = 64, n <= kFusedMaxN)
inline int64_t psi_tile_edge(int64_t n, int r) {
  const int R = psi_rows_per_thread(n, r);
  return R == 0 ? 64 : (int64_t)kPsiThreads * R;
}
inline int64_t psi_blocks(int64_t n, int r) { int64_t T = psi_tile_edge(n, r); return (n + T - 1) / T; }
inline int64_t psi_tiles(int64_t n, int r) { int64_t b = psi_blocks(n, r); return b * (b + 1) / 2; }
// the pass's schedulable work items for n samples (a function of n and r only): whole tiles, then
// -- with 2000 to 5000 tiles, psi.cu -- the kTailCols-column slices of the remainder tiles; launch_psi
// ranges and the multi-GPU shards (plugin_shard_tiles) count these.  psi_work_item: rows
// [out0, out1), columns [out2, out3) and weight out4 of one item (host)
constexpr int kTailCols = 64;
constexpr int kSchedSms = 148;  // SMs of a B200: the remainder is tiles mod kSchedSms (a constant, so items depend on n only)
int psi_sched_mode(int64_t tiles);  // 0 whole tiles, 1 remainder slices, 2 slices + per-SM quota of the whole tiles
int64_t psi_work_units(int64_t n, int r);
int64_t psi_tail_head(int64_t n, int r);
bool psi_work_item(int64_t n, int r, int64_t item, int64_t* out);

// order-preserving float bits <-> uint32 radix key (sort.cu, fused.cu)
__device__ __forceinline__ unsigned int bits2key(unsigned int b) {
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ unsigned int key2bits(unsigned int k) {
  return (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
}

// ---- signed 128-bit fixed point, value = hi + lo * 2^-64 ------------------------
struct Fx128 { unsigned long long lo; long long hi; };

// ---- workspace layout ----------------------------------------------------------
struct Ctrl {                       // zeroed at the start of every API call
  Fx128 acc[2];                     // psi accumulators (slot 0: r=6, slot 1: r=4 / psi_r)
  unsigned long long tile_counter[2];  // dynamic tile scheduler per slot (64-bit: n^2 tiles can pass 2^32)
  unsigned int step1_done;          // last-block-done counter of Step I
  int nonfinite;                    // set if any X is NaN/Inf
  unsigned int psi_done[2];         // last-CTA-done counters of the psi passes (PsiFin)
  long long distinct;               // number of distinct values of the sample (group.cu)
  int grouped;                      // 1: the passes run grouped by distinct value in fp64 (group.cu)
  unsigned int group_done;          // last-CTA-done counter of group_count_kernel
  unsigned int sm_cnt[2][kSchedSms];  // whole tiles claimed per SM and slot (scheduler mode 2, psi.cu)
  unsigned int smq_used[2];         // a quota pass ran on the slot and its counters are not yet reset
  unsigned int pad[4];
};
static_assert(sizeof(Ctrl) <= 2048, "ctrl block");

struct Layout {
  size_t ctrl, step1, xs, tmp, hist, result, fused, grp_heads, grp_v, grp_s, total;
  int64_t sort_blocks;
};
Layout layout(int64_t n);

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---- per-device, set-once host caches (launch geometry, function attributes) --------
// Keyed by the CURRENT device: occupancy, SM counts and cudaFuncSetAttribute are per device, so
// a process that calls the library on several GPUs gets each device's own values.  f(dev) must
// return a value >= 0 and must be idempotent (two threads may both compute it the first time).
constexpr int kMaxDevices = 64;
struct DevCache {
  std::atomic<int> v[kMaxDevices];  // value + 1; 0 = not yet computed (static storage: zeroed)
};
template <class F>
inline int dev_cached(DevCache& c, F f) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return f(dev < 0 ? 0 : dev);
  int v = c.v[dev].load(std::memory_order_acquire);
  if (v == 0) {
    v = f(dev) + 1;
    c.v[dev].store(v, std::memory_order_release);
  }
  return v - 1;
}
inline int device_sms(int dev) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 1;
}

// ---- launchers (each returns cudaGetLastError()) ----------------------------------
cudaError_t launch_step1(const float* x, int64_t n, Ctrl* ctrl, double* partials, plugin_result* out,
                         cudaStream_t s);
cudaError_t launch_sort(const float* x, int64_t n, float* xs, unsigned int* tmp, unsigned int* hist,
                        int64_t nblocks, cudaStream_t s);
// One pass of Steps IV/VI (or Psi_r for any even r <= 12) over work items [tile_begin, tile_end)
// (psi_work_units):
// g from *g_dev (a device bandwidth; the pass is skipped unless *status_dev == PLUGIN_OK) or,
// if g_dev is null, g_host.  skip != 0: skip tiles whose terms are all exactly 0 (NEXT 4).
// The pass's epilogue, run by its last CTA to finish (saves the finalize launch): what = -1
// none, 0 / 1 = Steps V / VII of Alg. 1 into *out, 2 = Psi_r(g) into *d_psi (as finalize_kernel).
struct PsiFin {
  int what = -1;
  plugin_result* out = nullptr;
  double g = 0.0;
  int r = 0;
  double* d_psi = nullptr;
};
cudaError_t launch_psi(const float* xs, int64_t n, int r, int skip, double g_host, const double* g_dev,
                       const int32_t* status_dev, Ctrl* ctrl, int slot, int64_t tile_begin, int64_t tile_end,
                       cudaStream_t s, PsiFin fin = PsiFin());
// |u| beyond which every fp32 term of a pass is exactly zero (psi.cu, fused.cu)
constexpr double kSkipU = 13.25;
// what: 0 = plugin r=6 finalize, 1 = plugin r=4 finalize, 2 = psi_r -> d_psi, 3 = export limbs
cudaError_t launch_finalize(int what, Ctrl* ctrl, int slot, const plugin_fx128* total, plugin_result* out,
                            int64_t n, double g_host, int r, double* d_psi, plugin_fx128* d_limbs,
                            cudaStream_t s);
// the whole of Alg. 1 in one thread-block-cluster launch for n <= kFusedMaxN (fused.cu); parts: 32 KB
// of workspace scratch (the sort's runs and ascending array; 2 * kFusedMaxGrid Fx128 in size).
// Returns cudaErrorNotSupported if the path does not apply (no cluster of 8 can be scheduled).
constexpr int kFusedMaxGrid = 1024;
cudaError_t launch_fused(const float* x, int64_t n, int skip, plugin_result* out, Fx128* parts, cudaStream_t s);
// many samples of 2 <= n_b <= kFusedMaxN, one CTA each (fused.cu): offsets[count + 1] on the device
cudaError_t launch_batch(const float* x, const int64_t* offsets, int count, int skip, plugin_result* out,
                         cudaStream_t s);
// the Q32.32 datapath (q32.cu): one pass over the Q32.32 sample zq with rg from rg_dev (or
// rg_host), its exact 128-bit total to out[2] (if out) and, with res, the PLUGIN finalize of
// pass `what` (rg_next <- encode(1/g2_z) after pass 0)
cudaError_t launch_psi_q32(const long long* zq, int64_t n, long long rg_host, const long long* rg_dev,
                           const int32_t* status_dev, int r, Ctrl* ctrl, int slot, long long* out, int what,
                           plugin_result* res, long long* rg_next, cudaStream_t s);
cudaError_t launch_q32_encode(const float* xs, int64_t n, const plugin_result* s1, long long* zq, cudaStream_t s);
cudaError_t launch_q32_rg1(const plugin_result* res, long long* rg, cudaStream_t s);
// the l-stage direct plug-in (dpi.cu)
constexpr int kDpiMaxStages = PLUGIN_DPI_MAX_STAGES;
cudaError_t launch_dpi_init(const plugin_result* s1, int stages, plugin_dpi_result* out, cudaStream_t s);
cudaError_t launch_dpi_finalize(Ctrl* ctrl, int slot, int j, plugin_dpi_result* out, cudaStream_t s);
// the grouped exact pass (group.cu): count the distinct values of the sorted copy and decide
// (ctrl->grouped), compact them (gv values, gs run starts with gs[m] = n); then per pass
cudaError_t launch_group_build(const float* xs, int64_t n, Ctrl* ctrl, unsigned int* chunk_heads, float* gv, long long* gs,
                               const plugin_result* s1, cudaStream_t s);
cudaError_t launch_group_psi(int64_t n, int r, double g_host, const double* g_dev, const int32_t* status_dev,
                             Ctrl* ctrl, int slot, int rank, int world, const float* gv, const long long* gs, cudaStream_t s,
                             PsiFin fin = PsiFin());
// KDE of Eq. 1-2 at m points over the sorted sample xs (kde.cu); `extra` holds
// kde_extra_bytes(n, m) bytes of workspace
size_t kde_extra_bytes(int64_t n, int64_t m);
int kde_segments(int64_t n, int64_t m);
cudaError_t launch_kde(const float* xs, int64_t n, double h, const float* pts, int64_t m, const Ctrl* ctrl,
                       void* extra, double* f, cudaStream_t s);

}  // namespace plg
