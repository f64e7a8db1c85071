// abi.cu -- the extern "C" boundary of libplugin.so (declared in include/plugin.h).
// Host-side argument checks, workspace layout and launch sequencing only; every step
// of the method runs in the kernels of scalar.cu / sort.cu / psi.cu.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>

#include "common.cuh"

namespace plg {

static thread_local char g_err[512] = "";

static plugin_status fail(plugin_status st, const char* fmt, const char* a = "", long long b = 0) {
  snprintf(g_err, sizeof(g_err), fmt, a, b);
  return st;
}
static plugin_status cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return PLUGIN_E_CUDA;
}

constexpr int64_t kMaxN = (int64_t)1 << 31;  // keeps tile indices and sort offsets in 32 bits

Layout layout(int64_t n) {
  Layout L;
  size_t off = 0;
  L.ctrl = off;
  off = align_up(off + sizeof(Ctrl), 256);
  L.step1 = off;
  off = align_up(off + sizeof(double) * 2 * kStep1Blocks, 256);
  L.xs = off;
  off = align_up(off + sizeof(float) * (size_t)(n > 0 ? n : 1), 256);
  L.tmp = off;
  off = align_up(off + sizeof(unsigned int) * (size_t)(n > 0 ? n : 1), 256);
  L.sort_blocks = (n + kSortTileSmall - 1) / kSortTileSmall;  // radix hist capacity (either tile)
  if (L.sort_blocks < 1) L.sort_blocks = 1;
  L.hist = off;
  off = align_up(off + sizeof(unsigned int) * 256 * (size_t)L.sort_blocks, 256);
  L.result = off;
  off = align_up(off + sizeof(plugin_result), 256);
  L.fused = off;
  off = align_up(off + sizeof(Fx128) * 2 * kFusedMaxGrid + 256, 256);  // fused.cu sort scratch (32 KB) + timing slots
  // group.cu: per-4096-chunk distinct counts, then at most n/4 distinct values and run starts (+1)
  const size_t nn = (size_t)(n > 0 ? n : 1);
  L.grp_heads = off;
  off = align_up(off + sizeof(unsigned int) * (nn / 4096 + 1), 256);
  L.grp_v = off;
  off = align_up(off + sizeof(float) * (nn / 4 + 1), 256);
  L.grp_s = off;
  off = align_up(off + sizeof(long long) * (nn / 4 + 2), 256);
  L.total = off;
  return L;
}

struct WS {
  Layout L;
  Ctrl* ctrl;
  double* step1;
  float* xs;
  unsigned int* tmp;
  unsigned int* hist;
  unsigned int* grp_heads;
  float* grp_v;
  long long* grp_s;
};

static plugin_status get_ws(void* d_ws, size_t ws_bytes, int64_t n, WS& w) {
  w.L = layout(n);
  if (!d_ws) return fail(PLUGIN_E_INVALID, "workspace pointer is null%s", "");
  if ((reinterpret_cast<uintptr_t>(d_ws) & 255u) != 0) return fail(PLUGIN_E_INVALID, "workspace not 256-byte aligned%s", "");
  if (ws_bytes < w.L.total)
    return fail(PLUGIN_E_INVALID, "workspace too small%s: need %lld bytes", "", (long long)w.L.total);
  char* b = static_cast<char*>(d_ws);
  w.ctrl = reinterpret_cast<Ctrl*>(b + w.L.ctrl);
  w.step1 = reinterpret_cast<double*>(b + w.L.step1);
  w.xs = reinterpret_cast<float*>(b + w.L.xs);
  w.tmp = reinterpret_cast<unsigned int*>(b + w.L.tmp);
  w.hist = reinterpret_cast<unsigned int*>(b + w.L.hist);
  w.grp_heads = reinterpret_cast<unsigned int*>(b + w.L.grp_heads);
  w.grp_v = reinterpret_cast<float*>(b + w.L.grp_v);
  w.grp_s = reinterpret_cast<long long*>(b + w.L.grp_s);
  return PLUGIN_OK;
}

static plugin_status check_n(int64_t n, int64_t nmin) {
  if (n < nmin || n > kMaxN) return fail(PLUGIN_E_INVALID, "n out of range%s (n=%lld)", "", (long long)n);
  return PLUGIN_OK;
}

// Step I..III + sort into the workspace
static plugin_status run_step1(const float* d_x, int64_t n, plugin_result* d_out, WS& w, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(w.ctrl, 0, sizeof(Ctrl), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset ctrl");
  // (step1_kernel's last block NaN-fills d_out before writing Steps I-III)
  // sort first: Step I then reads the sorted copy, so every result is a function of the
  // multiset of X only (bit-identical under any permutation of the input)
  if ((e = launch_sort(d_x, n, w.xs, w.tmp, w.hist, w.L.sort_blocks, s)) != cudaSuccess) return cuda_fail(e, "sort");
  if ((e = launch_step1(w.xs, n, w.ctrl, w.step1, d_out, s)) != cudaSuccess) return cuda_fail(e, "step1");
  // heavily tied samples: the passes run grouped by distinct value, exactly (group.cu)
  if ((e = launch_group_build(w.xs, n, w.ctrl, w.grp_heads, w.grp_v, w.grp_s, d_out, s)) != cudaSuccess)
    return cuda_fail(e, "group");
  return PLUGIN_OK;
}

// one pass over all of the pair triangle (or a rank's share): the fp32 tile pass and the grouped
// exact pass are both launched; the device runs the one ctrl->grouped selects
static cudaError_t pass(WS& w, int64_t n, int r, int skip, double g_host, const double* g_dev, const int32_t* status_dev,
                        int slot, int rank, int world, cudaStream_t s, PsiFin fin) {
  const int64_t tiles = psi_work_units(n, r);
  cudaError_t e = launch_psi(w.xs, n, r, skip, g_host, g_dev, status_dev, w.ctrl, slot, tiles * rank / world,
                             tiles * (rank + 1) / world, s, fin);
  if (e != cudaSuccess) return e;
  return launch_group_psi(n, r, g_host, g_dev, status_dev, w.ctrl, slot, rank, world, w.grp_v, w.grp_s, s, fin);
}

}  // namespace plg

using namespace plg;

extern "C" {

size_t plugin_workspace_bytes(int64_t n) { return layout(n).total; }

size_t plugin_host_workspace_bytes(int64_t n) {
  return layout(n).total + align_up(sizeof(float) * (size_t)(n > 0 ? n : 1), 256);
}

static bool valid_r(int r) { return r >= 0 && r <= 12 && !(r & 1); }

int64_t plugin_num_tiles(int64_t n, int r) { return n > 0 && valid_r(r) ? psi_work_units(n, r) : 0; }

int64_t plugin_tile_edge(int64_t n, int r) { return n > 0 && valid_r(r) ? psi_tile_edge(n, r) : 0; }

int plugin_work_item(int64_t n, int r, int64_t item, int64_t* out5) {
  if (!out5 || !valid_r(r)) return -1;
  return psi_work_item(n, r, item, out5) ? 0 : -1;
}

void plugin_shard_tiles(int64_t n, int r, int rank, int world, int64_t* begin, int64_t* end) {
  int64_t w = plugin_num_tiles(n, r);
  if (world < 1 || rank < 0 || rank >= world) {
    if (begin) *begin = 0;
    if (end) *end = 0;
    return;
  }
  // equal-work items (tiles for n <= 2048, else work units): contiguous, balanced to within one
  if (begin) *begin = (w * rank) / world;
  if (end) *end = (w * (rank + 1)) / world;
}

const char* plugin_last_error(void) { return g_err; }

const char* plugin_version(void) {
  return "libplugin 0.2 sm_100a (psi: f32x2 + MUFU.EX2, exact-staging centre, antithetic dither; "
         "grouped fp64 pass for tied samples; fx128 accumulation)";
}

plugin_status plugin_h(const float* d_x, int64_t n, plugin_result* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  return plugin_h_ex(d_x, n, d_out, 0u, d_ws, ws_bytes, stream);
}

plugin_status plugin_h_ex(const float* d_x, int64_t n, plugin_result* d_out, unsigned int flags, void* d_ws,
                          size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (flags & ~(unsigned int)(PLUGIN_SKIP_UNDERFLOW | PLUGIN_MULTI_KERNEL)) return fail(PLUGIN_E_INVALID, "unknown flags%s");
  const int skip = (flags & PLUGIN_SKIP_UNDERFLOW) ? 1 : 0;
  if (!d_x || !d_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (n <= kFusedMaxN && !(flags & PLUGIN_MULTI_KERNEL)) {
    // small n: the whole algorithm in one thread-block-cluster launch (fused.cu), bit-identical
    Fx128* parts = reinterpret_cast<Fx128*>(static_cast<char*>(d_ws) + w.L.fused);
    e = launch_fused(d_x, n, skip, d_out, parts, s);
    if (e == cudaSuccess) return PLUGIN_OK;
    if (e != cudaErrorNotSupported) return cuda_fail(e, "fused plugin");
    (void)cudaGetLastError();  // not applicable here: take the multi-kernel path
  }
  if ((st = run_step1(d_x, n, d_out, w, s)) != PLUGIN_OK) return st;
  // each pass finalises itself in its last CTA (Steps V / VII; PsiFin)
  PsiFin f6, f4;
  f6.what = 0, f6.out = d_out, f6.r = 6;
  f4.what = 1, f4.out = d_out, f4.r = 4;
  if ((e = pass(w, n, 6, skip, 0.0, &d_out->g1, &d_out->status, 0, 0, 1, s, f6)) != cudaSuccess)
    return cuda_fail(e, "psi6");
  if ((e = pass(w, n, 4, skip, 0.0, &d_out->g2, &d_out->status, 1, 0, 1, s, f4)) != cudaSuccess)
    return cuda_fail(e, "psi4");
  return PLUGIN_OK;
}

plugin_status plugin_h_sync(const float* d_x, int64_t n, plugin_result* h_out, void* d_ws, size_t ws_bytes,
                            void* stream) {
  if (!h_out) return fail(PLUGIN_E_INVALID, "null result pointer%s");
  WS w;
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  plugin_result* d_out = reinterpret_cast<plugin_result*>(static_cast<char*>(d_ws) + w.L.result);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = plugin_h(d_x, n, d_out, d_ws, ws_bytes, stream)) != PLUGIN_OK) return st;
  cudaError_t e = cudaMemcpyAsync(h_out, d_out, sizeof(plugin_result), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "copy result");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "sync");
  return static_cast<plugin_status>(h_out->status);
}

plugin_status plugin_h_host(const float* h_x, int64_t n, plugin_result* h_out, void* d_ws, size_t ws_bytes,
                            void* stream) {
  g_err[0] = 0;
  if (!h_x || !h_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  if (ws_bytes < plugin_host_workspace_bytes(n))
    return fail(PLUGIN_E_INVALID, "workspace too small%s: need %lld bytes", "", (long long)plugin_host_workspace_bytes(n));
  const Layout L = layout(n);
  const size_t base = L.total;
  char* b = static_cast<char*>(d_ws);
  float* d_x = reinterpret_cast<float*>(b + base);
  plugin_result* d_out = reinterpret_cast<plugin_result*>(b + L.result);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(d_x, h_x, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "copy X to device");
  if ((st = plugin_h(d_x, n, d_out, d_ws, base, stream)) != PLUGIN_OK) return st;
  if ((e = cudaMemcpyAsync(h_out, d_out, sizeof(plugin_result), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "copy result");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "sync");
  return static_cast<plugin_status>(h_out->status);
}

plugin_status psi_r(const float* d_x, int64_t n, double g, int r, double* d_psi, void* d_ws, size_t ws_bytes,
                    void* stream) {
  g_err[0] = 0;
  if (!d_x || !d_psi) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  if (r < 0 || r > 12 || (r & 1)) return fail(PLUGIN_E_INVALID, "r must be even, 0..12%s (r=%lld)", "", r);
  if (!(std::isfinite(g) && g > 0.0)) return fail(PLUGIN_E_INVALID, "g must be finite and > 0%s");
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(w.ctrl, 0, sizeof(Ctrl), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset ctrl");
  if ((e = launch_sort(d_x, n, w.xs, w.tmp, w.hist, w.L.sort_blocks, s)) != cudaSuccess) return cuda_fail(e, "sort");
  // Step I reduction only for its non-finite flag (a NaN/Inf sample makes Psi NaN); the distinct
  // count for the grouped exact pass
  plugin_result* scratch = reinterpret_cast<plugin_result*>(static_cast<char*>(d_ws) + w.L.result);
  if ((e = launch_step1(w.xs, n, w.ctrl, w.step1, scratch, s)) != cudaSuccess) return cuda_fail(e, "step1");
  if ((e = launch_group_build(w.xs, n, w.ctrl, w.grp_heads, w.grp_v, w.grp_s, scratch, s)) != cudaSuccess)
    return cuda_fail(e, "group");
  PsiFin fin;  // Psi_r(g) written by the pass's last CTA
  fin.what = 2, fin.g = g, fin.r = r, fin.d_psi = d_psi;
  if ((e = pass(w, n, r, 0, g, nullptr, nullptr, 1, 0, 1, s, fin)) != cudaSuccess) return cuda_fail(e, "psi");
  return PLUGIN_OK;
}

plugin_status plugin_step1(const float* d_x, int64_t n, plugin_result* d_out, void* d_ws, size_t ws_bytes,
                           void* stream) {
  g_err[0] = 0;
  if (!d_x || !d_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  return run_step1(d_x, n, d_out, w, static_cast<cudaStream_t>(stream));
}

plugin_status psi_r_shard(int64_t n, int r, int rank, int world, const plugin_result* d_out,
                          plugin_fx128* d_partial, void* d_ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_out || !d_partial) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  if (r < 0 || r > 12 || (r & 1)) return fail(PLUGIN_E_INVALID, "r must be even, 0..12%s (r=%lld)", "", r);
  if (world < 1 || rank < 0 || rank >= world) return fail(PLUGIN_E_INVALID, "bad rank/world%s");
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int slot = (r == 6) ? 0 : 1;
  cudaError_t e = pass(w, n, r, 0, 0.0, r == 6 ? &d_out->g1 : &d_out->g2, &d_out->status, slot, rank, world, s,
                       PsiFin());
  if (e != cudaSuccess) return cuda_fail(e, "psi shard");
  if ((e = launch_finalize(3, w.ctrl, slot, nullptr, nullptr, n, 0.0, r, nullptr, d_partial, s)) != cudaSuccess)
    return cuda_fail(e, "export partial");
  return PLUGIN_OK;
}

plugin_status plugin_prepare(const float* d_x, int64_t n, void* d_ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_x) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(w.ctrl, 0, sizeof(Ctrl), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset ctrl");
  if ((e = launch_sort(d_x, n, w.xs, w.tmp, w.hist, w.L.sort_blocks, s)) != cudaSuccess) return cuda_fail(e, "sort");
  plugin_result* scratch = reinterpret_cast<plugin_result*>(static_cast<char*>(d_ws) + w.L.result);
  if ((e = launch_step1(w.xs, n, w.ctrl, w.step1, scratch, s)) != cudaSuccess) return cuda_fail(e, "step1");
  if ((e = launch_group_build(w.xs, n, w.ctrl, w.grp_heads, w.grp_v, w.grp_s, scratch, s)) != cudaSuccess)
    return cuda_fail(e, "group");
  return PLUGIN_OK;
}

plugin_status psi_r_shard_g(int64_t n, double g, int r, int rank, int world, plugin_fx128* d_partial, void* d_ws,
                            size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_partial) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  if (r < 0 || r > 12 || (r & 1)) return fail(PLUGIN_E_INVALID, "r must be even, 0..12%s (r=%lld)", "", r);
  if (!(std::isfinite(g) && g > 0.0)) return fail(PLUGIN_E_INVALID, "g must be finite and > 0%s");
  if (world < 1 || rank < 0 || rank >= world) return fail(PLUGIN_E_INVALID, "bad rank/world%s");
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = pass(w, n, r, 0, g, nullptr, nullptr, 1, rank, world, s, PsiFin());
  if (e != cudaSuccess) return cuda_fail(e, "psi shard");
  if ((e = launch_finalize(3, w.ctrl, 1, nullptr, nullptr, n, 0.0, r, nullptr, d_partial, s)) != cudaSuccess)
    return cuda_fail(e, "export partial");
  return PLUGIN_OK;
}

plugin_status plugin_psi_from_total(const plugin_fx128* d_total, int64_t n, double g, int r, double* d_psi,
                                    void* stream) {
  g_err[0] = 0;
  if (!d_total || !d_psi) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  if (r < 0 || r > 12 || (r & 1)) return fail(PLUGIN_E_INVALID, "r must be even, 0..12%s (r=%lld)", "", r);
  if (!(std::isfinite(g) && g > 0.0)) return fail(PLUGIN_E_INVALID, "g must be finite and > 0%s");
  cudaError_t e = launch_finalize(2, nullptr, 0, d_total, nullptr, n, g, r, d_psi, nullptr,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "finalize");
  return PLUGIN_OK;
}

static plugin_status after(int what, const plugin_fx128* d_total, plugin_result* d_out, void* stream) {
  g_err[0] = 0;
  if (!d_total || !d_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  cudaError_t e = launch_finalize(what, nullptr, 0, d_total, d_out, 0, 0.0, what == 0 ? 6 : 4, nullptr, nullptr,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "finalize");
  return PLUGIN_OK;
}

plugin_status plugin_after_psi6(const plugin_fx128* d_total, plugin_result* d_out, void* stream) {
  return after(0, d_total, d_out, stream);
}
plugin_status plugin_after_psi4(const plugin_fx128* d_total, plugin_result* d_out, void* stream) {
  return after(1, d_total, d_out, stream);
}

plugin_status plugin_h_batch(const float* d_x, const int64_t* d_offsets, int count, plugin_result* d_out,
                             unsigned int flags, void* stream) {
  g_err[0] = 0;
  if (count < 0) return fail(PLUGIN_E_INVALID, "count must be >= 0%s");
  if (count == 0) return PLUGIN_OK;
  if (!d_x || !d_offsets || !d_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  if (flags & ~(unsigned int)PLUGIN_SKIP_UNDERFLOW) return fail(PLUGIN_E_INVALID, "unknown flags%s");
  cudaError_t e = launch_batch(d_x, d_offsets, count, (flags & PLUGIN_SKIP_UNDERFLOW) ? 1 : 0, d_out,
                               static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "batch");
  return PLUGIN_OK;
}

struct plugin_graph {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
};

plugin_status plugin_graph_create(const float* d_x, int64_t n, plugin_result* d_out, void* d_ws, size_t ws_bytes,
                                  unsigned int flags, plugin_graph** out_graph) {
  g_err[0] = 0;
  if (!out_graph) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  *out_graph = nullptr;
  cudaStream_t cs;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "graph stream");
  if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) {
    cudaStreamDestroy(cs);
    return cuda_fail(e, "begin capture");
  }
  plugin_status st = plugin_h_ex(d_x, n, d_out, flags, d_ws, ws_bytes, cs);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(cs, &graph);
  cudaStreamDestroy(cs);
  if (st != PLUGIN_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return cuda_fail(e, "end capture");
  cudaGraphExec_t exec;
  if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) {
    cudaGraphDestroy(graph);
    return cuda_fail(e, "instantiate");
  }
  plugin_graph* g = new (std::nothrow) plugin_graph{graph, exec};
  if (!g) {
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    return fail(PLUGIN_E_INVALID, "out of host memory%s");
  }
  *out_graph = g;
  return PLUGIN_OK;
}

plugin_status plugin_graph_launch(plugin_graph* g, void* stream) {
  g_err[0] = 0;
  if (!g) return fail(PLUGIN_E_INVALID, "null graph%s");
  cudaError_t e = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "graph launch");
  return PLUGIN_OK;
}

void plugin_graph_destroy(plugin_graph* g) {
  if (!g) return;
  cudaGraphExecDestroy(g->exec);
  cudaGraphDestroy(g->graph);
  delete g;
}

plugin_status plugin_sort(const float* d_x, int64_t n, float* d_sorted, void* d_ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_x || !d_sorted) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_sort(d_x, n, w.xs, w.tmp, w.hist, w.L.sort_blocks, s);
  if (e != cudaSuccess) return cuda_fail(e, "sort");
  if ((e = cudaMemcpyAsync(d_sorted, w.xs, sizeof(float) * (size_t)n, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "copy sorted");
  return PLUGIN_OK;
}

plugin_status plugin_dpi(const float* d_x, int64_t n, int stages, plugin_dpi_result* d_out, void* d_ws,
                         size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_x || !d_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  if (stages < 0 || stages > kDpiMaxStages) return fail(PLUGIN_E_INVALID, "stages must be 0..5%s");
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  plugin_result* s1 = reinterpret_cast<plugin_result*>(static_cast<char*>(d_ws) + w.L.result);
  if ((st = run_step1(d_x, n, s1, w, s)) != PLUGIN_OK) return st;
  cudaError_t e;
  if ((e = launch_dpi_init(s1, stages, d_out, s)) != cudaSuccess) return cuda_fail(e, "dpi init");
  for (int j = stages; j >= 1; --j) {
    const int slot = j & 1;
    if ((e = pass(w, n, 2 * j + 2, 0, 0.0, &d_out->g[j - 1], &d_out->status, slot, 0, 1, s, PsiFin())) !=
        cudaSuccess)
      return cuda_fail(e, "dpi pass");
    if ((e = launch_dpi_finalize(w.ctrl, slot, j, d_out, s)) != cudaSuccess) return cuda_fail(e, "dpi finalize");
  }
  return PLUGIN_OK;
}

size_t plugin_q32_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  return layout(n).total + align_up(sizeof(long long) * (size_t)n, 256) + 256;
}

plugin_status psi_r_q32(const int64_t* d_zq, int64_t n, int64_t rg_q, int r, int64_t* d_total, void* d_ws,
                        size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_zq || !d_total) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  if (r != 4 && r != 6) return fail(PLUGIN_E_INVALID, "r must be 4 or 6%s (r=%lld)", "", r);
  if (rg_q <= 0 || rg_q >= ((int64_t)1 << 52)) return fail(PLUGIN_E_INVALID, "rg_q must be in (0, 2^52)%s");
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(w.ctrl, 0, sizeof(Ctrl), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset ctrl");
  if ((e = launch_psi_q32(reinterpret_cast<const long long*>(d_zq), n, rg_q, nullptr, nullptr, r, w.ctrl, 1,
                          reinterpret_cast<long long*>(d_total), -1, nullptr, nullptr, s)) != cudaSuccess)
    return cuda_fail(e, "psi q32");
  return PLUGIN_OK;
}

plugin_status plugin_h_q32(const float* d_x, int64_t n, plugin_result* d_out, void* d_ws, size_t ws_bytes,
                           void* stream) {
  g_err[0] = 0;
  if (!d_x || !d_out) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 2);
  if (st != PLUGIN_OK) return st;
  if (ws_bytes < plugin_q32_workspace_bytes(n))
    return fail(PLUGIN_E_INVALID, "workspace too small%s: need %lld bytes", "", (long long)plugin_q32_workspace_bytes(n));
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  char* b = static_cast<char*>(d_ws);
  long long* zq = reinterpret_cast<long long*>(b + w.L.total);
  long long* rg = reinterpret_cast<long long*>(b + w.L.total + align_up(sizeof(long long) * (size_t)n, 256));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = run_step1(d_x, n, d_out, w, s)) != PLUGIN_OK) return st;
  cudaError_t e;
  if ((e = launch_q32_encode(w.xs, n, d_out, zq, s)) != cudaSuccess) return cuda_fail(e, "q32 encode");
  if ((e = launch_q32_rg1(d_out, rg, s)) != cudaSuccess) return cuda_fail(e, "q32 rg1");
  if ((e = launch_psi_q32(zq, n, 0, rg, &d_out->status, 6, w.ctrl, 0, nullptr, 0, d_out, rg + 1, s)) != cudaSuccess)
    return cuda_fail(e, "q32 psi6");
  if ((e = launch_psi_q32(zq, n, 0, rg + 1, &d_out->status, 4, w.ctrl, 1, nullptr, 1, d_out, nullptr, s)) !=
      cudaSuccess)
    return cuda_fail(e, "q32 psi4");
  return PLUGIN_OK;
}

size_t kde_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1) n = 1;
  if (m < 0) m = 0;
  return layout(n).total + kde_extra_bytes(n, m);
}

static plugin_status kde_check(int64_t n, double h, const float* d_points, int64_t m, double* d_f) {
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  if (m < 0 || m > kMaxN) return fail(PLUGIN_E_INVALID, "m out of range%s (m=%lld)", "", (long long)m);
  if (m > 0 && (!d_points || !d_f)) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  // h must be finite, > 0 and keep -log2(e)/(2 h^2) a normal float32
  if (!(std::isfinite(h) && h >= 1e-18 && h <= 1e18)) return fail(PLUGIN_E_INVALID, "h must be in [1e-18, 1e18]%s");
  return PLUGIN_OK;
}

plugin_status kde_prepare(const float* d_x, int64_t n, void* d_ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (!d_x) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  plugin_status st = check_n(n, 1);
  if (st != PLUGIN_OK) return st;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(w.ctrl, 0, sizeof(Ctrl), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset ctrl");
  if ((e = launch_sort(d_x, n, w.xs, w.tmp, w.hist, w.L.sort_blocks, s)) != cudaSuccess) return cuda_fail(e, "sort");
  // Step I reduction only for its non-finite flag (a NaN/Inf sample makes every f NaN)
  plugin_result* scratch = reinterpret_cast<plugin_result*>(static_cast<char*>(d_ws) + w.L.result);
  if ((e = launch_step1(w.xs, n, w.ctrl, w.step1, scratch, s)) != cudaSuccess) return cuda_fail(e, "step1");
  return PLUGIN_OK;
}

plugin_status kde_eval_prepared(int64_t n, double h, const float* d_points, int64_t m, double* d_f, void* d_ws,
                                size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  plugin_status st = kde_check(n, h, d_points, m, d_f);
  if (st != PLUGIN_OK) return st;
  if (m == 0) return PLUGIN_OK;
  WS w;
  if ((st = get_ws(d_ws, ws_bytes, n, w)) != PLUGIN_OK) return st;
  if (ws_bytes < kde_workspace_bytes(n, m))
    return fail(PLUGIN_E_INVALID, "workspace too small%s: need %lld bytes", "", (long long)kde_workspace_bytes(n, m));
  void* extra = static_cast<char*>(d_ws) + w.L.total;
  cudaError_t e = launch_kde(w.xs, n, h, d_points, m, w.ctrl, extra, d_f, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "kde");
  return PLUGIN_OK;
}

plugin_status kde_eval(const float* d_x, int64_t n, double h, const float* d_points, int64_t m, double* d_f,
                       void* d_ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  plugin_status st = kde_check(n, h, d_points, m, d_f);
  if (st != PLUGIN_OK) return st;
  if (!d_x) return fail(PLUGIN_E_INVALID, "null pointer argument%s");
  if (m == 0) return PLUGIN_OK;
  if (ws_bytes < kde_workspace_bytes(n, m))
    return fail(PLUGIN_E_INVALID, "workspace too small%s: need %lld bytes", "", (long long)kde_workspace_bytes(n, m));
  if ((st = kde_prepare(d_x, n, d_ws, ws_bytes, stream)) != PLUGIN_OK) return st;
  return kde_eval_prepared(n, h, d_points, m, d_f, d_ws, ws_bytes, stream);
}

}  // extern "C"
