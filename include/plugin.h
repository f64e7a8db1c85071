/*
 * plugin.h -- C ABI of libplugin.so, the B200 (sm_100a) hot path of the
 * two-stage Gaussian PLUGIN bandwidth selector of arXiv 1505.02100
 * (Algorithm 1).
 *
 * Problem statement: "data set X containing n elements" -> "value h
 * represents the optimal bandwidth for kernel density estimation".  The O(n^2)
 * part is Steps IV and VI, the pairwise functionals
 *     Psi_r(g) = (n^2 g^(r+1))^-1 sum_i sum_j K^(r)((X_i - X_j)/g),  r in {6, 4},
 * evaluated with the symmetry of Eq. 5-7; everything else is O(n)
 * (Step I) or O(1) (Steps II, III, V, VII, Eq. 4).
 *
 * Conventions for every entry point
 *  - Pointers named d_* are CUDA device pointers on the current device; h_* are
 *    host pointers.  `stream` is a cudaStream_t passed as void* (0 = legacy stream).
 *  - The caller owns all memory: the input sample, the result, the workspace.
 *    The library allocates nothing, keeps no global mutable state except a
 *    thread-local error string, and never synchronises the stream except in the
 *    *_sync / *_host calls; the asynchronous calls are CUDA-graph capturable.
 *  - Input X is float32, contiguous, not modified.  Workspace: at least
 *    plugin_workspace_bytes(n) bytes, 256-byte aligned, no initialisation needed;
 *    two calls may run concurrently only with distinct workspaces.
 *  - Return value (plugin_status): immediate errors only -- PLUGIN_E_INVALID for
 *    bad arguments (null pointer, n out of range, r not even in [0,12], g not finite
 *    and > 0, workspace too small, rank/world inconsistent) and PLUGIN_E_CUDA for
 *    a launch failure.  Data-dependent errors (non-finite sample, zero variance,
 *    psi6 >= 0, psi4 <= 0) are written by the device into plugin_result.status;
 *    fields that were not reached are NaN.  plugin_last_error() describes the
 *    last non-OK return of the calling thread.  Nothing aborts or throws.
 *  - Units: fields without suffix are in the data's own units (Eq. 4 applied);
 *    *_z fields are the paper's z-score units (Eq. 3).
 */
#ifndef PAPER_1505_02100_PLUGIN_H
#define PAPER_1505_02100_PLUGIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PLUGIN_OK = 0,
  PLUGIN_E_INVALID = 1,     /* bad argument (immediate)                                  */
  PLUGIN_E_NONFINITE = 2,   /* NaN/Inf in X (device status)                              */
  PLUGIN_E_DEGENERATE = 3,  /* Step I variance V <= 0, e.g. all X equal (device status)  */
  PLUGIN_E_DOMAIN = 4,      /* psi6 >= 0 (Step V) or psi4 <= 0 (Step VII) (device)       */
  PLUGIN_E_CUDA = 5         /* a CUDA launch / copy failed (immediate)                   */
} plugin_status;

/* plugin_result.path bits: how the device evaluated the O(n^2) steps */
#define PLUGIN_PATH_GROUPED 1  /* the exact fp64 pass over distinct values (heavily tied sample) */

/* Written by the device.  Layout is part of the ABI (int32,int32,int64, then doubles). */
typedef struct {
  int32_t status;     /* plugin_status of the data-dependent checks                          */
  int32_t path;       /* PLUGIN_PATH_* bits (plugin_h / psi_r; 0 from the multi-GPU calls)   */
  int64_t n;
  double mean;        /* Step I: sample mean                                       */
  double var;         /* Step I: V = sum X^2/(n-1) - (sum X)^2/(n(n-1)) (evaluated shifted)   */
  double sigma;       /* Step I: sigma = sqrt(V)                                             */
  double psi8_ns;     /* Step II: 105/(32 sqrt(pi) sigma^9)                        */
  double g1;          /* Step III                                                  */
  double psi6;        /* Step IV at g1                                            */
  double g2;          /* Step V                                                  */
  double psi4;        /* Step VI at g2                                           */
  double h;           /* Step VII with Eq. 4: h = h_z * sigma         */
  double g1_z, psi6_z, g2_z, psi4_z, h_z;   /* the same in z-score units (sigma_z = 1)       */
  double S6, S4;      /* sum_i sum_j P_r(t_ij) 2^(-t_ij log2(e)/2), t = ((X_i-X_j)/g)^2: the
                         full double sums of Steps IV/VI divided by phi(0) (diagnostics)     */
} plugin_result;

/* Fixed-point partial of a psi pass (multi-GPU building block):
 * the sum over this rank's pairs as a signed 128-bit integer in units of 2^-64,
 * stored as four 32-bit limbs held in int64 (limb k = bits [32k, 32k+32), limb 3
 * signed).  Integer addition is associative, so an NCCL allreduce(SUM, int64) of
 * these 4 words over any number of ranks gives the bit-identical total. */
typedef struct { int64_t limb[4]; } plugin_fx128;

/* Bytes of workspace needed for n samples (covers every call below). */
size_t plugin_workspace_bytes(int64_t n);

/*
 * plugin_h: the whole Algorithm 1 on the device, asynchronously on `stream`.
 *   d_x   : device float32[n], n >= 2 (Step I divides by n-1; reading s9 of DESIGN.md)
 *   d_out : device plugin_result, written when the stream reaches the end of the call
 * Launches: a sort of X into the workspace (summation order only), the Step I reduction,
 * the Step IV pass, its finalize (psi6, g2), the Step VI pass, its finalize (psi4, h);
 * for n <= 2048 all of it is one thread-block-cluster launch with the same results (plugin_h_ex).
 */
plugin_status plugin_h(const float* d_x, int64_t n, plugin_result* d_out,
                       void* d_ws, size_t ws_bytes, void* stream);

/* plugin_h with option flags (0 = plugin_h).  PLUGIN_SKIP_UNDERFLOW: in both passes, skip
 * the tiles of the sorted pair triangle in which every |X_i - X_j|/g exceeds 13.25: there
 * every fp32 term is exactly zero (the exponent is below -127 and MUFU.EX2 flushes), so the
 * result is bit-identical to plugin_h; only the work changes (the
 * headline pair rate is always measured without it).  Unknown bits -> PLUGIN_E_INVALID. */
#define PLUGIN_SKIP_UNDERFLOW 1u
/* PLUGIN_MULTI_KERNEL: for n <= 2048 plugin_h runs the whole algorithm in one cluster
 * launch (sort, Step I, both passes and the scalar steps; bit-identical to the multi-kernel
 * sequence); this flag forces the multi-kernel sequence instead (testing, timing). */
#define PLUGIN_MULTI_KERNEL 2u
plugin_status plugin_h_ex(const float* d_x, int64_t n, plugin_result* d_out, unsigned int flags,
                          void* d_ws, size_t ws_bytes, void* stream);

/* Many independent small samples in one launch (throughput for batches of the paper's sizes):
 * sample b is d_x[d_offsets[b] .. d_offsets[b+1]) (device float32 / int64[count + 1], ascending
 * offsets), 2 <= n_b <= 2048; d_out[b] (device plugin_result[count]) receives Algorithm 1 for it
 * (the same Step I as plugin_h; the passes use larger tiles, so psi/h agree with plugin_h to fp32
 * evaluation rounding, not bit for bit).  A sample outside [2, 2048] gets status
 * PLUGIN_E_INVALID in its result.  One CTA per sample, no workspace.  flags: 0 or
 * PLUGIN_SKIP_UNDERFLOW.  Asynchronous. */
plugin_status plugin_h_batch(const float* d_x, const int64_t* d_offsets, int count, plugin_result* d_out,
                             unsigned int flags, void* stream);

/* plugin_h as a CUDA graph, for repeated runs on the same buffers (the launch latency of the
 * kernel sequence -- or of the one cluster launch for n <= 2048 -- is paid once at
 * creation).  plugin_graph_create captures plugin_h_ex(d_x, n, d_out, flags, d_ws, ws_bytes)
 * with its arguments fixed: the caller keeps d_x, d_out and d_ws alive and may change the
 * CONTENTS of d_x between launches.  The handle (host memory, owned by the caller) is freed by
 * plugin_graph_destroy.  plugin_graph_launch runs it on `stream`, asynchronously. */
typedef struct plugin_graph plugin_graph;
plugin_status plugin_graph_create(const float* d_x, int64_t n, plugin_result* d_out, void* d_ws,
                                  size_t ws_bytes, unsigned int flags, plugin_graph** out_graph);
plugin_status plugin_graph_launch(plugin_graph* graph, void* stream);
void plugin_graph_destroy(plugin_graph* graph);

/* Same as plugin_h -- Algorithm 1, X -> h (Eq. 3-4) -- with the device result kept in
 * the workspace, then synchronises `stream`, copies the result to *h_out and returns its data
 * status (PLUGIN_OK or one of E_NONFINITE/E_DEGENERATE/E_DOMAIN). */
plugin_status plugin_h_sync(const float* d_x, int64_t n, plugin_result* h_out,
                            void* d_ws, size_t ws_bytes, void* stream);

/* End to end from HOST memory: copies h_x (float32[n], ideally pinned) into the
 * workspace, runs plugin_h, copies the result back to *h_out, synchronises and
 * returns the data status.  Needs plugin_host_workspace_bytes(n) bytes of workspace
 * (= plugin_workspace_bytes(n) plus room for the copy of X). */
size_t plugin_host_workspace_bytes(int64_t n);
plugin_status plugin_h_host(const float* h_x, int64_t n, plugin_result* h_out,
                            void* d_ws, size_t ws_bytes, void* stream);

/*
 * psi_r: Psi_r(g) of Steps IV/VI for a given bandwidth g (data units), r in {4,6} (and any
 * even r <= 12 with K^(r) = He_r(u) phi(u), the family of plugin_dpi):
 *   Psi_r(g) = (n^2 g^(r+1))^-1 sum_{i,j} K^(r)((x_i - x_j)/g), diagonal included,
 * evaluated as 2 sum_{i<j} + n K^(r)(0) (Eq. 6/7).  n >= 1, g finite > 0.
 * *d_psi (device double) is written; a non-finite sample makes it NaN.
 */
plugin_status psi_r(const float* d_x, int64_t n, double g, int r, double* d_psi,
                    void* d_ws, size_t ws_bytes, void* stream);

/* ---- multi-GPU building blocks (one process per GPU; the caller allreduces) ---- */

/* Steps I-III (V, sigma, Psi8^NS, g1) on this rank's full copy of X: fills mean, var,
 * sigma, psi8_ns, g1(_z), status in d_out and prepares the workspace (the sorted X, and the
 * distinct-value arrays of a heavily tied sample) for the psi shards.  Asynchronous. */
plugin_status plugin_step1(const float* d_x, int64_t n, plugin_result* d_out,
                           void* d_ws, size_t ws_bytes, void* stream);

/* One rank's share of a psi pass (Steps IV/VI, Eq. 6/7):
 * the work items [w*rank/world, w*(rank+1)/world) of the pair triangle (w = plugin_num_tiles(n, r)),
 * at the bandwidth of d_out (g1 for r=6, g2 for r=4 -- and g2 for the other even r <= 12 of
 * the plugin_dpi family, K^(r) = He_r phi), written as an unnormalised fixed-point
 * sum to *d_partial.  The items partition the pairs (sorted sample, upper block triangle,
 * diagonal tiles as full squares) identically for every world, and sums are exact integers:
 * any world gives the single-GPU bits.
 * Requires plugin_step1 (and plugin_after_psi6 for r=4) on the same workspace. */
plugin_status psi_r_shard(int64_t n, int r, int rank, int world, const plugin_result* d_out,
                          plugin_fx128* d_partial, void* d_ws, size_t ws_bytes, void* stream);

/* The same share at a bandwidth of the caller's choosing (SURVEY §8(b)'s psi_r_shard(x, n, g, r,
 * rank, world)): g (data units, finite > 0) from the host, any even r <= 12; the workspace must
 * hold d_x's preparation (plugin_prepare or plugin_step1).  Summing the partials of all ranks and
 * passing the total to plugin_psi_from_total gives psi_r(d_x, n, g, r) bit for bit. */
plugin_status psi_r_shard_g(int64_t n, double g, int r, int rank, int world, plugin_fx128* d_partial,
                            void* d_ws, size_t ws_bytes, void* stream);
/* Sort d_x into the workspace and run Step I (non-finite check) and the distinct-value count:
 * the preparation psi_r_shard_g needs.  Asynchronous. */
plugin_status plugin_prepare(const float* d_x, int64_t n, void* d_ws, size_t ws_bytes, void* stream);
/* Psi_r(g) = phi(0) S / (n^2 g^(r+1)) (Steps IV/VI) from the all-reduced fixed-point
 * total S of psi_r_shard_g, into *d_psi (device double).  Asynchronous; one thread. */
plugin_status plugin_psi_from_total(const plugin_fx128* d_total, int64_t n, double g, int r, double* d_psi,
                                    void* stream);

/* Finalize a pass from the all-reduced fixed-point total: Step IV's psi6 (Eq. 6) and
 * Step V's g2 for r=6, or Step VI's psi4 (Eq. 7), Step VII's h_z
 * and h = h_z sigma (Eq. 4) for r=4, into d_out (data status E_DOMAIN
 * if psi6 >= 0 or psi4 <= 0).  Asynchronous; one thread. */
plugin_status plugin_after_psi6(const plugin_fx128* d_total, plugin_result* d_out, void* stream);
plugin_status plugin_after_psi4(const plugin_fx128* d_total, plugin_result* d_out, void* stream);

/* The work items of the pass of order r (even, 0..12) for n samples -- a function of n and r
 * only: T x T tiles of the sorted sample's upper block triangle
 * (T = plugin_tile_edge(n, r): 64 for n <= 2048, else 256 R with R the rows per thread, which
 * depends on r: the r >= 6 passes use R <= 4); diagonal tiles are full squares, weight 1;
 * off-diagonal weight 2.  With 2000 to 5000 tiles (n ~ 32K-50K and 64.5K-101K) the last
 * tiles mod 148 tiles are split column-wise into items of 64 columns, so that a pass ends on fine
 * items (the A/B switch PLUGIN_PSI_TAIL=0 keeps every tile whole; 1 and 2 split from 148 tiles on).
 * plugin_num_tiles: the number of items;
 * plugin_shard_tiles: the item range [begin, end) that `rank` of `world` owns (what
 * psi_r_shard / psi_r_shard_g process for that r, balanced to one item; an empty range for a
 * bad rank, world or r); plugin_work_item: the pairs of one item, out5 = {row begin, row end,
 * column begin, column end, weight} (sorted indices), 0 on success, -1 if item or r is out of
 * range.  Host-only; no CUDA call. */
int64_t plugin_num_tiles(int64_t n, int r);
void plugin_shard_tiles(int64_t n, int r, int rank, int world, int64_t* begin, int64_t* end);
int plugin_work_item(int64_t n, int r, int64_t item, int64_t* out5);
int64_t plugin_tile_edge(int64_t n, int r);

/* ---- the l-stage direct plug-in family ---- */

/*
 * Algorithm 1 is the l = 2 member of the direct plug-in family of the book the paper follows
 * ("the symbols used are exactly such as in the book"):
 *     Psi_{2l+4} <- Psi^NS_{2l+4} = (-1)^(l+2) (2l+3)!! / (2^(l+3) sqrt(pi) sigma^(2l+5))
 *     for j = l..1:  g_j = (-2 K^(2j+2)(0) / (mu2 Psi_{2j+4} n))^(1/(2j+5)),
 *                    Psi_{2j+2} <- Psi_hat_{2j+2}(g_j)     (pair passes as Steps IV/VI)
 *     h = (R(K) / (mu2^2 Psi_4 n))^(1/5)                    (Step VII, Eq. 4)
 * l = 0 is the normal reference rule h = (4/(3n))^(1/5) sigma; l = 2 is plugin_h (bit-identical).
 * Arrays are indexed by stage: [j-1] holds g_j and Psi_{2j+2}(g_j).
 */
#define PLUGIN_DPI_MAX_STAGES 5
typedef struct {
  int32_t status;     /* plugin_status of the data-dependent checks (as plugin_result)          */
  int32_t stages;     /* l                                                                      */
  int64_t n;
  double mean, var, sigma;                 /* Step I                                             */
  double psi_ns_z;                         /* Psi^NS_{2l+4}, z units (sigma_z = 1)              */
  double g_z[PLUGIN_DPI_MAX_STAGES], g[PLUGIN_DPI_MAX_STAGES];       /* z and data units        */
  double psi_z[PLUGIN_DPI_MAX_STAGES], psi[PLUGIN_DPI_MAX_STAGES];   /* z and data units        */
  double h_z, h;
} plugin_dpi_result;

/* The l-stage direct plug-in bandwidth, 0 <= stages <= 5 (passes of order 2l+2 .. 4, each
 * over the i<j triangle like Steps IV/VI); n >= 2; asynchronous; d_out on the device.
 * Needs plugin_workspace_bytes(n).  Data errors in d_out->status as for plugin_h. */
plugin_status plugin_dpi(const float* d_x, int64_t n, int stages, plugin_dpi_result* d_out,
                         void* d_ws, size_t ws_bytes, void* stream);

/* ---- the paper's own Q32.32 fixed-point datapath ---- */

/*
 * The FPGA design computes in Q32.32 fixed point with a hoisted reciprocal and a
 * polynomial exp in the hot loop (Fig. 5 "fast").  Here the pair sums of Steps IV/VI
 * run in that arithmetic on the integer pipes (definitions Q1-Q7 of DESIGN.md §14: floor-
 * truncating 128-bit multiplies, a Q2.62 Taylor exp with the e^-21 clamp, the symmetric pair
 * term of |z_i - z_j|); sums are exact 128-bit integers, so results are order-free and equal the
 * oracle's bit for bit.  A Q32.32 value is an int64 raw r meaning r / 2^32.
 *
 * psi_r_q32: *d_total (device int64[2], low then high 64 bits of a two's-complement int128) =
 *   sum_i sum_j term(zq_i - zq_j) over ALL ordered pairs (Eq. 5-7's left side), r in {4, 6};
 *   d_zq device int64[n] (Q32.32, |z| < 2^20), rg_q = Q32.32 reciprocal bandwidth in (0, 2^52).
 *   Psi_r(g) = phi(0) (total / 2^32) / (n^2 g^(r+1)).  Needs plugin_workspace_bytes(n).
 * plugin_h_q32: Algorithm 1 with both pair passes in Q32.32 on the z-scored sample (Eq. 3,
 *   encoded on the device) and the O(1) steps in fp64 (as plugin_h); needs
 *   plugin_q32_workspace_bytes(n).  Its h agrees with the fp64 h to the paper's Table 4 bound.
 */
size_t plugin_q32_workspace_bytes(int64_t n);
plugin_status psi_r_q32(const int64_t* d_zq, int64_t n, int64_t rg_q, int r, int64_t* d_total,
                        void* d_ws, size_t ws_bytes, void* stream);
plugin_status plugin_h_q32(const float* d_x, int64_t n, plugin_result* d_out,
                           void* d_ws, size_t ws_bytes, void* stream);

/* ---- the estimate the bandwidth is for ---- */

/* Bytes of workspace kde_eval needs for n samples and m points (>= plugin_workspace_bytes(n)). */
size_t kde_workspace_bytes(int64_t n, int64_t m);

/*
 * kde_eval: the kernel density estimator of Eq. 1 with the Gaussian kernel of
 * Eq. 2 at m points:
 *     d_f[k] = f(x_k, h) = (1/(n h)) sum_{i=1..n} K((x_k - X_i)/h),   K(u) = e^{-u^2/2}/sqrt(2 pi)
 *   d_x      : device float32[n], n >= 1, not modified
 *   d_points : device float32[m], m >= 0, any order (sorted or clustered points are
 *              faster: each block of 1024 points only reads the samples that can reach it)
 *   d_f      : device double[m], written
 *   h        : finite, 1e-18 <= h <= 1e18 (else PLUGIN_E_INVALID)
 * Each term is evaluated in fp32 (difference first) with MUFU.EX2; terms whose exponent is
 * below -126.5 are exactly zero in that arithmetic and are not visited.  Accumulation is
 * fp32 over 64 terms, then fp64, in a fixed order (bit-reproducible).  A non-finite sample
 * makes every d_f[k] NaN; a NaN point gives NaN at that point.  Asynchronous on `stream`.
 */
plugin_status kde_eval(const float* d_x, int64_t n, double h, const float* d_points, int64_t m,
                       double* d_f, void* d_ws, size_t ws_bytes, void* stream);

/* kde_eval in two steps, for many point sets or bandwidths over one sample:
 * kde_prepare sorts X into the workspace (and records whether it is all finite);
 * kde_eval_prepared(n, h, ...) then evaluates on that workspace (same n, same results as
 * kde_eval; the workspace must hold kde_workspace_bytes(n, m) for the largest m used). */
plugin_status kde_prepare(const float* d_x, int64_t n, void* d_ws, size_t ws_bytes, void* stream);
plugin_status kde_eval_prepared(int64_t n, double h, const float* d_points, int64_t m, double* d_f,
                                void* d_ws, size_t ws_bytes, void* stream);

/* The ordering step of the path (not a step of Alg. 1: it fixes the summation order, DESIGN.md
 * §6.4): d_sorted (device float32[n]) = X in ascending order of the IEEE bits' total order
 * (-NaN < -Inf < ... < -0 < +0 < ... < +Inf < +NaN), i.e. the unique array the passes read
 * (for n <= 32768 the NaN with payload bits 0x7fffffff comes out as 0x7ffffffe, another NaN).
 * Needs plugin_workspace_bytes(n); asynchronous. */
plugin_status plugin_sort(const float* d_x, int64_t n, float* d_sorted, void* d_ws, size_t ws_bytes,
                          void* stream);

/* Text of the last non-OK return on this thread ("" if none).  Static storage. */
const char* plugin_last_error(void);

/* Library / build identification, e.g. "libplugin sm_100a tile=2048". */
const char* plugin_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PAPER_1505_02100_PLUGIN_H */
