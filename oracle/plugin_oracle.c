/*
 * plugin_oracle.c -- plain, slow, fp64 CPU oracle for the two-stage Gaussian
 * PLUGIN bandwidth selector of arXiv 1505.02100 (Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1505_02100_b200/) never links, imports or executes it, and
 * this file shares no code, header, constant table or helper with the CUDA path.
 *
 * What lives here is only the O(n) and O(n^2) arithmetic of Alg. 1, written
 * literally in binary64 with glibc exp/sqrt (no blocking, fusion, reordering
 * or fast-math; compile with -O2 -fno-fast-math -ffp-contract=off).  The O(1)
 * scalar steps (II, III, V, VII, Eq. 4) are written in plain Python in
 * oracle/oracle.py so they can be read against the paper line by line.
 *
 * Parity pins: see tests/test_oracle_pins.py (closed forms for n=1,2, toy data,
 * 50-digit mpmath brute force for n<=16, Hermite/finite-difference checks of K,
 * moment identities, the quadrature identity, naive-vs-halved, scale/shift
 * invariants, the normal-density expectation).  Nothing here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double ORACLE_PI = 3.14159265358979323846264338327950288;

/* Neumaier (improved Kahan-Babuska) compensated summation. */
typedef struct { double s, c; } neumaier_t;
static void neumaier_add(neumaier_t* a, double v) {
  double t = a->s + v;
  if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
  else                       a->c += (v - t) + a->s;
  a->s = t;
}
static double neumaier_value(const neumaier_t* a) { return a->s + a->c; }

/* Eq. 2: Gaussian kernel K(u) = exp(-u^2/2)/sqrt(2 pi). */
double oracle_phi(double u) { return exp(-0.5 * u * u) / sqrt(2.0 * ORACLE_PI); }

/* Alg. 1 Step IV: K^(6)(x) = (1/sqrt(2pi)) (x^6 - 15x^4 + 45x^2 - 15) e^{-x^2/2}. */
double oracle_K6(double x) {
  double x2 = x * x, x4 = x2 * x2, x6 = x4 * x2;
  return (x6 - 15.0 * x4 + 45.0 * x2 - 15.0) * exp(-0.5 * x2) / sqrt(2.0 * ORACLE_PI);
}

/* Alg. 1 Step VI: K^(4)(x) = (1/sqrt(2pi)) (x^4 - 6x^2 + 3) e^{-x^2/2}. */
double oracle_K4(double x) {
  double x2 = x * x, x4 = x2 * x2;
  return (x4 - 6.0 * x2 + 3.0) * exp(-0.5 * x2) / sqrt(2.0 * ORACLE_PI);
}

/*
 * K^(r)(x) = d^r/dx^r phi(x) for any even r >= 0 (the r-th derivative
 * reading R1 of the kernels of Steps IV/VI):  phi^(r)(x) = (-1)^r He_r(x) phi(x) with the
 * probabilists' Hermite polynomials He_0 = 1, He_1 = x, He_{k+1} = x He_k - k He_{k-1}.
 */
double oracle_K_hermite(int r, double x) {
  if (r < 0 || (r & 1)) return NAN;
  double hm1 = 1.0, h = x;  /* He_0, He_1 */
  if (r == 0) return oracle_phi(x);
  for (int k = 1; k < r; ++k) {
    double hp1 = x * h - (double)k * hm1;
    hm1 = h;
    h = hp1;
  }
  return h * oracle_phi(x);
}

/* r = 6, 4: the printed polynomials of Steps IV/VI; other even r: the Hermite form above. */
double oracle_K(int r, double x) {
  if (r == 6) return oracle_K6(x);
  if (r == 4) return oracle_K4(x);
  return oracle_K_hermite(r, x);
}

/*
 * Alg. 1 Step I on the exact float32 input widened to fp64.
 * out[0] = sum X_i            (Neumaier)
 * out[1] = sum X_i^2          (Neumaier)
 * out[2] = mean = sum X_i / n
 * out[3] = V_onepass = sum X^2/(n-1) - (sum X)^2/(n(n-1))   -- Step I printed form
 * out[4] = V_twopass = sum (X_i - mean)^2 / (n-1)          -- its definition (R3)
 * out[5] = sigma = sqrt(V_twopass)
 * Returns 0 ok, 1 n<2, 2 non-finite input, 3 V<=0 (degenerate).
 */
int oracle_step1(const float* x, int64_t n, double* out) {
  for (int k = 0; k < 6; ++k) out[k] = NAN;
  if (n < 2) return 1;
  neumaier_t s1 = {0, 0}, s2 = {0, 0};
  for (int64_t i = 0; i < n; ++i) {
    double xi = (double)x[i];
    if (!isfinite(xi)) return 2;
    neumaier_add(&s1, xi);
    neumaier_add(&s2, xi * xi);
  }
  double S1 = neumaier_value(&s1), S2 = neumaier_value(&s2);
  double nd = (double)n;
  double mean = S1 / nd;
  double v1 = S2 / (nd - 1.0) - (S1 * S1) / (nd * (nd - 1.0));
  neumaier_t q = {0, 0};
  for (int64_t i = 0; i < n; ++i) {
    double dlt = (double)x[i] - mean;
    neumaier_add(&q, dlt * dlt);
  }
  double v2 = neumaier_value(&q) / (nd - 1.0);
  out[0] = S1; out[1] = S2; out[2] = mean; out[3] = v1; out[4] = v2;
  if (!(v2 > 0.0)) return 3;
  out[5] = sqrt(v2);
  return 0;
}

/* Eq. 3: Z_i = (X_i - mu) / sigma, fp64. */
void oracle_zscore(const float* x, int64_t n, double mu, double sigma, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = ((double)x[i] - mu) / sigma;
}

/* Widen float32 -> fp64 (exact), for the raw-unit path. */
void oracle_widen(const float* x, int64_t n, double* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = (double)x[i];
}

/*
 * The halved double sum of Eq. 6/7, restricted to rows
 * i in [i0, i1):  sum_{i0<=i<i1} sum_{j>i} K^(r)((z_i - z_j)/g)
 * (the division is literal, as in Alg. 1 Steps IV/VI).
 * Each row is a Neumaier sum over j in index order; rows are then combined in
 * index order with Neumaier.  Rows are independent, so the OpenMP split over i
 * does not change the result (bit-identical for any thread count).
 * out[0], out[1] = Neumaier (sum, compensation) of the row range.
 */
void oracle_psi_rows(const double* z, int64_t n, double g, int r, int64_t i0, int64_t i1,
                     int nthreads, double* out) {
  if (i0 < 0) i0 = 0;
  if (i1 > n) i1 = n;
  out[0] = 0.0; out[1] = 0.0;
  if (i1 <= i0) return;
  int64_t m = i1 - i0;
  double* row = (double*)malloc(sizeof(double) * (size_t)m);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = i0 + k;
    neumaier_t acc = {0, 0};
    for (int64_t j = i + 1; j < n; ++j) neumaier_add(&acc, oracle_K(r, (z[i] - z[j]) / g));
    row[k] = neumaier_value(&acc);
  }
  neumaier_t tot = {0, 0};
  for (int64_t k = 0; k < m; ++k) neumaier_add(&tot, row[k]);
  free(row);
  out[0] = tot.s; out[1] = tot.c;
}

/*
 * A rectangular block of the literal double sum of Steps IV/VI:
 * sum_{i0<=i<i1} sum_{j0<=j<j1} K^(r)((z_i - z_j)/g), per-row Neumaier, rows combined
 * in index order (OpenMP over rows; bit-identical for any thread count).
 * Used to check sampled blocks of a full-size pass one by one.
 */
void oracle_psi_block(const double* z, int64_t n, double g, int r, int64_t i0, int64_t i1,
                      int64_t j0, int64_t j1, int nthreads, double* out) {
  if (i0 < 0) i0 = 0;
  if (j0 < 0) j0 = 0;
  if (i1 > n) i1 = n;
  if (j1 > n) j1 = n;
  out[0] = 0.0; out[1] = 0.0;
  if (i1 <= i0 || j1 <= j0) return;
  int64_t m = i1 - i0;
  double* row = (double*)malloc(sizeof(double) * (size_t)m);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = i0 + k;
    neumaier_t acc = {0, 0};
    for (int64_t j = j0; j < j1; ++j) neumaier_add(&acc, oracle_K(r, (z[i] - z[j]) / g));
    row[k] = neumaier_value(&acc);
  }
  neumaier_t tot = {0, 0};
  for (int64_t k = 0; k < m; ++k) neumaier_add(&tot, row[k]);
  free(row);
  out[0] = tot.s; out[1] = tot.c;
}

/*
 * The literal full double sum of Alg. 1 Step IV/VI:
 * sum_{i=1..n} sum_{j=1..n} K^(r)((z_i - z_j)/g), Neumaier in (i, j) order.
 * Used for small n to check the halving of Eq. 5-7.
 */
double oracle_psi_literal_sum(const double* z, int64_t n, double g, int r) {
  neumaier_t acc = {0, 0};
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) neumaier_add(&acc, oracle_K(r, (z[i] - z[j]) / g));
  return neumaier_value(&acc);
}

/*
 * Eq. 1 with the Gaussian kernel of Eq. 2: the kernel density
 * estimator f(x, h) = (1/(n h)) sum_{i=1..n} K((x - X_i)/h) at m points x_k.
 * Literal: for every point a Neumaier sum over i in index order of
 * exp(-u^2/2)/sqrt(2 pi) with u = (x_k - X_i)/h, then one division by n h.
 * OpenMP over points (independent; bit-identical for any thread count).
 */
void oracle_kde(const float* X, int64_t n, double h, const double* xk, int64_t m, int nthreads,
                double* f) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
  for (int64_t k = 0; k < m; ++k) {
    neumaier_t acc = {0, 0};
    for (int64_t i = 0; i < n; ++i) neumaier_add(&acc, oracle_phi((xk[k] - (double)X[i]) / h));
    f[k] = neumaier_value(&acc) / ((double)n * h);
  }
}

/* ======================================================================================
 * The paper's Q32.32 fixed-point datapath for Steps IV/VI (Fig. 5 "fast" loop;
 * SURVEY §8(f) NEXT 2), written from its definition in DESIGN.md §14 (readings Q1-Q7).
 * A Q32.32 number is an int64 raw value v, meaning v / 2^32.  Integer arithmetic only: the
 * result is exact and independent of summation order.
 * ====================================================================================== */
typedef __int128 i128;

/* Q1: multiplication = the 128-bit product shifted right by 32 (floor, i.e. truncation toward
 * -inf, the SPEC ledger's choice; P:208-213 fix Q32.32 but not the rounding) */
int64_t oracle_q32_mul(int64_t a, int64_t b) { return (int64_t)(((i128)a * (i128)b) >> 32); }
static int64_t q62_mul(int64_t a, int64_t b) { return (int64_t)(((i128)a * (i128)b) >> 62); }

/* Q3: e^x for x <= 0 (the only arguments Steps IV/VI need): x = k ln2 + w, k = round(x/ln2),
 * e^w by its Taylor polynomial of degree 9 in Q2.62 (coefficients round(2^62/i!)), then a
 * right shift by -k.  e^x = 0 below x = -21 (SPEC ledger underflow clamp). */
static const int64_t Q32_LN2 = 2977044472LL;         /* round(ln 2 * 2^32)  */
static const int64_t Q32_INV_LN2 = 6196328019LL;     /* round(2^32 / ln 2)  */

/* c_i = round(2^62 / i!), i = 0..9 (exact integer arithmetic, ties up) */
static void q32_taylor(int64_t* c) {
  i128 fact = 1;
  for (int i = 0; i < 10; ++i) {
    if (i > 0) fact *= i;
    const i128 num = ((i128)1) << 62;
    c[i] = (int64_t)((num + fact / 2) / fact);
  }
}

static int64_t q32_exp_c(const int64_t* c, int64_t x) {
  if (x < -21LL * 4294967296LL) return 0;
  const int64_t y = oracle_q32_mul(x, Q32_INV_LN2);
  const int64_t k = (y + 2147483648LL) >> 32;        /* round half up */
  const int64_t w = x - k * Q32_LN2;
  const int64_t w62 = w * 1073741824LL;               /* Q32.32 -> Q2.62 */
  int64_t p = c[9];
  for (int i = 8; i >= 0; --i) p = q62_mul(p, w62) + c[i];
  const int64_t sh = 30 - k;
  return sh >= 63 ? 0 : (p >> sh);
}

int64_t oracle_q32_exp(int64_t x) {
  int64_t c[10];
  q32_taylor(c);
  return q32_exp_c(c, x);
}

/* Q4-Q5: the pair term of Steps IV/VI in Q32.32, K^(r)(u)/phi(0) with u = |d| * rg:
 * t = u^2; 0 if t > 42 (e^{-t/2} = 0 below -21); else P_r(t) * e^{-t/2} with the printed
 * polynomials evaluated by Horner in Q32.32.  a = |d| is the exact
 * magnitude of the difference of two Q32.32 values (a uint64: no overflow for any pair). */
static int64_t q32_term_c(const int64_t* c, uint64_t a, int64_t rg, int r) {
  const int64_t one = 4294967296LL;
  /* u > 7 implies t = floor(u^2) > 42, so the term is 0 (reading Q4).  The test is made on the
   * exact 128-bit product, before u is narrowed to int64 (|d| rg can exceed 2^95), and keeps
   * floor(u*u / 2^32) inside int64 (it wraps for u >= 46341) */
  const unsigned __int128 ue = ((unsigned __int128)a * (unsigned __int128)(uint64_t)rg) >> 32;
  if (ue > (unsigned __int128)(7 * one)) return 0;
  const int64_t u = (int64_t)ue;
  const int64_t t = oracle_q32_mul(u, u);
  if (t > 42 * one) return 0;
  const int64_t e = q32_exp_c(c, -(t >> 1));
  int64_t P;
  if (r == 4) P = oracle_q32_mul(t, t) - 6 * t + 3 * one;
  else P = oracle_q32_mul(oracle_q32_mul(t - 15 * one, t) + 45 * one, t) - 15 * one;
  return oracle_q32_mul(P, e);
}

/* |x - y| of two int64 without overflow */
static uint64_t q32_absdiff(int64_t x, int64_t y) {
  return x >= y ? (uint64_t)x - (uint64_t)y : (uint64_t)y - (uint64_t)x;
}

int64_t oracle_q32_term(int64_t d, int64_t rg, int r) {
  int64_t c[10];
  q32_taylor(c);
  return q32_term_c(c, q32_absdiff(d, 0), rg, r);
}

/* The halved sum of Eq. 6/7 in Q32.32: out = sum_{i<j} term(z_i - z_j) as an exact int128
 * (out[0] = low 64 bits, out[1] = high 64 bits, two's complement).  Rows in parallel, each
 * an exact integer sum: identical for any thread count and any order. */
void oracle_q32_psi_sum(const int64_t* zq, int64_t n, int64_t rg, int r, int nthreads, int64_t* out) {
  i128 total = 0;
  int64_t c[10];
  q32_taylor(c);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  i128* row = (i128*)malloc(sizeof(i128) * (size_t)(n > 0 ? n : 1));
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t i = 0; i < n; ++i) {
    i128 acc = 0;
    for (int64_t j = i + 1; j < n; ++j) acc += q32_term_c(c, q32_absdiff(zq[i], zq[j]), rg, r);
    row[i] = acc;
  }
  for (int64_t i = 0; i < n; ++i) total += row[i];
  free(row);
  out[0] = (int64_t)(uint64_t)total;
  out[1] = (int64_t)(total >> 64);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
