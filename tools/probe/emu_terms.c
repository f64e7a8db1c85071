// Dev probe (not product, not oracle): CPU emulation of the psi pass's per-pair fp32
// arithmetic (psi_tile.cuh, centred form, T = 256 R tiles of the sorted sample), with each
// rounding switchable, to find which fp32 rounding dominates the error on discretised samples.
// The exp is exp2 of the (possibly rounded) argument in fp64 (the MUFU.EX2 table bias is a
// separate, measured effect: profiles/r01_numerics.md).
//   build: gcc -O2 -fopenmp -ffp-contract=off -o /tmp/emu tools/probe/emu_terms.c -lm
//   usage: emu <f32 sorted file> <n> <g> <r> <T> <flags> [variant]
// flags (bit): 1 dither s, 2 s in fp32, 4 round u (centred fma), 8 round t, 16 round a (fma,
// c2 fp32), 32 round e to fp32, 64 round P (fp32 Horner), 128 fp32 chunk accumulation,
// 256 c2 rounded to fp32 (exponent constant only), 512 round x'_i s_i only
// variant: 0 = current GPU, 1 = error-free u correction (t += 2 u u_lo), 2 = t from split
// prints: the weighted sum sum_w P(t) e^{-t/2} (w = 2 off-diagonal tiles, 1 diagonal: full squares)
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static unsigned int row_hash(int64_t i) { return (unsigned int)i * 2654435769u; }
static float row_phase(int64_t i) { return -1.0f - (float)(row_hash(i) >> 8) * (1.0f / 16777216.0f); }
static int row_scale_offset(int64_t i) {
  unsigned int h = ((unsigned int)i * 0x85EBCA6Bu) ^ 0x9E3779B9u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  return (int)(((h >> 16) * 15u) >> 16) - 7;
}
static int g_anti = 0;  // > 0: antithetic scale dither k_i in [-K, K], k_(2m+1) = -k_(2m)
static int anti_offset(int64_t i) {
  unsigned int h = ((unsigned int)(i >> 1) * 0x85EBCA6Bu) ^ 0x9E3779B9u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 13;
  int k = (int)(h % (unsigned)(2 * g_anti + 1)) - g_anti;
  return (i & 1) ? -k : k;
}
static float f32(double v) { return (float)v; }
static float u2f(unsigned int u) { float f; memcpy(&f, &u, 4); return f; }
static unsigned int f2u(float f) { unsigned int u; memcpy(&u, &f, 4); return u; }

static double poly(int r, double t) {
  if (r == 6) return ((t - 15) * t + 45) * t - 15;
  if (r == 4) return (t - 6) * t + 3;
  if (r == 8) return (((t - 28) * t + 210) * t - 420) * t + 105;
  return 1.0;
}
static float polyf(int r, float t) {
  if (r == 6) return fmaf(fmaf(t - 15.f, t, 45.f), t, -15.f);
  if (r == 4) return fmaf(t - 6.f, t, 3.f);
  if (r == 8) return fmaf(fmaf(fmaf(t - 28.f, t, 210.f), t, -420.f), t, 105.f);
  return 1.f;
}

int main(int argc, char** argv) {
  if (argc < 7) return 1;
  FILE* f = fopen(argv[1], "rb");
  int64_t n = atoll(argv[2]);
  double g = atof(argv[3]);
  int r = atoi(argv[4]);
  int T = atoi(argv[5]);
  int flags = atoi(argv[6]);
  int variant = argc > 7 ? atoi(argv[7]) : 0;
  if (argc > 8) g_anti = atoi(argv[8]);
  int cmode = argc > 9 ? atoi(argv[9]) : 0;
  int stride = argc > 10 ? atoi(argv[10]) : 1;  // evaluate rows i % stride == 0 only (sampled)  // tile centre: 0 x[i0], 1 x[i0] + random part of the row span, 2 zero, 3 difference first
  float* x = malloc(n * 4);
  if (fread(x, 4, n, f) != (size_t)n) return 2;
  fclose(f);
  const double LOG2E_2 = 0.72134752044448170368;  // log2(e)/2
  const float c2f = -0.72134752f;
  const double c2 = (flags & (16 | 256)) ? (double)c2f : -LOG2E_2;
  const float sf = f32(1.0 / g);
  int64_t nb = (n + T - 1) / T;
  double total = 0.0, comp = 0.0;
  const char* tb_env = getenv("EMU_TILE_BI");  // restrict to one tile (bi, bj)
  const int64_t only_bi = tb_env ? atoll(tb_env) : -1, only_bj = tb_env ? atoll(getenv("EMU_TILE_BJ")) : -1;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total)
  for (int64_t bi = 0; bi < nb; ++bi) {
    double tot_b = 0.0;
    if (only_bi >= 0 && bi != only_bi) continue;
    for (int64_t bj = bi; bj < nb; ++bj) {
      if (only_bj >= 0 && bj != only_bj) continue;
      const int64_t i0 = bi * T, j0 = bj * T;
      const double w = (bi == bj) ? 1.0 : 2.0;
      float cen = x[i0];
      int64_t ri0 = i0, rj0 = j0;  // register-side block, staged block
      if (cmode == 6) {  // the kernel's rule (psi_tile_centre), rows always in registers
        const int64_t jl = (j0 + T < n ? j0 + T : n) - 1;
        const float a = x[i0], q = x[jl];
        if (a >= 0.f) {
          const float uq = nextafterf(q, INFINITY) - q;
          cen = (q <= 2.f * a) ? a : truncf(a / uq) * uq;
        } else if (q <= 0.f) {
          const float ua = nextafterf(-a, INFINITY) + a;
          cen = (a >= 2.f * q) ? q : truncf(q / ua) * ua;
        } else {
          cen = 0.f;
        }
      }
      if (cmode == 5) {
        const int64_t il = (i0 + T < n ? i0 + T : n) - 1;
        const int64_t jl = (j0 + T < n ? j0 + T : n) - 1;
        const float a = x[i0], b = x[il], pp = x[j0], q = x[jl];
        if (a >= 0.f) {
          const float uq = nextafterf(q, INFINITY) - q;
          cen = truncf(a / uq) * uq;
        } else if (q <= 0.f) {
          const float ua = nextafterf(-a, INFINITY) + a;
          cen = truncf(q / ua) * ua;
          ri0 = j0; rj0 = i0;
        } else {
          cen = 0.f;
          if (!(b >= 0.f) && pp <= 0.f) { ri0 = j0; rj0 = i0; }
        }
      }
      if (cmode == 1) {
        const int64_t il = (i0 + T < n ? i0 + T : n) - 1;
        unsigned int h = (unsigned int)(bi * 7919 + bj) * 2654435769u;
        h ^= h >> 16;
        cen = x[i0] + (x[il] - x[i0]) * (float)(h & 0xffff) * (1.0f / 65536.0f);
      } else if (cmode == 2) {
        cen = 0.f;
      } else if (cmode == 4) {
        // exact-staging centre: every x - cen exact (rows and columns)
        const int64_t il = (i0 + T < n ? i0 + T : n) - 1;
        const int64_t jl = (j0 + T < n ? j0 + T : n) - 1;
        const float a = x[i0], b = x[il], q = x[jl];
        if (a > 0.f) {
          // a rounded toward zero to a multiple of ulp(q)
          const float uq = nextafterf(q, INFINITY) - q;
          cen = (q <= 2.f * a) ? a : floorf(a / uq) * uq;
        } else if (q < 0.f) {
          cen = (-(double)a * sf >= 32.0 + 2.0 * ((double)b - (double)a) * sf) ? a : 0.f;
        } else {
          cen = 0.f;
        }
      }
      double tile = 0.0;
      for (int64_t i = ri0; i < ri0 + T && i < n; ++i) {
        if (stride > 1 && ((i >> 1) % (stride >> 1)) != 0) continue;  // keep antithetic row pairs whole
        double si;
        float sif = sf;
        if (flags & 1) {
          const float ulps = u2f((f2u(sf) & 0x7f800000u) - (23u << 23));
          sif = g_anti ? fmaf((float)anti_offset(i), ulps, sf) : u2f(f2u(sf) + row_scale_offset(i));
        }
        si = (flags & (1 | 2)) ? (double)sif : 1.0 / g;
        const float p = row_phase(i);
        const float xi_c = x[i] - cen;  // fl(x_i - c)
        const float Xi = -(xi_c * sif);  // -fl(fl(x_i - c) s_i)
        double row = 0.0;
        float acc0 = 0.f, acc1 = 0.f;
        int64_t jend = rj0 + T < n ? rj0 + T : n;
        for (int64_t j = rj0; j < jend; ++j) {
          double u;
          float uf = 0.f, ulo = 0.f;
          if (flags & 4) {
            const float xj_c = x[j] - cen;
            uf = cmode == 3 ? (x[j] - x[i]) * sif : fmaf(xj_c, sif, Xi);
            u = uf;
            if (variant == 1) {
              // exact residual of the fma relative to the exact (x_j - x_i) s_i (for analysis)
              double ue = ((double)x[j] - (double)x[i]) * si;
              ulo = f32(ue - (double)uf);
            }
          } else if (flags & 512) {
            const float xj_c = x[j] - cen;
            u = cmode == 3 ? (double)(x[j] - x[i]) * si : (double)xj_c * si + (double)Xi;
          } else {
            u = ((double)x[j] - (double)x[i]) * si;
          }
          double t;
          float tf = 0.f;
          if (flags & 8) {
            tf = f32(u * u);
            if (variant == 1) tf = fmaf(2.f * uf, ulo, tf);
            t = tf;
          } else {
            t = u * u;
          }
          double a;
          if (flags & 16) a = fmaf(f32(t), c2f, p);
          else a = t * c2 + (double)p;
          double e = exp2(a) * exp2(-(double)p);
          if (flags & 32) e = (double)f32(exp2(a)) * exp2(-(double)p);
          double P = (flags & 64) ? (double)polyf(r, f32(t)) : poly(r, t);
          if (flags & 128) {
            float pe = f32(P) * f32(exp2(a));  // fp32 fma accumulate emulated below
            float* ac = ((j - rj0) & 1) == 0 ? &acc0 : &acc1;
            *ac = fmaf(f32(P), f32(exp2(a)), *ac);
            (void)pe;
            if (((j - rj0) & 63) == 63 || j == jend - 1) {
              row += (double)(acc0 + acc1) * exp2(-(double)p);
              acc0 = acc1 = 0.f;
            }
          } else {
            row += P * e;
          }
        }
        tile += row;
      }
      tot_b += w * tile;
    }
    total += tot_b;
  }
  (void)comp;
  printf("%.17g\n", total);
  return 0;
}
