/*
 * mpfem_oracle.c -- CPU restatement of the reference's hot-path algorithm.
 *
 * TEST INFRASTRUCTURE ONLY: this is the parity checker. The product never links it.
 * See mpfem_oracle.h for the contract. Reference citations are file:line into
 * /root/reference/proj. The restatement is pinned bit-for-bit against the compiled
 * reference (oracle/_ref) through the fixtures in tests/golden/.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (oracle/Makefile). FMA
 * contraction must stay off: the reference rounds every product and sum separately.
 */
#define _GNU_SOURCE
#include "mpfem_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define F_OVF 1u
#define F_UNF 2u
#define F_INV 4u
#define F_DZ 8u

static __thread char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ softfloat */
/* Format table: softfloat.hpp:50-56 */
typedef struct { int t; double min_normal, min_sub, max_finite, u; } fmtinfo;
static const fmtinfo FMT[4] = {
    {8, 0x1.0p-126, 0x1.0p-133, 0x1.fep127, 0x1.0p-8},
    {11, 0x1.0p-14, 0x1.0p-24, 65504.0, 0x1.0p-11},
    {24, 0x1.0p-126, 0x1.0p-149, 0x1.fffffep127, 0x1.0p-24},
    {53, 0x1.0p-1022, 0x1.0p-1074, 0x1.fffffffffffffp1023, 0x1.0p-53},
};

static double canonical_nan(void) {
  uint64_t b = 0x7ff8000000000000ull;
  double d;
  memcpy(&d, &b, 8);
  return d;
}
static uint64_t dbits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static double bitsd(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }

/* round_narrow: softfloat.hpp:72-112 */
static double round_narrow(double x, const fmtinfo* fi, uint32_t* fl, int ftz) {
  uint64_t bits = dbits(x);
  uint64_t mag = bits & 0x7fffffffffffffffull;
  if (mag >= 0x7ff0000000000000ull) {
    if (mag > 0x7ff0000000000000ull) { *fl |= F_INV; return canonical_nan(); }
    return x;
  }
  if (mag == 0) return x;
  double ax = bitsd(mag);
  if (ax < fi->min_normal) {
    if (ftz) { *fl |= F_UNF; return copysign(0.0, x); }
    double q = nearbyint(ax / fi->min_sub) * fi->min_sub;
    double r = copysign(q, x);
    if (r != x) *fl |= F_UNF;
    return r;
  }
  int drop = 53 - fi->t;
  uint64_t mask = (1ull << drop) - 1;
  uint64_t rem = bits & mask;
  uint64_t half = 1ull << (drop - 1);
  bits &= ~mask;
  if (rem > half || (rem == half && (bits & (1ull << drop)))) bits += 1ull << drop;
  double r = bitsd(bits);
  if (fabs(r) > fi->max_finite) { *fl |= F_OVF; return copysign(INFINITY, x); }
  return r;
}

/* round_fp32_native: softfloat.hpp:114-132 */
static double round_fp32(double x, uint32_t* fl, int ftz) {
  float g = (float)x;
  if (isnan(g)) { *fl |= F_INV; return canonical_nan(); }
  if (isinf(g)) { if (!isinf(x)) *fl |= F_OVF; return (double)g; }
  if (x != 0.0 && fabs(x) < 0x1.0p-126) {
    if (ftz) { *fl |= F_UNF; return copysign(0.0, x); }
    if ((double)g != x) *fl |= F_UNF;
  }
  return (double)g;
}

/* round_to: softfloat.hpp:147-157 */
double orc_round(double x, int fmt, int ftz, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  if (fmt == ORC_FP64) {
    if (isnan(x)) { *fl |= F_INV; return canonical_nan(); }
    return x;
  }
  if (fmt == ORC_FP32) return round_fp32(x, fl, ftz);
  return round_narrow(x, &FMT[fmt], fl, ftz);
}

/* fp_op: softfloat.hpp:170-186 (no fused multiply-add anywhere) */
double orc_op(double a, double b, int op, int fmt, int ftz, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  double r = 0.0;
  switch (op) {
    case 0: r = a + b; break;
    case 1: r = a - b; break;
    case 2: r = a * b; break;
    default:
      if (b == 0.0 && a != 0.0 && !isnan(a) && !isinf(a)) *fl |= F_DZ;
      r = a / b;
      break;
  }
  if (fmt == ORC_FP64 && isinf(r) && !isinf(a) && !isinf(b)) *fl |= F_OVF;
  return orc_round(r, fmt, ftz, fl);
}

#define RND(x, f) orc_round((x), (f), 0, fl)
#define ADD(a, b, f) orc_op((a), (b), 0, (f), 0, fl)
#define SUB(a, b, f) orc_op((a), (b), 1, (f), 0, fl)
#define MUL(a, b, f) orc_op((a), (b), 2, (f), 0, fl)
#define DIV(a, b, f) orc_op((a), (b), 3, (f), 0, fl)

/* ------------------------------------------------------------------ Rng */
/* common.hpp:21-35: std::mt19937_64 with uniform(a,b) = a + (b-a)*(next()>>11)*2^-53.
 * MT19937-64 as published by Matsumoto & Nishimura (the algorithm std::mt19937_64 names). */
#define MT_NN 312
#define MT_MM 156
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_NN;
}
uint64_t orc_rng_next(orc_rng* r) {
  static const uint64_t mag01[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (r->mti >= MT_NN) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ mag01[x & 1ull];
    }
    for (; i < MT_NN - 1; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[x & 1ull];
    }
    x = (r->mt[MT_NN - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[x & 1ull];
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}
double orc_rng_uniform(orc_rng* r, double a, double b) {
  double u01 = (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
  return a + (b - a) * u01;
}
void orc_rng_draws(uint64_t seed, int n, uint64_t* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = orc_rng_next(&r);
}

/* ------------------------------------------------------------------ quadrature */
static const double PI_D = 3.14159265358979323846;

/* legendre: quadrature.cpp:17-27 */
static void legendre(int n, double x, double* p, double* dp) {
  double p0 = 1.0, p1 = x;
  for (int j = 2; j <= n; ++j) {
    double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / (double)j;
    p0 = p1;
    p1 = p2;
  }
  *p = (n == 0) ? p0 : p1;
  *dp = (n == 0) ? 0.0 : (double)n * (x * p1 - p0) / (x * x - 1.0);
}

/* tridiag_ql: quadrature.cpp:31-81 (implicit-shift QL, z is n x n row-major) */
static int tridiag_ql(int n, double* d, double* e, double* z) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m = l;
    do {
      for (m = l; m < n - 1; ++m) {
        double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= 1e-300 + 2.3e-16 * dd) break;
      }
      if (m != l) {
        if (iter++ == 60) return fail(3, "internal error: tridiagonal QL stalled");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int deflated = 0;
        for (int i = m - 1; i >= l; --i) {
          double f = s * e[i];
          double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            deflated = 1;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int k = 0; k < n; ++k) {
            f = z[k * n + i + 1];
            z[k * n + i + 1] = s * z[k * n + i] + c * f;
            z[k * n + i] = c * z[k * n + i] - s * f;
          }
        }
        if (deflated) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return 0;
}

/* gauss_legendre_1d: quadrature.cpp:91-124 */
int orc_gauss_legendre_1d(int n, double* xs, double* ws) {
  if (n < 1 || n > 64) return fail(2, "quadrature point count must be in [1, 64]");
  if (n == 1) { xs[0] = 0.5; ws[0] = 1.0; return 0; }
  for (int k = 0; k < n; ++k) {
    double x = cos(PI_D * (k + 0.75) / (n + 0.5));
    double p = 0.0, dp = 1.0;
    for (int iter = 0;; ++iter) {
      if (iter >= 100) return fail(3, "internal error: Legendre Newton iteration stalled");
      legendre(n, x, &p, &dp);
      double step = p / dp;
      x -= step;
      if (fabs(step) < 1e-15) break;
    }
    legendre(n, x, &p, &dp);
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    xs[n - 1 - k] = 0.5 * (x + 1.0);
    ws[n - 1 - k] = 0.5 * w;
  }
  return 0;
}

/* gauss_jacobi_1d: quadrature.cpp:126-169 (Golub-Welsch) */
int orc_gauss_jacobi_1d(int n, int alpha, double* xs, double* ws) {
  if (n < 1 || n > 64) return fail(2, "quadrature point count must be in [1, 64]");
  if (alpha < 0) return fail(2, "Jacobi weight exponent must be nonnegative");
  double diag[64], off[64], z[64 * 64];
  for (int k = 0; k < n; ++k) off[k] = 0.0;
  diag[0] = -(double)alpha / (double)(alpha + 2);
  for (int k = 1; k < n; ++k) {
    double den = 2.0 * k + alpha;
    diag[k] = -(double)alpha * (double)alpha / (den * (den + 2.0));
    double bk = 4.0 * k * k * (k + alpha) * (k + alpha) / (den * den * (den * den - 1.0));
    off[k] = sqrt(bk);
  }
  for (int i = 0; i < n * n; ++i) z[i] = 0.0;
  for (int i = 0; i < n; ++i) z[i * n + i] = 1.0;
  int st = tridiag_ql(n, diag, off, z);
  if (st) return st;
  double mu0 = pow(2.0, alpha + 1) / (double)(alpha + 1);
  int order[64];
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) {
    int key = order[i];
    int j = i - 1;
    while (j >= 0 && diag[order[j]] > diag[key]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = key;
  }
  for (int i = 0; i < n; ++i) {
    int k = order[i];
    xs[i] = 0.5 * (diag[k] + 1.0);
    ws[i] = mu0 * z[0 * n + k] * z[0 * n + k] * pow(0.5, alpha + 1);
  }
  return 0;
}

/* rule_for, simplex branch, dim 3: quadrature.cpp:171-224 */
int orc_rule_simplex3(int p, double* pts, double* wts) {
  if (p < 1) return fail(2, "element degree must be at least 1");
  int n = p + 1;
  if (n > 64) return fail(2, "quadrature point count must be in [1, 64]");
  double fx[3][64], fw[3][64];
  for (int a = 0; a < 3; ++a) {
    int alpha = 3 - 1 - a;
    int st = alpha == 0 ? orc_gauss_legendre_1d(n, fx[a], fw[a])
                        : orc_gauss_jacobi_1d(n, alpha, fx[a], fw[a]);
    if (st) return st;
  }
  int nq = n * n * n;
  for (int q = 0; q < nq; ++q) {
    int idx[3], rem = q;
    for (int a = 0; a < 3; ++a) { idx[a] = rem % n; rem /= n; }
    double w = 1.0, xi[3];
    for (int a = 0; a < 3; ++a) { xi[a] = fx[a][idx[a]]; w *= fw[a][idx[a]]; }
    double shrink = 1.0;
    for (int a = 0; a < 3; ++a) { pts[q * 3 + a] = xi[a] * shrink; shrink *= (1.0 - xi[a]); }
    wts[q] = w;
  }
  return 0;
}

/* rule_for(box, p): quadrature.cpp:171-224, Gauss-Legendre on every axis, axis 0 fastest. */
static int orc_rule_box3_(int p, double* pts, double* wts) {
  if (p < 1) return fail(2, "element degree must be at least 1");
  int n = p + 1;
  double fx[64], fw[64];
  int st = orc_gauss_legendre_1d(n, fx, fw);
  if (st) return st;
  for (int q = 0; q < n * n * n; ++q) {
    int idx[3], rem = q;
    for (int a = 0; a < 3; ++a) { idx[a] = rem % n; rem /= n; }
    double w = 1.0;
    for (int a = 0; a < 3; ++a) { pts[q * 3 + a] = fx[idx[a]]; w *= fw[idx[a]]; }
    wts[q] = w;
  }
  return 0;
}
int orc_rule_box3(int p, double* pts, double* wts) { return orc_rule_box3_(p, pts, wts); }

/* ------------------------------------------------------------------ elements */
/* Product-form Lagrange basis on the unit tet: elements.cpp:89-147. */
typedef struct {
  int p, n_phi, m, box;
  double nodes[165][3];
  double weight[165];
  double fa[165][12][3]; /* factor linear coefficients (m <= 12: tets p <= 8, boxes p <= 4) */
  double fb[165][12];    /* factor constants */
  int fs[165][12][3];    /* derivative signs */
} basis_t;

int orc_nphi(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }
int orc_nq(int p) { return (p + 1) * (p + 1) * (p + 1); }

static int build_basis(int p, basis_t* B) {
  if (p < 1) return fail(2, "element degree must be at least 1");
  if (p > 8) return fail(2, "oracle supports p <= 8");
  memset(B, 0, sizeof *B);
  B->p = p;
  B->m = p;
  int count[3] = {0, 0, 0};
  int nf = 0;
  for (;;) {
    int sum = count[0] + count[1] + count[2];
    if (sum <= p) {
      int al[4] = {p - sum, count[0], count[1], count[2]};
      for (int a = 0; a < 3; ++a) B->nodes[nf][a] = (double)al[a + 1] / (double)p;
      double w = 1.0;
      int j = 0;
      for (int i = 0; i <= 3; ++i) {
        for (int k = 0; k < al[i]; ++k) {
          if (i == 0) {
            for (int a = 0; a < 3; ++a) { B->fa[nf][j][a] = -1.0; B->fs[nf][j][a] = -1; }
            B->fb[nf][j] = 1.0 - (double)k / (double)p;
          } else {
            B->fa[nf][j][i - 1] = 1.0;
            B->fs[nf][j][i - 1] = 1;
            B->fb[nf][j] = -(double)k / (double)p;
          }
          ++j;
          w *= (double)p / (double)(al[i] - k);
        }
      }
      B->weight[nf] = w;
      ++nf;
    }
    int a = 0;
    for (; a < 3; ++a) {
      if (++count[a] <= p) break;
      count[a] = 0;
    }
    if (a == 3) break;
  }
  B->n_phi = nf;
  return 0;
}

/* Tensor-product Lagrange basis on the unit box, equispaced nodes: elements.cpp:26-31,50-87.
 * Axis 0 fastest; per axis the p factors (x_a - x_j), j != i_a, weight 1 / prod (x_i - x_j). */
static int build_box_basis(int p, basis_t* B) {
  if (p < 1) return fail(2, "element degree must be at least 1");
  if (p > 4) return fail(2, "oracle supports box cells with p <= 4");
  memset(B, 0, sizeof *B);
  B->p = p;
  B->m = 3 * p;
  B->box = 1;
  int n1 = p + 1;
  double xs[5];
  for (int j = 0; j <= p; ++j) xs[j] = (double)j / (double)p;
  B->n_phi = n1 * n1 * n1;
  for (int idx = 0; idx < B->n_phi; ++idx) {
    int iax[3], rem = idx;
    for (int a = 0; a < 3; ++a) { iax[a] = rem % n1; rem /= n1; }
    double w = 1.0;
    int f = 0;
    for (int a = 0; a < 3; ++a) {
      B->nodes[idx][a] = xs[iax[a]];
      for (int j = 0; j <= p; ++j) {
        if (j == iax[a]) continue;
        B->fa[idx][f][a] = 1.0;
        B->fb[idx][f] = -xs[j];
        B->fs[idx][f][a] = 1;
        ++f;
        w /= xs[iax[a]] - xs[j];
      }
    }
    B->weight[idx] = w;
  }
  return 0;
}

/* factor_value: elements.cpp:165-169 */
static double factor_value(const basis_t* B, int i, int j, const double* x) {
  double v = B->fb[i][j];
  for (int a = 0; a < 3; ++a) v += B->fa[i][j][a] * x[a];
  return v;
}

/* eval_basis: elements.cpp:171-181 */
static double eval_basis(const basis_t* B, int i, const double* x, int f, uint32_t* fl) {
  double acc = RND(factor_value(B, i, 0, x), f);
  for (int j = 1; j < B->m; ++j) acc = MUL(acc, RND(factor_value(B, i, j, x), f), f);
  return MUL(acc, RND(B->weight[i], f), f);
}

/* eval_basis_gradient: elements.cpp:183-211 */
static void eval_basis_gradient(const basis_t* B, int i, const double* x, int f, double* g,
                                uint32_t* fl) {
  int m = B->m;
  double lhat[32];
  for (int j = 0; j < m; ++j) lhat[j] = RND(factor_value(B, i, j, x), f);
  double what = RND(B->weight[i], f);
  for (int s = 0; s < 3; ++s) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) {
      int sign = B->fs[i][j][s];
      if (sign == 0) continue;
      double prod = 1.0;
      int first = 1;
      for (int k = 0; k < m; ++k) {
        if (k == j) continue;
        prod = first ? lhat[k] : MUL(prod, lhat[k], f);
        first = 0;
      }
      acc = sign > 0 ? ADD(acc, prod, f) : SUB(acc, prod, f);
    }
    g[s] = MUL(acc, what, f);
  }
}

int orc_basis_nodes(int p, double* nodes) {
  basis_t B;
  int st = build_basis(p, &B);
  if (st) return st;
  for (int k = 0; k < B.n_phi; ++k)
    for (int a = 0; a < 3; ++a) nodes[k * 3 + a] = B.nodes[k][a];
  return 0;
}

/* tabulate: elements.cpp:249-274; layout (s*n_phi + k)*n_q + q */
static void tabulate_b(const basis_t* B, const double* pts, int nq, int ef, int sf, int grads,
                       double* out, uint32_t* fl) {
  int nphi = B->n_phi;
  for (int k = 0; k < nphi; ++k) {
    for (int q = 0; q < nq; ++q) {
      const double* xq = pts + 3 * q;
      if (grads) {
        double g[3];
        eval_basis_gradient(B, k, xq, ef, g, fl);
        for (int s = 0; s < 3; ++s) out[((size_t)s * nphi + k) * nq + q] = RND(g[s], sf);
      } else {
        out[(size_t)k * nq + q] = RND(eval_basis(B, k, xq, ef, fl), sf);
      }
    }
  }
}

int orc_tabulate(int p, int ef, int sf, int grads, double* out, uint32_t* fl) {
  basis_t B;
  int st = build_basis(p, &B);
  if (st) return st;
  int nq = orc_nq(p);
  double* pts = malloc(sizeof(double) * 3 * nq);
  double* w = malloc(sizeof(double) * nq);
  st = orc_rule_simplex3(p, pts, w);
  if (!st) tabulate_b(&B, pts, nq, ef, sf, grads, out, fl);
  free(pts);
  free(w);
  return st;
}

/* basis_condition_numbers: elements.cpp:278-359 (lebesgue, gradient parts) */
typedef struct {
  double lebesgue;
  double grad_lebesgue[3];
  double grad_kappa[165][3];
  double grad_kappa_max[3];
} cond_t;

static void basis_conditioning(const basis_t* B, const double* pts, int nq, cond_t* bc) {
  int m = B->m, nphi = B->n_phi;
  int n_random = 2000;
  int ns = nq + nphi + n_random;
  double* S = malloc(sizeof(double) * 3 * ns);
  int ip = 0;
  for (int q = 0; q < nq; ++q, ++ip)
    for (int a = 0; a < 3; ++a) S[ip * 3 + a] = pts[q * 3 + a];
  for (int k = 0; k < nphi; ++k, ++ip)
    for (int a = 0; a < 3; ++a) S[ip * 3 + a] = B->nodes[k][a];
  orc_rng rng;
  orc_rng_seed(&rng, 9001);
  for (int i = 0; i < n_random; ++i, ++ip) {
    double x[3];
    for (;;) {  /* sample_point: elements.cpp:279-289 */
      double sum = 0.0;
      for (int a = 0; a < 3; ++a) { x[a] = orc_rng_uniform(&rng, 0.0, 1.0); sum += x[a]; }
      if (B->box || sum <= 1.0) break;  /* sample_point: rejection for simplices only */
    }
    for (int a = 0; a < 3; ++a) S[ip * 3 + a] = x[a];
  }
  static double num_max[165][3], abs_max[165][3];
  memset(num_max, 0, sizeof num_max);
  memset(abs_max, 0, sizeof abs_max);
  bc->lebesgue = 1.0;
  for (int s = 0; s < 3; ++s) { bc->grad_lebesgue[s] = 0.0; bc->grad_kappa_max[s] = 0.0; }
  double lv[32], prefix[33], suffix[33];
  for (int si = 0; si < ns; ++si) {
    const double* x = S + 3 * si;
    double sum_abs_phi = 0.0, sum_abs_grad[3] = {0, 0, 0};
    for (int i = 0; i < nphi; ++i) {
      for (int j = 0; j < m; ++j) lv[j] = factor_value(B, i, j, x);
      prefix[0] = 1.0;
      for (int j = 0; j < m; ++j) prefix[j + 1] = prefix[j] * lv[j];
      suffix[m] = 1.0;
      for (int j = m - 1; j >= 0; --j) suffix[j] = suffix[j + 1] * lv[j];
      sum_abs_phi += fabs(B->weight[i] * prefix[m]);
      for (int s = 0; s < 3; ++s) {
        double grad = 0.0, numer = 0.0;
        for (int j = 0; j < m; ++j) {
          int sign = B->fs[i][j][s];
          if (sign == 0) continue;
          double complement = B->weight[i] * prefix[j] * suffix[j + 1];
          grad += sign * complement;
          numer += fabs(complement);
        }
        sum_abs_grad[s] += fabs(grad);
        if (fabs(grad) > abs_max[i][s]) abs_max[i][s] = fabs(grad);
        if (numer > num_max[i][s]) num_max[i][s] = numer;
      }
    }
    if (sum_abs_phi > bc->lebesgue) bc->lebesgue = sum_abs_phi;
    for (int s = 0; s < 3; ++s)
      if (sum_abs_grad[s] > bc->grad_lebesgue[s]) bc->grad_lebesgue[s] = sum_abs_grad[s];
  }
  for (int i = 0; i < nphi; ++i) {
    for (int s = 0; s < 3; ++s) {
      double numer = num_max[i][s], denom = abs_max[i][s];
      double kappa = 1.0;
      if (numer > 0.0) kappa = denom > 0.0 ? numer / denom : INFINITY;
      bc->grad_kappa[i][s] = kappa;
      if (kappa > bc->grad_kappa_max[s]) bc->grad_kappa_max[s] = kappa;
    }
  }
  free(S);
}

int orc_basis_conditioning(int p, double* leb, double* gleb, double* gk, double* gkmax) {
  basis_t B;
  int st = build_basis(p, &B);
  if (st) return st;
  int nq = orc_nq(p);
  double* pts = malloc(sizeof(double) * 3 * nq);
  double* w = malloc(sizeof(double) * nq);
  st = orc_rule_simplex3(p, pts, w);
  if (!st) {
    cond_t* bc = malloc(sizeof *bc);
    basis_conditioning(&B, pts, nq, bc);
    *leb = bc->lebesgue;
    for (int s = 0; s < 3; ++s) { gleb[s] = bc->grad_lebesgue[s]; gkmax[s] = bc->grad_kappa_max[s]; }
    for (int i = 0; i < B.n_phi; ++i)
      for (int s = 0; s < 3; ++s) gk[i * 3 + s] = bc->grad_kappa[i][s];
    free(bc);
  }
  free(pts);
  free(w);
  return st;
}

/* ------------------------------------------------------------------ geometry */
/* jacobian through the P1 geometry basis at the centroid: geometry.cpp:12-27 */
static void jacobian_at(const basis_t* G1, const double* verts, const double* xref, int f, double* jac,
                        uint32_t* fl) {
  for (int i = 0; i < 9; ++i) jac[i] = 0.0;
  for (int k = 0; k < G1->n_phi; ++k) {
    double g[3];
    eval_basis_gradient(G1, k, xref, f, g, fl);
    for (int i = 0; i < 3; ++i) {
      double x = RND(verts[k * 3 + i], f);
      for (int s = 0; s < 3; ++s) jac[i * 3 + s] = ADD(jac[i * 3 + s], MUL(x, g[s], f), f);
    }
  }
}
static void jacobian(const basis_t* G1, const double* verts, int f, double* jac, uint32_t* fl) {
  double centroid[3] = {0.25, 0.25, 0.25};
  jacobian_at(G1, verts, centroid, f, jac, fl);
}

/* lu_decompose: geometry.cpp:33-57 */
static int lu_decompose(double* lu, int* perm, int f, int* sign_out, uint32_t* fl) {
  int n = 3, sign = 1;
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    for (int r = col + 1; r < n; ++r)
      if (fabs(lu[r * 3 + col]) > fabs(lu[pivot * 3 + col])) pivot = r;
    if (lu[pivot * 3 + col] == 0.0) return fail(3, "singular cell geometry");
    if (pivot != col) {
      for (int c = 0; c < n; ++c) {
        double t = lu[pivot * 3 + c];
        lu[pivot * 3 + c] = lu[col * 3 + c];
        lu[col * 3 + c] = t;
      }
      int t = perm[pivot];
      perm[pivot] = perm[col];
      perm[col] = t;
      sign = -sign;
    }
    for (int r = col + 1; r < n; ++r) {
      double m = DIV(lu[r * 3 + col], lu[col * 3 + col], f);
      lu[r * 3 + col] = m;
      for (int c = col + 1; c < n; ++c)
        lu[r * 3 + c] = SUB(lu[r * 3 + c], MUL(m, lu[col * 3 + c], f), f);
    }
  }
  *sign_out = sign;
  return 0;
}

/* det_lu: geometry.cpp:61-68 */
static int det_lu(const double* jac, int f, double* det, uint32_t* fl) {
  double lu[9];
  int perm[3], sign;
  memcpy(lu, jac, sizeof lu);
  int st = lu_decompose(lu, perm, f, &sign, fl);
  if (st) return st;
  double d = (double)sign;
  for (int i = 0; i < 3; ++i) d = MUL(d, lu[i * 3 + i], f);
  *det = d;
  return 0;
}

/* inverse_lu: geometry.cpp:70-95 */
static int inverse_lu(const double* jac, int f, double* inv, uint32_t* fl) {
  double lu[9];
  int perm[3], sign;
  memcpy(lu, jac, sizeof lu);
  int st = lu_decompose(lu, perm, f, &sign, fl);
  if (st) return st;
  for (int i = 0; i < 9; ++i) inv[i] = 0.0;
  for (int k = 0; k < 3; ++k) {
    double y[3] = {0, 0, 0};
    for (int r = 0; r < 3; ++r) {
      double s = perm[r] == k ? 1.0 : 0.0;
      for (int c = 0; c < r; ++c) s = SUB(s, MUL(lu[r * 3 + c], y[c], f), f);
      y[r] = s;
    }
    for (int r = 2; r >= 0; --r) {
      double s = y[r];
      for (int c = r + 1; c < 3; ++c) s = SUB(s, MUL(lu[r * 3 + c], inv[c * 3 + k], f), f);
      inv[r * 3 + k] = DIV(s, lu[r * 3 + r], f);
    }
  }
  return 0;
}

/* sym_eigenvalues (cyclic Jacobi): geometry.cpp:120-154 */
static void sym_eigenvalues3(const double* sym, double* eig) {
  double a[9];
  memcpy(a, sym, sizeof a);
  int n = 3;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += a[p * 3 + q] * a[p * 3 + q];
    if (off <= 1e-300) break;
    for (int p = 0; p < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        if (a[p * 3 + q] == 0.0) continue;
        double theta = (a[q * 3 + q] - a[p * 3 + p]) / (2.0 * a[p * 3 + q]);
        double t = copysign(1.0, theta) / (fabs(theta) + sqrt(1.0 + theta * theta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = t * c;
        for (int k = 0; k < n; ++k) {
          double akp = a[k * 3 + p], akq = a[k * 3 + q];
          a[k * 3 + p] = c * akp - s * akq;
          a[k * 3 + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = a[p * 3 + k], aqk = a[q * 3 + k];
          a[p * 3 + k] = c * apk - s * aqk;
          a[q * 3 + k] = s * apk + c * aqk;
        }
      }
    }
  }
  for (int i = 0; i < 3; ++i) eig[i] = a[i * 3 + i];
  /* ascending sort */
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && eig[j - 1] > eig[j]; --j) {
      double t = eig[j]; eig[j] = eig[j - 1]; eig[j - 1] = t;
    }
}

/* kappa2_of: geometry.cpp:156-169 */
static double kappa2_of(const double* jac) {
  double jtj[9];
  for (int s = 0; s < 3; ++s)
    for (int t = 0; t < 3; ++t) {
      double dot = 0.0;
      for (int k = 0; k < 3; ++k) dot += jac[k * 3 + s] * jac[k * 3 + t];
      jtj[s * 3 + t] = dot;
    }
  double eig[3];
  sym_eigenvalues3(jtj, eig);
  if (eig[0] <= 0.0) return INFINITY;
  return sqrt(eig[2] / eig[0]);
}

/* kappa_cell_of: geometry.cpp:171-186 */
static double kappa_cell_nv(const double* verts, int nv, const double* jac) {
  double xnorm = 0.0;
  for (int i = 0; i < 3; ++i) {
    double row = 0.0;
    for (int v = 0; v < nv; ++v) row += fabs(verts[v * 3 + i]);
    if (row > xnorm) xnorm = row;
  }
  double jnorm = 0.0;
  for (int i = 0; i < 3; ++i) {
    double row = 0.0;
    for (int s = 0; s < 3; ++s) row += fabs(jac[i * 3 + s]);
    if (row > jnorm) jnorm = row;
  }
  return (double)nv * xnorm / jnorm;
}
static double kappa_cell_of(const double* verts, const double* jac) {
  return kappa_cell_nv(verts, 4, jac);
}

static basis_t g_geom1;
static int g_geom1_ready = 0;
static const basis_t* geom_basis(void) {
  if (!g_geom1_ready) { build_basis(1, &g_geom1); g_geom1_ready = 1; }
  return &g_geom1;
}

static basis_t g_geom1_box;
static int g_geom1_box_ready = 0;
static const basis_t* geom_basis_box(void) {
  if (!g_geom1_box_ready) { build_box_basis(1, &g_geom1_box); g_geom1_box_ready = 1; }
  return &g_geom1_box;
}

/* point_geometry: geometry.cpp:190-221 (J through the degree-1 geometry basis at xref). */
static int point_geometry(const basis_t* G1, const double* verts, const double* xref, int form,
                          int f, double* out, uint32_t* fl) {
  memset(out, 0, sizeof(double) * ORC_GEOM_SIZE);
  double* jac = out + 2;
  double* inv = out + 11;
  double* ten = out + 20;
  jacobian_at(G1, verts, xref, f, jac, fl);
  double det;
  int st = det_lu(jac, f, &det, fl);
  if (st) return st;
  out[0] = det;
  out[1] = fabs(det);
  st = inverse_lu(jac, f, inv, fl);
  if (st) return st;
  /* geometry_tensor: geometry.cpp:97-118 */
  if (form == ORC_MASS) {
    ten[0] = out[1];
  } else {
    for (int s = 0; s < 3; ++s)
      for (int t = s; t < 3; ++t) {
        double dot = 0.0;
        for (int k = 0; k < 3; ++k) dot = ADD(dot, MUL(inv[s * 3 + k], inv[t * 3 + k], f), f);
        double v = MUL(out[1], dot, f);
        ten[s * 3 + t] = v;
        ten[t * 3 + s] = v;
      }
  }
  /* binary64 diagnostics */
  uint32_t wide = 0;
  double jac64[9], inv64[9], det64;
  jacobian_at(G1, verts, xref, ORC_FP64, jac64, &wide);
  out[29] = kappa2_of(jac64);
  out[30] = kappa_cell_nv(verts, G1->n_phi, jac64);
  st = det_lu(jac64, ORC_FP64, &det64, &wide);
  if (st) return st;
  det64 = fabs(det64);
  double* tt = out + 31;
  if (form == ORC_MASS) {
    tt[0] = det64;
  } else {
    st = inverse_lu(jac64, ORC_FP64, inv64, &wide);
    if (st) return st;
    for (int s = 0; s < 3; ++s)
      for (int t = 0; t < 3; ++t) {
        double dot = 0.0;
        for (int k = 0; k < 3; ++k) dot += fabs(inv64[s * 3 + k]) * fabs(inv64[t * 3 + k]);
        tt[s * 3 + t] = det64 * dot;
      }
  }
  return 0;
}

/* cell_geometry, affine tets: geometry.cpp:226-245 (one point at the centroid). */
int orc_cell_geometry(const double* verts, int form, int f, double* out, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  double centroid[3] = {0.25, 0.25, 0.25};
  return point_geometry(geom_basis(), verts, centroid, form, f, out, fl);
}

/* ------------------------------------------------------------------ coefficients */
/* Quadrature-point coefficient path (SURVEY 8.0 "Q"): x_q = v0 + J xi_q in binary64 with
 * J[:, s] = v_{s+1} - v0, evaluated left to right. */
static void phys_point(const double* v, const double* xi, double* x) {
  for (int i = 0; i < 3; ++i) {
    double acc = v[i];
    for (int s = 0; s < 3; ++s) acc = acc + (v[(s + 1) * 3 + i] - v[i]) * xi[s];
    x[i] = acc;
  }
}
static double coef_sincosexp(const double* x) {
  const double two_pi = 6.283185307179586476925286766559;
  double s = sin(two_pi * x[0]);
  double c = cos(two_pi * x[1]);
  double e = exp(x[2]);
  return 1.0 + 0.5 * s * c * e;
}
static double coef_exp10_affine(const double* u4, const double* xi) {
  double l0 = ((1.0 - xi[0]) - xi[1]) - xi[2];
  double u = u4[0] * l0 + u4[1] * xi[0] + u4[2] * xi[1] + u4[3] * xi[2];
  return pow(10.0, 6.0 * u);
}

/* ------------------------------------------------------------------ kernels */
typedef struct {
  int p, form, up, ug, uq, us, engine;
  int nphi, nq, nd;
  basis_t B;
  double *pts, *wts;
  double* tab_store;  /* n_d x n_phi x n_q at (u_p -> u_s) */
  double* tab_values; /* n_phi x n_q at (u_p -> u_p) */
} setup_t;

static int orc_rule_box3_(int p, double* pts, double* wts);

/* make_setup: kernels.cpp:78-108 (box: tensor basis and Gauss-Legendre rule) */
static int make_setup_kind(int p, int form, const int* cfg, setup_t* S, int box);
static int make_setup(int p, int form, const int* cfg, setup_t* S) {
  return make_setup_kind(p, form, cfg, S, 0);
}
static int make_setup_kind(int p, int form, const int* cfg, setup_t* S, int box) {
  memset(S, 0, sizeof *S);
  S->p = p; S->form = form;
  S->up = cfg[0]; S->ug = cfg[1]; S->uq = cfg[2]; S->us = cfg[3]; S->engine = cfg[4];
  for (int i = 0; i < 4; ++i)
    if (cfg[i] < 0 || cfg[i] > 3) return fail(2, "unknown float format");
  /* validate_config: kernels.cpp:29-40 (matrix engine => u_s bf16, u_q fp32) */
  if (S->engine == 2 && (S->us != ORC_BF16 || S->uq != ORC_FP32))
    return fail(2, "matrix engine requires the unit's native formats: u_s = bf16, u_q = fp32");
  int st = box ? build_box_basis(p, &S->B) : build_basis(p, &S->B);
  if (st) return st;
  S->nphi = S->B.n_phi;
  S->nq = orc_nq(p);
  S->nd = form == ORC_POISSON ? 3 : 1;
  S->pts = malloc(sizeof(double) * 3 * S->nq);
  S->wts = malloc(sizeof(double) * S->nq);
  st = box ? orc_rule_box3_(p, S->pts, S->wts) : orc_rule_simplex3(p, S->pts, S->wts);
  if (st) return st;
  S->tab_store = malloc(sizeof(double) * S->nd * S->nphi * S->nq);
  S->tab_values = malloc(sizeof(double) * S->nphi * S->nq);
  uint32_t sf = 0;
  tabulate_b(&S->B, S->pts, S->nq, S->up, S->us, form == ORC_POISSON, S->tab_store, &sf);
  tabulate_b(&S->B, S->pts, S->nq, S->up, S->up, 0, S->tab_values, &sf);
  return 0;
}
static void free_setup(setup_t* S) {
  free(S->pts); free(S->wts); free(S->tab_store); free(S->tab_values);
}

/* zhat at u_g per quadrature point. Nodal path = eval_z_at_ug (kernels.cpp:114-136);
 * analytic path = c(x_q) in binary64 rounded once to u_g. Returns 0 if coefficient is one. */
static int coef_zhat(const setup_t* S, const double* verts, int kind, const double* coef,
                     double* zhat, uint32_t* fl) {
  int nq = S->nq, nphi = S->nphi;
  if (kind == ORC_COEF_ONE) return 0;
  if (kind == ORC_COEF_NODAL) {
    double zp[165];
    for (int i = 0; i < nphi; ++i) zp[i] = RND(coef[i], S->up);
    for (int q = 0; q < nq; ++q) {
      double acc = 0.0;
      for (int k = 0; k < nphi; ++k)
        acc = ADD(acc, MUL(zp[k], S->tab_values[(size_t)k * nq + q], S->up), S->up);
      zhat[q] = RND(acc, S->ug);
    }
    return 1;
  }
  for (int q = 0; q < nq; ++q) {
    double c;
    if (kind == ORC_COEF_SINCOSEXP) {
      double x[3];
      phys_point(verts, S->pts + 3 * q, x);
      c = coef_sincosexp(x);
    } else {
      c = coef_exp10_affine(coef, S->pts + 3 * q);
    }
    zhat[q] = RND(c, S->ug);
  }
  return 1;
}

int orc_coef_at_q(int p, const double* verts, int kind, const double* coef, double* cq) {
  int cfg[5] = {3, 3, 3, 3, 0};
  setup_t S;
  int st = make_setup(p, ORC_MASS, cfg, &S);
  if (!st) {
    uint32_t fl = 0;
    if (!coef_zhat(&S, verts, kind, coef, cq, &fl))
      for (int q = 0; q < S.nq; ++q) cq[q] = 1.0;
  }
  free_setup(&S);
  return st;
}

/* build_C: kernels.cpp:177-197 */
static int build_C_g(const setup_t* S, const double* geom, int gstride, const double* verts,
                     int kind, const double* coef, double* c, uint32_t* fl) {
  int nq = S->nq, nd = S->nd;
  double* zhat = malloc(sizeof(double) * nq);
  int have_z = coef_zhat(S, verts, kind, coef, zhat, fl);
  for (int q = 0; q < nq; ++q) {
    const double* ten = geom + (size_t)q * gstride + 20;
    double omega = RND(S->wts[q], S->ug);
    for (int s = 0; s < nd; ++s)
      for (int t = 0; t < nd; ++t) {
        double value = MUL(omega, ten[s * 3 + t], S->ug);
        if (have_z) value = MUL(value, zhat[q], S->ug);
        c[((size_t)s * nd + t) * nq + q] = RND(value, S->us);
      }
  }
  free(zhat);
  return 0;
}
static int build_C_s(const setup_t* S, const double* geom, const double* verts, int kind,
                     const double* coef, double* c, uint32_t* fl) {
  return build_C_g(S, geom, 0, verts, kind, coef, c, fl);
}

/* Geometry of one cell at every rule point: affine tets one point (stride 0), boxes one
 * point per rule point (cell_geometry, geometry.cpp:226-245). Caller frees *geo. */
static int cell_geometry_all(const setup_t* S, const double* verts, int f, double** geo,
                             int* stride, uint32_t* fl) {
  if (!S->B.box) {
    *geo = malloc(sizeof(double) * ORC_GEOM_SIZE);
    *stride = 0;
    return orc_cell_geometry(verts, S->form, f, *geo, fl);
  }
  *geo = malloc(sizeof(double) * ORC_GEOM_SIZE * S->nq);
  *stride = ORC_GEOM_SIZE;
  for (int q = 0; q < S->nq; ++q) {
    int st = point_geometry(geom_basis_box(), verts, S->pts + 3 * q, S->form, f,
                            *geo + (size_t)q * ORC_GEOM_SIZE, fl);
    if (st) return st;
  }
  return 0;
}

int orc_build_C(int p, int form, const int* cfg, const double* verts, int kind,
                const double* coef, double* c_out, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  setup_t S;
  int st = make_setup(p, form, cfg, &S);
  if (!st) {
    double geom[ORC_GEOM_SIZE];
    st = orc_cell_geometry(verts, form, S.ug, geom, fl);
    if (!st) st = build_C_s(&S, geom, verts, kind, coef, c_out, fl);
  }
  free_setup(&S);
  return st;
}

/* bilinear_kernel: kernels.cpp:242-267. H_cat fill at u_s (kernels.cpp:253-265) and the
 * depth-chained matmul at u_q (mm_units.cpp:76-88 scalar; the matrix engine of
 * mm_units.cpp:43-62,102-143 differs only by flushing subnormal accumulates). */
static int bilinear_one(const setup_t* S, const double* verts, int kind, const double* coef,
                        double* a, uint32_t* fl) {
  int nq = S->nq, nd = S->nd, nphi = S->nphi;
  int K = nd * nd * nq;
  double* geom = NULL;
  int gstride = 0;
  int st = cell_geometry_all(S, verts, S->ug, &geom, &gstride, fl);
  if (st) { free(geom); return st; }
  double* c = malloc(sizeof(double) * K);
  build_C_g(S, geom, gstride, verts, kind, coef, c, fl);
  free(geom);
  double* h = malloc(sizeof(double) * (size_t)K * nphi);
  for (int s = 0; s < nd; ++s)
    for (int t = 0; t < nd; ++t) {
      const double* cst = c + ((size_t)s * nd + t) * nq;
      int row0 = (s * nd + t) * nq;
      for (int q = 0; q < nq; ++q)
        for (int k = 0; k < nphi; ++k)
          h[(size_t)(row0 + q) * nphi + k] =
              MUL(cst[q], S->tab_store[((size_t)t * nphi + k) * nq + q], S->us);
    }
  int ftz = S->engine == 2;
  int uq = S->uq;
  for (int i = 0; i < nphi; ++i)
    for (int k = 0; k < nphi; ++k) {
      double acc = 0.0;
      for (int s = 0; s < nd; ++s)
        for (int t = 0; t < nd; ++t) {
          const double* bs = S->tab_store + ((size_t)s * nphi + i) * nq;
          int row0 = (s * nd + t) * nq;
          for (int q = 0; q < nq; ++q) {
            double prod = orc_op(bs[q], h[(size_t)(row0 + q) * nphi + k], 2, uq, 0, fl);
            acc = orc_op(acc, prod, 0, uq, ftz, fl);
          }
        }
      a[(size_t)i * nphi + k] = acc;
    }
  free(c);
  free(h);
  return 0;
}

int orc_bilinear(int p, int form, const int* cfg, int64_t m, const double* verts,
                 int kind, const double* coef, int coef_stride, double* a_out,
                 uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  setup_t S;
  int st = make_setup(p, form, cfg, &S);
  if (!st) {
    size_t n2 = (size_t)S.nphi * S.nphi;
    for (int64_t c = 0; c < m && !st; ++c)
      st = bilinear_one(&S, verts + 12 * c, kind, coef ? coef + coef_stride * c : NULL,
                        a_out + n2 * c, fl);
  }
  free_setup(&S);
  return st;
}

/* ------------------------------------------------------------------ bounds */
/* kernel_bounds, bilinear part: bounds.cpp:29-281. For the analytic coefficient path the
 * coefficient enters at >= u_g, so z_at = c(x_q) and theta_c = 0 (SURVEY 8.0, Q path). */
static int bound_impl(int p, int form, const int* cfg, const double* verts, int kind,
                      const double* coef, double* out4, double* a64, int box) {
  setup_t S;
  int st = make_setup_kind(p, form, cfg, &S, box);
  if (st) { free_setup(&S); return st; }
  int nq = S.nq, nd = S.nd, nphi = S.nphi;
  int poisson = form == ORC_POISSON;
  uint32_t scratch = 0;
  uint32_t* fl = &scratch;
  double* geom = NULL;
  int gstride = 0;
  st = cell_geometry_all(&S, verts, ORC_FP64, &geom, &gstride, fl);
  if (st) { free(geom); free_setup(&S); return st; }

  size_t nb = (size_t)nd * nphi * nq;
  double* tab = malloc(sizeof(double) * nb);
  tabulate_b(&S.B, S.pts, nq, ORC_FP64, ORC_FP64, poisson, tab, fl);
  cond_t* bc = malloc(sizeof *bc);
  basis_conditioning(&S.B, S.pts, nq, bc);
  double dp = 3.0 * p;
  double pd = pow((double)p, 3);
  double kv = bc->lebesgue;
  int z_const = kind == ORC_COEF_ONE;
  double z_norm = 0.0;
  if (kind == ORC_COEF_NODAL)
    for (int i = 0; i < nphi; ++i) if (fabs(coef[i]) > z_norm) z_norm = fabs(coef[i]);

  double* theta_b = calloc(nb, sizeof(double));
  if (poisson) {
    for (int s = 0; s < nd; ++s)
      for (int k = 0; k < nphi; ++k) {
        double peak = 0.0;
        for (int q = 0; q < nq; ++q) {
          double v = fabs(tab[((size_t)s * nphi + k) * nq + q]);
          if (v > peak) peak = v;
        }
        double budget = dp * bc->grad_kappa[k][s] * peak;
        for (int q = 0; q < nq; ++q) theta_b[((size_t)s * nphi + k) * nq + q] = budget;
      }
  } else {
    for (size_t i = 0; i < nb; ++i) theta_b[i] = dp * fabs(tab[i]);
  }

  double* z_at = malloc(sizeof(double) * nq);
  for (int q = 0; q < nq; ++q) z_at[q] = 1.0;
  if (kind == ORC_COEF_NODAL) {
    for (int q = 0; q < nq; ++q) {  /* eval_fe_function at fp64: elements.cpp:213-222 */
      double acc = 0.0;
      for (int i = 0; i < nphi; ++i) acc += coef[i] * eval_basis(&S.B, i, S.pts + 3 * q, ORC_FP64, fl);
      z_at[q] = acc;
    }
  } else if (kind == ORC_COEF_SINCOSEXP) {
    for (int q = 0; q < nq; ++q) {
      double x[3];
      phys_point(verts, S.pts + 3 * q, x);
      z_at[q] = coef_sincosexp(x);
    }
  } else if (kind == ORC_COEF_EXP10_AFFINE) {
    for (int q = 0; q < nq; ++q) z_at[q] = coef_exp10_affine(coef, S.pts + 3 * q);
  }

  size_t nc = (size_t)nd * nd * nq;
  double* cc = malloc(sizeof(double) * nc);
  double* thc = malloc(sizeof(double) * nc);
  double* gc = malloc(sizeof(double) * nc);
  for (int s = 0; s < nd; ++s)
    for (int t = 0; t < nd; ++t)
      for (int q = 0; q < nq; ++q) {
        double omega = S.wts[q];
        const double* gq = geom + (size_t)q * gstride;
        const double* ten = gq + 20;
        const double* tt = gq + 31;
        double kappa2 = gq[29], kcell = gq[30];
        size_t idx = ((size_t)s * nd + t) * nq + q;
        cc[idx] = omega * ten[s * 3 + t] * z_at[q];
        thc[idx] = (kind == ORC_COEF_NODAL && !z_const)
                       ? pd * kv * z_norm * fabs(omega * ten[s * 3 + t]) : 0.0;
        gc[idx] = kcell * kappa2 * fabs(omega * tt[s * 3 + t] * z_at[q]);
      }

  double amax = 0, samax = 0, tamax = 0, gamax = 0;
  for (int i = 0; i < nphi; ++i)
    for (int k = 0; k < nphi; ++k) {
      double acc = 0.0, sa = 0.0, ta = 0.0, ga = 0.0;
      for (int s = 0; s < nd; ++s)
        for (int t = 0; t < nd; ++t)
          for (int q = 0; q < nq; ++q) {
            size_t cidx = ((size_t)s * nd + t) * nq + q;
            double bval = tab[((size_t)t * nphi + k) * nq + q];
            double tbk = theta_b[((size_t)t * nphi + k) * nq + q];
            double h = cc[cidx] * bval;
            double th = thc[cidx] * fabs(bval) + fabs(cc[cidx]) * tbk;
            double gh = gc[cidx] * fabs(bval);
            double b = tab[((size_t)s * nphi + i) * nq + q];
            double tb = theta_b[((size_t)s * nphi + i) * nq + q];
            acc += b * h;
            sa += fabs(b) * fabs(h);
            ta += fabs(b) * th + tb * fabs(h);
            ga += fabs(b) * gh;
          }
      if (a64) a64[(size_t)i * nphi + k] = acc;
      if (fabs(acc) > amax) amax = fabs(acc);
      if (fabs(sa) > samax) samax = fabs(sa);
      if (fabs(ta) > tamax) tamax = fabs(ta);
      if (fabs(ga) > gamax) gamax = fabs(ga);
    }
  double u_p = FMT[S.up].u, u_g = FMT[S.ug].u, u_q = FMT[S.uq].u, u_s = FMT[S.us].u;
  if (amax > 0.0) {
    out4[1] = samax / amax;
    out4[2] = tamax / amax;
    out4[3] = gamax / amax;
    out4[0] = (u_s + nq * u_q) * out4[1] + u_p * out4[2] + u_g * out4[3];
  } else {
    out4[0] = out4[1] = out4[2] = out4[3] = NAN;
  }
  free(tab); free(bc); free(theta_b); free(z_at); free(cc); free(thc); free(gc); free(geom);
  free_setup(&S);
  return 0;
}

int orc_bound(int p, int form, const int* cfg, const double* verts, int kind,
              const double* coef, double* out4, double* a64) {
  return bound_impl(p, form, cfg, verts, kind, coef, out4, a64, 0);
}

/* ------------------------------------------------------------------ box cells */
/* Hexahedra: per-point geometry through the trilinear map (geometry.cpp:12-27,190-245 with the
 * degree-1 box basis), tensor Lagrange basis and Gauss-Legendre rule. Constant and nodal
 * coefficients (the reference's own coefficient path). */
static int box_coef_ok(int kind) {
  return kind == ORC_COEF_ONE || kind == ORC_COEF_NODAL
             ? 0 : fail(2, "box cells take constant or nodal coefficients");
}

int orc_bilinear_box(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                     const double* coef, int coef_stride, double* a_out, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  int st = box_coef_ok(kind);
  if (st) return st;
  setup_t S;
  st = make_setup_kind(p, form, cfg, &S, 1);
  if (!st) {
    size_t n2 = (size_t)S.nphi * S.nphi;
    for (int64_t c = 0; c < m && !st; ++c)
      st = bilinear_one(&S, verts + 24 * c, kind, coef ? coef + coef_stride * c : NULL,
                        a_out + n2 * c, fl);
  }
  free_setup(&S);
  return st;
}

int orc_build_C_box(int p, int form, const int* cfg, const double* verts, int kind,
                    const double* coef, double* c_out, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  int st = box_coef_ok(kind);
  if (st) return st;
  setup_t S;
  st = make_setup_kind(p, form, cfg, &S, 1);
  if (!st) {
    double* geom = NULL;
    int gstride = 0;
    st = cell_geometry_all(&S, verts, S.ug, &geom, &gstride, fl);
    if (!st) st = build_C_g(&S, geom, gstride, verts, kind, coef, c_out, fl);
    free(geom);
  }
  free_setup(&S);
  return st;
}

int orc_bound_box(int p, int form, const int* cfg, const double* verts, int kind,
                  const double* coef, double* out4, double* a64) {
  int st = box_coef_ok(kind);
  if (st) return st;
  return bound_impl(p, form, cfg, verts, kind, coef, out4, a64, 1);
}

/* ------------------------------------------------------------------ action (Algorithm 2) */
/* action_kernel (kernels.cpp:269-304) for one cell: w-evaluation eval_w_at_ug
 * (kernels.cpp:145-173: round w to u_s, k-ascending matmul against the u_s store slabs at
 * u_p, cast to u_g), the integrand r (kernels.cpp:280-301 / build_r 214-240: (G w)_s with t
 * ascending at u_g, times omega, times zhat, rounded to u_s) and v = b_cat_action r at u_q
 * ((s, q) ascending, kernels.cpp:303). The matrix engine flushes subnormal accumulates
 * (mm_units.cpp:43-62). Coefficient kinds as orc_build_C (Q path: zhat = c(x_q) at u_g). */
static int action_one(const setup_t* S, const double* verts, int kind, const double* coef,
                      const double* w, double* v, uint32_t* fl) {
  int nq = S->nq, nd = S->nd, nphi = S->nphi;
  double* geom = NULL;
  int gstride = 0;
  int st = cell_geometry_all(S, verts, S->ug, &geom, &gstride, fl);
  if (st) { free(geom); return st; }
  int ftz = S->engine == 2;
  double* zhat = malloc(sizeof(double) * nq);
  int have_z = coef_zhat(S, verts, kind, coef, zhat, fl);
  double wm[165];
  for (int k = 0; k < nphi; ++k) wm[k] = RND(w[k], S->us);
  double* what = malloc(sizeof(double) * nd * nq);
  for (int s = 0; s < nd; ++s)
    for (int q = 0; q < nq; ++q) {
      double acc = 0.0;
      for (int k = 0; k < nphi; ++k) {
        double prod = orc_op(wm[k], S->tab_store[((size_t)s * nphi + k) * nq + q], 2, S->up, 0, fl);
        acc = orc_op(acc, prod, 0, S->up, ftz, fl);
      }
      what[(size_t)s * nq + q] = RND(acc, S->ug);
    }
  double* r = malloc(sizeof(double) * nd * nq);
  for (int q = 0; q < nq; ++q) {
    double omega = RND(S->wts[q], S->ug);
    const double* ten = geom + (size_t)q * gstride + 20;
    for (int s = 0; s < nd; ++s) {
      double t1 = 0.0;
      for (int t = 0; t < nd; ++t)
        t1 = ADD(t1, MUL(ten[s * 3 + t], what[(size_t)t * nq + q], S->ug), S->ug);
      double m1 = MUL(omega, t1, S->ug);
      if (have_z) m1 = MUL(m1, zhat[q], S->ug);
      r[(size_t)s * nq + q] = RND(m1, S->us);
    }
  }
  for (int i = 0; i < nphi; ++i) {
    double acc = 0.0;
    for (int s = 0; s < nd; ++s)
      for (int q = 0; q < nq; ++q) {
        double prod = orc_op(S->tab_store[((size_t)s * nphi + i) * nq + q], r[(size_t)s * nq + q],
                             2, S->uq, 0, fl);
        acc = orc_op(acc, prod, 0, S->uq, ftz, fl);
      }
    v[i] = acc;
  }
  free(zhat); free(what); free(r); free(geom);
  return 0;
}

/* action_kernel on hexahedra (per-point geometry), constant or nodal coefficients. */
int orc_action_box(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                   const double* coef, int coef_stride, const double* w, int w_stride,
                   double* v_out, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  if (kind != ORC_COEF_ONE && kind != ORC_COEF_NODAL)
    return fail(2, "box cells take constant or nodal coefficients");
  setup_t S;
  int st = make_setup_kind(p, form, cfg, &S, 1);
  if (!st) {
    for (int64_t c = 0; c < m && !st; ++c)
      st = action_one(&S, verts + 24 * c, kind, coef ? coef + (int64_t)coef_stride * c : NULL,
                      w + (int64_t)w_stride * c, v_out + (int64_t)S.nphi * c, fl);
  }
  free_setup(&S);
  return st;
}

int orc_action(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
               const double* coef, int coef_stride, const double* w, int w_stride,
               double* v_out, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  setup_t S;
  int st = make_setup(p, form, cfg, &S);
  if (!st) {
    for (int64_t c = 0; c < m && !st; ++c)
      st = action_one(&S, verts + 12 * c, kind, coef ? coef + (int64_t)coef_stride * c : NULL,
                      w + (int64_t)w_stride * c, v_out + (int64_t)S.nphi * c, fl);
  }
  free_setup(&S);
  return st;
}

/* kernel_bounds, action part (bounds.cpp:29-281: the r stage 128-155 and the v
 * accumulation 222-240, bound_v 269-279). Q path as orc_bound: z_at = c(x_q), and the
 * coefficient-evaluation budget term (kv z_norm) is zero because c enters at >= u_g.
 * out4 = {bound_v, kappa_q_v, kappa_p_v, kappa_g_v}; v64 = the exact binary64 v. */
int orc_action_bound(int p, int form, const int* cfg, const double* verts, int kind,
                     const double* coef, const double* w, double* out4, double* v64) {
  setup_t S;
  int st = make_setup(p, form, cfg, &S);
  if (st) { free_setup(&S); return st; }
  int nq = S.nq, nd = S.nd, nphi = S.nphi;
  int poisson = form == ORC_POISSON;
  uint32_t scratch = 0;
  uint32_t* fl = &scratch;
  double geom[ORC_GEOM_SIZE];
  st = orc_cell_geometry(verts, form, ORC_FP64, geom, fl);
  if (st) { free_setup(&S); return st; }
  const double* ten = geom + 20;
  const double* tt = geom + 31;
  double kk2 = geom[30] * geom[29];
  size_t nb = (size_t)nd * nphi * nq;
  double* tab = malloc(sizeof(double) * nb);
  tabulate_b(&S.B, S.pts, nq, ORC_FP64, ORC_FP64, poisson, tab, fl);
  cond_t* bc = malloc(sizeof *bc);
  basis_conditioning(&S.B, S.pts, nq, bc);
  double dp = 3.0 * p, pd = pow((double)p, 3), kv = bc->lebesgue;
  double z_norm = 0.0, w_norm = 0.0;
  if (kind == ORC_COEF_NODAL)
    for (int i = 0; i < nphi; ++i) if (fabs(coef[i]) > z_norm) z_norm = fabs(coef[i]);
  for (int i = 0; i < nphi; ++i) if (fabs(w[i]) > w_norm) w_norm = fabs(w[i]);
  double* theta_b = calloc(nb, sizeof(double));
  if (poisson) {
    for (int s = 0; s < nd; ++s)
      for (int k = 0; k < nphi; ++k) {
        double peak = 0.0;
        for (int q = 0; q < nq; ++q) {
          double a = fabs(tab[((size_t)s * nphi + k) * nq + q]);
          if (a > peak) peak = a;
        }
        for (int q = 0; q < nq; ++q)
          theta_b[((size_t)s * nphi + k) * nq + q] = dp * bc->grad_kappa[k][s] * peak;
      }
  } else {
    for (size_t i = 0; i < nb; ++i) theta_b[i] = dp * fabs(tab[i]);
  }
  double* r = malloc(sizeof(double) * nd * nq);
  double* thr = malloc(sizeof(double) * nd * nq);
  double* gr = malloc(sizeof(double) * nd * nq);
  for (int q = 0; q < nq; ++q) {
    const double* x = S.pts + 3 * q;
    double z_at = 1.0;
    if (kind == ORC_COEF_NODAL) {
      z_at = 0.0;
      for (int i = 0; i < nphi; ++i) z_at += coef[i] * eval_basis(&S.B, i, x, ORC_FP64, fl);
    } else if (kind == ORC_COEF_SINCOSEXP) {
      double xp[3];
      phys_point(verts, x, xp);
      z_at = coef_sincosexp(xp);
    } else if (kind == ORC_COEF_EXP10_AFFINE) {
      z_at = coef_exp10_affine(coef, x);
    }
    double omega = S.wts[q];
    if (poisson) {
      double gw[3] = {0.0, 0.0, 0.0};  /* eval_fe_gradient (elements.cpp:224-236) */
      for (int i = 0; i < nphi; ++i) {
        double g[3];
        eval_basis_gradient(&S.B, i, x, ORC_FP64, g, fl);
        for (int a = 0; a < 3; ++a) gw[a] += w[i] * g[a];
      }
      for (int s = 0; s < 3; ++s) {
        double gw_s = 0.0, gtw_s = 0.0, kappa_s = 0.0;
        for (int t = 0; t < 3; ++t) {
          gw_s += ten[s * 3 + t] * gw[t];
          gtw_s += fabs(tt[s * 3 + t]) * fabs(gw[t]);
          kappa_s += fabs(ten[s * 3 + t]) * bc->grad_kappa_max[t] * bc->grad_lebesgue[t];
        }
        size_t idx = (size_t)s * nq + q;
        r[idx] = omega * z_at * gw_s;
        thr[idx] = pd * fabs(omega) * (kv * z_norm * fabs(gw_s) + fabs(z_at) * w_norm * kappa_s);
        gr[idx] = kk2 * fabs(omega * z_at) * gtw_s;
      }
    } else {
      double w_at = 0.0;
      for (int i = 0; i < nphi; ++i) w_at += w[i] * eval_basis(&S.B, i, x, ORC_FP64, fl);
      double g = ten[0];
      r[q] = omega * z_at * g * w_at;
      thr[q] = pd * kv * (fabs(w_at) * z_norm + fabs(z_at) * w_norm) * fabs(omega * g);
      gr[q] = kk2 * fabs(r[q]);
    }
  }
  double vmax = 0, svmax = 0, tvmax = 0, gvmax = 0;
  for (int i = 0; i < nphi; ++i) {
    double acc = 0.0, sv = 0.0, tv = 0.0, gv = 0.0;
    for (int s = 0; s < nd; ++s)
      for (int q = 0; q < nq; ++q) {
        double b = tab[((size_t)s * nphi + i) * nq + q];
        double tb = theta_b[((size_t)s * nphi + i) * nq + q];
        size_t idx = (size_t)s * nq + q;
        acc += b * r[idx];
        sv += fabs(b) * fabs(r[idx]);
        tv += fabs(b) * thr[idx] + tb * fabs(r[idx]);
        gv += fabs(b) * gr[idx];
      }
    if (v64) v64[i] = acc;
    if (fabs(acc) > vmax) vmax = fabs(acc);
    if (sv > svmax) svmax = sv;
    if (tv > tvmax) tvmax = tv;
    if (gv > gvmax) gvmax = gv;
  }
  double u_p = FMT[S.up].u, u_g = FMT[S.ug].u, u_q = FMT[S.uq].u, u_s = FMT[S.us].u;
  if (vmax > 0.0) {
    out4[1] = svmax / vmax;
    out4[2] = tvmax / vmax;
    out4[3] = gvmax / vmax;
    out4[0] = (u_s + nq * u_q) * out4[1] + u_p * out4[2] + u_g * out4[3];
  } else {
    out4[0] = out4[1] = out4[2] = out4[3] = NAN;
  }
  free(tab); free(bc); free(theta_b); free(r); free(thr); free(gr);
  free_setup(&S);
  return 0;
}

/* ------------------------------------------------------------------ synthetic inputs */
static double det3(const double j[3][3]) { /* mesh.cpp:21-25 */
  return j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
         j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
         j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
}

int orc_gen_tets(int kind, uint64_t seed, int64_t m, double* verts, double* coef_out) {
  static const double ref[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  for (int64_t c = 0; c < m; ++c) {
    double X[4][3];
    if (kind == 0) {
      for (;;) {
        for (int v = 0; v < 4; ++v)
          for (int a = 0; a < 3; ++a) X[v][a] = ref[v][a] + orc_rng_uniform(&rng, -0.15, 0.15);
        double e[3][3];
        for (int i = 0; i < 3; ++i) {
          e[i][0] = X[1][i] - X[0][i];
          e[i][1] = X[2][i] - X[0][i];
          e[i][2] = X[3][i] - X[0][i];
        }
        double d = det3(e);
        if (fabs(d) < 1e-3) continue;
        if (d < 0.0)
          for (int a = 0; a < 3; ++a) { double t = X[2][a]; X[2][a] = X[3][a]; X[3][a] = t; }
        break;
      }
    } else {
      double sa = orc_rng_uniform(&rng, 0.0, 4.0);
      double sb = orc_rng_uniform(&rng, 0.0, 4.0);
      /* rotation construction as test_geometry.cpp:20-40, angle in [0, 2 pi) */
      double axis[3];
      for (int a = 0; a < 3; ++a) axis[a] = orc_rng_uniform(&rng, -1.0, 1.0);
      double norm = sqrt(axis[0] * axis[0] + axis[1] * axis[1] + axis[2] * axis[2]);
      for (int a = 0; a < 3; ++a) axis[a] /= norm;
      double angle = orc_rng_uniform(&rng, 0.0, 6.283185307179586);
      double co = cos(angle), si = sin(angle);
      double R[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double cross = 0.0;
          if (i != j) {
            int k = 3 - i - j;
            double sign = ((j + 1) % 3 == i) ? 1.0 : -1.0;
            cross = sign * axis[k];
            if ((i + 1) % 3 == j) cross = -cross;
          }
          R[i][j] = co * (i == j ? 1.0 : 0.0) + si * cross + (1.0 - co) * axis[i] * axis[j];
        }
      double sc[3] = {1.0, pow(10.0, -sa), pow(10.0, -sb)};
      for (int v = 0; v < 4; ++v)
        for (int i = 0; i < 3; ++i) {
          double acc = 0.0;
          for (int j = 0; j < 3; ++j) acc += R[i][j] * (sc[j] * ref[v][j]);
          X[v][i] = acc;
        }
      for (int v = 0; v < 4; ++v) coef_out[c * 4 + v] = orc_rng_uniform(&rng, 0.0, 1.0);
    }
    for (int v = 0; v < 4; ++v)
      for (int a = 0; a < 3; ++a) verts[c * 12 + v * 3 + a] = X[v][a];
  }
  return 0;
}

/* ------------------------------------------------------------------ mesh */
int orc_tet_mesh_sizes(int nx, int ny, int nz, int64_t* nv, int64_t* nc) {
  *nv = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  *nc = (int64_t)nx * ny * nz * 6;
  return 0;
}

/* jittered_lattice + structured_tet_mesh: mesh.cpp:78-163 */
int orc_structured_tet_mesh(int nx, int ny, int nz, double extent, double jitter,
                            uint64_t seed, double* verts, int32_t* cells) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(2, "mesh must have at least one cell per axis");
  if (extent <= 0.0) return fail(2, "mesh extent must be positive");
  if (jitter < 0.0 || jitter > 0.45) return fail(2, "jitter fraction must be in [0, 0.45]");
  double h[3] = {extent / nx, extent / ny, extent / nz};
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  int64_t iv = 0;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        double v[3] = {i * h[0], j * h[1], k * h[2]};
        for (int a = 0; a < 3; ++a) v[a] += orc_rng_uniform(&rng, -jitter * h[a], jitter * h[a]);
        for (int a = 0; a < 3; ++a) verts[iv * 3 + a] = v[a];
        ++iv;
      }
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int64_t ic = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int hex[8];
        for (int b = 0; b < 8; ++b)
          hex[b] = (i + (b & 1)) + (nx + 1) * ((j + ((b >> 1) & 1)) + (ny + 1) * (k + ((b >> 2) & 1)));
        for (int pi = 0; pi < 6; ++pi) {
          int bits = 0, tet[4];
          tet[0] = hex[0];
          for (int step = 0; step < 3; ++step) {
            bits |= 1 << perms[pi][step];
            tet[step + 1] = hex[bits];
          }
          const double* a = verts + 3 * (int64_t)tet[0];
          const double* b = verts + 3 * (int64_t)tet[1];
          const double* c = verts + 3 * (int64_t)tet[2];
          const double* d = verts + 3 * (int64_t)tet[3];
          double e[3][3];
          for (int x = 0; x < 3; ++x) {
            e[x][0] = b[x] - a[x];
            e[x][1] = c[x] - a[x];
            e[x][2] = d[x] - a[x];
          }
          if (det3(e) < 0.0) { int t = tet[2]; tet[2] = tet[3]; tet[3] = t; }
          for (int v = 0; v < 4; ++v) cells[ic * 4 + v] = tet[v];
          ++ic;
        }
      }
  return 0;
}

/* ------------------------------------------------------------------ dofmap */
/* build_dofmap (continuous): mesh.cpp:204-298. Geometric identification with a
 * floor-keyed grid and 27-neighbour probing, first-encounter numbering. */
typedef struct { int64_t k[3]; int head; int used; } gslot;
typedef struct { double x[3]; int dof; int next; } gnode;

static uint64_t gkey_hash(const int64_t* k) { /* mesh.cpp:192-200 */
  uint64_t h = 0x9e3779b97f4a7c15ull;
  for (int a = 0; a < 3; ++a) h ^= (uint64_t)k[a] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h;
}

int orc_build_dofmap(int p, int64_t n_verts, const double* verts, int64_t n_cells,
                     const int32_t* cells, int32_t* cell_dofs, int32_t* n_dofs_out,
                     int32_t* max_mult_out) {
  (void)n_verts;
  basis_t B;
  int st = build_basis(p, &B);
  if (st) return st;
  const basis_t* G1 = geom_basis();
  int nphi = B.n_phi;
  double h = INFINITY;
  for (int64_t c = 0; c < n_cells; ++c) {
    double diam = 0.0;
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        const double* va = verts + 3 * (int64_t)cells[c * 4 + a];
        const double* vb = verts + 3 * (int64_t)cells[c * 4 + b];
        double d2 = 0.0;
        for (int i = 0; i < 3; ++i) d2 += (va[i] - vb[i]) * (va[i] - vb[i]);
        if (d2 > diam) diam = d2;
      }
    double s = sqrt(diam);
    if (s < h) h = s;
  }
  double tol = 1e-9 * h;
  double pitch = 100.0 * tol;
  int64_t total = n_cells * nphi;
  size_t cap = 1;
  while (cap < (size_t)total * 2 + 16) cap <<= 1;
  gslot* slots = calloc(cap, sizeof(gslot));
  gnode* nodes = malloc(sizeof(gnode) * (size_t)(total + 1));
  int32_t* mult = malloc(sizeof(int32_t) * (size_t)(total + 1));
  int nn = 0, nd = 0;
  double psi[165][4];
  uint32_t fl = 0;
  for (int k = 0; k < nphi; ++k)
    for (int g = 0; g < 4; ++g) psi[k][g] = eval_basis(G1, g, B.nodes[k], ORC_FP64, &fl);
  for (int64_t c = 0; c < n_cells && !st; ++c) {
    for (int k = 0; k < nphi; ++k) {
      double x[3] = {0, 0, 0};
      for (int g = 0; g < 4; ++g) {
        const double* xg = verts + 3 * (int64_t)cells[c * 4 + g];
        for (int i = 0; i < 3; ++i) x[i] += xg[i] * psi[k][g];
      }
      int64_t key[3];
      for (int a = 0; a < 3; ++a) key[a] = (int64_t)floor(x[a] / pitch);
      int found = -1;
      double best = INFINITY;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            int64_t pk[3] = {key[0] + dx, key[1] + dy, key[2] + dz};
            size_t s = gkey_hash(pk) & (cap - 1);
            while (slots[s].used) {
              if (slots[s].k[0] == pk[0] && slots[s].k[1] == pk[1] && slots[s].k[2] == pk[2]) {
                for (int e = slots[s].head; e >= 0; e = nodes[e].next) {
                  double d2 = 0.0;
                  for (int a = 0; a < 3; ++a) d2 += (x[a] - nodes[e].x[a]) * (x[a] - nodes[e].x[a]);
                  if (d2 < best) { best = d2; found = nodes[e].dof; }
                }
                break;
              }
              s = (s + 1) & (cap - 1);
            }
          }
      double dist = sqrt(best);
      int dofid;
      if (found >= 0 && dist <= 0.5 * tol) {
        dofid = found;
      } else if (found >= 0 && dist <= 100.0 * tol) {
        st = fail(3, "dof node collision: two basis nodes nearly coincide");
        break;
      } else {
        dofid = nd++;
        mult[dofid] = 0;
        size_t s = gkey_hash(key) & (cap - 1);
        while (slots[s].used && !(slots[s].k[0] == key[0] && slots[s].k[1] == key[1] &&
                                  slots[s].k[2] == key[2]))
          s = (s + 1) & (cap - 1);
        if (!slots[s].used) {
          slots[s].used = 1;
          slots[s].head = -1;
          memcpy(slots[s].k, key, sizeof key);
        }
        /* append at the tail to keep the reference's vector order */
        nodes[nn].dof = dofid;
        nodes[nn].next = -1;
        memcpy(nodes[nn].x, x, sizeof x);
        if (slots[s].head < 0) {
          slots[s].head = nn;
        } else {
          int e = slots[s].head;
          while (nodes[e].next >= 0) e = nodes[e].next;
          nodes[e].next = nn;
        }
        ++nn;
      }
      cell_dofs[c * nphi + k] = dofid;
      ++mult[dofid];
    }
  }
  if (!st) {
    int mm = 1;
    for (int i = 0; i < nd; ++i) if (mult[i] > mm) mm = mult[i];
    *n_dofs_out = nd;
    *max_mult_out = mm;
  }
  free(slots);
  free(nodes);
  free(mult);
  return st;
}

/* ------------------------------------------------------------------ assembly */
typedef struct { uint64_t key; int64_t seq; double v; } contrib_t;
static int cmp_contrib(const void* a, const void* b) {
  const contrib_t* x = a;
  const contrib_t* y = b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* assemble_matrix: assembly.cpp:41-88 -- per key, first contribution cast to fmt and
 * the rest added in (cell asc, i asc, j asc) order with one rounding each. */
int orc_assemble_matrix(int64_t n_cells, int n_loc, const int32_t* cd, int32_t n_dofs,
                        const double* locals, int fmt, int64_t* nnz, int32_t* rows,
                        int32_t* cols, double* values, uint32_t* fl) {
  uint32_t dummy = 0;
  if (!fl) fl = &dummy;
  if (n_loc <= 0) return fail(2, "dof map has no complete cells");
  size_t total = (size_t)n_cells * n_loc * n_loc;
  contrib_t* cs = malloc(sizeof(contrib_t) * (total ? total : 1));
  size_t idx = 0;
  for (int64_t c = 0; c < n_cells; ++c)
    for (int i = 0; i < n_loc; ++i) {
      int32_t gi = cd[c * n_loc + i];
      if (gi < 0 || gi >= n_dofs) { free(cs); return fail(3, "dof index out of range"); }
      for (int j = 0; j < n_loc; ++j) {
        int32_t gj = cd[c * n_loc + j];
        if (gj < 0 || gj >= n_dofs) { free(cs); return fail(3, "dof index out of range"); }
        cs[idx].key = (uint64_t)gi * (uint64_t)n_dofs + (uint64_t)gj;
        cs[idx].seq = (int64_t)idx;
        cs[idx].v = locals[((size_t)c * n_loc + i) * n_loc + j];
        ++idx;
      }
    }
  qsort(cs, total, sizeof(contrib_t), cmp_contrib);
  int64_t out = 0;
  for (size_t a = 0; a < total;) {
    size_t b = a;
    double acc = RND(cs[a].v, fmt);
    for (b = a + 1; b < total && cs[b].key == cs[a].key; ++b) acc = ADD(acc, RND(cs[b].v, fmt), fmt);
    if (rows) {
      rows[out] = (int32_t)(cs[a].key / (uint64_t)n_dofs);
      cols[out] = (int32_t)(cs[a].key % (uint64_t)n_dofs);
      values[out] = acc;
    }
    ++out;
    a = b;
  }
  *nnz = out;
  free(cs);
  return 0;
}
