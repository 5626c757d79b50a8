/* ulp errors of the device's fp64 coefficient functions (old Taylor vs new minimax/table
 * versions), restated in C with fma(), against long double references.
 * gcc -O2 scripts/coef_ulp_check.c -lm -o /tmp/coef_ulp && /tmp/coef_ulp */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static const double M = 6755399441055744.0;
static uint32_t lo32(double d) { uint64_t u; memcpy(&u, &d, 8); return (uint32_t)u; }
static double from_bits(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static double flip(double v, uint32_t n) { uint64_t u; memcpy(&u, &v, 8); u ^= (uint64_t)(n & 1u) << 63; return from_bits(u); }
static const double S13[13] = {3.141592653589793, -5.16771278004997, 2.5501640398773455, -0.5992645293207921, 0.08214588661112823, -0.0073704309457143504, 0.00046630280576761255, -2.1915353447830217e-05, 7.952054001475513e-07, -2.2948428997269873e-08, 5.392664662608129e-10, -1.0518471716932065e-11, 1.7302192458361107e-13};
static const double S9[9] = {3.141592653589793, -5.167712780049969, 2.5501640398773007, -0.5992645293189447, 0.0821458865731029, -0.007370430505916944, 0.0004662998161898394, -2.1903497074626018e-05, 7.697826768224191e-07};
static double poly_s(const double* c, int n, double r) { double s = r * r, p = c[n - 1]; for (int k = n - 2; k >= 0; --k) p = fma(p, s, c[k]); return r * p; }
static double sinpi_n(const double* c, int n, double a) { double t = a + M, k = t - M; return flip(poly_s(c, n, a - k), lo32(t)); }
static double cospi_n(const double* c, int n, double a) { double t = a + M, k = t - M; return flip(poly_s(c, n, 0.5 - fabs(a - k)), lo32(t)); }
static const double E15[15] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333, 0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10, 1.1470745597729725e-11};
static double exp_old(double z) {
  double t = z * 1.4426950408889634 + M, n = t - M;
  double r = fma(-n, 6.93147180369123816490e-01, z); r = fma(-n, 1.90821492927058770002e-10, r);
  double p = E15[14]; for (int k = 13; k >= 0; --k) p = fma(p, r, E15[k]);
  return p * from_bits((uint64_t)((int64_t)(int32_t)lo32(t) + 1023) << 52);
}
static double HI[32], LO[32];
static double exp_new(double z, int half) {  /* e^z (half: e^z / 2) */
  double t = z * 46.16624130844683 + M, n = t - M;
  double r = fma(-n, 0.021660849390173098, z); r = fma(-n, 2.325192846878874e-12, r);
  double q = 1.0 / 720; q = fma(q, r, 1.0 / 120); q = fma(q, r, 1.0 / 24); q = fma(q, r, 1.0 / 6);
  q = fma(q, r, 0.5); q = fma(q, r, 1.0); double p1 = q * r;       /* e^r - 1 */
  int32_t ni = (int32_t)lo32(t); int j = ni & 31, k = ni >> 5;
  double v = HI[j] + fma(HI[j], p1, LO[j]);
  return v * from_bits((uint64_t)(int64_t)(k - half + 1023) << 52);
}
static double ulp_err(double got, long double ref) {
  if (ref == 0) return got == 0 ? 0 : 1e9;
  int e; frexpl(fabsl(ref), &e);
  long double ulp = ldexpl(1.0L, e - 53);
  return (double)(fabsl((long double)got - ref) / ulp);
}
int main(void) {
  FILE* f = popen("python3 -c \"import mpmath as m; m.mp.dps=40; [print(repr(float(m.mpf(2)**(m.mpf(j)/32))), repr(float(m.mpf(2)**(m.mpf(j)/32)-m.mpf(float(m.mpf(2)**(m.mpf(j)/32)))))) for j in range(32)]\"", "r");
  for (int j = 0; j < 32; ++j) if (fscanf(f, "%lf %lf", &HI[j], &LO[j]) != 2) return 1;
  pclose(f);
  srand(7);
  double m_s13 = 0, m_s9 = 0, m_c13 = 0, m_c9 = 0, m_eo = 0, m_en = 0, m_co = 0, m_cn = 0;
  for (int i = 0; i < 2000000; ++i) {
    double x = ((double)rand() / RAND_MAX) * 4.0 - 2.0, y = ((double)rand() / RAND_MAX) * 4.0 - 2.0;
    double z = ((double)rand() / RAND_MAX) * 20.0 - 10.0;
    double a = 2 * x, b = 2 * y;
    const long double PI = 3.14159265358979323846264338327950288L;
    double na = rint(a), nb = rint(b);                     /* exact reductions */
    long double sr = sinl(PI * (long double)(a - na)) * (((int64_t)na & 1) ? -1 : 1);
    long double cr = sinl(PI * (long double)(0.5 - fabs(b - nb))) * (((int64_t)nb & 1) ? -1 : 1);
    long double er = expl((long double)z);
    if (sr != 0) { double e1 = ulp_err(sinpi_n(S13, 13, a), sr), e2 = ulp_err(sinpi_n(S9, 9, a), sr); if (e1 > m_s13) m_s13 = e1; if (e2 > m_s9) m_s9 = e2; }
    if (cr != 0) { double e1 = ulp_err(cospi_n(S13, 13, b), cr), e2 = ulp_err(cospi_n(S9, 9, b), cr); if (e1 > m_c13) m_c13 = e1; if (e2 > m_c9) m_c9 = e2; }
    { double e1 = ulp_err(exp_old(z), er), e2 = ulp_err(exp_new(z, 0), er); if (e1 > m_eo) m_eo = e1; if (e2 > m_en) m_en = e2; }
    long double cref = 1.0L + 0.5L * sr * cr * er;
    double c_old = 1.0 + ((0.5 * sinpi_n(S13, 13, a)) * cospi_n(S13, 13, b)) * exp_old(z);
    double c_new = fma(sinpi_n(S9, 9, a) * cospi_n(S9, 9, b), exp_new(z, 1), 1.0);
    /* absolute error in ulps of the larger of the two terms (cancellation-safe) */
    long double mag = fabsl(0.5L * sr * cr * er) > 1.0L ? fabsl(0.5L * sr * cr * er) : 1.0L;
    double e1 = ulp_err(c_old, cref) * (double)(fabsl(cref) / mag), e2 = ulp_err(c_new, cref) * (double)(fabsl(cref) / mag);
    if (e1 > m_co) m_co = e1; if (e2 > m_cn) m_cn = e2;
  }
  printf("max ulp: sinpi old %.3f new %.3f | cospi old %.3f new %.3f | exp old %.3f new %.3f | coef old %.3f new %.3f\n",
         m_s13, m_s9, m_c13, m_c9, m_eo, m_en, m_co, m_cn);
  return 0;
}
