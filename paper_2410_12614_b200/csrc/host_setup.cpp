// host_setup.cpp -- quadrature, basis and tabulation for a setup handle.
//
// The arithmetic follows the reference's published algorithms step for step so that
// the rule weights and tabulated values are bit-identical to make_setup's
// (tests/test_gpu_parity.py checks this against the oracle through the C-ABI):
//   * Gauss-Legendre by Newton on the three-term recurrence (quadrature.cpp:91-124)
//   * Gauss-Jacobi by Golub-Welsch with implicit-shift QL (quadrature.cpp:31-81,126-169)
//   * collapsed (Duffy) tensor rule, axis 0 fastest (quadrature.cpp:171-224)
//   * product-form Lagrange basis on the equispaced principal lattice
//     (elements.cpp:89-147), evaluated factor by factor (elements.cpp:165-211).
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <random>
#include <cstring>
#include <stdexcept>

namespace mpfem_b200 {

namespace {

constexpr double kPi = 3.14159265358979323846;

struct Narrow {
  int drop;
  double min_normal, min_sub, max_finite;
};
Narrow narrow_of(int fmt) {
  return fmt == 0 ? Narrow{45, 0x1.0p-126, 0x1.0p-133, 0x1.fep127}
                  : Narrow{42, 0x1.0p-14, 0x1.0p-24, 65504.0};
}

}  // namespace

double host_round(double x, int fmt, uint32_t& fl) {
  if (fmt == 3) {
    if (std::isnan(x)) { fl |= 4u; return std::nan(""); }
    return x;
  }
  if (fmt == 2) {
    float g = float(x);
    if (std::isnan(g)) { fl |= 4u; return std::nan(""); }
    if (std::isinf(g)) { if (!std::isinf(x)) fl |= 1u; return double(g); }
    if (x != 0.0 && std::fabs(x) < 0x1.0p-126 && double(g) != x) fl |= 2u;
    return double(g);
  }
  Narrow n = narrow_of(fmt);
  uint64_t bits;
  std::memcpy(&bits, &x, 8);
  uint64_t mag = bits & 0x7fffffffffffffffull;
  if (mag >= 0x7ff0000000000000ull) {
    if (mag > 0x7ff0000000000000ull) { fl |= 4u; return std::nan(""); }
    return x;
  }
  if (mag == 0) return x;
  double ax = std::fabs(x);
  if (ax < n.min_normal) {
    double r = std::copysign(std::nearbyint(ax / n.min_sub) * n.min_sub, x);
    if (r != x) fl |= 2u;
    return r;
  }
  uint64_t mask = (uint64_t(1) << n.drop) - 1, rem = bits & mask, half = uint64_t(1) << (n.drop - 1);
  bits &= ~mask;
  if (rem > half || (rem == half && (bits >> n.drop & 1u))) bits += uint64_t(1) << n.drop;
  double r;
  std::memcpy(&r, &bits, 8);
  if (std::fabs(r) > n.max_finite) { fl |= 1u; return std::copysign(INFINITY, x); }
  return r;
}

namespace {

// Legendre P_n and P_n' on [-1, 1].
void legendre_pair(int n, double x, double& p, double& dp) {
  double prev = 1.0, cur = x;
  for (int j = 2; j <= n; ++j) {
    double next = ((2.0 * j - 1.0) * x * cur - (j - 1.0) * prev) / double(j);
    prev = cur;
    cur = next;
  }
  p = (n == 0) ? prev : cur;
  dp = (n == 0) ? 0.0 : double(n) * (x * cur - prev) / (x * x - 1.0);
}

void gauss_legendre(int n, double* xs, double* ws) {
  if (n == 1) {
    xs[0] = 0.5;
    ws[0] = 1.0;
    return;
  }
  for (int k = 0; k < n; ++k) {
    double x = std::cos(kPi * (k + 0.75) / (n + 0.5));
    double p = 0.0, dp = 1.0;
    for (int it = 0;; ++it) {
      if (it >= 100) throw std::runtime_error("Legendre Newton iteration stalled");
      legendre_pair(n, x, p, dp);
      double step = p / dp;
      x -= step;
      if (std::fabs(step) < 1e-15) break;
    }
    legendre_pair(n, x, p, dp);
    xs[n - 1 - k] = 0.5 * (x + 1.0);
    ws[n - 1 - k] = 0.5 * (2.0 / ((1.0 - x * x) * dp * dp));
  }
}

// Eigen-decomposition of the Jacobi matrix (symmetric tridiagonal) by implicit QL;
// only the first row of the eigenvector matrix is needed for the weights, but the
// full rotation is accumulated to keep the arithmetic identical.
void jacobi_matrix_ql(int n, std::vector<double>& d, std::vector<double>& e,
                      std::vector<double>& z) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-300 + 2.3e-16 * dd) break;
      }
      if (m == l) break;
      if (iter++ == 60) throw std::runtime_error("tridiagonal QL stalled");
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      bool deflated = false;
      for (int i = m - 1; i >= l; --i) {
        double f = s * e[i], b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[m] = 0.0;
          deflated = true;
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
          double* row = &z[std::size_t(k) * n];
          f = row[i + 1];
          row[i + 1] = s * row[i] + c * f;
          row[i] = c * row[i] - s * f;
        }
      }
      if (deflated) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0.0;
    } while (m != l);
  }
}

void gauss_jacobi(int n, int alpha, double* xs, double* ws) {
  std::vector<double> d(n), e(n, 0.0), z(std::size_t(n) * n, 0.0);
  d[0] = -double(alpha) / double(alpha + 2);
  for (int k = 1; k < n; ++k) {
    double den = 2.0 * k + alpha;
    d[k] = -double(alpha) * double(alpha) / (den * (den + 2.0));
    e[k] = std::sqrt(4.0 * k * k * (k + alpha) * (k + alpha) / (den * den * (den * den - 1.0)));
  }
  for (int i = 0; i < n; ++i) z[std::size_t(i) * n + i] = 1.0;
  jacobi_matrix_ql(n, d, e, z);
  double mu0 = std::pow(2.0, alpha + 1) / double(alpha + 1);
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) {  // stable insertion sort by node
    int key = order[i], j = i - 1;
    for (; j >= 0 && d[order[j]] > d[key]; --j) order[j + 1] = order[j];
    order[j + 1] = key;
  }
  for (int i = 0; i < n; ++i) {
    int k = order[i];
    xs[i] = 0.5 * (d[k] + 1.0);
    ws[i] = mu0 * z[k] * z[k] * std::pow(0.5, alpha + 1);
  }
}

}  // namespace

Rule simplex_rule(int p) {
  int n = p + 1;
  double fx[3][64], fw[3][64];
  // collapse x = xi0, y = xi1 (1 - xi0), z = xi2 (1 - xi0)(1 - xi1): Jacobi exponents 2, 1, 0
  gauss_jacobi(n, 2, fx[0], fw[0]);
  gauss_jacobi(n, 1, fx[1], fw[1]);
  gauss_legendre(n, fx[2], fw[2]);
  Rule r;
  r.n_q = n * n * n;
  r.points.resize(std::size_t(r.n_q) * 3);
  r.weights.resize(r.n_q);
  for (int q = 0; q < r.n_q; ++q) {
    int ix[3] = {q % n, (q / n) % n, q / (n * n)};
    double w = 1.0, shrink = 1.0;
    for (int a = 0; a < 3; ++a) w *= fw[a][ix[a]];
    for (int a = 0; a < 3; ++a) {
      double xi = fx[a][ix[a]];
      r.points[std::size_t(q) * 3 + a] = xi * shrink;
      shrink *= (1.0 - xi);
    }
    r.weights[q] = w;
  }
  return r;
}

Basis simplex_basis(int p) {
  Basis b;
  b.p = p;
  // multi-indices (a1, a2, a3), a1 fastest, a0 = p - sum
  for (int a3 = 0; a3 <= p; ++a3)
    for (int a2 = 0; a2 <= p; ++a2)
      for (int a1 = 0; a1 <= p; ++a1) {
        if (a1 + a2 + a3 > p) continue;
        int al[4] = {p - a1 - a2 - a3, a1, a2, a3};
        std::vector<Factor> fs;
        double w = 1.0;
        for (int i = 0; i <= 3; ++i)
          for (int k = 0; k < al[i]; ++k) {
            Factor f;
            if (i == 0) {
              f.a = {-1.0, -1.0, -1.0};
              f.sign = {-1, -1, -1};
              f.b = 1.0 - double(k) / double(p);
            } else {
              f.a[i - 1] = 1.0;
              f.sign[i - 1] = 1;
              f.b = -double(k) / double(p);
            }
            fs.push_back(f);
            w *= double(p) / double(al[i] - k);
          }
        b.nodes.push_back({double(a1) / double(p), double(a2) / double(p), double(a3) / double(p)});
        b.weight.push_back(w);
        b.factors.push_back(std::move(fs));
      }
  b.n_phi = int(b.weight.size());
  b.m = p;
  return b;
}

Basis box_basis(int p) {
  Basis b;
  b.p = p;
  b.m = 3 * p;
  b.box = true;
  const int n1 = p + 1;
  std::vector<double> xs(n1);
  for (int j = 0; j <= p; ++j) xs[j] = double(j) / double(p);
  b.n_phi = n1 * n1 * n1;
  for (int idx = 0; idx < b.n_phi; ++idx) {
    int iax[3], rem = idx;
    for (int a = 0; a < 3; ++a) {
      iax[a] = rem % n1;
      rem /= n1;
    }
    std::vector<Factor> fs;
    double w = 1.0;
    for (int a = 0; a < 3; ++a)
      for (int j = 0; j <= p; ++j) {
        if (j == iax[a]) continue;
        Factor f;
        f.a[a] = 1.0;
        f.b = -xs[j];
        f.sign[a] = 1;
        fs.push_back(f);
        w /= xs[iax[a]] - xs[j];
      }
    b.nodes.push_back({xs[iax[0]], xs[iax[1]], xs[iax[2]]});
    b.weight.push_back(w);
    b.factors.push_back(std::move(fs));
  }
  return b;
}

Rule box_rule(int p) {
  const int n = p + 1;
  double fx[64], fw[64];
  gauss_legendre(n, fx, fw);
  Rule r;
  r.n_q = n * n * n;
  r.points.resize(std::size_t(r.n_q) * 3);
  r.weights.resize(r.n_q);
  for (int q = 0; q < r.n_q; ++q) {
    const int ix[3] = {q % n, (q / n) % n, q / (n * n)};
    double w = 1.0;
    for (int a = 0; a < 3; ++a) {
      r.points[std::size_t(q) * 3 + a] = fx[ix[a]];
      w *= fw[ix[a]];
    }
    r.weights[q] = w;
  }
  return r;
}

namespace {

double factor_at(const Factor& f, const double* x) {
  double v = f.b;
  for (int a = 0; a < 3; ++a) v += f.a[a] * x[a];
  return v;
}

double mul_at(double a, double b, int fmt, uint32_t& fl) { return host_round(a * b, fmt, fl); }

}  // namespace

std::vector<double> tabulate(const Basis& b, const Rule& r, int ef, int sf, bool grads,
                             uint32_t& fl) {
  int nd = grads ? 3 : 1, m = b.m, nphi = b.n_phi, nq = r.n_q;
  std::vector<double> out(std::size_t(nd) * nphi * nq);
  std::vector<double> l(m);
  for (int k = 0; k < nphi; ++k) {
    double w = host_round(b.weight[k], ef, fl);
    for (int q = 0; q < nq; ++q) {
      const double* x = &r.points[std::size_t(q) * 3];
      for (int j = 0; j < m; ++j) l[j] = host_round(factor_at(b.factors[k][j], x), ef, fl);
      if (!grads) {
        double acc = l[0];
        for (int j = 1; j < m; ++j) acc = mul_at(acc, l[j], ef, fl);
        out[std::size_t(k) * nq + q] = host_round(mul_at(acc, w, ef, fl), sf, fl);
        continue;
      }
      for (int s = 0; s < 3; ++s) {
        double acc = 0.0;
        for (int j = 0; j < m; ++j) {
          int sg = b.factors[k][j].sign[s];
          if (!sg) continue;
          double prod = 1.0;
          bool first = true;
          for (int i = 0; i < m; ++i) {
            if (i == j) continue;
            prod = first ? l[i] : mul_at(prod, l[i], ef, fl);
            first = false;
          }
          acc = host_round(sg > 0 ? acc + prod : acc - prod, ef, fl);
        }
        out[(std::size_t(s) * nphi + k) * nq + q] = host_round(mul_at(acc, w, ef, fl), sf, fl);
      }
    }
  }
  return out;
}

BasisCond basis_conditioning(const Basis& b, const Rule& r) {
  const int m = b.m, nphi = b.n_phi, nq = r.n_q, n_random = 2000;
  std::vector<std::array<double, 3>> pts;
  pts.reserve(size_t(nq + nphi + n_random));
  for (int q = 0; q < nq; ++q) pts.push_back({r.points[3 * q], r.points[3 * q + 1], r.points[3 * q + 2]});
  for (int k = 0; k < nphi; ++k) pts.push_back(b.nodes[k]);
  std::mt19937_64 eng(9001);  // common.hpp:21-35 Rng
  auto uniform = [&eng](double lo, double hi) { return lo + (hi - lo) * (double(eng() >> 11) * 0x1.0p-53); };
  for (int i = 0; i < n_random; ++i) {
    std::array<double, 3> x{};
    for (;;) {  // sample_point (elements.cpp:279-289)
      double sum = 0.0;
      for (int a = 0; a < 3; ++a) {
        x[a] = uniform(0.0, 1.0);
        sum += x[a];
      }
      if (b.box || sum <= 1.0) break;
    }
    pts.push_back(x);
  }
  BasisCond bc;
  std::vector<std::array<double, 3>> num_max(size_t(nphi), {0.0, 0.0, 0.0}), abs_max(size_t(nphi), {0.0, 0.0, 0.0});
  std::vector<double> lv(m), prefix(m + 1), suffix(m + 1);
  for (const auto& xs : pts) {
    const double* x = xs.data();
    double sum_abs_phi = 0.0, sum_abs_grad[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < nphi; ++i) {
      for (int j = 0; j < m; ++j) lv[j] = factor_at(b.factors[i][j], x);
      prefix[0] = 1.0;
      for (int j = 0; j < m; ++j) prefix[j + 1] = prefix[j] * lv[j];
      suffix[m] = 1.0;
      for (int j = m - 1; j >= 0; --j) suffix[j] = suffix[j + 1] * lv[j];
      sum_abs_phi += std::fabs(b.weight[i] * prefix[m]);
      for (int s = 0; s < 3; ++s) {
        double grad = 0.0, numer = 0.0;
        for (int j = 0; j < m; ++j) {
          const int sign = b.factors[i][j].sign[s];
          if (sign == 0) continue;
          const double complement = b.weight[i] * prefix[j] * suffix[j + 1];
          grad += sign * complement;
          numer += std::fabs(complement);
        }
        sum_abs_grad[s] += std::fabs(grad);
        abs_max[i][s] = std::max(abs_max[i][s], std::fabs(grad));
        num_max[i][s] = std::max(num_max[i][s], numer);
      }
    }
    bc.lebesgue = std::max(bc.lebesgue, sum_abs_phi);
    for (int s = 0; s < 3; ++s) bc.grad_lebesgue[s] = std::max(bc.grad_lebesgue[s], sum_abs_grad[s]);
  }
  bc.grad_kappa.resize(size_t(nphi));
  for (int i = 0; i < nphi; ++i)
    for (int s = 0; s < 3; ++s) {
      const double numer = num_max[i][s], denom = abs_max[i][s];
      double kappa = 1.0;
      if (numer > 0.0) kappa = denom > 0.0 ? numer / denom : INFINITY;
      bc.grad_kappa[i][s] = kappa;
      bc.grad_kappa_max[s] = std::max(bc.grad_kappa_max[s], kappa);
    }
  return bc;
}

}  // namespace mpfem_b200
