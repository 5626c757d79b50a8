// host_setup.hpp -- one-off host setup of a kernel configuration: the collapsed
// Gauss-Jacobi rule, the product-form Lagrange basis on the unit tet and its
// tabulations (the reference's make_setup, kernels.cpp:78-108). Runs once per setup
// handle; everything per-cell runs on the device.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

namespace mpfem_b200 {

// Reduced-precision rounding of a binary64 carrier on the host (softfloat.hpp:72-157),
// used for the u_p tabulations that feed the nodal-coefficient path.
double host_round(double x, int fmt, uint32_t& flags);

struct Rule {
  int n_q = 0;
  std::vector<double> points;   // n_q x 3
  std::vector<double> weights;  // n_q
};

// rule_for(simplex, p): quadrature.cpp:171-224 (collapsed Gauss-Jacobi, (p+1)^3 points).
Rule simplex_rule(int p);

// One product-form basis function: weight * prod_j (a_j . x + b_j).
struct Factor {
  std::array<double, 3> a{0.0, 0.0, 0.0};
  double b = 0.0;
  std::array<int8_t, 3> sign{0, 0, 0};
};
struct Basis {
  int p = 0;
  int m = 0;      // factors per function: p (tets), 3p (boxes)
  bool box = false;
  int n_phi = 0;
  std::vector<std::array<double, 3>> nodes;
  std::vector<double> weight;
  std::vector<std::vector<Factor>> factors;  // n_phi x p
};

// build_basis(simplex 3D, p): elements.cpp:89-147.
Basis simplex_basis(int p);
// build_basis(box 3D, p), equispaced nodes: elements.cpp:26-31,50-87 (axis 0 fastest).
Basis box_basis(int p);
// rule_for(box, p): Gauss-Legendre (p+1)^3 points, axis 0 fastest (quadrature.cpp:171-224).
Rule box_rule(int p);

// tabulate(basis, rule, eval_fmt, store_fmt, gradients): elements.cpp:171-274.
// Layout (s * n_phi + k) * n_q + q.
std::vector<double> tabulate(const Basis& b, const Rule& r, int eval_fmt, int store_fmt,
                             bool gradients, uint32_t& flags);

// basis_condition_numbers (elements.cpp:278-359): Lebesgue constant of the values, per-axis
// gradient Lebesgue constants and per-function gradient evaluation condition numbers, sampled
// at the rule points, the nodes and 2000 seeded points (Rng(9001), rejection in the unit tet).
// Host inputs of the GPU bound evaluation (kernel_bounds, bounds.cpp:29-281).
struct BasisCond {
  double lebesgue = 1.0;
  std::array<double, 3> grad_lebesgue{0.0, 0.0, 0.0};
  std::vector<std::array<double, 3>> grad_kappa;  // n_phi
  std::array<double, 3> grad_kappa_max{0.0, 0.0, 0.0};
};
BasisCond basis_conditioning(const Basis& b, const Rule& r);

}  // namespace mpfem_b200
