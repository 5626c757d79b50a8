// bounds.cuh -- KB: the reference's a-priori error bound kernel_bounds (bounds.cpp:29-281,
// bilinear part) evaluated per cell on the GPU in binary64, so that bound dominance can be
// checked on every cell of a full mesh instead of a host-side sample.
//
// Per cell: the binary64 geometry and its diagnostics (geometry.cpp:12-245: J, |det|, G,
// G~ = |det| |J^-1| |J^-T|, kappa_2(J) by cyclic Jacobi on J^T J, kappa_cell), the coefficient
// at the rule points, the scaled-weight stage budgets (c, theta_c, gamma_c; bounds.cpp:104-126)
// and the four accumulations of the output stage (exact A, sum |b||h|, theta, gamma;
// bounds.cpp:197-223) in the reference's (s, t, q) order. This translation unit is compiled
// with --fmad=false, so every value is the reference's binary64 result bit for bit (for
// constant and nodal coefficients; the analytic coefficient goes through CUDA's sin/cos/exp).
#pragma once
#include <cstdint>

#include "device_fp.cuh"

namespace mpfem_b200 {

struct BoundParams {
  const double* verts;
  const int32_t* cells;
  int64_t n_cells;
  int coef_kind;
  const double* coef;
  int64_t coef_stride;
  const double* tab;      // binary64 store tabulation (s n_phi + k) n_q + q (values / gradients)
  const double* theta_b;  // its evaluation budgets, same layout (bounds.cpp:75-95)
  const double* vals;     // binary64 value tabulation k n_q + q (nodal coefficient)
  const double* rule_w;   // binary64 weights
  const double* rule_x;   // [q][3]
  int n_phi, n_q, n_d, p;
  double lebesgue;        // basis_condition_numbers().lebesgue
  double u_p, u_g, u_q, u_s;
  double* out;            // n_cells x 4: bound_a, kappa_q, kappa_p, kappa_g
  double* a64;            // optional n_cells x n_phi^2: exact binary64 A (report.a)
  int* error;
  // action part (bound_v): w per cell and the gradient conditioning of the basis
  const double* w;        // n_cells rows of n_phi (row stride w_stride); NULL = bilinear
  int64_t w_stride;
  double grad_lebesgue[3], grad_kappa_max[3];
  // hexahedra: geometry at every rule point through the degree-1 box gradients (binary64)
  int box;
  const double* ggrad64;  // (s * 8 + k) * n_q + q
};

constexpr int kBoundThreads = 256;

// Host launchers (launch_bounds.cu). Return 0 or 4 (attribute failure). The action launcher
// evaluates the action part of kernel_bounds (bound_v, bounds.cpp:128-155,224-240,268-279)
// with a64 receiving the exact v (n_cells x n_phi).
int launch_bounds_kernel(const BoundParams& P, int sm_count, cudaStream_t st);
int launch_action_bounds_kernel(const BoundParams& P, int sm_count, cudaStream_t st);

}  // namespace mpfem_b200
