// geom_box.cuh -- K1 for hexahedral (box) cells: the scaled weights
// W = build_C (kernels.cpp:177-197) with the geometry evaluated at every rule point
// (cell_geometry, geometry.cpp:226-245, non-affine branch): J(xi_q) = sum_k x_k (x) grad phi_k(xi_q)
// through the degree-1 box basis at u_g (geometry.cpp:12-27), then LU, det, inverse and the
// geometry tensor at u_g (the shared jac_geometry_flagged). Bitwise the reference's values for
// constant and nodal coefficients; one thread per (cell, rule point). The GEMM (K2) is the
// tets' kernel unchanged: only W's values differ (per-point G instead of per-cell G).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "device_fp.cuh"

namespace mpfem_b200 {

struct GeomBoxParams {
  const double* verts;   // n_cells x 8 x 3 private, or the vertex table when cells != NULL
  const int32_t* cells;  // n_cells x 8 (lattice bit order, x fastest)
  int64_t n_cells;
  int coef_kind;         // 0 one, 3 nodal
  const double* coef;
  int64_t coef_stride;
  const double* rule_w_ug;  // omega_q at u_g
  const double* ggrad;      // degree-1 box basis gradients at u_g, (s * 8 + k) * n_q + q
  const double* tab_up;     // value tabulation at u_p, k * n_q + q
  int n_phi, n_q, nq_pad, n_blocks;
  int64_t k, k_pad;
  int up, ug, us;
  int poisson;
  void* W;
  uint32_t* flags;
  int* error;
};

// Host launcher (launch_geom_box.cu): w_type 0 fp16, 1 bf16, 2 fp32, 3 fp64.
void launch_geom_box(int w_type, const GeomBoxParams& P, int sm_count, cudaStream_t st);

}  // namespace mpfem_b200
