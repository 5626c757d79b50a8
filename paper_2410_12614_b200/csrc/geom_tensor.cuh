// geom_tensor.cuh -- parameters of K1 from precomputed geometry tensors (geom_tensor.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mpfem_b200 {

struct WTensorParams {
  const double* G;          // n_cells x n_pts x nd x nd geometry tensors at u_g (row-major)
  int n_pts;                // 1 (affine cells) or n_q (one entry per rule point)
  int64_t n_cells;
  const double* z;          // nodal coefficient rows (z_stride doubles apart; 0 = shared) or NULL
  int64_t z_stride;
  const double* rule_w_ug;  // omega_q rounded to u_g
  const double* tab_up;     // n_phi x n_q basis values evaluated at u_p
  int n_phi, n_q, nq_pad, nd, n_blocks;
  int up, ug, us;
  int64_t k_pad;
  void* W;
  uint32_t* flags;
};

void launch_w_from_tensor(int w_type, const WTensorParams& P, int sm_count, cudaStream_t st);

}  // namespace mpfem_b200
