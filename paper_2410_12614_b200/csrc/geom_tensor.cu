// geom_tensor.cu -- K1 from precomputed geometry: the drop-in path of the reference's own
// per-cell call bilinear_kernel(setup, geom, z, flags) (kernels.hpp:85-86), where the caller
// has already run cell_geometry (geometry.cpp:226-245) and hands over GeometryData.
//
//   W[c, b * nq_pad + q] = round_us(round_ug(round_ug(omega_q G_st(c, q)) zhat_q))
//
// is build_C (kernels.cpp:177-197) with the (s <= t) pairs packed as in geom_w.cuh; every
// product is the reference's binary64-then-round operation (fp_mul, softfloat.hpp:170-186),
// including its FP flags, so W is the reference's C bit for bit. zhat_q is eval_z_at_ug
// (kernels.cpp:114-136) over the u_p value tabulation. G is the cell's geometry tensor at
// u_g, one entry for affine cells or one per rule point. Any dimension (the pairs of an
// n_d x n_d tensor); the W layout and the GEMM (K2) are the vertex path's.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "geom_tensor.cuh"
#include "geom_w.cuh"

namespace mpfem_b200 {

template <typename T>
__global__ void __launch_bounds__(256) w_from_tensor_kernel(const WTensorParams P) {
  uint32_t fl = 0;
  const int64_t total = P.n_cells * P.nq_pad;
  const int nd2 = P.nd * P.nd;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = idx / P.nq_pad;
    const int q = int(idx - c * P.nq_pad);
    T* wrow = static_cast<T*>(P.W);
    const int64_t row = c * P.k_pad;
    if (q == 0)  // tail K..K_pad of the row
      for (int64_t k = int64_t(P.n_blocks) * P.nq_pad; k < P.k_pad; ++k) store_w<T>(wrow, row + k, 0.0);
    if (q >= P.n_q) {  // padding points: exact zeros
      for (int b = 0; b < P.n_blocks; ++b) store_w<T>(wrow, row + int64_t(b) * P.nq_pad + q, 0.0);
      continue;
    }
    double zq = 1.0;
    const bool have_z = P.z != nullptr;
    if (have_z) {
      const double* z = P.z + c * P.z_stride;
      double acc = 0.0;
      for (int k = 0; k < P.n_phi; ++k)
        acc = dadd(acc, dmul(dround(z[k], P.up, fl), P.tab_up[int64_t(k) * P.n_q + q], P.up, fl), P.up, fl);
      zq = dround(acc, P.ug, fl);
    }
    const double om = P.rule_w_ug[q];
    const double* g = P.G + (c * P.n_pts + (P.n_pts == 1 ? 0 : q)) * nd2;
    for (int b = 0; b < P.n_blocks; ++b) {
      int s, t;
      block_pair(b, P.nd, s, t);
      double v = dmul(om, g[s * P.nd + t], P.ug, fl);
      if (have_z) v = dmul(v, zq, P.ug, fl);
      v = dround(v, P.us, fl);
      store_w<T>(wrow, row + int64_t(b) * P.nq_pad + q, v);
    }
  }
  publish_flags(P.flags, fl);
}

void launch_w_from_tensor(int w_type, const WTensorParams& P, int sm_count, cudaStream_t st) {
  const int64_t total = P.n_cells * P.nq_pad;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, int64_t(sm_count) * 16)));
  switch (w_type) {
    case 0: w_from_tensor_kernel<__half><<<grid, 256, 0, st>>>(P); break;
    case 1: w_from_tensor_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(P); break;
    case 2: w_from_tensor_kernel<float><<<grid, 256, 0, st>>>(P); break;
    default: w_from_tensor_kernel<double><<<grid, 256, 0, st>>>(P); break;
  }
}

}  // namespace mpfem_b200
