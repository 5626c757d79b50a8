// launch_fused.cu -- instantiations of the fused small-degree kernel.
#include <cuda_runtime.h>

#include <stdexcept>

#include "cellmat_fused.cuh"

namespace mpfem_b200 {
namespace {
template <int P, int FORM, int UG, int US>
void launch_fused_coef(int coef, unsigned grid, cudaStream_t st, const FusedParams& F) {
  switch (coef) {
    case 0: cellmat_fused_kernel<P, FORM, UG, US, 0><<<grid, 128, 0, st>>>(F); break;
    case 1: cellmat_fused_kernel<P, FORM, UG, US, 1><<<grid, 128, 0, st>>>(F); break;
    case 2: cellmat_fused_kernel<P, FORM, UG, US, 2><<<grid, 128, 0, st>>>(F); break;
    default: cellmat_fused_kernel<P, FORM, UG, US, 3><<<grid, 128, 0, st>>>(F); break;
  }
}

template <int P, int FORM, int UG>
void launch_fused_us(int us, unsigned grid, cudaStream_t st, const FusedParams& F) {
  switch (us) {
    case 0: launch_fused_coef<P, FORM, UG, 0>(F.coef_kind, grid, st, F); break;
    case 1: launch_fused_coef<P, FORM, UG, 1>(F.coef_kind, grid, st, F); break;
    default: launch_fused_coef<P, FORM, UG, 2>(F.coef_kind, grid, st, F); break;
  }
}

}  // namespace

void launch_fused_dispatch(int key, int us, unsigned grid, cudaStream_t st, const FusedParams& F) {
  switch (key) {
    case 102: launch_fused_us<1, 0, 2>(us, grid, st, F); break;
    case 103: launch_fused_us<1, 0, 3>(us, grid, st, F); break;
    case 112: launch_fused_us<1, 1, 2>(us, grid, st, F); break;
    case 113: launch_fused_us<1, 1, 3>(us, grid, st, F); break;
    case 202: launch_fused_us<2, 0, 2>(us, grid, st, F); break;
    case 203: launch_fused_us<2, 0, 3>(us, grid, st, F); break;
    default: break;  // choose_path only selects the fused path for these keys
  }
}

}  // namespace mpfem_b200
