// launch_geom.cu -- instantiations of K1 (geom_w_kernel)
// for every (W element type, u_g, u_s, coefficient kind).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "geom_w.cuh"

#define CUDA_CHECK_K1(x)                                            \
  do {                                                              \
    if ((x) != cudaSuccess) return;  /* reported by the launch check */ \
  } while (0)

namespace mpfem_b200 {
namespace {
template <typename T, int UG, int US, int COEF>
void launch_one(unsigned grid, cudaStream_t st, const GeomWParams& P) {
  const size_t smem = geom_w_smem_bytes(P.nq_pad, P.geom_warps);
  static size_t smem_set = 0;
  if (smem > smem_set) {
    // P8 has nq_pad = 736 (23.5 KB); keep three CTAs per SM for every degree
    CUDA_CHECK_K1(cudaFuncSetAttribute(geom_w_kernel<T, UG, US, COEF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // full shared-memory carveout: an SM configured by K1 must still fit K2's 197 KB CTA
    // when the two run concurrently
    CUDA_CHECK_K1(cudaFuncSetAttribute(geom_w_kernel<T, UG, US, COEF>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout,
                                       int(cudaSharedmemCarveoutMaxShared)));
    smem_set = smem;
  }
  geom_w_kernel<T, UG, US, COEF><<<grid, kGeomThreads, smem, st>>>(P);
}

template <typename T, int US>
void launch_geom_ug(int ug, unsigned grid, cudaStream_t st, const GeomWParams& P) {
  switch (ug) {
#define MPFEM_K1(UGV)                                                   \
  switch (P.coef_kind) {                                                \
    case 0: launch_one<T, UGV, US, 0>(grid, st, P); break;              \
    case 1: launch_one<T, UGV, US, 1>(grid, st, P); break;              \
    case 2: launch_one<T, UGV, US, 2>(grid, st, P); break;              \
    default: launch_one<T, UGV, US, 3>(grid, st, P); break;             \
  }                                                                     \
  break;
    case 0: MPFEM_K1(0)
    case 1: MPFEM_K1(1)
    case 2: MPFEM_K1(2)
    default: MPFEM_K1(3)
#undef MPFEM_K1
  }
}

// W element type follows u_s except on the fp64 path, where any u_s is carried in fp64.
}  // namespace

void launch_geom_typed(int w_type, int ug, int us, unsigned grid, cudaStream_t st,
                       const GeomWParams& P) {
  switch (w_type) {
    case 0: launch_geom_ug<__half, 1>(ug, grid, st, P); break;
    case 1: launch_geom_ug<__nv_bfloat16, 0>(ug, grid, st, P); break;
    case 2: launch_geom_ug<float, 2>(ug, grid, st, P); break;
    default:
      switch (us) {
        case 0: launch_geom_ug<double, 0>(ug, grid, st, P); break;
        case 1: launch_geom_ug<double, 1>(ug, grid, st, P); break;
        case 2: launch_geom_ug<double, 2>(ug, grid, st, P); break;
        default: launch_geom_ug<double, 3>(ug, grid, st, P); break;
      }
  }
}


}  // namespace mpfem_b200
