// launch_geom.cu -- instantiations of K1 (cell_geometry_kernel + scaled_weights_kernel)
// for every (W element type, u_g, u_s, coefficient kind).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "geom_w.cuh"

namespace mpfem_b200 {
namespace {
template <typename T, int US>
void launch_geom_ug(int ug, unsigned grid_cells, unsigned grid_w, cudaStream_t st, const GeomWParams& P,
                    CellGeo* geo) {
  switch (ug) {
#define MPFEM_K1(UGV)                                                                       \
  cell_geometry_kernel<UGV><<<grid_cells, 256, 0, st>>>(P, geo);                            \
  switch (P.coef_kind) {                                                                    \
    case 0: scaled_weights_kernel<T, UGV, US, 0><<<grid_w, 256, 0, st>>>(P, geo); break;    \
    case 1: scaled_weights_kernel<T, UGV, US, 1><<<grid_w, 256, 0, st>>>(P, geo); break;    \
    case 2: scaled_weights_kernel<T, UGV, US, 2><<<grid_w, 256, 0, st>>>(P, geo); break;    \
    default: scaled_weights_kernel<T, UGV, US, 3><<<grid_w, 256, 0, st>>>(P, geo); break;   \
  }                                                                                         \
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

void launch_geom_typed(int w_type, int ug, int us, unsigned gc, unsigned gw, cudaStream_t st,
                       const GeomWParams& P, CellGeo* geo) {
  switch (w_type) {
    case 0: launch_geom_ug<__half, 1>(ug, gc, gw, st, P, geo); break;
    case 1: launch_geom_ug<__nv_bfloat16, 0>(ug, gc, gw, st, P, geo); break;
    case 2: launch_geom_ug<float, 2>(ug, gc, gw, st, P, geo); break;
    default:
      switch (us) {
        case 0: launch_geom_ug<double, 0>(ug, gc, gw, st, P, geo); break;
        case 1: launch_geom_ug<double, 1>(ug, gc, gw, st, P, geo); break;
        case 2: launch_geom_ug<double, 2>(ug, gc, gw, st, P, geo); break;
        default: launch_geom_ug<double, 3>(ug, gc, gw, st, P, geo); break;
      }
  }
}


}  // namespace mpfem_b200
