// mpfem/batched.hpp -- the B200 drop-in for the reference's hot path, C++ side.
//
// Link paper_2410_12614_b200/shim/mpfem_b200_shim.cpp (built against the reference's own
// headers, proj/include/mpfem) and libmpfem_b200.so in place of the reference definitions of
//   bilinear_kernel (kernels.hpp:85-86), action_kernel (kernels.hpp:90-92),
//   build_dofmap (mesh.hpp:61), assemble_matrix (assembly.hpp:29-30)
// and every existing caller keeps its code: the declarations are the reference's, unchanged.
// Each call runs on the GPU through the C-ABI (include/mpfem_b200.h); there is no CPU
// fallback -- configurations outside the B200 path raise ConfigError.
//
// This header adds the batched overloads, which amortise one launch over many cells (the
// per-cell calls above are batches of one).
#pragma once
#include <vector>

#include "mpfem/assembly.hpp"
#include "mpfem/kernels.hpp"
#include "mpfem/mesh.hpp"

namespace mpfem {

// bilinear_kernel for every geometry of `geoms` in one launch; z shared by all cells (empty:
// constant one). Result i equals bilinear_kernel(setup, geoms[i], z, flags).
std::vector<Mat> bilinear_kernel(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                                 const Coefficients& z, FpFlags& flags);

// Same with one nodal coefficient vector per cell (z.size() == geoms.size()).
std::vector<Mat> bilinear_kernel(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                                 const std::vector<Coefficients>& z, FpFlags& flags);

// Releases the device setups the shim created (cached per configuration, rule and
// tabulation). Optional: without it they live until the process exits.
void release_device_setups();

}  // namespace mpfem
