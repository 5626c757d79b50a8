// launch_action.cu -- instantiations and launch of KA (action.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "action.cuh"

namespace mpfem_b200 {
namespace {
constexpr size_t kActionSmemBudget = 100 * 1024;  // two CTAs per SM

template <int A>
void launch_one(const ActionParams& P0, int sm_count, cudaStream_t st) {
  ActionParams P = P0;
  // tile: as many cells as fit the budget, a multiple of the per-thread cell block
  int tile = 32;
  while (tile > kActionCB && action_smem_bytes<A, A>(tile, P.n_phi, P.n_q, P.n_d) > kActionSmemBudget)
    tile -= kActionCB;
  while (tile > 1 && action_smem_bytes<A, A>(tile, P.n_phi, P.n_q, P.n_d) > kActionSmemBudget) --tile;
  P.tile = tile;
  const size_t smem = action_smem_bytes<A, A>(tile, P.n_phi, P.n_q, P.n_d);
  static size_t smem_set = 0;
  if (smem > smem_set) {
    if (cudaFuncSetAttribute(action_kernel<A, A>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(std::max<size_t>(smem, 48 * 1024))) != cudaSuccess)
      return;  // reported by the caller's launch check
    smem_set = smem;
  }
  const int64_t tiles = (P.n_cells + tile - 1) / tile;
  const unsigned grid = unsigned(std::min<int64_t>(tiles, int64_t(sm_count) * 2));
  action_kernel<A, A><<<grid, kActionThreads, smem, st>>>(P);
}
}  // namespace

void launch_action(int ap, int aq, const ActionParams& P, int sm_count, cudaStream_t st) {
  const int a = ap == aq ? ap : kArGen;
  switch (a) {
    case kArF64: launch_one<kArF64>(P, sm_count, st); break;
    case kArF32: launch_one<kArF32>(P, sm_count, st); break;
    case kArF16: launch_one<kArF16>(P, sm_count, st); break;
    default: launch_one<kArGen>(P, sm_count, st); break;
  }
}

}  // namespace mpfem_b200
