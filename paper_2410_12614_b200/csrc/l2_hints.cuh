// l2_hints.cuh -- L2 eviction-priority hints shared by the scatter kernels (assembly.cuh) and the
// fused K2 epilogue (cellmat_tc2.cuh).
#pragma once
#include <cstdint>

namespace mpfem_b200 {
namespace asmb {

// red.global.add with an L2 evict-last hint: the CSR value lines are the only data of the
// order-free scatter that is touched more than once (by the neighbouring cells' reductions);
// the local matrices, the plan and W stream past them with evict-first.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void red_add_keep(float* addr, float v, uint64_t policy) {
  asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(addr), "f"(v), "l"(policy) : "memory");
}
__device__ __forceinline__ void red_add_keep(double* addr, double v, uint64_t policy) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(addr), "d"(v), "l"(policy) : "memory");
}

}  // namespace asmb
}  // namespace mpfem_b200
