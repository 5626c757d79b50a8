// launch_action.cu -- instantiations and launch of KA (action.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "action.cuh"

namespace mpfem_b200 {
namespace {
constexpr size_t kActionSmemMax = 227 * 1024;

// Tile height C (cells per CTA, a multiple of the per-thread block): both contractions run
// ceil(items / threads) rounds of a sequential loop (the reference's order forbids splitting
// an output's sum), so C is chosen to minimise the rounds per cell, e.g. P4: C = 28 gives
// 7 x 35 = 245 output items for 256 threads where C = 32 would need two rounds of 280.
template <int A, bool BOX>
int pick_tile(int n_phi, int n_q, int n_d, size_t budget, int threads) {
  const int n1 = n_d * n_q;
  int best = 0;
  double best_cost = 0.0;
  for (int c = kActionCBA; c <= 32; c += kActionCBA) {
    if (action_smem_bytes<A, BOX>(c, n_phi, n_q, n_d) > budget) break;
    const int g = c / kActionCB, ga = c / kActionCBA;
    const double rounds_a = double((ga * n1 + threads - 1) / threads) * n_phi;
    const double rounds_c = double((g * n_phi + threads - 1) / threads) * n1;
    const double rounds_b = double((c * n_q + threads - 1) / threads) * 8.0 * n_d;
    const double cost = (rounds_a + rounds_c + rounds_b) / c;
    if (!best || cost < best_cost * 0.999) {
      best = c;
      best_cost = cost;
    }
  }
  return best;
}

template <int A, bool FTZ, int UGK, bool BOX, bool FMA = false>
int launch_one(const ActionParams& P0, int sm_count, cudaStream_t st) {
  ActionParams P = P0;
  // measured (scripts/action_sweep.py, P4): mass 128 threads / 36 KB tiles (230 vs 291 us),
  // Poisson 256 threads / 70 KB tiles (710 vs 773 us)
  const int threads = P.n_d == 1 ? 128 : kActionThreads;
  const size_t budget = P.n_d == 1 ? 36 * 1024 : 70 * 1024;
  int tile = pick_tile<A, BOX>(P.n_phi, P.n_q, P.n_d, budget, threads);
  int per_sm = std::max(1, std::min(int(224 * 1024 / std::max<size_t>(1, action_smem_bytes<A, BOX>(tile ? tile : kActionCBA, P.n_phi, P.n_q, P.n_d) + 1024)), 2048 / threads));
  if (!tile) {  // high degree in fp64: one CTA of kActionCBA cells per SM
    tile = kActionCBA;
    per_sm = 1;
  }
  const size_t smem = action_smem_bytes<A, BOX>(tile, P.n_phi, P.n_q, P.n_d);
  if (smem > kActionSmemMax) return 2;  // tile does not fit shared memory (not reached for p <= 8)
  P.tile = tile;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    if (cudaFuncSetAttribute(action_kernel<A, FTZ, UGK, BOX, FMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(std::max<size_t>(smem, 48 * 1024))) != cudaSuccess)
      return 4;
    smem_set = smem;
  }
  const int64_t tiles = (P.n_cells + tile - 1) / tile;
  const unsigned grid = unsigned(std::min<int64_t>(tiles, int64_t(sm_count) * per_sm));
  action_kernel<A, FTZ, UGK, BOX, FMA><<<grid, threads, smem, st>>>(P);
  return 0;
}
}  // namespace

template <bool BOX>
int launch_kind(int ap, int aq, const ActionParams& P, int sm_count, cudaStream_t st) {
  const int a = ap == aq ? ap : kArGen;
  const bool ftz = P.ftz != 0;
  if (a == kArF64 && P.ug == kFP64) return launch_one<kArF64, false, kUg64, BOX>(P, sm_count, st);
  if (a == kArF16 && P.ug == kFP32) return launch_one<kArF16, false, kUg32, BOX>(P, sm_count, st);
  // fp32 accumulation over fp16-stored operands: products are exact, one FFMA per term (action.cuh madd)
  if (a == kArF32 && P.us == kFP16 && P.ug == kFP32)
    return ftz ? launch_one<kArF32, true, kUg32, BOX, true>(P, sm_count, st) : launch_one<kArF32, false, kUg32, BOX, true>(P, sm_count, st);
  if (a == kArF32 && P.us == kFP16 && P.ug == kFP64)
    return ftz ? launch_one<kArF32, true, kUg64, BOX, true>(P, sm_count, st) : launch_one<kArF32, false, kUg64, BOX, true>(P, sm_count, st);
  if (a == kArF32 && P.ug == kFP32)
    return ftz ? launch_one<kArF32, true, kUg32, BOX>(P, sm_count, st) : launch_one<kArF32, false, kUg32, BOX>(P, sm_count, st);
  if (a == kArF32 && P.ug == kFP64)
    return ftz ? launch_one<kArF32, true, kUg64, BOX>(P, sm_count, st) : launch_one<kArF32, false, kUg64, BOX>(P, sm_count, st);
  // every other format combination: binary64 carriers with the flagged emulation
  if (a == kArF64) return launch_one<kArF64, false, kUgGen, BOX>(P, sm_count, st);
  if (a == kArF32)
    return ftz ? launch_one<kArF32, true, kUgGen, BOX>(P, sm_count, st) : launch_one<kArF32, false, kUgGen, BOX>(P, sm_count, st);
  if (a == kArF16) return launch_one<kArF16, false, kUgGen, BOX>(P, sm_count, st);
  return ftz ? launch_one<kArGen, true, kUgGen, BOX>(P, sm_count, st) : launch_one<kArGen, false, kUgGen, BOX>(P, sm_count, st);
}

int launch_action(int ap, int aq, const ActionParams& P, int sm_count, cudaStream_t st) {
  return P.box ? launch_kind<true>(ap, aq, P, sm_count, st) : launch_kind<false>(ap, aq, P, sm_count, st);
}

}  // namespace mpfem_b200
