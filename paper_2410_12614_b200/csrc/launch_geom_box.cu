// launch_geom_box.cu -- K1 for box cells (geom_box.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "geom_box.cuh"

namespace mpfem_b200 {
namespace {

__device__ __forceinline__ double round_us_rt(double x, int f, uint32_t& fl) {
  switch (f) {
    case kBF16: return droundT<kBF16>(x, fl);
    case kFP16: return droundT<kFP16>(x, fl);
    case kFP32: return droundT<kFP32>(x, fl);
    default: return droundT<kFP64>(x, fl);
  }
}

template <typename T>
__device__ __forceinline__ T to_w(double v) {
  if constexpr (sizeof(T) == 8) return v;
  else if constexpr (sizeof(T) == 4) return float(v);
  else return T(float(v));  // v is already a u_s value: the conversion is exact
}

// u_s implied by the W element type (choose_path: fp16 / bf16 / fp32 W carry exactly that u_s;
// fp64 W carries any u_s, rounded at run time)
template <typename T> struct UsOf { static constexpr int v = -1; };
template <> struct UsOf<__half> { static constexpr int v = kFP16; };
template <> struct UsOf<__nv_bfloat16> { static constexpr int v = kBF16; };
template <> struct UsOf<float> { static constexpr int v = kFP32; };

template <typename T, int UG>
__global__ void __launch_bounds__(128) geom_w_box_kernel(const GeomBoxParams P) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // see geom_w_kernel
  uint32_t fl = 0;
  T* W = static_cast<T*>(P.W);
  const int64_t items = P.n_cells * P.nq_pad;
  // the u_g gradient table, (s * 8 + k) * n_q + q; held as float for u_g = fp32 (its values
  // are fp32 numbers, so the narrowing is exact and the per-point F2F conversions go away)
  using G = typename std::conditional<UG == kFP32, float, double>::type;
  extern __shared__ double s_raw[];
  G* s_gg = reinterpret_cast<G*>(s_raw);
  for (int e = threadIdx.x; e < 24 * P.n_q; e += blockDim.x) s_gg[e] = G(P.ggrad[e]);
  __syncthreads();
  using F = typename std::conditional<UG == kFP32, float, double>::type;
  // Warp-shared vertices need every lane of a warp on cells that start at a lane multiple of
  // min(nq_pad, 32): nq_pad a multiple of 32, or 8 / 16 (4 / 2 cells per warp). The item loop
  // then runs to a multiple of 32 so its trip count is warp-uniform; lanes past the last item
  // replay the last item's geometry and store nothing.
  const int grp = P.nq_pad >= 32 ? 32 : P.nq_pad;
  const bool warp_cell = UG == kFP32 && (P.nq_pad % 32 == 0 || grp == 8 || grp == 16);
  const int lane = threadIdx.x & 31;
  const int src0 = lane & ~(grp - 1);  // lane of the cell's first item (when warp_cell)
  const int64_t items_loop = warp_cell ? (items + 31) / 32 * 32 : items;
  for (int64_t it_raw = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; it_raw < items_loop;
       it_raw += int64_t(gridDim.x) * blockDim.x) {
    const bool live = it_raw < items;
    const int64_t it = live ? it_raw : items - 1;
    // 32-bit division while the item index fits (64-bit division is a long software sequence)
    const int64_t cell = items < (int64_t(1) << 31) ? int64_t(uint32_t(it) / uint32_t(P.nq_pad)) : it / P.nq_pad;
    const int q = int(it - cell * P.nq_pad);
    T* wrow = W + cell * P.k_pad;
    const int32_t* cv = P.cells ? P.cells + cell * 8 : nullptr;
    const double* pv = P.verts + cell * 24;
    auto vx = [&](int k, int i) {
      return cv ? P.verts[int64_t(cv[k]) * 3 + i] : pv[k * 3 + i];
    };
    // Warp-cooperative vertices (u_g = fp32, nq_pad a multiple of 32, so the warp's 32 items are
    // points of one cell and the loop trip count is warp-uniform): lane l < 24 loads, rounds and
    // screens coordinate l once and the native path takes it by shuffle. Every lane, padding
    // points included (at the clamped point n_q - 1, results discarded), runs the geometry so
    // that the shuffles see the full warp.
    TetGeometry geo;
    bool geo_ok;
    const bool pad = q >= P.n_q;
    const int qg = pad ? P.n_q - 1 : q;
    auto gq = [&](int s, int k) { return s_gg[(s * 8 + k) * P.n_q + qg]; };
    if (warp_cell && grp == 32) {
      // one cell per warp: lane l < 24 holds coordinate l
      const int l = lane < 24 ? lane : 0;
      const double xd = vx(l / 3, l % 3);
      const F xl = F(xd);
      const bool in_ok = __all_sync(0xffffffffu, box_input_ok<UG>(xd));
      auto xn = [&](int k, int i) { return __shfl_sync(0xffffffffu, xl, k * 3 + i); };
      geo_ok = box_point_geometry_pre<UG>(xn, in_ok, vx, gq, P.poisson != 0, geo, fl);
    } else if (warp_cell) {
      // 2 or 4 cells per warp: lane src0 + k holds vertex k of the lane's cell (three
      // coordinates); a tiny or non-finite coordinate anywhere in the warp sends the whole warp
      // to the exact fallback
      const int kv = (lane - src0) & 7;
      F xl[3];
      bool ok = true;
      #pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double xd = vx(kv, i);
        xl[i] = F(xd);
        ok = ok && box_input_ok<UG>(xd);
      }
      const bool in_ok = __all_sync(0xffffffffu, ok);
      auto xn = [&](int k, int i) { return __shfl_sync(0xffffffffu, xl[i], src0 + k); };
      geo_ok = box_point_geometry_pre<UG>(xn, in_ok, vx, gq, P.poisson != 0, geo, fl);
    } else if (!pad) {
      geo_ok = box_point_geometry<UG>(vx, gq, P.poisson != 0, geo, fl);
    }
    if (!live) continue;
    if (q == 0)
      for (int64_t e = P.k; e < P.k_pad; ++e) wrow[e] = T(0.0f);
    if (pad) {
      for (int b = 0; b < P.n_blocks; ++b) wrow[b * P.nq_pad + q] = T(0.0f);
      continue;
    }
    if (!geo_ok) {
      report_error(P.error, 3);
      #pragma unroll
      for (int b = 0; b < 6; ++b) geo.g[b] = __longlong_as_double(0x7ff8000000000000ll);  // singular: NaN row
    }
    double zq = 1.0;
    const bool have_z = P.coef_kind != 0;
    if (have_z) {  // eval_z_at_ug (kernels.cpp:114-136)
      const double* coef = P.coef + cell * P.coef_stride;
      double acc = 0.0;
      for (int k = 0; k < P.n_phi; ++k)
        acc = dadd(acc, dmul(dround(coef[k], P.up, fl), P.tab_up[size_t(k) * P.n_q + q], P.up, fl), P.up, fl);
      zq = droundT<UG>(acc, fl);
    }
    const double om = P.rule_w_ug[q];
    for (int b = 0; b < P.n_blocks; ++b) {
      double v = dmulT<UG>(om, geo.g[b], fl);
      if (have_z) v = dmulT<UG>(v, zq, fl);
      if constexpr (UsOf<T>::v >= 0) wrow[b * P.nq_pad + q] = to_w<T>(droundT<UsOf<T>::v>(v, fl));
      else wrow[b * P.nq_pad + q] = to_w<T>(round_us_rt(v, P.us, fl));
    }
  }
  publish_flags(P.flags, fl);
}

template <typename T>
void launch_ug(const GeomBoxParams& P, unsigned grid, cudaStream_t st) {
  const size_t smem = sizeof(double) * 24 * size_t(P.n_q);  // <= 24 KB for p <= 4
  switch (P.ug) {
    case kFP64: geom_w_box_kernel<T, kFP64><<<grid, 128, smem, st>>>(P); break;
    case kFP32: geom_w_box_kernel<T, kFP32><<<grid, 128, smem, st>>>(P); break;
    case kFP16: geom_w_box_kernel<T, kFP16><<<grid, 128, smem, st>>>(P); break;
    default: geom_w_box_kernel<T, kBF16><<<grid, 128, smem, st>>>(P); break;
  }
}

}  // namespace

void launch_geom_box(int w_type, const GeomBoxParams& P, int sm_count, cudaStream_t st) {
  const int64_t items = P.n_cells * P.nq_pad;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((items + 127) / 128, int64_t(sm_count) * 16)));
  switch (w_type) {
    case 0: launch_ug<__half>(P, grid, st); break;
    case 1: launch_ug<__nv_bfloat16>(P, grid, st); break;
    case 2: launch_ug<float>(P, grid, st); break;
    default: launch_ug<double>(P, grid, st); break;
  }
}

}  // namespace mpfem_b200
