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

// Native-precision twin of the geometry sequence for u_g = fp32 / fp64: IEEE fp32 / fp64
// +,-,*,/ (explicit _rn intrinsics, no contraction) are the correctly rounded results the
// emulation computes, so the values are bit-identical (as tet_geometry_f32 / _f64_fast).
// Returns false on a zero pivot or any non-finite value; the caller then reruns the flagged
// emulation, which also produces the reference's FP flags for those events.
template <typename F> struct NativeOps;
template <> struct NativeOps<float> {
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float div(float a, float b) { return __fdiv_rn(a, b); }
};
template <> struct NativeOps<double> {
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double div(double a, double b) { return __ddiv_rn(a, b); }
};

template <typename F>
__device__ __forceinline__ bool box_geometry_native(const F jac[3][3], bool poisson, TetGeometry& out) {
  using O = NativeOps<F>;
  F lu[3][3];
  int perm[3] = {0, 1, 2};
  int sign = 1;
  bool finite = true;
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) lu[i][s] = jac[i][s];
  #pragma unroll
  for (int col = 0; col < 3; ++col) {
    int pivot = col;
    F best = fabs(lu[col][col]);
    #pragma unroll
    for (int r = col + 1; r < 3; ++r)
      if (fabs(lu[r][col]) > best) { best = fabs(lu[r][col]); pivot = r; }
    F pv = lu[col][col];
    #pragma unroll
    for (int r = col + 1; r < 3; ++r)
      if (pivot == r) pv = lu[r][col];
    if (pv == F(0)) return false;
    #pragma unroll
    for (int r = col + 1; r < 3; ++r)
      if (pivot == r) {
        #pragma unroll
        for (int c = 0; c < 3; ++c) { const F t = lu[r][c]; lu[r][c] = lu[col][c]; lu[col][c] = t; }
        const int t = perm[r]; perm[r] = perm[col]; perm[col] = t;
        sign = -sign;
      }
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      const F m = O::div(lu[r][col], lu[col][col]);
      lu[r][col] = m;
      #pragma unroll
      for (int c = col + 1; c < 3; ++c) lu[r][c] = O::sub(lu[r][c], O::mul(m, lu[col][c]));
    }
  }
  F det = F(sign);
  #pragma unroll
  for (int i = 0; i < 3; ++i) det = O::mul(det, lu[i][i]);
  finite = finite && isfinite(det);
  const F adet = fabs(det);
  out.det = double(det);
  out.abs_det = double(adet);
  if (!poisson) {
    out.g[0] = double(adet);
    return finite;
  }
  F inv[3][3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    F y[3];
    #pragma unroll
    for (int r = 0; r < 3; ++r) {
      F s = perm[r] == k ? F(1) : F(0);
      #pragma unroll
      for (int c = 0; c < r; ++c) s = O::sub(s, O::mul(lu[r][c], y[c]));
      y[r] = s;
    }
    #pragma unroll
    for (int r = 2; r >= 0; --r) {
      F s = y[r];
      #pragma unroll
      for (int c = r + 1; c < 3; ++c) s = O::sub(s, O::mul(lu[r][c], inv[c][k]));
      inv[r][k] = O::div(s, lu[r][r]);
    }
  }
  int idx = 0;
  #pragma unroll
  for (int s = 0; s < 3; ++s)
    #pragma unroll
    for (int t = s; t < 3; ++t) {
      F dot = F(0);
      #pragma unroll
      for (int k = 0; k < 3; ++k) dot = O::add(dot, O::mul(inv[s][k], inv[t][k]));
      const F g = O::mul(adet, dot);
      finite = finite && isfinite(g);
      out.g[idx++] = double(g);
    }
  return finite;
}

template <typename T, int UG>
__global__ void __launch_bounds__(128) geom_w_box_kernel(const GeomBoxParams P) {
  uint32_t fl = 0;
  T* W = static_cast<T*>(P.W);
  const int64_t items = P.n_cells * P.nq_pad;
  for (int64_t it = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; it < items;
       it += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cell = it / P.nq_pad;
    const int q = int(it - cell * P.nq_pad);
    T* wrow = W + cell * P.k_pad;
    if (q == 0)
      for (int64_t e = P.k; e < P.k_pad; ++e) wrow[e] = T(0.0f);
    if (q >= P.n_q) {
      for (int b = 0; b < P.n_blocks; ++b) wrow[b * P.nq_pad + q] = T(0.0f);
      continue;
    }
    double vx[8][3], gq[3][8];
    #pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t base = P.cells ? int64_t(P.cells[cell * 8 + k]) * 3 : cell * 24 + k * 3;
      #pragma unroll
      for (int i = 0; i < 3; ++i) vx[k][i] = P.verts[base + i];
      #pragma unroll
      for (int s = 0; s < 3; ++s) gq[s][k] = P.ggrad[(size_t(s) * 8 + k) * P.n_q + q];
    }
    TetGeometry geo;
    bool done = false;
    if constexpr (UG == kFP32 || UG == kFP64) {
      using F = typename std::conditional<UG == kFP32, float, double>::type;
      using O = NativeOps<F>;
      F jn[3][3];
      bool fin = true;
      #pragma unroll
      for (int i = 0; i < 3; ++i)
        #pragma unroll
        for (int s = 0; s < 3; ++s) jn[i][s] = F(0);
      #pragma unroll
      for (int k = 0; k < 8; ++k)
        #pragma unroll
        for (int i = 0; i < 3; ++i) {
          const F x = F(vx[k][i]);  // one RNE rounding to u_g (exact for u_g = fp64)
          // tiny (fp32-subnormal) or non-finite inputs take the flagged path for exact flags
          fin = fin && isfinite(x) && (UG == kFP64 || vx[k][i] == 0.0 || fabs(vx[k][i]) >= 0x1.0p-126);
          #pragma unroll
          for (int s = 0; s < 3; ++s) jn[i][s] = O::add(jn[i][s], O::mul(x, F(gq[s][k])));
        }
      done = fin && box_geometry_native<F>(jn, P.poisson != 0, geo);
    }
    if (!done) {  // flagged emulation: rare events (zero pivot, non-finite, subnormal inputs)
      double jac[3][3];
      #pragma unroll
      for (int i = 0; i < 3; ++i)
        #pragma unroll
        for (int s = 0; s < 3; ++s) jac[i][s] = 0.0;
      #pragma unroll 1
      for (int k = 0; k < 8; ++k)
        #pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double x = droundT<UG>(vx[k][i], fl);
          #pragma unroll
          for (int s = 0; s < 3; ++s) jac[i][s] = daddT<UG>(jac[i][s], dmulT<UG>(x, gq[s][k], fl), fl);
        }
      if (!jac_geometry_flagged<UG>(jac, P.poisson != 0, geo, fl)) {
        atomicExch(P.error, 3);
        #pragma unroll
        for (int b = 0; b < 6; ++b) geo.g[b] = 0.0;
      }
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
      wrow[b * P.nq_pad + q] = to_w<T>(round_us_rt(v, P.us, fl));
    }
  }
  publish_flags(P.flags, fl);
}

template <typename T>
void launch_ug(const GeomBoxParams& P, unsigned grid, cudaStream_t st) {
  switch (P.ug) {
    case kFP64: geom_w_box_kernel<T, kFP64><<<grid, 128, 0, st>>>(P); break;
    case kFP32: geom_w_box_kernel<T, kFP32><<<grid, 128, 0, st>>>(P); break;
    case kFP16: geom_w_box_kernel<T, kFP16><<<grid, 128, 0, st>>>(P); break;
    default: geom_w_box_kernel<T, kBF16><<<grid, 128, 0, st>>>(P); break;
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
