// action.cuh -- KA: the reference's Algorithm 2 (action_kernel, kernels.cpp:269-304),
// batched over cells in one fused launch, bit-identical to the reference in every mode.
//
//   what[c][s][q] = round_ug( sum_k  round_us(w_ck) * Bs[s][k][q]   at u_p, k ascending )
//                   (eval_w_at_ug, kernels.cpp:145-173)
//   r[c][s][q]    = round_us( (omega_q * (sum_t G_st what_t)) * zhat_q   at u_g, t ascending )
//                   (kernels.cpp:280-301; build_r 214-240)
//   v[c][i]       = sum_(s,q) Bs[s][i][q] * r[c][s][q]   at u_q, (s, q) ascending
//                   (blocked_matmul(b_cat_action, r_cat), kernels.cpp:303)
//
// Bs is the setup's store tabulation (evaluated at u_p, stored at u_s). Every product and
// every sum is rounded once to its format, in the reference's order, so the results are
// the reference's bits: the two contractions are sequential per output and cannot use FMA
// or a tensor-core tree (both would change the rounding). The product is therefore an
// issue-bound SIMT kernel: a CTA holds a tile of cells in shared memory, each thread keeps
// CB cells of one output column in registers so that one coalesced tabulation load (L1/L2
// resident, shared by all cells) feeds CB multiply-adds.
//
// Arithmetic per format (exact-rounding arguments as device_fp.cuh):
//   fp64: hardware DMUL/DADD;  fp32: FMUL/FADD with _rn (no contraction) -- the binary64
//   product of two fp32 values is exact, so one fp32 rounding equals the reference's;
//   fp16: fp32 op then one RNE conversion to fp16 (24 >= 2*11+2: no double-rounding error)
//   for fp16-representable operands; anything else (bf16 accumulation, operands wider than
//   the accumulate format, FTZ fp64) runs the generic binary64-carrier emulation.
// The matrix engine (engine 2) flushes subnormal accumulates to signed zero
// (mm_units.cpp:43-62, flush_output_subnormals).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "device_fp.cuh"

namespace mpfem_b200 {

enum ArithKind : int { kArF64 = 0, kArF32 = 1, kArF16 = 2, kArGen = 3 };

struct ActionParams {
  const double* verts;
  const int32_t* cells;  // optional mesh indexing (n_cells x 4)
  int64_t n_cells;
  int coef_kind;
  const double* coef;
  int64_t coef_stride;
  const double* w;  // n_cells rows of n_phi fp64 (row stride w_stride)
  int64_t w_stride;
  const void* tab_a;  // [k][s * n_q + q]  store tabulation, u_p compute type
  const void* tab_c;  // [s * n_q + q][i]  store tabulation, u_q compute type
  const double* tab_up;    // value tabulation at u_p, [k][q] (nodal coefficient)
  const double* rule_w_ug; // omega_q rounded to u_g
  const double* rule_x;    // xi_q, [q][3]
  int n_phi, n_q, n_d;
  int up, ug, uq, us;
  int ftz;
  int tile;  // cells per CTA tile
  void* out;  // n_cells x out_pitch, fp32 (u_q != fp64) or fp64
  int64_t out_pitch;
  uint32_t* flags;
  int* error;
  int box;               // hexahedra: geometry at every rule point
  const double* ggrad;   // box: degree-1 gradients at u_g, (s * 8 + k) * n_q + q
  // Geometry given by the caller (the drop-in C++ API hands over GeometryData,
  // geometry.hpp:31-41): n_cells x g_pts x n_d x n_d tensors at u_g, g_pts = 1 (affine) or
  // n_q (one per rule point). NULL: evaluated from the vertices.
  const double* G;
  int g_pts;
};

constexpr int kActionThreads = 256;
constexpr int kActionCB = 4;   // cells per thread in the b_cat_action contraction (few outputs)
constexpr int kActionCBA = 4;  // cells per thread in the w evaluation (measured: 8 is slower)

template <int A>
struct Arith;
template <>
struct Arith<kArF64> {
  using T = double;
  __device__ static T mul(T a, T b, int, uint32_t&) { return __dmul_rn(a, b); }
  __device__ static T add(T a, T b, int, bool ftz, uint32_t&) {
    T r = __dadd_rn(a, b);
    if (ftz && fabs(r) < 0x1.0p-1022) r = copysign(0.0, r);
    return r;
  }
};
template <>
struct Arith<kArF32> {
  using T = float;
  __device__ static T mul(T a, T b, int, uint32_t&) { return __fmul_rn(a, b); }
  __device__ static T add(T a, T b, int, bool ftz, uint32_t&) {
    T r = __fadd_rn(a, b);
    if (ftz && fabsf(r) < 0x1.0p-126f) r = copysignf(0.0f, r);
    return r;
  }
};
template <>
struct Arith<kArF16> {
  using T = float;
  __device__ static T mul(T a, T b, int, uint32_t&) { return __half2float(__float2half_rn(__fmul_rn(a, b))); }
  __device__ static T add(T a, T b, int, bool ftz, uint32_t&) {
    T r = __half2float(__float2half_rn(__fadd_rn(a, b)));
    if (ftz && fabsf(r) < 0x1.0p-14f) r = copysignf(0.0f, r);
    return r;
  }
};
template <>
struct Arith<kArGen> {
  using T = double;
  __device__ static T mul(T a, T b, int f, uint32_t& fl) { return dmul(a, b, f, fl); }
  __device__ static T add(T a, T b, int f, bool ftz, uint32_t& fl) {
    T r = dadd(a, b, f, fl);
    if (ftz && r != 0.0 && fabs(r) < fmt_min_normal(f)) {
      fl |= kUnderflow;
      r = copysign(0.0, r);
    }
    return r;
  }
  __device__ static double fmt_min_normal(int f) {
    return f == kFP64 ? 0x1.0p-1022 : (f == kFP16 ? 0x1.0p-14 : 0x1.0p-126);
  }
};

// One multiply-add of a contraction. FMA (fp32 accumulation over fp16-stored operands only): the
// product of two fp16 values has at most 22 significant bits and an exponent within fp32's
// normal range, so it is exact in fp32 and round(a * b + acc) = round(round(a * b) + acc): one
// FFMA gives the bits of the reference's rounded product followed by its rounded sum.
template <int A, bool FMA>
__device__ __forceinline__ typename Arith<A>::T madd(typename Arith<A>::T acc, typename Arith<A>::T a,
                                                     typename Arith<A>::T b, int f, bool ftz, uint32_t& fl) {
  if constexpr (A == kArF32 && FMA) {
    float r = __fmaf_rn(a, b, acc);
    if (ftz && fabsf(r) < 0x1.0p-126f) r = copysignf(0.0f, r);
    return r;
  } else {
    return Arith<A>::add(acc, Arith<A>::mul(a, b, f, fl), f, ftz, fl);
  }
}

// The integrand stage at u_g: hardware ops when u_g is fp64 or fp32 (every operand -- G,
// what, omega, zhat -- is already a u_g value, so the fp32 op is the reference's rounded
// binary64 op), the flagged emulation otherwise.
enum UgKind : int { kUg64 = 0, kUg32 = 1, kUgGen = 2 };
template <int UGK>
__device__ __forceinline__ double ug_mul(double a, double b, int ug, uint32_t& fl) {
  if constexpr (UGK == kUg64) return __dmul_rn(a, b);
  else if constexpr (UGK == kUg32) return double(__fmul_rn(float(a), float(b)));
  else return dmul(a, b, ug, fl);
}
template <int UGK>
__device__ __forceinline__ double ug_add(double a, double b, int ug, uint32_t& fl) {
  if constexpr (UGK == kUg64) return __dadd_rn(a, b);
  else if constexpr (UGK == kUg32) return double(__fadd_rn(float(a), float(b)));
  else return dadd(a, b, ug, fl);
}

// round_to at a runtime format through the compile-time conversions (one cvt for fp16 /
// bf16 / fp32; bitwise dround, device_fp.cuh).
__device__ __forceinline__ double dround_fast(double x, int f, uint32_t& fl) {
  switch (f) {
    case kBF16: return droundT<kBF16>(x, fl);
    case kFP16: return droundT<kFP16>(x, fl);
    case kFP32: return droundT<kFP32>(x, fl);
    default: return droundT<kFP64>(x, fl);
  }
}

// Geometry at a runtime u_g (the op sequence of cell_geometry, geometry.cpp:12-118).
static __device__ __noinline__ bool action_geometry(const double v[4][3], bool poisson, int ug,
                                             TetGeometry& g, uint32_t& fl) {
  switch (ug) {
    case kFP64: return tet_geometry<kFP64>(v, poisson, g, fl);
    case kFP32: return tet_geometry<kFP32>(v, poisson, g, fl);
    case kFP16: return tet_geometry<kFP16>(v, poisson, g, fl);
    default: return tet_geometry<kBF16>(v, poisson, g, fl);
  }
}

// Shared-memory layout of one tile of C cells (C a multiple of kActionCBA; rows past the last
// cell are zeros), cell index fastest so that the CB cells of a thread are one vector load
// and the per-(cell, q) integrand stage is bank-conflict free:
//   sWm  [k][C]          TP      round_us(w)
//   sWH  [s n_q + q][C]  double  what at u_g
//   sR   [s n_q + q][C]  TQ      r at u_s (exact in the u_q compute type)
//   sGeo [C][18 | 24]    double  tets: G (6: G00 G01 G02 G11 G12 G22 / |det|), 2v0x 2v0y v0z,
//                                edges; boxes: the 8 vertices
// The row width is per cell kind (BOX is a template parameter, so the tet kernel carries
// none of the per-point box geometry: registers / stack / shared memory as before 8f.3).
template <bool BOX>
constexpr int geo_words() { return BOX ? 24 : 18; }

template <int A, bool BOX>
__host__ __device__ inline size_t action_smem_bytes(int tile, int n_phi, int n_q, int n_d) {
  using T = typename Arith<A>::T;
  const size_t n1 = size_t(n_d) * n_q;
  // a double r overwrites what in place (each (q, cell) item reads its own three what values
  // before writing its r values), so fp64 compute types need one n1 array per cell
  const size_t r_bytes = sizeof(T) == 8 ? 0 : sizeof(T);
  return size_t(tile) * (size_t(n_phi) * sizeof(T) + n1 * (sizeof(double) + r_bytes) +
                         geo_words<BOX>() * sizeof(double));
}

// Box cells: G at rule point q of a cell whose 8 vertices sit in geo (u_g runtime for the
// generic instantiation). False on a zero pivot.
template <int UGK>
__device__ __forceinline__ bool box_g_at(const ActionParams& P, const double* geo, int q,
                                         TetGeometry& g, uint32_t& fl) {
  auto vx = [&](int k, int a) { return geo[k * 3 + a]; };
  auto gq = [&](int s, int k) { return P.ggrad[(size_t(s) * 8 + k) * P.n_q + q]; };
  const bool poisson = P.n_d == 3;
  if constexpr (UGK == kUg64) return box_point_geometry<kFP64>(vx, gq, poisson, g, fl);
  else if constexpr (UGK == kUg32) return box_point_geometry<kFP32>(vx, gq, poisson, g, fl);
  else {
    switch (P.ug) {
      case kFP64: return box_point_geometry<kFP64>(vx, gq, poisson, g, fl);
      case kFP32: return box_point_geometry<kFP32>(vx, gq, poisson, g, fl);
      case kFP16: return box_point_geometry<kFP16>(vx, gq, poisson, g, fl);
      default: return box_point_geometry<kBF16>(vx, gq, poisson, g, fl);
    }
  }
}

// One cell's geometry row at u_g: G (6, upper triangle; mass: |det|), then K1's coefficient
// inputs (2 v0x, 2 v0y, v0z and the edges with x, y doubled).
template <bool BOX>
__device__ __forceinline__ void cell_geo_row(const ActionParams& P, int64_t cell, double* geo,
                                             uint32_t& fl) {
  if (P.G) {  // given tensors: packed upper triangle of the cell's (first) entry
    const int nd = P.n_d;
    const double* g = P.G + cell * P.g_pts * nd * nd;
    for (int b = 0; b < 6; ++b) geo[b] = 0.0;
    if (nd == 1) geo[0] = g[0];
    else
      for (int s = 0, b = 0; s < 3; ++s)
        for (int t = s; t < 3; ++t, ++b) geo[b] = g[s * 3 + t];
    for (int j = 6; j < geo_words<BOX>(); ++j) geo[j] = 0.0;
    return;
  }
  if constexpr (BOX) {  // hexahedra: the vertices; the geometry is evaluated per point in the r stage
    for (int k = 0; k < 8; ++k) {
      const int64_t base = P.cells ? int64_t(P.cells[cell * 8 + k]) * 3 : cell * 24 + k * 3;
      for (int a = 0; a < 3; ++a) geo[k * 3 + a] = P.verts[base + a];
    }
    return;
  }
  double v[4][3];
  #pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t base = P.cells ? int64_t(P.cells[cell * 4 + k]) * 3 : cell * 12 + k * 3;
    #pragma unroll
    for (int a = 0; a < 3; ++a) v[k][a] = P.verts[base + a];
  }
  TetGeometry g;
  if (!action_geometry(v, P.n_d == 3, P.ug, g, fl)) {
    report_error(P.error, 3);
    for (int b = 0; b < 6; ++b) g.g[b] = __longlong_as_double(0x7ff8000000000000ll);  // singular: NaN column
  }
  for (int b = 0; b < 6; ++b) geo[b] = g.g[b];
  #pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double sc = a < 2 ? 2.0 : 1.0;
    geo[6 + a] = sc * v[0][a];
    #pragma unroll
    for (int s2 = 0; s2 < 3; ++s2) geo[9 + s2 * 3 + a] = sc * __dsub_rn(v[s2 + 1][a], v[0][a]);
  }
}

template <typename T, int N>
__device__ __forceinline__ void load_cb(const T* p, T (&v)[N]) {
  #pragma unroll
  for (int h = 0; h < N / 4; ++h) {
    if constexpr (sizeof(T) == 4) {
      const float4 x = reinterpret_cast<const float4*>(p)[h];
      v[4 * h] = x.x; v[4 * h + 1] = x.y; v[4 * h + 2] = x.z; v[4 * h + 3] = x.w;
    } else {
      const double2 x = reinterpret_cast<const double2*>(p)[2 * h], y = reinterpret_cast<const double2*>(p)[2 * h + 1];
      v[4 * h] = x.x; v[4 * h + 1] = x.y; v[4 * h + 2] = y.x; v[4 * h + 3] = y.y;
    }
  }
}

// The two contractions as CB-cell x NB-column register tiles: one shared-memory vector of the
// cells and NB tabulation words feed CB * NB multiply-adds (each output still sums its terms in
// ascending order, so the bits are those of the one-column form). Measured at config 0 / 1
// (65,536 P4 tets, mixed): NB = 2 gains 6 % for Poisson (n1 = 375 columns) and loses 8 % for
// mass (n1 = 125: too few items per tile), NB = 4 loses everywhere (profiles/r2br_action_nb_ab.txt).
template <int A, bool FTZ, bool FMA, int NB>
__device__ __forceinline__ void what_stage(const ActionParams& P, const typename Arith<A>::T* sWm,
                                           double* sWH, const typename Arith<A>::T* tabA, int C,
                                           uint32_t& fl) {
  using T = typename Arith<A>::T;
  constexpr int kActionNB = NB;
  const int nphi = P.n_phi, n1 = P.n_d * P.n_q;
  // a thread keeps a CBA-cell x kActionNB-column register tile: one shared-memory vector of
  // the cells and kActionNB tabulation words feed CBA * kActionNB multiply-adds (each output
  // still sums k ascending, so the bits are unchanged)
  const int groups_a = C / kActionCBA;
  const int n1b = (n1 + kActionNB - 1) / kActionNB;
  for (int item = threadIdx.x; item < groups_a * n1b; item += blockDim.x) {
    const int cg = item / n1b, n = (item - cg * n1b) * kActionNB;
    T acc[kActionNB][kActionCBA];
    #pragma unroll
    for (int u = 0; u < kActionNB; ++u)
      #pragma unroll
      for (int j = 0; j < kActionCBA; ++j) acc[u][j] = T(0);
    // columns past n1 repeat the last one (computed, not stored)
    int col[kActionNB];
    #pragma unroll
    for (int u = 0; u < kActionNB; ++u) col[u] = min(n + u, n1 - 1);
    const T* bp = tabA;
    const T* wp = sWm + cg * kActionCBA;
    #pragma unroll 2
    for (int k = 0; k < nphi; ++k, bp += n1, wp += C) {
      T b[kActionNB];
      #pragma unroll
      for (int u = 0; u < kActionNB; ++u) b[u] = __ldg(bp + col[u]);
      T wv[kActionCBA];
      load_cb(wp, wv);
      #pragma unroll
      for (int u = 0; u < kActionNB; ++u)
        #pragma unroll
        for (int j = 0; j < kActionCBA; ++j)
          acc[u][j] = madd<A, FMA>(acc[u][j], wv[j], b[u], P.up, FTZ, fl);
    }
    #pragma unroll
    for (int u = 0; u < kActionNB; ++u)
      if (n + u < n1) {
        #pragma unroll
        for (int j = 0; j < kActionCBA; ++j)
          sWH[size_t(n + u) * C + cg * kActionCBA + j] = dround_fast(double(acc[u][j]), P.ug, fl);
      }
  }
}

template <int A, bool FTZ, bool FMA, int NB>
__device__ __forceinline__ void v_stage(const ActionParams& P, const typename Arith<A>::T* sR,
                                        const typename Arith<A>::T* tabC, int C, int64_t c0, int nc,
                                        uint32_t& fl) {
  using T = typename Arith<A>::T;
  constexpr int kActionNB = NB;
  const int nphi = P.n_phi, n1 = P.n_d * P.n_q;
  const int groups = C / kActionCB;
  const int nphib = (nphi + kActionNB - 1) / kActionNB;
  for (int item = threadIdx.x; item < groups * nphib; item += blockDim.x) {
    const int cg = item / nphib, i = (item - cg * nphib) * kActionNB;
    T acc[kActionNB][kActionCB];
    #pragma unroll
    for (int u = 0; u < kActionNB; ++u)
      #pragma unroll
      for (int j = 0; j < kActionCB; ++j) acc[u][j] = T(0);
    int col[kActionNB];
    #pragma unroll
    for (int u = 0; u < kActionNB; ++u) col[u] = min(i + u, nphi - 1);
    const T* bp = tabC;
    const T* rp = sR + cg * kActionCB;
    #pragma unroll 4
    for (int kk = 0; kk < n1; ++kk, bp += nphi, rp += C) {
      T b[kActionNB];
      #pragma unroll
      for (int u = 0; u < kActionNB; ++u) b[u] = __ldg(bp + col[u]);
      T rv[kActionCB];
      load_cb(rp, rv);
      #pragma unroll
      for (int u = 0; u < kActionNB; ++u)
        #pragma unroll
        for (int j = 0; j < kActionCB; ++j)
          acc[u][j] = madd<A, FMA>(acc[u][j], b[u], rv[j], P.uq, FTZ, fl);
    }
    #pragma unroll
    for (int u = 0; u < kActionNB; ++u) {
      if (i + u >= nphi) continue;
      #pragma unroll
      for (int j = 0; j < kActionCB; ++j) {
        const int c = cg * kActionCB + j;
        if (c < nc) {
          double v = double(acc[u][j]);
          if (!isfinite(v)) fl |= isnan(v) ? kInvalid : kOverflow;
          // NaN leaves as the reference's canonical quiet NaN (softfloat.hpp round_to)
          if (isnan(v)) v = canonical_nan_d();
          if (P.uq == kFP64)
            static_cast<double*>(P.out)[(c0 + c) * P.out_pitch + i + u] = v;
          else
            static_cast<float*>(P.out)[(c0 + c) * P.out_pitch + i + u] = float(v);
        }
      }
    }
  }
}

template <int A, bool FTZ, int UGK, bool BOX, bool FMA = false>
__global__ void __launch_bounds__(kActionThreads) action_kernel(const ActionParams P) {
  constexpr int kGeoWords = geo_words<BOX>();
  using T = typename Arith<A>::T;
  using Ar = Arith<A>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int C = P.tile, nphi = P.n_phi, nq = P.n_q, nd = P.n_d;
  const int n1 = nd * nq;
  T* sWm = reinterpret_cast<T*>(smem);
  double* sWH = reinterpret_cast<double*>(sWm + size_t(C) * nphi);
  T* sR = sizeof(T) == 8 ? reinterpret_cast<T*>(sWH) : reinterpret_cast<T*>(sWH + size_t(C) * n1);
  double* sGeo = sizeof(T) == 8 ? sWH + size_t(C) * n1 : reinterpret_cast<double*>(sR + size_t(C) * n1);
  const T* tabA = static_cast<const T*>(P.tab_a);
  const T* tabC = static_cast<const T*>(P.tab_c);
  const bool poisson = nd == 3;
  uint32_t fl = 0;
  const int64_t n_tiles = (P.n_cells + C - 1) / C;
  const int groups = C / kActionCB;

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t c0 = tile * C;
    const int nc = int((P.n_cells - c0 < int64_t(C) ? P.n_cells - c0 : int64_t(C)));
    // -- stage: geometry (one thread per cell) and the u_s-rounded w
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      if (c < nc) cell_geo_row<BOX>(P, c0 + c, sGeo + c * kGeoWords, fl);
      else for (int j = 0; j < kGeoWords; ++j) sGeo[c * kGeoWords + j] = 0.0;
    }
    for (int e = threadIdx.x; e < C * nphi; e += blockDim.x) {
      const int c = e / nphi, k = e - c * nphi;  // coalesced over the w rows
      const double wv = c < nc ? P.w[(c0 + c) * P.w_stride + k] : 0.0;
      sWm[k * C + c] = T(dround_fast(wv, P.us, fl));
    }
    __syncthreads();

    // -- what (eval_w_at_ug): column n = s n_q + q, CBA cells per thread, k ascending at u_p
    if (poisson) what_stage<A, FTZ, FMA, 2>(P, sWm, sWH, tabA, C, fl);
    else what_stage<A, FTZ, FMA, 1>(P, sWm, sWH, tabA, C, fl);
    __syncthreads();

    // -- integrand r at u_g, stored at u_s: one thread per (q, cell), cell fastest
    const bool have_z = P.coef_kind != 0;
    for (int item = threadIdx.x; item < C * nq; item += blockDim.x) {
      const int q = item / C, c = item - q * C;
      const double* geo = sGeo + c * kGeoWords;
      const double om = P.rule_w_ug[q];
      double zq = 1.0;
      if (c < nc && have_z) {
        const double xi[3] = {P.rule_x[3 * q], P.rule_x[3 * q + 1], P.rule_x[3 * q + 2]};
        const double* coef = P.coef ? P.coef + (c0 + c) * P.coef_stride : nullptr;
        if (P.coef_kind == 1) {
          zq = P.ug == kFP32 ? double(coef_sincosexp_f(geo + 6, geo + 9, xi))
                             : dround_fast(coef_sincosexp_e(geo + 6, geo + 9, xi), P.ug, fl);
        } else if (P.coef_kind == 2) {
          zq = dround_fast(coef_exp10_affine(coef, xi), P.ug, fl);
        } else {
          double acc = 0.0;  // eval_z_at_ug (kernels.cpp:114-136)
          for (int k = 0; k < nphi; ++k)
            acc = dadd(acc, dmul(dround_fast(coef[k], P.up, fl), P.tab_up[size_t(k) * nq + q], P.up, fl), P.up, fl);
          zq = dround_fast(acc, P.ug, fl);
        }
      }
      double wt[3] = {0.0, 0.0, 0.0};  // read before r overwrites what (fp64: aliased)
      for (int t = 0; t < nd; ++t) wt[t] = sWH[size_t(t * nq + q) * C + c];
      double gbox[6];
      const double* gsrc = geo;
      if (P.G && P.g_pts > 1) {  // given per-point tensors (non-affine cells)
        const double* g = P.G + ((c0 + (c < nc ? c : 0)) * P.g_pts + q) * nd * nd;
        if (nd == 1) gbox[0] = g[0];
        else
          for (int s = 0, b = 0; s < 3; ++s)
            for (int t = s; t < 3; ++t, ++b) gbox[b] = g[s * 3 + t];
        gsrc = gbox;
      } else if constexpr (BOX) {  // hexahedra: the geometry at this rule point
        TetGeometry tg;
        if (c < nc && !box_g_at<UGK>(P, geo, q, tg, fl)) {
          report_error(P.error, 3);
          for (int b = 0; b < 6; ++b) tg.g[b] = __longlong_as_double(0x7ff8000000000000ll);
        } else if (c >= nc) {
          for (int b = 0; b < 6; ++b) tg.g[b] = 0.0;
        }
        for (int b = 0; b < 6; ++b) gbox[b] = tg.g[b];
        gsrc = gbox;
      }
      for (int s = 0; s < nd; ++s) {
        double t1 = 0.0;
        if (poisson) {
          #pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int gi = s <= t ? (s * (5 - s)) / 2 + t : (t * (5 - t)) / 2 + s;  // upper-tri index
            t1 = ug_add<UGK>(t1, ug_mul<UGK>(gsrc[gi], wt[t], P.ug, fl), P.ug, fl);
          }
        } else {
          t1 = ug_add<UGK>(t1, ug_mul<UGK>(gsrc[0], wt[0], P.ug, fl), P.ug, fl);
        }
        double m1 = ug_mul<UGK>(om, t1, P.ug, fl);
        if (have_z) m1 = ug_mul<UGK>(m1, zq, P.ug, fl);
        const double r = c < nc ? dround_fast(m1, P.us, fl) : 0.0;
        sR[size_t(s * nq + q) * C + c] = T(r);
      }
    }
    __syncthreads();

    // -- v = b_cat_action r at u_q: output i, CB cells per thread, (s, q) ascending
    if (poisson) v_stage<A, FTZ, FMA, 2>(P, sR, tabC, C, c0, nc, fl);
    else v_stage<A, FTZ, FMA, 1>(P, sR, tabC, C, c0, nc, fl);
    __syncthreads();
  }
  publish_flags(P.flags, fl);
}

// Host launcher (launch_action.cu): picks the arithmetic instantiation and the tile.
// Returns 0, 2 (the tile does not fit shared memory) or 4 (attribute/launch failure).
int launch_action(int ap, int aq, const ActionParams& P, int sm_count, cudaStream_t st);

}  // namespace mpfem_b200
