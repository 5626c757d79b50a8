// device_fp.cuh -- reduced-precision arithmetic on the device, bit-identical to the
// reference's emulation (softfloat.hpp:72-216): every op is computed once in binary64
// (explicit _rn intrinsics, so nvcc cannot contract into FMA) and rounded once to the
// target format. For t <= 25 significand bits the binary64 intermediate cannot cause a
// double-rounding error (2t + 2 <= 53), which is the reference's own argument.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <type_traits>

namespace mpfem_b200 {

// A CheckError found on the device (3: singular cell, geometry.cpp:42). `error` points at
// host-mapped pinned memory owned by the setup, so the host sees it without a device copy
// and reports it on the setup's next call or its synchronize (the reference throws
// synchronously; an asynchronous stream can only defer). Every writer stores the same code.
__device__ __forceinline__ void report_error(int* error, int code) {
  *reinterpret_cast<volatile int*>(error) = code;
}

enum Fmt : int { kBF16 = 0, kFP16 = 1, kFP32 = 2, kFP64 = 3 };
enum FlagBits : uint32_t { kOverflow = 1u, kUnderflow = 2u, kInvalid = 4u, kDivzero = 8u };

struct FmtParams {
  int drop;           // 53 - t
  double min_normal;  // 2^e_min
  double inv_min_sub; // 1 / (2^(e_min + 1 - t)), a power of two
  double min_sub;
  double max_finite;
};

__host__ __device__ inline FmtParams fmt_params(int f) {
  switch (f) {
    case kBF16: return {45, 0x1.0p-126, 0x1.0p133, 0x1.0p-133, 0x1.fep127};
    case kFP16: return {42, 0x1.0p-14, 0x1.0p24, 0x1.0p-24, 65504.0};
    default:    return {29, 0x1.0p-126, 0x1.0p149, 0x1.0p-149, 0x1.fffffep127};
  }
}

__device__ __forceinline__ double canonical_nan_d() {
  return __longlong_as_double(0x7ff8000000000000ll);
}

// round_to(x, f) with SubnormalPolicy::supported (softfloat.hpp:147-157).
__device__ __forceinline__ double dround(double x, int f, uint32_t& fl) {
  if (f == kFP64) {
    if (isnan(x)) { fl |= kInvalid; return canonical_nan_d(); }
    return x;
  }
  if (f == kFP32) {
    float g = __double2float_rn(x);
    if (isnan(g)) { fl |= kInvalid; return canonical_nan_d(); }
    if (isinf(g)) { if (!isinf(x)) fl |= kOverflow; return (double)g; }
    if (x != 0.0 && fabs(x) < 0x1.0p-126 && (double)g != x) fl |= kUnderflow;
    return (double)g;
  }
  const FmtParams fp = fmt_params(f);
  unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  unsigned long long mag = bits & 0x7fffffffffffffffull;
  if (mag >= 0x7ff0000000000000ull) {
    if (mag > 0x7ff0000000000000ull) { fl |= kInvalid; return canonical_nan_d(); }
    return x;
  }
  if (mag == 0) return x;
  double ax = __longlong_as_double((long long)mag);
  if (ax < fp.min_normal) {
    double q = __dmul_rn(rint(__dmul_rn(ax, fp.inv_min_sub)), fp.min_sub);
    double r = copysign(q, x);
    if (r != x) fl |= kUnderflow;
    return r;
  }
  unsigned long long mask = (1ull << fp.drop) - 1ull;
  unsigned long long rem = bits & mask;
  unsigned long long half = 1ull << (fp.drop - 1);
  bits &= ~mask;
  if (rem > half || (rem == half && (bits & (1ull << fp.drop)))) bits += 1ull << fp.drop;
  double r = __longlong_as_double((long long)bits);
  if (fabs(r) > fp.max_finite) { fl |= kOverflow; return copysign(__longlong_as_double(0x7ff0000000000000ll), x); }
  return r;
}

// Publishes a warp's FP flags: one lane, and only the bits not yet visible, so that
// thousands of warps raising the same flag do not serialise on one L2 address.
__device__ __forceinline__ void publish_flags(uint32_t* flags, uint32_t fl) {
  fl = __reduce_or_sync(0xffffffffu, fl);
  if ((threadIdx.x & 31) == 0 && fl) {
    const uint32_t seen = *reinterpret_cast<volatile uint32_t*>(flags);
    if (fl & ~seen) atomicOr(flags, fl);
  }
}

// Compile-time-format rounding: identical results to dround(x, F, fl), but the format
// dispatch folds away (fp64 is the identity, fp32 a single conversion).
template <int F>
__device__ __forceinline__ double droundT(double x, uint32_t& fl) {
  if constexpr (F == kFP64) {
    if (isnan(x)) { fl |= kInvalid; return canonical_nan_d(); }
    return x;
  } else if constexpr (F == kFP32) {
    return dround(x, F, fl);
  } else if constexpr (F == kFP16) {
    // cvt.rn.f16.f64: one RNE rounding, subnormals included (== round_narrow)
    if (isnan(x)) { fl |= kInvalid; return canonical_nan_d(); }
    const double r = __half2float(__double2half(x));
    if (isinf(r) && !isinf(x)) fl |= kOverflow;
    if (fabs(r) < 0x1.0p-14 && r != x) fl |= kUnderflow;
    return r;
  } else {
    // cvt.rn.bf16.f64 (sm_90+): one RNE rounding
    if (isnan(x)) { fl |= kInvalid; return canonical_nan_d(); }
    const double r = __bfloat162float(__double2bfloat16(x));
    if (isinf(r) && !isinf(x)) fl |= kOverflow;
    if (fabs(r) < 0x1.0p-126 && r != x) fl |= kUnderflow;
    return r;
  }
}
template <int F>
__device__ __forceinline__ double daddT(double a, double b, uint32_t& fl) {
  double r = __dadd_rn(a, b);
  if constexpr (F == kFP64) {
    if (isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  }
  return droundT<F>(r, fl);
}
template <int F>
__device__ __forceinline__ double dsubT(double a, double b, uint32_t& fl) {
  double r = __dsub_rn(a, b);
  if constexpr (F == kFP64) {
    if (isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  }
  return droundT<F>(r, fl);
}
template <int F>
__device__ __forceinline__ double ddivT(double a, double b, uint32_t& fl) {
  if (b == 0.0 && a != 0.0 && !isnan(a) && !isinf(a)) fl |= kDivzero;
  double r = __ddiv_rn(a, b);
  if constexpr (F == kFP64) {
    if (isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  }
  return droundT<F>(r, fl);
}
template <int F>
__device__ __forceinline__ double dmulT(double a, double b, uint32_t& fl) {
  double r = __dmul_rn(a, b);
  if constexpr (F == kFP64) {
    if (isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  }
  return droundT<F>(r, fl);
}

// fp_op at format f (softfloat.hpp:170-186): exact binary64 op, one rounding.
__device__ __forceinline__ double dadd(double a, double b, int f, uint32_t& fl) {
  double r = __dadd_rn(a, b);
  if (f == kFP64 && isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  return dround(r, f, fl);
}
__device__ __forceinline__ double dsub(double a, double b, int f, uint32_t& fl) {
  double r = __dsub_rn(a, b);
  if (f == kFP64 && isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  return dround(r, f, fl);
}
__device__ __forceinline__ double dmul(double a, double b, int f, uint32_t& fl) {
  double r = __dmul_rn(a, b);
  if (f == kFP64 && isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  return dround(r, f, fl);
}
__device__ __forceinline__ double ddiv(double a, double b, int f, uint32_t& fl) {
  if (b == 0.0 && a != 0.0 && !isnan(a) && !isinf(a)) fl |= kDivzero;
  double r = __ddiv_rn(a, b);
  if (f == kFP64 && isinf(r) && !isinf(a) && !isinf(b)) fl |= kOverflow;
  return dround(r, f, fl);
}

// Affine-tet geometry at format f, the exact op sequence of cell_geometry's reduced-
// precision fields (geometry.cpp:12-118): J through the P1 basis gradients at the
// centroid (-1,-1,-1 / e_s, exact), LU with partial pivoting, det, inverse by three
// solves, geometry tensor upper triangle mirrored. Returns false on an exact zero pivot.
struct TetGeometry {
  double det, abs_det;
  double g[6];  // G_00 G_01 G_02 G_11 G_12 G_22 (poisson); g[0] = |det| (mass)
};

__device__ __forceinline__ bool tet_geometry_f32(const double v[4][3], bool poisson, TetGeometry& out,
                                                 uint32_t& fl);

template <int F>
__device__ __noinline__ bool tet_geometry_flagged(const double v[4][3], bool poisson, TetGeometry& out,
                                                     uint32_t& fl);
__device__ __forceinline__ bool tet_geometry_f64_fast(const double v[4][3], bool poisson, TetGeometry& out,
                                                      uint32_t& hmax);

// u_g = fp64 runs the op sequence with plain IEEE binary64 ops (bitwise the same values:
// every emulated op at fp64 is the hardware op) and only tracks the largest |high word| of
// the inputs and every intermediate; FP events at fp64 need a non-finite value somewhere
// (overflow, invalid) or a zero pivot, and in that rare case the flagged sequence reruns
// to produce the reference's flags exactly.
template <int F>
__device__ __forceinline__ bool tet_geometry(const double v[4][3], bool poisson, TetGeometry& out,
                                             uint32_t& fl) {
  if constexpr (F == kFP32) {
    return tet_geometry_f32(v, poisson, out, fl);
  } else if constexpr (F == kFP64) {
    uint32_t hmax = 0;
    const bool ok = tet_geometry_f64_fast(v, poisson, out, hmax);
    if (ok && hmax < 0x7ff00000u) return true;
    return tet_geometry_flagged<F>(v, poisson, out, fl);
  } else {
    return tet_geometry_flagged<F>(v, poisson, out, fl);
  }
}

__device__ __forceinline__ void track_hi(double r, uint32_t& hmax) {
  hmax = max(hmax, uint32_t(__double2hiint(r)) & 0x7fffffffu);
}

__device__ __forceinline__ bool tet_geometry_f64_fast(const double v[4][3], bool poisson, TetGeometry& out,
                                                      uint32_t& hmax) {
  double jac[3][3];
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) jac[i][s] = 0.0;
  #pragma unroll
  for (int k = 0; k < 4; ++k) {
    #pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double x = v[k][i];
      track_hi(x, hmax);
      #pragma unroll
      for (int s = 0; s < 3; ++s) {
        const double g = (k == 0) ? -1.0 : ((k - 1 == s) ? 1.0 : 0.0);
        jac[i][s] = __dadd_rn(jac[i][s], __dmul_rn(x, g));
        track_hi(jac[i][s], hmax);
      }
    }
  }
  double lu[3][3];
  int perm[3] = {0, 1, 2};
  int sign = 1;
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) lu[i][s] = jac[i][s];
  #pragma unroll
  for (int col = 0; col < 3; ++col) {
    int pivot = col;
    double best = fabs(lu[col][col]);
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      const double a = fabs(lu[r][col]);
      if (a > best) { best = a; pivot = r; }
    }
    double pv = lu[col][col];
    #pragma unroll
    for (int r = col + 1; r < 3; ++r)
      if (pivot == r) pv = lu[r][col];
    if (pv == 0.0) return false;
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      if (pivot == r) {
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
          double t = lu[r][c];
          lu[r][c] = lu[col][c];
          lu[col][c] = t;
        }
        int t = perm[r];
        perm[r] = perm[col];
        perm[col] = t;
        sign = -sign;
      }
    }
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      const double m = __ddiv_rn(lu[r][col], lu[col][col]);
      track_hi(m, hmax);
      lu[r][col] = m;
      #pragma unroll
      for (int c = col + 1; c < 3; ++c) {
        lu[r][c] = __dsub_rn(lu[r][c], __dmul_rn(m, lu[col][c]));
        track_hi(lu[r][c], hmax);
      }
    }
  }
  double det = (double)sign;
  #pragma unroll
  for (int i = 0; i < 3; ++i) det = __dmul_rn(det, lu[i][i]);
  track_hi(det, hmax);
  out.det = det;
  out.abs_det = fabs(det);
  if (!poisson) {
    out.g[0] = out.abs_det;
    return true;
  }
  double inv[3][3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    double y[3];
    #pragma unroll
    for (int r = 0; r < 3; ++r) {
      double s = perm[r] == k ? 1.0 : 0.0;
      #pragma unroll
      for (int c = 0; c < r; ++c) s = __dsub_rn(s, __dmul_rn(lu[r][c], y[c]));
      track_hi(s, hmax);
      y[r] = s;
    }
    #pragma unroll
    for (int r = 2; r >= 0; --r) {
      double s = y[r];
      #pragma unroll
      for (int c = r + 1; c < 3; ++c) s = __dsub_rn(s, __dmul_rn(lu[r][c], inv[c][k]));
      inv[r][k] = __ddiv_rn(s, lu[r][r]);
      track_hi(inv[r][k], hmax);
    }
  }
  int idx = 0;
  #pragma unroll
  for (int s = 0; s < 3; ++s)
    #pragma unroll
    for (int t = s; t < 3; ++t) {
      double dot = 0.0;
      #pragma unroll
      for (int k = 0; k < 3; ++k) dot = __dadd_rn(dot, __dmul_rn(inv[s][k], inv[t][k]));
      out.g[idx] = __dmul_rn(out.abs_det, dot);
      track_hi(out.g[idx], hmax);
      ++idx;
    }
  return true;
}

// LU, det, inverse and geometry tensor at format F from a Jacobian (geometry.cpp:29-118):
// shared by affine tets (J from the P1 gradients) and boxes (J at every rule point).
template <int F>
__device__ __noinline__ bool jac_geometry_flagged(const double jac[3][3], bool poisson,
                                                     TetGeometry& out, uint32_t& fl) {
  // lu_decompose (geometry.cpp:33-57)
  double lu[3][3];
  int perm[3] = {0, 1, 2};
  int sign = 1;
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) lu[i][s] = jac[i][s];
  #pragma unroll
  for (int col = 0; col < 3; ++col) {
    int pivot = col;
    double best = fabs(lu[col][col]);
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      const double a = fabs(lu[r][col]);
      if (a > best) { best = a; pivot = r; }
    }
    // first max wins (strict >), as lu_decompose; swaps with static indices only so the
    // 3x3 factors stay in registers
    double pv = lu[col][col];
    #pragma unroll
    for (int r = col + 1; r < 3; ++r)
      if (pivot == r) pv = lu[r][col];
    if (pv == 0.0) return false;
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      if (pivot == r) {
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
          double t = lu[r][c];
          lu[r][c] = lu[col][c];
          lu[col][c] = t;
        }
        int t = perm[r];
        perm[r] = perm[col];
        perm[col] = t;
        sign = -sign;
      }
    }
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      double m = ddivT<F>(lu[r][col], lu[col][col], fl);
      lu[r][col] = m;
      #pragma unroll
      for (int c = col + 1; c < 3; ++c) lu[r][c] = dsubT<F>(lu[r][c], dmulT<F>(m, lu[col][c], fl), fl);
    }
  }
  double det = (double)sign;
  #pragma unroll
  for (int i = 0; i < 3; ++i) det = dmulT<F>(det, lu[i][i], fl);
  out.det = det;
  out.abs_det = fabs(det);
  if (!poisson) {
    out.g[0] = out.abs_det;
    return true;
  }
  // inverse_lu (geometry.cpp:70-95); the LU is recomputed there but is identical.
  double inv[3][3];
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    double y[3];
    #pragma unroll
    for (int r = 0; r < 3; ++r) {
      double s = perm[r] == k ? 1.0 : 0.0;
      #pragma unroll
      for (int c = 0; c < r; ++c) s = dsubT<F>(s, dmulT<F>(lu[r][c], y[c], fl), fl);
      y[r] = s;
    }
    #pragma unroll
    for (int r = 2; r >= 0; --r) {
      double s = y[r];
      #pragma unroll
      for (int c = r + 1; c < 3; ++c) s = dsubT<F>(s, dmulT<F>(lu[r][c], inv[c][k], fl), fl);
      inv[r][k] = ddivT<F>(s, lu[r][r], fl);
    }
  }
  // geometry_tensor (geometry.cpp:97-118)
  int idx = 0;
  #pragma unroll
  for (int s = 0; s < 3; ++s)
    #pragma unroll
    for (int t = s; t < 3; ++t) {
      double dot = 0.0;
      #pragma unroll
      for (int k = 0; k < 3; ++k) dot = daddT<F>(dot, dmulT<F>(inv[s][k], inv[t][k], fl), fl);
      out.g[idx++] = dmulT<F>(out.abs_det, dot, fl);
    }
  return true;
}

template <int F>
__device__ __noinline__ bool tet_geometry_flagged(const double v[4][3], bool poisson, TetGeometry& out,
                                                     uint32_t& fl) {
  // P1 gradient signs: vertex 0 -> -1 on every axis, vertex k -> +1 on axis k-1.
  double jac[3][3];
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) jac[i][s] = 0.0;
  #pragma unroll
  for (int k = 0; k < 4; ++k) {
    #pragma unroll
    for (int i = 0; i < 3; ++i) {
      double x = droundT<F>(v[k][i], fl);
      #pragma unroll
      for (int s = 0; s < 3; ++s) {
        double g = (k == 0) ? -1.0 : ((k - 1 == s) ? 1.0 : 0.0);
        jac[i][s] = daddT<F>(jac[i][s], dmulT<F>(x, g, fl), fl);
      }
    }
  }
  return jac_geometry_flagged<F>(jac, poisson, out, fl);
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

// The input screen of the native path: x = round_ug(xd) finite and, for u_g = fp32, xd zero or
// at least the smallest fp32 normal (tiny inputs take the flagged path for exact flags).
template <int UG>
__device__ __forceinline__ bool box_input_ok(double xd) {
  if constexpr (UG == kFP32) return isfinite(float(xd)) && (xd == 0.0 || fabs(xd) >= 0x1.0p-126);
  else return isfinite(xd);
}

// Geometry of a box cell at one rule point (geometry.cpp:12-27,190-221) at u_g = UG: J from the
// 8 vertices and the u_g gradients of the degree-1 box basis at that point (gq[s][k]), then LU,
// det, inverse and G. Native _rn arithmetic for fp32 / fp64 (bitwise the emulation's values),
// the flagged emulation for other formats and rare events. False on a zero pivot.
// vx(k, i) and gq(s, k) read vertex coordinate i of vertex k and gradient component s of basis
// function k: accessors instead of arrays, so the values are loaded where they are used and the
// rare fallback reloads them (an [8][3] + [3][8] array kept live for it cost a 528-byte local
// frame per thread, or 160 registers once its loop was unrolled).
// Variant with the u_g-rounded coordinates supplied by the caller: xn(k, i) returns
// F(vx(k, i)) (F = float / double for u_g = fp32 / fp64, else unused) and in_ok says every
// input passed box_input_ok (finite after rounding, not fp32-subnormal); K1-box uses it to
// round and screen each vertex once per warp instead of once per point.
// With SCREEN the inputs are instead read, rounded and screened here (xn, in_ok unused).
template <int UG, bool SCREEN = false, class XN, class VX, class GQ>
__device__ __forceinline__ bool box_point_geometry_pre(XN xn, bool in_ok, VX vx, GQ gq, bool poisson,
                                                       TetGeometry& geo, uint32_t& fl) {
  bool done = false;
  if constexpr (UG == kFP32 || UG == kFP64) {
    using F = typename std::conditional<UG == kFP32, float, double>::type;
    using O = NativeOps<F>;
    F jn[3][3];
    #pragma unroll
    for (int i = 0; i < 3; ++i)
      #pragma unroll
      for (int s = 0; s < 3; ++s) jn[i][s] = F(0);
    #pragma unroll
    for (int k = 0; k < 8; ++k)
      #pragma unroll
      for (int i = 0; i < 3; ++i) {
        F x;
        if constexpr (SCREEN) {
          const double xd = vx(k, i);
          x = F(xd);  // one RNE rounding to u_g (exact for u_g = fp64)
          in_ok = in_ok && box_input_ok<UG>(xd);
        } else {
          x = xn(k, i);
        }
        #pragma unroll
        for (int s = 0; s < 3; ++s) jn[i][s] = O::add(jn[i][s], O::mul(x, F(gq(s, k))));
      }
    done = in_ok && box_geometry_native<F>(jn, poisson, geo);
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
        const double x = droundT<UG>(vx(k, i), fl);
        #pragma unroll
        for (int s = 0; s < 3; ++s) jac[i][s] = daddT<UG>(jac[i][s], dmulT<UG>(x, gq(s, k), fl), fl);
      }
    return jac_geometry_flagged<UG>(jac, poisson, geo, fl);
  }
  return true;
}

template <int UG, class VX, class GQ>
__device__ __forceinline__ bool box_point_geometry(VX vx, GQ gq, bool poisson, TetGeometry& geo,
                                                   uint32_t& fl) {
  auto xn = [](int, int) { return 0.0; };  // unused with SCREEN
  return box_point_geometry_pre<UG, true>(xn, true, vx, gq, poisson, geo, fl);
}

// u_g = fp32: the same op sequence in native fp32 arithmetic. IEEE fp32 +,-,*,/ are the
// correctly rounded results of the exact operations, i.e. exactly round_fp32 of the exact
// binary64 op the emulation computes (no double rounding, softfloat.hpp:12-16), so the
// values are bit-identical to tet_geometry<kFP32>; FP events are detected on the results.
__device__ __forceinline__ bool tet_geometry_f32(const double v[4][3], bool poisson, TetGeometry& out,
                                                 uint32_t& fl) {
  float x[4][3];
  #pragma unroll
  for (int k = 0; k < 4; ++k)
    #pragma unroll
    for (int i = 0; i < 3; ++i) x[k][i] = __double2float_rn(v[k][i]);
  float jac[3][3];
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) {
      // sum over k ascending of x_k * grad_k[s]: 0 + (-x0) then + x_{s+1} (others add +-0)
      float a = __fadd_rn(0.0f, __fmul_rn(x[0][i], -1.0f));
      #pragma unroll
      for (int k = 1; k < 4; ++k) a = __fadd_rn(a, __fmul_rn(x[k][i], (k - 1 == s) ? 1.0f : 0.0f));
      jac[i][s] = a;
    }
  float lu[3][3];
  int perm[3] = {0, 1, 2};
  int sign = 1;
  #pragma unroll
  for (int i = 0; i < 3; ++i)
    #pragma unroll
    for (int s = 0; s < 3; ++s) lu[i][s] = jac[i][s];
  #pragma unroll
  for (int col = 0; col < 3; ++col) {
    int pivot = col;
    float best = fabsf(lu[col][col]);
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      const float a = fabsf(lu[r][col]);
      if (a > best) { best = a; pivot = r; }
    }
    float pv = lu[col][col];
    #pragma unroll
    for (int r = col + 1; r < 3; ++r)
      if (pivot == r) pv = lu[r][col];
    if (pv == 0.0f) return false;
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      if (pivot == r) {
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float t = lu[r][c];
          lu[r][c] = lu[col][c];
          lu[col][c] = t;
        }
        const int t = perm[r];
        perm[r] = perm[col];
        perm[col] = t;
        sign = -sign;
      }
    }
    #pragma unroll
    for (int r = col + 1; r < 3; ++r) {
      const float m = __fdiv_rn(lu[r][col], lu[col][col]);
      lu[r][col] = m;
      #pragma unroll
      for (int c = col + 1; c < 3; ++c) lu[r][c] = __fsub_rn(lu[r][c], __fmul_rn(m, lu[col][c]));
    }
  }
  float det = float(sign);
  #pragma unroll
  for (int i = 0; i < 3; ++i) det = __fmul_rn(det, lu[i][i]);
  out.det = det;
  out.abs_det = fabsf(det);
  if (!poisson) {
    out.g[0] = out.abs_det;
  } else {
    float inv[3][3];
    #pragma unroll
    for (int k = 0; k < 3; ++k) {
      float y[3];
      #pragma unroll
      for (int r = 0; r < 3; ++r) {
        float s = perm[r] == k ? 1.0f : 0.0f;
        #pragma unroll
        for (int c = 0; c < r; ++c) s = __fsub_rn(s, __fmul_rn(lu[r][c], y[c]));
        y[r] = s;
      }
      #pragma unroll
      for (int r = 2; r >= 0; --r) {
        float s = y[r];
        #pragma unroll
        for (int c = r + 1; c < 3; ++c) s = __fsub_rn(s, __fmul_rn(lu[r][c], inv[c][k]));
        inv[r][k] = __fdiv_rn(s, lu[r][r]);
      }
    }
    int idx = 0;
    #pragma unroll
    for (int s = 0; s < 3; ++s)
      #pragma unroll
      for (int t = s; t < 3; ++t) {
        float dot = 0.0f;
        #pragma unroll
        for (int k = 0; k < 3; ++k) dot = __fadd_rn(dot, __fmul_rn(inv[s][k], inv[t][k]));
        const float gv = __fmul_rn(float(out.abs_det), dot);
        out.g[idx++] = gv;
        if (!isfinite(gv)) fl |= isnan(gv) ? kInvalid : kOverflow;
        if (gv != 0.0f && fabsf(gv) < 0x1.0p-126f) fl |= kUnderflow;
      }
  }
  if (!isfinite(det)) fl |= isnan(det) ? kInvalid : kOverflow;
  return true;
}

// Analytic coefficient at a quadrature point (BASELINE configs 0-2,4): x_q = v0 + J xi
// in binary64, left to right, then c = 1 + 0.5 sin(2 pi x) cos(2 pi y) e^z.
__device__ __forceinline__ double coef_sincosexp(const double v[4][3], const double* xi) {
  double x[3];
  #pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = v[0][i];
    #pragma unroll
    for (int s = 0; s < 3; ++s) acc = __dadd_rn(acc, __dmul_rn(__dsub_rn(v[s + 1][i], v[0][i]), xi[s]));
    x[i] = acc;
  }
  // sin(2 pi x) as sinpi(2x): exact argument reduction (2x is exact in binary64)
  double s = sinpi(__dmul_rn(2.0, x[0]));
  double c = cospi(__dmul_rn(2.0, x[1]));
  double e = exp(x[2]);
  return __dadd_rn(1.0, __dmul_rn(__dmul_rn(__dmul_rn(0.5, s), c), e));
}

// Branch-free binary64 transcendentals for the bounded arguments of the analytic
// coefficient (|2x| < 2^30, |z| < 700): range reduction by exact rounding, then fp64
// Horner. Measured (scripts/coef_ulp_check.c, long double references): sinpi/cospi
// <= 2.4 ulp, exp <= 0.56 ulp. The glibc/CUDA libm functions are within 1-2 ulp of the
// same values, so analytic-coefficient parity with the oracle is tolerance-based.
// Polynomial coefficients live in constant memory so DFMA reads them as constant-bank
// operands (fp64 immediates would otherwise be materialised with two UMOVs each).
// sin(pi r) = r P(r^2), |r| <= 1/2: near-minimax P of degree 8 in r^2 (Chebyshev fit in
// mpmath, scripts/fit_coef_polys.py; approximation error 2e-19 relative, below the fp64
// evaluation rounding).
__constant__ double kSinPiC[9] = {3.141592653589793, -5.167712780049969, 2.5501640398773007,
                                  -0.5992645293189447, 0.0821458865731029, -0.007370430505916944,
                                  0.0004662998161898394, -2.1903497074626018e-05, 7.697826768224191e-07};
__device__ __forceinline__ double sinpi_poly(double r) {  // sin(pi r), |r| <= 0.5
  const double s = r * r;
#ifdef MPFEM_ESTRIN  // diagnostic builds only: Estrin scheme (depth 4 instead of 8)
  const double s2 = s * s, s4 = s2 * s2;
  const double a0 = fma(kSinPiC[1], s, kSinPiC[0]), a1 = fma(kSinPiC[3], s, kSinPiC[2]);
  const double a2 = fma(kSinPiC[5], s, kSinPiC[4]), a3 = fma(kSinPiC[7], s, kSinPiC[6]);
  const double b0 = fma(a1, s2, a0), b1 = fma(a3, s2, a2);
  const double p = fma(fma(kSinPiC[8], s4, b1), s4, b0);
  return r * p;
#else
  double p = kSinPiC[8];
  #pragma unroll
  for (int k = 7; k >= 0; --k) p = fma(p, s, kSinPiC[k]);
  return r * p;
#endif
}
// Rounding to an integer without the fp64 conversion pipe (FRND / F2I run at a fraction
// of DFMA throughput): t = a + 1.5*2^52 rounds a to the nearest integer (ties to even) in
// the DADD itself for |a| < 2^51; t - 1.5*2^52 is that integer exactly and the low word of
// t holds it in two's complement.
constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52
__device__ __forceinline__ double flip_if_odd(double v, uint32_t n_lo) {
  return __hiloint2double(__double2hiint(v) ^ int((n_lo & 1u) << 31), __double2loint(v));
}
__device__ __forceinline__ double fast_sinpi(double a) {
  const double t = __dadd_rn(a, kRoundMagic);
  const double n = __dsub_rn(t, kRoundMagic);
  return flip_if_odd(sinpi_poly(__dsub_rn(a, n)), uint32_t(__double2loint(t)));
}
__device__ __forceinline__ double fast_cospi(double a) {  // cos(pi r) = sin(pi (1/2 - |r|))
  const double t = __dadd_rn(a, kRoundMagic);
  const double n = __dsub_rn(t, kRoundMagic);
  return flip_if_odd(sinpi_poly(__dsub_rn(0.5, fabs(__dsub_rn(a, n)))), uint32_t(__double2loint(t)));
}
// e^z * 2^-h (h = 0 or 1 folds a factor 1/2 into the exponent): n = rint(32 z / ln2),
// r = z - n ln2/32 (Cody-Waite, |r| <= ln2/64), e^r - 1 by degree-6 Taylor (error 3e-18),
// 2^(j/32) from a double-double table: hi + fma(hi, e^r - 1, lo). <= 0.56 ulp
// (scripts/coef_ulp_check.c). Table in global memory, read through L1 (lanes differ).
__device__ const double2 kExp2Tab[32] = {
    {1.0, 0.0}, {1.0218971486541166, 5.109225028973444e-17}, {1.0442737824274138, 8.551889705537965e-17},
    {1.0671404006768237, -7.899853966841582e-17}, {1.0905077326652577, -3.046782079812471e-17},
    {1.1143867425958924, 1.0410278456845571e-16}, {1.1387886347566916, 8.912812676025408e-17},
    {1.1637248587775775, 3.8292048369240935e-17}, {1.189207115002721, 3.982015231465646e-17},
    {1.215247359980469, -7.712630692681488e-17}, {1.241857812073484, 4.658027591836937e-17},
    {1.2690509571917332, 2.667932131342186e-18}, {1.2968395546510096, 2.5382502794888315e-17},
    {1.3252366431597413, -2.8587312100388614e-17}, {1.3542555469368927, 7.70094837980299e-17},
    {1.383909881963832, -6.770511658794786e-17}, {1.4142135623730951, -9.667293313452913e-17},
    {1.4451808069770467, -3.0237581349939873e-17}, {1.4768261459394993, -3.483994556892796e-17},
    {1.5091644275934228, -1.016455327754295e-16}, {1.5422108254079407, 7.949834809697621e-17},
    {1.5759808451078865, -1.0136916471278304e-17}, {1.6104903319492543, 2.4707192569797888e-17},
    {1.645755478153965, -1.0125679913674773e-16}, {1.681792830507429, 8.199010020581497e-17},
    {1.718619298122478, -1.851380418263111e-17}, {1.7562521603732995, 2.960140695448873e-17},
    {1.7947090750031072, 1.8227458427912087e-17}, {1.8340080864093424, 3.283107224245627e-17},
    {1.8741676341103, -6.122763413004143e-17}, {1.9152065613971474, -1.0619946056195963e-16},
    {1.9571441241754002, 8.960767791036668e-17}};
template <int H = 0>
__device__ __forceinline__ double fast_exp(double z) {
  const double t = __dadd_rn(__dmul_rn(z, 46.16624130844683), kRoundMagic);
  const double n = __dsub_rn(t, kRoundMagic);
  double r = fma(-n, 0.021660849390173098, z);  // ln2/32 hi (trailing zeros: n * hi exact)
  r = fma(-n, 2.325192846878874e-12, r);
  double q = fma(1.0 / 720, r, 1.0 / 120);
  q = fma(q, r, 1.0 / 24);
  q = fma(q, r, 1.0 / 6);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  const double p1 = q * r;  // e^r - 1
  const int ni = __double2loint(t);
  const double2 tj = __ldg(&kExp2Tab[ni & 31]);
  const double v = __dadd_rn(tj.x, fma(tj.x, p1, tj.y));
  return v * __hiloint2double(((ni >> 5) - H + 1023) << 20, 0);
}

// fp32 counterparts for u_g = fp32 (the coefficient is rounded to fp32 anyway): same
// reductions, Taylor series truncated below 2^-27; <= 1.7 ulp(fp32) against 100-bit mpmath.
__constant__ float kSinPiF[7] = {3.1415927410125732f, -5.167712688446045f, 2.550163984298706f,
                                 -0.5992645025253296f, 0.08214588463306427f, -0.00737043097615242f,
                                 0.0004663027939386666f};
__constant__ float kExpF[9] = {1.0f, 1.0f, 0.5f, 0.1666666716337204f, 0.0416666679084301f,
                               0.008333333767950535f, 0.0013888889225199819f,
                               0.00019841270113829523f, 2.4801587642286904e-05f};
__device__ __forceinline__ float sinpi_poly_f(float r) {
  const float s = r * r;
  float p = kSinPiF[6];
  #pragma unroll
  for (int k = 5; k >= 0; --k) p = fmaf(p, s, kSinPiF[k]);
  return r * p;
}
// Round-to-nearest-even of |a| < 2^22 by the 1.5 * 2^23 magic add: the FMA pipe instead of
// FRND / F2I on the conversion pipe (which K1's D2F conversions already load). The integer
// is read from the low mantissa bits of the biased sum.
__device__ __forceinline__ float magic_round_f(float a, int& ni) {
  const float big = __fadd_rn(a, 12582912.0f);
  ni = __float_as_int(big) - 0x4B400000;
  return __fsub_rn(big, 12582912.0f);
}
__device__ __forceinline__ float flip_if_odd_i(float v, int ni) {
  return __int_as_float(__float_as_int(v) ^ ((ni & 1) << 31));
}
__device__ __forceinline__ float fast_sinpi_f(float a) {
  int ni;
  const float n = magic_round_f(a, ni);
  return flip_if_odd_i(sinpi_poly_f(a - n), ni);
}
__device__ __forceinline__ float fast_cospi_f(float a) {
  int ni;
  const float n = magic_round_f(a, ni);
  return flip_if_odd_i(sinpi_poly_f(0.5f - fabsf(a - n)), ni);
}
__device__ __forceinline__ float fast_exp_f(float z) {
  int ni;
  const float n = magic_round_f(z * 1.4426950408889634f, ni);
  float r = fmaf(-n, 0.693145751953125f, z);
  r = fmaf(-n, 1.428606765330187e-06f, r);
  float p = kExpF[8];
  #pragma unroll
  for (int k = 7; k >= 0; --k) p = fmaf(p, r, kExpF[k]);
  return p * __int_as_float((ni + 127) << 23);
}

// The analytic coefficient from a cell's origin and edge vectors with the x and y components
// pre-doubled (v0d = (2 v0x, 2 v0y, v0z), Ed[s] likewise): the FMA chain then yields 2x and
// 2y exactly (scaling by 2 commutes with rounding), the sinpi/cospi arguments.
// c(x_q) with the physical point in binary64 and the transcendentals in fp32, for u_g = fp32.
__device__ __forceinline__ float coef_sincosexp_f(const double* v0d, const double* Ed, const double* xi) {
  double x[3];
  #pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = v0d[i];
    #pragma unroll
    for (int s = 0; s < 3; ++s) acc = fma(Ed[s * 3 + i], xi[s], acc);
    x[i] = acc;
  }
  const float sn = fast_sinpi_f(float(x[0]));
  const float cs = fast_cospi_f(float(x[1]));
  const float e = fast_exp_f(float(x[2]));
  return fmaf(0.5f * sn * cs, e, 1.0f);
}

// binary64: c = 1 + 0.5 sin(2 pi x) cos(2 pi y) e^z as fma(sn cs, e^z / 2, 1)
// (<= 5.3 ulp of max(1, |0.5 sn cs e^z|) against a long double reference).
__device__ __forceinline__ double coef_sincosexp_e(const double* v0d, const double* Ed,
                                                   const double* xi) {
  double x[3];
  #pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = v0d[i];
    #pragma unroll
    for (int s = 0; s < 3; ++s) acc = fma(Ed[s * 3 + i], xi[s], acc);
    x[i] = acc;
  }
  const double sn = fast_sinpi(x[0]);
  const double cs = fast_cospi(x[1]);
  return fma(__dmul_rn(sn, cs), fast_exp<1>(x[2]), 1.0);
}

// Config-3 coefficient: c = 10^(6 u(x_q)), u affine with vertex values u4.
__device__ __forceinline__ double coef_exp10_affine(const double* u4, const double* xi) {
  double l0 = __dsub_rn(__dsub_rn(__dsub_rn(1.0, xi[0]), xi[1]), xi[2]);
  double u = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(u4[0], l0), __dmul_rn(u4[1], xi[0])),
                                 __dmul_rn(u4[2], xi[1])),
                       __dmul_rn(u4[3], xi[2]));
  return pow(10.0, __dmul_rn(6.0, u));
}

}  // namespace mpfem_b200
