// geom_w.cuh -- K1: per-cell geometry + coefficient + scaled-weight pass.
//
// Geometry once per cell (one thread), then one warp per cell whose lanes stride over
// quadrature points and write the cell's row of the GEMM operand W:
//   W[c, b*n_q + q] = round_us(round_ug(round_ug(omega_q * G_b) * zhat_q))
// which is build_C (kernels.cpp:177-197) with the (s,t) pairs packed to the upper
// triangle b = (s<=t): (0,0),(0,1),(0,2),(1,1),(1,2),(2,2) (C is symmetric bitwise, so
// the packed GEMM operand T carries B_s B_t + B_t B_s for s<t).
// zhat_q is c(x_q) rounded to u_g for analytic coefficients, or eval_z_at_ug
// (kernels.cpp:114-136) for nodal coefficients. Entries K..K_pad are zero.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "device_fp.cuh"

namespace mpfem_b200 {

// x / d for 32-bit x by multiply-high with a precomputed magic (Granlund-Montgomery):
// m = ceil(2^(32+s) / d), s = ceil(log2 d); exact for all x < 2^31.
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  __host__ __device__ uint32_t div(uint32_t x) const {
    return s == 0 && m == 0 ? x : (__umulhi_compat(x, m) + ((x - __umulhi_compat(x, m)) >> 1)) >> (s - 1);
  }
  __host__ __device__ static uint32_t __umulhi_compat(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return uint32_t((uint64_t(a) * uint64_t(b)) >> 32);
#endif
  }
  static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d;
    if (d == 1) return f;
    uint32_t s = 0;
    while ((uint64_t(1) << s) < d) ++s;
    f.s = s;
    f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1);
    return f;
  }
};

struct GeomWParams {
  const double* verts;     // private: n_cells x 12 ; mesh: vertex table n_verts x 3
  const int32_t* cells;    // NULL or n_cells x 4
  int64_t n_cells;
  int coef_kind;
  const double* coef;
  int64_t coef_stride;
  const double* rule_w;    // n_q
  const double* rule_x;    // n_q x 3
  const double* tab_up;    // n_phi x n_q basis values at u_p (nodal path)
  int n_phi, n_q, up, ug, us;
  int poisson;
  int64_t k_pad;
  FastDiv div_nq;          // idx / groups-per-cell for the (cell, q-group) expansion
  int nq_pad;              // block stride of W and T along K: round_up(n_q, 8)
  int w_type;              // 0 fp16 bits, 1 bf16 bits, 2 fp32, 3 fp64
  void* W;
  uint32_t* flags;
  int* error;              // set to 3 on a singular cell
};

// Storage rounding round_us(v) (one RNE conversion, subnormals kept) of a u_g value held
// in double or float, returned in the element type T. FP events are accumulated cheaply
// from the stored bits: `amax` tracks the largest |bits| (>= inf pattern means an
// overflow or a NaN reached storage) and `tiny` a nonzero value stored as subnormal/zero
// (underflow). For T = double (the fp64 GEMM path) any US is carried exactly.
struct StoreFlags {
  uint32_t amax = 0;  // max |bits| in units of the storage format's inf pattern
  uint32_t tiny = 0;
};

template <typename T, int US, typename V>
__device__ __forceinline__ T to_storage(V v, StoreFlags& sf) {
  if constexpr (std::is_same_v<T, __half>) {
    const __half h = std::is_same_v<V, float> ? __float2half_rn(float(v)) : __double2half(double(v));
    const uint32_t a = __half_as_ushort(h) & 0x7fffu;
    sf.amax = max(sf.amax, a >= 0x7c00u ? (a == 0x7c00u ? 1u : 2u) : 0u);
    sf.tiny |= (a < 0x0400u) & (v != V(0));
    return h;
  } else if constexpr (std::is_same_v<T, __nv_bfloat16>) {
    const __nv_bfloat16 h = std::is_same_v<V, float> ? __float2bfloat16_rn(float(v)) : __double2bfloat16(double(v));
    const uint32_t a = __bfloat16_as_ushort(h) & 0x7fffu;
    sf.amax = max(sf.amax, a >= 0x7f80u ? (a == 0x7f80u ? 1u : 2u) : 0u);
    sf.tiny |= (a < 0x0080u) & (v != V(0));
    return h;
  } else if constexpr (std::is_same_v<T, float>) {
    const float f = float(v);  // v is float already, or a double rounded once here
    const uint32_t a = __float_as_uint(f) & 0x7fffffffu;
    sf.amax = max(sf.amax, a >= 0x7f800000u ? (a == 0x7f800000u ? 1u : 2u) : 0u);
    sf.tiny |= (a < 0x00800000u) & (double(f) != double(v) || false) & (v != V(0));
    return f;
  } else {
    uint32_t dummy = 0;
    const double d = droundT<US>(double(v), dummy);
    const bool fin = isfinite(d);
    sf.amax = max(sf.amax, fin ? 0u : (isnan(d) ? 2u : 1u));
    sf.tiny |= (dummy & kUnderflow) ? 1u : 0u;
    return d;
  }
}

__device__ __forceinline__ uint32_t store_flags_bits(const StoreFlags& sf) {
  return (sf.amax == 1u ? kOverflow : 0u) | (sf.amax >= 2u ? kInvalid : 0u) | (sf.tiny ? kUnderflow : 0u);
}

template <typename T>
__device__ __forceinline__ void store_w(void* W, int64_t idx, double v);
template <>
__device__ __forceinline__ void store_w<__half>(void* W, int64_t idx, double v) {
  static_cast<__half*>(W)[idx] = __float2half_rn(__double2float_rn(v));  // exact: v is fp16
}
template <>
__device__ __forceinline__ void store_w<__nv_bfloat16>(void* W, int64_t idx, double v) {
  static_cast<__nv_bfloat16*>(W)[idx] = __float2bfloat16_rn(__double2float_rn(v));  // exact
}
template <>
__device__ __forceinline__ void store_w<float>(void* W, int64_t idx, double v) {
  static_cast<float*>(W)[idx] = __double2float_rn(v);
}
template <>
__device__ __forceinline__ void store_w<double>(void* W, int64_t idx, double v) {
  static_cast<double*>(W)[idx] = v;
}

// K1 runs as two launches:
//  (a) cell_geometry_kernel: one thread per cell, the reference's LU/inverse/tensor
//      sequence at u_g (geometry.cpp:12-118) -> CellGeo (G, origin, edges) in a scratch array;
//  (b) scaled_weights_kernel: one thread per (cell, q): coefficient z_q and the cell's
//      W entries at q for every (s<=t) block.
// UG / US are compile-time, so the emulated rounding folds to the plain op for fp64 and a
// single conversion for fp32.
struct __align__(16) CellGeo {
  double g[6];  // G_00 G_01 G_02 G_11 G_12 G_22 (poisson) or |det| (mass)
  double v0[3];
  double e[9];  // e[s*3 + i] = v_{s+1}[i] - v0[i]
};

template <int UG>
__global__ void __launch_bounds__(256) cell_geometry_kernel(GeomWParams P, CellGeo* __restrict__ geo) {
  const int64_t cell = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t fl = 0;
  if (cell < P.n_cells) {
    double v[4][3];
    if (P.cells) {
      #pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t vid = P.cells[cell * 4 + k];
        #pragma unroll
        for (int a = 0; a < 3; ++a) v[k][a] = P.verts[vid * 3 + a];
      }
    } else {
      #pragma unroll
      for (int k = 0; k < 4; ++k)
        #pragma unroll
        for (int a = 0; a < 3; ++a) v[k][a] = P.verts[cell * 12 + k * 3 + a];
    }
    TetGeometry g;
    if (!tet_geometry<UG>(v, P.poisson != 0, g, fl)) {
      atomicExch(P.error, 3);
      #pragma unroll
      for (int b = 0; b < 6; ++b) g.g[b] = 0.0;
    }
    CellGeo& o = geo[cell];
    #pragma unroll
    for (int b = 0; b < 6; ++b) o.g[b] = g.g[b];
    #pragma unroll
    for (int a = 0; a < 3; ++a) {
      o.v0[a] = v[0][a];
      #pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) o.e[s2 * 3 + a] = __dsub_rn(v[s2 + 1][a], v[0][a]);
    }
  }
  publish_flags(P.flags, fl);
}

// One thread per (cell, group of kQPT = 8 consecutive quadrature points). The W row is
// laid out in blocks of nq_pad = round_up(n_q, 8) entries (entries q >= n_q are zero, as
// are the matching rows of T), so each thread writes each block with one 16-byte store
// and the per-cell state is loaded once per 8 points.
constexpr int kQPT = 8;

template <typename T>
struct Pack8 {
  T v[8];
};

template <typename T, int UG, int US, int COEF>
__global__ void __launch_bounds__(256, 3) scaled_weights_kernel(GeomWParams P,
                                                                const CellGeo* __restrict__ geo) {
  const int nq = P.n_q;
  const int nqp = P.nq_pad;
  const int ngroups = nqp / kQPT;  // P.div_nq divides by ngroups
  const int64_t total = P.n_cells * ngroups;
  const int nb = P.poisson ? 6 : 1;
  uint32_t fl = 0;
  StoreFlags sf;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t cell32 = P.div_nq.div(uint32_t(idx));
    const int64_t cell = cell32;
    const int q0 = int(uint32_t(idx) - cell32 * uint32_t(ngroups)) * kQPT;
    CellGeo cg;  // 9 x 16-byte loads, once per 8 points
    {
      const double2* src = reinterpret_cast<const double2*>(geo + cell);
      double2* dst = reinterpret_cast<double2*>(&cg);
      #pragma unroll
      for (int k = 0; k < 9; ++k) dst[k] = __ldg(src + k);
    }
    const double* coef = P.coef ? P.coef + cell * P.coef_stride : nullptr;
    double zq[kQPT], om[kQPT];
    #pragma unroll
    for (int j = 0; j < kQPT; ++j) {
      const int q = q0 + j;
      zq[j] = 1.0;
      om[j] = 0.0;  // padding points (q >= n_q) produce exact zeros
      if (q < nq) {
        om[j] = P.rule_w[q];  // already rounded to u_g on the host
        const double* xi = P.rule_x + 3 * q;
        if constexpr (COEF == 1 && UG == kFP32) {
          zq[j] = double(coef_sincosexp_f(cg.v0, cg.e, xi));
        } else if constexpr (COEF == 1) {
          zq[j] = droundT<UG>(coef_sincosexp_e(cg.v0, cg.e, xi), fl);
        } else if constexpr (COEF == 2) {
          zq[j] = droundT<UG>(coef_exp10_affine(coef, xi), fl);
        } else if constexpr (COEF == 3) {
          double acc = 0.0;
          for (int k = 0; k < P.n_phi; ++k)
            acc = dadd(acc, dmul(dround(coef[k], P.up, fl), P.tab_up[int64_t(k) * nq + q], P.up, fl), P.up, fl);
          zq[j] = droundT<UG>(acc, fl);
        }
      }
    }
    constexpr bool have_z = COEF != 0;
    T* wrow = static_cast<T*>(P.W) + cell * P.k_pad + q0;
    // C_stq = round_us(round_ug(round_ug(omega G_st) zhat_q))  (kernels.cpp:189-192)
    #pragma unroll
    for (int b = 0; b < 6; ++b) {
      if (b < nb) {
        Pack8<T> pk;
        #pragma unroll
        for (int j = 0; j < kQPT; ++j) {
          if constexpr (UG == kFP32) {
            float val = __fmul_rn(float(om[j]), float(cg.g[b]));  // fp32 values: exact-then-round
            if (have_z) val = __fmul_rn(val, float(zq[j]));
            pk.v[j] = to_storage<T, US>(val, sf);
          } else if constexpr (UG == kFP64) {
            double val = __dmul_rn(om[j], cg.g[b]);
            if (have_z) val = __dmul_rn(val, zq[j]);
            pk.v[j] = to_storage<T, US>(val, sf);
          } else {
            double val = droundT<UG>(__dmul_rn(om[j], cg.g[b]), fl);
            if (have_z) val = droundT<UG>(__dmul_rn(val, zq[j]), fl);
            pk.v[j] = to_storage<T, US>(val, sf);
          }
        }
        // one 16-byte store per block for 16-bit storage (2 / 4 for fp32 / fp64)
        const uint4* srcv = reinterpret_cast<const uint4*>(&pk);
        uint4* dstv = reinterpret_cast<uint4*>(wrow + int64_t(b) * nqp);
        #pragma unroll
        for (int k = 0; k < int(sizeof(Pack8<T>) / 16); ++k) dstv[k] = srcv[k];
      }
    }
    // tail K..K_pad of the row: zeros (the group that owns the last block's start writes it)
    if (q0 == 0) {
      T* tail = static_cast<T*>(P.W) + cell * P.k_pad;
      for (int64_t k = int64_t(nb) * nqp; k < P.k_pad; ++k) tail[k] = T(0.0f);
    }
  }
  publish_flags(P.flags, fl | store_flags_bits(sf));
}

// Shared basis-product operand T from the fp64 tabulation B (n_d x n_phi x n_q):
//   T[(b,q), (i,j)] = round_us(B_s[i,q] B_t[j,q] (+ B_t[i,q] B_s[j,q] if s<t)).
// transposed != 0 stores Tt[o][k] (K contiguous; the tcgen05 A operand), else T[k][o].
// rows: optional output-row table (tcgen05 path): row o computes entry (i, j) =
// (rows[o] & 0xffff, rows[o] >> 16), or nothing when rows[o] < 0; NULL means o = i*n_phi + j.
template <typename T>
__global__ void build_t_kernel(const double* B, int n_phi, int n_q, int nq_pad, int poisson, int us,
                               int64_t k_len, int64_t k_pad, int64_t n_out, int64_t n_out_pad,
                               int transposed, void* out, const int32_t* rows = nullptr) {
  const int64_t total = k_pad * n_out_pad;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t k, o;
    if (transposed) { o = idx / k_pad; k = idx % k_pad; }
    else { k = idx / n_out_pad; o = idx % n_out_pad; }
    double val = 0.0;
    const int b = int(k / nq_pad), q = int(k % nq_pad);
    int i = int(o / n_phi), j = int(o % n_phi);
    bool valid = o < n_out;
    if (rows) {
      const int32_t e = rows[o];
      valid = e >= 0;
      i = e & 0xffff;
      j = (e >> 16) & 0x3fff;
    }
    if (k < k_len && valid && q < n_q) {
      int s = 0, t = 0;
      if (poisson) {
        const int ss[6] = {0, 0, 0, 1, 1, 2}, tt[6] = {0, 1, 2, 1, 2, 2};
        s = ss[b];
        t = tt[b];
      }
      const double bsi = B[(int64_t(s) * n_phi + i) * n_q + q];
      const double btj = B[(int64_t(t) * n_phi + j) * n_q + q];
      val = __dmul_rn(bsi, btj);
      if (s != t) {
        const double bti = B[(int64_t(t) * n_phi + i) * n_q + q];
        const double bsj = B[(int64_t(s) * n_phi + j) * n_q + q];
        val = __dadd_rn(val, __dmul_rn(bti, bsj));
      }
      uint32_t fl = 0;
      val = dround(val, us, fl);
    }
    store_w<T>(out, idx, val);
  }
}

}  // namespace mpfem_b200
