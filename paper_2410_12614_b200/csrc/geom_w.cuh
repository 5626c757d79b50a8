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

// Two phases per CTA of kGeomCells cells:
//  (1) one thread per cell: geometry at u_g into shared memory (G, origin, edges);
//  (2) one warp per cell, lanes over quadrature points: coefficient + W row.
// UG / US are compile-time so the emulated rounding folds to the plain op for fp64 and a
// single conversion for fp32.
constexpr int kGeomCells = 64;     // cells per CTA
constexpr int kGeomThreads = 256;  // 8 warps share the (cell, q) expansion

template <typename T, int UG, int US>
__global__ void __launch_bounds__(kGeomThreads, 3) geom_w_kernel(GeomWParams P) {
  __shared__ double sG[kGeomCells][6];
  __shared__ double sV0[kGeomCells][3];
  __shared__ double sE[kGeomCells][9];
  __shared__ int sBad[kGeomCells];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t cell0 = int64_t(blockIdx.x) * kGeomCells;
  uint32_t fl = 0;
  if (tid < kGeomCells) {
    const int64_t cell = cell0 + tid;
    sBad[tid] = 1;
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
      const bool ok = tet_geometry<UG>(v, P.poisson != 0, g, fl);
      sBad[tid] = ok ? 0 : 2;
      if (!ok) atomicExch(P.error, 3);
      #pragma unroll
      for (int b = 0; b < 6; ++b) sG[tid][b] = g.g[b];
      #pragma unroll
      for (int a = 0; a < 3; ++a) {
        sV0[tid][a] = v[0][a];
        #pragma unroll
        for (int s = 0; s < 3; ++s) sE[tid][s * 3 + a] = __dsub_rn(v[s + 1][a], v[0][a]);
      }
    }
  }
  __syncthreads();
  const int nb = P.poisson ? 6 : 1;
  StoreFlags sf;
  for (int j = warp; j < kGeomCells; j += kGeomThreads / 32) {
    const int64_t cell = cell0 + j;
    if (cell >= P.n_cells || sBad[j]) continue;
    const int64_t row = cell * P.k_pad;
    const double* coef = P.coef ? P.coef + cell * P.coef_stride : nullptr;
    double G[6];
    #pragma unroll
    for (int b = 0; b < 6; ++b) G[b] = sG[j][b];
    const int nq = P.n_q;
    for (int q = lane; q < P.n_q; q += 32) {
      const double* xi = P.rule_x + 3 * q;
      double zq = 1.0;
      bool have_z = true;
      switch (P.coef_kind) {
        case 1: zq = droundT<UG>(coef_sincosexp_e(sV0[j], sE[j], xi), fl); break;
        case 2: zq = droundT<UG>(coef_exp10_affine(coef, xi), fl); break;
        case 3: {
          double acc = 0.0;
          for (int k = 0; k < P.n_phi; ++k)
            acc = dadd(acc, dmul(dround(coef[k], P.up, fl), P.tab_up[int64_t(k) * P.n_q + q], P.up, fl),
                       P.up, fl);
          zq = droundT<UG>(acc, fl);
          break;
        }
        default: have_z = false;
      }
      const double omega = P.rule_w[q];  // already rounded to u_g on the host
      T* wrow = static_cast<T*>(P.W) + row + q;
      // C_stq = round_us(round_ug(round_ug(omega G_st) zhat_q))  (kernels.cpp:189-192).
      if constexpr (UG == kFP32) {
        // fp32 operands: the hardware fp32 product is the correctly rounded binary64 one
        const float om = float(omega), zf = float(zq);
        #pragma unroll
        for (int b = 0; b < 6; ++b) {
          if (b < nb) {
            float val = __fmul_rn(om, float(G[b]));
            if (have_z) val = __fmul_rn(val, zf);
            wrow[b * nq] = to_storage<T, US>(val, sf);
          }
        }
      } else if constexpr (UG == kFP64) {
        #pragma unroll
        for (int b = 0; b < 6; ++b) {
          if (b < nb) {
            double val = __dmul_rn(omega, G[b]);
            if (have_z) val = __dmul_rn(val, zq);
            wrow[b * nq] = to_storage<T, US>(val, sf);
          }
        }
      } else {
        #pragma unroll
        for (int b = 0; b < 6; ++b) {
          if (b < nb) {
            double val = droundT<UG>(__dmul_rn(omega, G[b]), fl);
            if (have_z) val = droundT<UG>(__dmul_rn(val, zq), fl);
            wrow[b * nq] = to_storage<T, US>(val, sf);
          }
        }
      }
    }
    for (int64_t k = int64_t(nb) * P.n_q + lane; k < P.k_pad; k += 32) store_w<T>(P.W, row + k, 0.0);
  }
  fl |= store_flags_bits(sf);
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (lane == 0 && fl) atomicOr(P.flags, fl);
}

// Shared basis-product operand T from the fp64 tabulation B (n_d x n_phi x n_q):
//   T[(b,q), (i,j)] = round_us(B_s[i,q] B_t[j,q] (+ B_t[i,q] B_s[j,q] if s<t)).
// transposed != 0 stores Tt[o][k] (K contiguous; the tcgen05 A operand), else T[k][o].
template <typename T>
__global__ void build_t_kernel(const double* B, int n_phi, int n_q, int poisson, int us,
                               int64_t k_len, int64_t k_pad, int64_t n_out, int64_t n_out_pad,
                               int transposed, void* out) {
  const int64_t total = k_pad * n_out_pad;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t k, o;
    if (transposed) { o = idx / k_pad; k = idx % k_pad; }
    else { k = idx / n_out_pad; o = idx % n_out_pad; }
    double val = 0.0;
    if (k < k_len && o < n_out) {
      int b = int(k / n_q), q = int(k % n_q);
      int i = int(o / n_phi), j = int(o % n_phi);
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
