// cellmat_fused.cuh -- small-degree fused path (p = 1 mass/Poisson, p = 2 mass).
//
// For these degrees the GEMM depth K = n_blocks * n_q is 8..48 and a cell matrix has
// 16..100 entries: a cell's whole computation fits one thread's registers, and
// materialising W (and padding its rows to a 64-wide TMA box) would move several times
// more bytes than the output. One thread per cell therefore runs the complete hot path:
//   geometry at u_g (tet_geometry, bit-identical to cell_geometry) ->
//   for each quadrature point q: coefficient, W_(b,q) = round_us(round_ug(round_ug(omega G_b) z))
//   (bit-identical to build_C), A_o += W_(b,q) T[(b,q), o] with FFMA in fp32 (u_q = fp32)
//   -> 16-byte stores of the cell's row-major matrix.
// T (the shared basis products, rounded to u_s) lives in shared memory and is read as a
// broadcast (every thread reads the same T[k, o]). HBM traffic is 96 B in + 4 n_phi^2 B
// out per cell: the path's algorithmic bytes.
// Only the upper triangle (i <= j) is accumulated: T[k, (i, j)] and T[k, (j, i)] are the same
// bits (B_s[i] B_t[j] + B_t[i] B_s[j] is symmetric in (i, j)) and both entries would run the same
// fmaf sequence, so A[j, i] is A[i, j] bit for bit; the mirror happens at the store.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "device_fp.cuh"
#include "geom_w.cuh"

namespace mpfem_b200 {

struct FusedParams {
  const double* verts;
  const int32_t* cells;
  int64_t n_cells;
  int coef_kind;
  const double* coef;
  int64_t coef_stride;
  const double* rule_w_ug;  // n_q, rounded to u_g
  const double* rule_x;     // n_q x 3
  const double* tab_up;     // n_phi x n_q (nodal coefficient path)
  const float* T;           // K x n_out (fp32 carriers of u_s values)
  int us, up;
  float* out;
  int64_t out_pitch;
  uint32_t* flags;
  int* error;
};

template <int US>
__device__ __forceinline__ float round_storage_f(double v, StoreFlags& sf) {
  if constexpr (US == kFP16) return __half2float(to_storage<__half, kFP16>(v, sf));
  else if constexpr (US == kBF16) return __bfloat162float(to_storage<__nv_bfloat16, kBF16>(v, sf));
  else return to_storage<float, kFP32>(v, sf);
}

template <int P, int FORM, int UG, int US, int COEF>
__global__ void __launch_bounds__(128) cellmat_fused_kernel(FusedParams F) {
  constexpr int NPHI = (P + 1) * (P + 2) * (P + 3) / 6;
  constexpr int NQ = (P + 1) * (P + 1) * (P + 1);
  constexpr int NB = FORM ? 6 : 1;
  constexpr int K = NB * NQ;
  constexpr int NOUT = NPHI * NPHI;
  constexpr int NU = NPHI * (NPHI + 1) / 2;  // upper triangle, u(i, j) = i NPHI - i (i - 1) / 2 + j - i
  constexpr int NUP = (NU + 3) / 4 * 4;      // padded to whole float4
  __shared__ __align__(16) float sT[K * NUP];
  __shared__ double sW[NQ], sX[NQ * 3];
  for (int idx = threadIdx.x; idx < K * NUP; idx += blockDim.x) {
    const int k = idx / NUP, u = idx - k * NUP;
    float t = 0.0f;
    if (u < NU) {
      int i = 0, rem = u;
      while (rem >= NPHI - i) {
        rem -= NPHI - i;
        ++i;
      }
      t = F.T[k * NOUT + i * NPHI + i + rem];
    }
    sT[idx] = t;
  }
  for (int i = threadIdx.x; i < NQ; i += blockDim.x) sW[i] = F.rule_w_ug[i];
  for (int i = threadIdx.x; i < NQ * 3; i += blockDim.x) sX[i] = F.rule_x[i];
  __syncthreads();
  const int64_t cell = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t fl = 0;
  StoreFlags sf;
  if (cell < F.n_cells) {
    double v[4][3];
    if (F.cells) {
      #pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t vid = F.cells[cell * 4 + k];
        #pragma unroll
        for (int a = 0; a < 3; ++a) v[k][a] = F.verts[vid * 3 + a];
      }
    } else {
      const double2* src = reinterpret_cast<const double2*>(F.verts + cell * 12);
      double flat[12];
      #pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double2 t = __ldg(src + k);
        flat[2 * k] = t.x;
        flat[2 * k + 1] = t.y;
      }
      #pragma unroll
      for (int k = 0; k < 4; ++k)
        #pragma unroll
        for (int a = 0; a < 3; ++a) v[k][a] = flat[k * 3 + a];
    }
    TetGeometry g;
    if (!tet_geometry<UG>(v, FORM != 0, g, fl)) {
      report_error(F.error, 3);  // singular cell: NaN row (CheckError reported by the host)
      float* dst = F.out + cell * F.out_pitch;
      for (int o = 0; o < NOUT; ++o) dst[o] = __int_as_float(0x7fc00000);
    } else {
      double v0[3], E[9];  // x, y pre-doubled (coef_sincosexp_*)
      #pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double sc = a < 2 ? 2.0 : 1.0;
        v0[a] = sc * v[0][a];
        #pragma unroll
        for (int s = 0; s < 3; ++s) E[s * 3 + a] = sc * __dsub_rn(v[s + 1][a], v[0][a]);
      }
      const double* zc = F.coef ? F.coef + cell * F.coef_stride : nullptr;
      float acc[NUP];
      #pragma unroll
      for (int o = 0; o < NUP; ++o) acc[o] = 0.0f;
      // depth loop q-outer: W_(b,q) is generated and consumed immediately
      #pragma unroll 1
      for (int q = 0; q < NQ; ++q) {
        double zq = 1.0;
        const double* xi = sX + 3 * q;
        if constexpr (COEF == 1) {
          if constexpr (UG == kFP32) zq = double(coef_sincosexp_f(v0, E, xi));
          else zq = droundT<UG>(coef_sincosexp_e(v0, E, xi), fl);
        } else if constexpr (COEF == 2) {
          zq = droundT<UG>(coef_exp10_affine(zc, xi), fl);
        } else if constexpr (COEF == 3) {
          double a2 = 0.0;
          for (int k = 0; k < NPHI; ++k)
            a2 = dadd(a2, dmul(dround(zc[k], F.up, fl), F.tab_up[k * NQ + q], F.up, fl), F.up, fl);
          zq = droundT<UG>(a2, fl);
        }
        #pragma unroll
        for (int b = 0; b < NB; ++b) {
          double val;
          if constexpr (UG == kFP32) {
            float t = __fmul_rn(float(sW[q]), float(g.g[b]));
            if constexpr (COEF != 0) t = __fmul_rn(t, float(zq));
            val = t;
          } else {
            val = droundT<UG>(__dmul_rn(sW[q], g.g[b]), fl);
            if constexpr (COEF != 0) val = droundT<UG>(__dmul_rn(val, zq), fl);
          }
          const float wk = round_storage_f<US>(val, sf);
          const float4* trow = reinterpret_cast<const float4*>(sT + (b * NQ + q) * NUP);
          #pragma unroll
          for (int o4 = 0; o4 < NUP / 4; ++o4) {
            const float4 t = trow[o4];
            acc[4 * o4 + 0] = fmaf(wk, t.x, acc[4 * o4 + 0]);
            acc[4 * o4 + 1] = fmaf(wk, t.y, acc[4 * o4 + 1]);
            acc[4 * o4 + 2] = fmaf(wk, t.z, acc[4 * o4 + 2]);
            acc[4 * o4 + 3] = fmaf(wk, t.w, acc[4 * o4 + 3]);
          }
        }
      }
      uint32_t bad = 0;
      #pragma unroll
      for (int o = 0; o < NU; ++o) bad |= (__float_as_uint(acc[o]) & 0x7f800000u) == 0x7f800000u;
      if (bad) fl |= kInvalid;
      // entry o = i NPHI + j of the row-major matrix from the upper triangle (indices are
      // compile-time after unrolling: registers stay statically addressed)
      auto full = [&](int o) -> float {
        const int i = o / NPHI, j = o - i * NPHI;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        return acc[lo * NPHI - lo * (lo - 1) / 2 + hi - lo];
      };
      float* dst = F.out + cell * F.out_pitch;
      if ((F.out_pitch & 3) == 0) {
        #pragma unroll
        for (int o4 = 0; o4 < NOUT / 4; ++o4)
          __stcs(reinterpret_cast<float4*>(dst) + o4,
                 make_float4(full(4 * o4), full(4 * o4 + 1), full(4 * o4 + 2), full(4 * o4 + 3)));
      } else {
        #pragma unroll
        for (int o = 0; o < NOUT; ++o) __stcs(dst + o, full(o));
      }
    }
  }
  publish_flags(F.flags, fl | store_flags_bits(sf));
}

}  // namespace mpfem_b200
