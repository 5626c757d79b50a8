// cellmat_simt.cuh -- K2 for the fp32 reference mode (u_q = fp32 with fp32 operands): FFMA, no
// TF32 (the mode's products and sums are fp32). Same GEMM as the tcgen05 path,
//   A[c, o] = sum_k W[c, k] * T[k, o],   k ascending, one fma per term,
// as a register-blocked SGEMM:
//   * CTA tile 128 cells x 128 outputs, K block 16, 256 threads; a thread owns 8 x 8 results as
//     (4 + 4) x (4 + 4): cells ty*4.. and 64 + ty*4.., outputs tx*4.. and 64 + tx*4.., so every
//     operand fragment is one LDS.128 (4 per 64 FFMA) and a warp reads two distinct W fragments
//     (broadcast) and sixteen consecutive T fragments (conflict-free);
//   * the next K block's global loads (2 float4 of W, 2 of T per thread) are issued before the
//     current block is multiplied and stored to the other shared-memory buffer afterwards: one
//     __syncthreads per K block.
// The accumulation order of every output is that of the plain loop (k ascending), so the bits do
// not depend on the blocking.
#pragma once
#include <cstdint>

namespace mpfem_b200 {
namespace sg {

constexpr int BM = 128, BN = 128, BK = 16, THREADS = 256;
constexpr int LDA = BM + 4, LDB = BN + 4;  // rows stay 16-byte aligned

// W: n_cells x k_pad (row-major, k_pad % 16 == 0); Tm: k_pad x n_out_pad (row-major,
// n_out_pad % 128 == 0); out: n_cells x out_pitch.
__global__ void __launch_bounds__(THREADS, 2)
    cellmat_ffma_kernel(const float* __restrict__ W, const float* __restrict__ Tm, float* __restrict__ out,
                        int64_t n_cells, int n_out, int64_t n_out_pad, int64_t k_pad,
                        int64_t out_pitch, uint32_t* flags) {
  __shared__ __align__(16) float As[2][BK][LDA];  // [k][cell]
  __shared__ __align__(16) float Bs[2][BK][LDB];  // [k][output]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t c0 = int64_t(blockIdx.x) * BM;  // cell tiles on x (2^31 - 1 blocks)
  const int64_t o0 = int64_t(blockIdx.y) * BN;
  // global -> shared assignment: W rows a_row and a_row + 64, depth quad a_kq; T rows b_row and
  // b_row + 8, output quad b_c4
  const int a_row = tid >> 2, a_kq = tid & 3;
  const int b_row = tid >> 5, b_c4 = tid & 31;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* wp0 = W + (c0 + a_row) * k_pad + a_kq * 4;
  const float* wp1 = wp0 + 64 * k_pad;
  const bool w_ok0 = c0 + a_row < n_cells, w_ok1 = c0 + a_row + 64 < n_cells;
  const float* tp0 = Tm + int64_t(b_row) * n_out_pad + o0 + b_c4 * 4;
  const float* tp1 = tp0 + 8 * n_out_pad;

  float acc[8][8];
  #pragma unroll
  for (int i = 0; i < 8; ++i)
    #pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  float4 wa = w_ok0 ? *reinterpret_cast<const float4*>(wp0) : zero4;
  float4 wb = w_ok1 ? *reinterpret_cast<const float4*>(wp1) : zero4;
  float4 ta = *reinterpret_cast<const float4*>(tp0);
  float4 tb = *reinterpret_cast<const float4*>(tp1);
  auto stage = [&](int buf) {
    As[buf][a_kq * 4 + 0][a_row] = wa.x;
    As[buf][a_kq * 4 + 1][a_row] = wa.y;
    As[buf][a_kq * 4 + 2][a_row] = wa.z;
    As[buf][a_kq * 4 + 3][a_row] = wa.w;
    As[buf][a_kq * 4 + 0][a_row + 64] = wb.x;
    As[buf][a_kq * 4 + 1][a_row + 64] = wb.y;
    As[buf][a_kq * 4 + 2][a_row + 64] = wb.z;
    As[buf][a_kq * 4 + 3][a_row + 64] = wb.w;
    *reinterpret_cast<float4*>(&Bs[buf][b_row][b_c4 * 4]) = ta;
    *reinterpret_cast<float4*>(&Bs[buf][b_row + 8][b_c4 * 4]) = tb;
  };
  stage(0);
  __syncthreads();

  const int n_kb = int(k_pad / BK);
  for (int kb = 0; kb < n_kb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < n_kb) {  // next block's operands on their way while this one is multiplied
      const int64_t k1 = int64_t(kb + 1) * BK;
      wa = w_ok0 ? *reinterpret_cast<const float4*>(wp0 + k1) : zero4;
      wb = w_ok1 ? *reinterpret_cast<const float4*>(wp1 + k1) : zero4;
      ta = *reinterpret_cast<const float4*>(tp0 + k1 * n_out_pad);
      tb = *reinterpret_cast<const float4*>(tp1 + k1 * n_out_pad);
    }
    #pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      #pragma unroll
      for (int i = 0; i < 8; ++i)
        #pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kb + 1 < n_kb) {
      stage(buf ^ 1);  // the other buffer was last read before the previous barrier
      __syncthreads();
    }
  }

  uint32_t bad = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t c = c0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (c >= n_cells) continue;
    float* row = out + c * out_pitch;
    #pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t o = o0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (o < n_out) {
        bad |= isfinite(acc[i][j]) ? 0u : 1u;
        row[o] = acc[i][j];
      }
    }
  }
  if (bad && !(*reinterpret_cast<volatile uint32_t*>(flags) & 4u)) atomicOr(flags, 4u);
}

}  // namespace sg
}  // namespace mpfem_b200
