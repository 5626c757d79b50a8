// cellmat_simt.cuh -- K2 for the reference precision modes without a tensor-core
// format: fp32 (FFMA, no TF32) and fp64 (DFMA). Same GEMM as the tcgen05 path,
//   A[c, o] = sum_k W[c, k] * T[k, o],
// register-blocked: a CTA computes BM cells x BN outputs, each thread TM x TN with
// strided ownership so that a warp's stores hit consecutive output entries of a cell.
#pragma once
#include <cstdint>

namespace mpfem_b200 {

template <typename T, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    cellmat_simt_kernel(const T* __restrict__ W, const T* __restrict__ Tm, T* __restrict__ out,
                        int64_t n_cells, int n_out, int64_t n_out_pad, int64_t k_pad,
                        int64_t out_pitch, uint32_t* flags) {
  constexpr int TX = BN / TN;  // threads along outputs
  constexpr int TY = BM / TM;  // threads along cells
  constexpr int NT = TX * TY;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int64_t c0 = int64_t(blockIdx.x) * BM;  // cell tiles on x (2^31 - 1 blocks)
  const int64_t o0 = int64_t(blockIdx.y) * BN;
  T acc[TM][TN];
  #pragma unroll
  for (int i = 0; i < TM; ++i)
    #pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (int64_t k0 = 0; k0 < k_pad; k0 += BK) {
    // W tile: BM cells x BK depth (K contiguous in global) -> As[k][cell]
    for (int idx = tid; idx < BM * BK; idx += NT) {
      int r = idx / BK, kk = idx % BK;
      int64_t c = c0 + r;
      As[kk][r] = (c < n_cells) ? W[c * k_pad + k0 + kk] : T(0);
    }
    // T tile: BK depth x BN outputs (outputs contiguous)
    for (int idx = tid; idx < BK * BN; idx += NT) {
      int kk = idx / BN, n = idx % BN;
      Bs[kk][n] = Tm[(k0 + kk) * n_out_pad + o0 + n];
    }
    __syncthreads();
    #pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
      #pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + i * TY];
      #pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + j * TX];
      #pragma unroll
      for (int i = 0; i < TM; ++i)
        #pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  uint32_t bad = 0;
  #pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t c = c0 + ty + i * TY;
    if (c >= n_cells) continue;
    #pragma unroll
    for (int j = 0; j < TN; ++j) {
      int64_t o = o0 + tx + j * TX;
      if (o < n_out) {
        bad |= isfinite(acc[i][j]) ? 0u : 1u;
        out[c * out_pitch + o] = acc[i][j];
      }
    }
  }
  if (bad && !(*reinterpret_cast<volatile uint32_t*>(flags) & 4u)) atomicOr(flags, 4u);
}

}  // namespace mpfem_b200
