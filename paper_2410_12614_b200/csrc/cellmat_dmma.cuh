// cellmat_dmma.cuh -- K2 for the fp64 accumulation modes (u_q = fp64: the all-fp64 reference
// mode, reference_config of kernels.cpp:48-53, and 16-bit / fp32 storage with fp64
// accumulation) on the fp64 tensor cores:
//
//   D[c, o] = sum_k W[c, k] T[k, o]      (the all-cells GEMM of cellmat_tc.cuh, fp64 operands)
//
// with mma.sync.aligned.m16n8k4.row.col.f64 (SASS DMMA). The reference accumulates with the
// scalar engine (mm_units.cpp:76-88, one rounding per product and per sum, k ascending); the
// tensor core forms each k4 group's products exactly and rounds the dot products, so the
// result differs from the reference in the last bits and is checked, like every GEMM mode,
// against S * bound_a of the fp64 oracle (tests/test_gpu_cells.py).
//
// CTA tile 128 cells x 128 outputs, K block 16, 8 warps as 2 (M) x 4 (N) with 64 x 32 warp
// tiles (4 x 4 m16n8 accumulators = 64 doubles per thread). Operands are staged in shared
// memory transposed to [k][m] / [k][n] with rows padded to 136 doubles, so the fragment loads
// of a warp hit every bank pair exactly twice (the minimum for 256 bytes); the next K block is
// prefetched into registers while the current one is multiplied (double-buffered tiles).
#pragma once
#include <cstdint>

namespace mpfem_b200 {
namespace dm {

constexpr int BM = 128, BN = 128, BK = 16, THREADS = 256;
constexpr int PAD = 136;  // padded row (doubles) of the [k][m] and [k][n] tiles
constexpr int TILE = BK * PAD;
constexpr int SMEM_BYTES = 2 * 2 * TILE * 8;

__device__ __forceinline__ void mma_f64(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// W: n_cells x k_pad (row-major); T: k_pad x n_out_pad (row-major); out: n_cells x out_pitch.
__global__ void __launch_bounds__(THREADS, 1)
    cellmat_dmma_kernel(const double* __restrict__ W, const double* __restrict__ T,
                        double* __restrict__ out, int64_t n_cells, int n_out, int64_t n_out_pad,
                        int64_t k_pad, int64_t out_pitch, uint32_t* flags) {
  extern __shared__ double dsm[];
  double* As = dsm;              // [2][BK][PAD]: As[k][m]
  double* Bs = dsm + 2 * TILE;   // [2][BK][PAD]: Bs[k][n]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile (64 cells, 32 outputs)
  const int64_t c_base = int64_t(blockIdx.x) * BM;  // cell tiles on x (2^31 - 1 blocks)
  const int64_t o_base = int64_t(blockIdx.y) * BN;
  // global -> register staging: A row (tid / 2) columns (tid % 2) * 8 .. + 8; B row tid / 16
  // columns (tid % 16) * 8 .. + 8
  const int ar = tid >> 1, ac = (tid & 1) * 8;
  const int br = tid >> 4, bc = (tid & 15) * 8;
  const bool a_ok = c_base + ar < n_cells;
  const double* ag = W + (c_base + ar) * k_pad + ac;
  const double* bg = T + int64_t(br) * n_out_pad + o_base + bc;
  double2 ra[4], rb[4];
  auto load = [&](int kb) {
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
      ra[i] = a_ok ? __ldg(reinterpret_cast<const double2*>(ag + kb * BK) + i) : make_double2(0.0, 0.0);
      rb[i] = __ldg(reinterpret_cast<const double2*>(bg + int64_t(kb) * BK * n_out_pad) + i);
    }
  };
  auto stash = [&](int buf) {
    double* a = As + buf * TILE;
    double* b = Bs + buf * TILE;
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[(ac + 2 * i) * PAD + ar] = ra[i].x;
      a[(ac + 2 * i + 1) * PAD + ar] = ra[i].y;
      *reinterpret_cast<double2*>(b + br * PAD + bc + 2 * i) = rb[i];
    }
  };
  double acc[4][4][4];
  #pragma unroll
  for (int mi = 0; mi < 4; ++mi)
    #pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      #pragma unroll
      for (int e = 0; e < 4; ++e) acc[mi][ni][e] = 0.0;
  const int nkb = int(k_pad / BK);
  load(0);
  stash(0);
  __syncthreads();
  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) load(kb + 1);
    const double* a = As + buf * TILE + wm * 64 + gid;
    const double* b = Bs + buf * TILE + wn * 32 + gid;
    #pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4][2], bf[4];
      #pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        af[mi][0] = a[(kk + tig) * PAD + mi * 16];
        af[mi][1] = a[(kk + tig) * PAD + mi * 16 + 8];
      }
      #pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = b[(kk + tig) * PAD + ni * 8];
      #pragma unroll
      for (int mi = 0; mi < 4; ++mi)
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma_f64(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
    if (kb + 1 < nkb) {
      stash(buf ^ 1);
      __syncthreads();
    }
  }
  // epilogue: fragment (mi, ni) element e -> cell gid (+8 for e >= 2), output 2 tig (+1)
  uint32_t bad = 0;
  #pragma unroll
  for (int mi = 0; mi < 4; ++mi)
    #pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = c_base + wm * 64 + mi * 16 + gid + 8 * h;
      if (c >= n_cells) continue;
      double* row = out + c * out_pitch;
      #pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int64_t o = o_base + wn * 32 + ni * 8 + 2 * tig;
        #pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double v = acc[mi][ni][2 * h + e];
          bad |= !isfinite(v);
          if (o + e < n_out) __stcs(row + o + e, v);
        }
      }
    }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0 && bad && !(*reinterpret_cast<volatile uint32_t*>(flags) & 4u)) atomicOr(flags, 4u);
}

}  // namespace dm
}  // namespace mpfem_b200
