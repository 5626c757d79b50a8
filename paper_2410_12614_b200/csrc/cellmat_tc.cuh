// cellmat_tc.cuh -- K2: all-cells GEMM on the 5th-generation tensor cores (sm_100a).
//
//   D^T[o, c] = sum_k Tt[o, k] * W[c, k]      o = (i, j) output entry, c = cell
//
// which is reference Algorithm 1 (kernels.cpp:242-267: A = sum_st B_s C_st B_t^T, one
// depth-chained product over (s,t,q)) for every cell at once: the per-cell scaled
// weights W (K1) are the B operand, the shared basis products Tt the A operand.
//
// Warp-specialised persistent kernel, one CTA per SM:
//   warp 0      TMA producer: 128x64 Tt box + 256x64 W box per stage (SWIZZLE_128B)
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16,
//               fp32 (or f16) accumulators in TMEM, two 256-column buffers
//   warp 2      TMEM allocator (512 columns)
//   warps 4-11  epilogue (two per TMEM lane quarter, half the columns each):
//               tcgen05.ld 32x32b.x32 -> registers -> global. TMEM lane =
//               output entry, column = cell, so one warp store writes 32 consecutive
//               entries (128 B) of one cell's row-major matrix: coalesced, no staging.
// Output rows come from a table P.rows (entry (i, j) per TMEM lane; default row-major, so a
// warp store is 128 contiguous bytes of one cell). T is bitwise symmetric in (i, j), so
// A_ij == A_ji bitwise; an experimental table (MPFEM_B200_SYMMETRIC=1) covers only the
// upper triangle and writes each value to (i, j) and (j, i) -- fewer MMAs, but its 16/32-byte
// store pieces make the register-resident epilogue LSU-bound (slower).
// Tiles are ordered cell-block-major so the W block of a cell block is reused from L2
// by the CTAs that work on its output tiles at the same time.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdint>

namespace mpfem_b200 {
namespace tc {

#ifndef MPFEM_TC_BACKOFF_NS
#define MPFEM_TC_BACKOFF_NS 256
#endif
constexpr int BM = 128;  // output entries per tile (MMA M, TMEM lanes)
#ifndef MPFEM_TC_BN
#define MPFEM_TC_BN 256
#endif
#ifndef MPFEM_TC_STAGES
#define MPFEM_TC_STAGES 4
#endif
constexpr int BN = MPFEM_TC_BN;  // cells per tile (MMA N, TMEM columns per accumulator)
constexpr int BK = 64;   // 16-bit elements per K block = one 128-byte swizzle row
constexpr int STAGES = MPFEM_TC_STAGES;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 8;      // two warps per TMEM lane quarter, each half the columns
constexpr int EPI_SPLIT = EPI_WARPS / 4;
constexpr int THREADS = 128 + EPI_WARPS * 32;
constexpr int TMEM_COLS = 2 * BN >= 512 ? 512 : (2 * BN >= 256 ? 256 : 128);
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct Params {
  int64_t n_cells;
  int n_out;          // rows of Tt actually used (valid output rows)
  int n_phi;
  const int32_t* rows;  // output-row table: i | j << 16 | mirror << 30, or -1 (padding)
  int n_out_tiles;
  int n_cell_tiles;
  int num_k_blocks;
  float* out;
  int64_t out_pitch;
  uint32_t idesc;
  uint32_t* flags;
  // Concurrent K1/K2: per-K1-tile W stamps (NULL: W complete at launch, stream order)
  const uint32_t* ready;
  uint32_t epoch;
  int k1_tile;         // cells per K1 tile (stamp granularity)
  int* error;          // set to 5 if a stamp never arrives (K1 not co-resident); error[1]
                       // holds the epoch of the last timed-out call (later waits skip)
  unsigned long long* trace;  // debug timeline (slots 1024..2047), NULL normally
  // Fused CSR scatter (pair kernel, OUTK != 0): instead of storing, entry (i, j) of cell c
  // is added into values[pos_map[c * n_out + i * n_phi + j]] (fp32 or fp64 values).
  const int32_t* pos_map;
  void* values;
};

// Producer-side wait for K1's W rows [c0, c1): acquire each K1 tile stamp, then order the
// generic-proxy writes before this thread's async-proxy (TMA) reads. Bounded: after ~0.2 s
// without progress it flags error 5 and returns, so a scheduling failure cannot hang the GPU.
__device__ __forceinline__ void wait_w_ready(const Params& P, int64_t c0, int64_t c1) {
  if (!P.ready) return;
  if (c1 > P.n_cells) c1 = P.n_cells;
  if (c0 >= c1) return;
  const int64_t t0 = c0 / P.k1_tile, t1 = (c1 - 1) / P.k1_tile;
  uint64_t start = 0;
  for (int64_t t = t0; t <= t1; ++t) {
    if (reinterpret_cast<volatile uint32_t*>(P.error)[1] == P.epoch) return;  // this call timed out
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.ready + t) : "memory");
      if (v == P.epoch) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (!start) start = now;
      else if (now - start > 200000000ull) {
        atomicExch(P.error, 5);
        atomicExch(reinterpret_cast<uint32_t*>(P.error) + 1, P.epoch);
        return;
      }
      __nanosleep(200);
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Waits that are not on the MMA critical path back off with nanosleep, so warps parked on
// a barrier leave the issue slots to co-resident K1 CTAs.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) __nanosleep(MPFEM_TC_BACKOFF_NS);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand, 128-byte swizzle: rows of 128 B, 8-row atoms 1024 B apart (SBO).
__device__ __forceinline__ uint64_t make_smem_desc(const void* p) {
  uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;       // start address
  d |= uint64_t(1) << 16;              // leading byte offset (unused for SW128 K-major)
  d |= uint64_t(1024 >> 4) << 32;      // stride byte offset
  d |= uint64_t(1) << 46;              // descriptor version (sm_100)
  d |= uint64_t(2) << 61;              // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Instruction descriptor for kind::f16 (dense, K-major A and B).
__host__ __device__ constexpr uint32_t make_idesc(int ab_bf16, int d_f32, int m, int n) {
  return (uint32_t(d_f32 ? 1 : 0) << 4) | (uint32_t(ab_bf16) << 7) | (uint32_t(ab_bf16) << 10) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

template <bool ACC_F16>
__global__ void __launch_bounds__(THREADS, 1)
    cellmat_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const Params P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total_tiles = P.n_out_tiles * P.n_cell_tiles;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
        for (int kb = 0; kb < P.num_k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sA + stage * A_BYTES, &tmA, kb * BK, ot * BM, &full[stage]);
          tma_load_2d(sB + stage * B_BYTES, &tmB, kb * BK, ct * BN, &full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < P.num_k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = make_smem_desc(sA + stage * A_BYTES);
          const uint64_t bd = make_smem_desc(sB + stage * B_BYTES);
          #pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_f16(d_tmem, ad + uint64_t(2 * kk), bd + uint64_t(2 * kk), P.idesc, (kb | kk) != 0);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else if (warp >= 4) {
    // TMEM lane quarter = warp % 4 (hardware rule); the two warps of a quarter split the
    // accumulator's 256 columns (cells) in halves.
    const int quarter = warp & 3;
    const int half = (warp - 4) >> 2;  // which 1/EPI_SPLIT of the columns
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t expo_or = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int o = ot * BM + quarter * 32 + lane;
      const int32_t e = P.rows[o];
      const bool o_ok = e >= 0;
      const int ei = e & 0xffff, ej = (e >> 16) & 0x3fff;
      const int off_d = ei * P.n_phi + ej;                 // entry (i, j)
      const int off_m = ej * P.n_phi + ei;                 // its mirror (j, i)
      const bool mirror = o_ok && (e & (1 << 30));         // symmetric table only
      #pragma unroll 1
      for (int chunk = half * (BN / 32 / EPI_SPLIT); chunk < (half + 1) * (BN / 32 / EPI_SPLIT); ++chunk) {
        uint32_t r[32];
        tmem_ld_x32(tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN + chunk * 32), r);
        const int64_t cell0 = int64_t(ct) * BN + chunk * 32;
        if (o_ok) {
          float* dst = P.out + cell0 * P.out_pitch + off_d;
          const int64_t left = P.n_cells - cell0;
          if (left >= 32 && !mirror) {  // common case: full chunk, row-major table
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
              float v;
              if constexpr (ACC_F16) v = __half2float(__ushort_as_half(static_cast<unsigned short>(r[j] & 0xffffu)));
              else v = __uint_as_float(r[j]);
              expo_or |= (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
              __stcs(dst, v);
              dst += P.out_pitch;
            }
          } else {
            float* base = P.out + cell0 * P.out_pitch;
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (j < left) {
                float v;
                if constexpr (ACC_F16) v = __half2float(__ushort_as_half(static_cast<unsigned short>(r[j] & 0xffffu)));
                else v = __uint_as_float(r[j]);
                expo_or |= (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
                __stcs(base + off_d, v);
                if (mirror) __stcs(base + off_m, v);
              }
              base += P.out_pitch;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    expo_or = __reduce_or_sync(0xffffffffu, expo_or);
    if (lane == 0 && expo_or && !(*reinterpret_cast<volatile uint32_t*>(P.flags) & 4u)) atomicOr(P.flags, 4u);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tc
}  // namespace mpfem_b200
