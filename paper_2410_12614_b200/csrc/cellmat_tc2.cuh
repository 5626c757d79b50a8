// cellmat_tc2.cuh -- K2 on a CTA pair (tcgen05 cta_group::2), the default tcgen05 path.
//
// Same GEMM as cellmat_tc.cuh (D^T[o, c] = sum_k Tt[o, k] W[c, k]), but each 2-CTA cluster
// computes a 256-output x 256-cell tile with one M=256 MMA per K=16 step:
//   * each CTA stages its own 128 output rows of Tt and its own 128 cells of W per stage
//     (32 KB, 7 stages in 224 KB): per-SM operand traffic is 2/3 of the 1-CTA kernel's and
//     the pipeline holds 1.5x more MMA work in flight;
//   * only the leader (cluster rank 0) arms the full barriers (expect_tx of both CTAs'
//     bytes; the peer's TMA completes on the leader's barrier) and issues the MMAs;
//   * the MMA writes rows 0..127 of D into the leader's TMEM and rows 128..255 into the
//     peer's; commits multicast to both CTAs' barriers; both epilogues drain their own
//     TMEM and arrive on the leader's tmem-empty barrier.
#pragma once
#include "cellmat_tc.cuh"
#include "l2_hints.cuh"

namespace mpfem_b200 {
namespace tc2 {

constexpr int BM = 256;        // outputs per pair tile (MMA M)
constexpr int BMC = 128;       // outputs per CTA (TMEM lanes)
constexpr int BN = 256;        // cells per pair tile (MMA N; each CTA stages 128)
constexpr int BNC = 128;
constexpr int BK = 64;
#ifndef MPFEM_TC2_STAGES
#define MPFEM_TC2_STAGES 7  // 7 x 32 KB + barriers = 225 KB (measured 119 -> 115 us at config 1)
#endif
constexpr int STAGES = MPFEM_TC2_STAGES;
constexpr int A_BYTES = BMC * BK * 2;
constexpr int B_BYTES = BNC * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + EPI_WARPS * 32;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the CTA-rank bit of a cluster smem address

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int x, int y,
                                                 uint64_t* bar) {
  const uint32_t leader_bar = tc::smem_u32(bar) & kPeerMask;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
// same, with an L2 eviction-priority hint (createpolicy): streamed operands marked evict-first
// leave the L2 to the lines that are reused
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                      uint64_t* bar, uint64_t policy) {
  const uint32_t leader_bar = tc::smem_u32(bar) & kPeerMask;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar, uint16_t mask = 0x3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(tc::smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tc::smem_u32(bar) & kPeerMask)
               : "memory");
}

// OUTK: 0 = store the cell matrices (out, out_pitch); 1 / 2 = fused atomic CSR scatter into
// fp32 / fp64 values through pos_map (the local matrices never reach HBM).
template <bool ACC_F16, int OUTK = 0>
__global__ void __launch_bounds__(THREADS, 1)
    cellmat_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const tc::Params P) {
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
  const uint32_t rank = cluster_rank();  // CTA within its pair
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / 2, n_clusters = gridDim.x / 2;
  const int total_tiles = P.n_out_tiles * P.n_cell_tiles;  // pair tiles

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 2 * EPI_WARPS);  // both CTAs' epilogue warps (leader's copy used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(tmem_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any cross-CTA arrive / complete_tx
  tc::tc_fence_after();
  // Launched with programmatic stream serialisation behind K1: everything above overlaps
  // K1's tail; W, the flags word and the output are touched only after K1 has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      [[maybe_unused]] const uint64_t w_policy = OUTK != 0 ? policy_evict_first() : 0;
      for (int tile = cluster; tile < total_tiles; tile += n_clusters) {
        const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
        for (int kb = 0; kb < P.num_k_blocks; ++kb) {
          tc::mbar_wait_backoff(&empty[stage], phase ^ 1u);
          if (leader) tc::mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          tma_load_2d_pair(sA + stage * A_BYTES, &tmA, kb * BK, ot * BM + int(rank) * BMC, &full[stage]);
          // fused scatter: W is read once per output tile and must not push the CSR value
          // lines (the reductions' working set) out of the L2
          if constexpr (OUTK != 0)
            tma_load_2d_pair_hint(sB + stage * B_BYTES, &tmB, kb * BK, ct * BN + int(rank) * BNC, &full[stage], w_policy);
          else
            tma_load_2d_pair(sB + stage * B_BYTES, &tmB, kb * BK, ct * BN + int(rank) * BNC, &full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = cluster; tile < total_tiles; tile += n_clusters) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < P.num_k_blocks; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint64_t ad = tc::make_smem_desc(sA + stage * A_BYTES);
          const uint64_t bd = tc::make_smem_desc(sB + stage * B_BYTES);
          #pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_pair(d_tmem, ad + uint64_t(2 * kk), bd + uint64_t(2 * kk), P.idesc, (kb | kk) != 0);
          commit_pair(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        commit_pair(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else if (warp >= 4) {
    const int quarter = warp & 3;
    const int half = (warp - 4) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t expo_or = 0;
    [[maybe_unused]] const uint64_t keep = OUTK != 0 ? asmb::policy_evict_last() : 0;
    for (int tile = cluster; tile < total_tiles; tile += n_clusters) {
      const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
      tc::mbar_wait_backoff(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      const int o = ot * BM + int(rank) * BMC + quarter * 32 + lane;
      const int32_t e = P.rows[o];
      const bool o_ok = e >= 0;
      const int off = (e & 0xffff) * P.n_phi + ((e >> 16) & 0x3fff);
      #pragma unroll 1
      for (int chunk = half * (BN / 64); chunk < (half + 1) * (BN / 64); ++chunk) {
        uint32_t r[32];
        tc::tmem_ld_x32(tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN + chunk * 32), r);
        const int64_t cell0 = int64_t(ct) * BN + chunk * 32;
        if constexpr (OUTK != 0) {
          if (o_ok) {
            // all 32 positions first (independent coalesced loads), then the 32 reductions
            const int32_t* pm = P.pos_map + cell0 * P.n_out + off;
            const int64_t left = P.n_cells - cell0;
            int32_t pos[32];
            #pragma unroll
            for (int j = 0; j < 32; ++j) pos[j] = (left >= 32 || j < left) ? __ldcs(pm + j * P.n_out) : -1;
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (pos[j] >= 0) {
                float v;
                if constexpr (ACC_F16) v = __half2float(__ushort_as_half(static_cast<unsigned short>(r[j] & 0xffffu)));
                else v = __uint_as_float(r[j]);
                expo_or |= (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
                if constexpr (OUTK == 1) asmb::red_add_keep(static_cast<float*>(P.values) + pos[j], v, keep);
                else asmb::red_add_keep(static_cast<double*>(P.values) + pos[j], double(v), keep);
              }
            }
          }
        } else if (o_ok) {
          float* dst = P.out + cell0 * P.out_pitch + off;
          const int64_t left = P.n_cells - cell0;
          #pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (left >= 32 || j < left) {
              float v;
              if constexpr (ACC_F16) v = __half2float(__ushort_as_half(static_cast<unsigned short>(r[j] & 0xffffu)));
              else v = __uint_as_float(r[j]);
              expo_or |= (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
#ifndef MPFEM_TC2_NOSTORE  // diagnostic build only (make diag)
              __stcs(dst, v);
#endif
            }
            dst += P.out_pitch;
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    expo_or = __reduce_or_sync(0xffffffffu, expo_or);
    if (lane == 0 && expo_or && !(*reinterpret_cast<volatile uint32_t*>(P.flags) & 4u)) atomicOr(P.flags, 4u);
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();  // the pair's MMAs and peer arrivals are done before TMEM is released
  if (warp == 2) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tc2
}  // namespace mpfem_b200
