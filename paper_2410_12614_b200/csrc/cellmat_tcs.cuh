// cellmat_tcs.cuh -- K2 for the HBM-bound shapes (short GEMM depth: mass p <= 5, Poisson p = 2):
// the same tcgen05 GEMM as cellmat_tc2.cuh, with an epilogue built for the output stream.
//
// Measured on B200 (scripts/store_probe2.cu, store_probe3.cu; profiles/r2b_*, r2c_*): writing the
// 65,536 x 1225 fp32 cell matrices as 128-byte pieces (one warp store per cell and 32 outputs,
// the TMEM-lane = output layout of cellmat_tc2) reaches 3.2 TB/s; as 1 KB contiguous runs per
// cell it reaches 5.8 TB/s (7.5 TB/s is the write-only fill ceiling). So this kernel
//   * computes a 256-output x 128-cell tile per CTA (two M = 128 MMAs sharing the W tile,
//     two TMEM accumulators of 128 columns, double buffered = 512 columns), so that one CTA
//     owns 256 consecutive outputs = 1 KB of every cell of the tile;
//   * drains TMEM in 32-cell chunks into a shared-memory staging tile [cell][256 outputs]
//     (each row shifted by its cell's global 16-byte misalignment, so the staged row and the
//     global run have the same alignment), then writes every cell's run with 16-byte
//     stores (scalar head / tail): 512 contiguous bytes per warp store instruction.
// Warp roles: warp 0 TMA producer, warp 1 MMA issuer (one thread), warp 2 TMEM allocator,
// warps 4..11 drain TMEM into a 3-slot staging ring (TMEM lane quarter = warp % 4; warps 4-7
// drain M-tile 0, 8-11 M-tile 1), warps 12..15 store the staged rows (mbarrier full / empty per
// slot), so the TMEM-read and HBM-write phases overlap instead of alternating.
// The output-row table is the identity (row o = output entry o of the row-major cell matrix).
#pragma once
#include "cellmat_tc.cuh"

namespace mpfem_b200 {
namespace tcs {

constexpr int BM = 128;            // outputs per MMA (TMEM lanes)
constexpr int MT = 2;              // M-tiles per CTA tile: 256 consecutive outputs
constexpr int BO = BM * MT;        // outputs per tile
constexpr int BN = 128;            // cells per tile (MMA N)
constexpr int BK = 64;
constexpr int STAGES = 2;
constexpr int A_BYTES = BM * BK * 2;          // one M-tile's Tt box
constexpr int B_BYTES = BN * BK * 2;          // the W box
constexpr int STAGE_BYTES = MT * A_BYTES + B_BYTES;
constexpr int CHUNK = 32;                     // cells per epilogue chunk
constexpr int SROW = BO + 4;                  // staged row: 256 outputs + room for the shift
constexpr int STAGE_OUT_BYTES = CHUNK * SROW * 4;
constexpr int SLOTS = 3;                      // staging ring between drain and store warps
constexpr int EPI_WARPS = 8;                  // drain warps (TMEM -> staging)
constexpr int ST_WARPS = 16;                  // store warps (staging -> global)
constexpr int THREADS = 128 + (EPI_WARPS + ST_WARPS) * 32;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + SLOTS * STAGE_OUT_BYTES + 1024 + 512;

template <bool ACC_F16, bool PACKED>
__global__ void __launch_bounds__(THREADS, 1)
    cellmat_tcs_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const tc::Params P) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base, derived from the shared array itself (so plain C++ accesses below
  // compile to LDS / STS rather than generic loads)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                  // [stage][MT][A_BYTES]
  uint8_t* sB = smem + STAGES * MT * A_BYTES;          // [stage][B_BYTES]
  float* sOut = reinterpret_cast<float*>(sB + STAGES * B_BYTES);  // [SLOTS][CHUNK][SROW]
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + SLOTS * CHUNK * SROW);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;       // staging slot written (EPI_WARPS arrivals)
  uint64_t* sempty = sfull + SLOTS;   // staging slot stored (ST_WARPS arrivals)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + SLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total_tiles = P.n_out_tiles * P.n_cell_tiles;  // n_out_tiles counts 256-output tiles
  // PACKED: small matrices (n_out <= 256) stored densely, so a 32-cell chunk is one
  // contiguous span (the launcher selects it when n_out_tiles == 1 and pitch == n_out)
  constexpr bool packed = PACKED;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], EPI_WARPS);
    }
    for (int a = 0; a < SLOTS; ++a) {
      tc::mbar_init(&sfull[a], EPI_WARPS);
      tc::mbar_init(&sempty[a], ST_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(tmem_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // Launched with programmatic stream serialisation behind K1: everything above overlaps
  // K1's tail; W, the flags word and the output are touched only after K1 has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
        for (int kb = 0; kb < P.num_k_blocks; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1u);
          tc::mbar_expect_tx(&full[stage], STAGE_BYTES);
          #pragma unroll
          for (int m = 0; m < MT; ++m)
            tc::tma_load_2d(sA + (stage * MT + m) * A_BYTES, &tmA, kb * BK, ot * BO + m * BM, &full[stage]);
          tc::tma_load_2d(sB + stage * B_BYTES, &tmB, kb * BK, ct * BN, &full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc::tc_fence_after();
        for (int kb = 0; kb < P.num_k_blocks; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint64_t bd = tc::make_smem_desc(sB + stage * B_BYTES);
          #pragma unroll
          for (int m = 0; m < MT; ++m) {
            const uint64_t ad = tc::make_smem_desc(sA + (stage * MT + m) * A_BYTES);
            const uint32_t d_tmem = tmem_base + uint32_t((acc * MT + m) * BN);
            #pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              tc::mma_f16(d_tmem, ad + uint64_t(2 * kk), bd + uint64_t(2 * kk), P.idesc, (kb | kk) != 0);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        tc::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else if (warp >= 4 && warp < 4 + EPI_WARPS) {
    // drain warps: TMEM -> staging slot, row j (cell cell0 + j) shifted by its run's 16-byte
    // misalignment so that the staged row and the global run share their alignment
    const int ew = warp - 4;
    const int quarter = warp & 3;   // TMEM lane quarter (hardware rule: warp % 4)
    const int m = ew >> 2;          // M-tile drained by this warp
    const int o_loc = m * BM + quarter * 32 + lane;  // output within the 256-output tile
    const uint32_t s_out = tc::smem_u32(sOut);
    const int pitch3 = int(P.out_pitch & 3);
    int acc = 0, slot = 0;
    uint32_t acc_phase = 0, slot_phase = 0;
    uint32_t magmax = 0;  // max of (bits << 1): a value with an all-ones exponent gives >= 0xff000000
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
      const int o_base = ot * BO;
      tc::mbar_wait_backoff(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      #pragma unroll 1
      for (int ch = 0; ch < BN / CHUNK; ++ch) {
        const int64_t cell0 = int64_t(ct) * BN + ch * CHUNK;
        uint32_t r[32];
        tc::tmem_ld_x32(tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t((acc * MT + m) * BN + ch * CHUNK), r);
        if (ch == BN / CHUNK - 1) {  // this warp's last TMEM read of the tile
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        }
        tc::mbar_wait(&sempty[slot], slot_phase ^ 1u);
        const uint32_t sbuf = s_out + uint32_t(slot * CHUNK * SROW * 4);
        if constexpr (packed) {
          // whole, densely packed cell matrices: the chunk is one contiguous span in global
          // memory, staged in exactly that layout (row pitch n_out)
          if (o_loc < P.n_out) {
            uint32_t addr = sbuf + uint32_t(o_loc * 4);
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
              uint32_t bits = r[j];
              if constexpr (ACC_F16) bits = __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(bits & 0xffffu))));
              magmax = max(magmax, bits << 1);
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(bits) : "memory");
              addr += uint32_t(P.n_out * 4);
            }
          }
        } else {
          // the shift of row j depends on j mod 4 only (4 pitches are a multiple of 16 bytes):
          // four base addresses, the row offset is an immediate of the unrolled store
          const int shift0 = int((uint64_t(cell0) * uint64_t(P.out_pitch) + uint64_t(o_base)) & 3u);
          uint32_t* base4[4];  // derived from the shared array: the stores compile to STS
          #pragma unroll
          for (int k = 0; k < 4; ++k)
            base4[k] = reinterpret_cast<uint32_t*>(sOut) + slot * CHUNK * SROW + o_loc + ((shift0 + k * pitch3) & 3);
          #pragma unroll
          for (int j = 0; j < 32; ++j) {
            uint32_t bits = r[j];
            if constexpr (ACC_F16) bits = __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(bits & 0xffffu))));
            magmax = max(magmax, bits << 1);  // sign dropped: non-finite iff >= 0xff000000
            base4[j & 3][j * SROW] = bits;
          }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sfull[slot]);
        if (++slot == SLOTS) { slot = 0; slot_phase ^= 1u; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    const uint32_t bad = __reduce_max_sync(0xffffffffu, magmax) >= 0xff000000u;
    if (lane == 0 && bad && !(*reinterpret_cast<volatile uint32_t*>(P.flags) & 4u)) atomicOr(P.flags, 4u);
  } else if (warp >= 4 + EPI_WARPS) {
    // store warps: staging slot -> global, each warp CHUNK / ST_WARPS cells per chunk: scalar
    // head to the 16-byte boundary, float4 body (512 B per store instruction), scalar tail
    const int sw = warp - 4 - EPI_WARPS;
    const int64_t pitch = P.out_pitch;
    int slot = 0;
    uint32_t slot_phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int ct = tile / P.n_out_tiles, ot = tile % P.n_out_tiles;
      const int o_base = ot * BO;
      const int n_run = min(BO, P.n_out - o_base);  // valid outputs of the tile
      #pragma unroll 1
      for (int ch = 0; ch < BN / CHUNK; ++ch) {
        const int64_t cell0 = int64_t(ct) * BN + ch * CHUNK;
        tc::mbar_wait(&sfull[slot], slot_phase);
        const float* srow = sOut + slot * CHUNK * SROW;
        if constexpr (packed) {  // one contiguous span: float4 copy by all store warps (16-B aligned)
          const int64_t nc = P.n_cells - cell0 < CHUNK ? P.n_cells - cell0 : int64_t(CHUNK);
          const int total = int(nc) * P.n_out;
          float* dst = P.out + cell0 * P.n_out;
          const int n4 = total >> 2;
          for (int i = sw * 32 + lane; i < n4; i += ST_WARPS * 32)
            __stcs(reinterpret_cast<float4*>(dst) + i, reinterpret_cast<const float4*>(srow)[i]);
          for (int i = 4 * n4 + sw * 32 + lane; i < total; i += ST_WARPS * 32) __stcs(dst + i, srow[i]);
        } else
        #pragma unroll 1
        for (int jj = 0; jj < CHUNK / ST_WARPS; ++jj) {
          const int j = sw * (CHUNK / ST_WARPS) + jj;
          const int64_t cell = cell0 + j;
          if (cell >= P.n_cells || n_run <= 0) break;
          const int64_t g0 = cell * pitch + o_base;
          const int sh = int(g0 & 3);
          const int head = min((4 - sh) & 3, n_run);
          const int nb4 = (n_run - head) >> 2;
          const int tail0 = head + 4 * nb4;
          float* dst = P.out + g0;
          const float* rowp = srow + (j * SROW + sh);
          float4 v4[BO / 128];
          #pragma unroll
          for (int h = 0; h < BO / 128; ++h) {
            const int i = lane + 32 * h;
            if (i < nb4) v4[h] = reinterpret_cast<const float4*>(rowp + head)[i];
          }
          const float vh = lane < head ? rowp[lane] : 0.0f;
          const float vt = lane < n_run - tail0 ? rowp[tail0 + lane] : 0.0f;
          float4* dst4 = reinterpret_cast<float4*>(dst + head);
          #pragma unroll
          for (int h = 0; h < BO / 128; ++h) {
            const int i = lane + 32 * h;
            if (i < nb4) __stcs(dst4 + i, v4[h]);
          }
          if (lane < head) __stcs(dst + lane, vh);
          if (lane < n_run - tail0) __stcs(dst + tail0 + lane, vt);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sempty[slot]);
        if (++slot == SLOTS) { slot = 0; slot_phase ^= 1u; }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tcs
}  // namespace mpfem_b200
