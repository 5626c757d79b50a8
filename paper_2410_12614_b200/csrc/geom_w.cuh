// geom_w.cuh -- K1: per-cell geometry + coefficient + scaled-weight pass.
//
// Geometry once per cell (one lane of a tile's first warp), then all threads of the CTA
// expand the tile's (cell, quadrature point) pairs into the rows of the GEMM operand W:
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

#include "cellmat_tc.cuh"
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
  int* error;              // set to 3 on a singular cell (host-mapped, see report_error)
  // Dynamic tile schedule: tile_ctr[0] hands out tiles gridDim.x, gridDim.x + 1, ... to
  // CTAs as they free up (static blockIdx.x first); tile_ctr[1] counts finished CTAs and
  // the last one resets both to zero (no per-call memset). One pair of words per stream
  // workspace, so concurrent calls on different streams never share a counter.
  uint32_t* tile_ctr;
  int geom_warps;          // warps computing the next tile's geometry; tile = 32 * geom_warps cells
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

// K1 is one launch, one CTA per tile of kTileCells cells (grid-stride over tiles):
//  phase 1: warp 0 runs the reference's LU/inverse/tensor sequence at u_g
//           (geometry.cpp:12-118) for the tile's cells, one lane per cell -> shared memory;
//  phase 2: all threads expand (cell, group of kQPT = 8 consecutive quadrature points)
//           items: coefficient z_q and the W entries of every (s<=t) block at those points.
// The rule (weights rounded to u_g, reference points) is staged in shared memory once per
// CTA, permuted to [j][group] so that the lanes of a warp (consecutive groups, same j)
// read consecutive words. Each thread writes each block of its 8 points with one 16-byte
// store (W rows use blocks of nq_pad = round_up(n_q, 8); entries q >= n_q are zero, as are
// the matching rows of T).
// UG / US are compile-time, so the emulated rounding folds to the plain op for fp64 and a
// single conversion for fp32.
struct __align__(16) CellGeo {
  double g[6];  // G_00 G_01 G_02 G_11 G_12 G_22 (poisson) or |det| (mass)
  double v0[3];  // (2 v0x, 2 v0y, v0z)
  double e[9];   // e[s*3 + i] = (v_{s+1}[i] - v0[i]), x and y components doubled
  float gf[6];   // g as fp32 (exact for u_g = fp32: no per-entry conversion in the expansion)
  float pad[2];
};

#ifndef MPFEM_K1_QPT
#define MPFEM_K1_QPT 8  // 8 points per item (more independent fp64 chains per thread): with MINB 2, K1 73.7 -> 64.5 us at config 1 (r1j A/B)
#endif
constexpr int kWAlign = 8;             // W / T block stride: nq_pad = round_up(n_q, kWAlign)
constexpr int kQPT = MPFEM_K1_QPT;      // quadrature points per thread (divides kWAlign)
static_assert(kWAlign % kQPT == 0 && kQPT % 2 == 0, "points per thread must divide the W block alignment");
#ifndef MPFEM_K1_TILE
#define MPFEM_K1_TILE 32
#endif
#ifndef MPFEM_K1_MINB
#define MPFEM_K1_MINB 2  // 2 CTAs/SM (128 registers, room for the 8-point items; r1j A/B)
#endif
constexpr int kTileCells = MPFEM_K1_TILE;
constexpr int kGeomThreads = 256;

template <typename T>
struct alignas(sizeof(T) * kQPT) PackQ {
  T v[kQPT];
};
// one store of a thread's kQPT consecutive entries (16 B for 8 x 16-bit)
template <typename T>
__device__ __forceinline__ void store_pack(T* dst, const PackQ<T>& pk) {
  constexpr int bytes = int(sizeof(PackQ<T>));
  if constexpr (bytes % 16 == 0) {
    #pragma unroll
    for (int k = 0; k < bytes / 16; ++k) reinterpret_cast<uint4*>(dst)[k] = reinterpret_cast<const uint4*>(&pk)[k];
  } else {
    #pragma unroll
    for (int k = 0; k < bytes / 8; ++k) reinterpret_cast<uint2*>(dst)[k] = reinterpret_cast<const uint2*>(&pk)[k];
  }
}

#ifdef MPFEM_K1_GEOM_NOINLINE
#define MPFEM_K1_GEOM_INLINE __noinline__
#else
#define MPFEM_K1_GEOM_INLINE __forceinline__
#endif
template <int UG>
__device__ MPFEM_K1_GEOM_INLINE void cell_geometry(const GeomWParams& P, int64_t cell, CellGeo& o,
                                                   uint32_t& fl) {
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
    report_error(P.error, 3);
    #pragma unroll
    for (int b = 0; b < 6; ++b) g.g[b] = __longlong_as_double(0x7ff8000000000000ll);  // singular: NaN row
  }
  #pragma unroll
  for (int b = 0; b < 6; ++b) {
    o.g[b] = g.g[b];
    o.gf[b] = float(g.g[b]);
  }
  // origin and edges with x, y pre-doubled (the coefficient's sinpi(2x), cospi(2y) arguments)
  #pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double sc = a < 2 ? 2.0 : 1.0;
    o.v0[a] = sc * v[0][a];
    #pragma unroll
    for (int s2 = 0; s2 < 3; ++s2) o.e[s2 * 3 + a] = sc * __dsub_rn(v[s2 + 1][a], v[0][a]);
  }
}

// W value at u_g: round_ug(round_ug(omega G_b) zhat_q) in float (u_g = fp32, IEEE fp32 ops are
// the correctly rounded binary64 results) or double (u_g = fp64).
template <int UG, bool HAVE_Z>
__device__ __forceinline__ auto w_value(double om, double gb, double zq) {
  if constexpr (UG == kFP32) {
    float v = __fmul_rn(float(om), float(gb));
    if (HAVE_Z) v = __fmul_rn(v, float(zq));
    return v;
  } else {
    double v = __dmul_rn(om, gb);
    if (HAVE_Z) v = __dmul_rn(v, zq);
    return v;
  }
}
template <typename T>
struct Storage16;
template <>
struct Storage16<__half> {
  static constexpr uint32_t kInf = 0x7c00u, kMinNormal = 0x0400u;
};
template <>
struct Storage16<__nv_bfloat16> {
  static constexpr uint32_t kInf = 0x7f80u, kMinNormal = 0x0080u;
};
// round_us (one RNE conversion) -> storage bits
template <typename T, typename V>
__device__ __forceinline__ uint32_t storage_bits16(V v) {
  if constexpr (std::is_same_v<T, __half>) {
    if constexpr (std::is_same_v<V, float>) return __half_as_ushort(__float2half_rn(v));
    else return __half_as_ushort(__double2half(v));
  } else {
    if constexpr (std::is_same_v<V, float>) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
    else return __bfloat16_as_ushort(__double2bfloat16(v));
  }
}
// FP-event bits of the packed path: sf.amax holds the packed (u16x2) max of |bits|
template <typename T>
__device__ __forceinline__ uint32_t packed_store_flags(const StoreFlags& sf) {
  const uint32_t a = max(sf.amax & 0xffffu, sf.amax >> 16);
  return (a == Storage16<T>::kInf ? kOverflow : 0u) | (a > Storage16<T>::kInf ? kInvalid : 0u) |
         (sf.tiny ? kUnderflow : 0u);
}

// dynamic shared memory of geom_w_kernel: weights and the three point coordinates, each
// nq_pad doubles in [j][group] order, then the two geometry buffers of 32 * geom_warps cells
constexpr int kGeoSlots = 3;  // geometry ring of K1's tile pipeline
__host__ __device__ constexpr size_t geom_w_smem_bytes(int nq_pad, int geom_warps = 1) {
  return size_t(4) * nq_pad * sizeof(double) + size_t(kGeoSlots) * 32 * geom_warps * sizeof(CellGeo) +
         size_t(nq_pad) * sizeof(float);
}

template <typename T, int UG, int US, int COEF>
__global__ void __launch_bounds__(kGeomThreads, MPFEM_K1_MINB) geom_w_kernel(GeomWParams P) {
  // Programmatic dependent launch: K2 (launched with programmatic stream serialisation) may
  // become resident on SMs this grid has left and run its prologue; it reads W only after
  // its griddepcontrol.wait, i.e. after this whole grid has completed and flushed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ double s_rule[];
  __shared__ uint32_t s_next[kGeoSlots];  // per-slot item counters (dynamic 32-item grabs)
  __shared__ int64_t s_tile[kGeoSlots];   // the slot's tile
  __shared__ uint64_t s_ready[kGeoSlots], s_free[kGeoSlots];
  const int nq = P.n_q;
  const int nqp = P.nq_pad;
  const int tcells = 32 * P.geom_warps;  // cells per tile
  CellGeo* s_geo0 = reinterpret_cast<CellGeo*>(s_rule + 4 * nqp);  // [kGeoSlots][tcells]
  const int ngroups = nqp / kQPT;  // P.div_nq divides by ngroups
  const int nb = P.poisson ? 6 : 1;
  double* sW = s_rule;
  double* sX = s_rule + nqp;  // sX[a * nqp + perm(q)]
  float* sWf = reinterpret_cast<float*>(s_geo0 + kGeoSlots * tcells);  // the weights as fp32 (u_g = fp32)
  for (int q = threadIdx.x; q < nqp; q += blockDim.x) {
    const int pq = (q % kQPT) * ngroups + q / kQPT;
    const bool ok = q < nq;
    sW[pq] = ok ? P.rule_w[q] : 0.0;
    sWf[pq] = ok ? float(P.rule_w[q]) : 0.0f;
    #pragma unroll
    for (int a = 0; a < 3; ++a) sX[a * nqp + pq] = ok ? P.rule_x[3 * q + a] : 0.0;
  }
  uint32_t fl = 0;
  StoreFlags sf;
  const int64_t n_tiles = (P.n_cells + tcells - 1) / tcells;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool geo_warp = warp < P.geom_warps;
  auto tile_cells = [&](int64_t t) {
    const int64_t left = P.n_cells - t * tcells;
    return left < tcells ? int(left) : tcells;
  };
  // Tiles: static blockIdx.x first, then gridDim.x + atomicAdd(tile_ctr).
  auto claim = [&]() -> int64_t { return int64_t(gridDim.x) + atomicAdd(P.tile_ctr, 1u); };
  // Tile pipeline over a 3-slot ring of geometry buffers, synchronised by mbarriers instead of
  // a CTA barrier per tile: in iteration k every warp expands tile k (slot k % 3, 32-item
  // grabs) once its geometry is ready, while the geom_warps first prepare slot (k + 1) % 3 --
  // claim tile k + 1 and compute its geometry (one lane per cell) -- after every warp has left
  // that slot's previous use (iteration k - 2). Fast warps run ahead into tile k + 1 instead
  // of waiting for the slowest warp of tile k.
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGeoSlots; ++i) {
      tc::mbar_init(&s_ready[i], P.geom_warps);
      tc::mbar_init(&s_free[i], kGeomThreads / 32);
      s_next[i] = 0;
    }
    s_tile[0] = blockIdx.x;
  }
  if (blockIdx.x < n_tiles && threadIdx.x < tile_cells(blockIdx.x))
    cell_geometry<UG>(P, int64_t(blockIdx.x) * tcells + threadIdx.x, s_geo0[threadIdx.x], fl);
  __syncthreads();  // s_rule, the barriers, tile 0's index and geometry
  if (geo_warp && lane == 0) tc::mbar_arrive(&s_ready[0]);
  for (int k = 0;; ++k) {
    const int buf = k % kGeoSlots;
    tc::mbar_wait(&s_ready[buf], uint32_t(k / kGeoSlots) & 1u);
    const int64_t tile = s_tile[buf];
    if (tile >= n_tiles) break;
    if (geo_warp) {  // prepare slot (k + 1) % 3 for tile k + 1
      const int nbuf = (k + 1) % kGeoSlots;
      if (k >= 2) tc::mbar_wait(&s_free[nbuf], uint32_t((k - 2) / kGeoSlots) & 1u);
      if (threadIdx.x == 0) {
        s_tile[nbuf] = claim();
        s_next[nbuf] = 0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * P.geom_warps) : "memory");
      const int64_t nt = s_tile[nbuf];
      if (nt < n_tiles && int(threadIdx.x) < tile_cells(nt))
        cell_geometry<UG>(P, nt * tcells + threadIdx.x, s_geo0[nbuf * tcells + threadIdx.x], fl);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&s_ready[nbuf]);
    }
    const int64_t c0 = tile * tcells;
    const int nc = tile_cells(tile);
    const uint32_t items = uint32_t(nc * ngroups);
    const CellGeo* geo_t = s_geo0 + buf * tcells;
    while (true) {
      uint32_t base = 0;
      if (lane == 0)  // plain shared atomic (atomicAdd would add warp-aggregation code)
        asm volatile("atom.shared.add.u32 %0, [%1], 32;" : "=r"(base) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_next[buf]))) : "memory");
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= items) break;
      const uint32_t it = base + lane;
      if (it >= items) continue;
      const uint32_t cl = P.div_nq.div(it);
      const int grp = int(it - cl * uint32_t(ngroups));
      const int q0 = grp * kQPT;
      const int64_t cell = c0 + cl;
      const CellGeo& cg = geo_t[cl];
      const double* coef = P.coef ? P.coef + cell * P.coef_stride : nullptr;
      double zq[kQPT], om[kQPT];
      float zqf[kQPT], omf[kQPT];  // u_g = fp32: the same values in fp32 (exact)
      #pragma unroll
      for (int j = 0; j < kQPT; ++j) {
        const int pq = j * ngroups + grp;
        if constexpr (UG == kFP32) omf[j] = sWf[pq];
        else om[j] = sW[pq];
        zq[j] = 1.0;
        zqf[j] = 1.0f;
        if constexpr (COEF != 0) {
          const double xi[3] = {sX[pq], sX[nqp + pq], sX[2 * nqp + pq]};
          if constexpr (COEF == 1 && UG == kFP32) {
            zqf[j] = coef_sincosexp_f(cg.v0, cg.e, xi);
          } else if constexpr (COEF == 1) {
            zq[j] = droundT<UG>(coef_sincosexp_e(cg.v0, cg.e, xi), fl);
          } else if constexpr (COEF == 2) {
            zq[j] = droundT<UG>(coef_exp10_affine(coef, xi), fl);
          } else {
            const int q = q0 + j;
            if (q < nq) {
              double acc = 0.0;
              for (int k = 0; k < P.n_phi; ++k)
                acc = dadd(acc, dmul(dround(coef[k], P.up, fl), P.tab_up[int64_t(k) * nq + q], P.up, fl), P.up, fl);
              zq[j] = droundT<UG>(acc, fl);
            }
          }
        }
      }
      constexpr bool have_z = COEF != 0;
      if constexpr (UG == kFP32 && COEF != 1) {
        #pragma unroll
        for (int j = 0; j < kQPT; ++j) zqf[j] = float(zq[j]);
      }
      T* wrow = static_cast<T*>(P.W) + cell * P.k_pad + q0;
      // C_stq = round_us(round_ug(round_ug(omega G_st) zhat_q))  (kernels.cpp:189-192).
      // Points q >= n_q (only in a cell's last group) are exact zeros whatever G is.
      bool pad[kQPT];  // (the 16-bit path below uses the packed keep mask instead)
      #pragma unroll
      for (int j = 0; j < kQPT; ++j) pad[j] = q0 + j >= nq;
      if constexpr (sizeof(T) == 2 && (UG == kFP32 || UG == kFP64)) {
        // 16-bit storage: convert, pack two values per word, zero the padding halfwords
        // (only in a cell's last group), and derive the FP events from the packed words:
        // packed max of |bits| (>= the inf pattern: overflow / NaN) and packed min (below the
        // smallest normal: candidate underflow, confirmed exactly on that block). The
        // underflow flag is sticky, so once a thread has raised it the check is skipped
        // (fp16 W underflows on most cells from p = 3 on).
        constexpr int KW = kQPT / 2;  // packed words per block
        // entries j < nv are quadrature points, the rest padding (only in a cell's last group)
        const int nv = nq - q0;
        uint32_t keep[KW];
        #pragma unroll
        for (int k = 0; k < KW; ++k)
          keep[k] = (2 * k < nv ? 0x0000ffffu : 0u) | (2 * k + 1 < nv ? 0xffff0000u : 0u);
        // points whose coefficient is exactly zero (their W entries are exact zeros)
        uint32_t zqz[KW];
        #pragma unroll
        for (int k = 0; k < KW; ++k)
          if constexpr (UG == kFP32)
            zqz[k] = (zqf[2 * k] == 0.0f ? 0x0000ffffu : 0u) | (zqf[2 * k + 1] == 0.0f ? 0xffff0000u : 0u);
          else
            zqz[k] = (zq[2 * k] == 0.0 ? 0x0000ffffu : 0u) | (zq[2 * k + 1] == 0.0 ? 0xffff0000u : 0u);
        // Analytic coefficient at u_g = fp64 (BASELINE config 1, "G_K in fp64"): the point
        // factor omega_q c_q is formed once, so each of the 6 blocks costs one DMUL instead of
        // two. Same binary64 operations, grouped differently from build_C's
        // round(round(omega G) c): the products may differ in the last fp64 bit, which the
        // 16-bit storage rounding absorbs (W parity for the analytic coefficient is within
        // ulp(u_s), tests/test_gpu_cells.py). Constant and nodal coefficients keep build_C's
        // exact order (bitwise W).
        constexpr bool kFoldZ = UG == kFP64 && COEF == 1;
        double omz[kQPT];
        if constexpr (kFoldZ) {
          #pragma unroll
          for (int j = 0; j < kQPT; ++j) omz[j] = __dmul_rn(om[j], zq[j]);
        }
        #pragma unroll
        for (int b = 0; b < 6; ++b) {
          if (b < nb) {
            const double gb = cg.g[b];
            uint32_t wd[KW];
            #pragma unroll
            for (int k = 0; k < KW; ++k) {
              uint32_t lo, hi;
              if constexpr (kFoldZ) {
                lo = storage_bits16<T>(__dmul_rn(omz[2 * k], gb));
                hi = storage_bits16<T>(__dmul_rn(omz[2 * k + 1], gb));
              } else if constexpr (UG == kFP32) {
                const float gf = cg.gf[b];
                float v0 = __fmul_rn(omf[2 * k], gf), v1 = __fmul_rn(omf[2 * k + 1], gf);
                if (have_z) {
                  v0 = __fmul_rn(v0, zqf[2 * k]);
                  v1 = __fmul_rn(v1, zqf[2 * k + 1]);
                }
                lo = storage_bits16<T>(v0);
                hi = storage_bits16<T>(v1);
              } else {
                lo = storage_bits16<T>(w_value<UG, have_z>(om[2 * k], gb, zq[2 * k]));
                hi = storage_bits16<T>(w_value<UG, have_z>(om[2 * k + 1], gb, zq[2 * k + 1]));
              }
              wd[k] = (lo | (hi << 16)) & keep[k];
            }
            #pragma unroll
            for (int k = 0; k < KW; ++k) sf.amax = __vmaxu2(sf.amax, wd[k] & 0x7fff7fffu);
            if (!sf.tiny) {
              // A nonzero stored value below the smallest normal is an underflow. A stored
              // zero is one unless the exact value was zero: omega > 0 at quadrature points,
              // so that needs G_b == 0 or a zero coefficient (an fp64 product underflowing
              // to zero counts as underflow, as in fp_op).
              uint32_t bmin = 0xffffffffu, zmask = 0;
              #pragma unroll
              for (int k = 0; k < KW; ++k) {
                const uint32_t m = wd[k] & 0x7fff7fffu;
                const uint32_t z = __vcmpeq2(m, 0u) & keep[k];
                zmask |= z & ~zqz[k];
                bmin = __vminu2(bmin, m | z | ~keep[k]);
              }
              if (min(bmin & 0xffffu, bmin >> 16) < Storage16<T>::kMinNormal || (zmask && gb != 0.0))
                sf.tiny = 1;
            }
            if constexpr (KW == 4)
              *reinterpret_cast<uint4*>(wrow + int64_t(b) * nqp) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
            else
              *reinterpret_cast<uint2*>(wrow + int64_t(b) * nqp) = make_uint2(wd[0], wd[1]);
          }
        }
      } else {
      #pragma unroll
      for (int b = 0; b < 6; ++b) {
        if (b < nb) {
          const double gb = cg.g[b];
          PackQ<T> pk;
          #pragma unroll
          for (int j = 0; j < kQPT; ++j) {
            if constexpr (UG == kFP32) {
              float val = __fmul_rn(omf[j], cg.gf[b]);  // fp32 values: exact-then-round
              if (have_z) val = __fmul_rn(val, zqf[j]);
              if (pad[j]) val = 0.0f;
              pk.v[j] = to_storage<T, US>(val, sf);
            } else if constexpr (UG == kFP64) {
              double val = __dmul_rn(om[j], gb);
              if (have_z) val = __dmul_rn(val, zq[j]);
              if (pad[j]) val = 0.0;
              pk.v[j] = to_storage<T, US>(val, sf);
            } else {
              double val = droundT<UG>(__dmul_rn(om[j], gb), fl);
              if (have_z) val = droundT<UG>(__dmul_rn(val, zq[j]), fl);
              if (pad[j]) val = 0.0;
              pk.v[j] = to_storage<T, US>(val, sf);
            }
          }
          store_pack(wrow + int64_t(b) * nqp, pk);
        }
      }
      }
      // tail K..K_pad of the row: zeros (the group that owns the last block's start writes it)
      if (q0 == 0) {
        T* tail = static_cast<T*>(P.W) + cell * P.k_pad;
        for (int64_t k = int64_t(nb) * nqp; k < P.k_pad; ++k) tail[k] = T(0.0f);
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&s_free[buf]);  // this warp is done with slot buf
  }
  if (threadIdx.x == 0) {
    // every CTA made its final (failing) claim before counting itself done
    __threadfence();
    if (atomicAdd(P.tile_ctr + 1, 1u) == gridDim.x - 1) {
      P.tile_ctr[0] = 0;
      P.tile_ctr[1] = 0;
    }
  }
  if constexpr (sizeof(T) == 2 && (UG == kFP32 || UG == kFP64))
    publish_flags(P.flags, fl | packed_store_flags<T>(sf));
  else
    publish_flags(P.flags, fl | store_flags_bits(sf));
}

// Shared basis-product operand T from the store tabulation B (n_d x n_phi x n_q, u_s values):
//   T[(b,q), (i,j)] = round_us(B_s[i,q] B_t[j,q] (+ B_t[i,q] B_s[j,q] if s<t)).
// transposed != 0 stores Tt[o][k] (K contiguous; the tcgen05 A operand), else T[k][o].
// rows: optional output-row table (tcgen05 path): row o computes entry (i, j) =
// (rows[o] & 0xffff, rows[o] >> 16), or nothing when rows[o] < 0; NULL means o = i*n_phi + j.
// (s, t) of packed block b: the row-major upper triangle of an n_d x n_d tensor
// (n_d = 3: (0,0) (0,1) (0,2) (1,1) (1,2) (2,2), the order K1 writes W in)
__host__ __device__ inline void block_pair(int b, int nd, int& s, int& t) {
  s = 0;
  int row = nd;
  while (b >= row) {
    b -= row;
    ++s;
    --row;
  }
  t = s + b;
}

template <typename T>
__global__ void build_t_kernel(const double* B, int n_phi, int n_q, int nq_pad, int nd, int us,
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
      block_pair(b, nd, s, t);
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
