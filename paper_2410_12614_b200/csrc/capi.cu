// capi.cu -- the extern "C" boundary (include/mpfem_b200.h): setup handles, the
// batched cell-matrix driver (K1 geom_w -> K2 GEMM), host-buffer wrapper.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mpfem_b200.h"
#include "action.cuh"
#include "bounds.cuh"
#include "cellmat_fused.cuh"
#include "cellmat_dmma.cuh"
#include "cellmat_simt.cuh"
#include "cellmat_tc.cuh"
#include "cellmat_tc2.cuh"
#include "cellmat_tcs.cuh"
#include "geom_box.cuh"
#include "geom_tensor.cuh"
#include "geom_w.cuh"
#include "host_setup.hpp"

using namespace mpfem_b200;

namespace mpfem_b200 {
// K1 / fused-kernel instantiations live in launch_geom.cu / launch_fused.cu (separate
// translation units, compiled in parallel).
void launch_geom_typed(int w_type, int ug, int us, unsigned grid, cudaStream_t st,
                       const GeomWParams& P);
void launch_fused_dispatch(int key, int us, unsigned grid, cudaStream_t st, const FusedParams& F);
}  // namespace mpfem_b200

namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(expr)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw Error(MPFEM_B200_RUNTIME_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    f();
    return MPFEM_B200_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MPFEM_B200_RUNTIME_ERROR;
  }
}

// Device dispatch of a setup: which K2 runs and in which element types.
enum Path : int { kPathTC = 0, kPathF32 = 1, kPathF64 = 2, kPathFused = 3 };

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CUDA_OK(cudaMalloc(&p, n));
    bytes = n;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn tensor_map_encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!fn) throw Error(MPFEM_B200_RUNTIME_ERROR, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map_2d(const void* base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tensor_map_encoder()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(MPFEM_B200_RUNTIME_ERROR, "cuTensorMapEncodeTiled failed");
  return m;
}

int device_sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

}  // namespace

void mpfem_b200_set_last_error(const std::string& msg) { g_last_error = msg; }

// Per-stream scratch of a setup: the W operand, FP flags, K1's tile counter, host-API staging
// and the timing events. Calls on one stream are ordered by the stream, so they may share
// one workspace; calls on different streams get different workspaces and never race on
// device scratch (the setup itself is read-only after creation).
struct Workspace {
  DevBuf d_W, d_flags, d_tile_ctr, d_locals;
  DevBuf h_verts, h_cells, h_coef, h_out;  // device staging of the host-buffer API
  cudaEvent_t ev[8] = {};
  int n_ev = 0;
  ~Workspace() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  void mark(bool timing, cudaStream_t st) {
    if (!timing || n_ev >= 8) return;
    if (!ev[n_ev]) CUDA_OK(cudaEventCreate(&ev[n_ev]));
    CUDA_OK(cudaEventRecord(ev[n_ev++], st));
  }
};

struct mpfem_b200_setup_s {
  int p = 0, form = 0, up = 3, ug = 3, uq = 3, us = 3, engine = 0;
  int box = 0;         // hexahedral cells: per-point geometry in K1
  DevBuf d_ggrad;      // box: degree-1 basis gradients at u_g, (s * 8 + k) * n_q + q
  int n_phi = 0, n_q = 0, n_d = 1, n_blocks = 1, nq_pad = 0;
  int64_t k = 0, k_pad = 0, n_out = 0, n_out_pad = 0;
  int path = kPathF64;
  int acc_f16 = 0;
  int w_type = 3;  // element type of W / T: 0 fp16, 1 bf16, 2 fp32, 3 fp64
  // from_tab: created from the caller's rule and tabulations (mpfem_b200_setup_create_tab,
  // the C++ drop-in shim); such setups take geometry tensors, not vertices
  int from_tab = 0, dim = 3;
  std::vector<double> tab_store_host;  // the store tabulation (action contractions)
  Rule rule;
  // d_B: binary64 tabulation (bounds); d_Bs: the store tabulation (evaluated at u_p, stored at
  // u_s, tab_store of kernels.cpp:86-98) from which the GEMM operand T is built
  DevBuf d_rule_w, d_rule_w_ug, d_rule_x, d_tab_up, d_B, d_Bs, d_T, d_rows;
  int n_rows = 0;  // tcgen05 path: rows of Tt (output-row table, padded to the pair tile)
  // action (Algorithm 2): store tabulation in the u_p / u_q compute types, built on first use
  DevBuf d_act_a, d_act_c;
  int act_ap = -1, act_aq = -1;
  // GPU bound evaluation (kernel_bounds): binary64 budgets of the tabulation, built on first use
  DevBuf d_bnd_theta, d_bnd_vals, d_bnd_ggrad;
  double bnd_lebesgue = 0.0;
  double bnd_glebesgue[3] = {0.0, 0.0, 0.0}, bnd_gkmax[3] = {0.0, 0.0, 0.0};
  bool bnd_ready = false;
  int device = 0;
  // Host-side state is guarded by `mu`: every entry point holds it while it validates and
  // enqueues (the device work itself runs asynchronously on the caller's stream).
  std::mutex mu;
  std::map<cudaStream_t, std::unique_ptr<Workspace>> ws;
  Workspace* last_ws = nullptr;
  int last_launches = 0;
  int timing = 0;  // record CUDA events around K1 / K2 (mpfem_b200_set_timing)
  // CheckError word written by the kernels (report_error): pinned host memory mapped into
  // the device, read by the host without a copy.
  int* h_error = nullptr;
  int* d_error = nullptr;
  ~mpfem_b200_setup_s() {
    ws.clear();
    if (h_error) cudaFreeHost(h_error);
  }
  Workspace& workspace(cudaStream_t st) {
    auto& w = ws[st];
    if (!w) {
      auto n = std::make_unique<Workspace>();
      n->d_flags.ensure(16);
      n->d_tile_ctr.ensure(16);
      CUDA_OK(cudaMemset(n->d_flags.p, 0, 16));
      CUDA_OK(cudaMemset(n->d_tile_ctr.p, 0, 16));
      w = std::move(n);
    }
    last_ws = w.get();
    return *w;
  }
  // Raises a CheckError the device reported since the last check (the reference throws at
  // the failing cell, geometry.cpp:42; here the next call or synchronize reports it).
  void take_error(const char* when) {
    volatile int* e = h_error;
    const int code = *e;
    if (!code) return;
    *e = 0;
    throw Error(MPFEM_B200_CHECK_ERROR, std::string("singular cell geometry") + when);
  }
};

namespace {

size_t elem_size(int w_type) { return w_type <= 1 ? 2 : (w_type == 2 ? 4 : 8); }

void validate(int cell_kind, int dim, int p, int form, const int* fmts, int engine, int n_batch) {
  if ((cell_kind != 0 && cell_kind != 1) || dim != 3)
    throw Error(MPFEM_B200_CONFIG_ERROR, "the B200 path supports tetrahedra and hexahedra (dim 3)");
  if (p < 1 || p > 8) throw Error(MPFEM_B200_CONFIG_ERROR, "element degree must be in [1, 8]");
  if (cell_kind == 1 && p > 4) throw Error(MPFEM_B200_CONFIG_ERROR, "hexahedra support p <= 4");
  if (form != 0 && form != 1) throw Error(MPFEM_B200_CONFIG_ERROR, "unknown form");
  for (int i = 0; i < 4; ++i)
    if (fmts[i] < 0 || fmts[i] > 3) throw Error(MPFEM_B200_CONFIG_ERROR, "unknown float format");
  if (engine < 0 || engine > 2) throw Error(MPFEM_B200_CONFIG_ERROR, "unknown engine");
  // validate_config (kernels.cpp:29-40)
  if (n_batch < 1) throw Error(MPFEM_B200_CONFIG_ERROR, "batch size must be positive");
  if (engine == 2 && (fmts[3] != 0 || fmts[2] != 2))
    throw Error(MPFEM_B200_CONFIG_ERROR,
                "matrix engine requires the unit's native formats: u_s = bf16, u_q = fp32");
}

void choose_path(mpfem_b200_setup_s& S) {
  const int us = S.us, uq = S.uq;
  // Tiny GEMM depth (K <= 48) and small matrices: one thread per cell runs the whole
  // path in registers (cellmat_fused.cuh); fp32 accumulation of u_s-rounded operands.
  if (!S.box && !S.from_tab && uq == 2 && us <= 2 && (S.ug == 2 || S.ug == 3) && (S.p == 1 || (S.p == 2 && S.form == 0))) {
    S.path = kPathFused;
    S.w_type = us == 2 ? 2 : (us == 1 ? 0 : 1);
    return;
  }
  if ((us == 0 || us == 1) && uq == 2) {
    S.path = kPathTC;
    S.w_type = us == 1 ? 0 : 1;
  } else if (us == 1 && uq == 1) {
    S.path = kPathTC;
    S.w_type = 0;
    S.acc_f16 = 1;
  } else if (uq == 3) {
    S.path = kPathF64;  // any storage, fp64 accumulation; operands rounded to u_s
    S.w_type = 3;
  } else if (us == 2 && uq == 2) {
    S.path = kPathF32;
    S.w_type = 2;
  } else {
    throw Error(MPFEM_B200_CONFIG_ERROR,
                "unsupported accumulation: u_q must be fp32 or fp64, or fp16 with fp16 storage");
  }
}

// K1 tile height: one geometry lane per cell, so a tile of 32 G cells has G geometry warps.
// Low degrees have few quadrature groups per cell and would wait on a single geometry warp.
int k1_geom_warps(const mpfem_b200_setup_s& S) {
#ifdef MPFEM_K1_GW  // diagnostic builds only (scripts/build_variant.sh)
  return MPFEM_K1_GW;
#endif
  const int ngroups = S.nq_pad / kQPT;
  return std::max(1, std::min(4, 32 / ngroups));
}

// Optional fused CSR scatter of one call (mpfem_b200_cell_matrices_scatter).
struct Scatter {
  const int32_t* pos_map = nullptr;
  void* values = nullptr;
  bool fp64 = false;
};

void launch_geom_tet(mpfem_b200_setup_s& S, Workspace& ws, const double* verts, const int32_t* cells,
                     int64_t n, int coef_kind, const double* coef, int64_t coef_stride, void* W,
                     int64_t k_pad, int w_type, cudaStream_t st) {
  GeomWParams P;
  P.verts = verts;
  P.cells = cells;
  P.n_cells = n;
  P.coef_kind = coef_kind;
  P.coef = coef;
  P.coef_stride = coef_stride;
  P.rule_w = static_cast<const double*>(S.d_rule_w_ug.p);
  P.rule_x = static_cast<const double*>(S.d_rule_x.p);
  P.tab_up = static_cast<const double*>(S.d_tab_up.p);
  P.n_phi = S.n_phi;
  P.n_q = S.n_q;
  P.up = S.up;
  P.ug = S.ug;
  P.us = S.us;
  P.poisson = S.form;
  P.k_pad = k_pad;
  P.div_nq = FastDiv::make(uint32_t(S.nq_pad / kQPT));
  P.nq_pad = S.nq_pad;
  P.w_type = w_type;
  P.W = W;
  P.flags = static_cast<uint32_t*>(ws.d_flags.p);
  P.error = S.d_error;
  P.tile_ctr = static_cast<uint32_t*>(ws.d_tile_ctr.p);
  P.geom_warps = k1_geom_warps(S);
  const int64_t tile_cells = 32 * P.geom_warps;
  const int64_t tiles = (n + tile_cells - 1) / tile_cells;
  const unsigned grid = unsigned(std::min<int64_t>(tiles, int64_t(device_sm_count()) * MPFEM_K1_MINB));
  launch_geom_typed(w_type, S.ug, S.us, grid, st, P);
  CUDA_OK(cudaGetLastError());
}

// K1: per-cell geometry (tets, geom_w.cuh) or per-point geometry (boxes, geom_box.cuh).
void launch_geom(mpfem_b200_setup_s& S, Workspace& ws, const double* verts, const int32_t* cells,
                 int64_t n, int coef_kind, const double* coef, int64_t coef_stride, void* W,
                 int64_t k_pad, int w_type, cudaStream_t st) {
  if (!S.box)
    return launch_geom_tet(S, ws, verts, cells, n, coef_kind, coef, coef_stride, W, k_pad, w_type, st);
  GeomBoxParams P{};
  P.verts = verts;
  P.cells = cells;
  P.n_cells = n;
  P.coef_kind = coef_kind;
  P.coef = coef;
  P.coef_stride = coef_stride;
  P.rule_w_ug = static_cast<const double*>(S.d_rule_w_ug.p);
  P.ggrad = static_cast<const double*>(S.d_ggrad.p);
  P.tab_up = static_cast<const double*>(S.d_tab_up.p);
  P.n_phi = S.n_phi;
  P.n_q = S.n_q;
  P.nq_pad = S.nq_pad;
  P.n_blocks = S.n_blocks;
  P.k = S.k;
  P.k_pad = k_pad;
  P.up = S.up;
  P.ug = S.ug;
  P.us = S.us;
  P.poisson = S.form;
  P.W = W;
  P.flags = static_cast<uint32_t*>(ws.d_flags.p);
  P.error = S.d_error;
  launch_geom_box(w_type, P, device_sm_count(), st);
  CUDA_OK(cudaGetLastError());
}

void check_coef(const mpfem_b200_setup_s& S, int coef_kind, const double* coef, int64_t stride) {
  if (coef_kind < 0 || coef_kind > 3) throw Error(MPFEM_B200_CONFIG_ERROR, "unknown coefficient kind");
  if (S.box && (coef_kind == 1 || coef_kind == 2))
    throw Error(MPFEM_B200_CONFIG_ERROR, "hexahedra take constant or nodal coefficients");
  if (coef_kind == 2 && (!coef || stride < 4))
    throw Error(MPFEM_B200_CONFIG_ERROR, "affine coefficient needs 4 values per cell");
  if (coef_kind == 3 && (!coef || stride < S.n_phi))
    throw Error(MPFEM_B200_CONFIG_ERROR, "coefficient z needs one entry per basis function");
}

template <bool ACC_F16, int OUTK = 0>
void launch_tc2(const CUtensorMap& ta, const CUtensorMap& tb, const tc::Params& P, cudaStream_t st) {
  static int max_clusters = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // K2's prologue (barriers, TMEM allocation, cluster sync) overlaps K1's tail; the kernel
  // waits (griddepcontrol.wait) before it touches W
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(tc2::THREADS);
  cfg.dynamicSmemBytes = tc2::SMEM_BYTES;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (!max_clusters) {
    CUDA_OK(cudaFuncSetAttribute(tc2::cellmat_tc2_kernel<ACC_F16, OUTK>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM_BYTES));
    cfg.gridDim = dim3(unsigned(device_sm_count()));
    CUDA_OK(cudaOccupancyMaxActiveClusters(&max_clusters, tc2::cellmat_tc2_kernel<ACC_F16, OUTK>, &cfg));
    if (max_clusters < 1) throw Error(MPFEM_B200_RUNTIME_ERROR, "tcgen05 pair kernel does not fit an SM cluster");
  }
  const int64_t tiles = int64_t(P.n_out_tiles) * P.n_cell_tiles;
  cfg.gridDim = dim3(unsigned(2 * std::min<int64_t>(tiles, max_clusters)));
  CUDA_OK(cudaLaunchKernelEx(&cfg, tc2::cellmat_tc2_kernel<ACC_F16, OUTK>, ta, tb, P));
}

template <bool ACC_F16, bool PACKED>
void launch_tcs_t(const CUtensorMap& ta, const CUtensorMap& tb, const tc::Params& P, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    CUDA_OK(cudaFuncSetAttribute(tcs::cellmat_tcs_kernel<ACC_F16, PACKED>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tcs::SMEM_BYTES));
    attr = true;
  }
  const int64_t tiles = int64_t(P.n_out_tiles) * P.n_cell_tiles;
  const unsigned grid = unsigned(std::min<int64_t>(tiles, device_sm_count()));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see launch_tc2
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tcs::THREADS);
  cfg.dynamicSmemBytes = tcs::SMEM_BYTES;
  cfg.stream = st;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, tcs::cellmat_tcs_kernel<ACC_F16, PACKED>, ta, tb, P));
}
// packed: whole cell matrices in one 256-output tile, stored densely (pitch n_out)
template <bool ACC_F16>
void launch_tcs(const CUtensorMap& ta, const CUtensorMap& tb, const tc::Params& P, cudaStream_t st) {
  if (P.n_out_tiles == 1 && P.out_pitch == P.n_out) launch_tcs_t<ACC_F16, true>(ta, tb, P, st);
  else launch_tcs_t<ACC_F16, false>(ta, tb, P, st);
}

// The staged-epilogue kernel (cellmat_tcs.cuh) serves the HBM-bound shapes: short GEMM depth,
// where the output stream, not the operand stream, bounds K2.
bool use_tcs(const mpfem_b200_setup_s& S, const void* out) {
  return S.path == kPathTC && S.k_pad <= 256 && S.n_out_pad % tcs::BO == 0 &&
         (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
}

void launch_gemm(mpfem_b200_setup_s& S, Workspace& ws, void* W, int64_t n, void* out,
                 int64_t out_pitch, cudaStream_t st, const Scatter* sc) {
  if (S.path == kPathTC && !sc && use_tcs(S, out)) {
    const CUtensorMapDataType dt =
        S.w_type == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap ta = make_map_2d(S.d_T.p, dt, uint64_t(S.k_pad), uint64_t(S.n_out_pad), tc::BK, tcs::BM);
    CUtensorMap tb = make_map_2d(W, dt, uint64_t(S.k_pad), uint64_t(n), tc::BK, tcs::BN);
    tc::Params P{};
    P.n_cells = n;
    P.n_out = int(S.n_out);
    P.n_phi = S.n_phi;
    P.rows = static_cast<const int32_t*>(S.d_rows.p);
    P.n_out_tiles = int(S.n_out_pad / tcs::BO);
    P.n_cell_tiles = int((n + tcs::BN - 1) / tcs::BN);
    P.num_k_blocks = int(S.k_pad / tc::BK);
    P.out = static_cast<float*>(out);
    P.out_pitch = out_pitch;
    P.idesc = tc::make_idesc(S.w_type == 1, !S.acc_f16, tcs::BM, tcs::BN);
    P.flags = static_cast<uint32_t*>(ws.d_flags.p);
    if (S.acc_f16) launch_tcs<true>(ta, tb, P, st);
    else launch_tcs<false>(ta, tb, P, st);
  } else if (S.path == kPathTC) {
    const CUtensorMapDataType dt =
        S.w_type == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap ta = make_map_2d(S.d_T.p, dt, uint64_t(S.k_pad), uint64_t(S.n_out_pad), tc::BK, tc2::BMC);
    CUtensorMap tb = make_map_2d(W, dt, uint64_t(S.k_pad), uint64_t(n), tc::BK, tc2::BNC);
    tc::Params P{};
    P.n_cells = n;
    P.n_out = int(S.n_out);
    P.n_phi = S.n_phi;
    P.rows = static_cast<const int32_t*>(S.d_rows.p);
    P.n_out_tiles = int(S.n_out_pad / tc2::BM);
    P.n_cell_tiles = int((n + tc2::BN - 1) / tc2::BN);
    P.num_k_blocks = int(S.k_pad / tc::BK);
    P.out = static_cast<float*>(out);
    P.out_pitch = out_pitch;
    P.idesc = tc::make_idesc(S.w_type == 1, !S.acc_f16, tc2::BM, tc2::BN);
    P.flags = static_cast<uint32_t*>(ws.d_flags.p);
    if (sc) {
      // fused scatter: the local matrices go straight into the CSR values
      P.pos_map = sc->pos_map;
      P.values = sc->values;
      if (sc->fp64) {
        if (S.acc_f16) launch_tc2<true, 2>(ta, tb, P, st);
        else launch_tc2<false, 2>(ta, tb, P, st);
      } else {
        if (S.acc_f16) launch_tc2<true, 1>(ta, tb, P, st);
        else launch_tc2<false, 1>(ta, tb, P, st);
      }
    } else {
      if (S.acc_f16) launch_tc2<true>(ta, tb, P, st);
      else launch_tc2<false>(ta, tb, P, st);
    }
  } else if (S.path == kPathF32) {
    dim3 grid(unsigned((n + sg::BM - 1) / sg::BM), unsigned(S.n_out_pad / sg::BN));
    sg::cellmat_ffma_kernel<<<grid, sg::THREADS, 0, st>>>(
        static_cast<const float*>(W), static_cast<const float*>(S.d_T.p), static_cast<float*>(out),
        n, int(S.n_out), S.n_out_pad, S.k_pad, out_pitch, static_cast<uint32_t*>(ws.d_flags.p));
  } else {
    // fp64 accumulation: DMMA (cellmat_dmma.cuh)
    static bool attr = false;
    if (!attr) {
      CUDA_OK(cudaFuncSetAttribute(dm::cellmat_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   dm::SMEM_BYTES));
      attr = true;
    }
    dim3 grid(unsigned((n + dm::BM - 1) / dm::BM), unsigned(S.n_out_pad / dm::BN));
    dm::cellmat_dmma_kernel<<<grid, dm::THREADS, dm::SMEM_BYTES, st>>>(
        static_cast<const double*>(W), static_cast<const double*>(S.d_T.p), static_cast<double*>(out),
        n, int(S.n_out), S.n_out_pad, S.k_pad, out_pitch, static_cast<uint32_t*>(ws.d_flags.p));
  }
  CUDA_OK(cudaGetLastError());
}

void launch_fused(mpfem_b200_setup_s& S, Workspace& ws, const double* verts, const int32_t* cells,
                  int64_t n, int coef_kind, const double* coef, int64_t coef_stride, float* out,
                  int64_t out_pitch, cudaStream_t st) {
  FusedParams F;
  F.verts = verts;
  F.cells = cells;
  F.n_cells = n;
  F.coef_kind = coef_kind;
  F.coef = coef;
  F.coef_stride = coef_stride;
  F.rule_w_ug = static_cast<const double*>(S.d_rule_w_ug.p);
  F.rule_x = static_cast<const double*>(S.d_rule_x.p);
  F.tab_up = static_cast<const double*>(S.d_tab_up.p);
  F.T = static_cast<const float*>(S.d_T.p);
  F.us = S.us;
  F.up = S.up;
  F.out = out;
  F.out_pitch = out_pitch;
  F.flags = static_cast<uint32_t*>(ws.d_flags.p);
  F.error = S.d_error;
  const unsigned grid = unsigned((n + 127) / 128);
  launch_fused_dispatch(S.p * 100 + S.form * 10 + S.ug, S.us, grid, st, F);
  CUDA_OK(cudaGetLastError());
}

// Reads the FP flags of the call (flags != NULL synchronizes) and raises a CheckError the
// device reported.
void finish_call(mpfem_b200_setup_s& S, Workspace& ws, cudaStream_t st, uint32_t* flags) {
  if (!flags) return;
  uint32_t h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, ws.d_flags.p, 4, cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  *flags |= h;
  S.take_error("");
}

void run_cell_matrices(mpfem_b200_setup_s& S, Workspace& ws, const double* verts,
                       const int32_t* cells, int64_t n, int coef_kind, const double* coef,
                       int64_t coef_stride, void* out, int64_t out_pitch, cudaStream_t st,
                       uint32_t* flags, const Scatter* sc = nullptr) {
  S.take_error(" (reported on the device by an earlier call on this setup)");
  if (S.from_tab) throw Error(MPFEM_B200_CONFIG_ERROR, "this setup takes geometry tensors (mpfem_b200_bilinear_from_geometry)");
  check_coef(S, coef_kind, coef, coef_stride);
  if (n < 0) throw Error(MPFEM_B200_CONFIG_ERROR, "negative cell count");
  if (out_pitch < S.n_out) throw Error(MPFEM_B200_CONFIG_ERROR, "output pitch smaller than n_phi^2");
  if (n > 0 && !verts) throw Error(MPFEM_B200_CONFIG_ERROR, "null vertex buffer");
  S.last_launches = 0;
  ws.n_ev = 0;
  if (flags) CUDA_OK(cudaMemsetAsync(ws.d_flags.p, 0, 4, st));
  if (n > 0 && S.path == kPathFused) {
    if (n * int64_t(S.n_q) >= (int64_t(1) << 40)) throw Error(MPFEM_B200_CONFIG_ERROR, "batch too large");
    ws.mark(S.timing, st);
    launch_fused(S, ws, verts, cells, n, coef_kind, coef, coef_stride, static_cast<float*>(out), out_pitch, st);
    S.last_launches = 1;
    ws.mark(S.timing, st);
    ws.mark(S.timing, st);
  } else if (n > 0) {
    ws.d_W.ensure(size_t(n) * size_t(S.k_pad) * elem_size(S.w_type));
    ws.mark(S.timing, st);
    launch_geom(S, ws, verts, cells, n, coef_kind, coef, coef_stride, ws.d_W.p, S.k_pad, S.w_type, st);
    ws.mark(S.timing, st);
    launch_gemm(S, ws, ws.d_W.p, n, out, out_pitch, st, sc);
    ws.mark(S.timing, st);
    S.last_launches = 2;
  }
  finish_call(S, ws, st, flags);
}

// Compute type of a contraction accumulating at `acc` over operands stored at u_s
// (action.cuh): hardware fp64 / fp32, fp16 through fp32 for fp16 operands, else emulation.
int action_arith(int acc, int us) {
  if (acc == 3) return kArF64;
  if (acc == 2 && us <= 2) return kArF32;
  if (acc == 1 && us == 1) return kArF16;
  return kArGen;
}

template <typename T>
void upload_typed(DevBuf& buf, const std::vector<double>& v) {
  std::vector<T> t(v.begin(), v.end());
  buf.ensure(sizeof(T) * t.size());
  CUDA_OK(cudaMemcpy(buf.p, t.data(), sizeof(T) * t.size(), cudaMemcpyHostToDevice));
}

// make_setup's store tabulation (tab_store: evaluated at u_p, stored at u_s,
// kernels.cpp:86-98) in the two layouts of the action contractions.
void prepare_action(mpfem_b200_setup_s& S) {
  int ap = action_arith(S.up, S.us), aq = action_arith(S.uq, S.us);
  if (ap != aq) ap = aq = kArGen;
  if (ap == S.act_ap) return;
  const std::vector<double>& tab = S.tab_store_host;  // tab_store (kernels.cpp:86-98)
  const int nphi = S.n_phi, nq = S.n_q, nd = S.n_d, n1 = nd * nq;
  std::vector<double> a(size_t(nphi) * n1), c(size_t(n1) * nphi);
  for (int s = 0; s < nd; ++s)
    for (int k = 0; k < nphi; ++k)
      for (int q = 0; q < nq; ++q) {
        const double v = tab[(size_t(s) * nphi + k) * nq + q];
        a[size_t(k) * n1 + s * nq + q] = v;
        c[size_t(s * nq + q) * nphi + k] = v;
      }
  if (ap == kArF32 || ap == kArF16) {
    upload_typed<float>(S.d_act_a, a);
    upload_typed<float>(S.d_act_c, c);
  } else {
    upload_typed<double>(S.d_act_a, a);
    upload_typed<double>(S.d_act_c, c);
  }
  S.act_ap = ap;
  S.act_aq = aq;
}

void run_action(mpfem_b200_setup_s& S, Workspace& ws, const double* verts, const int32_t* cells,
                int64_t n, int coef_kind, const double* coef, int64_t coef_stride, const double* w,
                int64_t w_stride, void* out, int64_t out_pitch, cudaStream_t st, uint32_t* flags,
                const double* G = nullptr, int g_pts = 0) {
  S.take_error(" (reported on the device by an earlier call on this setup)");
  if (S.from_tab && !G) throw Error(MPFEM_B200_CONFIG_ERROR, "this setup takes geometry tensors (mpfem_b200_action_from_geometry)");
  if (G && S.dim != 3) throw Error(MPFEM_B200_CONFIG_ERROR, "the action kernel supports dimension 3");
  if (G && (coef_kind == 1 || coef_kind == 2)) throw Error(MPFEM_B200_CONFIG_ERROR, "geometry tensors take constant or nodal coefficients");
  // one nodal z may be shared by the batch (stride 0), as the reference's action_kernel takes it
  check_coef(S, coef_kind, coef, coef_kind == 3 && coef_stride == 0 ? S.n_phi : coef_stride);
  if (n < 0) throw Error(MPFEM_B200_CONFIG_ERROR, "negative batch");
  if (n > 0 && ((!verts && !G) || !w || !out)) throw Error(MPFEM_B200_CONFIG_ERROR, "null buffer");
  if (w_stride < S.n_phi) throw Error(MPFEM_B200_CONFIG_ERROR, "coefficient w needs one entry per basis function");
  if (out_pitch < S.n_phi) throw Error(MPFEM_B200_CONFIG_ERROR, "output pitch below n_phi");
  prepare_action(S);
  S.last_launches = 0;
  ws.n_ev = 0;
  if (flags) CUDA_OK(cudaMemsetAsync(ws.d_flags.p, 0, 4, st));
  if (n > 0) {
    ActionParams P{};
    P.verts = verts;
    P.cells = cells;
    P.n_cells = n;
    P.coef_kind = coef_kind;
    P.coef = coef;
    P.coef_stride = coef_stride;
    P.w = w;
    P.w_stride = w_stride;
    P.tab_a = S.d_act_a.p;
    P.tab_c = S.d_act_c.p;
    P.tab_up = static_cast<const double*>(S.d_tab_up.p);
    P.rule_w_ug = static_cast<const double*>(S.d_rule_w_ug.p);
    P.rule_x = static_cast<const double*>(S.d_rule_x.p);
    P.n_phi = S.n_phi;
    P.n_q = S.n_q;
    P.n_d = S.n_d;
    P.up = S.up;
    P.ug = S.ug;
    P.uq = S.uq;
    P.us = S.us;
    P.ftz = S.engine == 2;
    P.box = S.box;
    P.ggrad = static_cast<const double*>(S.d_ggrad.p);
    P.G = G;
    P.g_pts = g_pts;
    if (G) P.box = 0;  // geometry given: no per-point evaluation from vertices
    P.out = out;
    P.out_pitch = out_pitch;
    P.flags = static_cast<uint32_t*>(ws.d_flags.p);
    P.error = S.d_error;
    ws.mark(S.timing, st);
    const int rc = launch_action(S.act_ap, S.act_aq, P, device_sm_count(), st);
    if (rc == 2) throw Error(MPFEM_B200_CONFIG_ERROR, "action tile exceeds shared memory");
    if (rc) throw Error(MPFEM_B200_RUNTIME_ERROR, "action kernel attribute setup failed");
    CUDA_OK(cudaGetLastError());
    ws.mark(S.timing, st);
    S.last_launches = 1;
  }
  finish_call(S, ws, st, flags);
}

// kernel_bounds' setup-level inputs (bounds.cpp:60-95): theta_b of the binary64 tabulation
// (Poisson: 3p grad_kappa(k, s) max_q |d_s phi_k|; mass: 3p |phi_k(x_q)|), the binary64 value
// tabulation for nodal coefficients and the basis Lebesgue constant.
void prepare_bounds(mpfem_b200_setup_s& S) {
  if (S.bnd_ready) return;
  const Basis basis = S.box ? box_basis(S.p) : simplex_basis(S.p);
  const BasisCond bc = basis_conditioning(basis, S.rule);
  uint32_t fl = 0;
  const std::vector<double> tab = tabulate(basis, S.rule, 3, 3, S.form == 1, fl);
  const std::vector<double> vals = tabulate(basis, S.rule, 3, 3, false, fl);
  const int nphi = S.n_phi, nq = S.n_q, nd = S.n_d;
  const double dp = 3.0 * S.p;
  std::vector<double> theta(tab.size());
  for (int s = 0; s < nd; ++s)
    for (int k = 0; k < nphi; ++k) {
      const size_t row = (size_t(s) * nphi + k) * nq;
      if (S.form == 1) {
        double peak = 0.0;
        for (int q = 0; q < nq; ++q) peak = std::max(peak, std::fabs(tab[row + q]));
        const double budget = dp * bc.grad_kappa[k][s] * peak;
        for (int q = 0; q < nq; ++q) theta[row + q] = budget;
      } else {
        for (int q = 0; q < nq; ++q) theta[row + q] = dp * std::fabs(tab[row + q]);
      }
    }
  S.d_bnd_theta.ensure(sizeof(double) * theta.size());
  CUDA_OK(cudaMemcpy(S.d_bnd_theta.p, theta.data(), sizeof(double) * theta.size(), cudaMemcpyHostToDevice));
  S.d_bnd_vals.ensure(sizeof(double) * vals.size());
  CUDA_OK(cudaMemcpy(S.d_bnd_vals.p, vals.data(), sizeof(double) * vals.size(), cudaMemcpyHostToDevice));
  if (S.box) {  // degree-1 box gradients at binary64, for the per-point geometry
    const std::vector<double> gg = tabulate(box_basis(1), S.rule, 3, 3, true, fl);
    S.d_bnd_ggrad.ensure(sizeof(double) * gg.size());
    CUDA_OK(cudaMemcpy(S.d_bnd_ggrad.p, gg.data(), sizeof(double) * gg.size(), cudaMemcpyHostToDevice));
  }
  S.bnd_lebesgue = bc.lebesgue;
  for (int a = 0; a < 3; ++a) {
    S.bnd_glebesgue[a] = bc.grad_lebesgue[a];
    S.bnd_gkmax[a] = bc.grad_kappa_max[a];
  }
  S.bnd_ready = true;
}

double unit_roundoff(int f) {
  return f == 0 ? 0x1.0p-8 : (f == 1 ? 0x1.0p-11 : (f == 2 ? 0x1.0p-24 : 0x1.0p-53));
}

}  // namespace

extern "C" {

const char* mpfem_b200_last_error(void) { return g_last_error.c_str(); }
const char* mpfem_b200_version(void) { return "mpfem_b200 0.1 sm_100a"; }

}  // extern "C"

namespace {

// Device state of a setup from its host arrays: value tabulation at u_p (tab_up, n_phi x n_q),
// binary64 tabulation (B64, n_d x n_phi x n_q; may be empty: no GPU bounds), store tabulation
// (Bs, evaluated at u_p, stored at u_s), and the GEMM operand T built from Bs.
void finish_setup(mpfem_b200_setup_s& S, const std::vector<double>& tab_up,
                  const std::vector<double>& B64, const std::vector<double>& Bs) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(MPFEM_B200_RUNTIME_ERROR, "no CUDA device: the B200 path has no CPU fallback");
  CUDA_OK(cudaGetDevice(&S.device));
  S.n_blocks = S.n_d * (S.n_d + 1) / 2;
  S.nq_pad = (S.n_q + kWAlign - 1) / kWAlign * kWAlign;
  S.k = int64_t(S.n_blocks) * S.nq_pad;
  const int64_t kal = S.path == kPathTC ? tc::BK : 16;
  S.k_pad = (S.k + kal - 1) / kal * kal;
  S.n_out = int64_t(S.n_phi) * S.n_phi;
  S.n_out_pad = (S.n_out + 127) / 128 * 128;
  std::vector<int32_t> rows;
  if (S.path == kPathTC) {
    // full output, row-major (i, j): one warp store = 128 contiguous bytes of a cell
    for (int i = 0; i < S.n_phi; ++i)
      for (int j = 0; j < S.n_phi; ++j) rows.push_back(i | (j << 16));
    while (rows.size() % tc2::BM) rows.push_back(-1);
    S.n_out_pad = int64_t(rows.size());
    S.n_rows = int(rows.size());
    S.d_rows.ensure(sizeof(int32_t) * rows.size());
    CUDA_OK(cudaMemcpy(S.d_rows.p, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice));
  }
  uint32_t fl = 0;
  std::vector<double> w_ug(S.n_q);  // fp_cast(omega_q, fp64, u_g) (kernels.cpp:185)
  for (int q = 0; q < S.n_q; ++q) w_ug[q] = host_round(S.rule.weights[q], S.ug, fl);
  auto upload = [](DevBuf& d, const std::vector<double>& v) {
    d.ensure(sizeof(double) * std::max<size_t>(1, v.size()));
    if (!v.empty()) CUDA_OK(cudaMemcpy(d.p, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice));
  };
  upload(S.d_rule_w, S.rule.weights);
  upload(S.d_rule_w_ug, w_ug);
  upload(S.d_rule_x, S.rule.points);
  upload(S.d_tab_up, tab_up);
  upload(S.d_B, B64);
  upload(S.d_Bs, Bs);
  S.tab_store_host = Bs;
  CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&S.h_error), 16, cudaHostAllocMapped));
  std::memset(S.h_error, 0, 16);
  CUDA_OK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.d_error), S.h_error, 0));
  const int64_t t_rows = S.n_out_pad;
  size_t tbytes = size_t(S.k_pad) * size_t(t_rows) * elem_size(S.w_type);
  const double* dB = static_cast<const double*>(S.d_Bs.p);
  if (S.path == kPathFused) {
    // fp32 T[k][o] with k = block * n_q + q (no padding), values rounded to u_s
    const int64_t kf = int64_t(S.n_blocks) * S.n_q;
    S.d_T.ensure(sizeof(float) * size_t(kf) * size_t(S.n_out));
    const int64_t tot = kf * S.n_out;
    build_t_kernel<float><<<unsigned((tot + 255) / 256), 256>>>(dB, S.n_phi, S.n_q, S.n_q, S.n_d, S.us, kf, kf, S.n_out, S.n_out, 0, S.d_T.p);
    CUDA_OK(cudaGetLastError());
    tbytes = 0;
  }
  if (tbytes) S.d_T.ensure(tbytes);
  const int transposed = S.path == kPathTC;
  const int64_t total = tbytes ? S.k_pad * t_rows : 0;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 64)));
  const int32_t* rws = static_cast<const int32_t*>(S.d_rows.p);
  if (total) switch (S.w_type) {
    case 0: build_t_kernel<__half><<<grid, 256>>>(dB, S.n_phi, S.n_q, S.nq_pad, S.n_d, S.us, S.k, S.k_pad, S.n_out, t_rows, transposed, S.d_T.p, rws); break;
    case 1: build_t_kernel<__nv_bfloat16><<<grid, 256>>>(dB, S.n_phi, S.n_q, S.nq_pad, S.n_d, S.us, S.k, S.k_pad, S.n_out, t_rows, transposed, S.d_T.p, rws); break;
    case 2: build_t_kernel<float><<<grid, 256>>>(dB, S.n_phi, S.n_q, S.nq_pad, S.n_d, S.us, S.k, S.k_pad, S.n_out, S.n_out_pad, transposed, S.d_T.p); break;
    default: build_t_kernel<double><<<grid, 256>>>(dB, S.n_phi, S.n_q, S.nq_pad, S.n_d, S.us, S.k, S.k_pad, S.n_out, S.n_out_pad, transposed, S.d_T.p); break;
  }
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaDeviceSynchronize());
}

void init_config(mpfem_b200_setup_s& S, int cell_kind, int p, int form, const int* fmts, int engine) {
  S.p = p;
  S.form = form;
  S.up = fmts[0];
  S.ug = fmts[1];
  S.uq = fmts[2];
  S.us = fmts[3];
  S.engine = engine;
  S.box = cell_kind == 1;
  choose_path(S);
}

}  // namespace

extern "C" {

int mpfem_b200_setup_create(int cell_kind, int dim, int p, int form, int u_p, int u_g, int u_q,
                            int u_s, int engine, int n_batch, mpfem_b200_setup_t* out) {
  return guarded([&] {
    if (!out) throw Error(MPFEM_B200_CONFIG_ERROR, "null output handle");
    int fmts[4] = {u_p, u_g, u_q, u_s};
    validate(cell_kind, dim, p, form, fmts, engine, n_batch);
    auto S = std::make_unique<mpfem_b200_setup_s>();
    init_config(*S, cell_kind, p, form, fmts, engine);
    S->rule = S->box ? box_rule(p) : simplex_rule(p);
    Basis basis = S->box ? box_basis(p) : simplex_basis(p);
    S->n_phi = basis.n_phi;
    S->n_q = S->rule.n_q;
    S->n_d = form ? 3 : 1;
    uint32_t fl = 0;
    std::vector<double> tab_up = tabulate(basis, S->rule, u_p, u_p, false, fl);
    std::vector<double> B = tabulate(basis, S->rule, 3, 3, form == 1, fl);
    // T is built from the reference's own operand values: the tabulation evaluated at u_p
    // and stored at u_s (kernels.cpp:86-98). A format that cannot evaluate the basis (fp16 at
    // p >= 7 raises invalid, as in the reference) therefore yields the reference's NaN
    // matrices instead of silently better ones.
    std::vector<double> Bs = tabulate(basis, S->rule, u_p, u_s, form == 1, fl);
    if (S->box) {  // jacobian() at every rule point: degree-1 box gradients at u_g
      const std::vector<double> gg = tabulate(box_basis(1), S->rule, u_g, u_g, true, fl);
      S->d_ggrad.ensure(sizeof(double) * gg.size());
      CUDA_OK(cudaMemcpy(S->d_ggrad.p, gg.data(), sizeof(double) * gg.size(), cudaMemcpyHostToDevice));
    }
    finish_setup(*S, tab_up, B, Bs);
    *out = S.release();
  });
}

int mpfem_b200_setup_create_tab(int cell_kind, int dim, int p, int form, int u_p, int u_g,
                                int u_q, int u_s, int engine, int n_batch, int n_phi, int n_q,
                                const double* points, const double* weights,
                                const double* tab_store, const double* tab_up,
                                mpfem_b200_setup_t* out) {
  return guarded([&] {
    if (!out) throw Error(MPFEM_B200_CONFIG_ERROR, "null output handle");
    int fmts[4] = {u_p, u_g, u_q, u_s};
    if (dim != 2 && dim != 3) throw Error(MPFEM_B200_CONFIG_ERROR, "dimension must be 2 or 3");
    validate(cell_kind, 3, std::max(1, std::min(p, 4)), form, fmts, engine, n_batch);
    if (n_phi < 1 || n_q < 1 || !points || !weights || !tab_store || !tab_up)
      throw Error(MPFEM_B200_CONFIG_ERROR, "setup from tabulation needs the rule and both tabulations");
    auto S = std::make_unique<mpfem_b200_setup_s>();
    S->from_tab = 1;
    S->dim = dim;
    init_config(*S, cell_kind, p, form, fmts, engine);
    S->n_phi = n_phi;
    S->n_q = n_q;
    S->n_d = form ? dim : 1;
    S->rule.n_q = n_q;
    S->rule.weights.assign(weights, weights + n_q);
    S->rule.points.assign(size_t(3) * n_q, 0.0);
    for (int q = 0; q < n_q; ++q)
      for (int a = 0; a < dim; ++a) S->rule.points[size_t(3) * q + a] = points[size_t(dim) * q + a];
    std::vector<double> tu(tab_up, tab_up + size_t(n_phi) * n_q);
    std::vector<double> bs(tab_store, tab_store + size_t(S->n_d) * n_phi * n_q);
    finish_setup(*S, tu, {}, bs);
    *out = S.release();
  });
}

int mpfem_b200_setup_destroy(mpfem_b200_setup_t setup) {
  return guarded([&] { delete setup; });
}

int mpfem_b200_setup_info(mpfem_b200_setup_t S, int* n_phi, int* n_q, int* n_d, int64_t* k,
                          int64_t* k_pad, int* path) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    if (n_phi) *n_phi = S->n_phi;
    if (n_q) *n_q = S->n_q;
    if (n_d) *n_d = S->n_d;
    if (k) *k = S->k;
    if (k_pad) *k_pad = S->k_pad;
    if (path) *path = S->path;
  });
}

int mpfem_b200_setup_rule(mpfem_b200_setup_t S, double* points, double* weights) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    if (points) std::memcpy(points, S->rule.points.data(), sizeof(double) * 3 * S->n_q);
    if (weights) std::memcpy(weights, S->rule.weights.data(), sizeof(double) * S->n_q);
  });
}

int mpfem_b200_reserve(mpfem_b200_setup_t S, int64_t n_cells, void* stream) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace& ws = S->workspace(static_cast<cudaStream_t>(stream));
    ws.d_W.ensure(size_t(n_cells) * size_t(S->k_pad) * elem_size(S->w_type));
  });
}

int mpfem_b200_synchronize(mpfem_b200_setup_t S, void* stream) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    CUDA_OK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    std::lock_guard<std::mutex> lk(S->mu);
    S->take_error(" (reported on the device by a call on this setup)");
  });
}

int mpfem_b200_cell_matrices(mpfem_b200_setup_t S, const double* verts, const int32_t* cells,
                             int64_t n_cells, int coef_kind, const double* coef,
                             int64_t coef_stride, void* out, int64_t out_pitch, void* stream,
                             uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    run_cell_matrices(*S, S->workspace(st), verts, cells, n_cells, coef_kind, coef, coef_stride, out,
                      out_pitch, st, flags);
  });
}

int mpfem_b200_cell_matrices_scatter(mpfem_b200_setup_t S, const double* verts,
                                     const int32_t* cells, int64_t n_cells, int coef_kind,
                                     const double* coef, int64_t coef_stride,
                                     const int32_t* pos_map, void* values, int values_fmt,
                                     void* stream, uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    if (!pos_map || !values) throw Error(MPFEM_B200_CONFIG_ERROR, "scatter needs pos_map and values");
    if (values_fmt != 2 && values_fmt != 3) throw Error(MPFEM_B200_CONFIG_ERROR, "CSR values must be fp32 or fp64");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace& ws = S->workspace(st);
    if (S->path == kPathTC) {
      Scatter sc;
      sc.pos_map = pos_map;
      sc.values = values;
      sc.fp64 = values_fmt == 3;
      // out is unused by the fused epilogue (pitch n_out keeps the argument checks)
      run_cell_matrices(*S, ws, verts, cells, n_cells, coef_kind, coef, coef_stride, nullptr, S->n_out,
                        st, flags, &sc);
    } else {
      // other paths: stage the local matrices, then the atomic scatter (assemble mode 0)
      const int lf = S->path == kPathF64 ? 3 : 2;
      ws.d_locals.ensure(size_t(n_cells) * size_t(S->n_out) * (lf == 3 ? 8 : 4) + 16);
      run_cell_matrices(*S, ws, verts, cells, n_cells, coef_kind, coef, coef_stride, ws.d_locals.p,
                        S->n_out, st, flags);
      const int rc = mpfem_b200_assemble(ws.d_locals.p, lf, 0, n_cells, S->n_phi, nullptr, 0, pos_map,
                                         nullptr, nullptr, values, values_fmt, 0, 1, nullptr, 0, stream);
      if (rc) throw Error(rc, std::string("atomic scatter: ") + mpfem_b200_last_error());
    }
  });
}

namespace {
// Host-buffer API: H2D of the vertices (and cell table / coefficients) into the stream
// workspace's staging buffers. Returns the device (verts, cells, coef) pointers.
struct Staged {
  const double* verts = nullptr;
  const int32_t* cells = nullptr;
  const double* coef = nullptr;
};
Staged stage_inputs(mpfem_b200_setup_s& S, Workspace& ws, const double* verts, int64_t n_verts,
                    const int32_t* cells, int64_t n_cells, int coef_kind, const double* coef,
                    int64_t coef_stride, cudaStream_t st) {
  Staged d;
  const int nv = S.box ? 8 : 4;
  const size_t vbytes = sizeof(double) * size_t(cells ? n_verts * 3 : n_cells * 3 * nv);
  ws.h_verts.ensure(vbytes + 8);
  if (vbytes) CUDA_OK(cudaMemcpyAsync(ws.h_verts.p, verts, vbytes, cudaMemcpyHostToDevice, st));
  d.verts = static_cast<const double*>(ws.h_verts.p);
  if (cells) {
    ws.h_cells.ensure(sizeof(int32_t) * size_t(n_cells) * nv + 8);
    CUDA_OK(cudaMemcpyAsync(ws.h_cells.p, cells, sizeof(int32_t) * size_t(n_cells) * nv,
                            cudaMemcpyHostToDevice, st));
    d.cells = static_cast<const int32_t*>(ws.h_cells.p);
  }
  if (coef && (coef_kind == 2 || coef_kind == 3)) {
    const int64_t rows = coef_stride == 0 ? 1 : n_cells;
    const int64_t width = coef_stride == 0 ? S.n_phi : coef_stride;
    const size_t cb = sizeof(double) * size_t(rows) * size_t(width);
    ws.h_coef.ensure(cb + 8);
    CUDA_OK(cudaMemcpyAsync(ws.h_coef.p, coef, cb, cudaMemcpyHostToDevice, st));
    d.coef = static_cast<const double*>(ws.h_coef.p);
  }
  return d;
}
}  // namespace

int mpfem_b200_cell_matrices_host(mpfem_b200_setup_t S, const double* verts, int64_t n_verts,
                                  const int32_t* cells, int64_t n_cells, int coef_kind,
                                  const double* coef, int64_t coef_stride, void* out,
                                  int64_t out_pitch, void* stream, uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    check_coef(*S, coef_kind, coef, coef_stride);
    if (n_cells < 0) throw Error(MPFEM_B200_CONFIG_ERROR, "negative cell count");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace& ws = S->workspace(st);
    const Staged d = stage_inputs(*S, ws, verts, n_verts, cells, n_cells, coef_kind, coef, coef_stride, st);
    const size_t esz = S->path == kPathF64 ? 8 : 4;
    const size_t obytes = esz * size_t(n_cells) * size_t(out_pitch);
    ws.h_out.ensure(obytes + 16);
    run_cell_matrices(*S, ws, d.verts, d.cells, n_cells, coef_kind, d.coef, coef_stride, ws.h_out.p,
                      out_pitch, st, flags);
    if (obytes) CUDA_OK(cudaMemcpyAsync(out, ws.h_out.p, obytes, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    S->take_error("");  // the call synchronized: report this call's singular cells now
  });
}

int mpfem_b200_scaled_weights(mpfem_b200_setup_t S, const double* verts, const int32_t* cells,
                              int64_t n_cells, int coef_kind, const double* coef,
                              int64_t coef_stride, double* out, void* stream, uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    check_coef(*S, coef_kind, coef, coef_stride);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace& ws = S->workspace(st);
    S->take_error(" (reported on the device by an earlier call on this setup)");
    CUDA_OK(cudaMemsetAsync(ws.d_flags.p, 0, 4, st));
    if (n_cells > 0)
      launch_geom(*S, ws, verts, cells, n_cells, coef_kind, coef, coef_stride, out, S->k, 3, st);
    finish_call(*S, ws, st, flags);
  });
}

int mpfem_b200_action(mpfem_b200_setup_t S, const double* verts, const int32_t* cells,
                      int64_t n_cells, int coef_kind, const double* coef, int64_t coef_stride,
                      const double* w, int64_t w_stride, void* out, int64_t out_pitch,
                      void* stream, uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    run_action(*S, S->workspace(st), verts, cells, n_cells, coef_kind, coef, coef_stride, w, w_stride,
               out, out_pitch, st, flags);
  });
}

int mpfem_b200_action_host(mpfem_b200_setup_t S, const double* verts, int64_t n_verts,
                           const int32_t* cells, int64_t n_cells, int coef_kind, const double* coef,
                           int64_t coef_stride, const double* w, int64_t w_stride, void* out,
                           int64_t out_pitch, void* stream, uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    // one nodal z may be shared by the batch (stride 0), as in the device entry
    check_coef(*S, coef_kind, coef, coef_kind == 3 && coef_stride == 0 ? S->n_phi : coef_stride);
    if (w_stride < S->n_phi) throw Error(MPFEM_B200_CONFIG_ERROR, "coefficient w needs one entry per basis function");
    if (n_cells < 0) throw Error(MPFEM_B200_CONFIG_ERROR, "negative batch");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace& ws = S->workspace(st);
    const Staged d = stage_inputs(*S, ws, verts, n_verts, cells, n_cells, coef_kind, coef, coef_stride, st);
    // w and the result share one staging buffer: [w (n x w_stride fp64) | v]
    const size_t wbytes = sizeof(double) * size_t(n_cells) * size_t(w_stride);
    const size_t esz = S->uq == 3 ? 8 : 4;
    const size_t obytes = esz * size_t(n_cells) * size_t(out_pitch);
    ws.h_out.ensure(wbytes + obytes + 32);
    char* base = static_cast<char*>(ws.h_out.p);
    if (wbytes) CUDA_OK(cudaMemcpyAsync(base, w, wbytes, cudaMemcpyHostToDevice, st));
    void* dout = base + (wbytes + 15) / 16 * 16;
    run_action(*S, ws, d.verts, d.cells, n_cells, coef_kind, d.coef, coef_stride,
               reinterpret_cast<const double*>(base), w_stride, dout, out_pitch, st, flags);
    if (obytes) CUDA_OK(cudaMemcpyAsync(out, dout, obytes, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    S->take_error("");
  });
}

namespace {
void run_bounds(mpfem_b200_setup_s& S, const double* verts, const int32_t* cells, int64_t n_cells,
                int coef_kind, const double* coef, int64_t coef_stride, const double* w,
                int64_t w_stride, double* out, double* a64, cudaStream_t st) {
  S.take_error(" (reported on the device by an earlier call on this setup)");
  check_coef(S, coef_kind, coef, coef_stride);
  if (n_cells < 0 || (n_cells > 0 && (!verts || !out))) throw Error(MPFEM_B200_CONFIG_ERROR, "null buffer");
  if (w && w_stride < S.n_phi) throw Error(MPFEM_B200_CONFIG_ERROR, "coefficient w needs one entry per basis function");
  if (S.box && w) throw Error(MPFEM_B200_CONFIG_ERROR, "the action bound supports tetrahedra");
  if (S.from_tab) throw Error(MPFEM_B200_CONFIG_ERROR, "GPU bounds need a setup made from (cell, p, config)");
  prepare_bounds(S);
  if (n_cells == 0) return;
  BoundParams P{};
  P.verts = verts;
  P.cells = cells;
  P.n_cells = n_cells;
  P.coef_kind = coef_kind;
  P.coef = coef;
  P.coef_stride = coef_stride;
  P.tab = static_cast<const double*>(S.d_B.p);
  P.theta_b = static_cast<const double*>(S.d_bnd_theta.p);
  P.vals = static_cast<const double*>(S.d_bnd_vals.p);
  P.rule_w = static_cast<const double*>(S.d_rule_w.p);
  P.rule_x = static_cast<const double*>(S.d_rule_x.p);
  P.n_phi = S.n_phi;
  P.n_q = S.n_q;
  P.n_d = S.n_d;
  P.p = S.p;
  P.lebesgue = S.bnd_lebesgue;
  for (int a = 0; a < 3; ++a) {
    P.grad_lebesgue[a] = S.bnd_glebesgue[a];
    P.grad_kappa_max[a] = S.bnd_gkmax[a];
  }
  P.u_p = unit_roundoff(S.up);
  P.u_g = unit_roundoff(S.ug);
  P.u_q = unit_roundoff(S.uq);
  P.u_s = unit_roundoff(S.us);
  P.out = out;
  P.a64 = a64;
  P.w = w;
  P.w_stride = w_stride;
  P.box = S.box;
  P.ggrad64 = static_cast<const double*>(S.d_bnd_ggrad.p);
  P.error = S.d_error;
  const int rc = w ? launch_action_bounds_kernel(P, device_sm_count(), st)
                   : launch_bounds_kernel(P, device_sm_count(), st);
  if (rc) throw Error(MPFEM_B200_RUNTIME_ERROR, "bound kernel attribute setup failed");
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaStreamSynchronize(st));
  S.take_error("");
  S.last_launches = 1;
}
}  // namespace

namespace {
// Stages geometry tensors (and an optional nodal coefficient) of a host-buffer tensor call in
// the stream workspace: [G | z] in h_verts / h_coef.
void stage_tensor(mpfem_b200_setup_s& S, Workspace& ws, const double* G, int n_pts, int64_t n_cells,
                  const double* z, int64_t z_stride, cudaStream_t st, const double** dG,
                  const double** dz) {
  if (n_pts != 1 && n_pts != S.n_q)
    throw Error(MPFEM_B200_CONFIG_ERROR, "geometry needs one entry per cell (affine) or per rule point");
  const int nd = S.form ? S.dim : 1;
  const size_t gb = sizeof(double) * size_t(n_cells) * size_t(n_pts) * size_t(nd * nd);
  ws.h_verts.ensure(gb + 8);
  if (gb) CUDA_OK(cudaMemcpyAsync(ws.h_verts.p, G, gb, cudaMemcpyHostToDevice, st));
  *dG = static_cast<const double*>(ws.h_verts.p);
  *dz = nullptr;
  if (z) {
    const size_t zb = sizeof(double) * size_t(z_stride == 0 ? 1 : n_cells) * size_t(S.n_phi);
    ws.h_coef.ensure(zb + 8);
    if (z_stride == 0 || z_stride == S.n_phi) {
      CUDA_OK(cudaMemcpyAsync(ws.h_coef.p, z, zb, cudaMemcpyHostToDevice, st));
    } else {
      CUDA_OK(cudaMemcpy2DAsync(ws.h_coef.p, sizeof(double) * S.n_phi, z, sizeof(double) * z_stride,
                                sizeof(double) * S.n_phi, size_t(n_cells), cudaMemcpyHostToDevice, st));
    }
    *dz = static_cast<const double*>(ws.h_coef.p);
  }
}
}  // namespace

int mpfem_b200_bilinear_from_geometry(mpfem_b200_setup_t S, const double* G, int n_pts,
                                      int64_t n_cells, const double* z, int64_t z_stride,
                                      void* out, int64_t out_pitch, void* stream, uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    if (n_cells < 0 || (n_cells > 0 && (!G || !out))) throw Error(MPFEM_B200_CONFIG_ERROR, "null buffer");
    if (out_pitch < S->n_out) throw Error(MPFEM_B200_CONFIG_ERROR, "output pitch smaller than n_phi^2");
    if (z_stride != 0 && z_stride < S->n_phi)
      throw Error(MPFEM_B200_CONFIG_ERROR, "coefficient z needs one entry per basis function");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    S->take_error(" (reported on the device by an earlier call on this setup)");
    Workspace& ws = S->workspace(st);
    S->last_launches = 0;
    ws.n_ev = 0;
    CUDA_OK(cudaMemsetAsync(ws.d_flags.p, 0, 4, st));
    if (n_cells > 0) {
      const double *dG, *dz;
      stage_tensor(*S, ws, G, n_pts, n_cells, z, z_stride, st, &dG, &dz);
      ws.d_W.ensure(size_t(n_cells) * size_t(S->k_pad) * elem_size(S->w_type));
      const size_t esz = S->path == kPathF64 ? 8 : 4;
      const size_t obytes = esz * size_t(n_cells) * size_t(out_pitch);
      ws.h_out.ensure(obytes + 16);
      WTensorParams P{};
      P.G = dG;
      P.n_pts = n_pts;
      P.n_cells = n_cells;
      P.z = dz;
      P.z_stride = z_stride == 0 ? 0 : S->n_phi;
      P.rule_w_ug = static_cast<const double*>(S->d_rule_w_ug.p);
      P.tab_up = static_cast<const double*>(S->d_tab_up.p);
      P.n_phi = S->n_phi;
      P.n_q = S->n_q;
      P.nq_pad = S->nq_pad;
      P.nd = S->form ? S->dim : 1;
      P.n_blocks = S->n_blocks;
      P.up = S->up;
      P.ug = S->ug;
      P.us = S->us;
      P.k_pad = S->k_pad;
      P.W = ws.d_W.p;
      P.flags = static_cast<uint32_t*>(ws.d_flags.p);
      ws.mark(S->timing, st);
      launch_w_from_tensor(S->w_type, P, device_sm_count(), st);
      CUDA_OK(cudaGetLastError());
      ws.mark(S->timing, st);
      if (S->path == kPathFused) throw Error(MPFEM_B200_CONFIG_ERROR, "fused path takes vertices");
      launch_gemm(*S, ws, ws.d_W.p, n_cells, ws.h_out.p, out_pitch, st, nullptr);
      ws.mark(S->timing, st);
      S->last_launches = 2;
      CUDA_OK(cudaMemcpyAsync(out, ws.h_out.p, obytes, cudaMemcpyDeviceToHost, st));
    }
    uint32_t h = 0;
    CUDA_OK(cudaMemcpyAsync(&h, ws.d_flags.p, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (flags) *flags |= h;
  });
}

int mpfem_b200_action_from_geometry(mpfem_b200_setup_t S, const double* G, int n_pts,
                                    int64_t n_cells, const double* z, const double* w,
                                    int64_t w_stride, void* out, int64_t out_pitch, void* stream,
                                    uint32_t* flags) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    if (n_cells < 0 || (n_cells > 0 && (!G || !w || !out))) throw Error(MPFEM_B200_CONFIG_ERROR, "null buffer");
    if (w_stride < S->n_phi) throw Error(MPFEM_B200_CONFIG_ERROR, "coefficient w needs one entry per basis function");
    if (out_pitch < S->n_phi) throw Error(MPFEM_B200_CONFIG_ERROR, "output pitch below n_phi");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace& ws = S->workspace(st);
    const double *dG = nullptr, *dz = nullptr;
    if (n_cells > 0) stage_tensor(*S, ws, G, n_pts, n_cells, z, 0, st, &dG, &dz);
    const size_t wbytes = sizeof(double) * size_t(n_cells) * size_t(w_stride);
    const size_t esz = S->uq == 3 ? 8 : 4;
    const size_t obytes = esz * size_t(n_cells) * size_t(out_pitch);
    ws.h_out.ensure(wbytes + obytes + 32);
    char* base = static_cast<char*>(ws.h_out.p);
    if (wbytes) CUDA_OK(cudaMemcpyAsync(base, w, wbytes, cudaMemcpyHostToDevice, st));
    void* dout = base + (wbytes + 15) / 16 * 16;
    uint32_t fl = 0;
    run_action(*S, ws, nullptr, nullptr, n_cells, dz ? 3 : 0, dz, 0, reinterpret_cast<const double*>(base),
               w_stride, dout, out_pitch, st, &fl, dG, n_pts);
    if (obytes) CUDA_OK(cudaMemcpyAsync(out, dout, obytes, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (flags) *flags |= fl;
  });
}

int mpfem_b200_cell_bounds(mpfem_b200_setup_t S, const double* verts, const int32_t* cells,
                           int64_t n_cells, int coef_kind, const double* coef, int64_t coef_stride,
                           double* out, double* a64, void* stream) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    std::lock_guard<std::mutex> lk(S->mu);
    run_bounds(*S, verts, cells, n_cells, coef_kind, coef, coef_stride, nullptr, 0, out, a64,
               static_cast<cudaStream_t>(stream));
  });
}

int mpfem_b200_action_bounds(mpfem_b200_setup_t S, const double* verts, const int32_t* cells,
                             int64_t n_cells, int coef_kind, const double* coef, int64_t coef_stride,
                             const double* w, int64_t w_stride, double* out, double* v64,
                             void* stream) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    if (n_cells > 0 && !w) throw Error(MPFEM_B200_CONFIG_ERROR, "action bound needs w");
    std::lock_guard<std::mutex> lk(S->mu);
    run_bounds(*S, verts, cells, n_cells, coef_kind, coef, coef_stride, w, w_stride, out, v64,
               static_cast<cudaStream_t>(stream));
  });
}

int mpfem_b200_last_launch_count(mpfem_b200_setup_t S) { return S ? S->last_launches : 0; }

int mpfem_b200_set_timing(mpfem_b200_setup_t S, int enable) {
  return guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    std::lock_guard<std::mutex> lk(S->mu);
    S->timing = enable != 0;
    if (S->last_ws) S->last_ws->n_ev = 0;
  });
}

int mpfem_b200_last_timings(mpfem_b200_setup_t S, float* ms, int max_n) {
  int n = 0;
  int st = guarded([&] {
    if (!S) throw Error(MPFEM_B200_CONFIG_ERROR, "null setup");
    std::lock_guard<std::mutex> lk(S->mu);
    Workspace* w = S->last_ws;
    if (!w) return;
    for (int i = 0; i + 1 < w->n_ev && n < max_n; ++i) {
      CUDA_OK(cudaEventSynchronize(w->ev[i + 1]));
      CUDA_OK(cudaEventElapsedTime(&ms[n++], w->ev[i], w->ev[i + 1]));
    }
  });
  return st ? -st : n;
}

}  // extern "C"
