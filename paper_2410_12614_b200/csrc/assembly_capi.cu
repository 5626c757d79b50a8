// assembly_capi.cu -- C-ABI entry points of the dof map / CSR / scatter path
// (include/mpfem_b200.h), driving the kernels of assembly.cuh. Sorting and scans use CUB.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mpfem_b200.h"
#include "assembly.cuh"

using namespace mpfem_b200;

// shared with capi.cu: the ABI's single thread-local last-error string
void mpfem_b200_set_last_error(const std::string& msg);

namespace {

struct AsmError {
  int code;
  std::string msg;
};

#define ACUDA(expr)                                                                 \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) throw AsmError{4, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

template <typename F>
int aguard(F&& f) {
  try {
    mpfem_b200_set_last_error("");
    f();
    return 0;
  } catch (const AsmError& e) {
    mpfem_b200_set_last_error(e.msg);
    return e.code;
  }
}

// Stream-ordered scratch, released in stream order at scope exit.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {
    static bool pool_set = false;  // keep freed blocks cached: setup calls reuse GBs of scratch
    if (!pool_set) {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      pool_set = true;
    }
  }
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    ACUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

unsigned grid_for(int64_t n, int threads = 256) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32)));
}

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 62 && (int64_t(1) << b) <= maxval) ++b;
  return b;
}

template <typename T>
__global__ void iota_kernel(T* out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = T(i);
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                              T* __restrict__ dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[idx[i]];
}

template <typename T>
T read1(const T* dev, cudaStream_t st) {
  T h{};
  ACUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, st));
  ACUDA(cudaStreamSynchronize(st));
  return h;
}

// dof -> (cell*n_loc + local) lists, ascending position within each dof.
void build_incidence(const int32_t* cell_dofs, int64_t n, int32_t n_dofs, int64_t* inc_ptr,
                     int64_t* inc, Scratch& S) {
  cudaStream_t st = S.st;
  int64_t* counts = S.get<int64_t>(size_t(n_dofs) + 1);
  ACUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t(n_dofs) + 1), st));
  asmb::dof_count_kernel<<<grid_for(n), 256, 0, st>>>(cell_dofs, n, counts);
  size_t tb = 0;
  ACUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, inc_ptr, n_dofs + 1, st));
  void* tmp = S.get<char>(tb);
  ACUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, inc_ptr, n_dofs + 1, st));
  // stable LSD radix sort of (dof, position)
  int32_t* keys_out = S.get<int32_t>(n);
  int64_t* pos_in = S.get<int64_t>(n);
  iota_kernel<<<grid_for(n), 256, 0, st>>>(pos_in, n);
  size_t tb2 = 0;
  const int bits = bits_for(n_dofs);
  ACUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, cell_dofs, keys_out, pos_in, inc, n, 0, bits, st));
  void* tmp2 = S.get<char>(tb2);
  ACUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb2, cell_dofs, keys_out, pos_in, inc, n, 0, bits, st));
}

__global__ void max_diff_kernel(const int64_t* __restrict__ ptr, int32_t n, unsigned long long* out) {
  unsigned long long m = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x)
    m = max(m, (unsigned long long)(ptr[r + 1] - ptr[r]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

int64_t max_count(const int64_t* inc_ptr, int32_t n_dofs, Scratch& S) {
  unsigned long long* out = S.get<unsigned long long>(1);
  ACUDA(cudaMemsetAsync(out, 0, 8, S.st));
  max_diff_kernel<<<grid_for(n_dofs), 256, 0, S.st>>>(inc_ptr, n_dofs, out);
  return int64_t(read1(out, S.st));
}

}  // namespace

extern "C" {

int mpfem_b200_dofmap_cells(int cell_kind, int p, const int32_t* cells, int64_t n_cells,
                            int64_t n_verts, int32_t* cell_dofs, int32_t* n_dofs,
                            int32_t* max_multiplicity, void* stream) {
  return aguard([&] {
    if (cell_kind != 0 && cell_kind != 1) throw AsmError{2, "cell kind must be 0 (tets) or 1 (hexahedra)"};
    const bool box = cell_kind == 1;
    if (p < 1 || p > 8) throw AsmError{2, "element degree must be in [1, 8]"};
    if (n_cells < 1) throw AsmError{2, "dof map needs at least one cell"};
    if (n_verts >= (int64_t(1) << 21) - 1)
      throw AsmError{2, "vertex ids must fit 21 bits for the packed node keys"};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch S(st);
    const int n_phi = box ? (p + 1) * (p + 1) * (p + 1) : (p + 1) * (p + 2) * (p + 3) / 6;
    const int64_t n = n_cells * n_phi;
    if (n >= (int64_t(1) << 31)) throw AsmError{2, "n_cells * n_phi must fit int32"};
    uint64_t* hi = S.get<uint64_t>(n);
    uint64_t* lo = S.get<uint64_t>(n);
    int32_t* pos = S.get<int32_t>(n);
    if (box) {
      asmb::node_keys_box_kernel<<<grid_for(n), 256, 0, st>>>(cells, n_cells, p, hi, lo, pos);
    } else {
      std::vector<int8_t> al(size_t(n_phi) * 4);
      for (int k = 0; k < n_phi; ++k) {
        int a[4];
        asmb::node_alpha(p, k, a);
        for (int t = 0; t < 4; ++t) al[size_t(k) * 4 + t] = int8_t(a[t]);
      }
      int8_t* d_al = S.get<int8_t>(al.size());
      ACUDA(cudaMemcpyAsync(d_al, al.data(), al.size(), cudaMemcpyHostToDevice, st));
      asmb::node_keys_kernel<<<grid_for(n), 256, 0, st>>>(cells, n_cells, p, n_phi, d_al, hi, lo, pos);
    }
    ACUDA(cudaGetLastError());
    // LSD: stable sort by lo, then by hi -> order (hi, lo, position)
    uint64_t* k1 = S.get<uint64_t>(n);
    int32_t* p1 = S.get<int32_t>(n);
    size_t tb = 0;
    ACUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, lo, k1, pos, p1, n, 0, 64, st));
    void* tmp = S.get<char>(tb);
    ACUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, lo, k1, pos, p1, n, 0, 64, st));
    uint64_t* hi_g = S.get<uint64_t>(n);
    gather_kernel<<<grid_for(n), 256, 0, st>>>(hi, p1, n, hi_g);
    uint64_t* hi_s = S.get<uint64_t>(n);
    int32_t* p2 = S.get<int32_t>(n);
    size_t tb2 = 0;
    ACUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, hi_g, hi_s, p1, p2, n, 0, 64, st));
    void* tmp2 = S.get<char>(tb2);
    ACUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb2, hi_g, hi_s, p1, p2, n, 0, 64, st));
    uint64_t* lo_s = S.get<uint64_t>(n);
    gather_kernel<<<grid_for(n), 256, 0, st>>>(lo, p2, n, lo_s);
    // segment heads, first-encounter flags (in position order), numbering
    int32_t* first_flag = S.get<int32_t>(n);
    int32_t* seg_start = S.get<int32_t>(n);
    ACUDA(cudaMemsetAsync(first_flag, 0, sizeof(int32_t) * size_t(n), st));
    asmb::first_flags_kernel<<<grid_for(n), 256, 0, st>>>(hi_s, lo_s, p2, n, first_flag, seg_start);
    int32_t* seg_id = S.get<int32_t>(n);
    int32_t* scan_first = S.get<int32_t>(n);
    size_t tb3 = 0;
    ACUDA(cub::DeviceScan::InclusiveSum(nullptr, tb3, seg_start, seg_id, n, st));
    size_t tb4 = 0;
    ACUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb4, first_flag, scan_first, n, st));
    void* tmp3 = S.get<char>(std::max(tb3, tb4));
    ACUDA(cub::DeviceScan::InclusiveSum(tmp3, tb3, seg_start, seg_id, n, st));
    ACUDA(cub::DeviceScan::ExclusiveSum(tmp3, tb4, first_flag, scan_first, n, st));
    const int32_t n_seg = read1(seg_id + (n - 1), st);
    int32_t* seg_first_pos = S.get<int32_t>(n_seg);
    int32_t* seg_begin = S.get<int32_t>(n_seg);
    asmb::seg_first_kernel<<<grid_for(n), 256, 0, st>>>(p2, seg_start, seg_id, n, seg_first_pos, seg_begin);
    asmb::assign_dofs_kernel<<<grid_for(n), 256, 0, st>>>(p2, seg_id, seg_first_pos, scan_first, n, cell_dofs);
    int32_t* dmax = S.get<int32_t>(1);
    ACUDA(cudaMemsetAsync(dmax, 0, 4, st));
    asmb::seg_len_max_kernel<<<grid_for(n_seg), 256, 0, st>>>(seg_begin, n_seg, n, dmax);
    ACUDA(cudaGetLastError());
    if (n_dofs) *n_dofs = n_seg;
    if (max_multiplicity) *max_multiplicity = read1(dmax, st);
  });
}

int mpfem_b200_dofmap(int p, const int32_t* cells, int64_t n_cells, int64_t n_verts,
                      int32_t* cell_dofs, int32_t* n_dofs, int32_t* max_multiplicity,
                      void* stream) {
  return mpfem_b200_dofmap_cells(0, p, cells, n_cells, n_verts, cell_dofs, n_dofs, max_multiplicity,
                                 stream);
}

int mpfem_b200_csr_pattern(const int32_t* cell_dofs, int64_t n_cells, int n_loc, int32_t n_dofs,
                           int64_t* row_ptr, int32_t* col_idx, int64_t* nnz, void* stream) {
  return mpfem_b200_csr_pattern_cols(cell_dofs, nullptr, n_cells, n_loc, n_dofs, row_ptr, col_idx, nnz,
                                     stream);
}

int mpfem_b200_scatter_plan(const int32_t* cell_dofs, int64_t n_cells, int n_loc, int32_t n_dofs,
                            const int64_t* row_ptr, const int32_t* col_idx, int32_t* pos_map,
                            uint32_t* seg_ptr, uint32_t* perm, void* stream) {
  return mpfem_b200_scatter_plan_cols(cell_dofs, nullptr, n_cells, n_loc, n_dofs, row_ptr, col_idx,
                                      pos_map, seg_ptr, perm, stream);
}

int mpfem_b200_dofmap_table(const int32_t* key_dofs, const int32_t* val_dofs, int64_t n, int32_t* table,
                            void* stream) {
  return aguard([&] {
    if (n < 0) throw AsmError{2, "negative length"};
    if (n == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    asmb::dof_table_kernel<<<grid_for(n), 256, 0, st>>>(key_dofs, val_dofs, n, table);
    ACUDA(cudaGetLastError());
  });
}

int mpfem_b200_dofmap_globalize(const int32_t* local_dofs, int64_t n, const int32_t* table,
                                int32_t n_table, int32_t offset, int32_t* global_dofs, void* stream) {
  return aguard([&] {
    if (n < 0 || n_table < 0) throw AsmError{2, "negative length"};
    if (n == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    asmb::dof_globalize_kernel<<<grid_for(n), 256, 0, st>>>(local_dofs, n, table, n_table, offset, global_dofs);
    ACUDA(cudaGetLastError());
  });
}

int mpfem_b200_csr_find(const int64_t* row_ptr, const int32_t* col_idx, const int32_t* rows,
                        const int32_t* cols, int64_t n, int64_t* pos, void* stream) {
  return aguard([&] {
    if (n < 0) throw AsmError{2, "negative length"};
    if (n == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    asmb::csr_find_kernel<<<grid_for(n), 256, 0, st>>>(row_ptr, col_idx, rows, cols, n, pos);
    ACUDA(cudaGetLastError());
  });
}

int mpfem_b200_incidence(const int32_t* cell_dofs, int64_t n_cells, int n_loc, int32_t n_dofs,
                         int64_t* inc_ptr, int64_t* inc, void* stream) {
  return aguard([&] {
    if (n_loc < 1 || n_dofs < 1) throw AsmError{2, "dof map has no complete cells"};
    Scratch S(static_cast<cudaStream_t>(stream));
    build_incidence(cell_dofs, n_cells * n_loc, n_dofs, inc_ptr, inc, S);
    ACUDA(cudaGetLastError());
  });
}

int mpfem_b200_csr_pattern_cols(const int32_t* cell_dofs, const int32_t* col_dofs, int64_t n_cells,
                                int n_loc, int32_t n_dofs, int64_t* row_ptr, int32_t* col_idx,
                                int64_t* nnz, void* stream) {
  return aguard([&] {
    if (!col_dofs) col_dofs = cell_dofs;
    if (n_loc < 1 || n_dofs < 1) throw AsmError{2, "dof map has no complete cells"};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch S(st);
    const int64_t n = n_cells * n_loc;
    int64_t* inc_ptr = S.get<int64_t>(size_t(n_dofs) + 1);
    int64_t* inc = S.get<int64_t>(n);
    build_incidence(cell_dofs, n, n_dofs, inc_ptr, inc, S);
    const int64_t mmax = max_count(inc_ptr, n_dofs, S);
    if (mmax * n_loc > 8192) throw AsmError{2, "row candidate list exceeds 8192 (multiplicity x n_loc)"};
    // table of hcap slots + a sort list of hcap / 2 >= 32 (the bitonic sort pads to >= 32)
    int hcap = 64;
    while (hcap < 2 * mmax * n_loc) hcap <<= 1;
    const size_t per_warp = size_t(hcap + hcap / 2) * 4;
    const int warps = int(std::max<size_t>(1, std::min<size_t>(8, (48u << 10) / per_warp)));
    const size_t smem = size_t(warps) * per_warp;
    if (smem > (48u << 10))
      ACUDA(cudaFuncSetAttribute(asmb::csr_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const unsigned grid = unsigned(std::min<int64_t>((n_dofs + warps - 1) / warps, 148 * 32));
    int64_t* row_nnz = S.get<int64_t>(size_t(n_dofs) + 1);
    ACUDA(cudaMemsetAsync(row_nnz + n_dofs, 0, sizeof(int64_t), st));
    asmb::csr_rows_kernel<<<grid, warps * 32, smem, st>>>(col_dofs, n_loc, inc_ptr, inc, n_dofs, hcap,
                                                          0, row_nnz, nullptr, nullptr);
    ACUDA(cudaGetLastError());
    size_t tb = 0;
    ACUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, row_nnz, row_ptr, n_dofs + 1, st));
    void* tmp = S.get<char>(tb);
    ACUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, row_nnz, row_ptr, n_dofs + 1, st));
    const int64_t total = read1(row_ptr + n_dofs, st);
    if (total >= (int64_t(1) << 31)) throw AsmError{2, "nnz must fit int32 positions (split the mesh)"};
    if (nnz) *nnz = total;
    if (col_idx) {
      asmb::csr_rows_kernel<<<grid, warps * 32, smem, st>>>(col_dofs, n_loc, inc_ptr, inc, n_dofs,
                                                            hcap, 1, nullptr, row_ptr, col_idx);
      ACUDA(cudaGetLastError());
    }
  });
}

int mpfem_b200_scatter_plan_cols(const int32_t* cell_dofs, const int32_t* col_dofs, int64_t n_cells,
                                 int n_loc, int32_t n_dofs, const int64_t* row_ptr,
                                 const int32_t* col_idx, int32_t* pos_map, uint32_t* seg_ptr,
                                 uint32_t* perm, void* stream) {
  return mpfem_b200_scatter_plan_pull(cell_dofs, col_dofs, n_cells, n_loc, n_dofs, row_ptr, col_idx,
                                      pos_map, seg_ptr, perm, nullptr, stream);
}

int mpfem_b200_scatter_plan_pull(const int32_t* cell_dofs, const int32_t* col_dofs, int64_t n_cells,
                                 int n_loc, int32_t n_dofs, const int64_t* row_ptr,
                                 const int32_t* col_idx, int32_t* pos_map, uint32_t* seg_ptr,
                                 uint32_t* perm, uint16_t* pull_pos, void* stream) {
  return aguard([&] {
    if (!col_dofs) col_dofs = cell_dofs;
    if (n_loc < 1 || n_dofs < 1 || (!pos_map && !pull_pos))
      throw AsmError{2, "scatter plan needs a dof map and pos_map or pull_pos"};
    if (seg_ptr && !pos_map) throw AsmError{2, "the seg_ptr/perm plan needs pos_map"};
    const int64_t nk = n_cells * n_loc * n_loc;
    if (nk > int64_t(UINT32_MAX)) throw AsmError{2, "n_cells * n_loc^2 must fit 32 bits"};
    if ((seg_ptr == nullptr) != (perm == nullptr))
      throw AsmError{2, "deterministic plan needs both seg_ptr and perm"};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch S(st);
    const int64_t n = n_cells * n_loc;
    int64_t* inc_ptr = S.get<int64_t>(size_t(n_dofs) + 1);
    int64_t* inc = S.get<int64_t>(n);
    build_incidence(cell_dofs, n, n_dofs, inc_ptr, inc, S);
    int rcap = 32;
    const int64_t umax = max_count(row_ptr, n_dofs, S);
    while (rcap < umax) rcap <<= 1;
    // pull_pos holds uint16 offsets into 32-row blocks
    if (pull_pos && umax * 32 > 65536) throw AsmError{2, "pull_pos needs rows of at most 2048 entries"};
    const int64_t nnz = read1(row_ptr + n_dofs, st);
    uint32_t* counts = nullptr;
    if (seg_ptr) counts = S.get<uint32_t>(size_t(nnz) + 1);
    auto launch_dims = [&](size_t per_warp, const void* fn) {
      const int warps = int(std::max<size_t>(1, std::min<size_t>(8, (48u << 10) / per_warp)));
      const size_t smem = size_t(warps) * per_warp;
      if (smem > (48u << 10))
        ACUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      const unsigned grid = unsigned(std::min<int64_t>((n_dofs + warps - 1) / warps, 148 * 32));
      return std::make_tuple(grid, warps, smem);
    };
    {
      auto [grid, warps, smem] = launch_dims(size_t(rcap) * 8, reinterpret_cast<const void*>(asmb::plan_pos_kernel));
      asmb::plan_pos_kernel<<<grid, warps * 32, smem, st>>>(col_dofs, n_loc, inc_ptr, inc, row_ptr, col_idx,
                                                            n_dofs, rcap, pos_map, counts, pull_pos);
      ACUDA(cudaGetLastError());
    }
    if (!seg_ptr) return;
    ACUDA(cudaMemsetAsync(counts + nnz, 0, sizeof(uint32_t), st));
    size_t tb = 0;
    ACUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, seg_ptr, nnz + 1, st));
    void* tmp = S.get<char>(tb);
    ACUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, seg_ptr, nnz + 1, st));
    {
      auto [grid, warps, smem] = launch_dims(size_t(rcap) * 4, reinterpret_cast<const void*>(asmb::plan_perm_kernel));
      asmb::plan_perm_kernel<<<grid, warps * 32, smem, st>>>(n_loc, inc_ptr, inc, row_ptr, pos_map, seg_ptr,
                                                             n_dofs, rcap, perm);
      ACUDA(cudaGetLastError());
    }
  });
}

int mpfem_b200_assemble_pull(const void* locals, int locals_fmt, int64_t cell_begin,
                             int64_t cell_end, int n_loc, const int64_t* row_ptr, int32_t n_dofs,
                             const int64_t* inc_ptr, const int64_t* inc, const int32_t* pos_map,
                             const uint16_t* pull_pos, void* values, int fmt, int accumulate,
                             const int32_t* rows, int64_t n_rows, void* stream) {
  return aguard([&] {
    if (locals_fmt != 2 && locals_fmt != 3) throw AsmError{2, "local matrices must be fp32 or fp64"};
    if (fmt != 2 && fmt != 3) throw AsmError{2, "CSR values must be fp32 or fp64"};
    if (cell_end < cell_begin || n_loc < 1) throw AsmError{2, "bad cell range"};
    if (!row_ptr || !inc_ptr || !inc || (!pos_map && !pull_pos))
      throw AsmError{2, "row-pull assembly needs row_ptr, the incidence lists and pos_map or pull_pos"};
    if (pull_pos && reinterpret_cast<uintptr_t>(pull_pos) % 16 != 0)
      throw AsmError{2, "pull_pos must be 16-byte aligned"};
    if (n_dofs == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t per_cell = int64_t(n_loc) * n_loc;
    const size_t esz = locals_fmt == 2 ? 4 : 8;
    const char* base = static_cast<const char*>(locals) - size_t(cell_begin) * size_t(per_cell) * esz;
    const int init = accumulate ? 0 : 1;
    const int64_t nr = rows ? n_rows : int64_t(n_dofs);
    if (nr == 0) return;
    if (n_loc > 256) throw AsmError{2, "row-pull assembly supports n_loc <= 256"};
    const int64_t blocks32 = (nr + 31) / 32;  // a warp takes 32-row blocks
    // elements per cp.async: 4 / 2 / 1 by n_loc and the arrays' alignment
    auto aligned = [](const void* q, size_t a) { return reinterpret_cast<uintptr_t>(q) % a == 0; };
    int vec = 1;
    const bool p16 = pull_pos != nullptr;
    if (n_loc % 4 == 0 && aligned(base, 16) && (p16 || aligned(pos_map, 16))) vec = 4;
    else if (n_loc % 2 == 0 && aligned(base, std::min<size_t>(16, 2 * esz)) && (p16 || aligned(pos_map, 8))) vec = 2;
// Shared-memory carveout of the pull kernel: 75 % leaves the L1 large enough to keep the partly
// used sectors of neighbouring local rows until the next CSR row asks for them (measured at config 4,
// P3 fp32: carveout 100 % 9.3 ms, 75 % 6.0 ms, 50 % 6.5 ms, 25 % 12.1 ms).
#ifndef MPFEM_PULL_CARVEOUT
#define MPFEM_PULL_CARVEOUT 75
#endif
#define MPFEM_PULL_CARVE(...) ACUDA(cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributePreferredSharedMemoryCarveout, MPFEM_PULL_CARVEOUT));
#define MPFEM_PULL_P(TL, TV, CH, VEC, P16)                                                         \
  {                                                                                                \
    constexpr size_t smem = asmb::kPullWarps * asmb::pull_warp_bytes<TL, TV, CH, P16>();           \
    static bool attr = false;                                                                      \
    static int per_sm = 1;                                                                         \
    if (!attr) {                                                                                   \
      ACUDA(cudaFuncSetAttribute(asmb::assemble_pull_kernel<TL, TV, CH, VEC, P16>,                 \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));         \
      MPFEM_PULL_CARVE(asmb::assemble_pull_kernel<TL, TV, CH, VEC, P16>)                           \
      ACUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                         \
          &per_sm, asmb::assemble_pull_kernel<TL, TV, CH, VEC, P16>, asmb::kPullWarps * 32, smem)); \
      attr = true;                                                                                 \
    }                                                                                              \
    const unsigned grid = unsigned(std::max<int64_t>(                                              \
        1, std::min<int64_t>((blocks32 + asmb::kPullWarps - 1) / asmb::kPullWarps,                 \
                             int64_t(148) * std::max(per_sm, 1))));                                \
    asmb::assemble_pull_kernel<TL, TV, CH, VEC, P16><<<grid, asmb::kPullWarps * 32, smem, st>>>(   \
        reinterpret_cast<const TL*>(base), n_loc, row_ptr, inc_ptr, inc, pos_map, pull_pos, rows,  \
        nr, cell_begin, cell_end, init, static_cast<TV*>(values));                                 \
  }
#define MPFEM_PULL_V(TL, TV, CH, VEC)                                                              \
  {                                                                                                \
    if (p16) MPFEM_PULL_P(TL, TV, CH, VEC, true)                                                   \
    else MPFEM_PULL_P(TL, TV, CH, 1, false) /* pos_map fallback: 4-byte copies only */             \
  }
#define MPFEM_PULL_J(TL, TV, CH)                                                                   \
  {                                                                                                \
    if (vec == 4) MPFEM_PULL_V(TL, TV, CH, 4)                                                      \
    else if (vec == 2) MPFEM_PULL_V(TL, TV, CH, 2)                                                 \
    else MPFEM_PULL_V(TL, TV, CH, 1)                                                               \
  }
#define MPFEM_PULL(TL, TV)                                                                         \
  {                                                                                                \
    if (n_loc <= 64) MPFEM_PULL_J(TL, TV, 128)                                                     \
    else MPFEM_PULL_J(TL, TV, 256)                                                                 \
  }
    if (locals_fmt == 2 && fmt == 2) MPFEM_PULL(float, float)
    else if (locals_fmt == 2) MPFEM_PULL(float, double)
    else if (fmt == 2) MPFEM_PULL(double, float)
    else MPFEM_PULL(double, double)
#undef MPFEM_PULL_V
#undef MPFEM_PULL_P
#undef MPFEM_PULL_J
#undef MPFEM_PULL
    ACUDA(cudaGetLastError());
  });
}

int mpfem_b200_assemble(const void* locals, int locals_fmt, int64_t cell_begin, int64_t cell_end,
                        int n_loc, const int64_t* row_ptr, int32_t n_dofs, const int32_t* pos_map,
                        const uint32_t* seg_ptr, const uint32_t* perm, void* values, int fmt,
                        int mode, int accumulate, const int32_t* rows, int64_t n_rows,
                        void* stream) {
  return aguard([&] {
    if (locals_fmt != 2 && locals_fmt != 3) throw AsmError{2, "local matrices must be fp32 or fp64"};
    if (fmt != 2 && fmt != 3) throw AsmError{2, "CSR values must be fp32 or fp64"};
    if (mode != 0 && mode != 1) throw AsmError{2, "assembly mode must be 0 (atomic) or 1 (deterministic)"};
    if (cell_end < cell_begin || n_loc < 1) throw AsmError{2, "bad cell range"};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t per_cell = int64_t(n_loc) * n_loc;
    // locals[0] is cell_begin's matrix: rebase so kernels index by global local-entry id
    const size_t esz = locals_fmt == 2 ? 4 : 8;
    const char* base = static_cast<const char*>(locals) - size_t(cell_begin) * size_t(per_cell) * esz;
    if (mode == 0) {
      if (!pos_map) throw AsmError{2, "atomic assembly needs the scatter plan's pos_map"};
      if (!accumulate) {
        const int64_t nnz = read1(row_ptr + n_dofs, st);
        ACUDA(cudaMemsetAsync(values, 0, size_t(nnz) * (fmt == 2 ? 4 : 8), st));
      }
      const int64_t kb = cell_begin * per_cell, ke = cell_end * per_cell;
      const unsigned grid = grid_for(ke - kb);
      if (locals_fmt == 2 && fmt == 2)
        asmb::assemble_atomic_kernel<float, float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(base), pos_map, kb, ke, static_cast<float*>(values));
      else if (locals_fmt == 2)
        asmb::assemble_atomic_kernel<float, double><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(base), pos_map, kb, ke, static_cast<double*>(values));
      else if (fmt == 2)
        asmb::assemble_atomic_kernel<double, float><<<grid, 256, 0, st>>>(reinterpret_cast<const double*>(base), pos_map, kb, ke, static_cast<float*>(values));
      else
        asmb::assemble_atomic_kernel<double, double><<<grid, 256, 0, st>>>(reinterpret_cast<const double*>(base), pos_map, kb, ke, static_cast<double*>(values));
    } else {
      if (!seg_ptr || !perm) throw AsmError{2, "deterministic assembly needs the scatter plan (seg_ptr, perm)"};
      const int init = accumulate ? 0 : 1;
      if (rows) {
        if (n_rows == 0) return;
        const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((n_rows + 7) / 8, 148 * 64)));
#define MPFEM_SEG_ROWS(TL, TV) asmb::assemble_seg_rows_kernel<TL, TV><<<grid, 256, 0, st>>>(reinterpret_cast<const TL*>(base), per_cell, row_ptr, seg_ptr, perm, rows, n_rows, cell_begin, cell_end, init, static_cast<TV*>(values))
        if (locals_fmt == 2 && fmt == 2) MPFEM_SEG_ROWS(float, float);
        else if (locals_fmt == 2) MPFEM_SEG_ROWS(float, double);
        else if (fmt == 2) MPFEM_SEG_ROWS(double, float);
        else MPFEM_SEG_ROWS(double, double);
#undef MPFEM_SEG_ROWS
      } else {
        const int64_t nnz = read1(row_ptr + n_dofs, st);
        // block-staged segment gather (bitwise the per-entry sequential sum)
        const size_t vsz = fmt == 2 ? 4 : 8;
        const int cap = int((asmb::kSegSmem - asmb::kSegHeadBytes) / vsz);
        const size_t smem = asmb::kSegHeadBytes + size_t(cap) * vsz;
        const unsigned grid = unsigned(std::max<int64_t>(
            1, std::min<int64_t>((nnz + asmb::kSegBlock - 1) / asmb::kSegBlock, 148 * asmb::kSegCtasPerSm)));
#define MPFEM_SEG(TL, TV)                                                                          \
  asmb::assemble_seg_block_kernel<TL, TV><<<grid, 256, smem, st>>>(                                \
      reinterpret_cast<const TL*>(base), per_cell, seg_ptr, perm, nnz, cell_begin, cell_end, init, \
      cap, static_cast<TV*>(values))
        if (locals_fmt == 2 && fmt == 2) MPFEM_SEG(float, float);
        else if (locals_fmt == 2) MPFEM_SEG(float, double);
        else if (fmt == 2) MPFEM_SEG(double, float);
        else MPFEM_SEG(double, double);
#undef MPFEM_SEG
      }
    }
    ACUDA(cudaGetLastError());
  });
}

}  // extern "C"
