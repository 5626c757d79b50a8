// assembly_host.cu -- host-buffer dof map and assembly (the calls the C++ drop-in shim makes
// for build_dofmap, mesh.hpp:61, and assemble_matrix, assembly.hpp:29-30), on top of the
// device entry points of assembly_capi.cu. Every value and every index is computed on the
// GPU; the host side only stages buffers and validates dof ranges.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mpfem_b200.h"
#include "device_fp.cuh"

using namespace mpfem_b200;

void mpfem_b200_set_last_error(const std::string& msg);

struct mpfem_b200_asm_plan_s {
  int n_loc = 0;
  int64_t n_cells = 0;
  int32_t n_dofs = 0;
  int64_t nnz = 0;
  void* d_cell_dofs = nullptr;
  void* d_row_ptr = nullptr;
  void* d_col_idx = nullptr;
  void* d_pos_map = nullptr;
  void* d_seg_ptr = nullptr;
  void* d_perm = nullptr;
  ~mpfem_b200_asm_plan_s() {
    for (void* p : {d_cell_dofs, d_row_ptr, d_col_idx, d_pos_map, d_seg_ptr, d_perm})
      if (p) cudaFree(p);
  }
};

namespace {

struct HostError {
  int code;
  std::string msg;
};

#define HCUDA(expr)                                                                           \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) throw HostError{4, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
#define HCALL(expr)                                                   \
  do {                                                                \
    const int rc_ = (expr);                                           \
    if (rc_) throw HostError{rc_, std::string(mpfem_b200_last_error())}; \
  } while (0)

template <typename F>
int hguard(F&& f) {
  try {
    mpfem_b200_set_last_error("");
    f();
    return 0;
  } catch (const HostError& e) {
    mpfem_b200_set_last_error(e.msg);
    return e.code;
  }
}

struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t n) { HCUDA(cudaMalloc(&p, std::max<size_t>(n, 16))); }
  ~DevMem() { cudaFree(p); }
};

int n_local_of(int cell_kind, int dim, int p) {
  if (cell_kind == 1) {
    int n = 1;
    for (int a = 0; a < dim; ++a) n *= p + 1;
    return n;
  }
  return dim == 2 ? (p + 1) * (p + 2) / 2 : (p + 1) * (p + 2) * (p + 3) / 6;
}

__global__ void iota_dofs_kernel(int32_t* cd, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    cd[i] = int32_t(i);
}

// assemble_matrix at a 16-bit value format (assembly.cpp:41-69): every contribution cast to
// fmt, then each entry's contributions summed in the reference's order (seg_ptr / perm: cell
// asc, i asc, j asc) with one rounding to fmt per addition. Binary64 carriers; the binary64
// sum of two 16-bit values is exact, so dround gives the reference's fp_add bit for bit.
__global__ void assemble_fmt_kernel(const double* __restrict__ locals, const uint32_t* __restrict__ seg_ptr,
                                    const uint32_t* __restrict__ perm, int64_t nnz, int fmt,
                                    double* __restrict__ values, uint32_t* flags) {
  uint32_t fl = 0;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = seg_ptr[e], en = seg_ptr[e + 1];
    double acc = dround(locals[perm[b]], fmt, fl);
    for (int64_t t = b + 1; t < en; ++t) acc = dadd(acc, dround(locals[perm[t]], fmt, fl), fmt, fl);
    values[e] = acc;
  }
  publish_flags(flags, fl);
}

__global__ void widen_kernel(const float* in, double* out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = double(in[i]);
}

unsigned grid_of(int64_t n) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)));
}

}  // namespace

extern "C" {

int mpfem_b200_dofmap_host(int cell_kind, int dim, int p, int continuous, const int32_t* cells,
                           int64_t n_cells, int64_t n_verts, int32_t* cell_dofs, int32_t* n_dofs,
                           int32_t* max_multiplicity) {
  return hguard([&] {
    if (n_cells < 0 || p < 1 || (dim != 2 && dim != 3)) throw HostError{2, "bad dof map arguments"};
    const int n_loc = n_local_of(cell_kind, dim, p);
    const int64_t n = n_cells * n_loc;
    if (n > (int64_t(1) << 31) - 1) throw HostError{2, "dof map exceeds int range"};
    DevMem dcd(sizeof(int32_t) * size_t(n));
    if (!continuous) {  // discontinuous: every cell numbers its own dofs (mesh.cpp:208-215)
      iota_dofs_kernel<<<grid_of(n), 256>>>(static_cast<int32_t*>(dcd.p), n);
      HCUDA(cudaGetLastError());
      *n_dofs = int32_t(n);
      *max_multiplicity = 1;
    } else {
      if (dim != 3) throw HostError{2, "the B200 continuous dof map supports 3D meshes"};
      const int nv = cell_kind == 1 ? 8 : 4;
      DevMem dcells(sizeof(int32_t) * size_t(n_cells) * nv);
      HCUDA(cudaMemcpy(dcells.p, cells, sizeof(int32_t) * size_t(n_cells) * nv, cudaMemcpyHostToDevice));
      HCALL(mpfem_b200_dofmap_cells(cell_kind, p, static_cast<const int32_t*>(dcells.p), n_cells, n_verts,
                                    static_cast<int32_t*>(dcd.p), n_dofs, max_multiplicity, nullptr));
    }
    HCUDA(cudaMemcpy(cell_dofs, dcd.p, sizeof(int32_t) * size_t(n), cudaMemcpyDeviceToHost));
  });
}

int mpfem_b200_asm_plan_create(const int32_t* cell_dofs, int64_t n_cells, int n_loc, int32_t n_dofs,
                               mpfem_b200_asm_plan_t* out, int64_t* nnz) {
  return hguard([&] {
    if (!out || !nnz || n_cells < 0 || n_loc < 1) throw HostError{2, "bad assembly plan arguments"};
    const int64_t n = n_cells * n_loc;
    for (int64_t i = 0; i < n; ++i)  // checked_dof (assembly.cpp:31-37)
      if (cell_dofs[i] < 0 || cell_dofs[i] >= n_dofs) throw HostError{3, "dof index out of range"};
    auto P = new mpfem_b200_asm_plan_s();
    try {
      P->n_loc = n_loc;
      P->n_cells = n_cells;
      P->n_dofs = n_dofs;
      HCUDA(cudaMalloc(&P->d_cell_dofs, sizeof(int32_t) * std::max<int64_t>(n, 1)));
      HCUDA(cudaMemcpy(P->d_cell_dofs, cell_dofs, sizeof(int32_t) * size_t(n), cudaMemcpyHostToDevice));
      HCUDA(cudaMalloc(&P->d_row_ptr, sizeof(int64_t) * (size_t(n_dofs) + 1)));
      const int32_t* cd = static_cast<const int32_t*>(P->d_cell_dofs);
      int64_t* rp = static_cast<int64_t*>(P->d_row_ptr);
      HCALL(mpfem_b200_csr_pattern(cd, n_cells, n_loc, n_dofs, rp, nullptr, &P->nnz, nullptr));
      HCUDA(cudaMalloc(&P->d_col_idx, sizeof(int32_t) * std::max<int64_t>(P->nnz, 1)));
      HCALL(mpfem_b200_csr_pattern(cd, n_cells, n_loc, n_dofs, rp, static_cast<int32_t*>(P->d_col_idx),
                                   &P->nnz, nullptr));
      const int64_t nk = n * n_loc;
      HCUDA(cudaMalloc(&P->d_pos_map, sizeof(int32_t) * std::max<int64_t>(nk, 1)));
      HCUDA(cudaMalloc(&P->d_seg_ptr, sizeof(uint32_t) * (size_t(P->nnz) + 1)));
      HCUDA(cudaMalloc(&P->d_perm, sizeof(uint32_t) * std::max<int64_t>(nk, 1)));
      HCALL(mpfem_b200_scatter_plan(cd, n_cells, n_loc, n_dofs, rp, static_cast<const int32_t*>(P->d_col_idx),
                                    static_cast<int32_t*>(P->d_pos_map), static_cast<uint32_t*>(P->d_seg_ptr),
                                    static_cast<uint32_t*>(P->d_perm), nullptr));
      HCUDA(cudaDeviceSynchronize());
    } catch (...) {
      delete P;
      throw;
    }
    *nnz = P->nnz;
    *out = P;
  });
}

int mpfem_b200_asm_plan_pattern(mpfem_b200_asm_plan_t P, int64_t* row_ptr, int32_t* col_idx) {
  return hguard([&] {
    if (!P) throw HostError{2, "null plan"};
    if (row_ptr) HCUDA(cudaMemcpy(row_ptr, P->d_row_ptr, sizeof(int64_t) * (size_t(P->n_dofs) + 1), cudaMemcpyDeviceToHost));
    if (col_idx) HCUDA(cudaMemcpy(col_idx, P->d_col_idx, sizeof(int32_t) * size_t(P->nnz), cudaMemcpyDeviceToHost));
  });
}

int mpfem_b200_asm_plan_assemble(mpfem_b200_asm_plan_t P, const double* locals, int fmt,
                                 double* values, uint32_t* flags) {
  return hguard([&] {
    if (!P) throw HostError{2, "null plan"};
    if (fmt < 0 || fmt > 3) throw HostError{2, "unknown value format"};
    const int64_t nk = P->n_cells * P->n_loc * P->n_loc;
    DevMem dl(sizeof(double) * size_t(nk));
    HCUDA(cudaMemcpy(dl.p, locals, sizeof(double) * size_t(nk), cudaMemcpyHostToDevice));
    DevMem dv(sizeof(double) * size_t(P->nnz));
    DevMem df(16);
    HCUDA(cudaMemset(df.p, 0, 16));
    const int64_t* rp = static_cast<const int64_t*>(P->d_row_ptr);
    if (fmt >= 2) {
      HCALL(mpfem_b200_assemble(dl.p, 3, 0, P->n_cells, P->n_loc, rp, P->n_dofs,
                                static_cast<const int32_t*>(P->d_pos_map), static_cast<const uint32_t*>(P->d_seg_ptr),
                                static_cast<const uint32_t*>(P->d_perm), dv.p, fmt, 1, 0, nullptr, 0, nullptr));
      if (fmt == 2) {  // fp32 values -> binary64 carriers (exact)
        DevMem dw(sizeof(double) * size_t(P->nnz));
        widen_kernel<<<grid_of(P->nnz), 256>>>(static_cast<const float*>(dv.p), static_cast<double*>(dw.p), P->nnz);
        HCUDA(cudaGetLastError());
        HCUDA(cudaMemcpy(values, dw.p, sizeof(double) * size_t(P->nnz), cudaMemcpyDeviceToHost));
      } else {
        HCUDA(cudaMemcpy(values, dv.p, sizeof(double) * size_t(P->nnz), cudaMemcpyDeviceToHost));
      }
    } else {
      assemble_fmt_kernel<<<grid_of(P->nnz), 256>>>(static_cast<const double*>(dl.p),
                                                    static_cast<const uint32_t*>(P->d_seg_ptr),
                                                    static_cast<const uint32_t*>(P->d_perm), P->nnz, fmt,
                                                    static_cast<double*>(dv.p), static_cast<uint32_t*>(df.p));
      HCUDA(cudaGetLastError());
      HCUDA(cudaMemcpy(values, dv.p, sizeof(double) * size_t(P->nnz), cudaMemcpyDeviceToHost));
    }
    uint32_t h = 0;
    HCUDA(cudaMemcpy(&h, df.p, 4, cudaMemcpyDeviceToHost));
    if (flags) *flags |= h;
  });
}

int mpfem_b200_asm_plan_destroy(mpfem_b200_asm_plan_t P) {
  delete P;
  return 0;
}

}  // extern "C"
