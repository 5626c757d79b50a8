// assembly.cuh -- dof map, CSR pattern, incidence and scatter-add on the device.
//
// Reference: build_dofmap (mesh.cpp:204-298), assemble_matrix (assembly.cpp:41-88).
//
// Dof map. A Lagrange node of a tet is a lattice point with barycentric multi-index
// alpha (sum p) over the cell's 4 vertices; two cells' nodes coincide exactly when they
// lie on the same sub-simplex with the same alpha on its vertices. The key of node k of
// cell c is the sorted list of (vertex id, alpha_v) over alpha_v > 0, packed into 128 bits.
// Sorting the (key, position) pairs stably groups coincident nodes with the first
// encounter (cell asc, k asc) first; a scan over the "first occurrence" flags in position
// order numbers the dofs in first-encounter order -- the reference's numbering.
//
// CSR pattern. Row r's columns are the dofs of every cell incident to r (from the
// incidence lists), sorted and deduplicated per row by one warp in shared memory; the
// result is the reference COO key set in (row, col) order.
//
// Scatter. Deterministic mode is row-centric: one warp per row walks the row's incident
// (cell, local i) pairs in ascending cell order and adds local row i into the row's
// accumulators (lane j handles column dof(c, j)), so every CSR entry is the sequential
// ascending-cell sum of the reference, bit for bit. Atomic mode issues one red.global.add
// per local entry at the binary-searched CSR position.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mpfem_b200 {
namespace asmb {

// Multi-index of local node k for degree p, in build_basis order (elements.cpp:96-115):
// (a1, a2, a3) with a1 fastest, a0 = p - a1 - a2 - a3.
__host__ __device__ inline void node_alpha(int p, int k, int al[4]) {
  int idx = 0;
  for (int a3 = 0; a3 <= p; ++a3)
    for (int a2 = 0; a2 <= p; ++a2)
      for (int a1 = 0; a1 <= p; ++a1) {
        if (a1 + a2 + a3 > p) continue;
        if (idx == k) {
          al[0] = p - a1 - a2 - a3;
          al[1] = a1;
          al[2] = a2;
          al[3] = a3;
          return;
        }
        ++idx;
      }
}

// 128-bit node key: hi = up to 3 vertex ids (+1, 21 bits each, ascending), lo = alphas of
// those vertices (8 bits each) | sub-simplex size; interior nodes (4 vertices, p >= 4)
// are unique to their cell: hi = 2^63 | cell, lo = k.
__global__ void node_keys_kernel(const int32_t* __restrict__ cells, int64_t n_cells, int p,
                                 int n_phi, const int8_t* __restrict__ alphas /* n_phi x 4 */,
                                 uint64_t* __restrict__ key_hi, uint64_t* __restrict__ key_lo,
                                 int32_t* __restrict__ pos) {
  const int64_t total = n_cells * n_phi;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = i / n_phi;
    const int k = int(i % n_phi);
    int v[4], a[4], n = 0;
    for (int t = 0; t < 4; ++t) {
      const int al = alphas[k * 4 + t];
      if (al > 0) {
        v[n] = cells[c * 4 + t];
        a[n] = al;
        ++n;
      }
    }
    uint64_t hi, lo;
    if (n == 4) {
      hi = (uint64_t(1) << 63) | uint64_t(c);
      lo = uint64_t(k);
    } else {
      // sort the (vertex, alpha) pairs by vertex id (n <= 3)
      for (int x = 1; x < n; ++x)
        for (int y = x; y > 0 && v[y - 1] > v[y]; --y) {
          int tv = v[y]; v[y] = v[y - 1]; v[y - 1] = tv;
          int ta = a[y]; a[y] = a[y - 1]; a[y - 1] = ta;
        }
      hi = 0;
      lo = uint64_t(n);
      for (int t = 0; t < n; ++t) {
        hi |= uint64_t(v[t] + 1) << (21 * (2 - t));
        lo |= uint64_t(a[t]) << (8 * (t + 1));
      }
    }
    key_hi[i] = hi;
    key_lo[i] = lo;
    pos[i] = int32_t(i);
  }
}

// flags[pos] = 1 where the sorted entry starts a new key (first encounter).
__global__ void first_flags_kernel(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo,
                                   const int32_t* __restrict__ pos, int64_t n,
                                   int32_t* __restrict__ first_flag, int32_t* __restrict__ seg_start) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool head = i == 0 || hi[i] != hi[i - 1] || lo[i] != lo[i - 1];
    seg_start[i] = head ? 1 : 0;
    if (head) first_flag[pos[i]] = 1;
  }
}

// cell_dofs[pos] = dof id of the segment (the scan value at its first position); also
// segment lengths for the multiplicity.
__global__ void assign_dofs_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ seg_id,
                                   const int32_t* __restrict__ seg_first_pos,
                                   const int32_t* __restrict__ scan_first, int64_t n,
                                   int32_t* __restrict__ cell_dofs) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t s = seg_id[i] - 1;  // inclusive scan of heads -> 1-based
    cell_dofs[pos[i]] = scan_first[seg_first_pos[s]];
  }
}

__global__ void seg_first_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ seg_start,
                                 const int32_t* __restrict__ seg_id, int64_t n,
                                 int32_t* __restrict__ seg_first_pos, int32_t* __restrict__ seg_begin) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (seg_start[i]) {
      seg_first_pos[seg_id[i] - 1] = pos[i];
      seg_begin[seg_id[i] - 1] = int32_t(i);
    }
  }
}

__global__ void seg_len_max_kernel(const int32_t* __restrict__ seg_begin, int64_t n_seg, int64_t n,
                                   int32_t* __restrict__ max_len) {
  int32_t m = 0;
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n_seg;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t end = (s + 1 < n_seg) ? seg_begin[s + 1] : n;
    m = max(m, int32_t(end - seg_begin[s]));
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(max_len, m);
}

// Incidence: counts per dof, then (after a scan) positions. inc holds cell*n_loc + local
// in ascending position order, i.e. ascending (cell, local), per dof.
__global__ void dof_count_kernel(const int32_t* __restrict__ cell_dofs, int64_t n,
                                 int64_t* __restrict__ counts) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&counts[cell_dofs[i]]), 1ull);
}

// ---------------------------------------------------------------- CSR pattern
// One warp per row; shared-memory buffer of `cap` ints per warp. Pass 0 writes the unique
// count of row r to row_nnz[r]; pass 1 writes the sorted unique columns at row_ptr[r].
__device__ __forceinline__ void warp_bitonic_sort(int32_t* buf, int cap) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= cap; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < cap / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const int32_t a = buf[lo], b = buf[hi];
        if ((a > b) == up) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncwarp();
    }
  }
}

__global__ void csr_rows_kernel(const int32_t* __restrict__ cell_dofs, int n_loc,
                                const int64_t* __restrict__ inc_ptr, const int64_t* __restrict__ inc,
                                int32_t n_rows, int cap, int pass, int64_t* __restrict__ row_nnz,
                                const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx) {
  extern __shared__ int32_t sbuf[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* buf = sbuf + w * cap;
  for (int64_t r = int64_t(blockIdx.x) * warps + w; r < n_rows; r += int64_t(gridDim.x) * warps) {
    const int64_t b = inc_ptr[r], e = inc_ptr[r + 1];
    const int64_t total = (e - b) * n_loc;
    for (int i = lane; i < cap; i += 32) {
      int32_t v = INT32_MAX;
      if (i < total) {
        const int64_t pk = inc[b + i / n_loc];
        const int64_t cell = pk / n_loc;
        v = cell_dofs[cell * n_loc + (i % n_loc)];
      }
      buf[i] = v;
    }
    __syncwarp();
    warp_bitonic_sort(buf, cap);
    // unique count (and write)
    int64_t base = pass ? row_ptr[r] : 0;
    int64_t count = 0;
    for (int i0 = 0; i0 < cap; i0 += 32) {
      const int i = i0 + lane;
      const int32_t v = buf[i];
      const bool keep = v != INT32_MAX && (i == 0 || buf[i - 1] != v);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (pass && keep) col_idx[base + count + __popc(m & ((1u << lane) - 1u))] = v;
      count += __popc(m);
    }
    if (!pass && lane == 0) row_nnz[r] = count;
    __syncwarp();
  }
}

// ---------------------------------------------------------------- scatter-add
template <typename TL, typename TV>
__device__ __forceinline__ TV cast_value(TL x) {
  if constexpr (sizeof(TV) == 4 && sizeof(TL) == 8) return __double2float_rn(x);
  else return TV(x);
}

__device__ __forceinline__ int64_t find_col(const int32_t* __restrict__ cols, int64_t lo, int64_t hi,
                                            int32_t col) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cols[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Deterministic: one warp per row (rows list or all rows). The row's columns and its
// accumulators live in shared memory; the incident local rows are fetched in bulk
// (all lanes, independent loads, positions binary-searched in shared memory) and then
// added strictly in ascending incidence order, so each CSR entry is the reference's
// sequential ascending-cell sum. init != 0 starts every entry at -0.0 (the first
// contribution is then taken exactly, as the reference's cast); otherwise the sum
// continues from the current values (multi-GPU prefix partial sums).
template <typename TL, typename TV>
__global__ void assemble_det_kernel(const TL* __restrict__ locals, int n_loc,
                                    const int32_t* __restrict__ cell_dofs,
                                    const int64_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ col_idx,
                                    const int64_t* __restrict__ inc_ptr, const int64_t* __restrict__ inc,
                                    const int32_t* __restrict__ rows, int64_t n_rows,
                                    int64_t cell_begin, int64_t cell_end, int init,
                                    TV* __restrict__ values, int cap_cols, int cap_buf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = size_t(cap_cols) * (sizeof(int32_t) + sizeof(TV)) +
                          size_t(cap_buf) * (sizeof(int32_t) + sizeof(TV));
  unsigned char* base = smem_raw + w * per_warp;
  TV* acc = reinterpret_cast<TV*>(base);
  TV* bv = reinterpret_cast<TV*>(base + size_t(cap_cols) * sizeof(TV));
  int32_t* scol = reinterpret_cast<int32_t*>(base + size_t(cap_cols + cap_buf) * sizeof(TV));
  int32_t* bx = scol + cap_cols;
  const int chunk = cap_buf / n_loc;  // incidences per bulk fetch
  for (int64_t ri = int64_t(blockIdx.x) * warps + w; ri < n_rows; ri += int64_t(gridDim.x) * warps) {
    const int64_t r = rows ? rows[ri] : ri;
    const int64_t cb = row_ptr[r];
    const int nr = int(row_ptr[r + 1] - cb);
    for (int x = lane; x < nr; x += 32) {
      scol[x] = col_idx[cb + x];
      acc[x] = init ? TV(-0.0) : values[cb + x];
    }
    __syncwarp();
    const int64_t ib = inc_ptr[r], ie = inc_ptr[r + 1];
    for (int64_t t0 = ib; t0 < ie; t0 += chunk) {
      const int nt = int((ie - t0) < int64_t(chunk) ? (ie - t0) : int64_t(chunk));
      const int nf = nt * n_loc;
      for (int f = lane; f < nf; f += 32) {
        const int t = f / n_loc, j = f - t * n_loc;
        const int64_t pk = inc[t0 + t];
        const int64_t cell = pk / n_loc;
        int32_t x = -1;
        TV v = TV(0);
        if (cell >= cell_begin && cell < cell_end) {
          const int i = int(pk - cell * n_loc);
          const int32_t col = cell_dofs[cell * n_loc + j];
          v = cast_value<TL, TV>(locals[(cell * n_loc + i) * n_loc + j]);
          int lo = 0, hi = nr;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (scol[mid] < col) lo = mid + 1;
            else hi = mid;
          }
          x = lo;
        }
        bx[f] = x;
        bv[f] = v;
      }
      __syncwarp();
      for (int t = 0; t < nt; ++t) {
        for (int j = lane; j < n_loc; j += 32) {
          const int f = t * n_loc + j;
          const int32_t x = bx[f];
          if (x >= 0) acc[x] = acc[x] + bv[f];
        }
        __syncwarp();
      }
    }
    for (int x = lane; x < nr; x += 32) values[cb + x] = acc[x];
    __syncwarp();
  }
}

// Atomic: one warp per (cell, local row i); lanes over j.
template <typename TL, typename TV>
__global__ void assemble_atomic_kernel(const TL* __restrict__ locals, int n_loc,
                                       const int32_t* __restrict__ cell_dofs,
                                       const int64_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col_idx, int64_t cell_begin,
                                       int64_t cell_end, TV* __restrict__ values) {
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = (cell_end - cell_begin) * n_loc;
  for (int64_t t = int64_t(blockIdx.x) * warps + w; t < total; t += int64_t(gridDim.x) * warps) {
    const int64_t cell = cell_begin + t / n_loc;
    const int i = int(t % n_loc);
    const int32_t r = cell_dofs[cell * n_loc + i];
    const int64_t cb = row_ptr[r], ce = row_ptr[r + 1];
    const TL* lrow = locals + (cell * n_loc + i) * n_loc;
    for (int j = lane; j < n_loc; j += 32) {
      const int32_t col = cell_dofs[cell * n_loc + j];
      const int64_t x = find_col(col_idx, cb, ce, col);
      atomicAdd(&values[x], cast_value<TL, TV>(lrow[j]));
    }
  }
}

}  // namespace asmb
}  // namespace mpfem_b200
