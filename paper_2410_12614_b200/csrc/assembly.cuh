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
// Scatter plan (precomputed once per mesh, like the pattern): pos_map gives the CSR
// position of every local entry; perm lists the local entries sorted stably by that
// position (seg_ptr: nnz + 1 offsets into perm, uint32 -- n_cells n_loc^2 < 2^32 is required
// anyway), so within an entry's segment they appear in the reference's order (cell asc,
// i asc, j asc). Deterministic mode sums each segment sequentially at the value format --
// the reference's sum bit for bit; atomic mode issues one red.global.add per local entry.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "l2_hints.cuh"

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

// Node keys of hexahedral (box) cells: cells n x 8 vertex ids in lattice-bit order (mesh.hpp:
// 15-24), local node k = lattice point (c0, c1, c2) in [0, p]^3, axis 0 fastest (elements.cpp:
// 50-87). The node lies on the sub-entity spanned by its non-boundary axes; its key is that
// entity's vertices and the node's coordinates in a frame fixed by the vertex ids alone, so
// every cell sharing the entity computes the same key whatever its local orientation:
//   vertex: (v);  edge: (min, max, t measured from min);  face: (origin = min id, its two
//   face neighbours ordered by id, coordinates along those);  interior: (cell, k).
__global__ void node_keys_box_kernel(const int32_t* __restrict__ cells, int64_t n_cells, int p,
                                     uint64_t* __restrict__ key_hi, uint64_t* __restrict__ key_lo,
                                     int32_t* __restrict__ pos) {
  const int n1 = p + 1, n_phi = n1 * n1 * n1;
  const int64_t total = n_cells * n_phi;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = i / n_phi;
    const int k = int(i % n_phi);
    const int co[3] = {k % n1, (k / n1) % n1, k / (n1 * n1)};
    int fixed_bits = 0, free_ax[3], nf = 0;
    for (int a = 0; a < 3; ++a) {
      if (co[a] == p) fixed_bits |= 1 << a;
      else if (co[a] != 0) free_ax[nf++] = a;
    }
    auto vid = [&](int b) { return uint64_t(cells[c * 8 + b]) + 1; };
    uint64_t hi, lo;
    if (nf == 3) {
      hi = (uint64_t(1) << 63) | uint64_t(c);
      lo = uint64_t(k);
    } else if (nf == 0) {
      hi = vid(fixed_bits);
      lo = 1;
    } else if (nf == 1) {
      const int a = free_ax[0];
      uint64_t va = vid(fixed_bits), vb = vid(fixed_bits | (1 << a));
      int t = co[a];
      if (vb < va) {
        const uint64_t tmp = va; va = vb; vb = tmp;
        t = p - t;
      }
      hi = (va << 21) | vb;
      lo = 2 | (uint64_t(t) << 8);
    } else {
      const int a1 = free_ax[0], a2 = free_ax[1];
      uint64_t f[2][2];
      for (int s1 = 0; s1 < 2; ++s1)
        for (int s2 = 0; s2 < 2; ++s2) f[s1][s2] = vid(fixed_bits | (s1 << a1) | (s2 << a2));
      int o1 = 0, o2 = 0;
      for (int s1 = 0; s1 < 2; ++s1)
        for (int s2 = 0; s2 < 2; ++s2)
          if (f[s1][s2] < f[o1][o2]) { o1 = s1; o2 = s2; }
      int t1 = o1 ? p - co[a1] : co[a1], t2 = o2 ? p - co[a2] : co[a2];
      uint64_t nA = f[1 - o1][o2], nB = f[o1][1 - o2];
      if (nB < nA) {
        const uint64_t tmp = nA; nA = nB; nB = tmp;
        const int tt = t1; t1 = t2; t2 = tt;
      }
      hi = (f[o1][o2] << 42) | (nA << 21) | nB;
      lo = 3 | (uint64_t(t1) << 8) | (uint64_t(t2) << 16);
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

// ---------------------------------------------------------------- partitioned numbering
// (distributed.py) A rank numbers the nodes of its cells plus one halo layer
// first-encounter order; the nodes of a single cell layer are numbered the same way by both
// ranks that hold it, so a table layer-local id -> global id moves the numbering across.
// table[key[i]] = val[i] (every writer of one key writes the same value).
__global__ void dof_table_kernel(const int32_t* __restrict__ key, const int32_t* __restrict__ val,
                                 int64_t n, int32_t* __restrict__ table) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    table[key[i]] = val[i];
}
// global = local < n_table ? table[local] (halo nodes, numbered by the lower rank)
//                          : offset + local - n_table (the rank's own new nodes)
__global__ void dof_globalize_kernel(const int32_t* __restrict__ local, int64_t n,
                                     const int32_t* __restrict__ table, int32_t n_table,
                                     int32_t offset, int32_t* __restrict__ global) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t d = local[i];
    global[i] = d < n_table ? table[d] : offset + (d - n_table);
  }
}
// CSR position of (rows[i], cols[i]) by binary search in the row's sorted columns (-1: absent).
__global__ void csr_find_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                int64_t n, int64_t* __restrict__ pos) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = row_ptr[rows[i]], hi = row_ptr[rows[i] + 1];
    const int32_t c = cols[i];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col_idx[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    pos[i] = (lo < row_ptr[rows[i] + 1] && col_idx[lo] == c) ? lo : -1;
  }
}

// ---------------------------------------------------------------- CSR pattern
// One warp per row r. The row's candidate columns are the dofs of its incident cells
// (inc lists, ascending cell); duplicates are removed in a shared-memory open-addressing
// table sized to the row (H = next_pow2(2 * candidates)), so the count pass never sorts
// and the fill pass sorts only the row's unique columns (~50-70 at P3) instead of its
// candidate list (up to multiplicity x n_loc, 480 at P3).
__device__ __forceinline__ uint32_t next_pow2_u32(uint32_t v) {
  return v <= 1u ? 1u : 1u << (32 - __clz(v - 1u));
}

__device__ __forceinline__ int hash_insert(int32_t* table, uint32_t mask, int32_t v) {
  uint32_t h = (uint32_t(v) * 2654435761u) & mask;
  while (true) {
    const int32_t old = atomicCAS(&table[h], -1, v);
    if (old == -1) return 1;
    if (old == v) return 0;
    h = (h + 1u) & mask;
  }
}

__device__ __forceinline__ int warp_sum_i(int v) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Inserts the row's candidates; returns the number of unique columns (all lanes).
__device__ __forceinline__ int row_dedup(const int32_t* __restrict__ cell_dofs, int n_loc,
                                         const int64_t* __restrict__ inc, int64_t b, int64_t m,
                                         int32_t* table, uint32_t H) {
  const int lane = threadIdx.x & 31;
  for (uint32_t i = lane; i < H; i += 32) table[i] = -1;
  __syncwarp();
  int cnt = 0;
  for (int64_t k = 0; k < m; ++k) {
    const int64_t cell = inc[b + k] / n_loc;
    for (int j = lane; j < n_loc; j += 32) cnt += hash_insert(table, H - 1u, cell_dofs[cell * n_loc + j]);
  }
  __syncwarp();
  return warp_sum_i(cnt);
}

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

// pass 0: row_nnz[r] = unique count. pass 1: sorted unique columns at col_idx[row_ptr[r]].
// Shared memory per warp: hcap ints (table) + hcap / 2 ints (unique list).
__global__ void csr_rows_kernel(const int32_t* __restrict__ cell_dofs, int n_loc,
                                const int64_t* __restrict__ inc_ptr, const int64_t* __restrict__ inc,
                                int32_t n_rows, int hcap, int pass, int64_t* __restrict__ row_nnz,
                                const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx) {
  extern __shared__ int32_t sbuf[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* table = sbuf + int64_t(w) * (hcap + hcap / 2);
  int32_t* list = table + hcap;
  for (int64_t r = int64_t(blockIdx.x) * warps + w; r < n_rows; r += int64_t(gridDim.x) * warps) {
    const int64_t b = inc_ptr[r], m = inc_ptr[r + 1] - b;
    const int64_t t2 = 2 * m * n_loc;
    const uint32_t H = next_pow2_u32(uint32_t(t2 < 32 ? 32 : t2));
    const int u = row_dedup(cell_dofs, n_loc, inc, b, m, table, H);
    if (pass == 0) {
      if (lane == 0) row_nnz[r] = u;
      continue;
    }
    // compact the table (any order), pad to a power of two, sort, write
    int base = 0;
    for (uint32_t i0 = 0; i0 < H; i0 += 32) {
      const int32_t v = table[i0 + lane];
      const unsigned msk = __ballot_sync(0xffffffffu, v != -1);
      if (v != -1) list[base + __popc(msk & ((1u << lane) - 1u))] = v;
      base += __popc(msk);
    }
    const int cap = int(next_pow2_u32(uint32_t(max(u, 32))));
    for (int i = u + lane; i < cap; i += 32) list[i] = INT32_MAX;
    __syncwarp();
    warp_bitonic_sort(list, cap);
    const int64_t o = row_ptr[r];
    for (int i = lane; i < u; i += 32) col_idx[o + i] = list[i];
    __syncwarp();
  }
}

// ---------------------------------------------------------------- scatter plan
// Per row (one warp): the row's sorted columns in shared memory; every incident local row
// (cell, i) maps its n_loc entries by binary search -> pos_map, and (counts != NULL) the
// number of contributions per CSR position (distinct positions within one cell; the warp
// walks the incident cells in order, so plain shared-memory increments suffice). pull_pos
// (optional) receives the same positions as uint16 offsets from the first entry of the row's
// 32-row block (rows 32 b .. 32 b + 31), laid out in the order the row-pull kernel consumes
// them: entry (t, j) of incidence-list slot t.
__device__ __forceinline__ int lower_bound_i32(const int32_t* L, int n, int32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (L[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void plan_pos_kernel(const int32_t* __restrict__ cell_dofs, int n_loc,
                                const int64_t* __restrict__ inc_ptr, const int64_t* __restrict__ inc,
                                const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                int32_t n_rows, int rcap, int32_t* __restrict__ pos_map,
                                uint32_t* __restrict__ counts, uint16_t* __restrict__ pull_pos) {
  extern __shared__ int32_t sbuf[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* L = sbuf + int64_t(w) * 2 * rcap;
  int32_t* cnt = L + rcap;
  for (int64_t r = int64_t(blockIdx.x) * warps + w; r < n_rows; r += int64_t(gridDim.x) * warps) {
    const int64_t o = row_ptr[r];
    const int u = int(row_ptr[r + 1] - o);
    for (int i = lane; i < u; i += 32) {
      L[i] = col_idx[o + i];
      cnt[i] = 0;
    }
    __syncwarp();
    const int64_t b = inc_ptr[r], m = inc_ptr[r + 1] - b;
    const int blk_off = pull_pos ? int(o - row_ptr[r & ~int64_t(31)]) : 0;
    for (int64_t k = 0; k < m; ++k) {
      const int64_t pk = inc[b + k];
      const int64_t cell = pk / n_loc;
      for (int j = lane; j < n_loc; j += 32) {
        const int idx = lower_bound_i32(L, u, cell_dofs[cell * n_loc + j]);
        if (pos_map) pos_map[pk * n_loc + j] = int32_t(o + idx);
        // pull order: the pair's slot in the incidence list; position relative to the first
        // entry of the row's 32-row block
        if (pull_pos) pull_pos[(b + k) * n_loc + j] = uint16_t(blk_off + idx);
        if (counts) cnt[idx] += 1;
      }
      __syncwarp();
    }
    if (counts)
      for (int i = lane; i < u; i += 32) counts[o + i] = uint32_t(cnt[i]);
    __syncwarp();
  }
}

// perm: for every CSR position, its contributions' local indices (c*n_loc + i)*n_loc + j
// in ascending cell order (the reference's summation order), written through per-position
// cursors that start at seg_ptr. Same walk as plan_pos_kernel; positions from pos_map.
__global__ void plan_perm_kernel(int n_loc, const int64_t* __restrict__ inc_ptr,
                                 const int64_t* __restrict__ inc, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ pos_map, const uint32_t* __restrict__ seg_ptr,
                                 int32_t n_rows, int rcap, uint32_t* __restrict__ perm) {
  extern __shared__ uint32_t cursor_buf[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* cur = cursor_buf + int64_t(w) * rcap;
  for (int64_t r = int64_t(blockIdx.x) * warps + w; r < n_rows; r += int64_t(gridDim.x) * warps) {
    const int64_t o = row_ptr[r];
    const int u = int(row_ptr[r + 1] - o);
    for (int i = lane; i < u; i += 32) cur[i] = seg_ptr[o + i];
    __syncwarp();
    const int64_t b = inc_ptr[r], m = inc_ptr[r + 1] - b;
    for (int64_t k = 0; k < m; ++k) {
      const int64_t pk = inc[b + k];
      for (int j = lane; j < n_loc; j += 32) {
        const int64_t e = pk * n_loc + j;
        const int idx = int(pos_map[e] - o);
        perm[cur[idx]++] = uint32_t(e);
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- scatter-add
template <typename TL, typename TV>
__device__ __forceinline__ TV cast_value(TL x) {
  if constexpr (sizeof(TV) == 4 && sizeof(TL) == 8) return __double2float_rn(x);
  else return TV(x);
}

// Deterministic scatter: thread per CSR entry (all rows) walks its contributions in the
// reference order (perm is sorted by (entry, local index), local index ascending = cell
// asc, i asc, j asc) and sums them sequentially at the value format. Contributions of
// cells outside [cell_begin, cell_end) are skipped (multi-GPU slabs). init: first
// contribution taken exactly (start from -0.0); else continue from values[e].
template <typename TL, typename TV>
__device__ __forceinline__ void entry_sum(const TL* __restrict__ locals, int64_t per_cell,
                                          const uint32_t* __restrict__ seg_ptr,
                                          const uint32_t* __restrict__ perm, int64_t e,
                                          int64_t cell_begin, int64_t cell_end, int init,
                                          TV* __restrict__ values) {
  TV acc = init ? TV(-0.0) : values[e];
  const uint32_t b = seg_ptr[e], en = seg_ptr[e + 1];
  for (uint32_t t = b; t < en; ++t) {
    const int64_t k = perm[t];
    const int64_t cell = k / per_cell;
    if (cell < cell_begin || cell >= cell_end) continue;
    acc = acc + cast_value<TL, TV>(locals[k]);
  }
  values[e] = acc;
}

// Block-staged deterministic scatter: a CTA takes kSegBlock consecutive CSR entries, stages
// their segment offsets, gathers every contribution of the block into shared memory with
// independent coalesced perm loads (4 in flight per thread), then each thread sums its
// entries' segments sequentially from shared memory. Contributions of cells outside
// [cell_begin, cell_end) are replaced by -0.0, which leaves any IEEE sum unchanged
// (x + -0 == x, +0 + -0 == +0), so values are bitwise those of entry_sum. Blocks with more
// than `cap` contributions fall back to entry_sum.
#ifndef MPFEM_SEG_BLOCK
#define MPFEM_SEG_BLOCK 512
#endif
#ifndef MPFEM_SEG_SMEM_KB
#define MPFEM_SEG_SMEM_KB 24
#endif
#ifndef MPFEM_SEG_CTAS
#define MPFEM_SEG_CTAS 8
#endif
constexpr int kSegBlock = MPFEM_SEG_BLOCK;
constexpr int kSegSmem = MPFEM_SEG_SMEM_KB * 1024;  // dynamic shared memory per CTA
constexpr int kSegCtasPerSm = MPFEM_SEG_CTAS;
constexpr int kSegHeadBytes = ((kSegBlock + 1) * 4 + 15) / 16 * 16;  // staged segment offsets
template <typename TL, typename TV>
__global__ void __launch_bounds__(256) assemble_seg_block_kernel(
    const TL* __restrict__ locals, int64_t per_cell, const uint32_t* __restrict__ seg_ptr,
    const uint32_t* __restrict__ perm, int64_t nnz, int64_t cell_begin, int64_t cell_end, int init,
    int cap, TV* __restrict__ values) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_seg = reinterpret_cast<uint32_t*>(smem_raw);
  TV* s_val = reinterpret_cast<TV*>(smem_raw + kSegHeadBytes);
  const int64_t kb = cell_begin * per_cell, ke = cell_end * per_cell;
  const int64_t n_blocks = (nnz + kSegBlock - 1) / kSegBlock;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const int64_t e0 = blk * kSegBlock;
    const int n = int((nnz - e0 < kSegBlock ? nnz - e0 : int64_t(kSegBlock)));
    for (int i = threadIdx.x; i <= n; i += blockDim.x) s_seg[i] = seg_ptr[e0 + i];
    __syncthreads();
    const int64_t t0 = s_seg[0];
    const int64_t tn = int64_t(s_seg[n]) - t0;
    if (tn <= cap) {
      const int T = int(tn);
      for (int t = threadIdx.x; t < T; t += 4 * blockDim.x) {
        int64_t k[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tt = t + u * int(blockDim.x);
          k[u] = tt < T ? int64_t(perm[t0 + tt]) : -1;
        }
        TV x[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = (k[u] >= kb && k[u] < ke) ? cast_value<TL, TV>(locals[k[u]]) : TV(-0.0);
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tt = t + u * int(blockDim.x);
          if (tt < T) s_val[tt] = x[u];
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        TV acc = init ? TV(-0.0) : values[e0 + i];
        const int b = int(int64_t(s_seg[i]) - t0), en = int(int64_t(s_seg[i + 1]) - t0);
        for (int t = b; t < en; ++t) acc = acc + s_val[t];
        values[e0 + i] = acc;
      }
    } else {
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        entry_sum(locals, per_cell, seg_ptr, perm, e0 + i, cell_begin, cell_end, init, values);
    }
    __syncthreads();
  }
}

// Row-pull deterministic scatter (no seg_ptr/perm plan). A warp owns a batch of consecutive CSR
// rows whose entries fit its shared-memory accumulators. The batch's incident (cell, local row i)
// pairs are the contiguous run inc[inc_ptr[r0] .. inc_ptr[r1]) -- sorted by (dof, cell * n_loc + i),
// i.e. ascending cell order within every row. A pair's n_loc local entries are the contiguous row i
// of the cell's matrix and their CSR positions the matching n_loc words of pos_map, so both streams
// are read in contiguous runs (the seg_ptr/perm gather and the atomic scatter touch every
// contribution as a separate 4-byte sector access). Chunks of whole pairs are copied to a
// shared-memory ring with cp.async (kPullStages chunks in flight per warp, no registers held) and
// replayed pair by pair into the accumulators: every CSR entry receives its contributions in
// ascending cell order starting from -0.0 -- bitwise the reference's sequential sum
// (assembly.cpp:50-67) and entry_sum. A single row beyond the caps runs the same ordered replay on
// global memory. rows != NULL restricts the pass to those rows (runs of consecutive rows in the
// list form batches; multi-GPU slabs); pairs of cells outside [cell_begin, cell_end) are skipped.
constexpr int kPullWarps = 4;     // warps per CTA, each autonomous
#ifndef MPFEM_PULL_STAGES
#define MPFEM_PULL_STAGES 3
#define MPFEM_PULL_ACC 512
#define MPFEM_PULL_INC 128
#endif
#ifndef MPFEM_PULL_MINB
#define MPFEM_PULL_MINB 7
#endif
constexpr int kPullStages = MPFEM_PULL_STAGES;  // cp.async ring depth per warp
constexpr int kPullAccCap = MPFEM_PULL_ACC;     // accumulators (CSR entries) per batch
constexpr int kPullIncCap = MPFEM_PULL_INC;     // pairs per batch
// bytes of one stage's position slots: int32 CSR positions (pos_map) or uint16 row-relative
// positions (pull_pos; 8 entries of slack: the stream is copied from the 16-byte boundary below)
template <int CH, bool P16>
__host__ __device__ constexpr size_t pull_pos_stage_bytes() {
  return P16 ? size_t(CH + 8) * 2 : size_t(CH) * 4;
}
template <typename TL, typename TV, int CH, bool P16>
__host__ __device__ constexpr size_t pull_warp_bytes() {
  // + 128 bytes: the replay's operand prefetch runs up to 31 entries past the last staged pair
  return sizeof(TV) * (kPullAccCap + 32) + sizeof(int64_t) * kPullIncCap +
         size_t(kPullStages) * (CH * sizeof(TL) + pull_pos_stage_bytes<CH, P16>()) + 128;
}
template <int BYTES>
__device__ __forceinline__ void cp_async_bytes(void* smem_dst, const void* gsrc) {
  const uint32_t d = uint32_t(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(gsrc), "n"(BYTES) : "memory");
}
// VEC consecutive elements of T (VEC * sizeof(T) in {4, 8, 16, 32} bytes, both sides aligned to
// min(16, that))
template <typename T, int VEC>
__device__ __forceinline__ void cp_async_vec(T* smem_dst, const T* gsrc) {
  constexpr int bytes = int(sizeof(T)) * VEC;
  if constexpr (bytes <= 16) {
    cp_async_bytes<bytes>(smem_dst, gsrc);
  } else {
    #pragma unroll
    for (int h = 0; h < bytes / 16; ++h)
      cp_async_bytes<16>(reinterpret_cast<char*>(smem_dst) + 16 * h,
                         reinterpret_cast<const char*>(gsrc) + 16 * h);
  }
}
// VEC: elements per copy (n_loc % VEC == 0 and the arrays aligned accordingly; chosen by the host)
// P16: positions come from pull_pos (uint16 offsets into the row's 32-row block, in incidence-
// list order: one sequential stream, half the bytes of pos_map and no partly used sectors)
// instead of pos_map; batches then stay inside one 32-row block.
template <typename TL, typename TV, int CH, int VEC, bool P16>
__global__ void __launch_bounds__(kPullWarps * 32, MPFEM_PULL_MINB) assemble_pull_kernel(
    const TL* __restrict__ locals, int n_loc, const int64_t* __restrict__ row_ptr,
    const int64_t* __restrict__ inc_ptr, const int64_t* __restrict__ inc,
    const int32_t* __restrict__ pos_map, const uint16_t* __restrict__ pull_pos,
    const int32_t* __restrict__ rows, int64_t n_rows,
    int64_t cell_begin, int64_t cell_end, int init, TV* __restrict__ values) {
  extern __shared__ __align__(16) unsigned char pull_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = pull_smem + size_t(warp) * pull_warp_bytes<TL, TV, CH, P16>();
  int64_t* s_inc = reinterpret_cast<int64_t*>(base);  // first entry id of the pair, -1: skipped
  TV* s_acc = reinterpret_cast<TV*>(s_inc + kPullIncCap);
  TL* s_x = reinterpret_cast<TL*>(s_acc + kPullAccCap + 32);  // + one scratch slot per lane
  unsigned char* s_p = reinterpret_cast<unsigned char*>(s_x + kPullStages * CH);
  constexpr size_t kPosStage = pull_pos_stage_bytes<CH, P16>();
  const int64_t kb = cell_begin * n_loc, ke = cell_end * n_loc;  // pair ids of the cell range
  const int pairs_per_chunk = CH / n_loc;                          // >= 1 (host checks n_loc <= CH)
  const int upp = n_loc / VEC;                                     // copy units per pair
  const int dq = 32 / upp, dr = 32 - dq * upp;
  const int lane_t = lane / upp, lane_j = lane - lane_t * upp;
  const int64_t n_blocks = (n_rows + 31) >> 5;
  const int64_t wstride = int64_t(gridDim.x) * kPullWarps;
  for (int64_t blk = int64_t(blockIdx.x) * kPullWarps + warp; blk < n_blocks; blk += wstride) {
    // lane l holds row l of the 32-row block
    const int64_t ri = (blk << 5) + lane;
    const bool have = ri < n_rows;
    const int64_t r = have ? (rows ? int64_t(rows[ri]) : ri) : 0;
    const int64_t my_e0 = have ? row_ptr[r] : 0, my_e1 = have ? row_ptr[r + 1] : 0;
    const int64_t my_b0 = have ? inc_ptr[r] : 0, my_b1 = have ? inc_ptr[r + 1] : 0;
    // P16: first entry of the row's 32-row block (lane 0's row without a row list)
    int64_t my_blk0 = 0;
    if constexpr (P16) my_blk0 = rows ? (have ? row_ptr[r & ~int64_t(31)] : 0) : __shfl_sync(0xffffffffu, my_e0, 0);
    const int n_have = __popc(__ballot_sync(0xffffffffu, have));
    int start = 0;
    while (start < n_have) {
      const int64_t e0 = __shfl_sync(0xffffffffu, my_e0, start);
      const int64_t b0 = __shfl_sync(0xffffffffu, my_b0, start);
      // rows start .. start + nr - 1: a run of consecutive rows (always, without a row list)
      // that fits the caps
      const int64_t r_start = __shfl_sync(0xffffffffu, r, start);
      const bool fits = lane >= start && lane < n_have && r == r_start + (lane - start) &&
                        my_e1 - e0 <= kPullAccCap && my_b1 - b0 <= kPullIncCap &&
                        (!P16 || (r >> 5) == (r_start >> 5));
      const unsigned run = ~(__ballot_sync(0xffffffffu, fits) >> start);
      const int nr = run ? __ffs(run) - 1 : 32 - start;
      if (nr == 0) {
        // one long row: the same ordered replay on global memory
        const int64_t e1 = __shfl_sync(0xffffffffu, my_e1, start);
        const int64_t b1 = __shfl_sync(0xffffffffu, my_b1, start);
        const int64_t blk0 = __shfl_sync(0xffffffffu, my_blk0, start);
        if (init)
          for (int64_t e = e0 + lane; e < e1; e += 32) values[e] = TV(-0.0);
        __syncwarp();
        for (int64_t t = b0; t < b1; ++t) {
          const int64_t ki = inc[t];
          if (ki >= kb && ki < ke) {
            for (int j = lane; j < n_loc; j += 32) {
              const int64_t k = ki * n_loc + j;
              const int64_t pos = P16 ? blk0 + pull_pos[t * n_loc + j] : int64_t(pos_map[k]);
              values[pos] = values[pos] + cast_value<TL, TV>(locals[k]);
            }
          }
          __syncwarp();
        }
        start += 1;
        continue;
      }
      const int last = start + nr - 1;
      const int ne = int(__shfl_sync(0xffffffffu, my_e1, last) - e0);
      const int ni = int(__shfl_sync(0xffffffffu, my_b1, last) - b0);
      const int e0i = int(e0);  // pos_map is int32, so every position fits
      for (int t = lane; t < ni; t += 32) {
        const int64_t ki = __ldcs(inc + b0 + t);
        s_inc[t] = (ki >= kb && ki < ke) ? ki * n_loc : int64_t(-1);
      }
      for (int i = lane; i < ne; i += 32) s_acc[i] = init ? TV(-0.0) : values[e0 + i];
      __syncwarp();
      // P16: accumulator slot = staged block offset - (batch start - block start)
      const int cbase = P16 ? int(e0 - __shfl_sync(0xffffffffu, my_blk0, start)) : e0i;
      const uintptr_t pbytes0 = P16 ? reinterpret_cast<uintptr_t>(pull_pos + b0 * n_loc) : 0;
      const int n_chunks = (ni + pairs_per_chunk - 1) / pairs_per_chunk;
      auto issue = [&](int c) {
        if (c < n_chunks) {
          const int t0 = c * pairs_per_chunk;
          const int nu = min(ni - t0, pairs_per_chunk) * upp;
          TL* sx = s_x + (c % kPullStages) * CH;
          int32_t* sp = reinterpret_cast<int32_t*>(s_p + (c % kPullStages) * kPosStage);
          if constexpr (P16) {
            // the chunk's positions are one contiguous run of pull_pos: 16-byte copies from the
            // boundary below (the staged run keeps the stream's misalignment)
            const uintptr_t src = pbytes0 + uint32_t(2 * t0 * n_loc);
            const uintptr_t a0 = src & ~uintptr_t(15);
            const int units = (int(src & 15) + nu * VEC * 2 + 15) >> 4;
            for (int u = lane; u < units; u += 32)
              cp_async_bytes<16>(reinterpret_cast<unsigned char*>(sp) + 16 * u,
                                 reinterpret_cast<const unsigned char*>(a0) + 16 * u);
          }
          int t = lane_t, j = lane_j;
          for (int u = lane; u < nu; u += 32) {
            const int64_t k0 = s_inc[t0 + t];
            if (k0 >= 0) {
              cp_async_vec<TL, VEC>(sx + u * VEC, locals + k0 + j * VEC);
              if constexpr (!P16) cp_async_vec<int32_t, VEC>(sp + u * VEC, pos_map + k0 + j * VEC);
            } else {
              // a skipped pair adds -0.0 (to the batch's first entry without pull_pos): no
              // change in any bit
              #pragma unroll
              for (int v = 0; v < VEC; ++v) {
                sx[u * VEC + v] = TL(-0.0);
                if constexpr (!P16) sp[u * VEC + v] = e0i;
              }
            }
            t += dq;
            j += dr;
            if (j >= upp) {
              j -= upp;
              ++t;
            }
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      #pragma unroll
      for (int c = 0; c < kPullStages - 1; ++c) issue(c);
      for (int c = 0; c < n_chunks; ++c) {
        issue(c + kPullStages - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(kPullStages - 1) : "memory");
        __syncwarp();
        const int npairs = min(ni - c * pairs_per_chunk, pairs_per_chunk);
        const TL* sx = s_x + (c % kPullStages) * CH;
        const unsigned char* spb = s_p + (c % kPullStages) * kPosStage;
        const int32_t* sp = reinterpret_cast<const int32_t*>(spb);
        // P16: staged uint16 run, shifted by the stream's offset from its 16-byte boundary
        const uint16_t* sq = reinterpret_cast<const uint16_t*>(spb);
        if constexpr (P16) sq += int((pbytes0 + uint32_t(2 * c * pairs_per_chunk * n_loc)) & 15) >> 1;
        auto slot = [&](int idx) -> int {
          if constexpr (P16) return int(sq[idx]) - cbase;
          else return sp[idx] - cbase;
        };
        if (n_loc <= 32) {
          // one lane per local column, branch-free: lanes past n_loc update a scratch slot of
          // their own; the next pair's operands are fetched ahead of the dependent accumulator
          // update (the read after the chunk's last pair stays inside the warp's buffers and is
          // not used)
          const bool on = lane < n_loc;
          const int scratch = kPullAccCap + lane;
          int a = on ? slot(lane) : scratch;
          TV x = cast_value<TL, TV>(sx[lane]);
          int idx = lane;
          for (int t = 0; t < npairs; ++t) {
            idx += n_loc;
            const int a_next = on ? slot(idx) : scratch;
            const TV x_next = cast_value<TL, TV>(sx[idx]);
            s_acc[a] = s_acc[a] + x;
            __syncwarp();  // pairs are applied one after the other (ascending cell order per row)
            a = a_next;
            x = x_next;
          }
        } else {
          for (int t = 0; t < npairs; ++t) {
            for (int j = lane; j < n_loc; j += 32) {
              const int a = slot(t * n_loc + j);
              s_acc[a] = s_acc[a] + cast_value<TL, TV>(sx[t * n_loc + j]);
            }
            __syncwarp();
          }
        }
      }
      for (int i = lane; i < ne; i += 32) values[e0 + i] = s_acc[i];
      __syncwarp();
      start += nr;
    }
  }
}

template <typename TL, typename TV>
__global__ void assemble_seg_rows_kernel(const TL* __restrict__ locals, int64_t per_cell,
                                         const int64_t* __restrict__ row_ptr,
                                         const uint32_t* __restrict__ seg_ptr,
                                         const uint32_t* __restrict__ perm,
                                         const int32_t* __restrict__ rows, int64_t n_rows,
                                         int64_t cell_begin, int64_t cell_end, int init,
                                         TV* __restrict__ values) {
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t ri = int64_t(blockIdx.x) * warps + w; ri < n_rows; ri += int64_t(gridDim.x) * warps) {
    const int64_t r = rows[ri];
    for (int64_t e = row_ptr[r] + lane; e < row_ptr[r + 1]; e += 32)
      entry_sum(locals, per_cell, seg_ptr, perm, e, cell_begin, cell_end, init, values);
  }
}

// Atomic scatter: thread per local entry, red.global.add at its precomputed position. The
// local matrices and the plan are read once (streaming loads, evict-first) and the reductions
// carry an evict-last hint, so that the L2 keeps the CSR value lines the neighbouring cells
// return to (config 4 P3: 11.5 -> 7.5 ms, P2 2.23 -> 1.66 ms; profiles/r2_asm_order_experiment.txt).
// A Morton traversal of the cells on top of that gained <= 3 % at P3 and lost at P2 (same
// file): the kernel is bound by the streams it must read (locals, plan) at ~4.4 TB/s.
template <typename TL, typename TV>
__global__ void assemble_atomic_kernel(const TL* __restrict__ locals, const int32_t* __restrict__ pos_map,
                                       int64_t k_begin, int64_t k_end, TV* __restrict__ values) {
  const uint64_t keep = policy_evict_last();
  for (int64_t k = k_begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < k_end;
       k += int64_t(gridDim.x) * blockDim.x)
    red_add_keep(&values[__ldcs(pos_map + k)], cast_value<TL, TV>(__ldcs(locals + k)), keep);
}

}  // namespace asmb
}  // namespace mpfem_b200
