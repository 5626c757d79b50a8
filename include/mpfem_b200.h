/*
 * mpfem_b200.h -- C-ABI drop-in boundary of the B200-native hot path.
 *
 * Plain pointers, sizes and status codes; no torch or C++ types cross this boundary.
 * Each entry point names the reference interface it replaces (file:line into
 * /root/reference/proj). A reference-side binding (the mpfem C++ API re-implemented on
 * top of this ABI) is shown in INTEGRATION.md.
 *
 * Status codes mirror the reference CLI (mpfem_cli.cpp:517-527):
 *   0 ok, 2 ConfigError (bad name/shape/format/mode), 3 CheckError (singular cell,
 *   dof out of range, dof collision), 4 CUDA/runtime failure (no device, launch error).
 * FP exception flags (softfloat.hpp:22-36) are a bitmask: 1 overflow, 2 underflow,
 * 4 invalid, 8 divzero. On the GPU they are detected on rounding of the geometry and
 * scaled-weight stages and on non-finite outputs; this is coarser than the reference's
 * per-operation flags (documented in DESIGN.md).
 *
 * Formats (softfloat.hpp:17): 0 bf16, 1 fp16, 2 fp32, 3 fp64.
 * Forms (geometry.hpp:107): 0 mass, 1 poisson.  Engines (mm_units.hpp:31): 0 scalar,
 * 1 vector, 2 matrix (kept for validate_config parity; dispatch is on the formats).
 */
#ifndef MPFEM_B200_H
#define MPFEM_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpfem_b200_setup_s* mpfem_b200_setup_t;

enum {
  MPFEM_B200_OK = 0,
  MPFEM_B200_CONFIG_ERROR = 2,
  MPFEM_B200_CHECK_ERROR = 3,
  MPFEM_B200_RUNTIME_ERROR = 4
};

/* Coefficient kinds for cell_matrices:
 *   0 ONE            constant one (reference: empty z, multiplication skipped)
 *   1 SINCOSEXP      c(x) = 1 + 0.5 sin(2 pi x) cos(2 pi y) e^z at x_q = v0 + J xi_q (fp64),
 *                    rounded once to u_g  (BASELINE configs 0,1,2,4)
 *   2 EXP10_AFFINE   c = 10^(6 u(x_q)), u affine per cell from 4 vertex values
 *                    (coef: n_cells x 4 doubles)  (BASELINE config 3)
 *   3 NODAL          nodal FE coefficient z, n_phi doubles per cell, evaluated exactly as
 *                    eval_z_at_ug (kernels.cpp:114-136) */
enum { MPFEM_COEF_ONE = 0, MPFEM_COEF_SINCOSEXP = 1, MPFEM_COEF_EXP10_AFFINE = 2,
       MPFEM_COEF_NODAL = 3 };

/* Thread-local description of the last failure (empty when none). */
const char* mpfem_b200_last_error(void);

/* Library version and the compiled device architecture string ("sm_100a"). */
const char* mpfem_b200_version(void);

/* Replaces make_setup (kernels.hpp:60-62, kernels.cpp:78-108) + validate_config
 * (kernels.cpp:29-40). dim 3; cell_kind 0 (simplex, 1 <= p <= 8) or 1 (box / hexahedra,
 * 1 <= p <= 4: tensor Lagrange basis, Gauss-Legendre rule, geometry at every rule point;
 * vertices 8 per cell in lattice bit order, constant or nodal coefficients).
 * The handle owns device copies of the rule, the fp64 tabulations and the shared
 * basis-product operand T, which are read-only after creation. Per-call scratch (the W
 * operand, FP flags, the K1 tile counter, host-API staging) lives in one workspace per CUDA
 * stream, so a setup may be used from several threads and streams at once: calls on one
 * stream are ordered by the stream, calls on different streams use different scratch, and
 * the host-side bookkeeping of every call is serialized by a mutex of the setup.
 * CheckError semantics: a singular cell (geometry.cpp:42) is detected on the device. With
 * flags != NULL (or in the synchronizing host-buffer calls) the call itself returns 3;
 * otherwise the error is reported (status 3) by the next call on the setup or by
 * mpfem_b200_synchronize -- the asynchronous analogue of the reference's throw. */
int mpfem_b200_setup_create(int cell_kind, int dim, int p, int form, int u_p, int u_g,
                            int u_q, int u_s, int engine, int n_batch,
                            mpfem_b200_setup_t* out);
int mpfem_b200_setup_destroy(mpfem_b200_setup_t setup);

/* make_setup from the caller's own rule and tabulations (kernels.cpp:78-108 having run on the
 * reference side): the C++ drop-in shim (include/mpfem/batched.hpp) creates its device setup
 * from the reference KernelSetup this way, so any rule (the make_setup overload with an
 * explicit QuadratureRule, kernels.hpp:62) and dimension 2 or 3 are accepted.
 *   points:    n_q x dim rule points; weights: n_q
 *   tab_store: n_d x n_phi x n_q, KernelSetup::tab_store (evaluated at u_p, stored at u_s;
 *              n_d = dim for Poisson, 1 for mass)
 *   tab_up:    n_phi x n_q, KernelSetup::tab_values (basis values at u_p)
 * p is informational. Such a setup takes geometry tensors (the two calls below), not vertices;
 * GPU bounds need the vertex setup. */
int mpfem_b200_setup_create_tab(int cell_kind, int dim, int p, int form, int u_p, int u_g,
                                int u_q, int u_s, int engine, int n_batch, int n_phi, int n_q,
                                const double* points, const double* weights,
                                const double* tab_store, const double* tab_up,
                                mpfem_b200_setup_t* out);

/* bilinear_kernel(setup, geom, z, flags) (kernels.hpp:85-86) for n_cells cells whose geometry
 * the caller already evaluated (GeometryData, geometry.hpp:31-41), on HOST buffers:
 *   G:   n_cells x n_pts x n_d x n_d geometry tensors at u_g (GeometryPoint::tensor, row-major),
 *        n_pts = 1 (affine cells) or n_q (one entry per rule point)
 *   z:   NULL (constant one) or nodal coefficients, n_cells rows of z_stride doubles
 *        (z_stride = 0: one vector shared by every cell)
 *   out: n_cells x out_pitch, fp32 for u_q in {fp16, fp32}, fp64 for u_q = fp64
 * W is build_C's C bit for bit (kernels.cpp:177-197); the matrices meet the same tolerances as
 * mpfem_b200_cell_matrices. Synchronizes. */
int mpfem_b200_bilinear_from_geometry(mpfem_b200_setup_t setup, const double* G, int n_pts,
                                      int64_t n_cells, const double* z, int64_t z_stride,
                                      void* out, int64_t out_pitch, void* stream,
                                      uint32_t* flags);

/* action_kernel(setup, geoms, w, z, flags) (kernels.hpp:90-92) on HOST buffers with the caller's
 * geometry tensors (as above, dimension 3): z NULL or one nodal vector (n_phi) shared by the
 * batch; w n_cells rows of w_stride doubles; out n_cells x out_pitch (row c = the reference's
 * column c). Bit-identical to the reference in every mode. Synchronizes. */
int mpfem_b200_action_from_geometry(mpfem_b200_setup_t setup, const double* G, int n_pts,
                                    int64_t n_cells, const double* z, const double* w,
                                    int64_t w_stride, void* out, int64_t out_pitch, void* stream,
                                    uint32_t* flags);

/* Sizes: n_phi, n_q, n_d (1 mass, 3 poisson), K (GEMM depth = blocks x nq_pad), K_pad,
 * path (0 tcgen05, 1 fp32 FFMA, 2 fp64, 3 fused small-degree). */
int mpfem_b200_setup_info(mpfem_b200_setup_t setup, int* n_phi, int* n_q, int* n_d,
                          int64_t* k, int64_t* k_pad, int* path);

/* Host copies of the rule (n_q x 3 points, n_q weights) the setup uses; bitwise equal to
 * rule_for(simplex, p) (quadrature.cpp:171-224). */
int mpfem_b200_setup_rule(mpfem_b200_setup_t setup, double* points, double* weights);

/* Batched replacement for the per-cell loop cell_geometry (geometry.cpp:226-245) ->
 * bilinear_kernel (kernels.cpp:242-267) over n_cells affine tets, on DEVICE buffers.
 *   verts:  if cells == NULL, n_cells x 4 x 3 fp64 private vertices;
 *           else the mesh vertex table (n_verts x 3 fp64) indexed by cells (n_cells x 4 int32)
 *   coef:   per coefficient kind above (device, may be NULL for ONE/SINCOSEXP), row stride
 *           coef_stride doubles
 *   out:    n_cells rows of n_phi x n_phi row-major cell matrices with row pitch
 *           out_pitch elements (>= n_phi^2); fp32 for u_q in {fp16, fp32}, fp64 for fp64
 *   stream: cudaStream_t (NULL = legacy default)
 *   flags:  optional host pointer; OR-ed with the FP flag bitmask (forces a sync)
 * A singular cell makes its output row NaN and raises CheckError (3) as described at
 * mpfem_b200_setup_create. */
int mpfem_b200_cell_matrices(mpfem_b200_setup_t setup, const double* verts,
                             const int32_t* cells, int64_t n_cells, int coef_kind,
                             const double* coef, int64_t coef_stride, void* out,
                             int64_t out_pitch, void* stream, uint32_t* flags);

/* Same contract on HOST buffers: copies inputs in, runs, copies the matrices out (the
 * drop-in call a reference user makes). Host buffers should be pinned for full speed. */
int mpfem_b200_cell_matrices_host(mpfem_b200_setup_t setup, const double* verts,
                                  int64_t n_verts, const int32_t* cells, int64_t n_cells,
                                  int coef_kind, const double* coef, int64_t coef_stride,
                                  void* out, int64_t out_pitch, void* stream,
                                  uint32_t* flags);

/* Pre-size the scratch of `stream`'s workspace (scaled-weight operand W) for n_cells so that
 * later calls on this setup and stream allocate nothing (CUDA-graph capture safe). */
int mpfem_b200_reserve(mpfem_b200_setup_t setup, int64_t n_cells, void* stream);

/* Waits for `stream` and returns 3 (CheckError) if a call on this setup met a singular cell
 * since the last report (see the CheckError semantics at mpfem_b200_setup_create). */
int mpfem_b200_synchronize(mpfem_b200_setup_t setup, void* stream);

/* Debug/parity entry: the scaled weights W (kernels.cpp:177-197 build_C) in the GEMM
 * layout -- blocks (s<=t) of nq_pad = round_up(n_q, 8) entries, zero for q >= n_q -- as
 * fp64 carriers for n_cells cells (device out, n_cells x K doubles, K = blocks x nq_pad). */
int mpfem_b200_scaled_weights(mpfem_b200_setup_t setup, const double* verts,
                              const int32_t* cells, int64_t n_cells, int coef_kind,
                              const double* coef, int64_t coef_stride, double* out,
                              void* stream, uint32_t* flags);

/* Fused cell kernels + atomic CSR scatter (replaces run_assemble's per-cell
 * bilinear_kernel -> assemble_matrix loop, mpfem_cli.cpp:322-332, in the order-free atomic
 * mode): values[pos_map[c * n_phi^2 + i * n_phi + j]] += A_c[i][j] for the n_cells cells
 * (pos_map from mpfem_b200_scatter_plan, already offset to the first cell of this call).
 * On the tcgen05 path the local matrices never reach HBM (K2's epilogue adds from TMEM);
 * other paths stage them and run the atomic scatter. values_fmt 2 = fp32, 3 = fp64. */
int mpfem_b200_cell_matrices_scatter(mpfem_b200_setup_t setup, const double* verts,
                                     const int32_t* cells, int64_t n_cells, int coef_kind,
                                     const double* coef, int64_t coef_stride,
                                     const int32_t* pos_map, void* values, int values_fmt,
                                     void* stream, uint32_t* flags);

/* Batched replacement for action_kernel (kernels.hpp:90-92, kernels.cpp:269-304; Algorithm
 * 2 of the paper): v_c = sum_s B_s r_s for n_cells cells in ONE launch, on DEVICE buffers,
 * bit-identical to the reference in every mode (same op order and roundings: eval_w_at_ug
 * kernels.cpp:145-173, integrand kernels.cpp:280-301, b_cat_action contraction :303).
 *   verts/cells/coef: as mpfem_b200_cell_matrices (the reference takes one nodal z for the
 *           batch: pass coef_stride 0 to share it)
 *   w:      n_cells rows of n_phi fp64 FE coefficients (row stride w_stride >= n_phi)
 *   out:    n_cells rows of n_phi (row pitch out_pitch) -- row c is column c of the
 *           reference's n_phi x batch result; fp64 if u_q = fp64, else fp32 carriers of u_q
 * Errors as the reference: ConfigError (2) for a short w / coefficient, CheckError (3) for a
 * singular cell (see the CheckError semantics at mpfem_b200_setup_create). */
int mpfem_b200_action(mpfem_b200_setup_t setup, const double* verts, const int32_t* cells,
                      int64_t n_cells, int coef_kind, const double* coef, int64_t coef_stride,
                      const double* w, int64_t w_stride, void* out, int64_t out_pitch,
                      void* stream, uint32_t* flags);

/* Same on HOST buffers (H2D of vertices, coefficients and w; D2H of v inside the call). */
int mpfem_b200_action_host(mpfem_b200_setup_t setup, const double* verts, int64_t n_verts,
                           const int32_t* cells, int64_t n_cells, int coef_kind,
                           const double* coef, int64_t coef_stride, const double* w,
                           int64_t w_stride, void* out, int64_t out_pitch, void* stream,
                           uint32_t* flags);

/* Per-cell a-priori error bound on the GPU: replaces kernel_bounds (bounds.hpp, bounds.cpp:
 * 29-281, bilinear part) with basis_condition_numbers (elements.cpp:278-359) over n_cells cells
 * in binary64, so bound dominance can be checked on every cell of a mesh.
 *   out: n_cells x 4 doubles {bound_a, kappa_q_a, kappa_p_a, kappa_g_a} (NaN when A = 0)
 *   a64: optional n_cells x n_phi^2 doubles, the exact binary64 A of the report (report.a)
 * For constant and nodal coefficients every value is the reference's bit for bit; the
 * analytic coefficient (kinds 1, 2) enters at x_q as in the Q path (z_at = c(x_q),
 * theta_c = 0). Synchronizes (CheckError 3 for a singular cell). */
int mpfem_b200_cell_bounds(mpfem_b200_setup_t setup, const double* verts, const int32_t* cells,
                           int64_t n_cells, int coef_kind, const double* coef,
                           int64_t coef_stride, double* out, double* a64, void* stream);

/* The action part of kernel_bounds (bounds.cpp:128-155,224-240,268-279; the bound of Algorithm
 * 2) per cell on the GPU: out n_cells x 4 {bound_v, kappa_q_v, kappa_p_v, kappa_g_v}; v64
 * (optional) n_cells x n_phi, the exact binary64 v. w: n_cells rows of n_phi (stride w_stride).
 * Bitwise the reference's for constant and nodal coefficients. Synchronizes. */
int mpfem_b200_action_bounds(mpfem_b200_setup_t setup, const double* verts, const int32_t* cells,
                             int64_t n_cells, int coef_kind, const double* coef,
                             int64_t coef_stride, const double* w, int64_t w_stride, double* out,
                             double* v64, void* stream);

/* Number of kernel launches the last cell_matrices call on this setup issued. */
int mpfem_b200_last_launch_count(mpfem_b200_setup_t setup);

/* Per-kernel timing: when enabled, cell_matrices records CUDA events on its stream
 * around K1 (geometry/W) and K2 (GEMM); last_timings returns their durations in ms
 * (synchronizing on the events), count as return value (negative status on error). */
int mpfem_b200_set_timing(mpfem_b200_setup_t setup, int enable);
int mpfem_b200_last_timings(mpfem_b200_setup_t setup, float* ms, int max_n);


/* ---------------------------------------------------------------- mesh & assembly */

/* Seeded synthetic cells on the host (std::mt19937_64 = the reference Rng, common.hpp:21-35).
 * kind 0: BASELINE configs 0-2 tets (n x 4 x 3 doubles); kind 1: config-3 anisotropic
 * rotated tets plus 4 affine-field vertex values per cell in coef (n x 4). */
int mpfem_b200_gen_tets(int kind, uint64_t seed, int64_t n, double* verts, double* coef);

/* Replaces structured_tet_mesh (mesh.cpp:125-163) for the assembly config: host
 * arrays (n_verts = (nx+1)(ny+1)(nz+1) x 3, n_cells = 6 nx ny nz x 4). */
int mpfem_b200_structured_tet_mesh(int nx, int ny, int nz, double extent, double jitter,
                                   uint64_t seed, double* verts, int32_t* cells);

/* Replaces build_dofmap(mesh, basis, continuous) (mesh.cpp:204-298) on DEVICE buffers.
 * Nodes are identified topologically (sub-simplex vertex ids + lattice position), which
 * equals the reference's geometric identification on conforming meshes; dof ids are
 * assigned in first-encounter order over (cell asc, local k asc). cell_dofs: n_cells x
 * n_phi int32 (device). n_dofs / max_multiplicity written to host pointers. */
int mpfem_b200_dofmap(int p, const int32_t* cells, int64_t n_cells, int64_t n_verts,
                      int32_t* cell_dofs, int32_t* n_dofs, int32_t* max_multiplicity,
                      void* stream);

/* The same for either cell kind: cell_kind 0 tets (cells n_cells x 4), 1 hexahedra (cells
 * n_cells x 8 in lattice-bit order, tensor Lagrange nodes axis 0 fastest). Hexahedral nodes are
 * keyed by their sub-entity's vertex ids and coordinates in an id-fixed frame, so any
 * conforming mesh numbers like the reference's geometric identification. */
int mpfem_b200_dofmap_cells(int cell_kind, int p, const int32_t* cells, int64_t n_cells,
                            int64_t n_verts, int32_t* cell_dofs, int32_t* n_dofs,
                            int32_t* max_multiplicity, void* stream);

/* Sparsity pattern = the reference COO key set sorted by (row, col) (assembly.cpp:67-86)
 * as CSR. Two-phase: call with col_idx == NULL to get nnz into *nnz and row_ptr
 * (n_dofs + 1 int64, device) filled; then again with col_idx (nnz int32, device). */
int mpfem_b200_csr_pattern(const int32_t* cell_dofs, int64_t n_cells, int n_loc,
                           int32_t n_dofs, int64_t* row_ptr, int32_t* col_idx, int64_t* nnz,
                           void* stream);

/* Partitioned (multi-GPU) variants, SURVEY 8e / paper_2410_12614_b200/distributed.py: a rank
 * numbers its cells plus one halo layer locally (rows) while columns carry the global ids.
 * csr_pattern_cols / scatter_plan_cols: as csr_pattern / scatter_plan, with the row of local
 * entry (c, i) taken from cell_dofs and the column of (c, j) from col_dofs (NULL: cell_dofs). */
int mpfem_b200_csr_pattern_cols(const int32_t* cell_dofs, const int32_t* col_dofs, int64_t n_cells,
                                int n_loc, int32_t n_dofs, int64_t* row_ptr, int32_t* col_idx,
                                int64_t* nnz, void* stream);
int mpfem_b200_scatter_plan_cols(const int32_t* cell_dofs, const int32_t* col_dofs, int64_t n_cells,
                                 int n_loc, int32_t n_dofs, const int64_t* row_ptr,
                                 const int32_t* col_idx, int32_t* pos_map, uint32_t* seg_ptr,
                                 uint32_t* perm, void* stream);
/* scatter_plan_cols with the row-pull kernel's position stream: pull_pos[t * n_loc + j] is the
 * CSR position of local entry j of incidence-list slot t, as a uint16 offset from the first entry
 * of the row's 32-row block (rows 32 b .. 32 b + 31; status 2 when a row has more than 2,048
 * entries: use pos_map then). n_cells * n_loc^2 + 8 entries, 16-byte aligned -- the kernel copies
 * whole 16-byte units. pos_map may be NULL when only pull_pos is wanted (then seg_ptr and perm
 * too). */
int mpfem_b200_scatter_plan_pull(const int32_t* cell_dofs, const int32_t* col_dofs, int64_t n_cells,
                                 int n_loc, int32_t n_dofs, const int64_t* row_ptr,
                                 const int32_t* col_idx, int32_t* pos_map, uint32_t* seg_ptr,
                                 uint32_t* perm, uint16_t* pull_pos, void* stream);
/* table[key_dofs[i]] = val_dofs[i] for i < n (layer-local id -> global id). */
int mpfem_b200_dofmap_table(const int32_t* key_dofs, const int32_t* val_dofs, int64_t n, int32_t* table,
                            void* stream);
/* global[i] = local[i] < n_table ? table[local[i]] : offset + local[i] - n_table. */
int mpfem_b200_dofmap_globalize(const int32_t* local_dofs, int64_t n, const int32_t* table,
                                int32_t n_table, int32_t offset, int32_t* global_dofs, void* stream);
/* pos[i] = CSR position of (rows[i], cols[i]) in (row_ptr, col_idx), -1 when absent. */
int mpfem_b200_csr_find(const int64_t* row_ptr, const int32_t* col_idx, const int32_t* rows,
                        const int32_t* cols, int64_t n, int64_t* pos, void* stream);

/* Incidence (dof -> (cell, local) pairs in ascending cell order) used by the
 * deterministic assembly; inc_ptr: n_dofs + 1 int64, inc: n_cells x n_loc int64
 * (packed cell * n_loc + local). */
int mpfem_b200_incidence(const int32_t* cell_dofs, int64_t n_cells, int n_loc,
                         int32_t n_dofs, int64_t* inc_ptr, int64_t* inc, void* stream);

/* Scatter plan for a mesh (computed once, like the pattern):
 *   pos_map (n_cells x n_loc x n_loc int32): CSR position of every local entry;
 *   seg_ptr (nnz + 1 uint32) and perm (n_cells x n_loc^2 uint32): local-entry indices sorted
 *   stably by position -- each CSR entry's contributions in the reference's order
 *   (cell asc, i asc, j asc; assembly.cpp:50-67). seg_ptr/perm may be NULL (atomic only). */
int mpfem_b200_scatter_plan(const int32_t* cell_dofs, int64_t n_cells, int n_loc,
                            int32_t n_dofs, const int64_t* row_ptr, const int32_t* col_idx,
                            int32_t* pos_map, uint32_t* seg_ptr, uint32_t* perm, void* stream);

/* Replaces assemble_matrix (assembly.cpp:41-88): scatter-add of local matrices into
 * CSR values. mode 0 = atomic (red.global at pos_map, order-free), 1 = deterministic
 * (each entry summed sequentially in the reference's order at fmt: bitwise equal).
 *   locals: local matrices of cells [cell_begin, cell_end) (locals[0] is cell_begin's),
 *           n_loc x n_loc row-major each, fp32 (locals_fmt 2) or fp64 (3)
 *   values: CSR values, fp32 (fmt 2) or fp64 (fmt 3)
 *   rows/n_rows: mode 1 only -- restrict to these rows (NULL: every entry)
 *   accumulate: 0 = entries start empty (mode 1: first contribution taken exactly;
 *               mode 0: values zeroed), 1 = continue from the current contents (the
 *               prefix partial sums received from the rank owning lower cells). */
int mpfem_b200_assemble(const void* locals, int locals_fmt, int64_t cell_begin,
                        int64_t cell_end, int n_loc, const int64_t* row_ptr, int32_t n_dofs,
                        const int32_t* pos_map, const uint32_t* seg_ptr, const uint32_t* perm,
                        void* values, int fmt, int mode, int accumulate, const int32_t* rows,
                        int64_t n_rows, void* stream);

/* Deterministic assemble_matrix by row pull (no seg_ptr/perm plan needed): one warp per CSR row
 * replays the row's incident (cell, local row) pairs -- from the incidence lists
 * (mpfem_b200_incidence, ascending cell order) -- adding each pair's contiguous n_loc local
 * entries at their CSR positions (pos_map); values are bitwise those of mode 1 of
 * mpfem_b200_assemble (the reference's ascending-cell sequential sum, assembly.cpp:50-67).
 * rows/n_rows restrict the pass to those rows (NULL: every row); other arguments as
 * mpfem_b200_assemble. pull_pos (optional, from mpfem_b200_scatter_plan_pull) replaces pos_map
 * (which may then be NULL): the same positions as uint16 offsets into 32-row blocks, stored in
 * the order this kernel reads them, i.e. one sequential stream of half the bytes. */
int mpfem_b200_assemble_pull(const void* locals, int locals_fmt, int64_t cell_begin,
                             int64_t cell_end, int n_loc, const int64_t* row_ptr, int32_t n_dofs,
                             const int64_t* inc_ptr, const int64_t* inc, const int32_t* pos_map,
                             const uint16_t* pull_pos, void* values, int fmt, int accumulate,
                             const int32_t* rows, int64_t n_rows, void* stream);

/* ---------------------------------------------------------------- host-buffer assembly
 * The calls behind the C++ drop-in build_dofmap / assemble_matrix (include/mpfem/batched.hpp):
 * host arrays in and out, all index and value work on the GPU. */

/* build_dofmap(mesh, basis(cell_kind, dim, p), continuity) (mesh.hpp:61, mesh.cpp:204-298).
 * continuous: 3D tetrahedral or hexahedral meshes (cells n_cells x 4 or x 8 vertex ids), first-
 * encounter numbering as mpfem_b200_dofmap_cells; discontinuous: any cell kind, every cell
 * numbers its own n_loc dofs. cell_dofs: n_cells x n_loc int32 (host). */
int mpfem_b200_dofmap_host(int cell_kind, int dim, int p, int continuous, const int32_t* cells,
                           int64_t n_cells, int64_t n_verts, int32_t* cell_dofs, int32_t* n_dofs,
                           int32_t* max_multiplicity);

/* Assembly plan of a dof map: CSR pattern (the reference COO key set, assembly.cpp:67-86) and
 * the deterministic scatter plan, built on the GPU. CheckError (3) for a dof out of range
 * (assembly.cpp:31-37). */
typedef struct mpfem_b200_asm_plan_s* mpfem_b200_asm_plan_t;
int mpfem_b200_asm_plan_create(const int32_t* cell_dofs, int64_t n_cells, int n_loc, int32_t n_dofs,
                               mpfem_b200_asm_plan_t* out, int64_t* nnz);
/* row_ptr: n_dofs + 1 int64, col_idx: nnz int32 (host; either may be NULL). */
int mpfem_b200_asm_plan_pattern(mpfem_b200_asm_plan_t plan, int64_t* row_ptr, int32_t* col_idx);
/* assemble_matrix(locals, dofmap, fmt, flags) (assembly.cpp:41-88) in the deterministic mode:
 * locals n_cells x n_loc x n_loc binary64 (host), values nnz binary64 carriers of fmt (host),
 * bitwise the reference's sequential sum for every fmt (0 bf16, 1 fp16, 2 fp32, 3 fp64). */
int mpfem_b200_asm_plan_assemble(mpfem_b200_asm_plan_t plan, const double* locals, int fmt,
                                 double* values, uint32_t* flags);
int mpfem_b200_asm_plan_destroy(mpfem_b200_asm_plan_t plan);

#ifdef __cplusplus
}
#endif
#endif
