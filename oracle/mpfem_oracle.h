/*
 * mpfem_oracle.h -- CPU restatement of the reference algorithm (TEST INFRASTRUCTURE).
 *
 * This library is the parity CHECKER for the B200 product. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it. The product path (paper_2410_12614_b200) never links or calls it.
 *
 * Every function restates an algorithm of the reference artifact
 * (/root/reference/proj, "mpfem") and cites the file:line it follows. It is
 * pinned against the reference itself: oracle/ref_driver.cpp compiles the
 * reference sources out-of-tree (oracle/Makefile -> oracle/_ref/) and
 * tests/golden/make_golden.py dumps its outputs as fixtures that
 * tests/test_oracle_golden.py checks this restatement against bit for bit.
 *
 * Formats: 0 = bf16, 1 = fp16, 2 = fp32, 3 = fp64 (softfloat.hpp:17).
 * Flag bits: 1 overflow, 2 underflow, 4 invalid, 8 divzero (softfloat.hpp:22-36).
 * Status codes: 0 ok, 2 ConfigError, 3 CheckError (mpfem_cli.cpp:517-527).
 */
#ifndef MPFEM_ORACLE_H
#define MPFEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_BF16 = 0, ORC_FP16 = 1, ORC_FP32 = 2, ORC_FP64 = 3 };
enum { ORC_MASS = 0, ORC_POISSON = 1 };
/* Coefficient kinds (shared with the product's C-ABI):
 * 0 one (empty z), 1 c(x)=1+0.5 sin(2 pi x) cos(2 pi y) e^z at x_q,
 * 2 c=10^(6 u(x_q)) with u affine per cell (4 vertex values),
 * 3 nodal z (n_phi values per cell, reference eval_z_at_ug path). */
enum { ORC_COEF_ONE = 0, ORC_COEF_SINCOSEXP = 1, ORC_COEF_EXP10_AFFINE = 2,
       ORC_COEF_NODAL = 3 };

/* softfloat */
double orc_round(double x, int fmt, int ftz, uint32_t* flags);
double orc_op(double a, double b, int op /*0 add 1 sub 2 mul 3 div*/, int fmt, int ftz,
              uint32_t* flags);

/* Rng (common.hpp:21-35) */
typedef struct { uint64_t mt[312]; int mti; } orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double a, double b);
/* first n raw draws for pinning against std::mt19937_64 */
void orc_rng_draws(uint64_t seed, int n, uint64_t* out);

/* quadrature */
int orc_gauss_legendre_1d(int n, double* x, double* w);
int orc_gauss_jacobi_1d(int n, int alpha, double* x, double* w);
int orc_rule_simplex3(int p, double* points /* n_q x 3 */, double* weights /* n_q */);

/* elements (tets, dim 3) */
int orc_nphi(int p);
int orc_nq(int p);
int orc_basis_nodes(int p, double* nodes /* n_phi x 3 */);
int orc_tabulate(int p, int eval_fmt, int store_fmt, int gradients,
                 double* out /* n_d x n_phi x n_q */, uint32_t* flags);
int orc_basis_conditioning(int p, double* lebesgue, double* grad_lebesgue /*3*/,
                           double* grad_kappa /* n_phi x 3 */, double* grad_kappa_max /*3*/);

/* geometry of one affine tet (geometry.cpp). out layout (doubles):
 * [0] det, [1] abs_det, [2..10] jac, [11..19] inv, [20..28] tensor (3x3, mass: [20]),
 * [29] kappa2, [30] kappa_cell, [31..39] tensor_tilde. */
#define ORC_GEOM_SIZE 40
int orc_cell_geometry(const double* verts /* 4 x 3 */, int form, int fmt, double* out,
                      uint32_t* flags);

/* Kernel config: cfg[0..3] = u_p, u_g, u_q, u_s; cfg[4] = engine (0 scalar,1 vector,2 matrix) */

/* scaled weights C (kernels.cpp:177-197) for one cell; coef semantic per kind. */
int orc_build_C(int p, int form, const int* cfg, const double* verts, int coef_kind,
                const double* coef, double* c_out /* n_d^2 x n_q */, uint32_t* flags);

/* Reference Algorithm 1 (kernels.cpp:242-267): A (n_phi x n_phi) for M cells. */
int orc_bilinear(int p, int form, const int* cfg, int64_t m, const double* verts /* m x 12 */,
                 int coef_kind, const double* coef, int coef_stride, double* a_out,
                 uint32_t* flags);

/* Restated kernel_bounds (bounds.cpp:29-281), bilinear part; z_at from coef kind.
 * out[0] = bound_a, out[1] = kappa_q, out[2] = kappa_p, out[3] = kappa_g; a64 gets the
 * exact binary64 A (report.a). */
int orc_bound(int p, int form, const int* cfg, const double* verts, int coef_kind,
              const double* coef, double* out4, double* a64);

/* Reference Algorithm 2, action_kernel (kernels.cpp:269-304) incl. eval_w_at_ug
 * (kernels.cpp:145-173): v (n_phi per cell) for M cells, w (n_phi per cell, row stride
 * w_stride). Coefficient kinds as orc_bilinear. */
int orc_action(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
               const double* coef, int coef_stride, const double* w, int w_stride,
               double* v_out, uint32_t* flags);

/* Restated kernel_bounds, action part (bounds.cpp:128-155,222-279): out4 = {bound_v,
 * kappa_q_v, kappa_p_v, kappa_g_v}; v64 = exact binary64 v (report.v). */
int orc_action_bound(int p, int form, const int* cfg, const double* verts, int kind,
                     const double* coef, const double* w, double* out4, double* v64);

/* Box (hexahedral) cells: tensor Lagrange basis with equispaced nodes
 * (elements.cpp:50-87), Gauss-Legendre rule (quadrature.cpp:171-224), geometry at every rule
 * point through the trilinear map (geometry.cpp:12-27,190-245); p <= 4; coefficient kinds
 * ONE or NODAL. verts: 8 x 3 per cell in the lattice's bit order (x fastest). */
int orc_rule_box3(int p, double* points, double* weights);
int orc_bilinear_box(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                     const double* coef, int coef_stride, double* a_out, uint32_t* flags);
int orc_build_C_box(int p, int form, const int* cfg, const double* verts, int kind,
                    const double* coef, double* c_out, uint32_t* flags);
int orc_bound_box(int p, int form, const int* cfg, const double* verts, int kind,
                  const double* coef, double* out4, double* a64);
int orc_action_box(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                   const double* coef, int coef_stride, const double* w, int w_stride,
                   double* v_out, uint32_t* flags);

/* Physical quadrature points x_q = v0 + J (xi_q) in fp64 and the coefficient there. */
int orc_coef_at_q(int p, const double* verts, int coef_kind, const double* coef,
                  double* c_q /* n_q */);

/* Synthetic inputs. kind 0: config-0 tets (ref tet + U(-0.15,0.15) noise, reject
 * |det|<1e-3, swap 2<->3 if det<0); kind 1: config-3 anisotropic rotated tets with
 * 4 affine-field values per cell in coef_out (m x 4). */
int orc_gen_tets(int kind, uint64_t seed, int64_t m, double* verts, double* coef_out);

/* Mesh (mesh.cpp:78-163) */
int orc_tet_mesh_sizes(int nx, int ny, int nz, int64_t* n_verts, int64_t* n_cells);
int orc_structured_tet_mesh(int nx, int ny, int nz, double extent, double jitter,
                            uint64_t seed, double* verts, int32_t* cells);

/* Dofmap (mesh.cpp:204-298), continuous. Returns status; n_dofs, max_mult out. */
int orc_build_dofmap(int p, int64_t n_verts, const double* verts, int64_t n_cells,
                     const int32_t* cells, int32_t* cell_dofs, int32_t* n_dofs,
                     int32_t* max_mult);

/* assemble_matrix (assembly.cpp:41-88): returns nnz via *nnz; if rows==NULL only counts.
 * locals: n_cells x n_loc x n_loc doubles. */
int orc_assemble_matrix(int64_t n_cells, int n_loc, const int32_t* cell_dofs, int32_t n_dofs,
                        const double* locals, int fmt, int64_t* nnz, int32_t* rows,
                        int32_t* cols, double* values, uint32_t* flags);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
