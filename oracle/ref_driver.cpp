// ref_driver.cpp -- extern "C" harness around the UNMODIFIED reference library
// (TEST INFRASTRUCTURE). Compiled together with /root/reference/proj/src/*.cpp by
// oracle/Makefile into oracle/_ref/libmpfem_ref.so. Used to (1) generate the golden
// fixtures that pin the C restatement in oracle/mpfem_oracle.c and (2) time the
// reference CPU path for bench.py --impl reference / cpu_baseline.
//
// Only the reference's public API (proj/include/mpfem/*.hpp) is called. The
// quadrature-point coefficient path composes build_H + blocked_matmul exactly as
// bilinear_kernel does (kernels.cpp:242-267) with the scaled weights C built by the
// harness from the same formula as build_C (kernels.cpp:177-197), z_q := c(x_q).
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mpfem/assembly.hpp"
#include "mpfem/bounds.hpp"
#include "mpfem/common.hpp"
#include "mpfem/elements.hpp"
#include "mpfem/geometry.hpp"
#include "mpfem/kernels.hpp"
#include "mpfem/mesh.hpp"
#include "mpfem/mm_units.hpp"
#include "mpfem/quadrature.hpp"
#include "mpfem/softfloat.hpp"

using namespace mpfem;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const CheckError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

const ReferenceCell kTet{CellKind::simplex, 3};

KernelConfig make_cfg(int form, const int* cfg, ModeKind mode = ModeKind::bilinear) {
  KernelConfig c;
  c.form = form ? FormKind::poisson : FormKind::mass;
  c.mode = mode;
  c.u_p = Fmt(cfg[0]);
  c.u_g = Fmt(cfg[1]);
  c.u_q = Fmt(cfg[2]);
  c.u_s = Fmt(cfg[3]);
  c.engine = EngineKind(cfg[4]);
  return c;
}

Mesh single_tet(const double* v) {
  Mesh m;
  m.kind = CellKind::simplex;
  m.dim = 3;
  for (int k = 0; k < 4; ++k) m.vertices.push_back({v[3 * k], v[3 * k + 1], v[3 * k + 2]});
  m.cells.push_back({0, 1, 2, 3});
  return m;
}

// Harness coefficient c(x_q) at x_q = v0 + J xi_q (binary64, left to right).
double coef_at(int kind, const double* v, const double* coef, const double* xi) {
  if (kind == 1) {
    double x[3];
    for (int i = 0; i < 3; ++i) {
      double acc = v[i];
      for (int s = 0; s < 3; ++s) acc = acc + (v[(s + 1) * 3 + i] - v[i]) * xi[s];
      x[i] = acc;
    }
    const double two_pi = 6.283185307179586476925286766559;
    double s = std::sin(two_pi * x[0]);
    double c = std::cos(two_pi * x[1]);
    double e = std::exp(x[2]);
    return 1.0 + 0.5 * s * c * e;
  }
  double l0 = ((1.0 - xi[0]) - xi[1]) - xi[2];
  double u = coef[0] * l0 + coef[1] * xi[0] + coef[2] * xi[1] + coef[3] * xi[2];
  return std::pow(10.0, 6.0 * u);
}

// Same-mode cell matrix for one cell through the reference's public API.
Mat cell_matrix(const KernelSetup& setup, const double* v, int kind, const double* coef,
                FpFlags& flags) {
  Mesh mesh = single_tet(v);
  const KernelConfig& cfg = setup.config;
  GeometryData geom = cell_geometry(mesh, 0, setup.rule, cfg.form, cfg.u_g, flags);
  if (kind == 0) return bilinear_kernel(setup, geom, {}, flags);
  if (kind == 3) {
    Coefficients z(coef, coef + setup.basis.n_phi);
    return bilinear_kernel(setup, geom, z, flags);
  }
  int n_d = setup.n_d, n_q = setup.rule.n_points, n_phi = setup.basis.n_phi;
  std::vector<double> c(std::size_t(n_d) * n_d * n_q);
  for (int q = 0; q < n_q; ++q) {
    double zq = round_to(coef_at(kind, v, coef, setup.rule.point(q)), cfg.u_g, flags);
    double omega = fp_cast(setup.rule.weights[q], Fmt::fp64, cfg.u_g, flags);
    const GeometryPoint& gp = geom.at(q);
    for (int s = 0; s < n_d; ++s)
      for (int t = 0; t < n_d; ++t) {
        double value = fp_mul(omega, gp.tensor(s, t), cfg.u_g, flags);
        value = fp_mul(value, zq, cfg.u_g, flags);
        c[(std::size_t(s) * n_d + t) * n_q + q] = fp_cast(value, cfg.u_g, cfg.u_s, flags);
      }
  }
  Mat h_cat(n_d * n_d * n_q, n_phi);
  for (int s = 0; s < n_d; ++s)
    for (int t = 0; t < n_d; ++t) {
      Mat h = build_H(setup, c, s, t, flags);
      int row0 = (s * n_d + t) * n_q;
      for (int q = 0; q < n_q; ++q)
        for (int k = 0; k < n_phi; ++k) h_cat(row0 + q, k) = h(q, k);
    }
  return blocked_matmul(setup.b_cat_bilinear, h_cat, cfg.engine, cfg.u_q, flags);
}

// Same-mode action v (n_phi) for one cell through the reference's public API. Nodal /
// constant coefficients call action_kernel itself (kernels.cpp:269-304). The quadrature-
// point coefficient path composes the same stages from public pieces: the w evaluation as
// eval_w_at_ug does it (blocked_matmul of the u_s-rounded w against setup.store_slabs at
// u_p, cast to u_g; kernels.cpp:145-173), the integrand with z_q := c(x_q) at u_g
// (kernels.cpp:280-301), and blocked_matmul(setup.b_cat_action, r, engine, u_q).
std::vector<double> cell_action(const KernelSetup& setup, const double* v, int kind,
                                const double* coef, const double* w, FpFlags& flags) {
  Mesh mesh = single_tet(v);
  const KernelConfig& cfg = setup.config;
  GeometryData geom = cell_geometry(mesh, 0, setup.rule, cfg.form, cfg.u_g, flags);
  int n_d = setup.n_d, n_q = setup.rule.n_points, n_phi = setup.basis.n_phi;
  Coefficients wv(w, w + n_phi);
  if (kind == 0 || kind == 3) {
    Coefficients z;
    if (kind == 3) z.assign(coef, coef + n_phi);
    Mat out = action_kernel(setup, {geom}, {wv}, z, flags);
    return out.a;
  }
  Mat wmat(1, n_phi);
  for (int k = 0; k < n_phi; ++k) wmat(0, k) = fp_cast(w[k], Fmt::fp64, cfg.u_s, flags);
  std::vector<double> what(std::size_t(n_d) * n_q);
  for (int s = 0; s < n_d; ++s) {
    Mat vals = blocked_matmul(wmat, setup.store_slabs[s], cfg.engine, cfg.u_p, flags);
    for (int q = 0; q < n_q; ++q) what[std::size_t(s) * n_q + q] = fp_cast(vals(0, q), cfg.u_p, cfg.u_g, flags);
  }
  Mat r_cat(n_d * n_q, 1);
  for (int q = 0; q < n_q; ++q) {
    double zq = round_to(coef_at(kind, v, coef, setup.rule.point(q)), cfg.u_g, flags);
    double omega = fp_cast(setup.rule.weights[q], Fmt::fp64, cfg.u_g, flags);
    const GeometryPoint& gp = geom.at(q);
    for (int s = 0; s < n_d; ++s) {
      double t1 = 0.0;
      for (int t = 0; t < n_d; ++t)
        t1 = fp_add(t1, fp_mul(gp.tensor(s, t), what[std::size_t(t) * n_q + q], cfg.u_g, flags),
                    cfg.u_g, flags);
      double m1 = fp_mul(omega, t1, cfg.u_g, flags);
      m1 = fp_mul(m1, zq, cfg.u_g, flags);
      r_cat(s * n_q + q, 0) = fp_cast(m1, cfg.u_g, cfg.u_s, flags);
    }
  }
  return blocked_matmul(setup.b_cat_action, r_cat, cfg.engine, cfg.u_q, flags).a;
}

uint32_t pack(const FpFlags& f) {
  return (f.overflow ? 1u : 0u) | (f.underflow ? 2u : 0u) | (f.invalid ? 4u : 0u) |
         (f.divzero ? 8u : 0u);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_rng_draws(uint64_t seed, int n, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next();
}

double ref_round(double x, int fmt, int ftz, uint32_t* flags) {
  FpFlags f;
  double r = round_to(x, Fmt(fmt), f,
                      ftz ? SubnormalPolicy::flush_to_zero : SubnormalPolicy::supported);
  if (flags) *flags |= pack(f);
  return r;
}

int ref_rule_simplex3(int p, double* pts, double* wts) {
  return guard([&] {
    QuadratureRule r = rule_for(kTet, p);
    std::memcpy(pts, r.points.data(), sizeof(double) * r.points.size());
    std::memcpy(wts, r.weights.data(), sizeof(double) * r.weights.size());
  });
}

int ref_tabulate(int p, int ef, int sf, int grads, double* out) {
  return guard([&] {
    FpFlags f;
    LagrangeBasis b = build_basis(kTet, p);
    Tabulation t = tabulate(b, rule_for(kTet, p), Fmt(ef), Fmt(sf), grads != 0, f);
    std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
  });
}

int ref_basis_nodes(int p, double* nodes) {
  return guard([&] {
    LagrangeBasis b = build_basis(kTet, p);
    for (int k = 0; k < b.n_phi; ++k)
      for (int a = 0; a < 3; ++a) nodes[3 * k + a] = b.nodes[k][a];
  });
}

int ref_basis_conditioning(int p, double* leb, double* gleb, double* gk, double* gkmax) {
  return guard([&] {
    BasisConditioning bc = basis_condition_numbers(build_basis(kTet, p));
    *leb = bc.lebesgue;
    for (int s = 0; s < 3; ++s) {
      gleb[s] = bc.grad_lebesgue[s];
      gkmax[s] = bc.grad_kappa_max[s];
    }
    for (int i = 0; i < bc.grad_kappa.rows; ++i)
      for (int s = 0; s < 3; ++s) gk[3 * i + s] = bc.grad_kappa(i, s);
  });
}

// Same output layout as orc_cell_geometry.
int ref_cell_geometry(const double* verts, int form, int fmt, double* out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    Mesh mesh = single_tet(verts);
    QuadratureRule rule = rule_for(kTet, 1);
    GeometryData g = cell_geometry(mesh, 0, rule, form ? FormKind::poisson : FormKind::mass,
                                   Fmt(fmt), f);
    const GeometryPoint& gp = g.at(0);
    std::memset(out, 0, sizeof(double) * 40);
    out[0] = gp.det;
    out[1] = gp.abs_det;
    for (int i = 0; i < 9; ++i) out[2 + i] = gp.jac.a[i];
    for (int i = 0; i < 9; ++i) out[11 + i] = gp.inv.a[i];
    for (std::size_t i = 0; i < gp.tensor.a.size(); ++i) out[20 + i] = gp.tensor.a[i];
    out[29] = gp.kappa2;
    out[30] = gp.kappa_cell;
    for (std::size_t i = 0; i < gp.tensor_tilde.a.size(); ++i) out[31 + i] = gp.tensor_tilde.a[i];
    if (flags) *flags |= pack(f);
  });
}

// Scaled weights: nodal/one via the reference's build_C; analytic via the harness.
int ref_build_C(int p, int form, const int* cfg, const double* verts, int kind,
                const double* coef, double* c_out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kTet, p, make_cfg(form, cfg));
    Mesh mesh = single_tet(verts);
    GeometryData geom = cell_geometry(mesh, 0, setup.rule, setup.config.form,
                                      setup.config.u_g, f);
    std::vector<double> c;
    if (kind == 0) {
      c = build_C(setup, geom, {}, f);
    } else if (kind == 3) {
      c = build_C(setup, geom, Coefficients(coef, coef + setup.basis.n_phi), f);
    } else {
      const KernelConfig& k = setup.config;
      int n_d = setup.n_d, n_q = setup.rule.n_points;
      c.resize(std::size_t(n_d) * n_d * n_q);
      for (int q = 0; q < n_q; ++q) {
        double zq = round_to(coef_at(kind, verts, coef, setup.rule.point(q)), k.u_g, f);
        double omega = fp_cast(setup.rule.weights[q], Fmt::fp64, k.u_g, f);
        for (int s = 0; s < n_d; ++s)
          for (int t = 0; t < n_d; ++t) {
            double value = fp_mul(omega, geom.at(q).tensor(s, t), k.u_g, f);
            value = fp_mul(value, zq, k.u_g, f);
            c[(std::size_t(s) * n_d + t) * n_q + q] = fp_cast(value, k.u_g, k.u_s, f);
          }
      }
    }
    std::memcpy(c_out, c.data(), sizeof(double) * c.size());
    if (flags) *flags |= pack(f);
  });
}

int ref_bilinear(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                 const double* coef, int coef_stride, double* a_out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kTet, p, make_cfg(form, cfg));
    std::size_t n2 = std::size_t(setup.basis.n_phi) * setup.basis.n_phi;
    for (int64_t c = 0; c < m; ++c) {
      Mat a = cell_matrix(setup, verts + 12 * c, kind, coef ? coef + coef_stride * c : nullptr, f);
      std::memcpy(a_out + n2 * c, a.a.data(), sizeof(double) * n2);
    }
    if (flags) *flags |= pack(f);
  });
}

// kernel_bounds for constant / nodal coefficients (reference-native).
int ref_bound(int p, int form, const int* cfg, const double* verts, int kind,
              const double* coef, double* out4, double* a64) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kTet, p, make_cfg(form, cfg));
    BasisConditioning bc = basis_condition_numbers(setup.basis);
    Mesh mesh = single_tet(verts);
    GeometryData g64 = cell_geometry(mesh, 0, setup.rule, setup.config.form, Fmt::fp64, f);
    Coefficients z;
    if (kind == 3) z.assign(coef, coef + setup.basis.n_phi);
    BoundReport r = kernel_bounds(setup, bc, g64, z, {});
    out4[0] = r.bound_a;
    out4[1] = r.kappa_q_a;
    out4[2] = r.kappa_p_a;
    out4[3] = r.kappa_g_a;
    if (a64) std::memcpy(a64, r.a.a.data(), sizeof(double) * r.a.a.size());
  });
}

int ref_action(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
               const double* coef, int coef_stride, const double* w, int w_stride,
               double* v_out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kTet, p, make_cfg(form, cfg, ModeKind::action));
    int n_phi = setup.basis.n_phi;
    for (int64_t c = 0; c < m; ++c) {
      std::vector<double> v = cell_action(setup, verts + 12 * c, kind,
                                          coef ? coef + int64_t(coef_stride) * c : nullptr,
                                          w + int64_t(w_stride) * c, f);
      std::memcpy(v_out + int64_t(n_phi) * c, v.data(), sizeof(double) * n_phi);
    }
    if (flags) *flags |= pack(f);
  });
}

// kernel_bounds with w (bound_v, report.v) for constant / nodal coefficients.
int ref_action_bound(int p, int form, const int* cfg, const double* verts, int kind,
                     const double* coef, const double* w, double* out4, double* v64) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kTet, p, make_cfg(form, cfg, ModeKind::action));
    BasisConditioning bc = basis_condition_numbers(setup.basis);
    Mesh mesh = single_tet(verts);
    GeometryData g64 = cell_geometry(mesh, 0, setup.rule, setup.config.form, Fmt::fp64, f);
    Coefficients z;
    if (kind == 3) z.assign(coef, coef + setup.basis.n_phi);
    Coefficients wv(w, w + setup.basis.n_phi);
    BoundReport r = kernel_bounds(setup, bc, g64, z, wv);
    out4[0] = r.bound_v;
    out4[1] = r.kappa_q_v;
    out4[2] = r.kappa_p_v;
    out4[3] = r.kappa_g_v;
    if (v64) std::memcpy(v64, r.v.data(), sizeof(double) * r.v.size());
  });
}

// Box (hexahedral) cells through the reference's public API: a one-hex mesh, cell_geometry at
// every rule point, bilinear_kernel / build_C / kernel_bounds (constant or nodal z).
Mesh single_hex(const double* v) {
  Mesh m;
  m.kind = CellKind::box;
  m.dim = 3;
  for (int k = 0; k < 8; ++k) m.vertices.push_back({v[3 * k], v[3 * k + 1], v[3 * k + 2]});
  m.cells.push_back({0, 1, 2, 3, 4, 5, 6, 7});
  return m;
}
const ReferenceCell kHex{CellKind::box, 3};

int ref_bilinear_box(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                     const double* coef, int coef_stride, double* a_out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kHex, p, make_cfg(form, cfg));
    std::size_t n2 = std::size_t(setup.basis.n_phi) * setup.basis.n_phi;
    for (int64_t c = 0; c < m; ++c) {
      Mesh mesh = single_hex(verts + 24 * c);
      GeometryData geom = cell_geometry(mesh, 0, setup.rule, setup.config.form, setup.config.u_g, f);
      Coefficients z;
      if (kind == 3) z.assign(coef + coef_stride * c, coef + coef_stride * c + setup.basis.n_phi);
      Mat a = bilinear_kernel(setup, geom, z, f);
      std::memcpy(a_out + n2 * c, a.a.data(), sizeof(double) * n2);
    }
    if (flags) *flags |= pack(f);
  });
}

int ref_build_C_box(int p, int form, const int* cfg, const double* verts, int kind,
                    const double* coef, double* c_out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kHex, p, make_cfg(form, cfg));
    Mesh mesh = single_hex(verts);
    GeometryData geom = cell_geometry(mesh, 0, setup.rule, setup.config.form, setup.config.u_g, f);
    Coefficients z;
    if (kind == 3) z.assign(coef, coef + setup.basis.n_phi);
    std::vector<double> c = build_C(setup, geom, z, f);
    std::memcpy(c_out, c.data(), sizeof(double) * c.size());
    if (flags) *flags |= pack(f);
  });
}

int ref_bound_box(int p, int form, const int* cfg, const double* verts, int kind,
                  const double* coef, double* out4, double* a64) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kHex, p, make_cfg(form, cfg));
    BasisConditioning bc = basis_condition_numbers(setup.basis);
    Mesh mesh = single_hex(verts);
    GeometryData g64 = cell_geometry(mesh, 0, setup.rule, setup.config.form, Fmt::fp64, f);
    Coefficients z;
    if (kind == 3) z.assign(coef, coef + setup.basis.n_phi);
    BoundReport r = kernel_bounds(setup, bc, g64, z, {});
    out4[0] = r.bound_a;
    out4[1] = r.kappa_q_a;
    out4[2] = r.kappa_p_a;
    out4[3] = r.kappa_g_a;
    if (a64) std::memcpy(a64, r.a.a.data(), sizeof(double) * r.a.a.size());
  });
}

int ref_action_box(int p, int form, const int* cfg, int64_t m, const double* verts, int kind,
                   const double* coef, int coef_stride, const double* w, int w_stride,
                   double* v_out, uint32_t* flags) {
  return guard([&] {
    FpFlags f;
    KernelSetup setup = make_setup(kHex, p, make_cfg(form, cfg, ModeKind::action));
    int n_phi = setup.basis.n_phi;
    for (int64_t c = 0; c < m; ++c) {
      Mesh mesh = single_hex(verts + 24 * c);
      GeometryData geom = cell_geometry(mesh, 0, setup.rule, setup.config.form, setup.config.u_g, f);
      Coefficients z;
      if (kind == 3) z.assign(coef + coef_stride * c, coef + coef_stride * c + n_phi);
      Coefficients wv(w + int64_t(w_stride) * c, w + int64_t(w_stride) * c + n_phi);
      Mat v = action_kernel(setup, {geom}, {wv}, z, f);
      std::memcpy(v_out + int64_t(n_phi) * c, v.a.data(), sizeof(double) * n_phi);
    }
    if (flags) *flags |= pack(f);
  });
}

int ref_structured_tet_mesh(int nx, int ny, int nz, double extent, double jitter, uint64_t seed,
                            double* verts, int32_t* cells) {
  return guard([&] {
    Mesh m = structured_tet_mesh(nx, ny, nz, extent, jitter, seed);
    for (std::size_t v = 0; v < m.vertices.size(); ++v)
      for (int a = 0; a < 3; ++a) verts[3 * v + a] = m.vertices[v][a];
    for (std::size_t c = 0; c < m.cells.size(); ++c)
      for (int k = 0; k < 4; ++k) cells[4 * c + k] = m.cells[c][k];
  });
}

int ref_build_dofmap(int p, int64_t n_verts, const double* verts, int64_t n_cells,
                     const int32_t* cells, int32_t* cell_dofs, int32_t* n_dofs,
                     int32_t* max_mult) {
  return guard([&] {
    Mesh m;
    m.kind = CellKind::simplex;
    m.dim = 3;
    m.vertices.resize(std::size_t(n_verts));
    for (int64_t v = 0; v < n_verts; ++v)
      m.vertices[v] = {verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    m.cells.resize(std::size_t(n_cells));
    for (int64_t c = 0; c < n_cells; ++c)
      m.cells[c] = {cells[4 * c], cells[4 * c + 1], cells[4 * c + 2], cells[4 * c + 3]};
    DofMap d = build_dofmap(m, build_basis(kTet, p), Continuity::continuous);
    std::memcpy(cell_dofs, d.cell_dofs.data(), sizeof(int32_t) * d.cell_dofs.size());
    *n_dofs = d.n_dofs;
    *max_mult = d.max_multiplicity;
  });
}

int ref_assemble_matrix(int64_t n_cells, int n_loc, const int32_t* cd, int32_t n_dofs,
                        const double* locals, int fmt, int64_t* nnz, int32_t* rows,
                        int32_t* cols, double* values, uint32_t* flags) {
  return guard([&] {
    DofMap d;
    d.n_dofs = n_dofs;
    d.n_local = n_loc;
    d.cell_dofs.assign(cd, cd + n_cells * n_loc);
    std::vector<Mat> loc(std::size_t(n_cells), Mat(n_loc, n_loc));
    for (int64_t c = 0; c < n_cells; ++c)
      std::memcpy(loc[c].a.data(), locals + std::size_t(c) * n_loc * n_loc,
                  sizeof(double) * n_loc * n_loc);
    FpFlags f;
    SparseCoo coo = assemble_matrix(loc, d, Fmt(fmt), f);
    *nnz = coo.nnz();
    if (rows) {
      std::memcpy(rows, coo.row.data(), sizeof(int32_t) * coo.row.size());
      std::memcpy(cols, coo.col.data(), sizeof(int32_t) * coo.col.size());
      std::memcpy(values, coo.value.data(), sizeof(double) * coo.value.size());
    }
    if (flags) *flags |= pack(f);
  });
}

// CPU baseline: the reference's same-mode path (cell_geometry + kernel) over a bounded
// sample of cells, run with mpfem::parallel_for on `threads` workers (MPFEM_THREADS).
// Returns wall seconds in *seconds; outputs are discarded except a checksum.
int ref_cpu_baseline(int p, int form, const int* cfg, int64_t m, const double* verts,
                     int kind, const double* coef, int coef_stride, int threads,
                     double* seconds, double* checksum) {
  return guard([&] {
    std::string t = std::to_string(threads);
    setenv("MPFEM_THREADS", t.c_str(), 1);
    KernelSetup setup = make_setup(kTet, p, make_cfg(form, cfg));
    std::vector<double> sums(std::size_t(m), 0.0);
    auto t0 = std::chrono::steady_clock::now();
    parallel_for(int(m), [&](int c) {
      FpFlags f;
      Mat a = cell_matrix(setup, verts + 12 * c, kind, coef ? coef + coef_stride * c : nullptr, f);
      sums[c] = a.a[0];
    });
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    double s = 0.0;
    for (double v : sums) s += v;
    *checksum = s;
  });
}

}  // extern "C"
