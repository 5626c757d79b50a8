// mpfem_b200_shim.cpp -- the reference's hot-path C++ API re-implemented on the B200 C-ABI.
//
// Compiled against the reference's unchanged headers (proj/include/mpfem), this translation
// unit defines
//   mpfem::bilinear_kernel   kernels.hpp:85-86   (+ the batched overloads of batched.hpp)
//   mpfem::action_kernel     kernels.hpp:90-92
//   mpfem::build_dofmap      mesh.hpp:61
//   mpfem::assemble_matrix   assembly.hpp:29-30
// so a maintainer links it (and libmpfem_b200.so) instead of those reference definitions; every
// other reference function (make_setup, cell_geometry, build_C, ...) stays the reference's.
// The per-cell calls become GPU batches of one: correct, and the batched overloads are the
// fast path. Device setups are created from the caller's KernelSetup (its rule, tab_store and
// tab_values, mpfem_b200_setup_create_tab) and cached per configuration and tabulation.
// Errors map to the reference's exceptions: status 2 -> ConfigError, 3 -> CheckError.
#include <bit>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "mpfem/assembly.hpp"
#include "mpfem/batched.hpp"
#include "mpfem/kernels.hpp"
#include "mpfem/mesh.hpp"
#include "mpfem_b200.h"

namespace mpfem {
namespace {

void check(int status) {
  if (status == MPFEM_B200_OK) return;
  const std::string msg = mpfem_b200_last_error();
  if (status == MPFEM_B200_CONFIG_ERROR) throw ConfigError(msg);
  if (status == MPFEM_B200_CHECK_ERROR) throw CheckError(msg);
  throw std::runtime_error("mpfem_b200: " + msg);
}

void merge_flags(FpFlags& flags, uint32_t bits) {
  flags.overflow |= (bits & 1u) != 0;
  flags.underflow |= (bits & 2u) != 0;
  flags.invalid |= (bits & 4u) != 0;
  flags.divzero |= (bits & 8u) != 0;
}

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

using SetupKey = std::tuple<int, int, int, int, int, int, int, int, int, int, int, int, uint64_t>;

// Device setups live until release_device_setups() or process exit. The cache is never
// destroyed by a static destructor: at exit the CUDA runtime may already be torn down, and
// releasing device memory then corrupts its state; the driver reclaims everything anyway.
struct Cache {
  std::mutex mu;
  std::map<SetupKey, mpfem_b200_setup_t> setups;
};
Cache& cache() {
  static Cache* c = new Cache();
  return *c;
}

// The device setup of a reference KernelSetup: same config, rule and operand tabulations.
mpfem_b200_setup_t device_setup(const KernelSetup& setup) {
  const KernelConfig& c = setup.config;
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, setup.rule.points.data(), sizeof(double) * setup.rule.points.size());
  h = fnv(h, setup.rule.weights.data(), sizeof(double) * setup.rule.weights.size());
  h = fnv(h, setup.tab_store.data.data(), sizeof(double) * setup.tab_store.data.size());
  h = fnv(h, setup.tab_values.data.data(), sizeof(double) * setup.tab_values.data.size());
  const SetupKey key{int(setup.basis.cell.kind), setup.basis.cell.dim, setup.basis.p, int(c.form),
                     int(c.mode), int(c.u_p), int(c.u_g), int(c.u_q), int(c.u_s), int(c.engine),
                     c.n_batch, setup.rule.n_points, h};
  Cache& C = cache();
  std::lock_guard<std::mutex> lk(C.mu);
  auto it = C.setups.find(key);
  if (it != C.setups.end()) return it->second;
  mpfem_b200_setup_t s = nullptr;
  check(mpfem_b200_setup_create_tab(
      setup.basis.cell.kind == CellKind::box ? 1 : 0, setup.basis.cell.dim, setup.basis.p,
      int(c.form), int(c.u_p), int(c.u_g), int(c.u_q), int(c.u_s), int(c.engine), c.n_batch,
      setup.basis.n_phi, setup.rule.n_points, setup.rule.points.data(), setup.rule.weights.data(),
      setup.tab_store.data.data(), setup.tab_values.data.data(), &s));
  C.setups.emplace(key, s);
  return s;
}

// Geometry tensors of a batch, n_cells x n_pts x n_d x n_d (GeometryPoint::tensor).
std::vector<double> pack_geometry(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                                  int* n_pts_out) {
  const int n_q = setup.rule.n_points;
  const int nd = setup.n_d;
  int n_pts = 1;
  for (const GeometryData& g : geoms)
    if (!g.affine) n_pts = n_q;
  std::vector<double> G(geoms.size() * size_t(n_pts) * nd * nd);
  for (size_t c = 0; c < geoms.size(); ++c) {
    const GeometryData& g = geoms[c];
    if (!g.affine && g.n_entries() != n_q) throw ConfigError("geometry does not match the quadrature rule");
    for (int p = 0; p < n_pts; ++p) {
      const GeometryPoint& gp = g.at(p);
      if (gp.tensor.rows != nd || gp.tensor.cols != nd)
        throw ConfigError("geometry tensor does not match the form");
      std::memcpy(G.data() + (c * n_pts + p) * nd * nd, gp.tensor.a.data(), sizeof(double) * nd * nd);
    }
  }
  *n_pts_out = n_pts;
  return G;
}

std::vector<Mat> run_bilinear(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                              const double* z, int64_t z_stride, FpFlags& flags) {
  if (setup.config.mode != ModeKind::bilinear)
    throw ConfigError("configuration is not a bilinear-mode config");
  const int n_phi = setup.basis.n_phi;
  std::vector<Mat> out;
  if (geoms.empty()) return out;
  mpfem_b200_setup_t s = device_setup(setup);
  int n_pts = 1;
  const std::vector<double> G = pack_geometry(setup, geoms, &n_pts);
  const int64_t n2 = int64_t(n_phi) * n_phi;
  const bool f64 = setup.config.u_q == Fmt::fp64;
  std::vector<double> o64(f64 ? geoms.size() * n2 : 0);
  std::vector<float> o32(f64 ? 0 : geoms.size() * n2);
  uint32_t fl = 0;
  check(mpfem_b200_bilinear_from_geometry(s, G.data(), n_pts, int64_t(geoms.size()), z, z_stride,
                                          f64 ? static_cast<void*>(o64.data()) : o32.data(), n2,
                                          nullptr, &fl));
  merge_flags(flags, fl);
  out.reserve(geoms.size());
  for (size_t c = 0; c < geoms.size(); ++c) {
    Mat a(n_phi, n_phi);
    for (int64_t e = 0; e < n2; ++e) a.a[e] = f64 ? o64[c * n2 + e] : double(o32[c * n2 + e]);
    out.push_back(std::move(a));
  }
  return out;
}

}  // namespace

Mat bilinear_kernel(const KernelSetup& setup, const GeometryData& geom, const Coefficients& z,
                    FpFlags& flags) {
  if (setup.config.mode != ModeKind::bilinear)
    throw ConfigError("configuration is not a bilinear-mode config");
  if (!z.empty() && int(z.size()) != setup.basis.n_phi)
    throw ConfigError("coefficient z needs one entry per basis function");
  return run_bilinear(setup, {geom}, z.empty() ? nullptr : z.data(), 0, flags).front();
}

std::vector<Mat> bilinear_kernel(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                                 const Coefficients& z, FpFlags& flags) {
  if (!z.empty() && int(z.size()) != setup.basis.n_phi)
    throw ConfigError("coefficient z needs one entry per basis function");
  return run_bilinear(setup, geoms, z.empty() ? nullptr : z.data(), 0, flags);
}

std::vector<Mat> bilinear_kernel(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                                 const std::vector<Coefficients>& z, FpFlags& flags) {
  const int n_phi = setup.basis.n_phi;
  if (z.size() != geoms.size()) throw ConfigError("one coefficient vector per cell required");
  std::vector<double> zz(z.size() * size_t(n_phi));
  for (size_t c = 0; c < z.size(); ++c) {
    if (int(z[c].size()) != n_phi) throw ConfigError("coefficient z needs one entry per basis function");
    std::memcpy(zz.data() + c * n_phi, z[c].data(), sizeof(double) * n_phi);
  }
  return run_bilinear(setup, geoms, zz.data(), n_phi, flags);
}

Mat action_kernel(const KernelSetup& setup, const std::vector<GeometryData>& geoms,
                  const std::vector<Coefficients>& w, const Coefficients& z, FpFlags& flags) {
  if (setup.config.mode != ModeKind::action)
    throw ConfigError("configuration is not an action-mode config");
  if (geoms.size() != w.size()) throw ConfigError("action batch needs one coefficient vector per cell");
  const int n_phi = setup.basis.n_phi;
  if (!z.empty() && int(z.size()) != n_phi)
    throw ConfigError("coefficient z needs one entry per basis function");
  const int batch = int(geoms.size());
  Mat v(n_phi, batch);
  if (batch == 0) return v;
  std::vector<double> ww(size_t(batch) * n_phi);
  for (int j = 0; j < batch; ++j) {
    if (int(w[j].size()) != n_phi) throw ConfigError("coefficient w needs one entry per basis function");
    std::memcpy(ww.data() + size_t(j) * n_phi, w[j].data(), sizeof(double) * n_phi);
  }
  mpfem_b200_setup_t s = device_setup(setup);
  int n_pts = 1;
  const std::vector<double> G = pack_geometry(setup, geoms, &n_pts);
  const bool f64 = setup.config.u_q == Fmt::fp64;
  std::vector<double> o64(f64 ? size_t(batch) * n_phi : 0);
  std::vector<float> o32(f64 ? 0 : size_t(batch) * n_phi);
  uint32_t fl = 0;
  check(mpfem_b200_action_from_geometry(s, G.data(), n_pts, batch, z.empty() ? nullptr : z.data(),
                                        ww.data(), n_phi,
                                        f64 ? static_cast<void*>(o64.data()) : o32.data(), n_phi,
                                        nullptr, &fl));
  merge_flags(flags, fl);
  for (int j = 0; j < batch; ++j)
    for (int i = 0; i < n_phi; ++i)
      v(i, j) = f64 ? o64[size_t(j) * n_phi + i] : double(o32[size_t(j) * n_phi + i]);
  return v;
}

DofMap build_dofmap(const Mesh& mesh, const LagrangeBasis& basis, Continuity cont) {
  const int nv = geometry_vertex_count(basis.cell);
  std::vector<int32_t> cells(size_t(mesh.n_cells()) * nv);
  for (int c = 0; c < mesh.n_cells(); ++c) {
    if (int(mesh.cells[c].size()) != nv) throw ConfigError("mesh cells do not match the basis cell");
    for (int k = 0; k < nv; ++k) cells[size_t(c) * nv + k] = mesh.cells[c][k];
  }
  DofMap dm;
  dm.n_local = basis.n_phi;
  dm.cell_dofs.resize(size_t(mesh.n_cells()) * basis.n_phi);
  int32_t n_dofs = 0, mult = 0;
  check(mpfem_b200_dofmap_host(basis.cell.kind == CellKind::box ? 1 : 0, basis.cell.dim, basis.p,
                               cont == Continuity::continuous ? 1 : 0, cells.data(), mesh.n_cells(),
                               int64_t(mesh.vertices.size()), dm.cell_dofs.data(), &n_dofs, &mult));
  dm.n_dofs = n_dofs;
  dm.max_multiplicity = mult;
  return dm;
}

SparseCoo assemble_matrix(const std::vector<Mat>& local, const DofMap& dofmap, Fmt fmt,
                          FpFlags& flags) {
  if (dofmap.n_local <= 0 || dofmap.cell_dofs.size() % dofmap.n_local != 0)
    throw ConfigError("dof map has no complete cells");
  const int n_cells = int(dofmap.cell_dofs.size() / dofmap.n_local);
  if (int(local.size()) != n_cells) throw ConfigError("one local matrix per cell required");
  const int n_loc = dofmap.n_local;
  std::vector<double> loc(size_t(n_cells) * n_loc * n_loc);
  for (int c = 0; c < n_cells; ++c) {
    if (local[c].rows != n_loc || local[c].cols != n_loc)
      throw ConfigError("local matrix does not match the dof map");
    std::memcpy(loc.data() + size_t(c) * n_loc * n_loc, local[c].a.data(), sizeof(double) * n_loc * n_loc);
  }
  mpfem_b200_asm_plan_t plan = nullptr;
  int64_t nnz = 0;
  check(mpfem_b200_asm_plan_create(dofmap.cell_dofs.data(), n_cells, n_loc, dofmap.n_dofs, &plan, &nnz));
  struct Guard {
    mpfem_b200_asm_plan_t p;
    ~Guard() { mpfem_b200_asm_plan_destroy(p); }
  } guard{plan};
  std::vector<int64_t> row_ptr(size_t(dofmap.n_dofs) + 1);
  SparseCoo coo;
  coo.rows = coo.cols = dofmap.n_dofs;
  coo.col.resize(size_t(nnz));
  coo.value.resize(size_t(nnz));
  check(mpfem_b200_asm_plan_pattern(plan, row_ptr.data(), coo.col.data()));
  uint32_t fl = 0;
  check(mpfem_b200_asm_plan_assemble(plan, loc.data(), int(fmt), coo.value.data(), &fl));
  merge_flags(flags, fl);
  coo.row.resize(size_t(nnz));
  for (int r = 0; r < dofmap.n_dofs; ++r)
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) coo.row[size_t(e)] = r;
  return coo;
}

void release_device_setups() {
  Cache& C = cache();
  std::lock_guard<std::mutex> lk(C.mu);
  for (auto& kv : C.setups) mpfem_b200_setup_destroy(kv.second);
  C.setups.clear();
}

}  // namespace mpfem
