// host_mesh.cpp -- seeded synthetic inputs on the host (C++ std::mt19937_64, the
// reference Rng of common.hpp:21-35):
//   * BASELINE configs 0-2: reference tet + U(-0.15, 0.15) per coordinate, vertex-major,
//     |det J| < 1e-3 rejected, odd orientation repaired by swapping vertices 2 and 3
//     (the repair of mesh.cpp:157);
//   * BASELINE config 3: diag(1, 10^-a, 10^-b) scaled reference tet, a, b ~ U[0, 4], then
//     a random rotation (axis U(-1,1)^3 normalised, angle U(0, 2 pi)), plus 4 affine-field
//     vertex values U[0, 1];
//   * BASELINE config 4: structured_tet_mesh (mesh.cpp:78-163): jittered (nx+1)(ny+1)(nz+1)
//     lattice, draws in k, j, i, axis order, Kuhn split into 6 tets with orientation repair.
#include <cmath>
#include <cstdint>
#include <random>

#include "../../include/mpfem_b200.h"

namespace {

struct Draw {
  std::mt19937_64 eng;
  explicit Draw(uint64_t seed) : eng(seed) {}
  double uniform(double a, double b) { return a + (b - a) * (double(eng() >> 11) * 0x1.0p-53); }
};

double det3(const double e[3][3]) {
  return e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
         e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
         e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
}

const double kRefTet[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};

}  // namespace

extern "C" int mpfem_b200_gen_tets(int kind, uint64_t seed, int64_t n, double* verts,
                                   double* coef) {
  if (n < 0 || !verts || (kind == 1 && !coef) || kind < 0 || kind > 1) return MPFEM_B200_CONFIG_ERROR;
  Draw rng(seed);
  for (int64_t c = 0; c < n; ++c) {
    double* X = verts + 12 * c;
    if (kind == 0) {
      for (;;) {
        for (int v = 0; v < 4; ++v)
          for (int a = 0; a < 3; ++a) X[3 * v + a] = kRefTet[v][a] + rng.uniform(-0.15, 0.15);
        double e[3][3];
        for (int i = 0; i < 3; ++i)
          for (int s = 0; s < 3; ++s) e[i][s] = X[3 * (s + 1) + i] - X[i];
        double d = det3(e);
        if (std::fabs(d) < 1e-3) continue;
        if (d < 0.0)
          for (int a = 0; a < 3; ++a) std::swap(X[6 + a], X[9 + a]);
        break;
      }
      continue;
    }
    double sa = rng.uniform(0.0, 4.0), sb = rng.uniform(0.0, 4.0);
    double ax[3];
    for (double& a : ax) a = rng.uniform(-1.0, 1.0);
    double nrm = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    for (double& a : ax) a /= nrm;
    double ang = rng.uniform(0.0, 6.283185307179586);
    double co = std::cos(ang), si = std::sin(ang);
    double R[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double cross = 0.0;  // Rodrigues: (K)_ij of the cross-product matrix of the axis
        if (i != j) {
          int k = 3 - i - j;
          double sign = ((j + 1) % 3 == i) ? 1.0 : -1.0;
          cross = sign * ax[k];
          if ((i + 1) % 3 == j) cross = -cross;
        }
        R[i][j] = co * (i == j ? 1.0 : 0.0) + si * cross + (1.0 - co) * ax[i] * ax[j];
      }
    double sc[3] = {1.0, std::pow(10.0, -sa), std::pow(10.0, -sb)};
    for (int v = 0; v < 4; ++v)
      for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j) acc += R[i][j] * (sc[j] * kRefTet[v][j]);
        X[3 * v + i] = acc;
      }
    for (int v = 0; v < 4; ++v) coef[4 * c + v] = rng.uniform(0.0, 1.0);
  }
  return MPFEM_B200_OK;
}

extern "C" int mpfem_b200_structured_tet_mesh(int nx, int ny, int nz, double extent,
                                              double jitter, uint64_t seed, double* verts,
                                              int32_t* cells) {
  if (nx < 1 || ny < 1 || nz < 1 || extent <= 0.0 || jitter < 0.0 || jitter > 0.45)
    return MPFEM_B200_CONFIG_ERROR;
  const double h[3] = {extent / nx, extent / ny, extent / nz};
  Draw rng(seed);
  int64_t iv = 0;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i, ++iv) {
        double v[3] = {i * h[0], j * h[1], k * h[2]};
        for (int a = 0; a < 3; ++a) v[a] += rng.uniform(-jitter * h[a], jitter * h[a]);
        for (int a = 0; a < 3; ++a) verts[3 * iv + a] = v[a];
      }
  // Kuhn split: one tet per axis permutation along the main diagonal.
  static const int order[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  auto vid = [&](int i, int j, int k) -> int32_t {
    return int32_t(i + (nx + 1) * (j + (ny + 1) * int64_t(k)));
  };
  int64_t ic = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int32_t corner[8];
        for (int b = 0; b < 8; ++b) corner[b] = vid(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1));
        for (const auto& o : order) {
          int32_t t[4] = {corner[0], 0, 0, 0};
          int bits = 0;
          for (int s = 0; s < 3; ++s) {
            bits |= 1 << o[s];
            t[s + 1] = corner[bits];
          }
          double e[3][3];
          for (int x = 0; x < 3; ++x)
            for (int s = 0; s < 3; ++s) e[x][s] = verts[3 * int64_t(t[s + 1]) + x] - verts[3 * int64_t(t[0]) + x];
          if (det3(e) < 0.0) std::swap(t[2], t[3]);
          for (int v = 0; v < 4; ++v) cells[4 * ic + v] = t[v];
          ++ic;
        }
      }
  return MPFEM_B200_OK;
}
