// launch_bounds.cu -- KB kernel (bounds.cuh). Compiled with --fmad=false: every binary64
// product and sum is rounded separately, as in the reference's bounds.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "bounds.cuh"

namespace mpfem_b200 {
namespace {

// cyclic Jacobi eigenvalues of a symmetric 3x3 (geometry.cpp:120-154), ascending
__device__ void sym_eigenvalues3(const double* sym, double* eig) {
  double a[9];
  for (int i = 0; i < 9; ++i) a[i] = sym[i];
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) off += a[p * 3 + q] * a[p * 3 + q];
    if (off <= 1e-300) break;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p * 3 + q] == 0.0) continue;
        const double theta = (a[q * 3 + q] - a[p * 3 + p]) / (2.0 * a[p * 3 + q]);
        const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(1.0 + theta * theta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k * 3 + p], akq = a[k * 3 + q];
          a[k * 3 + p] = c * akp - s * akq;
          a[k * 3 + q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p * 3 + k], aqk = a[q * 3 + k];
          a[p * 3 + k] = c * apk - s * aqk;
          a[q * 3 + k] = s * apk + c * aqk;
        }
      }
  }
  for (int i = 0; i < 3; ++i) eig[i] = a[i * 3 + i];
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && eig[j - 1] > eig[j]; --j) {
      const double t = eig[j];
      eig[j] = eig[j - 1];
      eig[j - 1] = t;
    }
}

struct CellDiag {
  double ten[9], tt[9];
  double kk2;  // kappa_cell * kappa_2
  double v[8][3];
};

// Binary64 geometry and diagnostics at one point from its Jacobian (geometry.cpp:29-118,
// 156-221): G, G~, kappa_2(J), kappa_cell = nv ||X||_inf / ||J||_inf. False on a zero pivot.
__device__ bool diag_from_jac(const double jac[3][3], const double (*v)[3], int nv, bool poisson,
                              double* ten, double* tt, double& kk2) {
  double lu[3][3];
  int perm[3] = {0, 1, 2}, sign = 1;
  for (int i = 0; i < 3; ++i)
    for (int s = 0; s < 3; ++s) lu[i][s] = jac[i][s];
  for (int col = 0; col < 3; ++col) {
    int pivot = col;
    double best = fabs(lu[col][col]);
    for (int r = col + 1; r < 3; ++r)
      if (fabs(lu[r][col]) > best) { best = fabs(lu[r][col]); pivot = r; }
    if (lu[pivot][col] == 0.0) return false;
    if (pivot != col) {
      for (int c = 0; c < 3; ++c) { const double t = lu[pivot][c]; lu[pivot][c] = lu[col][c]; lu[col][c] = t; }
      const int t = perm[pivot]; perm[pivot] = perm[col]; perm[col] = t;
      sign = -sign;
    }
    for (int r = col + 1; r < 3; ++r) {
      const double m = lu[r][col] / lu[col][col];
      lu[r][col] = m;
      for (int c = col + 1; c < 3; ++c) lu[r][c] = lu[r][c] - m * lu[col][c];
    }
  }
  double det = double(sign);
  for (int i = 0; i < 3; ++i) det = det * lu[i][i];
  const double adet = fabs(det);
  double inv[3][3];
  for (int k = 0; k < 3; ++k) {
    double y[3];
    for (int r = 0; r < 3; ++r) {
      double s = perm[r] == k ? 1.0 : 0.0;
      for (int c = 0; c < r; ++c) s = s - lu[r][c] * y[c];
      y[r] = s;
    }
    for (int r = 2; r >= 0; --r) {
      double s = y[r];
      for (int c = r + 1; c < 3; ++c) s = s - lu[r][c] * inv[c][k];
      inv[r][k] = s / lu[r][r];
    }
  }
  for (int i = 0; i < 9; ++i) ten[i] = tt[i] = 0.0;
  if (!poisson) {
    ten[0] = adet;
    tt[0] = adet;
  } else {
    for (int s = 0; s < 3; ++s)
      for (int t = s; t < 3; ++t) {
        double dot = 0.0;
        for (int k = 0; k < 3; ++k) dot = dot + inv[s][k] * inv[t][k];
        ten[s * 3 + t] = ten[t * 3 + s] = adet * dot;
      }
    for (int s = 0; s < 3; ++s)
      for (int t = 0; t < 3; ++t) {
        double dot = 0.0;
        for (int k = 0; k < 3; ++k) dot += fabs(inv[s][k]) * fabs(inv[t][k]);
        tt[s * 3 + t] = adet * dot;
      }
  }
  double jtj[9], eig[3];
  for (int s = 0; s < 3; ++s)
    for (int t = 0; t < 3; ++t) {
      double dot = 0.0;
      for (int k = 0; k < 3; ++k) dot += jac[k][s] * jac[k][t];
      jtj[s * 3 + t] = dot;
    }
  sym_eigenvalues3(jtj, eig);
  const double kappa2 = eig[0] <= 0.0 ? INFINITY : sqrt(eig[2] / eig[0]);
  double xnorm = 0.0, jnorm = 0.0;
  for (int i = 0; i < 3; ++i) {
    double row = 0.0;
    for (int w = 0; w < nv; ++w) row += fabs(v[w][i]);
    xnorm = fmax(xnorm, row);
    double jr = 0.0;
    for (int s = 0; s < 3; ++s) jr += fabs(jac[i][s]);
    jnorm = fmax(jnorm, jr);
  }
  kk2 = double(nv) * xnorm / jnorm * kappa2;
  return true;
}

// Affine tets: one point (J through the P1 gradients at the centroid, exact +-1 / 0).
__device__ bool cell_diag(const BoundParams& P, int64_t cell, bool poisson, CellDiag& d) {
  const int nv = P.box ? 8 : 4;
  for (int k = 0; k < nv; ++k) {
    const int64_t base = P.cells ? int64_t(P.cells[cell * nv + k]) * 3 : cell * 3 * nv + k * 3;
    for (int a = 0; a < 3; ++a) d.v[k][a] = P.verts[base + a];
  }
  if (P.box) return true;  // boxes: per-point diagnostics in box_point_diag
  double jac[3][3];
  for (int i = 0; i < 3; ++i)
    for (int s = 0; s < 3; ++s) jac[i][s] = 0.0;
  for (int k = 0; k < 4; ++k)
    for (int i = 0; i < 3; ++i)
      for (int s = 0; s < 3; ++s) {
        const double g = (k == 0) ? -1.0 : ((k - 1 == s) ? 1.0 : 0.0);
        jac[i][s] = jac[i][s] + d.v[k][i] * g;
      }
  return diag_from_jac(jac, d.v, 4, poisson, d.ten, d.tt, d.kk2);
}

// Boxes: J(xi_q) = sum_k x_k (x) grad phi_k(xi_q) at binary64 (geometry.cpp:12-27).
__device__ bool box_point_diag(const BoundParams& P, const CellDiag& d, int q, bool poisson,
                               double* ten, double* tt, double& kk2) {
  double jac[3][3];
  for (int i = 0; i < 3; ++i)
    for (int s = 0; s < 3; ++s) jac[i][s] = 0.0;
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 3; ++i)
      for (int s = 0; s < 3; ++s)
        jac[i][s] = jac[i][s] + d.v[k][i] * P.ggrad64[(size_t(s) * 8 + k) * P.n_q + q];
  return diag_from_jac(jac, d.v, 8, poisson, ten, tt, kk2);
}

__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  v = l < int(blockDim.x >> 5) ? red[l] : 0.0;
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(kBoundThreads) cell_bounds_kernel(const BoundParams P) {
  extern __shared__ __align__(16) double sb[];
  const int nq = P.n_q, nd = P.n_d, nphi = P.n_phi;
  const int nc = nd * nd * nq;
  double* cc = sb;             // c_stq = omega G_st z_q          (bounds.cpp:118)
  double* thc = cc + nc;       // theta_c                         (bounds.cpp:119-122)
  double* gc = thc + nc;       // gamma_c                         (bounds.cpp:123-124)
  double* zat = gc + nc;       // z(x_q) in binary64
  double* red = zat + nq;      // 4 x 32 reduction scratch
  double* pten = red + 128;    // boxes: G, G~ and kappa_cell kappa_2 at every rule point
  double* ptt = pten + (P.box ? 9 * nq : 0);
  double* pkk = ptt + (P.box ? 9 * nq : 0);
  __shared__ CellDiag sd;
  __shared__ int s_ok;
  const bool poisson = nd == 3;
  const double pd = double(P.p) * double(P.p) * double(P.p);  // pow(p, d) for d = 3
  for (int64_t cell = blockIdx.x; cell < P.n_cells; cell += gridDim.x) {
    if (threadIdx.x == 0) {
      s_ok = cell_diag(P, cell, poisson, sd);
      if (!s_ok) report_error(P.error, 3);
    }
    __syncthreads();
    if (P.box) {
      for (int q = threadIdx.x; q < nq; q += blockDim.x)
        if (!box_point_diag(P, sd, q, poisson, pten + 9 * q, ptt + 9 * q, pkk[q])) {
          s_ok = 0;
          report_error(P.error, 3);
        }
      __syncthreads();
    }
    const double* coef = P.coef ? P.coef + cell * P.coef_stride : nullptr;
    double z_norm = 0.0;
    if (P.coef_kind == 3)
      for (int i = 0; i < nphi; ++i) z_norm = fmax(z_norm, fabs(coef[i]));
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      double z = 1.0;
      const double* xi = P.rule_x + 3 * q;
      if (P.coef_kind == 3) {  // eval_fe_function at binary64 (elements.cpp:213-222)
        z = 0.0;
        for (int i = 0; i < nphi; ++i) z += coef[i] * P.vals[size_t(i) * nq + q];
      } else if (P.coef_kind == 1) {
        double x[3];
        for (int i = 0; i < 3; ++i) {
          double acc = sd.v[0][i];
          for (int s = 0; s < 3; ++s) acc = acc + (sd.v[s + 1][i] - sd.v[0][i]) * xi[s];
          x[i] = acc;
        }
        const double two_pi = 6.283185307179586476925286766559;
        z = 1.0 + 0.5 * sin(two_pi * x[0]) * cos(two_pi * x[1]) * exp(x[2]);
      } else if (P.coef_kind == 2) {
        const double l0 = ((1.0 - xi[0]) - xi[1]) - xi[2];
        const double u = coef[0] * l0 + coef[1] * xi[0] + coef[2] * xi[1] + coef[3] * xi[2];
        z = pow(10.0, 6.0 * u);
      }
      zat[q] = z;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nc; e += blockDim.x) {
      const int st = e / nq, q = e - st * nq;
      const int s = st / nd, t = st - s * nd;
      const double omega = P.rule_w[q];
      const double ten = P.box ? pten[9 * q + s * 3 + t] : sd.ten[s * 3 + t];
      const double tt = P.box ? ptt[9 * q + s * 3 + t] : sd.tt[s * 3 + t];
      const double kk2 = P.box ? pkk[q] : sd.kk2;
      cc[e] = omega * ten * zat[q];
      thc[e] = P.coef_kind == 3 ? pd * P.lebesgue * z_norm * fabs(omega * ten) : 0.0;
      gc[e] = kk2 * fabs(omega * tt * zat[q]);
    }
    __syncthreads();
    double amax = 0.0, samax = 0.0, tamax = 0.0, gamax = 0.0;
    for (int e = threadIdx.x; e < nphi * nphi; e += blockDim.x) {
      const int i = e / nphi, k = e - i * nphi;
      double acc = 0.0, sa = 0.0, ta = 0.0, ga = 0.0;
      for (int s = 0; s < nd; ++s)
        for (int t = 0; t < nd; ++t) {
          const double* bk = P.tab + (size_t(t) * nphi + k) * nq;
          const double* tbk = P.theta_b + (size_t(t) * nphi + k) * nq;
          const double* bi = P.tab + (size_t(s) * nphi + i) * nq;
          const double* tbi = P.theta_b + (size_t(s) * nphi + i) * nq;
          const int base = (s * nd + t) * nq;
          for (int q = 0; q < nq; ++q) {
            const double bval = __ldg(bk + q);
            const double c = cc[base + q];
            const double h = c * bval;
            const double th = thc[base + q] * fabs(bval) + fabs(c) * __ldg(tbk + q);
            const double gh = gc[base + q] * fabs(bval);
            const double b = __ldg(bi + q);
            const double tb = __ldg(tbi + q);
            acc += b * h;
            sa += fabs(b) * fabs(h);
            ta += fabs(b) * th + tb * fabs(h);
            ga += fabs(b) * gh;
          }
        }
      if (P.a64) P.a64[cell * nphi * nphi + e] = acc;
      amax = fmax(amax, fabs(acc));
      samax = fmax(samax, fabs(sa));
      tamax = fmax(tamax, fabs(ta));
      gamax = fmax(gamax, fabs(ga));
    }
    amax = block_max(amax, red);
    samax = block_max(samax, red + 32);
    tamax = block_max(tamax, red + 64);
    gamax = block_max(gamax, red + 96);
    if (threadIdx.x == 0) {
      double* o = P.out + cell * 4;
      if (s_ok && amax > 0.0) {  // bounds.cpp:255-266
        o[1] = samax / amax;
        o[2] = tamax / amax;
        o[3] = gamax / amax;
        o[0] = (P.u_s + nq * P.u_q) * o[1] + P.u_p * o[2] + P.u_g * o[3];
      } else {
        o[0] = o[1] = o[2] = o[3] = __longlong_as_double(0x7ff8000000000000ll);
      }
    }
    __syncthreads();
  }
}

// Action part of kernel_bounds: one CTA per cell; threads over the rule points build r,
// theta_r, gamma_r (bounds.cpp:128-155) in shared memory, then one thread per output i runs the
// (s, q) accumulation (bounds.cpp:224-240).
__global__ void __launch_bounds__(kBoundThreads) cell_action_bounds_kernel(const BoundParams P) {
  extern __shared__ __align__(16) double sb[];
  const int nq = P.n_q, nd = P.n_d, nphi = P.n_phi;
  const int nr = nd * nq;
  double* rr = sb;        // r_sq
  double* thr = rr + nr;  // theta_r
  double* gr = thr + nr;  // gamma_r
  double* red = gr + nr;  // 4 x 32
  __shared__ CellDiag sd;
  __shared__ int s_ok;
  const bool poisson = nd == 3;
  const double pd = double(P.p) * double(P.p) * double(P.p);
  const double kv = P.lebesgue;
  for (int64_t cell = blockIdx.x; cell < P.n_cells; cell += gridDim.x) {
    if (threadIdx.x == 0) {
      s_ok = cell_diag(P, cell, poisson, sd);
      if (!s_ok) report_error(P.error, 3);
    }
    __syncthreads();
    const double* coef = P.coef ? P.coef + cell * P.coef_stride : nullptr;
    const double* w = P.w + cell * P.w_stride;
    double z_norm = 0.0, w_norm = 0.0;
    if (P.coef_kind == 3)
      for (int i = 0; i < nphi; ++i) z_norm = fmax(z_norm, fabs(coef[i]));
    for (int i = 0; i < nphi; ++i) w_norm = fmax(w_norm, fabs(w[i]));
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      double z = 1.0;
      const double* xi = P.rule_x + 3 * q;
      if (P.coef_kind == 3) {
        z = 0.0;
        for (int i = 0; i < nphi; ++i) z += coef[i] * P.vals[size_t(i) * nq + q];
      } else if (P.coef_kind == 1) {
        double x[3];
        for (int i = 0; i < 3; ++i) {
          double acc = sd.v[0][i];
          for (int s = 0; s < 3; ++s) acc = acc + (sd.v[s + 1][i] - sd.v[0][i]) * xi[s];
          x[i] = acc;
        }
        const double two_pi = 6.283185307179586476925286766559;
        z = 1.0 + 0.5 * sin(two_pi * x[0]) * cos(two_pi * x[1]) * exp(x[2]);
      } else if (P.coef_kind == 2) {
        const double l0 = ((1.0 - xi[0]) - xi[1]) - xi[2];
        const double u = coef[0] * l0 + coef[1] * xi[0] + coef[2] * xi[1] + coef[3] * xi[2];
        z = pow(10.0, 6.0 * u);
      }
      const double omega = P.rule_w[q];
      if (poisson) {
        double gw[3] = {0.0, 0.0, 0.0};  // eval_fe_gradient at binary64 (elements.cpp:224-236)
        for (int i = 0; i < nphi; ++i)
          for (int a = 0; a < 3; ++a) gw[a] += w[i] * P.tab[(size_t(a) * nphi + i) * nq + q];
        for (int s = 0; s < 3; ++s) {
          double gw_s = 0.0, gtw_s = 0.0, kappa_s = 0.0;
          for (int t = 0; t < 3; ++t) {
            gw_s += sd.ten[s * 3 + t] * gw[t];
            gtw_s += fabs(sd.tt[s * 3 + t]) * fabs(gw[t]);
            kappa_s += fabs(sd.ten[s * 3 + t]) * P.grad_kappa_max[t] * P.grad_lebesgue[t];
          }
          const int idx = s * nq + q;
          rr[idx] = omega * z * gw_s;
          thr[idx] = pd * fabs(omega) * (kv * z_norm * fabs(gw_s) + fabs(z) * w_norm * kappa_s);
          gr[idx] = sd.kk2 * fabs(omega * z) * gtw_s;
        }
      } else {
        double w_at = 0.0;
        for (int i = 0; i < nphi; ++i) w_at += w[i] * P.vals[size_t(i) * nq + q];
        const double g = sd.ten[0];
        rr[q] = omega * z * g * w_at;
        thr[q] = pd * kv * (fabs(w_at) * z_norm + fabs(z) * w_norm) * fabs(omega * g);
        gr[q] = sd.kk2 * fabs(rr[q]);
      }
    }
    __syncthreads();
    double vmax = 0.0, svmax = 0.0, tvmax = 0.0, gvmax = 0.0;
    for (int i = threadIdx.x; i < nphi; i += blockDim.x) {
      double acc = 0.0, sv = 0.0, tv = 0.0, gv = 0.0;
      for (int s = 0; s < nd; ++s) {
        const double* bi = P.tab + (size_t(s) * nphi + i) * nq;
        const double* tbi = P.theta_b + (size_t(s) * nphi + i) * nq;
        for (int q = 0; q < nq; ++q) {
          const double b = __ldg(bi + q), tb = __ldg(tbi + q);
          const int idx = s * nq + q;
          acc += b * rr[idx];
          sv += fabs(b) * fabs(rr[idx]);
          tv += fabs(b) * thr[idx] + tb * fabs(rr[idx]);
          gv += fabs(b) * gr[idx];
        }
      }
      if (P.a64) P.a64[cell * nphi + i] = acc;
      vmax = fmax(vmax, fabs(acc));
      svmax = fmax(svmax, sv);
      tvmax = fmax(tvmax, tv);
      gvmax = fmax(gvmax, gv);
    }
    vmax = block_max(vmax, red);
    svmax = block_max(svmax, red + 32);
    tvmax = block_max(tvmax, red + 64);
    gvmax = block_max(gvmax, red + 96);
    if (threadIdx.x == 0) {
      double* o = P.out + cell * 4;
      if (s_ok && vmax > 0.0) {  // bounds.cpp:268-279
        o[1] = svmax / vmax;
        o[2] = tvmax / vmax;
        o[3] = gvmax / vmax;
        o[0] = (P.u_s + nq * P.u_q) * o[1] + P.u_p * o[2] + P.u_g * o[3];
      } else {
        o[0] = o[1] = o[2] = o[3] = __longlong_as_double(0x7ff8000000000000ll);
      }
    }
    __syncthreads();
  }
}

}  // namespace

int launch_bounds_kernel(const BoundParams& P, int sm_count, cudaStream_t st) {
  const size_t nc = size_t(P.n_d) * P.n_d * P.n_q;
  const size_t smem = sizeof(double) * (3 * nc + P.n_q + 128 + (P.box ? 19 * size_t(P.n_q) : 0));
  static size_t smem_set = 0;
  if (smem > smem_set) {
    if (cudaFuncSetAttribute(cell_bounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(std::max<size_t>(smem, 48 * 1024))) != cudaSuccess)
      return 4;
    smem_set = smem;
  }
  const unsigned grid = unsigned(std::min<int64_t>(P.n_cells, int64_t(sm_count) * 4));
  cell_bounds_kernel<<<grid, kBoundThreads, smem, st>>>(P);
  return 0;
}

int launch_action_bounds_kernel(const BoundParams& P, int sm_count, cudaStream_t st) {
  const size_t smem = sizeof(double) * (3 * size_t(P.n_d) * P.n_q + 128);
  static size_t smem_set = 0;
  if (smem > smem_set) {
    if (cudaFuncSetAttribute(cell_action_bounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(std::max<size_t>(smem, 48 * 1024))) != cudaSuccess)
      return 4;
    smem_set = smem;
  }
  const unsigned grid = unsigned(std::min<int64_t>(P.n_cells, int64_t(sm_count) * 8));
  cell_action_bounds_kernel<<<grid, 128, smem, st>>>(P);
  return 0;
}

}  // namespace mpfem_b200
