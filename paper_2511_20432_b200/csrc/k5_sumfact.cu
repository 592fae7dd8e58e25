// K5 — sum-factorised superposition on tensor-grid point sets.
//
// The reference evaluates the flux integrand and the Dirichlet data pair by
// pair: superpose (proj/src/analytic.cpp:92-109) at every lateral face
// quadrature point (assemble_flux_load, proj/src/assembly.cpp:148-166) and at
// every bottom Greville point (dirichlet_values, proj/src/mesh.cpp:238-264).
// On an axis-aligned patch these point sets are tensor grids, and the point
// source factorises along the axes:
//   c e^{-r.r/s} = c e^{-dn^2/s} e^{-du^2/s} e^{-dv^2/s},
// so the sum over sources at all na x nb points of a face is one dense
// contraction  G = A B  with A[a][j] = c_j e^{-dn_j^2/s_j} (x the normal
// derivative factor -dn_j / (2 alpha dt_j) for the flux) e^{-du_aj^2/s_j} and
// B[j][b] = e^{-dv_bj^2/s_j}: (na + nb) exponentials per source instead of
// na nb, and 2 na nb flops per source on the FP64 tensor cores (DMMA, through
// cuBLAS: a plain library GEMM once A and B are formed).
//
// The pair-wise cull (skip iff r.r / s > cull) does not factorise, so only
// sources that cannot be culled anywhere in the set's bounding box take this
// path (sf_source_eligible; on a long scan that is every source older than a
// few hundredths of a second). The caller runs K1 with the exact cull on the
// remaining sources and adds the two parts, so exact zeros stay exact zeros.
// Accuracy: each factorised term is within a few ulps of the reference's term
// (three exponentials of partial arguments instead of one), plus <= 1e-12
// relative from the grid's coordinate rounding (bounded at eligibility), and
// the sum order differs: far inside the 1e-10 flux / T~ tolerance.
// Sums are deterministic: fixed chunking, fixed-order chunk reduction.
#include <cmath>

#include <algorithm>
#include <string>

#include "context.hpp"
#include "k5_sumfact.cuh"

namespace tgb {

namespace {

void cublas_ok(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS)
    throw cuda_error(std::string("cublas: ") + what + " failed (" + std::to_string(st) + ")");
}

struct Clusters {
  std::vector<double> rep, lo, hi;
  int find(double x) const {
    const long k = std::upper_bound(lo.begin(), lo.end(), x) - lo.begin() - 1;
    return (k >= 0 && x <= hi[k]) ? static_cast<int>(k) : -1;
  }
};

bool cluster_axis(std::vector<double> v, double tol, Clusters& c) {
  std::sort(v.begin(), v.end());
  size_t b = 0;
  for (size_t i = 1; i <= v.size(); ++i) {
    if (i < v.size() && v[i] - v[i - 1] <= tol) continue;
    if (v[i - 1] - v[b] > tol) return false;  // a chained cluster: not a grid line
    c.lo.push_back(v[b]);
    c.hi.push_back(v[i - 1]);
    c.rep.push_back(v[b + (i - 1 - b) / 2]);
    b = i;
  }
  return true;
}

// per source: fac = c e^{-dn^2/s} (x -dn / (2 alpha dt)), 1/s, the in-face
// coordinates; padded and causally inactive sources get fac = 0, 1/s = 0
__global__ void sf_prep_kernel(const double* __restrict__ src6, int J, int Jpad, double t,
                               double alpha, double rcp, SfDev g, bool grad, double* fac,
                               double* inv_s, double* su, double* sv) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Jpad) return;
  double f = 0.0, is = 0.0, u = 0.0, v = 0.0;
  if (j < J) {
    const double* p = src6 + 6 * static_cast<size_t>(j);  // position, energy, t_activate, tau
    const double dt = t - p[5];
    if (dt > 0.0) {
      const double spread = 4.0 * alpha * dt;
      const double c = p[3] / (rcp * pow(M_PI * spread, 1.5));
      const double dn = g.xf - p[g.axn];
      const double e = c * exp(-(dn * dn) / spread);
      f = grad ? dn * (-e / (2.0 * alpha * dt)) : e;
      is = 1.0 / spread;
      u = p[g.axu];
      v = p[g.axv];
    }
  }
  fac[j] = f;
  inv_s[j] = is;
  su[j] = u;
  sv[j] = v;
}

// A (na x Jpad, column-major): fac_j e^{-(U_a - u_j)^2 / s_j}; x: rows a,
// y: groups of kJA sources (2D grid, no 64-bit index division)
constexpr int kJA = 16;
__global__ void sf_build_a_kernel(SfDev g, int Jpad, const double* __restrict__ fac,
                                  const double* __restrict__ inv_s, const double* __restrict__ su,
                                  double* __restrict__ A) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= g.na) return;
  const double ua = g.U[a];
  const int j0 = blockIdx.y * kJA;
#pragma unroll 4
  for (int jj = 0; jj < kJA; ++jj) {
    const int j = j0 + jj;
    if (j >= Jpad) break;
    const double d = ua - su[j];
    A[static_cast<size_t>(j) * g.na + a] = fac[j] * exp(-(d * d) * inv_s[j]);
  }
}

// B, chunk c of Kc sources as a (Kc x nb) column-major block: e^{-(V_b - v_j)^2 / s_j};
// x: sources, y: groups of kBB rows b
constexpr int kBB = 8;
__global__ void sf_build_b_kernel(SfDev g, int Jpad, int Kc, const double* __restrict__ inv_s,
                                  const double* __restrict__ sv, double* __restrict__ B) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Jpad) return;
  const int c = j / Kc, jj = j - c * Kc;
  const double is = inv_s[j], v = sv[j];
  double* out = B + static_cast<size_t>(c) * Kc * g.nb + jj;
  const int b0 = blockIdx.y * kBB;
#pragma unroll 4
  for (int bb = 0; bb < kBB; ++bb) {
    const int b = b0 + bb;
    if (b >= g.nb) break;
    const double d = g.V[b] - v;
    out[static_cast<size_t>(b) * Kc] = exp(-(d * d) * is);
  }
}

__global__ void sf_reduce_kernel(int n, int C, const double* __restrict__ part,
                                 double* __restrict__ G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += part[static_cast<size_t>(c) * n + e];
  G[e] = s;
}

__global__ void sf_add_flux_kernel(int n, const int* __restrict__ pt_index, int n_base,
                                   const int* __restrict__ gcell, const int* __restrict__ gaxn,
                                   const double* __restrict__ G,
                                   const double* __restrict__ normals,
                                   const double* __restrict__ weights, double k,
                                   double* __restrict__ gq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int q = pt_index[i];
  if (q >= n_base) return;
  const int c = gcell[q];
  if (c < 0) return;
  const double dot = __dmul_rn(G[c], normals[3 * static_cast<size_t>(q) + gaxn[q]]);
  gq[i] = __dadd_rn(gq[i], __dmul_rn(__dmul_rn(-k, dot), weights[q]));
}

__global__ void sf_add_dirichlet_kernel(int n, const int* __restrict__ gcell,
                                        const double* __restrict__ G, double* __restrict__ g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  g[i] = __dsub_rn(g[i], G[gcell[i]]);
}

__global__ void sf_add_fine_kernel(int n, const int* __restrict__ pos,
                                   const int* __restrict__ ids, int n_base,
                                   const int* __restrict__ fa, const int* __restrict__ fb,
                                   const int* __restrict__ ff, const int* __restrict__ rect,
                                   const double* __restrict__ G,
                                   const double* __restrict__ normals,
                                   const double* __restrict__ weights, double k,
                                   double* __restrict__ gq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int q = ids[i];
  const int* r = rect + 5 * ff[q];
  const double gv = G[r[3] + (fa[q] - r[0]) + r[2] * (fb[q] - r[1])];
  const size_t qq = static_cast<size_t>(n_base) + q;
  const double dot = __dmul_rn(gv, normals[3 * qq + r[4]]);
  gq[pos[i]] = __dadd_rn(gq[pos[i]], __dmul_rn(__dmul_rn(-k, dot), weights[qq]));
}

__global__ void sf_scatter_add_kernel(int n, const int* __restrict__ pos,
                                      const double* __restrict__ tmp, double* __restrict__ gq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  gq[pos[i]] = __dadd_rn(gq[pos[i]], tmp[i]);
}

}  // namespace

bool sf_make_grid(const double* pts, long n, double tol, SfGrid& g) {
  if (n <= 0) return false;
  Clusters cl[3];
  for (int ax = 0; ax < 3; ++ax) {
    std::vector<double> v(n);
    for (long i = 0; i < n; ++i) v[i] = pts[3 * i + ax];
    if (!cluster_axis(std::move(v), tol, cl[ax])) return false;
    g.lo[ax] = cl[ax].lo.front();
    g.hi[ax] = cl[ax].hi.back();
  }
  int axn = -1;
  for (int ax = 0; ax < 3; ++ax)
    if (cl[ax].rep.size() == 1) {
      if (axn >= 0) return false;  // degenerate (a line of points)
      axn = ax;
    }
  if (axn < 0) return false;
  g.axn = axn;
  g.axu = axn == 0 ? 1 : 0;
  g.axv = axn == 2 ? 1 : 2;
  g.xf = cl[axn].rep[0];
  g.U = cl[g.axu].rep;
  g.V = cl[g.axv].rep;
  const long na = static_cast<long>(g.U.size()), nb = static_cast<long>(g.V.size());
  if (na * nb != n) return false;
  std::vector<char> seen(n, 0);
  g.cell.assign(n, -1);
  g.delta = 0.0;
  for (long i = 0; i < n; ++i) {
    const double* p = pts + 3 * i;
    const int a = cl[g.axu].find(p[g.axu]), b = cl[g.axv].find(p[g.axv]);
    if (a < 0 || b < 0) return false;
    const long c = a + na * b;
    if (seen[c]) return false;
    seen[c] = 1;
    g.cell[i] = static_cast<int>(c);
    g.delta = std::max({g.delta, std::fabs(p[axn] - g.xf), std::fabs(p[g.axu] - g.U[a]),
                        std::fabs(p[g.axv] - g.V[b])});
  }
  return true;
}

bool sf_source_eligible(const double* p, double t, double alpha, double cull, const double lo[3],
                        const double hi[3], double delta) {
  const double dt = t - p[5];
  if (!(dt > 0.0)) return true;  // skipped by the reference, zero column here
  const double spread = 4.0 * alpha * dt;
  double r2 = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    const double a = lo[ax] - p[ax], b = hi[ax] - p[ax];
    r2 += std::max(a * a, b * b);
  }
  if (!(r2 * (1.0 + 1e-9) <= cull * spread)) return false;
  // grid rounding: |d(arg)| <= sum over axes 2 |d| delta / s with |d| <= sqrt(cull s)
  return 36.0 * cull * delta * delta <= 1e-24 * spread;
}

bool sf_source_culled(const double* p, double t, double alpha, double cull, const double lo[3],
                      const double hi[3]) {
  const double dt = t - p[5];
  if (!(dt > 0.0)) return true;
  const double spread = 4.0 * alpha * dt;
  double r2 = 0.0;  // squared distance from the source to the box
  for (int ax = 0; ax < 3; ++ax) {
    const double d = std::max({lo[ax] - p[ax], p[ax] - hi[ax], 0.0});
    r2 += d * d;
  }
  return r2 * (1.0 - 1e-9) > cull * spread;
}

double sf_contract(cublasHandle_t h, const SfDev& g, bool grad, const double* d_src6, int J,
                   int Kc, double t, double alpha, double rcp, const SfScratch& w, double* d_G,
                   cudaStream_t s) {
  if (J <= 0) {  // nothing eligible: the callers add G
    TG_CUDA(cudaMemsetAsync(d_G, 0, sizeof(double) * g.na * g.nb, s));
    return 0.0;
  }
  const int C = (J + Kc - 1) / Kc;
  const int Jpad = C * Kc;
  constexpr int T = 256;
  sf_prep_kernel<<<(Jpad + T - 1) / T, T, 0, s>>>(d_src6, J, Jpad, t, alpha, rcp, g, grad, w.fac,
                                                   w.inv_s, w.su, w.sv);
  // (grid.y <= 65535: up to ~1e6 sources per contraction)
  const int TA = g.na >= 256 ? 256 : 128;
  sf_build_a_kernel<<<dim3((g.na + TA - 1) / TA, (Jpad + kJA - 1) / kJA), TA, 0, s>>>(
      g, Jpad, w.fac, w.inv_s, w.su, w.A);
  sf_build_b_kernel<<<dim3((Jpad + T - 1) / T, (g.nb + kBB - 1) / kBB), T, 0, s>>>(
      g, Jpad, Kc, w.inv_s, w.sv, w.B);
  const double one = 1.0, zero = 0.0;
  cublas_ok(cublasSetStream(h, s), "set stream");
  cublas_ok(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, g.na, g.nb, Kc, &one, w.A,
                                      g.na, static_cast<long long>(g.na) * Kc, w.B, Kc,
                                      static_cast<long long>(Kc) * g.nb, &zero, w.Cpart, g.na,
                                      static_cast<long long>(g.na) * g.nb, C),
            "dgemm strided batched");
  const int n = g.na * g.nb;
  sf_reduce_kernel<<<(n + T - 1) / T, T, 0, s>>>(n, C, w.Cpart, d_G);
  TG_CUDA(cudaGetLastError());
  return 2.0 * g.na * g.nb * static_cast<double>(Jpad);
}

void sf_add_flux(int n, const int* d_pt_index, int n_base, const int* d_gcell, const int* d_gaxn,
                 const double* d_G, const double* d_normals, const double* d_weights, double k,
                 double* d_gq, cudaStream_t s) {
  if (n <= 0) return;
  sf_add_flux_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, d_pt_index, n_base, d_gcell, d_gaxn, d_G,
                                                      d_normals, d_weights, k, d_gq);
}

void sf_add_dirichlet(int n, const int* d_gcell, const double* d_G, double* d_g, cudaStream_t s) {
  if (n <= 0) return;
  sf_add_dirichlet_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, d_gcell, d_G, d_g);
}

void sf_add_fine(int n, const int* d_pos, const int* d_ids, int n_base, const int* d_fa,
                 const int* d_fb, const int* d_ff, const int* d_rect, const double* d_G,
                 const double* d_normals, const double* d_weights, double k, double* d_gq,
                 cudaStream_t s) {
  if (n <= 0) return;
  sf_add_fine_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, d_pos, d_ids, n_base, d_fa, d_fb, d_ff,
                                                      d_rect, d_G, d_normals, d_weights, k, d_gq);
}

void sf_scatter_add(int n, const int* d_pos, const double* d_tmp, double* d_gq, cudaStream_t s) {
  if (n <= 0) return;
  sf_scatter_add_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, d_pos, d_tmp, d_gq);
}

}  // namespace tgb
