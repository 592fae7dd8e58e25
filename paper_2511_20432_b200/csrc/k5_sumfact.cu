// K5 host side: tensor-grid detection of the face / Greville point sets and
// the source tests of the region plan (restated on the device in
// k5_fused.cu, which holds the contraction itself).
//
// The reference evaluates the flux integrand and the Dirichlet data pair by
// pair (superpose, proj/src/analytic.cpp:92-109, from assemble_flux_load,
// proj/src/assembly.cpp:148-166, and dirichlet_values, proj/src/mesh.cpp:
// 238-264). On an axis-aligned patch those point sets are tensor grids up to
// ~1e-18 m of spline rounding; sf_make_grid finds the grid lines.
#include <cmath>

#include <algorithm>
#include <string>

#include "k5_sumfact.cuh"

namespace tgb {

namespace {

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

bool sf_region_ok(const double* p, double t, double alpha, double cull, const SfRegion& r) {
  const double dt = t - p[5];
  if (!(dt > 0.0)) return true;  // skipped by the reference: a zero column
  const double spread = 4.0 * alpha * dt;
  double r2 = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    const double a = r.lo[ax] - r.delta - p[ax], b = r.hi[ax] + r.delta - p[ax];
    r2 += std::max(a * a, b * b);
  }
  if (!(r2 * (1.0 + 1e-9) <= cull * spread)) return false;
  // grid rounding: |d(arg)| <= sum over axes 2 |d| delta / s with |d| <= sqrt(cull s)
  return 36.0 * cull * r.delta * r.delta <= 1e-24 * spread;
}

bool sf_region_culled(const double* p, double t, double alpha, double cull, const SfRegion& r) {
  const double dt = t - p[5];
  if (!(dt > 0.0)) return true;
  const double spread = 4.0 * alpha * dt;
  double r2 = 0.0;  // squared distance from the source to the box
  for (int ax = 0; ax < 3; ++ax) {
    const double d = std::max({r.lo[ax] - r.delta - p[ax], p[ax] - r.hi[ax] - r.delta, 0.0});
    r2 += d * d;
  }
  return r2 * (1.0 - 1e-9) > cull * spread;
}

}  // namespace tgb
