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
#include <unordered_map>

#include "host/parallel.hpp"
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

// The coordinates of one axis as sorted distinct values with multiplicities
// (a grid's points repeat each line coordinate many times: counting them in a
// hash map and sorting the few distinct values replaces a sort of all n);
// clusters of values within tol are the grid lines, each represented by its
// median element counting multiplicity (what a sort of all n values gives).
bool cluster_axis(const double* pts, long n, int ax, double tol, Clusters& c) {
  std::unordered_map<double, long> count;
  count.reserve(4096);
  for (long i = 0; i < n; ++i) ++count[pts[3 * i + ax]];
  std::vector<std::pair<double, long>> v(count.begin(), count.end());
  std::sort(v.begin(), v.end());
  size_t b = 0;
  long nb = 0;  // elements in the current cluster
  for (size_t i = 1; i <= v.size(); ++i) {
    nb += v[i - 1].second;
    if (i < v.size() && v[i].first - v[i - 1].first <= tol) continue;
    if (v[i - 1].first - v[b].first > tol) return false;  // a chained cluster: not a grid line
    c.lo.push_back(v[b].first);
    c.hi.push_back(v[i - 1].first);
    long k = (nb - 1) / 2;  // the median element's rank in the cluster
    size_t m = b;
    while (k >= v[m].second) k -= v[m++].second;
    c.rep.push_back(v[m].first);
    b = i;
    nb = 0;
  }
  return true;
}

}  // namespace

bool sf_make_grid(const double* pts, long n, double tol, SfGrid& g) {
  if (n <= 0) return false;
  Clusters cl[3];
  char ok[3] = {0, 0, 0};
  parallel_for(3, [&](long ax) {  // the three axes side by side
    ok[ax] = cluster_axis(pts, n, static_cast<int>(ax), tol, cl[ax]);
  }, 1);
  for (int ax = 0; ax < 3; ++ax) {
    if (!ok[ax]) return false;
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
  g.cell.assign(n, -1);
  // cells and the largest offset from the grid lines, in parallel chunks
  constexpr long kChunk = 1 << 16;
  const long nch = (n + kChunk - 1) / kChunk;
  std::vector<double> dmax(nch, 0.0);
  std::vector<char> bad(nch, 0);
  parallel_for(nch, [&](long ch) {
    double dm = 0.0;
    for (long i = ch * kChunk; i < std::min(n, (ch + 1) * kChunk); ++i) {
      const double* p = pts + 3 * i;
      const int a = cl[g.axu].find(p[g.axu]), b = cl[g.axv].find(p[g.axv]);
      if (a < 0 || b < 0) {
        bad[ch] = 1;
        return;
      }
      g.cell[i] = static_cast<int>(a + na * b);
      dm = std::max({dm, std::fabs(p[axn] - g.xf), std::fabs(p[g.axu] - g.U[a]),
                     std::fabs(p[g.axv] - g.V[b])});
    }
    dmax[ch] = dm;
  }, 1);
  g.delta = 0.0;
  for (long ch = 0; ch < nch; ++ch) {
    if (bad[ch]) return false;
    g.delta = std::max(g.delta, dmax[ch]);
  }
  std::vector<char> seen(n, 0);  // every cell exactly once
  for (long i = 0; i < n; ++i) {
    if (seen[g.cell[i]]) return false;
    seen[g.cell[i]] = 1;
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
