// K5 host side: tensor-grid detection and the region source tests (see k5_sumfact.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace tgb {

// A point set that is a tensor grid up to coordinate rounding: point i sits at
// (xf on axis axn, U[a] on axis axu, V[b] on axis axv), cell[i] = a + na * b.
// The spline maps of an axis-aligned cuboid give such sets (the lateral face
// quadrature points, the bottom Greville points), but only up to ~1e-18 m of
// rounding per coordinate; delta is the largest deviation from the grid.
struct SfGrid {
  int axn = 2, axu = 0, axv = 1;
  double xf = 0.0;
  std::vector<double> U, V;
  std::vector<int> cell;
  double delta = 0.0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
};

// Clusters each axis at gaps > tol; succeeds when one axis has a single
// cluster and the other two span exactly one point per (a, b) cell.
bool sf_make_grid(const double* pts, long n, double tol, SfGrid& out);

// Sources [0, J) may take the GEMM path for points in the box [lo, hi] at t
// when none of their pairs can be culled there (the reference skips a pair iff
// r.r / spread > cull) and the grid's coordinate rounding moves no term by
// more than ~1e-12 relative. Causally inactive sources are eligible (their
// terms are exact zeros on both paths).
bool sf_source_eligible(const double* src6, double t, double alpha, double cull,
                        const double lo[3], const double hi[3], double delta);

// Every pair of the source with a point in [lo, hi] is culled by the
// reference (or the source is causally inactive at t): its terms are exact
// zeros there, and K1 may skip it.
bool sf_source_culled(const double* src6, double t, double alpha, double cull,
                      const double lo[3], const double hi[3]);

}  // namespace tgb
