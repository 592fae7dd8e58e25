// K5 host side: tensor-grid detection and the region source tests (see k5_sumfact.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "k5_fused.cuh"

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

// The region tests of the K5 plan (restated on the device in k5_fused.cu's
// sf_source_ok / sf_source_culled): `ok` = no point of the region's box
// (+- delta) is in the source's cull range and the grid rounding moves no term
// by more than ~1e-12 relative (causally inactive sources are ok: zero
// columns); `culled` = every pair of the source with the box is culled.
bool sf_region_ok(const double* src6, double t, double alpha, double cull, const SfRegion& r);
bool sf_region_culled(const double* src6, double t, double alpha, double cull, const SfRegion& r);

}  // namespace tgb
