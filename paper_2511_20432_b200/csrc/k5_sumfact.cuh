// K5 — sum-factorised superposition on tensor-grid point sets (see k5_sumfact.cu).
#pragma once

#include <cublas_v2.h>
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

struct SfDev {
  int axn, axu, axv, na, nb;
  double xf;
  const double* U;
  const double* V;
};

struct SfScratch {  // caller-owned device scratch, sized by sf_scratch_doubles
  double* fac;      // Jpad
  double* inv_s;    // Jpad
  double* su;       // Jpad
  double* sv;       // Jpad
  double* A;        // na * Jpad
  double* B;        // Jpad * nb
  double* Cpart;    // C * na * nb
};

// G[e] (na x nb, column-major) = sum over sources j < J of
//   value: c_j e^{-dn^2/s} e^{-du_a^2/s} e^{-dv_b^2/s}
//   grad:  c_j e^{-dn^2/s} (-dn / (2 alpha dt)) e^{-du_a^2/s} e^{-dv_b^2/s}
// (dn, du, dv: grid point minus source along axn, axu, axv; s = 4 alpha dt;
// c_j = E / (rho c (pi s)^1.5)) as one strided-batched DGEMM over Kc-source
// chunks and a fixed-order chunk reduction. Returns the GEMM flops.
double sf_contract(cublasHandle_t h, const SfDev& g, bool grad, const double* d_src6, int J,
                   int Kc, double t, double alpha, double rcp, const SfScratch& w, double* d_G,
                   cudaStream_t s);

// gq[i] += (-k (G[gcell[q]] n_q[axn_q])) w_q for the compact points i whose
// quadrature point q = pt_index[i] is a gridded base point (gcell[q] >= 0)
void sf_add_flux(int n, const int* d_pt_index, int n_base, const int* d_gcell, const int* d_gaxn,
                 const double* d_G, const double* d_normals, const double* d_weights, double k,
                 double* d_gq, cudaStream_t s);
// g[c] -= G[gcell[c]] (g = -T~ at the Greville points)
void sf_add_dirichlet(int n, const int* d_gcell, const double* d_G, double* d_g, cudaStream_t s);
// fine-rule points: i < n, q = ids[i] (fine point index), face f = ff[q] with
// rect[5 f..] = a0, b0, na, G offset, normal axis of the step's rectangle:
//   gq[pos[i]] += (-k (G[off + (fa[q] - a0) + na (fb[q] - b0)] n[axn])) w
// (normals / weights indexed by n_base + q)
void sf_add_fine(int n, const int* d_pos, const int* d_ids, int n_base, const int* d_fa,
                 const int* d_fb, const int* d_ff, const int* d_rect, const double* d_G,
                 const double* d_normals, const double* d_weights, double k, double* d_gq,
                 cudaStream_t s);
// gq[pos[i]] += tmp[i]
void sf_scatter_add(int n, const int* d_pos, const double* d_tmp, double* d_gq, cudaStream_t s);

}  // namespace tgb
