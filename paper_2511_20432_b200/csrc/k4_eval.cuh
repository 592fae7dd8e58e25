// K4 — NURBS evaluation on the device for the observers (see k4_eval.cu).
#pragma once

#include <cuda_runtime.h>

namespace tgb {

constexpr int kNurbsMaxP = 7;

// The patch on the device: per-direction knot vectors and the control grid
// (x, y, z, w per point, first index fastest).
struct NurbsDev {
  int p[3];
  int n[3];          // basis counts
  const double* U[3];
  const double* pts;  // n[0] n[1] n[2] x 4
};

// Evaluation flags (OR-ed into *flags): parameter outside the knot range
// (find_span's domain_error), non-positive Jacobian determinant.
enum : int { kEvalDomain = 1, kEvalJacobian = 2, kEvalOutside = 4 };

// For each parametric point xi[3 i..]: x = map_point(xi).x (out_x, 3 per
// point) and, when coeffs is not null, the field value and its physical
// gradient (out_f, 4 per point: value, grad) — NurbsVolume::map_point /
// field_at (proj/src/splines.cpp:257-303) with the reference's association.
// strict01: flag kEvalOutside for xi outside [0, 1]^3 (the probe check of
// total_temperature, postproc.cpp:12-14).
void k4_eval(const NurbsDev& V, const double* d_xi, long n, const double* d_coeffs,
             double* d_x, double* d_f, int* d_flags, cudaStream_t s, bool strict01 = false);

// out (n x 12): x, y, z, T_total, T_tilde, T_hat, grad T_tilde, grad T_hat.
void k4_assemble_probe(long n, double t_c, const double* d_x, const double* d_f,
                       const double* d_val, const double* d_grad, double* d_out, cudaStream_t s);

}  // namespace tgb
