// K4 — NURBS geometry and field evaluation on the device, for the observers
// (SURVEY.md §8f "next": total_temperature, boundary_flux_profile,
// export_field and the driver's probes, proj/src/postproc.cpp:9-147,
// proj/src/driver.cpp:226-236).
//
// One thread per parametric point: find_span and the first-derivative
// Cox-de Boor table per direction ("The NURBS Book" A2.1/A2.3, as
// KnotVector::find_span / basis_ders, proj/src/splines.cpp:27-109), the
// rational tensor basis (basis_at, :212-255), then map_point (:257-278) and
// field_at (:280-303). Compiled with -fmad=false: every product and sum is
// rounded separately in the reference's order, so x is bit-identical to the
// host (and reference) map_point and feeds K1 unchanged.
#include "common.cuh"
#include "context.hpp"
#include "k4_eval.cuh"
#include "nurbs_dev.cuh"

namespace tgb {

namespace {

__global__ void k4_eval_kernel(NurbsDev V, const double* __restrict__ xi, long n,
                               const double* __restrict__ coeffs, double* __restrict__ out_x,
                               double* __restrict__ out_f, int* __restrict__ flags,
                               bool strict01) {
  const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (t >= n) return;
  if (strict01)
    for (int d = 0; d < 3; ++d)
      if (xi[3 * t + d] < 0.0 || xi[3 * t + d] > 1.0) {
        atomicOr(flags, kEvalOutside);
        return;
      }
  double tab[3][2 * (kNurbsMaxP + 1)];
  int sp[3];
  for (int d = 0; d < 3; ++d) {
    if (!find_span(V.U[d], V.p[d], V.n[d], xi[3 * t + d], sp[d])) {
      atomicOr(flags, kEvalDomain);
      return;
    }
    basis_ders1(V.U[d], V.p[d], xi[3 * t + d], sp[d], tab[d]);
  }
  const int p0 = V.p[0], p1 = V.p[1], p2 = V.p[2];
  auto grid_index = [&](int i, int j, int k) {
    return static_cast<long>(sp[0] - p0 + i) +
           static_cast<long>(V.n[0]) *
               (static_cast<long>(sp[1] - p1 + j) + static_cast<long>(V.n[1]) * (sp[2] - p2 + k));
  };
  // pass 1: weight sums (basis_at)
  double W = 0.0, dW[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k <= p2; ++k) {
    const double n3 = tab[2][k], d3 = tab[2][p2 + 1 + k];
    for (int j = 0; j <= p1; ++j) {
      const double n2 = tab[1][j], d2 = tab[1][p1 + 1 + j];
      for (int i = 0; i <= p0; ++i) {
        const double n1 = tab[0][i], d1 = tab[0][p0 + 1 + i];
        const double w = V.pts[4 * grid_index(i, j, k) + 3];
        W += w * n1 * n2 * n3;
        dW[0] += w * d1 * n2 * n3;
        dW[1] += w * n1 * d2 * n3;
        dW[2] += w * n1 * n2 * d3;
      }
    }
  }
  // pass 2: rational basis (recomputed bit-identically), map and field sums
  double x[3] = {0.0, 0.0, 0.0}, jac[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double value = 0.0, gp[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k <= p2; ++k) {
    const double n3 = tab[2][k], d3 = tab[2][p2 + 1 + k];
    for (int j = 0; j <= p1; ++j) {
      const double n2 = tab[1][j], d2 = tab[1][p1 + 1 + j];
      for (int i = 0; i <= p0; ++i) {
        const double n1 = tab[0][i], d1 = tab[0][p0 + 1 + i];
        const long g = grid_index(i, j, k);
        const double* c = V.pts + 4 * g;
        const double w = c[3];
        const double val = (w * n1 * n2 * n3) / W;
        const double dv[3] = {(w * d1 * n2 * n3 - dW[0] * val) / W,
                              (w * n1 * d2 * n3 - dW[1] * val) / W,
                              (w * n1 * n2 * d3 - dW[2] * val) / W};
        for (int r = 0; r < 3; ++r) {
          x[r] += c[r] * val;
          for (int q = 0; q < 3; ++q) jac[3 * r + q] += c[r] * dv[q];
        }
        if (coeffs) {
          const double cf = coeffs[g];
          value += cf * val;
          for (int q = 0; q < 3; ++q) gp[q] += dv[q] * cf;
        }
      }
    }
  }
  const double det = det3(jac);
  if (!(det > 0.0)) atomicOr(flags, kEvalJacobian);
  for (int r = 0; r < 3; ++r) out_x[3 * t + r] = x[r];
  if (coeffs) {
    const double* a = jac;
    const double d = det;
    const double inv[9] = {(a[4] * a[8] - a[5] * a[7]) / d, (a[2] * a[7] - a[1] * a[8]) / d,
                           (a[1] * a[5] - a[2] * a[4]) / d, (a[5] * a[6] - a[3] * a[8]) / d,
                           (a[0] * a[8] - a[2] * a[6]) / d, (a[2] * a[3] - a[0] * a[5]) / d,
                           (a[3] * a[7] - a[4] * a[6]) / d, (a[1] * a[6] - a[0] * a[7]) / d,
                           (a[0] * a[4] - a[1] * a[3]) / d};
    out_f[4 * t] = value;
    out_f[4 * t + 1] = inv[0] * gp[0] + inv[3] * gp[1] + inv[6] * gp[2];
    out_f[4 * t + 2] = inv[1] * gp[0] + inv[4] * gp[1] + inv[7] * gp[2];
    out_f[4 * t + 3] = inv[2] * gp[0] + inv[5] * gp[1] + inv[8] * gp[2];
  }
}

__global__ void k4_probe_kernel(long n, double t_c, const double* __restrict__ x,
                                const double* __restrict__ f, const double* __restrict__ val,
                                const double* __restrict__ grad, double* __restrict__ out) {
  const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (t >= n) return;
  double* o = out + 12 * t;
  o[0] = x[3 * t];
  o[1] = x[3 * t + 1];
  o[2] = x[3 * t + 2];
  o[3] = t_c + val[t] + f[4 * t];  // total_temperature (postproc.cpp:18)
  o[4] = val[t];
  o[5] = f[4 * t];
  o[6] = grad[3 * t];
  o[7] = grad[3 * t + 1];
  o[8] = grad[3 * t + 2];
  o[9] = f[4 * t + 1];
  o[10] = f[4 * t + 2];
  o[11] = f[4 * t + 3];
}

}  // namespace

void k4_eval(const NurbsDev& V, const double* d_xi, long n, const double* d_coeffs, double* d_x,
             double* d_f, int* d_flags, cudaStream_t s, bool strict01) {
  if (n <= 0) return;
  for (int d = 0; d < 3; ++d)
    if (V.p[d] > kNurbsMaxP) throw std::invalid_argument("degree > 7 not supported");
  const int threads = 128;
  k4_eval_kernel<<<static_cast<int>((n + threads - 1) / threads), threads, 0, s>>>(
      V, d_xi, n, d_coeffs, d_x, d_f, d_flags, strict01);
  TG_CUDA(cudaGetLastError());
}

void k4_assemble_probe(long n, double t_c, const double* d_x, const double* d_f,
                       const double* d_val, const double* d_grad, double* d_out, cudaStream_t s) {
  if (n <= 0) return;
  const int threads = 256;
  k4_probe_kernel<<<static_cast<int>((n + threads - 1) / threads), threads, 0, s>>>(
      n, t_c, d_x, d_f, d_val, d_grad, d_out);
  TG_CUDA(cudaGetLastError());
}

}  // namespace tgb
