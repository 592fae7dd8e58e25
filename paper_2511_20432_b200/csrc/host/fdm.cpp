#include "fdm.hpp"

#include <cmath>
#include <stdexcept>

namespace tgb {

void sym_eigen_jacobi(std::vector<double>& C, int n, std::vector<double>& w,
                      std::vector<double>& Q) {
  Q.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) Q[static_cast<size_t>(i) * n + i] = 1.0;
  auto c = [&](int i, int j) -> double& { return C[static_cast<size_t>(i) * n + j]; };
  double total = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) total += c(i, j) * c(i, j);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += c(i, j) * c(i, j);
    if (off <= 1e-34 * total) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = c(p, q);
        if (apq == 0.0) continue;
        const double theta = (c(q, q) - c(p, p)) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        // C <- J^T C J with J the (p, q) rotation
        for (int k = 0; k < n; ++k) {
          const double ckp = c(k, p), ckq = c(k, q);
          c(k, p) = cs * ckp - sn * ckq;
          c(k, q) = sn * ckp + cs * ckq;
        }
        for (int k = 0; k < n; ++k) {
          const double cpk = c(p, k), cqk = c(q, k);
          c(p, k) = cs * cpk - sn * cqk;
          c(q, k) = sn * cpk + cs * cqk;
        }
        c(p, q) = c(q, p) = 0.0;
        double* qp = &Q[static_cast<size_t>(p) * n];
        double* qq = &Q[static_cast<size_t>(q) * n];
        for (int k = 0; k < n; ++k) {
          const double a = qp[k], b = qq[k];
          qp[k] = cs * a - sn * b;
          qq[k] = sn * a + cs * b;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = c(i, i);
}

Fdm1D fdm_factor(const std::vector<double>& Mband, const std::vector<double>& Kband, int n_band,
                 int p, int first, int n) {
  const int W = 2 * p + 1;
  if (first < 0 || n < 1 || first + n > n_band) throw std::invalid_argument("fdm: bad range");
  std::vector<double> M(static_cast<size_t>(n) * n, 0.0), K(M.size(), 0.0);
  for (int i = 0; i < n; ++i)
    for (int d = -p; d <= p; ++d) {
      const int j = i + d;
      if (j < 0 || j >= n) continue;
      const size_t b = static_cast<size_t>(first + i) * W + p + d;
      M[static_cast<size_t>(i) * n + j] = Mband[b];
      K[static_cast<size_t>(i) * n + j] = Kband[b];
    }
  // Cholesky M = L L^T (row-major lower triangle)
  std::vector<double> L(M.size(), 0.0);
  for (int j = 0; j < n; ++j) {
    double s = M[static_cast<size_t>(j) * n + j];
    for (int k = 0; k < j; ++k) s -= L[static_cast<size_t>(j) * n + k] * L[static_cast<size_t>(j) * n + k];
    if (!(s > 0.0)) throw std::runtime_error("fdm: mass factor not positive definite");
    const double ljj = std::sqrt(s);
    L[static_cast<size_t>(j) * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double t = M[static_cast<size_t>(i) * n + j];
      for (int k = 0; k < j; ++k) t -= L[static_cast<size_t>(i) * n + k] * L[static_cast<size_t>(j) * n + k];
      L[static_cast<size_t>(i) * n + j] = t / ljj;
    }
  }
  // Y = L^-1 K (forward substitution per column), C = L^-1 Y^T = L^-1 K L^-T
  auto lsolve = [&](std::vector<double>& X) {  // X (row-major n x n) <- L^-1 X
    for (int col = 0; col < n; ++col)
      for (int i = 0; i < n; ++i) {
        double s = X[static_cast<size_t>(i) * n + col];
        for (int k = 0; k < i; ++k) s -= L[static_cast<size_t>(i) * n + k] * X[static_cast<size_t>(k) * n + col];
        X[static_cast<size_t>(i) * n + col] = s / L[static_cast<size_t>(i) * n + i];
      }
  };
  std::vector<double> Y = K;
  lsolve(Y);
  std::vector<double> C(Y.size());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) C[static_cast<size_t>(i) * n + j] = Y[static_cast<size_t>(j) * n + i];
  lsolve(C);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double s = 0.5 * (C[static_cast<size_t>(i) * n + j] + C[static_cast<size_t>(j) * n + i]);
      C[static_cast<size_t>(i) * n + j] = C[static_cast<size_t>(j) * n + i] = s;
    }
  Fdm1D out;
  out.n = n;
  std::vector<double> Q;
  sym_eigen_jacobi(C, n, out.lam, Q);
  // V = L^-T Q (back substitution per eigenvector), column-major
  out.V.assign(static_cast<size_t>(n) * n, 0.0);
  for (int col = 0; col < n; ++col) {
    const double* q = &Q[static_cast<size_t>(col) * n];
    double* v = &out.V[static_cast<size_t>(col) * n];
    for (int i = n - 1; i >= 0; --i) {
      double s = q[i];
      for (int k = i + 1; k < n; ++k) s -= L[static_cast<size_t>(k) * n + i] * v[k];
      v[i] = s / L[static_cast<size_t>(i) * n + i];
    }
  }
  return out;
}

}  // namespace tgb
