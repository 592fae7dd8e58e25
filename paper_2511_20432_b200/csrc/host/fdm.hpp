// Fast diagonalization of the separable theta-step operator (SURVEY.md §8f
// "stronger preconditioner"): per direction the generalized eigenproblem
// K_d v = lambda M_d v with V_d^T M_d V_d = I, so that
//   A = a Mz x My x Mx + b (Mz x My x Kx + Mz x Ky x Mx + Kz x My x Mx)
//     = (V^-T) [a + b (lx_i + ly_j + lz_k)] (V^-1),   V = Vz x Vy x Vx,
// and A^-1 = V diag(1 / (a + b (lx + ly + lz))) V^T exactly (up to rounding).
#pragma once

#include <vector>

namespace tgb {

struct Fdm1D {
  int n = 0;
  std::vector<double> V;    // n x n, column-major (column k = eigenvector k)
  std::vector<double> lam;  // n generalized eigenvalues
};

// From banded 1D factors (n_band x (2p+1), [i][p + (j - i)]); rows/columns
// [first, first + n) are kept (first = 1 drops a constrained first layer).
Fdm1D fdm_factor(const std::vector<double>& Mband, const std::vector<double>& Kband, int n_band,
                 int p, int first, int n);

// Symmetric eigen-decomposition C = Q diag(w) Q^T by cyclic Jacobi rotations
// (C: n x n row-major, overwritten; Q column-major). Exposed for tests.
void sym_eigen_jacobi(std::vector<double>& C, int n, std::vector<double>& w,
                      std::vector<double>& Q);

}  // namespace tgb
