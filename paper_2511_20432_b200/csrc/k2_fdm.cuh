// K2 option — Jacobi-free theta-step solve for separable patches: PCG with the
// fast-diagonalization preconditioner (SURVEY.md §8f "stronger
// preconditioner"; see host/fdm.hpp and k2_fdm.cu).
#pragma once

#include <functional>
#include <cuda_runtime.h>

#include "k2_kron.cuh"

namespace tgb {

struct FdmDev {
  int n[3];            // free-grid sizes
  const double* V[3];  // n_d x n_d column-major eigenvectors (V^T M V = I)
  const double* dinv;  // 1 / (a + b (lx_i + ly_j + lz_k)), free flat order
  const double* sinv;  // optional diagonal S^-1 (P = S^-1 V D V^T S^-1), null for none
};

// dinv from the eigenvalues (device arrays lam[3]).
void fdm_inverse_eigs(const int n[3], const double* lx, const double* ly, const double* lz,
                      double a, double b, double* dinv, cudaStream_t s);

// z = V diag(dinv) V^T r (= A^-1 r for the separable operator); t1, t2 are
// n_free scratch vectors. Six cuBLAS DGEMMs (mode products along x, y, z) and
// one scaling kernel.
void fdm_apply(const FdmDev& F, const double* r, double* z, double* t1, double* t2,
               cudaStream_t s);

// PCG (the reference's pcg_jacobi loop, sparse.cpp:41-100, with the Jacobi
// diagonal replaced by the fast-diagonalization inverse): warm start in x,
// stop test ||r||/||b|| <= tol before each matvec, b = 0 -> x = 0, status 3 /
// 4 as the reference. Host-driven; deterministic reductions.
struct FdmWork {
  double* r;
  double* z;
  double* p;
  double* Ap;
  double* t1;
  double* t2;
  double* partials;  // >= 2 * 512
  double* dots;      // device, 8 (the solve's scalars)
  double* h_dots;    // pinned host, 2
};
// x_map / p_map: TMA descriptors of x and w.p for the operator applies (or null)
// The reference's PCG loop (sparse.cpp:41-100: stop test, warm start, b = 0
// reset, failure semantics) with the preconditioner F in place of Jacobi and
// any operator apply (y = A v on the device).
PcgStatus pcg_precond_solve(const std::function<void(const double*, double*)>& apply,
                            const FdmDev& F, long n, const double* rhs, double* x,
                            const FdmWork& w, double tol, int max_iter, cudaStream_t s);
PcgStatus fdm_pcg_solve(const KronGrid& g, double a, double b, const FdmDev& F, const double* rhs,
                        double* x, const FdmWork& w, double tol, int max_iter, int sm_count,
                        cudaStream_t s, const TensorMap3* x_map = nullptr,
                        const TensorMap3* p_map = nullptr);

}  // namespace tgb
