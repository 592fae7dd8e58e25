// K2 general (assembled CSR) path — see k2_csr.cu.
#pragma once

#include <cuda_runtime.h>

#include "k2_kron.cuh"

namespace tgb {

struct DevCsr {
  int rows;
  const int* row_ptr;
  const int* col;
  const double* val;
};

// Sliced ELL (SELL-32) copy of a CSR matrix: rows in slices of 32; inside a
// slice, entry k of the 32 rows is contiguous (val/col[slice_ptr[s] + 32 k +
// lane]), so one thread per row reads coalesced while still summing its row
// in CSR order (the reference's CsrMatrix::multiply order). Slices are padded
// to their longest row; row_len masks the padding.
struct DevSell {
  int rows;
  const long long* slice_ptr;
  const int* row_len;
  const int* col;
  const double* val;
};

// Work vectors of an assembled-operator solve (stored Jacobi diagonal).
struct CsrWork {
  double* r;
  double* p;
  double* Ap;
  double* inv_diag;
  double* partials;  // >= 8 * max_blocks
  PcgStatus* status;
};

int csr_pcg_max_blocks(int sm_count);
void csr_inverse_diagonal(const DevCsr& A, double* inv_diag, PcgStatus* st, cudaStream_t s);
void csr_inverse_diagonal(const DevSell& A, double* inv_diag, PcgStatus* st, cudaStream_t s);
void csr_theta_rhs(const DevSell& Bf, const DevSell& Ac, const double* T, const double* g1,
                   const double* F0, const double* F1, const int* free_list, double theta,
                   double* rhs, cudaStream_t s);
void csr_pcg_solve(const DevCsr& A, const double* rhs, double* x, const CsrWork& w, double tol,
                   int max_iter, int blocks, cudaStream_t s);
void csr_pcg_solve(const DevSell& A, const double* rhs, double* x, const CsrWork& w, double tol,
                   int max_iter, int blocks, cudaStream_t s);
void csr_apply(const DevCsr& A, const double* x, double* y, cudaStream_t s);
void csr_apply(const DevSell& A, const double* x, double* y, cudaStream_t s);

}  // namespace tgb
