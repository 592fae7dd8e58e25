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

// The same rows with implicit columns, for operators on a structured free
// grid (a single patch whose constrained layer is a boundary plane, so the
// free rows are an nx x ny x nz box in flat order): row r couples to
// r + (dk nz-plane + dj nx + di), |di|, |dj|, |dk| <= p, and entry o of the
// (2p+1)^3 offsets, ascending = the CSR's ascending columns, sits at
// val[(slice * noff + o) * 32 + lane] (zero where the CSR row has no such
// column). 8 instead of 12 bytes per stored entry (SELL: value + column).
struct DevDia {
  int rows;
  int nx, nxy, p, noff;
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
// DIA copy of a SELL operator on the free box (nx, ny, nz); false (nothing
// written) when some entry lies outside the (2p+1)^3 stencil. val must hold
// ceil(rows / 32) * 32 * (2p+1)^3 doubles.
bool csr_make_dia(const DevSell& A, int nx, int ny, int nz, int p, double* val, int* d_flag,
                  DevDia* out, cudaStream_t s);
void csr_pcg_solve(const DevDia& A, const double* rhs, double* x, const CsrWork& w, double tol,
                   int max_iter, int blocks, cudaStream_t s);
void csr_apply(const DevDia& A, const double* x, double* y, cudaStream_t s);
void csr_apply(const DevCsr& A, const double* x, double* y, cudaStream_t s);
void csr_apply(const DevSell& A, const double* x, double* y, cudaStream_t s);

}  // namespace tgb
