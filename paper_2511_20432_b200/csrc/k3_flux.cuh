// K3 — Neumann load assembly kernels (see k3_flux.cu).
#pragma once

#include <cuda_runtime.h>

namespace tgb {

// Device view of the lateral face sets: per-element offsets into the base and
// fine quadrature arrays (n_fe + 1 entries each) and the basis tables
// (ndk kept DOF columns per element).
struct FaceTables {
  int n_fe, ndk;
  const int* qb_off;
  const int* qf_off;
  const double* Nb;
  const double* Nf;
};

// d_extra[r] = sum over the first r fine elements of (fine - base) rule size
void k3_point_index(const FaceTables& ft, const int* d_fine, const int* d_extra, int n_fine,
                    int* d_pt_index, int* d_elem_off, cudaStream_t s);
// local loads of the face elements [e_begin, e_end) (loc[e * ndk + a])
void k3_local(const FaceTables& ft, int e_begin, int e_end, const int* d_elem_off,
              const double* d_gq, double* d_loc, cudaStream_t s);
void k3_gather(int n, const int* d_ptr, const int* d_src, const double* d_loc, double* d_F,
               cudaStream_t s);

}  // namespace tgb
