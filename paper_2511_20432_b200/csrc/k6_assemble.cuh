// K6 — the general patch's θ-step operators assembled on the device (see
// k6_assemble.cu).
#pragma once

#include <cuda_runtime.h>

#include "k4_eval.cuh"

namespace tgb {

// The patch, its elements and the quadrature on the device.
struct AsmPatch {
  NurbsDev V;
  int n_el[3];
  const double* bp[3];    // breakpoints per direction (n_el + 1)
  const int* espan[3];    // knot span of each element per direction
  const int* elo[3];      // per basis index: the first / last element (per direction)
  const int* ehi[3];      //   whose span supports it
  int nq[3];
  const double* gn[3];    // Gauss nodes / weights per direction
  const double* gw[3];
  double rc, k;           // rho c, conductivity (the host's doubles)
};

// Free-row extraction maps (DofSplit): free row f is full row free_list[f];
// a full column c is free column free_index[c] / constrained column
// con_index[c] (-1 otherwise).
struct AsmMaps {
  const int* free_list;
  const int* free_index;
  const int* con_index;
  int n_free;
};

// Sliced-ELL output (k2_csr.cuh DevSell layout), slice pointers set.
struct SellOut {
  const long long* sp;
  int* col;
  double* val;
};

// Can K6 take this patch (basis block small enough for its per-thread
// element-matrix registers)?
bool k6_supported(const AsmPatch& P);
// Element matrices of the elements [e0, e0 + ne) (flat order, first index
// fastest): per element the lower triangles of M and K packed at a (a + 1) / 2
// + b. flags |= 1 on a non-positive Jacobian determinant or a span mismatch.
size_t k6_entries_per_element(const AsmPatch& P);
void k6_element_matrices(const AsmPatch& P, int e0, int ne, double* d_lm, double* d_lk,
                         int* d_flags, cudaStream_t s);
// Adds the contributions of the element layers [k0, k1) (their matrices from
// element e_base on, k6_element_matrices) to the tensor-pattern values M / K of
// the rows [r0, r1) (those the layers touch), per entry in element order.
void k6_gather(const AsmPatch& P, const int* d_row_ptr, int r0, int r1, int k0, int k1,
               int e_base, const double* d_lm, const double* d_lk, double* d_M, double* d_K,
               cudaStream_t s);
// Per free row: the entries of A_ff (free columns), A_fc (constrained
// columns) and B_f (all columns) in the pattern row.
void k6_row_lengths(const AsmPatch& P, const AsmMaps& m, int* d_lenA, int* d_lenAc, int* d_lenB,
                    cudaStream_t s);
// A = inv_dt M + th K, B = inv_dt M + mth K (assembly.cpp:194-199: inv_dt =
// 1 / dt, mth = -(1 - theta)) on the free rows, into the three SELL outputs
// (padding zeroed beforehand).
void k6_fill(const AsmPatch& P, const int* d_row_ptr, const AsmMaps& m, const double* d_M,
             const double* d_K, double inv_dt, double th, double mth, const SellOut& A,
             const SellOut& Ac, const SellOut& B, cudaStream_t s);

// ---------------------------------------------------------------------------
// Face quadrature sets on the device: build_face_sets (host/mesh.cpp; the
// reference's classify_boundary / build_face_element, proj/src/mesh.cpp:158-236,
// face_point, proj/src/splines.cpp:305-321), bit-identical to the host's.

// One lateral face element: face id (FaceId order), rule sizes, the element's
// parametric centre / half width along the face's two tangent axes.
struct FaceElemDev {
  int f, qu, qv;
  double mu, hu, mv, hv;
};

struct FaceSetDev {
  NurbsDev V;
  const FaceElemDev* el;
  int n_el, fm, nd;        // elements, fine-rule multiplier, basis block size
  const int* qb_off;       // n_el + 1 base / fine point offsets
  const int* qf_off;
  int tqb, tqf;
  const double* gnodes;    // Gauss rules n = 1 .. nmax at offset n (n - 1) / 2
  const double* gweights;
  double* x;               // 3 per point: base points, then fine points
  double* nrm;             // 3 per point (outward unit normals)
  double* w;               // 1 per point
  double* Nb;              // nd per base point (basis values, basis order)
  double* Nf;              // nd per fine point
  int* dofs;               // nd per element (grid indices of the basis block)
  double* centers;         // 3 per element
  int* flags;              // 1: non-positive det in the map, 2: degenerate surface point, 4: domain
};
void k6_face_sets(const FaceSetDev& F, cudaStream_t s);
// the columns of each element nonzero at one of its base or fine points, in
// order (keep: n_el x nd, nkeep: n_el)
void k6_face_keep(const FaceSetDev& F, int* d_keep, int* d_nkeep, cudaStream_t s);
// tables on the kept columns: Nbk / Nfk (ndk per point, zero padded), dofk
// (ndk per element, -1 padded)
void k6_face_compact(const FaceSetDev& F, const int* d_keep, const int* d_nkeep, int ndk,
                     double* d_Nbk, double* d_Nfk, int* d_dofk, cudaStream_t s);

}  // namespace tgb
