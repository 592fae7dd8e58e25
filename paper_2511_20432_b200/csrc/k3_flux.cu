// K3 — Neumann load assembly from the analytic flux (reference:
// assemble_boundary_load / assemble_flux_load, proj/src/assembly.cpp:117-166).
//
// Per step, on the device:
//   k3_point_index   compact list of the active face quadrature points: every
//                    lateral face element contributes its base rule, or its
//                    fine rule when it is within elevate_radius of the newest
//                    source (the host decides the fine set with the
//                    reference's exact arithmetic and uploads the sorted list
//                    plus the running extra-point counts);
//   (K1, flux mode)  g_q = (-k grad T~ . n_q) w_q at each active point;
//   k3_local         loc[e][a] = sum_q g_q N_q[a], q in the reference's order;
//   k3_gather        F[i] = sum of loc[e][a] over the (face, element, a)
//                    incidence list of DOF i, in the reference's scatter order
//                    (a deterministic gather instead of atomics: reruns are
//                    bitwise identical and match the serial scatter).
// Products and sums use explicit _rn intrinsics (no FMA contraction) so that
// K3 adds nothing beyond the flux values' own rounding differences.
#include "k3_flux.cuh"

namespace tgb {

__global__ void k3_point_index_kernel(FaceTables ft, const int* __restrict__ fine,
                                      const int* __restrict__ extra, int n_fine,
                                      int* __restrict__ pt_index, int* __restrict__ elem_off) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ft.n_fe) return;
  int lo = 0, hi = n_fine;  // rank = number of fine elements before e
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (fine[mid] < e) lo = mid + 1;
    else hi = mid;
  }
  const bool is_fine = lo < n_fine && fine[lo] == e;
  const int off = ft.qb_off[e] + extra[lo];
  const int nq = is_fine ? ft.qf_off[e + 1] - ft.qf_off[e] : ft.qb_off[e + 1] - ft.qb_off[e];
  const int base = is_fine ? ft.qb_off[ft.n_fe] + ft.qf_off[e] : ft.qb_off[e];
  for (int q = 0; q < nq; ++q) pt_index[off + q] = base + q;
  elem_off[e] = is_fine ? -(off + 1) : off;  // the sign carries the rule
}

__global__ void k3_local_kernel(FaceTables ft, int e_begin, int e_end,
                                const int* __restrict__ elem_off,
                                const double* __restrict__ gq, double* __restrict__ loc) {
  const int ndk = ft.ndk;
  const long t = e_begin * static_cast<long>(ndk) + blockIdx.x * static_cast<long>(blockDim.x) +
                 threadIdx.x;
  if (t >= static_cast<long>(e_end) * ndk) return;
  const int e = static_cast<int>(t / ndk), a = static_cast<int>(t % ndk);
  const int eo = elem_off[e];
  const bool fine = eo < 0;
  const int off = fine ? -eo - 1 : eo;
  const int q0 = fine ? ft.qf_off[e] : ft.qb_off[e];
  const int nq = (fine ? ft.qf_off[e + 1] : ft.qb_off[e + 1]) - q0;
  const double* N = (fine ? ft.Nf : ft.Nb) + static_cast<size_t>(q0) * ndk;
  const double* gp = gq + off;
  // the sum in q order (the reference's), its operands fetched 9 at a time:
  // the loads of a chunk are independent, so their latency overlaps instead
  // of serialising an 81-term fine-rule chain behind one load per term
  constexpr int C = 9;
  double s = 0.0;
  int q = 0;
  for (; q + C <= nq; q += C) {
    double g[C], n[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      g[c] = gp[q + c];
      n[c] = N[(q + c) * ndk + a];
    }
#pragma unroll
    for (int c = 0; c < C; ++c) s = __dadd_rn(s, __dmul_rn(g[c], n[c]));
  }
  for (; q < nq; ++q) s = __dadd_rn(s, __dmul_rn(gp[q], N[q * ndk + a]));
  loc[t] = s;
}

__global__ void k3_gather_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ src,
                                 const double* __restrict__ loc, double* __restrict__ F) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) s = __dadd_rn(s, loc[src[k]]);
  F[i] = s;
}

void k3_point_index(const FaceTables& ft, const int* d_fine, const int* d_extra, int n_fine,
                    int* d_pt_index, int* d_elem_off, cudaStream_t s) {
  if (ft.n_fe <= 0) return;
  k3_point_index_kernel<<<(ft.n_fe + 127) / 128, 128, 0, s>>>(ft, d_fine, d_extra, n_fine,
                                                              d_pt_index, d_elem_off);
}

void k3_local(const FaceTables& ft, int e_begin, int e_end, const int* d_elem_off,
              const double* d_gq, double* d_loc, cudaStream_t s) {
  const long n = static_cast<long>(e_end - e_begin) * ft.ndk;
  if (n <= 0) return;
  k3_local_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(ft, e_begin, e_end,
                                                                   d_elem_off, d_gq, d_loc);
}

void k3_gather(int n, const int* d_ptr, const int* d_src, const double* d_loc, double* d_F,
               cudaStream_t s) {
  if (n <= 0) return;
  k3_gather_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, d_ptr, d_src, d_loc, d_F);
}

}  // namespace tgb
