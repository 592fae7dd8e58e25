// K1 — point-source superposition kernels (see k1_superpose.cu).
#pragma once

#include <algorithm>
#include <cuda_runtime.h>

namespace tgb {

// Per-source, per-time constants (see src_exp in common.cuh); 96 bytes, read
// as three 32-byte broadcasts.
struct __align__(32) SrcRec {
  double sx, sy, sz;  // position (m)
  double nisp;        // -(1024/ln2) / spread, spread = 4 alpha (t - tau)
  double magicL;      // L + 1.5*2^52, L = rint((1024/ln2) log c), c = E/(rho c (pi spread)^1.5)
  double gfac;        // -1 / (2 alpha (t - tau))
  double thr;         // keep the pair iff r.r <= thr (cull and causality folded in)
  int thr_lo, thr_hi; // hi32(thr) - 1, hi32(thr) + 1: the fast-decision band
  double q0, q1, q2;  // C d_i, C = exp(log c - L ln2/1024)
  double pad;
};
static_assert(sizeof(SrcRec) == 96, "SrcRec must stay 96 bytes");

#ifndef K1_THREADS
#define K1_THREADS 256
#endif
#ifndef K1_CHUNK
#define K1_CHUNK 128
#endif
constexpr int kK1Threads = K1_THREADS;
constexpr int kK1Chunk = K1_CHUNK;  // sources per shared-memory stage (12 KB)
constexpr int kK1Stages = 3;
constexpr int kMaxSplits = 16;  // source splits of one launch (k1_choose_splits)

// Per-CTA source ranges (K5's remainder launch): CTA x takes only the sources
// [J[r], E[r]) of its region r = cta_region[x], split over grid.y; null =
// the launch's one range. okbits (when J[r] > 0): bit j - J[r] of row r
// (words per row) set = source j is in the region's contraction; skipped here.
struct K1Ranges {
  const int* cta_region = nullptr;
  const int* J = nullptr;
  const int* E = nullptr;
  const unsigned* okbits = nullptr;
  int words = 0;
};

void k1_upload_exp_table(cudaStream_t stream);
// the src_exp table (common.cuh) on the host: kExpTableSize doubles
void k1_exp_table_host(double* tab);
int k1_choose_splits(int n_pts, int n_src, int sm_count, int points_per_cta, int resident);
// CTAs of k1_partial<P> resident per SM (its launch bounds)
int k1_resident_ctas(int P);
void k1_prepare(const double* d_src6, int n, double t, double alpha, double rcp, double cull,
                SrcRec* d_rec, cudaStream_t stream);
// planar: all sources lie on z = zs (k1_partial's PLANAR variant)
void k1_launch_partial(const SrcRec* d_rec, int n_src, const double* d_pts, const int* d_index,
                       int n_pts, int S, bool grad, int P, double* d_part, cudaStream_t stream,
                       bool planar = false, double zs = 0.0, const K1Ranges& rg = K1Ranges{});
void k1_launch_combine_field(const double* d_part, int S, int n, double* d_val, double* d_grad,
                             cudaStream_t stream);
void k1_launch_combine_dirichlet(const double* d_part, int S, int n, double* d_out,
                                 cudaStream_t stream, bool negate = true);
void k1_launch_combine_flux(const double* d_part, int S, int n, const int* d_index,
                            const double* d_normals, const double* d_weights, double k,
                            double* d_gq, cudaStream_t stream);

}  // namespace tgb
