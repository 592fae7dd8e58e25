// K2 — matrix-free theta-step operator and Jacobi-PCG for separable
// (Kronecker) patches. See k2_kron.cu.
#pragma once

#include <cuda_runtime.h>

namespace tgb {

#ifndef K2_TX
#define K2_TX 32
#endif
constexpr int kKronTX = K2_TX;  // tile width along xi; 16x16 tiles: 100 us/iter (cfg 4) vs 93
#ifndef K2_TY
#define K2_TY 8
#endif
constexpr int kKronTY = K2_TY;  // tile height along eta; 16 (1 CTA/SM): 105 us/iter vs 93 (cfg 4)
constexpr int kKronMaxP = 3;

// A grid of control points (possibly the free sub-grid) with the banded 1D
// mass / stiffness factors of each direction: entry [i][P + (j - i)] of an
// (n x (2P+1)) row-major band array is the (i, j) coupling.
struct KronGrid {
  int p;  // spline degree (1..3); band width 2p+1
  int n[3];
  const double* M[3];
  const double* K[3];
};

// Opaque CUtensorMap (128 bytes, 64-byte aligned): a 3D TMA descriptor of one
// grid vector with a (32+2p) x (8+2p) x 2 box (halo'd plane tiles; 32 x 8 x 2
// with halo = false), zero fill outside the grid.
struct alignas(64) TensorMap3 {
  unsigned char bytes[128];
};
// Encode the descriptor for `base` (a vector over g's grid). Returns false
// when TMA cannot address the grid (row pitch not a multiple of 16 bytes);
// the kernels then load planes with ordinary loads.
// strip = true: the box of the transposed 8 x 32 strip tile (k2_kron.cu)
bool k2_make_map(const KronGrid& g, const double* base, TensorMap3* out, bool halo = true,
                 int planes = 2, bool strip = false);
// whether the single-sweep solve covers g's ragged last x columns with strip
// tiles (it then needs the strip maps of Cg1Maps)
bool k2_strip_applies(const KronGrid& g);

// y = Op(a1, b1) v1 + Op(a2, b2) v2 with Op(a, b) = a (Mz x My x Mx) +
//     b (Mz x My x Kx + Mz x Ky x Mx + Kz x My x Mx); v2 may be null.
struct KronTerms {
  double a1, b1, a2, b2;
};

// theta-step right-hand side on the free rows (assembly.cpp:245-272):
//   rhs_f = [B T_n - A g~]_f + theta F_{n+1,f} + (1-theta) F_{n,f}
struct RhsArgs {
  const double* T_full;    // expanded state at level n (free + constrained)
  const double* g_full;    // g_{n+1} on the constrained layer, zero elsewhere
  const double* F_n;       // full-size loads
  const double* F_np1;
  double theta;
  int bottom_axis, bottom_layer;  // constrained layer
  double* rhs;             // n_free, free flat order
};

struct PcgStatus {
  int iterations;
  int status;  // 0 ok, 3 no convergence, 4 indefinite direction, 2 bad diagonal
  double rel_residual;
  double bnorm;
};

// Work vectors of a solve; pA/pB are the ping-pong search directions,
// z = D^-1 r the preconditioned residual, inv_diag = 1 / diag(A) (set once
// per operator by k2_inverse_diagonal).
struct PcgWork {
  double* r;
  double* z;
  double* pA;
  double* pB;
  double* Ap;
  const double* inv_diag;
  double* partials;  // >= 8 * max_blocks
  PcgStatus* status;
  unsigned long long* trace;  // optional: per-phase %globaltimer stamps of CTA 0
};

// TMA descriptors of the vectors the PCG kernel sweeps (x, z, pA, pB), all
// over the free grid; valid = false -> plain loads.
struct PcgMaps {
  bool valid;
  TensorMap3 x, z, pA, pB;
};

// Work vectors of the single-sweep (Chronopoulos-Gear) solve: r, w = A u and
// s = A p ping-pong between two buffers (their halos are read while the sweep
// writes the next iterate); p is point-local. All over the free grid.
struct Cg1Work {
  double* p;
  double* r[2];
  double* w[2];
  double* s[2];
  const double* inv_diag;
  double* partials;  // >= 8 * max_blocks
  PcgStatus* status;
};
struct Cg1Maps {
  TensorMap3 x, inv_diag, r[2], w[2], s[2];
  TensorMap3 xc, pc;  // un-halo'd boxes of x and p (point-local inputs)
  // the same boxes for the strip tiles (valid when strip != 0)
  TensorMap3 sx, sr[2], sw[2], ss[2], sxc, spc;
  int strip;
};

void k2_theta_rhs(const KronGrid& full, double a_b, double b_b, double a_a, double b_a,
                  const RhsArgs& args, const TensorMap3* mT, const TensorMap3* mg, int sm_count,
                  cudaStream_t s);
// inv_diag = 1.0 / diag(Op(a, b)) (sparse.cpp:47-52); status = 2 when a
// diagonal entry is not positive.
void k2_inverse_diagonal(const KronGrid& g, double a, double b, double* inv_diag,
                         PcgStatus* status, cudaStream_t s);
int k2_pcg_max_blocks(int p, int sm_count, int nz);
// Jacobi-PCG on A = Op(a, b) over the free grid, one persistent cooperative
// launch per solve; x holds the warm start on entry.
void k2_pcg_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const PcgWork& w, const PcgMaps& maps, double tol, int max_iter, int blocks,
                  cudaStream_t s);
// The same solve with one tile sweep and one grid reduction per iteration
// (TMA only; see k2_kron.cu). Stop test, failure codes and warm start as
// k2_pcg_solve.
// planes per sweep step for this grid (2, or 4 for grids that cannot fill the
// GPU at 2 CTAs/SM); the maps of the solve must be made with that box depth
int k2_cg1_planes(const KronGrid& g, int sm_count);
int k2_cg1_max_blocks(int p, int sm_count, int nz, int pl);
void k2_cg1_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const Cg1Work& w, const Cg1Maps& maps, double tol, int max_iter, int blocks,
                  cudaStream_t s, int pl);
// The same solve with the solver state resident in shared memory (small
// grids, k2_resident.cu): one CTA per TX x TY x nz column block.
struct K2ResPlan {
  int TX, TY, ntx, nty;
  size_t smem;  // dynamic shared memory per CTA
};
struct K2ResWork {
  double* wx[2];     // w^ exchange buffers (free grid)
  double* ux;        // u_0 exchange buffer (free grid)
  double* partials;  // >= 8 * ntx * nty
  PcgStatus* status;
};
// false when no tile shape fits one cooperative wave (or TG_K2_NO_RESIDENT)
bool k2_res_plan(const KronGrid& g, int sm_count, int max_smem, K2ResPlan* out);
void k2_res_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const K2ResWork& w, const K2ResPlan& pl, double tol, int max_iter,
                  cudaStream_t s);

// plain y = Op(a, b) v (tests / the operator alone)
// v_map: TMA descriptor of v (k2_make_map) or null for plain loads
void k2_apply(const KronGrid& g, double a, double b, const double* v, double* y, int sm_count,
              cudaStream_t s, const TensorMap3* v_map = nullptr);

// ---- the single-sweep solve on one z-slab (multi-GPU; k2_kron.cu)
// Scalars carried from launch to launch (double-buffered by the caller).
struct SlabState {
  double alpha, beta, gamma, bnorm, rel;
  int it, status, stage, done;  // stage 1: init sums pending, 2: delta_0 pending, 3: iterating
};
struct SlabCtl {
  int phase;            // 0: r0 / u0 sweep, 1: w^0 sweep, 2: an iteration sweep
  int cur;              // the ping-pong buffers an iteration sweep reads
  int zo0, zo1;         // own planes (local indices) of the dot products
  int world;
  const double* gath;   // world x 4 partial sums of the previous launch, rank order
  double* mine;         // this launch's 4 partial sums
  const SlabState* sin;
  SlabState* sout;
  double* cta_part;     // >= 4 per CTA
  unsigned int* ticket; // zero between launches
};
int k2_slab_max_blocks(int p, int sm_count, int nz, int pl);
void k2_slab_launch(const KronGrid& g, double a, double b, const double* rhs, double* x,
                    const Cg1Work& w, const Cg1Maps& maps, double tol, int max_iter, int blocks,
                    const SlabCtl& ctl, cudaStream_t s, int pl);

}  // namespace tgb
