// K5 — sum-factorised superposition on tensor-grid point sets, fused
// (see k5_fused.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "k1_superpose.cuh"

namespace tgb {

// CTA output tile of the contraction (a rows x b columns of one grid) and the
// sources per shared-memory stage / per stream-K work item.
// measured (config 4, tools/k5_time.py): 64 x 96 / 256 threads / 2 CTAs per SM
// 5.97 ms per step's contraction, 128 x 96 / 512 / 1: 5.78, 64 x 192: 5.95,
// 128 x 192 / 512 / 1: 5.58
#ifndef K5_TA
#define K5_TA 128
#endif
#ifndef K5_TB
#define K5_TB 192
#endif
#ifndef K5_THREADS
#define K5_THREADS 512
#endif
#ifndef K5_MINB
#define K5_MINB 1
#endif
constexpr int kSfTA = K5_TA;
constexpr int kSfTB = K5_TB;
constexpr int kSfKS = 32;
constexpr int kSfItem = 1024;
constexpr int kSfThreads = K5_THREADS;  // 16 warps (4 x 4 of 32 x 48), 1 CTA per SM
constexpr int kSfMinBlocks = K5_MINB;
constexpr int kSfWarps = kSfThreads / 32;
constexpr int kSfWR = kSfTA / 32;                 // warp blocks per tile column (32 rows each)
constexpr int kSfWN = kSfWR * kSfTB / kSfWarps;   // columns per warp block

// Warp w of a CTA -> its block (rows [32 wa, +32), columns [kSfWN wb, +kSfWN)):
// the rows rotate with the column, so the blocks of one block row or column
// sit on different SM sub-partitions (w % 4, one FP64 pipe each) and a partial
// tile's active warps spread over the four pipes.
__host__ __device__ inline void sf_warp_block(int w, int& wa, int& wb) {
  wb = w / kSfWR;
  wa = (w + wb) % kSfWR;
}

// A point set that is a tensor grid up to coordinate rounding: point (a, b)
// sits at (xf on axis axn, U[a] on axu, V[b] on axv).
struct SfGridDesc {
  int axn, axu, axv, na, nb;
  int flux;     // 1: the normal derivative (flux integrand), 0: the value (Dirichlet)
  int vplane;   // 1: every source has V coordinate vs: the B exponent is cb[b] * nisp
  double xf;
  const double* U;
  const double* V;
  const double* cb;  // (V[b] - vs)^2 when vplane
};

// A CTA tile: rows [a0, a0 + na) x columns [b0, b0 + nb) of grid `grid`, whose
// sources come from region `region` (J = the contraction's prefix).
struct SfTile {
  int grid, a0, b0, na, nb, region;
};

// A region: points whose box [lo, hi] (+- delta per axis) decides which
// sources no cull can reach anywhere in it (the contraction's prefix [0, J))
// and which are culled everywhere in it (dropped from the pair-wise
// remainder [J, E)). npts: its point count (profitability; < 0: never contracted).
struct SfRegion {
  double lo[3], hi[3];
  double delta;
  double npts;
};

struct SfPlanArgs {
  const double* src6;
  int n_act;           // the causally active prefix (later sources are exact zeros)
  double t, alpha, cull;
  double min_pairs;    // J * npts below this and J below min_sources: no contraction for the
  int min_sources;     // region (its pairs are cheap on K1; a long J is not: one remainder CTA
                       // would run all of it over its points)
  bool gemm;           // false: J = 0 everywhere (every pair on K1)
};

// Per (grid, source) constants of the factors (64 bytes): u, v, nisp =
// -(1024/ln2)/spread, magicL = L + 1.5*2^52 and the folded cubic q0..q2, pad
// (= q3) of the A factor (src_exp's representation, common.cuh; zero for
// inactive sources).
struct SfConst {
  double u, v, nisp, magicL, q0, q1, q2, pad;
};

// Which regions a call computes: static flux tiles [0, nt_flux), Greville
// tiles [nt_flux, nt_static), the step's fine regions after n_static_regions;
// parts not requested, and (multi-GPU) regions r with r % world != rank, get
// J = E = 0 (no work; their outputs come out as zeros).
struct SfPlanMask {
  bool flux, dir;
  int nt_flux, nt_static;
  int rank, world;
};
// The sources of [J, E) that no cull reaches anywhere in the region's box
// either (a later source of the history can be eligible again: the prefix
// stops at the first failure) join the contraction: per region r with J > 0
// their indices in order, elist[r * cap + k] for k < Jc[r] - J[r], and their
// bits okbits[r * words + (j - J) / 32] (the remainder launch skips them).
struct SfLists {
  int* elist;
  unsigned* okbits;
  int* Jc;      // the contraction's source count: J + the eligible ones in [J, E)
  int* Jclast;  // Jc of the computed static regions (queries)
  int cap, words;
};

// regions' J, E (the computed static regions' also into Jlast / Elast, kept
// across calls for queries) and the eligible lists
void sf_plan(const SfPlanArgs& a, const SfRegion* d_regions, int n_regions, int* d_J, int* d_E,
             const SfPlanMask& mask, int n_static_regions, int* d_Jlast, int* d_Elast,
             int* d_Jraw, const SfLists& lists, cudaStream_t s);
// tiles' item prefix (n_tiles + 1) over their regions' contraction counts Jc
// and the call's contraction flops (2 na nb Jc summed over the tiles) added to
// stats[0]
void sf_items(const SfTile* d_tiles, int n_tiles, const int* d_Jc, int* d_prefix, double* stats,
              cudaStream_t s);
void sf_prep(const double* d_src6, int n_act, double t, double alpha, double rcp,
             const SfGridDesc* d_grids, int n_grids, int max_src, SfConst* d_cst, cudaStream_t s);

// The persistent stream-K contraction: the items (tile, 1024-source chunk) of
// all tiles split evenly over `ctas` CTAs; each CTA accumulates its run of
// items per tile in registers (DMMA m8n8k4) and writes one partial tile per
// (tile t, CTA c) to slot t + c of `scratch` (kSfTA * kSfTB doubles each, cell
// (a, b) at a + kSfTA * b). Deterministic: the split depends only on the item
// count and `ctas`. d_cst: one row of max_src SfConst per grid (sf_prep); entry
// max_src - 1 of every row must be a zero factor (max_src > the source count).
// Contraction position k of region r is source k for k < J[r], else
// lists.elist[r * cap + k - J[r]].
void sf_contract_fused(const SfGridDesc* d_grids, const SfTile* d_tiles, int n_tiles,
                       const int* d_prefix, const int* d_J, const SfLists& lists,
                       const SfConst* d_cst, int max_src, const double* d_tab, double* d_scratch,
                       int ctas, cudaStream_t s);
int sf_contract_max_ctas(int sm_count);

// Entries of the pair-wise remainder launch (K1 with per-region ranges): one
// per point, grouped by region and padded to whole K1 CTAs.
struct SfEntries {
  const int* q;      // point id (into the flux quadrature points, Greville after them)
  const int* pos;    // output slot (compact flux point / constrained DOF), -1 = none
  const int* tile;   // the point's contraction tile, -1 = none
  const int* cell;   // its cell in the tile
};

// positions of the static flux entries: pos = elem_off[e] + (q - qb_off[e])
// unless element e takes its fine rule this step (elem_off < 0, k3_flux.cu),
// or the entry is padding (tile < 0): then -1
void sf_base_positions(int n, const int* d_q, const int* d_tile, const int* d_qelem,
                       const int* d_qb_off, const int* d_elem_off, int* d_pos, cudaStream_t s);

// gq[pos] = (-k (grad.n)) w from the remainder's partials + (-k (G n_axn)) w,
// over entries [e0, e1) (flux); g[pos] = -v - G over [d0, d1) (Dirichlet).
// G = the sum over the tile's segments in CTA order (sf_contract_fused).
struct SfAddArgs {
  SfEntries ent;
  const double* part;  // K1 partial planes: S x 4 x n_entries
  int S, n_entries;
  const SfGridDesc* grids;
  const SfTile* tiles;
  const int* prefix;
  int n_tiles, ctas;
  const double* scratch;
  const double* normals;
  const double* weights;
  double k;
  double* gq;
  double* g;
};
void sf_add(const SfAddArgs& a, int e0, int e1, bool flux, cudaStream_t s);

}  // namespace tgb
