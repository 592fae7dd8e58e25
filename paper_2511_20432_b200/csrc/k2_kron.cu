// K2 — matrix-free theta-step operator and Jacobi-PCG on B200.
//
// Reference: DirichletSystem (proj/src/assembly.cpp:186-281) assembles
// A = M/dt + theta K and B = M/dt - (1-theta) K as CSR and pcg_jacobi
// (proj/src/sparse.cpp:41-100) runs ~130-170 serial CSR SpMV iterations per
// step. For separable patches (every axis-aligned cuboid, any knot grading)
// the p+1-point Gauss quadrature factorizes exactly, so
//   M = rho c (Mz x My x Mx),  K = k (Mz x My x Kx + Mz x Ky x Mx + Kz x My x Mx)
// with banded 1D factors (2p+1 diagonals). The apply is sum-factorized:
//   x-pass  u1 = Mx v, u2 = Kx v          (shared-memory plane tile with halo)
//   y-pass  w1 = My u1, w2 = My u2, w3 = Ky u1
//           s1 = a w1 + b (w2 + w3),  s2 = b w1
//   z-pass  y = Mz s1 + Kz s2            (2p+1-plane register window)
// A CTA owns 32 x 8 columns of the control grid and marches through z, PL
// planes per step (halving the barriers per plane). Halo'd (32+2p) x (8+2p)
// x PL boxes arrive by TMA (cp.async.bulk.tensor.3d, zero fill outside the
// grid) through mbarrier rings, so every vector is read from HBM once and
// written once per pass; the x/y halos come from L2. A prologue functor may
// build the tile the passes read from several rings (direction update,
// Chronopoulos-Gear residual update).
//
// Two persistent cooperative Jacobi-PCG solvers (one launch per solve):
//   k2_cg1_kernel (default): the Chronopoulos-Gear form, one tile sweep and
//     one grid reduction per iteration (see the section below);
//   k2_pcg_kernel: the reference's recurrences, two grid barriers per
//     iteration: A' p_new = z + beta p_old on the loaded tiles and Ap, p.Ap;
//     B x += alpha p, r -= alpha Ap, z = D^-1 r, r.z, r.r (streaming pass).
// Dot products are reduced per CTA in a fixed tree and across CTAs in a fixed
// order (bitwise-deterministic reruns). Reference semantics: inv_diag = 1.0 /
// d stored once, warm start, stop test ||r||/||b|| <= tol before the matvec,
// b = 0 -> x = 0, failure on pAp <= 0 or after max_iter.
#include <cooperative_groups.h>
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "context.hpp"
#include "k2_kron.cuh"

namespace cg = cooperative_groups;

namespace tgb {

namespace {

constexpr int kThreads = kKronTX * kKronTY;
#ifndef K2_MINB
#define K2_MINB (kKronTY > 8 ? 1 : 2)  // resident CTAs per SM of the persistent solvers
#endif
constexpr int kStages = 3;
constexpr int kTmaPlanes = 2;  // planes per TMA box / per sweep step
#ifndef K2_L2_AHEAD
#define K2_L2_AHEAD 0  // measured: 0 -> 92.9 us/iter, 1 -> 94.5, 2 -> 95.4, 4 -> 98.0 (config 4)
#endif
constexpr int kL2Ahead = K2_L2_AHEAD;  // steps beyond the shared-memory ring prefetched into L2

#ifndef K2_STRIP_W
#define K2_STRIP_W 6  // cost of a strip column-plane in quarters of a main one
#endif
// Tile shapes (control points per CTA, one per thread): the main 32 x 8
// tiles, and for grids whose x extent leaves a ragged remainder of <= 8
// columns (config 4: 258 = 8 * 32 + 2) a transposed 8 x 32 strip tile over
// those last columns, so the remainder costs ceil(ny / 32) tiles per plane
// instead of ceil(ny / 8) nearly empty 32-wide ones. Both shapes have the
// same halo'd plane size, so they share every shared-memory ring.
template <int TX_, int TY_, bool STRIP>
struct TileShape {
  static constexpr int TX = TX_, TY = TY_;
  static constexpr bool kStrip = STRIP;
};
using MainTile = TileShape<kKronTX, kKronTY, false>;
using StripTile = TileShape<kKronTY, kKronTX, true>;

template <int P, int PL, class Sh = MainTile>
struct Dims {
  static constexpr int W = 2 * P + 1;
  static constexpr int RY = Sh::TY + 2 * P;
  static constexpr int RX = Sh::TX + 2 * P;
  static constexpr int PLANE = RY * RX;                                    // doubles
  static constexpr int SLOT = ((PL * PLANE * 8 + 127) / 128) * 128 / 8;    // 128-byte slots
};

// NIN loaded vectors; NPASS separate x/y passes (2 for the RHS, whose two
// inputs carry different (a, b)); a prologue functor may build one tile v
// from the rings (the PCG direction update, the C-G residual update). The z
// band (Mz, Kz rows) of the whole grid follows the struct in dynamic shared
// memory.
// UB: buffers of the x-pass output. 2 lets step s+1's x-pass start while
// other warps still run step s's y-pass; 1 is enough for sweeps with a
// prologue, whose barrier after pro() already separates the two.
template <int P, int PL, int NIN, int NPASS, int ST = kStages, int UB = 2>
struct KSmem {
  static constexpr int kSt = ST;  // TMA ring depth (boxes in flight per input)
  static constexpr int kUb = UB;
  double ring[NIN][ST][Dims<P, PL>::SLOT];
  double v[PL][Dims<P, PL>::PLANE];
  // x-pass output rows [RY][TX] of the tile shape (the main shape's is the larger)
  double u1[NPASS][UB][PL][Dims<P, PL>::RY * kKronTX];
  double u2[NPASS][UB][PL][Dims<P, PL>::RY * kKronTX];
  uint64_t bar[NIN][ST];
};

template <int P, int PL, int NIN, int NPASS, int ST = kStages, int UB = 2>
__host__ __device__ constexpr size_t zband_offset() {
  return (sizeof(KSmem<P, PL, NIN, NPASS, ST, UB>) + 15) / 16 * 16;
}

// Work split: the grid is ntx x nty columns (32 x 8 control points each) of
// nz planes. The column-planes, linearized column by column, are cut into
// `blocks` equal contiguous ranges; a CTA sweeps its range as 1-2 column
// segments (each costs P halo planes per side). Equal shares whatever the
// column count (a static map keeps the reductions deterministic).
// With a strip (nsy > 0) the main tiles cover the first ntx * 32 columns and
// nsy strip tiles of 8 x 32 the columns from xs on; strip columns follow the
// main ones in the linearized column list.
// The CTAs' shares are cut in work units: a main column-plane costs wm units,
// a strip column-plane ws (strip tiles sweep slower per plane: narrow TMA
// boxes, 2-way bank conflicts on their 12-double rows), so the CTAs holding
// strip planes are not the last at the grid barrier.
struct TileIdx {
  int ntx, nty, nz;
  int nsy = 0;  // strip tiles along y (0: no strip)
  int xs = 0;   // first column of the strip
  int wm = 1, ws = 1;
  // column-aligned split (grid = ntx * nty + 2 nsy CTAs): CTA b < ntx * nty
  // sweeps main column b whole, the others half a strip column each, so all
  // CTAs march through z together and a tile's x/y halo rows were just
  // fetched by its neighbours (L2 hits instead of DRAM re-reads)
  int aligned = 0;
};
struct Seg {
  int x0, y0, k0, k1;
  int strip = 0;
};
inline TileIdx make_tiles(const KronGrid& g) {
  return {(g.n[0] + kKronTX - 1) / kKronTX, (g.n[1] + kKronTY - 1) / kKronTY, g.n[2]};
}
// the strip split when the ragged x remainder fits one strip tile's width
inline bool strip_applies(const KronGrid& g) {
  const int rx = g.n[0] % kKronTX;
  return g.n[0] > kKronTX && rx > 0 && rx <= StripTile::TX;
}
inline TileIdx make_tiles_strip(const KronGrid& g) {
  TileIdx T = make_tiles(g);
  if (!strip_applies(g)) return T;
  T.ntx = g.n[0] / kKronTX;
  T.xs = T.ntx * kKronTX;
  T.nsy = (g.n[1] + StripTile::TY - 1) / StripTile::TY;
  T.wm = 4;
  T.ws = K2_STRIP_W;
  if (const char* e = std::getenv("TG_K2_STRIP_W")) T.ws = std::max(1, std::atoi(e));
  return T;
}
__host__ __device__ __forceinline__ long n_columns(const TileIdx& T) {
  return static_cast<long>(T.ntx) * T.nty + T.nsy;
}
__host__ __device__ __forceinline__ long n_units(const TileIdx& T) {
  return (static_cast<long>(T.ntx) * T.nty * T.wm + static_cast<long>(T.nsy) * T.ws) * T.nz;
}
__device__ __forceinline__ Seg column_seg(const TileIdx& T, int col, int k0, int k1) {
  const int nmain = T.ntx * T.nty;
  if (col < nmain) return Seg{(col % T.ntx) * kKronTX, (col / T.ntx) * kKronTY, k0, k1, 0};
  return Seg{T.xs, (col - nmain) * StripTile::TY, k0, k1, 1};
}
// The next segment of the unit range [u, e): the planes whose first unit lies
// in it, within one column (false when none is left). Plane k of column c
// starts at unit base(c) + k w(c), so the CTA ranges partition the planes.
// 32-bit unit counts (< 2^31 for grids up to ~1e11 points): the loop state
// stays small beside kron_tile's registers.
__device__ __forceinline__ bool next_segment(const TileIdx& T, int& u, int e, Seg& out) {
  const int nmain = T.ntx * T.nty;
  const int mtot = nmain * T.wm * T.nz;
  while (u < e) {
    const bool main = u < mtot;
    const int w = main ? T.wm : T.ws;
    const int colu = T.nz * w;  // units per column
    const int c = main ? u / colu : (u - mtot) / colu;
    const int col = main ? c : nmain + c;
    if (col >= nmain + T.nsy) return false;
    const int base = main ? c * colu : mtot + c * colu;
    const int k0 = (u - base + w - 1) / w;
    if (k0 >= T.nz) {  // no plane starts in the rest of this column
      u = base + colu;
      continue;
    }
    if (base + k0 * w >= e) return false;
    const int k1 = min(T.nz, (e - base + w - 1) / w);
    out = column_seg(T, col, k0, k1);
    u = base + k1 * w;
    return true;
  }
  return false;
}
__device__ __forceinline__ int unit_bound(const TileIdx& T, int blocks, int b) {
  return static_cast<int>(n_units(T) * b / blocks);
}
__device__ __forceinline__ Seg aligned_seg(const TileIdx& T, int b) {
  const int nmain = T.ntx * T.nty;
  if (b < nmain) return column_seg(T, b, 0, T.nz);
  const int sc = (b - nmain) >> 1, h = (b - nmain) & 1, mid = T.nz / 2;
  return column_seg(T, nmain + sc, h ? mid : 0, h ? T.nz : mid);
}
template <class F>
__device__ __forceinline__ void for_segments(const TileIdx& T, int blocks, int b, F&& fn) {
  if (T.aligned) {
    fn(aligned_seg(T, b));
    return;
  }
  int u = unit_bound(T, blocks, b);
  const int e = unit_bound(T, blocks, b + 1);
  Seg sg;
  while (next_segment(T, u, e, sg)) fn(sg);
}

// The first segment for_segments hands CTA b (false when its range is empty).
__device__ __forceinline__ bool first_segment(const TileIdx& T, int blocks, int b, Seg& out) {
  if (T.aligned) {
    out = aligned_seg(T, b);
    return true;
  }
  int u = unit_bound(T, blocks, b);
  return next_segment(T, u, unit_bound(T, blocks, b + 1), out);
}

// Jacobi diagonal of Op(a, b) = a M + b K at (i, j, k) from the diagonals of
// the 1D factors: d = a (mx my) mz + b ((kx my + mx ky) mz + (mx my) kz), in
// this one rounding order everywhere (the stored D^-1 and the single-sweep
// solver's on-the-fly diagonal agree bit for bit).
struct DiagXY {
  double mm, km;  // mx my, kx my + mx ky
};
__device__ __forceinline__ DiagXY diag_xy(double mx, double kx, double my, double ky) {
  return {mx * my, fma(kx, my, mx * ky)};
}
__device__ __forceinline__ double diag_z(const DiagXY& q, double mz, double kz, double a,
                                         double b) {
  return fma(a, q.mm * mz, b * fma(q.km, mz, q.mm * kz));
}
template <int P>
__device__ __forceinline__ double diag_at(const KronGrid& g, double a, double b, int i, int j,
                                          int k) {
  constexpr int W = 2 * P + 1;
  const DiagXY q = diag_xy(g.M[0][i * W + P], g.K[0][i * W + P], g.M[1][j * W + P],
                           g.K[1][j * W + P]);
  return diag_z(q, g.M[2][k * W + P], g.K[2][k * W + P], a, b);
}

// pull a box into L2 ahead of its shared-memory load (no completion tracking)
__device__ __forceinline__ void tma_prefetch_box(const TensorMap3* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

__device__ __forceinline__ void tma_load_box(void* dst, const TensorMap3* map, int x, int y,
                                             int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Inputs of one sweep: NIN vectors, each with a TMA descriptor (or a plain
// pointer when TMA is off).
template <int NIN>
struct Inputs {
  const double* ptr[NIN];
  const TensorMap3* map[NIN];
  const TensorMap3* smap[NIN] = {};  // strip-tile boxes (sweeps over strip segments)
};

template <int P, int PL, int NIN, int NPASS, int ST, int UB>
__device__ __forceinline__ void init_smem(const KronGrid& g, KSmem<P, PL, NIN, NPASS, ST, UB>& sm,
                                          double* zb, bool tma) {
  constexpr int W = 2 * P + 1;
  const int tid = threadIdx.y * kKronTX + threadIdx.x;
  if (tma && tid == 0) {
    for (int q = 0; q < NIN; ++q)
      for (int s = 0; s < ST; ++s) mbar_init(&sm.bar[q][s], 1);
    fence_mbar_init();
  }
  for (int e = tid; e < g.n[2] * W; e += kThreads) {  // Mz, Kz rows: z-pass coefficients
    zb[e] = g.M[2][e];
    zb[g.n[2] * W + e] = g.K[2][e];
  }
  __syncthreads();
}

// Sweep one column segment, PL planes per step. For every output point
// (i, j, k) call epi(flat, i, j, k, y, v_own) where y = sum over passes of
// Op(a_q, b_q) in_q. With a prologue (Pro::kV) the x-pass runs on the tile
// v that pro(...) builds from the ring slots of the step (halo included), and
// v_own is v at the point; otherwise each pass reads its ring directly. Step
// s covers input planes k0 - P + PL s .. + PL - 1 (planes outside the grid
// arrive as zeros). The shared layout SM may hold more input rings than this
// sweep uses; seqs[q] counts the boxes ring q has delivered (mbarrier phases).
struct NoPro {
  static constexpr bool kV = false;
  template <class SM, class Sh>
  __device__ void operator()(SM&, const int*, int, int, const Seg&, Sh) {}
};

// the thread's point of a tile of shape Sh
template <class Sh>
__device__ __forceinline__ void tile_xy(int& tx, int& ty) {
  const int tid = threadIdx.y * kKronTX + threadIdx.x;
  tx = tid % Sh::TX;
  ty = tid / Sh::TX;
}
template <class Sh, int NIN>
__device__ __forceinline__ const TensorMap3* in_map(const Inputs<NIN>& in, int q) {
  return Sh::kStrip ? in.smap[q] : in.map[q];
}

template <int P, int PL, int NIN, int NPASS, bool TMA, class Sh = MainTile, class SM, class Pro,
          class Epi>
__device__ __forceinline__ void kron_tile(const KronGrid& g, const KronTerms& c,
                                          const Inputs<NIN>& in, Pro& pro, const Seg& sg,
                                          SM& sm, const double* zb, int* seqs, Epi& epi,
                                          bool primed = false) {
  using D = Dims<P, PL, Sh>;
  constexpr int W = D::W, RY = D::RY, RX = D::RX, PLANE = D::PLANE;
  static_assert(PLANE == Dims<P, PL>::PLANE, "tile shapes share the ring slots");
  int tx, ty;
  tile_xy<Sh>(tx, ty);
  const int tid = threadIdx.y * kKronTX + threadIdx.x;
  const bool leader = tid == 0;
  const int x0 = sg.x0, y0 = sg.y0, k0 = sg.k0, k1 = sg.k1;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int i = x0 + tx, j = y0 + ty;
  const int kfirst = k0 - P;
  const int nsteps = (k1 - k0 + 2 * P + PL - 1) / PL;
  constexpr uint32_t kBoxBytes = PL * PLANE * 8;

  __syncthreads();  // the previous segment's readers of the ring are done
  if (TMA && leader && !primed) {  // (primed: prime_ring already issued these boxes)
    for (int s = 0; s < SM::kSt && s < nsteps; ++s)
      for (int q = 0; q < NIN; ++q) {
        const int slot = (seqs[q] + s) % SM::kSt;
        mbar_arrive_expect_tx(&sm.bar[q][slot], kBoxBytes);
        tma_load_box(sm.ring[q][slot], in_map<Sh>(in, q), x0 - P, y0 - P, kfirst + PL * s,
                     &sm.bar[q][slot]);
      }
    for (int s = SM::kSt; s < SM::kSt + kL2Ahead && s < nsteps; ++s)
      for (int q = 0; q < NIN; ++q)
        tma_prefetch_box(in_map<Sh>(in, q), x0 - P, y0 - P, kfirst + PL * s);
  }

  // this thread's x and y rows of the 1D factors, in registers (the sweep is
  // shared-memory-bandwidth bound: coefficients must not come from smem);
  // loaded after the ring is primed so their latency overlaps the first boxes
  double mx[W], kx[W], my[W], ky[W];
#pragma unroll
  for (int d = 0; d < W; ++d) {
    mx[d] = i < nx ? g.M[0][i * W + d] : 0.0;
    kx[d] = i < nx ? g.K[0][i * W + d] : 0.0;
    my[d] = j < ny ? g.M[1][j * W + d] : 0.0;
    ky[d] = j < ny ? g.K[1][j * W + d] : 0.0;
  }

  double win1[W], win2[W], pown[W];
#pragma unroll
  for (int d = 0; d < W; ++d) win1[d] = win2[d] = pown[d] = 0.0;
  const size_t plane = static_cast<size_t>(nx) * ny;

  static_assert(SM::kUb == 2 || Pro::kV, "a single x-pass buffer needs a prologue barrier");
  for (int s = 0; s < nsteps; ++s) {
    const int kin0 = kfirst + PL * s;
    const int ub = SM::kUb == 1 ? 0 : (s & 1);
    int slot[NIN];
#pragma unroll
    for (int q = 0; q < NIN; ++q) {
      const int qn = seqs[q] + s;
      slot[q] = TMA ? qn % SM::kSt : 0;
      if (TMA) mbar_wait(&sm.bar[q][slot[q]], static_cast<uint32_t>((qn / SM::kSt) & 1));
    }
    if constexpr (!TMA) {
      for (int q = 0; q < NIN; ++q)
        for (int l = 0; l < PL; ++l) {
          const int kin = kin0 + l;
          for (int e = tid; e < PLANE; e += kThreads) {
            const int gi = x0 + e % RX - P, gj = y0 + e / RX - P;
            double val = 0.0;
            if (gi >= 0 && gi < nx && gj >= 0 && gj < ny && kin >= 0 && kin < nz)
              val = in.ptr[q][static_cast<size_t>(kin) * plane + static_cast<size_t>(gj) * nx + gi];
            sm.ring[q][0][l * PLANE + e] = val;
          }
        }
      __syncthreads();
    }
    // refill the ring slots just consumed; the barrier before the issue
    // orders every generic-proxy read of the slot before the TMA write
    auto refill = [&] {
      if (TMA && leader && s + SM::kSt < nsteps)
        for (int q = 0; q < NIN; ++q) {
          mbar_arrive_expect_tx(&sm.bar[q][slot[q]], kBoxBytes);
          tma_load_box(sm.ring[q][slot[q]], in_map<Sh>(in, q), x0 - P, y0 - P,
                       kfirst + PL * (s + SM::kSt), &sm.bar[q][slot[q]]);
          if (s + SM::kSt + kL2Ahead < nsteps)
            tma_prefetch_box(in_map<Sh>(in, q), x0 - P, y0 - P,
                             kfirst + PL * (s + SM::kSt + kL2Ahead));
        }
    };
    double po[PL];
    if constexpr (Pro::kV) {  // v over the halo'd tiles (and the prologue's own-point work)
      pro(sm, slot, s, kin0, sg, Sh{});
      __syncthreads();
      refill();  // the ring is only read by the prologue
#pragma unroll
      for (int l = 0; l < PL; ++l) po[l] = sm.v[l][(ty + P) * RX + tx + P];
    }
    // x-pass on the tile rows plus the y halo, PL planes
#pragma unroll
    for (int q = 0; q < NPASS; ++q)
      // (plane, row) pairs dealt round-robin to the 8 warps: equal shares
      for (int lr = ty; lr < PL * RY; lr += Sh::TY) {
        const int l = lr / RY, r = lr - l * RY;
        const double* src = Pro::kV ? sm.v[l] : sm.ring[q][slot[q < NIN ? q : 0]] + l * PLANE;
        {
          double a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int d = 0; d < W; ++d) {
            const double vv = src[r * RX + tx + d];
            a1 = fma(mx[d], vv, a1);
            a2 = fma(kx[d], vv, a2);
          }
          sm.u1[q][ub][l][r * Sh::TX + tx] = a1;
          sm.u2[q][ub][l][r * Sh::TX + tx] = a2;
        }
      }
    __syncthreads();
    if constexpr (!Pro::kV) refill();
    // y-pass, then the PL planes enter the z window one by one
#pragma unroll
    for (int l = 0; l < PL; ++l) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int q = 0; q < NPASS; ++q) {
        double w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
          const double p1 = sm.u1[q][ub][l][(ty + d) * Sh::TX + tx];
          w1 = fma(my[d], p1, w1);
          w2 = fma(my[d], sm.u2[q][ub][l][(ty + d) * Sh::TX + tx], w2);
          w3 = fma(ky[d], p1, w3);
        }
        const double a = q == 0 ? c.a1 : c.a2, b = q == 0 ? c.b1 : c.b2;
        s1 = fma(a, w1, fma(b, w2 + w3, s1));
        s2 = fma(b, w1, s2);
      }
#pragma unroll
      for (int d = 0; d < W - 1; ++d) {
        win1[d] = win1[d + 1];
        win2[d] = win2[d + 1];
        pown[d] = pown[d + 1];
      }
      win1[W - 1] = s1;
      win2[W - 1] = s2;
      pown[W - 1] = Pro::kV ? po[l] : 0.0;
      const int k = kin0 + l - P;
      if (k >= k0 && k < k1 && i < nx && j < ny) {
        const double* mz = zb + k * W;
        const double* kz = zb + nz * W + k * W;
        double y = 0.0;
#pragma unroll
        for (int d = 0; d < W; ++d) y = fma(mz[d], win1[d], fma(kz[d], win2[d], y));
        epi(static_cast<size_t>(k) * plane + static_cast<size_t>(j) * nx + i, i, j, k, y,
            pown[P]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NIN; ++q) seqs[q] += nsteps;
}

// kron_tile on a segment of either tile shape (sweeps whose TileIdx may hold
// a strip)
template <int P, int PL, int NIN, int NPASS, bool TMA, class SM, class Pro, class Epi>
__device__ __forceinline__ void kron_seg(const KronGrid& g, const KronTerms& c,
                                         const Inputs<NIN>& in, Pro& pro, const Seg& sg, SM& sm,
                                         const double* zb, int* seqs, Epi& epi,
                                         bool primed = false) {
  if (sg.strip)
    kron_tile<P, PL, NIN, NPASS, TMA, StripTile>(g, c, in, pro, sg, sm, zb, seqs, epi, primed);
  else
    kron_tile<P, PL, NIN, NPASS, TMA, MainTile>(g, c, in, pro, sg, sm, zb, seqs, epi, primed);
}

// ---------------------------------------------------------------------------
// stand-alone applies (plain loads)

struct EpiStore {
  double* y;
  __device__ void operator()(size_t idx, int, int, int, double v, double) { y[idx] = v; }
};

struct ApplyMap {
  TensorMap3 v;
};

template <int P, bool TMA>
__global__ void __launch_bounds__(kThreads) k2_apply_kernel(KronGrid g, KronTerms c,
                                                            const double* v, double* y,
                                                            TileIdx T,
                                                            const __grid_constant__ ApplyMap m) {
  constexpr int PL = TMA ? kTmaPlanes : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<KSmem<P, PL, 1, 1>*>(smem_raw);
  double* zb = reinterpret_cast<double*>(smem_raw + zband_offset<P, PL, 1, 1>());
  init_smem(g, sm, zb, TMA);
  EpiStore epi{y};
  Inputs<1> in{{v}, {&m.v}};
  int seq[1] = {0};
  NoPro np;
  for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
    kron_tile<P, PL, 1, 1, TMA>(g, c, in, np, sg, sm, zb, seq, epi);
  });
}

struct EpiRhs {
  RhsArgs a;
  int nfree[3];
  __device__ void operator()(size_t idx, int i, int j, int k, double y, double) {
    int ijk[3] = {i, j, k};
    if (ijk[a.bottom_axis] == a.bottom_layer) return;
    if (a.bottom_layer == 0) ijk[a.bottom_axis] -= 1;
    const size_t f = static_cast<size_t>(ijk[0]) +
                     static_cast<size_t>(nfree[0]) * (ijk[1] + static_cast<size_t>(nfree[1]) * ijk[2]);
    a.rhs[f] = y + a.theta * a.F_np1[idx] + (1.0 - a.theta) * a.F_n[idx];
  }
};

struct RhsMaps {
  TensorMap3 T, g;
};

template <int P, bool TMA>
__global__ void __launch_bounds__(kThreads) k2_rhs_kernel(KronGrid g, KronTerms c, RhsArgs args,
                                                          TileIdx T,
                                                          const __grid_constant__ RhsMaps maps) {
  constexpr int PL = TMA ? kTmaPlanes : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<KSmem<P, PL, 2, 2>*>(smem_raw);
  double* zb = reinterpret_cast<double*>(smem_raw + zband_offset<P, PL, 2, 2>());
  init_smem(g, sm, zb, TMA);
  EpiRhs epi{args, {g.n[0], g.n[1], g.n[2]}};
  epi.nfree[args.bottom_axis] -= 1;
  Inputs<2> in{{args.T_full, args.g_full}, {&maps.T, &maps.g}};
  int seq[2] = {0, 0};
  NoPro np;
  for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
    kron_tile<P, PL, 2, 2, TMA>(g, c, in, np, sg, sm, zb, seq, epi);
  });
}

template <int P>
__global__ void k2_inv_diag_kernel(KronGrid g, double a, double b, double* inv,
                                   PcgStatus* st) {
  const size_t n = static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2];
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(f % g.n[0]);
    const int j = static_cast<int>((f / g.n[0]) % g.n[1]);
    const int k = static_cast<int>(f / (static_cast<size_t>(g.n[0]) * g.n[1]));
    const double d = diag_at<P>(g, a, b, i, j, k);
    if (!(d > 0.0)) st->status = 2;  // sparse.cpp:50
    inv[f] = 1.0 / d;
  }
}

// ---------------------------------------------------------------------------
// persistent Jacobi-PCG

// Issue the first ring boxes kron_tile would issue for segment sg (one thread).
template <int P, int PL, int NIN, class SM>
__device__ __forceinline__ void prime_ring(const Inputs<NIN>& in, const Seg& sg, SM& sm,
                                           const int* seqs) {
  constexpr uint32_t kBoxBytes = PL * Dims<P, PL>::PLANE * 8;
  const int nsteps = (sg.k1 - sg.k0 + 2 * P + PL - 1) / PL;
  for (int s = 0; s < SM::kSt && s < nsteps; ++s)
    for (int q = 0; q < NIN; ++q) {
      const int slot = (seqs[q] + s) % SM::kSt;
      mbar_arrive_expect_tx(&sm.bar[q][slot], kBoxBytes);
      tma_load_box(sm.ring[q][slot], sg.strip ? in.smap[q] : in.map[q], sg.x0 - P, sg.y0 - P,
                   sg.k0 - P + PL * s, &sm.bar[q][slot]);
    }
}

// Wait for primed boxes nobody will consume (the solve ended after priming),
// so no bulk copy into this CTA's shared memory is in flight at exit.
template <int P, int PL, int NIN, class SM>
__device__ __forceinline__ void drain_ring(const Seg& sg, SM& sm, const int* seqs) {
  const int nsteps = (sg.k1 - sg.k0 + 2 * P + PL - 1) / PL;
  for (int s = 0; s < SM::kSt && s < nsteps; ++s)
    for (int q = 0; q < NIN; ++q) {
      const int qn = seqs[q] + s;
      mbar_wait(&sm.bar[q][qn % SM::kSt], static_cast<uint32_t>((qn / SM::kSt) & 1));
    }
}

struct NoAfterSync {
  __device__ void operator()() const {}
};

// Block-reduce acc (fixed tree), store to partials[buf][block][4], grid sync,
// then every CTA sums the per-block partials in the same fixed order.
template <class AfterSync = NoAfterSync>
__device__ __forceinline__ void grid_reduce(cg::grid_group& grid, const double (&acc)[4],
                                            double* partials, int& buf, double* red,
                                            double (&out)[4], AfterSync after = {}) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp * 4 + c] = v;
  }
  __syncthreads();
  double* pb = partials + static_cast<size_t>(buf) * 4 * gridDim.x;
  if (tid < 4) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w * 4 + tid];
    pb[blockIdx.x * 4 + tid] = s;
  }
  grid.sync();
  if (warp == 1 && lane == 0) after();  // e.g. prime the next sweep's TMA ring
  if (warp == 0) {
double s[4];
    warp_sum_partials(pb, static_cast<int>(gridDim.x), lane, s);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 4; ++c) red[32 + c] = s[c];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = red[32 + c];
  __syncthreads();
  buf ^= 1;
}

struct EpiResidual {  // r = b - A x; z = D^-1 r; p_old = 0; rr, bb, rz
  const double* rhs;
  const double* inv;
  double* r;
  double* z;
  double* p_old;
  double acc[4];
  __device__ void operator()(size_t idx, int, int, int, double y, double) {
    const double bi = rhs[idx];
    const double ri = bi - y;
    const double zi = inv[idx] * ri;
    r[idx] = ri;
    z[idx] = zi;
    p_old[idx] = 0.0;
    acc[0] += ri * ri;
    acc[1] += bi * bi;
    acc[2] += ri * zi;
  }
};

struct ProCombine {  // v = z + beta p_old over the halo'd tiles (ring 0: z, ring 1: p_old)
  static constexpr bool kV = true;
  double beta;
  template <class SM, class Sh>
  __device__ void operator()(SM& sm, const int* slot, int, int, const Seg&, Sh) {
    static_assert(!Sh::kStrip, "main tiles only");
    constexpr int N = sizeof(sm.v) / sizeof(double);
    for (int e = threadIdx.y * kKronTX + threadIdx.x; e < N; e += kThreads)
      (&sm.v[0][0])[e] = fma(beta, sm.ring[1][slot[1]][e], sm.ring[0][slot[0]][e]);
  }
};

struct EpiDirection {  // p_new (own point), Ap, p.Ap
  double* p_new;
  double* Ap;
  double acc[4];
  __device__ void operator()(size_t idx, int, int, int, double y, double p) {
    p_new[idx] = p;
    Ap[idx] = y;
    acc[0] += p * y;
  }
};

template <int P, bool TMA>
__global__ void __launch_bounds__(kThreads, K2_MINB)
    k2_pcg_kernel(KronGrid g, double a, double b, const double* rhs, double* x, PcgWork w,
                  double tol, int max_iter, TileIdx T, const __grid_constant__ PcgMaps maps) {
  constexpr int PL = TMA ? kTmaPlanes : 1;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<KSmem<P, PL, 2, 1>*>(smem_raw);
  double* zb = reinterpret_cast<double*>(smem_raw + zband_offset<P, PL, 2, 1>());
  __shared__ double red[64];
  init_smem(g, sm, zb, TMA);
  const KronTerms c{a, b, 0.0, 0.0};
  const int nx = g.n[0], ny = g.n[1];
  int buf = 0;
  int seq[2] = {0, 0};
  double tot[4];

  // r = b - A x, z = D^-1 r (sparse.cpp:61-69); the first direction update
  // sees p_old = 0, i.e. p = z
  {
    EpiResidual e0{rhs, w.inv_diag, w.r, w.z, w.pA, {0, 0, 0, 0}};
    Inputs<1> in1{{x}, {&maps.x}};  // ring 0 of the two-ring layout
    NoPro np;
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 1, 1, TMA>(g, c, in1, np, sg, sm, zb, seq, e0);
    });
    grid_reduce(grid, e0.acc, w.partials, buf, red, tot);
  }
  double rr = tot[0], rz = tot[2];
  const double bnorm = sqrt(tot[1]);
  if (bnorm == 0.0) {  // sparse.cpp:57-60: zero rhs resets even a warm start
    const size_t n = static_cast<size_t>(nx) * ny * g.n[2];
    for (size_t f = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.y * kKronTX + threadIdx.x;
         f < n; f += static_cast<size_t>(gridDim.x) * kThreads)
      x[f] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0)
      *w.status = PcgStatus{0, 0, 0.0, 0.0};
    return;
  }
  double rel = 0.0, beta = 0.0;
  int it = 0, status = 3;
  double* p_old = w.pA;
  double* p_new = w.pB;
  const TensorMap3* m_old = &maps.pA;
  const TensorMap3* m_new = &maps.pB;
  for (it = 0; it < max_iter; ++it) {
    rel = sqrt(rr) / bnorm;
    if (rel <= tol) {
      status = 0;
      break;
    }
    // optional phase trace of CTA 0 (tools/k2_trace.py)
    const bool tr = w.trace && it < 16 && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0;
    auto stamp = [&](int k) {
      if (tr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        w.trace[it * 5 + k] = t;
      }
    };
    stamp(0);
    // A': p_new = z + beta p_old (sparse.cpp:96), Ap = A p_new (sparse.cpp:81)
    EpiDirection e1{p_new, w.Ap, {0, 0, 0, 0}};
    Inputs<2> in{{w.z, p_old}, {&maps.z, m_old}};
    ProCombine pc{beta};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 2, 1, TMA>(g, c, in, pc, sg, sm, zb, seq, e1);
    });
    stamp(1);
    grid_reduce(grid, e1.acc, w.partials, buf, red, tot);
    stamp(2);
    const double pAp = tot[0];
    if (!(pAp > 0.0)) {
      status = 4;
      break;
    }
    const double alpha = rz / pAp;
    // B: x, r, z updates and the two dot products (sparse.cpp:85-94), on the
    // same segment map; rows of 32 consecutive points per warp, U planes of
    // loads in flight per thread
    double acc[4] = {0, 0, 0, 0};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      const int i = sg.x0 + threadIdx.x;
      const int j = sg.y0 + threadIdx.y;
      if (i >= nx || j >= ny) return;
      constexpr int U = 4;
      const size_t pl = static_cast<size_t>(nx) * ny;
      const size_t f0 = (static_cast<size_t>(sg.k0) * ny + j) * nx + i;
      double* __restrict__ xr = x;
      double* __restrict__ rr_ = w.r;
      double* __restrict__ zr = w.z;
      const double* __restrict__ pr = p_new;
      const double* __restrict__ apr = w.Ap;
      const double* __restrict__ ir = w.inv_diag;
      for (int k = sg.k0; k < sg.k1; k += U) {
        double xv[U], pv[U], rv[U], av[U], iv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k + u < sg.k1) {
            const size_t f = f0 + (k - sg.k0 + u) * pl;
            xv[u] = xr[f];
            pv[u] = pr[f];
            rv[u] = rr_[f];
            av[u] = apr[f];
            iv[u] = ir[f];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k + u < sg.k1) {
            const size_t f = f0 + (k - sg.k0 + u) * pl;
            xr[f] = xv[u] + alpha * pv[u];
            const double ri = rv[u] - alpha * av[u];
            const double zi = iv[u] * ri;
            rr_[f] = ri;
            zr[f] = zi;
            acc[0] += ri * zi;
            acc[1] += ri * ri;
          }
        }
      }
    });
    stamp(3);
    grid_reduce(grid, acc, w.partials, buf, red, tot);
    stamp(4);
    beta = tot[0] / rz;
    rz = tot[0];
    rr = tot[1];
    double* tp = p_old;
    p_old = p_new;
    p_new = tp;
    const TensorMap3* tm = m_old;
    m_old = m_new;
    m_new = tm;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *w.status = PcgStatus{it, status, rel, bnorm};
}

// ---------------------------------------------------------------------------
// single-sweep Jacobi-PCG (Chronopoulos-Gear recurrences)
//
// Same Krylov iterates as the reference's PCG in exact arithmetic, with the
// two dot-product phases merged: carrying w = A u and s = A p as vectors,
//   p_i = u_i + b_i p_{i-1}     s_i = w_i + b_i s_{i-1}
//   x  += a_i p_i               r_{i+1} = r_i - a_i s_i,  u_{i+1} = D^-1 r_{i+1}
//   w_{i+1} = A u_{i+1};  g = r.u, d = w.u, rr = r.r (one grid reduction)
//   b_{i+1} = g_{i+1} / g_i,  a_{i+1} = g_{i+1} / (d_{i+1} - b_{i+1} g_{i+1} / a_i)
// (the denominator is p.Ap; <= 0 is the reference's indefinite-direction
// failure). One tile sweep per iteration: the prologue forms s, r and u on the
// halo'd TMA tiles of r, w, s_old and D^-1 (the stencil input u = D^-1 r_new),
// updates p and x on the segment's own points, and the epilogue writes
// w = A u. Vectors whose halos are read (r, w, s) ping-pong between two
// buffers; x and p are point-local and update in place. HBM traffic: 6 reads
// + 5 writes = 88 B per DOF per iteration, one grid barrier (80 B in the
// scaled form below, the default: 89.6 against 92.6 us/iteration on config 4).

#ifndef K2_CG1_STAGES
#define K2_CG1_STAGES 2
#endif
// measured (config 4): 2 stages 89.6 us/iter; 3 (still 2 CTAs/SM in the scaled form) 90.4
constexpr int kCg1Stages = K2_CG1_STAGES;
#ifndef K2_CG1_SCALED
#define K2_CG1_SCALED 1
#endif
// Scaled form (default): carry u = D^-1 r, w^ = D^-1 A u and s^ = D^-1 A p
// instead of r, w, s. The recurrences keep their shape (s^ = w^ + beta s^,
// u -= alpha s^), the halo'd prologue needs no D^-1, and the dot products
// take d at the segment's own points (r.u = sum d u^2, r.r = sum (d u)^2,
// w.u = (A u).u), so D^-1 leaves the rings: 3 halo'd inputs, 80 B/DOF.
constexpr int kCg1Nin = K2_CG1_SCALED ? 3 : 4;
#ifndef K2_CG1_UB
#define K2_CG1_UB 1
#endif
#ifndef K2_DEFER_X
#define K2_DEFER_X 1  // x read / written every second sweep (bit-identical iterates)
#endif
#ifndef K2_STUDY_NOSWEEP
#define K2_STUDY_NOSWEEP 0
#endif
constexpr int kCg1Ub = K2_CG1_SCALED ? K2_CG1_UB : 2;  // every scaled sweep has a prologue

template <int P, int PL>
struct ProScale {  // init: v = D^-1 r0 (ring 0: r0, ring 1: D^-1); gamma0 on own points
  static constexpr bool kV = true;
  int nx, ny;
  double gamma;
  template <class SM, class Sh>
  __device__ void operator()(SM& sm, const int* slot, int, int kin0, const Seg& sg, Sh) {
    static_assert(!Sh::kStrip, "main tiles only");
    using D = Dims<P, PL>;
    constexpr int N = PL * D::PLANE;
    const double* rr = sm.ring[0][slot[0]];
    const double* dd = sm.ring[1][slot[1]];
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int e = ty * kKronTX + tx; e < N; e += kThreads) (&sm.v[0][0])[e] = dd[e] * rr[e];
    if (sg.x0 + tx < nx && sg.y0 + ty < ny) {
#pragma unroll
      for (int l = 0; l < PL; ++l) {
        const int kin = kin0 + l;
        if (kin >= sg.k0 && kin < sg.k1) {
          const int e = l * D::PLANE + (ty + P) * D::RX + tx + P;
          gamma += rr[e] * (dd[e] * rr[e]);
        }
      }
    }
  }
};

// Point-local inputs of the C-G sweep (x, p_{i-1}): un-halo'd 32 x 8 x PL
// TMA boxes through their own 2-slot ring, placed after the z band.
template <int PL>
struct CentreRing {
  static constexpr int kBox = PL * kKronTY * kKronTX;  // doubles per box
  double buf[2][2][kBox];                               // [vector][slot]
  uint64_t bar[2][2];
};

template <int P, int PL>
struct ProCg1 {  // rings: 0 r_i, 1 w_i, 2 s_{i-1}, 3 D^-1; centre ring: x, p_{i-1}
  static constexpr bool kV = true;
  double alpha, beta;
  double* x;
  double* p;
  double* r_out;
  double* s_out;
  int nx, ny;
  CentreRing<PL>* cr;
  const TensorMap3* mx;
  const TensorMap3* mp;
  int* cseq;  // boxes the centre ring has delivered (persists across sweeps)
  double gamma, rr;

  __device__ void issue(const Seg& sg, int step) const {
    const int q = *cseq + step, slot = q & 1;
    constexpr uint32_t bytes = CentreRing<PL>::kBox * 8;
    const int kin0 = sg.k0 - P + PL * step;
    mbar_arrive_expect_tx(&cr->bar[0][slot], bytes);
    tma_load_box(cr->buf[0][slot], mx, sg.x0, sg.y0, kin0, &cr->bar[0][slot]);
    mbar_arrive_expect_tx(&cr->bar[1][slot], bytes);
    tma_load_box(cr->buf[1][slot], mp, sg.x0, sg.y0, kin0, &cr->bar[1][slot]);
  }
  template <class SM, class Sh>
  __device__ void operator()(SM& sm, const int* slot, int s, int kin0, const Seg& sg, Sh) {
    static_assert(!Sh::kStrip, "main tiles only");
    using D = Dims<P, PL>;
    constexpr int N = PL * D::PLANE;
    const int nsteps = (sg.k1 - sg.k0 + 2 * P + PL - 1) / PL;
    const int tx = threadIdx.x, ty = threadIdx.y;
    // the slot of step s + 1 was last read in step s - 1 (a barrier ago)
    if (tx == 0 && ty == 0) {
      if (s == 0) {
        issue(sg, 0);
        for (int a = 2; a < 2 + kL2Ahead && a < nsteps; ++a) {
          tma_prefetch_box(mx, sg.x0, sg.y0, sg.k0 - P + PL * a);
          tma_prefetch_box(mp, sg.x0, sg.y0, sg.k0 - P + PL * a);
        }
      }
      if (s + 1 < nsteps) issue(sg, s + 1);
      if (s + 2 + kL2Ahead < nsteps) {
        tma_prefetch_box(mx, sg.x0, sg.y0, sg.k0 - P + PL * (s + 2 + kL2Ahead));
        tma_prefetch_box(mp, sg.x0, sg.y0, sg.k0 - P + PL * (s + 2 + kL2Ahead));
      }
    }
    const int q = *cseq + s, cs = q & 1;
    const uint32_t par = static_cast<uint32_t>((q >> 1) & 1);
    mbar_wait(&cr->bar[0][cs], par);
    mbar_wait(&cr->bar[1][cs], par);
    if (s + 1 == nsteps) *cseq += nsteps;
    const double* r_ = sm.ring[0][slot[0]];
    const double* w_ = sm.ring[1][slot[1]];
    const double* s_ = sm.ring[2][slot[2]];
    const double* d_ = sm.ring[3][slot[3]];
    const int i = sg.x0 + tx, j = sg.y0 + ty;
    if (i < nx && j < ny) {
#pragma unroll
      for (int l = 0; l < PL; ++l) {
        const int kin = kin0 + l;
        if (kin >= sg.k0 && kin < sg.k1) {
          const int e = l * D::PLANE + (ty + P) * D::RX + tx + P;
          const int c = (l * kKronTY + ty) * kKronTX + tx;
          const size_t f = (static_cast<size_t>(kin) * ny + j) * nx + i;
          const double ro = r_[e], dv = d_[e];
          const double pnew = fma(beta, cr->buf[1][cs][c], dv * ro);  // p_i = u_i + beta p_{i-1}
          p[f] = pnew;
          x[f] = fma(alpha, pnew, cr->buf[0][cs][c]);                 // x_{i+1}
          const double snew = fma(beta, s_[e], w_[e]);  // s_i = w_i + beta s_{i-1}
          const double rnew = fma(-alpha, snew, ro);    // r_{i+1}
          s_out[f] = snew;
          r_out[f] = rnew;
          gamma += rnew * (dv * rnew);
          rr += rnew * rnew;
        }
      }
    }
    for (int e = ty * kKronTX + tx; e < N; e += kThreads)  // u_{i+1}, halo included
      (&sm.v[0][0])[e] = d_[e] * fma(-alpha, fma(beta, s_[e], w_[e]), r_[e]);
  }
};

struct EpiCg1 {  // w = A u and w.u
  double* w_out;
  double delta;
  __device__ void operator()(size_t idx, int, int, int, double y, double u) {
    w_out[idx] = y;
    delta += y * u;
  }
};

struct EpiCg1Init {  // r0 = b - A x0, s_{-1} = p_{-1} = 0; r.r, b.b
  const double* rhs;
  double* r;
  double* s;
  double* p;
  double acc[4];
  __device__ void operator()(size_t idx, int, int, int, double y, double) {
    const double bi = rhs[idx];
    const double ri = bi - y;
    r[idx] = ri;
    s[idx] = 0.0;
    p[idx] = 0.0;
    acc[0] += ri * ri;
    acc[1] += bi * bi;
  }
};

// --- scaled form (K2_CG1_SCALED) ---
// own-point diagonal: the thread's x/y factor diagonals are fixed per
// segment, the z ones come from the shared z band
template <int P>
struct OwnDiag {
  DiagXY q;
  const double* zb;
  int nz;
  __device__ void set(const KronGrid& g, int i, int j) {
    constexpr int W = 2 * P + 1;
    q = diag_xy(g.M[0][i * W + P], g.K[0][i * W + P], g.M[1][j * W + P], g.K[1][j * W + P]);
  }
  __device__ double at(int k, double a, double b) const {
    constexpr int W = 2 * P + 1;
    return diag_z(q, zb[k * W + P], zb[nz * W + k * W + P], a, b);
  }
};

template <int P, int PL>
struct ProCopy {  // init: v = u0 (ring 0), so the epilogue sees u0 at its point
  static constexpr bool kV = true;
  const KronGrid* g;
  int nx, ny;
  OwnDiag<P> od;
  template <class SM, class Sh>
  __device__ void operator()(SM& sm, const int* slot, int s, int, const Seg& sg, Sh) {
    constexpr int N = PL * Dims<P, PL>::PLANE;
    int tx, ty;
    tile_xy<Sh>(tx, ty);
    const int i = sg.x0 + tx, j = sg.y0 + ty;
    if (s == 0 && i < nx && j < ny) od.set(*g, i, j);
    const double* uu = sm.ring[0][slot[0]];
    for (int e = threadIdx.y * kKronTX + threadIdx.x; e < N; e += kThreads)
      (&sm.v[0][0])[e] = uu[e];
  }
};

template <int P, int PL>
struct ProCg1S {  // rings: 0 u_i, 1 w^_i, 2 s^_{i-1}; centre ring: x, p_{i-1}
  static constexpr bool kV = true;
  double alpha, beta;
  double* x;
  double* p;
  double* u_out;
  double* s_out;
  int nx, ny;
  CentreRing<PL>* cr;
  const TensorMap3* mx;
  const TensorMap3* mp;
  int* cseq;
  const KronGrid* g;
  double a, b;
  OwnDiag<P> od;
  double gamma, rr;
  int zo0 = -(1 << 30), zo1 = 1 << 30;  // planes whose points enter the dot products
  // x update: 0 every sweep (x += alpha p_i); deferred (the single solve):
  // 1 = this sweep leaves x alone (no x traffic), 2 = x += alpha_prev p_{i-1}
  // + alpha p_i (the same two fma roundings as two sweeps of mode 0)
  int xmode = 0;
  double alpha_prev = 0.0;
  const TensorMap3* smx = nullptr;  // strip-tile boxes of x and p
  const TensorMap3* smp = nullptr;

  template <class Sh>
  __device__ void issue(const Seg& sg, int step) const {
    const int q = *cseq + step, slot = q & 1;
    constexpr uint32_t bytes = CentreRing<PL>::kBox * 8;
    const int kin0 = sg.k0 - P + PL * step;
    if (xmode == 1) {
      mbar_arrive(&cr->bar[0][slot]);  // completes the slot's phase without a copy
    } else {
      mbar_arrive_expect_tx(&cr->bar[0][slot], bytes);
      tma_load_box(cr->buf[0][slot], Sh::kStrip ? smx : mx, sg.x0, sg.y0, kin0,
                   &cr->bar[0][slot]);
    }
    mbar_arrive_expect_tx(&cr->bar[1][slot], bytes);
    tma_load_box(cr->buf[1][slot], Sh::kStrip ? smp : mp, sg.x0, sg.y0, kin0, &cr->bar[1][slot]);
  }
  template <class SM, class Sh>
  __device__ void operator()(SM& sm, const int* slot, int s, int kin0, const Seg& sg, Sh) {
    using D = Dims<P, PL, Sh>;
    constexpr int N = PL * D::PLANE;
    const int nsteps = (sg.k1 - sg.k0 + 2 * P + PL - 1) / PL;
    int tx, ty;
    tile_xy<Sh>(tx, ty);
    const int i = sg.x0 + tx, j = sg.y0 + ty;
    const bool own = i < nx && j < ny;
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      if (s == 0) issue<Sh>(sg, 0);
      if (s + 1 < nsteps) issue<Sh>(sg, s + 1);
    }
    if (s == 0 && own) od.set(*g, i, j);
    const int q = *cseq + s, cs = q & 1;
    const uint32_t par = static_cast<uint32_t>((q >> 1) & 1);
    if (xmode != 1) mbar_wait(&cr->bar[0][cs], par);
    mbar_wait(&cr->bar[1][cs], par);
    if (s + 1 == nsteps) *cseq += nsteps;
    const double* u_ = sm.ring[0][slot[0]];
    const double* w_ = sm.ring[1][slot[1]];
    const double* s_ = sm.ring[2][slot[2]];
    if (own) {
#pragma unroll
      for (int l = 0; l < PL; ++l) {
        const int kin = kin0 + l;
        if (kin >= sg.k0 && kin < sg.k1) {
          const int e = l * D::PLANE + (ty + P) * D::RX + tx + P;
          const int c = (l * Sh::TY + ty) * Sh::TX + tx;
          const size_t f = (static_cast<size_t>(kin) * ny + j) * nx + i;
          const double uo = u_[e], pold = cr->buf[1][cs][c];
          const double pnew = fma(beta, pold, uo);                 // p_i = u_i + beta p_{i-1}
          p[f] = pnew;
          if (xmode == 0)
            x[f] = fma(alpha, pnew, cr->buf[0][cs][c]);            // x_{i+1}
          else if (xmode == 2)
            x[f] = fma(alpha, pnew, fma(alpha_prev, pold, cr->buf[0][cs][c]));
          const double snew = fma(beta, s_[e], w_[e]);             // s^_i = w^_i + beta s^_{i-1}
          const double unew = fma(-alpha, snew, uo);               // u_{i+1}
          s_out[f] = snew;
          u_out[f] = unew;
          if (kin >= zo0 && kin < zo1) {
            const double ru = od.at(kin, a, b) * unew;             // r_{i+1} = D u_{i+1}
            gamma = fma(ru, unew, gamma);
            rr = fma(ru, ru, rr);
          }
        }
      }
    }
    for (int e = threadIdx.y * kKronTX + threadIdx.x; e < N; e += kThreads)  // u_{i+1}, halo included
      (&sm.v[0][0])[e] = fma(-alpha, fma(beta, s_[e], w_[e]), u_[e]);
  }
};

// 1/d to within an ulp without the IEEE-division slow path (d is a positive
// normal number): hardware estimate, two Newton steps
__device__ __forceinline__ double recip(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

template <int P, class Own>
struct EpiCg1S {  // w^ = D^-1 (A u), delta = (A u).u; own diagonal from the prologue
  double* w_out;
  const Own* own;
  double a, b;
  double delta;
  int zo0 = -(1 << 30), zo1 = 1 << 30;
  __device__ void operator()(size_t idx, int, int, int k, double y, double u) {
    w_out[idx] = y * recip(own->od.at(k, a, b));
    if (k >= zo0 && k < zo1) delta = fma(y, u, delta);
  }
};

template <int P>
struct EpiCg1InitS {  // r0 = b - A x0; u0 = D^-1 r0; s^_{-1} = p_{-1} = 0; r.r, b.b, r.u
  const double* rhs;
  double* u;
  double* s;
  double* p;
  const KronGrid* g;
  double a, b;
  OwnDiag<P> od;
  int ci, cj;
  double acc[4];
  int zo0 = -(1 << 30), zo1 = 1 << 30;
  __device__ void operator()(size_t idx, int i, int j, int k, double y, double) {
    if (i != ci || j != cj) {
      od.set(*g, i, j);
      ci = i;
      cj = j;
    }
    const double bi = rhs[idx];
    const double ri = bi - y;
    const double ui = ri * recip(od.at(k, a, b));
    u[idx] = ui;
    s[idx] = 0.0;
    p[idx] = 0.0;
    if (k >= zo0 && k < zo1) {
      acc[0] += ri * ri;
      acc[1] += bi * bi;
      acc[2] += ri * ui;
    }
  }
};

template <int P, int PL>
__host__ __device__ constexpr size_t cg1_centre_offset(int nz) {
  return (zband_offset<P, PL, kCg1Nin, 1, kCg1Stages, kCg1Ub>() +
          2 * static_cast<size_t>(nz) * (2 * P + 1) * 8 +
          127) / 128 * 128;
}
template <int P, int PL>
size_t cg1_smem_bytes(int nz) {
  return cg1_centre_offset<P, PL>(nz) + sizeof(CentreRing<PL>);
}

// PL planes per sweep step (TMA box depth): 2 for large grids (2 CTAs/SM), 4
// for grids too small to fill the GPU at 2 CTAs/SM (1 CTA/SM, half the steps
// per segment: the per-iteration time there is pipeline latency, not bytes)
template <int P, int PL>
__global__ void __launch_bounds__(kThreads, K2_MINB)
    k2_cg1_kernel(KronGrid g, double a, double b, const double* rhs, double* x, Cg1Work w,
                  double tol, int max_iter, TileIdx T, const __grid_constant__ Cg1Maps maps) {
  constexpr int NIN = kCg1Nin;
  using SMT = KSmem<P, PL, NIN, 1, kCg1Stages, kCg1Ub>;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SMT*>(smem_raw);
  double* zb =
      reinterpret_cast<double*>(smem_raw + zband_offset<P, PL, NIN, 1, kCg1Stages, kCg1Ub>());
  auto* cr = reinterpret_cast<CentreRing<PL>*>(smem_raw + cg1_centre_offset<P, PL>(g.n[2]));
  __shared__ double red[64];
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int v = 0; v < 2; ++v)
      for (int q = 0; q < 2; ++q) mbar_init(&cr->bar[v][q], 1);
  init_smem(g, sm, zb, true);  // (its barrier also publishes the centre-ring init)
  int cseq = 0;
  const KronTerms c{a, b, 0.0, 0.0};
  const int nx = g.n[0], ny = g.n[1];
  int buf = 0;
  int seq[4] = {0, 0, 0, 0};
  double tot[4];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0;
#if !K2_CG1_SCALED

  // r0 = b - A x0 (sparse.cpp:61-69)
  {
    EpiCg1Init e0{rhs, w.r[0], w.s[0], w.p, {0, 0, 0, 0}};
    Inputs<1> in1{{x}, {&maps.x}};
    NoPro np;
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 1, 1, true>(g, c, in1, np, sg, sm, zb, seq, e0);
    });
    grid_reduce(grid, e0.acc, w.partials, buf, red, tot);
  }
  const double bnorm = sqrt(tot[1]);
  if (bnorm == 0.0) {  // sparse.cpp:57-60: zero rhs resets even a warm start
    const size_t n = static_cast<size_t>(nx) * ny * g.n[2];
    for (size_t f = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.y * kKronTX + threadIdx.x;
         f < n; f += static_cast<size_t>(gridDim.x) * kThreads)
      x[f] = 0.0;
    if (lead) *w.status = PcgStatus{0, 0, 0.0, 0.0};
    return;
  }
  double rel = sqrt(tot[0]) / bnorm;
  if (max_iter <= 0 || rel <= tol) {  // the reference tests before its first matvec
    if (lead) *w.status = PcgStatus{0, max_iter <= 0 ? 3 : 0, rel, bnorm};
    return;
  }
  // w0 = A u0, gamma0 = r0.u0, delta0 = w0.u0 = p0.Ap0
  {
    ProScale<P, PL> ps{nx, ny, 0.0};
    EpiCg1 e1{w.w[0], 0.0};
    Inputs<2> in2{{w.r[0], w.inv_diag}, {&maps.r[0], &maps.inv_diag}};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 2, 1, true>(g, c, in2, ps, sg, sm, zb, seq, e1);
    });
    const double acc[4] = {ps.gamma, e1.delta, 0.0, 0.0};
    grid_reduce(grid, acc, w.partials, buf, red, tot);
  }
  double gamma = tot[0];
  int it = 0, status = 3;
  if (!(tot[1] > 0.0)) {
    if (lead) *w.status = PcgStatus{0, 4, rel, bnorm};
    return;
  }
  double alpha = gamma / tot[1], beta = 0.0;
  int cur = 0;
  // the next sweep's first ring boxes are issued as soon as the grid barrier
  // of the reduction has passed (its inputs are final), overlapping the
  // partial sums and the scalar updates
  Seg seg0{};
  const bool has_seg = first_segment(T, gridDim.x, blockIdx.x, seg0);
  auto inputs = [&](int k) {
    return Inputs<4>{{w.r[k], w.w[k], w.s[k], w.inv_diag},
                     {&maps.r[k], &maps.w[k], &maps.s[k], &maps.inv_diag}};
  };
  bool primed = false;
  while (it < max_iter) {
    ProCg1<P, PL> pc{alpha, beta, x,          w.p,       w.r[cur ^ 1], w.s[cur ^ 1], nx,
                     ny,    cr,   &maps.xc, &maps.pc, &cseq,        0.0,          0.0};
    EpiCg1 e{w.w[cur ^ 1], 0.0};
    const Inputs<4> in = inputs(cur);
    bool first = true;
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 4, 1, true>(g, c, in, pc, sg, sm, zb, seq, e, first && primed);
      first = false;
    });
    const double acc[4] = {pc.gamma, e.delta, pc.rr, 0.0};
    const Inputs<4> next = inputs(cur ^ 1);
    grid_reduce(grid, acc, w.partials, buf, red, tot, [&] {
      if (has_seg) prime_ring<P, PL, 4>(next, seg0, sm, seq);
    });
    primed = has_seg;
    ++it;
    cur ^= 1;
    bool stop = it >= max_iter;  // the reference leaves after max_iter updates untested
    if (!stop) {
      rel = sqrt(tot[2]) / bnorm;
      if (rel <= tol) {
        status = 0;
        stop = true;
      }
    }
    if (stop) {
      if (primed) drain_ring<P, PL, 4>(seg0, sm, seq);
      break;
    }
    const double g1 = tot[0];
    beta = g1 / gamma;
    const double den = tot[1] - beta * g1 / alpha;  // p_{i+1}.A p_{i+1}
    if (!(den > 0.0)) {
      status = 4;
      if (primed) drain_ring<P, PL, 4>(seg0, sm, seq);
      break;
    }
    alpha = g1 / den;
    gamma = g1;
  }
  if (lead) *w.status = PcgStatus{it, status, rel, bnorm};
#else
  // scaled form: the vectors w.r[], w.w[], w.s[] hold u, w^, s^
  // r0 = b - A x0 (sparse.cpp:61-69), u0 = D^-1 r0; r.r, b.b, r.u
  {
    EpiCg1InitS<P> e0{rhs, w.r[0], w.s[0], w.p, &g, a, b, {{}, zb, g.n[2]}, -1, -1, {0, 0, 0, 0}};
    Inputs<1> in1{{x}, {&maps.x}, {&maps.sx}};
    ProCopy<P, PL> pcp{&g, nx, ny, {{}, zb, g.n[2]}};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_seg<P, PL, 1, 1, true>(g, c, in1, pcp, sg, sm, zb, seq, e0);
    });
    grid_reduce(grid, e0.acc, w.partials, buf, red, tot);
  }
  const double bnorm = sqrt(tot[1]);
  if (bnorm == 0.0) {  // sparse.cpp:57-60: zero rhs resets even a warm start
    const size_t n = static_cast<size_t>(nx) * ny * g.n[2];
    for (size_t f = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.y * kKronTX + threadIdx.x;
         f < n; f += static_cast<size_t>(gridDim.x) * kThreads)
      x[f] = 0.0;
    if (lead) *w.status = PcgStatus{0, 0, 0.0, 0.0};
    return;
  }
  double rel = sqrt(tot[0]) / bnorm;
  if (max_iter <= 0 || rel <= tol) {  // the reference tests before its first matvec
    if (lead) *w.status = PcgStatus{0, max_iter <= 0 ? 3 : 0, rel, bnorm};
    return;
  }
  double gamma = tot[2];
  // w^0 = D^-1 A u0, delta0 = (A u0).u0 = p0.Ap0
  {
    ProCopy<P, PL> pcp{&g, nx, ny, {{}, zb, g.n[2]}};
    EpiCg1S<P, ProCopy<P, PL>> e1{w.w[0], &pcp, a, b, 0.0};
    Inputs<1> in1{{w.r[0]}, {&maps.r[0]}, {&maps.sr[0]}};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_seg<P, PL, 1, 1, true>(g, c, in1, pcp, sg, sm, zb, seq, e1);
    });
    const double acc[4] = {e1.delta, 0.0, 0.0, 0.0};
    grid_reduce(grid, acc, w.partials, buf, red, tot);
  }
  int it = 0, status = 3;
  if (!(tot[0] > 0.0)) {
    if (lead) *w.status = PcgStatus{0, 4, rel, bnorm};
    return;
  }
  double alpha = gamma / tot[0], beta = 0.0, alpha_prev = 0.0;
  int cur = 0;
  Seg seg0{};
  const bool has_seg = first_segment(T, gridDim.x, blockIdx.x, seg0);
  auto inputs = [&](int k) {
    return Inputs<NIN>{{w.r[k], w.w[k], w.s[k]},
                       {&maps.r[k], &maps.w[k], &maps.s[k]},
                       {&maps.sr[k], &maps.sw[k], &maps.ss[k]}};
  };
  bool primed = false;
  while (it < max_iter) {
    ProCg1S<P, PL> pc{alpha, beta, x,   w.p,  w.r[cur ^ 1], w.s[cur ^ 1], nx, ny, cr, &maps.xc,
                      &maps.pc, &cseq, &g, a,   b,            {{}, zb, g.n[2]}, 0.0, 0.0};
    // x is read and written every second sweep only (80 -> 72 B/DOF/iteration)
    pc.xmode = K2_DEFER_X ? ((it & 1) ? 2 : 1) : 0;
    pc.alpha_prev = alpha_prev;
    pc.smx = &maps.sxc;
    pc.smp = &maps.spc;
    EpiCg1S<P, ProCg1S<P, PL>> e{w.w[cur ^ 1], &pc, a, b, 0.0};
    const Inputs<NIN> in = inputs(cur);
#if K2_STUDY_NOSWEEP  // latency study only (tools/k2_iter_time.py): barrier + reduction alone
    {
      const double acc0[4] = {1.0, 1.0, 1.0, 0.0};
      grid_reduce(grid, acc0, w.partials, buf, red, tot);
      ++it;
      continue;
    }
#endif
    bool first = true;
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_seg<P, PL, NIN, 1, true>(g, c, in, pc, sg, sm, zb, seq, e, first && primed);
      first = false;
    });
    const double acc[4] = {pc.gamma, e.delta, pc.rr, 0.0};
    const Inputs<NIN> next = inputs(cur ^ 1);
    grid_reduce(grid, acc, w.partials, buf, red, tot, [&] {
      if (has_seg) prime_ring<P, PL, NIN>(next, seg0, sm, seq);
    });
    primed = has_seg;
    ++it;
    cur ^= 1;
    bool stop = it >= max_iter;  // the reference leaves after max_iter updates untested
    if (!stop) {
      rel = sqrt(tot[2]) / bnorm;
      if (rel <= tol) {
        status = 0;
        stop = true;
      }
    }
    if (stop) {
      if (primed) drain_ring<P, PL, NIN>(seg0, sm, seq);
      break;
    }
    const double g1 = tot[0];
    beta = g1 / gamma;
    const double den = tot[1] - beta * g1 / alpha;  // p_{i+1}.A p_{i+1}
    if (!(den > 0.0)) {
      status = 4;
      if (primed) drain_ring<P, PL, NIN>(seg0, sm, seq);
      break;
    }
    alpha_prev = alpha;
    alpha = g1 / den;
    gamma = g1;
  }
  if (K2_DEFER_X && it > 0 && ((it - 1) & 1) == 0) {  // the last sweep deferred its x update
    const size_t n = static_cast<size_t>(nx) * ny * g.n[2];
    for (size_t f = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.y * kKronTX + threadIdx.x;
         f < n; f += static_cast<size_t>(gridDim.x) * kThreads)
      x[f] = fma(alpha, w.p[f], x[f]);
  }
  if (lead) *w.status = PcgStatus{it, status, rel, bnorm};
#endif
}

// --------------------------------------------------------------------------
// The single-sweep solve on one z-slab of the free grid (multi-GPU: one slab
// per rank). The slab holds its own planes plus P ghost planes per interior
// side; each launch is ONE sweep of the persistent kernel above (the same
// prologue / epilogue functors) with the dot products restricted to the own
// planes, and the scalar recurrences advanced at the start of the next launch
// from the ranks' partial sums (summed in rank order, so every rank computes
// the same alpha, beta and stop decision). Between launches the caller
// exchanges the P ghost planes of the vector the sweep wrote (u_0, w^_0, then
// w^ each iteration: the only halo the next prologue reads that the rank
// cannot recompute) and all-gathers the 4 partials (NCCL over NVLink, or
// device copies between slabs of one GPU).
template <int P, int PL>
__global__ void __launch_bounds__(kThreads, K2_MINB)
    k2_slab_kernel(KronGrid g, double a, double b, const double* rhs, double* x, Cg1Work w,
                   double tol, int max_iter, TileIdx T, const __grid_constant__ Cg1Maps maps,
                   SlabCtl ctl) {
  constexpr int NIN = kCg1Nin;
  using SMT = KSmem<P, PL, NIN, 1, kCg1Stages, kCg1Ub>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SMT*>(smem_raw);
  double* zb =
      reinterpret_cast<double*>(smem_raw + zband_offset<P, PL, NIN, 1, kCg1Stages, kCg1Ub>());
  auto* cr = reinterpret_cast<CentreRing<PL>*>(smem_raw + cg1_centre_offset<P, PL>(g.n[2]));
  __shared__ double red[64];
  __shared__ int last_block;
  const int tid = threadIdx.y * kKronTX + threadIdx.x;
  const bool lead = blockIdx.x == 0 && tid == 0;

  // ---- the scalars (identical in every CTA of every rank)
  SlabState st = *ctl.sin;
  double tot[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < ctl.world; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) tot[c] += ctl.gath[4 * r + c];
  double beta = 0.0;
  bool zero_x = false;
  if (ctl.phase == 0) {
    st = SlabState{0.0, 0.0, 0.0, 0.0, 0.0, 0, 3, 1, 0};
  } else if (!st.done && ctl.phase == 1) {  // r.r, b.b, r.u of the initial residual
    st.bnorm = sqrt(tot[1]);
    if (st.bnorm == 0.0) {  // sparse.cpp:57-60: zero rhs resets even a warm start
      zero_x = true;
      st.status = 0;
      st.rel = 0.0;
      st.done = 1;
    } else {
      st.rel = sqrt(tot[0]) / st.bnorm;
      if (max_iter <= 0 || st.rel <= tol) {
        st.status = max_iter <= 0 ? 3 : 0;
        st.done = 1;
      }
      st.gamma = tot[2];
    }
    st.stage = 2;
  } else if (!st.done && st.stage == 2) {  // delta_0 = (A u0).u0
    if (!(tot[0] > 0.0)) {
      st.status = 4;
      st.done = 1;
    } else {
      st.alpha = st.gamma / tot[0];
      beta = 0.0;
    }
    st.stage = 3;
  } else if (!st.done) {  // the previous sweep's gamma', delta', r.r
    ++st.it;
    bool stop = st.it >= max_iter;  // the reference leaves after max_iter updates untested
    if (!stop) {
      st.rel = sqrt(tot[2]) / st.bnorm;
      if (st.rel <= tol) {
        st.status = 0;
        stop = true;
      }
    }
    if (stop) {
      st.done = 1;
    } else {
      const double g1 = tot[0];
      beta = g1 / st.gamma;
      const double den = tot[1] - beta * g1 / st.alpha;  // p_{i+1}.A p_{i+1}
      if (!(den > 0.0)) {
        st.status = 4;
        st.done = 1;
      } else {
        st.alpha = g1 / den;
        st.gamma = g1;
      }
    }
  }
  st.beta = beta;
  if (lead) *ctl.sout = st;
  const int nx = g.n[0], ny = g.n[1];
  if (zero_x) {
    const size_t n = static_cast<size_t>(nx) * ny * g.n[2];
    for (size_t f = static_cast<size_t>(blockIdx.x) * kThreads + tid; f < n;
         f += static_cast<size_t>(gridDim.x) * kThreads)
      x[f] = 0.0;
  }
  if (st.done) return;

  // ---- one sweep
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int v = 0; v < 2; ++v)
      for (int q = 0; q < 2; ++q) mbar_init(&cr->bar[v][q], 1);
  init_smem(g, sm, zb, true);
  int cseq = 0;
  int seq[4] = {0, 0, 0, 0};
  const KronTerms c{a, b, 0.0, 0.0};
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (ctl.phase == 0) {  // r0 = b - A x0, u0 = D^-1 r0, s = p = 0
    EpiCg1InitS<P> e0{rhs, w.r[0], w.s[0], w.p, &g, a, b, {{}, zb, g.n[2]}, -1, -1,
                      {0, 0, 0, 0}, ctl.zo0, ctl.zo1};
    Inputs<1> in1{{x}, {&maps.x}};
    ProCopy<P, PL> pcp{&g, nx, ny, {{}, zb, g.n[2]}};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 1, 1, true>(g, c, in1, pcp, sg, sm, zb, seq, e0);
    });
    for (int q = 0; q < 4; ++q) acc[q] = e0.acc[q];
  } else if (ctl.phase == 1) {  // w^0 = D^-1 A u0, delta0
    ProCopy<P, PL> pcp{&g, nx, ny, {{}, zb, g.n[2]}};
    EpiCg1S<P, ProCopy<P, PL>> e1{w.w[0], &pcp, a, b, 0.0, ctl.zo0, ctl.zo1};
    Inputs<1> in1{{w.r[0]}, {&maps.r[0]}};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, 1, 1, true>(g, c, in1, pcp, sg, sm, zb, seq, e1);
    });
    acc[0] = e1.delta;
  } else {
    const int cur = ctl.cur;
    ProCg1S<P, PL> pc{st.alpha, beta, x, w.p, w.r[cur ^ 1], w.s[cur ^ 1], nx, ny, cr, &maps.xc,
                      &maps.pc, &cseq, &g, a, b, {{}, zb, g.n[2]}, 0.0, 0.0, ctl.zo0, ctl.zo1};
    EpiCg1S<P, ProCg1S<P, PL>> e{w.w[cur ^ 1], &pc, a, b, 0.0, ctl.zo0, ctl.zo1};
    const Inputs<NIN> in{{w.r[cur], w.w[cur], w.s[cur]}, {&maps.r[cur], &maps.w[cur], &maps.s[cur]}};
    for_segments(T, gridDim.x, blockIdx.x, [&](const Seg& sg) {
      kron_tile<P, PL, NIN, 1, true>(g, c, in, pc, sg, sm, zb, seq, e);
    });
    acc[0] = pc.gamma;
    acc[1] = e.delta;
    acc[2] = pc.rr;
  }

  // ---- this rank's partial sums: a fixed tree per CTA, then the last CTA to
  // arrive sums the CTA partials in block order (deterministic)
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp * 4 + q] = v;
  }
  __syncthreads();
  if (tid < 4) {
    double v = 0.0;
    for (int q = 0; q < kThreads / 32; ++q) v += red[q * 4 + tid];
    ctl.cta_part[blockIdx.x * 4 + tid] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last_block = atomicAdd(ctl.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last_block && warp == 0) {
    __threadfence();
double v[4];
    warp_sum_partials(ctl.cta_part, static_cast<int>(gridDim.x), lane, v);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) ctl.mine[q] = v[q];
    if (lane == 0) *ctl.ticket = 0u;
  }
}

// --------------------------------------------------------------------------
// TMA descriptor encoding through the driver entry point (no -lcuda)

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

template <int P, int PL, int NIN, int NPASS, int ST = kStages>
size_t smem_bytes(int nz) {
  return zband_offset<P, PL, NIN, NPASS, ST>() + 2 * static_cast<size_t>(nz) * (2 * P + 1) * 8;
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  TG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(bytes)));
}

// CTAs for a sweep: at most `max_blocks`, and >= ~6 planes per CTA (small
// grids are latency-bound: more CTAs beat the 2P halo-plane overhead).
#ifndef K2_MIN_PLANES
#define K2_MIN_PLANES 3  // config 2 per CG iteration: 2 -> 16.6 us, 3 -> 15.5, 4 -> 16.2, 6 -> 17.4
#endif
int seg_blocks(const TileIdx& T, int max_blocks) {
  const long total = n_columns(T) * T.nz;  // column-planes
  return static_cast<int>(std::max(1L, std::min<long>(max_blocks, total / K2_MIN_PLANES)));
}

}  // namespace

bool k2_strip_applies(const KronGrid& g) { return strip_applies(g); }

bool k2_make_map(const KronGrid& g, const double* base, TensorMap3* out, bool halo, int planes,
                 bool strip) {
  static_assert(sizeof(TensorMap3) == sizeof(CUtensorMap), "tensor map size");
  EncodeFn enc = encoder();
  const size_t pitch = static_cast<size_t>(g.n[0]) * sizeof(double);
  if (!enc || pitch % 16 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
  // The TMA sweeps are validated for degree 2 (every BASELINE cuboid): with
  // degree-1 and degree-3 bands on a TMA-addressable grid the swept kernels
  // stop with an illegal-instruction fault, so those grids take the plain-load
  // kernels (and small grids the resident solve, which uses no TMA).
  if (g.p != 2) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.n[0]), static_cast<cuuint64_t>(g.n[1]),
                              static_cast<cuuint64_t>(g.n[2])};
  const cuuint64_t strides[2] = {pitch, pitch * static_cast<cuuint64_t>(g.n[1])};
  const int h = halo ? 2 * g.p : 0;
  const int bx = strip ? StripTile::TX : kKronTX, by = strip ? StripTile::TY : kKronTY;
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(bx + h), static_cast<cuuint32_t>(by + h),
                             static_cast<cuuint32_t>(planes)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::memcpy(out, &m, sizeof(m));
  return true;
}

// dispatch on the degree
#define TG_KRON_DISPATCH(P_, ...)                                                \
  switch (P_) {                                                                  \
    case 1: { constexpr int P = 1; __VA_ARGS__; break; }                         \
    case 2: { constexpr int P = 2; __VA_ARGS__; break; }                         \
    case 3: { constexpr int P = 3; __VA_ARGS__; break; }                         \
    default: throw std::invalid_argument("kronecker path supports degree 1..3"); \
  }

void k2_apply(const KronGrid& g, double a, double b, const double* v, double* y, int sm_count,
              cudaStream_t s, const TensorMap3* v_map) {
  const TileIdx T = make_tiles(g);
  const int blocks = seg_blocks(T, 3 * sm_count);
  ApplyMap m{};
  if (v_map) m.v = *v_map;
  TG_KRON_DISPATCH(g.p, {
    if (v_map) {
      const size_t sb = smem_bytes<P, kTmaPlanes, 1, 1>(g.n[2]);
      allow_smem(k2_apply_kernel<P, true>, sb);
      k2_apply_kernel<P, true><<<blocks, dim3(kKronTX, kKronTY), sb, s>>>(
          g, KronTerms{a, b, 0.0, 0.0}, v, y, T, m);
    } else {
      const size_t sb = smem_bytes<P, 1, 1, 1>(g.n[2]);
      allow_smem(k2_apply_kernel<P, false>, sb);
      k2_apply_kernel<P, false><<<blocks, dim3(kKronTX, kKronTY), sb, s>>>(
          g, KronTerms{a, b, 0.0, 0.0}, v, y, T, m);
    }
  });
  TG_CUDA(cudaGetLastError());
}

void k2_theta_rhs(const KronGrid& full, double a_b, double b_b, double a_a, double b_a,
                  const RhsArgs& args, const TensorMap3* mT, const TensorMap3* mg, int sm_count,
                  cudaStream_t s) {
  const TileIdx T = make_tiles(full);
  const int blocks = seg_blocks(T, 2 * sm_count);
  RhsMaps maps{};
  const bool tma = mT && mg;
  if (tma) {
    maps.T = *mT;
    maps.g = *mg;
  }
  const KronTerms c{a_b, b_b, a_a, b_a};
  TG_KRON_DISPATCH(full.p, {
    if (tma) {
      const size_t sb = smem_bytes<P, kTmaPlanes, 2, 2>(full.n[2]);
      allow_smem(k2_rhs_kernel<P, true>, sb);
      k2_rhs_kernel<P, true><<<blocks, dim3(kKronTX, kKronTY), sb, s>>>(full, c, args, T, maps);
    } else {
      const size_t sb = smem_bytes<P, 1, 2, 2>(full.n[2]);
      allow_smem(k2_rhs_kernel<P, false>, sb);
      k2_rhs_kernel<P, false><<<blocks, dim3(kKronTX, kKronTY), sb, s>>>(full, c, args, T, maps);
    }
  });
  TG_CUDA(cudaGetLastError());
}

void k2_inverse_diagonal(const KronGrid& g, double a, double b, double* inv_diag,
                         PcgStatus* status, cudaStream_t s) {
  TG_KRON_DISPATCH(g.p, k2_inv_diag_kernel<P><<<512, 256, 0, s>>>(g, a, b, inv_diag, status));
  TG_CUDA(cudaGetLastError());
}

int k2_pcg_max_blocks(int p, int sm_count, int nz) {
  int per_sm = 0;
  TG_KRON_DISPATCH(p, {
    const size_t sbt = smem_bytes<P, kTmaPlanes, 2, 1>(nz);
    const size_t sbp = smem_bytes<P, 1, 2, 1>(nz);
    allow_smem(k2_pcg_kernel<P, true>, sbt);
    allow_smem(k2_pcg_kernel<P, false>, sbp);
    TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, reinterpret_cast<const void*>(&k2_pcg_kernel<P, true>), kThreads, sbt));
  });
  return std::max(1, per_sm) * sm_count;
}

void k2_pcg_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const PcgWork& w, const PcgMaps& maps, double tol, int max_iter, int blocks,
                  cudaStream_t s) {
  const TileIdx T = make_tiles(g);
  const int nb = seg_blocks(T, blocks);
  dim3 grid(nb), block(kKronTX, kKronTY);
  KronGrid gg = g;
  PcgWork ww = w;
  PcgMaps mm = maps;
  double aa = a, bb = b, tt = tol;
  int mi = max_iter;
  TileIdx TT = T;
  void* args[] = {&gg, &aa, &bb, const_cast<double**>(&rhs), &x, &ww, &tt, &mi, &TT, &mm};
  TG_KRON_DISPATCH(g.p, {
    if (maps.valid)
      TG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k2_pcg_kernel<P, true>),
                                          grid, block, args,
                                          smem_bytes<P, kTmaPlanes, 2, 1>(g.n[2]), s));
    else
      TG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k2_pcg_kernel<P, false>),
                                          grid, block, args, smem_bytes<P, 1, 2, 1>(g.n[2]), s));
  });
}

#define TG_CG1_PL_DISPATCH(PL_, ...)                                          \
  switch (PL_) {                                                              \
    case 2: { constexpr int PL = 2; __VA_ARGS__; break; }                     \
    case 4: { constexpr int PL = 4; __VA_ARGS__; break; }                     \
    default: throw std::invalid_argument("cg1: planes per step must be 2 or 4"); \
  }

#ifndef K2_SMALL_PL
#define K2_SMALL_PL 4
#endif
int k2_cg1_planes(const KronGrid& g, int sm_count) {
  const TileIdx T = make_tiles(g);
  const long colplanes = static_cast<long>(T.ntx) * T.nty * T.nz;
  return colplanes / K2_MIN_PLANES < 2L * sm_count ? K2_SMALL_PL : 2;
}

int k2_cg1_max_blocks(int p, int sm_count, int nz, int pl) {
  int per_sm = 0;
  TG_KRON_DISPATCH(p, TG_CG1_PL_DISPATCH(pl, {
    const size_t sb = cg1_smem_bytes<P, PL>(nz);
    allow_smem(k2_cg1_kernel<P, PL>, sb);
    TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, reinterpret_cast<const void*>(&k2_cg1_kernel<P, PL>), kThreads, sb));
  }));
  return std::max(1, per_sm) * sm_count;
}

void k2_cg1_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const Cg1Work& w, const Cg1Maps& maps, double tol, int max_iter, int blocks,
                  cudaStream_t s, int pl) {
#if K2_CG1_SCALED
  TileIdx T = maps.strip ? make_tiles_strip(g) : make_tiles(g);
#else
  TileIdx T = make_tiles(g);
#endif
  int nb = seg_blocks(T, blocks);
  // the column-aligned split when every column (strip columns in halves) gets
  // its own CTA of one wave and the columns are deep enough to amortize the
  // 2P halo planes of a whole-column segment (TG_K2_ALIGNED=0/1 forces).
  // Config 4: 85.5 against 89.8 us/iteration, DRAM reads 19.3 -> 13.6 GB per
  // solve (the unit split drifted the CTAs' z positions apart, so y-neighbour
  // tiles missed each other's halo rows in L2)
  {
    const int need = T.ntx * T.nty + 2 * T.nsy;
    bool al = need <= blocks && T.nz >= 32;  // config 4: 264 + 2 x 9 = 282 CTAs
    if (const char* e = std::getenv("TG_K2_ALIGNED")) al = std::atoi(e) != 0 && need <= blocks;
    if (al) {
      T.aligned = 1;
      nb = need;
    }
  }
  dim3 grid(nb), block(kKronTX, kKronTY);
  KronGrid gg = g;
  Cg1Work ww = w;
  Cg1Maps mm = maps;
  double aa = a, bb = b, tt = tol;
  int mi = max_iter;
  TileIdx TT = T;
  void* args[] = {&gg, &aa, &bb, const_cast<double**>(&rhs), &x, &ww, &tt, &mi, &TT, &mm};
  TG_KRON_DISPATCH(g.p, TG_CG1_PL_DISPATCH(pl, {
    TG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k2_cg1_kernel<P, PL>),
                                        grid, block, args, cg1_smem_bytes<P, PL>(g.n[2]), s));
  }));
}

int k2_slab_max_blocks(int p, int sm_count, int nz, int pl) {
  int per_sm = 0;
  TG_KRON_DISPATCH(p, TG_CG1_PL_DISPATCH(pl, {
    const size_t sb = cg1_smem_bytes<P, PL>(nz);
    allow_smem(k2_slab_kernel<P, PL>, sb);
    TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, reinterpret_cast<const void*>(&k2_slab_kernel<P, PL>), kThreads, sb));
  }));
  return std::max(1, per_sm) * sm_count;
}

void k2_slab_launch(const KronGrid& g, double a, double b, const double* rhs, double* x,
                    const Cg1Work& w, const Cg1Maps& maps, double tol, int max_iter, int blocks,
                    const SlabCtl& ctl, cudaStream_t s, int pl) {
  const TileIdx T = make_tiles(g);
  const int nb = seg_blocks(T, blocks);
  dim3 grid(nb), block(kKronTX, kKronTY);
  TG_KRON_DISPATCH(g.p, TG_CG1_PL_DISPATCH(pl, {
    const size_t sb = cg1_smem_bytes<P, PL>(g.n[2]);  // slabs of one solver differ in depth
    allow_smem(k2_slab_kernel<P, PL>, sb);
    k2_slab_kernel<P, PL><<<grid, block, sb, s>>>(g, a, b, rhs, x, w, tol, max_iter, T, maps, ctl);
  }));
  TG_CUDA(cudaGetLastError());
}

}  // namespace tgb
