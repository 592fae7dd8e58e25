// K2 — matrix-free theta-step operator and Jacobi-PCG on B200.
//
// Reference: DirichletSystem (proj/src/assembly.cpp:186-281) assembles
// A = M/dt + theta K and B = M/dt - (1-theta) K as CSR and pcg_jacobi
// (proj/src/sparse.cpp:41-100) runs ~130-170 serial CSR SpMV iterations per
// step. For separable patches (every axis-aligned cuboid, any knot grading)
// the p+1-point Gauss quadrature factorizes exactly, so
//   M = rho c (Mz x My x Mx),  K = k (Mz x My x Kx + Mz x Ky x Mx + Kz x My x Mx)
// with banded 1D factors (2p+1 diagonals). The apply is sum-factorized:
//   x-pass  u1 = Mx v, u2 = Kx v          (shared-memory tile with halo)
//   y-pass  w1 = My u1, w2 = My u2, w3 = Ky u1
//           s1 = a w1 + b (w2 + w3),  s2 = b w1
//   z-pass  y = Mz s1 + Kz s2            (2p+1-plane register window)
// Each CTA owns a 32 x 8 column of the control grid and marches through a
// z-range, so v is read from HBM once and y written once per apply
// (16 B per DOF); the x/y halos come from L2.
//
// The whole PCG solve is one persistent cooperative launch: phases separated
// by grid-wide barriers, dot products reduced per CTA in a fixed tree and
// then across CTAs in a fixed order (bitwise-deterministic reruns), the
// convergence test evaluated on the device. The algorithm is the reference's:
// warm start, Jacobi preconditioner, stop test ||r||/||b|| <= tol before the
// matvec, b = 0 -> x = 0, failure on pAp <= 0 or after max_iter.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "context.hpp"
#include "k2_kron.cuh"

namespace cg = cooperative_groups;

namespace tgb {

namespace {

constexpr int kThreads = kKronTX * kKronTY;

template <int P, int NIN>
struct TileSmem {
  double v[NIN][kKronTY + 2 * P][kKronTX + 2 * P];
  double u1[NIN][kKronTY + 2 * P][kKronTX];
  double u2[NIN][kKronTY + 2 * P][kKronTX];
  double cx[2][kKronTX][2 * P + 1];  // Mx, Kx rows of the tile's xi range
  double cy[2][kKronTY][2 * P + 1];  // My, Ky rows of the tile's eta range
};

struct TileIdx {
  int ntx, nty, nzc, zlen;
  __device__ __host__ int count() const { return ntx * nty * nzc; }
};

// Tile layout for `blocks` co-resident CTAs. Each tile is a 32 x 8 column
// marching through zlen planes (+ P halo planes each side). With static
// tile -> CTA assignment (deterministic reductions), the cost is
// ceil(tiles / blocks) * (zlen + 2P); pick the z split that minimizes it.
inline TileIdx make_tiles(const KronGrid& g, int blocks, int P) {
  TileIdx best{};
  double best_cost = 1e300;
  const int ntx = (g.n[0] + kKronTX - 1) / kKronTX;
  const int nty = (g.n[1] + kKronTY - 1) / kKronTY;
  const int cap = std::max(1, g.n[2] / 4);  // >= 4 planes per chunk
  for (int nzc = 1; nzc <= std::min(cap, 16); ++nzc) {
    TileIdx t;
    t.ntx = ntx;
    t.nty = nty;
    t.zlen = (g.n[2] + nzc - 1) / nzc;
    t.nzc = (g.n[2] + t.zlen - 1) / t.zlen;
    const int rounds = (t.count() + blocks - 1) / blocks;
    const double cost = static_cast<double>(rounds) * (t.zlen + 2 * P) * 1.000001 +
                        1e-9 * t.count();  // ties: fewer tiles
    if (cost < best_cost) {
      best_cost = cost;
      best = t;
    }
  }
  return best;
}

// Sweep one tile: for every output point (i, j, k) of the tile call
// epi(flat_index, i, j, k, y) with y = sum over inputs of Op(a, b) v.
template <int P, int NIN, class Epi>
__device__ __forceinline__ void kron_tile(const KronGrid& g, const KronTerms& c,
                                          const double* __restrict__ v1,
                                          const double* __restrict__ v2, const TileIdx& T,
                                          int tile, TileSmem<P, NIN>& sm, Epi& epi) {
  constexpr int W = 2 * P + 1;
  constexpr int RY = kKronTY + 2 * P;
  constexpr int RX = kKronTX + 2 * P;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int txy = tile % (T.ntx * T.nty);
  const int zc = tile / (T.ntx * T.nty);
  const int x0 = (txy % T.ntx) * kKronTX, y0 = (txy / T.ntx) * kKronTY;
  const int k0 = zc * T.zlen, k1 = min(g.n[2], k0 + T.zlen);
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int i = x0 + tx, j = y0 + ty;

  // the tile's 1D rows in shared memory (zero beyond the grid); the barrier
  // retires the previous tile's readers, the first plane's barrier orders
  // these writes before any read
  __syncthreads();
  for (int q = ty * kKronTX + tx; q < kKronTX * W; q += kKronTX * kKronTY) {
    const int r = q / W, d = q % W, gi = x0 + r;
    sm.cx[0][r][d] = gi < nx ? g.M[0][gi * W + d] : 0.0;
    sm.cx[1][r][d] = gi < nx ? g.K[0][gi * W + d] : 0.0;
  }
  for (int q = ty * kKronTX + tx; q < kKronTY * W; q += kKronTX * kKronTY) {
    const int r = q / W, d = q % W, gj = y0 + r;
    sm.cy[0][r][d] = gj < ny ? g.M[1][gj * W + d] : 0.0;
    sm.cy[1][r][d] = gj < ny ? g.K[1][gj * W + d] : 0.0;
  }
  double win1[W], win2[W];
#pragma unroll
  for (int d = 0; d < W; ++d) win1[d] = win2[d] = 0.0;

  const size_t plane = static_cast<size_t>(nx) * ny;
  for (int kin = k0 - P; kin < k1 + P; ++kin) {
    double s1 = 0.0, s2 = 0.0;
    if (kin >= 0 && kin < nz) {
      // load the input plane tile(s) with a P-wide halo, zero outside the grid
#pragma unroll
      for (int q = 0; q < NIN; ++q) {
        const double* v = q == 0 ? v1 : v2;
        for (int r = ty; r < RY; r += kKronTY) {
          const int gj = y0 + r - P;
          for (int cc = tx; cc < RX; cc += kKronTX) {
            const int gi = x0 + cc - P;
            double val = 0.0;
            if (gi >= 0 && gi < nx && gj >= 0 && gj < ny)
              val = v[static_cast<size_t>(kin) * plane + static_cast<size_t>(gj) * nx + gi];
            sm.v[q][r][cc] = val;
          }
        }
      }
      __syncthreads();
      // x-pass on the rows of the tile plus the y halo
#pragma unroll
      for (int q = 0; q < NIN; ++q)
        for (int r = ty; r < RY; r += kKronTY) {
          double a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int d = 0; d < W; ++d) {
            const double vv = sm.v[q][r][tx + d];
            a1 = fma(sm.cx[0][tx][d], vv, a1);
            a2 = fma(sm.cx[1][tx][d], vv, a2);
          }
          sm.u1[q][r][tx] = a1;
          sm.u2[q][r][tx] = a2;
        }
      __syncthreads();
      // y-pass and the z-pass inputs
#pragma unroll
      for (int q = 0; q < NIN; ++q) {
        double w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
          const double p1 = sm.u1[q][ty + d][tx];
          const double my = sm.cy[0][ty][d];
          w1 = fma(my, p1, w1);
          w2 = fma(my, sm.u2[q][ty + d][tx], w2);
          w3 = fma(sm.cy[1][ty][d], p1, w3);
        }
        const double a = q == 0 ? c.a1 : c.a2, b = q == 0 ? c.b1 : c.b2;
        s1 = fma(a, w1, fma(b, w2 + w3, s1));
        s2 = fma(b, w1, s2);
      }
    }
#pragma unroll
    for (int d = 0; d < W - 1; ++d) {
      win1[d] = win1[d + 1];
      win2[d] = win2[d + 1];
    }
    win1[W - 1] = s1;
    win2[W - 1] = s2;
    const int k = kin - P;
    if (k >= k0 && i < nx && j < ny) {
      const double* mz = g.M[2] + k * W;
      const double* kz = g.K[2] + k * W;
      double y = 0.0;
#pragma unroll
      for (int d = 0; d < W; ++d) y = fma(mz[d], win1[d], fma(kz[d], win2[d], y));
      epi(static_cast<size_t>(k) * plane + static_cast<size_t>(j) * nx + i, i, j, k, y);
    }
  }
}

// ---------------------------------------------------------------------------
// stand-alone applies

template <int P>
struct EpiStore {
  double* y;
  __device__ void operator()(size_t idx, int, int, int, double v) { y[idx] = v; }
};

template <int P>
__global__ void __launch_bounds__(kThreads) k2_apply_kernel(KronGrid g, KronTerms c,
                                                            const double* v, double* y,
                                                            TileIdx T) {
  __shared__ TileSmem<P, 1> sm;
  EpiStore<P> epi{y};
  for (int t = blockIdx.x; t < T.count(); t += gridDim.x) kron_tile<P, 1>(g, c, v, nullptr, T, t, sm, epi);
}

template <int P>
struct EpiRhs {
  RhsArgs a;
  int nfree[3];
  __device__ void operator()(size_t idx, int i, int j, int k, double y) {
    int ijk[3] = {i, j, k};
    if (ijk[a.bottom_axis] == a.bottom_layer) return;
    if (a.bottom_layer == 0) ijk[a.bottom_axis] -= 1;
    const size_t f = static_cast<size_t>(ijk[0]) +
                     static_cast<size_t>(nfree[0]) * (ijk[1] + static_cast<size_t>(nfree[1]) * ijk[2]);
    a.rhs[f] = y + a.theta * a.F_np1[idx] + (1.0 - a.theta) * a.F_n[idx];
  }
};

template <int P>
__global__ void __launch_bounds__(kThreads) k2_rhs_kernel(KronGrid g, KronTerms c, RhsArgs args,
                                                          TileIdx T) {
  __shared__ TileSmem<P, 2> sm;
  EpiRhs<P> epi{args, {g.n[0], g.n[1], g.n[2]}};
  epi.nfree[args.bottom_axis] -= 1;
  for (int t = blockIdx.x; t < T.count(); t += gridDim.x)
    kron_tile<P, 2>(g, c, args.T_full, args.g_full, T, t, sm, epi);
}

// ---------------------------------------------------------------------------
// diagonal

template <int P>
__global__ void k2_diag_kernel(KronGrid g, double a, double b, double* inv_diag,
                               PcgStatus* st) {
  const size_t n = static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2];
  constexpr int W = 2 * P + 1;
  for (size_t f = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(f % g.n[0]);
    const int j = static_cast<int>((f / g.n[0]) % g.n[1]);
    const int k = static_cast<int>(f / (static_cast<size_t>(g.n[0]) * g.n[1]));
    const double mx = g.M[0][i * W + P], kx = g.K[0][i * W + P];
    const double my = g.M[1][j * W + P], ky = g.K[1][j * W + P];
    const double mz = g.M[2][k * W + P], kz = g.K[2][k * W + P];
    const double d = a * (mx * my * mz) + b * (kx * my * mz + mx * ky * mz + mx * my * kz);
    if (!(d > 0.0)) st->status = 2;
    inv_diag[f] = 1.0 / d;
  }
}

// ---------------------------------------------------------------------------
// persistent Jacobi-PCG

struct Acc4 {
  double v[4];
};

// Block-reduce acc (fixed tree), store to partials[buf][block][4], grid sync,
// then every CTA sums the per-block partials in the same fixed order.
__device__ __forceinline__ void grid_reduce(cg::grid_group& grid, double (&acc)[4],
                                            double* partials, int& buf, double* red,
                                            double (&out)[4]) {
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
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
      for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) s += pb[b * 4 + c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) red[32 + c] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = red[32 + c];
  __syncthreads();
  buf ^= 1;
}

template <int P>
struct EpiResidual {  // r = b - A x; z = D^-1 r; p = z; accumulate rr, bb, rz
  const double* rhs;
  const double* invd;
  double* r;
  double* p;
  double acc[4];
  __device__ void operator()(size_t idx, int, int, int, double y) {
    const double bi = rhs[idx];
    const double ri = bi - y;
    const double zi = invd[idx] * ri;
    r[idx] = ri;
    p[idx] = zi;
    acc[0] += ri * ri;
    acc[1] += bi * bi;
    acc[2] += ri * zi;
  }
};

template <int P>
struct EpiAp {
  const double* p;
  double* Ap;
  double acc[4];
  __device__ void operator()(size_t idx, int, int, int, double y) {
    Ap[idx] = y;
    acc[0] += p[idx] * y;
  }
};

template <int P>
__global__ void __launch_bounds__(kThreads, 3) k2_pcg_kernel(KronGrid g, double a, double b,
                                                          const double* rhs, double* x,
                                                          PcgWork w, double tol, int max_iter,
                                                          TileIdx T) {
  cg::grid_group grid = cg::this_grid();
  __shared__ TileSmem<P, 1> sm;
  __shared__ double red[64];
  const KronTerms c{a, b, 0.0, 0.0};
  const size_t n = static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2];
  const size_t gtid = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.y * kKronTX + threadIdx.x;
  const size_t gstride = static_cast<size_t>(gridDim.x) * kThreads;
  int buf = 0;
  double tot[4];

  // r = b - A x, z = D^-1 r, p = z   (sparse.cpp:61-70)
  EpiResidual<P> e0{rhs, w.inv_diag, w.r, w.p, {0, 0, 0, 0}};
  for (int t = blockIdx.x; t < T.count(); t += gridDim.x) kron_tile<P, 1>(g, c, x, nullptr, T, t, sm, e0);
  grid_reduce(grid, e0.acc, w.partials, buf, red, tot);
  double rr = tot[0], rz = tot[2];
  const double bnorm = sqrt(tot[1]);
  if (bnorm == 0.0) {  // sparse.cpp:57-60: zero rhs resets even a warm start
    for (size_t f = gtid; f < n; f += gstride) x[f] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0)
      *w.status = PcgStatus{0, 0, 0.0, 0.0};
    return;
  }
  double rel = 0.0;
  int it = 0, status = 3;
  for (it = 0; it < max_iter; ++it) {
    rel = sqrt(rr) / bnorm;
    if (rel <= tol) {
      status = 0;
      break;
    }
    EpiAp<P> e1{w.p, w.Ap, {0, 0, 0, 0}};
    for (int t = blockIdx.x; t < T.count(); t += gridDim.x) kron_tile<P, 1>(g, c, w.p, nullptr, T, t, sm, e1);
    grid_reduce(grid, e1.acc, w.partials, buf, red, tot);
    const double pAp = tot[0];
    if (!(pAp > 0.0)) {
      status = 4;
      break;
    }
    const double alpha = rz / pAp;
    double acc[4] = {0, 0, 0, 0};
    for (size_t f = gtid; f < n; f += gstride) {
      const double pi = w.p[f];
      x[f] += alpha * pi;
      const double ri = w.r[f] - alpha * w.Ap[f];
      w.r[f] = ri;
      const double zi = w.inv_diag[f] * ri;
      acc[0] += ri * zi;
      acc[1] += ri * ri;
    }
    grid_reduce(grid, acc, w.partials, buf, red, tot);
    const double beta = tot[0] / rz;
    rz = tot[0];
    rr = tot[1];
    for (size_t f = gtid; f < n; f += gstride) w.p[f] = w.inv_diag[f] * w.r[f] + beta * w.p[f];
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *w.status = PcgStatus{it, status, rel, bnorm};
}

template <int P>
const void* pcg_kernel_ptr() {
  return reinterpret_cast<const void*>(&k2_pcg_kernel<P>);
}

}  // namespace

// dispatch on the degree (stored in the band width)
#define TG_KRON_DISPATCH(P_, ...)                                      \
  switch (P_) {                                                        \
    case 1: { constexpr int P = 1; __VA_ARGS__; break; }               \
    case 2: { constexpr int P = 2; __VA_ARGS__; break; }               \
    case 3: { constexpr int P = 3; __VA_ARGS__; break; }               \
    default: throw std::invalid_argument("kronecker path supports degree 1..3"); \
  }

void k2_apply(const KronGrid& g, double a, double b, const double* v, double* y, int sm_count,
              cudaStream_t s) {
  const TileIdx T = make_tiles(g, 3 * sm_count, g.p);
  const int blocks = std::min(T.count(), 3 * sm_count);
  TG_KRON_DISPATCH(g.p, k2_apply_kernel<P><<<blocks, dim3(kKronTX, kKronTY), 0, s>>>(
                                 g, KronTerms{a, b, 0.0, 0.0}, v, y, T));
  TG_CUDA(cudaGetLastError());
}

void k2_theta_rhs(const KronGrid& full, double a_b, double b_b, double a_a, double b_a,
                  const RhsArgs& args, int sm_count, cudaStream_t s) {
  const TileIdx T = make_tiles(full, 2 * sm_count, full.p);
  const int blocks = std::min(T.count(), 2 * sm_count);
  TG_KRON_DISPATCH(full.p, k2_rhs_kernel<P><<<blocks, dim3(kKronTX, kKronTY), 0, s>>>(
                                 full, KronTerms{a_b, b_b, a_a, b_a}, args, T));
  TG_CUDA(cudaGetLastError());
}

void k2_inverse_diagonal(const KronGrid& g, double a, double b, double* inv_diag,
                         PcgStatus* status, cudaStream_t s) {
  TG_KRON_DISPATCH(g.p, k2_diag_kernel<P><<<256, 256, 0, s>>>(g, a, b, inv_diag, status));
  TG_CUDA(cudaGetLastError());
}

int k2_pcg_max_blocks(int p, int sm_count) {
  int per_sm = 0;
  TG_KRON_DISPATCH(p, TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                 &per_sm, pcg_kernel_ptr<P>(), kThreads, 0)));
  return std::max(1, per_sm) * sm_count;
}

void k2_pcg_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const PcgWork& w, double tol, int max_iter, int blocks, cudaStream_t s) {
  const TileIdx T = make_tiles(g, blocks, g.p);
  int nb = std::max(1, std::min(blocks, T.count()));
  dim3 grid(nb), block(kKronTX, kKronTY);
  KronGrid gg = g;
  PcgWork ww = w;
  double aa = a, bb = b, tt = tol;
  int mi = max_iter;
  TileIdx TT = T;
  void* args[] = {&gg, &aa, &bb, const_cast<double**>(&rhs), &x, &ww, &tt, &mi, &TT};
  TG_KRON_DISPATCH(g.p, TG_CUDA(cudaLaunchCooperativeKernel(pcg_kernel_ptr<P>(), grid,
                                                                  block, args, 0, s)));
}

}  // namespace tgb
