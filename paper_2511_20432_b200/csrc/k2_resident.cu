// K2 — the single-sweep Jacobi-PCG with the solver state resident in shared
// memory, for Kronecker grids small enough that every CTA of one cooperative
// wave can hold its own column block (config 0, config 2: 66 x 66 x 17 free
// DOF on 121 CTAs of 6 x 6 x 17).
//
// Reference: pcg_jacobi (proj/src/sparse.cpp:41-100) on A = M/dt + theta K
// (DirichletSystem, proj/src/assembly.cpp:186-281). The iterates are the
// scaled Chronopoulos-Gear recurrences of k2_cg1_kernel (k2_kron.cu): the
// reference's PCG in exact arithmetic, the same stop test, warm start, b = 0
// reset and failure codes, and per point the same band sums in the same
// order. On such grids the streaming kernel is latency bound (~15 us per
// iteration on config 2: a TMA pipeline of 3-plane segments per CTA plus the
// grid reduction). Here a CTA owns a TX x TY x nz column block and keeps u,
// s^ and w^ on the block plus a P-wide halo, and x, p, d, 1/d on the block, in
// shared memory for the whole solve. Per iteration:
//   prologue  s^ = w^ + beta s^, u -= alpha s^ on block + halo (the halo
//             copies are recomputed redundantly, so they equal the owner's),
//             p, x and the dot products r.u, r.r on the block;
//   stencil   w^ = D^-1 A u on the block (x-, y-, z-passes in shared memory);
//   exchange  the block's w^ to a global buffer (L2), one grid reduction of
//             (r.u, (Au).u, r.r) whose barrier also publishes the buffer, the
//             halo of w^ read back from it — the only value a CTA cannot
//             recompute (the same split as the multi-GPU slab solver).
// HBM is touched only for x, rhs and the L2-resident exchange buffers.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "context.hpp"
#include "k2_kron.cuh"

namespace cg = cooperative_groups;

namespace tgb {

namespace {

// threads per CTA: 512 on blocks of >= 6 x 6 columns (config 2: 8.9 against
// 10.4 us per iteration with 256), 256 on smaller ones
constexpr int res_threads(int tb) { return tb >= 6 ? 512 : 256; }

__device__ __forceinline__ double res_recip(double d) {  // as k2_kron.cu's recip
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// Shared-memory layout of one CTA (doubles), from the tile shape.
struct ResLayout {
  int TX, TY, nz, P;
  int RX, RY, RZ;  // halo'd extents
  int NH, N1, N2, NO;
  int u, s, w, u1, u2, s1, s2, x, p, d, rd, mx, kx, my, ky, mz, kz, red, total;
  __host__ __device__ void make(int tx, int ty, int z, int p_) {
    TX = tx;
    TY = ty;
    nz = z;
    P = p_;
    RX = TX + 2 * P;
    RY = TY + 2 * P;
    RZ = nz + 2 * P;
    NH = RX * RY * RZ;
    N1 = RZ * RY * TX;
    N2 = RZ * TY * TX;
    NO = nz * TY * TX;
    const int W = 2 * P + 1;
    int o = 0;
    auto take = [&](int n) {
      const int at = o;
      o += (n + 1) & ~1;  // 16-byte aligned arrays
      return at;
    };
    u = take(NH);
    s = take(NH);
    w = take(NH);
    u1 = take(N1);
    u2 = take(N1);
    s1 = take(N2);
    s2 = take(N2);
    x = take(NO);
    p = take(NO);
    d = take(NO);
    rd = take(NO);
    mx = take(TX * W);
    kx = take(TX * W);
    my = take(TY * W);
    ky = take(TY * W);
    mz = take(nz * W);
    kz = take(nz * W);
    red = take(64);
    total = o;
  }
};

struct ResArgs {
  double* wx[2];     // exchange buffers of w^ (free grid)
  double* ux;        // exchange buffer of u_0
  double* partials;  // >= 8 * blocks
  PcgStatus* status;
  int TX, TY, ntx, nty;
};

struct NoAfter {
  __device__ void operator()(int, int) const {}
};
// block-reduce acc (fixed tree), grid sync, sum the per-block partials in
// block order (k2_kron.cu's grid_reduce, deterministic). after(t, nt) runs on
// the other warps (t = 0 .. nt-1) while warp 0 sums the partials: the halo
// read-back overlaps the partial-sum read (both L2 round trips).
template <int NT, class After = NoAfter>
__device__ __forceinline__ void res_reduce(cg::grid_group& grid, const double (&acc)[4],
                                           double* partials, int& buf, double* red,
                                           double (&out)[4], After after = {}) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
    for (int w = 0; w < NT / 32; ++w) s += red[w * 4 + tid];
    pb[blockIdx.x * 4 + tid] = s;
  }
  grid.sync();
  if (warp == 0) {
double s[4];
    warp_sum_partials(pb, static_cast<int>(gridDim.x), lane, s);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 4; ++c) red[32 + c] = s[c];
  } else {
    after(tid - 32, NT - 32);
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = red[32 + c];
  // (no barrier here: red is next written by the following reduction, after
  // the block barriers of the prologue and the stencil passes)
  buf ^= 1;
}

// TB x TB column blocks (compile-time, so the index arithmetic of the
// flattened loops is by constants)
template <int P, int TB, int NT = res_threads(TB)>
__global__ void __launch_bounds__(NT, 1)
    k2_res_kernel(KronGrid g, double a, double b, const double* __restrict__ rhs, double* x,
                  ResArgs R, double tol, int max_iter) {
  constexpr int W = 2 * P + 1;
  constexpr int TX = TB, TY = TB, RX = TB + 2 * P, RY = TB + 2 * P;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  ResLayout L;
  L.make(TX, TY, g.n[2], P);
  const int tid = threadIdx.x;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int x0 = (blockIdx.x % R.ntx) * TX, y0 = (blockIdx.x / R.ntx) * TY;
  double* U = sm + L.u;
  double* S = sm + L.s;
  double* Wv = sm + L.w;
  double* U1 = sm + L.u1;
  double* U2 = sm + L.u2;
  double* S1 = sm + L.s1;
  double* S2 = sm + L.s2;
  double* X = sm + L.x;
  double* Pp = sm + L.p;
  double* Dd = sm + L.d;
  double* Rd = sm + L.rd;
  double* red = sm + L.red;
  const bool lead = blockIdx.x == 0 && tid == 0;

  // 1D band rows of the block, the z band, the block's diagonal, x
  for (int e = tid; e < TX * W; e += NT) {
    const int i = x0 + e / W;
    sm[L.mx + e] = i < nx ? g.M[0][x0 * W + e] : 0.0;
    sm[L.kx + e] = i < nx ? g.K[0][x0 * W + e] : 0.0;
  }
  for (int e = tid; e < TY * W; e += NT) {
    const int j = y0 + e / W;
    sm[L.my + e] = j < ny ? g.M[1][y0 * W + e] : 0.0;
    sm[L.ky + e] = j < ny ? g.K[1][y0 * W + e] : 0.0;
  }
  for (int e = tid; e < nz * W; e += NT) {
    sm[L.mz + e] = g.M[2][e];
    sm[L.kz + e] = g.K[2][e];
  }
  __syncthreads();
  // own point o = (k TY + ly) TX + lx; halo'd point h = ((k+P) RY + ly+P) RX + lx+P
  auto own_h = [&](int o) {
    const int lx = o % TX, t = o / TX, ly = t % TY, k = t / TY;
    return ((k + P) * RY + ly + P) * RX + lx + P;
  };
  auto own_f = [&](int o, bool& in) {
    const int lx = o % TX, t = o / TX, ly = t % TY, k = t / TY;
    const int i = x0 + lx, j = y0 + ly;
    in = i < nx && j < ny;
    return (static_cast<size_t>(k) * ny + j) * nx + i;
  };
  for (int o = tid; o < L.NO; o += NT) {
    bool in;
    const size_t f = own_f(o, in);
    const int lx = o % TX, t = o / TX, ly = t % TY, k = t / TY;
    double dv = 1.0;
    if (in) {  // d = a (mx my) mz + b ((kx my + mx ky) mz + (mx my) kz), k2_kron.cu's order
      const double mm = sm[L.mx + lx * W + P] * sm[L.my + ly * W + P];
      const double km = fma(sm[L.kx + lx * W + P], sm[L.my + ly * W + P],
                            sm[L.mx + lx * W + P] * sm[L.ky + ly * W + P]);
      const double mz = sm[L.mz + k * W + P], kz = sm[L.kz + k * W + P];
      dv = fma(a, mm * mz, b * fma(km, mz, mm * kz));
    }
    Dd[o] = dv;
    Rd[o] = res_recip(dv);
    X[o] = in ? x[f] : 0.0;
    Pp[o] = 0.0;
  }
  // halo'd load of a global vector (zero outside the grid); ring_only: keep
  // the block's own values
  auto load_halo_part = [&](double* dst, const double* src, bool ring_only, int t0, int nt) {
    // (the z halo planes lie outside the grid: zero from the start, skipped)
    for (int e = t0 + P * RX * RY; e < (P + nz) * RX * RY; e += nt) {
      const int hx = e % RX, t = e / RX, hy = t % RY, hz = t / RY;
      const bool own = hx >= P && hx < P + TX && hy >= P && hy < P + TY;
      if (ring_only && own) continue;
      const int i = x0 + hx - P, j = y0 + hy - P, k = hz - P;
      dst[e] = (i >= 0 && i < nx && j >= 0 && j < ny && k >= 0 && k < nz)
                   ? src[(static_cast<size_t>(k) * ny + j) * nx + i]
                   : 0.0;
    }
  };
  auto load_halo = [&](double* dst, const double* src, bool ring_only) {
    load_halo_part(dst, src, ring_only, tid, NT);
  };
  // y = Op(a, b) v on the block; epi(o, f, y) per own point in the grid
  auto stencil = [&](const double* v, auto&& epi) {
    for (int e = tid + P * RY * TX; e < (P + nz) * RY * TX; e += NT) {  // x-pass
      const int lx = e % TX, r = e / TX;             // r = hz RY + hy
      const double* row = v + r * RX + lx;
      double a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int d = 0; d < W; ++d) {
        const double vv = row[d];
        a1 = fma(sm[L.mx + lx * W + d], vv, a1);
        a2 = fma(sm[L.kx + lx * W + d], vv, a2);
      }
      U1[e] = a1;
      U2[e] = a2;
    }
    __syncthreads();
    for (int e = tid + P * TY * TX; e < (P + nz) * TY * TX; e += NT) {  // y-pass
      const int lx = e % TX, t = e / TX, ly = t % TY, hz = t / TY;
      const int base = (hz * RY + ly) * TX + lx;
      double w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
      for (int d = 0; d < W; ++d) {
        const double p1 = U1[base + d * TX];
        w1 = fma(sm[L.my + ly * W + d], p1, w1);
        w2 = fma(sm[L.my + ly * W + d], U2[base + d * TX], w2);
        w3 = fma(sm[L.ky + ly * W + d], p1, w3);
      }
      S1[e] = fma(a, w1, fma(b, w2 + w3, 0.0));
      S2[e] = fma(b, w1, 0.0);
    }
    __syncthreads();
    for (int o = tid; o < L.NO; o += NT) {  // z-pass
      bool in;
      const size_t f = own_f(o, in);
      if (!in) continue;
      const int lxy = o % (TX * TY), k = o / (TX * TY);
      double y = 0.0;
#pragma unroll
      for (int d = 0; d < W; ++d)
        y = fma(sm[L.mz + k * W + d], S1[(k + d) * TX * TY + lxy],
                fma(sm[L.kz + k * W + d], S2[(k + d) * TX * TY + lxy], y));
      epi(o, f, y);
    }
  };

  int buf = 0;
  double tot[4];
  // every halo'd array starts at zero (the z halo planes stay zero), then
  // r0 = b - A x0 (sparse.cpp:61-69), u0 = D^-1 r0; r.r, b.b, r.u
  for (int e = tid; e < L.x; e += NT) sm[e] = 0.0;
  __syncthreads();
  load_halo(U, x, false);
  __syncthreads();
  {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // (the epilogue writes U's own points after the x-pass has read them)
    stencil(U, [&](int o, size_t f, double y) {
      const double bi = rhs[f];
      const double ri = bi - y;
      const double ui = ri * Rd[o];
      U[own_h(o)] = ui;
      R.ux[f] = ui;
      acc[0] += ri * ri;
      acc[1] += bi * bi;
      acc[2] += ri * ui;
    });
    res_reduce<NT>(grid, acc, R.partials, buf, red, tot,
               [&](int t, int nt) { load_halo_part(U, R.ux, true, t, nt); });
  }
  const double bnorm = sqrt(tot[1]);
  auto write_x = [&] {
    for (int o = tid; o < L.NO; o += NT) {
      bool in;
      const size_t f = own_f(o, in);
      if (in) x[f] = X[o];
    }
  };
  if (bnorm == 0.0) {  // sparse.cpp:57-60: zero rhs resets even a warm start
    for (int o = tid; o < L.NO; o += NT) X[o] = 0.0;
    write_x();
    if (lead) *R.status = PcgStatus{0, 0, 0.0, 0.0};
    return;
  }
  double rel = sqrt(tot[0]) / bnorm;
  if (max_iter <= 0 || rel <= tol) {  // the reference tests before its first matvec
    if (lead) *R.status = PcgStatus{0, max_iter <= 0 ? 3 : 0, rel, bnorm};
    return;
  }
  double gamma = tot[2];
  // the halo of u0 (the rows outside the grid stay zero), then w^0 = D^-1 A u0
  // and delta0 = (A u0).u0
  {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    stencil(U, [&](int o, size_t f, double y) {
      const double wv = y * Rd[o];
      Wv[own_h(o)] = wv;
      R.wx[0][f] = wv;
      acc[0] = fma(y, U[own_h(o)], acc[0]);
    });
    res_reduce<NT>(grid, acc, R.partials, buf, red, tot,
               [&](int t, int nt) { load_halo_part(Wv, R.wx[0], true, t, nt); });
  }
  int it = 0, status = 3;
  if (!(tot[0] > 0.0)) {
    if (lead) *R.status = PcgStatus{0, 4, rel, bnorm};
    return;
  }
  double alpha = gamma / tot[0], beta = 0.0;
  int cur = 0;
  while (it < max_iter) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // prologue on block + halo: s^_i = w^_i + beta s^_{i-1}, u_{i+1} = u_i -
    // alpha s^_i; on the block also p_i, x_{i+1} and r.u, r.r of r_{i+1}
    for (int e = tid + P * RX * RY; e < (P + nz) * RX * RY; e += NT) {
      const double uo = U[e];
      const double sn = fma(beta, S[e], Wv[e]);
      const double un = fma(-alpha, sn, uo);
      S[e] = sn;
      U[e] = un;
      const int hx = e % RX, t = e / RX, hy = t % RY, hz = t / RY;
      const int lx = hx - P, ly = hy - P, k = hz - P;
      if (lx >= 0 && lx < TX && ly >= 0 && ly < TY && k >= 0 && k < nz && x0 + lx < nx &&
          y0 + ly < ny) {
        const int o = (k * TY + ly) * TX + lx;
        const double pn = fma(beta, Pp[o], uo);  // p_i = u_i + beta p_{i-1}
        Pp[o] = pn;
        X[o] = fma(alpha, pn, X[o]);             // x_{i+1}
        const double ru = Dd[o] * un;            // r_{i+1} = D u_{i+1}
        acc[0] = fma(ru, un, acc[0]);
        acc[2] = fma(ru, ru, acc[2]);
      }
    }
    __syncthreads();
    // w^_{i+1} = D^-1 A u_{i+1} and (A u).u on the block
    double* wout = R.wx[cur ^ 1];
    stencil(U, [&](int o, size_t f, double y) {
      const double wv = y * Rd[o];
      Wv[own_h(o)] = wv;
      wout[f] = wv;
      acc[1] = fma(y, U[own_h(o)], acc[1]);
    });
    res_reduce<NT>(grid, acc, R.partials, buf, red, tot,
               [&](int t, int nt) { load_halo_part(Wv, wout, true, t, nt); });
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
    if (stop) break;
    const double g1 = tot[0];
    beta = g1 / gamma;
    const double den = tot[1] - beta * g1 / alpha;  // p_{i+1}.A p_{i+1}
    if (!(den > 0.0)) {
      status = 4;
      break;
    }
    alpha = g1 / den;
    gamma = g1;
  }
  write_x();
  if (lead) *R.status = PcgStatus{it, status, rel, bnorm};
}

constexpr int kResShapes[] = {2, 4, 6, 8, 12};  // block edges instantiated

#define TG_RES_TB(TB_, ...)                                                 \
  switch (TB_) {                                                            \
    case 2: { constexpr int TB = 2; __VA_ARGS__; break; }                   \
    case 4: { constexpr int TB = 4; __VA_ARGS__; break; }                   \
    case 6: { constexpr int TB = 6; __VA_ARGS__; break; }                   \
    case 8: { constexpr int TB = 8; __VA_ARGS__; break; }                   \
    case 12: { constexpr int TB = 12; __VA_ARGS__; break; }                 \
    default: throw std::invalid_argument("resident solve: no such block"); \
  }
#define TG_RES_DISPATCH(P_, TB_, ...)                                            \
  switch (P_) {                                                                  \
    case 1: { constexpr int P = 1; TG_RES_TB(TB_, __VA_ARGS__); break; }         \
    case 2: { constexpr int P = 2; TG_RES_TB(TB_, __VA_ARGS__); break; }         \
    case 3: { constexpr int P = 3; TG_RES_TB(TB_, __VA_ARGS__); break; }         \
    default: throw std::invalid_argument("kronecker path supports degree 1..3"); \
  }

}  // namespace

// Tile shape for the resident solve: the smallest per-CTA block (then the
// squarest) whose tile count fits one cooperative wave at 1 CTA per SM and
// whose layout fits the shared memory; false when none does.
bool k2_res_plan(const KronGrid& g, int sm_count, int max_smem, K2ResPlan* out) {
  if (std::getenv("TG_K2_NO_RESIDENT")) return false;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  long best = -1;
  int bh = 0;
  K2ResPlan pl{};
  for (const int tx : kResShapes)
    for (const int ty : {tx}) {
      const int ntx = (nx + tx - 1) / tx, nty = (ny + ty - 1) / ty;
      if (static_cast<long>(ntx) * nty > sm_count) continue;
      ResLayout L;
      L.make(tx, ty, nz, g.p);
      if (static_cast<long>(L.total) * 8 > max_smem) continue;
      const long own = static_cast<long>(tx) * ty;
      if (best < 0 || own < best || (own == best && L.NH < bh)) {
        best = own;
        bh = L.NH;
        pl = K2ResPlan{tx, ty, ntx, nty, static_cast<size_t>(L.total) * 8};
      }
    }
  if (best < 0) return false;
  *out = pl;
  return true;
}

void k2_res_solve(const KronGrid& g, double a, double b, const double* rhs, double* x,
                  const K2ResWork& w, const K2ResPlan& pl, double tol, int max_iter,
                  cudaStream_t s) {
  ResArgs R{{w.wx[0], w.wx[1]}, w.ux, w.partials, w.status, pl.TX, pl.TY, pl.ntx, pl.nty};
  KronGrid gg = g;
  double aa = a, bb = b, tt = tol;
  int mi = max_iter;
  void* args[] = {&gg, &aa, &bb, const_cast<double**>(&rhs), &x, &R, &tt, &mi};
  dim3 grid(pl.ntx * pl.nty);
  TG_RES_DISPATCH(g.p, pl.TX, {
    TG_CUDA(cudaFuncSetAttribute(k2_res_kernel<P, TB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(pl.smem)));
    TG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k2_res_kernel<P, TB>),
                                        grid, dim3(res_threads(TB)), args, pl.smem, s));
  });
}

}  // namespace tgb
