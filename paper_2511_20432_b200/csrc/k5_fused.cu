// K5 — sum-factorised superposition on tensor-grid point sets, fused.
//
// The reference evaluates the flux integrand and the Dirichlet data pair by
// pair: superpose (proj/src/analytic.cpp:92-109) at every lateral face
// quadrature point (assemble_flux_load, proj/src/assembly.cpp:148-166) and at
// every bottom Greville point (dirichlet_values, proj/src/mesh.cpp:238-264).
// On an axis-aligned patch those point sets are tensor grids and the point
// source factorises along the axes,
//   c e^{-r.r/s} = c e^{-dn^2/s} e^{-du^2/s} e^{-dv^2/s},
// so over the na x nb points of a grid the sum over sources is one dense
// contraction G = A B with A[a][j] = c_j e^{-dn_j^2/s_j} (x -dn_j / (2 alpha
// dt_j) for the normal flux) e^{-du_aj^2/s_j} and B[j][b] = e^{-dv_bj^2/s_j}.
//
// The pair-wise cull (skip iff r.r/s > cull) does not factorise. Every grid
// is cut into regions (one per CTA tile of the contraction; per face, the
// step's fine-rule rectangle); per region, on the device:
//   J = the longest source prefix no cull can reach anywhere in the region's
//       box (sf_source_ok) -> the contraction;
//   E = one past the last source not culled on the whole box -> sources
//       [J, E) run pair by pair with the reference's exact cull (K1 with
//       per-CTA ranges); later sources are exact zeros there.
// Reference zeros therefore stay exact zeros, and a factorised term is within
// a few ulps of the reference's (table exponentials with a cubic, max relative
// error 1.1e-16, instead of one libm exp), far inside the 1e-10 flux / T~
// tolerance.
//
// The contraction never leaves the chip: A and B are generated per 32-source
// stage straight into shared memory (the exponential in 10 FP64 instructions
// per entry, 7 for B when every source lies on the grid's V plane) and
// contracted on the FP64 tensor cores with mma.sync m8n8k4 (DMMA; tcgen05 has
// no FP64 kind). DMMA and DFMA issue from one FP64 pipe on this part
// (tools/dmma_pipe.cu: 37.0 TF/s DMMA alone, 34.1 DFMA alone, ~35 mixed), so
// the generator's share is set by the tile shape (128 x 192: ~1/10 of the
// pipe time on exponentials), with 16 warps per SM issuing DMMA. Work is split stream-K style: the
// (tile, 1024-source) items of all tiles are cut evenly over one CTA per SM;
// a CTA accumulates its run of a tile's items in registers and writes one
// partial tile; the epilogue sums the partials in CTA order (deterministic).
#include <cmath>

#include <algorithm>

#include "common.cuh"
#include "context.hpp"
#include "k5_fused.cuh"

namespace tgb {

namespace {

// the cubic of sf_exp (below)
constexpr double kSfE0 = 0x1.fffffffffffffp-1;
constexpr double kSfE1 = 0x1.62e42fefa39efp-11;
constexpr double kSfE2 = 0x1.ebfbe046f706bp-23;
constexpr double kSfE3 = 0x1.c6b08d9bfb0bdp-35;

// ---------------------------------------------------------------- sources
// The region tests of the old host path (k5_sumfact.cu), on the device:
// eligible = no point of the box can be culled and the grid rounding moves
// no term by more than ~1e-12; culled = every point of the box is culled.
__device__ __forceinline__ bool sf_source_ok(const double* p, double t, double alpha,
                                             double cull, const SfRegion& r) {
  const double dt = t - p[5];
  if (!(dt > 0.0)) return true;  // skipped by the reference: a zero column here
  const double spread = 4.0 * alpha * dt;
  double r2 = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double a = r.lo[ax] - r.delta - p[ax], b = r.hi[ax] + r.delta - p[ax];
    r2 += fmax(a * a, b * b);
  }
  if (!(r2 * (1.0 + 1e-9) <= cull * spread)) return false;
  return 36.0 * cull * r.delta * r.delta <= 1e-24 * spread;
}

__device__ __forceinline__ bool sf_source_culled(const double* p, double t, double alpha,
                                                 double cull, const SfRegion& r) {
  const double dt = t - p[5];
  if (!(dt > 0.0)) return true;
  const double spread = 4.0 * alpha * dt;
  double r2 = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double d = fmax(fmax(r.lo[ax] - r.delta - p[ax], p[ax] - r.hi[ax] - r.delta), 0.0);
    r2 += d * d;
  }
  return r2 * (1.0 - 1e-9) > cull * spread;
}

__device__ __forceinline__ int block_min_int(int v, int* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int m = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = min(m, red[w]);
  __syncthreads();
  return m;
}

__device__ __forceinline__ int block_max_int(int v, int* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int m = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = max(m, red[w]);
  __syncthreads();
  return m;
}

// The plan in two passes over (region, source chunk) CTAs (integer min / max
// through atomics: order-independent, so deterministic):
//   pass 1: Jraw[r] = the first source failing sf_source_ok (n_act if none);
//   pass 2: J[r] = Jraw, or 0 when the contraction would not pay; E[r] = one
//           past the last source in [J, n_act) not culled on the box.
constexpr int kPlanChunks = 16;

__device__ __forceinline__ bool plan_active(const SfPlanMask& mask, int ri) {
  const bool part = ri < mask.nt_flux ? mask.flux : ri < mask.nt_static ? mask.dir : mask.flux;
  return part && ri % mask.world == mask.rank;
}

__global__ void sf_plan_init_kernel(int n, int n_act, int* __restrict__ Jraw,
                                    int* __restrict__ Eo) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) {
    Jraw[r] = n_act;
    Eo[r] = 0;
  }
}

__global__ void sf_plan_j_kernel(SfPlanArgs a, const SfRegion* __restrict__ regions,
                                 int* __restrict__ Jraw, SfPlanMask mask) {
  __shared__ int red[32];
  const int ri = blockIdx.x;
  if (!a.gemm || !plan_active(mask, ri)) return;
  const SfRegion r = regions[ri];
  const int L = (a.n_act + kPlanChunks - 1) / kPlanChunks;
  const int j0 = blockIdx.y * L, j1 = min(a.n_act, j0 + L);
  int J = a.n_act;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x)
    if (!sf_source_ok(a.src6 + 6 * static_cast<size_t>(j), a.t, a.alpha, a.cull, r)) {
      J = j;
      break;
    }
  J = block_min_int(J, red);
  if (threadIdx.x == 0 && J < a.n_act) atomicMin(&Jraw[ri], J);
}

__global__ void sf_plan_e_kernel(SfPlanArgs a, const SfRegion* __restrict__ regions,
                                 const int* __restrict__ Jraw, int* __restrict__ Jo,
                                 int* __restrict__ Eo, SfPlanMask mask, int n_static,
                                 int* __restrict__ Jl, int* __restrict__ El) {
  __shared__ int red[32];
  const int ri = blockIdx.x;
  const bool act = plan_active(mask, ri);
  const SfRegion r = regions[ri];
  int J = 0;
  if (act && a.gemm) {
    J = Jraw[ri];
    if (r.npts < 0.0 || (static_cast<double>(J) * r.npts < a.min_pairs && J < a.min_sources))
      J = 0;
  }
  int last = J - 1;
  if (act) {
    const int L = (a.n_act + kPlanChunks - 1) / kPlanChunks;
    const int j0 = max(J, blockIdx.y * L), j1 = min(a.n_act, (blockIdx.y + 1) * L);
    for (int j = j1 - 1 - static_cast<int>(threadIdx.x); j >= j0; j -= blockDim.x)
      if (!sf_source_culled(a.src6 + 6 * static_cast<size_t>(j), a.t, a.alpha, a.cull, r)) {
        last = j;
        break;
      }
    last = block_max_int(last, red);
  }
  if (threadIdx.x == 0) {
    if (blockIdx.y == 0) {
      Jo[ri] = act ? J : 0;
      if (Jl && ri < n_static && act) Jl[ri] = J;
    }
    if (act) atomicMax(&Eo[ri], max(J, last + 1));
  }
}

// the static regions' last computed E (queries), after pass 2
__global__ void sf_plan_keep_kernel(int n_static, const int* __restrict__ Eo, SfPlanMask mask,
                                    int* __restrict__ El) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n_static && El && plan_active(mask, r)) El[r] = Eo[r];
}

// the eligible sources of [J, E) per region, in order (one CTA per region)
__global__ void sf_plan_list_kernel(SfPlanArgs a, const SfRegion* __restrict__ regions,
                                    const int* __restrict__ Jo, const int* __restrict__ Eo,
                                    SfLists L, SfPlanMask mask, int n_static) {
  __shared__ int wcount[8];
  const int ri = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int J = Jo[ri], E = Eo[ri];
  int count = 0;
  if (J > 0) {
    const SfRegion r = regions[ri];
    int* el = L.elist + static_cast<size_t>(ri) * L.cap;
    unsigned* bits = L.okbits + static_cast<size_t>(ri) * L.words;
    for (int base = J; base < E; base += 256) {
      const int j = base + tid;
      const bool ok =
          j < E && sf_source_ok(a.src6 + 6 * static_cast<size_t>(j), a.t, a.alpha, a.cull, r);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) {
        wcount[warp] = __popc(m);
        if (base - J + 32 * warp < E - J) bits[((base - J) >> 5) + warp] = m;
      }
      __syncthreads();
      int pos = count + __popc(m & ((1u << lane) - 1u)), tot = 0;
      for (int w = 0; w < 8; ++w) {
        if (w < warp) pos += wcount[w];
        tot += wcount[w];
      }
      if (ok) el[pos] = j;
      count += tot;
      __syncthreads();
    }
  }
  if (tid == 0) {
    L.Jc[ri] = J + count;
    if (L.Jclast && ri < n_static && plan_active(mask, ri)) L.Jclast[ri] = J + count;
  }
}

// item prefix over the tiles (one CTA; a serial scan is plenty for <= a few
// thousand tiles)
__global__ void sf_items_kernel(const SfTile* __restrict__ tiles, int n, const int* __restrict__ Jc,
                                int* __restrict__ prefix, double* __restrict__ stats) {
  if (threadIdx.x != 0) return;
  int acc = 0;
  double flops = 0.0;
  for (int t = 0; t < n; ++t) {
    prefix[t] = acc;
    const SfTile tl = tiles[t];
    if (tl.na > 0 && tl.nb > 0) {
      const int j = Jc[tl.region];
      acc += (j + kSfItem - 1) / kSfItem;
      flops += 2.0 * tl.na * tl.nb * static_cast<double>(j);
    }
  }
  prefix[n] = acc;
  if (stats) stats[0] += flops;
}

// per (grid, source): the factor constants (SfConst)
__global__ void sf_prep_kernel(const double* __restrict__ src6, int n_act, double t, double alpha,
                               double rcp, const SfGridDesc* __restrict__ grids, int max_src,
                               SfConst* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const SfGridDesc g = grids[blockIdx.y];
  if (j >= max_src) return;
  SfConst c{0.0, 0.0, 0.0, kExpMagic, 0.0, 0.0, 0.0, 0.0};
  if (j < n_act) {
    const double* p = src6 + 6 * static_cast<size_t>(j);
    c.u = p[g.axu];
    c.v = p[g.axv];
    const double dt = t - p[5];
    const double dn = g.xf - p[g.axn];
    if (dt > 0.0 && p[3] > 0.0 && !(g.flux && dn == 0.0)) {
      const double spread = 4.0 * alpha * dt;
      const double lnc = log(p[3] / (rcp * pow(M_PI * spread, 1.5)));
      // |A factor| = exp(lnf): c e^{-dn^2/s} (x |dn| / (2 alpha dt) for the flux)
      double lnf = lnc - dn * dn / spread;
      double sign = 1.0;
      if (g.flux) {
        lnf += log(fabs(dn) / (2.0 * alpha * dt));
        sign = dn > 0.0 ? -1.0 : 1.0;  // fac = dn (-e / (2 alpha dt))
      }
      const double L = rint(lnf * kExpInvStep);
      double u = fma(-L, kExpStepHi, lnf);
      u = fma(-L, kExpStepLo, u);
      const double C = sign * exp(u);
      c.nisp = -kExpInvStep / spread;
      c.magicL = L + kExpMagic;
      c.q0 = C * kSfE0;
      c.q1 = C * kSfE1;
      c.q2 = C * kSfE2;
      c.pad = C * kSfE3;
    }
  }
  out[static_cast<size_t>(blockIdx.y) * max_src + j] = c;
}

// ---------------------------------------------------------------- contraction
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// C exp(y) with y = r2 nisp + (magicL - magic) ln2/1024: src_exp's
// representation (common.cuh) with a cubic instead of its quadratic, the
// near-minimax fit of 2^(f/1024) on |f| <= 1/2 (Chebyshev nodes, mpmath): max
// relative error 1.1e-16, so a factorised term stays within a few ulps of the
// reference's single libm exp
__device__ __forceinline__ double sf_exp(double r2, double nisp, double magicL, double q0,
                                         double q1, double q2, double q3,
                                         const double* __restrict__ tab) {
  const double kf = __fma_rn(r2, nisp, magicL);
  const double d = __dsub_rn(magicL, kf);  // L - k, exact
  const double f = __fma_rn(r2, nisp, d);
  const double q = __fma_rn(__fma_rn(__fma_rn(q3, f, q2), f, q1), f, q0);
  const int ki = __double2loint(kf);
  const double t = tab[ki & (kExpTableSize - 1)];
  const double sc = __hiloint2double(
      __double2hiint(t) + static_cast<int>(static_cast<unsigned>(ki) << (20 - kExpBits)),
      __double2loint(t));  // 2^(k/1024), exact
  return __dmul_rn(sc, q);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

constexpr int kLd = kSfKS + 4;  // row pitch (doubles) of the A / B stages: conflict-free frags
constexpr int kWarps = kSfWarps;
constexpr int kWR = kSfWR;
constexpr int kWN = kSfWN;
constexpr int kNT = kWN / 8;                  // n8 fragments per warp
static_assert(kSfTA % 32 == 0 && kWarps % kWR == 0 && kWN % 8 == 0, "warp tiling");

struct SfSmem {
  double tab[kExpTableSize];
  double A[2][kSfTA][kLd];
  double B[2][kSfTB][kLd];
  double cs[2][8][kSfKS];  // the stage's SfConst fields, field-major (conflict-free reads)
  double U[kSfTA];
  double V[kSfTB];  // V[b], or cb[b] for vplane grids
};

__global__ void __launch_bounds__(kSfThreads, kSfMinBlocks)
    sf_contract_kernel(const SfGridDesc* __restrict__ grids, const SfTile* __restrict__ tiles,
                       int n_tiles, const int* __restrict__ prefix, const int* __restrict__ J,
                       SfLists L, const SfConst* __restrict__ cst, int max_src,
                       const double* __restrict__ tab_g, double* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SfSmem& sm = *reinterpret_cast<SfSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp tile: rows [32 wa, +32), cols [kWN wb, +kWN); small warp tiles keep
  // the accumulators at 48 registers so 16 warps per SM issue DMMA (a warp
  // issues one only every few cycles: 2 warps per SM sub-partition left the
  // tensor pipe half idle)
  int wa, wb;
  sf_warp_block(warp, wa, wb);
  static_assert(kSfTB == kWN * (kWarps / kWR), "the warps tile the CTA tile");
  const int g8 = lane >> 2, q4 = lane & 3;
  for (int i = tid; i < kExpTableSize; i += kSfThreads) sm.tab[i] = tab_g[i];

  const int total = prefix[n_tiles];
  const int C = gridDim.x, c = blockIdx.x;
  const int lo = static_cast<int>(static_cast<long long>(total) * c / C);
  const int hi = static_cast<int>(static_cast<long long>(total) * (c + 1) / C);
  int it = lo;
  while (it < hi) {
    // the tile of item `it`
    int tl = 0, th = n_tiles;  // prefix[tl] <= it < prefix[th]
    while (th - tl > 1) {
      const int m = (tl + th) >> 1;
      if (prefix[m] <= it) tl = m; else th = m;
    }
    const int t = tl;
    const SfTile T = tiles[t];
    const SfGridDesc G = grids[T.grid];
    const int seg_end = min(hi, prefix[t + 1]);
    const int j0 = (it - prefix[t]) * kSfItem;
    const int j1 = min(L.Jc[T.region], (seg_end - prefix[t]) * kSfItem);
    const int jp = J[T.region];  // positions >= jp: the eligible list
    const int* el = L.elist + static_cast<size_t>(T.region) * L.cap;
    const SfConst* cg = cst + static_cast<size_t>(T.grid) * max_src;
    __syncthreads();  // the previous segment is done with U / V
    for (int i = tid; i < kSfTA; i += kSfThreads) sm.U[i] = i < T.na ? G.U[T.a0 + i] : 0.0;
    for (int i = tid; i < kSfTB; i += kSfThreads)
      sm.V[i] = i < T.nb ? (G.vplane ? G.cb[T.b0 + i] : G.V[T.b0 + i]) : 0.0;
    // a warp whose whole block lies outside the tile skips the MMAs
    // (warp-uniform); partial blocks multiply rows / columns nobody reads
    const bool active = 32 * wa < T.na && kWN * wb < T.nb;

    double acc[4][kNT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jn = 0; jn < kNT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;

    const int n_stage = (j1 - j0 + kSfKS - 1) / kSfKS;
    // stage constants: thread tid loads field tid & 7 of source tid >> 3
    // (coalesced); padded sources get zero columns
    // (cp.async: the copy lands while the stage's MMAs run; each thread waits
    // for its own copies before the stage barrier that publishes them)
    auto load_cst = [&](int st, int buf) {
      for (int e = tid; e < 8 * kSfKS; e += kSfThreads) {
        const int j = j0 + st * kSfKS + (e >> 3), f = e & 7;
        // padding columns (j >= j1) read entry max_src - 1: always a zero factor
        const int js = j >= j1 ? max_src - 1 : (j < jp ? j : el[j - jp]);
        const double* src = reinterpret_cast<const double*>(cg + js);
        cp_async8(&sm.cs[buf][f][e >> 3], src + f);
      }
    };
    auto generate = [&](int buf) {
      SfConst k;
      k.u = sm.cs[buf][0][lane];
      k.v = sm.cs[buf][1][lane];
      k.nisp = sm.cs[buf][2][lane];
      k.magicL = sm.cs[buf][3][lane];
      k.q0 = sm.cs[buf][4][lane];
      k.q1 = sm.cs[buf][5][lane];
      k.q2 = sm.cs[buf][6][lane];
      k.pad = sm.cs[buf][7][lane];
      // every row / column is generated (those outside the tile read U / V =
      // 0 and land in cells nobody reads): no divergence, 32 independent
      // exponentials per thread
#pragma unroll
      for (int r = 0; r < (kSfTA + kWarps - 1) / kWarps; ++r) {  // A: rows warp + kWarps r, column lane
        const int a = warp + kWarps * r;
        if (kSfTA % kWarps == 0 || a < kSfTA) {  // (compile-time true for the default shape)
          const double d = sm.U[a] - k.u;
          sm.A[buf][a][lane] = sf_exp(d * d, k.nisp, k.magicL, k.q0, k.q1, k.q2, k.pad, sm.tab);
        }
      }
      if (G.vplane) {
#pragma unroll
        for (int r = 0; r < (kSfTB + kWarps - 1) / kWarps; ++r) {
          const int b = warp + kWarps * r;
          if (kSfTB % kWarps == 0 || b < kSfTB)
            sm.B[buf][b][lane] =
                sf_exp(sm.V[b], k.nisp, kExpMagic, kSfE0, kSfE1, kSfE2, kSfE3, sm.tab);
        }
      } else {
#pragma unroll
        for (int r = 0; r < (kSfTB + kWarps - 1) / kWarps; ++r) {
          const int b = warp + kWarps * r;
          if (kSfTB % kWarps == 0 || b < kSfTB) {
            const double d = sm.V[b] - k.v;
            sm.B[buf][b][lane] =
                sf_exp(d * d, k.nisp, kExpMagic, kSfE0, kSfE1, kSfE2, kSfE3, sm.tab);
          }
        }
      }
    };
    auto contract = [&](int buf) {
#pragma unroll
      for (int kk = 0; kk < kSfKS; kk += 4) {
        double af[4], bf[kNT];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = sm.A[buf][32 * wa + 8 * i + g8][kk + q4];
#pragma unroll
        for (int jn = 0; jn < kNT; ++jn) bf[jn] = sm.B[buf][kWN * wb + 8 * jn + g8][kk + q4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jn = 0; jn < kNT; ++jn) dmma884(acc[i][jn][0], acc[i][jn][1], af[i], bf[jn]);
      }
    };

    if (n_stage > 0) {
      load_cst(0, 0);
      cp_async_wait_all();
      __syncthreads();
      generate(0);
      if (n_stage > 1) load_cst(1, 1);
      cp_async_wait_all();
      __syncthreads();
      // one barrier per stage: the constants of stage st + 2 go into cs[buf]
      // (read by generate(st) before the previous barrier), stage st + 1 is
      // generated into buffer buf ^ 1 (last read by contract(st - 1)) beside
      // stage st's MMAs on buffer buf
      for (int st = 0; st < n_stage; ++st) {
        const int buf = st & 1;
        if (st + 2 < n_stage) load_cst(st + 2, buf);
        if (st + 1 < n_stage) generate(buf ^ 1);
        if (active) contract(buf);
        cp_async_wait_all();
        __syncthreads();
      }
    }
    // partial tile -> slot t + c (cell (a, b) at a + kSfTA b)
    double* out = scratch + static_cast<size_t>(t + c) * (kSfTA * kSfTB);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jn = 0; jn < kNT; ++jn) {
        const int a = 32 * wa + 8 * i + g8;
        const int b = kWN * wb + 8 * jn + 2 * q4;
        out[a + kSfTA * b] = acc[i][jn][0];
        out[a + kSfTA * (b + 1)] = acc[i][jn][1];
      }
    it = seg_end;
  }
}

// ---------------------------------------------------------------- epilogue
__global__ void sf_base_positions_kernel(int n, const int* __restrict__ q_of,
                                         const int* __restrict__ tile,
                                         const int* __restrict__ qelem,
                                         const int* __restrict__ qb_off,
                                         const int* __restrict__ elem_off,
                                         int* __restrict__ pos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (tile[i] < 0) {
    pos[i] = -1;
    return;
  }
  const int q = q_of[i];
  const int e = qelem[q];
  const int eo = elem_off[e];
  pos[i] = eo < 0 ? -1 : eo + (q - qb_off[e]);
}

// G at a tile cell: the partial tiles of the CTAs that processed the tile's
// items, in CTA order
__device__ __forceinline__ double sf_tile_value(const SfAddArgs& a, int t, int cell) {
  const int total = a.prefix[a.n_tiles];
  const int p0 = a.prefix[t], p1 = a.prefix[t + 1];
  if (p1 <= p0 || total == 0) return 0.0;
  const int C = a.ctas;
  // first CTA whose range holds item p0: largest c with floor(total c / C) <= p0
  int c = static_cast<int>((static_cast<long long>(p0) * C) / total);
  while (c + 1 < C && static_cast<long long>(total) * (c + 1) / C <= p0) ++c;
  while (c > 0 && static_cast<long long>(total) * c / C > p0) --c;
  double G = 0.0;
  for (; c < C && static_cast<long long>(total) * c / C < p1; ++c) {
    const long long lo = static_cast<long long>(total) * c / C;
    const long long hi = static_cast<long long>(total) * (c + 1) / C;
    if (hi <= lo) continue;  // an empty CTA range wrote nothing
    G += a.scratch[static_cast<size_t>(t + c) * (kSfTA * kSfTB) + cell];
  }
  return G;
}

__global__ void sf_add_kernel(SfAddArgs a, int e0, int e1, bool flux) {
  const int i = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e1) return;
  const int pos = a.ent.pos[i];
  if (pos < 0) return;
  const size_t n = static_cast<size_t>(a.n_entries);
  double v = 0.0, x = 0.0, y = 0.0, z = 0.0;
  for (int s = 0; s < a.S; ++s) {  // split order, as k1_combine_*
    const double* p = a.part + static_cast<size_t>(s) * 4 * n;
    v += p[i];
    x += p[n + i];
    y += p[2 * n + i];
    z += p[3 * n + i];
  }
  const int t = a.ent.tile[i];
  const double G = t >= 0 ? sf_tile_value(a, t, a.ent.cell[i]) : 0.0;
  if (flux) {
    const int q = a.ent.q[i];
    const double* nn = a.normals + 3 * static_cast<size_t>(q);
    const double w = a.weights[q];
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(x, nn[0]), __dmul_rn(y, nn[1])),
                                 __dmul_rn(z, nn[2]));
    double gq = __dmul_rn(__dmul_rn(-a.k, dot), w);
    if (t >= 0) {
      const int axn = a.grids[a.tiles[t].grid].axn;
      gq = __dadd_rn(gq, __dmul_rn(__dmul_rn(-a.k, __dmul_rn(G, nn[axn])), w));
    }
    a.gq[pos] = gq;
  } else {
    a.g[pos] = __dsub_rn(-v, G);
  }
}

}  // namespace

void sf_plan(const SfPlanArgs& a, const SfRegion* d_regions, int n_regions, int* d_J, int* d_E,
             const SfPlanMask& mask, int n_static_regions, int* d_Jlast, int* d_Elast,
             int* d_Jraw, const SfLists& lists, cudaStream_t s) {
  if (n_regions <= 0) return;
  sf_plan_init_kernel<<<(n_regions + 127) / 128, 128, 0, s>>>(n_regions, a.n_act, d_Jraw, d_E);
  const dim3 grid(n_regions, kPlanChunks);
  sf_plan_j_kernel<<<grid, 256, 0, s>>>(a, d_regions, d_Jraw, mask);
  sf_plan_e_kernel<<<grid, 256, 0, s>>>(a, d_regions, d_Jraw, d_J, d_E, mask, n_static_regions,
                                        d_Jlast, d_Elast);
  sf_plan_keep_kernel<<<(n_static_regions + 127) / 128, 128, 0, s>>>(n_static_regions, d_E, mask,
                                                                      d_Elast);
  sf_plan_list_kernel<<<n_regions, 256, 0, s>>>(a, d_regions, d_J, d_E, lists, mask,
                                                n_static_regions);
}

void sf_items(const SfTile* d_tiles, int n_tiles, const int* d_Jc, int* d_prefix, double* stats,
              cudaStream_t s) {
  sf_items_kernel<<<1, 32, 0, s>>>(d_tiles, n_tiles, d_Jc, d_prefix, stats);
}

void sf_prep(const double* d_src6, int n_act, double t, double alpha, double rcp,
             const SfGridDesc* d_grids, int n_grids, int max_src, SfConst* d_cst,
             cudaStream_t s) {
  if (n_grids <= 0 || max_src <= 0) return;
  dim3 grid((max_src + 255) / 256, n_grids);
  sf_prep_kernel<<<grid, 256, 0, s>>>(d_src6, n_act, t, alpha, rcp, d_grids, max_src, d_cst);
}

int sf_contract_max_ctas(int sm_count) { return kSfMinBlocks * sm_count; }

void sf_contract_fused(const SfGridDesc* d_grids, const SfTile* d_tiles, int n_tiles,
                       const int* d_prefix, const int* d_J, const SfLists& lists,
                       const SfConst* d_cst, int max_src, const double* d_tab, double* d_scratch,
                       int ctas, cudaStream_t s) {
  static bool attr = false;
  const size_t bytes = sizeof(SfSmem);
  if (!attr) {
    TG_CUDA(cudaFuncSetAttribute(sf_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
    attr = true;
  }
  sf_contract_kernel<<<ctas, kSfThreads, bytes, s>>>(d_grids, d_tiles, n_tiles, d_prefix, d_J,
                                                     lists, d_cst, max_src, d_tab, d_scratch);
}

void sf_base_positions(int n, const int* d_q, const int* d_tile, const int* d_qelem,
                       const int* d_qb_off, const int* d_elem_off, int* d_pos, cudaStream_t s) {
  if (n <= 0) return;
  sf_base_positions_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, d_q, d_tile, d_qelem, d_qb_off,
                                                          d_elem_off, d_pos);
}

void sf_add(const SfAddArgs& a, int e0, int e1, bool flux, cudaStream_t s) {
  if (e1 <= e0) return;
  sf_add_kernel<<<(e1 - e0 + 255) / 256, 256, 0, s>>>(a, e0, e1, flux);
}

}  // namespace tgb
