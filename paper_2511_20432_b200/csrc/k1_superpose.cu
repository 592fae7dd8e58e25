// K1 — batched point-source superposition of the analytic field T~ and its
// gradient (reference: superpose, proj/src/analytic.cpp:92-109).
//
// Layout and schedule (sm_100a):
//   * per call, k1_prepare_sources turns the history {x, y, z, E, t_act, tau}
//     into 96-byte SrcRec records holding every per-source, per-time constant
//     (the reference recomputes pow(pi*spread, 1.5) per pair, analytic.cpp:104);
//   * k1_partial: one thread owns P points (registers), a CTA owns 256*P points
//     and one contiguous source range; source records stream through a 3-stage
//     shared-memory ring filled by TMA bulk copies (cp.async.bulk + mbarrier)
//     and are read as warp-wide broadcasts;
//   * the source dimension is split into S ranges (grid.y) so that the grid
//     holds >= ~16 waves of CTAs on 148 SMs; k1_combine_* sums the S partials in
//     a fixed order (deterministic reruns) and applies the caller's epilogue
//     (plain field, -k dT/dn * w flux integrand, or -T Dirichlet value).
//
// Exactness: the causality test (t - tau > 0), the spread 4*alpha*dt and the
// cull decision fl(r.r / spread) > cull reproduce the reference's discrete
// choices bit for bit: the cull threshold thr_j is the largest double a with
// fl(a / spread_j) <= cull, found with IEEE division in the prologue; the
// per-pair decision compares the high words of an FMA-formed r.r with thr_j's
// and, only inside the +-1 high-word band, re-forms r.r with the reference's
// association and no FMA for the exact compare.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "k1_superpose.cuh"

namespace tgb {

__constant__ double c_exp_table[kExpTableSize];

__global__ void k1_prepare_sources(const double* __restrict__ src6, int n, double t,
                                   double alpha4, double alpha2, double rcp, double cull,
                                   SrcRec* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double* s = src6 + 6 * static_cast<size_t>(j);
  SrcRec r;
  r.sx = s[0];
  r.sy = s[1];
  r.sz = s[2];
  const double E = s[3];
  const double dt = __dsub_rn(t, s[5]);  // analytic.cpp:97
  bool active = dt > 0.0 && E > 0.0;     // E == 0 contributes exact zeros
  double spread = 1.0, lnc = 0.0, thr = -1.0;
  if (active) {
    spread = __dmul_rn(alpha4, dt);  // 4.0 * alpha * dt
    const double c = E / (rcp * pow(M_PI * spread, 1.5));
    lnc = log(c);
    // largest a with fl(a / spread) <= cull (exact cull decision)
    double a = cull < 0.0 ? -1.0 : __dmul_rn(cull, spread);
    if (a >= 0.0 && isfinite(a)) {
      for (int it = 0; it < 16 && a > 0.0 && __ddiv_rn(a, spread) > cull; ++it)
        a = __longlong_as_double(__double_as_longlong(a) - 1);  // next down (a > 0)
      for (int it = 0; it < 16; ++it) {
        const double b = __longlong_as_double(__double_as_longlong(a) + 1);  // next up
        if (isfinite(b) && __ddiv_rn(b, spread) <= cull) a = b; else break;
      }
    }
    // keep exp(lnc - r2/spread) in the normal range: contributions below
    // e^-707 relative to nothing are flushed (only reachable without culling)
    const double lim = (lnc + 707.0) * spread;
    if (!(lim > 0.0) || !(lnc < 709.0)) active = false;
    thr = fmin(a, lim);
  }
  if (!active) {
    spread = 1.0;
    lnc = 0.0;
    thr = -1.0;
  }
  // exponent constants of src_exp (common.cuh)
  const double L = rint(__dmul_rn(lnc, kExpInvStep));
  double u = __fma_rn(-L, kExpStepHi, lnc);
  u = __fma_rn(-L, kExpStepLo, u);
  const double C = exp(u);
  r.nisp = active ? -kExpInvStep / spread : 0.0;
  r.magicL = __dadd_rn(L, kExpMagic);
  r.gfac = active ? -1.0 / __dmul_rn(alpha2, dt) : 0.0;
  r.thr = thr;
  r.thr_lo = __double2hiint(thr) - 1;
  r.thr_hi = __double2hiint(thr) + 1;
  r.q0 = __dmul_rn(C, kExpD0);
  r.q1 = __dmul_rn(C, kExpD1);
  r.q2 = __dmul_rn(C, kExpD2);
  r.pad = 0.0;
  out[j] = r;
}

// tuning knobs (tools/k1_variants.py builds and times the alternatives)
#ifndef K1_UNROLL
#define K1_UNROLL 3  // measured (config 1, chunk fast path): 1 0.977e12, 2 0.978e12, 3 0.981e12, 4 0.959e12, 8 0.962e12 pairs/s
#endif
#ifndef K1_MINB4
#define K1_MINB4 2
#endif
#ifndef K1_VOTE_LATE  // 1: exponentials before the band vote, 0: after it
#define K1_VOTE_LATE 1
#endif
constexpr int kK1Unroll = K1_UNROLL;

// PLANAR: every source of the history lies on one plane z = zs (a layer's
// scan paths; k1_run checks it). Then rz = z - zs and fl(rz * rz) are per
// point — the reference's own values for every pair of that point — and the
// z-gradient is rz * sum_j w_j: two FP64 instructions fewer per pair.
// BOX (K5's remainder launch): per source chunk the CTA first drops the
// sources whose every pair with the CTA's points is culled — the squared
// distance from the source to the bounding box of those points exceeds the
// source's exact keep threshold (with a relative margin far above the box
// arithmetic's rounding) — and loops over the kept ones only. The dropped
// pairs are exact zeros in the reference too, and a kept source's pairs run
// the exact per-pair test below, so the sums are unchanged.
template <int P, bool GRAD, bool PLANAR, bool BOX = false>
__global__ void __launch_bounds__(kK1Threads,
                                  P >= 6 ? 256 / kK1Threads : (P >= 4 ? K1_MINB4 : 3))
    k1_partial(const SrcRec* __restrict__ src, int n_src, int split_len,
               const double* __restrict__ pts, const int* __restrict__ pt_index, int n_pts,
               double* __restrict__ part, double zs, K1Ranges rg) {
  __shared__ __align__(128) SrcRec ring[kK1Stages][kK1Chunk];
  __shared__ double tab[kExpTableSize];
  __shared__ __align__(8) uint64_t bars[kK1Stages];
  __shared__ double boxs[BOX ? 6 : 1];
  __shared__ int keep_list[BOX ? kK1Chunk : 1];
  __shared__ int keep_n[BOX ? kK1Chunk / 32 + 1 : 1];

  const int tid = threadIdx.x;
  const int s = blockIdx.y;
  int begin = s * split_len;
  int len = max(0, min(n_src, begin + split_len) - begin);
  if (rg.cta_region) {  // this CTA's points take their region's range [J, E) only
    const int r = rg.cta_region[blockIdx.x];
    const int J = rg.J[r], E = min(rg.E[r], n_src);
    const int L = (max(0, E - J) + gridDim.y - 1) / gridDim.y;
    begin = J + s * L;
    len = max(0, min(E, begin + L) - begin);
  }
  const int n_chunks = (len + kK1Chunk - 1) / kK1Chunk;

  for (int q = tid; q < kExpTableSize; q += kK1Threads) tab[q] = c_exp_table[q];
  if (tid == 0) {
    for (int b = 0; b < kK1Stages; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int c = 0; c < kK1Stages && c < n_chunks; ++c) {
      const int cnt = min(kK1Chunk, len - c * kK1Chunk);
      const uint32_t bytes = static_cast<uint32_t>(cnt * sizeof(SrcRec));
      mbar_arrive_expect_tx(&bars[c], bytes);
      bulk_g2s(&ring[c][0], src + begin + c * kK1Chunk, bytes, &bars[c]);
    }
  }

  // this thread's points
  double px[P], py[P], pz[P], v[P], gx[P], gy[P], gz[P];
  const int base = blockIdx.x * (kK1Threads * P) + tid;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int i = base + k * kK1Threads;
    px[k] = py[k] = pz[k] = 0.0;
    if (i < n_pts) {
      const int pi = pt_index ? pt_index[i] : i;
      px[k] = pts[3 * static_cast<size_t>(pi)];
      py[k] = pts[3 * static_cast<size_t>(pi) + 1];
      pz[k] = pts[3 * static_cast<size_t>(pi) + 2];
    }
    v[k] = gx[k] = gy[k] = gz[k] = 0.0;
  }
  // PLANAR: pz holds rz = z - zs and gz accumulates sum_j w_j; rz2 = fl(rz rz)
  double rz2[PLANAR ? P : 1];
  if (PLANAR) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      pz[k] = __dsub_rn(pz[k], zs);
      rz2[k] = __dmul_rn(pz[k], pz[k]);
    }
  }
  {  // the bounding box of the CTA's points (PLANAR: z as rz)
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int k = 0; k < P; ++k)
      if (base + k * kK1Threads < n_pts) {
        lo[0] = fmin(lo[0], px[k]); hi[0] = fmax(hi[0], px[k]);
        lo[1] = fmin(lo[1], py[k]); hi[1] = fmax(hi[1], py[k]);
        lo[2] = fmin(lo[2], pz[k]); hi[2] = fmax(hi[2], pz[k]);
      }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
        hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
      }
    __shared__ double wbox[kK1Threads / 32][6];
    if ((tid & 31) == 0)
      for (int c = 0; c < 3; ++c) {
        wbox[tid >> 5][c] = lo[c];
        wbox[tid >> 5][3 + c] = hi[c];
      }
    __syncthreads();
    if (tid < 6) {
      double v = wbox[0][tid];
      for (int w = 1; w < kK1Threads / 32; ++w)
        v = tid < 3 ? fmin(v, wbox[w][tid]) : fmax(v, wbox[w][tid]);
      boxs[tid] = v;
    }
    __syncthreads();
  }

  for (int c = 0; c < n_chunks; ++c) {
    const int buf = c % kK1Stages;
    mbar_wait(&bars[buf], static_cast<uint32_t>((c / kK1Stages) & 1));
    const int cnt = min(kK1Chunk, len - c * kK1Chunk);
    const SrcRec* rb = ring[buf];
    int n_iter = cnt;
    // every source of the chunk keeps every pair with the CTA's points (the
    // farthest corner of their box within each source's exact keep threshold,
    // with a margin far above the box and r.r roundings): the pair loop then
    // skips the per-pair cull test — the same keep decisions, so the same sums
    bool full = false;
    if constexpr (!BOX) {
      bool f = true;
      if (tid < cnt) {
        const SrcRec& q = rb[tid];
        const double fx = fmax(fabs(boxs[0] - q.sx), fabs(boxs[3] - q.sx));
        const double fy = fmax(fabs(boxs[1] - q.sy), fabs(boxs[4] - q.sy));
        const double fz = PLANAR ? fmax(fabs(boxs[2]), fabs(boxs[5]))
                                 : fmax(fabs(boxs[2] - q.sz), fabs(boxs[5] - q.sz));
        f = (fx * fx + fy * fy + fz * fz) * (1.0 + 1e-9) <= q.thr;
      }
      full = __syncthreads_and(f) != 0;
    }
    if constexpr (BOX) {  // the chunk's sources that reach the CTA's box, in order
      bool keep = false;
      if (tid < cnt) {
        const SrcRec& q = rb[tid];
        const double dx = fmax(fmax(boxs[0] - q.sx, q.sx - boxs[3]), 0.0);
        const double dy = fmax(fmax(boxs[1] - q.sy, q.sy - boxs[4]), 0.0);
        const double dz = PLANAR ? fmax(fmax(boxs[2], -boxs[5]), 0.0)
                                 : fmax(fmax(boxs[2] - q.sz, q.sz - boxs[5]), 0.0);
        keep = (dx * dx + dy * dy + dz * dz) * (1.0 - 1e-9) <= q.thr;
        if (rg.okbits && keep) {  // in the region's contraction (k5_fused.cu's list)
          // (re-read per chunk: nothing stays live across the pair loop)
          const int r = rg.cta_region[blockIdx.x], Jr = rg.J[r];
          const int d = begin + c * kK1Chunk + tid - Jr;
          if (Jr > 0)
            keep = !((rg.okbits[static_cast<size_t>(r) * rg.words + (d >> 5)] >> (d & 31)) & 1u);
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (tid < kK1Chunk && (tid & 31) == 0) keep_n[tid >> 5] = __popc(m);
      __syncthreads();
      if (tid < kK1Chunk && keep) {
        int pos = __popc(m & ((1u << (tid & 31)) - 1u));
        for (int w = 0; w < (tid >> 5); ++w) pos += keep_n[w];
        keep_list[pos] = tid;
      }
      n_iter = 0;
      for (int w = 0; w < kK1Chunk / 32; ++w) n_iter += keep_n[w];
      __syncthreads();
    }
    auto pairs = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll kK1Unroll
    for (int jj = 0; jj < n_iter; ++jj) {
      const int j = BOX ? keep_list[jj] : jj;
      const double4 a = *reinterpret_cast<const double4*>(&rb[j].sx);      // sx sy sz nisp
      const double4 b = *reinterpret_cast<const double4*>(&rb[j].magicL);  // magicL gfac thr band
      const double4 q = *reinterpret_cast<const double4*>(&rb[j].q0);      // q0 q1 q2 -
      const int lo = __double2loint(b.w);  // hi32(thr) - 1
      double rx[P], ry[P], rz[P], r2[P], e[P];
      bool keep[P];
      unsigned band = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < P; ++k) {
        rx[k] = __dsub_rn(px[k], a.x);
        ry[k] = __dsub_rn(py[k], a.y);
        rz[k] = PLANAR ? pz[k] : __dsub_rn(pz[k], a.z);
        // r.r with FMA (3 roundings of non-negative terms: within a few ulp of
        // the reference's 5-rounding r.r, core.hpp:27)
        if (PLANAR)
          r2[k] = __fma_rn(ry[k], ry[k], __fma_rn(rx[k], rx[k], rz2[PLANAR ? k : 0]));
        else
          r2[k] = __fma_rn(rz[k], rz[k], __fma_rn(ry[k], ry[k], __dmul_rn(rx[k], rx[k])));
        // keep/cull decided on the high words (1 unit = 2^32 ulp >> the few-ulp
        // gap): thr < 0 (inactive source) lands in the cull branch; the band
        // hi32(r.r) in [lo, lo + 2] is re-decided exactly below
        if (!FULL) {
          const int h = __double2hiint(r2[k]);
          keep[k] = h < lo;
          band = min(band, static_cast<unsigned>(h - lo));
        }
        if (K1_VOTE_LATE) e[k] = src_exp(r2[k], a.w, b.x, q.x, q.y, q.z, tab);
      }
      if (!FULL && __any_sync(0xffffffffu, band <= 2u)) {  // warp-uniform, rare
        // the reference's exact r.r (association of core.hpp:27, no
        // contraction) and its exact compare, for every point of the warp
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const double zz = PLANAR ? rz2[PLANAR ? k : 0] : __dmul_rn(rz[k], rz[k]);
          const double e2 =
              __dadd_rn(__dadd_rn(__dmul_rn(rx[k], rx[k]), __dmul_rn(ry[k], ry[k])), zz);
          keep[k] = __double_as_longlong(e2) <= __double_as_longlong(b.z);
        }
      }
#pragma unroll
      for (int k = 0; k < P; ++k) {
        if (!K1_VOTE_LATE) e[k] = src_exp(r2[k], a.w, b.x, q.x, q.y, q.z, tab);
        const double T = (FULL || keep[k]) ? e[k] : 0.0;
        v[k] = __dadd_rn(v[k], T);
        if (GRAD) {
          const double w = __dmul_rn(T, b.y);
          gx[k] = __fma_rn(rx[k], w, gx[k]);
          gy[k] = __fma_rn(ry[k], w, gy[k]);
          gz[k] = PLANAR ? __dadd_rn(gz[k], w) : __fma_rn(rz[k], w, gz[k]);
        }
      }
    }
    };
    if (full)
      pairs(std::true_type{});
    else
      pairs(std::false_type{});
    __syncthreads();  // everyone is done with ring[buf]
    if (tid == 0 && c + kK1Stages < n_chunks) {
      const int cn = c + kK1Stages;
      const int cnt2 = min(kK1Chunk, len - cn * kK1Chunk);
      const uint32_t bytes = static_cast<uint32_t>(cnt2 * sizeof(SrcRec));
      mbar_arrive_expect_tx(&bars[buf], bytes);
      bulk_g2s(&ring[buf][0], src + begin + cn * kK1Chunk, bytes, &bars[buf]);
    }
  }

  const size_t plane = static_cast<size_t>(n_pts);
  double* pv = part + static_cast<size_t>(s) * (GRAD ? 4 : 1) * plane;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int i = base + k * kK1Threads;
    if (i < n_pts) {
      pv[i] = v[k];
      if (GRAD) {
        pv[plane + i] = gx[k];
        pv[2 * plane + i] = gy[k];
        pv[3 * plane + i] = PLANAR ? __dmul_rn(pz[k], gz[k]) : gz[k];
      }
    }
  }
}

// plain field: val[i], grad[3i..3i+2]
__global__ void k1_combine_field(const double* __restrict__ part, int S, int n,
                                 double* __restrict__ val, double* __restrict__ grad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t plane = static_cast<size_t>(n);
  double v = 0.0, x = 0.0, y = 0.0, z = 0.0;
#pragma unroll  // S <= kMaxSplits: all loads in flight, sums in split order
  for (int s = 0; s < kMaxSplits; ++s) {
    if (s < S) {
      const double* p = part + static_cast<size_t>(s) * 4 * plane;
      v += p[i];
      x += p[plane + i];
      y += p[2 * plane + i];
      z += p[3 * plane + i];
    }
  }
  val[i] = v;
  if (grad) {
    grad[3 * static_cast<size_t>(i)] = x;
    grad[3 * static_cast<size_t>(i) + 1] = y;
    grad[3 * static_cast<size_t>(i) + 2] = z;
  }
}

// Dirichlet values: out[i] = -T~ (mesh.cpp:261); partials are value-only.
// (negate = false: plain values, the field without its gradient)
__global__ void k1_combine_dirichlet(const double* __restrict__ part, int S, int n,
                                     double* __restrict__ out, bool negate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 0.0;
#pragma unroll
  for (int s = 0; s < kMaxSplits; ++s)
    if (s < S) v += part[static_cast<size_t>(s) * n + i];
  out[i] = negate ? -v : v;
}

// Flux integrand at face quadrature points (assembly.cpp:161-164, :135):
// g_q = (-k * grad.n) * w, with the qp addressed through pt_index.
__global__ void k1_combine_flux(const double* __restrict__ part, int S, int n,
                                const int* __restrict__ pt_index,
                                const double* __restrict__ normals,
                                const double* __restrict__ weights, double k,
                                double* __restrict__ gq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t plane = static_cast<size_t>(n);
  double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll
  for (int s = 0; s < kMaxSplits; ++s) {
    if (s < S) {
      const double* p = part + static_cast<size_t>(s) * 4 * plane;
      x += p[plane + i];
      y += p[2 * plane + i];
      z += p[3 * plane + i];
    }
  }
  const int q = pt_index ? pt_index[i] : i;
  const double* nn = normals + 3 * static_cast<size_t>(q);
  const double dot = __dadd_rn(__dadd_rn(__dmul_rn(x, nn[0]), __dmul_rn(y, nn[1])),
                               __dmul_rn(z, nn[2]));
  gq[i] = __dmul_rn(__dmul_rn(-k, dot), weights[q]);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

void k1_exp_table_host(double* tab) {
  // 2^(j/1024) with (j << 10) pre-subtracted from the high word (src_exp)
  for (int j = 0; j < kExpTableSize; ++j) {
    const double v = static_cast<double>(exp2l(static_cast<long double>(j) / kExpTableSize));
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    bits -= static_cast<uint64_t>(j) << (20 - kExpBits + 32);
    std::memcpy(&tab[j], &bits, 8);
  }
}

void k1_upload_exp_table(cudaStream_t stream) {
  static double tab[kExpTableSize];
  k1_exp_table_host(tab);
  cudaMemcpyToSymbolAsync(c_exp_table, tab, sizeof(tab), 0, cudaMemcpyHostToDevice, stream);
}

// The source splits depend on the source count only — never on the points —
// so every point's sum has the same association whichever subset of points a
// launch (or a shard of a multi-GPU run) evaluates: sharded loads reproduce
// the single-launch result bit for bit. >= 128 sources per split, <= 16 splits
// (enough CTAs for small point sets, few partial planes for large ones).
// The fewest source splits giving >= 12 waves of CTAs with the last one >= 95 %
// full (each split adds a partial plane of 4 doubles per point to write and
// combine; fewer, longer waves lose to the SMs' spread): config 1 (586 point
// blocks of 1792, one resident CTA per SM) takes 4 (15.8 waves; measured 1
// split 0.899e12 pairs/s, 4: 0.918e12, 16: 0.916e12); at most one per 128 sources.
int k1_choose_splits(int n_pts, int n_src, int sm_count, int points_per_cta, int resident) {
  const int smax = std::max(1, std::min(kMaxSplits, n_src / 128));
  if (const char* e = std::getenv("TG_K1_SPLITS")) return std::max(1, std::min(smax, std::atoi(e)));
  const long blocks = (static_cast<long>(n_pts) + points_per_cta - 1) / points_per_cta;
  const long slots = static_cast<long>(std::max(1, sm_count)) * std::max(1, resident);
  for (int S = 1; S <= smax; ++S) {
    const long ctas = blocks * S, waves = (ctas + slots - 1) / slots;
    if (ctas >= 12 * slots && static_cast<double>(ctas) >= 0.95 * static_cast<double>(waves * slots))
      return S;
  }
  return smax;
}

int k1_resident_ctas(int P) { return P >= 6 ? 256 / kK1Threads : (P >= 4 ? K1_MINB4 : 3); }

void k1_prepare(const double* d_src6, int n, double t, double alpha, double rcp, double cull,
                SrcRec* d_rec, cudaStream_t stream) {
  if (n <= 0) return;
  const int threads = 256;
  k1_prepare_sources<<<(n + threads - 1) / threads, threads, 0, stream>>>(
      d_src6, n, t, 4.0 * alpha, 2.0 * alpha, rcp, cull, d_rec);
}

void k1_launch_partial(const SrcRec* d_rec, int n_src, const double* d_pts,
                       const int* d_index, int n_pts, int S, bool grad, int P, double* d_part,
                       cudaStream_t stream, bool planar, double zs, const K1Ranges& rg) {
  const int split_len = (n_src + S - 1) / S;
  const int ppc = kK1Threads * P;
  dim3 grid((n_pts + ppc - 1) / ppc, S);
  if (rg.cta_region && grad && P == 7) {  // K5's remainder: per-CTA box culling of sources
    if (planar)
      k1_partial<7, true, true, true><<<grid, kK1Threads, 0, stream>>>(
          d_rec, n_src, split_len, d_pts, d_index, n_pts, d_part, zs, rg);
    else
      k1_partial<7, true, false, true><<<grid, kK1Threads, 0, stream>>>(
          d_rec, n_src, split_len, d_pts, d_index, n_pts, d_part, zs, rg);
    return;
  }
#define TG_K1_LAUNCH(PP, GG, PLN)                                                         \
  k1_partial<PP, GG, PLN><<<grid, kK1Threads, 0, stream>>>(d_rec, n_src, split_len, d_pts,     \
                                                          d_index, n_pts, d_part, zs, rg)
  // planar-history variants for the default shapes (P = 7 with gradient, 5 value-only;
  // measured best: gradient P=6/7/8 76.8/75.3/78.7 ms, value-only P=4/5/6 62.2/59.2/61.8)
  if (planar && grad && P == 7) {
    TG_K1_LAUNCH(7, true, true);
    return;
  }
  if (planar && !grad && P == 5) {
    TG_K1_LAUNCH(5, false, true);
    return;
  }
  switch (P) {
    case 1: if (grad) TG_K1_LAUNCH(1, true, false); else TG_K1_LAUNCH(1, false, false); break;
    case 2: if (grad) TG_K1_LAUNCH(2, true, false); else TG_K1_LAUNCH(2, false, false); break;
    case 3: if (grad) TG_K1_LAUNCH(3, true, false); else TG_K1_LAUNCH(3, false, false); break;
    case 5: if (grad) TG_K1_LAUNCH(5, true, false); else TG_K1_LAUNCH(5, false, false); break;
    case 6: if (grad) TG_K1_LAUNCH(6, true, false); else TG_K1_LAUNCH(6, false, false); break;
    case 7: if (grad) TG_K1_LAUNCH(7, true, false); else TG_K1_LAUNCH(7, false, false); break;
    case 8: if (grad) TG_K1_LAUNCH(8, true, false); else TG_K1_LAUNCH(8, false, false); break;
    default: if (grad) TG_K1_LAUNCH(4, true, false); else TG_K1_LAUNCH(4, false, false); break;
  }
#undef TG_K1_LAUNCH
}

void k1_launch_combine_field(const double* d_part, int S, int n, double* d_val, double* d_grad,
                             cudaStream_t stream) {
  k1_combine_field<<<(n + 255) / 256, 256, 0, stream>>>(d_part, S, n, d_val, d_grad);
}

void k1_launch_combine_dirichlet(const double* d_part, int S, int n, double* d_out,
                                 cudaStream_t stream, bool negate) {
  k1_combine_dirichlet<<<(n + 255) / 256, 256, 0, stream>>>(d_part, S, n, d_out, negate);
}

void k1_launch_combine_flux(const double* d_part, int S, int n, const int* d_index,
                            const double* d_normals, const double* d_weights, double k,
                            double* d_gq, cudaStream_t stream) {
  k1_combine_flux<<<(n + 255) / 256, 256, 0, stream>>>(d_part, S, n, d_index, d_normals,
                                                        d_weights, k, d_gq);
}

}  // namespace tgb
