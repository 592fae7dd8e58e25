// Shared device helpers for the sm_100a kernels: exact-rounding arithmetic
// wrappers, the table-driven fp64 exponential of the point-source kernels, and
// the TMA bulk-copy / mbarrier primitives that stage source tiles in shared
// memory.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tgb {

// ---------------------------------------------------------------------------
// Point-source exponential exp(lnc - r2 / spread), relative error < 1.7e-12.
//
// In units of ln2/1024 the exponent is y = r2 * nis' + lnc' with
// nis' = -(1024/ln2)/spread and lnc' = (1024/ln2) lnc, both per source.
// Per source, lnc' = L + l with L an integer and |l| <= 1/2; the factor
// C = 2^(l/1024) = exp(lnc - L ln2/1024) is folded into the polynomial:
//
//   k  = rint(r2 nis' + L)            (one DFMA against A = L + 1.5*2^52)
//   f  = r2 nis' + (L - k)            (exact integer L - k, one DFMA)
//   exp(..) = 2^(k >> 10) * 2^((k & 1023)/1024) * C 2^(f/1024),  |f| <= 1/2
//   C 2^(f/1024) ~= q0 + q1 f + q2 f^2 (q_i = C d_i, per source)
//
// 6 FP64-pipe instructions including the argument (3 DFMA + 1 DADD range
// reduction, 2 DFMA quadratic) plus 1 DMUL by the table entry 2^(k/1024),
// whose 2^(k>>10) part is an integer add into the exponent field. d_i is the relative
// minimax quadratic of exp(u) on |u| <= ln2/2048 in the variable f = 1024 u/ln2
// (Remez, mpmath): max relative error 1.62e-12, 60x below the 1e-10 parity
// tolerance (BASELINE.json north_star); the folded per-source rounding adds
// < 1e-15.
// ---------------------------------------------------------------------------
constexpr int kExpBits = 10;
constexpr int kExpTableSize = 1 << kExpBits;
constexpr double kExpInvStep = 0x1.71547652b82fep+10;   // 1024 / ln2
constexpr double kExpStepHi = 0x1.62e42fefa39efp-11;    // ln2 / 1024 (hi)
constexpr double kExpStepLo = 0x1.abc9e3b39803fp-66;    // ln2 / 1024 (lo)
constexpr double kExpMagic = 6755399441055744.0;        // 1.5 * 2^52
constexpr double kExpD0 = 0x1.0000000000002p+0;
constexpr double kExpD1 = 0x1.62e43044e4b97p-11;
constexpr double kExpD2 = 0x1.ebfbdfbd1456bp-23;

// e = exp(lnc - r2/spread) from the per-source constants (nisp = nis',
// magicL = L + 1.5*2^52, q0..q2) and the shared table. Entry j holds 2^(j/1024)
// with (j << 10) pre-subtracted from its high word, so that adding (k << 10)
// scales it by 2^(k >> 10) exactly (one IMAD; the entry is a bit container).
__device__ __forceinline__ double src_exp(double r2, double nisp, double magicL, double q0,
                                          double q1, double q2,
                                          const double* __restrict__ tab) {
  const double kf = __fma_rn(r2, nisp, magicL);
  const double d = __dsub_rn(magicL, kf);  // L - k, exact
  const double f = __fma_rn(r2, nisp, d);
  const double q = __fma_rn(__fma_rn(q2, f, q1), f, q0);
  const int ki = __double2loint(kf);
  const double t = tab[ki & (kExpTableSize - 1)];
  const double s = __hiloint2double(__double2hiint(t) + static_cast<int>(static_cast<unsigned>(ki) << (20 - kExpBits)),
                                    __double2loint(t));  // 2^(k/1024), exact
  return __dmul_rn(s, q);
}

// ---------------------------------------------------------------------------
// TMA bulk copy (cp.async.bulk, SASS UBLKCP) + mbarrier helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "TG_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra TG_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Deterministic block-wide sum (fixed tree order) of one double per thread;
// result valid in thread 0. `red` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (warp == 0) {
    v = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  return v;
}

// Warp-wide sum of the per-CTA partials pb[b*4 + c] (b < nb, c = 0..3), in
// the order of the loop it replaces — per lane s = 0 + pb[lane] + pb[lane+32]
// + ..., then a shuffle tree — so the sums are bit-identical to it. Every
// load of the first 32*K CTAs is issued (two 16-byte L2 reads per CTA, past
// L1) before the first add: one L2 round trip instead of one per component
// and per stride. Result valid in lane 0.
template <int K = 5>
__device__ __forceinline__ void warp_sum_partials(const double* pb, int nb, int lane,
                                                  double (&s)[4]) {
  double2 v[K][2];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int b = lane + 32 * k;
    if (b < nb) {
      v[k][0] = __ldcg(reinterpret_cast<const double2*>(pb + 4 * static_cast<size_t>(b)));
      v[k][1] = __ldcg(reinterpret_cast<const double2*>(pb + 4 * static_cast<size_t>(b) + 2));
    } else {  // + 0.0 leaves a sum that started at +0.0 unchanged
      v[k][0] = make_double2(0.0, 0.0);
      v[k][1] = make_double2(0.0, 0.0);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) s[c] = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    s[0] += v[k][0].x;
    s[1] += v[k][0].y;
    s[2] += v[k][1].x;
    s[3] += v[k][1].y;
  }
  for (int b = lane + 32 * K; b < nb; b += 32) {
    const double2 lo = __ldcg(reinterpret_cast<const double2*>(pb + 4 * static_cast<size_t>(b)));
    const double2 hi =
        __ldcg(reinterpret_cast<const double2*>(pb + 4 * static_cast<size_t>(b) + 2));
    s[0] += lo.x;
    s[1] += lo.y;
    s[2] += hi.x;
    s[3] += hi.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 4; ++c) s[c] += __shfl_down_sync(0xffffffffu, s[c], o);
}

}  // namespace tgb
