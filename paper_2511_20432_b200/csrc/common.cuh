// Shared device helpers for the sm_100a kernels: exact-rounding arithmetic
// wrappers, the table-driven fp64 exp used by the point-source kernels, and
// the TMA bulk-copy / mbarrier primitives that stage source tiles in shared
// memory.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tgb {

// ---------------------------------------------------------------------------
// Table-driven exp(x) for x in [-708, 709], relative error < 1e-13.
//
// x = (256 m + j) ln2/256 + r,  |r| <= ln2/512, j in [0,256)
// exp(x) = 2^m * 2^(j/256) * p(r),  p(r) = 1 + r + r^2 (c2 + c3 r)
//
// 7 FP64-pipe instructions (1 DFMA + 1 DADD + 1 DFMA range reduction, 3 DFMA
// polynomial, 1 DMUL table product) plus integer ops for j, m and the
// exponent add. The cubic is a Chebyshev fit of (e^r - 1 - r)/r^2 on
// [-ln2/512, ln2/512]: max relative error 7.0e-14 (mpmath), three orders
// below the 1e-10 parity tolerance (BASELINE.json north_star); the
// single-constant reduction adds < 2e-15 for |x| <= 80.
// ---------------------------------------------------------------------------
constexpr int kExpBits = 8;
constexpr int kExpTableSize = 1 << kExpBits;
constexpr double kExpInvStep = 369.32993046757462707;    // 256 / ln 2
constexpr double kExpStep = 0.0027076061740622863;       // ln 2 / 256
constexpr double kExpMagic = 6755399441055744.0;         // 1.5 * 2^52
constexpr double kExpC2 = 0x1.00000147fd40ap-1;
constexpr double kExpC3 = 0x1.5555565bb988ep-3;

// exp(x) with the 2^(j/256) table in shared memory.
__device__ __forceinline__ double fast_exp(double x, const double* __restrict__ tab) {
  const double kf = __fma_rn(x, kExpInvStep, kExpMagic);
  const double n = __dsub_rn(kf, kExpMagic);
  const int ki = __double2loint(kf);
  const double r = __fma_rn(n, -kExpStep, x);
  double p = __fma_rn(kExpC3, r, kExpC2);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  const double t = tab[ki & (kExpTableSize - 1)];
  const double e = __dmul_rn(t, p);
  // scale by 2^m: integer add into the exponent field of the high word
  const int m = ki >> kExpBits;
  const int hi = __double2hiint(e) + (m << 20);
  return __hiloint2double(hi, __double2loint(e));
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

}  // namespace tgb
