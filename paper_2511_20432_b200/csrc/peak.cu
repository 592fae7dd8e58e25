// FP64 peak microbenchmarks: independent DFMA chains (the FP64 pipe's issue
// limit; the roofline denominator of K1) and independent DMMA m8n8k4
// accumulators (the FP64 tensor-core rate; the denominator of K5's
// contraction). MEASURED_PEAKS.json carries no fp64 figure.
#include "context.hpp"

namespace tgb {

__global__ void __launch_bounds__(256) fp64_dfma_chains(double* out, int iters, double a,
                                                        double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = __fma_rn(x0, a, b);
      x1 = __fma_rn(x1, a, b);
      x2 = __fma_rn(x2, a, b);
      x3 = __fma_rn(x3, a, b);
      x4 = __fma_rn(x4, a, b);
      x5 = __fma_rn(x5, a, b);
      x6 = __fma_rn(x6, a, b);
      x7 = __fma_rn(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 1.2345) out[blockIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) fp64_dmma_chains(double* out, int iters, double a,
                                                        double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double x = a + threadIdx.x * 1e-9, y = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1])
                     : "d"(x), "d"(y));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[blockIdx.x] = s;
}

}  // namespace tgb

extern "C" int tg_dmma_peak(tg_ctx* ctx, double* out_tflops) {
  using namespace tgb;
  try {
    TG_CUDA(cudaSetDevice(ctx->device));
    DevBuf<double> sink;
    sink.ensure(1 << 16);
    const int blocks = ctx->sm_count * 2, threads = 256, iters = 2048;
    cudaEvent_t e0, e1;
    TG_CUDA(cudaEventCreate(&e0));
    TG_CUDA(cudaEventCreate(&e1));
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
      TG_CUDA(cudaEventRecord(e0, ctx->stream));
      fp64_dmma_chains<<<blocks, threads, 0, ctx->stream>>>(sink.p, iters, 1.0, 1e-7);
      TG_CUDA(cudaEventRecord(e1, ctx->stream));
      TG_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      TG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      // 512 flops per warp-level m8n8k4
      const double flops = 512.0 * 4 * 8 * static_cast<double>(iters) * blocks * (threads / 32);
      if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out_tflops = best;
    return TG_OK;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return TG_ECUDA;
  }
}

extern "C" int tg_fp64_peak(tg_ctx* ctx, double* out_tflops) {
  using namespace tgb;
  try {
    TG_CUDA(cudaSetDevice(ctx->device));
    DevBuf<double> sink;
    sink.ensure(1 << 16);
    const int blocks = ctx->sm_count * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    TG_CUDA(cudaEventCreate(&e0));
    TG_CUDA(cudaEventCreate(&e1));
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
      TG_CUDA(cudaEventRecord(e0, ctx->stream));
      fp64_dfma_chains<<<blocks, threads, 0, ctx->stream>>>(sink.p, iters, 0.999999, 1e-7);
      TG_CUDA(cudaEventRecord(e1, ctx->stream));
      TG_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      TG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
      if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out_tflops = best;
    return TG_OK;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return TG_ECUDA;
  }
}
