// Microbenchmark: FP64 tensor (DMMA m8n8k4) and FP64 vector (DFMA) issue
// rates on this GPU, alone and interleaved in the same warps — do the two
// pipes overlap? (sizes the K5 generator/MMA balance)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_pipe tools/dmma_pipe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NM, int NF>
__global__ void bench(double* out, int iters, double x) {
  double c[8][2];
  double f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0.0; f[i] = x + i; }
  const double a = x + threadIdx.x * 1e-3, b = x - threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int k = 0; k < NF; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  if (s == 1234.5) out[0] = s;
}

template <int NM, int NF>
void run(const char* name, int blocks, int threads) {
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 20000;
  bench<NM, NF><<<blocks, threads>>>(d, 100, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<NM, NF><<<blocks, threads>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(blocks) * threads / 32;
  const double mma_flops = warps * iters * NM * 512.0;
  const double fma_flops = warps * 32 * iters * NF * 8 * 2.0;
  printf("%-28s %8.3f ms  DMMA %6.2f TF/s  DFMA %6.2f TF/s  sum %6.2f\n", name, ms,
         mma_flops / ms * 1e-9, fma_flops / ms * 1e-9, (mma_flops + fma_flops) / ms * 1e-9);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {256, 512}) {
    printf("threads/CTA %d, %d CTAs\n", t, sms * 2);
    run<8, 0>("dmma only", sms * 2, t);
    run<0, 8>("dfma only", sms * 2, t);
    run<8, 1>("dmma 8 : dfma 8x1", sms * 2, t);
    run<8, 2>("dmma 8 : dfma 8x2", sms * 2, t);
    run<8, 4>("dmma 8 : dfma 8x4", sms * 2, t);
    run<4, 4>("dmma 4 : dfma 8x4", sms * 2, t);
  }
  return 0;
}
