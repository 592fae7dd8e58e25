// K2 option — PCG with the fast-diagonalization preconditioner for separable
// patches (SURVEY.md §8f "stronger preconditioner").
//
// For the Kronecker operator A = a Mz x My x Mx + b (...) the preconditioner
// P = V diag(1 / (a + b (lx + ly + lz))) V^T, V = Vz x Vy x Vx with
// K_d V_d = M_d V_d diag(l_d), V_d^T M_d V_d = I (host/fdm.cpp), is A^-1 up to
// rounding, so the reference's PCG loop stops after one or two iterations
// instead of ~64-170 with Jacobi. Applying P is six dense mode products (plain
// library GEMMs: cuBLAS DGEMM on the FP64 tensor cores) and one scaling; the
// operator apply is the sum-factorized TMA kernel of k2_kron.cu.
#include "context.hpp"
#include "k2_fdm.cuh"

namespace tgb {

namespace {

void cublas_check(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS)
    throw cuda_error(std::string("cublas: ") + what + " failed (" + std::to_string(st) + ")");
}
#define TG_CUBLAS(call) cublas_check((call), #call)

constexpr int kDotBlocks = 512;
constexpr int kDotThreads = 256;

__global__ void inv_eigs_kernel(int nx, int ny, int nz, const double* __restrict__ lx,
                                const double* __restrict__ ly, const double* __restrict__ lz,
                                double a, double b, double* __restrict__ dinv) {
  const long n = static_cast<long>(nx) * ny * nz;
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(f % nx);
    const int j = static_cast<int>((f / nx) % ny);
    const int k = static_cast<int>(f / (static_cast<long>(nx) * ny));
    dinv[f] = 1.0 / (a + b * (lx[i] + ly[j] + lz[k]));
  }
}

__global__ void scale_kernel(long n, const double* __restrict__ d, double* __restrict__ v) {
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x)
    v[f] *= d[f];
}

// r = b - y
__global__ void residual_kernel(long n, const double* __restrict__ b, const double* __restrict__ y,
                                double* __restrict__ r) {
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x)
    r[f] = b[f] - y[f];
}

// x += alpha p; r -= alpha Ap
__global__ void update_kernel(long n, double alpha, const double* __restrict__ p,
                              const double* __restrict__ Ap, double* __restrict__ x,
                              double* __restrict__ r) {
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x) {
    x[f] += alpha * p[f];
    r[f] -= alpha * Ap[f];
  }
}

// p = z + beta p
__global__ void direction_kernel(long n, double beta, const double* __restrict__ z,
                                 double* __restrict__ p) {
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x)
    p[f] = z[f] + beta * p[f];
}

// two dot products in a fixed order: per-block partials, then one block
__global__ void __launch_bounds__(kDotThreads) dot2_partial(long n, const double* __restrict__ a,
                                                            const double* __restrict__ b,
                                                            const double* __restrict__ c,
                                                            const double* __restrict__ d,
                                                            double* __restrict__ part) {
  __shared__ double s0[kDotThreads], s1[kDotThreads];
  double x0 = 0.0, x1 = 0.0;
  for (long f = blockIdx.x * static_cast<long>(kDotThreads) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * kDotThreads) {
    x0 += a[f] * b[f];
    if (c) x1 += c[f] * d[f];
  }
  s0[threadIdx.x] = x0;
  s1[threadIdx.x] = x1;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s0[threadIdx.x] += s0[threadIdx.x + w];
      s1[threadIdx.x] += s1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0[0];
    part[2 * blockIdx.x + 1] = s1[0];
  }
}

__global__ void __launch_bounds__(kDotThreads) dot2_final(int nb, const double* __restrict__ part,
                                                          double* __restrict__ out) {
  __shared__ double s0[kDotThreads], s1[kDotThreads];
  double x0 = 0.0, x1 = 0.0;
  for (int q = threadIdx.x; q < nb; q += kDotThreads) {
    x0 += part[2 * q];
    x1 += part[2 * q + 1];
  }
  s0[threadIdx.x] = x0;
  s1[threadIdx.x] = x1;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s0[threadIdx.x] += s0[threadIdx.x + w];
      s1[threadIdx.x] += s1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s0[0];
    out[1] = s1[0];
  }
}

int grid_for(long n) {
  return static_cast<int>(std::min<long>(4096, std::max<long>(1, (n + 255) / 256)));
}

// (a.b, c.d) on the host (synchronous)
void dot2(long n, const double* a, const double* b, const double* c, const double* d,
          const FdmWork& w, cudaStream_t s, double& o0, double& o1) {
  dot2_partial<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, c, d, w.partials);
  dot2_final<<<1, kDotThreads, 0, s>>>(kDotBlocks, w.partials, w.dots);
  TG_CUDA(cudaMemcpyAsync(w.h_dots, w.dots, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  o0 = w.h_dots[0];
  o1 = w.h_dots[1];
}

}  // namespace

void fdm_inverse_eigs(const int n[3], const double* lx, const double* ly, const double* lz,
                      double a, double b, double* dinv, cudaStream_t s) {
  const long N = static_cast<long>(n[0]) * n[1] * n[2];
  inv_eigs_kernel<<<grid_for(N), 256, 0, s>>>(n[0], n[1], n[2], lx, ly, lz, a, b, dinv);
  TG_CUDA(cudaGetLastError());
}

void fdm_apply(cublasHandle_t h, const FdmDev& F, const double* r, double* z, double* t1,
               double* t2, cudaStream_t s) {
  const int nx = F.n[0], ny = F.n[1], nz = F.n[2];
  const long nxy = static_cast<long>(nx) * ny;
  const double one = 1.0, zero = 0.0;
  TG_CUBLAS(cublasSetStream(h, s));
  // V^T r: x (t1 = Vx^T R), y (t2_k = t1_k Vy), z (t1 = t2 Vz)
  TG_CUBLAS(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nx, ny * nz, nx, &one, F.V[0], nx, r, nx,
                        &zero, t1, nx));
  TG_CUBLAS(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, nx, ny, ny, &one, t1, nx, nxy,
                                      F.V[1], ny, 0, &zero, t2, nx, nxy, nz));
  TG_CUBLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(nxy), nz, nz, &one, t2,
                        static_cast<int>(nxy), F.V[2], nz, &zero, t1, static_cast<int>(nxy)));
  const long N = nxy * nz;
  scale_kernel<<<grid_for(N), 256, 0, s>>>(N, F.dinv, t1);
  TG_CUDA(cudaGetLastError());
  // V w: z (t2 = t1 Vz^T), y (t1_k = t2_k Vy^T), x (z = Vx t1)
  TG_CUBLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, static_cast<int>(nxy), nz, nz, &one, t1,
                        static_cast<int>(nxy), F.V[2], nz, &zero, t2, static_cast<int>(nxy)));
  TG_CUBLAS(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_T, nx, ny, ny, &one, t2, nx, nxy,
                                      F.V[1], ny, 0, &zero, t1, nx, nxy, nz));
  TG_CUBLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, nx, ny * nz, nx, &one, F.V[0], nx, t1, nx,
                        &zero, z, nx));
}

PcgStatus fdm_pcg_solve(cublasHandle_t h, const KronGrid& g, double a, double b, const FdmDev& F,
                        const double* rhs, double* x, const FdmWork& w, double tol, int max_iter,
                        int sm_count, cudaStream_t s, const TensorMap3* x_map,
                        const TensorMap3* p_map) {
  const long n = static_cast<long>(g.n[0]) * g.n[1] * g.n[2];
  const int G = grid_for(n);
  double bb = 0.0, unused = 0.0;
  dot2(n, rhs, rhs, nullptr, nullptr, w, s, bb, unused);
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {  // sparse.cpp:57-60
    TG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    return PcgStatus{0, 0, 0.0, 0.0};
  }
  // r = b - A x (sparse.cpp:61-69); the preconditioned residual z = P r is
  // formed lazily after the stop test (same iterates as the reference's
  // order, one preconditioner apply fewer on the converged iteration)
  k2_apply(g, a, b, x, w.Ap, sm_count, s, x_map);
  residual_kernel<<<G, 256, 0, s>>>(n, rhs, w.Ap, w.r);
  double rr = 0.0, rz = 0.0, rz_old = 0.0;
  dot2(n, w.r, w.r, nullptr, nullptr, w, s, rr, unused);
  double rel = 0.0;
  for (int it = 0; it < max_iter; ++it) {
    rel = std::sqrt(rr) / bnorm;
    if (rel <= tol) return PcgStatus{it, 0, rel, bnorm};
    fdm_apply(h, F, w.r, w.z, w.t1, w.t2, s);
    dot2(n, w.r, w.z, nullptr, nullptr, w, s, rz, unused);
    if (it == 0) {
      TG_CUDA(cudaMemcpyAsync(w.p, w.z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    } else {
      direction_kernel<<<G, 256, 0, s>>>(n, rz / rz_old, w.z, w.p);  // p = z + beta p
    }
    rz_old = rz;
    k2_apply(g, a, b, w.p, w.Ap, sm_count, s, p_map);
    double pAp = 0.0;
    dot2(n, w.p, w.Ap, nullptr, nullptr, w, s, pAp, unused);
    if (!(pAp > 0.0)) return PcgStatus{it, 4, rel, bnorm};
    update_kernel<<<G, 256, 0, s>>>(n, rz / pAp, w.p, w.Ap, x, w.r);
    dot2(n, w.r, w.r, nullptr, nullptr, w, s, rr, unused);
  }
  return PcgStatus{max_iter, 3, rel, bnorm};
}

}  // namespace tgb
