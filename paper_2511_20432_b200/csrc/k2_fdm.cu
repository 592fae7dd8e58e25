// K2 option — PCG with the fast-diagonalization preconditioner for separable
// patches (SURVEY.md §8f "stronger preconditioner").
//
// For the Kronecker operator A = a Mz x My x Mx + b (...) the preconditioner
// P = V diag(1 / (a + b (lx + ly + lz))) V^T, V = Vz x Vy x Vx with
// K_d V_d = M_d V_d diag(l_d), V_d^T M_d V_d = I (host/fdm.cpp), is A^-1 up to
// rounding, so the reference's PCG loop stops after one or two iterations
// instead of ~64-170 with Jacobi. Applying P is six dense mode products
// (mode_gemm below: a strided-batched DMMA m8n8k4 GEMM on the FP64 tensor
// cores) and one scaling; the operator apply is the sum-factorized TMA kernel
// of k2_kron.cu (separable patches) or the sliced-ELL product of k2_csr.cu.
#include <functional>

#include "common.cuh"
#include "context.hpp"
#include "k2_fdm.cuh"

namespace tgb {

namespace {

// ---------------------------------------------------------------- mode GEMM
// C(m, n) = sum_k A(m, k) B(k, n) for a batch of independent products, every
// operand addressed through (row, column, batch) strides so that the six mode
// products of the preconditioner need no transposes. 64 x 64 output tile per
// CTA, 4 warps of 32 x 32 (DMMA m8n8k4), 16-wide k chunks staged in shared
// memory by coalesced loads along whichever index is contiguous.
struct GemmOp {
  int M, N, K, batch;
  const double* A;
  long sam, sak, sab;
  const double* B;
  long sbk, sbn, sbb;
  double* C;
  long scm, scn, scb;
};
constexpr int kGT = 64, kGK = 16, kGLd = kGK + 4;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) mode_gemm_kernel(GemmOp op) {
  __shared__ double As[kGT][kGLd];
  __shared__ double Bs[kGT][kGLd];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, q4 = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int m0 = blockIdx.x * kGT, n0 = blockIdx.y * kGT, bz = blockIdx.z;
  const double* A = op.A + bz * op.sab;
  const double* B = op.B + bz * op.sbb;
  double acc[4][4][2] = {};
  const bool a_kfast = op.sak == 1, b_kfast = op.sbk == 1;
  constexpr int kPer = kGT * kGK / 128;  // elements of each tile per thread
  double ra[kPer], rb[kPer];
  // the next k chunk into registers (its latency overlaps this chunk's MMAs)
  auto fetch = [&](int k0) {
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int e = tid + 128 * r;
      const int m = a_kfast ? e / kGK : e % kGT, k = a_kfast ? e % kGK : e / kGT;
      const int gm = m0 + m, gk = k0 + k;
      ra[r] = (gm < op.M && gk < op.K) ? A[gm * op.sam + gk * op.sak] : 0.0;
      const int n = b_kfast ? e / kGK : e % kGT, kb = b_kfast ? e % kGK : e / kGT;
      const int gn = n0 + n, gkb = k0 + kb;
      rb[r] = (gn < op.N && gkb < op.K) ? B[gkb * op.sbk + gn * op.sbn] : 0.0;
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < op.K; k0 += kGK) {
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int e = tid + 128 * r;
      As[a_kfast ? e / kGK : e % kGT][a_kfast ? e % kGK : e / kGT] = ra[r];
      Bs[b_kfast ? e / kGK : e % kGT][b_kfast ? e % kGK : e / kGT] = rb[r];
    }
    __syncthreads();
    if (k0 + kGK < op.K) fetch(k0 + kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[wm + 8 * i + g8][kk + q4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[wn + 8 * j + g8][kk + q4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* C = op.C + bz * op.scb;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + 8 * i + g8, gn = n0 + wn + 8 * j + 2 * q4 + h;
        if (gm < op.M && gn < op.N) C[gm * op.scm + gn * op.scn] = acc[i][j][h];
      }
}

void mode_gemm(const GemmOp& op, cudaStream_t s) {
  dim3 grid((op.M + kGT - 1) / kGT, (op.N + kGT - 1) / kGT, op.batch);
  mode_gemm_kernel<<<grid, 128, 0, s>>>(op);
  TG_CUDA(cudaGetLastError());
}

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

__global__ void diag_mul_kernel(long n, const double* __restrict__ d, const double* x,
                                double* y) {
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x)
    y[f] = d[f] * x[f];
}

void diag_mul(long n, const double* d, const double* x, double* y, cudaStream_t s) {
  diag_mul_kernel<<<grid_for(n), 256, 0, s>>>(n, d, x, y);
  TG_CUDA(cudaGetLastError());
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

void fdm_apply(const FdmDev& F, const double* r, double* z, double* t1, double* t2,
               cudaStream_t s) {
  const int nx = F.n[0], ny = F.n[1], nz = F.n[2];
  const long nxy = static_cast<long>(nx) * ny;
  const double *Vx = F.V[0], *Vy = F.V[1], *Vz = F.V[2];  // column-major: V(a, b) = V[a + n b]
  const double* in = r;
  if (F.sinv) {  // z = S^-1 P S^-1 r (diagonally scaled approximation, general patches)
    diag_mul(nxy * nz, F.sinv, r, z, s);
    in = z;
  }
  // V^T r: t1[k][j][b] = sum_a Vx(a, b) r[k][j][a]; t2[k][b][i] = sum_a Vy(a, b) t1[k][a][i];
  //        t1[b][j][i] = sum_a Vz(a, b) t2[a][j][i]
  mode_gemm({ny * nz, nx, nx, 1, in, nx, 1, 0, Vx, 1, nx, 0, t1, nx, 1, 0}, s);
  mode_gemm({ny, nx, ny, nz, Vy, ny, 1, 0, t1, nx, 1, nxy, t2, nx, 1, nxy}, s);
  mode_gemm({nz, static_cast<int>(nxy), nz, 1, Vz, nz, 1, 0, t2, nxy, 1, 0, t1, nxy, 1, 0}, s);
  const long N = nxy * nz;
  scale_kernel<<<grid_for(N), 256, 0, s>>>(N, F.dinv, t1);
  TG_CUDA(cudaGetLastError());
  // V w: t2[a][j][i] = sum_b Vz(a, b) t1[b][j][i]; t1[k][a][i] = sum_b Vy(a, b) t2[k][b][i];
  //      z[k][j][a] = sum_b Vx(a, b) t1[k][j][b]
  mode_gemm({nz, static_cast<int>(nxy), nz, 1, Vz, 1, nz, 0, t1, nxy, 1, 0, t2, nxy, 1, 0}, s);
  mode_gemm({ny, nx, ny, nz, Vy, 1, ny, 0, t2, nx, 1, nxy, t1, nx, 1, nxy}, s);
  mode_gemm({ny * nz, nx, nx, 1, t1, nx, 1, 0, Vx, nx, 1, 0, z, nx, 1, 0}, s);
  if (F.sinv) diag_mul(N, F.sinv, z, z, s);
}

namespace {
// device scalars of the preconditioned solve (FdmWork::dots, 8 doubles)
enum { kRz = 0, kRzOld = 1, kPap = 2, kRr = 3, kFail = 4 };

// p = z (first) or z + (rz / rz_old) p
__global__ void direction_dev_kernel(long n, bool first, const double* __restrict__ sc,
                                     const double* __restrict__ z, double* __restrict__ p) {
  const double beta = first ? 0.0 : sc[kRz] / sc[kRzOld];
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x)
    p[f] = first ? z[f] : z[f] + beta * p[f];
}

// x += alpha p, r -= alpha Ap with alpha = rz / pAp; pAp <= 0: no update, the
// failure flag is set (sparse.cpp:83-86); rz_old = rz for the next direction
__global__ void update_dev_kernel(long n, double* __restrict__ sc, const double* __restrict__ p,
                                  const double* __restrict__ Ap, double* __restrict__ x,
                                  double* __restrict__ r) {
  const double pAp = sc[kPap], rz = sc[kRz];
  if (!(pAp > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[kFail] = 1.0;
    return;
  }
  const double alpha = rz / pAp;
  for (long f = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<long>(gridDim.x) * blockDim.x) {
    x[f] += alpha * p[f];
    r[f] -= alpha * Ap[f];
  }
}

__global__ void shift_rz_kernel(double* sc) { sc[kRzOld] = sc[kRz]; }

// a.b into the device scalar slot (fixed-order reduction)
void dot_dev(long n, const double* a, const double* b, const FdmWork& w, double* slot,
             cudaStream_t s) {
  dot2_partial<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, nullptr, nullptr, w.partials);
  dot2_final<<<1, kDotThreads, 0, s>>>(kDotBlocks, w.partials, w.dots + 6);
  TG_CUDA(cudaMemcpyAsync(slot, w.dots + 6, sizeof(double), cudaMemcpyDeviceToDevice, s));
}
}  // namespace

// The reference's loop with every scalar kept on the device: per iteration
// one host synchronisation (the stop test on r.r), none for r.z and p.Ap.
PcgStatus pcg_precond_solve(const std::function<void(const double*, double*)>& apply,
                            const FdmDev& F, long n, const double* rhs, double* x,
                            const FdmWork& w, double tol, int max_iter, cudaStream_t s) {
  const int G = grid_for(n);
  double bb = 0.0, unused = 0.0;
  dot2(n, rhs, rhs, nullptr, nullptr, w, s, bb, unused);
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {  // sparse.cpp:57-60
    TG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    return PcgStatus{0, 0, 0.0, 0.0};
  }
  double* sc = w.dots;
  TG_CUDA(cudaMemsetAsync(sc, 0, 6 * sizeof(double), s));
  // r = b - A x (sparse.cpp:61-69); z = P r is formed after the stop test
  apply(x, w.Ap);
  residual_kernel<<<G, 256, 0, s>>>(n, rhs, w.Ap, w.r);
  double rr = 0.0;
  dot2(n, w.r, w.r, nullptr, nullptr, w, s, rr, unused);
  double rel = 0.0;
  for (int it = 0; it < max_iter; ++it) {
    rel = std::sqrt(rr) / bnorm;
    if (rel <= tol) return PcgStatus{it, 0, rel, bnorm};
    fdm_apply(F, w.r, w.z, w.t1, w.t2, s);
    dot_dev(n, w.r, w.z, w, sc + kRz, s);
    direction_dev_kernel<<<G, 256, 0, s>>>(n, it == 0, sc, w.z, w.p);  // p = z + beta p
    shift_rz_kernel<<<1, 1, 0, s>>>(sc);
    apply(w.p, w.Ap);
    dot_dev(n, w.p, w.Ap, w, sc + kPap, s);
    update_dev_kernel<<<G, 256, 0, s>>>(n, sc, w.p, w.Ap, x, w.r);
    dot_dev(n, w.r, w.r, w, sc + kRr, s);
    TG_CUDA(cudaMemcpyAsync(w.h_dots, sc + kRr, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if (w.h_dots[1] != 0.0) return PcgStatus{it, 4, rel, bnorm};
    rr = w.h_dots[0];
  }
  return PcgStatus{max_iter, 3, rel, bnorm};
}

PcgStatus fdm_pcg_solve(const KronGrid& g, double a, double b, const FdmDev& F, const double* rhs,
                        double* x, const FdmWork& w, double tol, int max_iter, int sm_count,
                        cudaStream_t s, const TensorMap3* x_map, const TensorMap3* p_map) {
  const long n = static_cast<long>(g.n[0]) * g.n[1] * g.n[2];
  return pcg_precond_solve(
      [&](const double* v, double* y) {
        k2_apply(g, a, b, v, y, sm_count, s, v == x ? x_map : (v == w.p ? p_map : nullptr));
      },
      F, n, rhs, x, w, tol, max_iter, s);
}

}  // namespace tgb
