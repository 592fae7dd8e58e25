// K2 general path — theta-step PCG on an assembled CSR operator, for patches
// that are not separable (rational geometry such as the reference's
// quarter-cylinder part, proj/src/splines.cpp:408-438). Same persistent
// cooperative structure and reductions as the Kronecker path (k2_kron.cu); the
// row products follow CsrMatrix::multiply (proj/src/sparse.cpp:25-31) term by
// term without contraction, so each matvec row equals the reference's bit for
// bit.
#include <cooperative_groups.h>

#include <algorithm>

#include "context.hpp"
#include "k2_csr.cuh"

namespace cg = cooperative_groups;

namespace tgb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double row_dot(const DevCsr& A, int r, const double* __restrict__ x) {
  double acc = 0.0;
  int k = A.row_ptr[r];
  const int e = A.row_ptr[r + 1];
  for (; k + 4 <= e; k += 4) {  // loads batched, adds in order
    double vv[4], xx[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) vv[u] = A.val[k + u];
#pragma unroll
    for (int u = 0; u < 4; ++u) xx[u] = x[A.col[k + u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(vv[u], xx[u]));
  }
  for (; k < e; ++k) acc = __dadd_rn(acc, __dmul_rn(A.val[k], x[A.col[k]]));
  return acc;
}

// the same sum over the sliced layout (coalesced across the 32 rows of a
// slice). The row's terms are added strictly in order, so the loads are
// batched (kBatch values, columns and gathered x in flight per thread) to
// hide memory latency behind the sequential add chain.
#ifndef K2_SELL_BATCH
#define K2_SELL_BATCH 16  // config 3 (302,974 rows): 4 -> 335, 8 -> 215, 16 -> 199 us per CG iteration
#endif
constexpr int kBatch = K2_SELL_BATCH;
__device__ __forceinline__ double row_dot(const DevSell& A, int r, const double* __restrict__ x) {
  const long long base = A.slice_ptr[r >> 5] + (r & 31);
  const int len = A.row_len[r];
  const double* __restrict__ v = A.val + base;
  const int* __restrict__ c = A.col + base;
  double acc = 0.0;
  int k = 0;
  for (; k + kBatch <= len; k += kBatch) {
    double vv[kBatch], xx[kBatch];
    int cc[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      vv[u] = __ldcs(v + 32 * (k + u));
      cc[u] = __ldcs(c + 32 * (k + u));
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) xx[u] = x[cc[u]];  // (x is written in-kernel: no .nc)
#pragma unroll
    for (int u = 0; u < kBatch; ++u) acc = __dadd_rn(acc, __dmul_rn(vv[u], xx[u]));
  }
  for (; k < len; ++k) acc = __dadd_rn(acc, __dmul_rn(__ldcs(v + 32 * k), x[__ldcs(c + 32 * k)]));
  return acc;
}

// the same sum over the implicit-column layout: the (2p+1)^3 offsets in
// ascending order (the CSR's column order); offsets a boundary row lacks hold
// exact zeros, whose products add nothing (+-0), and their x index is clamped
// into the vector. Loads go out K2_DIA_ROWS stencil rows (of 2p+1 terms) at a
// time ahead of the in-order adds.
#ifndef K2_DIA_ROWS
#define K2_DIA_ROWS 4  // config 3 per CG iteration: 1 -> 152.5 us, 2 -> 149.6, 3 -> 147.6, 4 -> 138.9, 7 -> 150.1
#endif
template <int P>
__device__ __forceinline__ double row_dot_dia(const DevDia& A, int r,
                                              const double* __restrict__ x) {
  constexpr int W = 2 * P + 1, RB = K2_DIA_ROWS, NB = RB * W;
  const double* __restrict__ v = A.val + static_cast<size_t>(r >> 5) * A.noff * 32 + (r & 31);
  const int n1 = A.rows - 1;
  double acc = 0.0;
#pragma unroll 1
  for (int dk = -P; dk <= P; ++dk) {
    const int kb = r + dk * A.nxy - P;
    const double* vk = v + 32 * ((dk + P) * W * W);
#pragma unroll
    for (int j0 = 0; j0 < W; j0 += RB) {
      double vv[NB], xx[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int jj = j0 + t / W, u = t % W;
        if (jj < W) {
          vv[t] = __ldcs(vk + 32 * (jj * W + u));
          xx[t] = x[min(max(kb + (jj - P) * A.nx + u, 0), n1)];
        }
      }
#pragma unroll
      for (int t = 0; t < NB; ++t)
        if (j0 + t / W < W) acc = __dadd_rn(acc, __dmul_rn(vv[t], xx[t]));
    }
  }
  return acc;
}
__device__ __forceinline__ double row_dot(const DevDia& A, int r, const double* __restrict__ x) {
  switch (A.p) {
    case 1: return row_dot_dia<1>(A, r, x);
    case 2: return row_dot_dia<2>(A, r, x);
    default: return row_dot_dia<3>(A, r, x);
  }
}

__device__ __forceinline__ double diag_of(const DevCsr& A, int r) {
  double d = 0.0;
  for (int k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k)
    if (A.col[k] == r) d = A.val[k];
  return d;
}
__device__ __forceinline__ double diag_of(const DevSell& A, int r) {
  const long long base = A.slice_ptr[r >> 5] + (r & 31);
  double d = 0.0;
  for (int k = 0; k < A.row_len[r]; ++k)
    if (A.col[base + 32 * k] == r) d = A.val[base + 32 * k];
  return d;
}

__device__ __forceinline__ void grid_reduce(cg::grid_group& grid, double (&acc)[4],
                                            double* partials, int& buf, double* red,
                                            double (&out)[4]) {
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

template <class Mat>
__global__ void __launch_bounds__(kThreads) csr_pcg_kernel(Mat A, const double* rhs, double* x,
                                                           CsrWork w, double tol, int max_iter) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[64];
  const int n = A.rows;
  const int gtid = blockIdx.x * kThreads + threadIdx.x;
  const int gstride = gridDim.x * kThreads;
  int buf = 0;
  double tot[4];
  double acc[4] = {0, 0, 0, 0};
  for (int f = gtid; f < n; f += gstride) {
    const double bi = rhs[f];
    const double ri = bi - row_dot(A, f, x);
    const double zi = w.inv_diag[f] * ri;
    w.r[f] = ri;
    w.p[f] = zi;
    acc[0] += ri * ri;
    acc[1] += bi * bi;
    acc[2] += ri * zi;
  }
  grid_reduce(grid, acc, w.partials, buf, red, tot);
  double rr = tot[0], rz = tot[2];
  const double bnorm = sqrt(tot[1]);
  if (bnorm == 0.0) {
    for (int f = gtid; f < n; f += gstride) x[f] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *w.status = PcgStatus{0, 0, 0.0, 0.0};
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
    double a1[4] = {0, 0, 0, 0};
    for (int f = gtid; f < n; f += gstride) {
      const double y = row_dot(A, f, w.p);
      w.Ap[f] = y;
      a1[0] += w.p[f] * y;
    }
    grid_reduce(grid, a1, w.partials, buf, red, tot);
    const double pAp = tot[0];
    if (!(pAp > 0.0)) {
      status = 4;
      break;
    }
    const double alpha = rz / pAp;
    double a2[4] = {0, 0, 0, 0};
    for (int f = gtid; f < n; f += gstride) {
      x[f] += alpha * w.p[f];
      const double ri = w.r[f] - alpha * w.Ap[f];
      w.r[f] = ri;
      const double zi = w.inv_diag[f] * ri;
      a2[0] += ri * zi;
      a2[1] += ri * ri;
    }
    grid_reduce(grid, a2, w.partials, buf, red, tot);
    const double beta = tot[0] / rz;
    rz = tot[0];
    rr = tot[1];
    for (int f = gtid; f < n; f += gstride) w.p[f] = w.inv_diag[f] * w.r[f] + beta * w.p[f];
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *w.status = PcgStatus{it, status, rel, bnorm};
}

template <class Mat>
__global__ void csr_diag_kernel(Mat A, double* inv_diag, PcgStatus* st) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= A.rows) return;
  const double d = diag_of(A, r);
  if (!(d > 0.0)) st->status = 2;
  inv_diag[r] = 1.0 / d;
}

// rhs_f = [B T]_f - [A g~]_f + theta F1 + (1 - theta) F0 (assembly.cpp:258-271)
__global__ void csr_rhs_kernel(DevSell Bf, DevSell Ac, const double* T, const double* g1,
                               const double* F0, const double* F1, const int* free_list,
                               double theta, double* rhs) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= Bf.rows) return;
  const int g = free_list[f];
  const double bt = row_dot(Bf, f, T);
  const double ag = row_dot(Ac, f, g1);
  rhs[f] = bt - ag + theta * F1[g] + (1.0 - theta) * F0[g];
}

}  // namespace

int csr_pcg_max_blocks(int sm_count) {
  int a = 0, b = 0;
  TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &a, reinterpret_cast<const void*>(&csr_pcg_kernel<DevCsr>), kThreads, 0));
  TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b, reinterpret_cast<const void*>(&csr_pcg_kernel<DevSell>), kThreads, 0));
  int c = 0;
  TG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &c, reinterpret_cast<const void*>(&csr_pcg_kernel<DevDia>), kThreads, 0));
  return std::max(1, std::min(std::min(a, b), c)) * sm_count;
}

template <class Mat>
void inverse_diagonal(const Mat& A, double* inv_diag, PcgStatus* st, cudaStream_t s) {
  if (A.rows <= 0) return;
  csr_diag_kernel<<<(A.rows + 255) / 256, 256, 0, s>>>(A, inv_diag, st);
  TG_CUDA(cudaGetLastError());
}
void csr_inverse_diagonal(const DevCsr& A, double* inv_diag, PcgStatus* st, cudaStream_t s) {
  inverse_diagonal(A, inv_diag, st, s);
}
void csr_inverse_diagonal(const DevSell& A, double* inv_diag, PcgStatus* st, cudaStream_t s) {
  inverse_diagonal(A, inv_diag, st, s);
}

void csr_theta_rhs(const DevSell& Bf, const DevSell& Ac, const double* T, const double* g1,
                   const double* F0, const double* F1, const int* free_list, double theta,
                   double* rhs, cudaStream_t s) {
  if (Bf.rows <= 0) return;
  csr_rhs_kernel<<<(Bf.rows + 255) / 256, 256, 0, s>>>(Bf, Ac, T, g1, F0, F1, free_list, theta,
                                                       rhs);
  TG_CUDA(cudaGetLastError());
}

template <class Mat>
void pcg_solve(const Mat& A, const double* rhs, double* x, const CsrWork& w, double tol,
               int max_iter, int blocks, cudaStream_t s) {
  const int need = (A.rows + kThreads - 1) / kThreads;
  const int nb = std::max(1, std::min(blocks, need));
  Mat AA = A;
  CsrWork ww = w;
  double tt = tol;
  int mi = max_iter;
  void* args[] = {&AA, const_cast<double**>(&rhs), &x, &ww, &tt, &mi};
  TG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&csr_pcg_kernel<Mat>),
                                      dim3(nb), dim3(kThreads), args, 0, s));
}
void csr_pcg_solve(const DevCsr& A, const double* rhs, double* x, const CsrWork& w, double tol,
                   int max_iter, int blocks, cudaStream_t s) {
  pcg_solve(A, rhs, x, w, tol, max_iter, blocks, s);
}
void csr_pcg_solve(const DevSell& A, const double* rhs, double* x, const CsrWork& w, double tol,
                   int max_iter, int blocks, cudaStream_t s) {
  pcg_solve(A, rhs, x, w, tol, max_iter, blocks, s);
}

void csr_pcg_solve(const DevDia& A, const double* rhs, double* x, const CsrWork& w, double tol,
                   int max_iter, int blocks, cudaStream_t s) {
  pcg_solve(A, rhs, x, w, tol, max_iter, blocks, s);
}

namespace {
// scatter every SELL entry of row r into its offset slot (flag: an entry
// outside the stencil)
__global__ void csr_to_dia_kernel(DevSell A, int nx, int ny, int p, double* val, int* flag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= A.rows) return;
  const int W = 2 * p + 1, noff = W * W * W;
  const int ri = r % nx, rj = (r / nx) % ny, rk = r / (nx * ny);
  const long long base = A.slice_ptr[r >> 5] + (r & 31);
  double* out = val + static_cast<size_t>(r >> 5) * noff * 32 + (r & 31);
  for (int k = 0; k < A.row_len[r]; ++k) {
    const int c = A.col[base + 32 * k];
    const int di = c % nx - ri, dj = (c / nx) % ny - rj, dk = c / (nx * ny) - rk;
    if (abs(di) > p || abs(dj) > p || abs(dk) > p) {
      atomicExch(flag, 1);
      return;
    }
    out[32 * (((dk + p) * W + dj + p) * W + di + p)] = A.val[base + 32 * k];
  }
}
}  // namespace

bool csr_make_dia(const DevSell& A, int nx, int ny, int nz, int p, double* val, int* d_flag,
                  DevDia* out, cudaStream_t s) {
  if (A.rows != nx * ny * nz || A.rows <= 0) return false;
  const int W = 2 * p + 1;
  const size_t n = static_cast<size_t>((A.rows + 31) / 32) * 32 * W * W * W;
  TG_CUDA(cudaMemsetAsync(val, 0, n * sizeof(double), s));
  TG_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
  csr_to_dia_kernel<<<(A.rows + 255) / 256, 256, 0, s>>>(A, nx, ny, p, val, d_flag);
  TG_CUDA(cudaGetLastError());
  int flag = 0;
  TG_CUDA(cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (flag) return false;
  *out = DevDia{A.rows, nx, nx * ny, p, W * W * W, val};
  return true;
}

namespace {
template <class Mat>
__global__ void csr_apply_kernel(Mat A, const double* x, double* y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < A.rows) y[r] = row_dot(A, r, x);
}
template <class Mat>
void apply(const Mat& A, const double* x, double* y, cudaStream_t s) {
  if (A.rows <= 0) return;
  csr_apply_kernel<<<(A.rows + 255) / 256, 256, 0, s>>>(A, x, y);
  TG_CUDA(cudaGetLastError());
}
}  // namespace

void csr_apply(const DevCsr& A, const double* x, double* y, cudaStream_t s) { apply(A, x, y, s); }
void csr_apply(const DevDia& A, const double* x, double* y, cudaStream_t s) { apply(A, x, y, s); }
void csr_apply(const DevSell& A, const double* x, double* y, cudaStream_t s) { apply(A, x, y, s); }

}  // namespace tgb
