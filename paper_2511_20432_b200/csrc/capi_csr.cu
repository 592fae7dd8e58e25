// C ABI for the sparse-LA layer on a caller matrix: pcg_jacobi and
// CsrMatrix::multiply (proj/include/thermiga/sparse.hpp:45-46,
// proj/src/sparse.cpp:25-100) on the context's GPU — the persistent CSR PCG
// kernel of k2_csr.cu behind the reference's signature and error behaviour.
#include <cstdio>
#include <stdexcept>

#include "context.hpp"
#include "k2_csr.cuh"

namespace {

using namespace tgb;

struct DevMatrix {
  DevBuf<int> rp, ci;
  DevBuf<double> v;
  DevCsr A{};
  void upload(int rows, const int* row_ptr, const int* col, const double* val, cudaStream_t s) {
    if (rows < 0 || (rows > 0 && (!row_ptr || !col || !val)))
      throw std::invalid_argument("csr: bad arguments");
    const int nnz = rows > 0 ? row_ptr[rows] : 0;
    rp.ensure(rows + 1);
    ci.ensure(nnz);
    v.ensure(nnz);
    TG_CUDA(cudaMemcpyAsync(rp.p, row_ptr, sizeof(int) * (rows + 1), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
      TG_CUDA(cudaMemcpyAsync(ci.p, col, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
      TG_CUDA(cudaMemcpyAsync(v.p, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    }
    A = DevCsr{rows, rp.p, ci.p, v.p};
  }
};

template <typename F>
int guarded(tg_ctx* ctx, F&& body) {
  try {
    body();
    return TG_OK;
  } catch (const numeric_error& e) {
    ctx->err = e.what();
    return TG_ENUMERIC;
  } catch (const cuda_error& e) {
    ctx->err = e.what();
    return TG_ECUDA;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return TG_ERROR;
  }
}

}  // namespace

extern "C" {

int tg_csr_multiply(tg_ctx* ctx, int rows, const int* row_ptr, const int* col, const double* val,
                    const double* x, double* y) {
  return guarded(ctx, [&] {
    TG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    DevMatrix M;
    M.upload(rows, row_ptr, col, val, s);
    if (rows == 0) return;
    DevBuf<double> dx, dy;
    dx.ensure(rows);
    dy.ensure(rows);
    TG_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * rows, cudaMemcpyHostToDevice, s));
    csr_apply(M.A, dx.p, dy.p, s);
    TG_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * rows, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
  });
}

int tg_pcg_jacobi(tg_ctx* ctx, int rows, const int* row_ptr, const int* col, const double* val,
                  const double* b, double* x, double tol, int max_iter, int* iterations,
                  double* rel_residual) {
  return guarded(ctx, [&] {
    if (!b || !x) throw std::invalid_argument("pcg: dimension mismatch");
    TG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    DevMatrix M;
    M.upload(rows, row_ptr, col, val, s);
    const int n = rows;
    DevBuf<double> db, dx, r, p, Ap, inv, part;
    DevBuf<PcgStatus> st;
    const int blocks = csr_pcg_max_blocks(ctx->sm_count);
    db.ensure(n);
    dx.ensure(n);
    r.ensure(n);
    p.ensure(n);
    Ap.ensure(n);
    inv.ensure(n);
    part.ensure(8 * static_cast<size_t>(blocks) + 8);
    st.ensure(1);
    TG_CUDA(cudaMemsetAsync(st.p, 0, sizeof(PcgStatus), s));
    if (n > 0) {
      TG_CUDA(cudaMemcpyAsync(db.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      TG_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      csr_inverse_diagonal(M.A, inv.p, st.p, s);  // sparse.cpp:47-52
    }
    PcgStatus h{};
    TG_CUDA(cudaMemcpyAsync(&h, st.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    if (h.status == 2) throw numeric_error("pcg: non-positive diagonal, matrix not SPD");
    if (n > 0) {
      const CsrWork w{r.p, p.p, Ap.p, inv.p, part.p, st.p};
      csr_pcg_solve(M.A, db.p, dx.p, w, tol, max_iter, blocks, s);
      TG_CUDA(cudaMemcpyAsync(&h, st.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
      TG_CUDA(cudaMemcpyAsync(x, dx.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      TG_CUDA(cudaStreamSynchronize(s));
    }
    if (iterations) *iterations = h.iterations;
    if (rel_residual) *rel_residual = h.rel_residual;
    if (h.status == 4) throw numeric_error("pcg: indefinite direction, matrix not SPD");
    if (h.status == 3) {
      char buf[64];
      std::snprintf(buf, sizeof(buf), "%.17g", h.rel_residual);
      throw numeric_error("pcg: no convergence in " + std::to_string(max_iter) +
                          " iterations, relative residual " + buf);
    }
  });
}

}  // extern "C"
