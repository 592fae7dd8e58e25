// C ABI entry points (include/thermiga_b200.h): argument checking, exception ->
// status mapping, host<->device staging. All arithmetic runs in the sm_100a
// kernels; there is no CPU fallback.
#include <cstring>
#include <exception>

#include "context.hpp"

namespace tgb {

namespace {

int fail(tg_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

template <typename F>
int guarded(tg_ctx* ctx, F&& body) {
  try {
    body();
    return TG_OK;
  } catch (const config_error& e) {
    return fail(ctx, TG_ECONFIG, e.what());
  } catch (const io_error& e) {
    return fail(ctx, TG_EIO, e.what());
  } catch (const numeric_error& e) {
    return fail(ctx, TG_ENUMERIC, e.what());
  } catch (const cuda_error& e) {
    return fail(ctx, TG_ECUDA, e.what());
  } catch (const std::exception& e) {
    return fail(ctx, TG_ERROR, e.what());
  }
}

Material to_material(const tg_material* m) {
  Material out;
  out.conductivity = m->conductivity;
  out.density = m->density;
  out.heat_capacity = m->heat_capacity;
  out.platform_temperature = m->platform_temperature;
  return out;
}

}  // namespace

void k1_run(tg_ctx* ctx, const double* d_src6, int n_src, const double* d_pts,
            const int* d_index, long n_pts_l, double t, double cull, K1Mode mode,
            double* d_out_a, double* d_out_b, const K1Flux& flux, cudaStream_t stream,
            int src_begin, int src_end) {
  if (n_pts_l <= 0) return;
  // launches of at most 2^28 points (int indexing, bounded partial buffers);
  // every point's sum is independent of the chunking
  constexpr long kChunk = 1L << 28;
  if (n_pts_l > kChunk) {
    for (long off = 0; off < n_pts_l; off += kChunk) {
      const long n = std::min(kChunk, n_pts_l - off);
      K1Flux f = flux;
      if (f.index) f.index += off;
      const bool fl = mode == K1Mode::flux;
      k1_run(ctx, d_src6, n_src, d_index || fl ? d_pts : d_pts + 3 * off,
             d_index ? d_index + off : nullptr, n, t, cull, mode, d_out_a + off,
             d_out_b ? d_out_b + 3 * off : nullptr, f, stream, src_begin, src_end);
    }
    return;
  }
  const int n_pts = static_cast<int>(n_pts_l);
  const Material& m = ctx->mat;
  const double alpha = m.diffusivity();
  const double rcp = m.volumetric_capacity();
  // gradients only where a caller reads them (flux integrand, or a field call
  // with a gradient output): value-only launches skip 4 of 17 FP64 ops per pair
  const bool grad = mode == K1Mode::flux || (mode == K1Mode::field && d_out_b != nullptr);
  const int P = grad ? ctx->k1_points_per_thread : ctx->k1_points_per_thread_value;
  const bool own_src = d_src6 == ctx->src6.p && static_cast<int>(ctx->tau_sufmin.size()) == n_src;
  if (own_src) n_src = ctx->active_prefix(t);  // trailing inactive sources: exact zeros
  // sources [src_begin, src_end) only (the K5 split hands the rest to a GEMM)
  if (src_end >= 0) n_src = std::min(n_src, src_end);
  src_begin = std::max(0, std::min(src_begin, n_src));
  d_src6 += 6 * static_cast<size_t>(src_begin);
  n_src -= src_begin;
  const bool planar = own_src && ctx->planar && !std::getenv("TG_K1_NO_PLANAR");
  int S = 1;
  if (n_src > 0) {
    k1_prepare(d_src6, n_src, t, alpha, rcp, cull, ctx->rec.ensure(n_src), stream);
    ++ctx->timer.launches;
    S = k1_choose_splits(n_pts, n_src, ctx->sm_count, kK1Threads * P, k1_resident_ctas(P));
  }
  double* part = ctx->part.ensure(static_cast<size_t>(S) * (grad ? 4 : 1) * n_pts);
  if (n_src > 0) {
    ctx->timer.timed(1, stream, [&] {
      k1_launch_partial(ctx->rec.p, n_src, d_pts, d_index, n_pts, S, grad, P, part, stream,
                        planar, ctx->planar_z);
    });
    ++ctx->timer.launches;
    ++ctx->timer.k1_launches;
    ctx->timer.k1_pairs += static_cast<double>(n_pts) * n_src;
  } else {
    TG_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * (grad ? 4 : 1) * n_pts, stream));
  }
  switch (mode) {
    case K1Mode::field:
      if (grad)
        k1_launch_combine_field(part, S, n_pts, d_out_a, d_out_b, stream);
      else
        k1_launch_combine_dirichlet(part, S, n_pts, d_out_a, stream, false);
      break;
    case K1Mode::dirichlet:
      k1_launch_combine_dirichlet(part, S, n_pts, d_out_a, stream);
      break;
    case K1Mode::flux:
      k1_launch_combine_flux(part, S, n_pts, flux.index, flux.normals, flux.weights, flux.k,
                             d_out_a, stream);
      break;
  }
  ++ctx->timer.launches;
  TG_CUDA(cudaGetLastError());
}

}  // namespace tgb

using namespace tgb;

extern "C" {

int tg_abi_version(void) { return 1; }

int tg_ctx_create(int device, tg_ctx** out) {
  if (!out) return TG_ERROR;
  *out = nullptr;
  auto* ctx = new tg_ctx();
  const int rc = guarded(ctx, [&] {
    int n = 0;
    TG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw cuda_error("cuda: no such device");
    cudaDeviceProp prop;
    TG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw cuda_error("cuda: device " + std::string(prop.name) + " is not sm_100-class");
    TG_CUDA(cudaSetDevice(device));
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    TG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    if (const char* p = std::getenv("TG_K1_P")) {  // points per thread: 1..8
      const int v = std::atoi(p);
      if (v >= 1 && v <= 8) ctx->k1_points_per_thread = v;
    }
    if (const char* p = std::getenv("TG_K1_P0")) {  // value-only launches: 1..8
      const int v = std::atoi(p);
      if (v >= 1 && v <= 8) ctx->k1_points_per_thread_value = v;
    }
    k1_upload_exp_table(ctx->stream);
    TG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
  if (rc != TG_OK) {
    // keep the context alive so the caller can read the error, then it must destroy it
    *out = ctx;
    return rc;
  }
  *out = ctx;
  return TG_OK;
}

void tg_ctx_destroy(tg_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

const char* tg_last_error(const tg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tg_set_profiling(tg_ctx* ctx, int on) {
  return guarded(ctx, [&] {
    ctx->timer.reset();
    ctx->timer.on = on != 0;
  });
}

int tg_profile_read(tg_ctx* ctx, double* out, int reset) {
  return guarded(ctx, [&] {
    TG_CUDA(cudaSetDevice(ctx->device));
    ctx->timer.collect();
    out[0] = ctx->timer.k1_ms;
    out[1] = static_cast<double>(ctx->timer.k1_launches);
    out[2] = ctx->timer.k1_pairs;
    out[3] = ctx->timer.k2_ms;
    out[4] = static_cast<double>(ctx->timer.k2_launches);
    out[5] = ctx->timer.k2_bytes;
    out[6] = static_cast<double>(ctx->timer.launches);
    out[7] = ctx->timer.step_ms;  // whole theta steps (expand + RHS + solve)
    out[8] = ctx->timer.k5_ms;    // K5 contraction launches
    out[9] = static_cast<double>(ctx->timer.k5_launches);
    out[10] = ctx->timer.run_ms;  // whole time steps (tg_sim_advance), device events
    if (reset) ctx->timer.reset();
  });
}

int tg_discretize_scan(const double* wp, int n_wp, double start_time, double plane_z,
                       const tg_laser* laser, const tg_material* mat, tg_point_source* out,
                       int max_out) {
  try {
    ScanPath path;
    for (int i = 0; i < n_wp; ++i) path.waypoints.push_back({wp[2 * i], wp[2 * i + 1]});
    path.start_time = start_time;
    path.plane_z = plane_z;
    LaserSpec ls;
    ls.power = laser->power;
    ls.speed = laser->speed;
    ls.spot_radius = laser->spot_radius;
    ls.absorptivity = laser->absorptivity;
    ls.dt = laser->dt;
    const auto src = discretize_scan(path, ls, to_material(mat));
    const int n = static_cast<int>(src.size());
    if (out && max_out > 0)
      std::memcpy(out, src.data(), sizeof(tg_point_source) * std::min(n, max_out));
    return n;
  } catch (const std::exception&) {
    return -TG_ERROR;
  }
}

int tg_set_sources(tg_ctx* ctx, const tg_point_source* src, int n, const tg_material* mat) {
  return guarded(ctx, [&] {
    if (n < 0 || (n > 0 && !src) || !mat) throw std::invalid_argument("set_sources: bad args");
    Material m = to_material(mat);
    m.validate();
    TG_CUDA(cudaSetDevice(ctx->device));
    ctx->mat = m;
    ctx->n_src = n;
    ctx->set_tau(reinterpret_cast<const double*>(src), n);
    double* d = ctx->src6.ensure(static_cast<size_t>(n) * 6);
    if (n > 0)
      TG_CUDA(cudaMemcpyAsync(d, src, sizeof(tg_point_source) * n, cudaMemcpyHostToDevice,
                              ctx->stream));
    TG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tg_superpose_batch(tg_ctx* ctx, const double* pts, long n, double t, double cull,
                       double* out_val, double* out_grad) {
  return guarded(ctx, [&] {
    if (n < 0 || (n > 0 && (!pts || !out_val)))
      throw std::invalid_argument("superpose: bad args");
    if (n == 0) return;
    TG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    double* dp = ctx->pts.ensure(3 * static_cast<size_t>(n));
    double* dv = ctx->val.ensure(n);
    double* dg = out_grad ? ctx->grad.ensure(3 * static_cast<size_t>(n)) : nullptr;
    TG_CUDA(cudaMemcpyAsync(dp, pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    k1_run(ctx, ctx->src6.p, ctx->n_src, dp, nullptr, n, t, cull, K1Mode::field, dv, dg, {}, s);
    TG_CUDA(cudaMemcpyAsync(out_val, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    if (out_grad)
      TG_CUDA(cudaMemcpyAsync(out_grad, dg, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
  });
}

int tg_superpose_batch_device(tg_ctx* ctx, const double* d_pts, long n, double t, double cull,
                              double* d_val, double* d_grad, void* stream) {
  return guarded(ctx, [&] {
    if (n < 0 || (n > 0 && (!d_pts || !d_val)))
      throw std::invalid_argument("superpose: bad args");
    TG_CUDA(cudaSetDevice(ctx->device));
    k1_run(ctx, ctx->src6.p, ctx->n_src, d_pts, nullptr, n, t, cull, K1Mode::field, d_val,
           d_grad, {}, ctx->pick(stream));
  });
}

}  // extern "C"
