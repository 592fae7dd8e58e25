// Simulation engine behind tg_sim_*: the host-side setup of the reference's
// prepare_simulation (proj/src/driver.cpp:66-95) in C++, and the per-step hot
// path of run_time_loop (driver.cpp:126-145) on the GPU:
//   F_{n+1} = assemble_flux_load(t)   K1 (flux mode) + K3
//   g_{n+1} = dirichlet_values(t)     K1 (value mode) at the Greville points
//   theta_step                        K2: RHS kernel + persistent Jacobi-PCG
// State (free coefficients, constrained values, loads) stays resident in HBM
// between steps; the host only decides the fine-rule element set per step
// (the reference's exact arithmetic) and reads back the PCG status.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>

#include "context.hpp"
#include "host/config.hpp"
#include "host/fdm.hpp"
#include "host/parallel.hpp"
#include "host/operator.hpp"
#include "k2_csr.cuh"
#include "k2_kron.cuh"
#include "k3_flux.cuh"
#include "sim.hpp"

namespace tgb {

namespace {

__global__ void expand_kernel(SimGeom g, const double* __restrict__ x,
                              const double* __restrict__ gc, double* __restrict__ T) {
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long n = static_cast<long>(g.n[0]) * g.n[1] * g.n[2];
  if (idx >= n) return;
  int ijk[3] = {static_cast<int>(idx % g.n[0]), static_cast<int>((idx / g.n[0]) % g.n[1]),
                static_cast<int>(idx / (static_cast<long>(g.n[0]) * g.n[1]))};
  if (ijk[g.ax] == g.layer) {
    T[idx] = gc[ijk[g.t0] + g.n[g.t0] * ijk[g.t1]];
  } else {
    if (g.layer == 0) ijk[g.ax] -= 1;
    int nf[3] = {g.n[0], g.n[1], g.n[2]};
    nf[g.ax] -= 1;
    T[idx] = x[ijk[0] + static_cast<long>(nf[0]) * (ijk[1] + static_cast<long>(nf[1]) * ijk[2])];
  }
}

__global__ void scatter_layer_kernel(SimGeom g, const double* __restrict__ gc,
                                     double* __restrict__ full) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int nc = g.n[g.t0] * g.n[g.t1];
  if (c >= nc) return;
  int ijk[3];
  ijk[g.ax] = g.layer;
  ijk[g.t0] = c % g.n[g.t0];
  ijk[g.t1] = c / g.n[g.t0];
  full[ijk[0] + static_cast<long>(g.n[0]) * (ijk[1] + static_cast<long>(g.n[1]) * ijk[2])] = gc[c];
}

template <typename T>
void upload(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.ensure(h.size());
  if (!h.empty())
    TG_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

}  // namespace

Sim::Sim(const std::string& path, const SimOptions& opt) {
  RunConfig c = parse_config(path);
  if (opt.t_end > 0.0) c.stepping.t_end = opt.t_end;
  if (opt.solver_tol > 0.0) c.stepping.solver_tol = opt.solver_tol;
  if (opt.max_iter > 0) c.stepping.max_iter = opt.max_iter;
  cfg = std::move(c);
  setup_host();
  sf_setup_host();
  if (!opt.host_only) setup_device(opt.device, opt.preconditioner);
}

Sim::~Sim() {
  if (cublas) cublasDestroy(cublas);
  if (h_dots) cudaFreeHost(h_dots);
  if (h_status) cudaFreeHost(h_status);
  if (h_fine) cudaFreeHost(h_fine);
  if (h_sf_fine) cudaFreeHost(h_sf_fine);
  if (h_sf_rect) cudaFreeHost(h_sf_rect);
  for (auto& ev : sf_ev)
    if (ev) cudaEventDestroy(ev);
  if (sf_stream) cudaStreamDestroy(sf_stream);
  if (ctx) tg_ctx_destroy(ctx);
}

namespace {
// TG_SETUP_TIMING=1: per-phase wall times of the setup on stderr
struct PhaseClock {
  bool on = std::getenv("TG_SETUP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-28s %8.3f s\n", what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  }
};
}  // namespace

void Sim::setup_host() {
  PhaseClock clk;
  // prepare_simulation (driver.cpp:66-95)
  vol = refine_for_spec(cfg.geometry, cfg.mesh);
  const auto p = vol.degrees();
  for (int d = 0; d < 3; ++d) quad[d] = cfg.mesh.quad_order > 0 ? cfg.mesh.quad_order : p[d] + 1;
  dofs = make_dof_map(vol, cfg.tags);
  sources = discretize_scan(cfg.scan, cfg.laser, cfg.material);
  tact_max.resize(sources.size());
  double m = -INFINITY;
  for (size_t i = 0; i < sources.size(); ++i) tact_max[i] = m = std::max(m, sources[i].t_activate);
  dt_solver = cfg.stepping.dt / cfg.stepping.substeps;
  n_steps = static_cast<int>(std::ceil(cfg.stepping.t_end / dt_solver - 1e-9));

  const auto n = vol.basis_counts();
  const FaceId bottom = cfg.tags.bottom_face();
  geom.n[0] = n[0];
  geom.n[1] = n[1];
  geom.n[2] = n[2];
  geom.ax = face_axis(bottom);
  geom.layer = face_is_min(bottom) ? 0 : n[geom.ax] - 1;
  const auto t = face_tangent_axes(bottom);
  geom.t0 = t[0];
  geom.t1 = t[1];
  n_full = vol.n_functions();
  n_free = dofs.n_free();
  n_con = dofs.n_constrained();

  // lateral face sets, with the columns that are exactly zero on every
  // quadrature point of an element dropped (their scatter adds +0, a no-op)
  clk.mark("volume, dofs, sources");
  FaceSets fs = build_face_sets(vol, cfg.tags, cfg.mesh.boundary_quad_multiplier);
  clk.mark("face sets");
  n_fe = fs.n_elems;
  const int nd = fs.n_dofs;
  const long tqb = fs.qb_off.back(), tqf = fs.qf_off.back();
  if (tqb + tqf > (1L << 31) - 1) throw std::invalid_argument("face quadrature set too large");
  h_qb_off.assign(fs.qb_off.begin(), fs.qb_off.end());
  h_qf_off.assign(fs.qf_off.begin(), fs.qf_off.end());
  nqb = nqf = 0;
  for (int e = 0; e < n_fe; ++e) {
    nqb = std::max(nqb, fs.nqb[e]);
    nqf = std::max(nqf, fs.nqf[e]);
  }
  std::vector<std::vector<int>> keep(n_fe);
  parallel_for(n_fe, [&](long e) {
    for (int a = 0; a < nd; ++a) {
      bool nz = false;
      for (long q = fs.qb_off[e]; q < fs.qb_off[e + 1] && !nz; ++q) nz = fs.Nb[q * nd + a] != 0.0;
      for (long q = fs.qf_off[e]; q < fs.qf_off[e + 1] && !nz; ++q) nz = fs.Nf[q * nd + a] != 0.0;
      if (nz) keep[e].push_back(a);
    }
  });
  ndk = 1;
  for (int e = 0; e < n_fe; ++e) ndk = std::max<int>(ndk, static_cast<int>(keep[e].size()));
  centers = fs.centers;
  h_qx = fs.xb;
  h_qx.insert(h_qx.end(), fs.xf.begin(), fs.xf.end());
  h_qn = fs.nb;
  h_qn.insert(h_qn.end(), fs.nf.begin(), fs.nf.end());
  h_qw = fs.wb;
  h_qw.insert(h_qw.end(), fs.wf.begin(), fs.wf.end());
  h_Nb.assign(static_cast<size_t>(tqb) * ndk, 0.0);
  h_Nf.assign(static_cast<size_t>(tqf) * ndk, 0.0);
  h_dofk.assign(static_cast<size_t>(n_fe) * ndk, -1);
  parallel_for(n_fe, [&](long e) {
    for (size_t kk = 0; kk < keep[e].size(); ++kk) {
      const int a = keep[e][kk];
      for (long q = fs.qb_off[e]; q < fs.qb_off[e + 1]; ++q) h_Nb[q * ndk + kk] = fs.Nb[q * nd + a];
      for (long q = fs.qf_off[e]; q < fs.qf_off[e + 1]; ++q) h_Nf[q * ndk + kk] = fs.Nf[q * nd + a];
      h_dofk[static_cast<size_t>(e) * ndk + kk] = fs.dofs[static_cast<size_t>(e) * nd + a];
    }
  });
  // incidence lists per DOF in the reference's scatter order (face, element, a):
  // a stable counting sort of the kept (element, column) slots by DOF
  h_inc_ptr.assign(n_full + 1, 0);
  for (size_t s2 = 0; s2 < h_dofk.size(); ++s2)
    if (h_dofk[s2] >= 0) ++h_inc_ptr[h_dofk[s2] + 1];
  for (int i = 0; i < n_full; ++i) h_inc_ptr[i + 1] += h_inc_ptr[i];
  h_inc_src.assign(h_inc_ptr[n_full], 0);
  {
    std::vector<int> fill(h_inc_ptr.begin(), h_inc_ptr.end() - 1);
    for (size_t s2 = 0; s2 < h_dofk.size(); ++s2)
      if (h_dofk[s2] >= 0) h_inc_src[fill[h_dofk[s2]]++] = static_cast<int>(s2);
  }

  clk.mark("face tables, incidence");
  grev = greville_points(vol, dofs, cfg.tags);
  clk.mark("greville points");

  // operator: Kronecker factors when separable, else the assembled CSR pair
  std::array<std::vector<double>, 3> coord;
  // the Kronecker kernels take equal degrees 1..kKronMaxP; mixed or higher
  // degrees use the assembled operator like any non-separable patch
  {
    const auto pd = vol.degrees();
    const bool eq = pd[0] == pd[1] && pd[1] == pd[2] && pd[0] >= 1 && pd[0] <= kKronMaxP;
    kron = eq && separable_coords(vol, coord);
  }
  const double dt = dt_solver, th = cfg.stepping.theta;
  if (!(dt > 0.0)) throw std::invalid_argument("theta scheme: dt must be > 0");
  if (!(th >= 0.0 && th <= 1.0)) throw std::invalid_argument("theta scheme: theta must be in [0,1]");
  if (kron) {
    for (int d = 0; d < 3; ++d) band[d] = assemble_band_1d(vol.knots(d), coord[d], quad[d]);
    const double rc = cfg.material.volumetric_capacity(), k = cfg.material.conductivity;
    coefA = {rc / dt, th * k};
    coefB = {rc / dt, -(1.0 - th) * k};
    clk.mark("kronecker factors");
  } else {
    Csr M, K;
    assemble_mass_stiffness(vol, quad, cfg.material, M, K);
    clk.mark("csr assembly (M, K)");
    // A = M/dt + theta K, B = M/dt - (1-theta) K (assembly.cpp:194-199)
    const long nnz = static_cast<long>(M.val.size());
    std::vector<double> Av(nnz), Bv(nnz);
    parallel_for((nnz + 4095) / 4096, [&](long blk) {
      const long e = std::min(nnz, (blk + 1) * 4096);
      for (long i2 = blk * 4096; i2 < e; ++i2) {
        Av[i2] = (1.0 / dt) * M.val[i2] + th * K.val[i2];
        Bv[i2] = (1.0 / dt) * M.val[i2] + -(1.0 - th) * K.val[i2];
      }
    }, 1);
    // free rows of the pattern with values v; columns renumbered by `map`
    // (entries with map < 0 dropped; all kept when map is null): count,
    // prefix, fill, row-parallel
    auto extract = [&](const std::vector<double>& v, const std::vector<int>* map, Csr& out) {
      const Csr& S = M;  // the shared pattern
      out.rows = n_free;
      out.row_ptr.assign(n_free + 1, 0);
      parallel_for(n_free, [&](long f) {
        const int r = dofs.free_list[f];
        int c = 0;
        for (int q = S.row_ptr[r]; q < S.row_ptr[r + 1]; ++q) c += !map || (*map)[S.col[q]] >= 0;
        out.row_ptr[f + 1] = c;
      }, 256);
      for (int f = 0; f < n_free; ++f) out.row_ptr[f + 1] += out.row_ptr[f];
      out.col.resize(out.row_ptr[n_free]);
      out.val.resize(out.row_ptr[n_free]);
      parallel_for(n_free, [&](long f) {
        const int r = dofs.free_list[f];
        int o = out.row_ptr[f];
        for (int q = S.row_ptr[r]; q < S.row_ptr[r + 1]; ++q) {
          const int c = map ? (*map)[S.col[q]] : S.col[q];
          if (c < 0) continue;
          out.col[o] = c;
          out.val[o++] = v[q];
        }
      }, 256);
    };
    extract(Av, &dofs.free_index, csrA);
    extract(Av, &dofs.constrained_index, csrAc);
    extract(Bv, nullptr, csrB);  // free rows of B, all columns
    clk.mark("csr theta operators");
  }
}

void Sim::setup_device(int device, int preconditioner) {
  const int rc = tg_ctx_create(device, &ctx);
  if (rc != TG_OK) {
    const std::string msg = ctx ? ctx->err : std::string("context creation failed");
    if (ctx) tg_ctx_destroy(ctx);
    ctx = nullptr;
    throw cuda_error(msg);
  }
  cudaStream_t s = ctx->stream;
  ctx->mat = cfg.material;
  ctx->n_src = static_cast<int>(sources.size());
  static_assert(sizeof(PointSource) == 6 * sizeof(double), "PointSource layout");
  ctx->set_tau(reinterpret_cast<const double*>(sources.data()), ctx->n_src);
  double* d = ctx->src6.ensure(6 * sources.size());
  if (!sources.empty())
    TG_CUDA(cudaMemcpyAsync(d, sources.data(), sources.size() * sizeof(PointSource),
                            cudaMemcpyHostToDevice, s));
  upload(d_qx, h_qx, s);
  upload(d_qn, h_qn, s);
  upload(d_qw, h_qw, s);
  upload(d_Nb, h_Nb, s);
  upload(d_Nf, h_Nf, s);
  upload(d_inc_ptr, h_inc_ptr, s);
  upload(d_inc_src, h_inc_src, s);
  upload(d_grev, grev, s);
  upload(d_qb_off, h_qb_off, s);
  upload(d_qf_off, h_qf_off, s);
  const size_t max_pts = static_cast<size_t>(std::max(h_qb_off.back(), h_qf_off.back())) + 1;
  d_pt_index.ensure(max_pts);
  d_elem_off.ensure(n_fe + 1);
  d_fine.ensure(2 * static_cast<size_t>(n_fe) + 2);
  d_gq.ensure(max_pts);
  d_loc.ensure(static_cast<size_t>(n_fe) * ndk + 1);
  TG_CUDA(cudaMallocHost(&h_fine, sizeof(int) * (2 * static_cast<size_t>(n_fe) + 2)));
  TG_CUDA(cudaMallocHost(&h_status, sizeof(PcgStatus)));

  d_x.ensure(n_free);
  d_r.ensure(n_free);
  d_p.ensure(n_free);
  d_Ap.ensure(n_free);
  d_invd.ensure(n_free);
  d_rhs.ensure(n_free);
  d_gn.ensure(n_con);
  d_g1.ensure(n_con);
  d_Fn.ensure(n_full);
  d_F1.ensure(n_full);
  d_T.ensure(n_full);
  d_gfull.ensure(n_full);
  d_status.ensure(1);
  d_trace.ensure(400);
  trace_on = std::getenv("TG_K2_TRACE") != nullptr;
  if (trace_on) {
    TG_CUDA(cudaMemsetAsync(d_trace.p, 0, 400 * sizeof(unsigned long long), s));
  }
  TG_CUDA(cudaMemsetAsync(d_gfull.p, 0, sizeof(double) * n_full, s));
  TG_CUDA(cudaMemsetAsync(d_status.p, 0, sizeof(PcgStatus), s));

  if (kron) {
    const int p = band[0].p;
    if (band[1].p != p || band[2].p != p || p < 1 || p > kKronMaxP)  // excluded in setup_host
      throw std::logic_error("kronecker path needs equal degrees 1..3 in all directions");
    const int W = 2 * p + 1;
    std::vector<double> all;
    for (int d = 0; d < 3; ++d) {
      all.insert(all.end(), band[d].M.begin(), band[d].M.end());
      all.insert(all.end(), band[d].K.begin(), band[d].K.end());
    }
    upload(d_band, all, s);
    size_t off = 0;
    for (int d = 0; d < 3; ++d) {
      const double* M = d_band.p + off;
      off += band[d].M.size();
      const double* K = d_band.p + off;
      off += band[d].K.size();
      gfull.M[d] = M;
      gfull.K[d] = K;
      gfull.n[d] = band[d].n;
      gfree.M[d] = M;
      gfree.K[d] = K;
      gfree.n[d] = band[d].n;
    }
    gfull.p = gfree.p = p;
    gfree.n[geom.ax] -= 1;
    if (geom.layer == 0) {  // drop row/col 0 of the constrained direction
      gfree.M[geom.ax] += W;
      gfree.K[geom.ax] += W;
    }
    k2_inverse_diagonal(gfree, coefA[0], coefA[1], d_invd.p, d_status.p, s);
    pcg_blocks = k2_pcg_max_blocks(p, ctx->sm_count, gfree.n[2]);
    d_p2.ensure(n_free);
    d_z.ensure(n_free);
    // TMA descriptors of the swept vectors (all persistent allocations)
    maps.valid = k2_make_map(gfree, d_x.p, &maps.x) && k2_make_map(gfree, d_z.p, &maps.z) &&
                 k2_make_map(gfree, d_p.p, &maps.pA) && k2_make_map(gfree, d_p2.p, &maps.pB);
    rhs_tma = k2_make_map(gfull, d_T.p, &map_T) && k2_make_map(gfull, d_gfull.p, &map_g);
    const char* algo = std::getenv("TG_K2_ALGO");
    if (maps.valid && !(algo && std::string(algo) == "pcg")) {
      // buffers: r = {d_r, d_z}, w = {d_Ap, d_w2}, s = {d_p2, d_s2}, p = d_p
      d_w2.ensure(n_free);
      d_s2.ensure(n_free);
      Cg1Maps& m = cg1maps;
      cg1_pl = k2_cg1_planes(gfree, ctx->sm_count);
      if (const char* e = std::getenv("TG_K2_PL")) cg1_pl = std::atoi(e);
      const int L = cg1_pl;
      use_cg1 = k2_make_map(gfree, d_x.p, &m.x, true, L) &&
                k2_make_map(gfree, d_invd.p, &m.inv_diag, true, L) &&
                k2_make_map(gfree, d_r.p, &m.r[0], true, L) &&
                k2_make_map(gfree, d_z.p, &m.r[1], true, L) &&
                k2_make_map(gfree, d_Ap.p, &m.w[0], true, L) &&
                k2_make_map(gfree, d_w2.p, &m.w[1], true, L) &&
                k2_make_map(gfree, d_p2.p, &m.s[0], true, L) &&
                k2_make_map(gfree, d_s2.p, &m.s[1], true, L) &&
                k2_make_map(gfree, d_x.p, &m.xc, false, L) &&
                k2_make_map(gfree, d_p.p, &m.pc, false, L);
      if (use_cg1) pcg_blocks = k2_cg1_max_blocks(p, ctx->sm_count, gfree.n[2], cg1_pl);
    }
    if (preconditioner == 1) {
      // V_d, lambda_d per direction on the free grid (host/fdm.cpp)
      std::vector<double> Vall, Lall;
      size_t offV[3], offL[3];
      for (int d = 0; d < 3; ++d) {
        const int first = (d == geom.ax && geom.layer == 0) ? 1 : 0;
        const Fdm1D f = fdm_factor(band[d].M, band[d].K, band[d].n, p, first, gfree.n[d]);
        offV[d] = Vall.size();
        offL[d] = Lall.size();
        Vall.insert(Vall.end(), f.V.begin(), f.V.end());
        Lall.insert(Lall.end(), f.lam.begin(), f.lam.end());
      }
      upload(d_fdmV, Vall, s);
      upload(d_fdmL, Lall, s);
      d_fdmDinv.ensure(n_free);
      fdm_inverse_eigs(gfree.n, d_fdmL.p + offL[0], d_fdmL.p + offL[1], d_fdmL.p + offL[2],
                       coefA[0], coefA[1], d_fdmDinv.p, s);
      for (int d = 0; d < 3; ++d) {
        fdm.n[d] = gfree.n[d];
        fdm.V[d] = d_fdmV.p + offV[d];
      }
      fdm.dinv = d_fdmDinv.p;
      if (cublasCreate(&cublas) != CUBLAS_STATUS_SUCCESS) throw cuda_error("cublas: create failed");
      d_w2.ensure(n_free);
      d_dots.ensure(2);
      TG_CUDA(cudaMallocHost(&h_dots, 2 * sizeof(double)));
      use_fdm = true;
      use_cg1 = false;
    }
  } else {
    auto up = [&](const Csr& C, SellBufs& b, DevSell& out) {
      const Sell h = to_sell(C);
      upload(b.sp, h.slice_ptr, s);
      upload(b.len, h.row_len, s);
      upload(b.col, h.col, s);
      upload(b.val, h.val, s);
      TG_CUDA(cudaStreamSynchronize(s));  // h dies here
      out = DevSell{C.rows, b.sp.p, b.len.p, b.col.p, b.val.p};
    };
    up(csrA, sA, devA);
    up(csrAc, sAc, devAc);
    up(csrB, sB, devB);
    csrAc = Csr{};  // host copies no longer needed (csrA stays: tg_sim_reduced_operator)
    csrB = Csr{};
    upload(d_free_list, dofs.free_list, s);
    csr_inverse_diagonal(devA, d_invd.p, d_status.p, s);
    pcg_blocks = csr_pcg_max_blocks(ctx->sm_count);
  }
  d_partials.ensure(std::max<size_t>(8 * static_cast<size_t>(pcg_blocks) + 8, 1024));
  TG_CUDA(cudaMemcpyAsync(h_status, d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  diag_ok = h_status->status != 2;
  sf_setup_device();
}

// K5 setup: are the lateral faces' base quadrature points and the Greville
// points tensor grids (up to coordinate rounding) with axis-aligned normals?
void Sim::sf_setup_host() {
  if (const char* e = std::getenv("TG_SF_KC")) sf_kc = std::max(64, std::atoi(e));
  if (const char* e = std::getenv("TG_SF_MIN_PAIRS")) sf_min_pairs = std::atof(e);
  if (const char* e = std::getenv("TG_SF_BANDS")) sf_bands = std::max(1, std::atoi(e));
  const int tqb = h_qb_off.empty() ? 0 : h_qb_off.back();
  // faces: base points grouped by the normal's axis and sign
  double ext = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    double lo = 1e300, hi = -1e300;
    for (int q = 0; q < tqb; ++q) {
      lo = std::min(lo, h_qx[3 * q + ax]);
      hi = std::max(hi, h_qx[3 * q + ax]);
    }
    ext = std::max(ext, hi - lo);
  }
  const double tol = 1e-12 * ext;
  auto& gcell = sf_h_gcell;
  auto& gaxn = sf_h_gaxn;
  gcell.assign(tqb, -1);
  gaxn.assign(tqb, 0);
  sf_flux_ok = tqb > 0;
  auto normal_key = [&](int q) {  // 2 axis + (sign > 0), or -1 off the axes
    const double* n = &h_qn[3 * static_cast<size_t>(q)];
    int ax = 0;
    for (int d = 1; d < 3; ++d)
      if (std::fabs(n[d]) > std::fabs(n[ax])) ax = d;
    const bool axis = std::fabs(std::fabs(n[ax]) - 1.0) <= 1e-12 &&
                      std::fabs(n[(ax + 1) % 3]) <= 1e-12 && std::fabs(n[(ax + 2) % 3]) <= 1e-12;
    return axis ? 2 * ax + (n[ax] > 0.0) : -1;
  };
  std::vector<int> qkey(tqb, -1);
  for (int q = 0; q < tqb && sf_flux_ok; ++q) {
    qkey[q] = normal_key(q);
    if (qkey[q] < 0) sf_flux_ok = false;
  }
  // elements by face (normal key), each face cut into up to sf_bands bands of
  // whole element rows (a band's box is smaller than the face's, so more of the
  // history is cull-free there and takes the GEMM); every band is a grid
  std::vector<int> ekey(n_fe, -1), eband(n_fe, -1);
  std::vector<std::vector<int>> kelems(6);
  for (int e = 0; e < n_fe && sf_flux_ok; ++e) {
    ekey[e] = qkey[h_qb_off[e]];
    for (int q = h_qb_off[e]; q < h_qb_off[e + 1]; ++q)
      if (qkey[q] != ekey[e]) sf_flux_ok = false;
    if (sf_flux_ok) kelems[ekey[e]].push_back(e);
  }
  int off = 0;
  auto grid_of = [&](const std::vector<int>& els, SfGrid& g) {
    std::vector<double> pts;
    for (int e : els)
      for (int q = h_qb_off[e]; q < h_qb_off[e + 1]; ++q)
        for (int d = 0; d < 3; ++d) pts.push_back(h_qx[3 * static_cast<size_t>(q) + d]);
    return sf_make_grid(pts.data(), static_cast<long>(pts.size() / 3), tol, g);
  };
  for (int k = 0; k < 6 && sf_flux_ok; ++k) {
    const std::vector<int>& E = kelems[k];
    if (E.empty()) continue;
    // row starts: where the slower-varying in-face centre coordinate changes
    const int ax = k / 2, u = ax == 0 ? 1 : 0, v = ax == 2 ? 1 : 2;
    auto changes = [&](int d) {
      int c = 0;
      for (size_t i = 1; i < E.size(); ++i)
        c += std::fabs(centers[3 * E[i] + d] - centers[3 * E[i - 1] + d]) > tol;
      return c;
    };
    const int slow = changes(u) <= changes(v) ? u : v;
    std::vector<size_t> rows{0};
    for (size_t i = 1; i < E.size(); ++i)
      if (std::fabs(centers[3 * E[i] + slow] - centers[3 * E[i - 1] + slow]) > tol)
        rows.push_back(i);
    std::vector<std::vector<int>> bands;
    for (int nb = std::max(1, std::min<int>(sf_bands, static_cast<int>(rows.size()))); nb >= 1;
         nb = nb > 1 ? 1 : 0) {
      bands.clear();
      size_t prev = 0;
      for (int b = 1; b <= nb; ++b) {
        const size_t end = b == nb ? E.size() : rows[rows.size() * b / nb];
        if (end > prev) bands.emplace_back(E.begin() + prev, E.begin() + end);
        prev = end;
      }
      std::vector<SfGrid> gs(bands.size());
      bool ok = true;
      for (size_t i = 0; i < bands.size() && ok; ++i)
        ok = grid_of(bands[i], gs[i]) && gs[i].axn == ax;
      if (!ok) {
        if (nb == 1) sf_flux_ok = false;
        continue;
      }
      for (size_t i = 0; i < bands.size(); ++i) {
        const int f = static_cast<int>(sf_faces.size());
        size_t c = 0;
        for (int e : bands[i]) {
          eband[e] = f;
          for (int q = h_qb_off[e]; q < h_qb_off[e + 1]; ++q, ++c) {
            gcell[q] = off + gs[i].cell[c];
            gaxn[q] = gs[i].axn;
          }
        }
        sf_faces_off.push_back(off);
        off += static_cast<int>(gs[i].U.size() * gs[i].V.size());
        sf_faces.push_back(std::move(gs[i]));
      }
      break;
    }
  }
  // fine-rule points: per face, the fine points of all its elements form a
  // finer grid; a step's fine elements take a rectangle of it
  const int tqf = h_qf_off.empty() ? 0 : h_qf_off.back();
  sf_fine_ok = sf_flux_ok && tqf > 0;
  auto& fa = sf_h_fa;
  auto& fb = sf_h_fb;
  auto& ff = sf_h_ff;
  fa.assign(tqf, 0);
  fb.assign(tqf, 0);
  ff.assign(tqf, 0);
  if (sf_fine_ok) {
    sf_elem_face.assign(n_fe, -1);
    sf_erect.assign(4 * static_cast<size_t>(n_fe), 0);
    std::vector<std::vector<int>> felems(sf_faces.size());
    for (int e = 0; e < n_fe && sf_fine_ok; ++e) {
      const int f = eband[e];
      for (int l = h_qf_off[e]; l < h_qf_off[e + 1]; ++l)
        if (normal_key(tqb + l) != ekey[e]) sf_fine_ok = false;
      sf_elem_face[e] = f;
      felems[f].push_back(e);
    }
    for (size_t f = 0; f < felems.size() && sf_fine_ok; ++f) {
      std::vector<double> pts;
      for (int e : felems[f])
        for (int l = h_qf_off[e]; l < h_qf_off[e + 1]; ++l)
          for (int d = 0; d < 3; ++d) pts.push_back(h_qx[3 * static_cast<size_t>(tqb + l) + d]);
      SfGrid g;
      if (!sf_make_grid(pts.data(), static_cast<long>(pts.size() / 3), tol, g) ||
          g.axn != sf_faces[f].axn) {
        sf_fine_ok = false;
        break;
      }
      const int na = static_cast<int>(g.U.size());
      size_t i = 0;
      for (int e : felems[f]) {
        int* r = &sf_erect[4 * static_cast<size_t>(e)];
        r[0] = r[1] = 1 << 30;
        r[2] = r[3] = -1;
        for (int l = h_qf_off[e]; l < h_qf_off[e + 1]; ++l, ++i) {
          const int a = g.cell[i] % na, b = g.cell[i] / na;
          fa[l] = a;
          fb[l] = b;
          ff[l] = static_cast<int>(f);
          r[0] = std::min(r[0], a);
          r[1] = std::min(r[1], b);
          r[2] = std::max(r[2], a);
          r[3] = std::max(r[3], b);
        }
      }
      sf_fine.push_back(std::move(g));
    }
    if (!sf_fine_ok) sf_fine.clear();
  }
  // per-face source prefixes need each face's elements contiguous (one K1
  // launch per face) and its fine points gridded (the GEMM covers them)
  sf_face_split = sf_fine_ok;
  if (sf_face_split) {
    const size_t nfc = sf_faces.size();
    sf_face_e.assign(2 * nfc, -1);
    for (int e = 0; e < n_fe; ++e) {
      const int f = sf_elem_face[e];
      if (sf_face_e[2 * f] < 0) sf_face_e[2 * f] = e;
      else if (sf_face_e[2 * f + 1] != e) sf_face_split = false;
      sf_face_e[2 * f + 1] = e + 1;
    }
    sf_face_box.assign(6 * nfc, 0.0);
    sf_face_delta.assign(nfc, 0.0);
    sf_pf_face.assign(nfc, SfPrefix{});
    for (size_t f = 0; f < nfc; ++f)
      for (int ax = 0; ax < 3; ++ax) {
        sf_face_box[6 * f + ax] = std::min(sf_faces[f].lo[ax], sf_fine[f].lo[ax]);
        sf_face_box[6 * f + 3 + ax] = std::max(sf_faces[f].hi[ax], sf_fine[f].hi[ax]);
        sf_face_delta[f] = std::max(sf_faces[f].delta, sf_fine[f].delta);
      }
  }
  if (sf_flux_ok) {
    for (int ax = 0; ax < 3; ++ax) {
      sf_lo[ax] = 1e300;
      sf_hi[ax] = -1e300;
    }
    for (const SfGrid& g : sf_fine) {  // the eligibility box covers the fine points too
      for (int ax = 0; ax < 3; ++ax) {
        sf_lo[ax] = std::min(sf_lo[ax], g.lo[ax]);
        sf_hi[ax] = std::max(sf_hi[ax], g.hi[ax]);
      }
      sf_delta = std::max(sf_delta, g.delta);
    }
    for (const SfGrid& g : sf_faces) {
      for (int ax = 0; ax < 3; ++ax) {
        sf_lo[ax] = std::min(sf_lo[ax], g.lo[ax]);
        sf_hi[ax] = std::max(sf_hi[ax], g.hi[ax]);
      }
      sf_delta = std::max(sf_delta, g.delta);
    }
  } else {
    sf_faces.clear();
    sf_faces_off.clear();
  }
  sf_dir_ok = n_con > 0 && sf_make_grid(grev.data(), n_con, tol, sf_dir);
  sf_g_total = off;
  if (std::getenv("TG_SF_DEBUG"))
    std::fprintf(stderr, "[k5] flux %d fine %d split %d groups %zu dir %d\n", sf_flux_ok,
                 sf_fine_ok, sf_face_split, sf_faces.size(), sf_dir_ok);
  const char* e = std::getenv("TG_SUMFACT");
  set_sumfact(!(e && std::string(e) == "0"));
}

void Sim::sf_setup_device() {
  cudaStream_t s = ctx->stream;
  const int off = sf_g_total;
  auto& gcell = sf_h_gcell;
  auto& gaxn = sf_h_gaxn;
  // grid lines on the device: faces then the Greville grid
  std::vector<double> uv;
  std::vector<size_t> at;
  auto push = [&](const SfGrid& g) {
    at.push_back(uv.size());
    uv.insert(uv.end(), g.U.begin(), g.U.end());
    uv.insert(uv.end(), g.V.begin(), g.V.end());
  };
  for (const SfGrid& g : sf_faces) push(g);
  for (const SfGrid& g : sf_fine) push(g);
  if (sf_dir_ok) push(sf_dir);
  if (uv.empty()) return;
  upload(d_sf_uv, uv, s);
  auto dev = [&](const SfGrid& g, size_t a) {
    const int na = static_cast<int>(g.U.size()), nb = static_cast<int>(g.V.size());
    return SfDev{g.axn, g.axu, g.axv, na, nb, g.xf, d_sf_uv.p + a, d_sf_uv.p + a + na};
  };
  for (size_t k = 0; k < sf_faces.size(); ++k) sf_faces_dev.push_back(dev(sf_faces[k], at[k]));
  for (size_t k = 0; k < sf_fine.size(); ++k)
    sf_fine_dev.push_back(dev(sf_fine[k], at[sf_faces.size() + k]));
  if (sf_fine_ok) {
    upload(d_sf_fa, sf_h_fa, s);
    upload(d_sf_fb, sf_h_fb, s);
    upload(d_sf_ff, sf_h_ff, s);
    d_sf_rect.ensure(5 * sf_fine.size());
    TG_CUDA(cudaMallocHost(&h_sf_rect, sizeof(int) * 5 * sf_fine.size()));
  }
  if (sf_dir_ok) {
    sf_dir_dev = dev(sf_dir, at.back());
    upload(d_sf_dcell, sf_dir.cell, s);
    d_sf_Gdir.ensure(sf_dir.U.size() * sf_dir.V.size());
  }
  if (sf_flux_ok) {
    upload(d_sf_gcell, gcell, s);
    upload(d_sf_gaxn, gaxn, s);
    d_sf_G.ensure(off);
    const size_t tqf = h_qf_off.back();
    d_sf_fine.ensure(2 * tqf + 2);
    d_sf_tmp.ensure(tqf + 1);
    TG_CUDA(cudaMallocHost(&h_sf_fine, sizeof(int) * (2 * tqf + 2)));
  }
  if (!cublas && cublasCreate(&cublas) != CUBLAS_STATUS_SUCCESS)
    throw cuda_error("cublas: create failed");
  const char* ser = std::getenv("TG_SF_SERIAL");
  if (sf_face_split && !(ser && std::string(ser) == "1")) {
    TG_CUDA(cudaStreamCreateWithFlags(&sf_stream, cudaStreamNonBlocking));
    for (auto& ev : sf_ev) TG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  TG_CUDA(cudaStreamSynchronize(s));
  for (auto* v : {&sf_h_gcell, &sf_h_gaxn, &sf_h_fa, &sf_h_fb, &sf_h_ff}) std::vector<int>().swap(*v);
}

void Sim::sf_prefixes(double t, int* out) {
  if (!sf_on) {
    out[0] = out[1] = 0;
    return;
  }
  out[0] = 0;
  if (sf_flux_ok) {
    SfPrefix c;
    out[0] = sf_prefix(t, sf_lo, sf_hi, sf_delta, c);
    if (sf_face_split) {
      out[0] = 1 << 30;
      for (size_t f = 0; f < sf_faces.size(); ++f) {
        c = SfPrefix{};
        out[0] = std::min(out[0], sf_prefix(t, &sf_face_box[6 * f], &sf_face_box[6 * f + 3],
                                            sf_face_delta[f], c));
      }
    }
  }
  SfPrefix c;
  out[1] = sf_dir_ok ? sf_prefix(t, sf_dir.lo, sf_dir.hi, sf_dir.delta, c) : 0;
}

// longest prefix [0, J) of the sources that sf_source_eligible admits for the
// box at t; a prefix of sources all active at an earlier t stays eligible
// (their spreads only grow), so the scan resumes there
int Sim::sf_prefix(double t, const double lo[3], const double hi[3], double delta, SfPrefix& c) {
  const double alpha = cfg.material.diffusivity();  // = ctx->mat's
  const double cull = cfg.superpose.cull_exponent;
  const double* src = reinterpret_cast<const double*>(sources.data());
  // (the GEMM builders' 2D grids address up to ~1e6 sources; later ones stay on K1)
  const int n = std::min(static_cast<int>(sources.size()), 1000000);
  int j = (c.valid && t >= c.t) ? c.J : 0;
  bool active = true;
  for (; j < n; ++j) {
    const double* p = src + 6 * static_cast<size_t>(j);
    if (!sf_source_eligible(p, t, alpha, cull, lo, hi, delta)) break;
    if (!(t - p[5] > 0.0)) active = false;
  }
  c = SfPrefix{j, t, active};
  return j;
}

int Sim::sf_suffix_end(double t, const double lo[3], const double hi[3], int begin) {
  const double alpha = ctx->mat.diffusivity();
  const double cull = cfg.superpose.cull_exponent;
  const double* src = reinterpret_cast<const double*>(sources.data());
  int end = ctx->active_prefix(t);
  while (end > begin &&
         sf_source_culled(src + 6 * static_cast<size_t>(end - 1), t, alpha, cull, lo, hi))
    --end;
  return end;
}

SfScratch Sim::sf_scratch(int na, int nb, int J) {
  const int C = (J + sf_kc - 1) / sf_kc;
  const size_t Jpad = static_cast<size_t>(C) * sf_kc;
  // sized for every source at once: the prefix only grows during a run
  const size_t Jmax = (sources.size() + sf_kc - 1) / sf_kc * static_cast<size_t>(sf_kc);
  const size_t Jcap = std::max(Jpad, Jmax);
  SfScratch w{};
  w.fac = d_sf_vec.ensure(4 * Jcap);
  w.inv_s = w.fac + Jcap;
  w.su = w.inv_s + Jcap;
  w.sv = w.su + Jcap;
  w.A = d_sf_A.ensure(static_cast<size_t>(na) * Jcap);
  w.B = d_sf_B.ensure(static_cast<size_t>(nb) * Jcap);
  w.Cpart = d_sf_C.ensure(static_cast<size_t>(na) * nb * (Jcap / sf_kc));
  return w;
}

// ---------------------------------------------------------------------------
// hot path pieces

bool Sim::focus_at(double t, Vec3& focus) const {
  // the newest source with t_activate <= t, scanning in order and stopping at
  // the first later one (assembly.cpp:153-157): first j with max(t_act[0..j]) > t
  const size_t k = std::upper_bound(tact_max.begin(), tact_max.end(), t) - tact_max.begin();
  if (k == 0) return false;
  focus = sources[k - 1].position;
  return true;
}

int Sim::fine_elements(double t, double radius) {
  Vec3 f;
  int nf = 0;
  if (!focus_at(t, f)) return 0;
  for (int e = 0; e < n_fe; ++e) {
    const Vec3 c{centers[3 * e], centers[3 * e + 1], centers[3 * e + 2]};
    if ((c - f).norm() < radius) h_fine[nf++] = e;
  }
  return nf;
}

void Sim::flux_load_device(double t, double radius, double* d_F, int e0, int e1) {
  cudaStream_t s = ctx->stream;
  // the pinned fine list is reused every step: order the last copy first
  TG_CUDA(cudaStreamSynchronize(s));
  const int nf = fine_elements(t, radius);
  // extra[r]: added points of the first r fine elements (fine minus base rule)
  int* extra = h_fine + n_fe + 1;
  extra[0] = 0;
  for (int r = 0; r < nf; ++r) {
    const int e = h_fine[r];
    extra[r + 1] = extra[r] + (h_qf_off[e + 1] - h_qf_off[e]) - (h_qb_off[e + 1] - h_qb_off[e]);
  }
  if (nf > 0) TG_CUDA(cudaMemcpyAsync(d_fine.p, h_fine, sizeof(int) * nf, cudaMemcpyHostToDevice, s));
  TG_CUDA(cudaMemcpyAsync(d_fine.p + n_fe + 1, extra, sizeof(int) * (nf + 1),
                          cudaMemcpyHostToDevice, s));
  // compact-list offset of element e: its base offset plus the extra points
  // of the fine elements before it
  auto offset_of = [&](int e) {
    const int r = static_cast<int>(std::lower_bound(h_fine, h_fine + nf, e) - h_fine);
    return static_cast<long>(h_qb_off[e]) + extra[r];
  };
  e0 = std::max(0, std::min(e0, n_fe));
  e1 = std::max(e0, std::min(e1, n_fe));
  const long p0 = offset_of(e0), p1 = e1 == n_fe ? h_qb_off.back() + extra[nf] : offset_of(e1);
  const FaceTables ft{n_fe, ndk, d_qb_off.p, d_qf_off.p, d_Nb.p, d_Nf.p};
  k3_point_index(ft, d_fine.p, d_fine.p + n_fe + 1, nf, d_pt_index.p, d_elem_off.p, s);
  ++ctx->timer.launches;
  K1Flux fl{d_pt_index.p + p0, d_qn.p, d_qw.p, cfg.material.conductivity};
  // K5 split (full-range calls): sources [0, J) by DGEMM on the face grids
  // (plus K1 on the fine-rule points, which are not on the grids), [J, n) by K1
  const bool full = e0 == 0 && e1 == n_fe;
  // per face the longest eligible prefix for that face's box (faces whose
  // elements are contiguous and gridded with their fine points), else one
  // prefix for the box of all faces
  const size_t nfc = sf_faces.size();
  std::vector<int> Jf(nfc, 0);
  int J = 0, Jmax = 0;
  if (sf_on && sf_flux_ok && full) {
    if (sf_face_split) {
      J = 1 << 30;
      for (size_t f = 0; f < nfc; ++f) {
        Jf[f] = sf_prefix(t, &sf_face_box[6 * f], &sf_face_box[6 * f + 3], sf_face_delta[f],
                          sf_pf_face[f]);
        J = std::min(J, Jf[f]);
        Jmax = std::max(Jmax, Jf[f]);
      }
    } else {
      J = Jmax = sf_prefix(t, sf_lo, sf_hi, sf_delta, sf_pf_flux);
      std::fill(Jf.begin(), Jf.end(), J);
    }
  }
  // profitability: a face's GEMM (a few launches, ~25 us) must save more K1
  // pair work than it costs (TG_SF_MIN_PAIRS moved pairs, default 3e7 ~ 30 us)
  if (Jmax > 0 && sf_face_split) {
    J = 1 << 30;
    Jmax = 0;
    for (size_t f = 0; f < nfc; ++f) {
      const double pts = static_cast<double>(sf_faces[f].U.size()) * sf_faces[f].V.size();
      if (static_cast<double>(Jf[f]) * pts < sf_min_pairs) Jf[f] = 0;
      J = std::min(J, Jf[f]);
      Jmax = std::max(Jmax, Jf[f]);
    }
  } else if (Jmax > 0) {  // one prefix for all faces: all kept or all dropped
    double pts = 0.0;
    for (const SfGrid& g : sf_faces) pts += static_cast<double>(g.U.size()) * g.V.size();
    if (static_cast<double>(J) * pts < sf_min_pairs) {
      J = Jmax = 0;
      std::fill(Jf.begin(), Jf.end(), 0);
    }
  }
  sf_last_j[0] = J;
  // the K1 remainder (FP64 pipe) runs on a side stream beside the GEMMs (DMMA)
  const bool conc = Jmax > 0 && sf_face_split && sf_stream != nullptr;
  cudaStream_t ks = conc ? sf_stream : s;
  if (conc) {
    TG_CUDA(cudaEventRecord(sf_ev[0], s));
    TG_CUDA(cudaStreamWaitEvent(sf_stream, sf_ev[0], 0));
  }
  if (Jmax > 0 && sf_face_split) {
    auto pos_of = [&](int e) { return e == n_fe ? p1 : offset_of(e); };
    for (size_t f = 0; f < nfc; ++f) {
      const long a = pos_of(sf_face_e[2 * f]), b = pos_of(sf_face_e[2 * f + 1]);
      K1Flux ff{d_pt_index.p + a, d_qn.p, d_qw.p, cfg.material.conductivity};
      const int end = sf_suffix_end(t, &sf_face_box[6 * f], &sf_face_box[6 * f + 3], Jf[f]);
      k1_run(ctx, ctx->src6.p, ctx->n_src, d_qx.p, d_pt_index.p + a, b - a, t,
             cfg.superpose.cull_exponent, K1Mode::flux, d_gq.p + a, nullptr, ff, ks, Jf[f], end);
    }
    if (conc) TG_CUDA(cudaEventRecord(sf_ev[1], sf_stream));
  } else {
    k1_run(ctx, ctx->src6.p, ctx->n_src, d_qx.p, d_pt_index.p + p0, p1 - p0, t,
           cfg.superpose.cull_exponent, K1Mode::flux, d_gq.p + p0, nullptr, fl, s, J);
  }
  int fine_n = 0;
  double* fine_G = nullptr;
  if (Jmax > 0) {
    const double alpha = ctx->mat.diffusivity(), rcp = ctx->mat.volumetric_capacity();
    const int tqb = h_qb_off.back();
    if (nf > 0 && sf_fine_ok) {
      // the step's fine elements: per face the bounding rectangle of their
      // cells in the face's fine grid, one GEMM each
      const size_t nF = sf_fine.size();
      std::vector<int> rc(4 * nF);
      for (size_t f = 0; f < nF; ++f) {
        rc[4 * f] = rc[4 * f + 1] = 1 << 30;
        rc[4 * f + 2] = rc[4 * f + 3] = -1;
      }
      int nfp = 0;
      for (int r = 0; r < nf; ++r) {
        const int e = h_fine[r], f = sf_elem_face[e];
        const int* er = &sf_erect[4 * static_cast<size_t>(e)];
        rc[4 * f] = std::min(rc[4 * f], er[0]);
        rc[4 * f + 1] = std::min(rc[4 * f + 1], er[1]);
        rc[4 * f + 2] = std::max(rc[4 * f + 2], er[2]);
        rc[4 * f + 3] = std::max(rc[4 * f + 3], er[3]);
        nfp += h_qf_off[e + 1] - h_qf_off[e];
      }
      size_t gtot = 0;
      for (size_t f = 0; f < nF; ++f) {
        int* hr = h_sf_rect + 5 * f;
        const bool any = rc[4 * f + 2] >= 0;
        hr[0] = rc[4 * f];
        hr[1] = rc[4 * f + 1];
        hr[2] = any ? rc[4 * f + 2] - rc[4 * f] + 1 : 0;
        hr[3] = static_cast<int>(gtot);
        hr[4] = sf_fine[f].axn;
        if (any) gtot += static_cast<size_t>(hr[2]) * (rc[4 * f + 3] - rc[4 * f + 1] + 1);
      }
      double* Gf = d_sf_Gf.ensure(gtot);
      for (size_t f = 0; f < nF; ++f) {
        const int* hr = h_sf_rect + 5 * f;
        if (hr[2] == 0) continue;
        SfDev g = sf_fine_dev[f];
        g.U += hr[0];
        g.V += hr[1];
        g.na = hr[2];
        g.nb = rc[4 * f + 3] - rc[4 * f + 1] + 1;
        sf_flops += sf_contract(cublas, g, true, ctx->src6.p, Jf[f], sf_kc, t, alpha, rcp,
                                sf_scratch(g.na, g.nb, Jf[f]), Gf + hr[3], s);
        sf_pairs += static_cast<double>(g.na) * g.nb * Jf[f];
        ctx->timer.launches += 5;
      }
      int* pos = h_sf_fine;
      int* ids = h_sf_fine + nfp;
      int m = 0;
      for (int r = 0; r < nf; ++r) {
        const int e = h_fine[r];
        const int o = h_qb_off[e] + extra[r], nq = h_qf_off[e + 1] - h_qf_off[e];
        for (int l = 0; l < nq; ++l, ++m) {
          pos[m] = o + l;
          ids[m] = h_qf_off[e] + l;
        }
      }
      TG_CUDA(cudaMemcpyAsync(d_sf_fine.p, h_sf_fine, sizeof(int) * 2 * nfp,
                              cudaMemcpyHostToDevice, s));
      TG_CUDA(cudaMemcpyAsync(d_sf_rect.p, h_sf_rect, sizeof(int) * 5 * nF,
                              cudaMemcpyHostToDevice, s));
      fine_n = nfp;  // added after the join with the K1 stream
      fine_G = Gf;
    } else if (nf > 0) {
      int nfp = 0;
      for (int r = 0; r < nf; ++r) nfp += h_qf_off[h_fine[r] + 1] - h_qf_off[h_fine[r]];
      int* pos = h_sf_fine;
      int* ids = h_sf_fine + nfp;
      int m = 0;
      for (int r = 0; r < nf; ++r) {
        const int e = h_fine[r];
        const int o = h_qb_off[e] + extra[r], nq = h_qf_off[e + 1] - h_qf_off[e];
        for (int l = 0; l < nq; ++l, ++m) {
          pos[m] = o + l;
          ids[m] = tqb + h_qf_off[e] + l;
        }
      }
      TG_CUDA(cudaMemcpyAsync(d_sf_fine.p, h_sf_fine, sizeof(int) * 2 * nfp,
                              cudaMemcpyHostToDevice, s));
      K1Flux ff{d_sf_fine.p + nfp, d_qn.p, d_qw.p, cfg.material.conductivity};
      k1_run(ctx, ctx->src6.p, ctx->n_src, d_qx.p, d_sf_fine.p + nfp, nfp, t,
             cfg.superpose.cull_exponent, K1Mode::flux, d_sf_tmp.p, nullptr, ff, s, 0, J);
      sf_scatter_add(nfp, d_sf_fine.p, d_sf_tmp.p, d_gq.p, s);
      ctx->timer.launches += 1;
    }
    for (size_t k = 0; k < sf_faces_dev.size(); ++k) {
      const SfDev& g = sf_faces_dev[k];
      sf_flops += sf_contract(cublas, g, true, ctx->src6.p, Jf[k], sf_kc, t, alpha, rcp,
                              sf_scratch(g.na, g.nb, Jf[k]), d_sf_G.p + sf_faces_off[k], s);
      sf_pairs += static_cast<double>(g.na) * g.nb * Jf[k];
      ctx->timer.launches += 5;
    }
    if (conc) TG_CUDA(cudaStreamWaitEvent(s, sf_ev[1], 0));  // K1 wrote gq
    if (fine_n > 0) {
      sf_add_fine(fine_n, d_sf_fine.p, d_sf_fine.p + fine_n, tqb, d_sf_fa.p, d_sf_fb.p,
                  d_sf_ff.p, d_sf_rect.p, fine_G, d_qn.p, d_qw.p, cfg.material.conductivity,
                  d_gq.p, s);
      ++ctx->timer.launches;
    }
    sf_add_flux(static_cast<int>(p1 - p0), d_pt_index.p, tqb, d_sf_gcell.p, d_sf_gaxn.p,
                d_sf_G.p, d_qn.p, d_qw.p, cfg.material.conductivity, d_gq.p, s);
    ++ctx->timer.launches;
  }
  k3_local(ft, e0, e1, d_elem_off.p, d_gq.p, d_loc.p, s);
  ++ctx->timer.launches;
  if (d_F) {
    k3_gather(n_full, d_inc_ptr.p, d_inc_src.p, d_loc.p, d_F, s);
    ++ctx->timer.launches;
  }
  TG_CUDA(cudaGetLastError());
}

void Sim::flux_gather_device(const double* d_loc_all, double* d_F) {
  k3_gather(n_full, d_inc_ptr.p, d_inc_src.p, d_loc_all, d_F, ctx->stream);
  ++ctx->timer.launches;
  TG_CUDA(cudaGetLastError());
}

void Sim::dirichlet_device(double t, double* d_g, int c0, int c1) {
  // constrained DOFs [c0, c1) (all by default): each value depends on its
  // Greville point only, so a range is the same bits as the full call
  if (c1 < 0) c1 = n_con;
  c0 = std::max(0, std::min(c0, n_con));
  c1 = std::max(c0, std::min(c1, n_con));
  int J = (sf_on && sf_dir_ok && c0 == 0 && c1 == n_con)
              ? sf_prefix(t, sf_dir.lo, sf_dir.hi, sf_dir.delta, sf_pf_dir)
              : 0;
  if (static_cast<double>(J) * n_con < sf_min_pairs) J = 0;  // not worth the launches
  sf_last_j[1] = J;
  const int end = J > 0 ? sf_suffix_end(t, sf_dir.lo, sf_dir.hi, J) : -1;
  k1_run(ctx, ctx->src6.p, ctx->n_src, d_grev.p + 3 * static_cast<size_t>(c0), nullptr, c1 - c0,
         t, cfg.superpose.cull_exponent, K1Mode::dirichlet, d_g, nullptr, {}, ctx->stream, J,
         end);
  if (J > 0) {  // g = -(K1 part) - (GEMM part)
    const SfDev& g = sf_dir_dev;
    sf_flops += sf_contract(cublas, g, false, ctx->src6.p, J, sf_kc, t, ctx->mat.diffusivity(),
                            ctx->mat.volumetric_capacity(), sf_scratch(g.na, g.nb, J),
                            d_sf_Gdir.p, ctx->stream);
    sf_add_dirichlet(n_con, d_sf_dcell.p, d_sf_Gdir.p, d_g, ctx->stream);
    ctx->timer.launches += 6;
    sf_pairs += static_cast<double>(n_con) * J;
  }
}

PcgStatus Sim::theta_step_device(double tol, int max_iter) {
  cudaStream_t s = ctx->stream;
  if (!diag_ok) throw numeric_error("pcg: non-positive diagonal, matrix not SPD");
  ctx->timer.timed(3, s, [&] { theta_step_launch(tol, max_iter); });
  TG_CUDA(cudaMemcpyAsync(h_status, d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  const PcgStatus st = *h_status;
  ctx->timer.k2_bytes += 104.0 * n_free * st.iterations;  // SURVEY.md §8d algorithmic bytes
  k2_iterations += st.iterations;
  if (st.status == 4) throw numeric_error("pcg: indefinite direction, matrix not SPD");
  if (st.status == 3) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", st.rel_residual);
    throw numeric_error("pcg: no convergence in " + std::to_string(max_iter) +
                        " iterations, relative residual " + buf);
  }
  return st;
}

// expand, RHS and the solve on the stream (theta_step, timestep.cpp:5-24)
void Sim::theta_step_launch(double tol, int max_iter) {
  cudaStream_t s = ctx->stream;
  const int threads = 256;
  expand_kernel<<<static_cast<int>((n_full + threads - 1) / threads), threads, 0, s>>>(
      geom, d_x.p, d_gn.p, d_T.p);
  ++ctx->timer.launches;
  const double th = cfg.stepping.theta;
  if (kron) {
    scatter_layer_kernel<<<(n_con + threads - 1) / threads, threads, 0, s>>>(geom, d_g1.p,
                                                                             d_gfull.p);
    RhsArgs ra{d_T.p, d_gfull.p, d_Fn.p, d_F1.p, th, geom.ax, geom.layer, d_rhs.p};
    k2_theta_rhs(gfull, coefB[0], coefB[1], -coefA[0], -coefA[1], ra, rhs_tma ? &map_T : nullptr,
                 rhs_tma ? &map_g : nullptr, ctx->sm_count, s);
    ctx->timer.launches += 2;
    if (use_fdm) {
      const FdmWork w{d_r.p, d_z.p, d_p.p, d_Ap.p, d_p2.p, d_w2.p, d_partials.p, d_dots.p, h_dots};
      ctx->timer.timed(2, s, [&] {
        *h_status = fdm_pcg_solve(cublas, gfree, coefA[0], coefA[1], fdm, d_rhs.p, d_x.p, w, tol,
                                  max_iter, ctx->sm_count, s, maps.valid ? &maps.x : nullptr,
                                  maps.valid ? &maps.pA : nullptr);
      });
      TG_CUDA(cudaMemcpyAsync(d_status.p, h_status, sizeof(PcgStatus), cudaMemcpyHostToDevice, s));
    } else if (use_cg1) {
      const Cg1Work w{d_p.p,    {d_r.p, d_z.p}, {d_Ap.p, d_w2.p}, {d_p2.p, d_s2.p},
                      d_invd.p, d_partials.p,   d_status.p};
      ctx->timer.timed(2, s, [&] {
        k2_cg1_solve(gfree, coefA[0], coefA[1], d_rhs.p, d_x.p, w, cg1maps, tol, max_iter,
                     pcg_blocks, s, cg1_pl);
      });
    } else {
      const PcgWork w{d_r.p,        d_z.p,      d_p.p,
                      d_p2.p,       d_Ap.p,     d_invd.p,
                      d_partials.p, d_status.p, trace_on ? d_trace.p : nullptr};
      ctx->timer.timed(2, s, [&] {
        k2_pcg_solve(gfree, coefA[0], coefA[1], d_rhs.p, d_x.p, w, maps, tol, max_iter,
                     pcg_blocks, s);
      });
    }
  } else {
    csr_theta_rhs(devB, devAc, d_T.p, d_g1.p, d_Fn.p, d_F1.p, d_free_list.p, th, d_rhs.p, s);
    ++ctx->timer.launches;
    const CsrWork w{d_r.p, d_p.p, d_Ap.p, d_invd.p, d_partials.p, d_status.p};
    ctx->timer.timed(2, s, [&] {
      csr_pcg_solve(devA, d_rhs.p, d_x.p, w, tol, max_iter, pcg_blocks, s);
    });
  }
  ++ctx->timer.launches;
  ++ctx->timer.k2_launches;
}

void Sim::reset() {
  cudaStream_t s = ctx->stream;
  TG_CUDA(cudaMemsetAsync(d_x.p, 0, sizeof(double) * n_free, s));
  dirichlet_device(0.0, d_gn.p);
  flux_load_device(0.0, cfg.mesh.elevate_radius, d_Fn.p);
  step = 0;
  TG_CUDA(cudaStreamSynchronize(s));
}

PcgStatus Sim::advance() {
  const int s1 = step + 1;
  const double t1 = s1 * dt_solver;  // driver.cpp:127
  static const bool timing = std::getenv("TG_STEP_TIMING") != nullptr;
  auto now = [&] {
    if (timing) TG_CUDA(cudaStreamSynchronize(ctx->stream));
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  flux_load_device(t1, cfg.mesh.elevate_radius, d_F1.p);
  const auto ta = now();
  dirichlet_device(t1, d_g1.p);
  const auto tb = now();
  const PcgStatus st = theta_step_device(cfg.stepping.solver_tol, cfg.stepping.max_iter);
  if (timing) {
    const auto tc = now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[step %d] flux %.3f ms, dirichlet %.3f ms, theta %.3f ms\n", s1,
                 ms(t0, ta), ms(ta, tb), ms(tb, tc));
  }
  std::swap(d_Fn.p, d_F1.p);
  std::swap(d_gn.p, d_g1.p);
  step = s1;
  return st;
}

PcgStatus Sim::advance_with_loads(const double* d_F1_in, const double* d_g1_in) {
  cudaStream_t s = ctx->stream;
  TG_CUDA(cudaMemcpyAsync(d_F1.p, d_F1_in, sizeof(double) * n_full, cudaMemcpyDeviceToDevice, s));
  TG_CUDA(cudaMemcpyAsync(d_g1.p, d_g1_in, sizeof(double) * n_con, cudaMemcpyDeviceToDevice, s));
  const PcgStatus st = theta_step_device(cfg.stepping.solver_tol, cfg.stepping.max_iter);
  std::swap(d_Fn.p, d_F1.p);
  std::swap(d_gn.p, d_g1.p);
  step += 1;
  return st;
}

// ---------------------------------------------------------------------------
// observers: K4 NURBS evaluation + K1 on the device

void Sim::upload_nurbs() {
  if (nurbs_up) return;
  cudaStream_t s = ctx->stream;
  std::vector<double> kn;
  size_t off[3];
  for (int d = 0; d < 3; ++d) {
    off[d] = kn.size();
    const auto& U = vol.knots(d).values();
    kn.insert(kn.end(), U.begin(), U.end());
  }
  upload(d_knots, kn, s);
  const ControlGrid& g = vol.grid();
  std::vector<double> cp(4 * static_cast<size_t>(g.count()));
  for (int i = 0; i < g.count(); ++i)
    for (int c = 0; c < 4; ++c) cp[4 * static_cast<size_t>(i) + c] = g.pts[i][c];
  upload(d_cpts, cp, s);
  const auto n = vol.basis_counts();
  for (int d = 0; d < 3; ++d) {
    nurbs.p[d] = vol.knots(d).degree();
    nurbs.n[d] = n[d];
    nurbs.U[d] = d_knots.p + off[d];
  }
  nurbs.pts = d_cpts.p;
  d_eflags.ensure(1);
  TG_CUDA(cudaStreamSynchronize(s));
  nurbs_up = true;
}

void Sim::field_eval_device(const double* d_coeffs, const double* d_xi, long n, double* d_xo,
                            double* d_f, cudaStream_t s) {
  if (n <= 0) return;
  upload_nurbs();
  TG_CUDA(cudaMemsetAsync(d_eflags.p, 0, sizeof(int), s));
  k4_eval(nurbs, d_xi, n, d_coeffs, d_xo, d_f, d_eflags.p, s);
  ++ctx->timer.launches;
  int flags = 0;
  TG_CUDA(cudaMemcpyAsync(&flags, d_eflags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (flags & kEvalOutside)  // postproc.cpp:12-14
    throw std::domain_error("probe parametric coordinates outside the patch");
  if (flags & kEvalDomain) throw std::domain_error("parameter outside knot range");
  if (flags & kEvalJacobian)
    throw numeric_error("non-positive Jacobian determinant in field evaluation");
}

void Sim::probe_device(const double* d_xi, long n, double* d_out, cudaStream_t s) {
  if (n <= 0) return;
  upload_nurbs();
  // full coefficients of the current state (DirichletSystem::expand,
  // assembly.cpp:274-281); d_T is rebuilt by every theta step
  const int threads = 256;
  expand_kernel<<<static_cast<int>((n_full + threads - 1) / threads), threads, 0, s>>>(
      geom, d_x.p, d_gn.p, d_T.p);
  ++ctx->timer.launches;
  double* xo = d_px.ensure(3 * static_cast<size_t>(n));
  double* fo = d_pf.ensure(4 * static_cast<size_t>(n));
  TG_CUDA(cudaMemsetAsync(d_eflags.p, 0, sizeof(int), s));
  k4_eval(nurbs, d_xi, n, d_T.p, xo, fo, d_eflags.p, s, true);
  ++ctx->timer.launches;
  int flags = 0;
  TG_CUDA(cudaMemcpyAsync(&flags, d_eflags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (flags & kEvalOutside)
    throw std::domain_error("probe parametric coordinates outside the patch");
  if (flags & kEvalDomain) throw std::domain_error("parameter outside knot range");
  if (flags & kEvalJacobian)
    throw numeric_error("non-positive Jacobian determinant in field evaluation");
  const double t = step * dt_solver;  // State::time (timestep.cpp:22)
  double* val = d_pval.ensure(n);
  double* grad = d_pgrad.ensure(3 * static_cast<size_t>(n));
  k1_run(ctx, ctx->src6.p, ctx->n_src, xo, nullptr, n, t, cfg.superpose.cull_exponent,
         K1Mode::field, val, grad, {}, s);
  k4_assemble_probe(n, cfg.material.platform_temperature, xo, fo, val, grad, d_out, s);
  ++ctx->timer.launches;
}

void Sim::flux_profile(FaceId face, int ns, double edge_v, const double* theta_axis,
                       double* out) {
  if (ns < 2) throw std::invalid_argument("flux profile needs >= 2 samples");
  const double k = cfg.material.conductivity;
  const auto tang = face_tangent_axes(face);
  // arc length along the edge: 4-point Gauss per interval, split at the
  // tangent direction's breakpoints (postproc.cpp:33-52)
  const GaussRule& quadr = gauss_rule(4);
  const auto breaks = vol.knots(tang[0]).breakpoints();
  auto segment_length = [&](double a, double b) {
    std::vector<double> cuts{a};
    for (double bp : breaks)
      if (bp > a && bp < b) cuts.push_back(bp);
    cuts.push_back(b);
    double len = 0.0;
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
      const double h = 0.5 * (cuts[c + 1] - cuts[c]), m = 0.5 * (cuts[c + 1] + cuts[c]);
      for (size_t q = 0; q < quadr.nodes.size(); ++q) {
        const auto pm = vol.map_point(face_param(face, m + h * quadr.nodes[q], edge_v));
        const Vec3 du{pm.jac(0, tang[0]), pm.jac(1, tang[0]), pm.jac(2, tang[0])};
        len += quadr.weights[q] * h * du.norm();
      }
    }
    return len;
  };
  std::vector<double> xi(3 * static_cast<size_t>(ns)), arc(ns);
  std::vector<Vec3> xs(ns), nrm(ns);
  double sacc = 0.0, u_prev = 0.0;
  for (int i = 0; i < ns; ++i) {
    const double u = static_cast<double>(i) / (ns - 1);
    if (i > 0) sacc += segment_length(u_prev, u);
    u_prev = u;
    const auto sp = vol.face_point(face, u, edge_v);
    for (int d = 0; d < 3; ++d) xi[3 * i + d] = sp.xi[d];
    xs[i] = sp.x;
    nrm[i] = sp.normal;
    arc[i] = sacc;
  }
  cudaStream_t s = ctx->stream;
  DevBuf<double> d_xi, d_o;
  upload(d_xi, xi, s);
  d_o.ensure(12 * static_cast<size_t>(ns));
  probe_device(d_xi.p, ns, d_o.p, s);
  std::vector<double> o(12 * static_cast<size_t>(ns));
  TG_CUDA(cudaMemcpyAsync(o.data(), d_o.p, sizeof(double) * o.size(), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < ns; ++i) {
    const double* r = &o[12 * static_cast<size_t>(i)];
    const Vec3 gt{r[6], r[7], r[8]}, gh{r[9], r[10], r[11]};
    double* row = out + 5 * static_cast<size_t>(i);
    row[0] = arc[i];
    row[1] = theta_axis ? std::atan2(-(xs[i].x - theta_axis[0]), xs[i].y - theta_axis[1])
                        : std::numeric_limits<double>::quiet_NaN();
    row[2] = -k * gt.dot(nrm[i]);
    row[3] = -k * gh.dot(nrm[i]);
    row[4] = row[2] + row[3];
  }
}

}  // namespace tgb
