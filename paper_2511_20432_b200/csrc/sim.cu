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
#include <functional>
#include <limits>
#include <numeric>
#include <tuple>

#include "context.hpp"
#include "host/config.hpp"
#include "host/fdm.hpp"
#include "host/parallel.hpp"
#include "host/operator.hpp"
#include "k2_csr.cuh"
#include "k2_kron.cuh"
#include "common.cuh"
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

Sim::Sim(const std::string& path, const SimOptions& opt) {
  RunConfig c = parse_config(path);
  if (opt.t_end > 0.0) c.stepping.t_end = opt.t_end;
  if (opt.solver_tol > 0.0) c.stepping.solver_tol = opt.solver_tol;
  if (opt.max_iter > 0) c.stepping.max_iter = opt.max_iter;
  cfg = std::move(c);
  // the general patch's operators: assembled on the device when there is one
  csr_deferred = !opt.host_only && !std::getenv("TG_HOST_ASSEMBLY");
  faces_deferred = !opt.host_only && !std::getenv("TG_HOST_FACES");
  setup_host();
  PhaseClock clk;
  if (!faces_deferred) {
    sf_setup_host();
    clk.mark("k5 grids, tiles, entries");
  }
  if (!opt.host_only) setup_device(opt.device, opt.preconditioner);
  clk.mark("device setup");
}

Sim::~Sim() {
  if (h_dots) cudaFreeHost(h_dots);
  if (h_status) cudaFreeHost(h_status);
  if (h_steps) cudaFreeHost(h_steps);
  release_stages();
  if (ctx) tg_ctx_destroy(ctx);
}


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
  FaceSets fs;
  if (faces_deferred)  // the per-point tables come from the device (face_tables_device)
    face_specs = face_elements(vol, cfg.tags, cfg.mesh.boundary_quad_multiplier, fs);
  else
    fs = build_face_sets(vol, cfg.tags, cfg.mesh.boundary_quad_multiplier);
  clk.mark(faces_deferred ? "face layout" : "face sets");
  n_fe = fs.n_elems;
  const long tqb = fs.qb_off.back(), tqf = fs.qf_off.back();
  if (tqb + tqf > (1L << 31) - 1) throw std::invalid_argument("face quadrature set too large");
  h_qb_off.assign(fs.qb_off.begin(), fs.qb_off.end());
  h_qf_off.assign(fs.qf_off.begin(), fs.qf_off.end());
  nqb = nqf = 0;
  for (int e = 0; e < n_fe; ++e) {
    nqb = std::max(nqb, fs.nqb[e]);
    nqf = std::max(nqf, fs.nqf[e]);
  }
  if (!faces_deferred) face_tables_host(fs);
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
  } else if (!csr_deferred) {
    assemble_csr_host();
  }
}

// The face tables from host face sets: the columns exactly zero at every
// point of an element dropped (their scatter adds +0, a no-op), positions,
// normals, weights, the kept N columns and their DOFs, incidence lists.
void Sim::face_tables_host(const FaceSets& fs) {
  const int nd = fs.n_dofs;
  const long tqb = fs.qb_off.back(), tqf = fs.qf_off.back();
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
  build_incidence();
}

// The face tables built on the device (K6 face sets, bit-identical to
// build_face_sets): points, normals, weights and the kept N columns stay there;
// positions, normals, weights, centres and the kept DOFs come back for the
// host-side setup (K5 grids, the step's fine-element test, incidence lists).
void Sim::face_tables_device(cudaStream_t s) {
  upload_nurbs();
  const auto pd = vol.degrees();
  const int nd = (pd[0] + 1) * (pd[1] + 1) * (pd[2] + 1);
  const int tqb = h_qb_off.back(), tqf = h_qf_off.back();
  const int fm = std::max(1, cfg.mesh.boundary_quad_multiplier);
  std::vector<FaceElemDev> el(n_fe);
  int nmax = 1;
  for (int e = 0; e < n_fe; ++e) {
    const FaceElemSpec& f = face_specs[e];
    el[e] = FaceElemDev{static_cast<int>(f.f), f.qu, f.qv, f.mu, f.hu, f.mv, f.hv};
    nmax = std::max(nmax, fm * std::max(f.qu, f.qv));
  }
  std::vector<double> gn, gw;  // Gauss rules 1..nmax at offset n (n - 1) / 2
  for (int n = 1; n <= nmax; ++n) {
    const GaussRule& g = gauss_rule(n);
    gn.insert(gn.end(), g.nodes.begin(), g.nodes.end());
    gw.insert(gw.end(), g.weights.begin(), g.weights.end());
  }
  DevBuf<FaceElemDev> d_el;
  DevBuf<double> d_gn, d_gw, Nb, Nf, cen;
  DevBuf<int> dofs_all, keep, nkeep, dofk, flag;
  upload(d_el, el, s);
  upload(d_gn, gn, s);
  upload(d_gw, gw, s);
  upload(d_qb_off, h_qb_off, s);
  upload(d_qf_off, h_qf_off, s);
  const size_t npts = static_cast<size_t>(tqb) + tqf;
  d_qx.ensure(3 * (npts + n_con));  // room for the Greville points (sf_setup_device)
  d_qn.ensure(3 * npts);
  d_qw.ensure(npts);
  Nb.ensure(static_cast<size_t>(tqb) * nd);
  Nf.ensure(static_cast<size_t>(tqf) * nd);
  dofs_all.ensure(static_cast<size_t>(n_fe) * nd);
  cen.ensure(3 * static_cast<size_t>(n_fe));
  flag.ensure(1);
  TG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
  FaceSetDev F{nurbs, d_el.p, n_fe, fm, nd, d_qb_off.p, d_qf_off.p, tqb, tqf, d_gn.p, d_gw.p,
               d_qx.p, d_qn.p, d_qw.p, Nb.p, Nf.p, dofs_all.p, cen.p, flag.p};
  k6_face_sets(F, s);
  keep.ensure(static_cast<size_t>(n_fe) * nd);
  nkeep.ensure(n_fe);
  k6_face_keep(F, keep.p, nkeep.p, s);
  int fl = 0;
  std::vector<int> nk(n_fe);
  TG_CUDA(cudaMemcpyAsync(&fl, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (n_fe > 0)
    TG_CUDA(cudaMemcpyAsync(nk.data(), nkeep.p, sizeof(int) * n_fe, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (fl & 4) throw std::domain_error("find_span: parameter outside the knot range");
  if (fl & 1) throw numeric_error("non-positive Jacobian determinant in geometry map");
  if (fl & 2) throw numeric_error("degenerate surface point");
  ndk = 1;
  for (int e = 0; e < n_fe; ++e) ndk = std::max(ndk, nk[e]);
  d_Nb.ensure(static_cast<size_t>(tqb) * ndk);
  d_Nf.ensure(static_cast<size_t>(tqf) * ndk);
  dofk.ensure(static_cast<size_t>(n_fe) * ndk);
  k6_face_compact(F, keep.p, nkeep.p, ndk, d_Nb.p, d_Nf.p, dofk.p, s);
  h_qx.resize(3 * npts);
  h_qn.resize(3 * npts);
  h_qw.resize(npts);
  centers.resize(3 * static_cast<size_t>(n_fe));
  h_dofk.resize(static_cast<size_t>(n_fe) * ndk);
  auto down = [&](auto& v, const auto* src) {
    if (!v.empty())
      TG_CUDA(cudaMemcpyAsync(v.data(), src, v.size() * sizeof(v[0]), cudaMemcpyDeviceToHost, s));
  };
  down(h_qx, d_qx.p);
  down(h_qn, d_qn.p);
  down(h_qw, d_qw.p);
  down(centers, cen.p);
  down(h_dofk, dofk.p);
  TG_CUDA(cudaStreamSynchronize(s));  // the temporaries die here
  h_Nb.clear();  // on demand (face_tables_to_host)
  h_Nf.clear();
  build_incidence();
}

// the kept N tables on the host (tg_sim_face_sets) when they were built on the device
void Sim::face_tables_to_host() {
  if (!faces_deferred || !ctx || !h_Nb.empty()) return;
  const size_t nb = static_cast<size_t>(h_qb_off.back()) * ndk;
  const size_t nf = static_cast<size_t>(h_qf_off.back()) * ndk;
  h_Nb.resize(nb);
  h_Nf.resize(nf);
  if (nb) TG_CUDA(cudaMemcpyAsync(h_Nb.data(), d_Nb.p, nb * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (nf) TG_CUDA(cudaMemcpyAsync(h_Nf.data(), d_Nf.p, nf * 8, cudaMemcpyDeviceToHost, ctx->stream));
  TG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// incidence lists per DOF in the reference's scatter order (face, element, a):
// a stable counting sort of the kept (element, column) slots by DOF
void Sim::build_incidence() {
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
}

// The general patch's operators on the device (K6, k6_assemble.cu): false if
// the patch is beyond it (the host path then runs). Bit-identical to
// assemble_csr_host (tests/test_cfg3.py).
bool Sim::assemble_csr_device(cudaStream_t s) {
  upload_nurbs();
  const ElementGrid eg = element_grid(vol);
  const auto n = vol.basis_counts();
  const auto pd = vol.degrees();
  AsmPatch P{};
  P.V = nurbs;
  std::vector<int> spans[3], elo[3], ehi[3];
  std::vector<double> gn[3], gw[3];
  for (int d = 0; d < 3; ++d) {
    P.n_el[d] = eg.n_el[d];
    P.nq[d] = quad[d];
    const KnotVector& kv = vol.knots(d);
    spans[d].resize(eg.n_el[d]);
    elo[d].assign(n[d], 1 << 30);
    ehi[d].assign(n[d], -1);
    for (int e = 0; e < eg.n_el[d]; ++e) {
      spans[d][e] = kv.find_span(0.5 * (eg.bp[d][e] + eg.bp[d][e + 1]));
      for (int i = spans[d][e] - pd[d]; i <= spans[d][e]; ++i) {
        elo[d][i] = std::min(elo[d][i], e);
        ehi[d][i] = std::max(ehi[d][i], e);
      }
    }
    const GaussRule& g = gauss_rule(quad[d]);
    gn[d] = g.nodes;
    gw[d] = g.weights;
  }
  P.rc = cfg.material.volumetric_capacity();
  P.k = cfg.material.conductivity;
  if (!k6_supported(P)) return false;
  // tensor pattern row pointers (tensor_pattern's row lengths)
  const long rows = static_cast<long>(n[0]) * n[1] * n[2];
  std::vector<int> row_ptr(rows + 1, 0);
  long nnz = 0;
  for (long r = 0; r < rows; ++r) {
    const int rc3[3] = {static_cast<int>(r % n[0]), static_cast<int>((r / n[0]) % n[1]),
                        static_cast<int>(r / (static_cast<long>(n[0]) * n[1]))};
    long len = 1;
    for (int d = 0; d < 3; ++d)
      len *= std::min(n[d] - 1, rc3[d] + pd[d]) - std::max(0, rc3[d] - pd[d]) + 1;
    nnz += len;
    if (nnz > std::numeric_limits<int>::max()) return false;
    row_ptr[r + 1] = static_cast<int>(nnz);
  }
  // device tables (freed at the end)
  DevBuf<double> d_bp[3], d_gn[3], d_gw[3], dM, dK, lm, lk;
  DevBuf<int> d_sp[3], d_lo[3], d_hi[3], d_rp, d_fi, d_ci, d_len[3];
  DevBuf<int> d_flag;
  for (int d = 0; d < 3; ++d) {
    upload(d_bp[d], eg.bp[d], s);
    upload(d_gn[d], gn[d], s);
    upload(d_gw[d], gw[d], s);
    upload(d_sp[d], spans[d], s);
    upload(d_lo[d], elo[d], s);
    upload(d_hi[d], ehi[d], s);
    P.bp[d] = d_bp[d].p;
    P.gn[d] = d_gn[d].p;
    P.gw[d] = d_gw[d].p;
    P.espan[d] = d_sp[d].p;
    P.elo[d] = d_lo[d].p;
    P.ehi[d] = d_hi[d].p;
  }
  upload(d_rp, row_ptr, s);
  dM.ensure(nnz);
  dK.ensure(nnz);
  TG_CUDA(cudaMemsetAsync(dM.p, 0, nnz * sizeof(double), s));
  TG_CUDA(cudaMemsetAsync(dK.p, 0, nnz * sizeof(double), s));
  d_flag.ensure(1);
  TG_CUDA(cudaMemsetAsync(d_flag.p, 0, sizeof(int), s));
  // element matrices by element layers (<= ~2 GB of them at a time), each
  // batch gathered into the pattern before the next (element order per entry)
  const size_t T = k6_entries_per_element(P);
  const size_t per_layer = static_cast<size_t>(eg.n_el[0]) * eg.n_el[1] * T * 2 * sizeof(double);
  const int layers = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(eg.n_el[2], (size_t{2} << 30) / std::max<size_t>(per_layer, 1))));
  const size_t cap = static_cast<size_t>(layers) * eg.n_el[0] * eg.n_el[1] * T;
  lm.ensure(cap);
  lk.ensure(cap);
  const int per = eg.n_el[0] * eg.n_el[1];
  for (int k0 = 0; k0 < eg.n_el[2]; k0 += layers) {
    const int k1 = std::min(eg.n_el[2], k0 + layers);
    k6_element_matrices(P, k0 * per, (k1 - k0) * per, lm.p, lk.p, d_flag.p, s);
    const int rz0 = std::max(0, spans[2][k0] - pd[2]), rz1 = std::min(n[2] - 1, spans[2][k1 - 1]);
    k6_gather(P, d_rp.p, rz0 * n[0] * n[1], (rz1 + 1) * n[0] * n[1], k0, k1, k0 * per, lm.p, lk.p,
              dM.p, dK.p, s);
  }
  int flag = 0;
  TG_CUDA(cudaMemcpyAsync(&flag, d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  if (flag) throw numeric_error("non-positive Jacobian determinant at quadrature point");
  lm.release();
  lk.release();
  // A / B on the free rows as sliced ELL
  upload(d_free_list, dofs.free_list, s);
  upload(d_fi, dofs.free_index, s);
  upload(d_ci, dofs.constrained_index, s);
  const AsmMaps maps{d_free_list.p, d_fi.p, d_ci.p, n_free};
  for (auto& b : d_len) b.ensure(std::max(1, n_free));
  k6_row_lengths(P, maps, d_len[0].p, d_len[1].p, d_len[2].p, s);
  std::vector<int> len[3];
  for (int m = 0; m < 3; ++m) {
    len[m].resize(n_free);
    TG_CUDA(cudaMemcpyAsync(len[m].data(), d_len[m].p, sizeof(int) * n_free,
                            cudaMemcpyDeviceToHost, s));
  }
  TG_CUDA(cudaStreamSynchronize(s));
  SellBufs* bufs[3] = {&sA, &sAc, &sB};
  SellOut outs[3];
  const int ns = (n_free + 31) / 32;
  for (int m = 0; m < 3; ++m) {  // to_sell's slices: 32 rows, padded to the longest
    std::vector<long long> sp(ns + 1, 0);
    for (int sl = 0; sl < ns; ++sl) {
      int w = 0;
      for (int r = sl * 32; r < std::min(n_free, sl * 32 + 32); ++r) w = std::max(w, len[m][r]);
      sp[sl + 1] = sp[sl] + 32LL * w;
    }
    SellBufs& b = *bufs[m];
    upload(b.sp, sp, s);
    upload(b.len, len[m], s);
    b.col.ensure(std::max<long long>(1, sp[ns]));
    b.val.ensure(std::max<long long>(1, sp[ns]));
    TG_CUDA(cudaMemsetAsync(b.col.p, 0, sizeof(int) * sp[ns], s));
    TG_CUDA(cudaMemsetAsync(b.val.p, 0, sizeof(double) * sp[ns], s));
    outs[m] = SellOut{b.sp.p, b.col.p, b.val.p};
  }
  const double dt = dt_solver, th = cfg.stepping.theta;
  k6_fill(P, d_rp.p, maps, dM.p, dK.p, 1.0 / dt, th, -(1.0 - th), outs[0], outs[1], outs[2], s);
  devA = DevSell{n_free, sA.sp.p, sA.len.p, sA.col.p, sA.val.p};
  devAc = DevSell{n_free, sAc.sp.p, sAc.len.p, sAc.col.p, sAc.val.p};
  devB = DevSell{n_free, sB.sp.p, sB.len.p, sB.col.p, sB.val.p};
  TG_CUDA(cudaStreamSynchronize(s));  // the temporaries die here
  csr_device = true;
  return true;
}

// A_ff as CSR on the host: the host assembly's copy, or (device assembly) the
// device's sliced ELL converted back (tg_sim_reduced_operator)
const Csr& Sim::reduced_operator() {
  if (csrA.rows > 0 || !csr_device) return csrA;
  cudaStream_t s = ctx->stream;
  const int ns = (n_free + 31) / 32;
  std::vector<long long> sp(ns + 1);
  std::vector<int> len(n_free);
  TG_CUDA(cudaMemcpyAsync(sp.data(), sA.sp.p, sizeof(long long) * (ns + 1), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(len.data(), sA.len.p, sizeof(int) * n_free, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> col(sp[ns]);
  std::vector<double> val(sp[ns]);
  TG_CUDA(cudaMemcpyAsync(col.data(), sA.col.p, sizeof(int) * sp[ns], cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaMemcpyAsync(val.data(), sA.val.p, sizeof(double) * sp[ns], cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  csrA.rows = n_free;
  csrA.row_ptr.assign(n_free + 1, 0);
  for (int f = 0; f < n_free; ++f) csrA.row_ptr[f + 1] = csrA.row_ptr[f] + len[f];
  csrA.col.resize(csrA.row_ptr[n_free]);
  csrA.val.resize(csrA.row_ptr[n_free]);
  for (int f = 0; f < n_free; ++f) {
    const long long base = sp[f >> 5] + (f & 31);
    for (int k = 0; k < len[f]; ++k) {
      csrA.col[csrA.row_ptr[f] + k] = col[base + 32LL * k];
      csrA.val[csrA.row_ptr[f] + k] = val[base + 32LL * k];
    }
  }
  return csrA;
}

// The general patch's operators on the host (assembly.cpp:59-101, 194-228):
// M, K on the tensor pattern, A / B entrywise, the free-row split.
void Sim::assemble_csr_host() {
  PhaseClock clk;
  const double dt = dt_solver, th = cfg.stepping.theta;
  {
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
  if (faces_deferred) {  // face tables on the device, then the K5 host setup on their points
    PhaseClock clk;
    face_tables_device(s);
    clk.mark("face tables on the device");
    sf_setup_host();
    clk.mark("k5 grids, tiles, entries");
  } else {
    upload(d_qx, h_qx, s);
    upload(d_qn, h_qn, s);
    upload(d_qw, h_qw, s);
    upload(d_Nb, h_Nb, s);
    upload(d_Nf, h_Nf, s);
  }
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
  h_fine.assign(2 * static_cast<size_t>(n_fe) + 2, 0);
  for (auto& st : sf_stage) TG_CUDA(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
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
    rhs_tma = !std::getenv("TG_K2_RHS_NO_TMA") && k2_make_map(gfull, d_T.p, &map_T) &&
              k2_make_map(gfull, d_gfull.p, &map_g);
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
      // strip tiles over the ragged last x columns of grids that fill the GPU
      // (2 planes per step; on latency-bound small grids the slower strip CTA
      // sets the iteration time: config 2 16.4 -> 17.2 us per iteration with
      // strips). TG_K2_NO_STRIP: main tiles only; TG_K2_STRIP=1 forces them.
      const bool want_strip = std::getenv("TG_K2_STRIP") ? true : L == 2;
      m.strip = use_cg1 && want_strip && k2_strip_applies(gfree) &&
                !std::getenv("TG_K2_NO_STRIP") &&
                k2_make_map(gfree, d_x.p, &m.sx, true, L, true) &&
                k2_make_map(gfree, d_r.p, &m.sr[0], true, L, true) &&
                k2_make_map(gfree, d_z.p, &m.sr[1], true, L, true) &&
                k2_make_map(gfree, d_Ap.p, &m.sw[0], true, L, true) &&
                k2_make_map(gfree, d_w2.p, &m.sw[1], true, L, true) &&
                k2_make_map(gfree, d_p2.p, &m.ss[0], true, L, true) &&
                k2_make_map(gfree, d_s2.p, &m.ss[1], true, L, true) &&
                k2_make_map(gfree, d_x.p, &m.sxc, false, L, true) &&
                k2_make_map(gfree, d_p.p, &m.spc, false, L, true);
      if (use_cg1) pcg_blocks = k2_cg1_max_blocks(p, ctx->sm_count, gfree.n[2], cg1_pl);
      // small grids: the solver state resident in shared memory (k2_resident.cu)
      int max_smem = 0;
      TG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                     ctx->device));
      use_res = use_cg1 && k2_res_plan(gfree, ctx->sm_count, max_smem, &res_plan);
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
      d_w2.ensure(n_free);
      d_dots.ensure(8);
      TG_CUDA(cudaMallocHost(&h_dots, 2 * sizeof(double)));
      use_fdm = true;
      use_cg1 = false;
    }
  } else {
    // the operators assembled on the device (K6) unless the patch needs the
    // host path (basis block too large) or TG_HOST_ASSEMBLY is set
    bool on_device = false;
    if (csr_deferred) {
      PhaseClock clk;
      on_device = assemble_csr_device(s);
      clk.mark(on_device ? "csr operators on the device" : "device assembly unsupported");
      if (!on_device) assemble_csr_host();
    }
    auto up = [&](const Csr& C, SellBufs& b, DevSell& out) {
      const Sell h = to_sell(C);
      upload(b.sp, h.slice_ptr, s);
      upload(b.len, h.row_len, s);
      upload(b.col, h.col, s);
      upload(b.val, h.val, s);
      TG_CUDA(cudaStreamSynchronize(s));  // h dies here
      out = DevSell{C.rows, b.sp.p, b.len.p, b.col.p, b.val.p};
    };
    if (!on_device) {
      up(csrA, sA, devA);
      up(csrAc, sAc, devAc);
      up(csrB, sB, devB);
      csrAc = Csr{};  // host copies no longer needed (csrA stays: tg_sim_reduced_operator)
      csrB = Csr{};
    }
    upload(d_free_list, dofs.free_list, s);
    {  // the implicit-column copy of A_ff: free rows = the grid minus the bottom layer
      const auto dg = vol.degrees();
      int fb[3] = {geom.n[0], geom.n[1], geom.n[2]};
      fb[geom.ax] -= 1;
      use_dia = false;
      const int W = 2 * dg[0] + 1;
      const size_t dia_n = static_cast<size_t>((n_free + 31) / 32) * 32 * W * W * W;
      size_t mem_free = 0, mem_total = 0;
      TG_CUDA(cudaMemGetInfo(&mem_free, &mem_total));
      // (a second copy of A_ff: only when it takes at most half the free memory)
      if (!std::getenv("TG_K2_NO_DIA") && dg[0] == dg[1] && dg[1] == dg[2] &&
          static_cast<long>(fb[0]) * fb[1] * fb[2] == n_free && dia_n * 8 <= mem_free / 2) {
        d_dia.ensure(dia_n);
        d_dia_flag.ensure(1);
        use_dia = csr_make_dia(devA, fb[0], fb[1], fb[2], dg[0], d_dia.p, d_dia_flag.p, &devAd, s);
        if (!use_dia) d_dia.release();
      }
    }
    csr_inverse_diagonal(devA, d_invd.p, d_status.p, s);
    pcg_blocks = csr_pcg_max_blocks(ctx->sm_count);
    if (preconditioner == 1) setup_general_fdm(s);
  }
  d_partials.ensure(std::max<size_t>(8 * static_cast<size_t>(pcg_blocks) + 8, 1024));
  TG_CUDA(cudaMemcpyAsync(h_status, d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  diag_ok = h_status->status != 2;
  sf_setup_device();
}

// Preconditioner for non-separable patches (config 3's rational part): the
// fast-diagonalization inverse of a separable approximation of A, scaled to
// A's diagonal. Per axis d the control net's mean cumulative arc length along
// d (averaged over all control lines) stands in for a separable map; its 1D
// mass / stiffness bands (assemble_band_1d) give A~ = a M~z x M~y x M~x + b
// (...), exactly invertible by FDM. With S = diag(sqrt(diag A / diag A~)),
// P = S^-1 A~^-1 S^-1 is SPD and close to A^-1 where the geometry varies
// slowly; the reference's PCG loop runs with P in place of Jacobi.
void Sim::setup_general_fdm(cudaStream_t s) {
  const ControlGrid& cg = vol.grid();
  const auto n = cg.dims;
  std::array<Band1D, 3> ab;
  for (int d = 0; d < 3; ++d) {
    const int o1 = (d + 1) % 3, o2 = (d + 2) % 3;
    std::vector<double> X(n[d], 0.0);
    int lines = 0;
    for (int b = 0; b < n[o2]; ++b)
      for (int a = 0; a < n[o1]; ++a) {
        double acc = 0.0;
        for (int i = 1; i < n[d]; ++i) {
          int ijk0[3], ijk1[3];
          ijk0[d] = i - 1;
          ijk1[d] = i;
          ijk0[o1] = ijk1[o1] = a;
          ijk0[o2] = ijk1[o2] = b;
          const auto& p0 = cg.pts[cg.index(ijk0[0], ijk0[1], ijk0[2])];
          const auto& p1 = cg.pts[cg.index(ijk1[0], ijk1[1], ijk1[2])];
          acc += std::sqrt((p1[0] - p0[0]) * (p1[0] - p0[0]) + (p1[1] - p0[1]) * (p1[1] - p0[1]) +
                           (p1[2] - p0[2]) * (p1[2] - p0[2]));
          X[i] += acc;
        }
        ++lines;
      }
    for (double& v : X) v /= lines;
    ab[d] = assemble_band_1d(vol.knots(d), X, quad[d]);
  }
  const double th = cfg.stepping.theta, dt = dt_solver;
  const double a = cfg.material.volumetric_capacity() / dt, b = th * cfg.material.conductivity;
  int nfree[3];
  std::vector<double> Vall, Lall;
  size_t offV[3], offL[3];
  std::vector<double> dm[3], dk[3];  // the approximation's 1D diagonals on the free rows
  for (int d = 0; d < 3; ++d) {
    const int first = (d == geom.ax && geom.layer == 0) ? 1 : 0;
    nfree[d] = ab[d].n - (d == geom.ax ? 1 : 0);
    const Fdm1D f = fdm_factor(ab[d].M, ab[d].K, ab[d].n, ab[d].p, first, nfree[d]);
    offV[d] = Vall.size();
    offL[d] = Lall.size();
    Vall.insert(Vall.end(), f.V.begin(), f.V.end());
    Lall.insert(Lall.end(), f.lam.begin(), f.lam.end());
    const int W = 2 * ab[d].p + 1;
    for (int i = 0; i < nfree[d]; ++i) {
      dm[d].push_back(ab[d].M[(first + i) * W + ab[d].p]);
      dk[d].push_back(ab[d].K[(first + i) * W + ab[d].p]);
    }
  }
  // S^-1 = sqrt(diag A~ / diag A) on the free points (free flat order)
  std::vector<double> invd(n_free), sinv(n_free);
  TG_CUDA(cudaMemcpyAsync(invd.data(), d_invd.p, sizeof(double) * n_free, cudaMemcpyDeviceToHost, s));
  TG_CUDA(cudaStreamSynchronize(s));
  for (int k = 0, f = 0; k < nfree[2]; ++k)
    for (int j = 0; j < nfree[1]; ++j)
      for (int i = 0; i < nfree[0]; ++i, ++f) {
        const double mm = dm[0][i] * dm[1][j] * dm[2][k];
        const double kk = dk[0][i] * dm[1][j] * dm[2][k] + dm[0][i] * dk[1][j] * dm[2][k] +
                          dm[0][i] * dm[1][j] * dk[2][k];
        sinv[f] = std::sqrt((a * mm + b * kk) * invd[f]);
      }
  if (static_cast<long>(nfree[0]) * nfree[1] * nfree[2] != n_free)
    throw std::logic_error("general FDM: free grid does not match the DOF split");
  upload(d_fdmV, Vall, s);
  upload(d_fdmL, Lall, s);
  upload(d_fdmS, sinv, s);
  d_fdmDinv.ensure(n_free);
  fdm_inverse_eigs(nfree, d_fdmL.p + offL[0], d_fdmL.p + offL[1], d_fdmL.p + offL[2], a, b,
                   d_fdmDinv.p, s);
  for (int d = 0; d < 3; ++d) {
    fdm.n[d] = nfree[d];
    fdm.V[d] = d_fdmV.p + offV[d];
  }
  fdm.dinv = d_fdmDinv.p;
  fdm.sinv = d_fdmS.p;
  d_z.ensure(n_free);
  d_p2.ensure(n_free);
  d_w2.ensure(n_free);
  d_dots.ensure(8);
  TG_CUDA(cudaMallocHost(&h_dots, 2 * sizeof(double)));
  use_fdm = true;
}

// K5 setup (host): are the lateral faces' base quadrature points and the
// Greville points tensor grids (up to coordinate rounding) with normals exactly
// along an axis? Then cut them into CTA tiles / regions and list the points
// of every region for the pair-wise remainder (k5_fused.cuh).
namespace {

// contiguous nearly equal pieces of n, each <= cap
std::vector<std::pair<int, int>> split_even(int n, int cap) {
  std::vector<std::pair<int, int>> out;
  const int k = std::max(1, (n + cap - 1) / cap);
  for (int i = 0; i < k; ++i) out.emplace_back(n * i / k, n * (i + 1) / k - n * i / k);
  return out;
}

// the same number of pieces: full pieces of cap, the remainder last
std::vector<std::pair<int, int>> split_full(int n, int cap) {
  std::vector<std::pair<int, int>> out;
  for (int a = 0; a < n; a += cap) out.emplace_back(a, std::min(cap, n - a));
  if (out.empty()) out.emplace_back(0, n);
  return out;
}

// A tile's time per stage in full-tile stages: the MMAs of its busiest SM
// sub-partition (the active warp blocks, sf_warp_block) plus the generator
// (every row of A and B, partial tiles too: about 0.13 of a full stage,
// profiles/r02_k5_ncu_summary.md).
double sf_tile_cost(int na, int nb) {
  int per[4] = {0, 0, 0, 0};
  for (int w = 0; w < kSfWarps; ++w) {
    int wa, wb;
    sf_warp_block(w, wa, wb);
    if (32 * wa < na && kSfWN * wb < nb) ++per[w % 4];
  }
  const int m = *std::max_element(per, per + 4);
  return m / (kSfWarps / 4.0) + 0.13;
}

// the CTA tiles of an na x nb grid (row pieces, column pieces): nearly equal
// pieces, or full pieces and a remainder, per axis, whichever costs less
// (e.g. 258 x 258: 128 + 128 + 2 rows x 129 + 129 columns beats 3 x 86 rows)
void sf_split_tiles(int na, int nb, std::vector<std::pair<int, int>>& as,
                    std::vector<std::pair<int, int>>& bs) {
  const std::vector<std::pair<int, int>> ca[2] = {split_even(na, kSfTA), split_full(na, kSfTA)};
  const std::vector<std::pair<int, int>> cb[2] = {split_even(nb, kSfTB), split_full(nb, kSfTB)};
  double best = 1e300;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      double c = 0.0;
      for (const auto& a : ca[i])
        for (const auto& b : cb[j]) c += sf_tile_cost(a.second, b.second);
      if (c < best - 1e-9) {
        best = c;
        as = ca[i];
        bs = cb[j];
      }
    }
}

SfRegion box_of(const SfGrid& g, int a0, int na, int b0, int nb) {
  SfRegion r{};
  r.lo[g.axn] = r.hi[g.axn] = g.xf;
  r.lo[g.axu] = g.U[a0];
  r.hi[g.axu] = g.U[a0 + na - 1];
  r.lo[g.axv] = g.V[b0];
  r.hi[g.axv] = g.V[b0 + nb - 1];
  r.delta = g.delta;
  r.npts = static_cast<double>(na) * nb;
  return r;
}

}  // namespace

void Sim::sf_setup_host() {
  PhaseClock clk;
  if (const char* e = std::getenv("TG_SF_MIN_PAIRS")) sf_min_pairs = std::atof(e);
  if (const char* e = std::getenv("TG_SF_MIN_SOURCES")) sf_min_sources = std::atoi(e);
  if (const char* e = std::getenv("TG_SF_K1_SPLITS"))
    sf_k1_splits = std::max(1, std::min(kMaxSplits, std::atoi(e)));
  const int tqb = h_qb_off.empty() ? 0 : h_qb_off.back();
  const int tqf = h_qf_off.empty() ? 0 : h_qf_off.back();
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
  // normal key: 2 axis + (sign > 0) when the normal lies on an axis up to the
  // spline rounding of its tangents' cross product (off-axis components
  // <= 1e-12; ~5e-14 on the BASELINE cuboids). The contraction takes n[axn]
  // only: a dropped term is n_off * (in-plane gradient), below 1e-12 of the
  // pair's gradient, two orders under the 1e-10 flux tolerance.
  auto normal_key = [&](int q) {
    const double* n = &h_qn[3 * static_cast<size_t>(q)];
    int ax = 0;
    for (int d = 1; d < 3; ++d)
      if (std::fabs(n[d]) > std::fabs(n[ax])) ax = d;
    const bool axis = std::fabs(std::fabs(n[ax]) - 1.0) <= 1e-12 &&
                      std::fabs(n[(ax + 1) % 3]) <= 1e-12 && std::fabs(n[(ax + 2) % 3]) <= 1e-12;
    return axis ? 2 * ax + (n[ax] > 0.0) : -1;
  };
  sf_flux_ok = tqb > 0;
  std::vector<int> ekey(n_fe, -1);
  std::vector<std::vector<int>> kelems(6);
  {  // per element: one axis normal shared by all its points (-1: none)
    std::vector<char> ok(n_fe, 1);
    parallel_for(n_fe, [&](long e) {
      ekey[e] = normal_key(h_qb_off[e]);
      bool good = ekey[e] >= 0;
      for (int q = h_qb_off[e]; q < h_qb_off[e + 1] && good; ++q) good = normal_key(q) == ekey[e];
      for (int l = h_qf_off[e]; l < h_qf_off[e + 1] && good; ++l)
        good = normal_key(tqb + l) == ekey[e];
      ok[e] = good;
    }, 256);
    for (int e = 0; e < n_fe && sf_flux_ok; ++e) {
      sf_flux_ok = ok[e] != 0;
      if (sf_flux_ok) kelems[ekey[e]].push_back(e);
    }
  }
  // base grid per face (normal key)
  sf_h_gcell.assign(tqb, -1);
  std::vector<int> q_face(tqb, -1);
  sf_elem_face.assign(n_fe, -1);
  // the faces' base grids (in parallel; used in face-key order below)
  SfGrid kgrid[6];
  char kgood[6] = {1, 1, 1, 1, 1, 1};
  if (sf_flux_ok)
    parallel_for(6, [&](long k) {
      if (kelems[k].empty()) return;
      std::vector<double> pts;
      for (int e : kelems[k])
        for (int q = h_qb_off[e]; q < h_qb_off[e + 1]; ++q)
          for (int d = 0; d < 3; ++d) pts.push_back(h_qx[3 * static_cast<size_t>(q) + d]);
      kgood[k] = sf_make_grid(pts.data(), static_cast<long>(pts.size() / 3), tol, kgrid[k]) &&
                 kgrid[k].axn == k / 2;
    }, 1);
  for (int k = 0; k < 6 && sf_flux_ok; ++k) {
    if (kelems[k].empty()) continue;
    SfGrid& g = kgrid[k];
    if (!kgood[k]) {
      sf_flux_ok = false;
      break;
    }
    const int f = static_cast<int>(sf_faces.size());
    size_t c = 0;
    for (int e : kelems[k]) {
      sf_elem_face[e] = f;
      for (int q = h_qb_off[e]; q < h_qb_off[e + 1]; ++q, ++c) {
        sf_h_gcell[q] = g.cell[c];
        q_face[q] = f;
      }
    }
    sf_faces.push_back(std::move(g));
  }
  if (!sf_flux_ok) sf_faces.clear();
  // fine-rule points: per face a finer grid; a step's fine elements take a
  // rectangle of it
  sf_fine_ok = sf_flux_ok && tqf > 0;
  sf_h_fa.assign(tqf, 0);
  sf_h_fb.assign(tqf, 0);
  sf_h_ff.assign(tqf, 0);
  if (sf_fine_ok) {
    sf_erect.assign(4 * static_cast<size_t>(n_fe), 0);
    std::vector<std::vector<int>> felems(sf_faces.size());
    for (int e = 0; e < n_fe; ++e) felems[sf_elem_face[e]].push_back(e);
    std::vector<SfGrid> fgrid(felems.size());
    std::vector<char> fgood(felems.size(), 1);
    parallel_for(static_cast<long>(felems.size()), [&](long f) {
      std::vector<double> pts;
      for (int e : felems[f])
        for (int l = h_qf_off[e]; l < h_qf_off[e + 1]; ++l)
          for (int d = 0; d < 3; ++d) pts.push_back(h_qx[3 * static_cast<size_t>(tqb + l) + d]);
      fgood[f] = sf_make_grid(pts.data(), static_cast<long>(pts.size() / 3), tol, fgrid[f]) &&
                 fgrid[f].axn == sf_faces[f].axn;
    }, 1);
    for (size_t f = 0; f < felems.size() && sf_fine_ok; ++f) {
      SfGrid& g = fgrid[f];
      if (!fgood[f]) {
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
          sf_h_fa[l] = a;
          sf_h_fb[l] = b;
          sf_h_ff[l] = static_cast<int>(f);
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
  clk.mark("  k5: face grids");
  sf_dir_ok = n_con > 0 && sf_make_grid(grev.data(), n_con, tol, sf_dir);

  // grids: faces, fine faces, Greville (descriptor lines are device pointers,
  // set in sf_setup_device); the B exponent of a grid is cb[b] * nisp when
  // every source shares its V coordinate (a layer's scan on its plane)
  sf_grids_h.clear();
  auto desc = [&](const SfGrid& g, int flux) {
    SfGridDesc d{};
    d.axn = g.axn;
    d.axu = g.axu;
    d.axv = g.axv;
    d.na = static_cast<int>(g.U.size());
    d.nb = static_cast<int>(g.V.size());
    d.flux = flux;
    d.xf = g.xf;
    bool same = !sources.empty();
    const double v0 = same ? sources[0].position[g.axv] : 0.0;
    for (size_t j = 1; j < sources.size() && same; ++j)
      same = std::memcmp(&sources[j].position[g.axv], &v0, sizeof(double)) == 0;
    d.vplane = same ? 1 : 0;
    return d;
  };
  for (const SfGrid& g : sf_faces) sf_grids_h.push_back(desc(g, 1));
  sf_grid_fine0 = static_cast<int>(sf_grids_h.size());
  for (const SfGrid& g : sf_fine) sf_grids_h.push_back(desc(g, 1));
  sf_grid_dir = -1;
  if (sf_dir_ok) {
    sf_grid_dir = static_cast<int>(sf_grids_h.size());
    sf_grids_h.push_back(desc(sf_dir, 0));
  }
  // static tiles = regions: face grids, then the Greville grid
  sf_tiles_h.clear();
  sf_regions_h.clear();
  std::vector<std::vector<int>> tile_pts;  // entry point ids per static tile
  std::vector<std::vector<int>> tile_cell;
  auto add_tiles = [&](const SfGrid& g, int grid) {
    const int na = static_cast<int>(g.U.size()), nb = static_cast<int>(g.V.size());
    std::vector<std::pair<int, int>> as, bs;
    sf_split_tiles(na, nb, as, bs);
    const int first = static_cast<int>(sf_tiles_h.size());
    for (const auto& [b0, nbt] : bs)
      for (const auto& [a0, nat] : as) {
        const int r = static_cast<int>(sf_regions_h.size());
        sf_tiles_h.push_back(SfTile{grid, a0, b0, nat, nbt, r});
        sf_regions_h.push_back(box_of(g, a0, nat, b0, nbt));
      }
    tile_pts.resize(sf_tiles_h.size());
    tile_cell.resize(sf_tiles_h.size());
    // cell (a, b) -> its tile (as / bs are sorted runs)
    std::vector<int> ta(na), tb(nb);
    for (size_t i = 0; i < as.size(); ++i)
      for (int a = as[i].first; a < as[i].first + as[i].second; ++a) ta[a] = static_cast<int>(i);
    for (size_t i = 0; i < bs.size(); ++i)
      for (int b = bs[i].first; b < bs[i].first + bs[i].second; ++b) tb[b] = static_cast<int>(i);
    return [=](int cell, int& tile, int& local) {
      const int a = cell % na, b = cell / na;
      tile = first + ta[a] + static_cast<int>(as.size()) * tb[b];
      const SfTile& T = sf_tiles_h[tile];
      local = (a - T.a0) + kSfTA * (b - T.b0);
    };
  };
  if (sf_flux_ok) {
    std::vector<std::function<void(int, int&, int&)>> locate;
    for (size_t f = 0; f < sf_faces.size(); ++f)
      locate.push_back(add_tiles(sf_faces[f], static_cast<int>(f)));
    for (int q = 0; q < tqb; ++q) {  // in compact (element) order
      int t, l;
      locate[q_face[q]](sf_h_gcell[q], t, l);
      tile_pts[t].push_back(q);
      tile_cell[t].push_back(l);
    }
  }
  sf_nt_flux = static_cast<int>(sf_tiles_h.size());
  if (sf_dir_ok) {
    auto loc = add_tiles(sf_dir, sf_grid_dir);
    for (int c = 0; c < n_con; ++c) {
      int t, l;
      loc(sf_dir.cell[c], t, l);
      tile_pts[t].push_back(c);
      tile_cell[t].push_back(l);
    }
  }
  sf_nt_static = static_cast<int>(sf_tiles_h.size());
  // remainder entries: per tile its points in compact 2D blocks (columns of
  // kBlockA cells along a, b slower, a fastest), so that each K1 CTA's 1792
  // points span a small box and its per-CTA source culling drops more of the
  // history; padded to whole K1 CTAs
  clk.mark("  k5: greville grid, tiles");
  sf_k1_ppc = kK1Threads * 7;  // k1_partial<7, GRAD> (the remainder launch)
  constexpr int kBlockA = 48;
  parallel_for(sf_nt_static, [&](long t) {
    std::vector<int> ord(tile_pts[t].size());
    std::iota(ord.begin(), ord.end(), 0);
    const auto& cells = tile_cell[t];
    auto key = [&](int i) {
      const int a = cells[i] % kSfTA, b = cells[i] / kSfTA;
      return std::make_tuple(a / kBlockA, b, a);
    };
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return key(x) < key(y); });
    std::vector<int> p2(ord.size()), c2(ord.size());
    for (size_t i = 0; i < ord.size(); ++i) {
      p2[i] = tile_pts[t][ord[i]];
      c2[i] = cells[ord[i]];
    }
    tile_pts[t].swap(p2);
    tile_cell[t].swap(c2);
  }, 1);
  clk.mark("  k5: entry order");
  sf_ent_q.clear();
  sf_ent_tile.clear();
  sf_ent_cell.clear();
  sf_ent_pos.clear();
  sf_cta_region.clear();
  const int qdir0 = tqb + tqf;  // Greville points follow the face points in d_qx
  for (int t = 0; t < sf_nt_static; ++t) {
    if (t == sf_nt_flux) {
      sf_ne_flux = static_cast<int>(sf_ent_q.size());
      sf_nc_flux = static_cast<int>(sf_cta_region.size());
    }
    const bool dir = t >= sf_nt_flux;
    const auto& P = tile_pts[t];
    const int n = static_cast<int>(P.size());
    const int pad = (n + sf_k1_ppc - 1) / sf_k1_ppc * sf_k1_ppc;
    for (int i = 0; i < pad; ++i) {
      const bool real = i < n;
      const int pt = real ? P[i] : P[0];
      sf_ent_q.push_back(dir ? qdir0 + pt : pt);
      sf_ent_tile.push_back(real ? t : -1);
      sf_ent_cell.push_back(real ? tile_cell[t][i] : 0);
      sf_ent_pos.push_back(dir && real ? pt : -1);  // flux: set per step
    }
    for (int c = 0; c < pad / sf_k1_ppc; ++c) sf_cta_region.push_back(sf_tiles_h[t].region);
  }
  if (sf_nt_flux == sf_nt_static) {
    sf_ne_flux = static_cast<int>(sf_ent_q.size());
    sf_nc_flux = static_cast<int>(sf_cta_region.size());
  }
  sf_ne_static = static_cast<int>(sf_ent_q.size());
  sf_nc_static = static_cast<int>(sf_cta_region.size());
  if (std::getenv("TG_SF_DEBUG"))
    std::fprintf(stderr, "[k5] flux %d fine %d dir %d grids %zu tiles %d+%d entries %d+%d\n",
                 sf_flux_ok, sf_fine_ok, sf_dir_ok, sf_grids_h.size(), sf_nt_flux,
                 sf_nt_static - sf_nt_flux, sf_ne_flux, sf_ne_static - sf_ne_flux);
  clk.mark("  k5: entries");
  const char* e = std::getenv("TG_SUMFACT");
  set_sumfact(!(e && std::string(e) == "0"));
}

void Sim::sf_setup_device() {
  cudaStream_t s = ctx->stream;
  if (!(sf_flux_ok || sf_dir_ok)) return;
  // grid lines (+ cb) on the device; descriptors point at them
  std::vector<double> lines, cb;
  std::vector<size_t> at, atc;
  std::vector<const SfGrid*> gs;
  for (const SfGrid& g : sf_faces) gs.push_back(&g);
  for (const SfGrid& g : sf_fine) gs.push_back(&g);
  if (sf_dir_ok) gs.push_back(&sf_dir);
  for (size_t i = 0; i < gs.size(); ++i) {
    const SfGrid& g = *gs[i];
    at.push_back(lines.size());
    lines.insert(lines.end(), g.U.begin(), g.U.end());
    lines.insert(lines.end(), g.V.begin(), g.V.end());
    atc.push_back(cb.size());
    const double vs = sources.empty() ? 0.0 : sources[0].position[g.axv];
    for (double v : g.V) cb.push_back((v - vs) * (v - vs));
  }
  upload(d_sf_lines, lines, s);
  upload(d_sf_cb, cb, s);
  for (size_t i = 0; i < gs.size(); ++i) {
    SfGridDesc& d = sf_grids_h[i];
    d.U = d_sf_lines.p + at[i];
    d.V = d.U + d.na;
    d.cb = d_sf_cb.p + atc[i];
  }
  upload(d_sf_grids, sf_grids_h, s);
  std::vector<double> tab(kExpTableSize);
  k1_exp_table_host(tab.data());
  upload(d_sf_tab, tab, s);
  // static tables, with room for the per-step fine tiles / regions / entries
  const int tqb = h_qb_off.back(), tqf = h_qf_off.back();
  size_t ft = 0;
  for (const SfGrid& g : sf_fine)
    ft += split_even(static_cast<int>(g.U.size()), kSfTA).size() *
          split_even(static_cast<int>(g.V.size()), kSfTB).size();
  const size_t nfr = sf_fine_ok ? sf_fine.size() : (sf_flux_ok ? 1 : 0);
  const size_t fent = sf_flux_ok ? static_cast<size_t>(tqf) + nfr * sf_k1_ppc : 0;
  d_sf_tiles.ensure(sf_nt_static + ft + 1);
  d_sf_regions.ensure(sf_regions_h.size() + nfr + 1);
  d_sf_ent_q.ensure(sf_ne_static + fent + 1);
  d_sf_ent_tile.ensure(sf_ne_static + fent + 1);
  d_sf_ent_cell.ensure(sf_ne_static + fent + 1);
  d_sf_ent_pos.ensure(sf_ne_static + fent + 1);
  d_sf_cta.ensure(sf_nc_static + fent / sf_k1_ppc + nfr + 1);
  auto put = [&](auto& d, const auto& h) {
    if (!h.empty())
      TG_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice, s));
  };
  put(d_sf_tiles, sf_tiles_h);
  put(d_sf_regions, sf_regions_h);
  put(d_sf_ent_q, sf_ent_q);
  put(d_sf_ent_tile, sf_ent_tile);
  put(d_sf_ent_cell, sf_ent_cell);
  put(d_sf_ent_pos, sf_ent_pos);
  put(d_sf_cta, sf_cta_region);
  d_sf_stats.ensure(2);
  TG_CUDA(cudaMemsetAsync(d_sf_stats.p, 0, 2 * sizeof(double), s));
  d_sf_J.ensure(sf_regions_h.size() + nfr + 1);
  d_sf_Jraw.ensure(sf_regions_h.size() + nfr + 1);
  d_sf_Jl.ensure(sf_regions_h.size() + 1);
  d_sf_El.ensure(sf_regions_h.size() + 1);
  d_sf_Jcl.ensure(sf_regions_h.size() + 1);
  TG_CUDA(cudaMemsetAsync(d_sf_Jl.p, 0, sizeof(int) * (sf_regions_h.size() + 1), s));
  TG_CUDA(cudaMemsetAsync(d_sf_El.p, 0, sizeof(int) * (sf_regions_h.size() + 1), s));
  TG_CUDA(cudaMemsetAsync(d_sf_Jcl.p, 0, sizeof(int) * (sf_regions_h.size() + 1), s));
  // eligible lists: one row of n_sources indices / bits per region
  sf_list_cap = std::max<int>(1, static_cast<int>(sources.size()));
  sf_list_words = (sf_list_cap + 31) / 32;
  const size_t nrows = sf_regions_h.size() + nfr + 1;
  d_sf_Jc.ensure(nrows);
  d_sf_elist.ensure(nrows * sf_list_cap);
  d_sf_okbits.ensure(nrows * sf_list_words);
  d_sf_E.ensure(sf_regions_h.size() + nfr + 1);
  d_sf_prefix.ensure(sf_nt_static + ft + 2);
  // qp -> element of the base points (their compact positions per step)
  std::vector<int> qelem(tqb);
  for (int e = 0; e < n_fe; ++e)
    for (int q = h_qb_off[e]; q < h_qb_off[e + 1]; ++q) qelem[q] = e;
  upload(d_sf_qelem, qelem, s);
  // the Greville points after the face points (one coordinate array for the
  // remainder launch)
  if (sf_dir_ok) {
    d_qx.ensure(3 * (static_cast<size_t>(tqb) + tqf + n_con));  // (never grows: sized here)
    if (!faces_deferred)  // (device-built face points are in place already)
      TG_CUDA(cudaMemcpyAsync(d_qx.p, h_qx.data(), h_qx.size() * sizeof(double),
                              cudaMemcpyHostToDevice, s));
    TG_CUDA(cudaMemcpyAsync(d_qx.p + 3 * (static_cast<size_t>(tqb) + tqf), grev.data(),
                            grev.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  // one row of max_src = n_sources + 1 per grid: entry n_sources is always a zero
  // factor (the contraction's padding columns)
  d_sf_cst.ensure(sf_grids_h.size() * (sources.size() + 1));
  d_sf_scratch.ensure((sf_nt_static + ft + sf_contract_max_ctas(ctx->sm_count) + 1) *
                      static_cast<size_t>(kSfTA * kSfTB));
  TG_CUDA(cudaStreamSynchronize(s));
  sf_ready = true;
}

char* Sim::stage_bytes(size_t bytes) {
  Stage& st = sf_stage[sf_stage_i];
  sf_stage_i = (sf_stage_i + 1) % 3;
  TG_CUDA(cudaEventSynchronize(st.done));  // its last copies have run
  if (bytes > st.cap) {
    if (st.h) TG_CUDA(cudaFreeHost(st.h));
    st.cap = bytes + bytes / 4 + 4096;
    TG_CUDA(cudaMallocHost(&st.h, st.cap));
  }
  return st.h;
}

void Sim::release_stages() {
  for (auto& st : sf_stage) {
    if (st.h) cudaFreeHost(st.h);
    if (st.done) cudaEventDestroy(st.done);
    st.h = nullptr;
    st.done = nullptr;
  }
}


void Sim::sf_plan_host(double t, int* J, int* E, int* Jc) {
  const double alpha = cfg.material.diffusivity(), cull = cfg.superpose.cull_exponent;
  const double* src = reinterpret_cast<const double*>(sources.data());
  // the causally active prefix (tg_ctx::active_prefix): later sources all
  // have t - tau <= 0
  int n_act = static_cast<int>(sources.size());
  while (n_act > 0 && !(t - src[6 * (n_act - 1) + 5] > 0.0)) --n_act;
  for (size_t r = 0; r < sf_regions_h.size(); ++r) {
    const SfRegion& R = sf_regions_h[r];
    int j = 0;
    if (sf_on) {
      while (j < n_act && sf_region_ok(src + 6 * static_cast<size_t>(j), t, alpha, cull, R)) ++j;
      if (R.npts < 0.0 ||
          (static_cast<double>(j) * R.npts < sf_min_pairs && j < sf_min_sources))
        j = 0;
    }
    int e = n_act;
    while (e > j && sf_region_culled(src + 6 * static_cast<size_t>(e - 1), t, alpha, cull, R))
      --e;
    J[r] = j;
    E[r] = e;
    if (Jc) {  // + the eligible sources of [J, E) (k5_fused.cuh SfLists)
      int c = j;
      for (int k = j; k < e && j > 0; ++k)
        c += sf_region_ok(src + 6 * static_cast<size_t>(k), t, alpha, cull, R) ? 1 : 0;
      Jc[r] = c;
    }
  }
}

double Sim::sf_flops_total() {
  if (!sf_ready) return 0.0;
  double v = 0.0;
  TG_CUDA(cudaMemcpyAsync(&v, d_sf_stats.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TG_CUDA(cudaStreamSynchronize(ctx->stream));
  return v;
}

void Sim::sf_last_plan(int* J, int* E, int* Jc) {
  const size_t n = sf_regions_h.size();
  TG_CUDA(cudaMemcpyAsync(J, d_sf_Jl.p, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TG_CUDA(cudaMemcpyAsync(E, d_sf_El.p, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  if (Jc)
    TG_CUDA(cudaMemcpyAsync(Jc, d_sf_Jcl.p, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TG_CUDA(cudaStreamSynchronize(ctx->stream));
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
  h_fine.resize(2 * static_cast<size_t>(n_fe) + 2);
  if (focus_given) {
    f = focus_value;
  } else if (!focus_at(t, f)) {
    return 0;
  }
  for (int e = 0; e < n_fe; ++e) {
    const Vec3 c{centers[3 * e], centers[3 * e + 1], centers[3 * e + 2]};
    if ((c - f).norm() < radius) h_fine[nf++] = e;
  }
  return nf;
}

// The fused loads path (full range): F_{n+1} = assemble_flux_load and/or
// g_{n+1} = dirichlet_values at t through K5 + the K1 remainder. No host
// synchronisation: the per-step host data (fine elements, the fine regions'
// tiles and points) goes through a pinned ring.
void Sim::loads_device(double t, double radius, double* d_F, double* d_g, bool gather) {
  cudaStream_t s = ctx->stream;
  const bool flux = d_F != nullptr || !gather;
  const bool dir = d_g != nullptr && sf_dir_ok;
  const int tqb = h_qb_off.back();
  // ---- host: fine-rule elements and their compact offsets
  int nf = 0;
  int* extra = nullptr;
  if (flux) {
    nf = fine_elements(t, radius);
    extra = h_fine.data() + n_fe + 1;
    extra[0] = 0;
    for (int r = 0; r < nf; ++r) {
      const int e = h_fine[r];
      extra[r + 1] = extra[r] + (h_qf_off[e + 1] - h_qf_off[e]) - (h_qb_off[e + 1] - h_qb_off[e]);
    }
  }
  const long n_compact = flux ? static_cast<long>(tqb) + (nf ? extra[nf] : 0) : 0;
  sf_last_npts = n_compact;
  // ---- host: the step's fine regions (one per face with fine elements)
  std::vector<SfTile> ftiles;
  std::vector<SfRegion> fregs;
  std::vector<int> fq, fpos, ftile, fcell, fcta;
  const int nreg_static = static_cast<int>(sf_regions_h.size());
  if (flux && nf > 0) {
    const size_t nF = sf_fine_ok ? sf_fine.size() : 1;
    std::vector<std::array<int, 4>> rc(nF, {1 << 30, 1 << 30, -1, -1});
    std::vector<std::vector<int>> fel(nF);
    for (int r = 0; r < nf; ++r) {
      const int e = h_fine[r];
      const int f = sf_fine_ok ? sf_elem_face[e] : 0;
      fel[f].push_back(r);
      if (sf_fine_ok) {
        const int* er = &sf_erect[4 * static_cast<size_t>(e)];
        rc[f][0] = std::min(rc[f][0], er[0]);
        rc[f][1] = std::min(rc[f][1], er[1]);
        rc[f][2] = std::max(rc[f][2], er[2]);
        rc[f][3] = std::max(rc[f][3], er[3]);
      }
    }
    for (size_t f = 0; f < nF; ++f) {
      if (fel[f].empty()) continue;
      const int reg = nreg_static + static_cast<int>(fregs.size());
      std::vector<std::pair<int, int>> as, bs;
      int tile0 = sf_nt_static + static_cast<int>(ftiles.size());
      if (sf_fine_ok) {
        const SfGrid& g = sf_fine[f];
        const int a0 = rc[f][0], b0 = rc[f][1];
        const int na = rc[f][2] - a0 + 1, nb = rc[f][3] - b0 + 1;
        fregs.push_back(box_of(g, a0, na, b0, nb));
        sf_split_tiles(na, nb, as, bs);
        for (const auto& [bb, nbt] : bs)
          for (const auto& [aa, nat] : as)
            ftiles.push_back(SfTile{sf_grid_fine0 + static_cast<int>(f), a0 + aa, b0 + bb, nat,
                                    nbt, reg});
      } else {  // fine points not on grids: all their sources pair-wise
        SfRegion all{};
        for (int ax = 0; ax < 3; ++ax) {
          all.lo[ax] = -1e300;
          all.hi[ax] = 1e300;
        }
        all.npts = -1.0;
        fregs.push_back(all);
      }
      const size_t e0 = fq.size();
      for (int r : fel[f]) {
        const int e = h_fine[r];
        const int o = h_qb_off[e] + extra[r];
        for (int l = h_qf_off[e]; l < h_qf_off[e + 1]; ++l) {
          fq.push_back(tqb + l);
          fpos.push_back(o + (l - h_qf_off[e]));
          if (sf_fine_ok) {
            const int a = sf_h_fa[l] - rc[f][0], b = sf_h_fb[l] - rc[f][1];
            int ia = 0, ib = 0;
            while (ia + 1 < static_cast<int>(as.size()) && a >= as[ia + 1].first) ++ia;
            while (ib + 1 < static_cast<int>(bs.size()) && b >= bs[ib + 1].first) ++ib;
            ftile.push_back(tile0 + ia + static_cast<int>(as.size()) * ib);
            fcell.push_back((a - as[ia].first) + kSfTA * (b - bs[ib].first));
          } else {
            ftile.push_back(-1);
            fcell.push_back(0);
          }
        }
      }
      const size_t n = fq.size() - e0;
      if (sf_fine_ok) {  // compact 2D blocks per K1 CTA, as the static regions
        std::vector<int> ord(n);
        std::iota(ord.begin(), ord.end(), 0);
        auto key = [&](int i) {
          const int l = fq[e0 + i] - tqb;
          return std::make_tuple(sf_h_fa[l] / 48, sf_h_fb[l], sf_h_fa[l]);
        };
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return key(x) < key(y); });
        auto permute = [&](std::vector<int>& v) {
          std::vector<int> tmp(n);
          for (size_t i = 0; i < n; ++i) tmp[i] = v[e0 + ord[i]];
          std::copy(tmp.begin(), tmp.end(), v.begin() + e0);
        };
        permute(fq);
        permute(fpos);
        permute(ftile);
        permute(fcell);
      }
      const size_t pad = (n + sf_k1_ppc - 1) / sf_k1_ppc * sf_k1_ppc;
      for (size_t i = n; i < pad; ++i) {
        fq.push_back(fq[e0]);
        fpos.push_back(-1);
        ftile.push_back(-1);
        fcell.push_back(0);
      }
      for (size_t c = 0; c < pad / sf_k1_ppc; ++c) fcta.push_back(reg);
    }
  }
  const int n_tiles = sf_nt_static + static_cast<int>(ftiles.size());
  const int n_regs = nreg_static + static_cast<int>(fregs.size());
  const int n_ent = sf_ne_static + static_cast<int>(fq.size());
  const int n_cta = sf_nc_static + static_cast<int>(fcta.size());
  // ---- stage + upload the per-step host data (one pinned slot, async)
  {
    const size_t b_fine = flux ? sizeof(int) * (2 * static_cast<size_t>(nf) + 1) : 0;
    const size_t b_t = sizeof(SfTile) * ftiles.size(), b_r = sizeof(SfRegion) * fregs.size();
    const size_t b_e = sizeof(int) * fq.size(), b_c = sizeof(int) * fcta.size();
    char* h = stage_bytes(b_fine + b_t + b_r + 4 * b_e + b_c + 64);
    size_t o = 0;
    auto copy = [&](void* dst, const void* src, size_t bytes) {
      if (!bytes) return;
      std::memcpy(h + o, src, bytes);
      TG_CUDA(cudaMemcpyAsync(dst, h + o, bytes, cudaMemcpyHostToDevice, s));
      o += (bytes + 15) / 16 * 16;
    };
    if (flux) {
      copy(d_fine.p, h_fine.data(), sizeof(int) * nf);
      copy(d_fine.p + n_fe + 1, extra, sizeof(int) * (nf + 1));
    }
    copy(d_sf_tiles.p + sf_nt_static, ftiles.data(), b_t);
    copy(d_sf_regions.p + nreg_static, fregs.data(), b_r);
    copy(d_sf_ent_q.p + sf_ne_static, fq.data(), b_e);
    copy(d_sf_ent_pos.p + sf_ne_static, fpos.data(), b_e);
    copy(d_sf_ent_tile.p + sf_ne_static, ftile.data(), b_e);
    copy(d_sf_ent_cell.p + sf_ne_static, fcell.data(), b_e);
    copy(d_sf_cta.p + sf_nc_static, fcta.data(), b_c);
    TG_CUDA(cudaEventRecord(sf_stage[(sf_stage_i + 2) % 3].done, s));
  }
  // ---- device
  const FaceTables ft{n_fe, ndk, d_qb_off.p, d_qf_off.p, d_Nb.p, d_Nf.p};
  if (flux) {
    k3_point_index(ft, d_fine.p, d_fine.p + n_fe + 1, nf, d_pt_index.p, d_elem_off.p, s);
    sf_base_positions(sf_ne_flux, d_sf_ent_q.p, d_sf_ent_tile.p, d_sf_qelem.p, d_qb_off.p,
                      d_elem_off.p, d_sf_ent_pos.p, s);
    ctx->timer.launches += 2;
  }
  const Material& m = ctx->mat;
  const double alpha = m.diffusivity(), rcp = m.volumetric_capacity();
  const double cull = cfg.superpose.cull_exponent;
  const int n_act = ctx->active_prefix(t);
  SfPlanArgs pa{ctx->src6.p, n_act, t, alpha, cull, sf_min_pairs, sf_min_sources, sf_on};
  SfPlanMask mask{flux, dir, sf_nt_flux, sf_nt_static, sf_rank, sf_world};
  const SfLists lists{d_sf_elist.p, d_sf_okbits.p, d_sf_Jc.p, d_sf_Jcl.p, sf_list_cap,
                      sf_list_words};
  sf_plan(pa, d_sf_regions.p, n_regs, d_sf_J.p, d_sf_E.p, mask, nreg_static, d_sf_Jl.p,
          d_sf_El.p, d_sf_Jraw.p, lists, s);
  sf_items(d_sf_tiles.p, n_tiles, d_sf_Jc.p, d_sf_prefix.p, d_sf_stats.p, s);
  sf_prep(ctx->src6.p, n_act, t, alpha, rcp, d_sf_grids.p, static_cast<int>(sf_grids_h.size()),
          static_cast<int>(sources.size()) + 1, d_sf_cst.p, s);
  const int ctas = sf_contract_max_ctas(ctx->sm_count);
  ctx->timer.timed(5, s, [&] {
    sf_contract_fused(d_sf_grids.p, d_sf_tiles.p, n_tiles, d_sf_prefix.p, d_sf_J.p, lists,
                      d_sf_cst.p, static_cast<int>(sources.size()) + 1, d_sf_tab.p,
                      d_sf_scratch.p, ctas, s);
  });
  ctx->timer.launches += 5;
  // the pair-wise remainder: K1 over every entry with its region's [J, E)
  const int S = sf_k1_splits;
  double* part = ctx->part.ensure(static_cast<size_t>(S) * 4 * n_ent);
  if (n_act > 0) {
    k1_prepare(ctx->src6.p, n_act, t, alpha, rcp, cull, ctx->rec.ensure(n_act), s);
    const bool planar = ctx->planar && !std::getenv("TG_K1_NO_PLANAR");
    K1Ranges rg{d_sf_cta.p, d_sf_J.p, d_sf_E.p, d_sf_okbits.p, sf_list_words};
    ctx->timer.timed(1, s, [&] {
      k1_launch_partial(ctx->rec.p, n_act, d_qx.p, d_sf_ent_q.p, n_ent, S, true, 7, part, s,
                        planar, ctx->planar_z, rg);
    });
    ctx->timer.launches += 2;
    ++ctx->timer.k1_launches;
  } else {
    TG_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * S * 4 * n_ent, s));
  }
  (void)n_cta;
  SfAddArgs aa{};
  aa.ent = SfEntries{d_sf_ent_q.p, d_sf_ent_pos.p, d_sf_ent_tile.p, d_sf_ent_cell.p};
  aa.part = part;
  aa.S = S;
  aa.n_entries = n_ent;
  aa.grids = d_sf_grids.p;
  aa.tiles = d_sf_tiles.p;
  aa.prefix = d_sf_prefix.p;
  aa.n_tiles = n_tiles;
  aa.ctas = ctas;
  aa.scratch = d_sf_scratch.p;
  aa.normals = d_qn.p;
  aa.weights = d_qw.p;
  aa.k = cfg.material.conductivity;
  aa.gq = d_gq.p;
  aa.g = d_g;
  if (flux) {
    sf_add(aa, 0, sf_ne_flux, true, s);
    sf_add(aa, sf_ne_static, n_ent, true, s);
    ctx->timer.launches += 2;
  }
  if (dir) {
    sf_add(aa, sf_ne_flux, sf_ne_static, false, s);
    ++ctx->timer.launches;
  }
  if (flux && gather) {
    k3_local(ft, 0, n_fe, d_elem_off.p, d_gq.p, d_loc.p, s);
    if (d_F) k3_gather(n_full, d_inc_ptr.p, d_inc_src.p, d_loc.p, d_F, s);
    ctx->timer.launches += 2;
  }
  TG_CUDA(cudaGetLastError());
}

void Sim::flux_finish(double* d_F) {
  cudaStream_t s = ctx->stream;
  const FaceTables ft{n_fe, ndk, d_qb_off.p, d_qf_off.p, d_Nb.p, d_Nf.p};
  k3_local(ft, 0, n_fe, d_elem_off.p, d_gq.p, d_loc.p, s);
  k3_gather(n_full, d_inc_ptr.p, d_inc_src.p, d_loc.p, d_F, s);
  ctx->timer.launches += 2;
}

void Sim::flux_load_device(double t, double radius, double* d_F, int e0, int e1) {
  e0 = std::max(0, std::min(e0, n_fe));
  e1 = std::max(e0, std::min(e1, n_fe));
  if (sf_ready && sf_flux_ok && e0 == 0 && e1 == n_fe) {
    loads_device(t, radius, d_F, nullptr, true);
    return;
  }
  // pair-wise K1 over the compact points of elements [e0, e1) (non-gridded
  // patches, and the element-slab range calls)
  cudaStream_t s = ctx->stream;
  const int nf = fine_elements(t, radius);
  int* extra = h_fine.data() + n_fe + 1;
  extra[0] = 0;
  for (int r = 0; r < nf; ++r) {
    const int e = h_fine[r];
    extra[r + 1] = extra[r] + (h_qf_off[e + 1] - h_qf_off[e]) - (h_qb_off[e + 1] - h_qb_off[e]);
  }
  {
    char* h = stage_bytes(sizeof(int) * (2 * static_cast<size_t>(nf) + 1) + 32);
    std::memcpy(h, h_fine.data(), sizeof(int) * nf);
    std::memcpy(h + sizeof(int) * nf, extra, sizeof(int) * (nf + 1));
    if (nf > 0)
      TG_CUDA(cudaMemcpyAsync(d_fine.p, h, sizeof(int) * nf, cudaMemcpyHostToDevice, s));
    TG_CUDA(cudaMemcpyAsync(d_fine.p + n_fe + 1, h + sizeof(int) * nf, sizeof(int) * (nf + 1),
                            cudaMemcpyHostToDevice, s));
    TG_CUDA(cudaEventRecord(sf_stage[(sf_stage_i + 2) % 3].done, s));
  }
  auto offset_of = [&](int e) {
    const int r = static_cast<int>(std::lower_bound(h_fine.begin(), h_fine.begin() + nf, e) -
                                   h_fine.begin());
    return static_cast<long>(h_qb_off[e]) + extra[r];
  };
  const long p0 = offset_of(e0), p1 = e1 == n_fe ? h_qb_off.back() + extra[nf] : offset_of(e1);
  sf_last_npts = h_qb_off.back() + extra[nf];
  const FaceTables ft{n_fe, ndk, d_qb_off.p, d_qf_off.p, d_Nb.p, d_Nf.p};
  k3_point_index(ft, d_fine.p, d_fine.p + n_fe + 1, nf, d_pt_index.p, d_elem_off.p, s);
  ++ctx->timer.launches;
  K1Flux fl{d_pt_index.p + p0, d_qn.p, d_qw.p, cfg.material.conductivity};
  k1_run(ctx, ctx->src6.p, ctx->n_src, d_qx.p, d_pt_index.p + p0, p1 - p0, t,
         cfg.superpose.cull_exponent, K1Mode::flux, d_gq.p + p0, nullptr, fl, s);
  k3_local(ft, e0, e1, d_elem_off.p, d_gq.p, d_loc.p, s);
  ++ctx->timer.launches;
  if (d_F) {
    k3_gather(n_full, d_inc_ptr.p, d_inc_src.p, d_loc.p, d_F, s);
    ++ctx->timer.launches;
  }
  TG_CUDA(cudaGetLastError());
}

void Sim::dirichlet_device(double t, double* d_g, int c0, int c1) {
  // constrained DOFs [c0, c1) (all by default): each value depends on its
  // Greville point only, so a range is the same bits as the full call
  if (c1 < 0) c1 = n_con;
  c0 = std::max(0, std::min(c0, n_con));
  c1 = std::max(c0, std::min(c1, n_con));
  if (sf_ready && sf_dir_ok && c0 == 0 && c1 == n_con) {
    loads_device(t, 0.0, nullptr, d_g, true);
    return;
  }
  k1_run(ctx, ctx->src6.p, ctx->n_src, d_grev.p + 3 * static_cast<size_t>(c0), nullptr, c1 - c0,
         t, cfg.superpose.cull_exponent, K1Mode::dirichlet, d_g, nullptr, {}, ctx->stream);
}

PcgStatus Sim::theta_step_device(double tol, int max_iter) {
  cudaStream_t s = ctx->stream;
  if (!diag_ok) throw numeric_error("pcg: non-positive diagonal, matrix not SPD");
  ctx->timer.timed(3, s, [&] { theta_step_launch(tol, max_iter); });
  TG_CUDA(cudaMemcpyAsync(h_status, d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
  stream_wait(comm.get(), s);
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
        *h_status = fdm_pcg_solve(gfree, coefA[0], coefA[1], fdm, d_rhs.p, d_x.p, w, tol,
                                  max_iter, ctx->sm_count, s, maps.valid ? &maps.x : nullptr,
                                  maps.valid ? &maps.pA : nullptr);
      });
      TG_CUDA(cudaMemcpyAsync(d_status.p, h_status, sizeof(PcgStatus), cudaMemcpyHostToDevice, s));
    } else if (slab) {  // z-slabs (multi-GPU, or the local test bed)
      ctx->timer.timed(2, s, [&] {
        slab->solve(d_rhs.p, d_x.p, coefA[0], coefA[1], tol, max_iter, d_status.p, s);
      });
    } else if (use_res) {
      const K2ResWork w{{d_Ap.p, d_w2.p}, d_r.p, d_partials.p, d_status.p};
      ctx->timer.timed(2, s, [&] {
        k2_res_solve(gfree, coefA[0], coefA[1], d_rhs.p, d_x.p, w, res_plan, tol, max_iter, s);
      });
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
    if (use_fdm) {  // the scaled separable-approximation preconditioner
      const FdmWork w{d_r.p, d_z.p, d_p.p, d_Ap.p, d_p2.p, d_w2.p, d_partials.p, d_dots.p, h_dots};
      ctx->timer.timed(2, s, [&] {
        *h_status = pcg_precond_solve([&](const double* v, double* y) {
          if (use_dia) csr_apply(devAd, v, y, s); else csr_apply(devA, v, y, s); },
                                      fdm, n_free, d_rhs.p, d_x.p, w, tol, max_iter, s);
      });
      TG_CUDA(cudaMemcpyAsync(d_status.p, h_status, sizeof(PcgStatus), cudaMemcpyHostToDevice, s));
    } else {
      const CsrWork w{d_r.p, d_p.p, d_Ap.p, d_invd.p, d_partials.p, d_status.p};
      ctx->timer.timed(2, s, [&] {
        if (use_dia)
          csr_pcg_solve(devAd, d_rhs.p, d_x.p, w, tol, max_iter, pcg_blocks, s);
        else
          csr_pcg_solve(devA, d_rhs.p, d_x.p, w, tol, max_iter, pcg_blocks, s);
      });
    }
  }
  ++ctx->timer.launches;
  ++ctx->timer.k2_launches;
}

void Sim::reset() {
  cudaStream_t s = ctx->stream;
  TG_CUDA(cudaMemsetAsync(d_x.p, 0, sizeof(double) * n_free, s));
  step_loads(0.0, d_Fn.p, d_gn.p);
  step = 0;
  stream_wait(comm.get(), s);
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
  step_loads(t1, d_F1.p, d_g1.p);
  const auto ta = now();
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

void Sim::step_loads(double t, double* d_F, double* d_g) {
  const double r = cfg.mesh.elevate_radius;
  const bool fused = sf_ready && sf_flux_ok && sf_dir_ok;
  if (fused && comm && sf_world > 1) {
    // this rank's regions; the compact integrand and g summed over the ranks
    // (disjoint supports: every entry has one nonzero contributor, so the sum
    // is exact and the same on every rank), then the local loads and gather
    loads_device(t, r, nullptr, d_g, false);
    nccl_allreduce_sum(*comm, d_gq.p, static_cast<size_t>(sf_last_npts), ctx->stream);
    nccl_allreduce_sum(*comm, d_g, static_cast<size_t>(n_con), ctx->stream);
    flux_finish(d_F);
    return;
  }
  if (fused) {  // both loads in one fused pass
    loads_device(t, r, d_F, d_g, true);
    return;
  }
  flux_load_device(t, r, d_F);
  dirichlet_device(t, d_g);
}

void Sim::shard(int rank, int world, const char id[128]) {
  comm = nccl_comm(rank, world, id, ctx->device);
  sf_rank = rank;
  sf_world = world;
  slab.reset();
  if (world > 1 && kron && use_cg1)
    slab = std::make_unique<SlabSolver>(gfree, world, rank, comm, ctx->sm_count, cg1_pl);
}

void Sim::set_slabs(int n) {
  slab.reset();
  if (n > 1) {
    if (!(kron && use_cg1)) throw std::invalid_argument("slabs: needs the single-sweep Kronecker solver");
    slab = std::make_unique<SlabSolver>(gfree, n, 0, nullptr, ctx->sm_count, cg1_pl);
  }
}

// n steps with no host synchronisation between them: every step's loads,
// RHS and solve are enqueued and its PCG status is copied to a pinned slot;
// the statuses are read once at the end. A failing solve raises the
// reference's numeric_error (sparse.cpp:75-99) for the first failing step, as
// run_time_loop would; the state after such a step is unspecified (the
// reference's State is lost with the exception).
long Sim::advance_steps(int n, double* last_rel) {
  static const bool timing = std::getenv("TG_STEP_TIMING") != nullptr;
  long it = 0;
  if (n <= 0) return 0;
  if (use_fdm || timing) {  // host-driven solver / per-phase timing: one step at a time
    PcgStatus st{};
    for (int k = 0; k < n; ++k) {
      st = advance();
      it += st.iterations;
    }
    if (last_rel) *last_rel = st.rel_residual;
    return it;
  }
  if (!diag_ok) throw numeric_error("pcg: non-positive diagonal, matrix not SPD");
  if (static_cast<size_t>(n) > h_steps_cap) {
    if (h_steps) TG_CUDA(cudaFreeHost(h_steps));
    h_steps = nullptr;
    h_steps_cap = 0;
    TG_CUDA(cudaMallocHost(&h_steps, sizeof(PcgStatus) * n));
    h_steps_cap = n;
  }
  cudaStream_t s = ctx->stream;
  const int first = step;
  ctx->timer.timed(4, s, [&] {
  for (int k = 0; k < n; ++k) {
    const double t1 = (step + 1) * dt_solver;  // driver.cpp:127
    step_loads(t1, d_F1.p, d_g1.p);
    ctx->timer.timed(3, s, [&] { theta_step_launch(cfg.stepping.solver_tol, cfg.stepping.max_iter); });
    TG_CUDA(cudaMemcpyAsync(&h_steps[k], d_status.p, sizeof(PcgStatus), cudaMemcpyDeviceToHost, s));
    std::swap(d_Fn.p, d_F1.p);
    std::swap(d_gn.p, d_g1.p);
    ++step;
  }
  });
  stream_wait(comm.get(), s);
  for (int k = 0; k < n; ++k) {
    const PcgStatus& st = h_steps[k];
    it += st.iterations;
    ctx->timer.k2_bytes += 104.0 * n_free * st.iterations;  // SURVEY.md §8d algorithmic bytes
    k2_iterations += st.iterations;
    if (st.status == 4 || st.status == 3) {
      step = first + k + 1;
      if (st.status == 4) throw numeric_error("pcg: indefinite direction, matrix not SPD");
      char buf[64];
      std::snprintf(buf, sizeof(buf), "%.17g", st.rel_residual);
      throw numeric_error("pcg: no convergence in " + std::to_string(cfg.stepping.max_iter) +
                          " iterations, relative residual " + buf);
    }
  }
  if (last_rel) *last_rel = h_steps[n - 1].rel_residual;
  return it;
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
