// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" harness over the UNMODIFIED reference library (thermiga), compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libthermiga_ref.so. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, and only as the
// checker or the CPU baseline. Every entry point calls the reference's own
// public API (proj/include/thermiga/*.hpp); nothing here re-implements the
// reference's arithmetic.

#include <chrono>
#include <cmath>
#include <optional>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "thermiga/assembly.hpp"
#include "thermiga/config.hpp"
#include "thermiga/driver.hpp"
#include "thermiga/mesh.hpp"
#include "thermiga/postproc.hpp"
#include "thermiga/sparse.hpp"
#include "thermiga/timestep.hpp"

using namespace thermiga;

namespace {

void put_err(char* err, int len, const std::string& msg) {
  if (err && len > 0) {
    std::snprintf(err, static_cast<size_t>(len), "%s", msg.c_str());
  }
}

Material make_mat(double k, double rho, double c) {
  Material m;
  m.conductivity = k;
  m.density = rho;
  m.heat_capacity = c;
  m.platform_temperature = 0.0;
  return m;
}

std::vector<PointSource> unpack_sources(const double* s6, int n) {
  std::vector<PointSource> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    v[i].position = {s6[6 * i + 0], s6[6 * i + 1], s6[6 * i + 2]};
    v[i].energy = s6[6 * i + 3];
    v[i].t_activate = s6[6 * i + 4];
    v[i].tau = s6[6 * i + 5];
  }
  return v;
}

// Reference run state: prepare_simulation + the pieces of run_time_loop
// (proj/src/driver.cpp:105-146), stepped one θ-step at a time so that every
// intermediate (F_n, g_n, free coefficients, CG iterations) can be dumped.
struct RefSim {
  Simulation sim;
  std::unique_ptr<DirichletSystem> dsys;
  State state;
  std::vector<double> load_n, load_np1;
  int step = 0;
};

}  // namespace

extern "C" {

int ref_abi_version() { return 3; }

// discretize_scan (proj/src/analytic.cpp:22-71). Returns the source count or
// -1 on error; writes at most max_out sources as {x,y,z,E,t_act,tau}.
int ref_discretize_scan(const double* wp, int n_wp, double start_time, double plane_z,
                        double power, double speed, double spot_radius, double absorptivity,
                        double laser_dt, double k, double rho, double c, double* out6,
                        int max_out, char* err, int errlen) {
  try {
    ScanPath path;
    for (int i = 0; i < n_wp; ++i) path.waypoints.push_back({wp[2 * i], wp[2 * i + 1]});
    path.start_time = start_time;
    path.plane_z = plane_z;
    LaserSpec laser{power, speed, spot_radius, absorptivity, laser_dt};
    const auto src = discretize_scan(path, laser, make_mat(k, rho, c));
    const int n = static_cast<int>(src.size());
    for (int i = 0; i < n && i < max_out; ++i) {
      out6[6 * i + 0] = src[i].position.x;
      out6[6 * i + 1] = src[i].position.y;
      out6[6 * i + 2] = src[i].position.z;
      out6[6 * i + 3] = src[i].energy;
      out6[6 * i + 4] = src[i].t_activate;
      out6[6 * i + 5] = src[i].tau;
    }
    return n;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return -1;
  }
}

// superpose (proj/src/analytic.cpp:92-109) at every point, threaded over
// points with the reference's own parallel_for (proj/src/core.cpp:67-85).
// grad may be null. Returns elapsed seconds.
double ref_superpose_batch(const double* src6, int n_src, double k, double rho, double c,
                           const double* pts, long n_pts, double t, double cull, double* val,
                           double* grad, int n_threads) {
  const auto sources = unpack_sources(src6, n_src);
  const Material mat = make_mat(k, rho, c);
  SuperposeOptions opts;
  opts.cull_exponent = cull;
  const auto t0 = std::chrono::steady_clock::now();
  parallel_for(static_cast<size_t>(n_pts), n_threads, [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      const Vec3 x{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
      const AnalyticField f = superpose(sources, mat, x, t, opts);
      val[i] = f.value;
      if (grad) {
        grad[3 * i] = f.grad.x;
        grad[3 * i + 1] = f.grad.y;
        grad[3 * i + 2] = f.grad.z;
      }
    }
  });
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// temp_point_source / grad_point_source (proj/src/analytic.cpp:73-90).
void ref_point_source(const double* s6, double k, double rho, double c, const double* x,
                      double t, double* out4) {
  const auto src = unpack_sources(s6, 1);
  const Material mat = make_mat(k, rho, c);
  const Vec3 p{x[0], x[1], x[2]};
  out4[0] = temp_point_source(src[0], mat, p, t);
  const Vec3 g = grad_point_source(src[0], mat, p, t);
  out4[1] = g.x;
  out4[2] = g.y;
  out4[3] = g.z;
}

// gauss_rule (proj/src/core.cpp:57-65).
void ref_gauss_rule(int n, double* nodes, double* weights) {
  const GaussRule& g = gauss_rule(n);
  for (int i = 0; i < n; ++i) {
    nodes[i] = g.nodes[i];
    weights[i] = g.weights[i];
  }
}

// --- simulation handle --------------------------------------------------

void* ref_sim_open(const char* cfg_path, int n_threads, double t_end_override,
                   double solver_tol_override, char* err, int errlen) {
  try {
    RunConfig cfg = parse_config(cfg_path);
    if (t_end_override > 0.0) cfg.stepping.t_end = t_end_override;
    if (solver_tol_override > 0.0) cfg.stepping.solver_tol = solver_tol_override;
    auto* rs = new RefSim{prepare_simulation(std::move(cfg), n_threads), nullptr, {}, {}, {}, 0};
    return rs;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

void ref_sim_close(void* h) { delete static_cast<RefSim*>(h); }

// out[0..]: n_full, n_free, n_constrained, n_steps, n_sources, n_lateral_face_elems,
// nx, ny, nz (basis counts), px, py, pz (degrees), n_elements, threads
int ref_sim_info(void* h, long* out) {
  auto* rs = static_cast<RefSim*>(h);
  const Simulation& s = rs->sim;
  long n_fe = 0;
  for (const auto& f : s.boundary.lateral) n_fe += static_cast<long>(f.elements.size());
  const auto n = s.volume().basis_counts();
  const auto p = s.volume().degrees();
  const long vals[] = {s.mesh.n_functions(), s.dofs.n_free(), s.dofs.n_constrained(),
                       s.n_steps, static_cast<long>(s.sources.size()), n_fe,
                       n[0], n[1], n[2], p[0], p[1], p[2], s.mesh.n_elements(), s.threads};
  std::memcpy(out, vals, sizeof(vals));
  return static_cast<int>(sizeof(vals) / sizeof(long));
}

// out: dt_solver, theta, solver_tol, elevate_radius, cull, k, rho, c, T_c
void ref_sim_params(void* h, double* out) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  out[0] = s.dt_solver;
  out[1] = s.cfg.stepping.theta;
  out[2] = s.cfg.stepping.solver_tol;
  out[3] = s.cfg.mesh.elevate_radius;
  out[4] = s.cfg.superpose.cull_exponent;
  out[5] = s.cfg.material.conductivity;
  out[6] = s.cfg.material.density;
  out[7] = s.cfg.material.heat_capacity;
  out[8] = s.cfg.material.platform_temperature;
}

int ref_sim_sources(void* h, double* out6) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  for (size_t i = 0; i < s.sources.size(); ++i) {
    out6[6 * i + 0] = s.sources[i].position.x;
    out6[6 * i + 1] = s.sources[i].position.y;
    out6[6 * i + 2] = s.sources[i].position.z;
    out6[6 * i + 3] = s.sources[i].energy;
    out6[6 * i + 4] = s.sources[i].t_activate;
    out6[6 * i + 5] = s.sources[i].tau;
  }
  return static_cast<int>(s.sources.size());
}

// Lateral face quadrature sets (proj/src/mesh.cpp:158-236), flattened in
// (face, element, q) order; the rule sizes differ between faces when the
// degrees differ per direction, so per-element counts are exported too.
// counts: [n_fe, total base qps, total fine qps, n_dofs_per_fe].
// With centers == null only counts are returned.
int ref_sim_face_sets(void* h, long* counts, int* nq_base, int* nq_fine, double* centers,
                      int* dofs, double* xb, double* nb, double* wb, double* Nb, double* xf,
                      double* nf, double* wf, double* Nf) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  long n_fe = 0, tqb = 0, tqf = 0, nd = 0;
  for (const auto& f : s.boundary.lateral)
    for (const auto& fe : f.elements) {
      ++n_fe;
      tqb += static_cast<long>(fe.qp_base.size());
      tqf += static_cast<long>(fe.qp_fine.size());
      nd = static_cast<long>(fe.dofs.size());
    }
  counts[0] = n_fe;
  counts[1] = tqb;
  counts[2] = tqf;
  counts[3] = nd;
  if (!centers) return 0;
  long e = 0, ob = 0, of = 0;
  auto put = [nd](const FaceQuadPoint& qp, const double* N, long o, double* x, double* n,
                  double* w, double* NN) {
    x[3 * o] = qp.x.x; x[3 * o + 1] = qp.x.y; x[3 * o + 2] = qp.x.z;
    n[3 * o] = qp.normal.x; n[3 * o + 1] = qp.normal.y; n[3 * o + 2] = qp.normal.z;
    w[o] = qp.weight;
    for (long a = 0; a < nd; ++a) NN[o * nd + a] = N[a];
  };
  for (const auto& f : s.boundary.lateral)
    for (const auto& fe : f.elements) {
      centers[3 * e] = fe.center.x;
      centers[3 * e + 1] = fe.center.y;
      centers[3 * e + 2] = fe.center.z;
      for (long a = 0; a < nd; ++a) dofs[e * nd + a] = fe.dofs[a];
      nq_base[e] = static_cast<int>(fe.qp_base.size());
      nq_fine[e] = static_cast<int>(fe.qp_fine.size());
      for (size_t q = 0; q < fe.qp_base.size(); ++q, ++ob)
        put(fe.qp_base[q], &fe.N_base[q * nd], ob, xb, nb, wb, Nb);
      for (size_t q = 0; q < fe.qp_fine.size(); ++q, ++of)
        put(fe.qp_fine[q], &fe.N_fine[q * nd], of, xf, nf, wf, Nf);
      ++e;
    }
  return 0;
}

// Physical Greville points of the constrained DOFs, in constrained order, as
// dirichlet_values (proj/src/mesh.cpp:238-264) evaluates them.
int ref_sim_greville_points(void* h, double* out3) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  const NurbsVolume& vol = s.volume();
  const FaceId bottom = s.cfg.tags.bottom_face();
  const auto tang = face_tangent_axes(bottom);
  const auto g0 = vol.knots(tang[0]).greville();
  const auto g1 = vol.knots(tang[1]).greville();
  const auto n = vol.basis_counts();
  for (int c = 0; c < s.dofs.n_constrained(); ++c) {
    const int g = s.dofs.constrained_list[c];
    const std::array<int, 3> ijk{g % n[0], (g / n[0]) % n[1], g / (n[0] * n[1])};
    const Vec3 x = vol.map_point(face_param(bottom, g0[ijk[tang[0]]], g1[ijk[tang[1]]])).x;
    out3[3 * c] = x.x;
    out3[3 * c + 1] = x.y;
    out3[3 * c + 2] = x.z;
  }
  return s.dofs.n_constrained();
}

// Knot vectors of the refined patch (normalized), per direction.
int ref_sim_knots(void* h, int dir, double* out) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  const auto& v = s.volume().knots(dir).values();
  if (out)
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  return static_cast<int>(v.size());
}

// assemble_flux_load (proj/src/assembly.cpp:148-166) at time t.
int ref_sim_flux_load(void* h, double t, double* F, int n_threads) {
  auto* rs = static_cast<RefSim*>(h);
  const Simulation& s = rs->sim;
  std::vector<double> load(s.mesh.n_functions());
  assemble_flux_load(s.boundary, s.sources, s.cfg.material, t, s.cfg.mesh.elevate_radius, load,
                     s.cfg.superpose, n_threads);
  std::memcpy(F, load.data(), load.size() * sizeof(double));
  return 0;
}

// assemble_flux_load with an explicit fine radius (0 = base rule only).
int ref_sim_flux_load_radius(void* h, double t, double radius, double* F) {
  auto* rs = static_cast<RefSim*>(h);
  const Simulation& s = rs->sim;
  std::vector<double> load(s.mesh.n_functions());
  assemble_flux_load(s.boundary, s.sources, s.cfg.material, t, radius, load, s.cfg.superpose, 1);
  std::memcpy(F, load.data(), load.size() * sizeof(double));
  return 0;
}

// dirichlet_values (proj/src/mesh.cpp:238-264) at time t.
int ref_sim_dirichlet(void* h, double t, double* g) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  const auto v = dirichlet_values(s.volume(), s.dofs, s.cfg.tags, s.sources, s.cfg.material, t,
                                  s.cfg.superpose);
  std::memcpy(g, v.data(), v.size() * sizeof(double));
  return 0;
}

// CSR export: which = 0 mass, 1 stiffness, 2 reduced operator A_ff.
// Pass null arrays to query nnz (returned) and rows (*rows).
long ref_sim_csr(void* h, int which, int* rows, int* row_ptr, int* col, double* val) {
  auto* rs = static_cast<RefSim*>(h);
  Simulation& s = rs->sim;
  if (which == 2 && !rs->dsys)
    rs->dsys = std::make_unique<DirichletSystem>(s.matrices, s.dofs, s.cfg.stepping.theta,
                                                 s.dt_solver);
  const CsrMatrix& m = which == 0   ? s.matrices.mass
                       : which == 1 ? s.matrices.stiffness
                                    : rs->dsys->reduced_operator();
  *rows = m.rows;
  if (row_ptr) {
    std::memcpy(row_ptr, m.row_ptr.data(), m.row_ptr.size() * sizeof(int));
    std::memcpy(col, m.col_idx.data(), m.col_idx.size() * sizeof(int));
    std::memcpy(val, m.vals.data(), m.vals.size() * sizeof(double));
  }
  return m.nnz();
}

// Initial state of run_time_loop (proj/src/driver.cpp:126-142): g_0 and F_0.
int ref_sim_reset(void* h, double* F0, double* g0, char* err, int errlen) {
  auto* rs = static_cast<RefSim*>(h);
  try {
    Simulation& s = rs->sim;
    const RunConfig& cfg = s.cfg;
    rs->dsys = std::make_unique<DirichletSystem>(s.matrices, s.dofs, cfg.stepping.theta,
                                                 s.dt_solver);
    rs->state = State{};
    rs->state.free_coeffs.assign(s.dofs.n_free(), 0.0);
    rs->state.constrained_values = dirichlet_values(s.volume(), s.dofs, cfg.tags, s.sources,
                                                    cfg.material, 0.0, cfg.superpose);
    const int n_full = s.mesh.n_functions();
    rs->load_n.assign(n_full, 0.0);
    rs->load_np1.assign(n_full, 0.0);
    assemble_flux_load(s.boundary, s.sources, cfg.material, 0.0, cfg.mesh.elevate_radius,
                       rs->load_n, cfg.superpose, s.threads);
    rs->step = 0;
    if (F0) std::memcpy(F0, rs->load_n.data(), n_full * sizeof(double));
    if (g0)
      std::memcpy(g0, rs->state.constrained_values.data(),
                  rs->state.constrained_values.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// One iteration of the run_time_loop body (proj/src/driver.cpp:145-164).
int ref_sim_step(void* h, double* F_np1, double* g_np1, double* free_out, int* iters,
                 double* rel, char* err, int errlen) {
  auto* rs = static_cast<RefSim*>(h);
  try {
    Simulation& s = rs->sim;
    const RunConfig& cfg = s.cfg;
    const int step = rs->step + 1;
    const double t1 = step * s.dt_solver;
    assemble_flux_load(s.boundary, s.sources, cfg.material, t1, cfg.mesh.elevate_radius,
                       rs->load_np1, cfg.superpose, s.threads);
    const std::vector<double> g1 = dirichlet_values(s.volume(), s.dofs, cfg.tags, s.sources,
                                                    cfg.material, t1, cfg.superpose);
    const PcgOptions pcg{cfg.stepping.solver_tol, cfg.stepping.max_iter};
    PcgResult res;
    rs->state = theta_step(*rs->dsys, rs->state, rs->load_n, rs->load_np1, g1, pcg, &res);
    if (F_np1) std::memcpy(F_np1, rs->load_np1.data(), rs->load_np1.size() * sizeof(double));
    if (g_np1) std::memcpy(g_np1, g1.data(), g1.size() * sizeof(double));
    if (free_out)
      std::memcpy(free_out, rs->state.free_coeffs.data(),
                  rs->state.free_coeffs.size() * sizeof(double));
    if (iters) *iters = res.iterations;
    if (rel) *rel = res.rel_residual;
    std::swap(rs->load_n, rs->load_np1);
    rs->step = step;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// theta_step (proj/src/timestep.cpp:5-24) alone, on caller-given inputs.
int ref_sim_theta_step(void* h, const double* free_n, const double* g_n, const double* F_n,
                       const double* F_np1, const double* g_np1, double tol, int max_iter,
                       double* free_out, int* iters, double* rel, char* err, int errlen) {
  auto* rs = static_cast<RefSim*>(h);
  try {
    Simulation& s = rs->sim;
    if (!rs->dsys)
      rs->dsys = std::make_unique<DirichletSystem>(s.matrices, s.dofs, s.cfg.stepping.theta,
                                                   s.dt_solver);
    const int nf = s.dofs.n_free(), nc = s.dofs.n_constrained(), n = s.mesh.n_functions();
    State st;
    st.free_coeffs.assign(free_n, free_n + nf);
    st.constrained_values.assign(g_n, g_n + nc);
    PcgResult res;
    const State out = theta_step(*rs->dsys, st, std::span<const double>(F_n, n),
                                 std::span<const double>(F_np1, n),
                                 std::span<const double>(g_np1, nc), {tol, max_iter}, &res);
    std::memcpy(free_out, out.free_coeffs.data(), nf * sizeof(double));
    if (iters) *iters = res.iterations;
    if (rel) *rel = res.rel_residual;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// field_at (proj/src/splines.cpp:280-303) of a full coefficient vector.
int ref_sim_field_at(void* h, const double* full, const double* xi, double* out4) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  const auto f = s.volume().field_at(std::span<const double>(full, s.mesh.n_functions()),
                                     Vec3{xi[0], xi[1], xi[2]});
  out4[0] = f.value;
  out4[1] = f.grad.x;
  out4[2] = f.grad.y;
  out4[3] = f.grad.z;
  return 0;
}

// total_temperature (proj/src/postproc.cpp:9-19) at t with caller coefficients.
int ref_sim_total_temperature(void* h, const double* full, const double* xi, double t,
                              double* out, char* err, int errlen) {
  try {
    const Simulation& s = static_cast<RefSim*>(h)->sim;
    *out = total_temperature(s.volume(), std::span<const double>(full, s.mesh.n_functions()),
                             s.sources, s.cfg.material, Vec3{xi[0], xi[1], xi[2]}, t,
                             s.cfg.superpose);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// boundary_flux_profile (postproc.cpp:21-79) + integrated_abs_flux (:81-95):
// out (n x 5) = s, theta, q_tilde, q_hat, q_net; metrics[3] = integral_net,
// integral_analytic, ratio (NaN when absent).
int ref_sim_flux_profile(void* h, const double* full, int face, int n, double t,
                         const double* theta_axis, double edge_v, double* out, double* metrics,
                         char* err, int errlen) {
  try {
    const Simulation& s = static_cast<RefSim*>(h)->sim;
    std::optional<std::array<double, 2>> ax;
    if (theta_axis) ax = std::array<double, 2>{theta_axis[0], theta_axis[1]};
    const FluxProfile p = boundary_flux_profile(
        s.volume(), std::span<const double>(full, s.mesh.n_functions()), s.sources,
        s.cfg.material, static_cast<FaceId>(face), n, t, ax, edge_v, s.cfg.superpose);
    for (int i = 0; i < n; ++i) {
      const auto& q = p.samples[i];
      const double row[5] = {q.s, q.theta, q.q_tilde, q.q_hat, q.q_net};
      std::memcpy(out + 5 * i, row, sizeof(row));
    }
    const FluxMetrics m = integrated_abs_flux(p);
    metrics[0] = m.integral_net;
    metrics[1] = m.integral_analytic;
    metrics[2] = m.ratio ? *m.ratio : std::nan("");
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// export_field (postproc.cpp:101-147) and export_profile_csv (:149-159) to a path.
int ref_sim_export_field(void* h, const double* full, const int* dims, double t,
                         const char* path, char* err, int errlen) {
  try {
    const Simulation& s = static_cast<RefSim*>(h)->sim;
    export_field(s.volume(), std::span<const double>(full, s.mesh.n_functions()), s.sources,
                 s.cfg.material, {dims[0], dims[1], dims[2]}, t, path, s.cfg.superpose);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

int ref_export_profile_csv(const double* rows, int n, const char* path, char* err, int errlen) {
  try {
    FluxProfile p;
    for (int i = 0; i < n; ++i)
      p.samples.push_back({rows[5 * i], rows[5 * i + 1], rows[5 * i + 2], rows[5 * i + 3],
                           rows[5 * i + 4]});
    export_profile_csv(p, path);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// face_point (proj/src/splines.cpp:305-321): out = x (3), normal (3), area scale.
int ref_sim_face_point(void* h, int face, double u, double v, double* out) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  const auto sp = s.volume().face_point(static_cast<FaceId>(face), u, v);
  const double o[7] = {sp.x.x, sp.x.y, sp.x.z, sp.normal.x, sp.normal.y, sp.normal.z,
                       sp.area_scale};
  std::memcpy(out, o, sizeof(o));
  return 0;
}

// face_point at n (u, v) pairs: out (n x 7).
int ref_sim_face_points(void* h, int face, int n, const double* uv, double* out) {
  for (int i = 0; i < n; ++i) ref_sim_face_point(h, face, uv[2 * i], uv[2 * i + 1], out + 7 * i);
  return 0;
}

// map_point (proj/src/splines.cpp:257-278).
int ref_sim_map_point(void* h, const double* xi, double* x) {
  const Simulation& s = static_cast<RefSim*>(h)->sim;
  const auto pm = s.volume().map_point(Vec3{xi[0], xi[1], xi[2]});
  x[0] = pm.x.x;
  x[1] = pm.x.y;
  x[2] = pm.x.z;
  return 0;
}

// pcg_jacobi (proj/src/sparse.cpp:41-100) on a caller CSR matrix.
int ref_pcg_csr(int n, const int* rp, const int* ci, const double* v, const double* b, double* x,
                double tol, int max_iter, int* iters, double* rel, char* err, int errlen) {
  try {
    CsrMatrix A;
    A.rows = A.cols = n;
    A.row_ptr.assign(rp, rp + n + 1);
    A.col_idx.assign(ci, ci + rp[n]);
    A.vals.assign(v, v + rp[n]);
    const PcgResult r =
        pcg_jacobi(A, std::span<const double>(b, n), std::span<double>(x, n), {tol, max_iter});
    if (iters) *iters = r.iterations;
    if (rel) *rel = r.rel_residual;
    return 0;
  } catch (const numeric_error& e) {
    put_err(err, errlen, e.what());
    return 3;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// Full run_time_loop (proj/src/driver.cpp:105-146) for CPU timing. timings:
// [time_assembly, time_loads, time_solve, cg_iterations, n_steps, wall].
int ref_sim_run(void* h, int n_steps, double* timings, char* err, int errlen) {
  auto* rs = static_cast<RefSim*>(h);
  try {
    Simulation& s = rs->sim;
    if (n_steps > 0) s.n_steps = n_steps;
    s.time_loads = s.time_solve = 0.0;
    s.cg_iterations = 0;
    const auto t0 = std::chrono::steady_clock::now();
    run_time_loop(s, [](const State&, const std::vector<double>&) {});
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    timings[0] = s.time_assembly;
    timings[1] = s.time_loads;
    timings[2] = s.time_solve;
    timings[3] = static_cast<double>(s.cg_iterations);
    timings[4] = s.n_steps;
    timings[5] = wall;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

}  // extern "C"
