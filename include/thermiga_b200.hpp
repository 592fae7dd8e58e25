// thermiga_b200.hpp — header-only C++ shim over the C ABI (thermiga_b200.h)
// with the reference's hot-path signatures (proj/include/thermiga/*.hpp), so a
// caller of the reference's run_time_loop can switch the hot path to the B200
// kernels by swapping these calls. C ABI status codes are re-raised as the
// reference's exception types (proj/include/thermiga/core.hpp:66-80).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "thermiga_b200.h"

namespace thermiga_b200 {

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
};

struct config_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct numeric_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// rc first, then the context's message (read only after the call returned)
inline void raise(int rc, const char* msg);
inline void check_ctx(int rc, tg_ctx* c) {
  if (rc != TG_OK) raise(rc, tg_last_error(c));
}

inline void raise(int rc, const char* msg) {
  switch (rc) {
    case TG_OK: return;
    case TG_ECONFIG: throw config_error(msg);
    case TG_EIO: throw io_error(msg);
    case TG_ENUMERIC: throw numeric_error(msg);
    case TG_ECUDA: throw device_error(msg);
    default: throw std::invalid_argument(msg);
  }
}

// analytic.hpp:10-40 (same layouts as the reference's records)
using Material = tg_material;
using LaserSpec = tg_laser;
using PointSource = tg_point_source;
struct ScanPath {
  std::vector<std::array<double, 2>> waypoints;
  double start_time = 0.0;
  double plane_z = 0.0;
};
struct SuperposeOptions {
  double cull_exponent = 60.0;
};
struct AnalyticField {
  double value = 0.0;
  Vec3 grad;
};

// discretize_scan (analytic.hpp:45-48)
inline std::vector<PointSource> discretize_scan(const ScanPath& path, const LaserSpec& laser,
                                                const Material& mat) {
  std::vector<double> wp;
  for (const auto& w : path.waypoints) wp.insert(wp.end(), {w[0], w[1]});
  const int n = tg_discretize_scan(wp.data(), static_cast<int>(path.waypoints.size()),
                                   path.start_time, path.plane_z, &laser, &mat, nullptr, 0);
  if (n < 0) throw std::invalid_argument("discretize_scan: invalid laser, material or path");
  std::vector<PointSource> out(n);
  tg_discretize_scan(wp.data(), static_cast<int>(path.waypoints.size()), path.start_time,
                     path.plane_z, &laser, &mat, out.data(), n);
  return out;
}

// A device context: the scan history resident in HBM plus scratch.
class Device {
 public:
  explicit Device(int device = 0) {
    tg_ctx* c = nullptr;
    const int rc = tg_ctx_create(device, &c);
    ctx_.reset(c);
    if (rc != TG_OK) raise(rc, tg_last_error(c));
  }
  tg_ctx* get() const { return ctx_.get(); }
  void set_sources(const std::vector<PointSource>& s, const Material& m) {
    check_ctx(tg_set_sources(get(), s.data(), static_cast<int>(s.size()), &m), get());
  }
  // superpose (analytic.hpp:73-75) at many points: values and gradients
  void superpose(const std::vector<Vec3>& x, double t, std::vector<AnalyticField>& out,
                 const SuperposeOptions& opts = {}) {
    std::vector<double> v(x.size()), g(3 * x.size());
    check_ctx(tg_superpose_batch(get(), &x[0].x, static_cast<long>(x.size()), t,
                                 opts.cull_exponent, v.data(), g.data()),
              get());
    out.resize(x.size());
    for (size_t i = 0; i < x.size(); ++i) out[i] = {v[i], {g[3 * i], g[3 * i + 1], g[3 * i + 2]}};
  }

 private:
  struct Del {
    void operator()(tg_ctx* c) const { tg_ctx_destroy(c); }
  };
  std::unique_ptr<tg_ctx, Del> ctx_;
};

// superpose for one point (analytic.hpp:73-75); uploads the history each call,
// use Device::superpose for batches.
inline AnalyticField superpose(const std::vector<PointSource>& sources, const Material& mat,
                               const Vec3& x, double t, const SuperposeOptions& opts = {}) {
  thread_local Device dev;
  dev.set_sources(sources, mat);
  std::vector<AnalyticField> out;
  dev.superpose({x}, t, out, opts);
  return out[0];
}

struct PcgOptions {  // sparse.hpp:32-35
  double tol = 1e-10;
  int max_iter = 5000;
};
struct PcgResult {  // sparse.hpp:37-40
  int iterations = 0;
  double rel_residual = 0.0;
};

namespace detail {
inline Device& thread_device() {
  thread_local Device dev;
  return dev;
}
}  // namespace detail

// CsrMatrix (sparse.hpp:14-30): same fields; multiply runs on the GPU.
struct CsrMatrix {
  int rows = 0, cols = 0;
  std::vector<int> row_ptr, col_idx;
  std::vector<double> vals;
  void multiply(const std::vector<double>& x, std::vector<double>& y) const {
    if (static_cast<int>(x.size()) != cols) throw std::invalid_argument("spmv: size mismatch");
    y.resize(rows);
    Device& d = detail::thread_device();
    check_ctx(tg_csr_multiply(d.get(), rows, row_ptr.data(), col_idx.data(), vals.data(),
                              x.data(), y.data()),
              d.get());
  }
};

// pcg_jacobi (sparse.hpp:45-46) on the GPU: x is the warm start and the result.
inline PcgResult pcg_jacobi(const CsrMatrix& A, const std::vector<double>& b,
                            std::vector<double>& x, const PcgOptions& opts = {}) {
  if (A.cols != A.rows || static_cast<int>(b.size()) != A.rows ||
      static_cast<int>(x.size()) != A.rows)
    throw std::invalid_argument("pcg: dimension mismatch");
  Device& d = detail::thread_device();
  PcgResult r;
  check_ctx(tg_pcg_jacobi(d.get(), A.rows, A.row_ptr.data(), A.col_idx.data(), A.vals.data(),
                          b.data(), x.data(), opts.tol, opts.max_iter, &r.iterations,
                          &r.rel_residual),
            d.get());
  return r;
}

// Geometry tooling (config 3; not in the reference): exact degree elevation of
// a geometry file, written in the reference's format.
inline void elevate_geometry(const std::string& in_path, const std::string& out_path,
                             const int elevate[3], const double* scale = nullptr) {
  char err[512] = {0};
  const int rc =
      tg_geometry_elevate(in_path.c_str(), elevate, scale, out_path.c_str(), err, sizeof(err));
  if (rc != TG_OK) raise(rc, err);
}

// postproc.hpp:17-44
struct FluxProfile {
  struct Sample {
    double s, theta, q_tilde, q_hat, q_net;
  };
  std::vector<Sample> samples;
};
struct FluxMetrics {
  double integral_net = 0.0, integral_analytic = 0.0;
  bool has_ratio = false;
  double ratio = 0.0;
};
// integrated_abs_flux (postproc.cpp:81-95)
inline FluxMetrics integrated_abs_flux(const FluxProfile& p) {
  if (p.samples.size() < 2) throw std::invalid_argument("flux metrics need >= 2 samples");
  FluxMetrics m;
  for (size_t i = 1; i < p.samples.size(); ++i) {
    const auto& a = p.samples[i - 1];
    const auto& b = p.samples[i];
    const double ds = b.s - a.s;
    m.integral_net += 0.5 * ds * (std::abs(a.q_net) + std::abs(b.q_net));
    m.integral_analytic += 0.5 * ds * (std::abs(a.q_tilde) + std::abs(b.q_tilde));
  }
  if (m.integral_analytic > 0.0) {
    m.has_ratio = true;
    m.ratio = m.integral_net / m.integral_analytic;
  }
  return m;
}
struct State {  // timestep.hpp:16-21
  std::vector<double> free_coeffs;
  std::vector<double> constrained_values;
  int step = 0;
  double time = 0.0;
};

// prepare_simulation (driver.hpp:49) + the hot-path calls of run_time_loop.
class Simulation {
 public:
  explicit Simulation(const std::string& config_path, tg_sim_options opt = {}) {
    tg_sim* s = nullptr;
    const int rc = tg_sim_create(config_path.c_str(), &opt, &s);
    sim_.reset(s);
    if (rc != TG_OK) raise(rc, tg_sim_last_error(s));
    long info[18];
    check(tg_sim_info(get(), info));
    n_full = info[0];
    n_free = info[1];
    n_constrained = info[2];
    n_steps = static_cast<int>(info[3]);
    double par[10];
    check(tg_sim_params(get(), par));
    dt_solver = par[0];
    tol = par[2];
    max_iter = static_cast<int>(par[9]);
  }
  tg_sim* get() const { return sim_.get(); }

  // assemble_flux_load (assembly.hpp:37-40); fine_radius < 0: config value
  void assemble_flux_load(double t, double fine_radius, std::vector<double>& load) {
    load.resize(n_full);
    check(tg_sim_flux_load(get(), t, nullptr, fine_radius, load.data()));
  }
  // dirichlet_values (mesh.hpp:121-125)
  std::vector<double> dirichlet_values(double t) {
    std::vector<double> g(n_constrained);
    check(tg_sim_dirichlet_values(get(), t, g.data()));
    return g;
  }
  // theta_step (timestep.hpp:26-29)
  State theta_step(const State& s, const std::vector<double>& load_n,
                   const std::vector<double>& load_np1, const std::vector<double>& g_np1,
                   const PcgOptions& o, PcgResult* stats = nullptr) {
    State next;
    next.free_coeffs.resize(n_free);
    int it = 0;
    double rel = 0.0;
    check(tg_sim_theta_step(get(), s.free_coeffs.data(), s.constrained_values.data(),
                            load_n.data(), load_np1.data(), g_np1.data(), o.tol, o.max_iter,
                            next.free_coeffs.data(), &it, &rel));
    if (stats) *stats = {it, rel};
    next.constrained_values = g_np1;
    next.step = s.step + 1;
    next.time = next.step * dt_solver;
    return next;
  }
  // run_time_loop (driver.hpp:45-47) with the state resident on the device;
  // on_state sees the state after every step (and once with the initial one).
  long run_time_loop(const std::function<void(const State&)>& on_state) {
    check(tg_sim_reset(get()));
    State st;
    pull(st);
    on_state(st);
    long total = 0;
    for (int s = 1; s <= n_steps; ++s) {
      long it = 0;
      check(tg_sim_advance(get(), 1, &it, nullptr));
      total += it;
      pull(st);
      on_state(st);
    }
    return total;
  }

  // observers on the current device state (postproc.cpp:9-79):
  // total_temperature at parametric points, boundary_flux_profile of a face
  std::vector<double> total_temperature(const std::vector<Vec3>& xi) {
    std::vector<double> out(12 * xi.size()), T(xi.size());
    if (!xi.empty()) check(tg_sim_probe(get(), &xi[0].x, static_cast<long>(xi.size()), out.data()));
    for (size_t i = 0; i < xi.size(); ++i) T[i] = out[12 * i + 3];
    return T;
  }
  FluxProfile boundary_flux_profile(int face, int n_samples, const double* theta_axis = nullptr,
                                    double edge_v = 1.0) {
    std::vector<double> rows(5 * static_cast<size_t>(std::max(0, n_samples)));
    check(tg_sim_flux_profile(get(), face, n_samples, edge_v, theta_axis, rows.data()));
    FluxProfile p;
    for (int i = 0; i < n_samples; ++i)
      p.samples.push_back({rows[5 * i], rows[5 * i + 1], rows[5 * i + 2], rows[5 * i + 3],
                           rows[5 * i + 4]});
    return p;
  }

  // DirichletSystem::reduced_operator() (assembly.hpp:56) of a non-separable
  // patch, as the reference's CsrMatrix (bit-identical values)
  CsrMatrix reduced_operator() {
    int rows = 0;
    const long nnz = tg_sim_reduced_operator(get(), &rows, nullptr, nullptr, nullptr);
    if (nnz < 0) raise(static_cast<int>(-nnz), tg_sim_last_error(get()));
    CsrMatrix A;
    A.rows = A.cols = rows;
    A.row_ptr.resize(rows + 1);
    A.col_idx.resize(nnz);
    A.vals.resize(nnz);
    tg_sim_reduced_operator(get(), nullptr, A.row_ptr.data(), A.col_idx.data(), A.vals.data());
    return A;
  }

  // the discretized history and material the simulation's config defines
  std::vector<PointSource> sources() const {
    long info[18];
    raise(tg_sim_info(get(), info), tg_sim_last_error(get()));
    std::vector<PointSource> out(info[4]);
    raise(tg_sim_sources(get(), out.data(), static_cast<int>(out.size())),
          tg_sim_last_error(get()));
    return out;
  }
  Material material() const {
    double par[10];
    raise(tg_sim_params(get(), par), tg_sim_last_error(get()));
    Material m{};
    m.conductivity = par[5];
    m.density = par[6];
    m.heat_capacity = par[7];
    m.platform_temperature = par[8];
    return m;
  }
  SuperposeOptions superpose_options() const {
    double par[10];
    raise(tg_sim_params(get(), par), tg_sim_last_error(get()));
    return SuperposeOptions{par[4]};
  }

  long n_full = 0, n_free = 0, n_constrained = 0;
  int n_steps = 0, max_iter = 5000;
  double dt_solver = 0.0, tol = 1e-10;

 private:
  void check(int rc) { raise(rc, tg_sim_last_error(get())); }
  void pull(State& st) {
    st.free_coeffs.resize(n_free);
    st.constrained_values.resize(n_constrained);
    check(tg_sim_state(get(), &st.step, &st.time, st.free_coeffs.data(),
                       st.constrained_values.data(), nullptr));
  }
  struct Del {
    void operator()(tg_sim* s) const { tg_sim_destroy(s); }
  };
  std::unique_ptr<tg_sim, Del> sim_;
};

// ---- the reference's free-function hot path (assembly.hpp:37-40,
// mesh.hpp:121-125, timestep.hpp:26-29) over the simulation's device data:
// BoundarySets stands for its lateral face quadrature sets, DirichletSystem
// for its θ-scheme operator. The history is the one the simulation's config
// discretized (it is resident in HBM); sources / mat / opts are checked
// against it rather than re-uploaded.
struct BoundarySets {
  Simulation* sim;
};
struct DirichletSystem {
  Simulation* sim;
};
inline BoundarySets boundary_sets(Simulation& s) { return {&s}; }
inline DirichletSystem dirichlet_system(Simulation& s) { return {&s}; }

namespace detail {
inline void same_history(const Simulation& s, const std::vector<PointSource>& src,
                         const Material& mat, const SuperposeOptions& opts) {
  long info[18];
  raise(tg_sim_info(s.get(), info), tg_sim_last_error(s.get()));
  double par[10];
  raise(tg_sim_params(s.get(), par), tg_sim_last_error(s.get()));
  if (static_cast<long>(src.size()) != info[4] || mat.conductivity != par[5] ||
      mat.density != par[6] || mat.heat_capacity != par[7] || opts.cull_exponent != par[4])
    throw std::invalid_argument(
        "sources / material / options differ from the simulation's (resident on the device)");
}
}  // namespace detail

// assemble_flux_load (assembly.hpp:37-40); the fine rule follows the newest
// source active at t; n_threads is accepted and ignored (core.cpp:67-85)
inline void assemble_flux_load(const BoundarySets& b, const std::vector<PointSource>& sources,
                               const Material& mat, double t, double fine_radius,
                               std::vector<double>& load, const SuperposeOptions& opts = {},
                               int n_threads = 1) {
  (void)n_threads;
  detail::same_history(*b.sim, sources, mat, opts);
  b.sim->assemble_flux_load(t, fine_radius, load);
}
// dirichlet_values (mesh.hpp:121-125)
inline std::vector<double> dirichlet_values(const BoundarySets& b,
                                            const std::vector<PointSource>& sources,
                                            const Material& mat, double t,
                                            const SuperposeOptions& opts = {}) {
  detail::same_history(*b.sim, sources, mat, opts);
  return b.sim->dirichlet_values(t);
}
// theta_step (timestep.hpp:26-29)
inline State theta_step(const DirichletSystem& sys, const State& s,
                        const std::vector<double>& load_n, const std::vector<double>& load_np1,
                        const std::vector<double>& constrained_np1, const PcgOptions& o,
                        PcgResult* stats = nullptr) {
  return sys.sim->theta_step(s, load_n, load_np1, constrained_np1, o, stats);
}

}  // namespace thermiga_b200
