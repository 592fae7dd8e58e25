// C ABI of the simulation engine: tg_sim_* (include/thermiga_b200.h).
#include <cstring>
#include <fstream>

#include "host/config.hpp"
#include "host/fdm.hpp"
#include "sim.hpp"

using namespace tgb;

namespace {

template <typename F>
int sim_guard(tg_sim* s, F&& body, bool needs_device = true) {
  try {
    if (!s || !s->sim) throw std::invalid_argument("null simulation handle");
    if (needs_device) {
      if (!s->sim->ctx) throw cuda_error("cuda: host-only simulation has no device context");
      TG_CUDA(cudaSetDevice(s->sim->ctx->device));
    }
    body(*s->sim);
    return TG_OK;
  } catch (const config_error& e) {
    if (s) s->err = e.what();
    return TG_ECONFIG;
  } catch (const io_error& e) {
    if (s) s->err = e.what();
    return TG_EIO;
  } catch (const numeric_error& e) {
    if (s) s->err = e.what();
    return TG_ENUMERIC;
  } catch (const cuda_error& e) {
    if (s) s->err = e.what();
    return TG_ECUDA;
  } catch (const std::exception& e) {
    if (s) s->err = e.what();
    return TG_ERROR;
  }
}

void d2h(double* h, const double* d, size_t n, cudaStream_t s) {
  if (h && n) TG_CUDA(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, s));
}
void h2d(double* d, const double* h, size_t n, cudaStream_t s) {
  if (n) TG_CUDA(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, s));
}

}  // namespace

extern "C" {

int tg_sim_create(const char* config_path, const tg_sim_options* opt, tg_sim** out) {
  if (!out) return TG_ERROR;
  auto* h = new tg_sim();
  *out = h;
  try {
    SimOptions o;
    if (opt) {
      o.t_end = opt->t_end;
      o.solver_tol = opt->solver_tol;
      o.max_iter = opt->max_iter;
      o.device = opt->device;
      o.host_only = opt->host_only != 0;
      o.preconditioner = opt->preconditioner;
    }
    h->sim = new Sim(config_path ? config_path : "", o);
    return TG_OK;
  } catch (const config_error& e) {
    h->err = e.what();
    return TG_ECONFIG;
  } catch (const io_error& e) {
    h->err = e.what();
    return TG_EIO;
  } catch (const numeric_error& e) {
    h->err = e.what();
    return TG_ENUMERIC;
  } catch (const cuda_error& e) {
    h->err = e.what();
    return TG_ECUDA;
  } catch (const std::exception& e) {
    h->err = e.what();
    return TG_ERROR;
  }
}

void tg_sim_destroy(tg_sim* s) {
  if (!s) return;
  delete s->sim;
  delete s;
}

const char* tg_sim_last_error(const tg_sim* s) { return s ? s->err.c_str() : "null simulation"; }

int tg_sim_kron_factors(tg_sim* s, int dir, double* M, double* K) {
  return sim_guard(s, [&](Sim& m) {
    if (!m.kron) throw std::invalid_argument("patch is not separable: no Kronecker factors");
    if (dir < 0 || dir > 2) throw std::invalid_argument("dir must be 0, 1 or 2");
    std::memcpy(M, m.band[dir].M.data(), m.band[dir].M.size() * sizeof(double));
    std::memcpy(K, m.band[dir].K.data(), m.band[dir].K.size() * sizeof(double));
  }, false);
}

long tg_sim_reduced_operator(tg_sim* s, int* rows, int* row_ptr, int* col, double* val) {
  long nnz = -TG_ERROR;
  const int rc = sim_guard(s, [&](Sim& m) {
    if (m.kron) throw std::invalid_argument("separable patch: the operator is not assembled");
    const Csr& A = m.reduced_operator();
    if (rows) *rows = A.rows;
    if (row_ptr) std::memcpy(row_ptr, A.row_ptr.data(), A.row_ptr.size() * sizeof(int));
    if (col) std::memcpy(col, A.col.data(), A.col.size() * sizeof(int));
    if (val) std::memcpy(val, A.val.data(), A.val.size() * sizeof(double));
    nnz = static_cast<long>(A.val.size());
  }, false);
  return rc == TG_OK ? nnz : -rc;
}

int tg_sim_context(tg_sim* s, tg_ctx** out) {
  return sim_guard(s, [&](Sim& m) { *out = m.ctx; });
}

int tg_sim_info(tg_sim* s, long* out) {
  return sim_guard(s, [&](Sim& m) {
    const auto n = m.vol.basis_counts();
    const auto p = m.vol.degrees();
    const long v[] = {m.n_full, m.n_free, m.n_con, m.n_steps, static_cast<long>(m.sources.size()),
                      m.n_fe, n[0], n[1], n[2], p[0], p[1], p[2], m.kron ? (m.use_fdm ? 3 : (m.use_cg1 ? 2 : 1)) : 0, m.nqb, m.nqf,
                      m.ndk, m.h_qb_off.back(), m.h_qf_off.back()};
    std::memcpy(out, v, sizeof(v));
  }, false);
}

int tg_sim_set_sumfact(tg_sim* s, int on) {
  return sim_guard(s, [&](Sim& m) { m.set_sumfact(on != 0); }, false);
}

int tg_sim_sumfact_stats(tg_sim* s, double* out) {
  return sim_guard(s, [&](Sim& m) {
    const int nr = m.sf_n_regions();
    double jf = 0.0, jd = 0.0;
    if (m.sf_fused_ready() && nr > 0) {  // the last call's device plan
      std::vector<int> J(nr), E(nr);
      m.sf_last_plan(J.data(), E.data());
      int mf = 1 << 30, md = 1 << 30;
      for (int r = 0; r < nr; ++r) {
        const bool dir = m.sf_dir_ok && r >= nr - m.sf_dir_regions();
        (dir ? md : mf) = std::min(dir ? md : mf, J[r]);
      }
      jf = mf == (1 << 30) ? 0.0 : mf;
      jd = md == (1 << 30) ? 0.0 : md;
    }
    const double v[] = {m.sf_on ? 1.0 : 0.0, m.sf_flux_ok ? 1.0 : 0.0, m.sf_dir_ok ? 1.0 : 0.0,
                        jf, jd, m.sf_flops_total(), static_cast<double>(nr),
                        static_cast<double>(kSfItem)};
    std::memcpy(out, v, sizeof(v));
  }, false);
}

int tg_nccl_unique_id(char* out128) {
  try {
    tgb::nccl_unique_id(out128);
    return TG_OK;
  } catch (const std::exception&) {
    return TG_ECUDA;
  }
}

int tg_slab_plan(int nz, int p, int world, int rank, int* out6) {
  try {
    const tgb::SlabPlan q = tgb::slab_plan(nz, p, world, rank);
    const int v[] = {q.gz0, q.nloc, q.zo0, q.zo1, q.lo, q.hi};
    std::memcpy(out6, v, sizeof(v));
    return TG_OK;
  } catch (const std::exception&) {
    return TG_ERROR;
  }
}

int tg_sim_shard(tg_sim* s, int rank, int world, const char* id128) {
  return sim_guard(s, [&](Sim& m) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard: bad rank");
    m.shard(rank, world, id128);
  });
}

int tg_sim_set_slabs(tg_sim* s, int n) {
  return sim_guard(s, [&](Sim& m) { m.set_slabs(n); });
}

int tg_sim_sumfact_regions(tg_sim* s, double* out) {
  return sim_guard(s, [&](Sim& m) {
    const auto& R = m.sf_regions();
    for (size_t r = 0; r < R.size(); ++r) {
      double* o = out + 8 * r;
      for (int a = 0; a < 3; ++a) {
        o[a] = R[r].lo[a];
        o[3 + a] = R[r].hi[a];
      }
      o[6] = R[r].delta;
      o[7] = R[r].npts;
    }
  }, false);
}

int tg_sim_sumfact_plan(tg_sim* s, double t, int* J, int* E) {
  return sim_guard(s, [&](Sim& m) { m.sf_plan_host(t, J, E); }, false);
}

int tg_sim_sumfact_counts(tg_sim* s, double t, int* Jc) {
  return sim_guard(s, [&](Sim& m) {
    std::vector<int> J(m.sf_n_regions()), E(m.sf_n_regions());
    m.sf_plan_host(t, J.data(), E.data(), Jc);
  }, false);
}

int tg_sim_sumfact_last_counts(tg_sim* s, int* Jc) {
  return sim_guard(s, [&](Sim& m) {
    if (!m.sf_fused_ready()) throw std::logic_error("no device plan (host-only simulation)");
    std::vector<int> J(m.sf_n_regions()), E(m.sf_n_regions());
    m.sf_last_plan(J.data(), E.data(), Jc);
  });
}

int tg_sim_sumfact_last_plan(tg_sim* s, int* J, int* E) {
  return sim_guard(s, [&](Sim& m) {
    if (!m.sf_fused_ready()) throw std::logic_error("no device plan (host-only simulation)");
    m.sf_last_plan(J, E);
  });
}

int tg_sim_params(tg_sim* s, double* out) {
  return sim_guard(s, [&](Sim& m) {
    const double v[] = {m.dt_solver, m.cfg.stepping.theta, m.cfg.stepping.solver_tol,
                        m.cfg.mesh.elevate_radius, m.cfg.superpose.cull_exponent,
                        m.cfg.material.conductivity, m.cfg.material.density,
                        m.cfg.material.heat_capacity, m.cfg.material.platform_temperature,
                        static_cast<double>(m.cfg.stepping.max_iter)};
    std::memcpy(out, v, sizeof(v));
  }, false);
}

int tg_sim_sources(tg_sim* s, tg_point_source* out, int max_out) {
  return sim_guard(s, [&](Sim& m) {
    const int n = std::min<int>(max_out, static_cast<int>(m.sources.size()));
    if (n > 0) std::memcpy(out, m.sources.data(), n * sizeof(tg_point_source));
  }, false);
}

int tg_sim_face_sets(tg_sim* s, int* qb_off, int* qf_off, double* centers, int* dofs,
                     double* xq, double* nq, double* wq, double* Nb, double* Nf) {
  return sim_guard(s, [&](Sim& m) {
    auto cp = [](auto* dst, const auto& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    if (Nb || Nf) m.face_tables_to_host();
    cp(qb_off, m.h_qb_off);
    cp(qf_off, m.h_qf_off);
    cp(centers, m.centers);
    cp(dofs, m.h_dofk);
    cp(xq, m.h_qx);
    cp(nq, m.h_qn);
    cp(wq, m.h_qw);
    cp(Nb, m.h_Nb);
    cp(Nf, m.h_Nf);
  }, false);
}

int tg_sim_last_local_loads(tg_sim* s, double* out) {
  return sim_guard(s, [&](Sim& m) {
    d2h(out, m.d_loc.p, static_cast<size_t>(m.n_fe) * m.ndk, m.ctx->stream);
    TG_CUDA(cudaStreamSynchronize(m.ctx->stream));
  });
}

int tg_sim_greville_points(tg_sim* s, double* out) {
  return sim_guard(s, [&](Sim& m) { std::memcpy(out, m.grev.data(), m.grev.size() * sizeof(double)); }, false);
}

int tg_sim_flux_load(tg_sim* s, double t, const double* focus_xyz, double fine_radius,
                     double* out_F) {
  return sim_guard(s, [&](Sim& m) {
    const double r = fine_radius < 0.0 ? m.cfg.mesh.elevate_radius : fine_radius;
    m.focus_given = focus_xyz != nullptr;
    if (focus_xyz) m.focus_value = Vec3{focus_xyz[0], focus_xyz[1], focus_xyz[2]};
    try {
      m.flux_load_device(t, r, m.d_T.p);
    } catch (...) {
      m.focus_given = false;
      throw;
    }
    m.focus_given = false;
    d2h(out_F, m.d_T.p, m.n_full, m.ctx->stream);
    TG_CUDA(cudaStreamSynchronize(m.ctx->stream));
  });
}

int tg_sim_dirichlet_values(tg_sim* s, double t, double* out_g) {
  return sim_guard(s, [&](Sim& m) {
    m.dirichlet_device(t, m.d_rhs.p);
    d2h(out_g, m.d_rhs.p, m.n_con, m.ctx->stream);
    TG_CUDA(cudaStreamSynchronize(m.ctx->stream));
  });
}

int tg_sim_theta_step(tg_sim* s, const double* free_n, const double* g_n, const double* F_n,
                      const double* F_np1, const double* g_np1, double tol, int max_iter,
                      double* free_out, int* iters, double* rel) {
  return sim_guard(s, [&](Sim& m) {
    cudaStream_t st = m.ctx->stream;
    h2d(m.d_x.p, free_n, m.n_free, st);
    h2d(m.d_gn.p, g_n, m.n_con, st);
    h2d(m.d_Fn.p, F_n, m.n_full, st);
    h2d(m.d_F1.p, F_np1, m.n_full, st);
    h2d(m.d_g1.p, g_np1, m.n_con, st);
    const PcgStatus r = m.theta_step_device(tol, max_iter);
    d2h(free_out, m.d_x.p, m.n_free, st);
    TG_CUDA(cudaStreamSynchronize(st));
    if (iters) *iters = r.iterations;
    if (rel) *rel = r.rel_residual;
  });
}

int tg_sim_reset(tg_sim* s) {
  return sim_guard(s, [&](Sim& m) { m.reset(); });
}

int tg_sim_advance(tg_sim* s, int n_steps, long* cg_iterations, double* last_rel) {
  return sim_guard(s, [&](Sim& m) {
    double rel = 0.0;
    const long it = m.advance_steps(n_steps, &rel);
    if (cg_iterations) *cg_iterations = it;
    if (last_rel) *last_rel = rel;
  });
}

int tg_sim_state(tg_sim* s, int* step, double* time, double* free_out, double* g_out,
                 double* F_out) {
  return sim_guard(s, [&](Sim& m) {
    cudaStream_t st = m.ctx->stream;
    d2h(free_out, m.d_x.p, m.n_free, st);
    d2h(g_out, m.d_gn.p, m.n_con, st);
    d2h(F_out, m.d_Fn.p, m.n_full, st);
    TG_CUDA(cudaStreamSynchronize(st));
    if (step) *step = m.step;
    if (time) *time = m.step * m.dt_solver;
  });
}

long tg_sim_last_integrand(tg_sim* s, double* out) {
  long n = -TG_ERROR;
  const int rc = sim_guard(s, [&](Sim& m) {
    n = m.sf_compact_points();
    if (out) {
      d2h(out, m.d_gq.p, static_cast<size_t>(n), m.ctx->stream);
      TG_CUDA(cudaStreamSynchronize(m.ctx->stream));
    }
  });
  return rc == TG_OK ? n : -rc;
}

int tg_sim_set_region_split(tg_sim* s, int rank, int world) {
  return sim_guard(s, [&](Sim& m) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("split: bad rank");
    m.sf_rank = rank;
    m.sf_world = world;
  }, false);
}

int tg_sim_debug_trace(tg_sim* s, unsigned long long* out, int n) {
  return sim_guard(s, [&](Sim& m) {
    TG_CUDA(cudaMemcpy(out, m.d_trace.p, sizeof(unsigned long long) * std::min(n, 400),
                       cudaMemcpyDeviceToHost));
  });
}

int tg_sim_operator_apply(tg_sim* s, const double* x_free, double* y_free) {
  return sim_guard(s, [&](Sim& m) {
    cudaStream_t st = m.ctx->stream;
    h2d(m.d_r.p, x_free, m.n_free, st);
    if (m.kron)
      k2_apply(m.gfree, m.coefA[0], m.coefA[1], m.d_r.p, m.d_Ap.p, m.ctx->sm_count, st);
    else
      csr_apply(m.devA, m.d_r.p, m.d_Ap.p, st);
    d2h(y_free, m.d_Ap.p, m.n_free, st);
    TG_CUDA(cudaStreamSynchronize(st));
  });
}

int tg_fdm_factor(const double* Mband, const double* Kband, int n_band, int p, int first, int n,
                  double* V, double* lam) {
  try {
    const size_t nb = static_cast<size_t>(n_band) * (2 * p + 1);
    const Fdm1D f = fdm_factor(std::vector<double>(Mband, Mband + nb),
                               std::vector<double>(Kband, Kband + nb), n_band, p, first, n);
    std::memcpy(V, f.V.data(), sizeof(double) * f.V.size());
    std::memcpy(lam, f.lam.data(), sizeof(double) * f.lam.size());
    return TG_OK;
  } catch (const std::exception&) {
    return TG_ERROR;
  }
}

int tg_geometry_elevate(const char* in_path, const int* elevate, const double* scale,
                        const char* out_path, char* err, int err_len) {
  auto fail = [&](int code, const char* msg) {
    if (err && err_len > 0) {
      std::strncpy(err, msg, static_cast<size_t>(err_len) - 1);
      err[err_len - 1] = '\0';
    }
    return code;
  };
  try {
    if (!in_path || !out_path) throw std::invalid_argument("geometry_elevate: null path");
    NurbsVolume v = read_geometry_file(in_path);
    if (scale) v = scaled(v, {scale[0], scale[1], scale[2]});
    if (elevate) v = elevate_degree(v, {elevate[0], elevate[1], elevate[2]});
    std::ofstream out(out_path);
    if (!out) throw io_error(std::string("cannot write '") + out_path + "'");
    out << "# written by tg_geometry_elevate (exact degree elevation)\n" << geometry_text(v);
    if (!out) throw io_error(std::string("cannot write '") + out_path + "'");
    return TG_OK;
  } catch (const config_error& e) {
    return fail(TG_ECONFIG, e.what());
  } catch (const io_error& e) {
    return fail(TG_EIO, e.what());
  } catch (const std::exception& e) {
    return fail(TG_ERROR, e.what());
  }
}

int tg_sim_probe(tg_sim* s, const double* xi, long n, double* out) {
  return sim_guard(s, [&](Sim& m) {
    if (n < 0 || (n > 0 && (!xi || !out))) throw std::invalid_argument("probe: bad args");
    if (n == 0) return;
    cudaStream_t st = m.ctx->stream;
    DevBuf<double> d_xi, d_o;
    d_xi.ensure(3 * static_cast<size_t>(n));
    d_o.ensure(12 * static_cast<size_t>(n));
    h2d(d_xi.p, xi, 3 * n, st);
    m.probe_device(d_xi.p, n, d_o.p, st);
    d2h(out, d_o.p, 12 * n, st);
    TG_CUDA(cudaStreamSynchronize(st));
  });
}

int tg_sim_probe_device(tg_sim* s, const double* d_xi, long n, double* d_out) {
  return sim_guard(s, [&](Sim& m) {
    if (n < 0 || (n > 0 && (!d_xi || !d_out))) throw std::invalid_argument("probe: bad args");
    m.probe_device(d_xi, n, d_out, m.ctx->stream);
    TG_CUDA(cudaStreamSynchronize(m.ctx->stream));
  });
}

int tg_sim_field_eval(tg_sim* s, const double* coeffs, const double* xi, long n, double* out_x,
                      double* out_f) {
  return sim_guard(s, [&](Sim& m) {
    if (n < 0 || (n > 0 && (!xi || !out_x)) || (out_f && !coeffs))
      throw std::invalid_argument("field_eval: bad args");
    if (n == 0) return;
    cudaStream_t st = m.ctx->stream;
    DevBuf<double> d_c, d_xi, d_x, d_f;
    d_xi.ensure(3 * static_cast<size_t>(n));
    d_x.ensure(3 * static_cast<size_t>(n));
    h2d(d_xi.p, xi, 3 * n, st);
    const double* dc = nullptr;
    if (out_f) {
      d_c.ensure(m.n_full);
      h2d(d_c.p, coeffs, m.n_full, st);
      d_f.ensure(4 * static_cast<size_t>(n));
      dc = d_c.p;
    }
    m.field_eval_device(dc, d_xi.p, n, d_x.p, out_f ? d_f.p : nullptr, st);
    d2h(out_x, d_x.p, 3 * n, st);
    if (out_f) d2h(out_f, d_f.p, 4 * n, st);
    TG_CUDA(cudaStreamSynchronize(st));
  });
}

int tg_sim_flux_profile(tg_sim* s, int face, int n_samples, double edge_v,
                        const double* theta_axis, double* out) {
  return sim_guard(s, [&](Sim& m) {
    if (face < 0 || face > 5 || !out) throw std::invalid_argument("flux_profile: bad args");
    m.flux_profile(static_cast<FaceId>(face), n_samples, edge_v, theta_axis, out);
  });
}

}  // extern "C"
