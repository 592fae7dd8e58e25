/* thermiga_b200 — C ABI of the B200-native hot path of the semi-analytical IGA
 * thermal solver (reference: "thermiga", /root/reference/proj).
 *
 * The reference has no FFI of its own: its boundary for this path is the C++
 * API in the headers under proj/include/thermiga/, called by run_time_loop
 * (proj/src/driver.cpp:105-146). Each entry point below replaces one of those
 * calls; the citation says which. The C++ shim include/thermiga_b200.hpp
 * re-exposes them with the reference's signatures.
 *
 * Conventions
 *  - Plain pointers and sizes only. "host" arrays are caller-owned CPU memory;
 *    "_device" variants take CUDA device pointers and a cudaStream_t (as void*,
 *    NULL = the legacy default stream, as everywhere in CUDA) and do not
 *    synchronize; host variants run on the context's own stream and return
 *    after the results are in host memory.
 *  - Vectors over control points use the reference's flat order, first index
 *    fastest (ControlGrid::index, proj/include/thermiga/splines.hpp:73-75).
 *  - Points are xyz-interleaved doubles (Vec3, proj/include/thermiga/core.hpp:14).
 *  - Every function returns a status code; the message of the last failure on a
 *    context is available from tg_last_error(). Codes mirror the reference CLI's
 *    exit codes (proj/tools/main.cpp:84-96).
 *  - One context per host thread; calls on a context are serialized by the caller.
 *  - There is no CPU fallback: without a usable sm_100a device every compute
 *    entry point fails with TG_ECUDA.
 */
#ifndef THERMIGA_B200_H
#define THERMIGA_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define TG_OK 0
#define TG_ERROR 1    /* std::invalid_argument / other std::exception (CLI exit 1) */
#define TG_ECONFIG 2  /* thermiga::config_error (CLI exit 2) */
#define TG_ENUMERIC 3 /* thermiga::numeric_error, e.g. PCG non-convergence (CLI exit 3) */
#define TG_EIO 4      /* thermiga::io_error (CLI exit 4) */
#define TG_ECUDA 5    /* CUDA runtime failure or no usable device */

typedef struct tg_ctx tg_ctx;
typedef struct tg_sim tg_sim;

/* thermiga::Material (proj/include/thermiga/analytic.hpp:10-20) */
typedef struct tg_material {
  double conductivity;
  double density;
  double heat_capacity;
  double platform_temperature;
} tg_material;

/* thermiga::LaserSpec (proj/include/thermiga/analytic.hpp:22-31) */
typedef struct tg_laser {
  double power;
  double speed;
  double spot_radius;
  double absorptivity;
  double dt;
} tg_laser;

/* thermiga::PointSource (proj/include/thermiga/analytic.hpp:35-40); same
 * 48-byte layout, so a std::vector<PointSource> can be passed as is. */
typedef struct tg_point_source {
  double x, y, z;
  double energy;
  double t_activate;
  double tau;
} tg_point_source;

/* ---- library / context ------------------------------------------------ */
int tg_abi_version(void);
int tg_ctx_create(int device, tg_ctx** out);
void tg_ctx_destroy(tg_ctx* ctx);
const char* tg_last_error(const tg_ctx* ctx);
/* Kernel-level profiling: when on, the main K1/K2 kernels are bracketed by
 * CUDA events; tg_profile_read returns the summed milliseconds since the last
 * reset, the number of this library's kernel launches, and the work counted:
 * out = {k1_ms, k1_launches, k1_pairs, k2_ms (solve), k2_launches, k2_bytes,
 *        launches, theta_step_ms (expand + RHS + solve), k5_ms (contraction),
 *        k5_launches, run_ms (whole tg_sim_advance steps: loads + theta step)}. */
int tg_set_profiling(tg_ctx* ctx, int on);
int tg_profile_read(tg_ctx* ctx, double* out /* [11] */, int reset);
/* FP64 issue-rate microbenchmark (independent DFMA chains over every SM);
 * the K1 roofline denominator. */
int tg_fp64_peak(tg_ctx* ctx, double* out_tflops);
/* Measured FP64 tensor-core (DMMA m8n8k4) rate of this GPU, TFLOP/s. */
int tg_dmma_peak(tg_ctx* ctx, double* out_tflops);

/* ---- analytic field (K1) ---------------------------------------------- */

/* discretize_scan (proj/src/analytic.cpp:22-71), host-side and bit-exact.
 * Returns the source count (>= 0) or -TG_ERROR; writes at most max_out. */
int tg_discretize_scan(const double* waypoints_xy, int n_waypoints, double start_time,
                       double plane_z, const tg_laser* laser, const tg_material* mat,
                       tg_point_source* out, int max_out);

/* Upload the scan history (replaces the std::vector<PointSource> argument of
 * superpose, proj/include/thermiga/analytic.hpp:73-75). */
int tg_set_sources(tg_ctx* ctx, const tg_point_source* src, int n, const tg_material* mat);

/* superpose (proj/src/analytic.cpp:92-109) at n points: value (degC rise) and
 * gradient (degC/m, xyz-interleaved, may be NULL). cull = SuperposeOptions::
 * cull_exponent (analytic.hpp:62-66). Host arrays; synchronous. */
int tg_superpose_batch(tg_ctx* ctx, const double* pts_xyz, long n, double t, double cull,
                       double* out_val, double* out_grad);
int tg_superpose_batch_device(tg_ctx* ctx, const double* d_pts_xyz, long n, double t,
                              double cull, double* d_val, double* d_grad, void* stream);

/* ---- simulation (K1 + K2 + K3 behind the reference's driver) ------------ */

/* Overrides for a parsed config; zero fields keep the config's value. */
typedef struct tg_sim_options {
  double t_end;      /* [stepping] t_end */
  double solver_tol; /* [stepping] solver_tol */
  int max_iter;      /* [stepping] max_iter */
  int device;        /* CUDA device ordinal */
  int host_only;     /* 1: host setup only (no device; compute calls fail) */
  int preconditioner; /* 0: Jacobi, the reference's pcg_jacobi (default);
                         1: fast diagonalization (separable patches; the
                         same PCG loop converges in 1-2 iterations) */
} tg_sim_options;

/* parse_config + prepare_simulation (proj/src/config.cpp:253-416,
 * proj/src/driver.cpp:66-95): the config format is the reference's. On
 * failure *out is still set so tg_sim_last_error can be read; destroy it. */
int tg_sim_create(const char* config_path, const tg_sim_options* opt, tg_sim** out);
void tg_sim_destroy(tg_sim* sim);
const char* tg_sim_last_error(const tg_sim* sim);
/* The simulation's device context (profiling counters, K1 sources). */
int tg_sim_context(tg_sim* sim, tg_ctx** out);
/* out[18]: n_full, n_free, n_constrained, n_steps, n_sources, n_face_elements,
 * nx, ny, nz, px, py, pz, operator (0 assembled CSR, 1 Kronecker, 2 Kronecker with the
 * single-sweep solver on the device, 3 Kronecker with the fast-diagonalization
 * preconditioner), max nq_base, max nq_fine,
 * ndofs_kept, total base qps, total fine qps */
int tg_sim_info(tg_sim* sim, long* out);
/* out[10]: dt_solver, theta, solver_tol, elevate_radius, cull_exponent,
 * conductivity, density, heat_capacity, platform_temperature, max_iter */
int tg_sim_params(tg_sim* sim, double* out);
int tg_sim_sources(tg_sim* sim, tg_point_source* out, int max_out);
/* Lateral face quadrature sets as uploaded (classify_boundary,
 * proj/src/mesh.cpp:158-236): per-element offsets into the base / fine rules
 * (n_face_elements + 1 each), centers, kept DOF columns (-1 = pad), base then
 * fine quadrature points, normals, weights and basis tables. */
int tg_sim_face_sets(tg_sim* sim, int* qb_off, int* qf_off, double* centers, int* dofs,
                     double* xq, double* nq, double* wq, double* Nb, double* Nf);
int tg_sim_greville_points(tg_sim* sim, double* out_xyz);
/* The per-element local loads of the last flux-load call (n_face_elements x
 * ndofs_kept, the columns of tg_sim_face_sets' dofs): assemble_boundary_load's
 * `local` (proj/src/assembly.cpp:123-137) before the scatter. */
int tg_sim_last_local_loads(tg_sim* sim, double* out);
/* Banded 1D factors of the Kronecker operator for axis dir (n x (2p+1),
 * [i][p + j - i]); TG_ERROR when the patch is not separable. */
int tg_sim_kron_factors(tg_sim* sim, int dir, double* M, double* K);
/* DirichletSystem::reduced_operator() (proj/include/thermiga/assembly.hpp:56,
 * proj/src/assembly.cpp:201-228) of a non-separable patch as assembled on the
 * host (bit-identical to the reference's): returns nnz (pass NULL arrays to
 * query), or -status (TG_ERROR for separable patches, whose operator is never
 * assembled). */
long tg_sim_reduced_operator(tg_sim* sim, int* rows, int* row_ptr, int* col, double* val);

/* assemble_flux_load (proj/src/assembly.cpp:148-166): F (n_full) at time t.
 * focus_xyz (nullable): the fine-rule focus; NULL = the newest source active
 * at t (assembly.cpp:153-157). fine_radius < 0 uses the config's
 * elevate_radius. */
int tg_sim_flux_load(tg_sim* sim, double t, const double* focus_xyz, double fine_radius,
                     double* out_F);
/* dirichlet_values (proj/src/mesh.cpp:238-264): g (n_constrained) at time t. */
int tg_sim_dirichlet_values(tg_sim* sim, double t, double* out_g);
/* theta_step (proj/src/timestep.cpp:5-24) with pcg_jacobi
 * (proj/src/sparse.cpp:41-100): warm-started from free_n. Returns TG_ENUMERIC
 * with the reference's message on non-convergence or a non-SPD operator. */
int tg_sim_theta_step(tg_sim* sim, const double* free_n, const double* g_n, const double* F_n,
                      const double* F_np1, const double* g_np1, double tol, int max_iter,
                      double* free_out, int* iters, double* rel);
/* y = A_ff x, the reduced theta-step operator (DirichletSystem::reduced_operator,
 * proj/include/thermiga/assembly.hpp:56). */
int tg_sim_operator_apply(tg_sim* sim, const double* x_free, double* y_free);

/* The compact flux integrand of the last flux-load call (the per-point
 * (-k grad T~ . n) w of assemble_boundary_load, assembly.cpp:133-135, in the
 * device's element order: base rules, fine rules of the step's fine
 * elements): returns the point count (pass NULL to query). */
long tg_sim_last_integrand(tg_sim* sim, double* out);
/* Restrict the fused loads to the K5 regions r with r % world == rank (the
 * split tg_sim_shard uses; a test hook to check that the ranks' integrands
 * and Dirichlet values sum to the unsplit ones bit for bit). */
int tg_sim_set_region_split(tg_sim* sim, int rank, int world);

/* Diagnostics: %globaltimer stamps of CTA 0 at the K2 phase boundaries of the
 * first 16 CG iterations of the last solve (5 per iteration; recorded only
 * when TG_K2_TRACE is set in the environment at tg_sim_create). */
int tg_sim_debug_trace(tg_sim* sim, unsigned long long* out, int n);

/* run_time_loop (proj/src/driver.cpp:105-146) with the state resident on the
 * device: reset = step 0 (free = 0, g_0, F_0); advance = n steps. */
int tg_sim_reset(tg_sim* sim);
int tg_sim_advance(tg_sim* sim, int n_steps, long* cg_iterations, double* last_rel);
/* Copy the current state to the host (any pointer may be NULL). */
int tg_sim_state(tg_sim* sim, int* step, double* time, double* free_out, double* g_out,
                 double* F_out);

/* ---- sparse LA on a caller matrix (proj/include/thermiga/sparse.hpp) ------
 * CSR: rows x rows, 0-based row_ptr (rows + 1) / col / val, host arrays.
 * tg_pcg_jacobi = pcg_jacobi (sparse.cpp:41-100) on this context's GPU: x
 * holds the warm start and receives the solution; the reference's options
 * default to tol = 1e-10, max_iter = 5000 (sparse.hpp:32-35). TG_ENUMERIC with
 * the reference's messages on a non-positive diagonal, an indefinite
 * direction, or the iteration cap (iterations / rel_residual still set).
 * tg_csr_multiply = CsrMatrix::multiply (sparse.cpp:25-31). */
int tg_pcg_jacobi(tg_ctx* ctx, int rows, const int* row_ptr, const int* col, const double* val,
                  const double* b, double* x, double tol, int max_iter, int* iterations,
                  double* rel_residual);
int tg_csr_multiply(tg_ctx* ctx, int rows, const int* row_ptr, const int* col, const double* val,
                    const double* x, double* y);

/* Host helper behind the fast-diagonalization preconditioner (exposed for
 * tests): K_d V = M_d V diag(lam), V^T M_d V = I for rows/cols
 * [first, first + n) of banded 1D factors (n_band x (2p+1), [i][p + j - i]).
 * V: n x n column-major. */
int tg_fdm_factor(const double* Mband, const double* Kband, int n_band, int p, int first, int n,
                  double* V, double* lam);

/* Geometry tooling (not in the reference):
 * read a geometry file (the reference's [geometry] format or `case =`,
 * proj/src/config.cpp:171-215), scale the control coordinates per axis
 * (scale[3], NULL = none), elevate the degree exactly by elevate[3] per
 * direction (Bezier extraction + Bernstein elevation on homogeneous points;
 * interior breakpoints end with multiplicity p + t, i.e. C0), and write the
 * result as a geometry file the reference reads. On failure the message is
 * copied to err (err_len bytes). */
int tg_geometry_elevate(const char* in_path, const int* elevate, const double* scale,
                        const char* out_path, char* err, int err_len);

/* ---- observers (proj/src/postproc.cpp, driver.cpp:226-254) --
 * The current state (after reset/advance, time = step * dt) at parametric
 * points xi (n x 3, each coordinate in [0, 1]; others fail like
 * total_temperature, postproc.cpp:12-14): out (n x 12) per point =
 *   x, y, z (map_point), T_total = T_c + T_tilde + T_hat (total_temperature),
 *   T_tilde (superpose), T_hat (field_at), grad T_tilde (3), grad T_hat (3).
 * The probes, export_field and boundary_flux_profile read these columns. */
int tg_sim_probe(tg_sim* sim, const double* xi, long n, double* out);
/* Same on device buffers (synchronous; runs on the simulation's stream). */
int tg_sim_probe_device(tg_sim* sim, const double* d_xi, long n, double* d_out);
/* map_point / field_at (proj/src/splines.cpp:257-303) with caller
 * coefficients (n_full, host, flat order): out_x (n x 3), out_f (n x 4 =
 * value, physical gradient). coeffs and out_f may be NULL (geometry only). */
int tg_sim_field_eval(tg_sim* sim, const double* coeffs, const double* xi, long n,
                      double* out_x, double* out_f);
/* boundary_flux_profile (postproc.cpp:21-79) of the current state on face
 * `face` (0 ximin, 1 ximax, 2 etamin, 3 etamax, 4 zetamin, 5 zetamax) at edge
 * parameter edge_v: out (n_samples x 5) = s, theta (NaN without theta_axis),
 * q_tilde, q_hat, q_net. theta_axis: NULL or 2 doubles. */
int tg_sim_flux_profile(tg_sim* sim, int face, int n_samples, double edge_v,
                        const double* theta_axis, double* out);

/* K5 sum-factorised superposition (no reference counterpart: an evaluation
 * strategy for assemble_flux_load, proj/src/assembly.cpp:148-166, and
 * dirichlet_values, proj/src/mesh.cpp:238-264, on axis-aligned patches whose
 * face quadrature / Greville points are tensor grids). On by default where
 * available; on = 0 makes every superposition a K1 pair loop. */
int tg_sim_set_sumfact(tg_sim* sim, int on);
/* out[8]: on, faces gridded, Greville grid, the last call's contraction
 * prefix J (the smallest over the flux regions; over the Greville regions),
 * contraction flops issued since setup, regions, sources per work item */
int tg_sim_sumfact_stats(tg_sim* sim, double* out);
/* ---- multi-GPU (one process per GPU; proj/src/driver.cpp:126-145 per rank).
 * tg_nccl_unique_id: rank 0 creates the communicator id (128 bytes) that the
 * caller hands to every rank (e.g. a torch.distributed broadcast).
 * tg_sim_shard: join the NCCL communicator as rank of world; from then on
 * tg_sim_advance splits the superposition regions over the ranks (loads
 * all-reduced) and the θ-step solve into z-slabs of the free grid (ghost
 * planes and the dot products' partial sums exchanged every iteration, x
 * broadcast after the solve): every rank ends each step with the same state.
 * tg_sim_set_slabs: the same slab solve with n slabs on this one GPU, halos
 * exchanged by device copies (n <= 1: off).
 * tg_slab_plan (host only): out6 = local first global plane, local planes,
 * own planes [zo0, zo1) in local indices, lower / upper neighbour (-1: none). */
int tg_nccl_unique_id(char* out128);
int tg_sim_shard(tg_sim* sim, int rank, int world, const char* id128);
int tg_sim_set_slabs(tg_sim* sim, int n);
int tg_slab_plan(int nz, int p, int world, int rank, int* out6);
/* K5 regions (one per contraction tile of the face grids, then of the
 * Greville grid): out (n_regions x 8) = lo[3], hi[3], delta, points. */
int tg_sim_sumfact_regions(tg_sim* sim, double* out);
/* The K5 plan at time t restated on the host (no device needed): per region
 * the contraction prefix J (sources [0, J)) and the end E of the pair-wise
 * remainder [J, E) (later sources are culled on the whole region box). */
int tg_sim_sumfact_plan(tg_sim* sim, double t, int* J, int* E);
/* The plan the device computed in the last flux-load / Dirichlet call. */
int tg_sim_sumfact_last_plan(tg_sim* sim, int* J, int* E);
/* Per region the contraction's source count Jc: J plus the sources of
 * [J, E) that no cull reaches anywhere in the region either (they join the
 * contraction; the pair-wise remainder skips them). Host restatement at t /
 * the last device plan. */
int tg_sim_sumfact_counts(tg_sim* sim, double t, int* Jc);
int tg_sim_sumfact_last_counts(tg_sim* sim, int* Jc);

#ifdef __cplusplus
}
#endif
#endif /* THERMIGA_B200_H */
