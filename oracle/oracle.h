/* TEST INFRASTRUCTURE — plain-C restatement of the reference hot path.
 * Used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg,
 * as the checker or the "port" CPU baseline; never by the product.
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj). */
#ifndef THERMIGA_ORACLE_H
#define THERMIGA_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Sources are packed as 6 doubles {x, y, z, energy, t_activate, tau}
 * (PointSource, include/thermiga/analytic.hpp:35-40). */

/* gauss_rule: src/core.cpp:28-65 */
void or_gauss_rule(int n, double* nodes, double* weights);

/* discretize_scan: src/analytic.cpp:22-71. Returns the source count, or -1 on
 * invalid input; writes at most max_out sources. */
int or_discretize_scan(const double* waypoints, int n_wp, double start_time, double plane_z,
                       double power, double speed, double spot_radius, double absorptivity,
                       double laser_dt, double k, double rho, double c, double* out6,
                       int max_out);

/* superpose: src/analytic.cpp:92-109, once per point, serial. grad may be NULL. */
void or_superpose_batch(const double* src6, int n_src, double k, double rho, double c,
                        const double* pts, long n_pts, double t, double cull, double* val,
                        double* grad);

/* CsrMatrix::multiply: src/sparse.cpp:25-31 */
void or_csr_spmv(int n, const int* row_ptr, const int* col, const double* val, const double* x,
                 double* y);

/* pcg_jacobi: src/sparse.cpp:41-100. Returns 0 on success, 2 for a
 * non-positive diagonal, 4 for an indefinite direction, 3 when max_iter is hit. */
int or_pcg_jacobi(int n, const int* row_ptr, const int* col, const double* val, const double* b,
                  double* x, double tol, int max_iter, int* iters, double* rel);

/* assemble_flux_load + assemble_boundary_load: src/assembly.cpp:117-166, on
 * face sets flattened in (face, element, q) order (mesh.hpp:84-113) with
 * per-element rule sizes nq_base[e], nq_fine[e]. */
void or_boundary_load(int n_fe, int n_dofs, const int* nq_base, const int* nq_fine,
                      const int* dofs, const double* centers, const double* xb, const double* nb,
                      const double* wb, const double* Nb, const double* xf, const double* nf,
                      const double* wf, const double* Nf, int n_src, const double* src6,
                      int n_full, double t, double fine_radius, double cull, double k,
                      double rho, double c, double* load);

/* Element-local loads of face elements [e0, e1) (assembly.cpp:126-139), no
 * scatter: loc[(e - e0) * n_dofs + a]. */
void or_boundary_local(int n_fe, int n_dofs, const int* nq_base, const int* nq_fine,
                       const double* centers, const double* xb, const double* nb,
                       const double* wb, const double* Nb, const double* xf, const double* nf,
                       const double* wf, const double* Nf, int n_src, const double* src6,
                       double t, double fine_radius, double cull, double k, double rho, double c,
                       int e0, int e1, double* loc);

#ifdef __cplusplus
}
#endif
#endif
