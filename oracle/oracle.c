/* TEST INFRASTRUCTURE — plain-C restatement of the reference hot path.
 *
 * This file is the oracle: a CPU restatement of the reference algorithm for
 * the path BASELINE.json's north_star names (point-source superposition, the
 * Neumann flux load and the Jacobi-PCG of the theta-step). It is pinned against
 * the unmodified reference library (oracle/_ref, tests/test_oracle_pins.py) and
 * the reference's own known-answer tests. It is compiled with
 * -ffp-contract=off so that its rounding matches the reference's x86-64 build
 * (no FMA). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* src/core.cpp:28-55 — Newton iteration on the Legendre recurrence, nodes
 * seeded by the Chebyshev-like guess cos(pi (i + 3/4) / (n + 1/2)). */
void or_gauss_rule(int n, double* nodes, double* weights) {
  for (int i = 0; i < n; ++i) {
    double x = cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double l0 = 1.0, l1 = x;
      for (int k = 2; k <= n; ++k) {
        const double l2 = ((2.0 * k - 1.0) * x * l1 - (k - 1.0) * l0) / k;
        l0 = l1;
        l1 = l2;
      }
      dp = n * (x * l1 - l0) / (x * x - 1.0);
      const double step = l1 / dp;
      x -= step;
      if (fabs(step) < 1e-15) break;
    }
    nodes[n - 1 - i] = x;
    weights[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

/* src/analytic.cpp:22-71 */
int or_discretize_scan(const double* wp, int n_wp, double start_time, double plane_z,
                       double power, double speed, double spot_radius, double absorptivity,
                       double laser_dt, double k, double rho, double c, double* out6,
                       int max_out) {
  if (n_wp < 1) return -1;
  if (!(power >= 0.0) || !(speed > 0.0) || !(spot_radius > 0.0) ||
      !(absorptivity > 0.0 && absorptivity <= 1.0) || !(laser_dt > 0.0))
    return -1;
  if (!(k > 0.0) || !(rho > 0.0) || !(c > 0.0)) return -1;
  const double alpha = k / (rho * c);
  const double energy = absorptivity * power * laser_dt;
  const double tau_shift = spot_radius * spot_radius / (8.0 * alpha);
#define EMIT(I, X, Y)                                        \
  do {                                                       \
    if ((I) < max_out) {                                     \
      double* o = out6 + 6 * (size_t)(I);                    \
      o[0] = (X);                                            \
      o[1] = (Y);                                            \
      o[2] = plane_z;                                        \
      o[3] = energy;                                         \
      o[4] = start_time + (I) * laser_dt;                    \
      o[5] = o[4] - tau_shift;                               \
    }                                                        \
  } while (0)
  if (n_wp == 1) {
    EMIT(0, wp[0], wp[1]);
    return 1;
  }
  const double spacing = speed * laser_dt;
  double* cum = (double*)calloc((size_t)n_wp, sizeof(double));
  for (int i = 1; i < n_wp; ++i)
    cum[i] = cum[i - 1] + hypot(wp[2 * i] - wp[2 * i - 2], wp[2 * i + 1] - wp[2 * i - 1]);
  const double total = cum[n_wp - 1];
  const int n_src = (int)floor(total / spacing * (1.0 + 1e-12)) + 1;
  int seg = 0;
  for (int I = 0; I < n_src; ++I) {
    double s = I * spacing;
    if (s > total) s = total;
    while (seg + 2 < n_wp && cum[seg + 1] < s) ++seg;
    const double len = cum[seg + 1] - cum[seg];
    const double f = len > 0.0 ? (s - cum[seg]) / len : 0.0;
    const double x = wp[2 * seg] + f * (wp[2 * seg + 2] - wp[2 * seg]);
    const double y = wp[2 * seg + 1] + f * (wp[2 * seg + 3] - wp[2 * seg + 1]);
    EMIT(I, x, y);
  }
#undef EMIT
  free(cum);
  return n_src;
}

/* src/analytic.cpp:92-109: causality skip dt <= 0, cull arg > cull, source order. */
static void superpose_one(const double* src6, int n_src, double alpha, double rcp,
                          const double* x, double t, double cull, double* val, double* g) {
  double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
  for (int j = 0; j < n_src; ++j) {
    const double* s = src6 + 6 * (size_t)j;
    const double dt = t - s[5];
    if (dt <= 0.0) continue;
    const double spread = 4.0 * alpha * dt;
    const double rx = x[0] - s[0], ry = x[1] - s[1], rz = x[2] - s[2];
    const double arg = (rx * rx + ry * ry + rz * rz) / spread;
    if (arg > cull) continue;
    const double T = s[3] / (rcp * pow(M_PI * spread, 1.5)) * exp(-arg);
    v += T;
    const double w = -T / (2.0 * alpha * dt);
    gx += rx * w;
    gy += ry * w;
    gz += rz * w;
  }
  *val = v;
  if (g) {
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
  }
}

void or_superpose_batch(const double* src6, int n_src, double k, double rho, double c,
                        const double* pts, long n_pts, double t, double cull, double* val,
                        double* grad) {
  const double alpha = k / (rho * c);
  const double rcp = rho * c;
  for (long i = 0; i < n_pts; ++i)
    superpose_one(src6, n_src, alpha, rcp, pts + 3 * i, t, cull, val + i,
                  grad ? grad + 3 * i : NULL);
}

/* src/sparse.cpp:25-31 */
void or_csr_spmv(int n, const int* rp, const int* col, const double* val, const double* x,
                 double* y) {
  for (int r = 0; r < n; ++r) {
    double acc = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) acc += val[k] * x[col[k]];
    y[r] = acc;
  }
}

/* src/sparse.cpp:41-100 */
int or_pcg_jacobi(int n, const int* rp, const int* col, const double* val, const double* b,
                  double* x, double tol, int max_iter, int* iters, double* rel_out) {
  double* inv_diag = (double*)malloc(sizeof(double) * (size_t)n);
  for (int r = 0; r < n; ++r) {
    double d = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k)
      if (col[k] == r) d = val[k];
    if (!(d > 0.0)) {
      free(inv_diag);
      return 2;
    }
    inv_diag[r] = 1.0 / d;
  }
  double bnorm = 0.0;
  for (int i = 0; i < n; ++i) bnorm += b[i] * b[i];
  bnorm = sqrt(bnorm);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    *iters = 0;
    *rel_out = 0.0;
    free(inv_diag);
    return 0;
  }
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* Ap = (double*)malloc(sizeof(double) * (size_t)n);
  or_csr_spmv(n, rp, col, val, x, r);
  for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  double rz = 0.0;
  for (int i = 0; i < n; ++i) {
    z[i] = inv_diag[i] * r[i];
    rz += r[i] * z[i];
  }
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rel = 0.0;
  int status = 3;
  int it = 0;
  for (it = 0; it < max_iter; ++it) {
    double rn = 0.0;
    for (int i = 0; i < n; ++i) rn += r[i] * r[i];
    rel = sqrt(rn) / bnorm;
    if (rel <= tol) {
      status = 0;
      break;
    }
    or_csr_spmv(n, rp, col, val, p, Ap);
    double pAp = 0.0;
    for (int i = 0; i < n; ++i) pAp += p[i] * Ap[i];
    if (!(pAp > 0.0)) {
      status = 4;
      break;
    }
    const double alpha = rz / pAp;
    for (int i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * Ap[i];
    }
    double rz_new = 0.0;
    for (int i = 0; i < n; ++i) {
      z[i] = inv_diag[i] * r[i];
      rz_new += r[i] * z[i];
    }
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  *iters = it;
  *rel_out = rel;
  free(inv_diag);
  free(r);
  free(z);
  free(p);
  free(Ap);
  return status;
}

/* src/assembly.cpp:117-166 — element-local accumulation in q order, then a
 * serial scatter in (face, element, a) order; the fine rule follows the newest
 * source with t_activate <= t (assembly.cpp:153-157). */
void or_boundary_load(int n_fe, int nd, const int* nq_base, const int* nq_fine, const int* dofs,
                      const double* centers, const double* xb, const double* nb,
                      const double* wb, const double* Nb, const double* xf, const double* nf,
                      const double* wf, const double* Nf, int n_src, const double* src6,
                      int n_full, double t, double fine_radius, double cull, double k,
                      double rho, double c, double* load) {
  const double alpha = k / (rho * c);
  const double rcp = rho * c;
  int have_focus = 0;
  double focus[3] = {0, 0, 0};
  for (int j = 0; j < n_src; ++j) {
    if (src6[6 * (size_t)j + 4] > t) break;
    focus[0] = src6[6 * (size_t)j];
    focus[1] = src6[6 * (size_t)j + 1];
    focus[2] = src6[6 * (size_t)j + 2];
    have_focus = 1;
  }
  memset(load, 0, sizeof(double) * (size_t)n_full);
  double* loc = (double*)malloc(sizeof(double) * (size_t)nd);
  size_t ob = 0, of = 0;
  for (int e = 0; e < n_fe; ++e) {
    const double* ce = centers + 3 * (size_t)e;
    int fine = 0;
    if (have_focus) {
      const double dx = ce[0] - focus[0], dy = ce[1] - focus[1], dz = ce[2] - focus[2];
      fine = sqrt(dx * dx + dy * dy + dz * dz) < fine_radius;
    }
    const int nq = fine ? nq_fine[e] : nq_base[e];
    const size_t o = fine ? of : ob;
    const double* X = (fine ? xf : xb) + 3 * o;
    const double* Nn = (fine ? nf : nb) + 3 * o;
    const double* W = (fine ? wf : wb) + o;
    const double* N = (fine ? Nf : Nb) + o * nd;
    for (int a = 0; a < nd; ++a) loc[a] = 0.0;
    for (int q = 0; q < nq; ++q) {
      double v, g[3];
      superpose_one(src6, n_src, alpha, rcp, X + 3 * q, t, cull, &v, g);
      const double* n = Nn + 3 * q;
      const double integrand = -k * (g[0] * n[0] + g[1] * n[1] + g[2] * n[2]);
      const double gq = integrand * W[q];
      for (int a = 0; a < nd; ++a) loc[a] += gq * N[(size_t)q * nd + a];
    }
    for (int a = 0; a < nd; ++a) load[dofs[(size_t)e * nd + a]] += loc[a];
    ob += (size_t)nq_base[e];
    of += (size_t)nq_fine[e];
  }
  free(loc);
}

/* The element-local half of assemble_boundary_load (src/assembly.cpp:126-139)
 * for face elements [e0, e1): loc[(e - e0) * nd + a], without the scatter.
 * (Test support for the sharded flux load: slabs of these, gathered in the
 * reference's order, must reproduce or_boundary_load bit for bit.) */
void or_boundary_local(int n_fe, int nd, const int* nq_base, const int* nq_fine,
                       const double* centers, const double* xb, const double* nb,
                       const double* wb, const double* Nb, const double* xf, const double* nf,
                       const double* wf, const double* Nf, int n_src, const double* src6,
                       double t, double fine_radius, double cull, double k, double rho, double c,
                       int e0, int e1, double* loc) {
  const double alpha = k / (rho * c);
  const double rcp = rho * c;
  int have_focus = 0;
  double focus[3] = {0, 0, 0};
  for (int j = 0; j < n_src; ++j) {
    if (src6[6 * (size_t)j + 4] > t) break;
    focus[0] = src6[6 * (size_t)j];
    focus[1] = src6[6 * (size_t)j + 1];
    focus[2] = src6[6 * (size_t)j + 2];
    have_focus = 1;
  }
  size_t ob = 0, of = 0;
  for (int e = 0; e < e0 && e < n_fe; ++e) {
    ob += (size_t)nq_base[e];
    of += (size_t)nq_fine[e];
  }
  for (int e = e0; e < e1 && e < n_fe; ++e) {
    const double* ce = centers + 3 * (size_t)e;
    int fine = 0;
    if (have_focus) {
      const double dx = ce[0] - focus[0], dy = ce[1] - focus[1], dz = ce[2] - focus[2];
      fine = sqrt(dx * dx + dy * dy + dz * dz) < fine_radius;
    }
    const int nq = fine ? nq_fine[e] : nq_base[e];
    const size_t o = fine ? of : ob;
    const double* X = (fine ? xf : xb) + 3 * o;
    const double* Nn = (fine ? nf : nb) + 3 * o;
    const double* W = (fine ? wf : wb) + o;
    const double* N = (fine ? Nf : Nb) + o * nd;
    double* l = loc + (size_t)(e - e0) * nd;
    for (int a = 0; a < nd; ++a) l[a] = 0.0;
    for (int q = 0; q < nq; ++q) {
      double v, g[3];
      superpose_one(src6, n_src, alpha, rcp, X + 3 * q, t, cull, &v, g);
      const double* n = Nn + 3 * q;
      const double gq = -k * (g[0] * n[0] + g[1] * n[1] + g[2] * n[2]) * W[q];
      for (int a = 0; a < nd; ++a) l[a] += gq * N[(size_t)q * nd + a];
    }
    ob += (size_t)nq_base[e];
    of += (size_t)nq_fine[e];
  }
}
