/* thermiga_b200 — C ABI of the B200-native hot path of the semi-analytical IGA
 * thermal solver (reference: "thermiga", /root/reference/proj).
 *
 * The reference has no FFI of its own: its boundary for this path is the C++
 * API in proj/include/thermiga/*.hpp, called by run_time_loop
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
 * reset, the number of this library's kernel launches, and the work counted. */
int tg_set_profiling(tg_ctx* ctx, int on);
int tg_profile_read(tg_ctx* ctx, double* out /* [8] */, int reset);
/* FP64 issue-rate microbenchmark (independent DFMA chains over every SM);
 * the K1 roofline denominator. */
int tg_fp64_peak(tg_ctx* ctx, double* out_tflops);

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

#ifdef __cplusplus
}
#endif
#endif /* THERMIGA_B200_H */
