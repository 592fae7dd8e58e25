// Simulation engine (see sim.cu).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "context.hpp"
#include "host/config.hpp"
#include "host/operator.hpp"
#include "k2_csr.cuh"
#include "k2_fdm.cuh"
#include "k2_kron.cuh"
#include "k4_eval.cuh"
#include "k5_sumfact.cuh"

namespace tgb {

// Control-grid geometry of the DOF split: grid dims, the constrained axis and
// layer, and the two in-face axes that order the constrained values.
struct SimGeom {
  int n[3];
  int ax, layer, t0, t1;
};

struct SimOptions {
  double t_end = 0.0;       // > 0 overrides the config
  double solver_tol = 0.0;  // > 0 overrides the config
  int max_iter = 0;         // > 0 overrides the config
  int device = 0;
  bool host_only = false;
  int preconditioner = 0;  // 0 Jacobi (reference), 1 fast diagonalization
};

class Sim {
 public:
  Sim(const std::string& config_path, const SimOptions& opt);
  ~Sim();
  Sim(const Sim&) = delete;
  Sim& operator=(const Sim&) = delete;

  // run_time_loop pieces (driver.cpp:105-146)
  void reset();          // state 0: free = 0, g_0, F_0
  PcgStatus advance();   // one step: F_{n+1}, g_{n+1}, theta step
  // one step with F_{n+1}, g_{n+1} supplied on the device (a multi-GPU driver
  // assembles them sharded, all-gathers, and every rank steps)
  PcgStatus advance_with_loads(const double* d_F1_in, const double* d_g1_in);

  // drop-in pieces on device buffers
  // assemble_flux_load; with [e0, e1) only those face elements' local loads
  // (d_loc) are computed, and d_F == nullptr skips the gather (sharded use)
  void flux_load_device(double t, double radius, double* d_F, int e0 = 0,
                        int e1 = 1 << 30);
  void flux_gather_device(const double* d_loc_all, double* d_F);
  void dirichlet_device(double t, double* d_g, int c0 = 0, int c1 = -1);
  PcgStatus theta_step_device(double tol, int max_iter);  // uses d_x, d_gn, d_g1, d_Fn, d_F1
  void theta_step_launch(double tol, int max_iter);      // its launches (no status read)

  // observers: the current state at parametric points, on
  // device buffers: d_out (n x 12) = x, T_total, T_tilde, T_hat, grad T_tilde,
  // grad T_hat (k4_eval.cuh); map_point / field_at with caller coefficients
  void probe_device(const double* d_xi, long n, double* d_out, cudaStream_t s);
  void field_eval_device(const double* d_coeffs, const double* d_xi, long n, double* d_x,
                         double* d_f, cudaStream_t s);
  // boundary_flux_profile (postproc.cpp:21-79): out (n_samples x 5) = s,
  // theta, q_tilde, q_hat, q_net
  void flux_profile(FaceId face, int n_samples, double edge_v, const double* theta_axis,
                    double* out);

  // K5 (k5_sumfact.cuh): the superposition on the gridded face / Greville
  // point sets of an axis-aligned patch as a DGEMM over the sources that no
  // cull can touch there; K1 keeps the rest. On by default where the sets are
  // grids (TG_SUMFACT=0 or set_sumfact(false) turns it off). Only the
  // full-range flux / Dirichlet calls use it (the sharded range calls are K1).
  void set_sumfact(bool on) { sf_on = on && (sf_flux_ok || sf_dir_ok); }
  // the GEMM source prefixes at t (flux: smallest over the faces; Dirichlet), host only
  void sf_prefixes(double t, int* out);
  bool sf_on = false, sf_flux_ok = false, sf_dir_ok = false;
  double sf_flops = 0.0;   // GEMM flops issued (2 na nb Jpad per set)
  double sf_pairs = 0.0;   // point x source pairs taken off K1
  int sf_last_j[2] = {0, 0};  // source prefix of the last flux / Dirichlet call
  int sf_kc = 2048;           // sources per GEMM chunk (one batch entry; TG_SF_KC)
  double sf_min_pairs = 3e7;  // smallest J x points worth a GEMM (TG_SF_MIN_PAIRS)
  int sf_bands = 1;           // bands of element rows per face (TG_SF_BANDS; see DESIGN K5)

  bool focus_at(double t, Vec3& focus) const;
  int fine_elements(double t, double radius);  // fills h_fine, returns the count

  // ---- host setup
  RunConfig cfg;
  NurbsVolume vol;
  DofMap dofs;
  std::array<int, 3> quad{0, 0, 0};
  std::vector<PointSource> sources;
  std::vector<double> tact_max;
  double dt_solver = 0.0;
  int n_steps = 0;
  SimGeom geom{};
  int n_full = 0, n_free = 0, n_con = 0;
  int n_fe = 0, nqb = 0, nqf = 0, ndk = 0;
  std::vector<double> centers, h_qx, h_qn, h_qw, h_Nb, h_Nf, grev;
  std::vector<int> h_dofk, h_inc_ptr, h_inc_src, h_qb_off, h_qf_off;
  bool kron = false;
  std::array<Band1D, 3> band;
  std::array<double, 2> coefA{0, 0}, coefB{0, 0};
  Csr csrA, csrAc, csrB;

  // ---- device
  tg_ctx* ctx = nullptr;
  DevBuf<double> d_qx, d_qn, d_qw, d_Nb, d_Nf, d_gq, d_loc, d_grev, d_band;
  DevBuf<int> d_inc_ptr, d_inc_src, d_pt_index, d_elem_off, d_fine, d_free_list, d_qb_off,
      d_qf_off;
  struct SellBufs {
    DevBuf<long long> sp;
    DevBuf<int> len, col;
    DevBuf<double> val;
  };
  SellBufs sA, sAc, sB;
  DevSell devA{}, devAc{}, devB{};
  KronGrid gfull{}, gfree{};
  DevBuf<double> d_x, d_r, d_z, d_p, d_p2, d_Ap, d_invd, d_rhs, d_gn, d_g1, d_Fn, d_F1, d_T, d_gfull,
      d_partials;
  PcgMaps maps{};
  // single-sweep solve (k2_cg1_solve): the default when TMA can address the
  // free grid; TG_K2_ALGO=pcg selects the two-phase kernel
  int cg1_pl = 2;  // planes per sweep step of the single-sweep solver
  bool use_cg1 = false;
  // fast-diagonalization preconditioner (k2_fdm.cuh), opt-in
  bool use_fdm = false;
  FdmDev fdm{};
  DevBuf<double> d_fdmV, d_fdmL, d_fdmDinv, d_dots;
  double* h_dots = nullptr;
  cublasHandle_t cublas = nullptr;
  Cg1Maps cg1maps{};
  DevBuf<double> d_w2, d_s2;
  // observers: the patch on the device (uploaded on first use) and scratch
  NurbsDev nurbs{};
  bool nurbs_up = false;
  DevBuf<double> d_knots, d_cpts, d_px, d_pf, d_pval, d_pgrad;
  DevBuf<int> d_eflags;
  void upload_nurbs();
  TensorMap3 map_T{}, map_g{};
  bool rhs_tma = false;
  DevBuf<PcgStatus> d_status;
  DevBuf<unsigned long long> d_trace;  // K2 phase stamps (TG_K2_TRACE)
  bool trace_on = false;
  PcgStatus* h_status = nullptr;
  int* h_fine = nullptr;
  int pcg_blocks = 1;
  bool diag_ok = true;
  int step = 0;
  long k2_iterations = 0;

 private:
  void setup_host();
  void setup_device(int device, int preconditioner);
  void sf_setup_host();    // grids, face boxes (host only)
  void sf_setup_device();  // uploads
  std::vector<int> sf_h_gcell, sf_h_gaxn, sf_h_fa, sf_h_fb, sf_h_ff;  // until uploaded
  int sf_g_total = 0;
  struct SfPrefix {
    int J = 0;
    double t = 0.0;
    bool valid = false;  // [0, J) were all causally active at t (reusable at later t)
  };
  int sf_prefix(double t, const double lo[3], const double hi[3], double delta, SfPrefix& c);
  // end of the K1 source range [begin, end): trailing sources culled on the whole box drop out
  int sf_suffix_end(double t, const double lo[3], const double hi[3], int begin);
  std::vector<SfGrid> sf_faces;
  std::vector<SfDev> sf_faces_dev;
  std::vector<int> sf_faces_off;
  bool sf_fine_ok = false;  // fine-rule points gridded per face too
  bool sf_face_split = false;  // per-face source prefixes (face boxes)
  std::vector<int> sf_face_e;  // per face: element range [begin, end)
  std::vector<double> sf_face_box, sf_face_delta;
  std::vector<SfPrefix> sf_pf_face;
  std::vector<SfGrid> sf_fine;
  std::vector<SfDev> sf_fine_dev;
  std::vector<int> sf_elem_face, sf_erect;  // per face element: face, fine-cell rectangle
  DevBuf<int> d_sf_fa, d_sf_fb, d_sf_ff, d_sf_rect;
  DevBuf<double> d_sf_Gf;
  int* h_sf_rect = nullptr;
  cudaStream_t sf_stream = nullptr;  // K1 remainder beside the GEMMs (TG_SF_SERIAL=1: one stream)
  cudaEvent_t sf_ev[2] = {nullptr, nullptr};
  SfGrid sf_dir;
  SfDev sf_dir_dev{};
  double sf_lo[3] = {0, 0, 0}, sf_hi[3] = {0, 0, 0}, sf_delta = 0.0;
  SfPrefix sf_pf_flux, sf_pf_dir;
  DevBuf<double> d_sf_uv, d_sf_G, d_sf_Gdir, d_sf_vec, d_sf_A, d_sf_B, d_sf_C, d_sf_tmp;
  DevBuf<int> d_sf_gcell, d_sf_gaxn, d_sf_dcell, d_sf_fine;
  int* h_sf_fine = nullptr;  // pinned: fine compact positions, then their qp ids
  SfScratch sf_scratch(int na, int nb, int J);
};

}  // namespace tgb

struct tg_sim {
  tgb::Sim* sim = nullptr;
  std::string err;
};
