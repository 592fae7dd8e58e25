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
#include "k5_fused.cuh"
#include "k6_assemble.cuh"
#include "k5_sumfact.cuh"
#include "slab.hpp"

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
  // n steps without host synchronisation between them (statuses read at the
  // end); returns the CG iterations
  long advance_steps(int n, double* last_rel);

  // drop-in pieces on device buffers
  // assemble_flux_load; with [e0, e1) only those face elements' local loads
  // (d_loc) are computed, and d_F == nullptr skips the gather (sharded use)
  void flux_load_device(double t, double radius, double* d_F, int e0 = 0,
                        int e1 = 1 << 30);
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

  // K5 (k5_fused.cuh): the superposition on the gridded face / Greville point
  // sets of an axis-aligned patch as a fused on-chip contraction over the
  // sources no cull can reach in each region, with the pair-wise remainder on
  // K1. On by default where the sets are grids (TG_SUMFACT=0 or
  // set_sumfact(false): every pair through K1, with the same per-region
  // source ranges).
  void set_sumfact(bool on) { sf_on = on && (sf_flux_ok || sf_dir_ok); }
  // host restatement of the device plan at t for the static regions (flux
  // tiles, then Greville tiles): J (contraction prefix), E (remainder end)
  void sf_plan_host(double t, int* J, int* E, int* Jc = nullptr);
  bool sf_on = false, sf_flux_ok = false, sf_dir_ok = false;
  // contraction flops (2 per point x source) since setup, read from the device
  double sf_flops_total();
  double sf_min_pairs = 3e7;  // smallest J x points worth a contraction (TG_SF_MIN_PAIRS)
  int sf_min_sources = 16384;  // ... unless J reaches this (TG_SF_MIN_SOURCES)
  int sf_k1_splits = 4;       // source splits of the remainder launch (TG_SF_K1_SPLITS)
  // the device plan of the static regions, each part (flux / Greville) as its
  // last call computed it, read back on request
  void sf_last_plan(int* J, int* E, int* Jc = nullptr);
  int sf_n_regions() const { return static_cast<int>(sf_regions_h.size()); }
  int sf_dir_regions() const { return sf_nt_static - sf_nt_flux; }
  const std::vector<SfRegion>& sf_regions() const { return sf_regions_h; }
  // multi-GPU: this rank computes the regions r with r % world == rank
  int sf_rank = 0, sf_world = 1;
  // the fused loads path: F (d_F may be null) and/or g at t. gather = false
  // leaves the (rank-partial) compact integrand in d_gq without the K3 local
  // loads and gather (multi-GPU: all-reduced by the caller, then flux_finish)
  void loads_device(double t, double radius, double* d_F, double* d_g, bool gather = true);
  void flux_finish(double* d_F);  // k3_local + gather over all elements from d_gq
  bool sf_fused_ready() const { return sf_ready; }
  long sf_compact_points() const { return sf_last_npts; }

  // multi-GPU (slab.hpp): shard(rank, world, id) joins an NCCL communicator;
  // the loads' K5 regions and the θ-step solve's z-slabs are then split over
  // the ranks (the loads all-reduced, x broadcast after each solve).
  // set_slabs(n): the same slab solve with n slabs on this one GPU.
  void shard(int rank, int world, const char id[128]);
  void set_slabs(int n);
  std::unique_ptr<SlabSolver> slab;
  std::shared_ptr<NcclComm> comm;
  // F_{n+1} and g_{n+1} of a step at t (fused / sharded / K1 paths)
  void step_loads(double t, double* d_F, double* d_g);

  bool focus_at(double t, Vec3& focus) const;
  // a caller-given fine-rule focus for the next flux-load call (tg_sim_flux_load's
  // focus_xyz) instead of the newest active source (assembly.cpp:153-157)
  bool focus_given = false;
  Vec3 focus_value{};
  int fine_elements(double t, double radius);  // fills h_fine, returns the count
  std::vector<int> h_fine;  // fine elements (sorted), then the running extra-point counts

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
  bool faces_deferred = false;  // face tables built on the device (face_tables_device)
  std::vector<FaceElemSpec> face_specs;
  void face_tables_host(const FaceSets& fs);
  void face_tables_device(cudaStream_t s);
  void face_tables_to_host();
  void build_incidence();
  bool csr_deferred = false;  // assemble the general operators on the device (setup_device)
  bool csr_device = false;    // ... and it did (csrA then only on demand: reduced_operator)
  void assemble_csr_host();
  bool assemble_csr_device(cudaStream_t s);
  const Csr& reduced_operator();

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
  // A_ff with implicit columns on the free box (k2_csr.cuh DevDia): the solve's
  // operator when every entry lies in the (2p+1)^3 stencil (TG_K2_NO_DIA: SELL)
  DevDia devAd{};
  bool use_dia = false;
  DevBuf<double> d_dia;
  DevBuf<int> d_dia_flag;
  KronGrid gfull{}, gfree{};
  DevBuf<double> d_x, d_r, d_z, d_p, d_p2, d_Ap, d_invd, d_rhs, d_gn, d_g1, d_Fn, d_F1, d_T, d_gfull,
      d_partials;
  PcgMaps maps{};
  // single-sweep solve (k2_cg1_solve): the default when TMA can address the
  // free grid; TG_K2_ALGO=pcg selects the two-phase kernel
  int cg1_pl = 2;  // planes per sweep step of the single-sweep solver
  bool use_cg1 = false;
  bool use_res = false;  // small grids: k2_res_solve (state resident in shared memory)
  K2ResPlan res_plan{};
  // fast-diagonalization preconditioner (k2_fdm.cuh), opt-in
  bool use_fdm = false;
  FdmDev fdm{};
  DevBuf<double> d_fdmV, d_fdmL, d_fdmDinv, d_fdmS, d_dots;
  double* h_dots = nullptr;
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
  PcgStatus* h_steps = nullptr;  // pinned per-step statuses of advance_steps
  size_t h_steps_cap = 0;
  int pcg_blocks = 1;
  bool diag_ok = true;
  int step = 0;
  long k2_iterations = 0;

 private:
  void setup_host();
  void setup_device(int device, int preconditioner);
  void setup_general_fdm(cudaStream_t s);
  void sf_setup_host();    // grids, tiles, regions, remainder entries (host only)
  void sf_setup_device();  // uploads
  std::vector<int> sf_h_gcell, sf_h_fa, sf_h_fb, sf_h_ff;  // until the entry lists are built
  std::vector<SfGrid> sf_faces;           // base grid per face
  std::vector<SfGrid> sf_fine;            // fine grid per face (sf_fine_ok)
  SfGrid sf_dir;
  bool sf_fine_ok = false;
  std::vector<int> sf_elem_face, sf_erect;  // per face element: face, fine-cell rectangle
  // static tables: grids (faces, fine faces, Greville), tiles / regions
  // (flux base tiles [0, sf_nt_flux), Greville tiles [sf_nt_flux, sf_nt_static)),
  // remainder entries (flux base [0, sf_ne_flux), Greville [.., sf_ne_static))
  std::vector<SfGridDesc> sf_grids_h;
  std::vector<SfTile> sf_tiles_h;
  std::vector<SfRegion> sf_regions_h;
  std::vector<int> sf_ent_q, sf_ent_tile, sf_ent_cell, sf_ent_pos, sf_cta_region;
  int sf_nt_flux = 0, sf_nt_static = 0, sf_ne_flux = 0, sf_ne_static = 0;
  int sf_nc_flux = 0, sf_nc_static = 0;  // remainder CTAs
  int sf_grid_fine0 = 0, sf_grid_dir = -1;
  double sf_vplane = 0.0;
  bool sf_ready = false;
  long sf_last_npts = 0;
  int sf_k1_ppc = 0;  // remainder points per K1 CTA
  DevBuf<double> d_sf_lines, d_sf_cb, d_sf_tab, d_sf_scratch, d_sf_stats;
  DevBuf<SfGridDesc> d_sf_grids;
  DevBuf<SfTile> d_sf_tiles;
  DevBuf<SfRegion> d_sf_regions;
  DevBuf<SfConst> d_sf_cst;
  DevBuf<int> d_sf_elist, d_sf_Jc, d_sf_Jcl;
  DevBuf<unsigned> d_sf_okbits;
  int sf_list_cap = 1, sf_list_words = 1;
  DevBuf<int> d_sf_J, d_sf_E, d_sf_Jl, d_sf_El, d_sf_Jraw, d_sf_prefix, d_sf_ent_q, d_sf_ent_tile, d_sf_ent_cell,
      d_sf_ent_pos, d_sf_cta, d_sf_qelem;
  // per-step host staging (pinned ring; an event marks when a slot's copies ran)
  struct Stage {
    char* h = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
  };
  Stage sf_stage[3];
  int sf_stage_i = 0;
  char* stage_bytes(size_t bytes);  // the next ring slot, grown / waited for as needed
  void release_stages();
};

}  // namespace tgb

struct tg_sim {
  tgb::Sim* sim = nullptr;
  std::string err;
};
