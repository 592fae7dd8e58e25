// Multi-GPU θ-step: the free grid cut into z-slabs, one per rank (see slab.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "context.hpp"
#include "k2_kron.cuh"

namespace tgb {

// One rank's slab of nz planes: own planes [z0, z1) (global), stored with P
// ghost planes on each interior side as local planes [0, nloc) = global
// [gz0, gz0 + nloc); own planes are local [zo0, zo1). lo / hi: the
// neighbouring ranks (-1 at the grid's ends).
struct SlabPlan {
  int gz0, nloc, zo0, zo1, lo, hi;
};
// Equal shares of the planes; needs nz / world >= P (ghosts come from the
// adjacent rank only). Pure host arithmetic.
SlabPlan slab_plan(int nz, int p, int world, int rank);

// NCCL, bound at run time (libnccl.so.2: the copy a torch process already
// loaded, else the system's): only the multi-GPU path needs it.
struct NcclComm;
bool nccl_available();
void nccl_unique_id(char out[128]);
std::shared_ptr<NcclComm> nccl_comm(int rank, int world, const char id[128], int device);
void nccl_allreduce_sum(NcclComm& c, double* buf, size_t n, cudaStream_t s);
// cudaStreamSynchronize, bounded in time when a multi-rank communicator is in
// use (the communicator is aborted and cuda_error thrown after TG_NCCL_TIMEOUT s)
void stream_wait(NcclComm* c, cudaStream_t s);
void nccl_broadcast_parts(NcclComm& c, double* buf, const std::vector<size_t>& off,
                          const std::vector<size_t>& count, cudaStream_t s);

class SlabSolver {
 public:
  // NCCL mode: this process is rank `rank` of `comm`; local mode (comm null):
  // this process runs all `world` slabs on its one GPU, in turn, and
  // exchanges halos / partials with device copies (the decomposition's test
  // bed: no kernel ever waits on another)
  SlabSolver(const KronGrid& gfree, int world, int rank, std::shared_ptr<NcclComm> comm,
             int sm_count, int pl);
  ~SlabSolver();
  // x (full free vector) in: warm start; out: the solution on every rank.
  // Writes the PcgStatus to d_status.
  void solve(const double* d_rhs, double* d_x, double a, double b, double tol, int max_iter,
             PcgStatus* d_status, cudaStream_t s);
  int world() const { return world_; }
  long launches = 0;

 private:
  struct Rank;
  void exchange(int vec_kind, int cur, cudaStream_t s);
  double* vec_of(Rank& r, int kind, int cur);
  KronGrid gfree_;
  int world_, rank_, pl_;
  size_t plane_;
  std::shared_ptr<NcclComm> comm_;
  std::vector<std::unique_ptr<Rank>> ranks_;  // 1 (NCCL) or world (local)
  SlabState* h_state_ = nullptr;
};

}  // namespace tgb
