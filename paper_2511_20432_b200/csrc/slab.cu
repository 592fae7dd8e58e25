// Multi-GPU θ-step solve: Jacobi-PCG (the reference's pcg_jacobi,
// proj/src/sparse.cpp:41-100, in the Chronopoulos-Gear single-sweep form of
// k2_cg1_kernel) on the free grid cut into z-slabs, one per GPU.
//
// Per iteration every rank runs one sweep of its slab (k2_slab_kernel: the
// prologue / stencil / epilogue of the single-GPU kernel, dot products over
// its own planes only) and then, on the same stream, one NCCL group: the P
// ghost planes of w^ = D^-1 A u to / from each neighbour (contiguous planes:
// no packing) and an all-gather of the 4 partial sums. The next launch sums
// the partials in rank order, so every rank takes the same alpha, beta and
// stop decision; the vectors' ghost planes hold bit-identical copies of the
// neighbours' own values. The host looks at the solver state every
// kCheckEvery sweeps. After the solve each rank broadcasts its own planes of
// x, so all ranks continue from the same full state.
//
// Local mode (no communicator): one process runs all slabs on its GPU in
// turn and exchanges the same halos / partials with device copies. It
// checks the decomposition on one GPU without any kernel waiting on another.
#include "slab.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

namespace tgb {

SlabPlan slab_plan(int nz, int p, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("slab: bad rank / world");
  if (nz / world < p) throw std::invalid_argument("slab: fewer own planes than the halo depth");
  const int z0 = static_cast<int>(static_cast<long>(nz) * rank / world);
  const int z1 = static_cast<int>(static_cast<long>(nz) * (rank + 1) / world);
  SlabPlan s{};
  s.gz0 = rank > 0 ? z0 - p : 0;
  const int gend = rank + 1 < world ? z1 + p : nz;
  s.nloc = gend - s.gz0;
  s.zo0 = z0 - s.gz0;
  s.zo1 = z1 - s.gz0;
  s.lo = rank > 0 ? rank - 1 : -1;
  s.hi = rank + 1 < world ? rank + 1 : -1;
  return s;
}

// ---------------------------------------------------------------- NCCL
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a = [] {
    NcclApi n;
    // TG_NCCL_LIB (the Python binding points it at torch's bundled copy), the
    // copy already in the process, else the loader's search path
    void* h = nullptr;
    if (const char* e = std::getenv("TG_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return n;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      return f != nullptr;
    };
    n.ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
           sym(n.CommDestroy, "ncclCommDestroy") && sym(n.Send, "ncclSend") &&
           sym(n.Recv, "ncclRecv") && sym(n.AllGather, "ncclAllGather") &&
           sym(n.AllReduce, "ncclAllReduce") && sym(n.Broadcast, "ncclBroadcast") &&
           sym(n.GroupStart, "ncclGroupStart") && sym(n.GroupEnd, "ncclGroupEnd") &&
           sym(n.ErrorString, "ncclGetErrorString") && sym(n.CommAbort, "ncclCommAbort");
    return n;
  }();
  return a;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw cuda_error(std::string("nccl: ") + what + ": " + api().ErrorString(r));
}

}  // namespace

struct NcclComm {
  ncclComm_t c = nullptr;
  int rank = 0, world = 1;
  ~NcclComm() {
    if (c) api().CommDestroy(c);
  }
};

bool nccl_available() { return api().ok; }

void nccl_unique_id(char out[128]) {
  if (!api().ok) throw cuda_error("nccl: libnccl.so.2 not found");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  nccl_ok(api().GetUniqueId(&id), "get unique id");
  std::memcpy(out, &id, 128);
}

std::shared_ptr<NcclComm> nccl_comm(int rank, int world, const char id[128], int device) {
  if (!api().ok) throw cuda_error("nccl: libnccl.so.2 not found");
  TG_CUDA(cudaSetDevice(device));
  auto c = std::make_shared<NcclComm>();
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  nccl_ok(api().CommInitRank(&c->c, world, uid, rank), "comm init");
  c->rank = rank;
  c->world = world;
  return c;
}

void stream_wait(NcclComm* c, cudaStream_t s) {
  if (!c || c->world == 1) {
    TG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  // a rank that never joins a collective must not hang the others forever:
  // poll, and abort the communicator after TG_NCCL_TIMEOUT seconds (120)
  static const double limit = [] {
    const char* e = std::getenv("TG_NCCL_TIMEOUT");
    return e ? std::atof(e) : 120.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) TG_CUDA(q);
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
      if (c->c) api().CommAbort(c->c);
      c->c = nullptr;
      throw cuda_error("multi-GPU step timed out (a rank missed a collective); NCCL aborted");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

void nccl_allreduce_sum(NcclComm& c, double* buf, size_t n, cudaStream_t s) {
  if (n == 0 || c.world == 1) return;
  nccl_ok(api().AllReduce(buf, buf, n, ncclDouble, ncclSum, c.c, s), "all-reduce");
}

void nccl_broadcast_parts(NcclComm& c, double* buf, const std::vector<size_t>& off,
                          const std::vector<size_t>& count, cudaStream_t s) {
  if (c.world == 1) return;
  nccl_ok(api().GroupStart(), "group start");
  for (int r = 0; r < c.world; ++r)
    nccl_ok(api().Broadcast(buf + off[r], buf + off[r], count[r], ncclDouble, r, c.c, s),
            "broadcast");
  nccl_ok(api().GroupEnd(), "group end");
}

// ---------------------------------------------------------------- solver
namespace {
constexpr int kCheckEvery = 4;  // sweeps between host looks at the solver state

__global__ void slab_status_kernel(const SlabState* st, PcgStatus* out) {
  *out = PcgStatus{st->it, st->status, st->rel, st->bnorm};
}
}  // namespace

struct SlabSolver::Rank {
  int rank = 0;
  SlabPlan plan{};
  KronGrid g{};
  DevBuf<double> x, rhs, u[2], w[2], s[2], p, gath, mine, cta;
  DevBuf<SlabState> st;
  DevBuf<unsigned int> ticket;
  Cg1Maps maps{};
  int blocks = 0;
};

SlabSolver::SlabSolver(const KronGrid& gfree, int world, int rank, std::shared_ptr<NcclComm> comm,
                       int sm_count, int pl)
    : gfree_(gfree), world_(world), rank_(rank), pl_(pl), comm_(std::move(comm)) {
  plane_ = static_cast<size_t>(gfree.n[0]) * gfree.n[1];
  const int W = 2 * gfree.p + 1;
  const int first = comm_ ? rank : 0, last = comm_ ? rank + 1 : world;
  for (int r = first; r < last; ++r) {
    auto R = std::make_unique<Rank>();
    R->rank = r;
    R->plan = slab_plan(gfree.n[2], gfree.p, world, r);
    R->g = gfree;
    R->g.n[2] = R->plan.nloc;
    R->g.M[2] = gfree.M[2] + static_cast<size_t>(R->plan.gz0) * W;
    R->g.K[2] = gfree.K[2] + static_cast<size_t>(R->plan.gz0) * W;
    const size_t n = plane_ * R->plan.nloc;
    for (auto* b : {&R->x, &R->rhs, &R->u[0], &R->u[1], &R->w[0], &R->w[1], &R->s[0], &R->s[1],
                    &R->p}) {
      b->ensure(n);
      TG_CUDA(cudaMemset(b->p, 0, n * sizeof(double)));
    }
    R->gath.ensure(4 * static_cast<size_t>(world));
    R->mine.ensure(4);
    R->st.ensure(2);
    R->ticket.ensure(1);
    TG_CUDA(cudaMemset(R->gath.p, 0, 4 * world * sizeof(double)));
    TG_CUDA(cudaMemset(R->ticket.p, 0, sizeof(unsigned int)));
    const KronGrid& g = R->g;
    const int L = pl;
    Cg1Maps& m = R->maps;
    const bool ok = k2_make_map(g, R->x.p, &m.x, true, L) &&
                    k2_make_map(g, R->u[0].p, &m.r[0], true, L) &&
                    k2_make_map(g, R->u[1].p, &m.r[1], true, L) &&
                    k2_make_map(g, R->w[0].p, &m.w[0], true, L) &&
                    k2_make_map(g, R->w[1].p, &m.w[1], true, L) &&
                    k2_make_map(g, R->s[0].p, &m.s[0], true, L) &&
                    k2_make_map(g, R->s[1].p, &m.s[1], true, L) &&
                    k2_make_map(g, R->x.p, &m.xc, false, L) &&
                    k2_make_map(g, R->p.p, &m.pc, false, L);
    if (!ok) throw std::invalid_argument("slab: TMA cannot address the slab grid");
    R->blocks = k2_slab_max_blocks(g.p, sm_count, g.n[2], pl);
    R->cta.ensure(4 * static_cast<size_t>(R->blocks) + 4);
    ranks_.push_back(std::move(R));
  }
  TG_CUDA(cudaMallocHost(&h_state_, sizeof(SlabState)));
}

SlabSolver::~SlabSolver() {
  if (h_state_) cudaFreeHost(h_state_);
}

double* SlabSolver::vec_of(Rank& r, int kind, int cur) {
  return kind == 0 ? r.u[cur].p : r.w[cur].p;
}

// after a sweep: the ghost planes of the vector it wrote, and the partials
void SlabSolver::exchange(int kind, int cur, cudaStream_t s) {
  const int P = gfree_.p;
  const size_t halo = static_cast<size_t>(P) * plane_;
  if (comm_) {
    Rank& r = *ranks_[0];
    double* v = vec_of(r, kind, cur);
    NcclApi& n = api();
    nccl_ok(n.GroupStart(), "group start");
    if (r.plan.lo >= 0) {
      nccl_ok(n.Send(v + r.plan.zo0 * plane_, halo, ncclDouble, r.plan.lo, comm_->c, s), "send");
      nccl_ok(n.Recv(v, halo, ncclDouble, r.plan.lo, comm_->c, s), "recv");
    }
    if (r.plan.hi >= 0) {
      nccl_ok(n.Send(v + (r.plan.zo1 - P) * plane_, halo, ncclDouble, r.plan.hi, comm_->c, s),
              "send");
      nccl_ok(n.Recv(v + r.plan.zo1 * plane_, halo, ncclDouble, r.plan.hi, comm_->c, s), "recv");
    }
    nccl_ok(n.AllGather(r.mine.p, r.gath.p, 4, ncclDouble, comm_->c, s), "all-gather");
    nccl_ok(n.GroupEnd(), "group end");
    return;
  }
  for (size_t i = 0; i < ranks_.size(); ++i) {
    Rank& r = *ranks_[i];
    double* v = vec_of(r, kind, cur);
    if (r.plan.lo >= 0) {
      Rank& q = *ranks_[i - 1];
      TG_CUDA(cudaMemcpyAsync(v, vec_of(q, kind, cur) + (q.plan.zo1 - P) * plane_,
                              halo * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    if (r.plan.hi >= 0) {
      Rank& q = *ranks_[i + 1];
      TG_CUDA(cudaMemcpyAsync(v + r.plan.zo1 * plane_, vec_of(q, kind, cur) + q.plan.zo0 * plane_,
                              halo * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    for (size_t q = 0; q < ranks_.size(); ++q)
      TG_CUDA(cudaMemcpyAsync(r.gath.p + 4 * q, ranks_[q]->mine.p, 4 * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
  }
}

void SlabSolver::solve(const double* d_rhs, double* d_x, double a, double b, double tol,
                       int max_iter, PcgStatus* d_status, cudaStream_t s) {
  for (auto& R : ranks_) {  // the slab of the warm start and of the right-hand side
    const size_t off = static_cast<size_t>(R->plan.gz0) * plane_, n = plane_ * R->plan.nloc;
    TG_CUDA(cudaMemcpyAsync(R->x.p, d_x + off, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    TG_CUDA(cudaMemcpyAsync(R->rhs.p, d_rhs + off, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  int launch = 0;
  auto sweep = [&](int phase, int cur) {
    for (auto& R : ranks_) {
      Cg1Work w{R->p.p, {R->u[0].p, R->u[1].p}, {R->w[0].p, R->w[1].p}, {R->s[0].p, R->s[1].p},
                nullptr, nullptr, nullptr};
      SlabCtl ctl{phase, cur, R->plan.zo0, R->plan.zo1, world_, R->gath.p, R->mine.p,
                  R->st.p + (launch & 1), R->st.p + ((launch + 1) & 1), R->cta.p, R->ticket.p};
      k2_slab_launch(R->g, a, b, R->rhs.p, R->x.p, w, R->maps, tol, max_iter, R->blocks, ctl, s,
                     pl_);
      ++launches;
    }
    ++launch;
  };
  sweep(0, 0);  // r0, u0
  exchange(0, 0, s);
  sweep(1, 0);  // w^0
  exchange(1, 0, s);
  int cur = 0;
  const int cap = max_iter + 2;
  for (int k = 0; k <= cap; ++k) {
    sweep(2, cur);
    exchange(1, cur ^ 1, s);
    cur ^= 1;
    if ((k + 1) % kCheckEvery == 0 || k == cap) {
      // the state the last launch wrote (identical on every slab)
      TG_CUDA(cudaMemcpyAsync(h_state_, ranks_[0]->st.p + (launch & 1), sizeof(SlabState),
                              cudaMemcpyDeviceToHost, s));
      stream_wait(comm_.get(), s);
      if (h_state_->done) break;
    }
  }
  // the final state: the launch after the deciding one copies it forward
  slab_status_kernel<<<1, 1, 0, s>>>(ranks_[0]->st.p + (launch & 1), d_status);
  // own planes back into the full vector; every rank ends with all of x
  std::vector<size_t> off(world_), cnt(world_);
  for (int r = 0; r < world_; ++r) {
    const SlabPlan q = slab_plan(gfree_.n[2], gfree_.p, world_, r);
    off[r] = static_cast<size_t>(q.gz0 + q.zo0) * plane_;
    cnt[r] = static_cast<size_t>(q.zo1 - q.zo0) * plane_;
  }
  for (auto& R : ranks_)
    TG_CUDA(cudaMemcpyAsync(d_x + off[R->rank], R->x.p + R->plan.zo0 * plane_,
                            cnt[R->rank] * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (comm_) nccl_broadcast_parts(*comm_, d_x, off, cnt, s);
  TG_CUDA(cudaGetLastError());
}

}  // namespace tgb
