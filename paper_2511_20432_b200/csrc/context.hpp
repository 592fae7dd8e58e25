// Device context behind the C ABI: one CUDA stream, grow-only device buffers,
// the uploaded scan history and the profiling counters.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/thermiga_b200.h"
#include "host/analytic.hpp"
#include "k1_superpose.cuh"

namespace tgb {

struct cuda_error : std::runtime_error {
  explicit cuda_error(const std::string& m) : std::runtime_error(m) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw cuda_error(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define TG_CUDA(call) ::tgb::cuda_check((call), #call)

// Grow-only device allocation.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  // grows with 25 % headroom once a buffer has been sized (per-step sizes
  // such as the flux-load point count vary by a few percent; a reallocation
  // synchronizes the device and costs milliseconds at config-4 sizes)
  T* ensure(size_t n) {
    if (n > cap) {
      const size_t want = cap > 0 ? n + n / 4 : n;
      if (p) TG_CUDA(cudaFree(p));
      p = nullptr;
      cap = 0;
      TG_CUDA(cudaMalloc(&p, std::max<size_t>(want, 1) * sizeof(T)));
      cap = want;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Per-kernel event timing for the roofline (CUDA events on the launch stream).
struct KernelTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> live;  // pending pairs
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  // kinds 1 (K1 main), 2 (K2 main), 3 (whole theta step), 4 (whole time
  // steps: loads + theta step), 5 (K5 contraction)
  double k1_ms = 0.0, k2_ms = 0.0, step_ms = 0.0, k5_ms = 0.0, run_ms = 0.0;
  std::vector<int> kinds;
  double k1_pairs = 0.0, k2_bytes = 0.0;
  long launches = 0, k1_launches = 0, k2_launches = 0, k5_launches = 0;

  std::pair<cudaEvent_t, cudaEvent_t> get() {
    if (!pool.empty()) {
      auto e = pool.back();
      pool.pop_back();
      return e;
    }
    std::pair<cudaEvent_t, cudaEvent_t> e;
    TG_CUDA(cudaEventCreate(&e.first));
    TG_CUDA(cudaEventCreate(&e.second));
    return e;
  }
  // Bracket one launch of kernel class `kind` (1 = K1 main, 2 = K2 main).
  template <typename F>
  void timed(int kind, cudaStream_t s, F&& launch) {
    if (!on) {
      launch();
      return;
    }
    auto e = get();
    TG_CUDA(cudaEventRecord(e.first, s));
    launch();
    TG_CUDA(cudaEventRecord(e.second, s));
    live.push_back(e);
    kinds.push_back(kind);
  }
  void collect() {
    for (size_t i = 0; i < live.size(); ++i) {
      TG_CUDA(cudaEventSynchronize(live[i].second));
      float ms = 0.f;
      TG_CUDA(cudaEventElapsedTime(&ms, live[i].first, live[i].second));
      (kinds[i] == 1 ? k1_ms : kinds[i] == 2 ? k2_ms : kinds[i] == 5 ? k5_ms
                                     : kinds[i] == 4 ? run_ms : step_ms) += ms;
      pool.push_back(live[i]);
    }
    live.clear();
    kinds.clear();
  }
  void reset() {
    collect();
    k1_ms = k2_ms = step_ms = k5_ms = run_ms = 0.0;
    k1_pairs = k2_bytes = 0.0;
    launches = k1_launches = k2_launches = k5_launches = 0;
  }
  ~KernelTimer() {
    for (auto& e : live) pool.push_back(e);
    for (auto& e : pool) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  }
};

}  // namespace tgb

struct tg_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  tgb::KernelTimer timer;

  // K1 state
  tgb::Material mat;
  int n_src = 0;
  // suffix minima of the sources' modified times tau: sources [j, n) are all
  // causally inactive at t (t - tau <= 0) iff tau_sufmin[j] >= t, so K1 runs
  // over the active prefix only (the skipped pairs are exact zeros)
  std::vector<double> tau_sufmin;
  int active_prefix(double t) const {
    const auto it = std::lower_bound(tau_sufmin.begin(), tau_sufmin.end(), t);
    return static_cast<int>(it - tau_sufmin.begin());
  }
  // all sources on one plane z = planar_z (k1_partial's PLANAR variant)
  bool planar = false;
  double planar_z = 0.0;
  void set_tau(const double* src6_host, int n) {
    planar = n > 0;
    planar_z = n > 0 ? src6_host[2] : 0.0;
    for (int j = 1; j < n && planar; ++j)
      planar = __builtin_memcmp(&src6_host[6 * j + 2], &planar_z, sizeof(double)) == 0;
    tau_sufmin.assign(n, 0.0);
    double m = INFINITY;
    for (int j = n - 1; j >= 0; --j) tau_sufmin[j] = m = std::min(m, src6_host[6 * j + 5]);
  }
  tgb::DevBuf<double> src6;
  tgb::DevBuf<tgb::SrcRec> rec;
  tgb::DevBuf<double> part;
  tgb::DevBuf<double> pts, val, grad;
  // measured (config 1, 17 FP64 ops/pair, unroll 4): P=7 82.4 ms, P=6 83.9, P=8 89.7, P=5 94.6
  int k1_points_per_thread = 7;
  // value-only launches (Dirichlet, field without grad), config 1: P=5 64.7 ms, 4 65.5, 7 67.2
  int k1_points_per_thread_value = 5;

  // device-pointer entry points run on the caller's stream (NULL = legacy default)
  static cudaStream_t pick(void* s) { return static_cast<cudaStream_t>(s); }
};

namespace tgb {

// K1 on device arrays: prepare the per-time source records, run the partial
// kernel over S source splits, then the epilogue selected by `mode`.
enum class K1Mode { field, dirichlet, flux };

struct K1Flux {
  const int* index = nullptr;      // qp ids of the points (nullable = identity)
  const double* normals = nullptr; // per qp
  const double* weights = nullptr; // per qp
  double k = 0.0;
};

void k1_run(tg_ctx* ctx, const double* d_src6, int n_src, const double* d_pts,
            const int* d_index, long n_pts, double t, double cull, K1Mode mode, double* d_out_a,
            double* d_out_b, const K1Flux& flux, cudaStream_t stream, int src_begin = 0,
            int src_end = -1);

}  // namespace tgb
