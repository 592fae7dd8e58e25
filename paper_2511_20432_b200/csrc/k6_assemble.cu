// K6 — the general (non-separable) patch's θ-step operators assembled on the
// device: SURVEY.md §8f "GPU setup path" (assemble_matrix / element_quad,
// proj/src/assembly.cpp:59-101, proj/src/mesh.cpp:65-117; the θ operators
// and the free-row split, assembly.cpp:194-228).
//
// Bit-identical to the host assembly (host/operator.cpp, itself bit-identical
// to the reference's CSR, tests/test_cfg3.py): this file is compiled with
// -fmad=false, so every product and sum rounds separately, in the host's
// order:
//   * element matrices, one CTA per element: per Gauss point the rational
//     basis (basis_at, splines.cpp:212-255: w n1 n2 n3, sums W / dW in basis
//     order, then the quotient rule), J = sum_m P_m dN_m^T (basis order),
//     det / inverse (Mat3), w = g0 g1 g2 |box| det, G = J^-T dN; then per
//     lower-triangle entry (a, b), over the points in order,
//     m += (wm N_a) N_b and k += wk ((G_a.x G_b.x + G_a.y G_b.y) + G_a.z G_b.z);
//   * the scatter as a gather: each pattern entry (r, c) adds, in element
//     order, the one entry of every element whose span supports both r and c
//     (the host's scatter order: element order per entry);
//   * A = (1/dt) M + theta K and B = (1/dt) M - (1 - theta) K entrywise on the
//     free rows, split into A_ff / A_fc / B_f and written as sliced ELL.
#include <stdexcept>

#include "common.cuh"
#include "context.hpp"
#include "k6_assemble.cuh"
#include "nurbs_dev.cuh"

namespace tgb {

namespace {

constexpr int kThreads = 256;

struct Layout {
  int nb, T, nqp, Q, maxq, tabw;
  int o_tab, o_val, o_dv, o_W, o_dW, o_J, o_inv, o_w;  // offsets in doubles
  int doubles;
};

__host__ __device__ inline Layout layout_of(const AsmPatch& P) {
  Layout L{};
  const int p0 = P.V.p[0], p1 = P.V.p[1], p2 = P.V.p[2];
  L.nb = (p0 + 1) * (p1 + 1) * (p2 + 1);
  L.T = L.nb * (L.nb + 1) / 2;
  L.nqp = P.nq[0] * P.nq[1] * P.nq[2];
  L.Q = L.nqp < 1024 / L.nb ? L.nqp : (1024 / L.nb > 1 ? 1024 / L.nb : 1);
  if (L.Q > 28) L.Q = 28;  // 9 Q threads form the Jacobians
  L.maxq = P.nq[0] > P.nq[1] ? P.nq[0] : P.nq[1];
  if (P.nq[2] > L.maxq) L.maxq = P.nq[2];
  int pm = p0 > p1 ? p0 : p1;
  if (p2 > pm) pm = p2;
  L.tabw = 2 * (pm + 1);
  int o = 0;
  L.o_tab = o;
  o += 3 * L.maxq * L.tabw;
  L.o_val = o;
  o += L.Q * L.nb;
  L.o_dv = o;
  o += 3 * L.Q * L.nb;
  L.o_W = o;
  o += L.Q;
  L.o_dW = o;
  o += 3 * L.Q;
  L.o_J = o;
  o += 9 * L.Q;
  L.o_inv = o;
  o += 9 * L.Q;
  L.o_w = o;
  o += L.Q;
  L.doubles = o;
  return L;
}

// entry t of a packed lower triangle -> (a, b), b <= a
__device__ __forceinline__ void tri_ab(int t, int& a, int& b) {
  int x = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (x * (x + 1) / 2 > t) --x;
  while ((x + 1) * (x + 2) / 2 <= t) ++x;
  a = x;
  b = t - x * (x + 1) / 2;
}

template <int EPT>
__global__ void __launch_bounds__(kThreads)
    k6_element_kernel(AsmPatch P, int e0, double* __restrict__ lm, double* __restrict__ lk,
                      int* __restrict__ flags) {
  extern __shared__ double sm[];
  __shared__ int spn[3];
  const Layout L = layout_of(P);
  const int tid = threadIdx.x;
  const int e = e0 + blockIdx.x;
  const int p0 = P.V.p[0], p1 = P.V.p[1], p2 = P.V.p[2];
  const int el[3] = {e % P.n_el[0], (e / P.n_el[0]) % P.n_el[1], e / (P.n_el[0] * P.n_el[1])};
  double half[3], mid[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    half[d] = 0.5 * (P.bp[d][el[d] + 1] - P.bp[d][el[d]]);
    mid[d] = 0.5 * (P.bp[d][el[d] + 1] + P.bp[d][el[d]]);
  }
  const double box = half[0] * half[1] * half[2];
  double* tab = sm + L.o_tab;
  // 1D basis tables at the element's Gauss nodes (all nodes of a direction
  // share the element's span)
  if (tid < 3) spn[tid] = P.espan[tid][el[tid]];
  __syncthreads();
  if (tid < P.nq[0] + P.nq[1] + P.nq[2]) {
    const int d = tid < P.nq[0] ? 0 : (tid < P.nq[0] + P.nq[1] ? 1 : 2);
    const int a = tid - (d == 0 ? 0 : (d == 1 ? P.nq[0] : P.nq[0] + P.nq[1]));
    const double u = mid[d] + half[d] * P.gn[d][a];
    int span;
    if (!find_span(P.V.U[d], P.V.p[d], P.V.n[d], u, span) || span != spn[d]) atomicOr(flags, 1);
    basis_ders1(P.V.U[d], P.V.p[d], u, spn[d], tab + (d * L.maxq + a) * L.tabw);
  }
  __syncthreads();
  double am[EPT], ak[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) am[i] = ak[i] = 0.0;
  double* val = sm + L.o_val;
  double* dv = sm + L.o_dv;
  double* W = sm + L.o_W;
  double* dW = sm + L.o_dW;
  double* J = sm + L.o_J;
  double* inv = sm + L.o_inv;
  double* wq = sm + L.o_w;
  const int w0 = p0 + 1, w1 = p1 + 1;
  const double* pts = P.V.pts;
  auto gidx = [&](int i, int j, int k) {
    return static_cast<long>(spn[0] - p0 + i) +
           static_cast<long>(P.V.n[0]) *
               (static_cast<long>(spn[1] - p1 + j) + static_cast<long>(P.V.n[1]) * (spn[2] - p2 + k));
  };
  for (int q0 = 0; q0 < L.nqp; q0 += L.Q) {
    const int nqc = min(L.Q, L.nqp - q0);
    // (1) w n1 n2 n3 and its derivatives per (point, basis)
    for (int idx = tid; idx < nqc * L.nb; idx += kThreads) {
      const int qc = idx / L.nb, m = idx - qc * L.nb, q = q0 + qc;
      const int qa = q % P.nq[0], qb = (q / P.nq[0]) % P.nq[1], qz = q / (P.nq[0] * P.nq[1]);
      const int i = m % w0, j = (m / w0) % w1, k = m / (w0 * w1);
      const double* t0 = tab + (0 * L.maxq + qa) * L.tabw;
      const double* t1 = tab + (1 * L.maxq + qb) * L.tabw;
      const double* t2 = tab + (2 * L.maxq + qz) * L.tabw;
      const double n1 = t0[i], d1 = t0[p0 + 1 + i];
      const double n2 = t1[j], d2 = t1[p1 + 1 + j];
      const double n3 = t2[k], d3 = t2[p2 + 1 + k];
      const double w = pts[4 * gidx(i, j, k) + 3];
      val[idx] = w * n1 * n2 * n3;
      dv[3 * idx] = w * d1 * n2 * n3;
      dv[3 * idx + 1] = w * n1 * d2 * n3;
      dv[3 * idx + 2] = w * n1 * n2 * d3;
    }
    __syncthreads();
    // (2) W, dW in basis order
    if (tid < 4 * nqc) {
      const int qc = tid >> 2, c = tid & 3;
      double acc = 0.0;
      if (c == 0)
        for (int m = 0; m < L.nb; ++m) acc += val[qc * L.nb + m];
      else
        for (int m = 0; m < L.nb; ++m) acc += dv[3 * (qc * L.nb + m) + c - 1];
      if (c == 0) W[qc] = acc;
      else dW[3 * qc + c - 1] = acc;
    }
    __syncthreads();
    // (3) quotient rule: val /= W; dv = (dv - dW val) / W
    for (int idx = tid; idx < nqc * L.nb; idx += kThreads) {
      const int qc = idx / L.nb;
      const double v = val[idx] / W[qc];
      val[idx] = v;
#pragma unroll
      for (int c = 0; c < 3; ++c) dv[3 * idx + c] = (dv[3 * idx + c] - dW[3 * qc + c] * v) / W[qc];
    }
    __syncthreads();
    // (4) J(r, s) += P_m[r] dN_m[s] in basis order
    if (tid < 9 * nqc) {
      const int qc = tid / 9, rs = tid - 9 * qc, r = rs / 3, s = rs - 3 * r;
      double acc = 0.0;
      for (int m = 0; m < L.nb; ++m) {
        const int i = m % w0, j = (m / w0) % w1, k = m / (w0 * w1);
        acc += pts[4 * gidx(i, j, k) + r] * dv[3 * (qc * L.nb + m) + s];
      }
      J[9 * qc + rs] = acc;
    }
    __syncthreads();
    // (5) det, inverse, weight (Mat3::det / inverse, element_quad)
    if (tid < nqc) {
      const double* a = J + 9 * tid;
      const double det = det3(a);
      if (!(det > 0.0)) atomicOr(flags, 1);
      const double d = det;
      double* r = inv + 9 * tid;
      r[0] = (a[4] * a[8] - a[5] * a[7]) / d;
      r[1] = (a[2] * a[7] - a[1] * a[8]) / d;
      r[2] = (a[1] * a[5] - a[2] * a[4]) / d;
      r[3] = (a[5] * a[6] - a[3] * a[8]) / d;
      r[4] = (a[0] * a[8] - a[2] * a[6]) / d;
      r[5] = (a[2] * a[3] - a[0] * a[5]) / d;
      r[6] = (a[3] * a[7] - a[4] * a[6]) / d;
      r[7] = (a[1] * a[6] - a[0] * a[7]) / d;
      r[8] = (a[0] * a[4] - a[1] * a[3]) / d;
      const int q = q0 + tid;
      const int qa = q % P.nq[0], qb = (q / P.nq[0]) % P.nq[1], qz = q / (P.nq[0] * P.nq[1]);
      wq[tid] = P.gw[0][qa] * P.gw[1][qb] * P.gw[2][qz] * box * det;
    }
    __syncthreads();
    // (6) physical gradients G = J^-T dN (Mat3::apply_transposed)
    for (int idx = tid; idx < nqc * L.nb; idx += kThreads) {
      const double* a = inv + 9 * (idx / L.nb);
      const double x = dv[3 * idx], y = dv[3 * idx + 1], z = dv[3 * idx + 2];
      dv[3 * idx] = a[0] * x + a[3] * y + a[6] * z;
      dv[3 * idx + 1] = a[1] * x + a[4] * y + a[7] * z;
      dv[3 * idx + 2] = a[2] * x + a[5] * y + a[8] * z;
    }
    __syncthreads();
    // (7) the entries this thread owns, over the chunk's points in order
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int t = tid + kThreads * i;
      if (t < L.T) {
        int a, b;
        tri_ab(t, a, b);
        for (int qc = 0; qc < nqc; ++qc) {
          const double wm = P.rc * wq[qc];
          const double wk = P.k * wq[qc];
          const double* N = val + qc * L.nb;
          const double* G = dv + 3 * qc * L.nb;
          const double ma = wm * N[a];
          am[i] += ma * N[b];
          ak[i] += wk * (G[3 * a] * G[3 * b] + G[3 * a + 1] * G[3 * b + 1] + G[3 * a + 2] * G[3 * b + 2]);
        }
      }
    }
    __syncthreads();
  }
  const size_t base = static_cast<size_t>(blockIdx.x) * L.T;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int t = tid + kThreads * i;
    if (t < L.T) {
      lm[base + t] = am[i];
      lk[base + t] = ak[i];
    }
  }
}

// one warp per pattern row r of the rows [r0, r1)
__global__ void k6_gather_kernel(AsmPatch P, const int* __restrict__ row_ptr, int r0, int r1,
                                 int k0, int k1, int e_base, const double* __restrict__ lm,
                                 const double* __restrict__ lk, double* __restrict__ M,
                                 double* __restrict__ K) {
  const int lane = threadIdx.x & 31;
  const int r = r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= r1) return;
  const int n0 = P.V.n[0], n1 = P.V.n[1];
  const int p0 = P.V.p[0], p1 = P.V.p[1], p2 = P.V.p[2];
  const int rc[3] = {r % n0, (r / n0) % n1, r / (n0 * n1)};
  int lo[3], w[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    lo[d] = max(0, rc[d] - P.V.p[d]);
    w[d] = min(P.V.n[d] - 1, rc[d] + P.V.p[d]) - lo[d] + 1;
  }
  const int len = w[0] * w[1] * w[2];
  const int nb = (p0 + 1) * (p1 + 1) * (p2 + 1);
  const size_t T = static_cast<size_t>(nb) * (nb + 1) / 2;
  const int ne0 = P.n_el[0], ne1 = P.n_el[1];
  for (int s = lane; s < len; s += 32) {
    const int cc[3] = {lo[0] + s % w[0], lo[1] + (s / w[0]) % w[1], lo[2] + s / (w[0] * w[1])};
    int eL[3], eH[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      eL[d] = max(P.elo[d][rc[d]], P.elo[d][cc[d]]);
      eH[d] = min(P.ehi[d][rc[d]], P.ehi[d][cc[d]]);
    }
    eL[2] = max(eL[2], k0);
    eH[2] = min(eH[2], k1 - 1);
    const size_t slot = static_cast<size_t>(row_ptr[r]) + s;
    double am = M[slot], ak = K[slot];
    for (int ek = eL[2]; ek <= eH[2]; ++ek) {
      const int sk = P.espan[2][ek] - p2;
      for (int ej = eL[1]; ej <= eH[1]; ++ej) {
        const int sj = P.espan[1][ej] - p1;
        for (int ei = eL[0]; ei <= eH[0]; ++ei) {
          const int si = P.espan[0][ei] - p0;
          const int a = (rc[0] - si) + (p0 + 1) * ((rc[1] - sj) + (p1 + 1) * (rc[2] - sk));
          const int b = (cc[0] - si) + (p0 + 1) * ((cc[1] - sj) + (p1 + 1) * (cc[2] - sk));
          const int A = max(a, b), B = min(a, b);
          const size_t e = static_cast<size_t>(ei) + static_cast<size_t>(ne0) * (ej + static_cast<size_t>(ne1) * ek);
          const size_t at = (e - e_base) * T + static_cast<size_t>(A) * (A + 1) / 2 + B;
          am += lm[at];
          ak += lk[at];
        }
      }
    }
    M[slot] = am;
    K[slot] = ak;
  }
}

// column c of slot s in the pattern row of r (tensor_pattern's order)
struct RowBox {
  int lo[3], w[3], len;
  __device__ RowBox(const AsmPatch& P, int r) {
    const int n0 = P.V.n[0], n1 = P.V.n[1];
    const int rc[3] = {r % n0, (r / n0) % n1, r / (n0 * n1)};
    for (int d = 0; d < 3; ++d) {
      lo[d] = max(0, rc[d] - P.V.p[d]);
      w[d] = min(P.V.n[d] - 1, rc[d] + P.V.p[d]) - lo[d] + 1;
    }
    len = w[0] * w[1] * w[2];
  }
  __device__ int col(const AsmPatch& P, int s) const {
    const int ii = lo[0] + s % w[0], jj = lo[1] + (s / w[0]) % w[1], kk = lo[2] + s / (w[0] * w[1]);
    return ii + P.V.n[0] * (jj + P.V.n[1] * kk);
  }
};

__global__ void k6_lengths_kernel(AsmPatch P, AsmMaps m, int* __restrict__ lenA,
                                  int* __restrict__ lenAc, int* __restrict__ lenB) {
  const int lane = threadIdx.x & 31;
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (f >= m.n_free) return;
  const RowBox rb(P, m.free_list[f]);
  int a = 0, ac = 0;
  for (int s = lane; s < rb.len; s += 32) {
    const int c = rb.col(P, s);
    a += m.free_index[c] >= 0;
    ac += m.con_index[c] >= 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    ac += __shfl_xor_sync(0xffffffffu, ac, o);
  }
  if (lane == 0) {
    lenA[f] = a;
    lenAc[f] = ac;
    lenB[f] = rb.len;
  }
}

__global__ void k6_fill_kernel(AsmPatch P, const int* __restrict__ row_ptr, AsmMaps m,
                               const double* __restrict__ M, const double* __restrict__ K,
                               double inv_dt, double th, double mth, SellOut A, SellOut Ac,
                               SellOut B) {
  const int lane = threadIdx.x & 31;
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (f >= m.n_free) return;
  const int r = m.free_list[f];
  const RowBox rb(P, r);
  const long long sl = f >> 5, ln = f & 31;
  const long long ba = A.sp[sl] + ln, bac = Ac.sp[sl] + ln, bb = B.sp[sl] + ln;
  int ka = 0, kac = 0;
  for (int s0 = 0; s0 < rb.len; s0 += 32) {
    const int s = s0 + lane;
    const bool in = s < rb.len;
    int c = 0, fi = -1, ci = -1;
    double av = 0.0, bv = 0.0;
    if (in) {
      c = rb.col(P, s);
      fi = m.free_index[c];
      ci = m.con_index[c];
      const size_t q = static_cast<size_t>(row_ptr[r]) + s;
      av = inv_dt * M[q] + th * K[q];
      bv = inv_dt * M[q] + mth * K[q];
      B.col[bb + 32LL * s] = c;
      B.val[bb + 32LL * s] = bv;
    }
    const unsigned mf = __ballot_sync(0xffffffffu, in && fi >= 0);
    const unsigned mc = __ballot_sync(0xffffffffu, in && ci >= 0);
    const unsigned below = (1u << lane) - 1u;
    if (in && fi >= 0) {
      const long long at = ba + 32LL * (ka + __popc(mf & below));
      A.col[at] = fi;
      A.val[at] = av;
    }
    if (in && ci >= 0) {
      const long long at = bac + 32LL * (kac + __popc(mc & below));
      Ac.col[at] = ci;
      Ac.val[at] = av;
    }
    ka += __popc(mf);
    kac += __popc(mc);
  }
}

// ---------------------------------------------------------------- face sets
// map_point + face_point at face parameters (u, v) of face f: x, the outward
// unit normal, the area scale |t_u x t_v|; N (nd basis values, nullable) and
// the basis block's grid indices (nullable)
__device__ void face_point_dev(const NurbsDev& V, int f, double u, double v, double* x,
                               double* nrm, double* area, double* N, int* idx, int* flags) {
  const int ax = f / 2;
  const bool is_min = (f % 2) == 0;
  const int t0 = ax == 0 ? 1 : 0, t1 = ax == 2 ? 1 : 2;
  double xi[3];
  xi[ax] = is_min ? 0.0 : 1.0;
  xi[t0] = u;
  xi[t1] = v;
  double tab[3][2 * (kNurbsMaxP + 1)];
  int sp[3];
  for (int d = 0; d < 3; ++d) {
    if (!find_span(V.U[d], V.p[d], V.n[d], xi[d], sp[d])) {
      atomicOr(flags, 4);
      return;
    }
    basis_ders1(V.U[d], V.p[d], xi[d], sp[d], tab[d]);
  }
  const int p0 = V.p[0], p1 = V.p[1], p2 = V.p[2];
  auto gidx = [&](int i, int j, int k) {
    return static_cast<long>(sp[0] - p0 + i) +
           static_cast<long>(V.n[0]) *
               (static_cast<long>(sp[1] - p1 + j) + static_cast<long>(V.n[1]) * (sp[2] - p2 + k));
  };
  // basis_at: weight sums in basis order, then the rational basis (as K4)
  double W = 0.0, dW[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k <= p2; ++k) {
    const double n3 = tab[2][k], d3 = tab[2][p2 + 1 + k];
    for (int j = 0; j <= p1; ++j) {
      const double n2 = tab[1][j], d2 = tab[1][p1 + 1 + j];
      for (int i = 0; i <= p0; ++i) {
        const double n1 = tab[0][i], d1 = tab[0][p0 + 1 + i];
        const double w = V.pts[4 * gidx(i, j, k) + 3];
        W += w * n1 * n2 * n3;
        dW[0] += w * d1 * n2 * n3;
        dW[1] += w * n1 * d2 * n3;
        dW[2] += w * n1 * n2 * d3;
      }
    }
  }
  double xs[3] = {0.0, 0.0, 0.0}, jac[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int m = 0;
  for (int k = 0; k <= p2; ++k) {
    const double n3 = tab[2][k], d3 = tab[2][p2 + 1 + k];
    for (int j = 0; j <= p1; ++j) {
      const double n2 = tab[1][j], d2 = tab[1][p1 + 1 + j];
      for (int i = 0; i <= p0; ++i, ++m) {
        const double n1 = tab[0][i], d1 = tab[0][p0 + 1 + i];
        const long g = gidx(i, j, k);
        const double* c = V.pts + 4 * g;
        const double w = c[3];
        const double val = (w * n1 * n2 * n3) / W;
        const double dv[3] = {(w * d1 * n2 * n3 - dW[0] * val) / W,
                              (w * n1 * d2 * n3 - dW[1] * val) / W,
                              (w * n1 * n2 * d3 - dW[2] * val) / W};
        for (int r = 0; r < 3; ++r) {
          xs[r] += c[r] * val;
          for (int q = 0; q < 3; ++q) jac[3 * r + q] += c[r] * dv[q];
        }
        if (N) N[m] = val;
        if (idx) idx[m] = static_cast<int>(g);
      }
    }
  }
  if (!(det3(jac) > 0.0)) atomicOr(flags, 1);
  const double tu[3] = {jac[t0], jac[3 + t0], jac[6 + t0]};
  const double tv[3] = {jac[t1], jac[3 + t1], jac[6 + t1]};
  const double ac[3] = {jac[ax], jac[3 + ax], jac[6 + ax]};
  const double cr[3] = {tu[1] * tv[2] - tu[2] * tv[1], tu[2] * tv[0] - tu[0] * tv[2],
                        tu[0] * tv[1] - tu[1] * tv[0]};
  const double ar = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
  if (!(ar > 0.0)) atomicOr(flags, 2);
  double n[3] = {cr[0] / ar, cr[1] / ar, cr[2] / ar};
  const double sdot = n[0] * ac[0] + n[1] * ac[1] + n[2] * ac[2];
  if ((is_min && sdot > 0.0) || (!is_min && sdot < 0.0))
    for (int c = 0; c < 3; ++c) n[c] = n[c] * -1.0;
  for (int c = 0; c < 3; ++c) {
    x[c] = xs[c];
    nrm[c] = n[c];
  }
  *area = ar;
}

__device__ __forceinline__ int elem_of(const int* off, int n_el, int q) {
  int lo = 0, hi = n_el;  // off[lo] <= q < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void k6_face_points_kernel(FaceSetDev F) {
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long>(F.tqb) + F.tqf) return;
  const bool base = i < F.tqb;
  const int q = static_cast<int>(base ? i : i - F.tqb);
  const int e = elem_of(base ? F.qb_off : F.qf_off, F.n_el, q);
  const FaceElemDev E = F.el[e];
  const int mult = base ? 1 : F.fm;
  const int nu = mult * E.qu, nv = mult * E.qv;
  const int loc = q - (base ? F.qb_off[e] : F.qf_off[e]);
  const int a = loc % nu, b = loc / nu;
  const double* gun = F.gnodes + nu * (nu - 1) / 2;
  const double* guw = F.gweights + nu * (nu - 1) / 2;
  const double* gvn = F.gnodes + nv * (nv - 1) / 2;
  const double* gvw = F.gweights + nv * (nv - 1) / 2;
  const double u = E.mu + E.hu * gun[a];
  const double v = E.mv + E.hv * gvn[b];
  double area;
  double* N = (base ? F.Nb : F.Nf) + static_cast<size_t>(q) * F.nd;
  int* idx = base && loc == 0 ? F.dofs + static_cast<size_t>(e) * F.nd : nullptr;
  face_point_dev(F.V, E.f, u, v, F.x + 3 * i, F.nrm + 3 * i, &area, N, idx, F.flags);
  F.w[i] = guw[a] * gvw[b] * E.hu * E.hv * area;
}

__global__ void k6_face_centers_kernel(FaceSetDev F) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= F.n_el) return;
  const FaceElemDev E = F.el[e];
  double nrm[3], area;
  face_point_dev(F.V, E.f, E.mu, E.mv, F.centers + 3 * static_cast<size_t>(e), nrm, &area,
                 nullptr, nullptr, F.flags);
}

__global__ void k6_face_keep_kernel(FaceSetDev F, int* __restrict__ keep, int* __restrict__ nkeep) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= F.n_el) return;
  int c = 0;
  for (int a = 0; a < F.nd; ++a) {
    bool nz = false;
    for (int q = F.qb_off[e]; q < F.qb_off[e + 1] && !nz; ++q)
      nz = F.Nb[static_cast<size_t>(q) * F.nd + a] != 0.0;
    for (int q = F.qf_off[e]; q < F.qf_off[e + 1] && !nz; ++q)
      nz = F.Nf[static_cast<size_t>(q) * F.nd + a] != 0.0;
    if (nz) keep[static_cast<size_t>(e) * F.nd + c++] = a;
  }
  nkeep[e] = c;
}

__global__ void k6_face_compact_kernel(FaceSetDev F, const int* __restrict__ keep,
                                       const int* __restrict__ nkeep, int ndk,
                                       double* __restrict__ Nbk, double* __restrict__ Nfk,
                                       int* __restrict__ dofk) {
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long npts = static_cast<long>(F.tqb) + F.tqf;
  if (i < npts * ndk) {
    const long pt = i / ndk;
    const int kk = static_cast<int>(i - pt * ndk);
    const bool base = pt < F.tqb;
    const int q = static_cast<int>(base ? pt : pt - F.tqb);
    const int e = elem_of(base ? F.qb_off : F.qf_off, F.n_el, q);
    const double* N = (base ? F.Nb : F.Nf) + static_cast<size_t>(q) * F.nd;
    const double val = kk < nkeep[e] ? N[keep[static_cast<size_t>(e) * F.nd + kk]] : 0.0;
    (base ? Nbk : Nfk)[static_cast<size_t>(q) * ndk + kk] = val;
  } else if (i < npts * ndk + static_cast<long>(F.n_el) * ndk) {
    const long j = i - npts * ndk;
    const int e = static_cast<int>(j / ndk), kk = static_cast<int>(j - static_cast<long>(e) * ndk);
    dofk[j] = kk < nkeep[e] ? F.dofs[static_cast<size_t>(e) * F.nd + keep[static_cast<size_t>(e) * F.nd + kk]]
                            : -1;
  }
}

int ept_of(const AsmPatch& P) {
  const Layout L = layout_of(P);
  const int need = (L.T + kThreads - 1) / kThreads;
  for (int e : {2, 4, 9, 16, 32})
    if (need <= e) return e;
  return 0;
}

}  // namespace

bool k6_supported(const AsmPatch& P) {
  for (int d = 0; d < 3; ++d)
    if (P.V.p[d] > kNurbsMaxP || P.nq[d] < 1 || P.nq[d] > 2 * (kNurbsMaxP + 1)) return false;
  const Layout L = layout_of(P);
  return ept_of(P) > 0 && L.doubles * 8 <= 200 * 1024 && 4 * L.Q >= 1 && 9 * L.Q <= kThreads &&
         3 * L.maxq <= kThreads;
}

size_t k6_entries_per_element(const AsmPatch& P) { return static_cast<size_t>(layout_of(P).T); }

void k6_element_matrices(const AsmPatch& P, int e0, int ne, double* d_lm, double* d_lk,
                         int* d_flags, cudaStream_t s) {
  if (ne <= 0) return;
  const Layout L = layout_of(P);
  const size_t bytes = static_cast<size_t>(L.doubles) * 8;
  auto go = [&](auto kern) {
    TG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
    kern<<<ne, kThreads, bytes, s>>>(P, e0, d_lm, d_lk, d_flags);
  };
  switch (ept_of(P)) {
    case 2: go(k6_element_kernel<2>); break;
    case 4: go(k6_element_kernel<4>); break;
    case 9: go(k6_element_kernel<9>); break;
    case 16: go(k6_element_kernel<16>); break;
    case 32: go(k6_element_kernel<32>); break;
    default: throw std::invalid_argument("k6: basis block too large for the device assembly");
  }
  TG_CUDA(cudaGetLastError());
}

void k6_gather(const AsmPatch& P, const int* d_row_ptr, int r0, int r1, int k0, int k1,
               int e_base, const double* d_lm, const double* d_lk, double* d_M, double* d_K,
               cudaStream_t s) {
  if (k1 <= k0 || r1 <= r0) return;
  const int warps = 8;
  k6_gather_kernel<<<(r1 - r0 + warps - 1) / warps, 32 * warps, 0, s>>>(
      P, d_row_ptr, r0, r1, k0, k1, e_base, d_lm, d_lk, d_M, d_K);
  TG_CUDA(cudaGetLastError());
}

void k6_face_sets(const FaceSetDev& F, cudaStream_t s) {
  for (int d = 0; d < 3; ++d)
    if (F.V.p[d] > kNurbsMaxP) throw std::invalid_argument("degree > 7 not supported");
  const long n = static_cast<long>(F.tqb) + F.tqf;
  if (n > 0)
    k6_face_points_kernel<<<static_cast<int>((n + 127) / 128), 128, 0, s>>>(F);
  if (F.n_el > 0) k6_face_centers_kernel<<<(F.n_el + 127) / 128, 128, 0, s>>>(F);
  TG_CUDA(cudaGetLastError());
}

void k6_face_keep(const FaceSetDev& F, int* d_keep, int* d_nkeep, cudaStream_t s) {
  if (F.n_el <= 0) return;
  k6_face_keep_kernel<<<(F.n_el + 127) / 128, 128, 0, s>>>(F, d_keep, d_nkeep);
  TG_CUDA(cudaGetLastError());
}

void k6_face_compact(const FaceSetDev& F, const int* d_keep, const int* d_nkeep, int ndk,
                     double* d_Nbk, double* d_Nfk, int* d_dofk, cudaStream_t s) {
  const long n = (static_cast<long>(F.tqb) + F.tqf + F.n_el) * ndk;
  if (n <= 0) return;
  k6_face_compact_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(F, d_keep, d_nkeep, ndk,
                                                                         d_Nbk, d_Nfk, d_dofk);
  TG_CUDA(cudaGetLastError());
}

void k6_row_lengths(const AsmPatch& P, const AsmMaps& m, int* d_lenA, int* d_lenAc, int* d_lenB,
                    cudaStream_t s) {
  if (m.n_free <= 0) return;
  const int warps = 8;
  k6_lengths_kernel<<<(m.n_free + warps - 1) / warps, 32 * warps, 0, s>>>(P, m, d_lenA, d_lenAc,
                                                                         d_lenB);
  TG_CUDA(cudaGetLastError());
}

void k6_fill(const AsmPatch& P, const int* d_row_ptr, const AsmMaps& m, const double* d_M,
             const double* d_K, double inv_dt, double th, double mth, const SellOut& A,
             const SellOut& Ac, const SellOut& B, cudaStream_t s) {
  if (m.n_free <= 0) return;
  const int warps = 8;
  k6_fill_kernel<<<(m.n_free + warps - 1) / warps, 32 * warps, 0, s>>>(P, d_row_ptr, m, d_M, d_K,
                                                                      inv_dt, th, mth, A, Ac, B);
  TG_CUDA(cudaGetLastError());
}

}  // namespace tgb
