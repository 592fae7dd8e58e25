#include "operator.hpp"

#include "parallel.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace tgb {

bool separable_coords(const NurbsVolume& vol, std::array<std::vector<double>, 3>& coord) {
  const auto& g = vol.grid();
  const auto n = g.dims;
  const double w0 = g.pts[0][3];
  for (int d = 0; d < 3; ++d) coord[d].assign(n[d], 0.0);
  for (int i = 0; i < n[0]; ++i) coord[0][i] = g.pts[g.index(i, 0, 0)][0];
  for (int j = 0; j < n[1]; ++j) coord[1][j] = g.pts[g.index(0, j, 0)][1];
  for (int k = 0; k < n[2]; ++k) coord[2][k] = g.pts[g.index(0, 0, k)][2];
  // Knot insertion (Boehm, on homogeneous points) perturbs coordinates that
  // are constant along a line by an ulp or two (a x + (1-a) x != x), so the
  // test allows a relative 1e-12 of the patch extent; the operator then
  // differs from the assembled one at the rounding level only.
  double ext = 0.0;
  for (int d = 0; d < 3; ++d)
    ext = std::max(ext, std::abs(coord[d].back() - coord[d].front()));
  const double tol = 1e-12 * (ext > 0.0 ? ext : 1.0);
  for (int k = 0; k < n[2]; ++k)
    for (int j = 0; j < n[1]; ++j)
      for (int i = 0; i < n[0]; ++i) {
        const auto& p = g.pts[g.index(i, j, k)];
        if (std::abs(p[3] - w0) > 1e-12 * std::abs(w0) || std::abs(p[0] - coord[0][i]) > tol ||
            std::abs(p[1] - coord[1][j]) > tol || std::abs(p[2] - coord[2][k]) > tol)
          return false;
      }
  return true;
}

// 1D factors on one axis: M_ab = sum_q w_q h J N_a N_b, K_ab = sum_q w_q h N'_a N'_b / J,
// with J = dx/du from the axis' control coordinates (Gauss nq points per span).
Band1D assemble_band_1d(const KnotVector& kv, const std::vector<double>& X, int nq) {
  Band1D b;
  b.p = kv.degree();
  b.n = kv.basis_count();
  const int p = b.p, W = 2 * p + 1;
  b.M.assign(static_cast<size_t>(b.n) * W, 0.0);
  b.K.assign(static_cast<size_t>(b.n) * W, 0.0);
  const auto bp = kv.breakpoints();
  const auto& g = gauss_rule(nq);
  std::vector<double> tab(2 * (p + 1));
  int sign = 0;
  for (std::size_t s = 0; s + 1 < bp.size(); ++s) {
    const double h = 0.5 * (bp[s + 1] - bp[s]), m = 0.5 * (bp[s + 1] + bp[s]);
    for (int q = 0; q < nq; ++q) {
      const double u = m + h * g.nodes[q];
      const int span = kv.find_span(u);
      kv.basis_ders(u, span, 1, tab.data());
      double J = 0.0;
      for (int a = 0; a <= p; ++a) J += tab[p + 1 + a] * X[span - p + a];
      const int sg = J > 0.0 ? 1 : (J < 0.0 ? -1 : 0);
      if (sg == 0 || (sign != 0 && sg != sign))
        throw numeric_error("non-positive Jacobian determinant at quadrature point");
      sign = sg;
      const double w = g.weights[q] * h;
      for (int a = 0; a <= p; ++a)
        for (int c = 0; c <= p; ++c) {
          const int ia = span - p + a, ic = span - p + c;
          const size_t slot = static_cast<size_t>(ia) * W + (p + ic - ia);
          b.M[slot] += w * J * tab[a] * tab[c];
          b.K[slot] += w * tab[p + 1 + a] * tab[p + 1 + c] / J;
        }
    }
  }
  return b;
}

namespace {

Csr tensor_pattern(const NurbsVolume& vol) {
  const auto n = vol.basis_counts();
  const auto p = vol.degrees();
  Csr m;
  m.rows = n[0] * n[1] * n[2];
  m.row_ptr.assign(m.rows + 1, 0);
  auto range = [](int c, int pd, int nd, int& lo, int& hi) {
    lo = std::max(0, c - pd);
    hi = std::min(nd - 1, c + pd);
  };
  for (int pass = 0; pass < 2; ++pass) {
    int r = 0;
    for (int k = 0; k < n[2]; ++k)
      for (int j = 0; j < n[1]; ++j)
        for (int i = 0; i < n[0]; ++i, ++r) {
          int il, ih, jl, jh, kl, kh;
          range(i, p[0], n[0], il, ih);
          range(j, p[1], n[1], jl, jh);
          range(k, p[2], n[2], kl, kh);
          if (pass == 0) {
            m.row_ptr[r + 1] = (ih - il + 1) * (jh - jl + 1) * (kh - kl + 1);
            continue;
          }
          int slot = m.row_ptr[r];
          for (int kk = kl; kk <= kh; ++kk)
            for (int jj = jl; jj <= jh; ++jj)
              for (int ii = il; ii <= ih; ++ii) m.col[slot++] = ii + n[0] * (jj + n[1] * kk);
        }
    if (pass == 0) {
      for (int r2 = 0; r2 < m.rows; ++r2) m.row_ptr[r2 + 1] += m.row_ptr[r2];
      m.col.resize(m.row_ptr[m.rows]);
      m.val.assign(m.row_ptr[m.rows], 0.0);
    }
  }
  return m;
}


}  // namespace

Sell to_sell(const Csr& m) {
  Sell s;
  s.rows = m.rows;
  const int ns = (m.rows + 31) / 32;
  s.row_len.assign(m.rows, 0);
  s.slice_ptr.assign(ns + 1, 0);
  for (int sl = 0; sl < ns; ++sl) {
    int w = 0;
    for (int r = sl * 32; r < std::min(m.rows, sl * 32 + 32); ++r) {
      s.row_len[r] = m.row_ptr[r + 1] - m.row_ptr[r];
      w = std::max(w, s.row_len[r]);
    }
    s.slice_ptr[sl + 1] = s.slice_ptr[sl] + 32LL * w;
  }
  s.col.assign(s.slice_ptr[ns], 0);
  s.val.assign(s.slice_ptr[ns], 0.0);
  parallel_for(ns, [&](long sl) {
    for (int r = static_cast<int>(sl) * 32; r < std::min(m.rows, static_cast<int>(sl) * 32 + 32);
         ++r) {
      const long long base = s.slice_ptr[sl] + (r & 31);
      for (int k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k) {
        s.col[base + 32LL * (k - m.row_ptr[r])] = m.col[k];
        s.val[base + 32LL * (k - m.row_ptr[r])] = m.val[k];
      }
    }
  }, 64);
  return s;
}

// Element matrices are formed in parallel in batches of consecutive elements;
// the scatter is parallel over the tensor index i of the row (each worker owns
// a range of i and walks the batch in element order), so every entry still
// receives its element contributions in element order, with the reference's
// per-element arithmetic (assembly.cpp:59-101): the values are bit-identical
// to a serial assembly for any thread count. CSR slots come from the tensor
// pattern directly (no search).
void assemble_mass_stiffness(const NurbsVolume& vol, std::array<int, 3> nq, const Material& mat,
                             Csr& M, Csr& K) {
  M = tensor_pattern(vol);
  K = M;
  const ElementGrid eg = element_grid(vol);
  const auto n = vol.basis_counts();
  const auto pd = vol.degrees();
  const int ne = eg.count();
  constexpr int kBatch = 2048;
  struct Local {
    int nb = 0;
    std::vector<int> dofs;
    std::vector<std::array<int, 3>> ijk;
    std::vector<double> lm, lk;  // nb x nb, lower triangle used
  };
  std::vector<Local> loc(std::min(kBatch, std::max(ne, 1)));
  const int nth = std::max(1, std::min(host_threads(), n[0]));
  double t_loc = 0.0, t_sc = 0.0;
  for (int e0 = 0; e0 < ne; e0 += kBatch) {
    auto c0 = std::chrono::steady_clock::now();
    const int nbt = std::min(kBatch, ne - e0);
    parallel_for(nbt, [&](long t) {
      thread_local ElementQuad quad;
      element_quad(vol, eg, e0 + static_cast<int>(t), nq, quad);
      Local& L = loc[t];
      const int nb = L.nb = quad.n_basis;
      L.dofs.assign(quad.dofs.begin(), quad.dofs.end());
      L.ijk.resize(nb);
      for (int a = 0; a < nb; ++a) {
        const int f = L.dofs[a];
        L.ijk[a] = {f % n[0], (f / n[0]) % n[1], f / (n[0] * n[1])};
      }
      L.lm.assign(static_cast<size_t>(nb) * nb, 0.0);
      L.lk.assign(static_cast<size_t>(nb) * nb, 0.0);
      // the reference's expressions, wm * N[a] * N[b] and wk * (G[a].dot(G[b])),
      // with (wm * N[a]) hoisted and G split by component so the b loop
      // vectorizes; same roundings in the same order
      thread_local std::vector<double> gx, gy, gz;
      gx.resize(nb);
      gy.resize(nb);
      gz.resize(nb);
      double* __restrict lm = L.lm.data();
      double* __restrict lk = L.lk.data();
      for (int q = 0; q < quad.n_qp; ++q) {
        const double wm = mat.volumetric_capacity() * quad.weight[q];
        const double wk = mat.conductivity * quad.weight[q];
        const double* __restrict N = &quad.N[static_cast<size_t>(q) * nb];
        const Vec3* G = &quad.dN[static_cast<size_t>(q) * nb];
        for (int a = 0; a < nb; ++a) {
          gx[a] = G[a].x;
          gy[a] = G[a].y;
          gz[a] = G[a].z;
        }
        const double* __restrict X = gx.data();
        const double* __restrict Y = gy.data();
        const double* __restrict Z = gz.data();
        for (int a = 0; a < nb; ++a) {
          const double ma = wm * N[a];
          const double xa = X[a], ya = Y[a], za = Z[a];
          double* __restrict rm = lm + static_cast<size_t>(a) * nb;
          double* __restrict rk = lk + static_cast<size_t>(a) * nb;
          for (int b = 0; b <= a; ++b) {
            rm[b] += ma * N[b];
            rk[b] += wk * (xa * X[b] + ya * Y[b] + za * Z[b]);
          }
        }
      }
    }, 8);
    auto c1 = std::chrono::steady_clock::now();
    t_loc += std::chrono::duration<double>(c1 - c0).count();
    parallel_for(nth, [&](long T) {
      const int i0 = static_cast<int>(static_cast<long>(n[0]) * T / nth);
      const int i1 = static_cast<int>(static_cast<long>(n[0]) * (T + 1) / nth);
      // slot of column c in the pattern row of r (tensor_pattern's order)
      auto slot = [&](int r, const std::array<int, 3>& ri, const std::array<int, 3>& ci) {
        int lo[3], w[3];
        for (int d = 0; d < 3; ++d) {
          lo[d] = std::max(0, ri[d] - pd[d]);
          w[d] = std::min(n[d] - 1, ri[d] + pd[d]) - lo[d] + 1;
        }
        return M.row_ptr[r] + ((ci[2] - lo[2]) * w[1] + (ci[1] - lo[1])) * w[0] + (ci[0] - lo[0]);
      };
      for (int t = 0; t < nbt; ++t) {
        const Local& L = loc[t];
        const int nb = L.nb;
        int imin = n[0], imax = -1;
        for (int a = 0; a < nb; ++a) {
          imin = std::min(imin, L.ijk[a][0]);
          imax = std::max(imax, L.ijk[a][0]);
        }
        if (imax < i0 || imin >= i1) continue;
        for (int a = 0; a < nb; ++a) {
          const bool own_a = L.ijk[a][0] >= i0 && L.ijk[a][0] < i1;
          for (int b = 0; b <= a; ++b) {
            const bool own_b = L.ijk[b][0] >= i0 && L.ijk[b][0] < i1;
            if (!own_a && !own_b) continue;
            const double vm = L.lm[static_cast<size_t>(a) * nb + b];
            const double vk = L.lk[static_cast<size_t>(a) * nb + b];
            if (own_a) {
              const int sl = slot(L.dofs[a], L.ijk[a], L.ijk[b]);
              M.val[sl] += vm;
              K.val[sl] += vk;
            }
            if (a != b && own_b) {
              const int sl = slot(L.dofs[b], L.ijk[b], L.ijk[a]);
              M.val[sl] += vm;
              K.val[sl] += vk;
            }
          }
        }
      }
    }, 1);
    t_sc += std::chrono::duration<double>(std::chrono::steady_clock::now() - c1).count();
  }
  if (std::getenv("TG_SETUP_TIMING")) std::fprintf(stderr, "[setup]   element matrices %.3f s, scatter %.3f s\n", t_loc, t_sc);
}

}  // namespace tgb
