#include "operator.hpp"

#include <algorithm>
#include <cmath>

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

double& at(Csr& m, int r, int c) {
  auto b = m.col.begin() + m.row_ptr[r], e = m.col.begin() + m.row_ptr[r + 1];
  auto it = std::lower_bound(b, e, c);
  if (it == e || *it != c) throw std::out_of_range("entry not in sparsity pattern");
  return m.val[it - m.col.begin()];
}

}  // namespace

void assemble_mass_stiffness(const NurbsVolume& vol, std::array<int, 3> nq, const Material& mat,
                             Csr& M, Csr& K) {
  M = tensor_pattern(vol);
  K = M;
  const ElementGrid eg = element_grid(vol);
  ElementQuad quad;
  std::vector<double> lm, lk;
  for (int e = 0; e < eg.count(); ++e) {
    element_quad(vol, eg, e, nq, quad);
    const int nb = quad.n_basis;
    lm.assign(static_cast<size_t>(nb) * nb, 0.0);
    lk.assign(static_cast<size_t>(nb) * nb, 0.0);
    for (int q = 0; q < quad.n_qp; ++q) {
      const double wm = mat.volumetric_capacity() * quad.weight[q];
      const double wk = mat.conductivity * quad.weight[q];
      const double* N = &quad.N[static_cast<size_t>(q) * nb];
      const Vec3* G = &quad.dN[static_cast<size_t>(q) * nb];
      for (int a = 0; a < nb; ++a)
        for (int b = 0; b <= a; ++b) {
          lm[static_cast<size_t>(a) * nb + b] += wm * N[a] * N[b];
          lk[static_cast<size_t>(a) * nb + b] += wk * G[a].dot(G[b]);
        }
    }
    // deterministic scatter in element order, symmetric by construction
    for (int a = 0; a < nb; ++a)
      for (int b = 0; b <= a; ++b) {
        const double vm = lm[static_cast<size_t>(a) * nb + b];
        const double vk = lk[static_cast<size_t>(a) * nb + b];
        at(M, quad.dofs[a], quad.dofs[b]) += vm;
        at(K, quad.dofs[a], quad.dofs[b]) += vk;
        if (a != b) {
          at(M, quad.dofs[b], quad.dofs[a]) += vm;
          at(K, quad.dofs[b], quad.dofs[a]) += vk;
        }
      }
  }
}

}  // namespace tgb
