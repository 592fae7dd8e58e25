#include "mesh.hpp"

#include <algorithm>
#include <cmath>

#include "parallel.hpp"

namespace tgb {

FaceId BoundaryTags::bottom_face() const {
  for (FaceId f : kFaces)
    if (role_of(f) == FaceRole::bottom) return f;
  throw config_error("boundary tags: no face tagged bottom");
}

void BoundaryTags::validate() const {
  int nb = 0, nl = 0;
  for (FaceId f : kFaces) {
    nb += role_of(f) == FaceRole::bottom;
    nl += role_of(f) == FaceRole::lateral;
  }
  if (nb != 1) throw config_error("boundary tags: exactly one face must be bottom");
  if (nl < 1) throw config_error("boundary tags: at least one face must be lateral");
}

BoundaryTags BoundaryTags::extruded_default() {
  BoundaryTags t;
  t.role.fill(FaceRole::lateral);
  t.role[static_cast<int>(FaceId::zetamin)] = FaceRole::bottom;
  t.role[static_cast<int>(FaceId::zetamax)] = FaceRole::top;
  return t;
}

DofMap make_dof_map(const NurbsVolume& vol, const BoundaryTags& tags) {
  tags.validate();
  const FaceId bottom = tags.bottom_face();
  const int ax = face_axis(bottom);
  const auto n = vol.basis_counts();
  const int layer = face_is_min(bottom) ? 0 : n[ax] - 1;
  DofMap m;
  m.free_index.assign(vol.n_functions(), -1);
  m.constrained_index.assign(vol.n_functions(), -1);
  for (int k = 0; k < n[2]; ++k)
    for (int j = 0; j < n[1]; ++j)
      for (int i = 0; i < n[0]; ++i) {
        const int ijk[3] = {i, j, k};
        const int g = vol.grid().index(i, j, k);
        if (ijk[ax] == layer) {
          m.constrained_index[g] = m.n_constrained();
          m.constrained_list.push_back(g);
        } else {
          m.free_index[g] = m.n_free();
          m.free_list.push_back(g);
        }
      }
  return m;
}

std::vector<FaceElemSpec> face_elements(const NurbsVolume& vol, const BoundaryTags& tags,
                                        int fine_mult, FaceSets& fs) {
  tags.validate();
  fine_mult = std::max(1, fine_mult);
  const auto p = vol.degrees();
  fs = FaceSets{};
  fs.n_dofs = (p[0] + 1) * (p[1] + 1) * (p[2] + 1);
  // element list in the reference's order (face, then v-interval, then
  // u-interval; mesh.cpp:158-236) with its rule offsets
  using Elem = FaceElemSpec;
  std::vector<Elem> el;
  fs.qb_off.push_back(0);
  fs.qf_off.push_back(0);
  for (FaceId f : kFaces) {
    if (tags.role_of(f) != FaceRole::lateral) continue;
    const auto t = face_tangent_axes(f);
    const auto bu = vol.knots(t[0]).breakpoints();
    const auto bv = vol.knots(t[1]).breakpoints();
    const int qu = p[t[0]] + 1, qv = p[t[1]] + 1;
    for (std::size_t jv = 0; jv + 1 < bv.size(); ++jv)
      for (std::size_t iu = 0; iu + 1 < bu.size(); ++iu) {
        el.push_back({f, 0.5 * (bu[iu + 1] + bu[iu]), 0.5 * (bu[iu + 1] - bu[iu]),
                      0.5 * (bv[jv + 1] + bv[jv]), 0.5 * (bv[jv + 1] - bv[jv]), qu, qv});
        fs.nqb.push_back(qu * qv);
        fs.nqf.push_back(fine_mult * qu * fine_mult * qv);
        fs.qb_off.push_back(fs.qb_off.back() + qu * qv);
        fs.qf_off.push_back(fs.qf_off.back() + fine_mult * qu * fine_mult * qv);
      }
  }
  fs.n_elems = static_cast<int>(el.size());
  return el;
}

FaceSets build_face_sets(const NurbsVolume& vol, const BoundaryTags& tags, int fine_mult) {
  FaceSets fs;
  const std::vector<FaceElemSpec> el = face_elements(vol, tags, fine_mult, fs);
  using Elem = FaceElemSpec;
  fine_mult = std::max(1, fine_mult);
  const int nd = fs.n_dofs;
  const size_t tqb = fs.qb_off.back(), tqf = fs.qf_off.back();
  fs.centers.assign(3 * el.size(), 0.0);
  fs.dofs.assign(nd * el.size(), 0);
  fs.xb.assign(3 * tqb, 0.0);
  fs.nb.assign(3 * tqb, 0.0);
  fs.wb.assign(tqb, 0.0);
  fs.Nb.assign(nd * tqb, 0.0);
  fs.xf.assign(3 * tqf, 0.0);
  fs.nf.assign(3 * tqf, 0.0);
  fs.wf.assign(tqf, 0.0);
  fs.Nf.assign(nd * tqf, 0.0);
  for (const Elem& e : el) {  // warm the (mutex-guarded) rule cache
    gauss_rule(e.qu);
    gauss_rule(e.qv);
    gauss_rule(fine_mult * e.qu);
    gauss_rule(fine_mult * e.qv);
  }
  parallel_for(static_cast<long>(el.size()), [&](long ei) {
    const Elem& e = el[ei];
    std::vector<int> idx;
    std::vector<double> val;
    std::vector<Vec3> dv;
    auto rule = [&](int nu, int nv, long q0, double* X, double* Nn, double* Wt, double* Nt,
                    bool first) {
      const auto& gu = gauss_rule(nu);
      const auto& gv = gauss_rule(nv);
      long q = q0;
      for (int b = 0; b < nv; ++b)
        for (int a = 0; a < nu; ++a, ++q) {
          const double u = e.mu + e.hu * gu.nodes[a];
          const double v = e.mv + e.hv * gv.nodes[b];
          const auto sp = vol.face_point(e.f, u, v);
          const int nbas = vol.basis_at(sp.xi, idx, val, dv);
          if (first && q == q0) std::copy(idx.begin(), idx.begin() + nbas, &fs.dofs[ei * nd]);
          X[3 * q] = sp.x.x;
          X[3 * q + 1] = sp.x.y;
          X[3 * q + 2] = sp.x.z;
          Nn[3 * q] = sp.normal.x;
          Nn[3 * q + 1] = sp.normal.y;
          Nn[3 * q + 2] = sp.normal.z;
          Wt[q] = gu.weights[a] * gv.weights[b] * e.hu * e.hv * sp.area_scale;
          std::copy(val.begin(), val.begin() + nbas, Nt + q * nd);
        }
    };
    rule(e.qu, e.qv, fs.qb_off[ei], fs.xb.data(), fs.nb.data(), fs.wb.data(), fs.Nb.data(), true);
    rule(fine_mult * e.qu, fine_mult * e.qv, fs.qf_off[ei], fs.xf.data(), fs.nf.data(),
         fs.wf.data(), fs.Nf.data(), false);
    const auto c = vol.face_point(e.f, e.mu, e.mv);
    fs.centers[3 * ei] = c.x.x;
    fs.centers[3 * ei + 1] = c.x.y;
    fs.centers[3 * ei + 2] = c.x.z;
  });
  return fs;
}

std::vector<double> greville_points(const NurbsVolume& vol, const DofMap& dofs,
                                    const BoundaryTags& tags) {
  const FaceId bottom = tags.bottom_face();
  const auto t = face_tangent_axes(bottom);
  const auto g0 = vol.knots(t[0]).greville();
  const auto g1 = vol.knots(t[1]).greville();
  const auto n = vol.basis_counts();
  std::vector<double> out;
  out.reserve(3 * dofs.n_constrained());
  for (int c = 0; c < dofs.n_constrained(); ++c) {
    const int g = dofs.constrained_list[c];
    const int ijk[3] = {g % n[0], (g / n[0]) % n[1], g / (n[0] * n[1])};
    const Vec3 x = vol.map_point(face_param(bottom, g0[ijk[t[0]]], g1[ijk[t[1]]])).x;
    out.insert(out.end(), {x.x, x.y, x.z});
  }
  return out;
}

ElementGrid element_grid(const NurbsVolume& vol) {
  ElementGrid eg;
  for (int d = 0; d < 3; ++d) {
    eg.bp[d] = vol.knots(d).breakpoints();
    eg.n_el[d] = static_cast<int>(eg.bp[d].size()) - 1;
  }
  return eg;
}

void element_quad(const NurbsVolume& vol, const ElementGrid& eg, int e, std::array<int, 3> nq,
                  ElementQuad& out) {
  const int ei = e % eg.n_el[0];
  const int ej = (e / eg.n_el[0]) % eg.n_el[1];
  const int ek = e / (eg.n_el[0] * eg.n_el[1]);
  const int el[3] = {ei, ej, ek};
  double half[3], mid[3];
  for (int d = 0; d < 3; ++d) {
    half[d] = 0.5 * (eg.bp[d][el[d] + 1] - eg.bp[d][el[d]]);
    mid[d] = 0.5 * (eg.bp[d][el[d] + 1] + eg.bp[d][el[d]]);
  }
  const double box = half[0] * half[1] * half[2];
  const auto& g0 = gauss_rule(nq[0]);
  const auto& g1 = gauss_rule(nq[1]);
  const auto& g2 = gauss_rule(nq[2]);
  out.n_qp = nq[0] * nq[1] * nq[2];
  const auto p = vol.degrees();
  out.n_basis = (p[0] + 1) * (p[1] + 1) * (p[2] + 1);
  out.weight.assign(out.n_qp, 0.0);
  out.N.assign(static_cast<size_t>(out.n_qp) * out.n_basis, 0.0);
  out.dN.assign(static_cast<size_t>(out.n_qp) * out.n_basis, Vec3{});
  std::vector<int> idx;
  std::vector<double> val;
  std::vector<Vec3> dv;
  int q = 0;
  for (int c = 0; c < nq[2]; ++c)
    for (int b = 0; b < nq[1]; ++b)
      for (int a = 0; a < nq[0]; ++a, ++q) {
        const Vec3 xi{mid[0] + half[0] * g0.nodes[a], mid[1] + half[1] * g1.nodes[b],
                      mid[2] + half[2] * g2.nodes[c]};
        const int nb = vol.basis_at(xi, idx, val, dv);
        if (nb != out.n_basis) throw numeric_error("basis block size mismatch");
        if (q == 0) out.dofs = idx;
        Mat3 J;
        for (int m = 0; m < nb; ++m) {
          const auto& cp = vol.grid().pts[idx[m]];
          for (int r = 0; r < 3; ++r)
            for (int s = 0; s < 3; ++s) J(r, s) += cp[r] * dv[m][s];
        }
        const double det = J.det();
        if (!(det > 0.0))
          throw numeric_error("non-positive Jacobian determinant at quadrature point");
        const Mat3 inv = J.inverse();
        out.weight[q] = g0.weights[a] * g1.weights[b] * g2.weights[c] * box * det;
        for (int m = 0; m < nb; ++m) {
          out.N[static_cast<size_t>(q) * nb + m] = val[m];
          out.dN[static_cast<size_t>(q) * nb + m] = inv.apply_transposed(dv[m]);
        }
      }
}

}  // namespace tgb
