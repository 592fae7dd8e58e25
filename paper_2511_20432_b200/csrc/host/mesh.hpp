// Host-side discretization setup: face roles, the free/constrained DOF split,
// the lateral-face quadrature sets (K1 flux points + K3 tables) and the
// bottom-face Greville collocation points (K1 Dirichlet points). Semantics of
// the reference's mesh module (proj/include/thermiga/mesh.hpp).
#pragma once

#include <array>
#include <vector>

#include "splines.hpp"

namespace tgb {

enum class FaceRole { bottom, lateral, top };

struct BoundaryTags {
  std::array<FaceRole, 6> role{};
  FaceRole role_of(FaceId f) const { return role[static_cast<int>(f)]; }
  FaceId bottom_face() const;
  void validate() const;
  static BoundaryTags extruded_default();
};

// Constrained = the control-point layer touching the bottom face
// (mesh.cpp:130-154); both lists are in flat (first index fastest) order.
struct DofMap {
  std::vector<int> free_index, constrained_index, free_list, constrained_list;
  int n_free() const { return static_cast<int>(free_list.size()); }
  int n_constrained() const { return static_cast<int>(constrained_list.size()); }
};
DofMap make_dof_map(const NurbsVolume& vol, const BoundaryTags& tags);

// Lateral face quadrature, flattened in (face, element, q) order with q
// v-outer / u-inner (mesh.cpp:158-205). Every face element carries the
// (p+1)^3 volume DOFs active at its first quadrature point and both rules;
// rule sizes differ between faces when the degrees differ per direction, so
// each element has its own counts and offsets into the flat arrays.
struct FaceSets {
  int n_elems = 0, n_dofs = 0;
  std::vector<int> nqb, nqf;            // per element rule sizes
  std::vector<long> qb_off, qf_off;     // per element offsets (n_elems + 1)
  std::vector<double> centers;          // 3 per element
  std::vector<int> dofs;                // n_dofs per element
  std::vector<double> xb, nb, wb, Nb;   // base rule: 3, 3, 1, n_dofs per qp
  std::vector<double> xf, nf, wf, Nf;   // fine rule
};
FaceSets build_face_sets(const NurbsVolume& vol, const BoundaryTags& tags, int fine_mult);
// The lateral face elements in the reference's order (face, v-interval,
// u-interval) and the layout fields of fs (n_elems, n_dofs, rule sizes and
// offsets; no per-point arrays): build_face_sets' first half, shared with the
// device builder (k6_assemble.cu).
struct FaceElemSpec {
  FaceId f;
  double mu, hu, mv, hv;
  int qu, qv;
};
std::vector<FaceElemSpec> face_elements(const NurbsVolume& vol, const BoundaryTags& tags,
                                        int fine_mult, FaceSets& fs);

// Physical positions of the Greville points of the constrained DOFs, in
// constrained order (mesh.cpp:238-264).
std::vector<double> greville_points(const NurbsVolume& vol, const DofMap& dofs,
                                    const BoundaryTags& tags);

// Per-element quadrature over all elements of the patch: used by the general
// (non-separable) operator path and by the det J > 0 check of build_mesh
// (mesh.cpp:65-128).
struct ElementQuad {
  int n_qp = 0, n_basis = 0;
  std::vector<int> dofs;
  std::vector<double> weight;  // gauss x box measure x det J
  std::vector<double> N;       // n_qp x n_basis
  std::vector<Vec3> dN;        // physical gradients
};
struct ElementGrid {
  std::array<std::vector<double>, 3> bp;  // breakpoints
  std::array<int, 3> n_el{0, 0, 0};
  int count() const { return n_el[0] * n_el[1] * n_el[2]; }
};
ElementGrid element_grid(const NurbsVolume& vol);
void element_quad(const NurbsVolume& vol, const ElementGrid& eg, int e, std::array<int, 3> nq,
                  ElementQuad& out);

}  // namespace tgb
