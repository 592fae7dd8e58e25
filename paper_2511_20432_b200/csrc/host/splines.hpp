// Host-side B-spline / NURBS geometry: the setup that produces the point sets
// (face quadrature points, Greville points) and the 1D operator tables the
// kernels consume. Same semantics as the reference's splines module
// (proj/include/thermiga/splines.hpp); the algorithms are the standard ones
// (span search, Cox-de Boor values and derivatives, Boehm knot insertion).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "analytic.hpp"

namespace tgb {

struct Mat3 {
  std::array<double, 9> a{};
  double& operator()(int r, int c) { return a[3 * r + c]; }
  double operator()(int r, int c) const { return a[3 * r + c]; }
  double det() const;
  Mat3 inverse() const;
  Vec3 apply_transposed(const Vec3& v) const;
};

// Gauss-Legendre rule on [-1, 1] (Newton on the Legendre recurrence); cached.
struct GaussRule {
  std::vector<double> nodes, weights;
};
const GaussRule& gauss_rule(int n);

class KnotVector {
 public:
  KnotVector() = default;
  KnotVector(std::vector<double> values, int degree);
  int degree() const { return p_; }
  const std::vector<double>& values() const { return u_; }
  int basis_count() const { return static_cast<int>(u_.size()) - p_ - 1; }
  double min_knot() const { return u_.front(); }
  double max_knot() const { return u_.back(); }
  int find_span(double u) const;
  // (nd+1) x (p+1) row-major: row k = k-th derivatives of the p+1 nonzero functions
  void basis_ders(double u, int span, int nd, double* out) const;
  std::vector<double> breakpoints() const;
  std::vector<double> greville() const;
  KnotVector normalized() const;

 private:
  std::vector<double> u_;
  int p_ = 0;
};

enum class FaceId { ximin = 0, ximax, etamin, etamax, zetamin, zetamax };
constexpr std::array<FaceId, 6> kFaces = {FaceId::ximin, FaceId::ximax, FaceId::etamin,
                                          FaceId::etamax, FaceId::zetamin, FaceId::zetamax};
const char* face_name(FaceId f);
FaceId face_from_name(const std::string& s);
inline int face_axis(FaceId f) { return static_cast<int>(f) / 2; }
inline bool face_is_min(FaceId f) { return static_cast<int>(f) % 2 == 0; }
std::array<int, 2> face_tangent_axes(FaceId f);
Vec3 face_param(FaceId f, double u, double v);

struct ControlGrid {
  std::array<int, 3> dims{0, 0, 0};
  std::vector<std::array<double, 4>> pts;  // x, y, z, w; first index fastest
  int index(int i, int j, int k) const { return i + dims[0] * (j + dims[1] * k); }
  int count() const { return dims[0] * dims[1] * dims[2]; }
};

class NurbsVolume {
 public:
  NurbsVolume() = default;
  NurbsVolume(std::array<KnotVector, 3> kvs, ControlGrid grid);
  const KnotVector& knots(int d) const { return kv_[d]; }
  const ControlGrid& grid() const { return grid_; }
  std::array<int, 3> degrees() const {
    return {kv_[0].degree(), kv_[1].degree(), kv_[2].degree()};
  }
  std::array<int, 3> basis_counts() const {
    return {kv_[0].basis_count(), kv_[1].basis_count(), kv_[2].basis_count()};
  }
  int n_functions() const { return grid_.count(); }

  // Rational basis at xi: flat indices, values, parametric gradients.
  int basis_at(const Vec3& xi, std::vector<int>& idx, std::vector<double>& val,
               std::vector<Vec3>& dval) const;
  struct PointMap {
    Vec3 x;
    Mat3 jac;
    double det_jac;
  };
  PointMap map_point(const Vec3& xi) const;
  struct SurfacePoint {
    Vec3 xi, x, normal;
    double area_scale;
  };
  SurfacePoint face_point(FaceId f, double u, double v) const;
  struct FieldEval {
    double value;
    Vec3 grad;
  };
  FieldEval field_at(const double* coeffs, const Vec3& xi) const;
  NurbsVolume refined(const std::array<std::vector<double>, 3>& new_knots) const;

 private:
  std::array<KnotVector, 3> kv_;
  ControlGrid grid_;
};

NurbsVolume quarter_cylinder_part();

// Geometry tooling (not in the reference): exact degree
// elevation by t[d] per direction, an optional per-axis scaling of the control
// coordinates, and the reference's geometry-file text ([geometry] degrees,
// knots_*, grid_dims, cp lines; proj/src/config.cpp:171-215).
NurbsVolume elevate_degree(const NurbsVolume& vol, std::array<int, 3> t);
NurbsVolume scaled(const NurbsVolume& vol, std::array<double, 3> s);
std::string geometry_text(const NurbsVolume& vol);

std::vector<double> graded_refinement_knots(const KnotVector& kv, int target_elements,
                                            double ratio, double focus);

}  // namespace tgb
