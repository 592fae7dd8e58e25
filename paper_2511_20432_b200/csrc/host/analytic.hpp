// Host-side analytic-field setup: material / laser records and the scan-path
// discretization that produces the point-source history K1 consumes.
#pragma once

#include <array>
#include <stdexcept>
#include <string>
#include <vector>

namespace tgb {

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  double& operator[](int i) { return (&x)[i]; }
  double operator[](int i) const { return (&x)[i]; }
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
  Vec3& operator+=(const Vec3& o) {
    x += o.x;
    y += o.y;
    z += o.z;
    return *this;
  }
  // association (x*x + y*y) + z*z, as thermiga::Vec3::dot (core.hpp:27)
  double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
  Vec3 cross(const Vec3& o) const {
    return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x};
  }
  double norm() const;
};

// Error categories of the reference (core.hpp:66-80); mapped to TG_* codes.
struct config_error : std::runtime_error {
  explicit config_error(const std::string& m, int line = 0)
      : std::runtime_error(line > 0 ? "config error (line " + std::to_string(line) + "): " + m
                                    : "config error: " + m) {}
};
struct io_error : std::runtime_error {
  explicit io_error(const std::string& m) : std::runtime_error("i/o error: " + m) {}
};
struct numeric_error : std::runtime_error {
  explicit numeric_error(const std::string& m) : std::runtime_error("numeric error: " + m) {}
};

struct Material {
  double conductivity = 0.0;
  double density = 0.0;
  double heat_capacity = 0.0;
  double platform_temperature = 0.0;
  double diffusivity() const { return conductivity / (density * heat_capacity); }
  double volumetric_capacity() const { return density * heat_capacity; }
  void validate() const;
};

struct LaserSpec {
  double power = 0.0, speed = 0.0, spot_radius = 0.0, absorptivity = 0.0, dt = 0.0;
  void validate() const;
};

// Same field order and size as thermiga::PointSource (analytic.hpp:35-40).
struct PointSource {
  Vec3 position;
  double energy = 0.0;
  double t_activate = 0.0;
  double tau = 0.0;
};
static_assert(sizeof(PointSource) == 48, "PointSource layout");

struct ScanPath {
  std::vector<std::array<double, 2>> waypoints;
  double start_time = 0.0;
  double plane_z = 0.0;
};

// Sources every speed*dt of arc length; source I activates at start + I*dt,
// carries A*P*dt and has tau = t_act - r^2/(8 alpha) (analytic.cpp:22-71).
std::vector<PointSource> discretize_scan(const ScanPath& path, const LaserSpec& laser,
                                         const Material& mat);

struct SuperposeOptions {
  double cull_exponent = 60.0;
};

}  // namespace tgb
