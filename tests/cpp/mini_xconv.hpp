// Minimal stand-ins with the member names and storage order of the reference
// types (proj/include/xconv/field.hpp, freq_filter.hpp, engine.hpp), used to
// compile the C++ drop-in shim without Eigen (absent in this image).  Grids
// are column-major like Eigen's default: values(y, x) at y + x * rows.
#pragma once
#include <complex>
#include <map>
#include <string>
#include <vector>

namespace mini {

template <class T>
struct Grid {
  std::vector<T> v;
  int r = 0, c = 0;
  Grid() = default;
  Grid(int rows, int cols) : v(size_t(rows) * cols), r(rows), c(cols) {}
  T& operator()(int row, int col) { return v[row + size_t(col) * r]; }
  const T& operator()(int row, int col) const { return v[row + size_t(col) * r]; }
  T* data() { return v.data(); }
  const T* data() const { return v.data(); }
  int rows() const { return r; }
  int cols() const { return c; }
};

enum class XformKind { rotation2, scale2, rotation3 };
enum class XMode { correlation, convolution };

template <class Real>
struct Field2 {
  Grid<std::complex<Real>> values;
  Field2() = default;
  Field2(int w, int h) : values(h, w) {}
  int width() const { return values.cols(); }
  int height() const { return values.rows(); }
};

template <class Real>
struct Field3 {  // field.hpp:66-85: x fastest
  int nx = 0, ny = 0, nz = 0;
  std::vector<std::complex<Real>> values;
  Field3() = default;
  Field3(int x, int y, int z) : nx(x), ny(y), nz(z), values(size_t(x) * y * z) {}
};

template <class Real>
struct Quaternion {  // the accessors of Eigen::Quaternion
  Real qw = 1, qx = 0, qy = 0, qz = 0;
  Real w() const { return qw; }
  Real x() const { return qx; }
  Real y() const { return qy; }
  Real z() const { return qz; }
};

template <class Real>
struct XformField {
  XformKind kind = XformKind::rotation2;
  Grid<Real> angle, scale;
  int nx = 0, ny = 0, nz = 0;
  std::vector<Quaternion<Real>> quats;
  int width() const { return kind == XformKind::scale2 ? scale.cols() : angle.cols(); }
  int height() const { return kind == XformKind::scale2 ? scale.rows() : angle.rows(); }
};

template <class Real>
struct FreqFilter2 {
  XformKind group = XformKind::rotation2;
  int K = 0;
  std::vector<int> ks;
  Grid<std::complex<Real>> comps;
  int n_radii = 0, n_angles = 0;
  Real r_max = 0, r_min = 0, r_domain = 0;
};

template <class Real>
struct SphFilter3 {  // sph.hpp:130-157
  int K = 0, n_radii = 0;
  Real r_max = 0;
  Grid<std::complex<Real>> coeffs;  // (n_radii, (K+1)^2)
};

struct XConvPlan {
  XMode mode = XMode::correlation;
  XformKind group = XformKind::rotation2;
  std::vector<int> components;
  bool periodic = false;
};

template <class Real>
struct Response2 {
  Field2<Real> output;
  XConvPlan plan;
  long long standard_ops = 0;
  std::map<std::string, double> seconds;
};

template <class Real>
struct Response3 {  // engine.hpp:31-37
  Field3<Real> output;
  XConvPlan plan;
  long long standard_ops = 0;
  std::map<std::string, double> seconds;
};

template <class Real>
struct SmoothResult {
  Field2<Real> output;
  long long standard_ops = 0;
  int clamped_pixels = 0;
};

template <class Real>
struct VoteFilter {  // vote_filter.hpp:8-26
  Grid<Real> weights;
  int radius = 0;
  Real eps = 0;
};

template <class Real>
struct Peak {  // vote_filter.hpp:99-102
  int x = 0, y = 0;
  Real value = 0;
};

template <class Real>
struct DetectionResult {  // vote_filter.hpp:137-142
  Field2<Real> response;
  std::vector<Peak<Real>> peaks;
  long long standard_ops = 0;
};

}  // namespace mini
