// Host side of the boundary: filter band decomposition and per-band rendering.
// These run once per filter on the CPU (north star: "Filter band decomposition
// stays on the host and runs once per filter"); the rendered components feed
// the device spectrum cache.  Reference: proj/include/xconv/freq_filter.hpp,
// polar.hpp, field.hpp.
#pragma once
#include <complex>
#include <stdexcept>
#include <string>
#include <vector>

namespace xcb {

using cplx = std::complex<double>;

struct HostFilter {  // FreqFilter2, freq_filter.hpp:21-46
  int group = 0;     // 0 rotation2, 1 scale2
  int K = 0;
  std::vector<int> ks;
  std::vector<cplx> comps;  // row-major [n_rows][nc]
  int n_radii = 0, n_angles = 0;
  double r_max = 0, r_min = 0, r_domain = 0;

  int nc() const { return int(ks.size()); }
  int n_rows() const { return group == 0 ? n_radii : n_angles; }
  const cplx& comp(int row, int ci) const { return comps[size_t(row) * nc() + ci]; }
  double domain_top() const { return r_domain > 0 ? r_domain : r_max; }
  double omega() const;
  int index_of(int k) const;
  int render_radius() const;  // engine.hpp:255-258
  // F_{-k} = conj(F_k) for every retained k (a real filter's angular /
  // log-radial bands), to 1e-12 of the largest coefficient
  bool hermitian() const;
};

// Field2 view of a complex image, row-major [y][x].
struct ImageView {
  const cplx* data;
  int width, height;
  cplx sample(double x, double y) const;  // field.hpp:51-62
};

HostFilter decompose_rotation2(const ImageView& f, double cx, double cy, int K,
                               int n_radii, int n_angles, double r_max);
HostFilter decompose_scale2(const ImageView& f, double cx, double cy, int K,
                            int n_radii, int n_angles, double r_min, double r_max,
                            double r_domain);
// the validated metadata of a decomposition (ks, sampling, radii) without the
// coefficients: the device decomposition (xc_decompose_*_device) fills comps
HostFilter rotation2_shell(int K, int n_radii, int n_angles, double r_max);
HostFilter scale2_shell(int K, int n_radii, int n_angles, double r_min, double r_max,
                        double r_domain);
cplx component_value(const HostFilter& f, int ci, double r, double theta);
cplx inner_dc_value(const HostFilter& f);
// (2R+1)^2-style rendering, row-major [y][x]; transpose=true renders f(y,x)
// (used when the caller's grids are column-major).
void render_component(const HostFilter& f, int ci, int width, int height, double cx,
                      double cy, bool transpose, cplx* out);
void reconstruct(const HostFilter& f, int width, int height, double cx, double cy,
                 const int* subset, int nsub, bool transpose, cplx* out);

// Vote filters of the generalized-Hough detector (vote_filter.hpp:8-95):
// (2R+1)^2 non-negative weights, row-major [y][x], origin at the centre,
// R = ceil(eps).  Inputs are row-major [h][w] real grids.
struct VoteFilterHost {
  std::vector<double> weights;
  int radius = 0;
  double eps = 0;
};
VoteFilterHost build_vote_filter(const double* weight, const double* frame, int h, int w,
                                 double px, double py, double eps, bool nearest);
VoteFilterHost build_optimal_filter(const double* pattern, int h, int w, double px, double py,
                                    double eps, bool nearest);
// central-difference gradient, one-sided at the borders (field.hpp:204-237)
void gradient_host(const double* img, int h, int w, double* mag, double* dir);

}  // namespace xcb
