// Host-side filter decomposition and rendering (see host_filter.h).
#include "host_filter.h"

#include <algorithm>
#include <cmath>

namespace xcb {

namespace {
constexpr double kPi = 3.14159265358979323846264338327950288;  // EIGEN_PI
constexpr double kTwoPi = 2.0 * kPi;

// polar.hpp:36-43
void check_polar_params(int n_radii, int n_angles, double r_max) {
  if (n_radii < 1) throw std::invalid_argument("n_radii must be >= 1");
  if (n_angles < 4 || n_angles % 2 != 0)
    throw std::invalid_argument("n_angles must be >= 4 and even");
  if (!(r_max > 0.0)) throw std::invalid_argument("r_max must be > 0");
}

// freq_filter.hpp:52-59: K -> k in [-K/2, K/2]
std::vector<int> retained(int K, int n_periodic) {
  const int kh = K / 2;
  if (kh > n_periodic / 2)
    throw std::invalid_argument("band limit too large for sampling rate");
  std::vector<int> ks;
  for (int k = -kh; k <= kh; ++k) ks.push_back(k);
  return ks;
}

// Bilinear polar / log-polar resampling, polar.hpp:46-83: rows = radius
// r_j, columns = angle 2 pi m / n_angles.
std::vector<cplx> polar_samples(const ImageView& f, double cx, double cy, int n_radii,
                                int n_angles, bool log_radial, double r_min,
                                double r_max) {
  std::vector<cplx> p(size_t(n_radii) * n_angles);
  for (int j = 0; j < n_radii; ++j) {
    const double r = log_radial ? r_min * std::pow(r_max / r_min, (j + 0.5) / n_radii)
                                : (j + 0.5) * r_max / n_radii;
    for (int m = 0; m < n_angles; ++m) {
      const double th = kTwoPi * m / n_angles;
      p[size_t(j) * n_angles + m] = f.sample(cx + r * std::cos(th), cy + r * std::sin(th));
    }
  }
  return p;
}
}  // namespace

double HostFilter::omega() const {  // freq_filter.hpp:44-45
  return kTwoPi / std::log(domain_top() / r_min);
}

int HostFilter::index_of(int k) const {  // freq_filter.hpp:35-39
  for (int i = 0; i < nc(); ++i)
    if (ks[i] == k) return i;
  throw std::invalid_argument("frequency not retained");
}

int HostFilter::render_radius() const { return int(std::ceil(r_max)); }

cplx ImageView::sample(double x, double y) const {
  const double fx = std::floor(x), fy = std::floor(y);
  const int x0 = int(fx), y0 = int(fy);
  const double tx = x - fx, ty = y - fy;
  auto tap = [&](int xi, int yi) {
    return (xi < 0 || yi < 0 || xi >= width || yi >= height) ? cplx(0)
                                                             : data[size_t(yi) * width + xi];
  };
  return (1.0 - ty) * ((1.0 - tx) * tap(x0, y0) + tx * tap(x0 + 1, y0)) +
         ty * ((1.0 - tx) * tap(x0, y0 + 1) + tx * tap(x0 + 1, y0 + 1));
}

// freq_filter.hpp:63-89: per-radius angular DFT of the polar resampling;
// the |k| = n_angles/2 coefficient is halved (split over +-k).
HostFilter rotation2_shell(int K, int n_radii, int n_angles, double r_max) {
  check_polar_params(n_radii, n_angles, r_max);
  HostFilter f;
  f.group = 0;
  f.K = K;
  f.ks = retained(K, n_angles);
  f.n_radii = n_radii;
  f.n_angles = n_angles;
  f.r_max = r_max;
  return f;
}

HostFilter decompose_rotation2(const ImageView& img, double cx, double cy, int K,
                               int n_radii, int n_angles, double r_max) {
  HostFilter f = rotation2_shell(K, n_radii, n_angles, r_max);
  const auto p = polar_samples(img, cx, cy, n_radii, n_angles, false, 0.0, r_max);
  const int nc = f.nc();
  f.comps.assign(size_t(n_radii) * nc, cplx(0));
  for (int ci = 0; ci < nc; ++ci) {
    const int k = f.ks[ci];
    const double half = (2 * std::abs(k) == n_angles) ? 0.5 : 1.0;
    for (int j = 0; j < n_radii; ++j) {
      cplx acc(0);
      for (int m = 0; m < n_angles; ++m) {
        const double ph = -kTwoPi * k * m / n_angles;
        acc += p[size_t(j) * n_angles + m] * cplx(std::cos(ph), std::sin(ph));
      }
      f.comps[size_t(j) * nc + ci] = acc * half / double(n_angles);
    }
  }
  return f;
}

// freq_filter.hpp:91-129: per-angle log-radial DFT with basis phase
// 2 pi k (j + 1/2) / n_radii.
HostFilter scale2_shell(int K, int n_radii, int n_angles, double r_min, double r_max,
                        double r_domain) {
  if (!(r_min > 0.0))
    throw std::invalid_argument("r_min must be > 0 (log-polar excludes the origin)");
  if (r_domain != 0.0 && r_domain < r_max)
    throw std::invalid_argument("basis domain must reach the support radius");
  const double D = r_domain > 0 ? r_domain : r_max;
  check_polar_params(n_radii, n_angles, D);
  if (!(r_min < D)) throw std::invalid_argument("log-polar sampling needs 0 < r_min < r_max");
  HostFilter f;
  f.group = 1;
  f.K = K;
  f.ks = retained(K, n_radii);
  f.n_radii = n_radii;
  f.n_angles = n_angles;
  f.r_max = r_max;
  f.r_min = r_min;
  f.r_domain = D;
  return f;
}

HostFilter decompose_scale2(const ImageView& img, double cx, double cy, int K,
                            int n_radii, int n_angles, double r_min, double r_max,
                            double r_domain) {
  HostFilter f = scale2_shell(K, n_radii, n_angles, r_min, r_max, r_domain);
  const double D = f.r_domain;
  const auto p = polar_samples(img, cx, cy, n_radii, n_angles, true, r_min, D);
  const int nc = f.nc();
  f.comps.assign(size_t(n_angles) * nc, cplx(0));
  for (int ci = 0; ci < nc; ++ci) {
    const int k = f.ks[ci];
    const double half = (2 * std::abs(k) == n_radii) ? 0.5 : 1.0;
    for (int m = 0; m < n_angles; ++m) {
      cplx acc(0);
      for (int j = 0; j < n_radii; ++j) {
        const double ph = -kTwoPi * k * (j + 0.5) / n_radii;
        acc += p[size_t(j) * n_angles + m] * cplx(std::cos(ph), std::sin(ph));
      }
      f.comps[size_t(m) * nc + ci] = acc * half / double(n_radii);
    }
  }
  return f;
}

// freq_filter.hpp:131-159
cplx component_value(const HostFilter& f, int ci, double r, double theta) {
  const int k = f.ks[ci];
  if (f.group == 0) {
    if (r <= 1e-9 && k != 0) return cplx(0);
    double u = r / f.r_max * f.n_radii - 0.5;
    u = std::min(std::max(u, 0.0), double(f.n_radii - 1));
    const int j0 = int(u), j1 = std::min(j0 + 1, f.n_radii - 1);
    const double t = u - j0;
    return ((1 - t) * f.comp(j0, ci) + t * f.comp(j1, ci)) * std::polar(1.0, k * theta);
  }
  const int na = f.n_angles;
  double v = theta / kTwoPi * na;
  v -= std::floor(v / na) * na;
  const int m0 = int(v) % na, m1 = (m0 + 1) % na;
  const double t = v - std::floor(v);
  if (r < f.r_min) return cplx(0);
  return ((1 - t) * f.comp(m0, ci) + t * f.comp(m1, ci)) *
         std::polar(1.0, k * f.omega() * std::log(r / f.r_min));
}

// freq_filter.hpp:165-169: sum over bands of the angular mean.
cplx inner_dc_value(const HostFilter& f) {
  if (f.group != 1) return cplx(0);
  cplx s(0);
  for (int ci = 0; ci < f.nc(); ++ci) {
    cplx m(0);
    for (int row = 0; row < f.n_angles; ++row) m += f.comp(row, ci);
    s += m / double(f.n_angles);
  }
  return s;
}

// freq_filter.hpp:172-184 (y points down; zero beyond r_max)
void render_component(const HostFilter& f, int ci, int width, int height, double cx,
                      double cy, bool transpose, cplx* out) {
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < width; ++x) {
      const double dx = double(x) - cx, dy = double(y) - cy;
      const double r = std::sqrt(dx * dx + dy * dy);
      const cplx v = r > f.r_max ? cplx(0) : component_value(f, ci, r, std::atan2(dy, dx));
      out[transpose ? size_t(x) * height + y : size_t(y) * width + x] = v;
    }
}

// freq_filter.hpp:216-235
void reconstruct(const HostFilter& f, int width, int height, double cx, double cy,
                 const int* subset, int nsub, bool transpose, cplx* out) {
  const size_t n = size_t(width) * height;
  std::fill(out, out + n, cplx(0));
  std::vector<cplx> tmp(n);
  for (int ci = 0; ci < f.nc(); ++ci) {
    if (subset && nsub >= 0 && std::find(subset, subset + nsub, f.ks[ci]) == subset + nsub)
      continue;
    render_component(f, ci, width, height, cx, cy, transpose, tmp.data());
    for (size_t i = 0; i < n; ++i) out[i] += tmp[i];
  }
  if (f.group == 1) {
    const cplx dc = inner_dc_value(f);
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) {
        const double dx = double(x) - cx, dy = double(y) - cy;
        if (dx * dx + dy * dy < f.r_min * f.r_min)
          out[transpose ? size_t(x) * height + y : size_t(y) * width + x] = dc;
      }
  }
}

bool HostFilter::hermitian() const {
  double mx = 0;
  for (const cplx& c : comps) mx = std::max(mx, std::abs(c));
  const double tol = 1e-12 * std::max(mx, 1e-300);
  for (int ci = 0; ci < nc(); ++ci) {
    int cj = -1;
    for (int j = 0; j < nc(); ++j)
      if (ks[j] == -ks[ci]) cj = j;
    if (cj < 0) return false;
    for (int r = 0; r < n_rows(); ++r)
      if (std::abs(comp(r, cj) - std::conj(comp(r, ci))) > tol) return false;
  }
  return true;
}

// ------------------------------------------------------------------ vote filters
void gradient_host(const double* img, int h, int w, double* mag, double* dir) {
  auto I = [&](int y, int x) { return img[size_t(y) * w + x]; };
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const double gx = w == 1 ? 0.0
                        : x == 0 ? I(y, 1) - I(y, 0)
                        : x == w - 1 ? I(y, w - 1) - I(y, w - 2)
                                     : 0.5 * (I(y, x + 1) - I(y, x - 1));
      const double gy = h == 1 ? 0.0
                        : y == 0 ? I(1, x) - I(0, x)
                        : y == h - 1 ? I(h - 1, x) - I(h - 2, x)
                                     : 0.5 * (I(y + 1, x) - I(y - 1, x));
      const double m = std::sqrt(gx * gx + gy * gy);
      mag[size_t(y) * w + x] = m;
      dir[size_t(y) * w + x] = m > 0.0 ? std::atan2(gy, gx) : 0.0;
    }
}

// vote_filter.hpp:43-81: every q with weight(q) > 0 within eps of the centre
// p votes at (p - q) rotated into q's frame (x-axis = frame angle), bilinear
// or nearest splat
VoteFilterHost build_vote_filter(const double* weight, const double* frame, int h, int w,
                                 double px, double py, double eps, bool nearest) {
  if (!(eps > 0.0)) throw std::invalid_argument("support radius must be > 0");
  VoteFilterHost f;
  f.eps = eps;
  f.radius = int(std::ceil(eps));
  const int side = 2 * f.radius + 1;
  f.weights.assign(size_t(side) * side, 0.0);
  auto add = [&](int xi, int yi, double v) {
    if (xi >= 0 && yi >= 0 && xi < side && yi < side) f.weights[size_t(yi) * side + xi] += v;
  };
  bool any = false;
  for (int qy = 0; qy < h; ++qy)
    for (int qx = 0; qx < w; ++qx) {
      const double m = weight[size_t(qy) * w + qx];
      if (m <= 0.0) continue;
      const double ox = px - qx, oy = py - qy;
      if (ox * ox + oy * oy > eps * eps) continue;
      const double a = -frame[size_t(qy) * w + qx];
      const double ca = std::cos(a), sa = std::sin(a);
      const double vx = ca * ox - sa * oy + f.radius, vy = sa * ox + ca * oy + f.radius;
      if (nearest) {
        add(int(std::lround(vx)), int(std::lround(vy)), m);
      } else {
        const int x0 = int(std::floor(vx)), y0 = int(std::floor(vy));
        const double tx = vx - x0, ty = vy - y0;
        add(x0, y0, m * (1 - tx) * (1 - ty));
        add(x0 + 1, y0, m * tx * (1 - ty));
        add(x0, y0 + 1, m * (1 - tx) * ty);
        add(x0 + 1, y0 + 1, m * tx * ty);
      }
      any = true;
    }
  if (!any) throw std::invalid_argument("degenerate pattern: no votes in support");
  return f;
}

// vote_filter.hpp:83-91
VoteFilterHost build_optimal_filter(const double* pattern, int h, int w, double px, double py,
                                    double eps, bool nearest) {
  if (px < 0 || py < 0 || px >= w || py >= h)
    throw std::invalid_argument("center must lie inside the pattern");
  std::vector<double> mag(size_t(h) * w), dir(size_t(h) * w);
  gradient_host(pattern, h, w, mag.data(), dir.data());
  return build_vote_filter(mag.data(), dir.data(), h, w, px, py, eps, nearest);
}

}  // namespace xcb
