// xconv_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see xconv_oracle.h).
//
// Double-precision CPU restatement of the reference 2D path
// (/root/reference/proj/include/xconv/{fft,freq_filter,polar,field,engine,
// vote_filter,contour}.hpp).  Every function cites the reference lines it
// restates.  Grids are row-major [y][x]; the reference stores Eigen
// column-major values(y,x) -- element-for-element the same grid.
//
// FFT: the reference calls Eigen's unsupported FFT module with its default
// kissfft backend (fft.hpp:3, 19-53; Eigen >= 3.4, version unpinned).  Its
// published algorithm is restated below: recursive mixed-radix
// decimation-in-time with radix-4 first, then 2, 3, 5, generic odd factors,
// forward e^{-2 pi i jk/n} unscaled, inverse e^{+} scaled by 1/n (Eigen's
// default, round trip pinned by proj/tests/test_fft.cpp:40-47).

#include "xconv_oracle.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846264338327950288;  // Real(EIGEN_PI)

thread_local std::string g_err;

struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// ---------------------------------------------------------------- FFT (kissfft)

struct KissPlan {
  int n = 0;
  std::vector<int> radix, remain;  // stage radix p and remaining length m
  std::vector<cd> tw[2];           // [0] forward e^{-}, [1] inverse e^{+}
};

std::mutex g_plan_mu;
std::map<int, std::shared_ptr<KissPlan>> g_plans;

std::shared_ptr<KissPlan> kiss_plan(int n) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find(n);
  if (it != g_plans.end()) return it->second;
  auto p = std::make_shared<KissPlan>();
  p->n = n;
  for (int inv = 0; inv < 2; ++inv) {
    p->tw[inv].resize(n);
    for (int i = 0; i < n; ++i) {
      const double phase = (inv ? 2.0 : -2.0) * kPi * i / n;
      p->tw[inv][i] = cd(std::cos(phase), std::sin(phase));
    }
  }
  // factorization order of kissfft: 4 first, then 2, 3, 5, 7, ...
  int m = n, f = 4;
  do {
    while (m % f) {
      if (f == 4) f = 2;
      else if (f == 2) f = 3;
      else f += 2;
      if (f * f > m) f = m;
    }
    m /= f;
    p->radix.push_back(f);
    p->remain.push_back(m);
  } while (m > 1);
  g_plans[n] = p;
  return p;
}

void kiss_bfly(const KissPlan& pl, bool inv, cd* F, size_t fstride, int P, int m) {
  const cd* tw = pl.tw[inv].data();
  const int n = pl.n;
  if (P == 2) {
    for (int k = 0; k < m; ++k) {
      const cd t = F[m + k] * tw[k * fstride];
      F[m + k] = F[k] - t;
      F[k] += t;
    }
  } else if (P == 4) {
    for (int k = 0; k < m; ++k) {
      const cd s0 = F[k + m] * tw[k * fstride];
      const cd s1 = F[k + 2 * m] * tw[2 * k * fstride];
      const cd s2 = F[k + 3 * m] * tw[3 * k * fstride];
      const cd s5 = F[k] - s1;
      const cd a = F[k] + s1;
      const cd s3 = s0 + s2, s4 = s0 - s2;
      F[k + 2 * m] = a - s3;
      F[k] = a + s3;
      // forward multiplies (s0-s2) by -i, inverse by +i
      const cd rot = inv ? cd(-s4.imag(), s4.real()) : cd(s4.imag(), -s4.real());
      F[k + m] = s5 + rot;
      F[k + 3 * m] = s5 - rot;
    }
  } else if (P == 3) {
    const double s3 = tw[fstride * m].imag();  // sin(-+2pi/3)
    for (int k = 0; k < m; ++k) {
      const cd a = F[k];
      const cd b = F[k + m] * tw[k * fstride];
      const cd c = F[k + 2 * m] * tw[2 * k * fstride];
      const cd sum = b + c, dif = b - c;
      const cd mid = a - 0.5 * sum;
      const cd rot(-s3 * dif.imag(), s3 * dif.real());  // i*s3*dif
      F[k] = a + sum;
      F[k + m] = mid + rot;
      F[k + 2 * m] = mid - rot;
    }
  } else {
    // generic odd radix (5 and above): direct P-point DFT of twiddled inputs
    std::vector<cd> scratch(P);
    for (int k = 0; k < m; ++k) {
      for (int q = 0; q < P; ++q) scratch[q] = F[k + q * m] * tw[(size_t(q) * k * fstride) % n];
      for (int u = 0; u < P; ++u) {
        cd acc = scratch[0];
        for (int q = 1; q < P; ++q)
          acc += scratch[q] * tw[(size_t(q) * u * m * fstride) % n];
        F[k + u * m] = acc;
      }
    }
  }
}

void kiss_work(const KissPlan& pl, bool inv, int stage, cd* out, const cd* in,
               size_t fstride, size_t in_stride) {
  const int P = pl.radix[stage], m = pl.remain[stage];
  if (m == 1) {
    for (int j = 0; j < P; ++j) out[j] = in[j * fstride * in_stride];
  } else {
    for (int j = 0; j < P; ++j)
      kiss_work(pl, inv, stage + 1, out + j * m, in + j * fstride * in_stride,
                fstride * P, in_stride);
  }
  kiss_bfly(pl, inv, out, fstride, P, m);
}

// One 1D transform of n elements at `base` with element stride `stride`
// (Eigen::FFT::fwd / ::inv on a copied vector, fft.hpp:20-47).
void fft1d(cd* base, int n, size_t stride, bool inverse, std::vector<cd>& in,
           std::vector<cd>& out) {
  if (n <= 1) return;
  auto pl = kiss_plan(n);
  in.resize(n);
  out.resize(n);
  for (int i = 0; i < n; ++i) in[i] = base[i * stride];
  kiss_work(*pl, inverse, 0, out.data(), in.data(), 1, 1);
  const double s = inverse ? 1.0 / n : 1.0;
  for (int i = 0; i < n; ++i) base[i * stride] = out[i] * s;
}

// fft.hpp:49-53: columns then rows.
void fft2(std::vector<cd>& a, int h, int w, bool inverse) {
  std::vector<cd> in, out;
  for (int x = 0; x < w; ++x) fft1d(a.data() + x, h, w, inverse, in, out);
  for (int y = 0; y < h; ++y) fft1d(a.data() + size_t(y) * w, w, 1, inverse, in, out);
}

int next_fast_size(int n) {  // fft.hpp:9-17
  if (n < 1) return 1;
  for (int s = n;; ++s) {
    int m = s;
    for (int f : {2, 3, 5})
      while (m % f == 0) m /= f;
    if (m == 1) return s;
  }
}

// fft.hpp:59-69
std::vector<cd> wrap_filter(const cd* f, int fh, int fw, int fcx, int fcy, int ph,
                            int pw) {
  std::vector<cd> out(size_t(ph) * pw, cd(0));
  for (int y = 0; y < fh; ++y)
    for (int x = 0; x < fw; ++x) {
      const int u = ((x - fcx) % pw + pw) % pw;
      const int v = ((y - fcy) % ph + ph) % ph;
      out[size_t(v) * pw + u] += f[size_t(y) * fw + x];
    }
  return out;
}

// fft.hpp:78-100
std::vector<cd> filter2_fft(const cd* sig, int h, int w, const cd* filt, int fh,
                            int fw, int fcx, int fcy, bool correlate, bool periodic) {
  const int ph = periodic ? h : next_fast_size(h + fh);
  const int pw = periodic ? w : next_fast_size(w + fw);
  std::vector<cd> A(size_t(ph) * pw, cd(0));
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) A[size_t(y) * pw + x] = sig[size_t(y) * w + x];
  std::vector<cd> B = wrap_filter(filt, fh, fw, fcx, fcy, ph, pw);
  fft2(A, ph, pw, false);
  fft2(B, ph, pw, false);
  for (size_t i = 0; i < A.size(); ++i) A[i] *= correlate ? std::conj(B[i]) : B[i];
  fft2(A, ph, pw, true);
  std::vector<cd> out(size_t(h) * w);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) out[size_t(y) * w + x] = A[size_t(y) * pw + x];
  return out;
}

// ---------------------------------------------------------------- fields

double normalize_angle(double a) {  // field.hpp:121-127
  const double two_pi = 2.0 * kPi;
  a = std::fmod(a + kPi, two_pi);
  if (a < 0) a += two_pi;
  return a - kPi;
}

// Field2::sample, field.hpp:51-62 (reads outside the grid are 0)
cd sample(const cd* f, int w, int h, double x, double y) {
  const double fx = std::floor(x), fy = std::floor(y);
  const int x0 = int(fx), y0 = int(fy);
  const double tx = x - fx, ty = y - fy;
  auto tap = [&](int xi, int yi) -> cd {
    if (xi < 0 || yi < 0 || xi >= w || yi >= h) return cd(0);
    return f[size_t(yi) * w + xi];
  };
  return (1.0 - ty) * ((1.0 - tx) * tap(x0, y0) + tx * tap(x0 + 1, y0)) +
         ty * ((1.0 - tx) * tap(x0, y0 + 1) + tx * tap(x0 + 1, y0 + 1));
}

// XformField (field.hpp:133-158): angle normalized, or scale + log_scale.
struct Xform {
  int kind = 0;
  int w = 0, h = 0;
  std::vector<double> angle, scale, log_scale;
};

Xform make_xform(int kind, const double* param, int h, int w) {
  Xform T;
  T.kind = kind;
  T.w = w;
  T.h = h;
  const size_t n = size_t(h) * w;
  if (kind == 0) {
    T.angle.resize(n);
    for (size_t i = 0; i < n; ++i) T.angle[i] = normalize_angle(param[i]);
  } else {
    for (size_t i = 0; i < n; ++i)
      if (!(param[i] > 0) || !std::isfinite(param[i]))
        throw InvalidArg("scale field must be strictly positive and finite");
    T.scale.assign(param, param + n);
    T.log_scale.resize(n);
    for (size_t i = 0; i < n; ++i) T.log_scale[i] = std::log(param[i]);
  }
  return T;
}

// ---------------------------------------------------------------- filters

struct Filter {
  int group = 0, K = 0;
  std::vector<int> ks;
  std::vector<cd> comps;  // [n_rows][nc]
  int n_radii = 0, n_angles = 0;
  double r_max = 0, r_min = 0, r_domain = 0;
  int nc() const { return int(ks.size()); }
  int n_rows() const { return group == 0 ? n_radii : n_angles; }
  const cd& c(int row, int ci) const { return comps[size_t(row) * nc() + ci]; }
  int index_of(int k) const {  // freq_filter.hpp:35-39
    for (int i = 0; i < nc(); ++i)
      if (ks[i] == k) return i;
    throw InvalidArg("frequency not retained");
  }
  double domain_top() const { return r_domain > 0 ? r_domain : r_max; }  // :42
  double log_period() const { return std::log(domain_top() / r_min); }    // :44
  double omega() const { return 2.0 * kPi / log_period(); }               // :45
};

Filter to_filter(const or_filter* f) {
  Filter F;
  F.group = f->group;
  F.K = f->K;
  F.ks.assign(f->ks, f->ks + f->nc);
  F.n_radii = f->n_radii;
  F.n_angles = f->n_angles;
  F.r_max = f->r_max;
  F.r_min = f->r_min;
  F.r_domain = f->r_domain;
  const size_t n = size_t(F.n_rows()) * f->nc;
  F.comps.resize(n);
  for (size_t i = 0; i < n; ++i) F.comps[i] = cd(f->comps[2 * i], f->comps[2 * i + 1]);
  return F;
}

// polar.hpp:11-34 (radius of sample row j)
double polar_radius(bool log_radial, double r_min, double r_max, int n_radii, int j) {
  if (log_radial) return r_min * std::pow(r_max / r_min, (double(j) + 0.5) / n_radii);
  return (double(j) + 0.5) * r_max / n_radii;
}

void check_polar_params(int n_radii, int n_angles, double r_max) {  // polar.hpp:37-43
  if (n_radii < 1) throw InvalidArg("n_radii must be >= 1");
  if (n_angles < 4 || n_angles % 2 != 0)
    throw InvalidArg("n_angles must be >= 4 and even");
  if (!(r_max > 0.0)) throw InvalidArg("r_max must be > 0");
}

// freq_filter.hpp:52-59
std::vector<int> retained_ks(int K, int n_periodic) {
  const int kh = K / 2;
  if (kh > n_periodic / 2) throw InvalidArg("band limit too large for sampling rate");
  std::vector<int> ks;
  for (int k = -kh; k <= kh; ++k) ks.push_back(k);
  return ks;
}

// resample_polar (polar.hpp:46-61) + decompose_rotation2 (freq_filter.hpp:63-89)
Filter decompose_rotation2(const cd* filt, int fw, int fh, double cx, double cy, int K,
                           int n_radii, int n_angles, double r_max) {
  check_polar_params(n_radii, n_angles, r_max);
  std::vector<cd> p(size_t(n_radii) * n_angles);
  for (int j = 0; j < n_radii; ++j) {
    const double r = polar_radius(false, 0, r_max, n_radii, j);
    for (int m = 0; m < n_angles; ++m) {
      const double th = 2.0 * kPi * m / n_angles;
      p[size_t(j) * n_angles + m] =
          sample(filt, fw, fh, cx + r * std::cos(th), cy + r * std::sin(th));
    }
  }
  Filter f;
  f.group = 0;
  f.K = K;
  f.ks = retained_ks(K, n_angles);
  f.n_radii = n_radii;
  f.n_angles = n_angles;
  f.r_max = r_max;
  const int nc = f.nc();
  f.comps.assign(size_t(n_radii) * nc, cd(0));
  const double two_pi = 2.0 * kPi;
  for (int ci = 0; ci < nc; ++ci) {
    const int k = f.ks[ci];
    const double half = (2 * std::abs(k) == n_angles) ? 0.5 : 1.0;
    for (int j = 0; j < n_radii; ++j) {
      cd acc(0);
      for (int m = 0; m < n_angles; ++m) {
        const double ph = -two_pi * k * m / n_angles;
        acc += p[size_t(j) * n_angles + m] * cd(std::cos(ph), std::sin(ph));
      }
      f.comps[size_t(j) * nc + ci] = acc * half / double(n_angles);
    }
  }
  return f;
}

// resample_polar_log (polar.hpp:63-83) + decompose_scale2 (freq_filter.hpp:91-129)
Filter decompose_scale2(const cd* filt, int fw, int fh, double cx, double cy, int K,
                        int n_radii, int n_angles, double r_min, double r_max,
                        double r_domain) {
  if (!(r_min > 0.0))
    throw InvalidArg("r_min must be > 0 (log-polar excludes the origin)");
  if (r_domain != 0.0 && r_domain < r_max)
    throw InvalidArg("basis domain must reach the support radius");
  const double D = r_domain > 0 ? r_domain : r_max;
  check_polar_params(n_radii, n_angles, D);
  if (!(r_min > 0.0) || !(r_min < D))
    throw InvalidArg("log-polar sampling needs 0 < r_min < r_max");
  std::vector<cd> p(size_t(n_radii) * n_angles);
  for (int j = 0; j < n_radii; ++j) {
    const double r = polar_radius(true, r_min, D, n_radii, j);
    for (int m = 0; m < n_angles; ++m) {
      const double th = 2.0 * kPi * m / n_angles;
      p[size_t(j) * n_angles + m] =
          sample(filt, fw, fh, cx + r * std::cos(th), cy + r * std::sin(th));
    }
  }
  Filter f;
  f.group = 1;
  f.K = K;
  f.ks = retained_ks(K, n_radii);
  f.n_radii = n_radii;
  f.n_angles = n_angles;
  f.r_max = r_max;
  f.r_min = r_min;
  f.r_domain = D;
  const int nc = f.nc();
  f.comps.assign(size_t(n_angles) * nc, cd(0));
  const double two_pi = 2.0 * kPi;
  for (int ci = 0; ci < nc; ++ci) {
    const int k = f.ks[ci];
    const double half = (2 * std::abs(k) == n_radii) ? 0.5 : 1.0;
    for (int m = 0; m < n_angles; ++m) {
      cd acc(0);
      for (int j = 0; j < n_radii; ++j) {
        const double ph = -two_pi * k * (j + 0.5) / n_radii;
        acc += p[size_t(j) * n_angles + m] * cd(std::cos(ph), std::sin(ph));
      }
      f.comps[size_t(m) * nc + ci] = acc * half / double(n_radii);
    }
  }
  return f;
}

// freq_filter.hpp:131-159
cd component_value(const Filter& f, int ci, double r, double theta) {
  const int k = f.ks[ci];
  if (f.group == 0) {
    if (r <= 1e-9 && k != 0) return cd(0);
    double u = r / f.r_max * f.n_radii - 0.5;
    if (u < 0) u = 0;
    if (u > f.n_radii - 1) u = double(f.n_radii - 1);
    const int j0 = int(u);
    const int j1 = std::min(j0 + 1, f.n_radii - 1);
    const double t = u - j0;
    const cd prof = (1 - t) * f.c(j0, ci) + t * f.c(j1, ci);
    return prof * std::polar(1.0, k * theta);
  }
  const int na = f.n_angles;
  double v = theta / (2.0 * kPi) * na;
  v = v - std::floor(v / na) * na;
  const int m0 = int(v) % na;
  const int m1 = (m0 + 1) % na;
  const double t = v - std::floor(v);
  if (r < f.r_min) return cd(0);
  const cd prof = (1 - t) * f.c(m0, ci) + t * f.c(m1, ci);
  return prof * std::polar(1.0, f.ks[ci] * f.omega() * std::log(r / f.r_min));
}

// freq_filter.hpp:165-169
cd inner_dc_value(const Filter& f) {
  if (f.group != 1) return cd(0);
  cd s(0);
  for (int ci = 0; ci < f.nc(); ++ci) {
    cd m(0);
    for (int row = 0; row < f.n_angles; ++row) m += f.c(row, ci);
    s += m / double(f.n_angles);
  }
  return s;
}

// freq_filter.hpp:172-184
std::vector<cd> render_component(const Filter& f, int ci, int width, int height,
                                 double cx, double cy) {
  std::vector<cd> out(size_t(width) * height, cd(0));
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < width; ++x) {
      const double dx = double(x) - cx, dy = double(y) - cy;
      const double r = std::sqrt(dx * dx + dy * dy);
      if (r > f.r_max) continue;
      out[size_t(y) * width + x] = component_value(f, ci, r, std::atan2(dy, dx));
    }
  return out;
}

bool in_subset(const int* subset, int nsub, int k) {
  if (nsub < 0 || subset == nullptr) return true;
  return std::find(subset, subset + nsub, k) != subset + nsub;
}

// freq_filter.hpp:216-235
std::vector<cd> reconstruct(const Filter& f, int width, int height, double cx,
                            double cy, const int* subset = nullptr, int nsub = -1) {
  std::vector<cd> out(size_t(width) * height, cd(0));
  for (int ci = 0; ci < f.nc(); ++ci) {
    if (!in_subset(subset, nsub, f.ks[ci])) continue;
    auto rc = render_component(f, ci, width, height, cx, cy);
    for (size_t i = 0; i < out.size(); ++i) out[i] += rc[i];
  }
  if (f.group == 1) {
    const cd dc = inner_dc_value(f);
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) {
        const double dx = double(x) - cx, dy = double(y) - cy;
        if (dx * dx + dy * dy < f.r_min * f.r_min) out[size_t(y) * width + x] = dc;
      }
  }
  return out;
}

// ---------------------------------------------------------------- engine

std::vector<int> plan_components(const std::vector<int>& available,
                                  const int* comps, int ncomp) {  // engine.hpp:51-58
  if (comps == nullptr || ncomp <= 0) return available;
  for (int i = 0; i < ncomp; ++i)
    if (std::find(available.begin(), available.end(), comps[i]) == available.end())
      throw InvalidArg("plan retains a component the filter lacks");
  return std::vector<int>(comps, comps + ncomp);
}

void check_scale_guard(const Xform& T, const Filter& F) {  // engine.hpp:267-279
  const double lo = F.r_min / F.domain_top(), hi = F.domain_top() / F.r_min;
  for (int y = 0; y < T.h; ++y)
    for (int x = 0; x < T.w; ++x) {
      const double s = T.scale[size_t(y) * T.w + x];
      if (s < lo || s > hi)
        throw InvalidArg("scale factor " + std::to_string(s) + " at pixel (" +
                         std::to_string(x) + "," + std::to_string(y) +
                         ") outside guard band [" + std::to_string(lo) + "," +
                         std::to_string(hi) + "]");
    }
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// xcorr_fast (engine.hpp:286-326) / xconv_fast (engine.hpp:331-373).
// nthreads > 1: contiguous band ranges per thread, partials summed in
// thread order ("deterministic ordered reduction").
std::vector<cd> xfast(int mode, const std::vector<cd>& H, int h, int w, const Xform& T,
                      const Filter& F, const int* comps, int ncomp, bool periodic,
                      long long* ops, double* secs, int nthreads) {
  if (T.kind != F.group) throw InvalidArg("transformation/filter group mismatch");
  if (T.w != w || T.h != h) throw InvalidArg("signal and transformation field dims differ");
  if (T.kind == 1) check_scale_guard(T, F);
  const int R = int(std::ceil(F.r_max));  // engine.hpp:255-258
  const auto ks = plan_components(F.ks, comps, ncomp);
  const size_t N = size_t(h) * w;
  const int nb = int(ks.size());
  nthreads = std::max(1, std::min(nthreads, nb));
  std::vector<std::vector<cd>> part(nthreads, std::vector<cd>(N, cd(0)));
  std::vector<std::array<double, 4>> tsec(nthreads, {0, 0, 0, 0});
  auto run = [&](int tid) {
    const int b0 = int((long long)nb * tid / nthreads);
    const int b1 = int((long long)nb * (tid + 1) / nthreads);
    std::vector<cd>& out = part[tid];
    for (int bi = b0; bi < b1; ++bi) {
      const int k = ks[bi];
      auto t0 = std::chrono::steady_clock::now();
      auto Fk = render_component(F, F.index_of(k), 2 * R + 1, 2 * R + 1, double(R),
                                 double(R));
      tsec[tid][0] += secs_since(t0);
      // steer_phase (engine.hpp:261-265)
      auto phase = [&](size_t i) {
        return T.kind == 0 ? double(k) * T.angle[i]
                           : double(k) * F.omega() * T.log_scale[i];
      };
      if (mode == 0) {
        t0 = std::chrono::steady_clock::now();
        auto Gk = filter2_fft(H.data(), h, w, Fk.data(), 2 * R + 1, 2 * R + 1, R, R,
                              true, periodic);
        tsec[tid][1] += secs_since(t0);
        t0 = std::chrono::steady_clock::now();
        for (size_t i = 0; i < N; ++i) {
          const double a = phase(i);
          out[i] += Gk[i] * cd(std::cos(a), std::sin(a));
        }
        tsec[tid][2] += secs_since(t0);
      } else {
        t0 = std::chrono::steady_clock::now();
        std::vector<cd> Gk(N);
        for (size_t i = 0; i < N; ++i) {
          const double a = phase(i);
          Gk[i] = H[i] * cd(std::cos(-a), std::sin(-a));
        }
        tsec[tid][3] += secs_since(t0);
        t0 = std::chrono::steady_clock::now();
        Gk = filter2_fft(Gk.data(), h, w, Fk.data(), 2 * R + 1, 2 * R + 1, R, R, false,
                         periodic);
        tsec[tid][1] += secs_since(t0);
        t0 = std::chrono::steady_clock::now();
        for (size_t i = 0; i < N; ++i) out[i] += Gk[i];
        tsec[tid][2] += secs_since(t0);
      }
    }
  };
  if (nthreads == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(run, t);
    for (auto& t : th) t.join();
    for (int t = 1; t < nthreads; ++t)
      for (size_t i = 0; i < N; ++i) part[0][i] += part[t][i];
  }
  std::vector<cd> out = std::move(part[0]);
  if (T.kind == 1) {  // engine.hpp:320-324 / 369-371
    const cd dc = inner_dc_value(F);
    for (size_t i = 0; i < N; ++i) out[i] += (mode == 0 ? std::conj(dc) : dc) * H[i];
  }
  if (ops) *ops = nb;
  if (secs)
    for (int s = 0; s < 4; ++s) {
      secs[s] = 0;
      for (int t = 0; t < nthreads; ++t) secs[s] += tsec[t][s];
    }
  return out;
}

// ---------------------------------------------------------------- brute force

struct PolarTable {  // polar.hpp:11-34
  std::vector<cd> values;  // [n_radii][n_angles]
  int nr = 0, na = 0;
  double r_max = 0, r_min = 0;
  bool log_radial = false;
  cd inner_dc{0};
  double radial_index(double r) const {
    if (log_radial) return std::log(r / r_min) / std::log(r_max / r_min) * nr - 0.5;
    return r / r_max * nr - 0.5;
  }
};

// polar.hpp:85-106
cd polar_sample(const PolarTable& g, double r, double theta) {
  if (r > g.r_max) return cd(0);
  if (r <= 1e-9) {
    cd m(0);
    for (int i = 0; i < g.na; ++i) m += g.values[i];
    return m / double(g.na);
  }
  const int nr = g.nr, na = g.na;
  double u = g.radial_index(r);
  if (u < 0) u = 0;
  if (u > nr - 1) u = double(nr - 1);
  const int j0 = std::min(int(u), nr - 1);
  const int j1 = std::min(j0 + 1, nr - 1);
  const double tu = u - j0;
  double v = theta / (2.0 * kPi) * na;
  v = v - std::floor(v / na) * na;
  const int m0 = int(v) % na;
  const int m1 = (m0 + 1) % na;
  const double tv = v - std::floor(v);
  auto at = [&](int j, int m) { return g.values[size_t(j) * na + m]; };
  return (1 - tu) * ((1 - tv) * at(j0, m0) + tv * at(j0, m1)) +
         tu * ((1 - tv) * at(j1, m0) + tv * at(j1, m1));
}

// engine.hpp:95-124
PolarTable synthesis_table(const Filter& F, int n_radii, int n_angles) {
  const bool log_radial = F.group == 1;
  if (n_radii <= 0)
    n_radii = log_radial ? 512 : std::max(64, 16 * int(std::ceil(F.r_max)));
  if (n_angles <= 0) n_angles = 512;
  PolarTable g;
  g.nr = n_radii;
  g.na = n_angles;
  g.r_max = log_radial ? F.domain_top() : F.r_max;
  if (log_radial) {
    g.log_radial = true;
    g.r_min = F.r_min;
    g.inner_dc = inner_dc_value(F);
  }
  g.values.assign(size_t(n_radii) * n_angles, cd(0));
  for (int j = 0; j < n_radii; ++j) {
    const double r = polar_radius(g.log_radial, g.r_min, g.r_max, n_radii, j);
    for (int m = 0; m < n_angles; ++m) {
      const double th = 2.0 * kPi * m / n_angles;
      cd acc(0);
      for (int ci = 0; ci < F.nc(); ++ci) acc += component_value(F, ci, r, th);
      g.values[size_t(j) * n_angles + m] = acc;
    }
  }
  return g;
}

// engine.hpp:130-146
cd table_sample(const PolarTable& t, int kind, double param, double dx, double dy) {
  const double r = std::hypot(dx, dy);
  const double th = std::atan2(dy, dx);
  if (kind == 0) return polar_sample(t, r, th - param);
  if (t.log_radial) {
    if (r < t.r_min) return t.inner_dc;
    const double L = std::log(t.r_max / t.r_min);
    double tt = std::log(r / (param * t.r_min));
    tt -= std::floor(tt / L) * L;
    return polar_sample(t, t.r_min * std::exp(tt), th);
  }
  return polar_sample(t, r / param, th);
}

// engine.hpp:148-208
std::vector<cd> brute(int mode, const std::vector<cd>& H, int h, int w, const Xform& T,
                      const PolarTable& table, double eps) {
  std::vector<cd> out(size_t(h) * w, cd(0));
  auto par = [&](int y, int x) {
    const size_t i = size_t(y) * w + x;
    return T.kind == 0 ? T.angle[i] : T.scale[i];
  };
  if (mode == 0) {
    for (int py = 0; py < h; ++py)
      for (int px = 0; px < w; ++px) {
        const double param = par(py, px);
        const double reach = T.kind == 1 && !table.log_radial ? eps * param : eps;
        const int R = int(std::ceil(reach));
        cd acc(0);
        for (int qy = std::max(0, py - R); qy <= std::min(h - 1, py + R); ++qy)
          for (int qx = std::max(0, px - R); qx <= std::min(w - 1, px + R); ++qx) {
            const double dx = qx - px, dy = qy - py;
            if (dx * dx + dy * dy > reach * reach) continue;
            acc += H[size_t(qy) * w + qx] *
                   std::conj(table_sample(table, T.kind, param, dx, dy));
          }
        out[size_t(py) * w + px] = acc;
      }
  } else {
    for (int qy = 0; qy < h; ++qy)
      for (int qx = 0; qx < w; ++qx) {
        const cd hv = H[size_t(qy) * w + qx];
        if (hv == cd(0)) continue;
        const double param = par(qy, qx);
        const double reach = T.kind == 1 && !table.log_radial ? eps * param : eps;
        const int R = int(std::ceil(reach));
        for (int py = std::max(0, qy - R); py <= std::min(h - 1, qy + R); ++py)
          for (int px = std::max(0, qx - R); px <= std::min(w - 1, qx + R); ++px) {
            const double dx = px - qx, dy = py - qy;
            if (dx * dx + dy * dy > reach * reach) continue;
            out[size_t(py) * w + px] += hv * table_sample(table, T.kind, param, dx, dy);
          }
      }
  }
  return out;
}

std::vector<cd> to_cd(const double* a, size_t n) {
  std::vector<cd> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = cd(a[2 * i], a[2 * i + 1]);
  return v;
}

void from_cd(const std::vector<cd>& v, double* a) {
  for (size_t i = 0; i < v.size(); ++i) {
    a[2 * i] = v[i].real();
    a[2 * i + 1] = v[i].imag();
  }
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

// ==================================================================== C API

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }
int or_next_fast_size(int n) { return next_fast_size(n); }

void or_fft2(double* a, int h, int w, int inverse) {
  auto v = to_cd(a, size_t(h) * w);
  fft2(v, h, w, inverse != 0);
  from_cd(v, a);
}

void or_filter2_fft(const double* sig, int h, int w, const double* filt, int fh,
                    int fw, int fcx, int fcy, int correlate, int periodic,
                    double* out) {
  auto s = to_cd(sig, size_t(h) * w);
  auto f = to_cd(filt, size_t(fh) * fw);
  from_cd(filter2_fft(s.data(), h, w, f.data(), fh, fw, fcx, fcy, correlate != 0,
                      periodic != 0),
          out);
}

// proj/tests/test_fft.cpp:9-22
void or_correlate_direct(const double* Hd, int h, int w, const double* Fd, int fh,
                         int fw, int fcx, int fcy, double* outd) {
  auto H = to_cd(Hd, size_t(h) * w);
  auto F = to_cd(Fd, size_t(fh) * fw);
  std::vector<cd> out(size_t(h) * w, cd(0));
  for (int py = 0; py < h; ++py)
    for (int px = 0; px < w; ++px)
      for (int qy = 0; qy < h; ++qy)
        for (int qx = 0; qx < w; ++qx) {
          const int ux = qx - px + fcx, uy = qy - py + fcy;
          if (ux < 0 || uy < 0 || ux >= fw || uy >= fh) continue;
          out[size_t(py) * w + px] += H[size_t(qy) * w + qx] * std::conj(F[size_t(uy) * fw + ux]);
        }
  from_cd(out, outd);
}

// proj/tests/test_fft.cpp:24-36
void or_convolve_direct(const double* Hd, int h, int w, const double* Fd, int fh,
                        int fw, int fcx, int fcy, double* outd) {
  auto H = to_cd(Hd, size_t(h) * w);
  auto F = to_cd(Fd, size_t(fh) * fw);
  std::vector<cd> out(size_t(h) * w, cd(0));
  for (int py = 0; py < h; ++py)
    for (int px = 0; px < w; ++px)
      for (int qy = 0; qy < h; ++qy)
        for (int qx = 0; qx < w; ++qx) {
          const int ux = px - qx + fcx, uy = py - qy + fcy;
          if (ux < 0 || uy < 0 || ux >= fw || uy >= fh) continue;
          out[size_t(py) * w + px] += H[size_t(qy) * w + qx] * F[size_t(uy) * fw + ux];
        }
  from_cd(out, outd);
}

static void export_filter(const Filter& f, int* ks_out, double* comps_out, int* nc_out) {
  for (int i = 0; i < f.nc(); ++i) ks_out[i] = f.ks[i];
  from_cd(f.comps, comps_out);
  *nc_out = f.nc();
}

int or_decompose_rotation2(const double* filt, int fw, int fh, double cx, double cy,
                           int K, int n_radii, int n_angles, double r_max,
                           int* ks_out, double* comps_out, int* nc_out) {
  return guarded([&] {
    auto f = to_cd(filt, size_t(fw) * fh);
    export_filter(decompose_rotation2(f.data(), fw, fh, cx, cy, K, n_radii, n_angles, r_max),
                  ks_out, comps_out, nc_out);
  });
}

int or_decompose_scale2(const double* filt, int fw, int fh, double cx, double cy, int K,
                        int n_radii, int n_angles, double r_min, double r_max,
                        double r_domain, int* ks_out, double* comps_out, int* nc_out) {
  return guarded([&] {
    auto f = to_cd(filt, size_t(fw) * fh);
    export_filter(decompose_scale2(f.data(), fw, fh, cx, cy, K, n_radii, n_angles, r_min,
                                   r_max, r_domain),
                  ks_out, comps_out, nc_out);
  });
}

void or_component_value(const or_filter* F, int ci, double r, double theta, double* out2) {
  const cd v = component_value(to_filter(F), ci, r, theta);
  out2[0] = v.real();
  out2[1] = v.imag();
}

void or_render_component(const or_filter* F, int ci, int width, int height, double cx,
                         double cy, double* out) {
  from_cd(render_component(to_filter(F), ci, width, height, cx, cy), out);
}

void or_inner_dc_value(const or_filter* F, double* out2) {
  const cd v = inner_dc_value(to_filter(F));
  out2[0] = v.real();
  out2[1] = v.imag();
}

void or_reconstruct(const or_filter* F, int width, int height, double cx, double cy,
                    const int* subset, int nsub, double* out) {
  from_cd(reconstruct(to_filter(F), width, height, cx, cy, subset, nsub), out);
}

// freq_filter.hpp:187-213
void or_synthesize_polar(const or_filter* Fc, const int* subset, int nsub, double* out) {
  const Filter f = to_filter(Fc);
  std::vector<cd> g(size_t(f.n_radii) * f.n_angles, cd(0));
  const double two_pi = 2.0 * kPi;
  for (int ci = 0; ci < f.nc(); ++ci) {
    const int k = f.ks[ci];
    if (!in_subset(subset, nsub, k)) continue;
    for (int j = 0; j < f.n_radii; ++j)
      for (int m = 0; m < f.n_angles; ++m) {
        const double ph = f.group == 0 ? two_pi * k * m / f.n_angles
                                       : two_pi * k * (j + 0.5) / f.n_radii;
        const cd& prof = f.group == 0 ? f.c(j, ci) : f.c(m, ci);
        g[size_t(j) * f.n_angles + m] += prof * cd(std::cos(ph), std::sin(ph));
      }
  }
  from_cd(g, out);
}

int or_xfast(int mode, const double* Hd, int h, int w, int kind, const double* param,
             const or_filter* Fc, const int* components, int ncomp, int periodic,
             double* out, long long* ops_out, double* seconds_out, int nthreads) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const Xform T = make_xform(kind, param, h, w);
    auto H = to_cd(Hd, size_t(h) * w);
    from_cd(xfast(mode, H, h, w, T, F, components, ncomp, periodic != 0, ops_out,
                  seconds_out, nthreads),
            out);
  });
}

int or_smooth_adaptive(const double* Hd, int h, int w, int kind, const double* param,
                       const or_filter* Fc, int normalize, double* out_real,
                       long long* ops_out, int* clamped_out, int nthreads) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const Xform T = make_xform(kind, param, h, w);
    const size_t N = size_t(h) * w;
    auto H = to_cd(Hd, N);
    // engine.hpp:388-392
    const int R = int(std::ceil(F.r_max));
    auto full = reconstruct(F, 2 * R + 1, 2 * R + 1, double(R), double(R));
    cd integral(0);
    double mx = 0;
    for (auto& v : full) {
      integral += v;
      mx = std::max(mx, std::abs(v));
    }
    if (std::abs(integral) < 1e-12 * std::max(1.0, mx))
      throw InvalidArg("normalization undefined: filter has zero integral");
    // engine.hpp:394-401
    std::vector<cd> Ht = H, ones(N, cd(1));
    if (normalize && T.kind == 1) {
      for (size_t i = 0; i < N; ++i) {
        const double inv = 1.0 / (T.scale[i] * T.scale[i]);
        Ht[i] = H[i] * cd(inv);
        ones[i] = cd(inv);
      }
    }
    long long o1 = 0, o2 = 0;
    auto num = xfast(1, Ht, h, w, T, F, nullptr, 0, false, &o1, nullptr, nthreads);
    auto den = xfast(1, ones, h, w, T, F, nullptr, 0, false, &o2, nullptr, nthreads);
    // engine.hpp:405-418
    double dmax = 0;
    for (auto& d : den) dmax = std::max(dmax, std::abs(d));
    const double floor_ = 1e-9 * dmax;
    int clamped = 0;
    for (size_t i = 0; i < N; ++i) {
      if (std::abs(den[i]) < floor_) {
        ++clamped;
        out_real[i] = 0;
        continue;
      }
      out_real[i] = std::real(num[i] / den[i]);
    }
    if (ops_out) *ops_out = o1 + o2;
    if (clamped_out) *clamped_out = clamped;
  });
}

int or_xbrute(int mode, const double* Hd, int h, int w, int kind, const double* param,
              const or_filter* Fc, double eps, int table_radii, int table_angles,
              double* out) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const Xform T = make_xform(kind, param, h, w);
    if (eps <= 0) eps = F.r_max;  // engine.hpp:237
    auto H = to_cd(Hd, size_t(h) * w);
    from_cd(brute(mode, H, h, w, T, synthesis_table(F, table_radii, table_angles), eps), out);
  });
}

// test_engine2d.cpp:33-61 (rotation) and test_engine_scale.cpp:37-78 (scale)
int or_spectral_oracle(int mode, const double* Hd, int h, int w, int kind,
                       const double* param, const or_filter* Fc, double* outd) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const Xform T = make_xform(kind, param, h, w);
    auto H = to_cd(Hd, size_t(h) * w);
    const int R = int(std::ceil(F.r_max));
    std::vector<cd> out(size_t(h) * w, cd(0));
    const double om = kind == 1 ? F.omega() : 0.0;
    const cd dc = inner_dc_value(F);
    for (int py = 0; py < h; ++py)
      for (int px = 0; px < w; ++px)
        for (int dy = -R; dy <= R; ++dy)
          for (int dx = -R; dx <= R; ++dx) {
            const double r = std::hypot(double(dx), double(dy));
            if (r > F.r_max) continue;
            const double th = std::atan2(double(dy), double(dx));
            const int qx = mode == 0 ? px + dx : px - dx;
            const int qy = mode == 0 ? py + dy : py - dy;
            if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
            const size_t pi = size_t(mode == 0 ? py : qy) * w + (mode == 0 ? px : qx);
            cd acc(0);
            if (kind == 0) {
              for (int ci = 0; ci < F.nc(); ++ci)
                acc += component_value(F, ci, r, th - T.angle[pi]);
              if (mode == 0) acc = std::conj(acc);
            } else {
              const double ls = std::log(T.scale[pi]);
              if (r < F.r_min) {
                acc = mode == 0 ? std::conj(dc) : dc;
              } else {
                for (int ci = 0; ci < F.nc(); ++ci) {
                  const cd cv = component_value(F, ci, r, th);
                  acc += mode == 0 ? std::conj(cv) * std::polar(1.0, F.ks[ci] * om * ls)
                                   : cv * std::polar(1.0, -F.ks[ci] * om * ls);
                }
              }
            }
            out[size_t(py) * w + px] += H[size_t(qy) * w + qx] * acc;
          }
    from_cd(out, outd);
  });
}

// Spectral oracle evaluated only at the listed pixels (test_engine2d.cpp:33-61
// / test_engine_scale.cpp:37-78 restricted to p in `pix`): full-size parity
// checks sample pixels instead of running the whole O(N R^2 B) loop.
// H and param are float32 (the arrays the GPU consumed), upcast to double.
int or_spectral_oracle_at(int mode, const float* Hf, int h, int w, int kind,
                          const float* paramf, const or_filter* Fc, const int* pys,
                          const int* pxs, int npix, double* outd) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const int R = int(std::ceil(F.r_max));
    const double om = kind == 1 ? F.omega() : 0.0;
    const cd dc = inner_dc_value(F);
    // per-offset component values for rotation are angle dependent; precompute
    // r, theta per offset only
    for (int t = 0; t < npix; ++t) {
      const int py = pys[t], px = pxs[t];
      cd acc_out(0);
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          const double r = std::hypot(double(dx), double(dy));
          if (r > F.r_max) continue;
          const double th = std::atan2(double(dy), double(dx));
          const int qx = mode == 0 ? px + dx : px - dx;
          const int qy = mode == 0 ? py + dy : py - dy;
          if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
          const size_t pi = size_t(mode == 0 ? py : qy) * w + (mode == 0 ? px : qx);
          const double prm = double(paramf[pi]);
          cd acc(0);
          if (kind == 0) {
            const double a = normalize_angle(prm);
            for (int ci = 0; ci < F.nc(); ++ci) acc += component_value(F, ci, r, th - a);
            if (mode == 0) acc = std::conj(acc);
          } else {
            const double ls = std::log(prm);
            if (r < F.r_min) {
              acc = mode == 0 ? std::conj(dc) : dc;
            } else {
              for (int ci = 0; ci < F.nc(); ++ci) {
                const cd cv = component_value(F, ci, r, th);
                acc += mode == 0 ? std::conj(cv) * std::polar(1.0, F.ks[ci] * om * ls)
                                 : cv * std::polar(1.0, -F.ks[ci] * om * ls);
              }
            }
          }
          acc_out += cd(double(Hf[size_t(qy) * w + qx]), 0.0) * acc;
        }
      outd[2 * t] = acc_out.real();
      outd[2 * t + 1] = acc_out.imag();
    }
  });
}

// vote_filter.hpp:105-134
int or_find_peaks(const double* resp, int h, int w, double radius, double threshold_frac,
                  int* xs, int* ys, double* vals, int max_out) {
  struct Pk {
    int x, y;
    double v;
  };
  std::vector<Pk> peaks;
  double mx = -INFINITY;
  for (size_t i = 0; i < size_t(h) * w; ++i) mx = std::max(mx, resp[i]);
  const double thresh = threshold_frac * mx;
  const int R = std::max(1, int(std::ceil(radius)));
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const double v = resp[size_t(y) * w + x];
      if (v < thresh) continue;
      bool best = true;
      for (int dy = -R; dy <= R && best; ++dy)
        for (int dx = -R; dx <= R && best; ++dx) {
          if (dx == 0 && dy == 0) continue;
          if (dx * dx + dy * dy > radius * radius) continue;
          const int xi = x + dx, yi = y + dy;
          if (xi < 0 || yi < 0 || xi >= w || yi >= h) continue;
          const double o = resp[size_t(yi) * w + xi];
          if (o > v || (o == v && (dy < 0 || (dy == 0 && dx < 0)))) best = false;
        }
      if (best) peaks.push_back({x, y, v});
    }
  std::sort(peaks.begin(), peaks.end(), [](const Pk& a, const Pk& b) {
    if (a.v != b.v) return a.v > b.v;
    return a.y != b.y ? a.y < b.y : a.x < b.x;
  });
  const int n = int(peaks.size());
  for (int i = 0; i < std::min(n, max_out); ++i) {
    xs[i] = peaks[i].x;
    ys[i] = peaks[i].y;
    vals[i] = peaks[i].v;
  }
  return n;
}

// contour.hpp:28-55
void or_gaussian_blur(const double* in, int h, int w, double sigma, double* out) {
  const int R = std::max(1, int(std::ceil(3 * sigma)));
  std::vector<double> k(2 * R + 1);
  double ks = 0;
  for (int i = -R; i <= R; ++i) {
    k[i + R] = std::exp(-double(i * i) / (2 * sigma * sigma));
  }
  for (double v : k) ks += v;
  for (double& v : k) v /= ks;
  std::vector<double> tmp(size_t(h) * w, 0.0);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0;
      for (int i = -R; i <= R; ++i) {
        const int xi = x + i;
        if (xi >= 0 && xi < w) acc += k[i + R] * in[size_t(y) * w + xi];
      }
      tmp[size_t(y) * w + x] = acc;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0;
      for (int i = -R; i <= R; ++i) {
        const int yi = y + i;
        if (yi >= 0 && yi < h) acc += k[i + R] * tmp[size_t(yi) * w + x];
      }
      out[size_t(y) * w + x] = acc;
    }
}

// field.hpp:202-237
void or_gradient(const double* I, int h, int w, double* mag, double* dir) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      auto at = [&](int yy, int xx) { return I[size_t(yy) * w + xx]; };
      double gx, gy;
      if (w == 1) gx = 0;
      else if (x == 0) gx = at(y, 1) - at(y, 0);
      else if (x == w - 1) gx = at(y, w - 1) - at(y, w - 2);
      else gx = (at(y, x + 1) - at(y, x - 1)) / 2.0;
      if (h == 1) gy = 0;
      else if (y == 0) gy = at(1, x) - at(0, x);
      else if (y == h - 1) gy = at(h - 1, x) - at(h - 2, x);
      else gy = (at(y + 1, x) - at(y - 1, x)) / 2.0;
      const double m = std::sqrt(gx * gx + gy * gy);
      mag[size_t(y) * w + x] = m;
      dir[size_t(y) * w + x] = m > 0.0 ? std::atan2(gy, gx) : 0.0;
    }
}

// vote_filter.hpp:27-40 (bilinear splat), 45-60 (splat_vote), 62-81
// (build_vote_filter); row-major [y][x] grids, radius R = ceil(eps)
static void vote_splat_bilinear(std::vector<double>& g, int side, double x, double y, double w) {
  const int x0 = int(std::floor(x)), y0 = int(std::floor(y));
  const double tx = x - x0, ty = y - y0;
  for (int dy = 0; dy < 2; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      const int xi = x0 + dx, yi = y0 + dy;
      if (xi < 0 || yi < 0 || xi >= side || yi >= side) continue;
      g[size_t(yi) * side + xi] += w * (dx ? tx : 1 - tx) * (dy ? ty : 1 - ty);
    }
}

int or_build_vote_filter(const double* weight, const double* frame, int h, int w, double px,
                         double py, double eps, int nearest, double* weights_out,
                         int* radius_out) {
  return guarded([&] {
    if (!(eps > 0.0)) throw InvalidArg("support radius must be > 0");
    const int R = int(std::ceil(eps)), side = 2 * R + 1;
    std::vector<double> g(size_t(side) * side, 0.0);
    bool any = false;
    for (int qy = 0; qy < h; ++qy)
      for (int qx = 0; qx < w; ++qx) {
        const double m = weight[size_t(qy) * w + qx];
        if (m <= 0.0) continue;
        const double dx = px - qx, dy = py - qy;
        if (dx * dx + dy * dy > eps * eps) continue;
        const double a = frame[size_t(qy) * w + qx];
        const double c = std::cos(-a), sn = std::sin(-a);
        const double vx = c * dx - sn * dy + R, vy = sn * dx + c * dy + R;
        if (nearest) {
          const int xi = int(std::lround(vx)), yi = int(std::lround(vy));
          if (xi >= 0 && yi >= 0 && xi < side && yi < side) g[size_t(yi) * side + xi] += m;
        } else {
          vote_splat_bilinear(g, side, vx, vy, m);
        }
        any = true;
      }
    if (!any) throw InvalidArg("degenerate pattern: no votes in support");
    std::copy(g.begin(), g.end(), weights_out);
    *radius_out = R;
  });
}

// vote_filter.hpp:83-91 (build_optimal_filter)
int or_build_optimal_filter(const double* pattern, int h, int w, double px, double py,
                            double eps, int nearest, double* weights_out, int* radius_out) {
  return guarded([&] {
    if (px < 0 || py < 0 || px >= w || py >= h)
      throw InvalidArg("center must lie inside the pattern");
    std::vector<double> mag(size_t(h) * w), dir(size_t(h) * w);
    or_gradient(pattern, h, w, mag.data(), dir.data());
    const int rc = or_build_vote_filter(mag.data(), dir.data(), h, w, px, py, eps, nearest,
                                        weights_out, radius_out);
    if (rc) throw InvalidArg(g_err);
  });
}

// vote_filter.hpp:146-168 (detect_pattern): gradient magnitude votes through
// the vote filter (decomposed with K bands), steered by the gradient
// direction; response = Re(xconv_fast); peaks within eps/2, 0.5 max
int or_detect_pattern(const double* image, int h, int w, const double* vote_weights,
                      int radius, double eps, int K, int n_radii, int n_angles,
                      double* response, int* xs, int* ys, double* vals, int max_peaks,
                      int* n_peaks, long long* ops_out) {
  return guarded([&] {
    if (K < 1) throw InvalidArg("K must be >= 1");
    std::vector<double> mag(size_t(h) * w), dir(size_t(h) * w);
    or_gradient(image, h, w, mag.data(), dir.data());
    const int R = radius, side = 2 * R + 1;
    if (n_radii == 0) n_radii = std::max(4, 2 * R);
    if (n_angles == 0) n_angles = std::max(16, 8 * ((R + 1) / 2) * 2);
    std::vector<cd> vf(size_t(side) * side);
    for (size_t i = 0; i < vf.size(); ++i) vf[i] = cd(vote_weights[i], 0.0);
    const Filter F = decompose_rotation2(vf.data(), side, side, double(R), double(R), K, n_radii,
                                         n_angles, double(R) + 0.5);
    const Xform T = make_xform(0, dir.data(), h, w);
    std::vector<cd> H(size_t(h) * w);
    for (size_t i = 0; i < H.size(); ++i) H[i] = cd(mag[i], 0.0);
    long long ops = 0;
    const auto out = xfast(1, H, h, w, T, F, nullptr, 0, false, &ops, nullptr, 1);
    for (size_t i = 0; i < out.size(); ++i) response[i] = out[i].real();
    *n_peaks = or_find_peaks(response, h, w, eps / 2, 0.5, xs, ys, vals, max_peaks);
    *ops_out = ops;
  });
}

// SURVEY 8(a) A9 / BASELINE config 3.  No reference function exists; the
// per-angle sum follows the gather steering e^{+ik alpha} of engine.hpp:313-316
// with alpha_s = -2 pi s / n_angles, i.e. sum_k e^{-i k 2 pi s/n} G_k(p)
// (the angle grid of contour.hpp:119-138 / PAPER.md:700-704).
void or_anglemax(const double* G, const int* ks, int nc, int h, int w, int n_angles,
                 double* score, int* argmax) {
  const size_t N = size_t(h) * w;
  std::vector<cd> tw(static_cast<size_t>(n_angles));
  for (int s = 0; s < n_angles; ++s) {
    const double a = -2.0 * kPi * s / n_angles;
    tw[s] = cd(std::cos(a), std::sin(a));
  }
  for (size_t p = 0; p < N; ++p) {
    double best = -1;
    int arg = 0;
    for (int s = 0; s < n_angles; ++s) {
      cd acc(0);
      for (int c = 0; c < nc; ++c) {
        const long long e = ((long long)ks[c] * s) % n_angles;
        const cd z = tw[(e + n_angles) % n_angles];
        acc += z * cd(G[2 * (size_t(c) * N + p)], G[2 * (size_t(c) * N + p) + 1]);
      }
      const double m = std::abs(acc);
      if (m > best) {
        best = m;
        arg = s;
      }
    }
    score[p] = best;
    argmax[p] = arg;
  }
}

// ---------------------------------------------------------------- full-size checks
// Helpers for the full-size parity tests (test infrastructure).  Each is the
// reference arithmetic above, split across threads where the reference loop
// is independent per band or per pixel.

// G_k = filter2_fft(H, F_k, correlate) for each selected band (the per-band
// term of xcorr_fast before steering, engine.hpp:301-311), threads over bands.
int or_band_responses(const double* Hd, int h, int w, const or_filter* Fc, const int* ks,
                      int nk, int nthreads, double* Gout) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const int R = int(std::ceil(F.r_max));
    const size_t N = size_t(h) * w;
    auto H = to_cd(Hd, N);
    nthreads = std::max(1, std::min(nthreads, nk));
    auto run = [&](int tid) {
      for (int bi = tid; bi < nk; bi += nthreads) {
        auto Fk = render_component(F, F.index_of(ks[bi]), 2 * R + 1, 2 * R + 1, double(R),
                                   double(R));
        auto Gk = filter2_fft(H.data(), h, w, Fk.data(), 2 * R + 1, 2 * R + 1, R, R, true,
                              false);
        std::memcpy(Gout + 2 * N * size_t(bi), Gk.data(), N * sizeof(cd));
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(run, t);
    for (auto& t : th) t.join();
  });
}

// or_anglemax with rows split across threads and the e^{-i k 2 pi s / n}
// factors tabulated per (s, band); same max / first-argmax rule.
void or_anglemax_mt(const double* G, const int* ks, int nc, int h, int w, int n_angles,
                    int nthreads, double* score, int* argmax) {
  const size_t N = size_t(h) * w;
  std::vector<cd> tab(size_t(n_angles) * nc);
  for (int s = 0; s < n_angles; ++s)
    for (int c = 0; c < nc; ++c) {
      const long long e = (((long long)ks[c] * s) % n_angles + n_angles) % n_angles;
      const double a = -2.0 * kPi * double(e) / n_angles;
      tab[size_t(s) * nc + c] = cd(std::cos(a), std::sin(a));
    }
  nthreads = std::max(1, std::min(nthreads, h));
  auto run = [&](int tid) {
    std::vector<cd> g(nc);
    for (int y = tid; y < h; y += nthreads)
      for (int x = 0; x < w; ++x) {
        const size_t p = size_t(y) * w + x;
        for (int c = 0; c < nc; ++c)
          g[c] = cd(G[2 * (size_t(c) * N + p)], G[2 * (size_t(c) * N + p) + 1]);
        double best = -1;
        int arg = 0;
        for (int s = 0; s < n_angles; ++s) {
          const cd* t = tab.data() + size_t(s) * nc;
          double re = 0, im = 0;
          for (int c = 0; c < nc; ++c) {
            re += t[c].real() * g[c].real() - t[c].imag() * g[c].imag();
            im += t[c].real() * g[c].imag() + t[c].imag() * g[c].real();
          }
          const double m = std::sqrt(re * re + im * im);
          if (m > best) {
            best = m;
            arg = s;
          }
        }
        score[p] = best;
        argmax[p] = arg;
      }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) th.emplace_back(run, t);
  for (auto& t : th) t.join();
}

// xcorr_fast / xconv_fast evaluated directly (no FFT) at selected pixels:
// the bands are rendered once (render_component, freq_filter.hpp:173-184) and
// the zero-padded linear filtering of fft.hpp:74-77 is summed tap by tap,
// then steered as engine.hpp:312-317 / 353-366 (+ the inner-DC term).
int or_direct_at(int mode, const double* Hd, int h, int w, int kind, const double* param,
                 const or_filter* Fc, const int* pys, const int* pxs, int npix, int nthreads,
                 double* outd) {
  return guarded([&] {
    const Filter F = to_filter(Fc);
    const Xform T = make_xform(kind, param, h, w);
    const int R = int(std::ceil(F.r_max)), S = 2 * R + 1;
    const int nb = F.nc();
    std::vector<std::vector<cd>> Fk(nb);
    for (int ci = 0; ci < nb; ++ci)
      Fk[ci] = render_component(F, ci, S, S, double(R), double(R));
    const cd dc = inner_dc_value(F);
    auto phase = [&](int ci, size_t i) {
      return T.kind == 0 ? double(F.ks[ci]) * T.angle[i]
                         : double(F.ks[ci]) * F.omega() * T.log_scale[i];
    };
    auto Hat = [&](int x, int y) {
      return cd(Hd[2 * (size_t(y) * w + x)], Hd[2 * (size_t(y) * w + x) + 1]);
    };
    nthreads = std::max(1, std::min(nthreads, npix));
    auto run = [&](int tid) {
      for (int t = tid; t < npix; t += nthreads) {
        const int py = pys[t], px = pxs[t];
        cd acc(0);
        for (int ci = 0; ci < nb; ++ci) {
          cd band(0);
          for (int dy = -R; dy <= R; ++dy)
            for (int dx = -R; dx <= R; ++dx) {
              const cd fv = Fk[ci][size_t(dy + R) * S + (dx + R)];
              if (mode == 0) {  // out(p) = sum_u conj(F(u)) H(p+u)
                const int qx = px + dx, qy = py + dy;
                if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                band += std::conj(fv) * Hat(qx, qy);
              } else {  // out(p) = sum_u F(u) (H e^{-i phi})(p-u)
                const int qx = px - dx, qy = py - dy;
                if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                const double a = phase(ci, size_t(qy) * w + qx);
                band += fv * Hat(qx, qy) * cd(std::cos(-a), std::sin(-a));
              }
            }
          if (mode == 0) {
            const double a = phase(ci, size_t(py) * w + px);
            acc += band * cd(std::cos(a), std::sin(a));
          } else {
            acc += band;
          }
        }
        if (T.kind == 1) acc += (mode == 0 ? std::conj(dc) : dc) * Hat(px, py);
        outd[2 * t] = acc.real();
        outd[2 * t + 1] = acc.imag();
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(run, t);
    for (auto& t : th) t.join();
  });
}

// ---------------------------------------------------------------- fixtures
// proj/tests/helpers.hpp; the argument-evaluation order of
// Cx<double>(u(rng), u(rng)) is the compiler's, as in the reference build.

void* or_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void or_rng_free(void* rng) { delete static_cast<std::mt19937_64*>(rng); }
uint64_t or_rng_next(void* rng) { return (*static_cast<std::mt19937_64*>(rng))(); }
double or_rng_uniform(void* rng, double a, double b) {
  std::uniform_real_distribution<double> u(a, b);
  return u(*static_cast<std::mt19937_64*>(rng));
}

// helpers.hpp:29-36
void or_random_field(void* rngp, int w, int h, int complex_valued, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rngp);
  std::uniform_real_distribution<double> u(-1, 1);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const cd v = complex_valued ? cd(u(rng), u(rng)) : cd(u(rng), 0);
      out[2 * (size_t(y) * w + x)] = v.real();
      out[2 * (size_t(y) * w + x) + 1] = v.imag();
    }
}

// helpers.hpp:38-64
void or_random_smooth_filter(void* rngp, int radius, int n_bumps, double envelope_frac,
                             double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rngp);
  std::uniform_real_distribution<double> u(-1, 1);
  const int S = 2 * radius + 1;
  struct Bump {
    double x, y, a, s;
  };
  std::vector<Bump> bumps;
  for (int i = 0; i < n_bumps; ++i)
    bumps.push_back({u(rng) * radius * 0.5, u(rng) * radius * 0.5, u(rng),
                     1.2 + 0.8 * std::abs(u(rng))});
  const double env = envelope_frac * radius;
  for (int y = -radius; y <= radius; ++y)
    for (int x = -radius; x <= radius; ++x) {
      double v = 0;
      for (const auto& b : bumps) {
        const double dx = x - b.x, dy = y - b.y;
        v += b.a * std::exp(-(dx * dx + dy * dy) / (2 * b.s * b.s));
      }
      v *= std::exp(-(double(x) * x + double(y) * y) / (2 * env * env));
      const size_t i = size_t(y + radius) * S + (x + radius);
      out[2 * i] = v;
      out[2 * i + 1] = 0;
    }
}

// test_engine_scale.cpp:9-28 (and acceptance.cpp:61-79 with 0.354, 0.044)
void or_annular_filter(void* rngp, int R, double r0_frac, double sr_frac, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rngp);
  std::uniform_real_distribution<double> u(-1, 1);
  const int S = 2 * R + 1;
  const double r0 = r0_frac * R, sr = sr_frac * R;
  const double a1 = u(rng), b1 = u(rng), a2 = 0.5 * u(rng);
  for (int y = -R; y <= R; ++y)
    for (int x = -R; x <= R; ++x) {
      const double r = std::hypot(double(x), double(y));
      const double th = std::atan2(double(y), double(x));
      const double radial = std::exp(-(r - r0) * (r - r0) / (2 * sr * sr));
      const double v = radial * (1.0 + 0.6 * (a1 * std::cos(th) + b1 * std::sin(th)) +
                                 0.4 * a2 * std::cos(2 * th));
      const size_t i = size_t(y + R) * S + (x + R);
      out[2 * i] = v;
      out[2 * i + 1] = 0;
    }
}

// helpers.hpp:110-116 (raw angles; normalization happens in make_xform)
void or_random_rotation_field(void* rngp, int w, int h, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rngp);
  std::uniform_real_distribution<double> u(-kPi, kPi);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) out[size_t(y) * w + x] = u(rng);
}

// helpers.hpp:118-125
void or_random_scale_field(void* rngp, int w, int h, double lo, double hi, double* out) {
  auto& rng = *static_cast<std::mt19937_64*>(rngp);
  std::uniform_real_distribution<double> u(std::log(lo), std::log(hi));
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) out[size_t(y) * w + x] = std::exp(u(rng));
}

}  // extern "C"

// 3D rotation pipeline
#include "xconv_oracle3d.inc"
