// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C entry layer over the REFERENCE implementation itself: the reference's
// headers (/root/reference/proj/include/xconv/*.hpp) are compiled unchanged
// against the Eigen-subset shim in oracle/ref_shim and wrapped here with
// plain pointers, so Python tests can run the reference's xcorr_fast /
// xconv_fast / smooth_adaptive / decompose_* / find_peaks / detect_pattern on
// the same inputs as the CPU restatement (oracle/xconv_oracle.cpp) and the
// GPU product.  Built by `make -C oracle ref` into oracle/_ref/ (git-ignored;
// it travels to the GPU box as a prebuilt library).  Nothing here is product
// code and the product never loads it.
//
// Grids are row-major [y][x] here (element (x, y) of the reference's
// column-major Field2::values(y, x)); complex data is interleaved (re, im).
// FreqFilter2 comps are column-major (n_rows x nc) like the reference's CGrid.
#include <xconv/engine.hpp>
#include <xconv/vote_filter.hpp>

#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace xconv;

namespace {

thread_local std::string g_err;

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
    return 13;
  }
}

Field2d field_c(const double* d, int h, int w) {
  Field2d f(w, h);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x)
      f.at(x, y) = Cx<double>(d[2 * (size_t(y) * w + x)], d[2 * (size_t(y) * w + x) + 1]);
  return f;
}

RGrid<double> grid_r(const double* d, int h, int w) {
  RGrid<double> g(h, w);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) g(y, x) = d[size_t(y) * w + x];
  return g;
}

void put_c(const CGrid<double>& g, double* out) {
  const int h = int(g.rows()), w = int(g.cols());
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      out[2 * (size_t(y) * w + x)] = g(y, x).real();
      out[2 * (size_t(y) * w + x) + 1] = g(y, x).imag();
    }
}

FreqFilter2d make_filter(int group, int K, const int* ks, int nc, const double* comps,
                         int n_radii, int n_angles, double r_max, double r_min, double r_domain) {
  FreqFilter2d f;
  f.group = group == 0 ? XformKind::rotation2 : XformKind::scale2;
  f.K = K;
  f.ks.assign(ks, ks + nc);
  f.n_radii = n_radii;
  f.n_angles = n_angles;
  f.r_max = r_max;
  f.r_min = r_min;
  f.r_domain = r_domain;
  const int rows = group == 0 ? n_radii : n_angles;
  f.comps.resize(rows, nc);
  for (int c = 0; c < nc; ++c)
    for (int r = 0; r < rows; ++r)
      f.comps(r, c) = Cx<double>(comps[2 * (size_t(c) * rows + r)],
                                 comps[2 * (size_t(c) * rows + r) + 1]);
  return f;
}

void export_filter(const FreqFilter2d& f, int* ks_out, double* comps_out, int* nc_out) {
  const int nc = f.n_components(), rows = int(f.comps.rows());
  for (int i = 0; i < nc; ++i) ks_out[i] = f.ks[i];
  for (int c = 0; c < nc; ++c)
    for (int r = 0; r < rows; ++r) {
      comps_out[2 * (size_t(c) * rows + r)] = f.comps(r, c).real();
      comps_out[2 * (size_t(c) * rows + r) + 1] = f.comps(r, c).imag();
    }
  *nc_out = nc;
}

XformFieldd make_xform(int kind, const double* param, int h, int w) {
  return kind == 0 ? XformFieldd::rotation(grid_r(param, h, w))
                   : XformFieldd::scaling(grid_r(param, h, w));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_next_fast_size(int n) { return next_fast_size(n); }

// fft.hpp:79-100
int ref_filter2_fft(const double* sig, int h, int w, const double* filt, int fh, int fw,
                    int fcx, int fcy, int correlate, int periodic, double* out) {
  return guarded([&] {
    auto S = field_c(sig, h, w), F = field_c(filt, fh, fw);
    put_c(filter2_fft(S.values, F.values, fcx, fcy, correlate != 0, periodic != 0), out);
  });
}

// fft.hpp:20-53 (Eigen FFT through the shim: kissfft order, inverse 1/n)
int ref_fft2(const double* a, int h, int w, int inverse, double* out) {
  return guarded([&] {
    auto A = field_c(a, h, w).values;
    fft2(A, inverse != 0);
    put_c(A, out);
  });
}

// freq_filter.hpp:63-89
int ref_decompose_rotation2(const double* filt, int h, int w, double cx, double cy, int K,
                            int n_radii, int n_angles, double r_max, int* ks_out,
                            double* comps_out, int* nc_out) {
  return guarded([&] {
    export_filter(decompose_rotation2(field_c(filt, h, w), cx, cy, K, n_radii, n_angles, r_max),
                  ks_out, comps_out, nc_out);
  });
}

// freq_filter.hpp:92-129
int ref_decompose_scale2(const double* filt, int h, int w, double cx, double cy, int K,
                         int n_radii, int n_angles, double r_min, double r_max, double r_domain,
                         int* ks_out, double* comps_out, int* nc_out) {
  return guarded([&] {
    export_filter(decompose_scale2(field_c(filt, h, w), cx, cy, K, n_radii, n_angles, r_min, r_max,
                                   r_domain),
                  ks_out, comps_out, nc_out);
  });
}

// freq_filter.hpp:173-184
int ref_render_component(int group, int K, const int* ks, int nc, const double* comps,
                         int n_radii, int n_angles, double r_max, double r_min, double r_domain,
                         int ci, int width, int height, double cx, double cy, double* out) {
  return guarded([&] {
    auto F = make_filter(group, K, ks, nc, comps, n_radii, n_angles, r_max, r_min, r_domain);
    put_c(render_component(F, ci, width, height, cx, cy).values, out);
  });
}

// xcorr_fast (engine.hpp:286-326) / xconv_fast (engine.hpp:331-373).  nthreads
// > 1 calls the reference on contiguous band subsets (XConvPlan::components)
// in parallel and sums the outputs in thread order (the scale inner-DC term,
// added by every call, is removed from all but the first).
int ref_xfast(int mode, const double* Hd, int h, int w, int kind, const double* param,
              int group, int K, const int* ks, int nc, const double* comps, int n_radii,
              int n_angles, double r_max, double r_min, double r_domain, const int* components,
              int ncomp, int periodic, int nthreads, double* out, long long* ops_out) {
  return guarded([&] {
    const Field2d H = field_c(Hd, h, w);
    const XformFieldd T = make_xform(kind, param, h, w);
    const FreqFilter2d F = make_filter(group, K, ks, nc, comps, n_radii, n_angles, r_max, r_min,
                                       r_domain);
    XConvPlan plan;
    plan.periodic = periodic != 0;
    if (components && ncomp > 0) plan.components.assign(components, components + ncomp);
    auto run = [&](const XConvPlan& p) {
      return mode == 0 ? xcorr_fast(H, T, F, p) : xconv_fast(H, T, F, p);
    };
    std::vector<int> all = plan.components.empty() ? F.ks : plan.components;
    const int nt = std::max(1, std::min(nthreads, int(all.size())));
    if (nt == 1) {
      auto r = run(plan);
      put_c(r.output.values, out);
      if (ops_out) *ops_out = r.standard_ops;
      return;
    }
    std::vector<Response2<double>> parts(static_cast<size_t>(nt));
    std::vector<std::string> errs(static_cast<size_t>(nt));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        try {
          XConvPlan p = plan;
          const size_t a = all.size() * size_t(t) / size_t(nt);
          const size_t b = all.size() * size_t(t + 1) / size_t(nt);
          p.components.assign(all.begin() + long(a), all.begin() + long(b));
          parts[size_t(t)] = run(p);
        } catch (const std::exception& e) {
          errs[size_t(t)] = e.what();
        }
      });
    for (auto& x : th) x.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
    CGrid<double> acc = parts[0].output.values;
    long long ops = parts[0].standard_ops;
    const Cx<double> dc = inner_dc_value(F);
    for (int t = 1; t < nt; ++t) {
      acc += parts[size_t(t)].output.values;
      ops += parts[size_t(t)].standard_ops;
      if (kind == 1) acc -= (mode == 0 ? std::conj(dc) : dc) * H.values;
    }
    put_c(acc, out);
    if (ops_out) *ops_out = ops;
  });
}

// smooth_adaptive (engine.hpp:385-419); H real [h][w]
int ref_smooth_adaptive(const double* Hr, int h, int w, int kind, const double* param, int group,
                        int K, const int* ks, int nc, const double* comps, int n_radii,
                        int n_angles, double r_max, double r_min, double r_domain, int normalize,
                        double* out, long long* ops_out, int* clamped_out) {
  return guarded([&] {
    Field2d H(w, h);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) H.at(x, y) = Hr[size_t(y) * w + x];
    const XformFieldd T = make_xform(kind, param, h, w);
    const FreqFilter2d F = make_filter(group, K, ks, nc, comps, n_radii, n_angles, r_max, r_min,
                                       r_domain);
    auto r = smooth_adaptive(H, T, F, normalize != 0);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) out[size_t(y) * w + x] = r.output.at(x, y).real();
    *ops_out = r.standard_ops;
    *clamped_out = r.clamped_pixels;
  });
}

// find_peaks (vote_filter.hpp:107-134); returns the number found
int ref_find_peaks(const double* resp, int h, int w, double radius, double threshold_frac,
                   int* xs, int* ys, double* vals, int max_out) {
  const auto pk = find_peaks<double>(grid_r(resp, h, w), radius, threshold_frac);
  for (int i = 0; i < int(pk.size()) && i < max_out; ++i) {
    xs[i] = pk[size_t(i)].x;
    ys[i] = pk[size_t(i)].y;
    vals[i] = pk[size_t(i)].value;
  }
  return int(pk.size());
}

// build_optimal_filter (vote_filter.hpp:83-91) + detect_pattern (146-168):
// real pattern / image [h][w]; response [h][w]; peaks (x, y, value)
int ref_detect_pattern(const double* pattern, int ph, int pw, double px, double py, double eps,
                       const double* image, int h, int w, int K, double* response, int* xs,
                       int* ys, double* vals, int max_out, int* n_found, long long* ops_out) {
  return guarded([&] {
    Field2d P(pw, ph), I(w, h);
    for (int y = 0; y < ph; ++y)
      for (int x = 0; x < pw; ++x) P.at(x, y) = pattern[size_t(y) * pw + x];
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) I.at(x, y) = image[size_t(y) * w + x];
    const auto vf = build_optimal_filter(P, px, py, eps);
    const auto det = detect_pattern(I, vf, K);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) response[size_t(y) * w + x] = det.response.at(x, y).real();
    for (int i = 0; i < int(det.peaks.size()) && i < max_out; ++i) {
      xs[i] = det.peaks[size_t(i)].x;
      ys[i] = det.peaks[size_t(i)].y;
      vals[i] = det.peaks[size_t(i)].value;
    }
    *n_found = int(det.peaks.size());
    *ops_out = det.standard_ops;
  });
}

}  // extern "C"
