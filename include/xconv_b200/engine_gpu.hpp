// engine_gpu.hpp -- C++ host-side drop-in for the reference's 2D fast paths.
//
// Header-only, templated over the reference's own types (Field2<Real>,
// XformField<Real>, FreqFilter2<Real>, XConvPlan, Response2<Real>,
// SmoothResult<Real> from proj/include/xconv/{field,freq_filter,engine}.hpp),
// so the reference keeps its signatures and replaces its per-band CPU loop by
// the C ABI of include/xconv_b200.h:
//
//   xconv::gpu::xcorr_fast(H, T, F, plan)        <- engine.hpp:286-326
//   xconv::gpu::xconv_fast(H, T, F, plan)        <- engine.hpp:331-373
//   xconv::gpu::smooth_adaptive(H, T, F, norm)   <- engine.hpp:385-419
//   xconv::gpu::build_optimal_filter(P, px, py, eps, nearest)
//                                                <- vote_filter.hpp:83-91
//   xconv::gpu::detect_pattern(I, vf, K, n_radii, n_angles)
//                                                <- vote_filter.hpp:146-168
//   xconv::gpu::xcorr_fast_3d / xconv_fast_3d(H, T, F, plan)
//                                                <- engine3d.hpp:270-335
//
// Eigen's default column-major storage (field.hpp:15) is passed as
// XC_COL_MAJOR with the caller's complex<double> / double buffers
// (XC_C128 / XC_F64); std::invalid_argument is rethrown with the reference's
// message for XC_EINVAL, std::runtime_error otherwise.  The device-side filter
// spectra are cached per filter content (exact key, 4-entry LRU), per thread.
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../xconv_b200.h"

namespace xconv {
namespace gpu {

namespace detail {

inline void check(int rc, xc_context ctx) {
  if (rc == XC_OK) return;
  const std::string msg = xc_last_error(ctx);
  if (rc == XC_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("xconv_b200: " + msg);
}

// Decomposed filters uploaded to the library, keyed by their full content
// (group, K, n_radii, n_angles, radii, ks, coefficients) and compared byte for
// byte on a hit.  Each handle keeps its device spectra (nb * Ph * Pw * 8 bytes,
// ~9.7 GB for BASELINE config 5) alive, so the cache is a small LRU.
struct FilterCache {
  static constexpr size_t kCapacity = 4;
  struct Entry {
    std::vector<unsigned char> key;
    xc_filter handle;
  };
  std::vector<Entry> entries;  // most recently used last
  ~FilterCache() {
    for (auto& e : entries) xc_filter_destroy(e.handle);
  }
  xc_filter find(const std::vector<unsigned char>& key) {
    for (size_t i = 0; i < entries.size(); ++i)
      if (entries[i].key == key) {
        Entry e = std::move(entries[i]);
        entries.erase(entries.begin() + long(i));
        entries.push_back(std::move(e));
        return entries.back().handle;
      }
    return nullptr;
  }
  void insert(std::vector<unsigned char> key, xc_filter h) {
    if (entries.size() >= kCapacity) {
      xc_filter_destroy(entries.front().handle);
      entries.erase(entries.begin());
    }
    entries.push_back(Entry{std::move(key), h});
  }
};

// One library context per host thread (contexts are not shared across
// threads, include/xconv_b200.h).  The devices it runs on come from
// XCB_DEVICES ("0,1,2,3"; default: device 0); with several devices xc_run
// shards the bands (gather/scatter) over them and reduces with NCCL.
inline std::vector<int> env_devices() {
  std::vector<int> ids;
  if (const char* e = std::getenv("XCB_DEVICES")) {
    std::string s(e);
    size_t pos = 0;
    while (pos < s.size()) {
      size_t end = s.find(',', pos);
      if (end == std::string::npos) end = s.size();
      if (end > pos) ids.push_back(std::atoi(s.substr(pos, end - pos).c_str()));
      pos = end + 1;
    }
  }
  if (ids.empty()) ids.push_back(0);
  return ids;
}

struct Context {
  xc_context ctx = nullptr;
  FilterCache filters;
  Context() {
    const std::vector<int> ids = env_devices();
    if (ids.size() == 1)
      check(xc_context_create(ids[0], &ctx), nullptr);
    else
      check(xc_context_create_multi(int(ids.size()), ids.data(), &ctx), nullptr);
  }
  ~Context() {
    for (auto& e : filters.entries) xc_filter_destroy(e.handle);  // before the context
    filters.entries.clear();
    xc_context_destroy(ctx);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
};

inline Context& context() {
  thread_local Context c;
  return c;
}

inline void append(std::vector<unsigned char>& k, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  k.insert(k.end(), b, b + n);
}

// FreqFilter2<Real> -> xc_filter (cached by content)
template <class F>
xc_filter filter_handle(const F& f) {
  Context& c = context();
  const int nc = static_cast<int>(f.ks.size());
  const int rows = static_cast<int>(f.comps.rows());
  std::vector<double> comps(size_t(2) * nc * rows);
  for (int ci = 0; ci < nc; ++ci)
    for (int r = 0; r < rows; ++r) {  // Eigen column-major (row + ci * n_rows)
      comps[2 * (size_t(ci) * rows + r)] = double(std::real(f.comps(r, ci)));
      comps[2 * (size_t(ci) * rows + r) + 1] = double(std::imag(f.comps(r, ci)));
    }
  const int group = static_cast<int>(f.group);
  const double sc[3] = {double(f.r_max), double(f.r_min), double(f.r_domain)};
  const int ints[5] = {group, f.K, f.n_radii, f.n_angles, nc};
  std::vector<unsigned char> key;
  key.reserve(sizeof(ints) + sizeof(sc) + f.ks.size() * sizeof(int) + comps.size() * 8);
  append(key, ints, sizeof(ints));
  append(key, sc, sizeof(sc));
  append(key, f.ks.data(), f.ks.size() * sizeof(int));
  append(key, comps.data(), comps.size() * sizeof(double));
  if (xc_filter hit = c.filters.find(key)) return hit;
  xc_filter out = nullptr;
  check(xc_filter_create(c.ctx, group, f.K, f.ks.data(), nc, comps.data(), f.n_radii,
                         f.n_angles, sc[0], sc[1], sc[2], &out),
        nullptr);
  c.filters.insert(std::move(key), out);
  return out;
}

template <class Real>
constexpr int signal_dtype() {
  return sizeof(Real) == 8 ? XC_C128 : XC_C64;
}
template <class Real>
constexpr int real_dtype() {
  return sizeof(Real) == 8 ? XC_F64 : XC_F32;
}

// engine.hpp:288-291 checks (the ABI repeats them; these keep the order of
// the reference's messages for the fields only the host sees)
template <class Field, class Xform, class F>
void validate(const Field& H, const Xform& T, const F& Fl) {
  if (static_cast<int>(T.kind) != static_cast<int>(Fl.group))
    throw std::invalid_argument("transformation/filter group mismatch");
  if (static_cast<int>(T.kind) == XC_ROTATION3)
    throw std::invalid_argument("2D pipeline needs a 2D field");
  if (H.width() != T.width() || H.height() != T.height())
    throw std::invalid_argument("signal and transformation field dims differ");
}

template <class Response, class Field, class Xform, class F, class Plan>
Response run(int mode, const Field& H, const Xform& T, const F& Fl, Plan plan) {
  using Real = typename std::remove_cv<typename std::remove_reference<
      decltype(std::real(H.values(0, 0)))>::type>::type;
  validate(H, T, Fl);
  Context& c = context();
  xc_filter fh = filter_handle(Fl);
  const bool scale = static_cast<int>(T.kind) == XC_SCALE2;
  xc_image_desc d{};
  d.height = H.height();
  d.width = H.width();
  d.batch = 1;
  d.signal_dtype = signal_dtype<Real>();
  d.param_dtype = real_dtype<Real>();
  d.out_dtype = signal_dtype<Real>();
  d.layout = XC_COL_MAJOR;
  d.memory = XC_HOST;
  d.param_per_image = 1;
  d.xform_kind = static_cast<int>(T.kind);
  Response r;
  plan.mode = decltype(plan.mode)(mode);
  plan.group = T.kind;
  r.plan = plan;
  r.output = Field(H.width(), H.height());
  const void* param = scale ? static_cast<const void*>(T.scale.data())
                            : static_cast<const void*>(T.angle.data());
  std::vector<int> comps(plan.components.begin(), plan.components.end());
  xc_stats st{};
  check(xc_run(c.ctx, fh, mode, &d, H.values.data(), param, comps.empty() ? nullptr : comps.data(),
               static_cast<int>(comps.size()), plan.periodic ? XC_FLAG_PERIODIC : 0u,
               r.output.values.data(), &st),
        c.ctx);
  r.standard_ops = st.standard_ops;
  r.seconds["render"] = st.seconds_render;
  r.seconds["fft"] = st.seconds_fft;
  r.seconds["combine"] = st.seconds_combine;
  if (mode == XC_CONVOLUTION) r.seconds["premultiply"] = st.seconds_premultiply;
  return r;
}

}  // namespace detail

// engine.hpp:286-287
template <class Response, class Field, class Xform, class F, class Plan>
Response xcorr_fast(const Field& H, const Xform& T, const F& Fl, Plan plan) {
  return detail::run<Response>(XC_CORRELATION, H, T, Fl, plan);
}

// engine.hpp:331-332
template <class Response, class Field, class Xform, class F, class Plan>
Response xconv_fast(const Field& H, const Xform& T, const F& Fl, Plan plan) {
  return detail::run<Response>(XC_CONVOLUTION, H, T, Fl, plan);
}

// engine.hpp:385-387 (SmoothResult: output, standard_ops, clamped_pixels)
template <class Result, class Field, class Xform, class F>
Result smooth_adaptive(const Field& H, const Xform& T, const F& Fl, bool normalize_signal = true) {
  using Real = typename std::remove_cv<typename std::remove_reference<
      decltype(std::real(H.values(0, 0)))>::type>::type;
  detail::Context& c = detail::context();
  xc_filter fh = detail::filter_handle(Fl);
  if (H.width() != T.width() || H.height() != T.height())
    throw std::invalid_argument("signal and transformation field dims differ");
  const bool scale = static_cast<int>(T.kind) == XC_SCALE2;
  xc_image_desc d{};
  d.height = H.height();
  d.width = H.width();
  d.batch = 1;
  d.signal_dtype = detail::signal_dtype<Real>();
  d.param_dtype = detail::real_dtype<Real>();
  d.out_dtype = detail::real_dtype<Real>();
  d.layout = XC_COL_MAJOR;
  d.memory = XC_HOST;
  d.param_per_image = 1;
  d.xform_kind = static_cast<int>(T.kind);
  std::vector<Real> real_out(size_t(H.width()) * H.height());
  const void* param = scale ? static_cast<const void*>(T.scale.data())
                            : static_cast<const void*>(T.angle.data());
  xc_stats st{};
  detail::check(xc_smooth(c.ctx, fh, &d, H.values.data(), param, normalize_signal ? 1 : 0,
                          real_out.data(), &st),
                c.ctx);
  Result out;
  out.standard_ops = st.standard_ops;
  out.clamped_pixels = st.clamped_pixels;
  out.output = decltype(out.output)(H.width(), H.height());
  for (size_t i = 0; i < real_out.size(); ++i) out.output.values.data()[i] = real_out[i];
  return out;
}

// vote_filter.hpp:83-91 (VoteFilter<Real>: weights (2R+1)^2 column-major,
// radius, eps); the pattern must be real-valued (field.hpp:206)
template <class VF, class Field, class Real>
VF build_optimal_filter(const Field& pattern, Real px, Real py, Real eps, bool nearest = false) {
  const int h = pattern.height(), w = pattern.width();
  std::vector<double> p(size_t(h) * w);
  for (size_t i = 0; i < p.size(); ++i) {
    if (std::imag(pattern.values.data()[i]) != 0)
      throw std::invalid_argument("gradient requires real field");
    p[i] = double(std::real(pattern.values.data()[i]));
  }
  const int R = eps > 0 ? static_cast<int>(std::ceil(double(eps))) : 0;
  std::vector<double> wts(size_t(2 * R + 1) * (2 * R + 1));
  int radius = 0;
  detail::check(xc_build_optimal_filter(p.data(), h, w, XC_COL_MAJOR, double(px), double(py),
                                        double(eps), nearest ? 1 : 0, wts.data(), &radius),
                nullptr);
  VF f;
  f.eps = eps;
  f.radius = radius;
  f.weights = decltype(f.weights)(2 * radius + 1, 2 * radius + 1);
  for (size_t i = 0; i < wts.size(); ++i) f.weights.data()[i] = wts[i];
  return f;
}

// vote_filter.hpp:146-168 (DetectionResult<Real>: response Field2, peaks
// {x, y, value} sorted by value desc / y / x, standard_ops)
template <class Result, class Field, class VF>
Result detect_pattern(const Field& image, const VF& filter, int K, int n_radii = 0,
                      int n_angles = 0) {
  detail::Context& c = detail::context();
  const int h = image.height(), w = image.width();
  std::vector<double> img(size_t(h) * w);
  for (size_t i = 0; i < img.size(); ++i) {
    if (std::imag(image.values.data()[i]) != 0)
      throw std::invalid_argument("gradient requires real field");
    img[i] = double(std::real(image.values.data()[i]));
  }
  const int side = 2 * filter.radius + 1;
  std::vector<double> wts(size_t(side) * side);
  for (size_t i = 0; i < wts.size(); ++i) wts[i] = double(filter.weights.data()[i]);
  xc_image_desc d{};
  d.height = h;
  d.width = w;
  d.batch = 1;
  d.signal_dtype = XC_F64;
  d.param_dtype = XC_F64;
  d.out_dtype = XC_F64;
  d.layout = XC_COL_MAJOR;
  d.memory = XC_HOST;
  d.param_per_image = 1;
  d.xform_kind = XC_ROTATION2;
  std::vector<double> resp(img.size());
  const int max_peaks = static_cast<int>(img.size());
  std::vector<int> px(max_peaks), py(max_peaks);
  std::vector<double> pv(max_peaks);
  int n = 0;
  xc_stats st{};
  detail::check(xc_detect_pattern(c.ctx, &d, img.data(), wts.data(), filter.radius,
                                  double(filter.eps), K, n_radii, n_angles, resp.data(),
                                  px.data(), py.data(), pv.data(), max_peaks, &n, &st),
                c.ctx);
  Result out;
  out.standard_ops = st.standard_ops;
  out.response = decltype(out.response)(w, h);
  for (size_t i = 0; i < resp.size(); ++i) out.response.values.data()[i] = resp[i];
  for (int i = 0; i < n && i < max_peaks; ++i) {
    typename decltype(out.peaks)::value_type pk;
    pk.x = px[i];
    pk.y = py[i];
    pk.value = pv[i];
    out.peaks.push_back(pk);
  }
  return out;
}

// engine3d.hpp:270-335 (Field3<Real>: nx, ny, nz, values x fastest;
// XformField<Real>: kind, nx, ny, nz, quats with w() x() y() z();
// SphFilter3<Real>: K, n_radii, r_max, coeffs (n_radii x (K+1)^2, Eigen
// column-major); Response3<Real>: output, plan, standard_ops, seconds)
namespace detail {

template <class Result, class Field3T, class Xform, class SphF, class Plan>
Result run3(int mode, const Field3T& H, const Xform& T, const SphF& F, Plan plan) {
  if (T.nx != H.nx || T.ny != H.ny || T.nz != H.nz)  // engine3d.hpp:274-275
    throw std::invalid_argument("signal and transformation field dims differ");
  Context& c = context();
  const size_t n = H.values.size();
  std::vector<double> sig(2 * n), q(4 * n), out(2 * n);
  for (size_t i = 0; i < n; ++i) {
    sig[2 * i] = double(std::real(H.values[i]));
    sig[2 * i + 1] = double(std::imag(H.values[i]));
    const auto& qq = T.quats[i];
    q[4 * i] = double(qq.w());
    q[4 * i + 1] = double(qq.x());
    q[4 * i + 2] = double(qq.y());
    q[4 * i + 3] = double(qq.z());
  }
  const int rows = static_cast<int>(F.coeffs.rows()), cols = static_cast<int>(F.coeffs.cols());
  std::vector<double> co(size_t(2) * rows * cols);
  for (int cc = 0; cc < cols; ++cc)
    for (int r = 0; r < rows; ++r) {
      co[2 * (size_t(cc) * rows + r)] = double(std::real(F.coeffs(r, cc)));
      co[2 * (size_t(cc) * rows + r) + 1] = double(std::imag(F.coeffs(r, cc)));
    }
  xc_filter3 f = nullptr;
  check(xc_filter3_create(F.K, F.n_radii, double(F.r_max), co.data(), &f), nullptr);
  std::unique_ptr<xc_filter3_s, void (*)(xc_filter3)> guard(f, xc_filter3_destroy);
  std::vector<int> deg(plan.components.begin(), plan.components.end());
  xc_stats st{};
  check(xc_run3(c.ctx, f, mode, H.nx, H.ny, H.nz, sig.data(), XC_C128, q.data(),
                deg.empty() ? nullptr : deg.data(), int(deg.size()), XC_HOST, out.data(), &st),
        c.ctx);
  Result res;
  res.plan = plan;
  res.standard_ops = st.standard_ops;
  res.seconds["fft"] = st.seconds_fft;
  res.seconds["total"] = st.seconds_total;
  res.output = decltype(res.output)(H.nx, H.ny, H.nz);
  for (size_t i = 0; i < n; ++i)
    res.output.values[i] = typename decltype(res.output.values)::value_type(out[2 * i],
                                                                           out[2 * i + 1]);
  return res;
}

}  // namespace detail

template <class Result, class Field3T, class Xform, class SphF, class Plan>
Result xcorr_fast_3d(const Field3T& H, const Xform& T, const SphF& F, Plan plan) {
  plan.mode = decltype(plan.mode)(0);
  return detail::run3<Result>(XC_CORRELATION, H, T, F, plan);
}

template <class Result, class Field3T, class Xform, class SphF, class Plan>
Result xconv_fast_3d(const Field3T& H, const Xform& T, const SphF& F, Plan plan) {
  plan.mode = decltype(plan.mode)(1);
  return detail::run3<Result>(XC_CONVOLUTION, H, T, F, plan);
}

}  // namespace gpu
}  // namespace xconv
