// The C++ drop-in path end to end: reference-shaped types -> engine_gpu.hpp ->
// C ABI -> sm_100a kernels, checked against the CPU oracle (test
// infrastructure).  Exit 0 iff every case is within 1e-5 relative L2.
#include <cmath>
#include <cstdio>
#include <random>

#include "../../include/xconv_b200/engine_gpu.hpp"
#include "../../oracle/xconv_oracle.h"
#include "mini_xconv.hpp"

using namespace mini;
using cd = std::complex<double>;

static double rel(const std::vector<cd>& a, const std::vector<cd>& b) {
  double n = 0, d = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    n += std::norm(a[i] - b[i]);
    d += std::norm(b[i]);
  }
  return std::sqrt(n / d);
}

int main() {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1, 1);
  const int h = 37, w = 53, R = 6;
  // filter: decompose a random smooth image with the product's host ABI
  std::vector<double> filt(2 * (2 * R + 1) * (2 * R + 1));
  for (size_t i = 0; i < filt.size(); i += 2) filt[i] = u(rng);
  const int K = 16, nr = 12, na = 34;
  std::vector<int> ks(K + 1);
  std::vector<double> comps(2 * size_t(nr) * (K + 1));
  int nc = 0;
  if (xc_decompose_rotation2(filt.data(), 2 * R + 1, 2 * R + 1, XC_ROW_MAJOR, R, R, K, nr, na,
                             double(R), ks.data(), comps.data(), &nc) != XC_OK)
    return 2;
  FreqFilter2<double> F;
  F.group = XformKind::rotation2;
  F.K = K;
  F.ks = ks;
  F.comps = Grid<std::complex<double>>(nr, nc);
  for (int ci = 0; ci < nc; ++ci)
    for (int r = 0; r < nr; ++r)
      F.comps(r, ci) = cd(comps[2 * (size_t(ci) * nr + r)], comps[2 * (size_t(ci) * nr + r) + 1]);
  F.n_radii = nr;
  F.n_angles = na;
  F.r_max = R;
  // signal / angles, column-major like Eigen
  Field2<double> H(w, h);
  XformField<double> T;
  T.kind = XformKind::rotation2;
  T.angle = Grid<double>(h, w);
  for (int x = 0; x < w; ++x)
    for (int y = 0; y < h; ++y) {
      H.values(y, x) = cd(u(rng), u(rng));
      T.angle(y, x) = 3.14159 * u(rng);
    }
  // oracle inputs (row-major)
  std::vector<double> Ho(2 * size_t(h) * w), To(size_t(h) * w), rowc(2 * size_t(nr) * nc);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      Ho[2 * (size_t(y) * w + x)] = H.values(y, x).real();
      Ho[2 * (size_t(y) * w + x) + 1] = H.values(y, x).imag();
      To[size_t(y) * w + x] = T.angle(y, x);
    }
  for (int r = 0; r < nr; ++r)
    for (int ci = 0; ci < nc; ++ci) {
      rowc[2 * (size_t(r) * nc + ci)] = F.comps(r, ci).real();
      rowc[2 * (size_t(r) * nc + ci) + 1] = F.comps(r, ci).imag();
    }
  or_filter of{0, K, nc, ks.data(), rowc.data(), nr, na, double(R), 0, 0};
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int periodic = 0; periodic < 2; ++periodic) {
      XConvPlan plan;
      plan.periodic = periodic != 0;
      Response2<double> r =
          mode == 0 ? xconv::gpu::xcorr_fast<Response2<double>>(H, T, F, plan)
                    : xconv::gpu::xconv_fast<Response2<double>>(H, T, F, plan);
      std::vector<double> ref(2 * size_t(h) * w);
      long long ops = 0;
      if (or_xfast(mode, Ho.data(), h, w, 0, To.data(), &of, nullptr, 0, periodic, ref.data(),
                   &ops, nullptr, 1) != 0)
        return 3;
      std::vector<cd> a(size_t(h) * w), b(size_t(h) * w);
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          a[size_t(y) * w + x] = r.output.values(y, x);
          b[size_t(y) * w + x] = cd(ref[2 * (size_t(y) * w + x)], ref[2 * (size_t(y) * w + x) + 1]);
        }
      const double e = rel(a, b);
      const bool ok = e < 1e-5 && r.standard_ops == ops && r.standard_ops == nc &&
                      r.plan.mode == (mode ? XMode::convolution : XMode::correlation);
      std::printf("mode %d periodic %d: rel_l2 %.3e ops %lld %s\n", mode, periodic, e,
                  r.standard_ops, ok ? "ok" : "FAIL");
      fails += !ok;
    }
  // error behaviour: the reference's std::invalid_argument text
  try {
    XConvPlan plan;
    plan.components = {99};
    xconv::gpu::xcorr_fast<Response2<double>>(H, T, F, plan);
    ++fails;
  } catch (const std::invalid_argument& e) {
    const bool ok = std::string(e.what()) == "plan retains a component the filter lacks";
    std::printf("invalid plan: \"%s\" %s\n", e.what(), ok ? "ok" : "FAIL");
    fails += !ok;
  }
  // detect_pattern through the shim (vote_filter.hpp:146-168) vs the oracle
  {
    const int Rp = 6, n = 48;
    Field2<double> pat(2 * Rp + 1, 2 * Rp + 1);
    for (int y = -Rp; y <= Rp; ++y)
      for (int x = -Rp; x <= Rp; ++x)
        pat.values(y + Rp, x + Rp) =
            std::exp(-((x + 1.5) * (x + 1.5) + (y - 0.5) * (y - 0.5)) / 4.0) -
            0.7 * std::exp(-((x - 2.0) * (x - 2.0) + (y + 2.0) * (y + 2.0)) / 3.0);
    auto vf = xconv::gpu::build_optimal_filter<VoteFilter<double>>(pat, 6.0, 6.0, 6.0);
    Field2<double> img(n, n);
    for (int y = 0; y < 2 * Rp + 1; ++y)
      for (int x = 0; x < 2 * Rp + 1; ++x) {
        img.values(y + 10, x + 14) += pat.values(y, x);
        img.values(x + 27, 2 * Rp - y + 20) += 0.8 * pat.values(y, x);  // weaker 90-degree copy
      }
    auto det = xconv::gpu::detect_pattern<DetectionResult<double>>(img, vf, 12);
    std::vector<double> imo(size_t(n) * n), wo(size_t(2 * Rp + 1) * (2 * Rp + 1));
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x) imo[size_t(y) * n + x] = img.values(y, x).real();
    for (int y = 0; y < 2 * Rp + 1; ++y)
      for (int x = 0; x < 2 * Rp + 1; ++x) wo[size_t(y) * (2 * Rp + 1) + x] = vf.weights(y, x);
    std::vector<double> resp(size_t(n) * n), pvv(64);
    std::vector<int> pxx(64), pyy(64);
    int np = 0;
    long long ops = 0;
    if (or_detect_pattern(imo.data(), n, n, wo.data(), vf.radius, vf.eps, 12, 0, 0, resp.data(),
                          pxx.data(), pyy.data(), pvv.data(), 64, &np, &ops) != 0)
      return 4;
    std::vector<cd> a(size_t(n) * n), b(size_t(n) * n);
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x) {
        a[size_t(y) * n + x] = det.response.values(y, x);
        b[size_t(y) * n + x] = resp[size_t(y) * n + x];
      }
    const double e = rel(a, b);
    const bool ok = e < 1e-5 && det.standard_ops == ops && !det.peaks.empty() && np > 0 &&
                    det.peaks[0].x == pxx[0] && det.peaks[0].y == pyy[0];
    std::printf("detect_pattern: rel_l2 %.3e peak (%d,%d) %s\n", e,
                det.peaks.empty() ? -1 : det.peaks[0].x, det.peaks.empty() ? -1 : det.peaks[0].y,
                ok ? "ok" : "FAIL");
    fails += !ok;
  }
  // 3D rotation (engine3d.hpp:270-335) through the shim vs the oracle
  {
    void* rg = or_rng_new(83);
    const int R3 = 2, K3 = 2, nx = 7, ny = 6, nz = 5, S3 = 2 * R3 + 1, nc3 = (K3 + 1) * (K3 + 1);
    std::vector<double> vol(2 * size_t(S3) * S3 * S3), c3(2 * size_t(2 * R3) * nc3);
    or_random_smooth_filter3(rg, R3, 6, 0.4, vol.data());
    if (or_decompose_rotation3(vol.data(), S3, S3, S3, R3, R3, R3, K3, 2 * R3, double(R3), 12, 12,
                               c3.data()) != 0)
      return 5;
    SphFilter3<double> F3;
    F3.K = K3;
    F3.n_radii = 2 * R3;
    F3.r_max = R3;
    F3.coeffs = Grid<std::complex<double>>(2 * R3, nc3);
    for (int j = 0; j < 2 * R3; ++j)
      for (int c = 0; c < nc3; ++c)
        F3.coeffs(j, c) = cd(c3[2 * (size_t(j) * nc3 + c)], c3[2 * (size_t(j) * nc3 + c) + 1]);
    const size_t n3 = size_t(nx) * ny * nz;
    std::vector<double> h3(2 * n3), q3(4 * n3);
    or_random_field3(rg, nx, ny, nz, 1, h3.data());
    or_random_rotation3_field(rg, int(n3), q3.data());
    or_rng_free(rg);
    Field3<double> H3(nx, ny, nz);
    XformField<double> T3;
    T3.kind = XformKind::rotation3;
    T3.nx = nx;
    T3.ny = ny;
    T3.nz = nz;
    for (size_t i = 0; i < n3; ++i) {
      H3.values[i] = cd(h3[2 * i], h3[2 * i + 1]);
      T3.quats.push_back({q3[4 * i], q3[4 * i + 1], q3[4 * i + 2], q3[4 * i + 3]});
    }
    for (int mode = 0; mode < 2; ++mode) {
      XConvPlan plan;
      plan.group = XformKind::rotation3;
      Response3<double> r = mode == 0
                                ? xconv::gpu::xcorr_fast_3d<Response3<double>>(H3, T3, F3, plan)
                                : xconv::gpu::xconv_fast_3d<Response3<double>>(H3, T3, F3, plan);
      std::vector<double> ref(2 * n3);
      long long ops = 0;
      if (or_xfast3(mode, h3.data(), nx, ny, nz, q3.data(), K3, 2 * R3, double(R3), c3.data(),
                    nullptr, 0, ref.data(), &ops) != 0)
        return 6;
      std::vector<cd> a(n3), b(n3);
      for (size_t i = 0; i < n3; ++i) {
        a[i] = r.output.values[i];
        b[i] = cd(ref[2 * i], ref[2 * i + 1]);
      }
      const double e = rel(a, b);
      const bool ok = e < 1e-5 && r.standard_ops == ops && ops == 35 &&
                      r.plan.mode == (mode ? XMode::convolution : XMode::correlation);
      std::printf("3D mode %d: rel_l2 %.3e ops %lld %s\n", mode, e, r.standard_ops,
                  ok ? "ok" : "FAIL");
      fails += !ok;
    }
  }
  return fails ? 1 : 0;
}
