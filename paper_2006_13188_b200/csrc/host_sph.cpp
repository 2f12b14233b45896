// Host side of the 3D rotation pipeline: SH band decomposition and
// rendering of a 3D filter (sph.hpp), Wigner-D coefficients (wigner.hpp).
#include "host_sph.h"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace xcb {
namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;

// sph.hpp:13-33: fully normalized P_l^m(cos theta) with Condon-Shortley phase
std::vector<double> legendre(int lmax, double ct) {
  const double st = std::sqrt(std::max(0.0, 1 - ct * ct));
  auto at = [](int l, int m) { return l * (l + 1) / 2 + m; };
  std::vector<double> P(size_t(at(lmax, lmax)) + 1);
  P[0] = std::sqrt(1.0 / (4 * kPi));
  for (int m = 1; m <= lmax; ++m)
    P[at(m, m)] = -std::sqrt(double(2 * m + 1) / double(2 * m)) * st * P[at(m - 1, m - 1)];
  for (int m = 0; m < lmax; ++m) P[at(m + 1, m)] = std::sqrt(double(2 * m + 3)) * ct * P[at(m, m)];
  for (int m = 0; m <= lmax; ++m)
    for (int l = m + 2; l <= lmax; ++l) {
      const double a = std::sqrt(double(4 * l * l - 1) / double(l * l - m * m));
      const double b =
          std::sqrt(double((l - 1) * (l - 1) - m * m) / double(4 * (l - 1) * (l - 1) - 1));
      P[at(l, m)] = a * (ct * P[at(l - 1, m)] - b * P[at(l - 2, m)]);
    }
  return P;
}

// Quadrature weights of the equiangular theta midpoints: sum_i w_i P_n(cos
// theta_i) = 2 delta_n0 for n < nt (sph.hpp:59-84), Gaussian elimination with
// partial pivoting
std::vector<double> theta_weights(int nt, std::vector<double>& theta) {
  theta.resize(nt);
  for (int i = 0; i < nt; ++i) theta[i] = kPi * (i + 0.5) / nt;
  std::vector<double> A(size_t(nt) * nt), b(nt, 0.0);
  b[0] = 2;
  for (int i = 0; i < nt; ++i) {
    const double x = std::cos(theta[i]);
    double p0 = 1, p1 = x;
    A[i] = p0;
    if (nt > 1) A[size_t(nt) + i] = p1;
    for (int n = 2; n < nt; ++n) {
      const double p2 = ((2 * n - 1) * x * p1 - (n - 1) * p0) / n;
      A[size_t(n) * nt + i] = p2;
      p0 = p1;
      p1 = p2;
    }
  }
  for (int k = 0; k < nt; ++k) {
    int p = k;
    for (int i = k + 1; i < nt; ++i)
      if (std::abs(A[size_t(i) * nt + k]) > std::abs(A[size_t(p) * nt + k])) p = i;
    if (p != k) {
      for (int j = 0; j < nt; ++j) std::swap(A[size_t(k) * nt + j], A[size_t(p) * nt + j]);
      std::swap(b[k], b[p]);
    }
    const double piv = A[size_t(k) * nt + k];
    for (int i = k + 1; i < nt; ++i) {
      const double f = A[size_t(i) * nt + k] / piv;
      for (int j = k; j < nt; ++j) A[size_t(i) * nt + j] -= f * A[size_t(k) * nt + j];
      b[i] -= f * b[k];
    }
  }
  std::vector<double> w(nt);
  for (int k = nt - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j < nt; ++j) s -= A[size_t(k) * nt + j] * w[j];
    w[k] = s / A[size_t(k) * nt + k];
  }
  return w;
}

// Field3::sample (field.hpp:94-113): trilinear, 0 outside the grid
cplx sample3(const cplx* f, int nx, int ny, int nz, double x, double y, double z) {
  const int x0 = int(std::floor(x)), y0 = int(std::floor(y)), z0 = int(std::floor(z));
  const double tx = x - x0, ty = y - y0, tz = z - z0;
  cplx out(0);
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double w = (dx ? tx : 1 - tx) * (dy ? ty : 1 - ty) * (dz ? tz : 1 - tz);
        const int xi = x0 + dx, yi = y0 + dy, zi = z0 + dz;
        if (w == 0 || xi < 0 || yi < 0 || zi < 0 || xi >= nx || yi >= ny || zi >= nz) continue;
        out += w * f[(size_t(zi) * ny + yi) * nx + xi];
      }
  return out;
}

double log_fact(int n) {
  double s = 0;
  for (int i = 2; i <= n; ++i) s += std::log(double(i));
  return s;
}

}  // namespace

int HostFilter3::render_radius() const { return int(std::ceil(r_max)); }

cplx HostFilter3::radial(int l, int m, double r) const {
  double u = r / r_max * n_radii - 0.5;
  u = std::min(std::max(u, 0.0), double(n_radii - 1));
  const int j0 = int(u), j1 = std::min(j0 + 1, n_radii - 1);
  const double t = u - j0;
  return (1 - t) * coeff(j0, l, m) + t * coeff(j1, l, m);
}

cplx sph_harm(int l, int m, double theta, double phi) {
  const int am = std::abs(m);
  if (am > l) throw std::invalid_argument("|m| must be <= l");
  const double p = legendre(l, std::cos(theta))[l * (l + 1) / 2 + am];
  cplx y = p * std::polar(1.0, am * phi);
  if (m < 0) y = (am % 2 ? -1.0 : 1.0) * std::conj(y);
  return y;
}

HostFilter3 decompose_rotation3(const cplx* vol, int nx, int ny, int nz, double cx, double cy,
                                double cz, int K, int n_radii, double r_max, int n_theta,
                                int n_phi) {
  if (K < 0) throw std::invalid_argument("band limit must be >= 0");
  if (n_radii < 1) throw std::invalid_argument("n_radii must be >= 1");
  if (n_theta == 0) n_theta = 2 * (K + 1);
  if (n_phi == 0) n_phi = 2 * (K + 1);
  if (n_theta < 2 * (K + 1) || n_phi < 2 * (K + 1))
    throw std::invalid_argument("insufficient angular sampling for band limit");
  std::vector<double> theta;
  const std::vector<double> wt = theta_weights(n_theta, theta);
  const double dphi = 2 * kPi / n_phi;
  HostFilter3 f;
  f.K = K;
  f.n_radii = n_radii;
  f.r_max = r_max;
  f.coeffs.assign(size_t(n_radii) * f.ncol(), cplx(0));
  std::vector<cplx> az(2 * K + 1);
  for (int j = 0; j < n_radii; ++j) {
    const double r = (j + 0.5) * r_max / n_radii;
    cplx* c = f.coeffs.data() + size_t(j) * f.ncol();
    // sh_analyze (sph.hpp:90-113): azimuthal sums, then Legendre weights
    for (int i = 0; i < n_theta; ++i) {
      const double th = theta[i];
      std::fill(az.begin(), az.end(), cplx(0));
      for (int jj = 0; jj < n_phi; ++jj) {
        const double ph = 2 * kPi * jj / n_phi;
        const cplx v = sample3(vol, nx, ny, nz, cx + r * std::sin(th) * std::cos(ph),
                               cy + r * std::sin(th) * std::sin(ph), cz + r * std::cos(th));
        for (int m = -K; m <= K; ++m) az[m + K] += v * std::polar(1.0, -m * ph);
      }
      const std::vector<double> P = legendre(K, std::cos(th));
      for (int l = 0; l <= K; ++l)
        for (int m = -l; m <= l; ++m) {
          const int am = std::abs(m);
          double p = P[l * (l + 1) / 2 + am];
          if (m < 0 && (am % 2)) p = -p;
          c[l * (l + 1) + m] += wt[i] * dphi * p * az[m + K];
        }
    }
  }
  return f;
}

void render_sph_component(const HostFilter3& f, int l, int m_radial, int m_angular, int nx,
                          int ny, int nz, double cx, double cy, double cz, cplx* out) {
  if (l < 0 || l > f.K || std::abs(m_radial) > l || std::abs(m_angular) > l)
    throw std::invalid_argument("component outside the filter's band limit");
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        cplx& o = out[(size_t(z) * ny + y) * nx + x];
        o = 0;
        const double dx = x - cx, dy = y - cy, dz = z - cz;
        const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
        if (r > f.r_max || (r <= 1e-9 && l > 0)) continue;
        const double theta = r > 0 ? std::acos(std::clamp(dz / r, -1.0, 1.0)) : 0.0;
        o = f.radial(l, m_radial, r) * sph_harm(l, m_angular, theta, std::atan2(dy, dx));
      }
}

void reconstruct3(const HostFilter3& f, int nx, int ny, int nz, double cx, double cy, double cz,
                  const int* degrees, int ndeg, cplx* out) {
  const size_t n = size_t(nx) * ny * nz;
  std::fill(out, out + n, cplx(0));
  std::vector<cplx> c(n);
  for (int l = 0; l <= f.K; ++l) {
    if (degrees && std::find(degrees, degrees + ndeg, l) == degrees + ndeg) continue;
    for (int m = -l; m <= l; ++m) {
      render_sph_component(f, l, m, m, nx, ny, nz, cx, cy, cz, c.data());
      for (size_t i = 0; i < n; ++i) out[i] += c[i];
    }
  }
}

SmallD small_d_coeffs(int l, int m1, int m2) {
  SmallD s;
  if (l > 16) throw std::invalid_argument("degree above 16 is not supported");
  const int s_lo = std::max(0, m2 - m1), s_hi = std::min(l - m1, l + m2);
  if (s_hi < s_lo) return s;
  const double pref = 0.5 * (log_fact(l + m1) + log_fact(l - m1) + log_fact(l + m2) +
                             log_fact(l - m2));
  // term_s = sign exp(lg_s) cb^(2l+m2-m1-2s) sb^(m1-m2+2s): with k = s - s_lo,
  // cb^pc sb^ps = cb^pc_end sb^ps0 u^(n-k) v^k
  s.n = s_hi - s_lo;
  s.pc_end = 2 * l + m2 - m1 - 2 * s_hi;
  s.ps0 = m1 - m2 + 2 * s_lo;
  for (int k = 0; k <= s.n; ++k) {
    const int sv = s_lo + k;
    const double lg = pref - log_fact(l + m2 - sv) - log_fact(sv) - log_fact(m1 - m2 + sv) -
                      log_fact(l - m1 - sv);
    s.c[k] = ((m1 - m2 + sv) % 2 ? -1.0 : 1.0) * std::exp(lg);
  }
  return s;
}

double small_d_eval(const SmallD& s, double beta) {
  if (s.n < 0) return 0;
  const double cb = std::cos(beta / 2), sb = std::sin(beta / 2);
  const double u = cb * cb, v = sb * sb;
  double acc = s.c[0], vk = 1;
  for (int k = 1; k <= s.n; ++k) {
    vk *= v;
    acc = acc * u + s.c[k] * vk;
  }
  double p = 1;
  for (int i = 0; i < s.pc_end; ++i) p *= cb;
  for (int i = 0; i < s.ps0; ++i) p *= sb;
  return p * acc;
}

void euler_zyz(const double* q, double* abg) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  // Eigen Quaternion::toRotationMatrix
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w, txx = tx * x, txy = ty * x,
               txz = tz * x, tyy = ty * y, tyz = tz * y, tzz = tz * z;
  const double M00 = 1 - (tyy + tzz), M02 = txz + twy, M10 = txy + twz, M12 = tyz - twx,
               M20 = txz - twy, M21 = tyz + twx, M22 = 1 - (txx + tyy);
  const double sb = std::sqrt(M02 * M02 + M12 * M12);
  abg[1] = std::atan2(sb, M22);
  if (sb > 1e-12) {
    abg[0] = std::atan2(M12, M02);
    abg[2] = std::atan2(M21, -M20);
  } else {
    abg[0] = std::atan2(M10, M00);
    if (M22 < 0) abg[0] = -abg[0];
    abg[2] = 0;
  }
}

void wigner_d(int l, const double* q, cplx* D) {
  if (l < 0) throw std::invalid_argument("degree must be >= 0");
  const double nr = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (std::abs(nr - 1.0) > 1e-9) throw std::invalid_argument("rotation quaternion must be unit norm");
  const double qn[4] = {q[0] / nr, q[1] / nr, q[2] / nr, q[3] / nr};
  double abg[3];
  euler_zyz(qn, abg);
  const int n = 2 * l + 1;
  for (int m1 = -l; m1 <= l; ++m1)
    for (int m2 = -l; m2 <= l; ++m2)
      D[size_t(m1 + l) * n + (m2 + l)] = std::polar(1.0, -m1 * abg[0]) *
                                         small_d_eval(small_d_coeffs(l, m1, m2), abg[1]) *
                                         std::polar(1.0, -m2 * abg[2]);
}

}  // namespace xcb
