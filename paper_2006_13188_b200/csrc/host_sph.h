// Host side of the 3D rotation pipeline: the spherical
// harmonic band decomposition of a 3D filter and its per-band rendering, run
// once per filter (sph.hpp), and the Wigner-D coefficients the steering
// kernels evaluate per voxel (wigner.hpp).  Volumes are x fastest,
// index (z*ny + y)*nx + x (field.hpp:67-85).
#pragma once
#include <complex>
#include <vector>

namespace xcb {

using cplx = std::complex<double>;

// SphFilter3 (sph.hpp:130-157): coeffs row-major [shell][l*(l+1)+m]
struct HostFilter3 {
  int K = 0, n_radii = 0;
  double r_max = 0;
  std::vector<cplx> coeffs;
  int ncol() const { return (K + 1) * (K + 1); }
  int render_radius() const;  // ceil(r_max) (engine3d.hpp:283)
  cplx coeff(int shell, int l, int m) const {
    return coeffs[size_t(shell) * ncol() + l * (l + 1) + m];
  }
  cplx radial(int l, int m, double r) const;  // sph.hpp:142-151
};

// sph.hpp:37-47
cplx sph_harm(int l, int m, double theta, double phi);
// sph.hpp:161-188 (n_theta / n_phi 0 = 2(K+1)); throws std::invalid_argument
HostFilter3 decompose_rotation3(const cplx* vol, int nx, int ny, int nz, double cx, double cy,
                                double cz, int K, int n_radii, double r_max, int n_theta,
                                int n_phi);
// sph.hpp:194-212: f_l^{m_radial}(r) Y_l^{m_angular} on an nx*ny*nz grid
void render_sph_component(const HostFilter3& f, int l, int m_radial, int m_angular, int nx,
                          int ny, int nz, double cx, double cy, double cz, cplx* out);
// sph.hpp:215-221 (degrees == nullptr: all)
void reconstruct3(const HostFilter3& f, int nx, int ny, int nz, double cx, double cy, double cz,
                  const int* degrees, int ndeg, cplx* out);

// d^l_{m1 m2}(beta) = pref(beta) * sum_k c_k u^{n-k} v^k, u = cos^2(beta/2),
// v = sin^2(beta/2), pref = cos(beta/2)^pc_end sin(beta/2)^ps0 (wigner.hpp:18-37
// regrouped so a kernel evaluates it with one Horner loop, no pow)
struct SmallD {
  int pc_end = 0, ps0 = 0, n = -1;  // n < 0: the entry is identically 0
  double c[2 * 16 + 1];
};
SmallD small_d_coeffs(int l, int m1, int m2);
double small_d_eval(const SmallD& s, double beta);
// wigner.hpp:40-57 on a unit quaternion (w, x, y, z)
void euler_zyz(const double* q, double* abg);
// wigner.hpp:64-88: D[(m_to + l)(2l+1) + m_from + l]; throws on l < 0 or a
// non-unit quaternion
void wigner_d(int l, const double* q, cplx* D);

}  // namespace xcb
