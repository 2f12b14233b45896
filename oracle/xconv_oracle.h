/*
 * xconv_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (double precision, no Eigen) of the reference 2D extended
 * correlation / convolution path of arXiv 2006.13188 (`xconv`, mounted at
 * /root/reference).  This library is the *checker* for the B200 product in
 * paper_2006_13188_b200/: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product never links
 * or calls it.
 *
 * The reference itself cannot be compiled here (it needs Eigen >= 3.4,
 * proj/CMakeLists.txt:10, which is absent), so parity is pinned by porting the
 * reference's own implementation-independent known-answer tests (direct-loop
 * FFT filtering, spectral oracles, brute-force oracles, constant-field
 * reductions) onto this restatement -- see tests/test_oracle_kat.py.
 *
 * Storage convention: every 2D grid is ROW-MAJOR [y][x] (y = row, height), the
 * transpose of the reference's Eigen column-major storage (field.hpp:15).  The
 * reference's `values(y,x)` is element y*W + x here.  Complex arrays are
 * interleaved (re, im) doubles.  All loops follow the reference's loop order
 * (fft2 does columns then rows, fft.hpp:50-53), so arithmetic is unchanged.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FreqFilter2 (freq_filter.hpp:21-46).  comps is row-major [n_rows][nc]
 * complex, n_rows = n_radii (rotation2) or n_angles (scale2). */
typedef struct {
  int group; /* 0 = rotation2, 1 = scale2 (field.hpp:129) */
  int K;
  int nc;
  const int* ks;
  const double* comps;
  int n_radii, n_angles;
  double r_max, r_min, r_domain;
} or_filter;

const char* or_last_error(void);
int or_next_fast_size(int n);

/* fft.hpp:49-53: in-place 2D FFT (columns then rows), kissfft semantics. */
void or_fft2(double* a, int h, int w, int inverse);
/* fft.hpp:78-100 */
void or_filter2_fft(const double* sig, int h, int w, const double* filt, int fh,
                    int fw, int fcx, int fcy, int correlate, int periodic,
                    double* out);
/* test_fft.cpp:9-36 direct-loop references */
void or_correlate_direct(const double* H, int h, int w, const double* F, int fh,
                         int fw, int fcx, int fcy, double* out);
void or_convolve_direct(const double* H, int h, int w, const double* F, int fh,
                        int fw, int fcx, int fcy, double* out);

/* freq_filter.hpp:63-129.  ks_out needs 2*(K/2)+1 ints, comps_out
 * n_rows*nc complex.  Return 0 ok, 2 invalid argument (or_last_error). */
int or_decompose_rotation2(const double* filt, int fw, int fh, double cx,
                           double cy, int K, int n_radii, int n_angles,
                           double r_max, int* ks_out, double* comps_out,
                           int* nc_out);
int or_decompose_scale2(const double* filt, int fw, int fh, double cx, double cy,
                        int K, int n_radii, int n_angles, double r_min,
                        double r_max, double r_domain, int* ks_out,
                        double* comps_out, int* nc_out);
void or_component_value(const or_filter* F, int ci, double r, double theta,
                        double* out2);
void or_render_component(const or_filter* F, int ci, int width, int height,
                         double cx, double cy, double* out);
void or_inner_dc_value(const or_filter* F, double* out2);
void or_reconstruct(const or_filter* F, int width, int height, double cx,
                    double cy, const int* subset, int nsub, double* out);
void or_synthesize_polar(const or_filter* F, const int* subset, int nsub,
                         double* out);

/* engine.hpp:286-373.  mode 0 = correlation (xcorr_fast), 1 = convolution
 * (xconv_fast).  kind 0 = rotation2 (param = raw angle, normalized as
 * XformField::rotation does, field.hpp:143-148), 1 = scale2 (param = scale
 * factor, field.hpp:150-158).  components: subset of ks (NULL/0 = all).
 * seconds_out[4] = render, fft, combine, premultiply (engine.hpp:41-49).
 * nthreads > 1 runs contiguous band ranges on threads (ordered reduction). */
int or_xfast(int mode, const double* H, int h, int w, int kind,
             const double* param, const or_filter* F, const int* components,
             int ncomp, int periodic, double* out, long long* ops_out,
             double* seconds_out, int nthreads);
/* engine.hpp:385-419 */
int or_smooth_adaptive(const double* H, int h, int w, int kind,
                       const double* param, const or_filter* F, int normalize,
                       double* out_real, long long* ops_out, int* clamped_out,
                       int nthreads);
/* engine.hpp:233-249 (brute force over synthesis_table) */
int or_xbrute(int mode, const double* H, int h, int w, int kind,
              const double* param, const or_filter* F, double eps,
              int table_radii, int table_angles, double* out);
/* test_engine2d.cpp:33-61 / test_engine_scale.cpp:37-78 spectral oracles */
int or_spectral_oracle(int mode, const double* H, int h, int w, int kind,
                       const double* param, const or_filter* F, double* out);

/* spectral oracle at selected pixels; real float32 signal / param */
int or_spectral_oracle_at(int mode, const float* H, int h, int w, int kind,
                          const float* param, const or_filter* F, const int* pys,
                          const int* pxs, int npix, double* out);
/* vote_filter.hpp:107-134.  Returns number of peaks (<= max_out written). */
int or_find_peaks(const double* resp, int h, int w, double radius,
                  double threshold_frac, int* xs, int* ys, double* vals,
                  int max_out);
/* contour.hpp:29-55 */
void or_gaussian_blur(const double* in, int h, int w, double sigma, double* out);
/* field.hpp:203-237 (real image in, magnitude/direction out) */
void or_gradient(const double* img, int h, int w, double* mag, double* dir);
/* vote_filter.hpp:62-91: vote filters (row-major [y][x]; weights_out holds
 * (2R+1)^2 values, R = ceil(eps) returned in *radius_out) */
int or_build_vote_filter(const double* weight, const double* frame, int h, int w, double px,
                         double py, double eps, int nearest, double* weights_out,
                         int* radius_out);
int or_build_optimal_filter(const double* pattern, int h, int w, double px, double py,
                            double eps, int nearest, double* weights_out, int* radius_out);
/* vote_filter.hpp:146-168: response (h*w, Re of xconv_fast) and NMS peaks */
int or_detect_pattern(const double* image, int h, int w, const double* vote_weights,
                      int radius, double eps, int K, int n_radii, int n_angles,
                      double* response, int* xs, int* ys, double* vals, int max_peaks,
                      int* n_peaks, long long* ops_out);
/* BASELINE config 3 / SURVEY 8(a) A9: score(p) = max_s |sum_k e^{-i k 2 pi s/n}
 * G_k(p)| over s in [0,n_angles); argmax = first s attaining the max.
 * G is [nc][h][w] complex. */
void or_anglemax(const double* G, const int* ks, int nc, int h, int w,
                 int n_angles, double* score, int* argmax);

/* Seeded fixtures of proj/tests/helpers.hpp (std::mt19937_64 +
 * std::uniform_real_distribution, bit-identical to the reference tests when
 * built with the same libstdc++). */
void* or_rng_new(uint64_t seed);
void or_rng_free(void* rng);
void or_random_field(void* rng, int w, int h, int complex_valued, double* out);
void or_random_smooth_filter(void* rng, int radius, int n_bumps,
                             double envelope_frac, double* out);
void or_annular_filter(void* rng, int R, double r0_frac, double sr_frac,
                       double* out);
void or_random_rotation_field(void* rng, int w, int h, double* out);
void or_random_scale_field(void* rng, int w, int h, double lo, double hi,
                           double* out);
uint64_t or_rng_next(void* rng);
double or_rng_uniform(void* rng, double a, double b);


/* ---- 3D rotation pipeline (xconv_oracle3d.inc; sph.hpp, wigner.hpp,
 * engine3d.hpp).  Volumes x fastest, complex interleaved; quaternions
 * (w, x, y, z); SphFilter3 coefficients row-major [shell][l(l+1)+m]. */
int or_decompose_rotation3(const double* vol, int nx, int ny, int nz, double cx, double cy,
                           double cz, int K, int n_radii, double r_max, int n_theta, int n_phi,
                           double* coeffs_out);
int or_xfast3(int mode, const double* H, int nx, int ny, int nz, const double* quats, int K,
              int n_radii, double r_max, const double* coeffs, const int* degrees, int ndeg,
              double* out, long long* ops);
void or_random_field3(void* rng, int nx, int ny, int nz, int complex_valued, double* out);
void or_random_smooth_filter3(void* rng, int radius, int n_bumps, double envelope_frac,
                              double* out);
void or_random_rotation3_field(void* rng, int n, double* out);

/* Full-size parity helpers (threaded; same arithmetic as the loops above). */
/* G: nk planes [h][w] complex, G_k = filter2_fft(H, F_k, correlate). */
int or_band_responses(const double* H, int h, int w, const or_filter* F, const int* ks,
                      int nk, int nthreads, double* G);
void or_anglemax_mt(const double* G, const int* ks, int nc, int h, int w, int n_angles,
                    int nthreads, double* score, int* argmax);
/* xcorr_fast / xconv_fast by direct summation at npix pixels (no FFT). */
int or_direct_at(int mode, const double* H, int h, int w, int kind, const double* param,
                 const or_filter* F, const int* pys, const int* pxs, int npix, int nthreads,
                 double* out);

#ifdef __cplusplus
}
#endif
