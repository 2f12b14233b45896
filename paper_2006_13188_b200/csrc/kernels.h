// Device pipeline stages of the extended correlation / convolution hot path.
//
// Data layouts in HBM (complex fp32 = float2, per image):
//   signal   [H][W]  as the caller stores it (transposed problems are handled
//                    by rendering the filter transposed)
//   T1       layout B': [u/2][y][u%2], Hx2 rows  -- row-FFT output (F1, S1)
//   spectra  layout B : [u/2][v][u%2], Ph rows   -- H^, F^_k, Sigma
//   T2       layout A : [y/2][u][y%2], H2 rows   -- column-IFFT output (I1, S2)
// Every kernel reads its input block contiguously (a column pair of B/B' or a
// row pair of A) and writes its output as 32-byte sector-complete scatters.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "fft_plan.h"

namespace xcb {

struct Geo {
  int H, W;    // output (= signal) extent, as stored
  int Hx, Wx;  // transform input extent: H, W (zero pad) or H+2R, W+2R (periodic)
  int Hx2;     // Hx rounded up to even (rows of T1)
  int H2;      // H rounded up to even (rows of T2)
  int off;     // crop offset: 0, or R (periodic)
  int Ph, Pw;  // transform size
  int R;       // render radius
  int periodic;
};

// SIG_PACK (smoothing): the real signal h and weight w (1 when wgt is null)
// packed as one complex signal (h w, alpha w), alpha = the power of two nearest
// max|h| (from *amax, float bits), so num and den of smooth_adaptive come out of
// one scatter as its real and imaginary parts (alpha keeps both at the same
// scale, so each carries the other's rounding at its own relative size)
enum SigMode { SIG_PLAIN = 0, SIG_TIMES_W = 1, SIG_W_ONLY = 2, SIG_PACK = 3 };

struct SigSrc {
  const void* sig;  // float [H][W] (real) or float2 (complex)
  int is_complex;
  const float* wgt; // per-pixel real weight (smooth: 1/s^2) or null
  int mode;         // SigMode
  const unsigned* amax = nullptr;  // SIG_PACK: max|h| as float bits
};

struct Bands {
  const int* k;     // band frequencies (device)
  const int* spec;  // index of each band's spectrum in the filter cache
  int n;
};

// out accumulator element type
enum OutKind { OUT_C64 = 0, OUT_C128 = 1 };

struct LaunchCounter {
  int n = 0;
};

// Per-pixel steering base: rotation theta, scale omega*log(s) (double), the
// smooth weight 1/s^2 (float, optional) and the scale guard-band check.
// bad[0] = first pixel (true y-major index) with s <= 0 or non-finite,
// bad[1] = first pixel outside [lo, hi].  transposed: stored [x][y].
void launch_prep(const void* param, int param_is_f64, int kind, double omega, double lo,
                 double hi, int H, int W, int transposed, double* base, float* wgt,
                 unsigned long long* bad, cudaStream_t st, LaunchCounter& lc);

void launch_convert_signal(const void* src, int dtype, size_t n, void* dst,
                           cudaStream_t st, LaunchCounter& lc);

// F1: row FFT of the (zero-padded / periodically extended) signal -> T1.
void launch_rows_fwd(const FftPlan& prow, const Geo& g, const SigSrc& s, float2* T1,
                     cudaStream_t st, LaunchCounter& lc);
// F2: column FFT of T1 -> spectrum (layout B).
void launch_cols_fwd(const FftPlan& pcol, const Geo& g, const float2* T1, float2* spec,
                     cudaStream_t st, LaunchCounter& lc);
// I1: per band, column IFFT of H^ . conj(F^_k) -> T2_b (band planes, H2*Pw each).
void launch_cols_inv_corr(const FftPlan& pcol, const Geo& g, const float2* Hhat,
                          const float2* Fhat, size_t spec_stride, const Bands& b,
                          float2* T2, cudaStream_t st, LaunchCounter& lc);
// I2: per band, row IFFT of T2_b, crop, steer e^{+i k phi}, accumulate.
void launch_rows_inv_steer(const FftPlan& prow, const Geo& g, const float2* T2,
                           const Bands& b, const double* base, int out_kind, void* out,
                           int accumulate, const SigSrc& dc_sig, double dc_re,
                           double dc_im, cudaStream_t st, LaunchCounter& lc);
// I2 variant for the angle max: per band, row IFFT of T2_b, crop -> G planes.
void launch_rows_inv_planes(const FftPlan& prow, const Geo& g, const float2* T2,
                            int nbands, float2* planes, cudaStream_t st,
                            LaunchCounter& lc);
// S1: per band, row FFT of signal . e^{-i k phi} -> T1_b planes (Hx2*Pw each).
void launch_rows_fwd_premul(const FftPlan& prow, const Geo& g, const SigSrc& s,
                            const double* base, const Bands& b, float2* T1,
                            cudaStream_t st, LaunchCounter& lc);
// S2: per column pair, sum over bands of FFT_y(T1_b) . F^_b, then IFFT_y -> T2.
void launch_cols_fwd_mac_inv(const FftPlan& pcol, const Geo& g, const float2* T1,
                             const float2* Fhat, size_t spec_stride, const Bands& b,
                             float2* Sigma, float2* T2, cudaStream_t st, LaunchCounter& lc);
// S4: row IFFT of T2, crop (+ dc * signal) -> out.
void launch_rows_inv_out(const FftPlan& prow, const Geo& g, const float2* T2,
                         int out_kind, void* out, int accumulate, const SigSrc& dc_sig,
                         double dc_re, double dc_im, cudaStream_t st, LaunchCounter& lc,
                         const float2* T2b = nullptr);

// Filter spectra: rendered (2R+1)^2 components (nb bands, c64) -> F^ (layout B).
void launch_filter_spectra(const FftPlan& prow, const FftPlan& pcol, const Geo& g,
                           const float2* comps, int nb, float2* T1f, float2* Fhat,
                           cudaStream_t st, LaunchCounter& lc);

// smooth: max |den| (as float bits) then divide with the 1e-9 floor.
// max|x| of a real fp32 field as float bits (atomicMax; *bits zeroed by the caller)
void launch_absmax(const float* x, size_t n, unsigned* bits, cudaStream_t st, LaunchCounter& lc);
// smooth_adaptive's divide from one packed scatter z = num + i alpha den
// (SIG_PACK): floor 1e-9 max|den|, out = num / den
void launch_smooth_finish_packed(const float2* z, size_t n, const unsigned* amax, int out_f64,
                                 void* out, unsigned* maxbits, unsigned* clamped, cudaStream_t st,
                                 LaunchCounter& lc);
void launch_smooth_finish(const float2* num, const float2* den, size_t n, int out_f64,
                          void* out, unsigned* maxbits, unsigned* clamped,
                          cudaStream_t st, LaunchCounter& lc);

// angle max over n_angles of |sum_b G_b e^{-i k_b 2 pi s/n}|.
void launch_anglemax(const float2* planes, const int* ks_host, int nb, size_t npix,
                     int n_angles, int score_f64, void* score, int* argmax,
                     cudaStream_t st, LaunchCounter& lc);

// Hermitian half-band angle max (real signal, F_{-k} = conj F_k): planes of
// bands k = 0..KH only (ks_host: their k values, plane order); 360 angles.
void launch_anglemax_herm(const float2* planes, const int* ks_host, int nb, size_t npix,
                          int score_f64, void* score, int* argmax, cudaStream_t st,
                          LaunchCounter& lc);
int anglemax_herm_kh(int kh);  // 1 if KH has a half-band kernel (4, 8, 16)
// the same half-band angle max (360 angles, KH <= 16) as two tf32 GEMMs per
// 128-pixel tile on the tensor cores, 3xTF32 (k_anglemax_tc.cu)
bool anglemax_tc_ok(int kh);
void launch_anglemax_tc(const float2* planes, const int* ks_host, int nb, size_t npix,
                        int score_f64, void* score, int* argmax, cudaStream_t st,
                        LaunchCounter& lc);

// Upload the plan's twiddles; returns device pointer (owned by caller).
float2* upload_twiddles(const FftPlan& p);

}  // namespace xcb

namespace xcb {
// Fast band-loop variants (k_fast.cu): plans from make_fast_plan.  fast_smem
// returns the dynamic smem a stage needs, or 0 if it does not fit (stage 0 =
// I1, 1 = I2, 2 = S1, 3 = S2, 4 = planes); callers fall back to the generic
// kernels.
size_t fast_smem(int stage, const FftPlan& pl, const Geo& g);
void launch_cols_inv_corr_fast(const FftPlan& pc, const Geo& g, const float2* Hhat,
                               const float2* Fhat, size_t sstride, const Bands& b, float2* T2,
                               cudaStream_t st, LaunchCounter& lc);
// parts: scratch for band-chunked partial sums (fast_steer_chunks(g, nb) x
// H x W float2), or null for one CTA per row pair over all bands
void launch_rows_inv_steer_fast(const FftPlan& pr, const Geo& g, const float2* T2,
                                const Bands& b, const double* base, int out_kind, void* out,
                                int accumulate, const SigSrc& dcs, double dcr, double dci,
                                float2* parts, cudaStream_t st, LaunchCounter& lc);
int fast_steer_chunks(const Geo& g, int nb);
// F1 / F2 with the compile-time plans (stage 5 of fast_smem)
void launch_rows_fwd_fast(const FftPlan& pr, const Geo& g, const SigSrc& s, float2* T1,
                          cudaStream_t st, LaunchCounter& lc);
void launch_cols_fwd_fast(const FftPlan& pc, const Geo& g, const float2* T1, float2* spec,
                          cudaStream_t st, LaunchCounter& lc);
void launch_rows_inv_planes_fast(const FftPlan& pr, const Geo& g, const float2* T2,
                                 int nbands, float2* planes, cudaStream_t st,
                                 LaunchCounter& lc);
void launch_rows_fwd_premul_fast(const FftPlan& pr, const Geo& g, const SigSrc& s,
                                 const double* base, const Bands& b, float2* T1,
                                 cudaStream_t st, LaunchCounter& lc);
void launch_cols_fwd_mac_inv_fast(const FftPlan& pc, const Geo& g, const float2* T1,
                                  const float2* Fhat, size_t sstride, const Bands& b,
                                  float2* T2, cudaStream_t st, LaunchCounter& lc);
// the same over conjugate band pairs (launch_cols_fwd_mac_inv_cpair); fast_smem stage 6
void launch_cols_fwd_mac_inv_cpair_fast(const FftPlan& pc, const Geo& g, const float2* T1,
                                        const float2* Fhat, const float2* Ghat, size_t sstride,
                                        const Bands& b, const int* gspec, float2* T2,
                                        size_t t2plane, cudaStream_t st, LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// Pair-engine variants (k_pair.cu, lengths of XCB_PAIR_TABLE in fft_pair.cuh):
// pair_smem returns the dynamic smem of stage 0 (I1) / 1 (I2) / 2 (planes) / 3 (S1) /
// 4 (S2), or 0 when the
// length has no pair plan; callers then use the fast or generic kernels.
size_t pair_smem(int stage, int L, const Geo& g);
// nimg (1 or 2; 2 only on the interleaved engine) images per launch: Hhat and
// T2 of image i at Hhat + i * hstride, T2 + i * tstride (float2 units); the
// staged filter spectrum column is shared by the images.
void launch_cols_inv_corr_pair(const Geo& g, const float2* Hhat, const float2* Fhat,
                               size_t sstride, const Bands& b, float2* T2, cudaStream_t st,
                               LaunchCounter& lc, int nimg = 1, size_t hstride = 0,
                               size_t tstride = 0);
// scatter stages S1 / S2 on the pair engine (stages 3 / 4 of pair_smem)
void launch_rows_fwd_premul_pair(const Geo& g, const SigSrc& s, const double* base,
                                 const Bands& b, float2* T1, cudaStream_t st, LaunchCounter& lc);
// the transform lengths served by the pair engine (k_pair.cu XCB_PAIR_TABLE)
std::vector<int> pair_plan_lengths();
// half0: Hermitian half-band mode (bands k >= 0; the k = 0 band weighted 1/2)
void launch_cols_fwd_mac_inv_pair(const Geo& g, const float2* T1, const float2* Fhat,
                                  size_t sstride, const Bands& b, int half0, float2* T2,
                                  cudaStream_t st, LaunchCounter& lc);
// Conjugate band pairs (real signal, any filter): T1 holds the bands k >= 0
// only, since H e^{+ik phi} = conj(H e^{-ik phi}).  Per band k the column FFT X
// feeds two sums, A += X F^_k and (k > 0) B += X G_k with G_k the spectrum of
// conj(f_{-k}) (plane gspec[bi] of Ghat, launch_spec_conj_reflect); both are
// inverse transformed into T2 and T2 + t2plane, and S4 writes a + conj(b).
void launch_cols_fwd_mac_inv_cpair(const Geo& g, const float2* T1, const float2* Fhat,
                                   const float2* Ghat, size_t sstride, const Bands& b,
                                   const int* gspec, float2* T2, size_t t2plane,
                                   cudaStream_t st, LaunchCounter& lc);
// G_i[v, u] = conj(F^_i[-v, -u]) for nb spectra in layout B: the spectrum of
// the conjugated filter component
void launch_spec_conj_reflect(const float2* Fhat, float2* Ghat, int nb, int Ph, int Pw,
                              cudaStream_t st, LaunchCounter& lc);
// single transforms on the pair engine: F1 (stage 5), F2 (6), S4 (7)
void launch_rows_fwd_pair(const Geo& g, const SigSrc& s, float2* T1, cudaStream_t st,
                          LaunchCounter& lc);
void launch_cols_fwd_pair(const Geo& g, const float2* T1, float2* spec, cudaStream_t st,
                          LaunchCounter& lc);
// real2: out = 2 Re(IFFT) (+ dc H), the Hermitian half-band scatter
// T2b (conjugate band pairs, else nullptr): out = IFFT(T2) + conj(IFFT(T2b))
void launch_rows_inv_out_pair(const Geo& g, const float2* T2, int out_kind, void* out,
                              int accumulate, int real2, const SigSrc& dcs, double dcr,
                              double dci, cudaStream_t st, LaunchCounter& lc,
                              const float2* T2b = nullptr);
// planes stage (angle max) on the interleaved engine; stage 2 of pair_smem
void launch_rows_inv_planes_pair(const Geo& g, const float2* T2, int nbands, float2* planes,
                                 cudaStream_t st, LaunchCounter& lc);
// images per I1 launch the pair engine supports for this geometry
int pair_i1_images();
// I1 of one image (Hhat -> T2w) and I2 of the previous one (T2r -> out) in one
// launch with interleaved CTAs (needs Ph == Pw and both pair plans)
bool dual_pair_ok(const Geo& g);
void launch_dual_pair(const Geo& g, const float2* Hhat, const float2* Fhat, size_t sstride,
                      const Bands& b, float2* T2w, const float2* T2r, int half,
                      const double* base, int out_kind, void* out, int accumulate,
                      const SigSrc& dcs, double dcr, double dci, cudaStream_t st,
                      LaunchCounter& lc);
// half: Hermitian half-band mode (bands k >= 0, k = 0 weighted 1/2, out = 2 Re)
void launch_rows_inv_steer_pair(const Geo& g, const float2* T2, const Bands& b, int half,
                                const double* base, int out_kind, void* out, int accumulate,
                                const SigSrc& dcs, double dcr, double dci, cudaStream_t st,
                                LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// detect_pattern (vote_filter.hpp:146-168): gradient magnitude / direction of
// a real image (f32 or f64, row- or column-major) -> fp32 in the same order;
// real part of a complex field.
void launch_gradient(const void* img, int img_f64, int h, int w, int colmajor, float* mag,
                     float* dir, cudaStream_t st, LaunchCounter& lc);
void launch_real_part(const float2* in, size_t n, int out_f64, void* out, cudaStream_t st,
                      LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// find_peaks (vote_filter.hpp:107-134) on a device response: global max, then
// every local maximum within the disk above frac * max appended (x, y, value)
// to the first `cap` slots; *count = number found (the host sorts).
void launch_find_peaks(const void* resp, int f64, int h, int w, int colmajor, double radius,
                       double frac, int cap, unsigned long long* mx, unsigned* count, int* px,
                       int* py, double* pv, cudaStream_t st, LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// Render every band of a decomposed filter on the (2R+1)^2 grid on the GPU
// (freq_filter.hpp:133-184): comps [n_rows][nb] complex fp64, ks [nb];
// out [nb][S][S] c64 (transposed grids when `transpose`).
void launch_render(const double2* comps, const int* ks, int nb, int group, int n_radii,
                   int n_angles, double r_max, double r_min, double omega, int S, int R,
                   int transpose, float2* out, cudaStream_t st, LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// dst[i] += src[i] over n floats (f64 = 0) or doubles (f64 = 1): the ordered
// partial sums of the multi-device band reduce without NCCL (peer copies).
void launch_accumulate(void* dst, const void* src, size_t n, int f64, cudaStream_t st,
                       LaunchCounter& lc);
// dst += slots[0] + ... + slots[ns - 1] in slot order; n, stride in scalars (even)
void launch_sum_slots(void* dst, const void* slots, size_t stride, int ns, size_t n, int f64,
                      cudaStream_t st, LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// decompose_rotation2 (group 0) / decompose_scale2 (group 1) on the device
// (freq_filter.hpp:63-129): img row-major [h][w] complex fp64; samples scratch
// [nr][na]; comps [n_rows][nc] complex fp64.  r_top = r_max (rotation) or the
// basis domain top (scale).
void launch_decompose(const double2* img, int w, int h, double cx, double cy, int nr, int na,
                      int group, double r_min, double r_top, const int* ks, int nc,
                      double2* samples, double2* comps, cudaStream_t st, LaunchCounter& lc);
}  // namespace xcb

namespace xcb {
// fft2 (fft.hpp:20-53) on the device: input staging to c64 (conjugated for the
// inverse) and the F2 spectrum (layout B) to row-major c64 / c128 (conjugated
// and scaled 1/(Ph Pw) for the inverse)
// (tr: the caller's rows x cols grid is transformed as its transpose, so that
// the staged row length, which the engine pairs, is even)
void launch_fft2_in(const void* src, int c128, int rows, int cols, int tr, int conj_in,
                    float2* dst, cudaStream_t st, LaunchCounter& lc);
void launch_fft2_out(const float2* hh, int rows, int cols, int tr, int inverse, int c128,
                     void* out, cudaStream_t st, LaunchCounter& lc);
}  // namespace xcb
