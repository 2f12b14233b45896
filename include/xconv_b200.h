/*
 * xconv_b200.h -- C ABI of the B200-native extended correlation / convolution
 * hot path (arXiv 2006.13188).  This is the drop-in boundary: the reference's
 * C++ host API (proj/include/xconv/engine.hpp) keeps its signatures and calls
 * these entry points instead of its per-band CPU loop (INTEGRATION.md shows
 * the shim).  Plain pointers and sizes only; no C++ or torch types.
 *
 * Entry points and the reference interface each one replaces:
 *   xc_run(mode = XC_CORRELATION)  <- xcorr_fast   engine.hpp:286-326
 *   xc_run(mode = XC_CONVOLUTION)  <- xconv_fast   engine.hpp:331-373
 *   xc_smooth                      <- smooth_adaptive engine.hpp:385-419
 *   xc_anglemax                    <- (new; BASELINE config 3)
 *   xc_find_peaks                  <- find_peaks   vote_filter.hpp:107-134
 *   xc_build_vote_filter / xc_build_optimal_filter
 *                                  <- build_vote_filter / build_optimal_filter
 *                                     vote_filter.hpp:62-91
 *   xc_detect_pattern              <- detect_pattern vote_filter.hpp:146-168
 *   xc_filter_create               <- FreqFilter2  freq_filter.hpp:21-46 (the
 *                                     per-band filter spectra are built once
 *                                     per filter and pad size and cached)
 *   xc_decompose_rotation2/scale2  <- decompose_rotation2 / decompose_scale2
 *                                     freq_filter.hpp:63-129 (host, once per
 *                                     filter)
 *   xc_fft2                        <- fft2 fft.hpp:20-53 (the pipelines' own
 *                                     row / column transforms)
 *   xc_decompose_*_device          <- the same on the GPU (per-call builds:
 *                                     detect_pattern, contour matching)
 *   xc_render_component / xc_reconstruct / xc_inner_dc_value
 *                                  <- freq_filter.hpp:165-235 (host)
 *   3D rotation pipeline:
 *   xc_run3(mode = XC_CORRELATION) <- xcorr_fast_3d engine3d.hpp:270-302
 *   xc_run3(mode = XC_CONVOLUTION) <- xconv_fast_3d engine3d.hpp:306-335
 *   xc_filter3_create              <- SphFilter3   sph.hpp:130-157
 *   xc_decompose_rotation3         <- decompose_rotation3 sph.hpp:161-188 (host)
 *   xc_render_sph_component / xc_reconstruct3 / xc_sph_harm
 *                                  <- sph.hpp:37-47, 194-221 (host)
 *   xc_wigner_d                    <- wigner_d     wigner.hpp:64-88 (host)
 *   xc_white_noise                 <- white_noise  lic.hpp:9-17 (host; the
 *                                     seeded input of lic, lic.hpp:37-55)
 *
 * Conventions
 *   - Status codes: XC_OK; XC_EINVAL for the reference's std::invalid_argument
 *     (the message text is the reference's, readable with xc_last_error);
 *     >= 10 for CUDA / allocation / NCCL failures.  A context that cannot
 *     reach a CUDA device fails loudly at xc_context_create: there is no CPU
 *     fallback.
 *   - Grids: `layout` XC_COL_MAJOR is Eigen's default storage used by the
 *     reference (values(y,x) at y + x*height, field.hpp:15); XC_ROW_MAJOR is
 *     [y][x].  Complex data is interleaved (re, im).
 *   - FreqFilter2 comps are passed column-major like the reference's Eigen
 *     CGrid (n_rows x nc, element (row, ci) at row + ci*n_rows), n_rows =
 *     n_radii for rotation2 and n_angles for scale2.
 *   - The caller owns all buffers passed in.  With memory == XC_HOST, host
 *     buffers (pinned or pageable) are copied in and out inside the call; with
 *     XC_DEVICE the pointers are device pointers on the context's device.
 *     Calls are synchronous with respect to the host.
 *   - One context per host thread, or external locking.
 */
#ifndef XCONV_B200_H
#define XCONV_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define XC_ABI_VERSION 2 /* 2: xc_stats::band_mode */

enum xc_status {
  XC_OK = 0,
  XC_EINVAL = 2,      /* std::invalid_argument in the reference */
  XC_ECUDA = 10,
  XC_ENOMEM = 11,
  XC_ENCCL = 12,
  XC_EINTERNAL = 13
};

enum xc_group { XC_ROTATION2 = 0, XC_SCALE2 = 1, XC_ROTATION3 = 2 }; /* field.hpp:129 */
enum xc_mode { XC_CORRELATION = 0, XC_CONVOLUTION = 1 };            /* engine.hpp:10 */
enum xc_dtype { XC_F32 = 0, XC_F64 = 1, XC_C64 = 2, XC_C128 = 3 };
enum xc_layout { XC_ROW_MAJOR = 0, XC_COL_MAJOR = 1 };
enum xc_memory { XC_HOST = 0, XC_DEVICE = 1 };

/* xc_run flags */
#define XC_FLAG_PERIODIC 1u      /* XConvPlan::periodic, engine.hpp:20 */
#define XC_FLAG_NO_INNER_DC 2u   /* omit the scale inner-DC term (engine.hpp:320-324,
                                    369-371): set on all but one rank when bands
                                    are sharded across GPUs */
#define XC_FLAG_ACCUMULATE 4u    /* out += result (device memory only) */
#define XC_FLAG_ASYNC 8u         /* device memory only.  Rank contexts: return once
                                    this rank's bands are computed, with the reduce
                                    (and rank 0's write of `out`) queued on an
                                    internal stream that overlaps the next call.
                                    Single-device contexts, rotation group: return
                                    with the kernels queued on the context's stream
                                    (no host sync; the call can be captured in a
                                    CUDA graph).  xc_context_synchronize waits. */

typedef struct xc_context_s* xc_context;
typedef struct xc_filter_s* xc_filter;

/* Image batch descriptor: `batch` images of height x width, contiguous. */
typedef struct {
  int height, width, batch;
  int signal_dtype; /* XC_F32 / XC_F64 (real) or XC_C64 / XC_C128 (complex) */
  int param_dtype;  /* XC_F32 or XC_F64: angle (rotation2) or scale (scale2) */
  int out_dtype;    /* XC_C64 / XC_C128 for xc_run; XC_F32 / XC_F64 for xc_smooth */
  int layout;       /* XC_ROW_MAJOR or XC_COL_MAJOR */
  int memory;       /* XC_HOST or XC_DEVICE, for every data pointer of the call */
  int param_per_image; /* 1: param has `batch` planes; 0: one plane shared */
  int xform_kind;   /* XformField::kind (field.hpp:129): what param holds --
                       XC_ROTATION2 angles or XC_SCALE2 scale factors */
} xc_image_desc;

/* Response2 counters and StageTimer keys (engine.hpp:23-29, 41-49). */
typedef struct {
  long long standard_ops;  /* bands executed (engine.hpp:318, 367; smooth: num+den) */
  int clamped_pixels;      /* SmoothResult::clamped_pixels, engine.hpp:381 */
  int pad_h, pad_w;        /* transform size used */
  double seconds_render, seconds_fft, seconds_combine, seconds_premultiply;
  double seconds_h2d, seconds_d2h, seconds_total;
  int gpu_launches;        /* kernels launched by this call */
  int bands_run;           /* bands transformed per image (the Hermitian half-band
                              mode transforms k >= 0 only; summed over devices) */
  int band_mode;           /* 0: every band transformed; 1: Hermitian half-band (real
                              signal, F_{-k} = conj F_k); 2: conjugate band pairs of the
                              scatter (real signal, any filter: bands k >= 0 transformed,
                              each fed into the F_k and the conj(f_{-k}) sums) */
} xc_stats;

int xc_abi_version(void);

/* ---- contexts ---------------------------------------------------------- */
int xc_context_create(int device, xc_context* out);

/* Multi-GPU contexts (the band loop of engine.hpp:300-319 /
 * 345-368 split across devices).  xc_run and xc_smooth on such a context split
 * the bands into contiguous ranges (balanced to +-1), run one range per
 * device and sum the partial outputs onto the first device with one NCCL
 * reduce (smooth: numerator and denominator, divided on the root).  The scale
 * group's inner-DC term is added once.  Other entry points run on the first
 * device.  Pointers with memory == XC_DEVICE live on the first device.
 *
 * xc_context_create_multi: one process, n_dev devices (ncclCommInitAll).  A
 *   device listed twice (or XCB_REDUCE=peer) reduces with peer copies and an
 *   ordered device-side sum instead of NCCL.
 * xc_context_create_rank: one process per GPU; all ranks call xc_run /
 *   xc_smooth with the same arguments and their own inputs, rank 0's `out`
 *   receives the result (ncclCommInitRank; the 128-byte id comes from
 *   xc_nccl_unique_id on one rank, shared by the caller). */
enum xc_shard { XC_SHARD_BANDS = 0, XC_SHARD_BATCH = 1 };
int xc_nccl_unique_id(void* id128);
int xc_context_create_multi(int n_dev, const int* dev_ids, xc_context* out);
int xc_context_create_rank(int device, const void* nccl_id128, int rank, int nranks,
                           xc_context* out);
/* XC_SHARD_BANDS (default; reduce) or XC_SHARD_BATCH (images split across the
 * devices of a create_multi context, no collective). */
int xc_context_set_sharding(xc_context ctx, int shard);
/* wait for every stream of the context (XC_FLAG_ASYNC reduces included) */
int xc_context_synchronize(xc_context ctx);
/* devices (or ranks) of a context and whether its reduce is NCCL */
int xc_context_devices(xc_context ctx, int* n_dev, int* uses_nccl);
void xc_context_destroy(xc_context ctx);
/* Message of the last failed call on this context (or thread if ctx NULL). */
const char* xc_last_error(xc_context ctx);
/* Launch on a caller-owned cudaStream_t (NULL restores the internal stream). */
int xc_context_set_stream(xc_context ctx, void* cuda_stream);
/* Release cached device scratch (filter spectra stay with their filters). */
int xc_context_trim(xc_context ctx);

/* Per-stage device-time profile (CUDA events on the launch stream around each
 * pipeline stage; reference: StageTimer, engine.hpp:41-49).  xc_profile_get
 * returns the number of stages recorded and fills entry idx if it exists. */
int xc_profile_enable(xc_context ctx, int on);
int xc_profile_reset(xc_context ctx);
int xc_profile_get(xc_context ctx, int idx, char* name, int name_len, double* total_ms,
                   long long* launches);

/* fft2 (fft.hpp:20-53) on the device with the pipeline's own transforms: the
 * 2D DFT of a rows x cols complex grid (XC_C64 / XC_C128, row-major, host or
 * device memory), forward unscaled, inverse scaled 1/(rows cols).  One extent
 * must be even (the engine pairs rows / columns); lengths must be 2,3,5-smooth
 * and <= 32768, as for the pipelines' pads. */
int xc_fft2(xc_context ctx, int rows, int cols, int dtype, int memory, int inverse,
            const void* in, void* out);

/* Out-of-bounds debug mode (no compute-sanitizer on the GPU pool).  With the
 * environment variable XCB_GUARD=<bytes> set before the first allocation, every
 * context buffer gets a guard zone of that size on each side and the whole
 * allocation is poisoned with 0xFF bytes (NaN in fp32 / fp64).
 * xc_debug_check_guards synchronizes the device and counts the guard zones
 * that changed (*n_bad; the first one's buffer name in first_bad); a stray or
 * uninitialised read surfaces as NaN in the result.  xc_debug_guard_bytes
 * returns the active guard size (0 = off). */
int xc_debug_check_guards(xc_context ctx, int* n_bad, char* first_bad, int len);
int xc_debug_guard_bytes(void);

/* The transform length the 2D pipelines pick for an axis that needs at least n
 * points (extent + R; fft.hpp:85-86 takes next_fast_size(extent + 2R + 1), any
 * length >= extent + R filters identically): host logic, no GPU needed.
 * xc_debug_tile_count: the number of halo tiles along an image axis of `extent`
 * points with render radius R (1 = not tiled; rotation group, DESIGN 5). */
int xc_debug_pick_pad(int n);
int xc_debug_tile_count(int extent, int R);

/* ---- filters (FreqFilter2) -------------------------------------------- */
/* Filters are host objects (ctx may be NULL); device spectra are built on first
 * use per (device, pad size, layout) and freed by xc_filter_destroy.  Errors of
 * filter-only calls are reported by xc_last_error(NULL). */
int xc_filter_create(xc_context ctx, int group, int K, const int* ks, int nc,
                     const double* comps, int n_radii, int n_angles, double r_max,
                     double r_min, double r_domain, xc_filter* out);
void xc_filter_destroy(xc_filter f);
int xc_filter_num_components(xc_filter f);

/* ---- host-side decomposition / synthesis (once per filter) ------------ */
/* filter image: height x width complex<double> in `layout`.  Outputs: ks
 * (2*(K/2)+1 ints), comps column-major (n_rows x nc) complex<double>. */
int xc_decompose_rotation2(const double* filt, int height, int width, int layout,
                           double cx, double cy, int K, int n_radii, int n_angles,
                           double r_max, int* ks_out, double* comps_out, int* nc_out);
int xc_decompose_scale2(const double* filt, int height, int width, int layout,
                        double cx, double cy, int K, int n_radii, int n_angles,
                        double r_min, double r_max, double r_domain, int* ks_out,
                        double* comps_out, int* nc_out);
/* The same decompositions computed on the context's device (per-call filter
 * builds; freq_filter.hpp:63-129): polar / log-polar bilinear
 * resampling and the band DFT as two kernels, fp64; identical validation and
 * error texts, outputs in host memory as above. */
int xc_decompose_rotation2_device(xc_context ctx, const double* filt, int height, int width,
                                  int layout, double cx, double cy, int K, int n_radii,
                                  int n_angles, double r_max, int* ks_out, double* comps_out,
                                  int* nc_out);
int xc_decompose_scale2_device(xc_context ctx, const double* filt, int height, int width,
                               int layout, double cx, double cy, int K, int n_radii,
                               int n_angles, double r_min, double r_max, double r_domain,
                               int* ks_out, double* comps_out, int* nc_out);
int xc_render_component(xc_filter f, int ci, int width, int height, double cx,
                        double cy, int layout, double* out);
int xc_reconstruct(xc_filter f, int width, int height, double cx, double cy,
                   const int* subset, int nsub, int layout, double* out);
int xc_inner_dc_value(xc_filter f, double* out2);

/* ---- the hot path ------------------------------------------------------ */
/* xcorr_fast / xconv_fast.  components: XConvPlan::components (NULL/0 = all
 * retained bands, in the filter's ascending order). */
int xc_run(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d,
           const void* signal, const void* param, const int* components,
           int n_components, unsigned flags, void* out, xc_stats* stats);

/* smooth_adaptive: out is real (d->out_dtype XC_F32 or XC_F64). */
int xc_smooth(xc_context ctx, xc_filter f, const xc_image_desc* d,
              const void* signal, const void* param, int normalize_signal,
              void* out, xc_stats* stats);

/* Rotation-invariant matching score: for every pixel,
 * score = max over s < n_angles of |sum_k e^{-i k 2 pi s / n_angles} G_k(p)|,
 * G_k = H (*) F_k the per-band correlations of xcorr_fast; argmax = first s
 * attaining the max (int32).  d->out_dtype selects the score type (XC_F32 /
 * XC_F64).  argmax may be NULL. */
int xc_anglemax(xc_context ctx, xc_filter f, const xc_image_desc* d,
                const void* signal, const int* components, int n_components,
                int n_angles, void* score, int* argmax, xc_stats* stats);

/* find_peaks (vote_filter.hpp:107-134) on a real response (host memory). */
int xc_find_peaks(const void* resp, int dtype, int height, int width, int layout,
                  double radius, double threshold_frac, int* xs, int* ys,
                  double* values, int max_peaks, int* n_found);

/* find_peaks on a response in device memory (same result as xc_find_peaks):
 * the NMS runs on the GPU, the sort on the host; outputs in host memory. */
int xc_find_peaks_device(xc_context ctx, const void* resp, int dtype, int height, int width,
                         int layout, double radius, double threshold_frac, int* xs, int* ys,
                         double* values, int max_peaks, int* n_found);

/* ---- pattern detection (vote_filter.hpp) ------------- */
/* build_vote_filter / build_optimal_filter (vote_filter.hpp:62-91): real
 * height x width grids in `layout`; weights_out receives (2R+1)^2 doubles in
 * the same layout, R = ceil(eps) in *radius_out. */
int xc_build_vote_filter(const double* weight, const double* frame, int height, int width,
                         int layout, double px, double py, double eps, int nearest,
                         double* weights_out, int* radius_out);
int xc_build_optimal_filter(const double* pattern, int height, int width, int layout,
                            double px, double py, double eps, int nearest,
                            double* weights_out, int* radius_out);
/* detect_pattern (vote_filter.hpp:146-168): one real image (d->signal_dtype
 * XC_F32 / XC_F64, d->batch 1), vote weights (2R+1)^2 in d->layout, K bands
 * (n_radii / n_angles 0 = the reference defaults).  response: real
 * (d->out_dtype) Re(xconv_fast(|grad I|, rotation(dir grad I), F)); peaks: NMS
 * within eps/2 at 0.5 of the max, sorted (value desc, y, x), up to max_peaks
 * written, *n_peaks = number found. */
int xc_detect_pattern(xc_context ctx, const xc_image_desc* d, const void* image,
                      const double* vote_weights, int radius, double eps, int K, int n_radii,
                      int n_angles, void* response, int* peak_x, int* peak_y, double* peak_v,
                      int max_peaks, int* n_peaks, xc_stats* stats);

/* ------------------------------------------------------------------ 3D rotation
 * Volumes are x fastest: element (x, y, z) at (z*ny + y)*nx + x (Field3,
 * field.hpp:67-85).  Quaternion fields are 4 doubles (w, x, y, z) per voxel;
 * non-unit quaternions are renormalized (XformField::rotation3d).  SphFilter3
 * coefficients are column-major like the reference's Eigen CGrid (n_radii x
 * (K+1)^2, element (shell, l(l+1)+m) at shell + (l(l+1)+m)*n_radii). */
typedef struct xc_filter3_s* xc_filter3;

int xc_filter3_create(int K, int n_radii, double r_max, const double* coeffs, xc_filter3* out);
void xc_filter3_destroy(xc_filter3 f);
/* sph.hpp:161-188; coeffs_out: n_radii * (K+1)^2 complex, column-major.
 * n_theta / n_phi = 0 select 2(K+1). */
int xc_decompose_rotation3(const double* volume, int nx, int ny, int nz, double cx, double cy,
                           double cz, int K, int n_radii, double r_max, int n_theta, int n_phi,
                           double* coeffs_out);
/* f_l^{m_radial}(r) Y_l^{m_angular} on an nx*ny*nz grid (sph.hpp:194-212) */
int xc_render_sph_component(xc_filter3 f, int l, int m_radial, int m_angular, int nx, int ny,
                            int nz, double cx, double cy, double cz, double* out);
/* sph.hpp:215-221; degrees == NULL (or ndeg < 0) keeps every degree */
int xc_reconstruct3(xc_filter3 f, int nx, int ny, int nz, double cx, double cy, double cz,
                    const int* degrees, int ndeg, double* out);
int xc_sph_harm(int l, int m, double theta, double phi, double* out2);
/* D[(m_to + l)(2l+1) + (m_from + l)], (2l+1)^2 complex (wigner.hpp:64-88) */
int xc_wigner_d(int l, const double* quat, double* out);

/* ---- line integral convolution input (lic.hpp) ------- */
/* white_noise (lic.hpp:9-17): std::mt19937_64(seed), value (rng() >> 11) *
 * 2^-53 per pixel in y-major order (y outer, x inner); height x width
 * doubles written in `layout`.  Host only: no device needed. */
int xc_white_noise(unsigned long long seed, int height, int width, int layout, double* out);
/* xcorr_fast_3d / xconv_fast_3d: signal (signal_dtype XC_F32 / XC_F64 /
 * XC_C64 / XC_C128), quats and out (complex128) in `memory`; degrees selects a
 * subset of l (XConvPlan::components over degrees, engine3d.hpp:11-16);
 * stats->standard_ops = sum over the kept degrees of (2l+1)^2. */
int xc_run3(xc_context ctx, xc_filter3 f, int mode, int nx, int ny, int nz, const void* signal,
            int signal_dtype, const double* quats, const int* degrees, int ndeg, int memory,
            double* out, xc_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* XCONV_B200_H */
