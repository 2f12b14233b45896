// Device stages of the 3D rotation pipeline (k_3d.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

namespace xcb {

struct Geo3 {
  int nx, ny, nz;  // signal extent (x fastest)
  int px, py, pz;  // transform size
  int R;           // render radius ceil(r_max)
};

// One band (l, m, m'): the Wigner entry D^l_{m' m} = e^{-i(m' alpha + m gamma)}
// d^l_{m' m}(beta), d from host_sph.h SmallD (Horner coefficients c[0..n]).
struct Band3 {
  int l, m, mp;
  int n, pc_end, ps0;
  double c[33];
};

// signal (XC_F32 / XC_F64 / XC_C64 / XC_C128) -> complex fp32
void launch3_signal(const void* src, int dtype, size_t n, float2* dst, cudaStream_t st,
                    LaunchCounter& lc);
void launch3_euler(const double* quats, size_t n, double4* eul, cudaStream_t st,
                   LaunchCounter& lc);
// in-place forward line transforms along axis (0 x, 1 y, 2 z) of nvol volumes
void launch3_pass(const FftPlan& pl, const Geo3& g, int axis, float2* buf, size_t vstride,
                  int nvol, cudaStream_t st, LaunchCounter& lc);
// x-pass of the (zero-padded) signal, times D_b when premul, for nb bands
void launch3_x_signal(const FftPlan& pl, const Geo3& g, const float2* sig, const double4* eul,
                      const Band3* bands, int nb, int premul, float2* work, size_t vstride,
                      cudaStream_t st, LaunchCounter& lc);
// x-pass of nb rendered filter bands ((2R+1)^3 each), wrapped to the origin
void launch3_x_filter(const FftPlan& pl, const Geo3& g, const float2* comps, int nb,
                      float2* spec, size_t vstride, cudaStream_t st, LaunchCounter& lc);
// z-pass loading conj(H^) V^_sidx[b] (mode 0, nb bands) or conj(H^) (mode 1)
void launch3_z_load(const FftPlan& pl, const Geo3& g, const float2* Hh, const float2* spec,
                    const int* sidx, int nb, size_t vstride, int mode, float2* work,
                    cudaStream_t st, LaunchCounter& lc);
// x-pass finishing an inverse, crop; mode 0: per-band planes part_b =
// conj(D_b) G_b for nb bands; mode 1: out (+)= G (one volume)
void launch3_x_out(const FftPlan& pl, const Geo3& g, const float2* work, size_t vstride, int nb,
                   const double4* eul, const Band3* bands, int mode, float2* part,
                   int accumulate, double2* out, cudaStream_t st, LaunchCounter& lc);
// out (+)= sum of nb planes of n voxels (band order)
void launch3_reduce_parts(const float2* part, int nb, size_t n, int accumulate, double2* out,
                          cudaStream_t st, LaunchCounter& lc);
// sum += sum_b work_b V^_sidx[b] over nb transformed scatter bands of P points
void launch3_mac(const float2* work, int nb, size_t P, const float2* spec, const int* sidx,
                 float2* sum, cudaStream_t st, LaunchCounter& lc);
// dynamic shared memory of a 16-line tile CTA for line length L
size_t tile3_smem(int L);

}  // namespace xcb
