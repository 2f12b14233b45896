// 3D rotation pipeline on the GPU (engine3d.hpp:267-335).
//
// Bands are the (l, m, m') triples of the SH decomposition, sum (2l+1)^2 of
// them.  Volumes are x fastest, index (z*py + y)*px + x for padded
// (px, py, pz) volumes.  Every 3D FFT is three passes of line transforms
// (k3_* below), each CTA transforming a pair of lines in shared memory with
// the runtime-planned Stockham engine of fft_core.cuh.  Inverse transforms
// are conj(FFT(conj(.)))/P with the conjugations folded into the first load
// and the last store.
//   gather  : H^ = FFT3(H) once; per band z-pass of conj(H^) V^_b (the
//             spectral multiply fused into the load), y-pass, then an x-pass
//             that crops and accumulates conj(D^l_{m' m}(voxel)) G_b into a
//             shared-memory line accumulator across the bands of a chunk
//   scatter : per band x-pass of H D_b(voxel) (premultiply fused into the
//             load), y-pass, z-pass whose store accumulates FFT3(H D_b) V^_b
//             into one spectrum; one inverse 3D FFT at the end (the
//             reference's per-band inverse FFTs collapse into one)
// The per-voxel Wigner entry D = e^{-i(m' alpha + m gamma)} d^l_{m' m}(beta)
// is evaluated in fp64 from the voxel's (alpha, gamma, cos beta/2, sin beta/2)
// with the band's Horner coefficients (host_sph.h SmallD).
#include "kernels3d.h"
#include "stages_common.cuh"

namespace xcb {
namespace {

// ---------------------------------------------------------------- per voxel

// XformField::rotation3d normalization (field.hpp:168-171) + euler_zyz
// (wigner.hpp:40-57) -> (alpha, gamma, cos(beta/2), sin(beta/2))
__global__ void k3_euler(const double4* __restrict__ q, size_t n, double4* __restrict__ e) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    double4 v = q[i];  // (w, x, y, z)
    const double nr = sqrt(v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w);
    if (fabs(nr - 1.0) > 1e-12) {
      v.x /= nr;
      v.y /= nr;
      v.z /= nr;
      v.w /= nr;
    }
    const double w = v.x, x = v.y, y = v.z, z = v.w;
    const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w, txx = tx * x, txy = ty * x,
                 txz = tz * x, tyy = ty * y, tyz = tz * y, tzz = tz * z;
    const double M00 = 1 - (tyy + tzz), M02 = txz + twy, M10 = txy + twz, M12 = tyz - twx,
                 M20 = txz - twy, M21 = tyz + twx, M22 = 1 - (txx + tyy);
    const double sb = sqrt(M02 * M02 + M12 * M12);
    const double beta = atan2(sb, M22);
    double alpha, gamma;
    if (sb > 1e-12) {
      alpha = atan2(M12, M02);
      gamma = atan2(M21, -M20);
    } else {
      alpha = atan2(M10, M00);
      if (M22 < 0) alpha = -alpha;
      gamma = 0;
    }
    double s, c;
    sincos(0.5 * beta, &s, &c);
    e[i] = make_double4(alpha, gamma, c, s);
  }
}

// signal of any dtype (0 f32, 1 f64, 2 c64, 3 c128) -> complex fp32
__global__ void k3_to_c64(const void* __restrict__ src, int dtype, size_t n,
                          float2* __restrict__ dst) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    float2 v;
    if (dtype == 0) v = make_float2(static_cast<const float*>(src)[i], 0.f);
    else if (dtype == 1) v = make_float2(float(static_cast<const double*>(src)[i]), 0.f);
    else if (dtype == 2) v = static_cast<const float2*>(src)[i];
    else {
      const double2 d = static_cast<const double2*>(src)[i];
      v = make_float2(float(d.x), float(d.y));
    }
    dst[i] = v;
  }
}

// D^l_{m' m} (sign = -1) or its conjugate (sign = +1) at a voxel
__device__ __forceinline__ float2 wigner_at(const Band3& b, const double4& e, float sign) {
  if (b.n < 0) return make_float2(0.f, 0.f);
  const double u = e.z * e.z, v = e.w * e.w;
  double acc = b.c[0], vk = 1;
  for (int k = 1; k <= b.n; ++k) {
    vk *= v;
    acc = fma(acc, u, b.c[k] * vk);
  }
  for (int i = 0; i < b.pc_end; ++i) acc *= e.z;
  for (int i = 0; i < b.ps0; ++i) acc *= e.w;
  const double ph = double(b.mp) * e.x + double(b.m) * e.y;
  const double q = rint(ph * kInvTwoPi);
  double r = fma(-q, kTwoPiHi, ph);
  r = fma(-q, kTwoPiLo, r);
  float sn, cs;
  sincosf(float(r), &sn, &cs);
  const float d = float(acc);
  return make_float2(d * cs, sign * d * sn);
}

// ---------------------------------------------------------------- line geometry
// line li of axis a in a (px, py, pz) volume: element n at base + n * stride
struct Lines {
  int px, py, pz, axis;
  __device__ __forceinline__ int count() const {
    return axis == 0 ? py * pz : axis == 1 ? px * pz : px * py;
  }
  __device__ __forceinline__ size_t base(int li) const {
    if (axis == 0) return size_t(li) * px;
    if (axis == 1) return size_t(li % px) + size_t(li / px) * px * py;
    return size_t(li);
  }
  __device__ __forceinline__ size_t stride() const {
    return axis == 0 ? 1 : axis == 1 ? size_t(px) : size_t(px) * py;
  }
};

// plain in-place forward pass along `axis` of nb volumes (grid.y = volume)
__global__ void __launch_bounds__(kMaxThreads)
    k3_pass(FftPlanD p, Lines ln, float2* __restrict__ buf, size_t vstride) {
  extern __shared__ float2 sm[];
  float2* v = buf + blockIdx.y * vstride;
  const int li0 = 2 * blockIdx.x, nl = ln.count();
  const size_t st = ln.stride();
  const size_t b0 = ln.base(li0), b1 = li0 + 1 < nl ? ln.base(li0 + 1) : b0;
  auto load = [&](int n, int g) -> float2 { return v[(g ? b1 : b0) + n * st]; };
  auto store = [&](int k, int g, float2 x) {
    if (g == 0 || li0 + 1 < nl) v[(g ? b1 : b0) + k * st] = x;
  };
  fft_block(p, sm, load, store);
}

// x-pass from the signal (zero-padded), optionally times D_b(voxel) (the
// scatter premultiply, engine3d.hpp:317-321); grid.y = band of the chunk
__global__ void __launch_bounds__(kMaxThreads)
    k3_x_signal(FftPlanD p, Geo3 g, const float2* __restrict__ sig,
                const double4* __restrict__ eul, const Band3* __restrict__ bands, int premul,
                float2* __restrict__ work, size_t vstride) {
  extern __shared__ float2 sm[];
  const Band3& b = bands[blockIdx.y];
  float2* v = work + blockIdx.y * vstride;
  const int li0 = 2 * blockIdx.x, nl = g.py * g.pz;
  auto load = [&](int n, int gi) -> float2 {
    const int li = li0 + gi, y = li % g.py, z = li / g.py;
    if (li >= nl || n >= g.nx || y >= g.ny || z >= g.nz) return make_float2(0.f, 0.f);
    const size_t i = (size_t(z) * g.ny + y) * g.nx + n;
    float2 h = sig[i];
    if (premul) h = c_mul(h, wigner_at(b, eul[i], -1.f));
    return h;
  };
  auto store = [&](int k, int gi, float2 x) {
    if (li0 + gi < nl) v[size_t(li0 + gi) * g.px + k] = x;
  };
  fft_block(p, sm, load, store);
}

// x-pass of the filter bands: rendered (2R+1)^3 components wrapped to the
// origin (fft.hpp:186-194); grid.y = band
__global__ void __launch_bounds__(kMaxThreads)
    k3_x_filter(FftPlanD p, Geo3 g, const float2* __restrict__ comps, float2* __restrict__ spec,
                size_t vstride) {
  extern __shared__ float2 sm[];
  const int S = 2 * g.R + 1;
  const float2* f = comps + size_t(blockIdx.y) * S * S * S;
  float2* v = spec + blockIdx.y * vstride;
  const int li0 = 2 * blockIdx.x, nl = g.py * g.pz;
  auto src = [&](int n, int P) { int s = n + g.R; return s >= P ? s - P : s; };
  auto load = [&](int n, int gi) -> float2 {
    const int li = li0 + gi;
    if (li >= nl) return make_float2(0.f, 0.f);
    const int x = src(n, g.px), y = src(li % g.py, g.py), z = src(li / g.py, g.pz);
    if (x >= S || y >= S || z >= S) return make_float2(0.f, 0.f);
    return f[(size_t(z) * S + y) * S + x];
  };
  auto store = [&](int k, int gi, float2 x) {
    if (li0 + gi < nl) v[size_t(li0 + gi) * g.px + k] = x;
  };
  fft_block(p, sm, load, store);
}

// gather z-pass: conj(H^) V^_b (conj of the correlation product H^ conj(V^),
// fft.hpp:195-197) -> work_b; grid.y = band of the chunk.  mode 1 instead
// loads conj(src) of one volume (the scatter's final inverse).
__global__ void __launch_bounds__(kMaxThreads)
    k3_z_load(FftPlanD p, Geo3 g, const float2* __restrict__ Hh, const float2* __restrict__ spec,
              const int* __restrict__ sidx, size_t vstride, int mode, float2* __restrict__ work) {
  extern __shared__ float2 sm[];
  const int li0 = 2 * blockIdx.x, nl = g.px * g.py;
  const size_t st = size_t(g.px) * g.py;
  const float2* V = mode == 0 ? spec + size_t(sidx[blockIdx.y]) * vstride : nullptr;
  float2* w = work + blockIdx.y * vstride;
  auto load = [&](int n, int gi) -> float2 {
    const int li = li0 + gi;
    if (li >= nl) return make_float2(0.f, 0.f);
    const size_t i = size_t(li) + n * st;
    return mode == 0 ? c_mul(c_conj(Hh[i]), V[i]) : c_conj(Hh[i]);
  };
  auto store = [&](int k, int gi, float2 x) {
    if (li0 + gi < nl) w[size_t(li0 + gi) + k * st] = x;
  };
  fft_block(p, sm, load, store);
}

// gather x-pass: per band of the chunk, row transform of work_b, crop, steer
// with conj(D_b) and accumulate in shared memory; out (+)= the sum
// (engine3d.hpp:290-298).  mode 1: one volume, no steering (the scatter's
// final inverse).  The inverse is conj(Y) / P.
__global__ void __launch_bounds__(kMaxThreads)
    k3_x_steer(FftPlanD p, Geo3 g, const float2* __restrict__ work, size_t vstride, int nb,
               const double4* __restrict__ eul, const Band3* __restrict__ bands, int mode,
               float inv_p, int accumulate, double2* __restrict__ out) {
  extern __shared__ float2 sm[];
  float2* acc = sm + 2 * kG * p.Lp;  // [2][nx]
  const int li0 = 2 * blockIdx.x, nl = g.ny * g.nz;
  for (int i = threadIdx.x; i < 2 * g.nx; i += blockDim.x) acc[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int bi = 0; bi < nb; ++bi) {
    const float2* w = work + bi * vstride;
    const Band3& b = bands[bi];
    auto load = [&](int n, int gi) -> float2 {
      const int li = li0 + gi;
      if (li >= nl) return make_float2(0.f, 0.f);
      const int y = li % g.ny, z = li / g.ny;
      return w[(size_t(z) * g.py + y) * g.px + n];
    };
    auto store = [&](int k, int gi, float2 x) {
      const int li = li0 + gi;
      if (k >= g.nx || li >= nl) return;
      float2 v = c_scale(c_conj(x), inv_p);
      if (mode == 0) {
        const size_t vi = size_t(li) * g.nx + k;  // (z*ny + y)*nx + x
        v = c_mul(wigner_at(b, eul[vi], 1.f), v);
      }
      acc[gi * g.nx + k] = c_add(acc[gi * g.nx + k], v);
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < 2 * g.nx; i += blockDim.x) {
    const int li = li0 + i / g.nx;
    if (li >= nl) continue;
    const size_t o = size_t(li) * g.nx + i % g.nx;
    double2 v = make_double2(acc[i].x, acc[i].y);
    if (accumulate) {
      v.x += out[o].x;
      v.y += out[o].y;
    }
    out[o] = v;
  }
}

// scatter z-pass: per band of the chunk, column transform of work_b, then
// sum += FFT3(H D_b) V^_b (fft.hpp:195-197 with the band sum in frequency)
__global__ void __launch_bounds__(kMaxThreads)
    k3_z_mac(FftPlanD p, Geo3 g, const float2* __restrict__ work, size_t vstride, int nb,
             const float2* __restrict__ spec, const int* __restrict__ sidx,
             float2* __restrict__ sum) {
  extern __shared__ float2 sm[];
  const int li0 = 2 * blockIdx.x, nl = g.px * g.py;
  const size_t st = size_t(g.px) * g.py;
  for (int bi = 0; bi < nb; ++bi) {
    const float2* w = work + bi * vstride;
    const float2* V = spec + size_t(sidx[bi]) * vstride;
    auto load = [&](int n, int gi) -> float2 {
      const int li = li0 + gi;
      return li < nl ? w[size_t(li) + n * st] : make_float2(0.f, 0.f);
    };
    auto store = [&](int k, int gi, float2 x) {
      const int li = li0 + gi;
      if (li >= nl) return;
      const size_t i = size_t(li) + k * st;
      sum[i] = c_add(sum[i], c_mul(x, V[i]));
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
}

template <class K>
void smem_attr(K k, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

unsigned pairs(long long lines) { return unsigned((lines + 1) / 2); }

}  // namespace

void launch3_signal(const void* src, int dtype, size_t n, float2* dst, cudaStream_t st,
                    LaunchCounter& lc) {
  k3_to_c64<<<grid_for(n, 256), 256, 0, st>>>(src, dtype, n, dst);
  ++lc.n;
}

void launch3_euler(const double* quats, size_t n, double4* eul, cudaStream_t st,
                   LaunchCounter& lc) {
  k3_euler<<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const double4*>(quats), n, eul);
  ++lc.n;
}

void launch3_pass(const FftPlan& pl, const Geo3& g, int axis, float2* buf, size_t vstride,
                  int nvol, cudaStream_t st, LaunchCounter& lc) {
  const Lines ln{g.px, g.py, g.pz, axis};
  const long long nl = axis == 0 ? 1LL * g.py * g.pz : axis == 1 ? 1LL * g.px * g.pz
                                                                  : 1LL * g.px * g.py;
  smem_attr(k3_pass, pl.smem_bytes());
  k3_pass<<<dim3(pairs(nl), nvol), pl.d.nt, pl.smem_bytes(), st>>>(pl.d, ln, buf, vstride);
  ++lc.n;
}

void launch3_x_signal(const FftPlan& pl, const Geo3& g, const float2* sig, const double4* eul,
                      const Band3* bands, int nb, int premul, float2* work, size_t vstride,
                      cudaStream_t st, LaunchCounter& lc) {
  smem_attr(k3_x_signal, pl.smem_bytes());
  k3_x_signal<<<dim3(pairs(1LL * g.py * g.pz), nb), pl.d.nt, pl.smem_bytes(), st>>>(
      pl.d, g, sig, eul, bands, premul, work, vstride);
  ++lc.n;
}

void launch3_x_filter(const FftPlan& pl, const Geo3& g, const float2* comps, int nb,
                      float2* spec, size_t vstride, cudaStream_t st, LaunchCounter& lc) {
  smem_attr(k3_x_filter, pl.smem_bytes());
  k3_x_filter<<<dim3(pairs(1LL * g.py * g.pz), nb), pl.d.nt, pl.smem_bytes(), st>>>(
      pl.d, g, comps, spec, vstride);
  ++lc.n;
}

void launch3_z_load(const FftPlan& pl, const Geo3& g, const float2* Hh, const float2* spec,
                    const int* sidx, int nb, size_t vstride, int mode, float2* work,
                    cudaStream_t st, LaunchCounter& lc) {
  smem_attr(k3_z_load, pl.smem_bytes());
  k3_z_load<<<dim3(pairs(1LL * g.px * g.py), nb), pl.d.nt, pl.smem_bytes(), st>>>(
      pl.d, g, Hh, spec, sidx, vstride, mode, work);
  ++lc.n;
}

void launch3_x_steer(const FftPlan& pl, const Geo3& g, const float2* work, size_t vstride,
                     int nb, const double4* eul, const Band3* bands, int mode, int accumulate,
                     double2* out, cudaStream_t st, LaunchCounter& lc) {
  const size_t smem = pl.smem_bytes() + 2 * size_t(g.nx) * sizeof(float2);
  smem_attr(k3_x_steer, smem);
  const float inv_p = float(1.0 / (double(g.px) * g.py * g.pz));
  k3_x_steer<<<pairs(1LL * g.ny * g.nz), pl.d.nt, smem, st>>>(pl.d, g, work, vstride, nb, eul,
                                                              bands, mode, inv_p, accumulate,
                                                              out);
  ++lc.n;
}

void launch3_z_mac(const FftPlan& pl, const Geo3& g, const float2* work, size_t vstride, int nb,
                   const float2* spec, const int* sidx, float2* sum, cudaStream_t st,
                   LaunchCounter& lc) {
  smem_attr(k3_z_mac, pl.smem_bytes());
  k3_z_mac<<<pairs(1LL * g.px * g.py), pl.d.nt, pl.smem_bytes(), st>>>(pl.d, g, work, vstride,
                                                                       nb, spec, sidx, sum);
  ++lc.n;
}

}  // namespace xcb
