// 3D rotation pipeline on the GPU (engine3d.hpp:267-335).
//
// Bands are the (l, m, m') triples of the SH decomposition, sum (2l+1)^2 of
// them.  Volumes are x fastest, index (z*py + y)*px + x for padded
// (px, py, pz) volumes.  Every 3D FFT is three passes of line transforms.
// A CTA transforms a tile of 16 lines held in shared memory as [line][n]
// with an odd row stride (conflict-free for the line-fast butterfly order),
// using the runtime-planned Stockham codelets of fft_core.cuh:
//   x tiles: 16 rows (contiguous lines), copied in and out n-fast
//   y / z tiles: 16 adjacent x at one (z) / (y), copied line-fast, so every
//   global access covers 128 contiguous bytes
// Grids are (tiles, bands of the chunk), so short lines still fill the GPU.
// Inverse transforms are conj(FFT(conj(.)))/P with the conjugations folded
// into the first load and the last store.
//   gather  : H^ = FFT3(H) once; per band a z-pass loading conj(H^) V^_b
//             (the spectral multiply fused into the load), a y-pass, and an
//             x-pass that crops and steers with conj(D^l_{m'm}(voxel)) into a
//             per-band plane; one reduction sums the planes (fixed order)
//   scatter : per band an x-pass of H D_b(voxel) (premultiply fused), y- and
//             z-passes, one multiply-accumulate kernel sum += FFT3(H D_b) V^_b
//             over the chunk; one inverse 3D FFT at the end (the reference's
//             per-band inverse FFTs collapse into one)
// The Wigner entry D = e^{-i(m' alpha + m gamma)} d^l_{m' m}(beta) is
// evaluated in fp64 from the voxel's (alpha, gamma, cos beta/2, sin beta/2)
// with the band's Horner coefficients (host_sph.h SmallD).
#include <algorithm>

#include "kernels3d.h"
#include "stages_common.cuh"

namespace xcb {
namespace {

constexpr int kTL = 16;    // lines per tile
constexpr int kT3 = 256;   // threads per tile CTA

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

// ---------------------------------------------------------------- tile FFT
// Row stride of a tile buffer: odd (mod 16), so 16 lanes on consecutive
// lines hit distinct bank pairs.
__host__ __device__ constexpr int tile_stride(int L) { return L % 2 ? L : L + 1; }

// Radices of the tile plans (make_fft_plan_maxr(L, 10)): a small dispatch set
// keeps the register demand low.  The tile kernels are bounded to 5 CTAs of
// 256 threads per SM (48 registers, ~150 B of spills): 64^3 xcorr 2.31 ->
// 2.08 ms against 64 registers (4 CTAs); 6 CTAs (40 registers) was slower.
template <class F>
__device__ __forceinline__ void radix_dispatch10(int R, F&& f) {
  switch (R) {
    case 2: f(IntC<2>{}); break;
    case 3: f(IntC<3>{}); break;
    case 4: f(IntC<4>{}); break;
    case 5: f(IntC<5>{}); break;
    case 6: f(IntC<6>{}); break;
    case 8: f(IntC<8>{}); break;
    case 9: f(IntC<9>{}); break;
    case 10: f(IntC<10>{}); break;
    default: break;
  }
}

// Forward transform of kTL sequences held in A ([line][Lp]); ping-pong with B.
// Returns the buffer holding the result.  Called by every thread; A must be
// complete (a barrier) on entry.
__device__ float2* tile_fft_rt(const FftPlanD& p, float2* A, float2* B, int Lp) {
  float2* src = A;
  float2* dst = B;
  for (int q = 0; q < p.npass; ++q) {
    radix_dispatch10(p.radix[q], [&](auto rc) {
      constexpr int R = decltype(rc)::value;
      const int nb = p.L / R, Ns = p.ns[q];
      const float2* tw = p.tw + p.tw_off[q];
      for (int w = threadIdx.x; w < kTL * nb; w += blockDim.x) {
        const int line = w % kTL, j = w / kTL;
        const int jm = q == 0 ? 0 : j - Ns * int(__umulhi(unsigned(j), p.magic[q]));
        const float2* s = src + line * Lp + j;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = s[r * nb];
        if (q > 0) {
#pragma unroll
          for (int r = 1; r < R; ++r) v[r] = c_mul(v[r], __ldg(tw + (r - 1) * Ns + jm));
        }
        Dft<R>::run(v);
        float2* d = dst + line * Lp + (j - jm) * R + jm;
#pragma unroll
        for (int r = 0; r < R; ++r) d[r * Ns] = v[Dft<R>::pos(r)];
      }
    });
    __syncthreads();
    float2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

// The same transform with the first pass reading through load(line, n) and
// the last pass writing through store(line, k, value) (global memory for the
// y / z tiles, where the line-fast order is coalesced): one barrier per pass
// boundary and no separate copy-in / copy-out.
template <class Ld, class St>
__device__ void tile_fft_io_rt(const FftPlanD& p, float2* A, float2* B, int Lp, Ld&& load,
                               St&& store) {
  if (p.npass == 0) {  // L == 1
    for (int line = threadIdx.x; line < kTL; line += blockDim.x) store(line, 0, load(line, 0));
    return;
  }
  float2* src = A;
  float2* dst = B;
  for (int q = 0; q < p.npass; ++q) {
    const bool first = q == 0, last = q == p.npass - 1;
    radix_dispatch10(p.radix[q], [&](auto rc) {
      constexpr int R = decltype(rc)::value;
      const int nb = p.L / R, Ns = p.ns[q];
      const float2* tw = p.tw + p.tw_off[q];
      for (int w = threadIdx.x; w < kTL * nb; w += blockDim.x) {
        const int line = w % kTL, j = w / kTL;
        const int jm = first ? 0 : j - Ns * int(__umulhi(unsigned(j), p.magic[q]));
        float2 v[R];
        if (first) {
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = load(line, j + r * nb);
        } else {
          const float2* s = src + line * Lp + j;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = s[r * nb];
#pragma unroll
          for (int r = 1; r < R; ++r) v[r] = c_mul(v[r], __ldg(tw + (r - 1) * Ns + jm));
        }
        Dft<R>::run(v);
        if (last) {  // Ns = L / R: output k = j + r nb
#pragma unroll
          for (int r = 0; r < R; ++r) store(line, j + r * nb, v[Dft<R>::pos(r)]);
        } else {
          float2* d = dst + line * Lp + (j - jm) * R + jm;
#pragma unroll
          for (int r = 0; r < R; ++r) d[r * Ns] = v[Dft<R>::pos(r)];
        }
      }
    });
    if (last) break;
    __syncthreads();
    float2* tmp = src;
    src = dst;
    dst = tmp;
  }
}

// ------------------------------------------------ compile-time tile plans
// The same Stockham passes with the plan's radices, lengths and strides as
// template constants, so index arithmetic folds into immediates and
// constant-divisor multiplies (the runtime plan above costs about 114 thread
// instructions per point per line transform at 72 points).  Used when the
// runtime plan equals one of CtPlan's instantiations (tile_dispatch).
struct NoIo {
  __device__ float2 operator()(int, int) const { return make_float2(0.f, 0.f); }
  __device__ void operator()(int, int, float2) const {}
};

// pass with radix R over sequences of length L, NS = product of the earlier
// radices; LD: inputs through load(line, n) (else src smem); ST: outputs
// through store(line, k, v) (else dst smem)
template <int L, int R, int NS, bool LD, bool ST, class Ld, class St>
__device__ __forceinline__ void ct_pass(const float2* __restrict__ tw, const float2* src,
                                        float2* dst, int Lp, Ld& load, St& store) {
  constexpr int nb = L / R;
  for (int w = threadIdx.x; w < kTL * nb; w += blockDim.x) {
    const int line = w % kTL, j = w / kTL;
    const int jm = NS == 1 ? 0 : j % NS;
    float2 v[R];
    if constexpr (LD) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = load(line, j + r * nb);
    } else {
      const float2* sp = src + line * Lp + j;
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = sp[r * nb];
    }
    if constexpr (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = c_mul(v[r], __ldg(tw + (r - 1) * NS + jm));
    }
    Dft<R>::run(v);
    if constexpr (ST) {
#pragma unroll
      for (int r = 0; r < R; ++r) store(line, j + r * nb, v[Dft<R>::pos(r)]);
    } else {
      float2* d = dst + line * Lp + (j - jm) * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) d[r * NS] = v[Dft<R>::pos(r)];
    }
  }
}

// two- or three-pass plan (R2 = 1: two passes), radices in the host plan's
// order (make_fft_plan_maxr: larger first)
template <int R0, int R1, int R2>
struct CtPlan {
  static constexpr int L = R0 * R1 * R2;
  __device__ static bool match(const FftPlanD& p) {
    return p.L == L && p.npass == (R2 == 1 ? 2 : 3) && p.radix[0] == R0 &&
           p.radix[1] == R1 && (R2 == 1 || p.radix[2] == R2);
  }
  // IO: first pass from load, last pass to store; else smem A -> result
  // buffer (returned)
  template <bool IO, class Ld, class St>
  __device__ static float2* run(const FftPlanD& p, float2* A, float2* B, int Lp, Ld& load,
                                St& store) {
    const float2* tw1 = p.tw + p.tw_off[1];
    ct_pass<L, R0, 1, IO, false>(nullptr, A, B, Lp, load, store);
    __syncthreads();
    if constexpr (R2 == 1) {
      ct_pass<L, R1, R0, false, IO>(tw1, B, A, Lp, load, store);
      if constexpr (!IO) __syncthreads();
      return A;
    } else {
      ct_pass<L, R1, R0, false, false>(tw1, B, A, Lp, load, store);
      __syncthreads();
      ct_pass<L, R2, R0 * R1, false, IO>(p.tw + p.tw_off[2], A, B, Lp, load, store);
      if constexpr (!IO) __syncthreads();
      return B;
    }
  }
};

// f(CtPlan<...>{}) for the first instantiation matching p; false if none.
// Covers the pads of the 64^3 / 128^3 benchmarks (72, 135, 144) and their
// neighbours.
template <class F>
__device__ __forceinline__ bool tile_dispatch(const FftPlanD& p, F&& f) {
  if (CtPlan<9, 8, 1>::match(p)) return f(CtPlan<9, 8, 1>{}), true;
  if (CtPlan<10, 8, 1>::match(p)) return f(CtPlan<10, 8, 1>{}), true;
  if (CtPlan<10, 9, 1>::match(p)) return f(CtPlan<10, 9, 1>{}), true;
  if (CtPlan<9, 5, 3>::match(p)) return f(CtPlan<9, 5, 3>{}), true;
  if (CtPlan<6, 6, 4>::match(p)) return f(CtPlan<6, 6, 4>{}), true;
  return false;
}

__device__ float2* tile_fft(const FftPlanD& p, float2* A, float2* B, int Lp) {
  float2* res = nullptr;
  NoIo io;
  if (tile_dispatch(p, [&](auto pl) { res = decltype(pl)::template run<false>(p, A, B, Lp, io, io); }))
    return res;
  return tile_fft_rt(p, A, B, Lp);
}

template <class Ld, class St>
__device__ void tile_fft_io(const FftPlanD& p, float2* A, float2* B, int Lp, Ld&& load,
                            St&& store) {
  if (tile_dispatch(p, [&](auto pl) { decltype(pl)::template run<true>(p, A, B, Lp, load, store); }))
    return;
  tile_fft_io_rt(p, A, B, Lp, load, store);
}

// y / z tiles: 16 adjacent x at one (z) for axis 1, at one (y) for axis 2
struct YZTile {
  int x0, c;
  __device__ __forceinline__ size_t base(const Geo3& g, int axis, int n) const {
    return axis == 1 ? (size_t(c) * g.py + n) * g.px + x0 : (size_t(n) * g.py + c) * g.px + x0;
  }
};
__device__ __forceinline__ YZTile yz_tile(const Geo3& g) {
  const int xt = (g.px + kTL - 1) / kTL;
  return YZTile{int(blockIdx.x % xt) * kTL, int(blockIdx.x / xt)};
}

// in-place forward y- or z-pass of nvol volumes; grid (tiles, volume)
__global__ void __launch_bounds__(kT3, 5) k3t_yz(FftPlanD p, Geo3 g, int axis,
                                              float2* __restrict__ buf, size_t vstride) {
  extern __shared__ float2 sm[];
  const int L = p.L, Lp = tile_stride(L);
  float2* A = sm;
  float2* B = sm + kTL * Lp;
  float2* v = buf + blockIdx.y * vstride;
  const YZTile t = yz_tile(g);
  const bool full = t.x0 + kTL <= g.px;
  tile_fft_io(
      p, A, B, Lp,
      [&](int line, int n) {
        return full || t.x0 + line < g.px ? v[t.base(g, axis, n) + line] : make_float2(0.f, 0.f);
      },
      [&](int line, int k, float2 x) {
        if (full || t.x0 + line < g.px) v[t.base(g, axis, k) + line] = x;
      });
}

// z-pass loading conj(H^) V^_sidx[b] (mode 0, gather) or conj(H^) (mode 1,
// the scatter's final inverse) -> work_b; grid (tiles, band of the chunk)
__global__ void __launch_bounds__(kT3, 5)
    k3t_z_load(FftPlanD p, Geo3 g, const float2* __restrict__ Hh, const float2* __restrict__ spec,
               const int* __restrict__ sidx, size_t vstride, int mode, float2* __restrict__ work) {
  extern __shared__ float2 sm[];
  const int L = p.L, Lp = tile_stride(L);
  float2* A = sm;
  float2* B = sm + kTL * Lp;
  const float2* V = mode == 0 ? spec + size_t(sidx[blockIdx.y]) * vstride : nullptr;
  float2* w = work + blockIdx.y * vstride;
  const YZTile t = yz_tile(g);
  tile_fft_io(
      p, A, B, Lp,
      [&](int line, int n) {
        if (t.x0 + line >= g.px) return make_float2(0.f, 0.f);
        const size_t i = t.base(g, 2, n) + line;
        return mode == 0 ? c_mul(c_conj(Hh[i]), __ldg(V + i)) : c_conj(Hh[i]);
      },
      [&](int line, int k, float2 x) {
        if (t.x0 + line < g.px) w[t.base(g, 2, k) + line] = x;
      });
}

// x tiles: rows li0 .. li0 + 15 of nl lines, copied in n-fast (contiguous)
template <class Ld>
__device__ __forceinline__ void x_load(int L, int nl, float2* A, int Lp, Ld&& ld) {
  const int li0 = blockIdx.x * kTL;
  for (int w = threadIdx.x; w < kTL * L; w += blockDim.x) {
    const int n = w % L, line = w / L;
    A[line * Lp + n] = li0 + line < nl ? ld(li0 + line, n) : make_float2(0.f, 0.f);
  }
  __syncthreads();
}
__device__ __forceinline__ void x_store_rows(int L, int nl, int px, const float2* Y, int Lp,
                                             float2* v) {
  const int li0 = blockIdx.x * kTL;
  for (int w = threadIdx.x; w < kTL * L; w += blockDim.x) {
    const int n = w % L, line = w / L;
    if (li0 + line < nl) v[size_t(li0 + line) * px + n] = Y[line * Lp + n];
  }
}

// x-pass from the signal (zero-padded), times D_b when premul (the scatter
// premultiply, engine3d.hpp:317-321); grid (tiles over py*pz rows, band)
__global__ void __launch_bounds__(kT3, 5)
    k3t_x_signal(FftPlanD p, Geo3 g, const float2* __restrict__ sig,
                 const double4* __restrict__ eul, const Band3* __restrict__ bands, int premul,
                 float2* __restrict__ work, size_t vstride) {
  extern __shared__ float2 sm[];
  const int L = p.L, Lp = tile_stride(L), nl = g.py * g.pz;
  float2* A = sm;
  float2* B = sm + kTL * Lp;
  const Band3& b = bands[blockIdx.y];
  x_load(L, nl, A, Lp, [&](int li, int n) -> float2 {
    const int y = li % g.py, z = li / g.py;
    if (n >= g.nx || y >= g.ny || z >= g.nz) return make_float2(0.f, 0.f);
    const size_t i = (size_t(z) * g.ny + y) * g.nx + n;
    float2 h = sig[i];
    if (premul) h = c_mul(h, wigner_at(b, eul[i], -1.f));
    return h;
  });
  const float2* Y = tile_fft(p, A, B, Lp);
  x_store_rows(L, nl, g.px, Y, Lp, work + blockIdx.y * vstride);
}

// x-pass of the filter bands: rendered (2R+1)^3 components wrapped to the
// origin (fft.hpp:186-194); grid (tiles over py*pz rows, band)
__global__ void __launch_bounds__(kT3, 5)
    k3t_x_filter(FftPlanD p, Geo3 g, const float2* __restrict__ comps, float2* __restrict__ spec,
                 size_t vstride) {
  extern __shared__ float2 sm[];
  const int L = p.L, Lp = tile_stride(L), nl = g.py * g.pz, S = 2 * g.R + 1;
  float2* A = sm;
  float2* B = sm + kTL * Lp;
  const float2* f = comps + size_t(blockIdx.y) * S * S * S;
  auto src = [&](int n, int P) {
    const int s = n + g.R;
    return s >= P ? s - P : s;
  };
  x_load(L, nl, A, Lp, [&](int li, int n) -> float2 {
    const int x = src(n, g.px), y = src(li % g.py, g.py), z = src(li / g.py, g.pz);
    if (x >= S || y >= S || z >= S) return make_float2(0.f, 0.f);
    return f[(size_t(z) * S + y) * S + x];
  });
  const float2* Y = tile_fft(p, A, B, Lp);
  x_store_rows(L, nl, g.px, Y, Lp, spec + blockIdx.y * vstride);
}

// x-pass finishing an inverse: rows (y, z) < (ny, nz) of work_b, crop x < nx;
// mode 0: part_b = conj(D_b) G_b (gather steering, engine3d.hpp:290-298);
// mode 1: out (+)= G (the scatter's single inverse).  G = conj(Y) / P.
__global__ void __launch_bounds__(kT3, 5)
    k3t_x_out(FftPlanD p, Geo3 g, const float2* __restrict__ work, size_t vstride,
              const double4* __restrict__ eul, const Band3* __restrict__ bands, int mode,
              float inv_p, float2* __restrict__ part, int accumulate, double2* __restrict__ out) {
  extern __shared__ float2 sm[];
  const int L = p.L, Lp = tile_stride(L), nl = g.ny * g.nz;
  float2* A = sm;
  float2* B = sm + kTL * Lp;
  const float2* w = work + blockIdx.y * vstride;
  x_load(L, nl, A, Lp, [&](int li, int n) -> float2 {
    const int y = li % g.ny, z = li / g.ny;
    return w[(size_t(z) * g.py + y) * g.px + n];
  });
  const float2* Y = tile_fft(p, A, B, Lp);
  const size_t N = size_t(g.nx) * g.ny * g.nz;
  const int li0 = blockIdx.x * kTL;
  for (int e = threadIdx.x; e < kTL * g.nx; e += blockDim.x) {
    const int x = e % g.nx, line = e / g.nx, li = li0 + line;
    if (li >= nl) continue;
    const size_t vi = size_t(li) * g.nx + x;  // (z*ny + y)*nx + x
    const float2 G = c_scale(c_conj(Y[line * Lp + x]), inv_p);
    if (mode == 0) {
      part[blockIdx.y * N + vi] = c_mul(wigner_at(bands[blockIdx.y], eul[vi], 1.f), G);
    } else {
      double2 v = make_double2(G.x, G.y);
      if (accumulate) {
        v.x += out[vi].x;
        v.y += out[vi].y;
      }
      out[vi] = v;
    }
  }
}

// out (+)= sum over the chunk's nb band planes, in band order (deterministic)
__global__ void k3_reduce_parts(const float2* __restrict__ part, int nb, size_t n,
                                int accumulate, double2* __restrict__ out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    double2 acc = accumulate ? out[i] : make_double2(0.0, 0.0);
    for (int b = 0; b < nb; ++b) {
      const float2 v = part[b * n + i];
      acc.x += v.x;
      acc.y += v.y;
    }
    out[i] = acc;
  }
}

// scatter: sum += sum over the chunk's bands of FFT3(H D_b) V^_sidx[b]
__global__ void k3_mac(const float2* __restrict__ work, int nb, size_t P,
                       const float2* __restrict__ spec, const int* __restrict__ sidx,
                       float2* __restrict__ sum) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < P;
       i += size_t(gridDim.x) * blockDim.x) {
    float2 acc = sum[i];
    for (int b = 0; b < nb; ++b)
      acc = c_add(acc, c_mul(work[b * P + i], __ldg(spec + size_t(sidx[b]) * P + i)));
    sum[i] = acc;
  }
}


size_t tile_smem(int L) { return 2 * size_t(kTL) * tile_stride(L) * sizeof(float2); }
// threads of a tile CTA: one per butterfly of the widest pass (16 lines x
// L / R), so short lines do not leave half the CTA idle
int tile_threads(const FftPlanD& p) {
  int nb = 1;
  for (int q = 0; q < p.npass; ++q) nb = std::max(nb, p.L / p.radix[q]);
  const int t = (kTL * nb + 31) / 32 * 32;
  return std::min(kT3, std::max(64, t));
}
unsigned ntiles(long long lines) { return unsigned((lines + kTL - 1) / kTL); }
unsigned yz_tiles(const Geo3& g, int axis) {
  return unsigned((g.px + kTL - 1) / kTL) * unsigned(axis == 1 ? g.pz : g.py);
}

}  // namespace

size_t tile3_smem(int L) { return tile_smem(L); }

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
  const size_t sm = tile_smem(pl.d.L);
  set_smem(k3t_yz, sm);
  k3t_yz<<<dim3(yz_tiles(g, axis), nvol), tile_threads(pl.d), sm, st>>>(pl.d, g, axis, buf, vstride);
  ++lc.n;
}

void launch3_x_signal(const FftPlan& pl, const Geo3& g, const float2* sig, const double4* eul,
                      const Band3* bands, int nb, int premul, float2* work, size_t vstride,
                      cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = tile_smem(pl.d.L);
  set_smem(k3t_x_signal, sm);
  k3t_x_signal<<<dim3(ntiles(1LL * g.py * g.pz), nb), tile_threads(pl.d), sm, st>>>(pl.d, g, sig, eul, bands,
                                                                     premul, work, vstride);
  ++lc.n;
}

void launch3_x_filter(const FftPlan& pl, const Geo3& g, const float2* comps, int nb,
                      float2* spec, size_t vstride, cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = tile_smem(pl.d.L);
  set_smem(k3t_x_filter, sm);
  k3t_x_filter<<<dim3(ntiles(1LL * g.py * g.pz), nb), tile_threads(pl.d), sm, st>>>(pl.d, g, comps, spec,
                                                                     vstride);
  ++lc.n;
}

void launch3_z_load(const FftPlan& pl, const Geo3& g, const float2* Hh, const float2* spec,
                    const int* sidx, int nb, size_t vstride, int mode, float2* work,
                    cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = tile_smem(pl.d.L);
  set_smem(k3t_z_load, sm);
  k3t_z_load<<<dim3(yz_tiles(g, 2), nb), tile_threads(pl.d), sm, st>>>(pl.d, g, Hh, spec, sidx, vstride, mode,
                                                        work);
  ++lc.n;
}

void launch3_x_out(const FftPlan& pl, const Geo3& g, const float2* work, size_t vstride, int nb,
                   const double4* eul, const Band3* bands, int mode, float2* part,
                   int accumulate, double2* out, cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = tile_smem(pl.d.L);
  set_smem(k3t_x_out, sm);
  const float inv_p = float(1.0 / (double(g.px) * g.py * g.pz));
  k3t_x_out<<<dim3(ntiles(1LL * g.ny * g.nz), nb), tile_threads(pl.d), sm, st>>>(
      pl.d, g, work, vstride, eul, bands, mode, inv_p, part, accumulate, out);
  ++lc.n;
}

void launch3_reduce_parts(const float2* part, int nb, size_t n, int accumulate, double2* out,
                          cudaStream_t st, LaunchCounter& lc) {
  k3_reduce_parts<<<grid_for(n, 256), 256, 0, st>>>(part, nb, n, accumulate, out);
  ++lc.n;
}

void launch3_mac(const float2* work, int nb, size_t P, const float2* spec, const int* sidx,
                 float2* sum, cudaStream_t st, LaunchCounter& lc) {
  k3_mac<<<grid_for(P, 256), 256, 0, st>>>(work, nb, P, spec, sidx, sum);
  ++lc.n;
}

}  // namespace xcb
