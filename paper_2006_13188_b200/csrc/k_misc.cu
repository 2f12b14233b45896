#include <cstdlib>
// Per-pixel stages: steering base / guard band, dtype conversion, smooth divide, angle max.
#include <algorithm>

#include "stages_common.cuh"

namespace xcb {
namespace {

// ------------------------------------------------------------------ prep
template <class TP>
__global__ void k_prep(const TP* __restrict__ param, int kind, double omega, double lo,
                       double hi, int H, int W, int transposed, double* __restrict__ base,
                       float* __restrict__ wgt, unsigned long long* bad) {
  pdl_wait();
  const size_t n = size_t(H) * W;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double v = double(param[i]);
    if (kind == 0) {
      base[i] = v;
      if (wgt) wgt[i] = 1.f;
      continue;
    }
    // true y-major index of the pixel (the reference scans y, then x)
    const size_t r = i / W, cidx = i % W;
    const unsigned long long ti = transposed ? (unsigned long long)cidx * H + r : i;
    if (!(v > 0.0) || !isfinite(v)) {
      atomicMin(bad, ti);
      base[i] = 0.0;
      if (wgt) wgt[i] = 0.f;
      continue;
    }
    if (v < lo || v > hi) atomicMin(bad + 1, ti);
    base[i] = omega * log(v);
    if (wgt) wgt[i] = float(1.0 / (v * v));
  }
}

template <class TS, class TD>
__global__ void k_convert(const TS* __restrict__ s, TD* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    d[i] = TD(s[i]);
}
__global__ void k_convert_c(const double2* __restrict__ s, float2* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    d[i] = make_float2(float(s[i].x), float(s[i].y));
}

// ------------------------------------------------------------------ smooth
__global__ void k_smooth_max(const float2* __restrict__ den, size_t n, unsigned* maxbits) {
  float m = 0.f;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    m = fmaxf(m, hypotf(den[i].x, den[i].y));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(maxbits, __float_as_uint(m));
  }
}

// block max of m >= 0, one atomicMax on the float bits per block (non-negative
// floats order as their bit patterns)
__device__ __forceinline__ void block_max_atomic(float m, unsigned* bits) {
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(bits, __float_as_uint(m));
  }
}

__global__ void k_absmax(const float* __restrict__ x, size_t n, int aligned, unsigned* bits) {
  float m = 0.f;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const size_t n4 = aligned ? n / 4 : 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
       i += size_t(gridDim.x) * blockDim.x) {
    const float4 v = x4[i];
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  // the tail (or, unaligned, everything) element-wise over the whole grid
  for (size_t i = 4 * n4 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    m = fmaxf(m, fabsf(x[i]));
  block_max_atomic(m, bits);
}

// packed smoothing (SIG_PACK): z = num + i alpha den with num, den real
__global__ void k_smooth_max_packed(const float2* __restrict__ z, size_t n, unsigned* maxbits) {
  float m = 0.f;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    m = fmaxf(m, fabsf(z[i].y));
  block_max_atomic(m, maxbits);
}

// floor 1e-9 max|den| (alpha cancels: |z.y| < 1e-9 max|z.y|), out = alpha z.x / z.y
template <class TO>
__global__ void k_smooth_div_packed(const float2* __restrict__ z, size_t n,
                                    const unsigned* amax, const unsigned* maxbits,
                                    TO* __restrict__ out, unsigned* clamped) {
  const double floor_ = 1e-9 * double(__uint_as_float(*maxbits));
  const double alpha = double(pack_alpha(amax));
  const bool zero = *amax == 0u;  // h == 0: num is exactly 0 (the packed z.x is rounding)
  unsigned cnt = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double dy = z[i].y;
    if (fabs(dy) < floor_) {
      ++cnt;
      out[i] = TO(0);
      continue;
    }
    out[i] = zero ? TO(0) : TO(alpha * double(z[i].x) / dy);
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(clamped, cnt);
}

template <class TO>
__global__ void k_smooth_div(const float2* __restrict__ num, const float2* __restrict__ den,
                             size_t n, const unsigned* maxbits, TO* __restrict__ out,
                             unsigned* clamped) {
  const double floor_ = 1e-9 * double(__uint_as_float(*maxbits));
  unsigned cnt = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double dx = den[i].x, dy = den[i].y;
    const double ad = sqrt(dx * dx + dy * dy);
    if (ad < floor_) {
      ++cnt;
      out[i] = TO(0);
      continue;
    }
    out[i] = TO((double(num[i].x) * dx + double(num[i].y) * dy) / (dx * dx + dy * dy));
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(clamped, cnt);
}

// ------------------------------------------------------------------ angle max
constexpr int kMaxDense = 256;
struct AngleMap {
  int nd;                 // dense coefficient count (kmax - kmin + 1)
  int idx[kMaxDense];     // plane index of dense slot d, or -1
};

template <class TO>
__global__ void __launch_bounds__(128)
    k_anglemax(const float2* __restrict__ planes, AngleMap m, size_t npix, int n,
               TO* __restrict__ score, int* __restrict__ argmax) {
  extern __shared__ float2 sa[];
  float2* tw = sa;                   // [n] e^{-2 pi i s / n}
  float2* co = sa + n;               // [nd][blockDim]
  const int bd = blockDim.x, t = threadIdx.x;
  for (int s = t; s < n; s += bd) {
    double sn, cs;
    sincospi(-2.0 * s / n, &sn, &cs);
    tw[s] = make_float2(float(cs), float(sn));
  }
  const size_t p = blockIdx.x * size_t(bd) + t;
  for (int d = 0; d < m.nd; ++d)
    co[d * bd + t] = (p < npix && m.idx[d] >= 0) ? planes[size_t(m.idx[d]) * npix + p]
                                                 : make_float2(0.f, 0.f);
  __syncthreads();
  if (p >= npix) return;
  constexpr int CH = 12;
  float best = -1.f;
  int arg = 0;
  for (int s0 = 0; s0 < n; s0 += CH) {
    float2 acc[CH], z[CH];
    const float2 top = co[(m.nd - 1) * bd + t];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      z[c] = tw[min(s0 + c, n - 1)];
      acc[c] = top;
    }
    for (int d = m.nd - 2; d >= 0; --d) {
      const float2 gv = co[d * bd + t];
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = c_add(c_mul(acc[c], z[c]), gv);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const float m2 = fmaf(acc[c].x, acc[c].x, acc[c].y * acc[c].y);
      if (s0 + c < n && m2 > best) {
        best = m2;
        arg = s0 + c;
      }
    }
  }
  score[p] = TO(sqrtf(best));
  if (argmax) argmax[p] = arg;
}

// Angle max by FFT (n_angles = 360, bands k in [-KH, KH]): with s = s1 + N1 s2
// (N1 N2 = 360, N2 >= 2 KH + 1),
//   X(s) = sum_k G_k e^{-2 pi i k s / 360}
//        = DFT_N2[ m -> G_k w^{k s1}, m = k mod N2 ](s2),  w = e^{-2 pi i / 360},
// so each pixel costs N1 twiddled N2-point DFTs instead of 360 x (2 KH + 1)
// complex MACs.  Ties keep the smallest s (the oracle's first maximum).
// 360-angle max for bands inside [-KH, KH]: S(s1 + N1 s2) =
// DFT_N2[ G_d w^{d s1} ] (w = e^{-2 pi i / 360}, d = k mod N2), N1 = 360 / N2.
// The s1 loop runs U trips per unrolled body (the body must stay small enough
// for the instruction cache); twiddles are smem broadcast reads; the running
// max takes the first angle in scan order (s1-major) on exact ties.
template <int KH, int N2, class TO, int U>
__device__ __forceinline__ void anglemax_fft_body(const float2* __restrict__ planes,
                                                  const AngleMap& m, size_t npix,
                                                  TO* __restrict__ score,
                                                  int* __restrict__ argmax) {
  constexpr int ND = 2 * KH + 1, N = 360, N1 = N / N2;
  static_assert(N1 * N2 == N && N2 >= ND && N1 % U == 0, "bad angle-max split");
  // twiddles w^{(d - KH) s1}, [s1][d] (broadcast reads)
  __shared__ float2 tws[N1 * ND];
  for (int i = threadIdx.x; i < N1 * ND; i += blockDim.x) {
    const int s1 = i / ND, d = i % ND;
    double sn, cs;
    sincospi(-2.0 * double((d - KH) * s1) / N, &sn, &cs);
    tws[i] = make_float2(float(cs), float(sn));
  }
  __syncthreads();
  const size_t p = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (p >= npix) return;
  float2 G[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d)
    G[d] = m.idx[d] >= 0 ? planes[size_t(m.idx[d]) * npix + p] : make_float2(0.f, 0.f);
  float best = -1.f;
  int arg = 0;
#pragma unroll U
  for (int s1 = 0; s1 < N1; ++s1) {
    float2 v[N2];
#pragma unroll
    for (int q = 0; q < N2; ++q) v[q] = make_float2(0.f, 0.f);
    const float2* tw = tws + s1 * ND;
#pragma unroll
    for (int d = 0; d < ND; ++d) v[((d - KH) % N2 + N2) % N2] = c_mul(G[d], tw[d]);
    Dft<N2>::run(v);
#pragma unroll
    for (int s2 = 0; s2 < N2; ++s2) {
      const float2 x = v[Dft<N2>::pos(s2)];
      const float m2 = fmaf(x.x, x.x, x.y * x.y);
      if (m2 > best) {
        best = m2;
        arg = s1 + N1 * s2;
      }
    }
  }
  score[p] = TO(sqrtf(best));
  if (argmax) argmax[p] = arg;
}

#define XCB_AM_KERNEL(NAME, U)                                                        \
  template <int KH, int N2, class TO>                                                 \
  __global__ void __launch_bounds__(128)                                              \
      NAME(const float2* __restrict__ planes, AngleMap m, size_t npix,                \
           TO* __restrict__ score, int* __restrict__ argmax) {                        \
    anglemax_fft_body<KH, N2, TO, U>(planes, m, npix, score, argmax);                 \
  }
// measured on config 3 (KH = 16): one s1 per loop trip 4.83 ms, two 4.91,
// five 6.59 (instruction-cache misses), fully unrolled 5.45
XCB_AM_KERNEL(k_anglemax_fft, 1)
#undef XCB_AM_KERNEL

// Hermitian half-band angle max: for a real signal and a filter with
// F_{-k} = conj(F_k) the band responses satisfy G_{-k} = conj(G_k), so
// S(s) = sum_k G_k w^{ks} = G_0 + 2 Re(sum_{k=1}^{KH} G_k w^{ks}) is real and
// only the planes k = 0..KH are needed (half the I1 / planes work), and one
// complex DFT_N2 evaluates two rows s1 of real outputs.  m.idx[k] = plane of
// band k (k = 0..KH).
template <int KH, int N2, class TO>
__global__ void __launch_bounds__(128)
    k_anglemax_herm(const float2* __restrict__ planes, AngleMap m, size_t npix,
                    TO* __restrict__ score, int* __restrict__ argmax) {
  constexpr int N = 360, N1 = N / N2;
  static_assert(N1 * N2 == N && N2 > 2 * KH && N1 % 2 == 0, "bad angle-max split");
  __shared__ float2 tws[N1 * KH];  // w^{k s1}, [s1][k-1]
  for (int i = threadIdx.x; i < N1 * KH; i += blockDim.x) {
    const int s1 = i / KH, k = i % KH + 1;
    double sn, cs;
    sincospi(-2.0 * double(k * s1) / N, &sn, &cs);
    tws[i] = make_float2(float(cs), float(sn));
  }
  __syncthreads();
  const size_t p = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (p >= npix) return;
  const float g0 = m.idx[0] >= 0 ? planes[size_t(m.idx[0]) * npix + p].x : 0.f;
  float2 G[KH];
#pragma unroll
  for (int k = 1; k <= KH; ++k)
    G[k - 1] = m.idx[k] >= 0 ? planes[size_t(m.idx[k]) * npix + p] : make_float2(0.f, 0.f);
  float best = -1.f;
  int arg = 0;
  // Two s1 per DFT: with X_k = G_k w^{k sa}, Y_k = G_k w^{k sb} (k = -KH..KH,
  // X_{-k} = conj X_k) both DFTs are real, so DFT(X + iY) = S(sa + N1 s2) +
  // i S(sb + N1 s2): one N2-point DFT per pair of s1 instead of two.
#pragma unroll 1
  for (int sa = 0; sa < N1; sa += 2) {
    float2 v[N2];
#pragma unroll
    for (int q = 0; q < N2; ++q) v[q] = make_float2(0.f, 0.f);
    v[0] = make_float2(g0, g0);
    const float2* ta = tws + sa * KH;
    const float2* tb = ta + KH;
#pragma unroll
    for (int k = 1; k <= KH; ++k) {
      const float2 x = c_mul(G[k - 1], ta[k - 1]), y = c_mul(G[k - 1], tb[k - 1]);
      v[k] = make_float2(x.x - y.y, x.y + y.x);            // X_k + i Y_k
      v[N2 - k] = make_float2(x.x + y.y, y.x - x.y);       // conj X_k + i conj Y_k
    }
    Dft<N2>::run(v);
    // scan in the s1-major order (sa, then sb): the first maximum wins
#pragma unroll
    for (int s2 = 0; s2 < N2; ++s2) {
      const float a = fabsf(v[Dft<N2>::pos(s2)].x);
      if (a > best) {
        best = a;
        arg = sa + N1 * s2;
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < N2; ++s2) {
      const float a = fabsf(v[Dft<N2>::pos(s2)].y);
      if (a > best) {
        best = a;
        arg = sa + 1 + N1 * s2;
      }
    }
  }
  score[p] = TO(best);
  if (argmax) argmax[p] = arg;
}

// Looped variant (twiddles from a smem table) for wide band spans, where the
// unrolled kernel would not fit in registers.
template <int KH, int N2, class TO>
__global__ void __launch_bounds__(128)
    k_anglemax_fft_loop(const float2* __restrict__ planes, AngleMap m, size_t npix,
                   TO* __restrict__ score, int* __restrict__ argmax) {
  constexpr int ND = 2 * KH + 1, N = 360, N1 = N / N2;
  static_assert(N1 * N2 == N && N2 >= ND, "bad angle-max split");
  __shared__ float2 tw[ND * N1];
  for (int i = threadIdx.x; i < ND * N1; i += blockDim.x) {
    const int d = i / N1, s1 = i % N1;
    double sn, cs;
    sincospi(-2.0 * double((d - KH) * s1) / N, &sn, &cs);
    tw[i] = make_float2(float(cs), float(sn));
  }
  __syncthreads();
  const size_t p = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (p >= npix) return;
  float2 G[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d)
    G[d] = m.idx[d] >= 0 ? planes[size_t(m.idx[d]) * npix + p] : make_float2(0.f, 0.f);
  float best = -1.f;
  int arg = 0;
#pragma unroll 1
  for (int s1 = 0; s1 < N1; ++s1) {
    float2 v[N2];
#pragma unroll
    for (int q = 0; q < N2; ++q) v[q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int d = 0; d < ND; ++d) v[((d - KH) % N2 + N2) % N2] = c_mul(G[d], tw[d * N1 + s1]);
    Dft<N2>::run(v);
#pragma unroll
    for (int s2 = 0; s2 < N2; ++s2) {
      const float2 x = v[Dft<N2>::pos(s2)];
      const float m2 = fmaf(x.x, x.x, x.y * x.y);
      const int s = s1 + N1 * s2;
      if (m2 > best || (m2 == best && s < arg)) {
        best = m2;
        arg = s;
      }
    }
  }
  score[p] = TO(sqrtf(best));
  if (argmax) argmax[p] = arg;
}

}  // namespace

float2* upload_twiddles(const FftPlan& p) {
  float2* d = nullptr;
  if (cudaMalloc(&d, p.tw_host.size() * sizeof(float2)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, p.tw_host.data(), p.tw_host.size() * sizeof(float2), cudaMemcpyHostToDevice);
  return d;
}

void launch_prep(const void* param, int param_is_f64, int kind, double omega, double lo,
                 double hi, int H, int W, int transposed, double* base, float* wgt,
                 unsigned long long* bad, cudaStream_t st, LaunchCounter& lc) {
  const int g = grid_for(size_t(H) * W, 256);
  if (param_is_f64)
    launch_k(k_prep<double>, g, 256, 0, st, static_cast<const double*>(param), kind, omega, lo, hi,
                                      H, W, transposed, base, wgt, bad);
  else
    launch_k(k_prep<float>, g, 256, 0, st, static_cast<const float*>(param), kind, omega, lo, hi,
                                     H, W, transposed, base, wgt, bad);
  ++lc.n;
}

void launch_convert_signal(const void* src, int dtype, size_t n, void* dst, cudaStream_t st,
                           LaunchCounter& lc) {
  const int g = grid_for(n, 256);
  if (dtype == 1)  // f64 real -> f32
    k_convert<double, float><<<g, 256, 0, st>>>(static_cast<const double*>(src),
                                                static_cast<float*>(dst), n);
  else  // c128 -> c64
    k_convert_c<<<g, 256, 0, st>>>(static_cast<const double2*>(src), static_cast<float2*>(dst),
                                   n);
  ++lc.n;
}

template <class T>
__global__ void k_accumulate(T* __restrict__ dst, const T* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

void launch_accumulate(void* dst, const void* src, size_t n, int f64, cudaStream_t st,
                       LaunchCounter& lc) {
  const int g = grid_for(n, 256);
  if (f64)
    k_accumulate<double><<<g, 256, 0, st>>>(static_cast<double*>(dst),
                                            static_cast<const double*>(src), n);
  else
    k_accumulate<float><<<g, 256, 0, st>>>(static_cast<float*>(dst),
                                           static_cast<const float*>(src), n);
  ++lc.n;
}

// dst += slots[0] + slots[1] + ... in slot order (the order of the sequential
// accumulate, so both reduces give the same bits); slots `stride` elements apart
template <class T>
__global__ void k_sum_slots(T* __restrict__ dst, const T* __restrict__ slots, size_t stride,
                            int ns, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    T a = dst[i];
    for (int s = 0; s < ns; ++s) {
      const T b = slots[size_t(s) * stride + i];
      a.x += b.x;
      a.y += b.y;
    }
    dst[i] = a;
  }
}

void launch_sum_slots(void* dst, const void* slots, size_t stride, int ns, size_t n, int f64,
                      cudaStream_t st, LaunchCounter& lc) {
  // n, stride: scalar counts (even: complex or (num, den) pairs)
  const int g = grid_for(n / 2, 256);
  if (f64)
    k_sum_slots<double2><<<g, 256, 0, st>>>(static_cast<double2*>(dst),
                                            static_cast<const double2*>(slots), stride / 2, ns,
                                            n / 2);
  else
    k_sum_slots<float2><<<g, 256, 0, st>>>(static_cast<float2*>(dst),
                                           static_cast<const float2*>(slots), stride / 2, ns,
                                           n / 2);
  ++lc.n;
}

void launch_absmax(const float* x, size_t n, unsigned* bits, cudaStream_t st, LaunchCounter& lc) {
  // 4 CTAs per SM loop over the field: one atomic per CTA (float4 loads need
  // 16-byte alignment: the staged fields are cudaMalloc'd)
  const int al = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  k_absmax<<<std::min(grid_for(n / 4 + 1, 256), 4 * 148), 256, 0, st>>>(x, n, al, bits);
  ++lc.n;
}

void launch_smooth_finish_packed(const float2* z, size_t n, const unsigned* amax, int out_f64,
                                 void* out, unsigned* maxbits, unsigned* clamped, cudaStream_t st,
                                 LaunchCounter& lc) {
  const int g = grid_for(n, 256);
  k_smooth_max_packed<<<g, 256, 0, st>>>(z, n, maxbits);
  if (out_f64)
    k_smooth_div_packed<double><<<g, 256, 0, st>>>(z, n, amax, maxbits,
                                                   static_cast<double*>(out), clamped);
  else
    k_smooth_div_packed<float><<<g, 256, 0, st>>>(z, n, amax, maxbits, static_cast<float*>(out),
                                                  clamped);
  lc.n += 2;
}

void launch_smooth_finish(const float2* num, const float2* den, size_t n, int out_f64,
                          void* out, unsigned* maxbits, unsigned* clamped, cudaStream_t st,
                          LaunchCounter& lc) {
  const int g = grid_for(n, 256);
  k_smooth_max<<<g, 256, 0, st>>>(den, n, maxbits);
  if (out_f64)
    k_smooth_div<double><<<g, 256, 0, st>>>(num, den, n, maxbits, static_cast<double*>(out),
                                            clamped);
  else
    k_smooth_div<float><<<g, 256, 0, st>>>(num, den, n, maxbits, static_cast<float*>(out),
                                           clamped);
  lc.n += 2;
}

void launch_anglemax_herm(const float2* planes, const int* ks_host, int nb, size_t npix,
                          int score_f64, void* score, int* argmax, cudaStream_t st,
                          LaunchCounter& lc) {
  int kh = 0;
  for (int i = 0; i < nb; ++i) kh = std::max(kh, ks_host[i]);
  AngleMap m{};
  m.nd = kh + 1;
  for (int k = 0; k <= kh; ++k) m.idx[k] = -1;
  for (int i = 0; i < nb; ++i) m.idx[ks_host[i]] = i;
  const int bs = 128;
  const int grid = int((npix + bs - 1) / bs);
#define XCB_AMH(KHV, N2V)                                                                   \
  if (kh == KHV) {                                                                         \
    if (score_f64)                                                                         \
      k_anglemax_herm<KHV, N2V, double><<<grid, bs, 0, st>>>(planes, m, npix,              \
                                                            static_cast<double*>(score), argmax); \
    else                                                                                   \
      k_anglemax_herm<KHV, N2V, float><<<grid, bs, 0, st>>>(planes, m, npix,               \
                                                           static_cast<float*>(score), argmax);  \
  }
  XCB_AMH(4, 12) XCB_AMH(8, 18) XCB_AMH(16, 36)
#undef XCB_AMH
  ++lc.n;
}

int anglemax_herm_kh(int kh) { return kh == 4 || kh == 8 || kh == 16; }

void launch_anglemax(const float2* planes, const int* ks_host, int nb, size_t npix,
                     int n_angles, int score_f64, void* score, int* argmax, cudaStream_t st,
                     LaunchCounter& lc) {
  AngleMap m{};
  int kmin = ks_host[0], kmax = ks_host[0];
  for (int i = 0; i < nb; ++i) {
    kmin = ks_host[i] < kmin ? ks_host[i] : kmin;
    kmax = ks_host[i] > kmax ? ks_host[i] : kmax;
  }
  m.nd = kmax - kmin + 1;
  for (int d = 0; d < m.nd && d < kMaxDense; ++d) m.idx[d] = -1;
  for (int i = 0; i < nb; ++i) m.idx[ks_host[i] - kmin] = i;
  const int bs = 128;
  const int grid = int((npix + bs - 1) / bs);
  // FFT evaluation for 360 angles and a band set inside [-KH, KH]
  const int kh = std::max(-kmin, kmax);
  int KH = 0;
  for (int c : {4, 8, 16, 32})
    if (kh <= c) {
      KH = c;
      break;
    }
  if (n_angles == 360 && KH > 0) {
    AngleMap fm{};
    fm.nd = 2 * KH + 1;
    for (int d = 0; d < fm.nd; ++d) fm.idx[d] = -1;
    for (int i = 0; i < nb; ++i) fm.idx[ks_host[i] + KH] = i;
#define XCB_AM(KHV, N2V, KER)                                                                \
  if (KH == KHV) {                                                                         \
    if (score_f64)                                                                         \
      KER<KHV, N2V, double><<<grid, bs, 0, st>>>(planes, fm, npix,                         \
                                                static_cast<double*>(score), argmax);      \
    else                                                                                   \
      KER<KHV, N2V, float><<<grid, bs, 0, st>>>(planes, fm, npix,                          \
                                               static_cast<float*>(score), argmax);        \
  }
    XCB_AM(4, 12, k_anglemax_fft) XCB_AM(8, 18, k_anglemax_fft)
    XCB_AM(16, 36, k_anglemax_fft) XCB_AM(32, 72, k_anglemax_fft_loop)
#undef XCB_AM
    ++lc.n;
    return;
  }
  const size_t smem = (size_t(n_angles) + size_t(m.nd) * bs) * sizeof(float2);
  if (score_f64) {
    set_smem(k_anglemax<double>, smem);
    k_anglemax<double><<<grid, bs, smem, st>>>(planes, m, npix, n_angles,
                                               static_cast<double*>(score), argmax);
  } else {
    set_smem(k_anglemax<float>, smem);
    k_anglemax<float><<<grid, bs, smem, st>>>(planes, m, npix, n_angles,
                                              static_cast<float*>(score), argmax);
  }
  ++lc.n;
}

// ------------------------------------------------------------------ detect_pattern
namespace {
// central-difference gradient, one-sided at the borders (field.hpp:204-237),
// in double, of a real image stored row- or column-major; magnitude and
// direction written in the same storage order as fp32 (the xconv inputs)
template <class TI>
__global__ void k_gradient(const TI* __restrict__ img, int h, int w, int colmajor,
                           float* __restrict__ mag, float* __restrict__ dir) {
  const size_t n = size_t(h) * w;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int y = colmajor ? int(i % h) : int(i / w), x = colmajor ? int(i / h) : int(i % w);
    auto I = [&](int yy, int xx) -> double {
      return double(img[colmajor ? size_t(xx) * h + yy : size_t(yy) * w + xx]);
    };
    const double gx = w == 1 ? 0.0
                      : x == 0 ? I(y, 1) - I(y, 0)
                      : x == w - 1 ? I(y, w - 1) - I(y, w - 2)
                                   : 0.5 * (I(y, x + 1) - I(y, x - 1));
    const double gy = h == 1 ? 0.0
                      : y == 0 ? I(1, x) - I(0, x)
                      : y == h - 1 ? I(h - 1, x) - I(h - 2, x)
                                   : 0.5 * (I(y + 1, x) - I(y - 1, x));
    const double m = sqrt(gx * gx + gy * gy);
    mag[i] = float(m);
    dir[i] = m > 0.0 ? float(atan2(gy, gx)) : 0.f;
  }
}

template <class TO>
__global__ void k_real_part(const float2* __restrict__ in, size_t n, TO* __restrict__ out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = TO(in[i].x);
}
}  // namespace

void launch_gradient(const void* img, int img_f64, int h, int w, int colmajor, float* mag,
                     float* dir, cudaStream_t st, LaunchCounter& lc) {
  const int g = grid_for(size_t(h) * w, 256);
  if (img_f64)
    k_gradient<double><<<g, 256, 0, st>>>(static_cast<const double*>(img), h, w, colmajor, mag,
                                          dir);
  else
    k_gradient<float><<<g, 256, 0, st>>>(static_cast<const float*>(img), h, w, colmajor, mag,
                                         dir);
  ++lc.n;
}

void launch_real_part(const float2* in, size_t n, int out_f64, void* out, cudaStream_t st,
                      LaunchCounter& lc) {
  const int g = grid_for(n, 256);
  if (out_f64)
    k_real_part<double><<<g, 256, 0, st>>>(in, n, static_cast<double*>(out));
  else
    k_real_part<float><<<g, 256, 0, st>>>(in, n, static_cast<float*>(out));
  ++lc.n;
}

// ------------------------------------------------------------------ find_peaks (device)
namespace {
// order-preserving map of a float / double to an unsigned key (max = max key)
__device__ __forceinline__ unsigned long long okey(double v) {
  unsigned long long b = __double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unkey(unsigned long long k) {
  return __longlong_as_double((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k);
}

template <class T>
__global__ void k_max_key(const T* __restrict__ r, size_t n, unsigned long long* mx) {
  unsigned long long best = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    best = max(best, okey(double(r[i])));
  for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, best);
}

// vote_filter.hpp:107-134: a pixel at or above threshold_frac * max is a peak
// if no pixel within the disk beats it (ties: the earlier one in y-major scan
// order wins); peaks are appended unordered, the host sorts them
template <class T>
__global__ void k_nms(const T* __restrict__ r, int h, int w, int colmajor, double radius,
                      double frac, const unsigned long long* mx, int R, int cap,
                      unsigned* count, int* px, int* py, double* pv) {
  const double thresh = frac * unkey(*mx);
  const size_t n = size_t(h) * w;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int y = int(i / w), x = int(i % w);
    auto at = [&](int yy, int xx) -> double {
      return double(r[colmajor ? size_t(xx) * h + yy : size_t(yy) * w + xx]);
    };
    const double v = at(y, x);
    if (v < thresh) continue;
    bool best = true;
    for (int dy = -R; dy <= R && best; ++dy)
      for (int dx = -R; dx <= R && best; ++dx) {
        if (dx == 0 && dy == 0) continue;
        if (double(dx * dx + dy * dy) > radius * radius) continue;
        const int xi = x + dx, yi = y + dy;
        if (xi < 0 || yi < 0 || xi >= w || yi >= h) continue;
        const double o = at(yi, xi);
        if (o > v || (o == v && (dy < 0 || (dy == 0 && dx < 0)))) best = false;
      }
    if (best) {
      const unsigned k = atomicAdd(count, 1u);
      if (int(k) < cap) {
        px[k] = x;
        py[k] = y;
        pv[k] = v;
      }
    }
  }
}
}  // namespace

void launch_find_peaks(const void* resp, int f64, int h, int w, int colmajor, double radius,
                       double frac, int cap, unsigned long long* mx, unsigned* count, int* px,
                       int* py, double* pv, cudaStream_t st, LaunchCounter& lc) {
  const size_t n = size_t(h) * w;
  const int R = radius > 1.0 ? int(ceil(radius)) : 1;
  cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st);
  cudaMemsetAsync(count, 0, sizeof(unsigned), st);
  const int g = grid_for(n, 256);
  if (f64) {
    k_max_key<double><<<g, 256, 0, st>>>(static_cast<const double*>(resp), n, mx);
    k_nms<double><<<g, 256, 0, st>>>(static_cast<const double*>(resp), h, w, colmajor, radius,
                                     frac, mx, R, cap, count, px, py, pv);
  } else {
    k_max_key<float><<<g, 256, 0, st>>>(static_cast<const float*>(resp), n, mx);
    k_nms<float><<<g, 256, 0, st>>>(static_cast<const float*>(resp), h, w, colmajor, radius,
                                    frac, mx, R, cap, count, px, py, pv);
  }
  lc.n += 2;
}

// ------------------------------------------------------------------ filter rendering
// Per-band rendering of a decomposed filter on the (2R+1)^2 grid centred at
// (R, R) (freq_filter.hpp:133-184, component_value / render_component):
//   rotation: linear interpolation of the radial profile at half-integer
//             radii x e^{i k phi}; r <= 1e-9 keeps only k = 0
//   scale:    linear interpolation of the angular profile (wrapped) x
//             e^{i k omega log(r / r_min)}; 0 inside r_min
// zero outside r_max; phi = atan2(dy, dx) with y down.  fp64 math, fp32 out,
// layout [band][y][x] (transpose: [band][x][y]).
namespace {
__global__ void k_render(const double2* __restrict__ comps, const int* __restrict__ ks, int nb,
                         int group, int n_radii, int n_angles, double r_max, double r_min,
                         double omega, int S, int R, int transpose, float2* __restrict__ out) {
  const size_t n = size_t(nb) * S * S;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int ci = int(i / (size_t(S) * S));
    const int rem = int(i % (size_t(S) * S));
    const int y = rem / S, x = rem % S;
    const double dx = double(x - R), dy = double(y - R);
    const double r = sqrt(dx * dx + dy * dy);
    const int k = ks[ci];
    double vr = 0, vi = 0;
    if (r <= r_max) {
      const double th = atan2(dy, dx);
      double ar, ai, ph;
      bool zero = false;
      if (group == 0) {
        if (r <= 1e-9 && k != 0) zero = true;
        double u = r / r_max * n_radii - 0.5;
        u = fmin(fmax(u, 0.0), double(n_radii - 1));
        const int j0 = int(u), j1 = min(j0 + 1, n_radii - 1);
        const double t = u - j0;
        const double2 c0 = comps[size_t(j0) * nb + ci], c1 = comps[size_t(j1) * nb + ci];
        ar = (1 - t) * c0.x + t * c1.x;
        ai = (1 - t) * c0.y + t * c1.y;
        ph = k * th;
      } else {
        const double twopi = 6.283185307179586476925286766559;
        double v = th / twopi * n_angles;
        v -= floor(v / n_angles) * n_angles;
        const int m0 = int(v) % n_angles, m1 = (m0 + 1) % n_angles;
        const double t = v - floor(v);
        if (r < r_min) zero = true;
        const double2 c0 = comps[size_t(m0) * nb + ci], c1 = comps[size_t(m1) * nb + ci];
        ar = (1 - t) * c0.x + t * c1.x;
        ai = (1 - t) * c0.y + t * c1.y;
        ph = zero ? 0.0 : k * omega * log(r / r_min);
      }
      if (!zero) {
        double sn, cs;
        sincos(ph, &sn, &cs);
        vr = ar * cs - ai * sn;
        vi = ar * sn + ai * cs;
      }
    }
    out[size_t(ci) * S * S + (transpose ? size_t(x) * S + y : size_t(y) * S + x)] =
        make_float2(float(vr), float(vi));
  }
}
}  // namespace

void launch_render(const double2* comps, const int* ks, int nb, int group, int n_radii,
                   int n_angles, double r_max, double r_min, double omega, int S, int R,
                   int transpose, float2* out, cudaStream_t st, LaunchCounter& lc) {
  const int g = grid_for(size_t(nb) * S * S, 256);
  k_render<<<g, 256, 0, st>>>(comps, ks, nb, group, n_radii, n_angles, r_max, r_min, omega, S, R,
                              transpose, out);
  ++lc.n;
}

}  // namespace xcb

// ------------------------------------------------------------------ decomposition
// decompose_rotation2 / decompose_scale2 on the device (freq_filter.hpp:63-129,
// polar.hpp:46-83): the polar (log-polar) bilinear resampling of the filter
// image, one thread per sample, then the DFT over the periodic axis, one thread
// per (row, band).  fp64 throughout; the band phase 2 pi k (s + off) / L is
// evaluated with sincospi of an exactly formed quotient.
namespace xcb {
namespace {
__global__ void k_polar_samples(const double2* __restrict__ img, int w, int h, double cx,
                                double cy, int nr, int na, int log_radial, double r_min,
                                double r_max, double2* __restrict__ p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr * na) return;
  const int j = i / na, m = i % na;
  const double r = log_radial ? r_min * pow(r_max / r_min, (j + 0.5) / nr)
                              : (j + 0.5) * r_max / nr;
  const double two_pi = 6.283185307179586476925286766559;  // 2 * EIGEN_PI
  const double th = two_pi * m / na;
  double sn, cs;
  sincos(th, &sn, &cs);
  const double x = cx + r * cs, y = cy + r * sn;
  // Field2::sample (field.hpp:51-62): bilinear, zero outside the grid
  const double fx = floor(x), fy = floor(y);
  const int x0 = int(fx), y0 = int(fy);
  const double tx = x - fx, ty = y - fy;
  auto tap = [&](int xi, int yi) {
    return (xi < 0 || yi < 0 || xi >= w || yi >= h) ? make_double2(0.0, 0.0)
                                                     : img[size_t(yi) * w + xi];
  };
  const double2 a = tap(x0, y0), b = tap(x0 + 1, y0), c = tap(x0, y0 + 1), d = tap(x0 + 1, y0 + 1);
  p[i] = make_double2((1.0 - ty) * ((1.0 - tx) * a.x + tx * b.x) + ty * ((1.0 - tx) * c.x + tx * d.x),
                      (1.0 - ty) * ((1.0 - tx) * a.y + tx * b.y) + ty * ((1.0 - tx) * c.y + tx * d.y));
}

// comps[row][ci] = half_k / L * sum_s P(row, s) e^{-2 pi i k (s + off) / L}:
// rotation (group 0): rows = radii j, s = angle m, P = p[j][m], off = 0;
// scale (group 1): rows = angles m, s = radius j, P = p[j][m], off = 1/2.
__global__ void k_band_dft(const double2* __restrict__ p, int nr, int na, int group,
                           const int* __restrict__ ks, int nc, double2* __restrict__ comps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = group == 0 ? nr : na, L = group == 0 ? na : nr;
  if (i >= rows * nc) return;
  const int row = i / nc, ci = i % nc, k = ks[ci];
  double ar = 0.0, ai = 0.0;
  for (int s = 0; s < L; ++s) {
    const double2 v = group == 0 ? p[size_t(row) * na + s] : p[size_t(s) * na + row];
    // e^{-2 pi i k (s + off) / L}: 2 k (s + off) is exact (an integer)
    const long long num = group == 0 ? 2LL * k * s : (2LL * s + 1) * k;
    double sn, cs;
    sincospi(-double(num) / double(L), &sn, &cs);
    ar += v.x * cs - v.y * sn;
    ai += v.x * sn + v.y * cs;
  }
  const double half = (2 * abs(k) == L) ? 0.5 : 1.0;
  comps[size_t(row) * nc + ci] = make_double2(ar * half / L, ai * half / L);
}
}  // namespace

void launch_decompose(const double2* img, int w, int h, double cx, double cy, int nr, int na,
                      int group, double r_min, double r_top, const int* ks, int nc,
                      double2* samples, double2* comps, cudaStream_t st, LaunchCounter& lc) {
  const int n = nr * na, rows = (group == 0 ? nr : na) * nc;
  k_polar_samples<<<(n + 127) / 128, 128, 0, st>>>(img, w, h, cx, cy, nr, na, group == 1, r_min,
                                                   r_top, samples);
  k_band_dft<<<(rows + 127) / 128, 128, 0, st>>>(samples, nr, na, group, ks, nc, comps);
  lc.n += 2;
}
}  // namespace xcb

// ------------------------------------------------------------------ fft2 (fft.hpp:20-53)
// input staging (c64 / c128 -> c64, conjugated for the inverse) and the
// spectrum's layout B [u/2][v][u%2] -> row-major [v][u] (conjugated and scaled
// 1/(Ph Pw) for the inverse, as Eigen's inverse FFT: conj(FFT(conj x)) / n)
namespace xcb {
namespace {
// tr: the transform runs on the transposed grid (the caller's rows x cols is
// stored row-major; the staged grid is cols x rows)
__global__ void k_fft2_in(const void* __restrict__ src, int c128, int rows, int cols, int tr,
                          int conj_in, float2* __restrict__ dst) {
  const size_t n = size_t(rows) * cols;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const size_t j = tr ? (i % rows) * cols + i / rows : i;
    float2 v = c128 ? make_float2(float(static_cast<const double2*>(src)[j].x),
                                  float(static_cast<const double2*>(src)[j].y))
                    : static_cast<const float2*>(src)[j];
    if (conj_in) v.y = -v.y;
    dst[i] = v;
  }
}

__global__ void k_fft2_out(const float2* __restrict__ hh, int rows, int cols, int tr,
                           int inverse, double scale, int c128, void* __restrict__ out) {
  const size_t n = size_t(rows) * cols;
  const int ph = tr ? cols : rows;  // column-transform length of the staged grid
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int r = int(i / cols), c = int(i % cols);
    const int u = tr ? r : c, v = tr ? c : r;  // staged (row-transform, column-transform) index
    float2 x = hh[(size_t(u >> 1) * ph + v) * 2 + (u & 1)];
    double re = x.x, im = x.y;
    if (inverse) {
      re *= scale;
      im *= -scale;
    }
    if (c128)
      static_cast<double2*>(out)[i] = make_double2(re, im);
    else
      static_cast<float2*>(out)[i] = make_float2(float(re), float(im));
  }
}
}  // namespace

void launch_fft2_in(const void* src, int c128, int rows, int cols, int tr, int conj_in,
                    float2* dst, cudaStream_t st, LaunchCounter& lc) {
  k_fft2_in<<<grid_for(size_t(rows) * cols, 256), 256, 0, st>>>(src, c128, rows, cols, tr,
                                                                conj_in, dst);
  ++lc.n;
}

void launch_fft2_out(const float2* hh, int rows, int cols, int tr, int inverse, int c128,
                     void* out, cudaStream_t st, LaunchCounter& lc) {
  k_fft2_out<<<grid_for(size_t(rows) * cols, 256), 256, 0, st>>>(
      hh, rows, cols, tr, inverse, 1.0 / (double(rows) * cols), c128, out);
  ++lc.n;
}
}  // namespace xcb

// ------------------------------------------------------------------ conjugated spectra
// The DFT of conj(a) is conj(A[-v, -u]): the spectra of the conjugated filter
// components from the cached ones (layout B: ((u / 2) Ph + v) 2 + u % 2), for
// the scatter's conjugate band pairs (kernels.h launch_cols_fwd_mac_inv_cpair).
namespace xcb {
namespace {
__global__ void k_spec_conj_reflect(const float2* __restrict__ F, float2* __restrict__ G, int ph,
                                    int pw, size_t total) {
  const size_t plane = size_t(ph) * pw;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const size_t b = i / plane, e = i - b * plane;
    const int gq = int(e & 1), v = int((e >> 1) % ph), u = int((e >> 1) / ph) * 2 + gq;
    const int vs = v ? ph - v : 0, us = u ? pw - u : 0;
    const float2 x = F[b * plane + (size_t(us >> 1) * ph + vs) * 2 + (us & 1)];
    G[i] = make_float2(x.x, -x.y);
  }
}
}  // namespace

void launch_spec_conj_reflect(const float2* Fhat, float2* Ghat, int nb, int Ph, int Pw,
                              cudaStream_t st, LaunchCounter& lc) {
  const size_t total = size_t(nb) * Ph * Pw;
  k_spec_conj_reflect<<<grid_for(total, 256), 256, 0, st>>>(Fhat, Ghat, Ph, Pw, total);
  ++lc.n;
}
}  // namespace xcb
