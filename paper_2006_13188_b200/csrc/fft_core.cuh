// Shared-memory mixed-radix Stockham FFT for sm_100a (device side).
//
// Forward transform only (e^{-2 pi i nk/L}); inverse transforms are computed as
// conj(FFT(conj(x))) with the conjugations and the 1/L scale folded into the
// load / store functors of each kernel.  Codelets are compile-time: radices
// 2, 3, 4, 5 hand-written, composites built by Cooley-Tukey in registers with
// constexpr twiddles (folded to immediates after unrolling).
#pragma once
#include <cuda_runtime.h>

#include "fft_plan.h"

namespace xcb {

// ------------------------------------------------------------ complex helpers
// sm_100 issues two fp32 lanes per instruction (FADD2 / FMUL2 / FFMA2,
// PTX add / mul / fma .rn.f32x2 on a 64-bit register pair).  A complex value
// is such a pair, so a complex add is one instruction and a complex multiply
// two; ptxas folds the lane swaps, lane broadcasts and single-lane negations
// that complex arithmetic needs into the operand modifiers (.LO_HI, .F32
// broadcast, partial negate), so they cost nothing.  The band kernels are
// instruction-issue bound (DESIGN 6a), so halving their FP32 instructions is
// the lever.  XCB_F32X2=0 builds the scalar forms (A/B).
#ifndef XCB_F32X2
#define XCB_F32X2 1
#endif
#if XCB_F32X2
__device__ __forceinline__ unsigned long long f2_u(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 u_f2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// lane-wise a + b, a - b, a * b, a * b + c (round to nearest, no ftz)
__device__ __forceinline__ float2 v_add(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u(a)), "l"(f2_u(b)));
  return u_f2(r);
}
__device__ __forceinline__ float2 v_sub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u(a)), "l"(f2_u(b)));
  return u_f2(r);
}
__device__ __forceinline__ float2 v_mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u(a)), "l"(f2_u(b)));
  return u_f2(r);
}
__device__ __forceinline__ float2 v_fma(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_u(a)), "l"(f2_u(b)), "l"(f2_u(c)));
  return u_f2(r);
}
#else
__device__ __forceinline__ float2 v_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 v_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 v_mul(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 v_fma(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
#endif
__device__ __forceinline__ float2 v_bc(float s) { return make_float2(s, s); }  // broadcast
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return v_add(a, b); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return v_sub(a, b); }
// a b = a b.re + (-a.im, a.re) b.im
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return v_fma(make_float2(-a.y, a.x), v_bc(b.y), v_mul(a, v_bc(b.x)));
}
// a * conj(b) = a b.re + (a.im, -a.re) b.im
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {
  return v_fma(make_float2(a.y, -a.x), v_bc(b.y), v_mul(a, v_bc(b.x)));
}
// acc + a b
__device__ __forceinline__ float2 c_fma(float2 a, float2 b, float2 acc) {
  return v_fma(make_float2(-a.y, a.x), v_bc(b.y), v_fma(a, v_bc(b.x), acc));
}
__device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return v_mul(a, v_bc(s)); }
__device__ __forceinline__ float2 c_mi(float2 a) { return make_float2(a.y, -a.x); }  // -i * a

// ------------------------------------------------------ constexpr twiddles
__host__ __device__ constexpr double cx_sin_poly(double x) {
  double x2 = x * x, term = x, sum = x;
  for (int i = 1; i < 12; ++i) {
    term *= -x2 / double((2 * i) * (2 * i + 1));
    sum += term;
  }
  return sum;
}
__host__ __device__ constexpr double cx_cos_poly(double x) {
  double x2 = x * x, term = 1.0, sum = 1.0;
  for (int i = 1; i < 12; ++i) {
    term *= -x2 / double((2 * i - 1) * (2 * i));
    sum += term;
  }
  return sum;
}
// cos / sin of 2 pi a / b, octant-reduced
__host__ __device__ constexpr double cx_cos_frac(long a, long b) {
  a %= b;
  if (a < 0) a += b;
  const long q = (4 * a) / b;                      // quadrant 0..3
  const double x = 6.283185307179586476925286766559 * double(4 * a - q * b) / double(4 * b);
  const double c = x <= 0.78539816339744830962 ? cx_cos_poly(x)
                                               : cx_sin_poly(1.5707963267948966192 - x);
  const double s = x <= 0.78539816339744830962 ? cx_sin_poly(x)
                                               : cx_cos_poly(1.5707963267948966192 - x);
  return q == 0 ? c : q == 1 ? -s : q == 2 ? -c : s;
}
__host__ __device__ constexpr double cx_sin_frac(long a, long b) {
  return cx_cos_frac(4 * a - b, 4 * b);  // sin t = cos(t - pi/2)
}

template <int R>
struct CTw {  // e^{-2 pi i e / R}
  float re[R], im[R];
  __host__ __device__ constexpr CTw() : re(), im() {
    for (int e = 0; e < R; ++e) {
      re[e] = float(cx_cos_frac(e, R));
      im[e] = float(-cx_sin_frac(e, R));
    }
  }
};

__host__ __device__ constexpr int first_factor(int R) {
  return (R % 4 == 0 && R > 4) ? 4 : (R % 2 == 0 && R > 2) ? 2 : (R % 3 == 0 && R > 3) ? 3
                                   : (R % 5 == 0 && R > 5) ? 5 : R;
}

// x * e^{-2 pi i e / R} with the trivial angles (multiples of pi/4) done by
// swaps / negations / one scale instead of a full complex multiply
template <int R>
__device__ __forceinline__ float2 tw_apply(float2 x, int e, const CTw<R>& tw) {
  if (e == 0) return x;
  if ((4 * e) % R == 0) {
    const int q = (4 * e) / R;  // e^{-i pi q / 2}
    return q == 1 ? make_float2(x.y, -x.x) : q == 2 ? make_float2(-x.x, -x.y)
                                                     : make_float2(-x.y, x.x);
  }
  if ((8 * e) % R == 0) {
    constexpr float h = 0.70710678118654752440f;
    const int q = (8 * e) / R;  // odd: e^{-i pi q / 4}
    return q == 1 ? v_mul(v_add(x, c_mi(x)), v_bc(h))
         : q == 3 ? v_mul(v_sub(c_mi(x), x), v_bc(h))
         : q == 5 ? v_mul(v_add(x, c_mi(x)), v_bc(-h))
                  : v_mul(v_sub(x, c_mi(x)), v_bc(h));
  }
  return c_mul(x, make_float2(tw.re[e], tw.im[e]));
}

// ---------------------------------------------------------------- codelets
__host__ __device__ constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
__host__ __device__ constexpr int inv_mod(int a, int m) {  // a^{-1} mod m (gcd(a, m) = 1)
  int r = 1;
  while ((a * r) % m != 1) ++r;
  return r;
}

// Dft<R>::run(v) transforms v in place; output X[k] ends at v[Dft<R>::pos(k)]
// (compile-time permutation), so composites need no second R-element array.
// R = A B with gcd(A, B) = 1 uses the prime-factor (Good-Thomas) mapping:
// input n = (A n2 + B n1) mod R, output k = k1 (mod A), k2 (mod B): no
// twiddle multiplies.  Other composites use Cooley-Tukey with constexpr
// twiddles.
template <int R>
struct Dft {
  static constexpr int A = first_factor(R);
  static constexpr int B = R / A;
  static constexpr bool kPfa = A > 1 && B > 1 && cgcd(A, B) == 1;
  __host__ __device__ static constexpr int pos(int k) {
    // CT: X[k1 + A k2] sits at v[B k1 + pos_B(k2)] after the B-point stage;
    // PFA: X[k] with k1 = k mod A, k2 = k mod B sits at v[B k1 + pos_B(k2)]
    return kPfa ? B * (k % A) + Dft<B>::pos(k % B) : B * (k % A) + Dft<B>::pos(k / A);
  }
  __device__ __forceinline__ static void run(float2* v) {
    if constexpr (kPfa) {
      float2 t[R];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) {
        float2 a[A];
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) a[n1] = v[(A * n2 + B * n1) % R];
        Dft<A>::run(a);
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) t[B * k1 + n2] = a[Dft<A>::pos(k1)];
      }
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) Dft<B>::run(t + B * k1);
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = t[i];
    } else {
      constexpr CTw<R> tw{};
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) {
        float2 a[A];
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) a[n1] = v[B * n1 + n2];
        Dft<A>::run(a);
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) {
          const int e = (n2 * k1) % R;
          const float2 x = a[Dft<A>::pos(k1)];
          v[B * k1 + n2] = tw_apply<R>(x, e, tw);
        }
      }
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) Dft<B>::run(v + B * k1);
    }
  }
};

template <>
struct Dft<1> {
  __host__ __device__ static constexpr int pos(int k) { return k; }
  __device__ __forceinline__ static void run(float2*) {}
};

template <>
struct Dft<2> {
  __host__ __device__ static constexpr int pos(int k) { return k; }
  __device__ __forceinline__ static void run(float2* v) {
    const float2 a = v[0], b = v[1];
    v[0] = c_add(a, b);
    v[1] = c_sub(a, b);
  }
};

template <>
struct Dft<3> {
  __host__ __device__ static constexpr int pos(int k) { return k; }
  __device__ __forceinline__ static void run(float2* v) {
    constexpr float s = 0.86602540378443864676f;  // sin(2 pi / 3)
    const float2 t1 = c_add(v[1], v[2]), t2 = c_sub(v[1], v[2]);
    const float2 m = v_fma(t1, v_bc(-0.5f), v[0]);
    const float2 n = v_mul(c_mi(t2), v_bc(s));  // -i s (x1 - x2)
    v[0] = c_add(v[0], t1);
    v[1] = c_add(m, n);
    v[2] = c_sub(m, n);
  }
};

template <>
struct Dft<4> {
  __host__ __device__ static constexpr int pos(int k) { return k; }
  __device__ __forceinline__ static void run(float2* v) {
    const float2 a = c_add(v[0], v[2]), b = c_sub(v[0], v[2]);
    const float2 c = c_add(v[1], v[3]), d = c_sub(v[1], v[3]);
    v[0] = c_add(a, c);
    v[2] = c_sub(a, c);
    v[1] = c_add(b, c_mi(d));
    v[3] = c_sub(b, c_mi(d));
  }
};

template <>
struct Dft<5> {
  __host__ __device__ static constexpr int pos(int k) { return k; }
  __device__ __forceinline__ static void run(float2* v) {
    constexpr float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
    constexpr float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
    const float2 t1 = c_add(v[1], v[4]), t2 = c_add(v[2], v[3]);
    const float2 t3 = c_sub(v[1], v[4]), t4 = c_sub(v[2], v[3]);
    const float2 x0 = v[0];
    const float2 a1 = v_fma(t1, v_bc(c1), v_fma(t2, v_bc(c2), x0));
    const float2 a2 = v_fma(t1, v_bc(c2), v_fma(t2, v_bc(c1), x0));
    const float2 b1 = v_fma(t3, v_bc(s1), v_mul(t4, v_bc(s2)));
    const float2 b2 = v_fma(t3, v_bc(s2), v_mul(t4, v_bc(-s1)));
    v[0] = c_add(x0, c_add(t1, t2));
    v[1] = c_add(a1, c_mi(b1));
    v[4] = c_sub(a1, c_mi(b1));
    v[2] = c_add(a2, c_mi(b2));
    v[3] = c_sub(a2, c_mi(b2));
  }
};

// --------------------------------------------------------- radix dispatch
template <int N>
struct IntC {
  static constexpr int value = N;
};

// Every radix make_fft_plan may choose (fft_plan.cpp kRadices).
template <class F>
__device__ __forceinline__ void radix_dispatch(int R, F&& f) {
  switch (R) {
    case 2: f(IntC<2>{}); break;
    case 3: f(IntC<3>{}); break;
    case 4: f(IntC<4>{}); break;
    case 5: f(IntC<5>{}); break;
    case 6: f(IntC<6>{}); break;
    case 8: f(IntC<8>{}); break;
    case 9: f(IntC<9>{}); break;
    case 10: f(IntC<10>{}); break;
    case 12: f(IntC<12>{}); break;
    case 15: f(IntC<15>{}); break;
    case 16: f(IntC<16>{}); break;
    case 18: f(IntC<18>{}); break;
    case 20: f(IntC<20>{}); break;
    default: break;
  }
}

__device__ __forceinline__ int sm_phys(int n) { return n + (n >> 4); }

// ------------------------------------------------------------------ passes
// Out-of-place (ping-pong) Stockham: pass q reads buffer q&1 and writes the
// other, so threads loop over butterflies freely.  Butterfly (j, g): inputs
// j + r*L/R, twiddle W_{Ns R}^{(j mod Ns) r}, outputs (j - jm) R + jm + r Ns.

template <int R, class Load>
__device__ __forceinline__ void pass_first(const FftPlanD& p, float2* dst, Load& load) {
  const int nb = p.L / R;
  const int items = nb * kG;
  for (int w = threadIdx.x; w < items; w += blockDim.x) {
    const int g = w & (kG - 1), j = w >> 1;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = load(j + r * nb, g);
    Dft<R>::run(v);
    float2* d = dst + g * p.Lp;
#pragma unroll
    for (int r = 0; r < R; ++r) d[sm_phys(j * R + r)] = v[Dft<R>::pos(r)];
  }
}

__host__ __device__ constexpr int tw_split(int R) {  // smallest A with A*A >= R
  int a = 1;
  while (a * a < R) ++a;
  return a;
}

// Reads the butterfly's R inputs and applies W_{Ns R}^{jm r}, r = A a + b:
// only W^{jm b} (b < A) and W^{jm A a} are loaded from the exact table and
// W^{jm r} = W^{jm A a} W^{jm b} (one rounding), which keeps ~2 sqrt(R)
// twiddles live instead of R - 1.
template <int R>
__device__ __forceinline__ void load_twiddled(const FftPlanD& p, int q, const float2* src,
                                              int j, int jm, float2* v) {
  constexpr int A = tw_split(R);
  constexpr int NA = (R + A - 1) / A;
  const int nb = p.L / R, Ns = p.ns[q];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = src[sm_phys(j + r * nb)];
  const float2* tw = p.tw + p.tw_off[q] + jm;  // entry (r-1)*Ns: W^{jm r}
  float2 lo[A], hi[NA];
  lo[0] = make_float2(1.f, 0.f);
  hi[0] = make_float2(1.f, 0.f);
#pragma unroll
  for (int b = 1; b < A; ++b) lo[b] = __ldg(tw + (b - 1) * Ns);
#pragma unroll
  for (int a = 1; a < NA; ++a) hi[a] = __ldg(tw + (A * a - 1) * Ns);
#pragma unroll
  for (int r = 1; r < R; ++r) {
    const int a = r / A, b = r % A;
    const float2 t = a == 0 ? lo[b] : b == 0 ? hi[a] : c_mul(hi[a], lo[b]);
    v[r] = c_mul(v[r], t);
  }
}

template <int R>
__device__ __noinline__ void pass_mid(const FftPlanD& p, int q, const float2* src,
                                      float2* dst) {
  const int nb = p.L / R, Ns = p.ns[q];
  const int items = nb * kG;
  for (int w = threadIdx.x; w < items; w += blockDim.x) {
    const int g = w & (kG - 1), j = w >> 1;
    const int jm = j - Ns * int(__umulhi(unsigned(j), p.magic[q]));
    float2 v[R];
    load_twiddled<R>(p, q, src + g * p.Lp, j, jm, v);
    Dft<R>::run(v);
    float2* d = dst + g * p.Lp;
    const int base = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) d[sm_phys(base + r * Ns)] = v[Dft<R>::pos(r)];
  }
}

// Last pass (Ns = L/R, so jm = j): output k = j + r*nb -> store(k, g, value).
template <int R, class Store>
__device__ __forceinline__ void pass_last(const FftPlanD& p, int q, const float2* src,
                                          Store& store) {
  const int nb = p.L / R;
  const int items = nb * kG;
  for (int w = threadIdx.x; w < items; w += blockDim.x) {
    const int g = w & (kG - 1), j = w >> 1;
    float2 v[R];
    load_twiddled<R>(p, q, src + g * p.Lp, j, j, v);
    Dft<R>::run(v);
#pragma unroll
    for (int r = 0; r < R; ++r) store(j + r * nb, g, v[Dft<R>::pos(r)]);
  }
}

template <int R, class Load, class Store>
__device__ __forceinline__ void pass_single(Load& load, Store& store) {
  const int g = threadIdx.x;
  if (g < kG) {
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = load(r, g);
    Dft<R>::run(v);
#pragma unroll
    for (int r = 0; r < R; ++r) store(r, g, v[Dft<R>::pos(r)]);
  }
}

// Full forward transform of the CTA's kG sequences: load -> FFT -> store.
// Every thread of the CTA must call it; `sm` holds 2 * kG * p.Lp float2.
// Begins and ends with a barrier-free region: callers reusing `sm` for a
// following transform must __syncthreads() in between.
template <class Load, class Store>
__device__ __forceinline__ void fft_block(const FftPlanD& p, float2* sm, Load& load,
                                          Store& store) {
  if (p.npass == 0) {  // L == 1
    if (threadIdx.x < kG) store(0, threadIdx.x, load(0, threadIdx.x));
    return;
  }
  if (p.npass == 1) {
    radix_dispatch(p.radix[0], [&](auto rc) { pass_single<decltype(rc)::value>(load, store); });
    return;
  }
  float2* buf[2] = {sm, sm + kG * p.Lp};
  radix_dispatch(p.radix[0], [&](auto rc) { pass_first<decltype(rc)::value>(p, buf[0], load); });
  __syncthreads();
  int cur = 0;
  for (int q = 1; q < p.npass - 1; ++q) {
    radix_dispatch(p.radix[q], [&](auto rc) {
      pass_mid<decltype(rc)::value>(p, q, buf[cur], buf[cur ^ 1]);
    });
    cur ^= 1;
    __syncthreads();
  }
  const int ql = p.npass - 1;
  radix_dispatch(p.radix[ql],
                 [&](auto rc) { pass_last<decltype(rc)::value>(p, ql, buf[cur], store); });
}

}  // namespace xcb

namespace xcb {

// ------------------------------------------------------------------ fast path
// Single in-place buffer W ([g][phys(n)], kG * Lp float2):
//   first : load functor -> W            (loops over butterflies)
//   mid   : W -> W in place               (one butterfly per thread, staged
//                                         through registers between barriers)
//   last  : W -> store(k, g, r, value)    (one butterfly per thread: the
//                                         (thread, r) -> k map is the same on
//                                         every call, so callers accumulate
//                                         across bands in registers)
// Plans come from make_fast_plan(L) (XCB_FAST_TABLE in fft_plan.h).

template <int R>
__device__ __forceinline__ void pass_mid_ip(const FftPlanD& p, int q, float2* buf) {
  const int nb = p.L / R, Ns = p.ns[q];
  const int w = threadIdx.x;
  const bool act = w < nb * kG;
  float2 v[R];
  int g = 0, j = 0, jm = 0;
  if (act) {
    g = w & (kG - 1);
    j = w >> 1;
    jm = j - Ns * int(__umulhi(unsigned(j), p.magic[q]));
    load_twiddled<R>(p, q, buf + g * p.Lp, j, jm, v);
    Dft<R>::run(v);
  }
  __syncthreads();
  if (act) {
    float2* d = buf + g * p.Lp;
    const int base = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) d[sm_phys(base + r * Ns)] = v[Dft<R>::pos(r)];
  }
  __syncthreads();
}

__host__ __device__ constexpr int fast_lp(int L) {  // host finalize_plan's stride rule
  int lp = (L - 1) + ((L - 1) >> 4) + 1;
  while (lp % 16 != 8) ++lp;
  return lp;
}

// Compile-time fast plan for length L = R0 * R1 * RL (R1 = 1: two passes):
// every extent, stride, twiddle offset and j mod Ns divisor is a constant, so
// the index arithmetic folds into immediates.  Only the twiddle table pointer
// comes from the host plan (same table layout as finalize_plan).
template <int L_, int R0, int R1, int RL>
struct FastFft {
  static constexpr int L = L_;
  static constexpr int Lp = fast_lp(L_);
  static constexpr int kLast = RL;
  static constexpr int NS1 = R0;                    // Ns of the middle pass
  static constexpr int NSL = R1 > 1 ? R0 * R1 : R0;  // Ns of the last pass
  static_assert(R0 * R1 * RL == L_, "bad fast plan");

  // compact twiddle tables (fft_plan.cpp finalize_plan, fast): per pass,
  // (A-1 + NA-1) entry rows of Ns values, kept in shared memory
  template <int R>
  __host__ __device__ static constexpr int tw_rows() {
    return (tw_split(R) - 1) + ((R + tw_split(R) - 1) / tw_split(R) - 1);
  }
  static constexpr int TWM = R1 > 1 ? tw_rows<R1>() * NS1 : 0;  // mid-pass entries
  static constexpr int TWN = TWM + tw_rows<RL>() * NSL;          // total entries
  static constexpr size_t kTwBytes = size_t(TWN) * sizeof(float2);

  // cooperative copy of the table into smem (call once, then __syncthreads)
  __device__ __forceinline__ static void load_twiddles(float2* sm_tw, const float2* gtw) {
    for (int i = threadIdx.x; i < TWN; i += blockDim.x) sm_tw[i] = __ldg(gtw + i);
  }

  template <int R, int NS, int TWO>
  __device__ __forceinline__ static void load_tw(const float2* twt, const float2* src, int j,
                                                 int jm, float2* v) {
    constexpr int nb = L / R;
    constexpr int A = tw_split(R);
    constexpr int NA = (R + A - 1) / A;
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[sm_phys(j + r * nb)];
    const float2* tw = twt + TWO + jm;
    float2 lo[A], hi[NA];
    lo[0] = make_float2(1.f, 0.f);
    hi[0] = make_float2(1.f, 0.f);
#pragma unroll
    for (int b = 1; b < A; ++b) lo[b] = tw[(b - 1) * NS];
#pragma unroll
    for (int a = 1; a < NA; ++a) hi[a] = tw[(A - 1 + a - 1) * NS];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const int a = r / A, b = r % A;
      const float2 t = a == 0 ? lo[b] : b == 0 ? hi[a] : c_mul(hi[a], lo[b]);
      v[r] = c_mul(v[r], t);
    }
  }

  template <class Load>
  __device__ __forceinline__ static void first(const FftPlanD&, float2* W, Load& load) {
    constexpr int nb = L / R0;
    for (int w = threadIdx.x; w < nb * kG; w += blockDim.x) {
      const int g = w & 1, j = w >> 1;
      float2 v[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) v[r] = load(j + r * nb, g);
      Dft<R0>::run(v);
      float2* d = W + g * Lp;
#pragma unroll
      for (int r = 0; r < R0; ++r) d[sm_phys(j * R0 + r)] = v[Dft<R0>::pos(r)];
    }
  }

  __device__ __forceinline__ static void mid(const float2* twt, float2* W) {
    if constexpr (R1 > 1) {
      constexpr int nb = L / R1;
      const int w = threadIdx.x;
      const bool act = w < nb * kG;
      float2 v[R1];
      int g = 0, j = 0, jm = 0;
      if (act) {
        g = w & 1;
        j = w >> 1;
        jm = j % NS1;
        load_tw<R1, NS1, 0>(twt, W + g * Lp, j, jm, v);
        Dft<R1>::run(v);
      }
      __syncthreads();
      if (act) {
        float2* d = W + g * Lp;
        const int base = (j - jm) * R1 + jm;
#pragma unroll
        for (int r = 0; r < R1; ++r) d[sm_phys(base + r * NS1)] = v[Dft<R1>::pos(r)];
      }
      __syncthreads();
    }
  }

  template <class Store>
  __device__ __forceinline__ static void last(const float2* twt, const float2* W, Store& store) {
    constexpr int nb = L / RL;
    const int w = threadIdx.x;
    if (w < nb * kG) {
      const int g = w & 1, j = w >> 1;
      float2 v[RL];
      load_tw<RL, NSL, TWM>(twt, W + g * Lp, j, j, v);
      Dft<RL>::run(v);
#pragma unroll
      for (int r = 0; r < RL; ++r) store(j + r * nb, g, r, v[Dft<RL>::pos(r)]);
    }
  }
};

}  // namespace xcb
