// Pair engine: one CTA transforms the two interleaved sequences of a row pair
// (layout A) or column pair (layout B) with every thread owning both halves of
// its butterflies, so each element moves as one 16-byte float4 and each
// twiddle serves two points.
//
// Length L = R0 * R1 * R2, three Stockham passes, T = max(L / Rq) threads:
//   pass 0 (Ns = 1)       : inputs through a functor (the band's input block,
//                           TMA-staged into W0 while the previous band's
//                           pass 2 ran), -> registers, barrier, -> W0
//   pass 1 (Ns = R0)      : W0 -> W1, twiddles W_{R0 R1}^{(j mod R0) r} (smem)
//   pass 2 (Ns = R0 R1)   : W1 -> outputs k = j + r L/R2, twiddles W_L^{j r}
// Ping-pong buffers: the next band's input is copied into W0 as soon as
// pass 1 has consumed it, overlapping pass 2; three barriers per band.  Twiddles of pass 2 depend on
// the thread only (j = thread), so they live in registers for the whole band
// loop.  The float4 swizzle keeps every pass's loads and stores conflict-free
// for the tabled radix orders (checked with a bank simulator: 4 wavefronts
// per 512-byte warp access).  Buffers hold LP = L + L/16 float4.
#pragma once
#include <cuda_runtime.h>

#include "fft_core.cuh"

namespace xcb {

// v, opaque to the optimizer: the passes derive their addresses from an
// opaque thread index so that they are recomputed each band instead of being
// hoisted out of the band loop into (spilled) registers
__device__ __forceinline__ int opaque_i(int v) {
  asm volatile("" : "+r"(v));
  return v;
}

__host__ __device__ constexpr int cmax3(int a, int b, int c) {
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

__device__ __forceinline__ float4 ldg_stream4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// predicated 8-byte global store (one STG, no branch)
__device__ __forceinline__ void st_pred(float2* p, float2 v, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.global.v2.f32 [%0], {%1, %2};\n}" ::"l"(p),
      "f"(v.x), "f"(v.y), "r"(int(pred))
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int L_, int R0_, int R1_, int R2_>
struct PairFft {
  static constexpr int L = L_, R0 = R0_, R1 = R1_, R2 = R2_;
  static constexpr int NB0 = L / R0, NB1 = L / R1, NB2 = L / R2;
  static constexpr int T = (cmax3(NB0, NB1, NB2) + 31) / 32 * 32;
  static constexpr int TWM = (R1 - 1) * R0;  // mid-pass twiddle entries [r-1][jm]
  static constexpr int TWL = (R2 - 1) * NB2;  // last-pass twiddle entries [r-1][j]
  static_assert(R0 * R1 * R2 == L, "bad pair plan");

  // float4 element n -> slot: one pad slot per 16 elements.  For the tabled
  // radix orders every pass's index is (thread term) + (compile-time r term)
  // with the r term a multiple of 16, so the offsets stay immediates.
  static constexpr int LP = L + L / 16;
  __device__ __forceinline__ static int phys(int n) { return n + (n >> 4); }

  __device__ __forceinline__ static void split(float4 v, float2& a, float2& b) {
    a = make_float2(v.x, v.y);
    b = make_float2(v.z, v.w);
  }

  // twiddles of pass 2 for thread j, split r = A a + b: lo[b] = W_L^{j b},
  // hi[a] = W_L^{j A a} (kept in registers by the caller; W^{j r} = hi lo)
  static constexpr int TA = tw_split(R2), TNA = (R2 + TA - 1) / TA;
  struct LastTw {
    float2 lo[TA], hi[TNA];
  };
  __device__ __forceinline__ static void load_last_tw(const float2* __restrict__ twl, int j,
                                                      LastTw& tl) {
    tl.lo[0] = tl.hi[0] = make_float2(1.f, 0.f);
#pragma unroll
    for (int b = 1; b < TA; ++b) tl.lo[b] = j < NB2 ? __ldg(twl + (b - 1) * NB2 + j) : tl.lo[0];
#pragma unroll
    for (int a = 1; a < TNA; ++a)
      tl.hi[a] = j < NB2 ? __ldg(twl + (TA * a - 1) * NB2 + j) : tl.lo[0];
  }

  // pass 0 in two halves so that its input may live in W0 itself (TMA
  // staging): compute reads every input into registers, the caller
  // barriers, then store writes W0.  load(n) -> float4, n = j + r NB0.
  struct P0Regs {
    float2 a[R0], b[R0];
  };
  template <class Load>
  __device__ __forceinline__ static void pass0_compute(Load& load, P0Regs& v) {
    const int j = opaque_i(threadIdx.x);
    if (j < NB0) {
#pragma unroll
      for (int r = 0; r < R0; ++r) split(load(j + r * NB0), v.a[r], v.b[r]);
      Dft<R0>::run(v.a);
      Dft<R0>::run(v.b);
    }
  }
  __device__ __forceinline__ static void pass0_store(float4* W0, const P0Regs& v) {
    const int j = opaque_i(threadIdx.x);
    if (j < NB0) {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int p = Dft<R0>::pos(r);
        W0[phys(j * R0 + r)] = make_float4(v.a[p].x, v.a[p].y, v.b[p].x, v.b[p].y);
      }
    }
  }

  __device__ __forceinline__ static void pass1(const float4* W0, float4* W1, const float2* TWs) {
    const int j = opaque_i(threadIdx.x);
    if (j < NB1) {
      const int jm = j % R0;
      float2 a[R1], b[R1];
#pragma unroll
      for (int r = 0; r < R1; ++r) split(W0[phys(j + r * NB1)], a[r], b[r]);
#pragma unroll
      for (int r = 1; r < R1; ++r) {
        const float2 w = TWs[(r - 1) * R0 + jm];
        a[r] = c_mul(a[r], w);
        b[r] = c_mul(b[r], w);
      }
      Dft<R1>::run(a);
      Dft<R1>::run(b);
      const int base = (j - jm) * R1 + jm;
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        const int p = Dft<R1>::pos(r);
        W1[phys(base + r * R0)] = make_float4(a[p].x, a[p].y, b[p].x, b[p].y);
      }
    }
  }

  // pass 2 handing every output of the butterfly to f(a, b) at once:
  // output k = j + r NB2 is a[Dft<R2>::pos(r)] (caller checks j < NB2 itself
  // only if NB2 < T; f runs for all threads so it may use warp-collective ops)
  template <class F>
  __device__ __forceinline__ static void pass2_all(const float4* W1, const LastTw& tl, F& f) {
    const int j = opaque_i(threadIdx.x < NB2 ? threadIdx.x : 0);
    float2 a[R2], b[R2];
#pragma unroll
    for (int r = 0; r < R2; ++r) split(W1[phys(j + r * NB2)], a[r], b[r]);
#pragma unroll
    for (int r = 1; r < R2; ++r) {
      const int ta = r / TA, tb = r % TA;
      const float2 w = ta == 0 ? tl.lo[tb] : tb == 0 ? tl.hi[ta] : c_mul(tl.hi[ta], tl.lo[tb]);
      a[r] = c_mul(a[r], w);
      b[r] = c_mul(b[r], w);
    }
    Dft<R2>::run(a);
    Dft<R2>::run(b);
    f(a, b);
  }

  // pass 2: store(k, r, a, b) for output k = j + r NB2 (same (thread, r) -> k
  // map every call, so callers accumulate in registers indexed by r)
  template <class Store>
  __device__ __forceinline__ static void pass2(const float4* W1, const LastTw& tl,
                                               Store& store) {
    const int j = opaque_i(threadIdx.x);
    if (j < NB2) {
      float2 a[R2], b[R2];
#pragma unroll
      for (int r = 0; r < R2; ++r) split(W1[phys(j + r * NB2)], a[r], b[r]);
#pragma unroll
      for (int r = 1; r < R2; ++r) {
        const int ta = r / TA, tb = r % TA;
        const float2 w = ta == 0 ? tl.lo[tb] : tb == 0 ? tl.hi[ta] : c_mul(tl.hi[ta], tl.lo[tb]);
        a[r] = c_mul(a[r], w);
        b[r] = c_mul(b[r], w);
      }
      Dft<R2>::run(a);
      Dft<R2>::run(b);
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        const int p = Dft<R2>::pos(r);
        store(j + r * NB2, r, a[p], b[p]);
      }
    }
  }
};

// Interleaved variant of the pair engine: same smem layout (float4 = both
// sequences of the pair at one index) and passes, but each sequence of a
// butterfly goes to its own thread (thread t: sequence g = t & 1, butterfly
// j = t >> 1), so T doubles (18 warps for 4320) and per-thread registers
// halve.  Adjacent threads read the two halves of the same float4, so every
// warp access still covers whole 16-byte slots (conflict-free as above).
template <int L_, int R0_, int R1_, int R2_>
struct IlvFft {
  static constexpr int L = L_, R0 = R0_, R1 = R1_, R2 = R2_;
  static constexpr int NB0 = L / R0, NB1 = L / R1, NB2 = L / R2;
  static constexpr int T = 2 * ((cmax3(NB0, NB1, NB2) + 15) / 16 * 16);
  static constexpr int TWM = (R1 - 1) * R0;
  static constexpr int TWL = (R2 - 1) * NB2;
  static constexpr int LP = L + L / 16;
  static_assert(R0 * R1 * R2 == L, "bad pair plan");
  __device__ __forceinline__ static int phys(int n) { return n + (n >> 4); }
  // float2 index of (element n, sequence g) in a float4-pair buffer
  __device__ __forceinline__ static int at(int n, int g) { return 2 * phys(n) + g; }
  // phys(a + b) = phys(a) + b + b / 16 when b is a multiple of 16 (or a is
  // and b < 16): the per-r offsets below are then compile-time immediates
  template <int B>
  __device__ __forceinline__ static constexpr int lin() { return 2 * (B + B / 16); }
  static_assert(R0 % 16 == 0 && NB1 % 16 == 0 && NB2 % 16 == 0,
                "radix order must keep every pass index linear in r (see lin)");

  static constexpr int TA = tw_split(R2), TNA = (R2 + TA - 1) / TA;
  struct LastTw {
    float2 lo[TA], hi[TNA];
  };
  __device__ __forceinline__ static void load_last_tw(const float2* __restrict__ twl,
                                                      LastTw& tl) {
    const int j = threadIdx.x >> 1;
    tl.lo[0] = tl.hi[0] = make_float2(1.f, 0.f);
#pragma unroll
    for (int b = 1; b < TA; ++b) tl.lo[b] = j < NB2 ? __ldg(twl + (b - 1) * NB2 + j) : tl.lo[0];
#pragma unroll
    for (int a = 1; a < TNA; ++a)
      tl.hi[a] = j < NB2 ? __ldg(twl + (TA * a - 1) * NB2 + j) : tl.lo[0];
  }

  struct P0Regs {
    float2 a[R0];
  };
  // load(r, n, g) -> float2 (input n = j + r NB0 of sequence g)
  template <class Load>
  __device__ __forceinline__ static void pass0_compute(Load& load, P0Regs& v) {
    const int t = opaque_i(threadIdx.x), g = t & 1, j = t >> 1;
    if (j < NB0) {
#pragma unroll
      for (int r = 0; r < R0; ++r) v.a[r] = load(r, j + r * NB0, g);
      Dft<R0>::run(v.a);
    }
  }
  __device__ __forceinline__ static void pass0_store(float2* W0, const P0Regs& v) {
    const int t = opaque_i(threadIdx.x), g = t & 1, j = t >> 1;
    if (j < NB0) {
      float2* d = W0 + at(j * R0, g);
#pragma unroll
      for (int r = 0; r < R0; ++r) d[2 * r + 2 * (r / 16)] = v.a[Dft<R0>::pos(r)];
    }
  }

  __device__ __forceinline__ static void pass1(const float2* W0, float2* W1, const float2* TWs) {
    const int t = opaque_i(threadIdx.x), g = t & 1, j = t >> 1;
    if (j < NB1) {
      const int jm = j % R0;
      float2 a[R1];
      const float2* s = W0 + at(j, g);
#pragma unroll
      for (int r = 0; r < R1; ++r) a[r] = s[r * lin<NB1>()];
#pragma unroll
      for (int r = 1; r < R1; ++r) a[r] = c_mul(a[r], TWs[(r - 1) * R0 + jm]);
      Dft<R1>::run(a);
      float2* d = W1 + at((j - jm) * R1 + jm, g);
#pragma unroll
      for (int r = 0; r < R1; ++r) d[r * lin<R0>()] = a[Dft<R1>::pos(r)];
    }
  }

  // f(a) with every output of the butterfly: k = j + r NB2 is a[pos(r)];
  // runs on every thread (threads past NB2 compute a dummy butterfly)
  // pass 2 with the thread's full twiddle row w[r] = W_L^{j r}, r = 1..R2-1
  // (read from TMEM by the caller; w[0] unused)
  template <class F>
  __device__ __forceinline__ static void pass2_all_w(const float2* W1, const float2* w, F& f) {
    const int t = opaque_i(threadIdx.x), g = t & 1;
    const int j = (t >> 1) < NB2 ? (t >> 1) : 0;
    float2 a[R2];
    const float2* s = W1 + at(j, g);
#pragma unroll
    for (int r = 0; r < R2; ++r) a[r] = s[r * lin<NB2>()];
#pragma unroll
    for (int r = 1; r < R2; ++r) a[r] = c_mul(a[r], w[r]);
    Dft<R2>::run(a);
    f(a);
  }
  static constexpr int kTwCols = 2 * (R2 - 1);  // TMEM columns of the full twiddle row
  static constexpr int kTwColsPad = (kTwCols + 3) / 4 * 4;

  template <class F>
  __device__ __forceinline__ static void pass2_all(const float2* W1, const LastTw& tl, F& f) {
    const int t = opaque_i(threadIdx.x), g = t & 1;
    const int j = (t >> 1) < NB2 ? (t >> 1) : 0;
    float2 a[R2];
    const float2* s = W1 + at(j, g);
#pragma unroll
    for (int r = 0; r < R2; ++r) a[r] = s[r * lin<NB2>()];
#pragma unroll
    for (int r = 1; r < R2; ++r) {
      const int ta = r / TA, tb = r % TA;
      const float2 w = ta == 0 ? tl.lo[tb] : tb == 0 ? tl.hi[ta] : c_mul(tl.hi[ta], tl.lo[tb]);
      a[r] = c_mul(a[r], w);
    }
    Dft<R2>::run(a);
    f(a);
  }
};

// Transform lengths with a pair plan: X(L, R0, R1, R2).  Radix orders are the
// bank-conflict-free ones for the float4 swizzle.
#define XCB_PAIR_TABLE(X) X(4320, 16, 18, 15)

}  // namespace xcb
