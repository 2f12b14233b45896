// Pair engine (device side): one CTA transforms the two interleaved sequences
// of a row pair (layout A) or column pair (layout B / B') of length
// L = R0 * R1 * R2 in three Stockham passes.
//
//   thread t: sequence g = t & 1, butterfly j = t >> 1; T = 2 max(L / Rq)
//   pass 0 (Ns = 1)       : inputs through a functor (a TMA-staged block, TMEM
//                           operands, ...) -> registers -> W0
//   pass 1 (Ns = R0)      : W0 -> W1, twiddles W_{R0 R1}^{(j mod R0) r} (smem)
//   pass 2 (Ns = R0 R1)   : W1 -> outputs k = j + r L/R2, twiddles W_L^{j r}
//                           (per-thread constants: registers or TMEM)
//
// Shared memory keeps the pair interleaved (one float4 = both sequences at one
// index), so adjacent threads read the two halves of the same 16-byte slot
// and every warp access covers whole slots.  One pad slot follows every P
// elements: with R0, L/R1 and L/R2 multiples of P every pass index is
// (thread term) + (compile-time r term), so the per-r offsets are immediates.
// The radix orders and P of XCB_PAIR_TABLE were picked with a bank simulator
// over all passes (4320: conflict-free; 2160: 1.2 wavefronts per ideal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

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

template <int L_, int R0_, int R1_, int R2_, int P_>
struct IlvFft {
  static constexpr int L = L_, R0 = R0_, R1 = R1_, R2 = R2_, P = P_;
  static constexpr int NB0 = L / R0, NB1 = L / R1, NB2 = L / R2;
  static constexpr int T = 2 * ((cmax3(NB0, NB1, NB2) + 15) / 16 * 16);
  static constexpr int TWM = (R1 - 1) * R0;   // pass-1 twiddles [r-1][jm]
  static constexpr int TWL = (R2 - 1) * NB2;  // pass-2 twiddles [r-1][j]
  static constexpr int LP = L + L / P;        // float4 slots per buffer
  // CTAs per SM the band kernels ask for (__launch_bounds__): two when two
  // CTAs' buffers fit in shared memory (short transforms), else one
  // (and two CTAs' warps fit the register file at ~80 registers: T <= 384)
  static constexpr int MINB = (L + 2 * LP) * 16 + TWM * 8 <= 112 * 1024 && T <= 384 ? 2 : 1;
  static constexpr int WPQ = (T / 32 + 3) / 4;  // max warps sharing a TMEM lane quadrant
  // TMEM allocation (power of two >= 32 columns) for kThr columns per thread
  __host__ __device__ static constexpr uint32_t tmem_cols(int kThr) {
    return kThr * WPQ <= 32 ? 32 : kThr * WPQ <= 64 ? 64 : kThr * WPQ <= 128 ? 128
         : kThr * WPQ <= 256 ? 256 : 512;
  }
  static_assert(R0 * R1 * R2 == L, "bad pair plan");
  static_assert(R0 % P == 0 && NB1 % P == 0 && NB2 % P == 0,
                "every pass index must stay linear in r (see lin)");
  __device__ __forceinline__ static int phys(int n) { return n + n / P; }
  // float2 index of (element n, sequence g) in a float4-pair buffer
  __device__ __forceinline__ static int at(int n, int g) { return 2 * phys(n) + g; }
  // float2 offset of + B elements when B is a multiple of P
  template <int B>
  __device__ __forceinline__ static constexpr int lin() { return 2 * (B + B / P); }

  // pass-2 twiddles of thread j in split form r = A a + b: lo[b] = W_L^{j b},
  // hi[a] = W_L^{j A a} (from the split table twl)
  static constexpr int TA = tw_split(R2), TNA = (R2 + TA - 1) / TA;
  static constexpr int TWLS = (TA - 1 + TNA - 1) * NB2;  // split table entries
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
  static constexpr int kTwCols = 2 * (R2 - 1);  // TMEM columns of a full twiddle row
  static constexpr int kTwColsPad = (kTwCols + 3) / 4 * 4;

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
      for (int r = 0; r < R0; ++r) d[2 * (r + r / P)] = v.a[Dft<R0>::pos(r)];
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

  // pass 2: f(a) gets every output of the butterfly, k = j + r NB2 is
  // a[Dft<R2>::pos(r)]; runs on every thread (threads past NB2 compute a
  // dummy butterfly) so f may use warp-collective operations
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
  // the same with the full twiddle row w[r] = W_L^{j r}, r = 1..R2-1 (w[0] unused)
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
};

// Transform lengths with a pair plan: X(L, R0, R1, R2, P).  4320 serves
// configs 3 and 5, 2160 config 4, 1152 config 2.
// XCB_PLAN_1152_ALT (A/B builds, tools/ab_build.py AB_DEFS) selects another
// 1152 plan
#if defined(XCB_PLAN_1152_ALT) && XCB_PLAN_1152_ALT == 1
#define XCB_PAIR_1152(X) X(1152, 8, 12, 12, 8)
#elif defined(XCB_PLAN_1152_ALT) && XCB_PLAN_1152_ALT == 2
#define XCB_PAIR_1152(X) X(1152, 8, 16, 9, 8)
#else
#define XCB_PAIR_1152(X) X(1152, 16, 9, 8, 16)
#endif
// Further lengths (session 5) so that most image sizes find a pair plan within
// ~25% per axis (api.cu pick_pad2d): natural radix orders, R0 = P
#define XCB_PAIR_MORE(X)                                                                 \
  X(288, 8, 6, 6, 8) X(576, 8, 9, 8, 8) X(768, 8, 12, 8, 8) X(1024, 16, 8, 8, 16)          \
  X(1280, 16, 10, 8, 16)                                                                   \
  X(1536, 16, 12, 8, 16) X(1920, 16, 12, 10, 16) X(2048, 16, 16, 8, 16)                    \
  X(2304, 16, 12, 12, 16) X(2560, 16, 16, 10, 16) X(2880, 16, 15, 12, 16)                  \
  X(3072, 16, 16, 12, 16) X(3456, 16, 18, 12, 16)                                          \
  X(4096, 16, 16, 16, 16)
#define XCB_PAIR_TABLE(X) \
  X(4320, 16, 18, 15, 16) X(2160, 12, 15, 12, 12) XCB_PAIR_1152(X) XCB_PAIR_MORE(X)

}  // namespace xcb
