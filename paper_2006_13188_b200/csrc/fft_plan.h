// Host-built plans for the shared-memory Stockham FFT (fft_core.cuh).
//
// One CTA transforms kG = 2 sequences of length L held in shared memory
// ([g][phys(n)], phys(n) = n + n/16 to break power-of-two bank strides), in
// two ping-pong buffers.  L = R_0 * R_1 * ... with radices from a
// compile-time codelet set (2..20, 2/3/5-smooth).  The first pass reads the
// input through a functor (global memory), the last pass writes through a
// functor; middle passes go smem -> smem.
#pragma once
#include <cuda_runtime.h>

#include <vector>

namespace xcb {

constexpr int kG = 2;            // sequences per CTA (= interleave of the layouts)
constexpr int kMaxPasses = 6;
constexpr int kMaxThreads = 512;  // __launch_bounds__ of every FFT kernel

struct FftPlanD {
  int L;        // transform length
  int Lp;       // smem stride per sequence (float2 units)
  int npass;
  int nt;       // threads per CTA
  int radix[kMaxPasses];
  int ns[kMaxPasses];            // product of the radices before pass q
  unsigned magic[kMaxPasses];    // ceil(2^32 / ns) for j / ns
  int tw_off[kMaxPasses];        // offset of pass q in the twiddle table
  const float2* tw;              // device twiddles: pass q entry (r-1)*ns + jm
};

struct FftPlan {
  FftPlanD d{};
  std::vector<float2> tw_host;
  bool fast = false;
  size_t smem_bytes() const { return (fast ? 1 : 2) * size_t(kG) * d.Lp * sizeof(float2); }
};

bool is_smooth235(int n);
// Builds a plan for length L (2/3/5-smooth); false if no factorization fits
// the codelet set and thread budget.
bool make_fft_plan(int L, FftPlan* out);
// the same with radices <= max_radix (the 3D tile kernels dispatch 2..10 only)
bool make_fft_plan_maxr(int L, int max_radix, FftPlan* out);
// Fast path (k_fast.cu): transform lengths with a compile-time plan
// (R0 first pass, R1 middle pass or 1, RL last pass).  One kernel instance per
// entry keeps each kernel to a single radix per pass, which is what lets the
// band accumulators stay in registers.  Constraints: one butterfly per thread
// after the first pass, <= 512 threads (128 registers per thread).
#define XCB_FAST_TABLE(X)                                                              \
  X(64, 4, 1, 16) X(128, 8, 1, 16) X(256, 16, 1, 16) X(288, 18, 1, 16)               \
  X(512, 2, 16, 16) X(576, 4, 9, 16) X(1024, 4, 16, 16) X(1152, 8, 9, 16)            \
  X(2048, 8, 16, 16) X(2160, 9, 15, 16) X(2304, 9, 16, 16) X(2880, 12, 15, 16)       \
  X(3072, 12, 16, 16) X(3456, 12, 18, 16)                                            \
  X(4096, 16, 16, 16) X(4320, 12, 18, 20)
bool make_fast_plan(int L, FftPlan* out);
constexpr int kFastMaxThreads = 512;
// Smallest plannable 2/3/5-smooth length >= n (the pad size rule).
int pick_fft_length(int n);

}  // namespace xcb
