// Host-side helpers of the pair-engine kernels shared by k_pair.cu (f32x2
// arithmetic) and k_pair_sc.cu (scalar arithmetic): twiddle tables, the
// length dispatch, the tail split, and the TMEM twiddle parking (device).
#pragma once
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "fft_pair.cuh"
#include "tmem.cuh"

namespace xcb {
namespace {

// the thread's full pass-2 twiddle row W_L^{j r} (r = 1..R2-1) into TMEM at ta
// (2 columns each; table twf is [r-1][j], j < NB2); warp-collective
template <class PF>
__device__ __forceinline__ void park_last_tw(const float2* __restrict__ twf, uint32_t ta) {
  const int j = threadIdx.x >> 1;
#pragma unroll
  for (int r = 1; r < PF::R2; ++r)
    tmem_st2(ta + 2 * (r - 1), j < PF::NB2 ? __ldg(twf + (r - 1) * PF::NB2 + j)
                                           : make_float2(1.f, 0.f));
}

constexpr size_t kSmemLimitP = 232448;

// exact twiddle tables of a pair plan (fp64 -> fp32), per device: pass 1
// [r-1][jm] (W_{R0 R1}^{jm r}) and pass 2 [r-1][j] (W_L^{j r}, full rows)
struct PairTw {
  float2* mid = nullptr;
  float2* last = nullptr;
};

template <class PF>
PairTw pair_tables() {
  static std::mutex mu;
  static std::map<int, PairTw> cache;  // device -> tables
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  std::vector<float2> m(PF::TWM), l(PF::TWL);
  const double tp = 6.283185307179586476925286766559;
  auto w = [&](long e, long n) {
    e %= n;
    const double a = -tp * double(e) / double(n);
    return make_float2(float(std::cos(a)), float(std::sin(a)));
  };
  for (int r = 1; r < PF::R1; ++r)
    for (int jm = 0; jm < PF::R0; ++jm) m[(r - 1) * PF::R0 + jm] = w(long(jm) * r, PF::R0 * PF::R1);
  for (int r = 1; r < PF::R2; ++r)
    for (int j = 0; j < PF::NB2; ++j) l[(r - 1) * PF::NB2 + j] = w(long(j) * r, PF::L);
  PairTw p;
  if (cudaMalloc(&p.mid, m.size() * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&p.last, l.size() * sizeof(float2)) != cudaSuccess)
    return PairTw{};
  cudaMemcpy(p.mid, m.data(), m.size() * sizeof(float2), cudaMemcpyHostToDevice);
  cudaMemcpy(p.last, l.data(), l.size() * sizeof(float2), cudaMemcpyHostToDevice);
  cache[dev] = p;
  return p;
}

}  // namespace

#define XCB_PAIR_DISPATCH(LEN, BODY)                                               \
  switch (LEN) {                                                                   \
    XCB_PAIR_TABLE(BODY)                                                           \
    default: break;                                                                \
  }


// Grid of a band-loop kernel with its last, partial wave split into band
// chunks (k_pair.cu tail_split)
struct TailSplit {
  int grid, full, split;
  int slots = 0;  // resident CTAs of the device (SMs * per_sm)
};
// threads: the CTA size, for the co-residency estimate of sub-wave grids
TailSplit tail_split(int units, int per_sm, int nb, int threads = 0);

}  // namespace xcb
