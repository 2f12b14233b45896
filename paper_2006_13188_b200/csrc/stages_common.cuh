// Shared device helpers of the pipeline stages (included by k_*.cu).
#pragma once
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include "fft_core.cuh"
#include "kernels.h"

namespace xcb {
namespace {

constexpr double kTwoPiHi = 6.283185307179586232;
constexpr double kTwoPiLo = 2.4492935982947064e-16;
constexpr double kInvTwoPi = 0.15915494309189533577;
constexpr double kInvPi = 0.31830988618379067154;

// e^{sign * i * k * base}: the product is formed and reduced to half turns in
// [-1, 1] in double (k*theta is exact for fp32 theta), then evaluated with
// sincospif (accurate to ~1 ulp, no range reduction left to do).
__device__ __forceinline__ float2 steer(int k, double base, float sign) {
  const double ph = double(k) * base;
  const double q = rint(ph * kInvTwoPi);
  double r = fma(-q, kTwoPiHi, ph);
  r = fma(-q, kTwoPiLo, r);
  float s, c;
  sincospif(float(r * kInvPi), &s, &c);
  return make_float2(c, sign * s);
}

// transform-input row/column y' -> source index, or -1 for the zero pad
__device__ __forceinline__ int src_index(int yp, int ext, int n, int R, int periodic) {
  if (yp >= ext) return -1;
  if (!periodic) return yp;
  int y = (yp - R) % n;
  return y < 0 ? y + n : y;
}

// alpha of SIG_PACK: the power of two nearest max|h| (1 for an all-zero h)
__device__ __forceinline__ float pack_alpha(const unsigned* amax) {
  const float m = __uint_as_float(*amax);
  return m > 0.f ? exp2f(rintf(log2f(m))) : 1.f;
}

__device__ __forceinline__ float2 sig_value(const SigSrc& s, size_t i) {
  if (s.mode == SIG_W_ONLY) return make_float2(s.wgt ? s.wgt[i] : 1.f, 0.f);
  if (s.mode == SIG_PACK) {
    const float w = s.wgt ? s.wgt[i] : 1.f;
    return make_float2(static_cast<const float*>(s.sig)[i] * w, pack_alpha(s.amax) * w);
  }
  float2 v = s.is_complex ? static_cast<const float2*>(s.sig)[i]
                          : make_float2(static_cast<const float*>(s.sig)[i], 0.f);
  if (s.mode == SIG_TIMES_W) v = c_scale(v, s.wgt[i]);
  return v;
}

template <class TO>
struct OutOps;
template <>
struct OutOps<float2> {
  __device__ static void put(float2* o, size_t i, float2 v, bool acc, float2 extra) {
    float2 t = c_add(v, extra);
    if (acc) t = c_add(o[i], t);
    o[i] = t;
  }
};
template <>
struct OutOps<double2> {
  __device__ static void put(double2* o, size_t i, float2 v, bool acc, float2 extra) {
    double2 t = make_double2(double(v.x) + double(extra.x), double(v.y) + double(extra.y));
    if (acc) {
      t.x += o[i].x;
      t.y += o[i].y;
    }
    o[i] = t;
  }
};

__device__ __forceinline__ float2 dc_term(const SigSrc& s, size_t i, double dr, double di) {
  if (dr == 0.0 && di == 0.0) return make_float2(0.f, 0.f);
  const float2 h = sig_value(s, i);
  return make_float2(float(dr * h.x - di * h.y), float(dr * h.y + di * h.x));
}

// ------------------------------------------------------------------ programmatic dependent launch
// The pipeline's kernels run back to back on one stream, each consuming the
// previous one's output.  Launched with programmatic stream serialization, a
// kernel's launch and block scheduling overlap the tail and completion of its
// predecessor; pdl_wait() (griddepcontrol.wait, the first statement of every
// kernel launched this way) then blocks until the predecessor grid has
// completed and its writes are visible.  No kernel triggers early, so a
// dependent grid never takes SM slots from blocks of the primary that have not
// run yet.  It shortens the launch-latency-bound small configs (config 1: five
// kernels in a CUDA graph); XCB_PDL=0 uses plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool use_pdl() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class... KArgs, class... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              Args&&... args) {
  if (!use_pdl()) {
    kernel<<<grid, block, smem, st>>>(KArgs(args)...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}

// ------------------------------------------------------------------ launch helpers
// Raise a kernel's dynamic shared memory limit once per (device, kernel) and
// size: the attribute call costs a driver round trip on every launch otherwise.
template <class K>
void set_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(dev, reinterpret_cast<const void*>(kernel));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[key];
  if (have >= bytes) return;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) ==
      cudaSuccess)
    have = bytes;
}

int grid_for(size_t n, int bs) {
  size_t g = (n + bs - 1) / bs;
  if (g > 148 * 32) g = 148 * 32;
  return int(g < 1 ? 1 : g);
}

}  // namespace
}  // namespace xcb
