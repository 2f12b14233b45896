// Tensor memory (TMEM, 512 columns x 128 lanes x 32 bit per SM) used as
// per-thread scratch: with the 32x32b access shape each thread of a warp
// reads/writes its own lane (lane = 32 * (warp % 4) + laneid), so warps that
// share a lane quadrant take disjoint column ranges.  The band-loop kernels
// keep their per-thread band accumulators / operands here instead of in
// registers (sm_100a: tcgen05.alloc / ld / st; SASS LDTM / STTM).
#pragma once
#include <cstdint>

#include "tma.cuh"

namespace xcb {

// one full warp: allocate ncols (power of 2, >= 32) columns; base -> *dst
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

// one full warp (the allocating one), after every warp's last TMEM access
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tmem_fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// this warp's lane quadrant in a TMEM address (lane field = bits 31:16)
__device__ __forceinline__ uint32_t tmem_warp_base(uint32_t base) {
  return base + ((32u * ((threadIdx.x >> 5) & 3u)) << 16);
}

// this warp's kThr-column block: lane quadrant warp % 4, column block warp / 4
// (warps of a quadrant side by side).  Broadcast from lane 0 so that ptxas
// keeps it in a uniform register: a per-thread value costs one R2UR per TMEM
// access.
__device__ __forceinline__ uint32_t tmem_warp_cols(uint32_t base, int kThr) {
  const uint32_t a = tmem_warp_base(base) + uint32_t((threadIdx.x >> 7) * kThr);
  return __shfl_sync(0xffffffffu, a, 0);
}

// 4 consecutive columns of this thread's lane (warp-collective)
__device__ __forceinline__ float4 tmem_ld4(uint32_t taddr) {
  uint32_t a, b, c, d;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(taddr)
               : "memory");
  return make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c),
                     __uint_as_float(d));
}

// 2 consecutive columns (one complex value per thread)
__device__ __forceinline__ float2 tmem_ld2(uint32_t taddr) {
  uint32_t a, b;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
               : "=r"(a), "=r"(b)
               : "r"(taddr)
               : "memory");
  return make_float2(__uint_as_float(a), __uint_as_float(b));
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr),
               "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y))
               : "memory");
}
__device__ __forceinline__ void tmem_dep(float2& v) { asm volatile("" : "+f"(v.x), "+f"(v.y)); }

__device__ __forceinline__ void tmem_st4(uint32_t taddr, float4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
               "r"(__float_as_uint(v.w))
               : "memory");
}

// N = 8 / 16 consecutive columns into v[0..N) (warp-collective)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
// N consecutive columns (N a multiple of 4) as the fewest x16 / x8 / x4
// accesses; pair with one tmem_wait_ld / tmem_wait_st
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float* v) {
  static_assert(N % 4 == 0, "columns in multiples of 4");
  int o = 0;
#pragma unroll
  for (; o + 16 <= N; o += 16) tmem_ld16(taddr + o, v + o);
  if constexpr (N % 16 >= 8) {
    tmem_ld8(taddr + (N / 16) * 16, v + (N / 16) * 16);
  }
  if constexpr (N % 8 == 4) {
    const float4 q = tmem_ld4(taddr + N - 4);
    v[N - 4] = q.x;
    v[N - 3] = q.y;
    v[N - 2] = q.z;
    v[N - 1] = q.w;
  }
}
template <int N>
__device__ __forceinline__ void tmem_stn(uint32_t taddr, const float* v) {
  static_assert(N % 4 == 0, "columns in multiples of 4");
#pragma unroll
  for (int o = 0; o + 16 <= N; o += 16) tmem_st16(taddr + o, v + o);
  if constexpr (N % 16 >= 8) tmem_st8(taddr + (N / 16) * 16, v + (N / 16) * 16);
  if constexpr (N % 8 == 4)
    tmem_st4(taddr + N - 4, make_float4(v[N - 4], v[N - 3], v[N - 2], v[N - 1]));
}
template <int N>
__device__ __forceinline__ void tmem_depn(float* v) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+f"(v[i]));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// ties v to the preceding wait::ld so its uses cannot be scheduled above it
__device__ __forceinline__ void tmem_dep(float4& v) {
  asm volatile("" : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w));
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

}  // namespace xcb
