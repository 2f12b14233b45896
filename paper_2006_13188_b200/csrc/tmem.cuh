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
