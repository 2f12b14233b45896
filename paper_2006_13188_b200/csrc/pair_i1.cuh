// I1 device body (column IFFT of conj(H^) F^_k per band -> T2), shared by
// the I1 kernel (k_pair_sc.cu) and the opt-in dual kernel (k_pair.cu).
#pragma once
#include "fft_pair.cuh"
#include "pair_host.cuh"
#include "stages_common.cuh"
#include "tma.cuh"
#include "tmem.cuh"

namespace xcb {
namespace {

// ------------------------------------------------------------------ I1 (interleaved)
// conj(H^) of NI images at the thread's pass-0 inputs is parked in TMEM for
// the whole band loop; F^_k is TMA-staged once per band and applied to all NI
// images (the filter spectrum is image-independent, so its HBM read is shared).
// Per (band, image): two barriers (after pass 0, after pass 1).
template <class PF, int NI>
__device__ __forceinline__ void i1_body(int c, int b0, int b1, const Geo& g,
                                        const float4* __restrict__ Hh,
                                        size_t hstride4, const float4* __restrict__ Fh,
                                        size_t sstride4, const Bands& bl,
                                        float2* __restrict__ T2, size_t tstride,
                                        const float2* __restrict__ twm,
                                        const float2* __restrict__ twf) {
  constexpr int L = PF::L;  // = Ph
  // TMEM per thread: conj(H^) (2 R0 columns per image), then the pass-2
  // twiddle row; warps of a lane quadrant side by side (up to 5 of 18)
  constexpr int kThr = NI * 2 * PF::R0 + PF::kTwColsPad;
  constexpr uint32_t kCols = PF::tmem_cols(kThr);
  static_assert(kThr * PF::WPQ <= 512, "TMEM budget");
  extern __shared__ __align__(16) float4 smp[];
  float4* ST4 = smp;  // staged F^_k column pair, natural order
  float4* W04 = ST4 + L;
  float4* W14 = W04 + PF::LP;
  float2* TWs = reinterpret_cast<float2*>(W14 + PF::LP);
  const float2* ST = reinterpret_cast<const float2*>(ST4);
  float2* W0 = reinterpret_cast<float2*>(W04);
  float2* W1 = reinterpret_cast<float2*>(W14);
  const int t = threadIdx.x;
  const size_t plane = size_t(g.H2) * g.Pw;  // float2 per T2 band plane
  constexpr unsigned kBytes = unsigned(L * sizeof(float4));
  auto fsrc = [&](int bi) { return Fh + size_t(bl.spec[bi]) * sstride4 + size_t(c) * L; };
  __shared__ __align__(8) uint64_t bar;
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, kBytes);
    bulk_copy(ST4, fsrc(b0), kBytes, &bar);
    if (b0 + 1 < b1) prefetch_l2(fsrc(b0 + 1), kBytes);
  }
  // conj(H^) at this thread's pass-0 inputs n = j + r NB0, parked in TMEM
  // (2 columns per r and image; warps of a lane quadrant side by side)
  __shared__ uint32_t tbase;
  if (t < 32) tmem_alloc(&tbase, kCols);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t thc = tmem_warp_base(tbase) + uint32_t((t >> 7) * kThr);
  const uint32_t ttw = thc + NI * 2 * PF::R0;
  {
    const int gi = t & 1, j = t >> 1;
#pragma unroll
    for (int im = 0; im < NI; ++im) {
      const float2* hcol = reinterpret_cast<const float2*>(Hh + im * hstride4 + size_t(c) * L) + gi;
#pragma unroll
      for (int r = 0; r < PF::R0; ++r)
        tmem_st2(thc + 2 * (im * PF::R0 + r),
                 j < PF::NB0 ? c_conj(__ldg(hcol + 2 * (j + r * PF::NB0))) : make_float2(0.f, 0.f));
    }
    park_last_tw<PF>(twf, ttw);
    tmem_wait_st();
  }
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  __syncthreads();
  unsigned phase = 0;
  for (int bi = b0; bi < b1; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
#pragma unroll 1
    for (int im = 0; im < NI; ++im) {
      // conj(H^ conj(F^)) = conj(H^) F^ : inverse via conj-FFT-conj
      {
        float2 hc[PF::R0];
        const uint32_t ta = thc + 2 * PF::R0 * opaque_i(im);
        tmem_ldn<2 * PF::R0>(ta, reinterpret_cast<float*>(hc));
        tmem_wait_ld();
        tmem_depn<2 * PF::R0>(reinterpret_cast<float*>(hc));
        auto load = [&](int r, int n, int gi) -> float2 { return c_mul(hc[r], ST[2 * n + gi]); };
        typename PF::P0Regs v;
        PF::pass0_compute(load, v);
        PF::pass0_store(W0, v);
      }
      __syncthreads();
      if (t == 0 && im == NI - 1 && bi + 1 < b1) {
        fence_proxy_async();
        mbar_expect_tx(&bar, kBytes);
        bulk_copy(ST4, fsrc(bi + 1), kBytes, &bar);
        if (bi + 2 < b1) prefetch_l2(fsrc(bi + 2), kBytes);
      }
      PF::pass1(W0, W1, TWs);
      __syncthreads();
      const int tt = opaque_i(t), gi = tt & 1, j = tt >> 1;
      // output y = j + r NB2 - off: NB2 is even, so y & 1 is fixed and y >> 1
      // advances by NB2 / 2 rows of T2 per r
      const int y0 = j - g.off;
      const int rstride = (PF::NB2 / 2) * 2 * g.Pw;  // float2 per r step (< 2^31: one plane)
      float2* o = T2 + im * tstride + size_t(bi) * plane + 2 * (2 * c + gi) +
                  (ptrdiff_t(y0 >> 1) * (2 * g.Pw) + (y0 & 1));
      const bool act = j < PF::NB2;
      auto store = [&](float2 (&a)[PF::R2]) {
        int y = opaque_i(y0);
        float2* p = o;
#pragma unroll
        for (int r = 0; r < PF::R2; ++r) {
          st_pred(p, c_conj(a[Dft<PF::R2>::pos(r)]), act && unsigned(y) < unsigned(g.H));
          y += PF::NB2;
          p += rstride;
        }
      };
      float2 w[PF::kTwColsPad / 2 + 1];
      tmem_ldn<PF::kTwColsPad>(ttw, reinterpret_cast<float*>(w + 1));
      tmem_wait_ld();
      tmem_depn<PF::kTwColsPad>(reinterpret_cast<float*>(w + 1));
      PF::pass2_all_w(W1, w, store);
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (t < 32) {
    tmem_fence_after_sync();
    tmem_dealloc(tbase, kCols);
  }
}

}  // namespace
}  // namespace xcb
