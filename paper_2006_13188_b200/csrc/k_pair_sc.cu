// Pair-engine stages built with scalar fp32 arithmetic (XCB_F32X2 = 0):
// I1 (k_cols_inv_corr_ilv) and the angle-max planes (k_rows_inv_planes_ilv).
// Both end in predicated global stores of conj(FFT) outputs; with the packed
// FADD2 / FFMA2 forms (fft_core.cuh) they measured slower at base clocks
// (config 5 I1 6225 -> 6656 us, planes 1314 -> 1402 us) while I2 / S1 / S2
// gained (4939 -> 4786, 142 -> 139, 133 -> 127 us), so each translation unit
// picks its form.  Device code is compiled per unit (no -rdc), so the two
// definitions of the inline helpers never meet.
#define XCB_F32X2 0
#include <cstdlib>

#include "fft_pair.cuh"
#include "kernels.h"
#include "pair_host.cuh"
#include "pair_i1.cuh"
#include "stages_common.cuh"
#include "tma.cuh"
#include "tmem.cuh"

namespace xcb {
namespace {

template <class PF, int NI>
__global__ void __launch_bounds__(PF::T, PF::MINB)
    k_cols_inv_corr_ilv(Geo g, const float4* __restrict__ Hh, size_t hstride4,
                        const float4* __restrict__ Fh, size_t sstride4, Bands bl,
                        float2* __restrict__ T2, size_t tstride,
                        const float2* __restrict__ twm, const float2* __restrict__ twf,
                        int full, int split) {
  pdl_wait();
  // CTAs below `full` run every band of column pair blockIdx.x; the column
  // pairs of the last, partial wave are split into `split` band chunks so the
  // tail spreads over all SMs (CTAs are dispatched in blockIdx order)
  int c = blockIdx.x, b0 = 0, b1 = bl.n;
  if (c >= full) {
    const int u = c - full, ch = u % split;
    c = full + u / split;
    b0 = ch * bl.n / split;
    b1 = (ch + 1) * bl.n / split;
  }
  i1_body<PF, NI>(c, b0, b1, g, Hh, hstride4, Fh, sstride4, bl, T2, tstride, twm, twf);
}

// ------------------------------------------------------------------ planes (interleaved)
// Angle-max front end: per band, row IFFT of T2_b, crop, store the band plane
// G_b = H * F_b (engine.hpp:304-311 per band); k_anglemax_* then reads all
// bands per pixel.  Same engine as I2 without the steering; a warp's store
// covers 16 consecutive pixels of both rows (two full 128-byte lines).
template <class PF>
__global__ void __launch_bounds__(PF::T, PF::MINB)
    k_rows_inv_planes_ilv(Geo g, const float4* __restrict__ T2, int nbands,
                          float2* __restrict__ planes, float scale,
                          const float2* __restrict__ twm, const float2* __restrict__ twl) {
  pdl_wait();
  constexpr int L = PF::L;  // = Pw
  constexpr int R2 = PF::R2;
  extern __shared__ __align__(16) float4 smp[];
  float4* ST4 = smp;
  float4* W04 = ST4 + L;
  float4* W14 = W04 + PF::LP;
  float2* TWs = reinterpret_cast<float2*>(W14 + PF::LP);
  const float2* ST = reinterpret_cast<const float2*>(ST4);
  float2* W0 = reinterpret_cast<float2*>(W04);
  float2* W1 = reinterpret_cast<float2*>(W14);
  const int b = blockIdx.x, t = threadIdx.x;
  const size_t plane4 = size_t(g.H2 / 2) * g.Pw;
  const float4* rowp = T2 + size_t(b) * g.Pw;
  constexpr unsigned kBytes = unsigned(L * sizeof(float4));
  __shared__ __align__(8) uint64_t bar;
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, kBytes);
    bulk_copy(ST4, rowp, kBytes, &bar);
    if (nbands > 1) prefetch_l2(rowp + plane4, kBytes);
  }
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  typename PF::LastTw tl;
  PF::load_last_tw(twl, tl);
  __syncthreads();
  const size_t npix = size_t(g.H) * g.W;
  unsigned phase = 0;
  for (int bi = 0; bi < nbands; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    auto load = [&](int, int n, int gi) -> float2 { return c_conj(ST[2 * n + gi]); };
    {
      typename PF::P0Regs v;
      PF::pass0_compute(load, v);
      PF::pass0_store(W0, v);
    }
    __syncthreads();
    if (t == 0 && bi + 1 < nbands) {
      fence_proxy_async();
      mbar_expect_tx(&bar, kBytes);
      bulk_copy(ST4, rowp + size_t(bi + 1) * plane4, kBytes, &bar);
      if (bi + 2 < nbands) prefetch_l2(rowp + size_t(bi + 2) * plane4, kBytes);
    }
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    const int tt = opaque_i(t), gi = tt & 1, j = tt >> 1, y = 2 * b + gi;
    const int x0 = j - g.off;
    float2* o = planes + size_t(bi) * npix + size_t(y) * g.W + x0;
    const bool act = j < PF::NB2 && y < g.H;
    auto store = [&](float2 (&a)[R2]) {
      int x = opaque_i(x0);
      float2* p = o;
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        st_pred(p, c_scale(c_conj(a[Dft<R2>::pos(r)]), scale),
                act && unsigned(x) < unsigned(g.W));
        x += PF::NB2;
        p += PF::NB2;
      }
    };
    PF::pass2_all(W1, tl, store);
  }
}
}  // namespace

void launch_cols_inv_corr_pair(const Geo& g, const float2* Hhat, const float2* Fhat,
                               size_t sstride, const Bands& b, float2* T2, cudaStream_t st,
                               LaunchCounter& lc, int nimg, size_t hstride, size_t tstride) {
  const size_t sm = pair_smem(0, g.Ph, g);
  const float4* hh = reinterpret_cast<const float4*>(Hhat);
  const float4* fh = reinterpret_cast<const float4*>(Fhat);
  const int ncol = g.Pw / 2;
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    const TailSplit ts = tail_split(ncol, PF::MINB, b.n, PF::T);                                   \
    if (nimg == 2) {                                                                        \
      set_smem(k_cols_inv_corr_ilv<PF, 2>, sm);                                             \
      launch_k(k_cols_inv_corr_ilv<PF, 2>, ts.grid, PF::T, sm, st,                                \
          g, hh, hstride / 2, fh, sstride / 2, b, T2, tstride, tw.mid, tw.last, ts.full,    \
          ts.split);                                                                        \
    } else {                                                                                \
      set_smem(k_cols_inv_corr_ilv<PF, 1>, sm);                                             \
      launch_k(k_cols_inv_corr_ilv<PF, 1>, ts.grid, PF::T, sm, st,                                \
          g, hh, hstride / 2, fh, sstride / 2, b, T2, tstride, tw.mid, tw.last, ts.full,    \
          ts.split);                                                                        \
    }                                                                                       \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Ph, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_rows_inv_planes_pair(const Geo& g, const float2* T2, int nbands, float2* planes,
                                 cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = pair_smem(2, g.Pw, g);
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    set_smem(k_rows_inv_planes_ilv<PF>, sm);                                                \
    launch_k(k_rows_inv_planes_ilv<PF>, g.H2 / 2, PF::T, sm, st,                                  \
        g, reinterpret_cast<const float4*>(T2), nbands, planes, scale, tw.mid, tw.last);    \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Pw, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

}  // namespace xcb
