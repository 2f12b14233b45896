// Band-loop stages on the pair engine (fft_pair.cuh) for the lengths of
// XCB_PAIR_TABLE.  One CTA per SM transforms a row pair or column pair; the
// next band's input block is TMA-staged (cp.async.bulk + mbarrier) while the
// current band's passes run, and the band after that is prefetched into L2.
// Per-thread operands that are fixed for the whole band loop live in TMEM
// (tcgen05.alloc / ld / st, tmem.cuh) instead of registers.
//   I1 k_cols_inv_corr_ilv  : per band, column IFFT of conj(H^) F^_k (the
//        spectral multiply of fft.hpp:94-97 fused into pass 0) -> T2_k
//   I2 k_rows_inv_steer_ilv : per band, row IFFT of T2_k, crop, Horner steering
//        over the bands sorted by descending k (engine.hpp:312-317), band sums
//        in TMEM; the output is written once
//   planes k_rows_inv_planes_ilv : per band, row IFFT of T2_k -> G_k planes
//        (angle max)
//   S1 k_rows_fwd_premul_ilv : per band, row FFT of H e^{-i k phi}
//        (engine.hpp:353-358) with the phasor recurrence in TMEM -> T1_k
//   S2 k_cols_fwd_mac_ilv    : per band, column FFT of T1_k times F^_k summed
//        over the bands in TMEM (the reference's B inverse FFTs collapse into
//        one, engine.hpp:359-366), then one inverse column FFT -> T2
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "fft_pair.cuh"
#include "pair_host.cuh"
#include "pair_i1.cuh"
#include "stages_common.cuh"
#include "tma.cuh"
#include "tmem.cuh"

namespace xcb {
namespace {


// ------------------------------------------------------------------ I2 (interleaved)
// TMEM per thread: the band accumulator and the steering phasor z = e^{i phi}
// of each pass-2 output (4 columns per output r), then the pass-2 twiddle row
// W_L^{j r} (one x28 load per band instead of products of split-table
// entries: 0.6% faster at fixed clocks); warps of a lane quadrant side by side.
template <class PF, class TO>
__device__ __forceinline__ void i2_body(int b, const Geo& g, const float4* __restrict__ T2,
                                        const Bands& bl, int half,
                                        const double* __restrict__ base, TO* __restrict__ out,
                                        int accumulate, const SigSrc& dcs, double dcr,
                                        double dci, float scale,
                                        const float2* __restrict__ twm,
                                        const float2* __restrict__ twl) {
  constexpr int L = PF::L;  // = Pw
  constexpr int R2 = PF::R2;
  static_assert(2 * PF::NB2 <= PF::T, "pass 2: one butterfly per thread");
  // TMEM columns per thread: (acc, z) per output r, then the pass-2 twiddle row
  constexpr int kThr = 4 * R2 + PF::kTwColsPad;
  static_assert(kThr * PF::WPQ <= 512, "TMEM budget");
  extern __shared__ __align__(16) float4 smp[];
  float4* ST4 = smp;  // staged T2 row pair, natural order
  float4* W04 = ST4 + L;
  float4* W14 = W04 + PF::LP;
  float2* TWs = reinterpret_cast<float2*>(W14 + PF::LP);
  const float2* ST = reinterpret_cast<const float2*>(ST4);
  float2* W0 = reinterpret_cast<float2*>(W04);
  float2* W1 = reinterpret_cast<float2*>(W14);
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  const size_t plane4 = size_t(g.H2 / 2) * g.Pw;  // float4 per band plane
  const float4* rowp = T2 + size_t(b) * g.Pw;
  constexpr unsigned kBytes = unsigned(L * sizeof(float4));
  __shared__ __align__(8) uint64_t bar;
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, kBytes);
    bulk_copy(ST4, rowp, kBytes, &bar);
    if (bl.n > 1) prefetch_l2(rowp + plane4, kBytes);
  }
  if (t < 32) tmem_alloc(&tbase, PF::tmem_cols(kThr));
  const int gi = t & 1, j = t >> 1, y = 2 * b + gi;
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  // per output r: columns [acc.re, acc.im, z.re, z.im], z = e^{i phi}
  const uint32_t tacc = tmem_warp_cols(tbase, kThr);
  park_last_tw<PF>(twl, tacc + 4 * R2);
  // the thread's R2 phases: one batch of independent loads (the TMEM stores
  // are asm volatile, so loads interleaved with them would serialise)
  auto in_image = [&](int r) {
    const int x = j + r * PF::NB2 - g.off;
    return j < PF::NB2 && x >= 0 && x < g.W && y < g.H;
  };
  auto load_phases = [&](double (&th)[R2]) {
#pragma unroll
    for (int r = 0; r < R2; ++r)
      th[r] = in_image(r) ? __ldg(base + size_t(y) * g.W + (j + r * PF::NB2 - g.off)) : 0.0;
  };
  {
    double th[R2];
    load_phases(th);
#pragma unroll
    for (int r = 0; r < R2; ++r)
      tmem_st2(tacc + 4 * r + 2, in_image(r) ? steer(1, th[r], 1.f) : make_float2(1.f, 0.f));
  }
  tmem_wait_st();
  unsigned phase = 0;
  for (int bi = 0; bi < bl.n; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    auto load = [&](int, int n, int gi2) -> float2 { return c_conj(ST[2 * n + gi2]); };
    {
      typename PF::P0Regs v;
      PF::pass0_compute(load, v);
      PF::pass0_store(W0, v);
    }
    __syncthreads();
    if (t == 0 && bi + 1 < bl.n) {
      fence_proxy_async();
      mbar_expect_tx(&bar, kBytes);
      bulk_copy(ST4, rowp + size_t(bi + 1) * plane4, kBytes, &bar);
      if (bi + 2 < bl.n) prefetch_l2(rowp + size_t(bi + 2) * plane4, kBytes);
    }
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    const int dk = bi == 0 ? 0 : bl.k[bi - 1] - bl.k[bi];
    // Hermitian half-band mode: the k = 0 band enters with weight 1/2 (a
    // CTA-uniform branch, so the other bands carry no scaling multiplies)
    const bool hz = half && bl.k[bi] == 0;
    // acc = acc z^dk + conj(v)  (Horner over descending k; IFFT = conj FFT conj)
    auto horner = [&](float2 (&a)[R2]) {
      if (hz) {
#pragma unroll
        for (int r = 0; r < R2; ++r) a[r] = c_scale(a[r], 0.5f);
      }
      constexpr int C = 5;  // outputs per TMEM round trip
#pragma unroll
      for (int r0 = 0; r0 < R2; r0 += C) {
        float4 az[C];  // (acc, z)
        float2 acc[C];
        if (bi > 0) {
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) az[i] = tmem_ld4(tacc + 4 * (r0 + i));
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) tmem_dep(az[i]);
        }
#pragma unroll
        for (int i = 0; i < C; ++i) {
          const int r = r0 + i;
          if (r >= R2) break;
          const float2 va = a[Dft<R2>::pos(r)];
          if (bi == 0) {
            acc[i] = c_conj(va);
            continue;
          }
          float2 pa = make_float2(az[i].x, az[i].y);
          const float2 zr = make_float2(az[i].z, az[i].w);
          if (dk == 1) {
            pa = c_fma(pa, zr, c_conj(va));
          } else {
            float2 za = zr;
            int d = dk;
            if (d < 0) {
              za = c_conj(za);
              d = -d;
            }
            for (int s = 0; s < d; ++s) pa = c_mul(pa, za);
            pa = c_add(pa, c_conj(va));
          }
          acc[i] = pa;
        }
#pragma unroll
        for (int i = 0; i < C; ++i)
          if (r0 + i < R2) tmem_st2(tacc + 4 * (r0 + i), acc[i]);
      }
      tmem_wait_st();
    };
    float2 w[PF::kTwColsPad / 2 + 1];
    tmem_ldn<PF::kTwColsPad>(tacc + 4 * R2, reinterpret_cast<float*>(w + 1));
    tmem_wait_ld();
    tmem_depn<PF::kTwColsPad>(reinterpret_cast<float*>(w + 1));
    PF::pass2_all_w(W1, w, horner);
  }
  // out = scale * z^{k_last} * acc (+ conj(dc) H for the scale group)
  {
    const int klast = bl.k[bl.n - 1];
    constexpr int C = 5;  // outputs per batch of loads
#pragma unroll
    for (int r0 = 0; r0 < R2; r0 += C) {
      double th[C];
      float az[4 * C];  // (acc, z) per output
#pragma unroll
      for (int i = 0; i < C; ++i)
        th[i] = r0 + i < R2 && in_image(r0 + i)
                    ? __ldg(base + size_t(y) * g.W + (j + (r0 + i) * PF::NB2 - g.off))
                    : 0.0;
      tmem_ldn<4 * C>(tacc + 4 * r0, az);
      tmem_wait_ld();
      tmem_depn<4 * C>(az);
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int r = r0 + i;
        if (r >= R2 || !in_image(r)) continue;
        const float2 acc = make_float2(az[4 * i], az[4 * i + 1]);
        const size_t o = size_t(y) * g.W + (j + r * PF::NB2 - g.off);
        float2 v = c_scale(c_mul(acc, steer(klast, th[i], 1.f)), scale);
        if (half) v = make_float2(2.f * v.x, 0.f);  // out = G_0 + 2 Re sum_{k>0} (real)
        OutOps<TO>::put(out, o, v, accumulate != 0, dc_term(dcs, o, dcr, dci));
      }
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (t < 32) {
    tmem_fence_after_sync();
    tmem_dealloc(tbase, PF::tmem_cols(kThr));
  }
}

template <class PF, class TO>
__global__ void __launch_bounds__(PF::T, PF::MINB)
    k_rows_inv_steer_ilv(Geo g, const float4* __restrict__ T2, Bands bl, int half,
                         const double* __restrict__ base, TO* __restrict__ out, int accumulate,
                         SigSrc dcs, double dcr, double dci, float scale,
                         const float2* __restrict__ twm, const float2* __restrict__ twl) {
  pdl_wait();
  i2_body<PF, TO>(blockIdx.x, g, T2, bl, half, base, out, accumulate, dcs, dcr, dci, scale, twm,
                  twl);
}

// ------------------------------------------------------------------ I1 + I2 (dual)
// One launch runs I1 of image n+1 and I2 of image n, their CTAs interleaved
// by block index, so every SM alternates between the HBM-heavy I1 (filter
// spectra in, T2 out) and the FP32-bound I2: the two kernels' bottlenecks
// overlap instead of following each other.  Same engine, same shared-memory
// layout and TMEM budget; n1 I1 column pairs, n2 I2 row pairs.
struct I1Args {
  const float4* Hh;
  const float4* Fh;
  size_t sstride4;
  Bands bl;
  float2* T2;
};
template <class TO>
struct I2Args {
  const float4* T2;
  Bands bl;
  int half;
  const double* base;
  TO* out;
  int accumulate;
  SigSrc dcs;
  double dcr, dci;
  float scale;
};

template <class PF, class TO>
__global__ void __launch_bounds__(PF::T, 1)
    k_dual_ilv(Geo g, I1Args a, I2Args<TO> b, int n1, int n2, const float2* __restrict__ twm,
               const float2* __restrict__ twl, const float2* __restrict__ twf) {
  pdl_wait();
  const int x = blockIdx.x, m = n1 < n2 ? n1 : n2;
  bool first;
  int item;
  if (x < 2 * m) {
    first = (x & 1) == 0;
    item = x >> 1;
  } else {
    first = n1 > m;
    item = x - m;
  }
  if (first)
    i1_body<PF, 1>(item, 0, a.bl.n, g, a.Hh, 0, a.Fh, a.sstride4, a.bl, a.T2, 0, twm, twf);
  else
    i2_body<PF, TO>(item, g, b.T2, b.bl, b.half, b.base, b.out, b.accumulate, b.dcs, b.dcr, b.dci,
                    b.scale, twm, twl);
}


// ------------------------------------------------------------------ S1 (interleaved)
// TMEM per thread, for each pass-0 input r: [cur.re, cur.im, mul.re, mul.im]
// with cur = H e^{-i k phi} of the current band and mul = e^{-i phi}.
// TWR (short rows, S1Occ): the pass-2 twiddles stay in registers in split
// form instead of TMEM, so the TMEM allocation admits 3 CTAs per SM
template <class PF>
struct S1Occ {
  static constexpr bool kTwReg = PF::L < 2048;
  static constexpr int kMinB = kTwReg && PF::T <= 288 ? 3 : PF::MINB;
};

template <class PF>
__global__ void __launch_bounds__(PF::T, S1Occ<PF>::kMinB)
    k_rows_fwd_premul_ilv(Geo g, SigSrc s, const double* __restrict__ base, Bands bl,
                          float2* __restrict__ T1, const float2* __restrict__ twm,
                          const float2* __restrict__ twl, int full, int split) {
  pdl_wait();
  constexpr int R0 = PF::R0, R2 = PF::R2;
  constexpr bool TWR = S1Occ<PF>::kTwReg;
  // TMEM columns per thread: [cur, mul] per pass-0 input, then (unless TWR)
  // the pass-2 twiddle row (out of the registers: no spills at 2 CTAs per SM)
  constexpr int kThr = 4 * R0 + (TWR ? 0 : PF::kTwColsPad);
  static_assert(kThr * PF::WPQ <= 512, "TMEM budget");
  extern __shared__ __align__(16) float4 smp[];
  float4* W04 = smp;
  float4* W14 = W04 + PF::LP;
  float2* TWs = reinterpret_cast<float2*>(W14 + PF::LP);
  float2* W0 = reinterpret_cast<float2*>(W04);
  float2* W1 = reinterpret_cast<float2*>(W14);
  __shared__ uint32_t tbase;
  // row pairs below `full` run every band; the pairs of the last, partial
  // wave are split into `split` band chunks (tail_split) so the tail fills
  // the SMs
  int b = blockIdx.x, b0 = 0, b1 = bl.n;
  if (b >= full) {
    const int u = b - full, ch = u % split;
    b = full + u / split;
    b0 = ch * bl.n / split;
    b1 = (ch + 1) * bl.n / split;
  }
  const int t = threadIdx.x;
  if (t < 32) tmem_alloc(&tbase, PF::tmem_cols(kThr));
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const int gi = t & 1, j = t >> 1;
  const uint32_t tc = tmem_warp_cols(tbase, kThr);
  const uint32_t ttw = tc + 4 * R0;
  typename PF::LastTw tl;
  if constexpr (TWR)
    PF::load_last_tw(twl, tl);
  else
    park_last_tw<PF>(twl, ttw);
  {
    const int ys = src_index(2 * b + gi, g.Hx, g.H, g.R, g.periodic);
    const int k0 = bl.k[b0];
    // batches of independent loads (the asm volatile TMEM stores would
    // otherwise serialise one load latency per r)
    constexpr int C = 4;
#pragma unroll
    for (int r0 = 0; r0 < R0; r0 += C) {
      double ph[C];
      float2 sv[C];
      bool ok[C];
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int r = r0 + i;
        const int xs = r < R0 && j < PF::NB0
                           ? src_index(j + r * PF::NB0, g.Wx, g.W, g.R, g.periodic) : -1;
        ok[i] = ys >= 0 && xs >= 0;
        const size_t idx = ok[i] ? size_t(ys) * g.W + xs : 0;
        ph[i] = ok[i] ? __ldg(base + idx) : 0.0;
        sv[i] = ok[i] ? sig_value(s, idx) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < C; ++i) {
        if (r0 + i >= R0) break;
        float4 cm = make_float4(0.f, 0.f, 1.f, 0.f);
        if (ok[i]) {
          const float2 cur = c_mul(sv[i], steer(k0, ph[i], -1.f));  // H e^{-i k0 phi}
          const float2 mul = steer(1, ph[i], -1.f);
          cm = make_float4(cur.x, cur.y, mul.x, mul.y);
        }
        tmem_st4(tc + 4 * (r0 + i), cm);
      }
    }
    tmem_wait_st();
  }
  const size_t plane = size_t(g.Hx2) * g.Pw;  // float2 per T1 band plane
  for (int bi = b0; bi < b1; ++bi) {
    {
      // pass-0 inputs of this band, then advance cur to the next band's k:
      // bands run in descending k, so the step is almost always -1 (one
      // multiply by conj(mul), a CTA-uniform branch); other steps loop
      const int dk = bi + 1 < b1 ? bl.k[bi + 1] - bl.k[bi] : 0;
      const bool unit = dk == -1;  // CTA-uniform
      typename PF::P0Regs v;  // the pass-0 inputs, read straight from TMEM
#pragma unroll
      for (int r0 = 0; r0 < R0; r0 += 4) {
        float4 cm[4];
        tmem_ldn<16>(tc + 4 * r0, reinterpret_cast<float*>(cm));
        tmem_wait_ld();
        tmem_depn<16>(reinterpret_cast<float*>(cm));
#pragma unroll
        for (int i = 0; i < 4; ++i) v.a[r0 + i] = make_float2(cm[i].x, cm[i].y);
        if (unit) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 nx = c_mul(v.a[r0 + i], make_float2(cm[i].z, -cm[i].w));
            cm[i].x = nx.x;
            cm[i].y = nx.y;
          }
          tmem_stn<16>(tc + 4 * r0, reinterpret_cast<const float*>(cm));
        }
      }
      if (!unit && dk != 0) {
        // other band steps (band subsets): one rolled loop, kept out of the
        // unrolled hot path (its code would otherwise sit in the band loop
        // once per input and crowd the instruction cache)
        const int n = dk < 0 ? -dk : dk;
#pragma unroll 1
        for (int r = 0; r < R0; ++r) {
          float4 cm = tmem_ld4(tc + 4 * r);
          tmem_wait_ld();
          tmem_dep(cm);
          float2 nx = make_float2(cm.x, cm.y);
          const float2 mm = dk < 0 ? make_float2(cm.z, -cm.w) : make_float2(cm.z, cm.w);
#pragma unroll 1
          for (int q = 0; q < n; ++q) nx = c_mul(nx, mm);
          tmem_st4(tc + 4 * r, make_float4(nx.x, nx.y, cm.z, cm.w));
        }
      }
      tmem_wait_st();
      if ((opaque_i(t) >> 1) < PF::NB0) Dft<R0>::run(v.a);
      PF::pass0_store(W0, v);
    }
    __syncthreads();
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    const int tt = opaque_i(t), g2 = tt & 1, jj = tt >> 1, y = 2 * b + g2;
    // T1 layout B' [u/2][y][u%2]: u = jj + r NB2 (NB2 even: parity fixed)
    float2* o = T1 + size_t(bi) * plane + (size_t(jj >> 1) * g.Hx2 + y) * 2 + (jj & 1);
    const size_t ostep = size_t(PF::NB2 / 2) * g.Hx2 * 2;
    const bool act = jj < PF::NB2;
    auto store = [&](float2 (&a)[R2]) {
      float2* p = o;
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        st_pred(p, a[Dft<R2>::pos(r)], act);
        p += ostep;
      }
    };
    if constexpr (TWR) {
      PF::pass2_all(W1, tl, store);
    } else {
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
    tmem_dealloc(tbase, PF::tmem_cols(kThr));
  }
}

// ------------------------------------------------------------------ S2 (interleaved)
// Per band: the T1_k column pair (TMA) and F^_k column pair (TMA, double
// buffered: read in pass 2) -> column FFT -> acc += X F^_k in TMEM (2 columns
// per pass-2 output).  After the bands: conj(acc) -> W1 -> FFT -> conj -> T2
// (layout A, rows y = k - off).  The 1/(Ph Pw) scale is applied by S4.
template <class PF>
__global__ void __launch_bounds__(PF::T, 1)
    k_cols_fwd_mac_ilv(Geo g, const float4* __restrict__ T1, const float4* __restrict__ Fh,
                       size_t sstride4, Bands bl, int half0, float2* __restrict__ T2,
                       const float2* __restrict__ twm, const float2* __restrict__ twl) {
  pdl_wait();
  constexpr int L = PF::L, R2 = PF::R2;  // L = Ph
  constexpr int kThr = 2 * R2;
  static_assert(kThr * PF::WPQ <= 512, "TMEM budget");
  extern __shared__ __align__(16) float4 smp[];
  float4* ST4 = smp;              // T1_k column pair (Hx2 <= L rows)
  float4* SF4 = ST4 + L;          // F^_k column pair, two copies by band parity
  float4* W04 = SF4 + 2 * L;
  float4* W14 = W04 + PF::LP;
  float2* TWs = reinterpret_cast<float2*>(W14 + PF::LP);
  const float2* ST = reinterpret_cast<const float2*>(ST4);
  float2* W0 = reinterpret_cast<float2*>(W04);
  float2* W1 = reinterpret_cast<float2*>(W14);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int c = blockIdx.x, t = threadIdx.x;
  const size_t plane1 = size_t(g.Hx2 / 2) * g.Pw;  // float4 per T1 band plane
  const float4* colT = T1 + size_t(c) * g.Hx2;     // [u/2][y] pairs
  const unsigned bytesT = unsigned(g.Hx2) * unsigned(sizeof(float4));
  constexpr unsigned kBytesF = unsigned(L * sizeof(float4));
  auto fsrc = [&](int bi) { return Fh + size_t(bl.spec[bi]) * sstride4 + size_t(c) * L; };
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytesT + kBytesF);
    bulk_copy(ST4, colT, bytesT, &bar);
    bulk_copy(SF4, fsrc(0), kBytesF, &bar);
    if (bl.n > 1) {
      prefetch_l2(colT + plane1, bytesT);
      prefetch_l2(fsrc(1), kBytesF);
    }
  }
  if (t < 32) tmem_alloc(&tbase, PF::tmem_cols(kThr));
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  typename PF::LastTw tl;
  PF::load_last_tw(twl, tl);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tacc = tmem_warp_cols(tbase, kThr);
  const int hx2 = g.Hx2;
  unsigned phase = 0;
  for (int bi = 0; bi < bl.n; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    {
      auto load = [&](int, int n, int gi) -> float2 {
        return n < hx2 ? ST[2 * n + gi] : make_float2(0.f, 0.f);
      };
      typename PF::P0Regs v;
      PF::pass0_compute(load, v);
      PF::pass0_store(W0, v);
    }
    __syncthreads();
    if (t == 0 && bi + 1 < bl.n) {
      fence_proxy_async();
      mbar_expect_tx(&bar, bytesT + kBytesF);
      bulk_copy(ST4, colT + size_t(bi + 1) * plane1, bytesT, &bar);
      bulk_copy(SF4 + ((bi + 1) & 1) * L, fsrc(bi + 1), kBytesF, &bar);
      if (bi + 2 < bl.n) {
        prefetch_l2(colT + size_t(bi + 2) * plane1, bytesT);
        prefetch_l2(fsrc(bi + 2), kBytesF);
      }
    }
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    const float2* SF = reinterpret_cast<const float2*>(SF4 + (bi & 1) * L);
    // Hermitian half-band mode: the k = 0 band enters with weight 1/2 (S4
    // then takes 2 Re)
    const float wk = half0 && bl.k[bi] == 0 ? 0.5f : 1.f;
    const int tt = opaque_i(t);
    const float2* fp = SF + tt;  // F^[k] of this thread's sequence: 2 k + g, k = j + r NB2
    auto mac = [&](float2 (&a)[R2]) {
      constexpr int C = 5;
#pragma unroll
      for (int r0 = 0; r0 < R2; r0 += C) {
        float2 acc[C];
        if (bi > 0) {
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) acc[i] = tmem_ld2(tacc + 2 * (r0 + i));
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) tmem_dep(acc[i]);
        }
#pragma unroll
        for (int i = 0; i < C; ++i) {
          const int r = r0 + i;
          if (r >= R2) break;
          const float2 x = c_scale(c_mul(a[Dft<R2>::pos(r)], fp[2 * r * PF::NB2]), wk);
          acc[i] = bi > 0 ? c_add(acc[i], x) : x;
        }
#pragma unroll
        for (int i = 0; i < C; ++i)
          if (r0 + i < R2) tmem_st2(tacc + 2 * (r0 + i), acc[i]);
      }
      tmem_wait_st();
    };
    PF::pass2_all(W1, tl, mac);
  }
  // inverse column transform of the band sum: conj(acc) -> W1 (natural
  // order) -> FFT -> conj -> T2
  __syncthreads();  // every thread is past the last band's pass-2 reads of W1
  {
    const int gi = t & 1, j = t >> 1;
#pragma unroll
    for (int r = 0; r < R2; ++r) {
      const float2 a = tmem_ld2(tacc + 2 * r);
      tmem_wait_ld();
      float2 v = a;
      tmem_dep(v);
      if (j < PF::NB2) W1[2 * (j + r * PF::NB2) + gi] = c_conj(v);
    }
  }
  __syncthreads();
  {
    const float2* S = W1;
    auto load = [&](int, int n, int gi) -> float2 { return S[2 * n + gi]; };
    typename PF::P0Regs v;
    PF::pass0_compute(load, v);
    PF::pass0_store(W0, v);
  }
  __syncthreads();
  PF::pass1(W0, W1, TWs);
  __syncthreads();
  {
    const int tt = opaque_i(t), gi = tt & 1, j = tt >> 1;
    const int y0 = j - g.off;
    const int rstride = (PF::NB2 / 2) * 2 * g.Pw;
    float2* o = T2 + 2 * (2 * c + gi) + (ptrdiff_t(y0 >> 1) * (2 * g.Pw) + (y0 & 1));
    const bool act = j < PF::NB2;
    auto store = [&](float2 (&a)[R2]) {
      int y = opaque_i(y0);
      float2* p = o;
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        st_pred(p, c_conj(a[Dft<R2>::pos(r)]), act && unsigned(y) < unsigned(g.H));
        y += PF::NB2;
        p += rstride;
      }
    };
    PF::pass2_all(W1, tl, store);
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (t < 32) {
    tmem_fence_after_sync();
    tmem_dealloc(tbase, PF::tmem_cols(kThr));
  }
}

// ------------------------------------------------------------------ S2, conjugate band pairs
// Real signal, any filter: H e^{+ik phi} = conj(H e^{-ik phi}), so S1 transforms
// the bands k >= 0 only and the -k term of the scatter is
//   (H e^{+ik phi}) * f_{-k} = conj((H e^{-ik phi}) * conj(f_{-k})).
// Per band k this kernel feeds the column FFT X of T1_k into two sums in TMEM,
// A += X F^_k and (k > 0) B += X G_k with G_k the spectrum of conj(f_{-k}); both
// are inverse transformed (T2, T2 + t2plane) and S4 writes a + conj(b).  F^_k
// and G_k are staged side by side (single buffers) by one TMA pair per band:
// every warp arrives on `bard` when its pass-2 reads of the buffers are done,
// thread 0 then issues the next band's pair, which lands during that band's
// passes 0 and 1.  Same shared memory as k_cols_fwd_mac_ilv.
// two CTAs per SM when two sets of buffers fit in shared memory (1152): the
// register file then allows 80 per thread (warps are allocated in fours)
template <class PF>
__global__ void __launch_bounds__(PF::T)
    __maxnreg__((3 * PF::L + 2 * PF::LP) * 16 + PF::TWM * 8 <= 112 * 1024 ? 80 : 112)
        k_cols_fwd_mac_cpair_ilv(Geo g, const float4* __restrict__ T1, const float4* __restrict__ Fh,
                             const float4* __restrict__ Gh, size_t sstride4, Bands bl,
                             const int* __restrict__ gspec, float2* __restrict__ T2,
                             size_t t2plane, const float2* __restrict__ twm,
                             const float2* __restrict__ twl) {
  pdl_wait();
  constexpr int L = PF::L, R2 = PF::R2;  // L = Ph
  constexpr int kThr = 4 * R2;           // A then B, 2 columns per pass-2 output
  static_assert(kThr * PF::WPQ <= 512, "TMEM budget");
  extern __shared__ __align__(16) float4 smp[];
  float4* ST4 = smp;      // T1_k column pair (Hx2 <= L rows)
  float4* SF4 = ST4 + L;  // F^_k column pair
  float4* SG4 = SF4 + L;  // G_k column pair
  float4* W04 = SG4 + L;
  float4* W14 = W04 + PF::LP;
  float2* TWs = reinterpret_cast<float2*>(W14 + PF::LP);
  const float2* ST = reinterpret_cast<const float2*>(ST4);
  float2* W0 = reinterpret_cast<float2*>(W04);
  float2* W1 = reinterpret_cast<float2*>(W14);
  __shared__ __align__(8) uint64_t bar, barf, bard;
  __shared__ uint32_t tbase;
  const int c = blockIdx.x, t = threadIdx.x;
  const size_t plane1 = size_t(g.Hx2 / 2) * g.Pw;  // float4 per T1 band plane
  const float4* colT = T1 + size_t(c) * g.Hx2;     // [u/2][y] pairs
  const unsigned bytesT = unsigned(g.Hx2) * unsigned(sizeof(float4));
  constexpr unsigned kBytesF = unsigned(L * sizeof(float4));
  auto fsrc = [&](int bi) { return Fh + size_t(bl.spec[bi]) * sstride4 + size_t(c) * L; };
  auto gsrc = [&](int bi) { return Gh + size_t(gspec[bi]) * sstride4 + size_t(c) * L; };
  // F^ and G of band bi -> SF4, SG4 (thread 0)
  auto stage_fg = [&](int bi) {
    const bool pb = bl.k[bi] != 0;
    mbar_expect_tx(&barf, pb ? 2 * kBytesF : kBytesF);
    bulk_copy(SF4, fsrc(bi), kBytesF, &barf);
    if (pb) bulk_copy(SG4, gsrc(bi), kBytesF, &barf);
  };
  if (t == 0) {
    mbar_init(&bar, 1);
    mbar_init(&barf, 1);
    mbar_init(&bard, PF::T / 32);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytesT);
    bulk_copy(ST4, colT, bytesT, &bar);
    stage_fg(0);
    if (bl.n > 1) {
      prefetch_l2(colT + plane1, bytesT);
      prefetch_l2(fsrc(1), kBytesF);
      if (bl.k[1] != 0) prefetch_l2(gsrc(1), kBytesF);
    }
  }
  if (t < 32) tmem_alloc(&tbase, PF::tmem_cols(kThr));
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  typename PF::LastTw tl;
  PF::load_last_tw(twl, tl);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tacc = tmem_warp_cols(tbase, kThr);
#pragma unroll
  for (int r = 0; r < 2 * R2; ++r) tmem_st2(tacc + 2 * r, make_float2(0.f, 0.f));
  tmem_wait_st();
  const int hx2 = g.Hx2;
  unsigned phase = 0;
  for (int bi = 0; bi < bl.n; ++bi) {
    const bool pairb = bl.k[bi] != 0;  // CTA-uniform: the k = 0 band has no partner
    mbar_wait(&bar, phase);
    {
      auto load = [&](int, int n, int gi) -> float2 {
        return n < hx2 ? ST[2 * n + gi] : make_float2(0.f, 0.f);
      };
      typename PF::P0Regs v;
      PF::pass0_compute(load, v);
      PF::pass0_store(W0, v);
    }
    __syncthreads();
    if (t == 0 && bi + 1 < bl.n) {
      fence_proxy_async();
      mbar_expect_tx(&bar, bytesT);
      bulk_copy(ST4, colT + size_t(bi + 1) * plane1, bytesT, &bar);
      if (bi + 2 < bl.n) {
        prefetch_l2(colT + size_t(bi + 2) * plane1, bytesT);
        prefetch_l2(fsrc(bi + 2), kBytesF);
        if (bl.k[bi + 2] != 0) prefetch_l2(gsrc(bi + 2), kBytesF);
      }
    }
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    mbar_wait(&barf, phase);
    const int tt = opaque_i(t);
    // F^[k], G[k] of this thread's sequence: 2 k + g, k = j + r NB2
    const float2* fp = reinterpret_cast<const float2*>(SF4) + tt;
    const float2* gp = reinterpret_cast<const float2*>(SG4) + tt;
    auto mac = [&](float2 (&a)[R2]) {
      constexpr int C = 4;
      // one sum at a time (A with F^, then B with G) to bound the live registers
#pragma unroll 1
      for (int h = 0; h < (pairb ? 2 : 1); ++h) {
        const uint32_t ta = tacc + 2 * R2 * opaque_i(h);
        const float2* sp = h ? gp : fp;
#pragma unroll
        for (int r0 = 0; r0 < R2; r0 += C) {
          float2 acc[C];
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) acc[i] = tmem_ld2(ta + 2 * (r0 + i));
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) tmem_dep(acc[i]);
#pragma unroll
          for (int i = 0; i < C; ++i) {
            const int r = r0 + i;
            if (r >= R2) break;
            acc[i] = c_add(acc[i], c_mul(a[Dft<R2>::pos(r)], sp[2 * r * PF::NB2]));
          }
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (r0 + i < R2) tmem_st2(ta + 2 * (r0 + i), acc[i]);
        }
      }
      tmem_wait_st();
    };
    PF::pass2_all(W1, tl, mac);
    // the staged spectra are free once every warp is past its pass 2
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(&bard);
    if (t == 0 && bi + 1 < bl.n) {
      mbar_wait(&bard, phase);
      fence_proxy_async();
      stage_fg(bi + 1);
    }
    phase ^= 1;
  }
  // inverse column transforms of the two band sums: conj(acc) -> W1 (natural
  // order) -> FFT -> conj -> T2 plane
#pragma unroll 1
  for (int p = 0; p < 2; ++p) {
    __syncthreads();  // every thread is past the previous pass-2 reads of W1
    {
      const int gi = t & 1, j = t >> 1;
      const uint32_t ta = tacc + 2 * R2 * opaque_i(p);
#pragma unroll
      for (int r = 0; r < R2; ++r) {
        float2 v = tmem_ld2(ta + 2 * r);
        tmem_wait_ld();
        tmem_dep(v);
        if (j < PF::NB2) W1[2 * (j + r * PF::NB2) + gi] = c_conj(v);
      }
    }
    __syncthreads();
    {
      const float2* S = W1;
      auto load = [&](int, int n, int gi) -> float2 { return S[2 * n + gi]; };
      typename PF::P0Regs v;
      PF::pass0_compute(load, v);
      PF::pass0_store(W0, v);
    }
    __syncthreads();
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    {
      const int tt = opaque_i(t), gi = tt & 1, j = tt >> 1;
      const int y0 = j - g.off;
      const int rstride = (PF::NB2 / 2) * 2 * g.Pw;
      float2* o = T2 + size_t(p) * t2plane + 2 * (2 * c + gi) +
                  (ptrdiff_t(y0 >> 1) * (2 * g.Pw) + (y0 & 1));
      const bool act = j < PF::NB2;
      auto store = [&](float2 (&a)[R2]) {
        int y = opaque_i(y0);
        float2* q = o;
#pragma unroll
        for (int r = 0; r < R2; ++r) {
          st_pred(q, c_conj(a[Dft<R2>::pos(r)]), act && unsigned(y) < unsigned(g.H));
          y += PF::NB2;
          q += rstride;
        }
      };
      PF::pass2_all(W1, tl, store);
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (t < 32) {
    tmem_fence_after_sync();
    tmem_dealloc(tbase, PF::tmem_cols(kThr));
  }
}

// ------------------------------------------------------------------ single transforms
// F1 (row FFT of the zero-padded / periodically extended signal -> T1), F2
// (column FFT of T1 -> spectrum, layout B) and S4 (row IFFT of T2, crop,
// + dc H -> out) on the pair engine: one transform per CTA, inputs read
// straight from global memory (F1, S4) or TMA-staged (F2).
template <class PF>
__global__ void __launch_bounds__(PF::T, PF::MINB)
    k_rows_fwd_ilv(Geo g, SigSrc s, float2* __restrict__ T1, const float2* __restrict__ twm,
                   const float2* __restrict__ twl) {
  pdl_wait();
  extern __shared__ __align__(16) float4 smp[];
  float2* W0 = reinterpret_cast<float2*>(smp);
  float2* W1 = reinterpret_cast<float2*>(smp + PF::LP);
  float2* TWs = reinterpret_cast<float2*>(smp + 2 * PF::LP);
  const int b = blockIdx.x, t = threadIdx.x;
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  typename PF::LastTw tl;
  PF::load_last_tw(twl, tl);
  const int ys = src_index(2 * b + (t & 1), g.Hx, g.H, g.R, g.periodic);
  auto load = [&](int, int n, int) -> float2 {
    const int xs = src_index(n, g.Wx, g.W, g.R, g.periodic);
    return ys < 0 || xs < 0 ? make_float2(0.f, 0.f) : sig_value(s, size_t(ys) * g.W + xs);
  };
  typename PF::P0Regs v;
  PF::pass0_compute(load, v);
  PF::pass0_store(W0, v);
  __syncthreads();
  PF::pass1(W0, W1, TWs);
  __syncthreads();
  const int gi = t & 1, j = t >> 1, y = 2 * b + gi;
  float2* o = T1 + (size_t(j >> 1) * g.Hx2 + y) * 2 + (j & 1);  // layout B' (NB2 even)
  const size_t ostep = size_t(PF::NB2 / 2) * g.Hx2 * 2;
  auto store = [&](float2 (&a)[PF::R2]) {
    float2* p = o;
#pragma unroll
    for (int r = 0; r < PF::R2; ++r) {
      st_pred(p, a[Dft<PF::R2>::pos(r)], j < PF::NB2);
      p += ostep;
    }
  };
  PF::pass2_all(W1, tl, store);
}

template <class PF>
__global__ void __launch_bounds__(PF::T, PF::MINB)
    k_cols_fwd_ilv(Geo g, const float4* __restrict__ T1, float2* __restrict__ spec,
                   const float2* __restrict__ twm, const float2* __restrict__ twl) {
  pdl_wait();
  constexpr int L = PF::L;  // = Ph
  extern __shared__ __align__(16) float4 smp[];
  float4* ST4 = smp;
  float2* W0 = reinterpret_cast<float2*>(smp + L);
  float2* W1 = reinterpret_cast<float2*>(smp + L + PF::LP);
  float2* TWs = reinterpret_cast<float2*>(smp + L + 2 * PF::LP);
  const float2* ST = reinterpret_cast<const float2*>(ST4);
  __shared__ __align__(8) uint64_t bar;
  const int c = blockIdx.x, t = threadIdx.x;
  const unsigned bytes = unsigned(g.Hx2) * unsigned(sizeof(float4));
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytes);
    bulk_copy(ST4, T1 + size_t(c) * g.Hx2, bytes, &bar);
  }
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  typename PF::LastTw tl;
  PF::load_last_tw(twl, tl);
  __syncthreads();
  mbar_wait(&bar, 0);
  const int hx2 = g.Hx2;
  auto load = [&](int, int n, int gi) -> float2 {
    return n < hx2 ? ST[2 * n + gi] : make_float2(0.f, 0.f);
  };
  typename PF::P0Regs v;
  PF::pass0_compute(load, v);
  PF::pass0_store(W0, v);
  __syncthreads();
  PF::pass1(W0, W1, TWs);
  __syncthreads();
  const int tt = t, j = tt >> 1;
  float2* o = spec + size_t(c) * L * 2 + tt;  // layout B: (c Ph + k) 2 + g
  auto store = [&](float2 (&a)[PF::R2]) {
#pragma unroll
    for (int r = 0; r < PF::R2; ++r) st_pred(o + 2 * r * PF::NB2, a[Dft<PF::R2>::pos(r)], j < PF::NB2);
  };
  PF::pass2_all(W1, tl, store);
}

template <class PF, class TO>
__global__ void __launch_bounds__(PF::T, PF::MINB)
    k_rows_inv_out_ilv(Geo g, const float4* __restrict__ T2, const float4* __restrict__ T2b,
                       TO* __restrict__ out, int accumulate, int real2, SigSrc dcs, double dcr,
                       double dci, float scale, const float2* __restrict__ twm,
                       const float2* __restrict__ twl) {
  pdl_wait();
  extern __shared__ __align__(16) float4 smp[];
  float2* W0 = reinterpret_cast<float2*>(smp);
  float2* W1 = reinterpret_cast<float2*>(smp + PF::LP);
  float2* TWs = reinterpret_cast<float2*>(smp + 2 * PF::LP);
  const int b = blockIdx.x, t = threadIdx.x;
  for (int i = t; i < PF::TWM; i += blockDim.x) TWs[i] = twm[i];
  typename PF::LastTw tl;
  PF::load_last_tw(twl, tl);
  // conjugate band pairs: the second plane's term is conj(IFFT(T2b)) =
  // FFT(conj T2b) / (Ph Pw), kept in registers and added to the first plane's
  float2 kb[PF::R2];
#pragma unroll
  for (int r = 0; r < PF::R2; ++r) kb[r] = make_float2(0.f, 0.f);
  if (T2b) {  // CTA-uniform
    const float2* srcb = reinterpret_cast<const float2*>(T2b + size_t(b) * g.Pw);
    auto loadb = [&](int, int n, int gi) -> float2 { return c_conj(__ldg(srcb + 2 * n + gi)); };
    typename PF::P0Regs vb;
    PF::pass0_compute(loadb, vb);
    PF::pass0_store(W0, vb);
    __syncthreads();
    PF::pass1(W0, W1, TWs);
    __syncthreads();
    auto keep = [&](float2 (&a)[PF::R2]) {
#pragma unroll
      for (int r = 0; r < PF::R2; ++r) kb[r] = a[Dft<PF::R2>::pos(r)];
    };
    PF::pass2_all(W1, tl, keep);
    __syncthreads();  // W0 / W1 are reused by the first plane
  }
  const float2* src = reinterpret_cast<const float2*>(T2 + size_t(b) * g.Pw);
  auto load = [&](int, int n, int gi) -> float2 { return c_conj(__ldg(src + 2 * n + gi)); };
  typename PF::P0Regs v;
  PF::pass0_compute(load, v);
  PF::pass0_store(W0, v);
  __syncthreads();
  PF::pass1(W0, W1, TWs);
  __syncthreads();
  const int gi = t & 1, j = t >> 1, y = 2 * b + gi;
  auto store = [&](float2 (&a)[PF::R2]) {
    if (j >= PF::NB2 || y >= g.H) return;
#pragma unroll
    for (int r = 0; r < PF::R2; ++r) {
      const int x = j + r * PF::NB2 - g.off;
      if (x < 0 || x >= g.W) continue;
      const size_t i = size_t(y) * g.W + x;
      float2 v = c_scale(c_add(c_conj(a[Dft<PF::R2>::pos(r)]), kb[r]), scale);
      if (real2) v = make_float2(2.f * v.x, 0.f);  // Hermitian half-band: out = 2 Re
      OutOps<TO>::put(out, i, v, accumulate != 0, dc_term(dcs, i, dcr, dci));
    }
  };
  PF::pass2_all(W1, tl, store);
}


}  // namespace

// S1 at 1152 (config 2): the pair kernel (8 * 16 * 9, S1Plan) unless
// XCB_S1_PAIR=0 selects the fast one
bool s1_pair_small() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_S1_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// S1's own plan per length: S1's pass 0 reads its inputs from TMEM, so a
// short first radix that keeps every thread busy in pass 0 pays off there.
// 1152 = 8 * 16 * 9 (288 threads: 100% / 50% / 89% busy per pass) measured
// S1 164.6 -> 144.6 us on config 2 at base clocks; the other stages keep
// 16 * 9 * 8 (S2 130.9 against 139.7 us, S4 12.7 against 14.7 us).
template <class PF>
struct S1Plan {
  using type = PF;
};
template <>
struct S1Plan<IlvFft<1152, 16, 9, 8, 16>> {
  using type = IlvFft<1152, 8, 16, 9, 8>;
};
// the same for the other lengths whose common plan starts with radix 16 and
// whose S1 would otherwise spill (pass-0 inputs and phasors of 16 points)
#define XCB_S1_PLAN(LL, A1, A2, B0, B1, B2)       \
  template <>                                     \
  struct S1Plan<IlvFft<LL, 16, A1, A2, 16>> {     \
    using type = IlvFft<LL, B0, B1, B2, 8>;       \
  };
XCB_S1_PLAN(1024, 8, 8, 8, 16, 8)
XCB_S1_PLAN(1280, 10, 8, 8, 16, 10)
XCB_S1_PLAN(1536, 12, 8, 8, 16, 12)
XCB_S1_PLAN(1920, 12, 10, 8, 16, 15)
XCB_S1_PLAN(2048, 16, 8, 8, 16, 16)
#undef XCB_S1_PLAN

// the transform lengths with a pair plan (ascending)
std::vector<int> pair_plan_lengths() {
  std::vector<int> v;
#define XCB_PAIR_LEN(LL, R0, R1, R2, PP) v.push_back(LL);
  XCB_PAIR_TABLE(XCB_PAIR_LEN)
#undef XCB_PAIR_LEN
  std::sort(v.begin(), v.end());
  return v;
}

// 0 if no pair plan for L (or the stage does not fit); else the dynamic smem.
// stage 0 I1, 1 I2, 2 planes, 3 S1, 4 S2, 5 F1, 6 F2, 7 S4
size_t pair_smem(int stage, int L, const Geo& g) {
  size_t s = 0;
#define XCB_PAIR_SMEM(LL, R0, R1, R2, PP)                                          \
  if (L == LL) {                                                                   \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                         \
    const size_t tw = size_t(PF::TWM) * sizeof(float2);                            \
    const size_t w = 2 * size_t(PF::LP) * sizeof(float4);                          \
    if (stage <= 2) s = size_t(LL) * sizeof(float4) + w + tw;                      \
    if (stage == 3 && (LL >= 2048 || s1_pair_small())) {                           \
      using P1 = typename S1Plan<PF>::type;                                        \
      s = 2 * size_t(P1::LP) * sizeof(float4) + size_t(P1::TWM) * sizeof(float2);  \
    }                                                                              \
    if (stage == 4 && g.Hx2 <= LL) s = 3 * size_t(LL) * sizeof(float4) + w + tw;   \
    if (stage == 5 || stage == 7) s = w + tw;                                      \
    if (stage == 6 && g.Hx2 <= LL) s = size_t(LL) * sizeof(float4) + w + tw;      \
  }
  XCB_PAIR_TABLE(XCB_PAIR_SMEM)
#undef XCB_PAIR_SMEM
  return s <= kSmemLimitP ? s : 0;
}

// Two images per I1 launch halve the filter-spectrum reads, but I1 is issue-
// bound, not HBM-bound, so it measured slower (4.35 vs 3.88 ms per image on
// config 5): off unless XCB_I1_IMAGES=2.
int pair_i1_images() {
  static const int n = [] {
    const char* e = std::getenv("XCB_I1_IMAGES");
    return e && e[0] == '2' ? 2 : 1;
  }();
  return n;
}

// Grid of a band-loop kernel over `units` independent units (column pairs)
// with `per_sm` resident CTAs per SM: whole waves run every band; the units of
// the last, partial wave are split into band chunks so that the tail fills
// the SMs.  The split minimises ceil(rem * s / slots) * (ceil(nb / s) + 1)
// (one band-equivalent of per-CTA setup per chunk).  XCB_TAIL_SPLIT=0 turns
// it off.
TailSplit tail_split(int units, int per_sm, int nb, int threads) {
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  static const bool off = [] {
    const char* e = std::getenv("XCB_TAIL_SPLIT");
    return e && e[0] == '0';
  }();
  const int slots = sms * per_sm;
  const int full = units / slots * slots, rem = units - full;
  if (off || nb < 4) return {units, units, 1, slots};
  if (full == 0) {
    // under one wave (small images): every unit's bands go to s chunks, s CTAs
    // small CTAs co-reside beyond the launch bound (registers: ~640 threads per SM)
    const int occ = threads > 0 ? std::max(per_sm, std::min(6, 640 / threads)) : per_sm;
    const int s = std::min(sms * occ / std::max(units, 1), nb / 2);
    if (s < 2) return {units, units, 1, slots};
    return {units * s, 0, s, slots};
  }
  if (rem == 0) return {units, units, 1, slots};
  int best = 1;
  long best_cost = long(nb) + 1;
  for (int s = 2; s <= nb / 2; ++s) {
    const long waves = (long(rem) * s + slots - 1) / slots;
    const long cost = waves * ((nb + s - 1) / s + 1);
    if (cost < best_cost) {
      best_cost = cost;
      best = s;
    }
  }
  return {full + rem * best, full, best, slots};
}

void launch_rows_inv_steer_pair(const Geo& g, const float2* T2, const Bands& b, int half,
                                const double* base, int out_kind, void* out, int accumulate,
                                const SigSrc& dcs, double dcr, double dci, cudaStream_t st,
                                LaunchCounter& lc) {
  const size_t sm = pair_smem(1, g.Pw, g);
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  const float4* t2 = reinterpret_cast<const float4*>(T2);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    if (out_kind == OUT_C64) {                                                              \
      set_smem(k_rows_inv_steer_ilv<PF, float2>, sm);                                       \
      launch_k(k_rows_inv_steer_ilv<PF, float2>, g.H2 / 2, PF::T, sm, st,                         \
          g, t2, b, half, base, static_cast<float2*>(out), accumulate, dcs, dcr, dci, scale, \
          tw.mid, tw.last);                                                                 \
    } else {                                                                                \
      set_smem(k_rows_inv_steer_ilv<PF, double2>, sm);                                      \
      launch_k(k_rows_inv_steer_ilv<PF, double2>, g.H2 / 2, PF::T, sm, st,                        \
          g, t2, b, half, base, static_cast<double2*>(out), accumulate, dcs, dcr, dci,      \
          scale,                                                                            \
          tw.mid, tw.last);                                                                 \
    }                                                                                       \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Pw, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

bool dual_pair_ok(const Geo& g) {
  return g.Ph == g.Pw && pair_smem(0, g.Ph, g) && pair_smem(1, g.Pw, g);
}

void launch_dual_pair(const Geo& g, const float2* Hhat, const float2* Fhat, size_t sstride,
                      const Bands& b, float2* T2w, const float2* T2r, int half,
                      const double* base, int out_kind, void* out, int accumulate,
                      const SigSrc& dcs, double dcr, double dci, cudaStream_t st,
                      LaunchCounter& lc) {
  const size_t sm = pair_smem(0, g.Ph, g);
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  const I1Args a{reinterpret_cast<const float4*>(Hhat), reinterpret_cast<const float4*>(Fhat),
                 sstride / 2, b, T2w};
  const int n1 = g.Pw / 2, n2 = g.H2 / 2;
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    if (out_kind == OUT_C64) {                                                              \
      const I2Args<float2> i2{reinterpret_cast<const float4*>(T2r), b, half, base,          \
                              static_cast<float2*>(out), accumulate, dcs, dcr, dci, scale}; \
      set_smem(k_dual_ilv<PF, float2>, sm);                                                 \
      launch_k(k_dual_ilv<PF, float2>, n1 + n2, PF::T, sm, st, g, a, i2, n1, n2, tw.mid, tw.last, \
                                                         tw.last);                          \
    } else {                                                                                \
      const I2Args<double2> i2{reinterpret_cast<const float4*>(T2r), b, half, base,         \
                               static_cast<double2*>(out), accumulate, dcs, dcr, dci,       \
                               scale};                                                      \
      set_smem(k_dual_ilv<PF, double2>, sm);                                                \
      launch_k(k_dual_ilv<PF, double2>, n1 + n2, PF::T, sm, st, g, a, i2, n1, n2, tw.mid,         \
                                                          tw.last, tw.last);                \
    }                                                                                       \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Pw, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_rows_fwd_premul_pair(const Geo& g, const SigSrc& s, const double* base,
                                 const Bands& b, float2* T1, cudaStream_t st,
                                 LaunchCounter& lc) {
  const size_t sm = pair_smem(3, g.Pw, g);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = typename S1Plan<IlvFft<LL, R0, R1, R2, PP>>::type;                           \
    const PairTw tw = pair_tables<PF>();                                                    \
    /* tail split only under two waves (config 2: 512 row pairs on 444 slots); config 4's  \
       3.5 waves measured 0.306 ms split, 0.297 ms not */                                   \
    const int rows2 = g.Hx2 / 2;                                                            \
    TailSplit ts = tail_split(rows2, S1Occ<PF>::kMinB, b.n, PF::T);                                \
    if (rows2 >= 2 * ts.slots) ts = TailSplit{rows2, rows2, 1, ts.slots};                   \
    set_smem(k_rows_fwd_premul_ilv<PF>, sm);                                                \
    launch_k(k_rows_fwd_premul_ilv<PF>, ts.grid, PF::T, sm, st, g, s, base, b, T1, tw.mid,        \
                                                          tw.last, ts.full, ts.split);      \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Pw, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_cols_fwd_mac_inv_pair(const Geo& g, const float2* T1, const float2* Fhat,
                                  size_t sstride, const Bands& b, int half0, float2* T2,
                                  cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = pair_smem(4, g.Ph, g);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    set_smem(k_cols_fwd_mac_ilv<PF>, sm);                                                   \
    launch_k(k_cols_fwd_mac_ilv<PF>, g.Pw / 2, PF::T, sm, st,                                     \
        g, reinterpret_cast<const float4*>(T1), reinterpret_cast<const float4*>(Fhat),      \
        sstride / 2, b, half0, T2, tw.mid, tw.last);                                        \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Ph, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_cols_fwd_mac_inv_cpair(const Geo& g, const float2* T1, const float2* Fhat,
                                   const float2* Ghat, size_t sstride, const Bands& b,
                                   const int* gspec, float2* T2, size_t t2plane,
                                   cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = pair_smem(4, g.Ph, g);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    set_smem(k_cols_fwd_mac_cpair_ilv<PF>, sm);                                             \
    launch_k(k_cols_fwd_mac_cpair_ilv<PF>, g.Pw / 2, PF::T, sm, st,                               \
        g, reinterpret_cast<const float4*>(T1), reinterpret_cast<const float4*>(Fhat),      \
        reinterpret_cast<const float4*>(Ghat), sstride / 2, b, gspec, T2, t2plane, tw.mid,  \
        tw.last);                                                                           \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Ph, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_rows_fwd_pair(const Geo& g, const SigSrc& s, float2* T1, cudaStream_t st,
                          LaunchCounter& lc) {
  const size_t sm = pair_smem(5, g.Pw, g);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    set_smem(k_rows_fwd_ilv<PF>, sm);                                                       \
    launch_k(k_rows_fwd_ilv<PF>, g.Hx2 / 2, PF::T, sm, st, g, s, T1, tw.mid, tw.last);            \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Pw, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_cols_fwd_pair(const Geo& g, const float2* T1, float2* spec, cudaStream_t st,
                          LaunchCounter& lc) {
  const size_t sm = pair_smem(6, g.Ph, g);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    set_smem(k_cols_fwd_ilv<PF>, sm);                                                       \
    launch_k(k_cols_fwd_ilv<PF>, g.Pw / 2, PF::T, sm, st, g, reinterpret_cast<const float4*>(T1), \
                                                    spec, tw.mid, tw.last);                 \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Ph, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

void launch_rows_inv_out_pair(const Geo& g, const float2* T2, int out_kind, void* out,
                              int accumulate, int real2, const SigSrc& dcs, double dcr,
                              double dci, cudaStream_t st, LaunchCounter& lc, const float2* T2b) {
  const size_t sm = pair_smem(7, g.Pw, g);
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  const float4* t2 = reinterpret_cast<const float4*>(T2);
  const float4* t2b = reinterpret_cast<const float4*>(T2b);
#define XCB_BODY(LL, R0, R1, R2, PP)                                                         \
  case LL: {                                                                                \
    using PF = IlvFft<LL, R0, R1, R2, PP>;                                                  \
    const PairTw tw = pair_tables<PF>();                                                    \
    if (out_kind == OUT_C64) {                                                              \
      set_smem(k_rows_inv_out_ilv<PF, float2>, sm);                                         \
      launch_k(k_rows_inv_out_ilv<PF, float2>, g.H2 / 2, PF::T, sm, st,                           \
          g, t2, t2b, static_cast<float2*>(out), accumulate, real2, dcs, dcr, dci, scale,   \
          tw.mid, tw.last);                                                                 \
    } else {                                                                                \
      set_smem(k_rows_inv_out_ilv<PF, double2>, sm);                                        \
      launch_k(k_rows_inv_out_ilv<PF, double2>, g.H2 / 2, PF::T, sm, st,                          \
          g, t2, t2b, static_cast<double2*>(out), accumulate, real2, dcs, dcr, dci, scale,  \
          tw.mid, tw.last);                                                                 \
    }                                                                                       \
    break;                                                                                  \
  }
  XCB_PAIR_DISPATCH(g.Pw, XCB_BODY)
#undef XCB_BODY
  ++lc.n;
}

}  // namespace xcb
