// Fast band-loop stages for the transform lengths of XCB_FAST_TABLE (one
// compile-time FastFft<R0, R1, RL> instance per length): one CTA per SM with
//   * the next band's input block prefetched by TMA (cp.async.bulk + mbarrier)
//     into a staging buffer while the current band's FFT passes run,
//   * an in-place FFT buffer (FastFft::first / mid / last),
//   * per-band results accumulated in registers across the band loop (the
//     radix-RL last pass maps (thread, r) to the same output every band).
// Steering uses Horner's rule over the bands sorted by descending k:
//   sum_k z^k G_k = z^{k_min} * (((G_{k0} z^{k0-k1} + G_{k1}) z^{k1-k2} + ...)
// so each band costs one complex FMA per pixel instead of a sincos
// (z = e^{i phi(p)}; engine.hpp:312-317 / 353-358 for the reference steering).
#include <algorithm>

#include <cstdlib>

#include "stages_common.cuh"
#include "tma.cuh"

namespace xcb {
namespace {

// Returns v, but opaque to the optimizer: used inside the band loops so that
// per-output address arithmetic is recomputed each band instead of being
// hoisted out of the loop into (spilled) registers.
__device__ __forceinline__ int opaque(int v) {
  asm volatile("" : "+r"(v));
  return v;
}

__device__ __forceinline__ float2 cpow_step(float2 a, float2 z, int d) {
  if (d == -1) return c_mul(a, c_conj(z));  // descending consecutive bands
  if (d < 0) {
    z = c_conj(z);
    d = -d;
  }
  for (int t = 0; t < d; ++t) a = c_mul(a, z);
  return a;
}

// ------------------------------------------------------------------ I1 fast
template <class FF>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_cols_inv_corr_fast(FftPlanD p, Geo g, const float2* __restrict__ Hh,
                         const float2* __restrict__ Fh, size_t sstride, Bands bl,
                         float2* __restrict__ T2) {
  // band chunk blockIdx.y of gridDim.y (small images: the bands of a column
  // pair are spread over several CTAs so the grid fills the GPU)
  const int b0 = int(blockIdx.y) * bl.n / int(gridDim.y);
  const int b1 = int(blockIdx.y + 1) * bl.n / int(gridDim.y);
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int L = FF::L;  // = Ph
  float2* Hc = reinterpret_cast<float2*>(smraw);
  float2* S = Hc + 2 * L;
  float2* W = S + 2 * L;
  float2* TW = W + 2 * FF::Lp;
  FF::load_twiddles(TW, p.tw);
  const int c = blockIdx.x, tid = threadIdx.x;
  const size_t colb = size_t(c) * L * 2;
  const unsigned bytes = unsigned(L) * 2u * unsigned(sizeof(float2));
  const size_t plane = size_t(g.H2) * g.Pw;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, 2 * bytes);
    bulk_copy(Hc, Hh + colb, bytes, &bar);
    bulk_copy(S, Fh + size_t(bl.spec[b0]) * sstride + colb, bytes, &bar);
  }
  __syncthreads();
  unsigned phase = 0;
  for (int bi = b0; bi < b1; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    // conj(H^ conj(F^)) = conj(H^) F^ : inverse via conj-FFT-conj
    auto load = [&](int n, int gi) -> float2 {
      const int i = n * 2 + gi;
      return c_mul(c_conj(Hc[i]), S[i]);
    };
    FF::first(p, W, load);
    __syncthreads();
    if (tid == 0 && bi + 1 < b1) {
      fence_proxy_async();
      mbar_expect_tx(&bar, bytes);
      bulk_copy(S, Fh + size_t(bl.spec[bi + 1]) * sstride + colb, bytes, &bar);
    }
    FF::mid(TW, W);
    float2* out = T2 + size_t(bi) * plane;
    const int pw = opaque(g.Pw), off = opaque(g.off);
    auto store = [&](int k, int gi, int, float2 v) {
      const int y = k - off;
      if (y >= 0 && y < g.H) out[(size_t(y >> 1) * pw + 2 * c + gi) * 2 + (y & 1)] = c_conj(v);
    };
    FF::last(TW, W, store);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ I2 fast
template <class FF, class TO>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_rows_inv_steer_fast(FftPlanD p, Geo g, const float2* __restrict__ T2, Bands bl,
                          const double* __restrict__ base, TO* __restrict__ out,
                          int accumulate, SigSrc dcs, double dcr, double dci, float scale,
                          float2* __restrict__ parts) {
  // band chunk blockIdx.y of gridDim.y: with several chunks each CTA writes
  // its chunk's steered partial sum to parts[chunk] and k_reduce_chunks adds
  // them in chunk order (small images: fills the GPU)
  const int b0 = int(blockIdx.y) * bl.n / int(gridDim.y);
  const int b1 = int(blockIdx.y + 1) * bl.n / int(gridDim.y);
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int L = FF::L;  // = Pw
  const int zs = g.W + ((8 - (g.W % 16) + 16) % 16);  // Z row stride = 8 (mod 16)
  float2* S = reinterpret_cast<float2*>(smraw);
  float2* W = S + 2 * L;
  float2* Z = W + 2 * FF::Lp;
  float2* TW = Z + 2 * zs;
  FF::load_twiddles(TW, p.tw);
  const int b = blockIdx.x, tid = threadIdx.x;
  const unsigned bytes = unsigned(L) * 2u * unsigned(sizeof(float2));
  const size_t plane = size_t(g.H2) * g.Pw;
  const size_t rowb = size_t(b) * L * 2;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytes);
    bulk_copy(S, T2 + size_t(b0) * plane + rowb, bytes, &bar);
  }
  // z = e^{i phi} of the CTA's two output rows
  for (int i = tid; i < 2 * g.W; i += blockDim.x) {
    const int gi = i >= g.W, x = i - gi * g.W, y = 2 * b + gi;
    Z[gi * zs + x] = y < g.H ? steer(1, base[size_t(y) * g.W + x], 1.f) : make_float2(1.f, 0.f);
  }
  __syncthreads();
  constexpr int RL = FF::kLast;
  float2 acc[RL];
#pragma unroll
  for (int r = 0; r < RL; ++r) acc[r] = make_float2(0.f, 0.f);
  unsigned phase = 0;
  for (int bi = b0; bi < b1; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    auto load = [&](int n, int gi) -> float2 { return c_conj(S[n * 2 + gi]); };
    FF::first(p, W, load);
    __syncthreads();
    if (tid == 0 && bi + 1 < b1) {
      fence_proxy_async();
      mbar_expect_tx(&bar, bytes);
      bulk_copy(S, T2 + size_t(bi + 1) * plane + rowb, bytes, &bar);
    }
    FF::mid(TW, W);
    const int dk = bi == b0 ? 0 : bl.k[bi - 1] - bl.k[bi];
    const int zso = opaque(zs), off = opaque(g.off);
    auto store = [&](int k, int gi, int r, float2 v) {
      const float2 val = c_scale(c_conj(v), scale);
      const int x = k - off;
      const float2 z = (x >= 0 && x < g.W) ? Z[gi * zso + x] : make_float2(1.f, 0.f);
      acc[r] = c_add(cpow_step(acc[r], z, dk), val);
    };
    FF::last(TW, W, store);
    __syncthreads();
  }
  // out = z^{k_last} * acc (+ conj(dc) H for the scale group)
  const int nb = L / RL, w = tid;
  if (w < nb * kG) {
    const int gi = w & 1, j = w >> 1, y = 2 * b + gi;
    const int klast = bl.k[b1 - 1];
    const size_t npix = size_t(g.H) * g.W;
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int x = j + r * nb - g.off;
      if (x < 0 || x >= g.W || y >= g.H) continue;
      const size_t i = size_t(y) * g.W + x;
      const float2 v = c_mul(acc[r], steer(klast, base[i], 1.f));
      if (gridDim.y > 1)
        parts[size_t(blockIdx.y) * npix + i] = v;
      else
        OutOps<TO>::put(out, i, v, accumulate != 0, dc_term(dcs, i, dcr, dci));
    }
  }
}

// the chunks' partial sums in chunk order, then the output rule of I2
template <class TO>
__global__ void k_reduce_chunks(const float2* __restrict__ parts, int nch, size_t npix,
                                TO* __restrict__ out, int accumulate, SigSrc dcs, double dcr,
                                double dci) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < npix;
       i += size_t(gridDim.x) * blockDim.x) {
    float2 v = parts[i];
    for (int c = 1; c < nch; ++c) v = c_add(v, parts[size_t(c) * npix + i]);
    OutOps<TO>::put(out, i, v, accumulate != 0, dc_term(dcs, i, dcr, dci));
  }
}

// ------------------------------------------------------------- F1 / F2 fast
// The single forward transforms of the gather front end (F1 rows of the
// signal -> T1, F2 columns of T1 -> H^) with the compile-time plans: the
// generic kernels' runtime radix dispatch is instruction-cache bound at
// small sizes (config 1: ncu no_instruction 25 cycles per issue).
template <class FF>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_rows_fwd_fast(FftPlanD p, Geo g, SigSrc s, float2* __restrict__ T1) {
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* W = reinterpret_cast<float2*>(smraw);
  float2* TW = W + 2 * FF::Lp;
  FF::load_twiddles(TW, p.tw);
  __syncthreads();
  const int b = blockIdx.x;
  auto load = [&](int n, int gi) -> float2 {
    const int ys = src_index(2 * b + gi, g.Hx, g.H, g.R, g.periodic);
    const int xs = src_index(n, g.Wx, g.W, g.R, g.periodic);
    if (ys < 0 || xs < 0) return make_float2(0.f, 0.f);
    return sig_value(s, size_t(ys) * g.W + xs);
  };
  FF::first(p, W, load);
  __syncthreads();
  FF::mid(TW, W);
  const int hx2 = opaque(g.Hx2);
  auto store = [&](int k, int gi, int, float2 v) {
    T1[(size_t(k >> 1) * hx2 + 2 * b + gi) * 2 + (k & 1)] = v;
  };
  FF::last(TW, W, store);
}

template <class FF>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_cols_fwd_fast(FftPlanD p, Geo g, const float2* __restrict__ T1, float2* __restrict__ spec) {
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* W = reinterpret_cast<float2*>(smraw);
  float2* TW = W + 2 * FF::Lp;
  FF::load_twiddles(TW, p.tw);
  __syncthreads();
  const int c = blockIdx.x;
  const float2* src = T1 + size_t(c) * g.Hx2 * 2;
  float2* dst = spec + size_t(c) * FF::L * 2;
  auto load = [&](int n, int gi) -> float2 {
    return n < g.Hx2 ? src[n * 2 + gi] : make_float2(0.f, 0.f);
  };
  FF::first(p, W, load);
  __syncthreads();
  FF::mid(TW, W);
  auto store = [&](int k, int gi, int, float2 v) { dst[k * 2 + gi] = v; };
  FF::last(TW, W, store);
}

// ------------------------------------------------------------- planes fast
// Angle-max front end: per band, row IFFT of T2_b, crop, store the band plane
// G_b (k_anglemax_* then reads all bands per pixel).
template <class FF>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_rows_inv_planes_fast(FftPlanD p, Geo g, const float2* __restrict__ T2, int nbands,
                           float2* __restrict__ planes, float scale) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int L = FF::L;  // = Pw
  float2* S = reinterpret_cast<float2*>(smraw);
  float2* W = S + 2 * L;
  float2* TW = W + 2 * FF::Lp;
  FF::load_twiddles(TW, p.tw);
  const int b = blockIdx.x, tid = threadIdx.x;
  const unsigned bytes = unsigned(L) * 2u * unsigned(sizeof(float2));
  const size_t plane = size_t(g.H2) * g.Pw;
  const size_t rowb = size_t(b) * L * 2;
  const size_t npix = size_t(g.H) * g.W;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytes);
    bulk_copy(S, T2 + rowb, bytes, &bar);
  }
  __syncthreads();
  unsigned phase = 0;
  for (int bi = 0; bi < nbands; ++bi) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    auto load = [&](int n, int gi) -> float2 { return c_conj(S[n * 2 + gi]); };
    FF::first(p, W, load);
    __syncthreads();
    if (tid == 0 && bi + 1 < nbands) {
      fence_proxy_async();
      mbar_expect_tx(&bar, bytes);
      bulk_copy(S, T2 + size_t(bi + 1) * plane + rowb, bytes, &bar);
    }
    FF::mid(TW, W);
    float2* dst = planes + size_t(bi) * npix;
    const int off = opaque(g.off), wd = opaque(g.W);
    auto store = [&](int k, int gi, int, float2 v) {
      const int x = k - off, y = 2 * b + gi;
      if (x >= 0 && x < wd && y < g.H) dst[size_t(y) * wd + x] = c_scale(c_conj(v), scale);
    };
    FF::last(TW, W, store);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ S1 fast
template <class FF>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_rows_fwd_premul_fast(FftPlanD p, Geo g, SigSrc s, const double* __restrict__ base,
                           Bands bl, float2* __restrict__ T1) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int xs_ = g.Wx + ((8 - (g.Wx % 16) + 16) % 16);
  float2* W = reinterpret_cast<float2*>(smraw);
  float2* CUR = W + 2 * FF::Lp;
  float2* MUL = CUR + 2 * xs_;
  float2* TW = MUL + 2 * xs_;
  FF::load_twiddles(TW, p.tw);
  const int b = blockIdx.x, tid = threadIdx.x;
  const size_t plane = size_t(g.Hx2) * g.Pw;
  const int k0 = bl.k[0];
  for (int i = tid; i < 2 * g.Wx; i += blockDim.x) {
    const int gi = i >= g.Wx, xp = i - gi * g.Wx;
    const int ys = src_index(2 * b + gi, g.Hx, g.H, g.R, g.periodic);
    const int xs = src_index(xp, g.Wx, g.W, g.R, g.periodic);
    float2 cur = make_float2(0.f, 0.f), mul = make_float2(1.f, 0.f);
    if (ys >= 0 && xs >= 0) {
      const size_t idx = size_t(ys) * g.W + xs;
      const double ph = base[idx];
      cur = c_mul(sig_value(s, idx), steer(k0, ph, -1.f));  // H e^{-i k0 phi}
      mul = steer(1, ph, -1.f);
    }
    CUR[gi * xs_ + xp] = cur;
    MUL[gi * xs_ + xp] = mul;
  }
  __syncthreads();
  for (int bi = 0; bi < bl.n; ++bi) {
    auto load = [&](int n, int gi) -> float2 {
      return n < g.Wx ? CUR[gi * xs_ + n] : make_float2(0.f, 0.f);
    };
    FF::first(p, W, load);
    __syncthreads();
    if (bi + 1 < bl.n) {  // advance H e^{-i k phi} to the next band
      const int dk = bl.k[bi + 1] - bl.k[bi];
      for (int i = tid; i < 2 * g.Wx; i += blockDim.x) {
        const int gi = i >= g.Wx, xp = i - gi * g.Wx;
        CUR[gi * xs_ + xp] = cpow_step(CUR[gi * xs_ + xp], MUL[gi * xs_ + xp], dk);
      }
    }
    FF::mid(TW, W);
    float2* dst = T1 + size_t(bi) * plane;
    const int hx2 = opaque(g.Hx2);
    auto store = [&](int k, int gi, int, float2 v) {
      dst[(size_t(k >> 1) * hx2 + 2 * b + gi) * 2 + (k & 1)] = v;
    };
    FF::last(TW, W, store);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ S2 fast
// CP: conjugate band pairs (kernels.h launch_cols_fwd_mac_inv_cpair): the bands
// are k >= 0 of a real signal; a second sum accB += X G_k (k > 0), G_k = plane
// gspec[bi] of Gh staged beside F^_k, and a second inverse transform into
// T2 + t2plane
template <class FF, bool CP>
__global__ void __launch_bounds__(kFastMaxThreads, 1)
    k_cols_fwd_mac_inv_fast(FftPlanD p, Geo g, const float2* __restrict__ T1,
                            const float2* __restrict__ Fh, const float2* __restrict__ Gh,
                            size_t sstride, Bands bl, const int* __restrict__ gspec,
                            float2* __restrict__ T2, size_t t2plane) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t barS, barF;
  constexpr int L = FF::L;  // = Ph
  const int sl = g.Hx2 > L ? g.Hx2 : L;
  float2* S = reinterpret_cast<float2*>(smraw);
  float2* SF = S + 2 * sl;
  float2* SG = SF + 2 * L;  // CP only
  float2* W = SF + (CP ? 4 : 2) * L;
  float2* TW = W + 2 * FF::Lp;
  FF::load_twiddles(TW, p.tw);
  const int c = blockIdx.x, tid = threadIdx.x;
  const size_t plane1 = size_t(g.Hx2) * g.Pw;
  const size_t col1 = size_t(c) * g.Hx2 * 2, colF = size_t(c) * L * 2;
  const unsigned bytesS = unsigned(g.Hx2) * 2u * unsigned(sizeof(float2));
  const unsigned bytesF = unsigned(L) * 2u * unsigned(sizeof(float2));
  if (tid == 0) {
    mbar_init(&barS, 1);
    mbar_init(&barF, 1);
    fence_mbar_init();
    mbar_expect_tx(&barS, bytesS);
    bulk_copy(S, T1 + col1, bytesS, &barS);
    const bool pb0 = CP && bl.k[0] != 0;
    mbar_expect_tx(&barF, pb0 ? 2 * bytesF : bytesF);
    bulk_copy(SF, Fh + size_t(bl.spec[0]) * sstride + colF, bytesF, &barF);
    if (pb0) bulk_copy(SG, Gh + size_t(gspec[0]) * sstride + colF, bytesF, &barF);
  }
  __syncthreads();
  constexpr int RL = FF::kLast;
  float2 acc[RL], accB[CP ? RL : 1];
#pragma unroll
  for (int r = 0; r < RL; ++r) acc[r] = make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < (CP ? RL : 1); ++r) accB[r] = make_float2(0.f, 0.f);
  unsigned phS = 0, phF = 0;
  for (int bi = 0; bi < bl.n; ++bi) {
    const bool pairb = CP && bl.k[bi] != 0;  // CTA-uniform
    mbar_wait(&barS, phS);
    phS ^= 1;
    auto load = [&](int n, int gi) -> float2 {
      return n < g.Hx2 ? S[n * 2 + gi] : make_float2(0.f, 0.f);
    };
    FF::first(p, W, load);
    __syncthreads();
    if (tid == 0 && bi + 1 < bl.n) {
      fence_proxy_async();
      mbar_expect_tx(&barS, bytesS);
      bulk_copy(S, T1 + size_t(bi + 1) * plane1 + col1, bytesS, &barS);
    }
    FF::mid(TW, W);
    mbar_wait(&barF, phF);
    phF ^= 1;
    const int two = opaque(2);
    auto store = [&](int k, int gi, int r, float2 v) {
      acc[r] = c_add(acc[r], c_mul(v, SF[k * two + gi]));
      if constexpr (CP) {
        if (pairb) accB[r] = c_add(accB[r], c_mul(v, SG[k * two + gi]));
      }
    };
    FF::last(TW, W, store);
    __syncthreads();
    if (tid == 0 && bi + 1 < bl.n) {
      fence_proxy_async();
      const bool pb = CP && bl.k[bi + 1] != 0;
      mbar_expect_tx(&barF, pb ? 2 * bytesF : bytesF);
      bulk_copy(SF, Fh + size_t(bl.spec[bi + 1]) * sstride + colF, bytesF, &barF);
      if (pb) bulk_copy(SG, Gh + size_t(gspec[bi + 1]) * sstride + colF, bytesF, &barF);
    }
  }
  // inverse column transform of each band sum: conj(acc) -> S -> FFT -> conj
#pragma unroll
  for (int pl = 0; pl < (CP ? 2 : 1); ++pl) {
    if (pl) __syncthreads();  // the first plane's last pass is done with W
    {
      const int nb = L / RL, w = tid;
      if (w < nb * kG) {
        const int gi = w & 1, j = w >> 1;
#pragma unroll
        for (int r = 0; r < RL; ++r)
          S[(j + r * nb) * 2 + gi] = c_conj(CP && pl ? accB[r] : acc[r]);
      }
    }
    __syncthreads();
    auto load = [&](int n, int gi) -> float2 { return S[n * 2 + gi]; };
    FF::first(p, W, load);
    __syncthreads();
    FF::mid(TW, W);
    float2* dst = T2 + size_t(pl) * t2plane;
    auto store = [&](int k, int gi, int, float2 v) {
      const int y = k - g.off;
      if (y >= 0 && y < g.H) dst[(size_t(y >> 1) * g.Pw + 2 * c + gi) * 2 + (y & 1)] = c_conj(v);
    };
    FF::last(TW, W, store);
  }
}

constexpr size_t kSmemLimit = 232448;  // 227 KB opt-in per CTA on sm_100

}  // namespace

// smem needs of each fast kernel (0 if the stage has no fast variant)
size_t fast_smem(int stage, const FftPlan& pl, const Geo& g) {
  const size_t f2 = sizeof(float2);
  const size_t Wb = pl.smem_bytes() + pl.tw_host.size() * f2;  // W + smem twiddles
  const size_t L = pl.d.L;
  size_t s = 0;
  switch (stage) {
    case 0: s = 4 * L * f2 + Wb; break;                                   // I1
    case 1: s = 2 * L * f2 + Wb + 2 * (g.W + 16) * f2; break;            // I2 (+ Z)
    case 2: s = Wb + 4 * (g.Wx + 16) * f2; break;                         // S1
    case 3: s = 2 * (g.Hx2 > int(L) ? g.Hx2 : L) * f2 + 2 * L * f2 + Wb; break;  // S2
    case 6: s = 2 * (g.Hx2 > int(L) ? g.Hx2 : L) * f2 + 4 * L * f2 + Wb; break;  // S2, pairs
    case 4: s = 2 * L * f2 + Wb; break;                                   // planes
    case 5: s = Wb; break;                                                // F1 / F2
  }
  return s <= kSmemLimit ? s : 0;
}

#define XCB_FAST_CASE(LL, R0, R1, RL) \
  case LL: {                          \
    using FF = FastFft<LL, R0, R1, RL>; \
    XCB_FAST_BODY;                    \
    break;                            \
  }

// band chunks for a grid of `units` CTAs: small images (fewer units than
// 2 per SM) spread each unit's bands over up to 4 * SMs / units CTAs
int fast_band_chunks(int units, int nb) {
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  static const bool off = [] {
    const char* e = std::getenv("XCB_BAND_CHUNKS");
    return e && e[0] == '0';
  }();
  if (off || units >= 2 * sms || nb < 2) return 1;
  const int c = (4 * sms + units - 1) / units;
  return c < nb ? c : nb;
}

void launch_cols_inv_corr_fast(const FftPlan& pc, const Geo& g, const float2* Hhat,
                               const float2* Fhat, size_t sstride, const Bands& b, float2* T2,
                               cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(0, pc, g);
  const dim3 grid(g.Pw / 2, fast_band_chunks(g.Pw / 2, b.n));
#define XCB_FAST_BODY                                                                      \
  set_smem(k_cols_inv_corr_fast<FF>, sm);                                                  \
  k_cols_inv_corr_fast<FF><<<grid, pc.d.nt, sm, st>>>(pc.d, g, Hhat, Fhat, sstride, b, T2)
  switch (pc.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

void launch_rows_inv_steer_fast(const FftPlan& pr, const Geo& g, const float2* T2,
                                const Bands& b, const double* base, int out_kind, void* out,
                                int accumulate, const SigSrc& dcs, double dcr, double dci,
                                float2* parts, cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(1, pr, g);
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  const int nch = parts ? fast_band_chunks(g.H2 / 2, b.n) : 1;
  const dim3 grid(g.H2 / 2, nch);
  const size_t npix = size_t(g.H) * g.W;
  if (out_kind == OUT_C64) {
#define XCB_FAST_BODY                                                                      \
  set_smem(k_rows_inv_steer_fast<FF, float2>, sm);                                         \
  k_rows_inv_steer_fast<FF, float2><<<grid, pr.d.nt, sm, st>>>(                            \
      pr.d, g, T2, b, base, static_cast<float2*>(out), accumulate, dcs, dcr, dci, scale, parts)
    switch (pr.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
    if (nch > 1)
      k_reduce_chunks<float2><<<grid_for(npix, 256), 256, 0, st>>>(
          parts, nch, npix, static_cast<float2*>(out), accumulate, dcs, dcr, dci);
  } else {
#define XCB_FAST_BODY                                                                      \
  set_smem(k_rows_inv_steer_fast<FF, double2>, sm);                                        \
  k_rows_inv_steer_fast<FF, double2><<<grid, pr.d.nt, sm, st>>>(                           \
      pr.d, g, T2, b, base, static_cast<double2*>(out), accumulate, dcs, dcr, dci, scale, parts)
    switch (pr.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
    if (nch > 1)
      k_reduce_chunks<double2><<<grid_for(npix, 256), 256, 0, st>>>(
          parts, nch, npix, static_cast<double2*>(out), accumulate, dcs, dcr, dci);
  }
  lc.n += nch > 1 ? 2 : 1;
}

int fast_steer_chunks(const Geo& g, int nb) { return fast_band_chunks(g.H2 / 2, nb); }

void launch_rows_fwd_fast(const FftPlan& pr, const Geo& g, const SigSrc& s, float2* T1,
                          cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(5, pr, g);
#define XCB_FAST_BODY                                                                      \
  set_smem(k_rows_fwd_fast<FF>, sm);                                                       \
  k_rows_fwd_fast<FF><<<g.Hx2 / 2, pr.d.nt, sm, st>>>(pr.d, g, s, T1)
  switch (pr.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

void launch_cols_fwd_fast(const FftPlan& pc, const Geo& g, const float2* T1, float2* spec,
                          cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(5, pc, g);
#define XCB_FAST_BODY                                                                      \
  set_smem(k_cols_fwd_fast<FF>, sm);                                                       \
  k_cols_fwd_fast<FF><<<g.Pw / 2, pc.d.nt, sm, st>>>(pc.d, g, T1, spec)
  switch (pc.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

void launch_rows_inv_planes_fast(const FftPlan& pr, const Geo& g, const float2* T2,
                                 int nbands, float2* planes, cudaStream_t st,
                                 LaunchCounter& lc) {
  const size_t sm = fast_smem(4, pr, g);
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
#define XCB_FAST_BODY                                                                      \
  set_smem(k_rows_inv_planes_fast<FF>, sm);                                                \
  k_rows_inv_planes_fast<FF><<<g.H2 / 2, pr.d.nt, sm, st>>>(pr.d, g, T2, nbands, planes, scale)
  switch (pr.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

void launch_rows_fwd_premul_fast(const FftPlan& pr, const Geo& g, const SigSrc& s,
                                 const double* base, const Bands& b, float2* T1,
                                 cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(2, pr, g);
#define XCB_FAST_BODY                                                                      \
  set_smem(k_rows_fwd_premul_fast<FF>, sm);                                                \
  k_rows_fwd_premul_fast<FF><<<g.Hx2 / 2, pr.d.nt, sm, st>>>(pr.d, g, s, base, b, T1)
  switch (pr.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

void launch_cols_fwd_mac_inv_fast(const FftPlan& pc, const Geo& g, const float2* T1,
                                  const float2* Fhat, size_t sstride, const Bands& b,
                                  float2* T2, cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(3, pc, g);
#define XCB_FAST_BODY                                                                      \
  set_smem(k_cols_fwd_mac_inv_fast<FF, false>, sm);                                        \
  k_cols_fwd_mac_inv_fast<FF, false><<<g.Pw / 2, pc.d.nt, sm, st>>>(                       \
      pc.d, g, T1, Fhat, nullptr, sstride, b, nullptr, T2, 0)
  switch (pc.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

void launch_cols_fwd_mac_inv_cpair_fast(const FftPlan& pc, const Geo& g, const float2* T1,
                                        const float2* Fhat, const float2* Ghat, size_t sstride,
                                        const Bands& b, const int* gspec, float2* T2,
                                        size_t t2plane, cudaStream_t st, LaunchCounter& lc) {
  const size_t sm = fast_smem(6, pc, g);
#define XCB_FAST_BODY                                                                      \
  set_smem(k_cols_fwd_mac_inv_fast<FF, true>, sm);                                         \
  k_cols_fwd_mac_inv_fast<FF, true><<<g.Pw / 2, pc.d.nt, sm, st>>>(                        \
      pc.d, g, T1, Fhat, Ghat, sstride, b, gspec, T2, t2plane)
  switch (pc.d.L) { XCB_FAST_TABLE(XCB_FAST_CASE) }
#undef XCB_FAST_BODY
  ++lc.n;
}

}  // namespace xcb
