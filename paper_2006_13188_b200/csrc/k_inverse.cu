// Inverse stages: I1, I2 (steer / planes), S2 (band MAC + column IFFT), S4.
#include "stages_common.cuh"

namespace xcb {
namespace {

// ------------------------------------------------------------------ I1
__global__ void __launch_bounds__(kMaxThreads)
    k_cols_inv_corr(FftPlanD p, Geo g, const float2* __restrict__ Hh,
                    const float2* __restrict__ Fh, size_t sstride, Bands bl,
                    float2* __restrict__ T2) {
  extern __shared__ float2 sm[];
  const int c = blockIdx.x;
  const size_t colb = size_t(c) * g.Ph * 2;
  const size_t plane = size_t(g.H2) * g.Pw;
  const float2* Hc = Hh + colb;
  for (int bi = 0; bi < bl.n; ++bi) {
    const float2* F = Fh + size_t(bl.spec[bi]) * sstride + colb;
    float2* out = T2 + size_t(bi) * plane;
    // conj(H^ conj(F^)) = conj(H^) F^ : inverse via conj-FFT-conj
    auto load = [&](int n, int gi) -> float2 {
      const int i = n * 2 + gi;
      return c_mul(c_conj(Hc[i]), F[i]);
    };
    auto store = [&](int k, int gi, float2 v) {
      const int y = k - g.off;
      if (y >= 0 && y < g.H)
        out[(size_t(y >> 1) * g.Pw + 2 * c + gi) * 2 + (y & 1)] = c_conj(v);
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ I2
template <class TO>
__global__ void __launch_bounds__(kMaxThreads)
    k_rows_inv_steer(FftPlanD p, Geo g, const float2* __restrict__ T2, Bands bl,
                     const double* __restrict__ base, TO* __restrict__ out, int accumulate,
                     SigSrc dcs, double dcr, double dci, float scale) {
  extern __shared__ float2 sm[];
  const int b = blockIdx.x;
  const size_t plane = size_t(g.H2) * g.Pw;
  for (int bi = 0; bi < bl.n; ++bi) {
    const int kf = bl.k[bi];
    const float2* src = T2 + size_t(bi) * plane + size_t(b) * g.Pw * 2;
    const bool first = bi == 0, last = bi == bl.n - 1;
    auto load = [&](int n, int gi) -> float2 { return c_conj(src[n * 2 + gi]); };
    auto store = [&](int k, int gi, float2 v) {
      const int x = k - g.off, y = 2 * b + gi;
      if (x < 0 || x >= g.W || y >= g.H) return;
      const size_t i = size_t(y) * g.W + x;
      const float2 val = c_mul(c_scale(c_conj(v), scale), steer(kf, base[i], 1.f));
      const float2 extra = last ? dc_term(dcs, i, dcr, dci) : make_float2(0.f, 0.f);
      OutOps<TO>::put(out, i, val, !first || accumulate, extra);
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kMaxThreads)
    k_rows_inv_planes(FftPlanD p, Geo g, const float2* __restrict__ T2, int nb,
                      float2* __restrict__ planes, float scale) {
  extern __shared__ float2 sm[];
  const int b = blockIdx.x;
  const size_t plane = size_t(g.H2) * g.Pw;
  const size_t npix = size_t(g.H) * g.W;
  for (int bi = 0; bi < nb; ++bi) {
    const float2* src = T2 + size_t(bi) * plane + size_t(b) * g.Pw * 2;
    float2* dst = planes + size_t(bi) * npix;
    auto load = [&](int n, int gi) -> float2 { return c_conj(src[n * 2 + gi]); };
    auto store = [&](int k, int gi, float2 v) {
      const int x = k - g.off, y = 2 * b + gi;
      if (x < 0 || x >= g.W || y >= g.H) return;
      dst[size_t(y) * g.W + x] = c_scale(c_conj(v), scale);
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ S2
__global__ void __launch_bounds__(kMaxThreads)
    k_cols_fwd_mac_inv(FftPlanD p, Geo g, const float2* __restrict__ T1,
                       const float2* __restrict__ Fh, size_t sstride, Bands bl,
                       float2* __restrict__ Sigma, float2* __restrict__ T2) {
  extern __shared__ float2 sm[];
  const int c = blockIdx.x;
  const size_t plane1 = size_t(g.Hx2) * g.Pw;
  const size_t colS = size_t(c) * g.Ph * 2;
  float2* S = Sigma + colS;
  for (int bi = 0; bi < bl.n; ++bi) {
    const float2* src = T1 + size_t(bi) * plane1 + size_t(c) * g.Hx2 * 2;
    const float2* F = Fh + size_t(bl.spec[bi]) * sstride + colS;
    const bool first = bi == 0;
    auto load = [&](int n, int gi) -> float2 {
      return n < g.Hx2 ? src[n * 2 + gi] : make_float2(0.f, 0.f);
    };
    auto store = [&](int k, int gi, float2 v) {
      const int i = k * 2 + gi;
      const float2 t = c_mul(v, F[i]);
      S[i] = first ? t : c_add(S[i], t);
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
  // inverse column transform of the band sum (same thread wrote each S[i])
  auto load = [&](int n, int gi) -> float2 { return c_conj(S[n * 2 + gi]); };
  auto store = [&](int k, int gi, float2 v) {
    const int y = k - g.off;
    if (y >= 0 && y < g.H) T2[(size_t(y >> 1) * g.Pw + 2 * c + gi) * 2 + (y & 1)] = c_conj(v);
  };
  fft_block(p, sm, load, store);
}

// ------------------------------------------------------------------ S4
template <class TO>
__global__ void __launch_bounds__(kMaxThreads)
    k_rows_inv_out(FftPlanD p, Geo g, const float2* __restrict__ T2, TO* __restrict__ out,
                   int accumulate, int conjb, SigSrc dcs, double dcr, double dci, float scale) {
  extern __shared__ float2 sm[];
  const int b = blockIdx.x;
  const float2* src = T2 + size_t(b) * g.Pw * 2;
  auto load = [&](int n, int gi) -> float2 { return c_conj(src[n * 2 + gi]); };
  auto store = [&](int k, int gi, float2 v) {
    const int x = k - g.off, y = 2 * b + gi;
    if (x < 0 || x >= g.W || y >= g.H) return;
    const size_t i = size_t(y) * g.W + x;
    // conjb (second plane of the conjugate band pairs): out += conj(IFFT(T2)),
    // i.e. the forward transform of conj(T2) without the final conjugation
    if (conjb)
      OutOps<TO>::put(out, i, c_scale(v, scale), true, make_float2(0.f, 0.f));
    else
      OutOps<TO>::put(out, i, c_scale(c_conj(v), scale), accumulate != 0,
                      dc_term(dcs, i, dcr, dci));
  };
  fft_block(p, sm, load, store);
}

}  // namespace

void launch_cols_inv_corr(const FftPlan& pcol, const Geo& g, const float2* Hhat,
                          const float2* Fhat, size_t spec_stride, const Bands& b, float2* T2,
                          cudaStream_t st, LaunchCounter& lc) {
  set_smem(k_cols_inv_corr, pcol.smem_bytes());
  k_cols_inv_corr<<<g.Pw / 2, pcol.d.nt, pcol.smem_bytes(), st>>>(pcol.d, g, Hhat, Fhat,
                                                                  spec_stride, b, T2);
  ++lc.n;
}

void launch_rows_inv_steer(const FftPlan& prow, const Geo& g, const float2* T2,
                           const Bands& b, const double* base, int out_kind, void* out,
                           int accumulate, const SigSrc& dcs, double dcr, double dci,
                           cudaStream_t st, LaunchCounter& lc) {
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  if (out_kind == OUT_C64) {
    set_smem(k_rows_inv_steer<float2>, prow.smem_bytes());
    k_rows_inv_steer<float2><<<g.H2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(
        prow.d, g, T2, b, base, static_cast<float2*>(out), accumulate, dcs, dcr, dci, scale);
  } else {
    set_smem(k_rows_inv_steer<double2>, prow.smem_bytes());
    k_rows_inv_steer<double2><<<g.H2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(
        prow.d, g, T2, b, base, static_cast<double2*>(out), accumulate, dcs, dcr, dci, scale);
  }
  ++lc.n;
}

void launch_rows_inv_planes(const FftPlan& prow, const Geo& g, const float2* T2, int nbands,
                            float2* planes, cudaStream_t st, LaunchCounter& lc) {
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  set_smem(k_rows_inv_planes, prow.smem_bytes());
  k_rows_inv_planes<<<g.H2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(prow.d, g, T2, nbands,
                                                                    planes, scale);
  ++lc.n;
}

void launch_cols_fwd_mac_inv(const FftPlan& pcol, const Geo& g, const float2* T1,
                             const float2* Fhat, size_t spec_stride, const Bands& b,
                             float2* Sigma, float2* T2, cudaStream_t st, LaunchCounter& lc) {
  set_smem(k_cols_fwd_mac_inv, pcol.smem_bytes());
  k_cols_fwd_mac_inv<<<g.Pw / 2, pcol.d.nt, pcol.smem_bytes(), st>>>(
      pcol.d, g, T1, Fhat, spec_stride, b, Sigma, T2);
  ++lc.n;
}

void launch_rows_inv_out(const FftPlan& prow, const Geo& g, const float2* T2, int out_kind,
                         void* out, int accumulate, const SigSrc& dcs, double dcr, double dci,
                         cudaStream_t st, LaunchCounter& lc, const float2* T2b) {
  const float scale = float(1.0 / (double(g.Ph) * double(g.Pw)));
  // T2b: a second launch adds conj(IFFT(T2b)) to the first one's output
  for (int pl = 0; pl < (T2b ? 2 : 1); ++pl) {
    const float2* src = pl ? T2b : T2;
    if (out_kind == OUT_C64) {
      set_smem(k_rows_inv_out<float2>, prow.smem_bytes());
      k_rows_inv_out<float2><<<g.H2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(
          prow.d, g, src, static_cast<float2*>(out), accumulate, pl, dcs, dcr, dci, scale);
    } else {
      set_smem(k_rows_inv_out<double2>, prow.smem_bytes());
      k_rows_inv_out<double2><<<g.H2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(
          prow.d, g, src, static_cast<double2*>(out), accumulate, pl, dcs, dcr, dci, scale);
    }
    ++lc.n;
  }
}

}  // namespace xcb
