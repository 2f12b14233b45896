// Forward row/column stages: F1, F2, S1 and the filter-spectrum build (K2).
#include "stages_common.cuh"

namespace xcb {
namespace {

// ------------------------------------------------------------------ F1
__global__ void __launch_bounds__(kMaxThreads) k_rows_fwd(FftPlanD p, Geo g, SigSrc s,
                                                          float2* __restrict__ T1) {
  extern __shared__ float2 sm[];
  const int b = blockIdx.x;
  auto load = [&](int n, int gi) -> float2 {
    const int ys = src_index(2 * b + gi, g.Hx, g.H, g.R, g.periodic);
    const int xs = src_index(n, g.Wx, g.W, g.R, g.periodic);
    if (ys < 0 || xs < 0) return make_float2(0.f, 0.f);
    return sig_value(s, size_t(ys) * g.W + xs);
  };
  auto store = [&](int k, int gi, float2 v) {
    T1[(size_t(k >> 1) * g.Hx2 + 2 * b + gi) * 2 + (k & 1)] = v;
  };
  fft_block(p, sm, load, store);
}

// ------------------------------------------------------------------ F2
__global__ void __launch_bounds__(kMaxThreads) k_cols_fwd(FftPlanD p, Geo g,
                                                          const float2* __restrict__ T1,
                                                          float2* __restrict__ spec) {
  extern __shared__ float2 sm[];
  const int c = blockIdx.x;
  const float2* src = T1 + size_t(c) * g.Hx2 * 2;
  float2* dst = spec + size_t(c) * g.Ph * 2;
  auto load = [&](int n, int gi) -> float2 {
    return n < g.Hx2 ? src[n * 2 + gi] : make_float2(0.f, 0.f);
  };
  auto store = [&](int k, int gi, float2 v) { dst[k * 2 + gi] = v; };
  fft_block(p, sm, load, store);
}

// ------------------------------------------------------------------ S1
__global__ void __launch_bounds__(kMaxThreads)
    k_rows_fwd_premul(FftPlanD p, Geo g, SigSrc s, const double* __restrict__ base,
                      Bands bl, float2* __restrict__ T1) {
  extern __shared__ float2 sm[];
  const int b = blockIdx.x;
  const size_t plane = size_t(g.Hx2) * g.Pw;
  for (int bi = 0; bi < bl.n; ++bi) {
    const int kf = bl.k[bi];
    float2* dst = T1 + size_t(bi) * plane;
    auto load = [&](int n, int gi) -> float2 {
      const int ys = src_index(2 * b + gi, g.Hx, g.H, g.R, g.periodic);
      const int xs = src_index(n, g.Wx, g.W, g.R, g.periodic);
      if (ys < 0 || xs < 0) return make_float2(0.f, 0.f);
      const size_t i = size_t(ys) * g.W + xs;
      return c_mul(sig_value(s, i), steer(kf, base[i], -1.f));  // H e^{-i k phi}
    };
    auto store = [&](int k, int gi, float2 v) {
      dst[(size_t(k >> 1) * g.Hx2 + 2 * b + gi) * 2 + (k & 1)] = v;
    };
    fft_block(p, sm, load, store);
    __syncthreads();
  }
}

// ------------------------------------------------------------ filter spectra
__global__ void __launch_bounds__(kMaxThreads)
    k_filter_rows(FftPlanD p, Geo g, const float2* __restrict__ comps,
                  float2* __restrict__ T1f) {
  extern __shared__ float2 sm[];
  const int b = blockIdx.x, band = blockIdx.y;
  const int S = 2 * g.R + 1, Hf2 = S + 1;
  const float2* f = comps + size_t(band) * S * S;
  float2* dst = T1f + size_t(band) * Hf2 * g.Pw;
  auto load = [&](int n, int gi) -> float2 {
    const int dy = 2 * b + gi;
    int x = n + g.R;
    if (x >= g.Pw) x -= g.Pw;
    return (dy < S && x < S) ? f[dy * S + x] : make_float2(0.f, 0.f);
  };
  auto store = [&](int k, int gi, float2 v) {
    dst[(size_t(k >> 1) * Hf2 + 2 * b + gi) * 2 + (k & 1)] = v;
  };
  fft_block(p, sm, load, store);
}

__global__ void __launch_bounds__(kMaxThreads)
    k_filter_cols(FftPlanD p, Geo g, const float2* __restrict__ T1f, size_t sstride,
                  float2* __restrict__ Fhat) {
  extern __shared__ float2 sm[];
  const int c = blockIdx.x, band = blockIdx.y;
  const int S = 2 * g.R + 1, Hf2 = S + 1;
  const float2* src = T1f + size_t(band) * Hf2 * g.Pw + size_t(c) * Hf2 * 2;
  float2* dst = Fhat + size_t(band) * sstride + size_t(c) * g.Ph * 2;
  auto load = [&](int n, int gi) -> float2 {
    int dy = n + g.R;
    if (dy >= g.Ph) dy -= g.Ph;
    return dy < S ? src[dy * 2 + gi] : make_float2(0.f, 0.f);
  };
  auto store = [&](int k, int gi, float2 v) { dst[k * 2 + gi] = v; };
  fft_block(p, sm, load, store);
}

}  // namespace

void launch_rows_fwd(const FftPlan& prow, const Geo& g, const SigSrc& s, float2* T1,
                     cudaStream_t st, LaunchCounter& lc) {
  set_smem(k_rows_fwd, prow.smem_bytes());
  k_rows_fwd<<<g.Hx2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(prow.d, g, s, T1);
  ++lc.n;
}

void launch_cols_fwd(const FftPlan& pcol, const Geo& g, const float2* T1, float2* spec,
                     cudaStream_t st, LaunchCounter& lc) {
  set_smem(k_cols_fwd, pcol.smem_bytes());
  k_cols_fwd<<<g.Pw / 2, pcol.d.nt, pcol.smem_bytes(), st>>>(pcol.d, g, T1, spec);
  ++lc.n;
}

void launch_rows_fwd_premul(const FftPlan& prow, const Geo& g, const SigSrc& s,
                            const double* base, const Bands& b, float2* T1, cudaStream_t st,
                            LaunchCounter& lc) {
  set_smem(k_rows_fwd_premul, prow.smem_bytes());
  k_rows_fwd_premul<<<g.Hx2 / 2, prow.d.nt, prow.smem_bytes(), st>>>(prow.d, g, s, base, b,
                                                                     T1);
  ++lc.n;
}

void launch_filter_spectra(const FftPlan& prow, const FftPlan& pcol, const Geo& g,
                           const float2* comps, int nb, float2* T1f, float2* Fhat,
                           cudaStream_t st, LaunchCounter& lc) {
  const int S = 2 * g.R + 1;
  set_smem(k_filter_rows, prow.smem_bytes());
  k_filter_rows<<<dim3((S + 1) / 2, nb), prow.d.nt, prow.smem_bytes(), st>>>(prow.d, g, comps,
                                                                            T1f);
  set_smem(k_filter_cols, pcol.smem_bytes());
  k_filter_cols<<<dim3(g.Pw / 2, nb), pcol.d.nt, pcol.smem_bytes(), st>>>(
      pcol.d, g, T1f, size_t(g.Ph) * g.Pw, Fhat);
  lc.n += 2;
}

}  // namespace xcb
