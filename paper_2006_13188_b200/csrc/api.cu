// C ABI implementation (include/xconv_b200.h): contexts, filter spectrum cache,
// and the gather / scatter / smooth / angle-max pipelines.
//
// Pipeline per image (kernels.h for the layouts):
//   gather  (xcorr_fast, engine.hpp:286-326):
//     prep(base) -> F1 rows -> F2 cols (H^) -> I1 cols^-1 per band (x conj F^_k)
//     -> I2 rows^-1 per band, steer e^{+i k phi}, accumulate (+ conj(dc) H)
//   scatter (xconv_fast, engine.hpp:331-373):
//     prep -> S1 rows per band of H e^{-i k phi} -> S2 cols per band, x F^_k,
//     summed in frequency (the B inverse FFTs of the reference collapse into
//     one), col^-1 -> S4 rows^-1 (+ dc H)
//   smooth  (smooth_adaptive, engine.hpp:385-419): scatter(H w), scatter(w),
//     max|den|, floored divide
//   anglemax: gather's per-band responses G_k -> max_s |sum_k e^{-iks} G_k|
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <functional>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/xconv_b200.h"
#include "fft_plan.h"
#include "host_filter.h"
#include "kernels.h"
#include "host_sph.h"
#include "kernels3d.h"

namespace {

using xcb::cplx;

struct CudaError : std::runtime_error {
  int code;
  CudaError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = e == cudaErrorMemoryAllocation ? XC_ENOMEM : XC_ECUDA;
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e), code);
  }
}

thread_local std::string g_thread_err;

struct PlanEntry {
  xcb::FftPlan plan;
  float2* tw = nullptr;
};

struct DevBuf {
  void* p = nullptr;   // the allocation
  size_t n = 0;        // usable bytes (after the leading guard)
  size_t guard = 0;    // guard bytes on each side (XCB_GUARD)
  void* user() const { return static_cast<char*>(p) + guard; }
};

// XCB_GUARD=<bytes>: debug mode for out-of-bounds checks (compute-sanitizer is
// not available on the GPU pool).  Every context buffer gets a guard zone on
// each side, and the whole allocation is poisoned with 0xFF bytes (a NaN in
// fp32 and fp64): a stray write shows up as a changed guard byte
// (xc_debug_check_guards), a stray or uninitialised read as NaN in the output,
// which the parity tests compare with the oracle.
size_t guard_bytes() {
  static const size_t g = [] {
    const char* e = std::getenv("XCB_GUARD");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? (size_t(v) + 255) / 256 * 256 : size_t(0);
  }();
  return g;
}

struct StageEvents {
  const char* name;
  cudaEvent_t a, b;
};

struct StageTotal {
  double ms = 0;
  long long launches = 0;
};

// multi-device / multi-rank state of a context (defined with the group layer)
struct Group;
void destroy_group(Group* g);

}  // namespace

struct xc_context_s {
  int device = 0;
  Group* group = nullptr;  // set for xc_context_create_multi / _rank contexts
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t cp_in = nullptr, cp_out = nullptr;  // host-memory copy pipeline
  std::string err;
  std::mutex mu;
  std::map<int, PlanEntry> plans;
  std::map<int, PlanEntry> fast_plans;  // L -> in-place radix-16-last plan (or tw == null)
  std::map<std::string, DevBuf> bufs;
  // device copies of band tables (ks, spectrum indices), uploaded once per
  // distinct table: no per-call host->device copy, so device-memory calls
  // can be captured in a CUDA graph
  std::map<std::vector<int>, int*> band_tables;
  // detect_pattern's decomposed vote filters, by content (xc_detect_pattern)
  std::map<uint64_t, std::unique_ptr<xc_filter_s, void (*)(xc_filter_s*)>> det_filters;
  // events reused across calls (HostPipe slots, call timing)
  std::vector<cudaEvent_t> ev_sync, ev_timing;
  size_t ev_sync_used = 0, ev_timing_used = 0;
  cudaEvent_t event(bool timing) {
    auto& pool = timing ? ev_timing : ev_sync;
    size_t& used = timing ? ev_timing_used : ev_sync_used;
    if (used == pool.size()) {
      cudaEvent_t e;
      ck(timing ? cudaEventCreate(&e) : cudaEventCreateWithFlags(&e, cudaEventDisableTiming),
         "event");
      pool.push_back(e);
    }
    return pool[used++];
  }
  void release_events() { ev_sync_used = ev_timing_used = 0; }
  // per-stage CUDA-event profile (xc_profile_*): events are recorded on the
  // launch stream around each stage and resolved at the call's sync points
  bool profiling = false;
  std::vector<StageEvents> pending;
  std::vector<std::pair<std::string, StageTotal>> prof;

  void resolve_profile() {
    for (auto& e : pending) {
      float ms = 0;
      cudaEventElapsedTime(&ms, e.a, e.b);
      auto it = std::find_if(prof.begin(), prof.end(),
                             [&](const std::pair<std::string, StageTotal>& p) {
                               return p.first == e.name;
                             });
      if (it == prof.end()) it = prof.insert(prof.end(), {e.name, StageTotal{}});
      it->second.ms += ms;
      it->second.launches += 1;
    }
    pending.clear();
  }

  ~xc_context_s() {
    if (group) destroy_group(group);
    cudaSetDevice(device);
    for (auto& kv : plans) cudaFree(kv.second.tw);
    for (auto& kv : fast_plans) cudaFree(kv.second.tw);
    for (auto& kv : bufs) cudaFree(kv.second.p);
    for (auto& kv : band_tables) cudaFree(kv.second);
    for (cudaEvent_t e : ev_sync) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_timing) cudaEventDestroy(e);
    if (own) cudaStreamDestroy(own);
    if (cp_in) cudaStreamDestroy(cp_in);
    if (cp_out) cudaStreamDestroy(cp_out);
  }

  const xcb::FftPlan& plan(int L) {
    auto it = plans.find(L);
    if (it != plans.end()) return it->second.plan;
    PlanEntry e;
    if (!xcb::make_fft_plan(L, &e.plan)) throw std::invalid_argument("unsupported transform length");
    e.tw = xcb::upload_twiddles(e.plan);
    if (!e.tw) throw CudaError("twiddle upload failed", XC_ENOMEM);
    e.plan.d.tw = e.tw;
    return plans.emplace(L, std::move(e)).first->second.plan;
  }

  // plans with radices <= 10 for the 3D tile kernels (k_3d.cu), keyed -L
  const xcb::FftPlan& plan3(int L) {
    auto it = plans.find(-L);
    if (it != plans.end()) return it->second.plan;
    PlanEntry e;
    if (!xcb::make_fft_plan_maxr(L, 10, &e.plan))
      throw std::invalid_argument("unsupported transform length");
    e.tw = xcb::upload_twiddles(e.plan);
    if (!e.tw) throw CudaError("twiddle upload failed", XC_ENOMEM);
    e.plan.d.tw = e.tw;
    return plans.emplace(-L, std::move(e)).first->second.plan;
  }

  // nullptr if L has no fast plan
  const xcb::FftPlan* fast_plan(int L) {
    auto it = fast_plans.find(L);
    if (it == fast_plans.end()) {
      PlanEntry e;
      if (xcb::make_fast_plan(L, &e.plan)) {
        e.tw = xcb::upload_twiddles(e.plan);
        if (!e.tw) throw CudaError("twiddle upload failed", XC_ENOMEM);
        e.plan.d.tw = e.tw;
      }
      it = fast_plans.emplace(L, std::move(e)).first;
    }
    return it->second.tw ? &it->second.plan : nullptr;
  }

  int* band_table(const std::vector<int>& hb) {
    auto it = band_tables.find(hb);
    if (it != band_tables.end()) return it->second;
    int* d = nullptr;
    ck(cudaMalloc(&d, std::max<size_t>(hb.size(), 1) * sizeof(int)), "cudaMalloc bands");
    ck(cudaMemcpy(d, hb.data(), hb.size() * sizeof(int), cudaMemcpyHostToDevice), "upload bands");
    return band_tables.emplace(hb, d).first->second;
  }

  template <class T>
  T* buf(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    DevBuf& b = bufs[name];
    if (b.n < bytes) {
      if (b.p) {
        ck(cudaStreamSynchronize(stream), "sync before realloc");
        cudaFree(b.p);
        b.p = nullptr;
        b.n = 0;
      }
      const size_t g = guard_bytes();
      ck(cudaMalloc(&b.p, bytes + 2 * g), ("cudaMalloc " + name).c_str());
      b.n = bytes;
      b.guard = g;
      if (g) ck(cudaMemsetAsync(b.p, 0xff, bytes + 2 * g, stream), "poison");
    }
    return static_cast<T*>(b.user());
  }
};

// A filter is host data plus per-(device, pad, orientation) spectrum caches;
// it is not bound to a context, so host-only calls need no GPU.
struct xc_filter_s {
  xcb::HostFilter hf;
  // A filter handle may be shared by callers on several threads, each with its
  // own context: `mu` guards the spectrum cache and the integral check.
  std::mutex mu;
  std::map<std::tuple<int, int, int, int>, float2*> spectra;  // (dev, Ph, Pw, transposed)
  int integral_state = -1;  // smooth_adaptive zero-integral check cache
  ~xc_filter_s() {
    for (auto& kv : spectra) {
      cudaSetDevice(std::get<0>(kv.first));
      cudaFree(kv.second);
    }
  }
};

namespace {

template <class Fn>
int guarded(xc_context ctx, Fn&& fn) {
  std::string* err = ctx ? &ctx->err : &g_thread_err;
  try {
    fn();
    return XC_OK;
  } catch (const CudaError& e) {
    *err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    *err = e.what();
    return XC_EINVAL;
  } catch (const std::bad_alloc&) {
    *err = "host allocation failed";
    return XC_ENOMEM;
  } catch (const std::exception& e) {
    *err = e.what();
    return XC_EINTERNAL;
  }
}

size_t dtype_size(int dt) {
  switch (dt) {
    case XC_F32: return 4;
    case XC_F64: return 8;
    case XC_C64: return 8;
    case XC_C128: return 16;
  }
  throw std::invalid_argument("unknown dtype");
}

std::vector<cplx> to_rowmajor(const double* data, int height, int width, int layout) {
  std::vector<cplx> v(size_t(height) * width);
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < width; ++x) {
      const size_t s = layout == XC_COL_MAJOR ? size_t(x) * height + y : size_t(y) * width + x;
      v[size_t(y) * width + x] = cplx(data[2 * s], data[2 * s + 1]);
    }
  return v;
}

void export_filter(const xcb::HostFilter& f, int* ks, double* comps, int* nc) {
  const int n = f.nc(), rows = f.n_rows();
  for (int i = 0; i < n; ++i) ks[i] = f.ks[i];
  for (int ci = 0; ci < n; ++ci)
    for (int r = 0; r < rows; ++r) {  // Eigen column-major (row + ci * n_rows)
      comps[2 * (size_t(ci) * rows + r)] = f.comp(r, ci).real();
      comps[2 * (size_t(ci) * rows + r) + 1] = f.comp(r, ci).imag();
    }
  *nc = n;
}

// Resolved geometry and per-call state shared by the pipelines.
struct Call {
  bool packed = false;  // smoothing: num + i alpha den from one scatter (SIG_PACK)
  xc_context ctx;
  xc_filter f;
  xc_image_desc d;
  int rows, cols, transposed;
  xcb::Geo g;
  const xcb::FftPlan* prow;
  const xcb::FftPlan* pcol;
  const xcb::FftPlan* frow;  // fast plans (nullptr: generic kernels)
  const xcb::FftPlan* fcol;
  std::vector<int> ks;     // selected band frequencies
  std::vector<int> sidx;   // spectrum index of each
  xcb::Bands bands;
  float2* Fhat;
  size_t sstride;
  xcb::LaunchCounter lc;
  cudaStream_t st;
  double h2d_s = 0, d2h_s = 0;
  bool out_dev = false;  // outputs are device buffers even when d.memory == XC_HOST
  int nb_run = 0;        // bands transformed per image (Hermitian half-band: k >= 0)
  int band_mode = 0;     // xc_stats::band_mode
};

std::vector<int> plan_components(const xcb::HostFilter& hf, const int* comps, int n) {
  // engine.hpp:51-58
  if (comps == nullptr || n <= 0) return hf.ks;
  std::vector<int> out(comps, comps + n);
  for (int k : out)
    if (std::find(hf.ks.begin(), hf.ks.end(), k) == hf.ks.end())
      throw std::invalid_argument("plan retains a component the filter lacks");
  return out;
}

float2* filter_spectra(Call& c) {
  const auto key = std::make_tuple(c.ctx->device, c.g.Ph, c.g.Pw, c.transposed);
  std::lock_guard<std::mutex> flk(c.f->mu);  // one build per key across threads
  auto it = c.f->spectra.find(key);
  if (it != c.f->spectra.end()) return it->second;
  const xcb::HostFilter& hf = c.f->hf;
  const int R = c.g.R, S = 2 * R + 1, nb = hf.nc();
  // render every band once on the GPU (freq_filter.hpp:173-184; the host
  // render_component is the same formula), fp64 -> fp32
  std::vector<double2> hc(hf.comps.size());
  for (size_t i = 0; i < hc.size(); ++i) hc[i] = make_double2(hf.comps[i].real(), hf.comps[i].imag());
  double2* dtab = c.ctx->buf<double2>("filter_table", hc.size());
  int* dks = c.ctx->buf<int>("filter_ks", size_t(nb));
  ck(cudaMemcpyAsync(dtab, hc.data(), hc.size() * sizeof(double2), cudaMemcpyHostToDevice, c.st),
     "upload filter table");
  ck(cudaMemcpyAsync(dks, hf.ks.data(), size_t(nb) * sizeof(int), cudaMemcpyHostToDevice, c.st),
     "upload ks");
  float2* dcomps = c.ctx->buf<float2>("filter_comps", size_t(nb) * S * S);
  xcb::launch_render(dtab, dks, nb, hf.group, hf.n_radii, hf.n_angles, hf.r_max, hf.r_min,
                     hf.group == 1 ? hf.omega() : 0.0, S, R, c.transposed != 0, dcomps, c.st,
                     c.lc);
  float2* T1f = c.ctx->buf<float2>("filter_T1", size_t(nb) * (S + 1) * c.g.Pw);
  float2* spec = nullptr;
  ck(cudaMalloc(&spec, size_t(nb) * c.g.Ph * c.g.Pw * sizeof(float2)), "cudaMalloc spectra");
  if (guard_bytes())  // XCB_GUARD: poisoned, so a spectrum element never written reads NaN
    ck(cudaMemsetAsync(spec, 0xff, size_t(nb) * c.g.Ph * c.g.Pw * sizeof(float2), c.st),
       "poison");
  xcb::launch_filter_spectra(*c.prow, *c.pcol, c.g, dcomps, nb, T1f, spec, c.st, c.lc);
  ck(cudaGetLastError(), "filter spectra launch");
  ck(cudaStreamSynchronize(c.st), "filter spectra");  // host table lifetime
  c.f->spectra[key] = spec;
  return spec;
}

// Spectra of the conjugated components, G_i = FFT2(conj f_i) = conj(F^_i[-v, -u]),
// built from the cached F^ on first use by a real-signal scatter (conjugate
// band pairs, run_scatter); cached beside F^ under (dev, Ph, Pw, transposed + 2).
float2* filter_spectra_conj(Call& c) {
  const auto key = std::make_tuple(c.ctx->device, c.g.Ph, c.g.Pw, c.transposed + 2);
  std::lock_guard<std::mutex> flk(c.f->mu);
  auto it = c.f->spectra.find(key);
  if (it != c.f->spectra.end()) return it->second;
  const int nb = c.f->hf.nc();
  float2* spec = nullptr;
  ck(cudaMalloc(&spec, size_t(nb) * c.g.Ph * c.g.Pw * sizeof(float2)), "cudaMalloc spectra");
  xcb::launch_spec_conj_reflect(c.Fhat, spec, nb, c.g.Ph, c.g.Pw, c.st, c.lc);
  // complete before the entry is published: another context (its own stream)
  // may find it in the shared filter's cache right after
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
  if (e != cudaSuccess) {
    cudaFree(spec);
    ck(e, "conjugated spectra");
  }
  c.f->spectra[key] = spec;
  return spec;
}

// XCB_CPAIR=0 disables the scatter's conjugate band pairs (A/B timing, tests)
bool use_cpair() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_CPAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Pad (transform length) for an extent needing >= n points: any length >= n
// gives the same zero-padded linear filtering (fft.hpp:85-86 uses
// next_fast_size(extent + 2R + 1)); prefer a length with a fast plan (k_fast.cu)
// when it costs at most 15% over the smallest 2/3/5-smooth length.
int pick_pad_uncached(int n);
// pad sizes are cached: the search builds candidate plans
int pick_pad(int n) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  return cache[n] = pick_pad_uncached(n);
}

int pick_pad_uncached(int n) {
  const int L0 = xcb::pick_fft_length(n);
  if (L0 < 0) return L0;
  for (int s = n; s <= L0 + L0 / 7; ++s) {
    if (s % 2 || !xcb::is_smooth235(s)) continue;
    xcb::FftPlan p;
    if (xcb::make_fast_plan(s, &p)) return s;
  }
  return L0;
}

bool use_pair();

// Pad of a 2D pipeline axis needing >= n points.  The three kernel families
// cost very different amounts per transformed point: measured with
// tools/pad_sweep.py (17 bands, device-resident), per point of the padded
// grid, the pair engine (k_pair.cu) 1.0, the fast kernels (k_fast.cu) ~1.6,
// the generic kernels ~8 (xconv 800^2 at pad 810: 0.555 ms; 900^2 at pad
// 1152: 0.128 ms).  Per axis that is 1 / 1.25 / 2.8, so the pad is the
// candidate (smallest generic length, every fast length, every pair length)
// with the least length x weight.  XCB_PAD_RULE=0 keeps pick_pad's choice.
int pick_pad2d(int n) {
  static const bool on = [] {
    const char* e = std::getenv("XCB_PAD_RULE");
    return !(e && e[0] == '0');
  }();
  const int p = pick_pad(n);
  if (!on || p < 0) return p;
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  xcb::FftPlan tmp;
  int best = p;
  double cost = double(p) * (xcb::make_fast_plan(p, &tmp) ? 1.25 : 2.8);
  auto consider = [&](int L, double w) {
    if (L >= n && L % 2 == 0 && L * w < cost) {
      cost = L * w;
      best = L;
    }
  };
#define XCB_PAD_FAST(LL, R0, R1, RL) consider(LL, 1.25);
  XCB_FAST_TABLE(XCB_PAD_FAST)
#undef XCB_PAD_FAST
  if (use_pair())
    for (int L : xcb::pair_plan_lengths()) consider(L, 1.0);
  return cache[n] = best;
}

Call setup(xc_context ctx, xc_filter f, const xc_image_desc* d, int group_required,
           const int* components, int ncomp, bool periodic) {
  if (!ctx || !f || !d) throw std::invalid_argument("null argument");
  Call c{};
  c.ctx = ctx;
  c.f = f;
  c.d = *d;
  c.st = ctx->stream;
  if (d->height < 1 || d->width < 1 || d->batch < 1)
    throw std::invalid_argument("image dims must be positive");
  // engine.hpp:288-291
  const int kind = group_required >= 0 ? group_required : d->xform_kind;
  if (kind != f->hf.group) throw std::invalid_argument("transformation/filter group mismatch");
  if (kind == XC_ROTATION3) throw std::invalid_argument("2D pipeline needs a 2D field");
  c.transposed = d->layout == XC_COL_MAJOR;
  c.rows = c.transposed ? d->width : d->height;
  c.cols = c.transposed ? d->height : d->width;
  const int R = f->hf.render_radius();
  xcb::Geo& g = c.g;
  g.H = c.rows;
  g.W = c.cols;
  g.R = R;
  g.periodic = periodic ? 1 : 0;
  g.Hx = periodic ? c.rows + 2 * R : c.rows;
  g.Wx = periodic ? c.cols + 2 * R : c.cols;
  g.Hx2 = (g.Hx + 1) & ~1;
  g.H2 = (g.H + 1) & ~1;
  g.off = periodic ? R : 0;
  // zero-padded linear filtering needs P >= extent + R and no wrap of the
  // 2R+1 taps (fft.hpp:85-86 uses next_fast_size(extent + 2R + 1))
  g.Ph = pick_pad2d(std::max(g.Hx + R, 2 * R + 1));
  g.Pw = pick_pad2d(std::max(g.Wx + R, 2 * R + 1));
  if (g.Ph < 0 || g.Pw < 0) throw std::invalid_argument("image too large for the FFT planner");
  while (g.Pw % 2) g.Pw = xcb::pick_fft_length(g.Pw + 1);
  c.prow = &ctx->plan(g.Pw);
  c.pcol = &ctx->plan(g.Ph);
  c.frow = ctx->fast_plan(g.Pw);
  c.fcol = ctx->fast_plan(g.Ph);
  // bands in descending k: the fast kernels steer with Horner's rule (the
  // reference sums in ascending order; only the rounding order differs)
  std::vector<int> ks = plan_components(f->hf, components, ncomp);
  std::stable_sort(ks.begin(), ks.end(), [](int a, int b) { return a > b; });
  c.ks = ks;
  for (int k : c.ks) c.sidx.push_back(f->hf.index_of(k));
  c.Fhat = filter_spectra(c);
  c.sstride = size_t(g.Ph) * g.Pw;
  std::vector<int> hb(c.ks);
  hb.insert(hb.end(), c.sidx.begin(), c.sidx.end());
  int* dband = ctx->band_table(hb);
  c.bands = xcb::Bands{dband, dband + c.ks.size(), int(c.ks.size())};
  return c;
}

// Wrap one stage's launches in profiling events (no-op unless enabled).
template <class Fn>
void stage(Call& c, const char* name, Fn&& fn) {
  // NVTX range per stage (the reference's StageTimer, engine.hpp:41-49): free
  // without a tool attached, named ranges under ncu --nvtx / nsys
  struct Range {
    explicit Range(const char* n) { nvtxRangePushA(n); }
    ~Range() { nvtxRangePop(); }
  } range(name);
  if (!c.ctx->profiling) {
    fn();
    return;
  }
  StageEvents e{name, c.ctx->event(true), c.ctx->event(true)};  // pooled, reused after resolve
  ck(cudaEventRecord(e.a, c.st), "event");
  fn();
  ck(cudaEventRecord(e.b, c.st), "event");
  c.ctx->pending.push_back(e);
}

double event_seconds(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e-3;
}

// Stage one image's signal / param on the device; returns device pointers.
struct Staged {
  xcb::SigSrc sig;
  const void* param;
  int param_f64;
};

// Host-memory batches run a two-slot pipeline: H2D of image i+1 (cp_in) and
// D2H of image i-1 (cp_out) overlap the kernels of image i (compute stream).
struct HostPipe {
  Call* c = nullptr;
  bool host = false;      // inputs in host memory
  bool host_out = false;  // outputs in host memory
  static constexpr int NS = 4;  // slots: two groups of up to two images in flight
  cudaEvent_t in_done[NS]{}, comp_done[NS]{}, out_done[NS]{}, t0{}, t1{};
  int issued = 0;
  // events come from the context's pool (released when the call returns)
  explicit HostPipe(Call& call)
      : c(&call), host(call.d.memory == XC_HOST), host_out(call.d.memory == XC_HOST && !call.out_dev) {
    if (!host && !host_out) return;
    for (int s = 0; s < NS; ++s) {
      in_done[s] = call.ctx->event(false);
      comp_done[s] = call.ctx->event(false);
      out_done[s] = call.ctx->event(false);
    }
  }
  size_t npix() const { return size_t(c->rows) * c->cols; }
  static std::string slot_name(const char* b, int s) { return b + std::to_string(s); }
  // issue the H2D copies of image img into slot img % NS (host memory only)
  void h2d(const void* signal, const void* param, int img) {
    if (!host || img >= c->d.batch) return;
    const int s = img % NS;
    const size_t ss = dtype_size(c->d.signal_dtype), ps = dtype_size(c->d.param_dtype);
    void* bs = c->ctx->buf<char>(slot_name("sig_raw", s), npix() * ss);
    void* bp = param ? c->ctx->buf<char>(slot_name("param_raw", s), npix() * ps) : nullptr;
    if (img >= NS) ck(cudaStreamWaitEvent(c->ctx->cp_in, comp_done[s], 0), "wait");
    ck(cudaMemcpyAsync(bs, static_cast<const char*>(signal) + size_t(img) * npix() * ss,
                       npix() * ss, cudaMemcpyHostToDevice, c->ctx->cp_in),
       "H2D signal");
    if (param) {
      const char* src = static_cast<const char*>(param) +
                        (c->d.param_per_image ? size_t(img) * npix() * ps : 0);
      ck(cudaMemcpyAsync(bp, src, npix() * ps, cudaMemcpyHostToDevice, c->ctx->cp_in),
         "H2D param");
    }
    ck(cudaEventRecord(in_done[s], c->ctx->cp_in), "event");
  }
  // device pointers of image img's inputs, ready on the compute stream
  Staged inputs(const void* signal, const void* param, int img) {
    const xc_image_desc& d = c->d;
    const size_t ss = dtype_size(d.signal_dtype), ps = dtype_size(d.param_dtype);
    const bool cplx_sig = d.signal_dtype == XC_C64 || d.signal_dtype == XC_C128;
    const int s = img % NS;
    Staged st{};
    const void* dsig;
    const void* dpar = nullptr;
    if (host) {
      ck(cudaStreamWaitEvent(c->st, in_done[s], 0), "wait");
      dsig = c->ctx->buf<char>(slot_name("sig_raw", s), npix() * ss);
      if (param) dpar = c->ctx->buf<char>(slot_name("param_raw", s), npix() * ps);
    } else {
      dsig = static_cast<const char*>(signal) + size_t(img) * npix() * ss;
      if (param)
        dpar = static_cast<const char*>(param) + (d.param_per_image ? size_t(img) * npix() * ps : 0);
    }
    if (d.signal_dtype == XC_F64 || d.signal_dtype == XC_C128) {
      void* b = c->ctx->buf<char>(slot_name("sig_f32_", s), npix() * (cplx_sig ? 8 : 4));
      xcb::launch_convert_signal(dsig, d.signal_dtype, npix(), b, c->st, c->lc);
      dsig = b;
    }
    st.sig = xcb::SigSrc{dsig, cplx_sig ? 1 : 0, nullptr, xcb::SIG_PLAIN};
    st.param = dpar;
    st.param_f64 = d.param_dtype == XC_F64;
    return st;
  }
  // output buffer of image img (device: the caller's; host: a slot stage)
  void* out_buffer(void* out, int img, size_t os) {
    if (!host_out) return static_cast<char*>(out) + size_t(img) * npix() * os;
    const int s = img % NS;
    if (img >= NS) ck(cudaStreamWaitEvent(c->st, out_done[s], 0), "wait");
    return c->ctx->buf<char>(slot_name("out_stage", s), npix() * os);
  }
  // after image img's kernels: start its D2H (host memory)
  void done(void* out, int img, void* dout, size_t os) {
    if (!host && !host_out) return;
    const int s = img % NS;
    ck(cudaEventRecord(comp_done[s], c->st), "event");  // input slot s free again
    if (!host_out) return;
    ck(cudaStreamWaitEvent(c->ctx->cp_out, comp_done[s], 0), "wait");
    ck(cudaMemcpyAsync(static_cast<char*>(out) + size_t(img) * npix() * os, dout, npix() * os,
                       cudaMemcpyDeviceToHost, c->ctx->cp_out),
       "D2H");
    ck(cudaEventRecord(out_done[s], c->ctx->cp_out), "event");
  }
  void finish() {
    if (host_out) ck(cudaStreamSynchronize(c->ctx->cp_out), "D2H");
    ck(cudaStreamSynchronize(c->st), "compute");
  }
};

Staged stage_inputs(Call& c, const void* signal, const void* param, int img) {
  // synchronous single-image staging (smooth / anglemax paths)
  HostPipe hp(c);
  hp.h2d(signal, param, img);
  Staged s = hp.inputs(signal, param, img);
  if (hp.host) ck(cudaStreamSynchronize(c.st), "H2D");
  return s;
}

// base (steering phase per pixel) + optional weights.  For scale fields the
// kernel also records, per image, the first y-major pixel that is not positive
// and finite and the first outside the guard band (engine.hpp:267-279,
// field.hpp:150-153); guard_check() reads all images' slots back once per call.
void guard_begin(Call& c) {
  if (c.f->hf.group != XC_SCALE2) return;
  unsigned long long* bad = c.ctx->buf<unsigned long long>("bad", 2 * size_t(c.d.batch));
  ck(cudaMemsetAsync(bad, 0xff, 2 * size_t(c.d.batch) * sizeof(unsigned long long), c.st),
     "memset");
}

void prep(Call& c, const Staged& s, bool want_wgt, double** base_out, float** wgt_out,
          int slot = 0, int img = 0) {
  const size_t npix = size_t(c.rows) * c.cols;
  double* base = c.ctx->buf<double>("base" + std::to_string(slot), npix);
  float* wgt = want_wgt ? c.ctx->buf<float>("wgt" + std::to_string(slot), npix) : nullptr;
  const xcb::HostFilter& hf = c.f->hf;
  const bool scale = hf.group == 1;
  unsigned long long* bad =
      scale ? c.ctx->buf<unsigned long long>("bad", 2 * size_t(c.d.batch)) + 2 * size_t(img)
            : nullptr;
  const double lo = scale ? hf.r_min / hf.domain_top() : 0, hi = scale ? hf.domain_top() / hf.r_min : 0;
  stage(c, "prep", [&] {
    xcb::launch_prep(s.param, s.param_f64, hf.group, scale ? hf.omega() : 0.0, lo, hi, c.rows,
                     c.cols, c.transposed, base, wgt, bad, c.st, c.lc);
  });
  *base_out = base;
  if (wgt_out) *wgt_out = wgt;
}

// One readback per call: throw the reference's error for the first image (in
// batch order) whose scale field failed, naming its first offending pixel.
// `param` is the caller's pointer (d.memory), not a staging slot.
void guard_check(Call& c, const void* param) {
  if (c.f->hf.group != XC_SCALE2) return;
  const int B = c.d.batch;
  std::vector<unsigned long long> hbad(2 * size_t(B));
  ck(cudaMemcpyAsync(hbad.data(), c.ctx->buf<unsigned long long>("bad", 2 * size_t(B)),
                     hbad.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.st),
     "guard readback");
  ck(cudaStreamSynchronize(c.st), "guard");
  const xcb::HostFilter& hf = c.f->hf;
  const double lo = hf.r_min / hf.domain_top(), hi = hf.domain_top() / hf.r_min;
  const size_t npix = size_t(c.rows) * c.cols, ps = dtype_size(c.d.param_dtype);
  for (int img = 0; img < B; ++img) {
    if (hbad[2 * img] != ~0ull)
      throw std::invalid_argument("scale field must be strictly positive and finite");
    if (hbad[2 * img + 1] != ~0ull) {
      const unsigned long long ti = hbad[2 * img + 1];
      const int W = c.d.width;  // true (un-transposed) width
      const int x = int(ti % W), y = int(ti / W);
      const size_t si = (c.transposed ? size_t(x) * c.d.height + y : size_t(y) * c.d.width + x) +
                        (c.d.param_per_image ? size_t(img) * npix : 0);
      double sv = 0;
      const char* src = static_cast<const char*>(param) + si * ps;
      if (c.d.memory == XC_HOST)
        std::memcpy(&sv, src, ps);
      else
        ck(cudaMemcpy(&sv, src, ps, cudaMemcpyDeviceToHost), "guard value");
      if (ps == 4) {
        float fv;
        std::memcpy(&fv, &sv, 4);
        sv = fv;
      }
      throw std::invalid_argument("scale factor " + std::to_string(sv) + " at pixel (" +
                                  std::to_string(x) + "," + std::to_string(y) +
                                  ") outside guard band [" + std::to_string(lo) + "," +
                                  std::to_string(hi) + "]");
    }
  }
}

// XCB_PAIR=0 selects the previous (fast) band-loop kernels, for A/B timing
bool use_pair() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// F1 / F2 / S4 (single transforms): pair engine when the length has a plan
void run_f1(Call& c, const xcb::SigSrc& sig, float2* T1) {
  if (use_pair() && xcb::pair_smem(5, c.g.Pw, c.g))
    xcb::launch_rows_fwd_pair(c.g, sig, T1, c.st, c.lc);
  else if (c.frow && xcb::fast_smem(5, *c.frow, c.g))
    xcb::launch_rows_fwd_fast(*c.frow, c.g, sig, T1, c.st, c.lc);
  else
    xcb::launch_rows_fwd(*c.prow, c.g, sig, T1, c.st, c.lc);
}
void run_f2(Call& c, const float2* T1, float2* Hh) {
  if (use_pair() && xcb::pair_smem(6, c.g.Ph, c.g))
    xcb::launch_cols_fwd_pair(c.g, T1, Hh, c.st, c.lc);
  else if (c.fcol && xcb::fast_smem(5, *c.fcol, c.g))
    xcb::launch_cols_fwd_fast(*c.fcol, c.g, T1, Hh, c.st, c.lc);
  else
    xcb::launch_cols_fwd(*c.pcol, c.g, T1, Hh, c.st, c.lc);
}

// XCB_ANGLE_TC=0: the Hermitian angle max on the CUDA cores (k_anglemax_herm)
// instead of the tensor cores (k_anglemax_tc.cu)
bool use_angle_tc() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_ANGLE_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

// XCB_HERM=0 disables the Hermitian half-band paths (A/B timing, tests)
bool use_herm() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_HERM");
    return !(e && e[0] == '0');
  }();
  return on;
}

xcb::Bands half_bands(Call& c, bool real_sig);

// half: Hermitian half-band mode (bands = half_bands(), pair-engine I2 only)
void launch_i2(Call& c, const xcb::SigSrc& sig, const float2* T2, const xcb::Bands& bands,
               bool half, const double* base, void* out, int out_kind, bool accumulate, bool dc) {
  const xcb::Geo& g = c.g;
  const cplx dcv = dc ? std::conj(xcb::inner_dc_value(c.f->hf)) : cplx(0);  // engine.hpp:323
  if (half || (use_pair() && xcb::pair_smem(1, g.Pw, g))) {
    stage(c, "I2_rows_inv_steer", [&] {
      xcb::launch_rows_inv_steer_pair(g, T2, bands, half ? 1 : 0, base, out_kind, out, accumulate ? 1 : 0,
                                      sig, dcv.real(), dcv.imag(), c.st, c.lc);
    });
  } else if (c.frow && xcb::fast_smem(1, *c.frow, g)) {
    stage(c, "I2_rows_inv_steer", [&] {
      const int nch = xcb::fast_steer_chunks(g, c.bands.n);
      float2* parts = nch > 1 ? c.ctx->buf<float2>("steer_parts", size_t(nch) * g.H * g.W)
                              : nullptr;
      xcb::launch_rows_inv_steer_fast(*c.frow, g, T2, c.bands, base, out_kind, out,
                                      accumulate ? 1 : 0, sig, dcv.real(), dcv.imag(), parts,
                                      c.st, c.lc);
    });
  } else {
    stage(c, "I2_rows_inv_steer", [&] {
      xcb::launch_rows_inv_steer(*c.prow, g, T2, c.bands, base, out_kind, out,
                                 accumulate ? 1 : 0, sig, dcv.real(), dcv.imag(), c.st, c.lc);
    });
  }
}

// gather bands: the Hermitian half-band subset (k >= 0) when every signal is
// real, the filter hermitian() and the pair-engine I2 applies, else c.bands
xcb::Bands gather_bands(Call& c, const xcb::SigSrc* sig, int nsig, bool* half) {
  *half = false;
  if (!use_pair() || !xcb::pair_smem(1, c.g.Pw, c.g)) return c.bands;
  bool real = true;
  for (int i = 0; i < nsig; ++i) real = real && !sig[i].is_complex;
  const xcb::Bands hb = half_bands(c, real);
  if (hb.n == 0) return c.bands;
  *half = true;
  return hb;
}

void run_gather(Call& c, const xcb::SigSrc& sig, const double* base, void* out, int out_kind,
                bool accumulate, bool dc) {
  const xcb::Geo& g = c.g;
  bool half;
  const xcb::Bands bands = gather_bands(c, &sig, 1, &half);
  c.nb_run = bands.n;
  c.band_mode = half ? 1 : 0;
  float2* T1 = c.ctx->buf<float2>("T1", size_t(g.Hx2) * g.Pw);
  float2* Hh = c.ctx->buf<float2>("Hhat", size_t(g.Ph) * g.Pw);
  float2* T2 = c.ctx->buf<float2>("T2", size_t(bands.n) * g.H2 * g.Pw);
  stage(c, "F1_rows_fwd", [&] { run_f1(c, sig, T1); });
  stage(c, "F2_cols_fwd", [&] { run_f2(c, T1, Hh); });
  if (use_pair() && xcb::pair_smem(0, g.Ph, g)) {
    stage(c, "I1_cols_inv_corr", [&] {
      xcb::launch_cols_inv_corr_pair(g, Hh, c.Fhat, c.sstride, bands, T2, c.st, c.lc);
    });
  } else if (c.fcol && xcb::fast_smem(0, *c.fcol, g)) {
    stage(c, "I1_cols_inv_corr", [&] {
      xcb::launch_cols_inv_corr_fast(*c.fcol, g, Hh, c.Fhat, c.sstride, bands, T2, c.st, c.lc);
    });
  } else {
    stage(c, "I1_cols_inv_corr", [&] {
      xcb::launch_cols_inv_corr(*c.pcol, g, Hh, c.Fhat, c.sstride, bands, T2, c.st, c.lc);
    });
  }
  launch_i2(c, sig, T2, bands, half, base, out, out_kind, accumulate, dc);
}

// images per I1 launch for a gather call: the pair engine shares each staged
// filter spectrum column between two images (halving its HBM reads)
int gather_group(const Call& c) {
  return use_pair() && xcb::pair_smem(0, c.g.Ph, c.g) ? xcb::pair_i1_images() : 1;
}

// gather over two images: F1/F2 per image, one I1 launch for both, I2 per image
void run_gather2(Call& c, const xcb::SigSrc* sig, double* const* base, void* const* out,
                 int out_kind, bool accumulate, bool dc) {
  const xcb::Geo& g = c.g;
  bool half;
  const xcb::Bands bands = gather_bands(c, sig, 2, &half);
  c.nb_run = bands.n;
  c.band_mode = half ? 1 : 0;
  const size_t P = size_t(g.Ph) * g.Pw, tstride = size_t(bands.n) * g.H2 * g.Pw;
  float2* T1 = c.ctx->buf<float2>("T1", size_t(g.Hx2) * g.Pw);
  float2* Hh = c.ctx->buf<float2>("Hhat2", 2 * P);
  float2* T2 = c.ctx->buf<float2>("T2g", 2 * tstride);
  for (int i = 0; i < 2; ++i) {
    stage(c, "F1_rows_fwd", [&] { run_f1(c, sig[i], T1); });
    stage(c, "F2_cols_fwd", [&] { run_f2(c, T1, Hh + i * P); });
  }
  stage(c, "I1_cols_inv_corr", [&] {
    xcb::launch_cols_inv_corr_pair(g, Hh, c.Fhat, c.sstride, bands, T2, c.st, c.lc, 2, P,
                                   tstride);
  });
  for (int i = 0; i < 2; ++i)
    launch_i2(c, sig[i], T2 + i * tstride, bands, half, base[i], out[i], out_kind, accumulate,
              dc);
}

// Bands k >= 0 of the call (descending, as in c.bands) on the device, or an
// empty Bands when the Hermitian half-band mode does not apply: real signal,
// F_{-k} = conj(F_k) (hermitian()), and a symmetric band selection.
xcb::Bands half_bands(Call& c, bool real_sig) {
  if (!use_herm() || !real_sig || !c.f->hf.hermitian()) return xcb::Bands{nullptr, nullptr, 0};
  for (int k : c.ks)
    if (std::count(c.ks.begin(), c.ks.end(), -k) != 1) return xcb::Bands{nullptr, nullptr, 0};
  std::vector<int> hk, hs;
  for (size_t i = 0; i < c.ks.size(); ++i)
    if (c.ks[i] >= 0) {
      hk.push_back(c.ks[i]);
      hs.push_back(c.sidx[i]);
    }
  hk.insert(hk.end(), hs.begin(), hs.end());
  int* db = c.ctx->band_table(hk);
  const int n = int(hs.size());
  return xcb::Bands{db, db + n, n};
}

void run_scatter(Call& c, const xcb::SigSrc& sig, const double* base, void* out, int out_kind,
                 bool accumulate, bool dc) {
  const xcb::Geo& g = c.g;
  // Hermitian half-band mode (real signal, real filter): the -k terms are the
  // conjugates of the +k terms, so out = 2 Re(sum_{k>=0} w_k ...) with w_0 = 1/2;
  // it needs the pair-engine S2 and S4 (half weights, 2 Re)
  xcb::Bands bands = c.bands;
  bool half = use_pair() && xcb::pair_smem(4, g.Ph, g) && xcb::pair_smem(7, g.Pw, g);
  if (half) {
    const xcb::Bands hb = half_bands(c, !sig.is_complex);
    half = hb.n > 0;
    if (half) bands = hb;
  }
  // Conjugate band pairs (real signal, any filter, symmetric band selection):
  // H e^{+ik phi} = conj(H e^{-ik phi}), so S1 transforms the bands k >= 0 only
  // and S2 feeds each into two sums (k_pair.cu k_cols_fwd_mac_cpair_ilv)
  const int* gspec = nullptr;
  const float2* Ghat = nullptr;
  // S2 on the pair engine or the fast kernels; S1 and S4 on any engine
  const bool s2_pair = use_pair() && xcb::pair_smem(4, g.Ph, g);
  const bool s2_fast = !s2_pair && c.fcol && xcb::fast_smem(6, *c.fcol, g);
  // long columns (>= 3456): the staged G_k does not fit beside F^_k, so the fast
  // S2 runs twice over the same T1 planes (F^_k -> first plane; G_k, k > 0 ->
  // second plane); S1's halving is kept
  const bool s2_split = !s2_pair && !s2_fast && c.fcol && xcb::fast_smem(3, *c.fcol, g);
  bool cpair = !half && use_cpair() && !sig.is_complex && !c.packed &&
               (s2_pair || s2_fast || s2_split) && c.ks.size() > 1;
  xcb::Bands bands_g{nullptr, nullptr, 0};  // split S2: the bands k > 0 with G_k's planes
  if (cpair) {
    std::vector<int> hk, hs, hg;
    for (size_t i = 0; i < c.ks.size() && cpair; ++i) {
      const auto neg = std::find(c.ks.begin(), c.ks.end(), -c.ks[i]);
      cpair = neg != c.ks.end() && std::count(c.ks.begin(), c.ks.end(), c.ks[i]) == 1;
      if (cpair && c.ks[i] >= 0) {
        hk.push_back(c.ks[i]);
        hs.push_back(c.sidx[i]);
        hg.push_back(c.sidx[size_t(neg - c.ks.begin())]);
      }
    }
    if (cpair) {
      const int n = int(hk.size());
      hk.insert(hk.end(), hs.begin(), hs.end());
      hk.insert(hk.end(), hg.begin(), hg.end());
      int* db = c.ctx->band_table(hk);
      bands = xcb::Bands{db, db + n, n};
      gspec = db + 2 * n;
      Ghat = filter_spectra_conj(c);
      if (s2_split) {
        // T1 plane bi belongs to band hk[bi]; k = 0, if selected, must be the
        // last plane so that the bands k > 0 are a prefix of the planes
        int npos = 0;
        while (npos < n && hk[size_t(npos)] > 0) ++npos;
        for (int i = npos; i < n && cpair; ++i) cpair = hk[size_t(i)] == 0 && i == n - 1;
        bands_g = xcb::Bands{db, gspec, npos};
        if (!cpair) bands = c.bands;  // (setup sorts the bands in descending k: not reached)
      }
    }
  }
  c.nb_run = bands.n;
  c.band_mode = half ? 1 : cpair ? 2 : 0;
  const size_t t2plane = size_t(g.H2) * g.Pw;
  float2* T1 = c.ctx->buf<float2>("T1b", size_t(bands.n) * g.Hx2 * g.Pw);
  float2* Sg = c.ctx->buf<float2>("Sigma", size_t(g.Ph) * g.Pw);
  float2* T2 = c.ctx->buf<float2>("T2s", (cpair ? 2 : 1) * t2plane);
  if (use_pair() && xcb::pair_smem(3, g.Pw, g)) {
    stage(c, "S1_rows_fwd_premul", [&] {
      xcb::launch_rows_fwd_premul_pair(g, sig, base, bands, T1, c.st, c.lc);
    });
  } else if (c.frow && xcb::fast_smem(2, *c.frow, g)) {
    stage(c, "S1_rows_fwd_premul", [&] {
      xcb::launch_rows_fwd_premul_fast(*c.frow, g, sig, base, bands, T1, c.st, c.lc);
    });
  } else {
    stage(c, "S1_rows_fwd_premul", [&] {
      xcb::launch_rows_fwd_premul(*c.prow, g, sig, base, bands, T1, c.st, c.lc);
    });
  }
  if (cpair) {
    stage(c, "S2_cols_fwd_mac_inv", [&] {
      if (s2_pair) {
        xcb::launch_cols_fwd_mac_inv_cpair(g, T1, c.Fhat, Ghat, c.sstride, bands, gspec, T2,
                                           t2plane, c.st, c.lc);
      } else if (s2_fast) {
        xcb::launch_cols_fwd_mac_inv_cpair_fast(*c.fcol, g, T1, c.Fhat, Ghat, c.sstride, bands,
                                                gspec, T2, t2plane, c.st, c.lc);
      } else {
        xcb::launch_cols_fwd_mac_inv_fast(*c.fcol, g, T1, c.Fhat, c.sstride, bands, T2, c.st,
                                          c.lc);
        if (bands_g.n > 0)
          xcb::launch_cols_fwd_mac_inv_fast(*c.fcol, g, T1, Ghat, c.sstride, bands_g,
                                            T2 + t2plane, c.st, c.lc);
        else
          ck(cudaMemsetAsync(T2 + t2plane, 0, t2plane * sizeof(float2), c.st), "memset");
      }
    });
  } else if (use_pair() && xcb::pair_smem(4, g.Ph, g)) {
    stage(c, "S2_cols_fwd_mac_inv", [&] {
      xcb::launch_cols_fwd_mac_inv_pair(g, T1, c.Fhat, c.sstride, bands, half ? 1 : 0, T2, c.st,
                                        c.lc);
    });
  } else if (c.fcol && xcb::fast_smem(3, *c.fcol, g)) {
    stage(c, "S2_cols_fwd_mac_inv", [&] {
      xcb::launch_cols_fwd_mac_inv_fast(*c.fcol, g, T1, c.Fhat, c.sstride, bands, T2, c.st,
                                        c.lc);
    });
  } else {
    stage(c, "S2_cols_fwd_mac_inv", [&] {
      xcb::launch_cols_fwd_mac_inv(*c.pcol, g, T1, c.Fhat, c.sstride, bands, Sg, T2, c.st,
                                   c.lc);
    });
  }
  const cplx dcv = dc ? xcb::inner_dc_value(c.f->hf) : cplx(0);  // engine.hpp:370
  stage(c, "S4_rows_inv_out", [&] {
    if (use_pair() && xcb::pair_smem(7, g.Pw, g))
      xcb::launch_rows_inv_out_pair(g, T2, out_kind, out, accumulate ? 1 : 0, half ? 1 : 0, sig,
                                    dcv.real(), dcv.imag(), c.st, c.lc,
                                    cpair ? T2 + t2plane : nullptr);
    else
      xcb::launch_rows_inv_out(*c.prow, g, T2, out_kind, out, accumulate ? 1 : 0, sig, dcv.real(),
                               dcv.imag(), c.st, c.lc, cpair ? T2 + t2plane : nullptr);
  });
}

// XCB_DUAL=1 enables the interleaved I1 + I2 launches of gather batches.
// Measured on config 5 it is not faster (2 images: 155.1k against 156.1k
// Mpixel.bands/s; 16 images: 143.0k against 144.1k): with one CTA per SM an
// SM runs either an I1 or an I2 CTA, and both are limited per SM (barriers,
// issue), not by a resource the other kernel leaves idle.  Off by default.
bool use_dual() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_DUAL");
    return e && e[0] == '1';
  }();
  return on;
}

// Gather over a batch, software-pipelined: while image i's kernels are issued,
// one launch runs I1 of image i and I2 of image i-1 with interleaved CTAs
// (k_pair.cu k_dual_ilv), so the HBM-heavy column transforms and the
// FP32-bound row transforms share the SMs.  Two Hhat / T2 / base slots.
void run_gather_dual(Call& c, HostPipe& hp, const void* signal, const void* param, void* out,
                     size_t os, int out_kind, bool accumulate, bool dc) {
  const xcb::Geo& g = c.g;
  const int B = c.d.batch;
  const cplx dcv = dc ? std::conj(xcb::inner_dc_value(c.f->hf)) : cplx(0);  // engine.hpp:323
  bool half = false;
  xcb::Bands bands{};
  float2* T1 = c.ctx->buf<float2>("T1", size_t(g.Hx2) * g.Pw);
  float2* Hh[2] = {c.ctx->buf<float2>("Hhat_d0", size_t(g.Ph) * g.Pw),
                   c.ctx->buf<float2>("Hhat_d1", size_t(g.Ph) * g.Pw)};
  float2* T2[2] = {nullptr, nullptr};
  double* base[2] = {nullptr, nullptr};
  xcb::SigSrc sg[2]{};
  for (int img = 0; img <= B; ++img) {
    const int s = img & 1, p = s ^ 1;
    if (img < B) {
      hp.h2d(signal, param, img + 1);
      Staged st = hp.inputs(signal, param, img);
      prep(c, st, false, &base[s], nullptr, s, img);
      if (img == 0) {
        bands = gather_bands(c, &st.sig, 1, &half);
        c.nb_run = bands.n;
        c.band_mode = half ? 1 : 0;
        for (int i = 0; i < 2; ++i)
          T2[i] = c.ctx->buf<float2>("T2_d" + std::to_string(i), size_t(bands.n) * g.H2 * g.Pw);
      }
      sg[s] = st.sig;
      stage(c, "F1_rows_fwd", [&] { run_f1(c, sg[s], T1); });
      stage(c, "F2_cols_fwd", [&] { run_f2(c, T1, Hh[s]); });
    }
    if (img == 0) {
      stage(c, "I1_cols_inv_corr", [&] {
        xcb::launch_cols_inv_corr_pair(g, Hh[0], c.Fhat, c.sstride, bands, T2[0], c.st, c.lc);
      });
      continue;
    }
    void* dout = hp.out_buffer(out, img - 1, os);
    if (img < B) {
      stage(c, "I1_I2_dual", [&] {
        xcb::launch_dual_pair(g, Hh[s], c.Fhat, c.sstride, bands, T2[s], T2[p], half ? 1 : 0,
                              base[p], out_kind, dout, accumulate ? 1 : 0, sg[p], dcv.real(),
                              dcv.imag(), c.st, c.lc);
      });
    } else {
      launch_i2(c, sg[p], T2[p], bands, half, base[p], dout, out_kind, accumulate, dc);
    }
    ck(cudaGetLastError(), "kernel launch");
    hp.done(out, img - 1, dout, os);
  }
}

void fill_stats(Call& c, xc_stats* st, double gpu_s, double total_s, long long ops) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  st->standard_ops = ops;
  st->pad_h = c.g.Ph;
  st->pad_w = c.g.Pw;
  st->seconds_fft = gpu_s;
  st->seconds_h2d = c.h2d_s;
  st->seconds_d2h = c.d2h_s;
  st->seconds_total = total_s;
  st->gpu_launches = c.lc.n;
  st->bands_run = c.nb_run;
  st->band_mode = c.band_mode;
}

void run_single(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d,
                const void* signal, const void* param, const int* components, int n_components,
                unsigned flags, void* out, xc_stats* stats, bool out_dev);
void run_group(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d,
               const void* signal, const void* param, const int* components, int n_components,
               unsigned flags, void* out, xc_stats* stats);
void smooth_group(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                  const void* param, int normalize_signal, void* out, xc_stats* stats);
int tile_count(int n, int R);

}  // namespace

// ======================================================================= C ABI
extern "C" {

int xc_abi_version(void) { return XC_ABI_VERSION; }

int xc_context_create(int device, xc_context* out) {
  return guarded(nullptr, [&] {
    if (!out) throw std::invalid_argument("null argument");
    int n = 0;
    ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) throw CudaError("no such CUDA device", XC_ECUDA);
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new xc_context_s();
    c->device = device;
    ck(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&c->cp_in, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&c->cp_out, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own;
    *out = c;
  });
}

void xc_context_destroy(xc_context ctx) { delete ctx; }

const char* xc_last_error(xc_context ctx) {
  return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

int xc_context_set_stream(xc_context ctx, void* s) {
  return guarded(ctx, [&] { ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own; });
}

int xc_context_trim(xc_context ctx) {
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaSetDevice(ctx->device);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    for (auto& kv : ctx->bufs) cudaFree(kv.second.p);
    ctx->bufs.clear();
    ctx->det_filters.clear();  // their cached spectra
  });
}

// fft2 (fft.hpp:20-53): the 2D DFT of a rows x cols complex grid on the
// device with the pipeline's own transforms (F1 row FFT -> layout B', F2
// column FFT -> layout B), forward unscaled, inverse scaled 1/n as Eigen's
// FFT.  The engine pairs the staged rows' columns, so an odd width runs as
// the transposed problem; both extents odd is rejected.
int xc_fft2(xc_context ctx, int rows, int cols, int dtype, int memory, int inverse,
            const void* in, void* out) {
  return guarded(ctx, [&] {
    if (!ctx || !in || !out) throw std::invalid_argument("null argument");
    if (rows < 1 || cols < 1) throw std::invalid_argument("image dims must be positive");
    if (dtype != XC_C64 && dtype != XC_C128)
      throw std::invalid_argument("xc_fft2 takes complex data (XC_C64 / XC_C128)");
    const bool tr = cols % 2 != 0;
    if (tr && rows % 2 != 0) throw std::invalid_argument("xc_fft2 needs one even extent");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    Call c{};
    c.ctx = ctx;
    c.st = ctx->stream;
    const int R0 = tr ? cols : rows, C0 = tr ? rows : cols;  // staged grid
    xcb::Geo& g = c.g;
    g.H = g.Hx = R0;
    g.W = g.Wx = C0;
    g.Hx2 = g.H2 = (R0 + 1) & ~1;
    g.off = g.R = g.periodic = 0;
    g.Ph = R0;
    g.Pw = C0;
    c.prow = &ctx->plan(g.Pw);
    c.pcol = &ctx->plan(g.Ph);
    const size_t n = size_t(rows) * cols, es = dtype == XC_C128 ? 16 : 8;
    const void* src = in;
    if (memory == XC_HOST) {
      void* b = ctx->buf<char>("fft2_in", n * es);
      ck(cudaMemcpyAsync(b, in, n * es, cudaMemcpyHostToDevice, c.st), "H2D");
      src = b;
    }
    float2* x = ctx->buf<float2>("fft2_x", n);
    xcb::launch_fft2_in(src, dtype == XC_C128, rows, cols, tr, inverse != 0, x, c.st, c.lc);
    float2* T1 = ctx->buf<float2>("fft2_T1", size_t(g.Hx2) * g.Pw);
    float2* Hh = ctx->buf<float2>("fft2_H", size_t(g.Ph) * g.Pw);
    run_f1(c, xcb::SigSrc{x, 1, nullptr, xcb::SIG_PLAIN}, T1);
    run_f2(c, T1, Hh);
    void* dst = memory == XC_HOST ? ctx->buf<char>("fft2_out", n * es) : out;
    xcb::launch_fft2_out(Hh, rows, cols, tr, inverse != 0, dtype == XC_C128, dst, c.st, c.lc);
    ck(cudaGetLastError(), "fft2 launch");
    if (memory == XC_HOST)
      ck(cudaMemcpyAsync(out, dst, n * es, cudaMemcpyDeviceToHost, c.st), "D2H");
    ck(cudaStreamSynchronize(c.st), "fft2");
  });
}

int xc_debug_check_guards(xc_context ctx, int* n_bad, char* first_bad, int len) {
  return guarded(ctx, [&] {
    if (!ctx || !n_bad) throw std::invalid_argument("null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    ck(cudaDeviceSynchronize(), "sync");
    int bad = 0;
    std::string first;
    std::vector<unsigned char> h;
    for (auto& kv : ctx->bufs) {
      const DevBuf& b = kv.second;
      if (!b.guard) continue;
      h.resize(b.guard);
      for (int side = 0; side < 2; ++side) {
        const char* z = static_cast<const char*>(b.p) + (side ? b.guard + b.n : 0);
        ck(cudaMemcpy(h.data(), z, b.guard, cudaMemcpyDeviceToHost), "D2H guard");
        if (std::any_of(h.begin(), h.end(), [](unsigned char c) { return c != 0xff; })) {
          if (first.empty()) first = kv.first + (side ? " (after)" : " (before)");
          ++bad;
        }
      }
    }
    *n_bad = bad;
    if (first_bad && len > 0) {
      std::strncpy(first_bad, first.c_str(), size_t(len) - 1);
      first_bad[len - 1] = 0;
    }
  });
}

int xc_debug_guard_bytes(void) { return int(guard_bytes()); }

int xc_debug_pick_pad(int n) { return pick_pad2d(std::max(n, 1)); }

int xc_debug_tile_count(int extent, int R) { return tile_count(extent, R); }

int xc_profile_enable(xc_context ctx, int on) {
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->profiling = on != 0;
  });
}

int xc_profile_reset(xc_context ctx) {
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->prof.clear();
  });
}

int xc_profile_get(xc_context ctx, int idx, char* name, int name_len, double* total_ms,
                   long long* launches) {
  if (!ctx) return -1;
  std::lock_guard<std::mutex> lk(ctx->mu);
  const int n = int(ctx->prof.size());
  if (idx < 0 || idx >= n) return n;
  const auto& p = ctx->prof[idx];
  if (name && name_len > 0) {
    std::strncpy(name, p.first.c_str(), size_t(name_len) - 1);
    name[name_len - 1] = 0;
  }
  if (total_ms) *total_ms = p.second.ms;
  if (launches) *launches = p.second.launches;
  return n;
}

int xc_filter_create(xc_context ctx, int group, int K, const int* ks, int nc,
                     const double* comps, int n_radii, int n_angles, double r_max,
                     double r_min, double r_domain, xc_filter* out) {
  return guarded(ctx, [&] {
    if (!out || (nc > 0 && (!ks || !comps))) throw std::invalid_argument("null argument");
    if (group == XC_ROTATION3) throw std::invalid_argument("2D pipeline needs a 2D field");
    if (group != XC_ROTATION2 && group != XC_SCALE2) throw std::invalid_argument("unknown group");
    if (!(r_max > 0)) throw std::invalid_argument("r_max must be > 0");
    if (group == XC_SCALE2 && !(r_min > 0))
      throw std::invalid_argument("r_min must be > 0 (log-polar excludes the origin)");
    auto f = std::make_unique<xc_filter_s>();
    xcb::HostFilter& h = f->hf;
    h.group = group;
    h.K = K;
    h.ks.assign(ks, ks + nc);
    h.n_radii = n_radii;
    h.n_angles = n_angles;
    h.r_max = r_max;
    h.r_min = r_min;
    h.r_domain = r_domain;
    const int rows = h.n_rows();
    if (rows < 1) throw std::invalid_argument("n_radii must be >= 1");
    h.comps.resize(size_t(rows) * nc);
    for (int ci = 0; ci < nc; ++ci)
      for (int r = 0; r < rows; ++r)
        h.comps[size_t(r) * nc + ci] =
            cplx(comps[2 * (size_t(ci) * rows + r)], comps[2 * (size_t(ci) * rows + r) + 1]);
    *out = f.release();
  });
}

void xc_filter_destroy(xc_filter f) { delete f; }

int xc_filter_num_components(xc_filter f) { return f ? f->hf.nc() : 0; }

int xc_decompose_rotation2(const double* filt, int height, int width, int layout, double cx,
                           double cy, int K, int n_radii, int n_angles, double r_max,
                           int* ks_out, double* comps_out, int* nc_out) {
  return guarded(nullptr, [&] {
    auto img = to_rowmajor(filt, height, width, layout);
    auto f = xcb::decompose_rotation2(xcb::ImageView{img.data(), width, height}, cx, cy, K,
                                      n_radii, n_angles, r_max);
    export_filter(f, ks_out, comps_out, nc_out);
  });
}

int xc_decompose_scale2(const double* filt, int height, int width, int layout, double cx,
                        double cy, int K, int n_radii, int n_angles, double r_min,
                        double r_max, double r_domain, int* ks_out, double* comps_out,
                        int* nc_out) {
  return guarded(nullptr, [&] {
    auto img = to_rowmajor(filt, height, width, layout);
    auto f = xcb::decompose_scale2(xcb::ImageView{img.data(), width, height}, cx, cy, K,
                                   n_radii, n_angles, r_min, r_max, r_domain);
    export_filter(f, ks_out, comps_out, nc_out);
  });
}

}  // extern "C"

namespace {
// decompose_* on the context's device: the shell carries the
// validated metadata (host_filter.cpp rotation2_shell / scale2_shell); the
// polar resampling and the band DFT run as two kernels (k_misc.cu
// launch_decompose) and the small coefficient table comes back to the host.
// The caller holds ctx->mu.
void decompose_on_device(xc_context ctx, xcb::HostFilter& f, const std::vector<cplx>& img,
                         int width, int height, double cx, double cy) {
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int nr = f.n_radii, na = f.n_angles, nc = f.nc(), rows = f.n_rows();
  double2* dimg = ctx->buf<double2>("dec_img", std::max<size_t>(1, img.size()));
  double2* samples = ctx->buf<double2>("dec_samples", size_t(nr) * na);
  double2* comps = ctx->buf<double2>("dec_comps", size_t(rows) * nc);
  int* dks = ctx->buf<int>("dec_ks", size_t(nc));
  cudaStream_t st = ctx->stream;
  if (!img.empty())
    ck(cudaMemcpyAsync(dimg, img.data(), img.size() * sizeof(cplx), cudaMemcpyHostToDevice, st),
       "H2D filter");
  ck(cudaMemcpyAsync(dks, f.ks.data(), size_t(nc) * sizeof(int), cudaMemcpyHostToDevice, st),
     "H2D ks");
  xcb::LaunchCounter lc;
  xcb::launch_decompose(dimg, width, height, cx, cy, nr, na, f.group,
                        f.group == 1 ? f.r_min : 0.0, f.group == 1 ? f.domain_top() : f.r_max,
                        dks, nc, samples, comps, st, lc);
  ck(cudaGetLastError(), "decompose launch");
  f.comps.assign(size_t(rows) * nc, cplx(0));
  ck(cudaMemcpyAsync(f.comps.data(), comps, f.comps.size() * sizeof(cplx),
                     cudaMemcpyDeviceToHost, st),
     "D2H comps");
  ck(cudaStreamSynchronize(st), "decompose");
}
}  // namespace

extern "C" {

int xc_decompose_rotation2_device(xc_context ctx, const double* filt, int height, int width,
                                  int layout, double cx, double cy, int K, int n_radii,
                                  int n_angles, double r_max, int* ks_out, double* comps_out,
                                  int* nc_out) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    auto f = xcb::rotation2_shell(K, n_radii, n_angles, r_max);
    decompose_on_device(ctx, f, to_rowmajor(filt, height, width, layout), width, height, cx, cy);
    export_filter(f, ks_out, comps_out, nc_out);
  });
}

int xc_decompose_scale2_device(xc_context ctx, const double* filt, int height, int width,
                               int layout, double cx, double cy, int K, int n_radii,
                               int n_angles, double r_min, double r_max, double r_domain,
                               int* ks_out, double* comps_out, int* nc_out) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    auto f = xcb::scale2_shell(K, n_radii, n_angles, r_min, r_max, r_domain);
    decompose_on_device(ctx, f, to_rowmajor(filt, height, width, layout), width, height, cx, cy);
    export_filter(f, ks_out, comps_out, nc_out);
  });
}

int xc_render_component(xc_filter f, int ci, int width, int height, double cx, double cy,
                        int layout, double* out) {
  return guarded(nullptr, [&] {
    if (ci < 0 || ci >= f->hf.nc()) throw std::invalid_argument("component index out of range");
    xcb::render_component(f->hf, ci, width, height, cx, cy, layout == XC_COL_MAJOR,
                          reinterpret_cast<cplx*>(out));
  });
}

int xc_reconstruct(xc_filter f, int width, int height, double cx, double cy,
                   const int* subset, int nsub, int layout, double* out) {
  return guarded(nullptr, [&] {
    xcb::reconstruct(f->hf, width, height, cx, cy, subset, subset ? nsub : -1,
                     layout == XC_COL_MAJOR, reinterpret_cast<cplx*>(out));
  });
}

int xc_inner_dc_value(xc_filter f, double* out2) {
  return guarded(nullptr, [&] {
    const cplx v = xcb::inner_dc_value(f->hf);
    out2[0] = v.real();
    out2[1] = v.imag();
  });
}

}  // extern "C"

namespace {

// xcorr_fast / xconv_fast on one device (the caller holds ctx->mu).  out_dev:
// `out` is a device buffer even when d->memory == XC_HOST (multi-device partials).
// ---------------------------------------------------------------- tiles
// Images beyond the longest planned transform (4320) used to fall on the
// generic kernels, ~8x slower per point (pick_pad2d).  Both pipelines are
// local: out(p) reads the signal and the transformation field within
// R = ceil(r_max) of p only (engine.hpp:300-319, 345-368; zero padding outside
// the image), so the image is cut into balanced tiles whose inputs carry an
// R-pixel halo, each tile runs the planned pipelines, and the tile interiors
// are copied into the output.  The result is the same sum per pixel (the halo
// supplies exactly the samples the full transform would have used; rounding
// differs as between any two pads).  Rotation group only (the scale group's
// guard message names image pixels), not for periodic or accumulating calls.
// XCB_TILE=0 turns it off.
constexpr int kTileMaxLen = 4320;

// tiles along an axis of n points: one while n + R fits the longest plan, else
// balanced tiles of at most kTileMaxLen - 3R interior points (halo R each side
// and R more for the pad)
int tile_count(int n, int R) {
  if (n + R <= kTileMaxLen || 6 * R > kTileMaxLen) return 1;
  const int cap = kTileMaxLen - 3 * R;
  return (n + cap - 1) / cap;
}

bool needs_tiles(xc_filter f, const xc_image_desc* d, unsigned flags) {
  static const bool on = [] {
    const char* e = std::getenv("XCB_TILE");
    return !(e && e[0] == '0');
  }();
  if (!on || !use_pair() || !f || !d) return false;
  if (flags & (XC_FLAG_PERIODIC | XC_FLAG_ACCUMULATE)) return false;
  if (f->hf.group != XC_ROTATION2 || d->xform_kind != XC_ROTATION2) return false;
  const int R = f->hf.render_radius();
  if (6 * R > kTileMaxLen) return false;
  return std::max(d->height, d->width) + R > kTileMaxLen;
}

void run_tiled(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d, const void* signal,
               const void* param, const int* components, int n_components, unsigned flags,
               void* out, xc_stats* stats) {
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  const auto t_start = std::chrono::steady_clock::now();
  if (!signal || !param || !out) throw std::invalid_argument("null argument");
  if (d->height < 1 || d->width < 1 || d->batch < 1)
    throw std::invalid_argument("image dims must be positive");
  const int R = f->hf.render_radius();
  const bool cm = d->layout == XC_COL_MAJOR;
  // the grid as it lies in memory: MR rows of MC elements
  const int MR = cm ? d->width : d->height, MC = cm ? d->height : d->width;
  auto split = [&](int n, int* nt, int* t) {
    *nt = tile_count(n, R);
    *t = (n + *nt - 1) / *nt;
  };
  int ntr, tr, ntc, tc;
  split(MR, &ntr, &tr);
  split(MC, &ntc, &tc);
  const size_t ss = dtype_size(d->signal_dtype), ps = dtype_size(d->param_dtype),
               os = dtype_size(d->out_dtype);
  const size_t npix = size_t(MR) * MC;
  const size_t tmax = size_t(std::min(MR, tr + 2 * R)) * size_t(std::min(MC, tc + 2 * R));
  char* tsig = ctx->buf<char>("tile_sig", tmax * ss);
  char* tpar = ctx->buf<char>("tile_par", tmax * ps);
  char* tout = ctx->buf<char>("tile_out", tmax * os);
  cudaStream_t st = ctx->stream;
  xc_stats agg{};
  for (int img = 0; img < d->batch; ++img) {
    const char* sg = static_cast<const char*>(signal) + size_t(img) * npix * ss;
    const char* pr = static_cast<const char*>(param) +
                     (d->param_per_image ? size_t(img) * npix * ps : 0);
    char* po = static_cast<char*>(out) + size_t(img) * npix * os;
    for (int i = 0; i < ntr; ++i)
      for (int j = 0; j < ntc; ++j) {
        const int r0 = i * tr, r1 = std::min(MR, r0 + tr);
        const int c0 = j * tc, c1 = std::min(MC, c0 + tc);
        if (r0 >= r1 || c0 >= c1) continue;
        const int a0 = std::max(0, r0 - R), a1 = std::min(MR, r1 + R);  // with the halo
        const int b0 = std::max(0, c0 - R), b1 = std::min(MC, c1 + R);
        const int h = a1 - a0, w = b1 - b0;
        const size_t off = size_t(a0) * MC + b0;
        ck(cudaMemcpy2DAsync(tsig, size_t(w) * ss, sg + off * ss, size_t(MC) * ss, size_t(w) * ss,
                             size_t(h), cudaMemcpyDefault, st),
           "tile signal");
        ck(cudaMemcpy2DAsync(tpar, size_t(w) * ps, pr + off * ps, size_t(MC) * ps, size_t(w) * ps,
                             size_t(h), cudaMemcpyDefault, st),
           "tile param");
        xc_image_desc dt = *d;
        dt.batch = 1;
        dt.memory = XC_DEVICE;
        dt.param_per_image = 1;
        dt.height = cm ? w : h;
        dt.width = cm ? h : w;
        xc_stats s1{};
        run_single(ctx, f, mode, &dt, tsig, tpar, components, n_components,
                   flags & ~unsigned(XC_FLAG_ASYNC), tout, &s1, false);
        const size_t in_off = size_t(r0 - a0) * w + size_t(c0 - b0);
        ck(cudaMemcpy2DAsync(po + (size_t(r0) * MC + c0) * os, size_t(MC) * os,
                             tout + in_off * os, size_t(w) * os, size_t(c1 - c0) * os,
                             size_t(r1 - r0), cudaMemcpyDefault, st),
           "tile output");
        agg.standard_ops = s1.standard_ops;
        agg.pad_h = std::max(agg.pad_h, s1.pad_h);
        agg.pad_w = std::max(agg.pad_w, s1.pad_w);
        agg.seconds_fft += s1.seconds_fft;
        agg.gpu_launches += s1.gpu_launches;
        agg.bands_run = s1.bands_run;
        agg.band_mode = s1.band_mode;
      }
  }
  ck(cudaStreamSynchronize(st), "tiles");
  if (stats) {
    *stats = agg;
    stats->seconds_total =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
}

void run_single(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d,
                const void* signal, const void* param, const int* components, int n_components,
                unsigned flags, void* out, xc_stats* stats, bool out_dev) {
    if (needs_tiles(f, d, flags)) {
      if (mode != XC_CORRELATION && mode != XC_CONVOLUTION)
        throw std::invalid_argument("unknown mode");
      if (d->out_dtype != XC_C64 && d->out_dtype != XC_C128)
        throw std::invalid_argument("xc_run output must be complex (XC_C64 / XC_C128)");
      run_tiled(ctx, f, mode, d, signal, param, components, n_components, flags, out, stats);
      return;
    }
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const auto t_start = std::chrono::steady_clock::now();
    if (mode != XC_CORRELATION && mode != XC_CONVOLUTION) throw std::invalid_argument("unknown mode");
    if (!signal || !param || !out) throw std::invalid_argument("null argument");
    if (d && d->out_dtype != XC_C64 && d->out_dtype != XC_C128)
      throw std::invalid_argument("xc_run output must be complex (XC_C64 / XC_C128)");
    Call c = setup(ctx, f, d, -1, components, n_components, (flags & XC_FLAG_PERIODIC) != 0);
    c.out_dev = out_dev;
    guard_begin(c);
    const bool accumulate = (flags & XC_FLAG_ACCUMULATE) != 0;
    if (accumulate && d->memory != XC_DEVICE && !out_dev)
      throw std::invalid_argument("XC_FLAG_ACCUMULATE needs device memory");
    const bool dc = c.f->hf.group == XC_SCALE2 && !(flags & XC_FLAG_NO_INNER_DC);
    const size_t npix = size_t(c.rows) * c.cols, os = dtype_size(d->out_dtype);
    const int out_kind = d->out_dtype == XC_C64 ? xcb::OUT_C64 : xcb::OUT_C128;
    ctx->release_events();
    cudaEvent_t e0 = ctx->event(true), e1 = ctx->event(true);
    double gpu_s = 0;
    HostPipe hp(c);
    const int G = mode == XC_CORRELATION ? gather_group(c) : 1;
    for (int i = 0; i < G; ++i) hp.h2d(signal, param, i);
    ck(cudaEventRecord(e0, c.st), "event");
    const bool dual = mode == XC_CORRELATION && G == 1 && d->batch >= 2 && use_pair() &&
                      use_dual() && xcb::dual_pair_ok(c.g);
    if (dual) run_gather_dual(c, hp, signal, param, out, os, out_kind, accumulate, dc);
    for (int img = dual ? d->batch : 0; img < d->batch;) {
      const int n = std::min(G, d->batch - img);
      for (int i = 0; i < n; ++i) hp.h2d(signal, param, img + G + i);  // next group
      if (n == 2) {
        Staged s[2];
        double* base[2];
        void* dout[2];
        xcb::SigSrc sg[2];
        for (int i = 0; i < 2; ++i) {
          s[i] = hp.inputs(signal, param, img + i);
          prep(c, s[i], false, &base[i], nullptr, i, img + i);
          dout[i] = hp.out_buffer(out, img + i, os);
          sg[i] = s[i].sig;
        }
        run_gather2(c, sg, base, dout, out_kind, accumulate, dc);
        ck(cudaGetLastError(), "kernel launch");
        for (int i = 0; i < 2; ++i) hp.done(out, img + i, dout[i], os);
      } else {
        Staged s = hp.inputs(signal, param, img);
        double* base = nullptr;
        prep(c, s, false, &base, nullptr, 0, img);
        void* dout = hp.out_buffer(out, img, os);
        if (mode == XC_CORRELATION)
          run_gather(c, s.sig, base, dout, out_kind, accumulate, dc);
        else
          run_scatter(c, s.sig, base, dout, out_kind, accumulate, dc);
        ck(cudaGetLastError(), "kernel launch");
        hp.done(out, img, dout, os);
      }
      img += n;
    }
    ck(cudaEventRecord(e1, c.st), "event");
    // XC_FLAG_ASYNC with device memory and nothing to read back (no scale
    // guard): return with the work queued on the stream (capturable in a
    // CUDA graph); the caller synchronizes
    const bool async = (flags & XC_FLAG_ASYNC) && d->memory == XC_DEVICE && !out_dev &&
                       c.f->hf.group != XC_SCALE2 && !ctx->profiling;
    if (!async) {
      hp.finish();
      guard_check(c, param);
      gpu_s = event_seconds(e0, e1);
    }
    ctx->resolve_profile();
    fill_stats(c, stats, gpu_s,
               std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(),
               (long long)c.ks.size());
}

}  // namespace

extern "C" {

int xc_run(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d, const void* signal,
           const void* param, const int* components, int n_components, unsigned flags,
           void* out, xc_stats* stats) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->group)
      run_group(ctx, f, mode, d, signal, param, components, n_components, flags, out, stats);
    else
      run_single(ctx, f, mode, d, signal, param, components, n_components, flags, out, stats,
                 false);
  });
}

}  // extern "C"

namespace {

// engine.hpp:388-392: zero-integral filters cannot be normalized (cached per filter)
void check_integral(xc_filter f) {
  if (!f) throw std::invalid_argument("null argument");
  std::lock_guard<std::mutex> flk(f->mu);
  if (f->integral_state < 0) {
    const xcb::HostFilter& hf = f->hf;
    const int R = hf.render_radius(), S = 2 * R + 1;
    std::vector<cplx> full(size_t(S) * S);
    xcb::reconstruct(hf, S, S, R, R, nullptr, -1, false, full.data());
    cplx integral(0);
    double mx = 0;
    for (auto& v : full) {
      integral += v;
      mx = std::max(mx, std::abs(v));
    }
    f->integral_state = std::abs(integral) < 1e-12 * std::max(1.0, mx) ? 0 : 1;
  }
  if (f->integral_state == 0)
    throw std::invalid_argument("normalization undefined: filter has zero integral");
}

struct SmoothPart {
  double gpu_s = 0, h2d_s = 0;
  int launches = 0, pad_h = 0, pad_w = 0, bands_run = 0;
  long long bands = 0;
  bool packed = false;  // num + i alpha den in numden[img][0] (SIG_PACK)
};

// num and den of smooth_adaptive from ONE scatter (SIG_PACK): with a real
// signal, real weights and a filter whose selected bands satisfy
// F_{-k} = conj(F_k) (and a real inner DC), num and den are real, so the
// complex signal h w + i alpha w scatters to num + i alpha den.  It replaces
// the reference's two xconv_fast calls (engine.hpp:402-403) by one over the
// full band set: num and den share every staged F^_k column, T1 pass and the
// single inverse transform, and the divide reads one array.  XCB_PACK=0 runs
// the two scatters (each in the Hermitian half-band mode).
bool smooth_packable(const Call& c, const xcb::SigSrc& sig, bool dc) {
  static const bool on = [] {
    const char* e = std::getenv("XCB_PACK");
    return !(e && e[0] == '0');
  }();
  if (!on || sig.is_complex || !c.f->hf.hermitian()) return false;
  for (int k : c.ks)
    if (std::count(c.ks.begin(), c.ks.end(), -k) != 1) return false;
  if (dc) {
    const cplx v = xcb::inner_dc_value(c.f->hf);
    if (std::abs(v.imag()) > 1e-12 * std::max(1.0, std::abs(v))) return false;
  }
  return true;
}

// The two extended convolutions of smooth_adaptive (engine.hpp:394-403),
// num = xconv(H~) and den = xconv(1~), for every image of the batch over the
// selected bands, into numden[img][0 | 1][npix] (device memory of ctx).
// Inputs stream through the HostPipe slots (H2D of image i+1 overlaps image
// i); the scale guard is read back once for the whole batch.  on_image(img)
// is called after image img's kernels are queued (the single-device path
// queues its divide and D2H there).
template <class OnImage>
SmoothPart smooth_partials(xc_context ctx, xc_filter f, const xc_image_desc* d,
                           const void* signal, const void* param, int normalize_signal,
                           const int* comps, int ncomp, bool dc, float2* numden,
                           OnImage&& on_image, unsigned* amax = nullptr) {
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  Call c = setup(ctx, f, d, -1, comps, ncomp, false);
  c.out_dev = true;
  const bool scale = c.f->hf.group == XC_SCALE2;
  const bool weighted = normalize_signal && scale;  // engine.hpp:396-401
  const size_t npix = size_t(c.rows) * c.cols;
  guard_begin(c);
  ctx->release_events();
  cudaEvent_t e0 = ctx->event(true), e1 = ctx->event(true);
  HostPipe hp(c);
  hp.h2d(signal, param, 0);
  ck(cudaEventRecord(e0, c.st), "event");
  bool packed = false;
  for (int img = 0; img < d->batch; ++img) {
    hp.h2d(signal, param, img + 1);
    Staged s = hp.inputs(signal, param, img);
    double* base = nullptr;
    float* wgt = nullptr;
    prep(c, s, weighted, &base, weighted ? &wgt : nullptr, 0, img);
    packed = c.packed = amax && smooth_packable(c, s.sig, dc);
    if (packed) {
      xcb::SigSrc sp = s.sig;
      sp.mode = xcb::SIG_PACK;
      sp.wgt = wgt;  // null: w = 1
      sp.amax = amax + img;
      sp.is_complex = 1;  // a complex signal: the full band set
      stage(c, "absmax", [&] {
        xcb::launch_absmax(static_cast<const float*>(s.sig.sig), npix, amax + img, c.st, c.lc);
      });
      run_scatter(c, sp, base, numden + 2 * size_t(img) * npix, xcb::OUT_C64, false, dc);
      ck(cudaGetLastError(), "kernel launch");
      hp.done(nullptr, img, nullptr, 0);
      on_image(c, img);
      continue;
    }
    xcb::SigSrc sn = s.sig, sd = s.sig;
    sn.wgt = wgt;
    sn.mode = weighted ? xcb::SIG_TIMES_W : xcb::SIG_PLAIN;
    sd.wgt = wgt;
    sd.mode = xcb::SIG_W_ONLY;  // the all-ones signal (times 1/s^2 when weighted)
    float2* num = numden + 2 * size_t(img) * npix;
    run_scatter(c, sn, base, num, xcb::OUT_C64, false, dc);
    run_scatter(c, sd, base, num + npix, xcb::OUT_C64, false, dc);
    ck(cudaGetLastError(), "kernel launch");
    hp.done(nullptr, img, nullptr, 0);
    on_image(c, img);
  }
  ck(cudaEventRecord(e1, c.st), "event");
  hp.finish();
  guard_check(c, param);
  SmoothPart r;
  r.packed = packed;
  r.bands_run = c.nb_run;  // bands each scatter transformed (packed: one full-band scatter)
  r.gpu_s = event_seconds(e0, e1);
  r.launches = c.lc.n;
  r.pad_h = c.g.Ph;
  r.pad_w = c.g.Pw;
  r.bands = (long long)c.ks.size();
  return r;
}

// engine.hpp:405-418 for image img: floor 1e-9 max|den|, out = Re(num / den);
// red[img] holds image img's max bits, red[batch] the clamped total.
void smooth_divide(xc_context ctx, cudaStream_t st, const float2* numden, size_t npix, int img,
                   int batch, int out_f64, void* dout, unsigned* red, xcb::LaunchCounter& lc) {
  const float2* num = numden + 2 * size_t(img) * npix;
  xcb::launch_smooth_finish(num, num + npix, npix, out_f64, dout, red + img, red + batch, st, lc);
  ck(cudaGetLastError(), "kernel launch");
}

void smooth_single(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                   const void* param, int normalize_signal, void* out, xc_stats* stats) {
  const auto t_start = std::chrono::steady_clock::now();
  const bool host_out = d->memory == XC_HOST;
  const size_t npix = size_t(d->height) * d->width, os = dtype_size(d->out_dtype);
  float2* numden = ctx->buf<float2>("smooth_numden", 2 * npix * size_t(d->batch));
  // red[0..batch]: per-image max|den| bits and the clamped count; then the
  // per-image max|h| bits of the packed path
  unsigned* red = ctx->buf<unsigned>("smooth_red", 2 * size_t(d->batch) + 1);
  unsigned* amax = red + d->batch + 1;
  char* stage_out = host_out ? ctx->buf<char>("smooth_out", npix * os * size_t(d->batch)) : nullptr;
  ck(cudaMemsetAsync(red, 0, (2 * size_t(d->batch) + 1) * sizeof(unsigned), ctx->stream),
     "memset");
  std::vector<cudaEvent_t> done;
  xcb::LaunchCounter flc;
  Call* cp = nullptr;
  SmoothPart part = smooth_partials(
      ctx, f, d, signal, param, normalize_signal, nullptr, 0, f->hf.group == XC_SCALE2, numden,
      [&](Call& c, int img) {
        cp = &c;
        char* dout = host_out ? stage_out + size_t(img) * npix * os
                              : static_cast<char*>(out) + size_t(img) * npix * os;
        stage(c, "smooth_finish", [&] {
          if (c.packed) {
            xcb::launch_smooth_finish_packed(numden + 2 * size_t(img) * npix, npix, amax + img,
                                             d->out_dtype == XC_F64, dout, red + img,
                                             red + d->batch, c.st, flc);
            ck(cudaGetLastError(), "kernel launch");
          } else {
            smooth_divide(ctx, c.st, numden, npix, img, d->batch, d->out_dtype == XC_F64, dout,
                          red, flc);
          }
        });
        if (host_out) {  // D2H of image img overlaps the next image's kernels
          cudaEvent_t e = ctx->event(false);
          ck(cudaEventRecord(e, c.st), "event");
          ck(cudaStreamWaitEvent(ctx->cp_out, e, 0), "wait");
          ck(cudaMemcpyAsync(static_cast<char*>(out) + size_t(img) * npix * os, dout, npix * os,
                             cudaMemcpyDeviceToHost, ctx->cp_out),
             "D2H");
        }
      },
      amax);
  (void)cp;
  unsigned clamped = 0;
  ck(cudaMemcpyAsync(&clamped, red + d->batch, sizeof(unsigned), cudaMemcpyDeviceToHost,
                     ctx->stream),
     "readback");
  ck(cudaStreamSynchronize(ctx->stream), "smooth");
  if (host_out) ck(cudaStreamSynchronize(ctx->cp_out), "D2H");
  ctx->resolve_profile();
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->standard_ops = 2 * part.bands;  // engine.hpp:406 num + den
    stats->clamped_pixels = int(clamped);
    stats->pad_h = part.pad_h;
    stats->pad_w = part.pad_w;
    stats->seconds_fft = part.gpu_s;
    stats->seconds_total =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    stats->gpu_launches = part.launches + flc.n;
    stats->bands_run = part.bands_run;
  }
}

}  // namespace

extern "C" {

int xc_smooth(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
              const void* param, int normalize_signal, void* out, xc_stats* stats) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!signal || !param || !out || !d) throw std::invalid_argument("null argument");
    if (d->out_dtype != XC_F32 && d->out_dtype != XC_F64)
      throw std::invalid_argument("xc_smooth output must be real (XC_F32 / XC_F64)");
    check_integral(f);
    if (ctx->group)
      smooth_group(ctx, f, d, signal, param, normalize_signal, out, stats);
    else
      smooth_single(ctx, f, d, signal, param, normalize_signal, out, stats);
  });
}

}  // extern "C"

namespace {

void anglemax_tiled(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                    const int* components, int n_components, int n_angles, void* score,
                    int* argmax, xc_stats* stats);

void anglemax_single(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                     const int* components, int n_components, int n_angles, void* score,
                     int* argmax, xc_stats* stats) {
  {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const auto t_start = std::chrono::steady_clock::now();
    if (!signal || !score || !d) throw std::invalid_argument("null argument");
    if (n_angles < 1) throw std::invalid_argument("n_angles must be >= 1");
    if (d->out_dtype != XC_F32 && d->out_dtype != XC_F64)
      throw std::invalid_argument("xc_anglemax score must be real (XC_F32 / XC_F64)");
    // the score at p reads the signal within R of p only: tiles as in run_tiled
    if (f && needs_tiles(f, d, 0) && d->xform_kind == XC_ROTATION2) {
      anglemax_tiled(ctx, f, d, signal, components, n_components, n_angles, score, argmax, stats);
      return;
    }
    Call c = setup(ctx, f, d, XC_ROTATION2, components, n_components, false);
    const int span = *std::max_element(c.ks.begin(), c.ks.end()) -
                     *std::min_element(c.ks.begin(), c.ks.end()) + 1;
    if (span > 256) throw std::invalid_argument("band span too large for the angle max");
    const size_t npix = size_t(c.rows) * c.cols, os = dtype_size(d->out_dtype);
    // Hermitian half-band mode: real signal and F_{-k} = conj(F_k) over the
    // selected bands give G_{-k} = conj(G_k); only k >= 0 is transformed
    const bool real_sig = d->signal_dtype == XC_F32 || d->signal_dtype == XC_F64;
    bool herm = real_sig && n_angles == 360 && use_herm() && f->hf.hermitian() &&
                xcb::anglemax_herm_kh(*std::max_element(c.ks.begin(), c.ks.end()));
    for (int k : c.ks) herm = herm && std::count(c.ks.begin(), c.ks.end(), -k) == 1;
    xcb::Bands bands = c.bands;
    std::vector<int> hk;
    if (herm) {
      std::vector<int> hs;
      for (size_t i = 0; i < c.ks.size(); ++i)
        if (c.ks[i] >= 0) {
          hk.push_back(c.ks[i]);
          hs.push_back(c.sidx[i]);
        }
      std::vector<int> hb(hk);
      hb.insert(hb.end(), hs.begin(), hs.end());
      int* db = ctx->band_table(hb);
      bands = xcb::Bands{db, db + hk.size(), int(hk.size())};
    }
    c.nb_run = bands.n;
    c.band_mode = herm ? 1 : 0;
    float2* planes = ctx->buf<float2>("planes", size_t(bands.n) * npix);
    float2* T1 = ctx->buf<float2>("T1", size_t(c.g.Hx2) * c.g.Pw);
    float2* Hh = ctx->buf<float2>("Hhat", size_t(c.g.Ph) * c.g.Pw);
    float2* T2 = ctx->buf<float2>("T2", size_t(bands.n) * c.g.H2 * c.g.Pw);
    ctx->release_events();
    cudaEvent_t e0 = ctx->event(true), e1 = ctx->event(true);
    double gpu_s = 0;
    for (int img = 0; img < d->batch; ++img) {
      Staged s = stage_inputs(c, signal, nullptr, img);
      ck(cudaEventRecord(e0, c.st), "event");
      stage(c, "F1_rows_fwd", [&] { run_f1(c, s.sig, T1); });
      stage(c, "F2_cols_fwd", [&] { run_f2(c, T1, Hh); });
      stage(c, "I1_cols_inv_corr", [&] {
        if (use_pair() && xcb::pair_smem(0, c.g.Ph, c.g))
          xcb::launch_cols_inv_corr_pair(c.g, Hh, c.Fhat, c.sstride, bands, T2, c.st, c.lc);
        else if (c.fcol && xcb::fast_smem(0, *c.fcol, c.g))
          xcb::launch_cols_inv_corr_fast(*c.fcol, c.g, Hh, c.Fhat, c.sstride, bands, T2, c.st,
                                         c.lc);
        else
          xcb::launch_cols_inv_corr(*c.pcol, c.g, Hh, c.Fhat, c.sstride, bands, T2, c.st, c.lc);
      });
      stage(c, "I2_rows_inv_planes", [&] {
        if (use_pair() && xcb::pair_smem(2, c.g.Pw, c.g))
          xcb::launch_rows_inv_planes_pair(c.g, T2, bands.n, planes, c.st, c.lc);
        else if (c.frow && xcb::fast_smem(4, *c.frow, c.g))
          xcb::launch_rows_inv_planes_fast(*c.frow, c.g, T2, bands.n, planes, c.st, c.lc);
        else
          xcb::launch_rows_inv_planes(*c.prow, c.g, T2, bands.n, planes, c.st, c.lc);
      });
      char* dsc = d->memory == XC_DEVICE ? static_cast<char*>(score) + size_t(img) * npix * os
                                         : ctx->buf<char>("score_stage", npix * os);
      int* darg = nullptr;
      if (argmax)
        darg = d->memory == XC_DEVICE ? argmax + size_t(img) * npix
                                      : ctx->buf<int>("arg_stage", npix);
      stage(c, "anglemax", [&] {
        if (herm && use_angle_tc() &&
            xcb::anglemax_tc_ok(*std::max_element(hk.begin(), hk.end())))
          xcb::launch_anglemax_tc(planes, hk.data(), bands.n, npix, d->out_dtype == XC_F64, dsc,
                                  darg, c.st, c.lc);
        else if (herm)
          xcb::launch_anglemax_herm(planes, hk.data(), bands.n, npix, d->out_dtype == XC_F64, dsc,
                                    darg, c.st, c.lc);
        else
          xcb::launch_anglemax(planes, c.ks.data(), c.bands.n, npix, n_angles,
                               d->out_dtype == XC_F64, dsc, darg, c.st, c.lc);
      });
      ck(cudaGetLastError(), "kernel launch");
      ck(cudaEventRecord(e1, c.st), "event");
      ck(cudaEventSynchronize(e1), "anglemax");
      gpu_s += event_seconds(e0, e1);
      if (d->memory == XC_HOST) {
        auto t0 = std::chrono::steady_clock::now();
        ck(cudaMemcpy(static_cast<char*>(score) + size_t(img) * npix * os, dsc, npix * os,
                      cudaMemcpyDeviceToHost),
           "D2H");
        if (argmax)
          ck(cudaMemcpy(argmax + size_t(img) * npix, darg, npix * sizeof(int),
                        cudaMemcpyDeviceToHost),
             "D2H");
        c.d2h_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
    ctx->resolve_profile();
    fill_stats(c, stats, gpu_s,
               std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(),
               (long long)c.ks.size());
  }
}

// xc_anglemax over halo-extended tiles (see run_tiled): the tile interiors of
// the score and of the argmax are copied into the outputs
void anglemax_tiled(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                    const int* components, int n_components, int n_angles, void* score,
                    int* argmax, xc_stats* stats) {
  const auto t_start = std::chrono::steady_clock::now();
  if (d->height < 1 || d->width < 1 || d->batch < 1)
    throw std::invalid_argument("image dims must be positive");
  const int R = f->hf.render_radius();
  const bool cm = d->layout == XC_COL_MAJOR;
  const int MR = cm ? d->width : d->height, MC = cm ? d->height : d->width;
  auto split = [&](int n, int* nt, int* t) {
    *nt = tile_count(n, R);
    *t = (n + *nt - 1) / *nt;
  };
  int ntr, tr, ntc, tc;
  split(MR, &ntr, &tr);
  split(MC, &ntc, &tc);
  const size_t ss = dtype_size(d->signal_dtype), os = dtype_size(d->out_dtype);
  const size_t npix = size_t(MR) * MC;
  const size_t tmax = size_t(std::min(MR, tr + 2 * R)) * size_t(std::min(MC, tc + 2 * R));
  char* tsig = ctx->buf<char>("tile_sig", tmax * ss);
  char* tsc = ctx->buf<char>("tile_score", tmax * os);
  int* targ = argmax ? ctx->buf<int>("tile_arg", tmax) : nullptr;
  cudaStream_t st = ctx->stream;
  xc_stats agg{};
  for (int img = 0; img < d->batch; ++img) {
    const char* sg = static_cast<const char*>(signal) + size_t(img) * npix * ss;
    char* po = static_cast<char*>(score) + size_t(img) * npix * os;
    int* pa = argmax ? argmax + size_t(img) * npix : nullptr;
    for (int i = 0; i < ntr; ++i)
      for (int j = 0; j < ntc; ++j) {
        const int r0 = i * tr, r1 = std::min(MR, r0 + tr);
        const int c0 = j * tc, c1 = std::min(MC, c0 + tc);
        if (r0 >= r1 || c0 >= c1) continue;
        const int a0 = std::max(0, r0 - R), a1 = std::min(MR, r1 + R);
        const int b0 = std::max(0, c0 - R), b1 = std::min(MC, c1 + R);
        const int h = a1 - a0, w = b1 - b0;
        ck(cudaMemcpy2DAsync(tsig, size_t(w) * ss, sg + (size_t(a0) * MC + b0) * ss,
                             size_t(MC) * ss, size_t(w) * ss, size_t(h), cudaMemcpyDefault, st),
           "tile signal");
        xc_image_desc dt = *d;
        dt.batch = 1;
        dt.memory = XC_DEVICE;
        dt.height = cm ? w : h;
        dt.width = cm ? h : w;
        xc_stats s1{};
        anglemax_single(ctx, f, &dt, tsig, components, n_components, n_angles, tsc, targ, &s1);
        const size_t in_off = size_t(r0 - a0) * w + size_t(c0 - b0);
        const size_t out_off = size_t(r0) * MC + c0;
        ck(cudaMemcpy2DAsync(po + out_off * os, size_t(MC) * os, tsc + in_off * os,
                             size_t(w) * os, size_t(c1 - c0) * os, size_t(r1 - r0),
                             cudaMemcpyDefault, st),
           "tile score");
        if (pa)
          ck(cudaMemcpy2DAsync(pa + out_off, size_t(MC) * sizeof(int), targ + in_off,
                               size_t(w) * sizeof(int), size_t(c1 - c0) * sizeof(int),
                               size_t(r1 - r0), cudaMemcpyDefault, st),
             "tile argmax");
        agg.standard_ops = s1.standard_ops;
        agg.pad_h = std::max(agg.pad_h, s1.pad_h);
        agg.pad_w = std::max(agg.pad_w, s1.pad_w);
        agg.seconds_fft += s1.seconds_fft;
        agg.gpu_launches += s1.gpu_launches;
        agg.bands_run = s1.bands_run;
        agg.band_mode = s1.band_mode;
      }
  }
  ck(cudaStreamSynchronize(st), "tiles");
  if (stats) {
    *stats = agg;
    stats->seconds_total =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
}

}  // namespace

extern "C" {

int xc_anglemax(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                const int* components, int n_components, int n_angles, void* score,
                int* argmax, xc_stats* stats) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    anglemax_single(ctx, f, d, signal, components, n_components, n_angles, score, argmax, stats);
  });
}

// vote_filter.hpp:105-134
int xc_find_peaks(const void* resp, int dtype, int height, int width, int layout, double radius,
                  double threshold_frac, int* xs, int* ys, double* values, int max_peaks,
                  int* n_found) {
  return guarded(nullptr, [&] {
    if (!resp || !n_found) throw std::invalid_argument("null argument");
    if (dtype != XC_F32 && dtype != XC_F64) throw std::invalid_argument("response must be real");
    auto at = [&](int y, int x) -> double {
      const size_t i = layout == XC_COL_MAJOR ? size_t(x) * height + y : size_t(y) * width + x;
      return dtype == XC_F32 ? double(static_cast<const float*>(resp)[i])
                             : static_cast<const double*>(resp)[i];
    };
    double mx = -INFINITY;
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) mx = std::max(mx, at(y, x));
    const double thresh = threshold_frac * mx;
    const int R = std::max(1, int(std::ceil(radius)));
    struct Pk {
      int x, y;
      double v;
    };
    std::vector<Pk> peaks;
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) {
        const double v = at(y, x);
        if (v < thresh) continue;
        bool best = true;
        for (int dy = -R; dy <= R && best; ++dy)
          for (int dx = -R; dx <= R && best; ++dx) {
            if (dx == 0 && dy == 0) continue;
            if (dx * dx + dy * dy > radius * radius) continue;
            const int xi = x + dx, yi = y + dy;
            if (xi < 0 || yi < 0 || xi >= width || yi >= height) continue;
            const double o = at(yi, xi);
            if (o > v || (o == v && (dy < 0 || (dy == 0 && dx < 0)))) best = false;
          }
        if (best) peaks.push_back({x, y, v});
      }
    std::sort(peaks.begin(), peaks.end(), [](const Pk& a, const Pk& b) {
      if (a.v != b.v) return a.v > b.v;
      return a.y != b.y ? a.y < b.y : a.x < b.x;
    });
    const int n = int(peaks.size());
    for (int i = 0; i < std::min(n, max_peaks); ++i) {
      if (xs) xs[i] = peaks[i].x;
      if (ys) ys[i] = peaks[i].y;
      if (values) values[i] = peaks[i].v;
    }
    *n_found = n;
  });
}

// ---- find_peaks on a device response ---------------------------------------

namespace {
// NMS on the GPU, sort (value desc, y, x) on the host; returns the count
int device_peaks(xc_context ctx, const void* dresp, int dtype, int h, int w, int layout,
                 double radius, double frac, int* xs, int* ys, double* vals, int max_peaks) {
  cudaStream_t st = ctx->stream;
  xcb::LaunchCounter lc;
  int cap = 1 << 16;
  for (;;) {
    unsigned long long* mx = ctx->buf<unsigned long long>("nms_max", 1);
    unsigned* cnt = ctx->buf<unsigned>("nms_count", 1);
    int* px = ctx->buf<int>("nms_x", cap);
    int* py = ctx->buf<int>("nms_y", cap);
    double* pv = ctx->buf<double>("nms_v", cap);
    xcb::launch_find_peaks(dresp, dtype == XC_F64, h, w, layout == XC_COL_MAJOR, radius, frac, cap,
                           mx, cnt, px, py, pv, st, lc);
    ck(cudaGetLastError(), "find_peaks launch");
    unsigned n = 0;
    ck(cudaMemcpyAsync(&n, cnt, sizeof(n), cudaMemcpyDeviceToHost, st), "D2H count");
    ck(cudaStreamSynchronize(st), "find_peaks");
    if (int(n) > cap) {  // more local maxima than slots: rerun with room for all
      cap = int(n);
      continue;
    }
    struct Pk {
      int x, y;
      double v;
    };
    std::vector<int> hx(n), hy(n);
    std::vector<double> hv(n);
    if (n) {
      ck(cudaMemcpy(hx.data(), px, n * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
      ck(cudaMemcpy(hy.data(), py, n * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
      ck(cudaMemcpy(hv.data(), pv, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    }
    std::vector<Pk> pk(n);
    for (unsigned i = 0; i < n; ++i) pk[i] = {hx[i], hy[i], hv[i]};
    std::sort(pk.begin(), pk.end(), [](const Pk& a, const Pk& b) {
      if (a.v != b.v) return a.v > b.v;
      return a.y != b.y ? a.y < b.y : a.x < b.x;
    });
    for (int i = 0; i < std::min(int(n), max_peaks); ++i) {
      if (xs) xs[i] = pk[i].x;
      if (ys) ys[i] = pk[i].y;
      if (vals) vals[i] = pk[i].v;
    }
    return int(n);
  }
}
}  // namespace

int xc_find_peaks_device(xc_context ctx, const void* resp, int dtype, int height, int width,
                         int layout, double radius, double threshold_frac, int* xs, int* ys,
                         double* values, int max_peaks, int* n_found) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (!resp || !n_found) throw std::invalid_argument("null argument");
    if (dtype != XC_F32 && dtype != XC_F64) throw std::invalid_argument("response must be real");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    *n_found = device_peaks(ctx, resp, dtype, height, width, layout, radius, threshold_frac, xs,
                            ys, values, max_peaks);
  });
}

// ---- pattern detection (vote_filter.hpp) --------------------------------

namespace {
std::vector<double> real_rowmajor(const double* data, int height, int width, int layout) {
  std::vector<double> v(size_t(height) * width);
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < width; ++x)
      v[size_t(y) * width + x] =
          data[layout == XC_COL_MAJOR ? size_t(x) * height + y : size_t(y) * width + x];
  return v;
}
void export_vote(const xcb::VoteFilterHost& f, int layout, double* weights_out,
                 int* radius_out) {
  const int side = 2 * f.radius + 1;
  for (int y = 0; y < side; ++y)
    for (int x = 0; x < side; ++x)
      weights_out[layout == XC_COL_MAJOR ? size_t(x) * side + y : size_t(y) * side + x] =
          f.weights[size_t(y) * side + x];
  *radius_out = f.radius;
}
}  // namespace

int xc_build_vote_filter(const double* weight, const double* frame, int height, int width,
                         int layout, double px, double py, double eps, int nearest,
                         double* weights_out, int* radius_out) {
  return guarded(nullptr, [&] {
    if (!weight || !frame || !weights_out || !radius_out) throw std::invalid_argument("null argument");
    const auto wr = real_rowmajor(weight, height, width, layout);
    const auto fr = real_rowmajor(frame, height, width, layout);
    export_vote(xcb::build_vote_filter(wr.data(), fr.data(), height, width, px, py, eps,
                                       nearest != 0),
                layout, weights_out, radius_out);
  });
}

int xc_build_optimal_filter(const double* pattern, int height, int width, int layout, double px,
                            double py, double eps, int nearest, double* weights_out,
                            int* radius_out) {
  return guarded(nullptr, [&] {
    if (!pattern || !weights_out || !radius_out) throw std::invalid_argument("null argument");
    const auto pr = real_rowmajor(pattern, height, width, layout);
    export_vote(xcb::build_optimal_filter(pr.data(), height, width, px, py, eps, nearest != 0),
                layout, weights_out, radius_out);
  });
}

// detect_pattern (vote_filter.hpp:146-168): the vote filter is decomposed on
// the device (once per distinct pattern; the reference does it per call), the
// gradient runs on the GPU, the scatter is xc_run's pipeline, and the NMS peaks are found on the
// host.  The context lock is taken by the inner xc_run only.
int xc_detect_pattern(xc_context ctx, const xc_image_desc* d, const void* image,
                      const double* vote_weights, int radius, double eps, int K, int n_radii,
                      int n_angles, void* response, int* peak_x, int* peak_y, double* peak_v,
                      int max_peaks, int* n_peaks, xc_stats* stats) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (!d || !image || !vote_weights || !response || !n_peaks)
      throw std::invalid_argument("null argument");
    if (K < 1) throw std::invalid_argument("K must be >= 1");
    if (d->batch != 1) throw std::invalid_argument("detect_pattern takes one image");
    if (d->signal_dtype != XC_F32 && d->signal_dtype != XC_F64)
      throw std::invalid_argument("gradient requires real field");
    if (d->out_dtype != XC_F32 && d->out_dtype != XC_F64)
      throw std::invalid_argument("detect_pattern response must be real (XC_F32 / XC_F64)");
    if (radius < 0) throw std::invalid_argument("radius must be >= 0");
    const auto t_start = std::chrono::steady_clock::now();
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int h = d->height, w = d->width, R = radius, side = 2 * R + 1;
    const size_t npix = size_t(h) * w;
    // the vote filter's decomposition parameters (engine defaults of
    // vote_filter.hpp:157-160)
    if (n_radii == 0) n_radii = std::max(4, 2 * R);
    if (n_angles == 0) n_angles = std::max(16, 8 * ((R + 1) / 2) * 2);
    std::vector<cplx> vf(size_t(side) * side);
    for (int y = 0; y < side; ++y)
      for (int x = 0; x < side; ++x)
        vf[size_t(y) * side + x] = cplx(
            vote_weights[d->layout == XC_COL_MAJOR ? size_t(x) * side + y : size_t(y) * side + x],
            0.0);
    // the decomposed vote filter (and its device spectra) is cached per
    // context by content, so repeated detections with one pattern reuse it
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](const void* p, size_t n) {
      const unsigned char* b = static_cast<const unsigned char*>(p);
      for (size_t i = 0; i < n; ++i) key = (key ^ b[i]) * 1099511628211ull;
    };
    mix(vf.data(), vf.size() * sizeof(cplx));
    const int params[4] = {R, K, n_radii, n_angles};
    mix(params, sizeof(params));
    auto it = ctx->det_filters.find(key);
    if (it == ctx->det_filters.end()) {
      if (ctx->det_filters.size() >= 4) ctx->det_filters.clear();
      std::unique_ptr<xc_filter_s, void (*)(xc_filter_s*)> nf(new xc_filter_s(),
                                                              xc_filter_destroy);
      // per-call filter build on the device (freq_filter.hpp:63-89)
      nf->hf = xcb::rotation2_shell(K, n_radii, n_angles, double(R) + 0.5);
      {
        std::lock_guard<std::mutex> lk(ctx->mu);
        decompose_on_device(ctx, nf->hf, vf, side, side, double(R), double(R));
      }
      it = ctx->det_filters.emplace(key, std::move(nf)).first;
    }
    xc_filter_s* f = it->second.get();
    // device: gradient of the image
    cudaStream_t st = ctx->stream;
    xcb::LaunchCounter lc;
    const size_t is = dtype_size(d->signal_dtype), os = dtype_size(d->out_dtype);
    const void* dimg = image;
    if (d->memory == XC_HOST) {
      void* b = ctx->buf<char>("det_image", npix * is);
      ck(cudaMemcpyAsync(b, image, npix * is, cudaMemcpyHostToDevice, st), "H2D image");
      dimg = b;
    }
    float* mag = ctx->buf<float>("det_mag", npix);
    float* dir = ctx->buf<float>("det_dir", npix);
    xcb::launch_gradient(dimg, d->signal_dtype == XC_F64, h, w, d->layout == XC_COL_MAJOR, mag,
                         dir, st, lc);
    ck(cudaGetLastError(), "gradient launch");
    // scatter: xconv_fast(|grad|, rotation(direction), F)
    float2* out = ctx->buf<float2>("det_out", npix);
    xc_image_desc dd{h, w, 1, XC_F32, XC_F32, XC_C64, d->layout, XC_DEVICE, 1, XC_ROTATION2};
    xc_stats rs{};
    if (xc_run(ctx, f, XC_CONVOLUTION, &dd, mag, dir, nullptr, 0, 0, out, &rs) != XC_OK)
      throw std::runtime_error(ctx->err);
    // response = Re(out); NMS on the host
    void* dresp = d->memory == XC_DEVICE ? response : ctx->buf<char>("det_resp", npix * os);
    xcb::launch_real_part(out, npix, d->out_dtype == XC_F64, dresp, st, lc);
    ck(cudaGetLastError(), "real part launch");
    *n_peaks = device_peaks(ctx, dresp, d->out_dtype, h, w, d->layout, eps / 2, 0.5, peak_x,
                            peak_y, peak_v, max_peaks);
    if (d->memory == XC_HOST)
      ck(cudaMemcpy(response, dresp, npix * os, cudaMemcpyDeviceToHost), "D2H response");
    if (stats) {
      *stats = rs;
      stats->gpu_launches += lc.n;
      stats->seconds_total =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
  });
}

}  // extern "C"

// ================================================================ 3D rotation
// xcorr_fast_3d / xconv_fast_3d (engine3d.hpp:270-335) on the
// k_3d.cu stages.  The per-band spectra of a filter are built once per
// (device, pad) and cached; bands are (l, m, m') in the reference's loop order.

struct xc_filter3_s {
  xcb::HostFilter3 hf;
  std::mutex mu;  // guards the spectrum cache (handles may be shared across threads)
  std::map<std::tuple<int, int, int, int>, float2*> spectra;  // (dev, px, py, pz)
  ~xc_filter3_s() {
    for (auto& kv : spectra) {
      cudaSetDevice(std::get<0>(kv.first));
      cudaFree(kv.second);
    }
  }
};

namespace {

int band_offset(int l) {  // bands of degrees < l: sum (2l'+1)^2
  int n = 0;
  for (int d = 0; d < l; ++d) n += (2 * d + 1) * (2 * d + 1);
  return n;
}

// every band of the filter rendered on (2R+1)^3, x-, y-, z-transformed
float2* filter3_spectra(xc_context ctx, xc_filter3 f, const xcb::Geo3& g, const xcb::FftPlan& pxp,
                        const xcb::FftPlan& pyp, const xcb::FftPlan& pzp, cudaStream_t st,
                        xcb::LaunchCounter& lc) {
  const auto key = std::make_tuple(ctx->device, g.px, g.py, g.pz);
  std::lock_guard<std::mutex> flk(f->mu);
  auto it = f->spectra.find(key);
  if (it != f->spectra.end()) return it->second;
  const xcb::HostFilter3& hf = f->hf;
  const int S = 2 * g.R + 1, nb = band_offset(hf.K + 1);
  const size_t S3 = size_t(S) * S * S, P = size_t(g.px) * g.py * g.pz;
  std::vector<float2> comps(S3 * nb);
  std::vector<cplx> tmp(S3);
  int b = 0;
  for (int l = 0; l <= hf.K; ++l)
    for (int m = -l; m <= l; ++m)
      for (int mp = -l; mp <= l; ++mp, ++b) {  // engine3d.hpp:286-289
        xcb::render_sph_component(hf, l, m, mp, S, S, S, g.R, g.R, g.R, tmp.data());
        for (size_t i = 0; i < S3; ++i)
          comps[b * S3 + i] = make_float2(float(tmp[i].real()), float(tmp[i].imag()));
      }
  float2* dcomps = ctx->buf<float2>("f3_comps", comps.size());
  ck(cudaMemcpyAsync(dcomps, comps.data(), comps.size() * sizeof(float2), cudaMemcpyHostToDevice,
                     st),
     "upload 3D filter bands");
  float2* spec = nullptr;
  ck(cudaMalloc(&spec, P * nb * sizeof(float2)), "cudaMalloc 3D spectra");
  xcb::launch3_x_filter(pxp, g, dcomps, nb, spec, P, st, lc);
  xcb::launch3_pass(pyp, g, 1, spec, P, nb, st, lc);
  xcb::launch3_pass(pzp, g, 2, spec, P, nb, st, lc);
  ck(cudaGetLastError(), "3D filter spectra launch");
  ck(cudaStreamSynchronize(st), "3D filter spectra");  // host staging lifetime
  f->spectra[key] = spec;
  return spec;
}

xcb::Band3 make_band3(int l, int m, int mp) {
  // D^l_{m' m}: wigner_d_entry(l, mp, m, ...) (engine3d.hpp:296, 320)
  const xcb::SmallD d = xcb::small_d_coeffs(l, mp, m);
  xcb::Band3 b{};
  b.l = l;
  b.m = m;
  b.mp = mp;
  b.n = d.n;
  b.pc_end = d.pc_end;
  b.ps0 = d.ps0;
  for (int k = 0; k <= d.n; ++k) b.c[k] = d.c[k];
  return b;
}

}  // namespace

extern "C" {

int xc_filter3_create(int K, int n_radii, double r_max, const double* coeffs, xc_filter3* out) {
  return guarded(nullptr, [&] {
    if (!out || !coeffs) throw std::invalid_argument("null argument");
    if (K < 0 || K > 16) throw std::invalid_argument("band limit must be in [0, 16]");
    if (n_radii < 1) throw std::invalid_argument("n_radii must be >= 1");
    if (!(r_max > 0)) throw std::invalid_argument("r_max must be > 0");
    auto f = std::make_unique<xc_filter3_s>();
    xcb::HostFilter3& h = f->hf;
    h.K = K;
    h.n_radii = n_radii;
    h.r_max = r_max;
    const int nc = h.ncol();
    h.coeffs.resize(size_t(n_radii) * nc);
    for (int c = 0; c < nc; ++c)
      for (int r = 0; r < n_radii; ++r)
        h.coeffs[size_t(r) * nc + c] =
            cplx(coeffs[2 * (size_t(c) * n_radii + r)], coeffs[2 * (size_t(c) * n_radii + r) + 1]);
    *out = f.release();
  });
}

void xc_filter3_destroy(xc_filter3 f) { delete f; }

int xc_decompose_rotation3(const double* volume, int nx, int ny, int nz, double cx, double cy,
                           double cz, int K, int n_radii, double r_max, int n_theta, int n_phi,
                           double* coeffs_out) {
  return guarded(nullptr, [&] {
    if (!volume || !coeffs_out) throw std::invalid_argument("null argument");
    auto f = xcb::decompose_rotation3(reinterpret_cast<const cplx*>(volume), nx, ny, nz, cx, cy,
                                      cz, K, n_radii, r_max, n_theta, n_phi);
    const int nc = f.ncol();
    for (int c = 0; c < nc; ++c)
      for (int r = 0; r < n_radii; ++r) {
        coeffs_out[2 * (size_t(c) * n_radii + r)] = f.coeffs[size_t(r) * nc + c].real();
        coeffs_out[2 * (size_t(c) * n_radii + r) + 1] = f.coeffs[size_t(r) * nc + c].imag();
      }
  });
}

int xc_render_sph_component(xc_filter3 f, int l, int m_radial, int m_angular, int nx, int ny,
                            int nz, double cx, double cy, double cz, double* out) {
  return guarded(nullptr, [&] {
    xcb::render_sph_component(f->hf, l, m_radial, m_angular, nx, ny, nz, cx, cy, cz,
                              reinterpret_cast<cplx*>(out));
  });
}

int xc_reconstruct3(xc_filter3 f, int nx, int ny, int nz, double cx, double cy, double cz,
                    const int* degrees, int ndeg, double* out) {
  return guarded(nullptr, [&] {
    xcb::reconstruct3(f->hf, nx, ny, nz, cx, cy, cz, ndeg >= 0 ? degrees : nullptr, ndeg,
                      reinterpret_cast<cplx*>(out));
  });
}

int xc_sph_harm(int l, int m, double theta, double phi, double* out2) {
  return guarded(nullptr, [&] {
    const cplx v = xcb::sph_harm(l, m, theta, phi);
    out2[0] = v.real();
    out2[1] = v.imag();
  });
}

int xc_white_noise(unsigned long long seed, int height, int width, int layout, double* out) {
  return guarded(nullptr, [&] {
    if (!out) throw std::invalid_argument("null argument");
    if (height < 0 || width < 0) throw std::invalid_argument("dims must be non-negative");
    std::mt19937_64 rng(seed);
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) {
        const double v = double(rng() >> 11) * 0x1p-53;
        out[layout == XC_COL_MAJOR ? size_t(x) * height + y : size_t(y) * width + x] = v;
      }
  });
}

int xc_wigner_d(int l, const double* quat, double* out) {
  return guarded(nullptr, [&] { xcb::wigner_d(l, quat, reinterpret_cast<cplx*>(out)); });
}

int xc_run3(xc_context ctx, xc_filter3 f, int mode, int nx, int ny, int nz, const void* signal,
            int signal_dtype, const double* quats, const int* degrees, int ndeg, int memory,
            double* out, xc_stats* stats) {
  return guarded(ctx, [&] {
    const auto t_start = std::chrono::steady_clock::now();
    if (!ctx || !f || !signal || !quats || !out) throw std::invalid_argument("null argument");
    if (mode != XC_CORRELATION && mode != XC_CONVOLUTION) throw std::invalid_argument("unknown mode");
    if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("volume dims must be positive");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const xcb::HostFilter3& hf = f->hf;
    // plan_degrees (engine3d.hpp:11-16 over engine.hpp:51-58)
    std::vector<int> ls;
    if (degrees && ndeg > 0) {
      for (int i = 0; i < ndeg; ++i) {
        if (degrees[i] < 0 || degrees[i] > hf.K)
          throw std::invalid_argument("plan retains a component the filter lacks");
        ls.push_back(degrees[i]);
      }
    } else {
      for (int l = 0; l <= hf.K; ++l) ls.push_back(l);
    }
    std::vector<xcb::Band3> bands;
    std::vector<int> sidx;
    for (int l : ls)
      for (int m = -l; m <= l; ++m)
        for (int mp = -l; mp <= l; ++mp) {
          bands.push_back(make_band3(l, m, mp));
          sidx.push_back(band_offset(l) + (m + l) * (2 * l + 1) + (mp + l));
        }
    const int nb = int(bands.size());
    xcb::Geo3 g{nx, ny, nz, 0, 0, 0, hf.render_radius()};
    const int R = g.R;
    g.px = pick_pad(std::max(nx + R, 2 * R + 1));
    g.py = pick_pad(std::max(ny + R, 2 * R + 1));
    g.pz = pick_pad(std::max(nz + R, 2 * R + 1));
    if (g.px < 0 || g.py < 0 || g.pz < 0) throw std::invalid_argument("volume too large for the FFT planner");
    if (xcb::tile3_smem(std::max({g.px, g.py, g.pz})) > 200 * 1024)
      throw std::invalid_argument("volume too large for the 3D line transforms");
    const xcb::FftPlan& pxp = ctx->plan3(g.px);
    const xcb::FftPlan& pyp = ctx->plan3(g.py);
    const xcb::FftPlan& pzp = ctx->plan3(g.pz);
    cudaStream_t st = ctx->stream;
    xcb::LaunchCounter lc;
    const size_t N = size_t(nx) * ny * nz, P = size_t(g.px) * g.py * g.pz;
    float2* spec = filter3_spectra(ctx, f, g, pxp, pyp, pzp, st, lc);
    ctx->release_events();
    cudaEvent_t e0 = ctx->event(true), e1 = ctx->event(true);
    ck(cudaEventRecord(e0, st), "event");
    // inputs: signal -> complex fp32, quaternions -> per-voxel Euler data
    const size_t ss = dtype_size(signal_dtype);
    const void* dsig_raw = signal;
    const double* dq = quats;
    if (memory == XC_HOST) {
      void* b = ctx->buf<char>("v3_sig_raw", N * ss);
      ck(cudaMemcpyAsync(b, signal, N * ss, cudaMemcpyHostToDevice, st), "H2D signal");
      dsig_raw = b;
      double* q = ctx->buf<double>("v3_quats", 4 * N);
      ck(cudaMemcpyAsync(q, quats, 4 * N * sizeof(double), cudaMemcpyHostToDevice, st), "H2D quats");
      dq = q;
    }
    float2* dsig = ctx->buf<float2>("v3_sig", N);
    xcb::launch3_signal(dsig_raw, signal_dtype, N, dsig, st, lc);
    double4* eul = ctx->buf<double4>("v3_euler", N);
    xcb::launch3_euler(dq, N, eul, st, lc);
    xcb::Band3* dbands = ctx->buf<xcb::Band3>("v3_bands", size_t(nb));
    int* dsidx = ctx->buf<int>("v3_sidx", size_t(nb));
    ck(cudaMemcpyAsync(dbands, bands.data(), nb * sizeof(xcb::Band3), cudaMemcpyHostToDevice, st),
       "upload bands");
    ck(cudaMemcpyAsync(dsidx, sidx.data(), nb * sizeof(int), cudaMemcpyHostToDevice, st),
       "upload band spectra");
    double2* dout = memory == XC_DEVICE ? reinterpret_cast<double2*>(out)
                                        : ctx->buf<double2>("v3_out", N);
    // bands per chunk: work volumes (and gather planes) within a budget
    // (XCB_3D_CHUNK_MB, default 4 GB)
    static const size_t chunk_budget = [] {
      const char* e = std::getenv("XCB_3D_CHUNK_MB");
      return e && std::atol(e) > 0 ? size_t(std::atol(e)) << 20 : size_t(4) << 30;
    }();
    const size_t per_band = (P + (mode == XC_CORRELATION ? N : 0)) * sizeof(float2);
    const int cb = int(std::max<size_t>(1, std::min<size_t>(nb, chunk_budget / per_band)));
    float2* work = ctx->buf<float2>("v3_work", P * cb);
    if (mode == XC_CORRELATION) {
      float2* Hh = ctx->buf<float2>("v3_Hhat", P);
      float2* part = ctx->buf<float2>("v3_part", N * cb);
      xcb::launch3_x_signal(pxp, g, dsig, eul, dbands, 1, 0, Hh, P, st, lc);
      xcb::launch3_pass(pyp, g, 1, Hh, P, 1, st, lc);
      xcb::launch3_pass(pzp, g, 2, Hh, P, 1, st, lc);
      for (int b0 = 0; b0 < nb; b0 += cb) {
        const int n = std::min(cb, nb - b0);
        xcb::launch3_z_load(pzp, g, Hh, spec, dsidx + b0, n, P, 0, work, st, lc);
        xcb::launch3_pass(pyp, g, 1, work, P, n, st, lc);
        xcb::launch3_x_out(pxp, g, work, P, n, eul, dbands + b0, 0, part, 0, nullptr, st, lc);
        xcb::launch3_reduce_parts(part, n, N, b0 > 0, dout, st, lc);
      }
    } else {
      float2* sum = ctx->buf<float2>("v3_sum", P);
      ck(cudaMemsetAsync(sum, 0, P * sizeof(float2), st), "memset");
      for (int b0 = 0; b0 < nb; b0 += cb) {
        const int n = std::min(cb, nb - b0);
        xcb::launch3_x_signal(pxp, g, dsig, eul, dbands + b0, n, 1, work, P, st, lc);
        xcb::launch3_pass(pyp, g, 1, work, P, n, st, lc);
        xcb::launch3_pass(pzp, g, 2, work, P, n, st, lc);
        xcb::launch3_mac(work, n, P, spec, dsidx + b0, sum, st, lc);
      }
      xcb::launch3_z_load(pzp, g, sum, nullptr, nullptr, 1, P, 1, work, st, lc);
      xcb::launch3_pass(pyp, g, 1, work, P, 1, st, lc);
      xcb::launch3_x_out(pxp, g, work, P, 1, eul, dbands, 1, nullptr, 0, dout, st, lc);
    }
    ck(cudaGetLastError(), "3D kernel launch");
    ck(cudaEventRecord(e1, st), "event");
    if (memory == XC_HOST)
      ck(cudaMemcpyAsync(out, dout, N * sizeof(double2), cudaMemcpyDeviceToHost, st), "D2H out");
    ck(cudaStreamSynchronize(st), "xc_run3");
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->standard_ops = nb;  // engine3d.hpp:299, 331
      stats->pad_h = g.py;
      stats->pad_w = g.px;
      stats->seconds_fft = event_seconds(e0, e1);
      stats->seconds_total =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      stats->gpu_launches = lc.n;
    }
  });
}

}  // extern "C"

// ================================================================ multi-device
// the bands are independent terms of the extended sum
// (engine.hpp:300-319, 345-368) and XConvPlan::components (engine.hpp:19)
// selects a band subset, so a context over several GPUs splits the bands in
// contiguous ranges (balanced to +-1), runs each range on its device and sums
// the partial outputs with one NCCL reduce onto the first device.  The scale
// group's inner-DC term (engine.hpp:320-324 / 369-371) is added by the first
// device only.  smooth_adaptive (engine.hpp:385-419) is nonlinear: the
// numerator and denominator partials are reduced, then divided on the root.
//
//   xc_context_create_multi: one process drives several devices (one child
//     context and one NCCL communicator per device, ncclCommInitAll).  A device
//     listed twice (or XCB_REDUCE=peer) uses the peer-copy reduce instead: the
//     partials are copied to the root with cudaMemcpyPeerAsync and summed in
//     device order by launch_accumulate -- the same orchestration, testable
//     on one GPU.
//   xc_context_create_rank: one process per GPU; every rank calls xc_run /
//     xc_smooth with the same arguments and its own copy of the inputs, and
//     rank 0 receives the result (ncclCommInitRank over a shared unique id).
//
// XC_SHARD_BATCH splits the images of a batch across the devices instead (no
// collective; single-process contexts only).

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int,
                         ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is loaded on first use, so single-device use never needs it.  An NCCL
// already mapped into the process (torch's) is reused; else XCB_NCCL_LIBRARY,
// else the loader's libnccl.so.2.  (Loading an older libnccl.so.2 first would
// shadow a newer one that a later `import torch` needs: the Python binding
// imports torch before creating a multi-GPU context.)
const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* p = std::getenv("XCB_NCCL_LIBRARY")) h = dlopen(p, RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Reduce = reinterpret_cast<decltype(a.Reduce)>(sym("ncclReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitAll && a.CommInitRank && a.CommDestroy && a.Reduce &&
           a.GroupStart && a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

const NcclApi& nccl_or_throw() {
  const NcclApi& a = nccl();
  if (!a.ok) throw CudaError(a.why, XC_ENCCL);
  return a;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r), XC_ENCCL);
}

struct Group {
  std::vector<xc_context> kids;   // single-process: one child context per device
  std::vector<ncclComm_t> comms;  // one per kid, or the rank's one; empty = peer reduce
  bool rank_mode = false;
  // every kid's device can store into kids[0]'s memory (same device or peer
  // access over NVLink): partials are written straight into the root (peer_slots)
  bool peer_write = false;
  int rank = 0, nranks = 1;
  int shard = XC_SHARD_BANDS;
  // XC_FLAG_ASYNC (rank contexts): the reduce of call i runs on `comm` while
  // call i + 1 computes into the other partial buffer
  int device = 0;
  cudaStream_t comm = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};
  int slot = 0;
  ~Group() {
    if (comm) {
      cudaSetDevice(device);
      cudaStreamSynchronize(comm);
      for (cudaEvent_t e : done)
        if (e) cudaEventDestroy(e);
      cudaStreamDestroy(comm);
    }
    for (ncclComm_t c : comms)
      if (c) nccl().CommDestroy(c);
    for (xc_context k : kids) delete k;
  }
};

void destroy_group(Group* g) { delete g; }

// contiguous ranges balanced to +-1: 65 bands over 8 devices -> 8,8,8,8,8,8,8,9
std::pair<int, int> shard_range(int n, int r, int world) {
  return {int((long long)n * r / world), int((long long)n * (r + 1) / world)};
}

// pairs (shard_in_pairs): the bands k >= 0 are split in contiguous ranges and
// each rank takes its k and -k, so its share stays symmetric
std::vector<int> shard_bands(const std::vector<int>& ks, int r, int world, bool pairs = false) {
  if (!pairs) {
    const auto ab = shard_range(int(ks.size()), r, world);
    return std::vector<int>(ks.begin() + ab.first, ks.begin() + ab.second);
  }
  std::vector<int> nn;
  for (int k : ks)
    if (k >= 0) nn.push_back(k);
  const auto ab = shard_range(int(nn.size()), r, world);
  std::vector<int> mine;
  for (int k : ks)
    if (std::find(nn.begin() + ab.first, nn.begin() + ab.second, k < 0 ? -k : k) !=
        nn.begin() + ab.second)
      mine.push_back(k);
  return mine;
}

// Real signals run symmetric band selections in +-k pairs, transforming the
// bands k >= 0 only (the Hermitian half-band mode when F_{-k} = conj F_k; the
// scatter's conjugate band pairs for any filter), so a device's share must
// hold whole pairs and the load is the number of its bands k >= 0.
bool shard_in_pairs(xc_filter f, int mode, const xc_image_desc* d, const std::vector<int>& ks) {
  if (d->signal_dtype != XC_F32 && d->signal_dtype != XC_F64) return false;
  const bool herm = use_herm() && f->hf.hermitian();
  if (!(herm || (mode == XC_CONVOLUTION && use_cpair()))) return false;
  for (int k : ks)
    if (std::count(ks.begin(), ks.end(), -k) != 1 || std::count(ks.begin(), ks.end(), k) != 1)
      return false;
  return true;
}

// error of a worker thread, rethrown on the calling thread in device order
struct KidError {
  int code = XC_OK;
  std::string msg;
  void run(const std::function<void(int)>& fn, int i) {
    try {
      fn(i);
    } catch (const CudaError& e) {
      code = e.code;
      msg = e.what();
    } catch (const std::invalid_argument& e) {
      code = XC_EINVAL;
      msg = e.what();
    } catch (const std::bad_alloc&) {
      code = XC_ENOMEM;
      msg = "host allocation failed";
    } catch (const std::exception& e) {
      code = XC_EINTERNAL;
      msg = e.what();
    }
  }
};

struct KidRunner {
  KidError* e;
  const std::function<void(int)>* fn;
  int i;
  void operator()() const { e->run(*fn, i); }
};

// fn(i) for every device i, each on its own host thread (kid 0 on this one)
void for_each_kid(int n, const std::function<void(int)>& fn) {
  std::vector<KidError> errs(static_cast<size_t>(n));
  std::vector<std::thread> th;
  for (int i = 1; i < n; ++i) th.emplace_back(KidRunner{&errs[i], &fn, i});
  errs[0].run(fn, 0);
  for (auto& t : th) t.join();
  for (auto& e : errs) {
    if (e.code == XC_EINVAL) throw std::invalid_argument(e.msg);
    if (e.code != XC_OK) throw CudaError(e.msg, e.code);
  }
}

// The reduce of `n` per-device buffers of `count` floats / doubles onto
// bufs[0] (on kids[0]'s device).
void reduce_to_root(Group& G, const std::vector<void*>& bufs, size_t count, bool f64) {
  const int n = int(bufs.size());
  if (n <= 1) return;
  if (!G.comms.empty()) {
    const NcclApi& a = nccl_or_throw();
    nck(a.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < n; ++i) {
      ck(cudaSetDevice(G.kids[i]->device), "cudaSetDevice");
      nck(a.Reduce(bufs[i], bufs[i], count, f64 ? ncclDouble : ncclFloat, ncclSum, 0,
                   G.comms[i], G.kids[i]->stream),
          "ncclReduce");
    }
    nck(a.GroupEnd(), "ncclGroupEnd");
    for (int i = 0; i < n; ++i) {
      ck(cudaSetDevice(G.kids[i]->device), "cudaSetDevice");
      ck(cudaStreamSynchronize(G.kids[i]->stream), "band reduce");
    }
    ck(cudaSetDevice(G.kids[0]->device), "cudaSetDevice");
    return;
  }
  // peer reduce: partials copied to the root and summed in device order
  xc_context root = G.kids[0];
  ck(cudaSetDevice(root->device), "cudaSetDevice");
  const size_t bytes = count * (f64 ? 8 : 4);
  void* tmp = root->buf<char>("grp_peer_tmp", bytes);
  xcb::LaunchCounter lc;
  for (int i = 1; i < n; ++i) {
    // the kid's partial is complete: its run synchronized its stream
    ck(cudaMemcpyPeerAsync(tmp, root->device, bufs[i], G.kids[i]->device, bytes, root->stream),
       "peer copy");
    xcb::launch_accumulate(bufs[0], tmp, count, f64 ? 1 : 0, root->stream, lc);
    ck(cudaGetLastError(), "kernel launch");
  }
  ck(cudaStreamSynchronize(root->stream), "peer reduce");
}

// XCB_PEER_WRITE=0: partials stay on their devices and are reduced by NCCL (or
// the peer-copy reduce) instead of being written into the root's memory
bool use_peer_write() {
  static const bool on = [] {
    const char* e = std::getenv("XCB_PEER_WRITE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Fused partial delivery (single-process multi-device contexts).  The last
// kernel of a device's share (I2's steering sum, S4, the smoothing scatters)
// takes its output pointer from here: slot i - 1 of a buffer in the ROOT's
// memory, so its stores go over NVLink as the rows are produced and overlap
// the transforms still running; no partial is staged locally and no separate
// collective moves it.  The root then adds the slots in device order
// (sum_peer_slots).  Returns nullptr when the topology has no peer access
// (reduce_to_root then runs NCCL).
char* peer_slots(Group& G, const char* name, size_t bytes) {
  const int n = int(G.kids.size());
  if (n <= 1 || !G.peer_write || !use_peer_write()) return nullptr;
  xc_context root = G.kids[0];
  std::lock_guard<std::mutex> lk(root->mu);
  ck(cudaSetDevice(root->device), "cudaSetDevice");
  return root->buf<char>(name, size_t(n - 1) * bytes);
}

// parts[0] += slot 0 + slot 1 + ... (one kernel on the root; every kid's run
// has synchronized its stream, so its remote stores are complete)
void sum_peer_slots(Group& G, void* part0, const char* slots, size_t count, bool f64,
                    xcb::LaunchCounter& lc) {
  xc_context root = G.kids[0];
  ck(cudaSetDevice(root->device), "cudaSetDevice");
  xcb::launch_sum_slots(part0, slots, count, int(G.kids.size()) - 1, count, f64 ? 1 : 0,
                        root->stream, lc);
  ck(cudaGetLastError(), "kernel launch");
  ck(cudaStreamSynchronize(root->stream), "peer slot sum");
}

// Inputs of images [a, b) on kid k: the caller's pointers when they are host
// memory or already on k's device, else peer copies from the root device.
void kid_inputs(xc_context root, xc_context k, const xc_image_desc& d, const void* signal,
                const void* param, int a, int b, const void** sg, const void** pr) {
  const size_t npix = size_t(d.height) * d.width;
  const size_t ss = dtype_size(d.signal_dtype), ps = dtype_size(d.param_dtype);
  const char* s0 = static_cast<const char*>(signal) + size_t(a) * npix * ss;
  const char* p0 = param ? static_cast<const char*>(param) +
                               (d.param_per_image ? size_t(a) * npix * ps : 0)
                         : nullptr;
  *sg = s0;
  *pr = p0;
  if (d.memory == XC_HOST || k->device == root->device) return;
  const size_t sb = size_t(b - a) * npix * ss;
  const size_t pb = (d.param_per_image ? size_t(b - a) : 1) * npix * ps;
  void* bs = k->buf<char>("grp_sig", sb);
  ck(cudaMemcpyPeerAsync(bs, k->device, s0, root->device, sb, k->stream), "peer copy signal");
  *sg = bs;
  if (p0) {
    void* bp = k->buf<char>("grp_par", pb);
    ck(cudaMemcpyPeerAsync(bp, k->device, p0, root->device, pb, k->stream), "peer copy param");
    *pr = bp;
  }
}

// out (d.memory) <- buf (device, on ctx's device): copy, or add for XC_FLAG_ACCUMULATE
void deliver(xc_context ctx, const xc_image_desc& d, const void* buf, void* out, size_t bytes,
             bool accumulate, bool f64, xcb::LaunchCounter& lc) {
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (buf == out) return;
  if (d.memory == XC_HOST) {
    ck(cudaMemcpyAsync(out, buf, bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  } else if (accumulate) {
    xcb::launch_accumulate(out, buf, bytes / (f64 ? 8 : 4), f64 ? 1 : 0, ctx->stream, lc);
    ck(cudaGetLastError(), "kernel launch");
  } else {
    ck(cudaMemcpyAsync(out, buf, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
  }
  ck(cudaStreamSynchronize(ctx->stream), "deliver");
}

void merge_stats(xc_stats* out, const std::vector<xc_stats>& st, long long ops, double t0_s) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->standard_ops = ops;
  for (const auto& s : st) {
    out->pad_h = std::max(out->pad_h, s.pad_h);
    out->pad_w = std::max(out->pad_w, s.pad_w);
    out->seconds_fft = std::max(out->seconds_fft, s.seconds_fft);
    out->seconds_h2d = std::max(out->seconds_h2d, s.seconds_h2d);
    out->seconds_d2h = std::max(out->seconds_d2h, s.seconds_d2h);
    out->clamped_pixels += s.clamped_pixels;
    out->gpu_launches += s.gpu_launches;
    out->bands_run += s.bands_run;
    out->band_mode = std::max(out->band_mode, s.band_mode);
  }
  out->seconds_total = t0_s;
}

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void run_group(xc_context ctx, xc_filter f, int mode, const xc_image_desc* d,
               const void* signal, const void* param, const int* components, int n_components,
               unsigned flags, void* out, xc_stats* stats) {
  const auto t_start = std::chrono::steady_clock::now();
  Group& G = *ctx->group;
  if (!f || !d || !signal || !param || !out) throw std::invalid_argument("null argument");
  if (mode != XC_CORRELATION && mode != XC_CONVOLUTION) throw std::invalid_argument("unknown mode");
  if (d->out_dtype != XC_C64 && d->out_dtype != XC_C128)
    throw std::invalid_argument("xc_run output must be complex (XC_C64 / XC_C128)");
  if (d->height < 1 || d->width < 1 || d->batch < 1)
    throw std::invalid_argument("image dims must be positive");
  const std::vector<int> ks = plan_components(f->hf, components, n_components);
  const bool pairs = shard_in_pairs(f, mode, d, ks);
  const bool accumulate = (flags & XC_FLAG_ACCUMULATE) != 0;
  if (accumulate && d->memory != XC_DEVICE)
    throw std::invalid_argument("XC_FLAG_ACCUMULATE needs device memory");
  const size_t npix = size_t(d->height) * d->width, os = dtype_size(d->out_dtype);
  const size_t bytes = npix * size_t(d->batch) * os;
  const bool f64 = d->out_dtype == XC_C128;
  const unsigned kid_flags = flags & ~(XC_FLAG_ACCUMULATE | XC_FLAG_ASYNC);
  xcb::LaunchCounter lc;

  if (G.rank_mode && (flags & XC_FLAG_ASYNC) && d->memory == XC_DEVICE) {
    // compute into partial slot s (host-synchronous, like every call), then
    // queue the reduce and the root's delivery on the comm stream and return;
    // slot s is reused two calls later, after its reduce completed
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!G.comm) {
      G.device = ctx->device;
      ck(cudaStreamCreateWithFlags(&G.comm, cudaStreamNonBlocking), "cudaStreamCreate");
      for (auto& e : G.done) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    const int s = G.slot;
    G.slot ^= 1;
    ck(cudaEventSynchronize(G.done[s]), "previous reduce");
    const std::vector<int> mine = shard_bands(ks, G.rank, G.nranks, pairs);
    void* part = ctx->buf<char>("grp_part" + std::to_string(s), bytes);
    xc_stats st{};
    if (mine.empty()) {
      ck(cudaMemsetAsync(part, 0, bytes, ctx->stream), "memset");
      ck(cudaStreamSynchronize(ctx->stream), "memset");
    } else {
      run_single(ctx, f, mode, d, signal, param, mine.data(), int(mine.size()),
                 (kid_flags & ~XC_FLAG_ASYNC) | (G.rank ? XC_FLAG_NO_INNER_DC : 0u), part, &st,
                 true);
    }
    const NcclApi& a = nccl_or_throw();
    nck(a.Reduce(part, part, bytes / (f64 ? 8 : 4), f64 ? ncclDouble : ncclFloat, ncclSum, 0,
                 G.comms[0], G.comm),
        "ncclReduce");
    if (G.rank == 0) {
      if (accumulate)
        xcb::launch_accumulate(out, part, bytes / (f64 ? 8 : 4), f64 ? 1 : 0, G.comm, lc);
      else
        ck(cudaMemcpyAsync(out, part, bytes, cudaMemcpyDeviceToDevice, G.comm), "D2D");
      ck(cudaGetLastError(), "deliver");
    }
    ck(cudaEventRecord(G.done[s], G.comm), "event");
    st.gpu_launches += lc.n;
    merge_stats(stats, {st}, (long long)ks.size(), since(t_start));
    return;
  }

  if (G.rank_mode) {  // one process per GPU: this rank's bands, then ncclReduce to rank 0
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const std::vector<int> mine = shard_bands(ks, G.rank, G.nranks, pairs);
    void* part = ctx->buf<char>("grp_part", bytes);
    xc_stats st{};
    if (mine.empty())
      ck(cudaMemsetAsync(part, 0, bytes, ctx->stream), "memset");
    else
      run_single(ctx, f, mode, d, signal, param, mine.data(), int(mine.size()),
                 kid_flags | (G.rank ? XC_FLAG_NO_INNER_DC : 0u), part, &st, true);
    const NcclApi& a = nccl_or_throw();
    nck(a.Reduce(part, part, bytes / (f64 ? 8 : 4), f64 ? ncclDouble : ncclFloat, ncclSum, 0,
                 G.comms[0], ctx->stream),
        "ncclReduce");
    ck(cudaStreamSynchronize(ctx->stream), "band reduce");
    if (G.rank == 0) deliver(ctx, *d, part, out, bytes, accumulate, f64, lc);
    st.gpu_launches += lc.n;
    merge_stats(stats, {st}, (long long)ks.size(), since(t_start));
    return;
  }

  const int n = int(G.kids.size());
  std::vector<xc_stats> st(static_cast<size_t>(n));
  if (G.shard == XC_SHARD_BATCH) {  // images split across devices, no collective
    if (accumulate) throw std::invalid_argument("XC_FLAG_ACCUMULATE needs band sharding");
    const int nuse = std::min(n, d->batch);
    st.resize(size_t(nuse));
    for_each_kid(nuse, [&](int i) {
      xc_context k = G.kids[i];
      std::lock_guard<std::mutex> lk(k->mu);
      ck(cudaSetDevice(k->device), "cudaSetDevice");
      const auto ab = shard_range(d->batch, i, nuse);
      xc_image_desc di = *d;
      di.batch = ab.second - ab.first;
      const void *sg, *pr;
      kid_inputs(ctx, k, *d, signal, param, ab.first, ab.second, &sg, &pr);
      char* o = static_cast<char*>(out) + size_t(ab.first) * npix * os;
      const bool local = d->memory == XC_HOST || k->device == ctx->device;
      void* ko = local ? static_cast<void*>(o) : k->buf<char>("grp_part", size_t(di.batch) * npix * os);
      run_single(k, f, mode, &di, sg, pr, components, n_components, kid_flags, ko, &st[i], !local);
      if (!local) {
        ck(cudaMemcpyPeerAsync(o, ctx->device, ko, k->device, size_t(di.batch) * npix * os,
                               k->stream),
           "peer copy out");
        ck(cudaStreamSynchronize(k->stream), "peer copy out");
      }
    });
    merge_stats(stats, st, (long long)ks.size(), since(t_start));
    if (stats) stats->bands_run = st[0].bands_run;  // every device ran all bands
    return;
  }

  // band sharding: every device runs its band range (empty ranges add zeros)
  std::vector<void*> parts(static_cast<size_t>(n), nullptr);
  char* slots = peer_slots(G, "grp_slots", bytes);
  for_each_kid(n, [&](int i) {
    xc_context k = G.kids[i];
    std::lock_guard<std::mutex> lk(k->mu);
    ck(cudaSetDevice(k->device), "cudaSetDevice");
    const std::vector<int> mine = shard_bands(ks, i, n, pairs);
    const bool direct = i == 0 && d->memory == XC_DEVICE && !accumulate;
    void* part = direct             ? out
                 : (slots && i > 0) ? static_cast<void*>(slots + size_t(i - 1) * bytes)
                                    : k->buf<char>("grp_part", bytes);
    parts[i] = part;
    if (mine.empty()) {
      ck(cudaMemsetAsync(part, 0, bytes, k->stream), "memset");
      ck(cudaStreamSynchronize(k->stream), "memset");
      return;
    }
    const void *sg, *pr;
    kid_inputs(ctx, k, *d, signal, param, 0, d->batch, &sg, &pr);
    xc_image_desc di = *d;
    if (sg != signal) di.memory = XC_DEVICE;  // peer-copied inputs
    run_single(k, f, mode, &di, sg, pr, mine.data(), int(mine.size()),
               kid_flags | (i ? XC_FLAG_NO_INNER_DC : 0u), part, &st[i], true);
  });
  if (slots)
    sum_peer_slots(G, parts[0], slots, bytes / (f64 ? 8 : 4), f64, lc);
  else
    reduce_to_root(G, parts, bytes / (f64 ? 8 : 4), f64);
  deliver(G.kids[0], *d, parts[0], out, bytes, accumulate, f64, lc);
  st[0].gpu_launches += lc.n;
  merge_stats(stats, st, (long long)ks.size(), since(t_start));
}

// root: out[img] = floored Re(num / den) for every image of numden (device)
void smooth_divide_all(xc_context ctx, const xc_image_desc& d, const float2* numden, void* out,
                       xc_stats* st) {
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  const size_t npix = size_t(d.height) * d.width, os = dtype_size(d.out_dtype);
  unsigned* red = ctx->buf<unsigned>("smooth_red", size_t(d.batch) + 1);
  ck(cudaMemsetAsync(red, 0, (size_t(d.batch) + 1) * sizeof(unsigned), ctx->stream), "memset");
  char* dst = d.memory == XC_HOST ? ctx->buf<char>("smooth_out", npix * os * size_t(d.batch))
                                  : static_cast<char*>(out);
  xcb::LaunchCounter lc;
  for (int img = 0; img < d.batch; ++img)
    smooth_divide(ctx, ctx->stream, numden, npix, img, d.batch, d.out_dtype == XC_F64,
                  dst + size_t(img) * npix * os, red, lc);
  unsigned clamped = 0;
  ck(cudaMemcpyAsync(&clamped, red + d.batch, sizeof(unsigned), cudaMemcpyDeviceToHost,
                     ctx->stream),
     "readback");
  if (d.memory == XC_HOST)
    ck(cudaMemcpyAsync(out, dst, npix * os * size_t(d.batch), cudaMemcpyDeviceToHost,
                       ctx->stream),
       "D2H");
  ck(cudaStreamSynchronize(ctx->stream), "smooth divide");
  st->clamped_pixels = int(clamped);
  st->gpu_launches += lc.n;
}

void smooth_group(xc_context ctx, xc_filter f, const xc_image_desc* d, const void* signal,
                  const void* param, int normalize_signal, void* out, xc_stats* stats) {
  const auto t_start = std::chrono::steady_clock::now();
  Group& G = *ctx->group;
  const size_t npix = size_t(d->height) * d->width;
  const size_t count = 4 * npix * size_t(d->batch);  // floats of numden
  const std::vector<int>& all = f->hf.ks;
  // num and den are scatters of real fields when the signal is real
  const bool pairs = shard_in_pairs(f, XC_CONVOLUTION, d, all);
  const bool scale = f->hf.group == XC_SCALE2;
  auto no_op = [](Call&, int) {};
  auto part_stats = [](const SmoothPart& p) {
    xc_stats s{};
    s.pad_h = p.pad_h;
    s.pad_w = p.pad_w;
    s.seconds_fft = p.gpu_s;
    s.gpu_launches = p.launches;
    s.bands_run = p.bands_run;
    return s;
  };

  if (G.rank_mode) {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const std::vector<int> mine = shard_bands(all, G.rank, G.nranks, pairs);
    float2* nd = ctx->buf<float2>("grp_numden", count / 2);
    xc_stats st{};
    if (mine.empty())
      ck(cudaMemsetAsync(nd, 0, count * 4, ctx->stream), "memset");
    else
      st = part_stats(smooth_partials(ctx, f, d, signal, param, normalize_signal, mine.data(),
                                      int(mine.size()), scale && G.rank == 0, nd, no_op));
    const NcclApi& a = nccl_or_throw();
    nck(a.Reduce(nd, nd, count, ncclFloat, ncclSum, 0, G.comms[0], ctx->stream), "ncclReduce");
    ck(cudaStreamSynchronize(ctx->stream), "smooth reduce");
    if (G.rank == 0) smooth_divide_all(ctx, *d, nd, out, &st);
    merge_stats(stats, {st}, 2 * (long long)all.size(), since(t_start));
    return;
  }

  const int n = int(G.kids.size());
  std::vector<xc_stats> st(static_cast<size_t>(n));
  if (G.shard == XC_SHARD_BATCH) {
    const int nuse = std::min(n, d->batch);
    st.resize(size_t(nuse));
    for_each_kid(nuse, [&](int i) {
      xc_context k = G.kids[i];
      std::lock_guard<std::mutex> lk(k->mu);
      ck(cudaSetDevice(k->device), "cudaSetDevice");
      const auto ab = shard_range(d->batch, i, nuse);
      xc_image_desc di = *d;
      di.batch = ab.second - ab.first;
      const void *sg, *pr;
      kid_inputs(ctx, k, *d, signal, param, ab.first, ab.second, &sg, &pr);
      const size_t os = dtype_size(d->out_dtype);
      char* o = static_cast<char*>(out) + size_t(ab.first) * npix * os;
      const bool local = d->memory == XC_HOST || k->device == ctx->device;
      if (!local) di.memory = XC_DEVICE;
      void* ko = local ? static_cast<void*>(o) : k->buf<char>("grp_part", size_t(di.batch) * npix * os);
      smooth_single(k, f, &di, sg, pr, normalize_signal, ko, &st[i]);
      if (!local) {
        ck(cudaMemcpyPeerAsync(o, ctx->device, ko, k->device, size_t(di.batch) * npix * os,
                               k->stream),
           "peer copy out");
        ck(cudaStreamSynchronize(k->stream), "peer copy out");
      }
    });
    merge_stats(stats, st, 2 * (long long)all.size(), since(t_start));
    if (stats) stats->bands_run = st[0].bands_run;
    return;
  }

  std::vector<void*> parts(static_cast<size_t>(n), nullptr);
  char* slots = peer_slots(G, "grp_nd_slots", count * 4);
  for_each_kid(n, [&](int i) {
    xc_context k = G.kids[i];
    std::lock_guard<std::mutex> lk(k->mu);
    ck(cudaSetDevice(k->device), "cudaSetDevice");
    const std::vector<int> mine = shard_bands(all, i, n, pairs);
    float2* nd = k->buf<float2>("grp_numden", count / 2);
    parts[i] = nd;
    if (mine.empty()) {
      ck(cudaMemsetAsync(nd, 0, count * 4, k->stream), "memset");
      ck(cudaStreamSynchronize(k->stream), "memset");
      return;
    }
    const void *sg, *pr;
    kid_inputs(ctx, k, *d, signal, param, 0, d->batch, &sg, &pr);
    xc_image_desc di = *d;
    if (sg != signal) di.memory = XC_DEVICE;
    st[i] = part_stats(smooth_partials(k, f, &di, sg, pr, normalize_signal, mine.data(),
                                       int(mine.size()), scale && i == 0, nd, no_op));
  });
  reduce_to_root(G, parts, count, false);
  smooth_divide_all(G.kids[0], *d, static_cast<const float2*>(parts[0]), out, &st[0]);
  merge_stats(stats, st, 2 * (long long)all.size(), since(t_start));
}

}  // namespace

extern "C" {

int xc_nccl_unique_id(void* id_out) {
  return guarded(nullptr, [&] {
    if (!id_out) throw std::invalid_argument("null argument");
    ncclUniqueId id;
    nck(nccl_or_throw().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int xc_context_create_multi(int n_dev, const int* dev_ids, xc_context* out) {
  return guarded(nullptr, [&] {
    if (!out || !dev_ids || n_dev < 1) throw std::invalid_argument("null argument");
    xc_context root = nullptr;
    if (int rc = xc_context_create(dev_ids[0], &root)) throw CudaError(g_thread_err, rc);
    std::unique_ptr<xc_context_s> guard(root);
    auto* G = new Group();
    root->group = G;
    for (int i = 0; i < n_dev; ++i) {
      xc_context k = nullptr;
      if (int rc = xc_context_create(dev_ids[i], &k)) throw CudaError(g_thread_err, rc);
      G->kids.push_back(k);
    }
    bool distinct = true;
    for (int i = 0; i < n_dev; ++i)
      for (int j = 0; j < i; ++j) distinct = distinct && dev_ids[i] != dev_ids[j];
    const char* e = std::getenv("XCB_REDUCE");
    const bool peer = !distinct || (e && std::string(e) == "peer");
    if (!peer) {
      const NcclApi& a = nccl_or_throw();
      G->comms.assign(size_t(n_dev), nullptr);
      nck(a.CommInitAll(G->comms.data(), n_dev, dev_ids), "ncclCommInitAll");
    }
    if (!peer || n_dev > 1) {
      // direct peer access where the topology allows it (NVLink); the peer
      // copies work either way
      for (int i = 0; i < n_dev; ++i)
        for (int j = 0; j < n_dev; ++j) {
          int can = 0;
          if (dev_ids[i] == dev_ids[j]) continue;
          cudaDeviceCanAccessPeer(&can, dev_ids[i], dev_ids[j]);
          if (can) {
            cudaSetDevice(dev_ids[i]);
            cudaDeviceEnablePeerAccess(dev_ids[j], 0);
            cudaGetLastError();  // already enabled is fine
          }
        }
      cudaSetDevice(dev_ids[0]);
    }
    G->peer_write = true;  // kid i stores its partial into kids[0]'s memory
    for (int i = 1; i < n_dev; ++i) {
      int can = dev_ids[i] == dev_ids[0];
      if (!can) cudaDeviceCanAccessPeer(&can, dev_ids[i], dev_ids[0]);
      G->peer_write = G->peer_write && can;
    }
    *out = guard.release();
  });
}

int xc_context_create_rank(int device, const void* nccl_id, int rank, int nranks,
                           xc_context* out) {
  return guarded(nullptr, [&] {
    if (!out || !nccl_id || nranks < 1 || rank < 0 || rank >= nranks)
      throw std::invalid_argument("invalid rank arguments");
    xc_context c = nullptr;
    if (int rc = xc_context_create(device, &c)) throw CudaError(g_thread_err, rc);
    std::unique_ptr<xc_context_s> guard(c);
    auto* G = new Group();
    c->group = G;
    G->rank_mode = true;
    G->rank = rank;
    G->nranks = nranks;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    const NcclApi& a = nccl_or_throw();
    G->comms.assign(1, nullptr);
    ck(cudaSetDevice(device), "cudaSetDevice");
    nck(a.CommInitRank(&G->comms[0], nranks, id, rank), "ncclCommInitRank");
    *out = guard.release();
  });
}

int xc_context_set_sharding(xc_context ctx, int shard) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (shard != XC_SHARD_BANDS && shard != XC_SHARD_BATCH)
      throw std::invalid_argument("unknown sharding");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!ctx->group) throw std::invalid_argument("sharding needs a multi-device context");
    if (ctx->group->rank_mode && shard == XC_SHARD_BATCH)
      throw std::invalid_argument("rank contexts shard bands (split batches per rank instead)");
    ctx->group->shard = shard;
  });
}

int xc_context_synchronize(xc_context ctx) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    if (Group* G = ctx->group) {
      if (G->comm) ck(cudaStreamSynchronize(G->comm), "sync comm");
      for (xc_context k : G->kids) {
        ck(cudaSetDevice(k->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(k->stream), "sync");
      }
      ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    }
  });
}

int xc_context_devices(xc_context ctx, int* n_dev, int* uses_nccl) {
  return guarded(ctx, [&] {
    if (!ctx) throw std::invalid_argument("null context");
    const Group* G = ctx->group;
    if (n_dev) *n_dev = G ? (G->rank_mode ? G->nranks : int(G->kids.size())) : 1;
    if (uses_nccl) *uses_nccl = G && !G->comms.empty() ? 1 : 0;
  });
}

}  // extern "C"
