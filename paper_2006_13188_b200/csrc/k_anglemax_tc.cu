// Per-pixel 360-angle maximum on the 5th-
// generation tensor cores, for the Hermitian half-band planes (real signal,
// real template): with G_k the band responses k = 0..KH (KH <= 16),
//
//   S(n) = G_0 + 2 Re sum_{k>=1} G_k w^{kn},  w = e^{-2 pi i / 360},
//   score = max_n |S(n)|, argmax = the first n attaining it (n = 0..359).
//
// The sum splits by the parity of k: E(n) (G_0 and the even k) has period 180
// and O(n) (odd k) is anti-periodic, so S(n) = E(n) + O(n) and
// S(n + 180) = E(n) - O(n) for n < 180.  E and O over n < 180 are two real
// GEMMs per tile of 128 pixels:
//
//   E[p][n] = sum_kk AE[p][kk] BE[n][kk]   (kk: G_0.re, then Re/Im G_2..G_16;
//                                           BE = 1, 2 cos(k t_n), 2 sin(k t_n))
//   O[p][n] = sum_kk AO[p][kk] BO[n][kk]   (Re/Im G_1..G_15)
//
// K = 24 (17 used) and 16, N = 192 (180 used) in two chunks of 96, M = 128,
// kind::tf32 with fp32 accumulators in TMEM.  fp32 accuracy from 3xTF32:
// A = Ah + Al, B = Bh + Bl (tf32 hi parts and their fp32 residuals),
// D = Al Bh + Ah Bl + Ah Bh (the dropped Al Bl is ~2^-22 of each product).
//
// One persistent CTA per SM, 256 threads: every thread converts (one pixel's
// E or O coefficients), one thread issues the MMAs (tcgen05.mma, committed to
// an mbarrier), and all 8 warps run the epilogue (tcgen05.ld of the warp's
// lane quadrant; warps w and w + 4 take the two halves of a chunk's columns).
// Two TMEM accumulator buffers (one per chunk) and two smem A buffers: the
// MMAs of chunk c + 1 run while the epilogue of chunk c reads TMEM, and the
// global loads of the next tile are in flight during both.
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "stages_common.cuh"
#include "tmem.cuh"

namespace xcb {
namespace {

constexpr int kTM = 128;     // pixels per tile (MMA M)
constexpr int kNT = 192;     // angles n per tile (180 used), in chunks of NC (MMA N)
constexpr int kNH = 180;     // angles n of E / O (the other 180 are E - O)
constexpr int kKE = 24, kKO = 16;
constexpr int kThreads = 256;
// smem (bytes), K-major with the hardware swizzles (conflict-free tensor-core
// reads; the interleaved no-swizzle layout measured ~45 B/cycle): E rows are
// 128 B (SWIZZLE_128B atom 8 rows x 128 B, K padded to 32), O rows 64 B
// (SWIZZLE_64B atom 8 x 64 B).  The 16-byte chunk index of an element is
// XORed with the row's position in its atom (128B: r % 8; 64B: (r % 8) / 2).
constexpr uint32_t kSboE = 1024, kSboO = 512;                  // 8-row group strides
constexpr uint32_t kAE = kTM * 128, kAO = kTM * 64;            // 16384, 8192
constexpr uint32_t kBE = kNT * 128, kBO = kNT * 64;            // 24576, 12288
constexpr uint32_t kABuf = 2 * kAE + 2 * kAO;                  // hi, lo of E, O
constexpr uint32_t kOffBEh = 0, kOffBEl = kBE, kOffBOh = 2 * kBE, kOffBOl = 2 * kBE + kBO;
constexpr uint32_t kOffA = 2 * kBE + 2 * kBO;                  // two A buffers follow
constexpr uint32_t kSmem = kOffA + 2 * kABuf + 1024;           // + alignment slack
constexpr uint32_t kTmemCols = 512;  // NC = 96: 2 buffers x (E 96 + O 96); 192: 1 x 384
constexpr uint64_t kSw128 = 2, kSw64 = 4;                      // descriptor layout types

struct PlaneMap {
  int idx[17];  // plane index of band k = 0..16, or -1
};

__device__ __forceinline__ uint32_t kmaj_e(int r, int kk) {
  return uint32_t(r >> 3) * kSboE + uint32_t(r & 7) * 128u +
         (uint32_t((kk >> 2) ^ (r & 7)) << 4) + uint32_t(kk & 3) * 4u;
}
__device__ __forceinline__ uint32_t kmaj_o(int r, int kk) {
  return uint32_t(r >> 3) * kSboO + uint32_t(r & 7) * 64u +
         (uint32_t((kk >> 2) ^ ((r & 7) >> 1)) << 4) + uint32_t(kk & 3) * 4u;
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// K-major swizzled shared-memory matrix descriptor (sm_100 layout: start >> 4
// [0,14), LBO >> 4 [16,30) (unused for swizzled K-major: 1), SBO >> 4 [32,46),
// version 1 [46,48), layout type [61,64)); a K step of 8 tf32 moves the start
// 32 bytes along the swizzled row
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t sbo, uint64_t layout) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46) | (layout << 61);
}

// instruction descriptor: fp32 accumulate, tf32 A and B, both K-major
template <int NC>
constexpr uint32_t idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(NC >> 3) << 17) |
         (uint32_t(kTM >> 4) << 24);
}

template <int NC>
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc<NC>()), "r"(acc)
      : "memory");
}

// mbarrier wait that traps instead of spinning forever (a lost MMA commit
// surfaces as a launch error, not a hung GPU)
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, unsigned phase) {
  for (unsigned spins = 0;; ++spins) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (done) return;
    if (spins > (1u << 24)) __trap();
  }
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// one chunk (angles [NC h, NC h + NC)) of one tile: 3xTF32 over the K steps of
// E and O into TMEM columns dcol (E) and dcol + NC (O).  IL interleaves the E
// and O MMAs (two independent accumulator chains) instead of E then O.
template <int NC, bool IL>
__device__ __forceinline__ void issue_chunk(uint32_t sbase, uint32_t abuf, int h, uint32_t dcol) {
  const uint32_t ae = sbase + abuf, ao = ae + 2 * kAE;
  auto step = [&](int part, int ks, int prod) {
    const uint32_t sbo = part == 0 ? kSboE : kSboO;
    const uint32_t ah = part == 0 ? ae : ao, al = ah + (part == 0 ? kAE : kAO);
    const uint32_t bh = sbase + (part == 0 ? kOffBEh : kOffBOh) + uint32_t(h) * (NC / 8) * sbo;
    const uint32_t bl = bh + (part == 0 ? kBE : kBO);
    const uint32_t d = dcol + uint32_t(part) * NC;
    const uint32_t o = uint32_t(ks) * 32u;  // 8 tf32 along the swizzled row
    const uint32_t a = prod == 0 ? al : ah, b = prod == 1 ? bl : bh;
    const uint64_t lt = part == 0 ? kSw128 : kSw64;
    mma_tf32<NC>(d, umma_desc(a + o, sbo, lt), umma_desc(b + o, sbo, lt), ks > 0 || prod > 0);
  };
  if (IL) {
#pragma unroll
    for (int i = 0; i < 3 * (kKE / 8); ++i) {
      step(0, i / 3, i % 3);
      if (i < 3 * (kKO / 8)) step(1, i / 3, i % 3);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 3 * (kKE / 8); ++i) step(0, i / 3, i % 3);
#pragma unroll
    for (int i = 0; i < 3 * (kKO / 8); ++i) step(1, i / 3, i % 3);
  }
}

template <class TO, int NC, bool IL>
__global__ void __launch_bounds__(kThreads, 1)
    k_anglemax_tc(const float2* __restrict__ planes, PlaneMap m, size_t npix,
                  TO* __restrict__ score, int* __restrict__ argmax, int probe) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tbase;
  __shared__ float mrg_v[2][kTM];
  __shared__ int mrg_j[2][kTM];
  const int t = threadIdx.x, warp = t >> 5;
  const uint32_t sraw = smem_u32(sm), sbase = (sraw + 1023u) & ~1023u;  // swizzle atoms
  unsigned char* const sa = sm + (sbase - sraw);
  const size_t ntiles = (npix + kTM - 1) / kTM;
  if (blockIdx.x >= ntiles) return;

  if (warp == 0) tmem_alloc(&tbase, kTmemCols);
  if (t == 32) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  // B (every chunk): rows n < 180 hold the trig table, rows 180..191 zero
  for (int i = t; i < kNT * (kKE + kKO); i += kThreads) {
    const bool e = i < kNT * kKE;
    const int j = e ? i : i - kNT * kKE, K = e ? kKE : kKO;
    const int n = j / K, kk = j % K;
    double v = 0.0;
    if (n < kNH) {
      int k = -1, im = 0;
      if (e) {
        if (kk == 0) v = 1.0;
        else if (kk <= 16) k = 2 * ((kk - 1) / 2 + 1), im = (kk - 1) & 1;
      } else {
        k = 2 * (kk / 2) + 1, im = kk & 1;
      }
      if (k >= 0) {
        double sn, cs;
        sincospi(2.0 * double(k * n) / 360.0, &sn, &cs);
        v = 2.0 * (im ? sn : cs);
      }
    }
    const float f = float(v), hi = tf32_hi(f);
    const uint32_t off = e ? kmaj_e(n, kk) : kmaj_o(n, kk);
    *reinterpret_cast<float*>(sa + (e ? kOffBEh : kOffBOh) + off) = hi;
    *reinterpret_cast<float*>(sa + (e ? kOffBEl : kOffBOl) + off) = f - hi;
  }

  // this thread's pixel row and coefficient set: threads < 128 convert E
  // (planes k = 0, 2, ..., 16: 9 loads), the others O (k = 1, 3, ..., 15: 8)
  const int row = t & (kTM - 1);
  const bool isE = t < kTM;
  float2 g[9];
  auto load_tile = [&](size_t tile) {
    const size_t p = tile * kTM + row;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = isE ? 2 * i : 2 * i + 1;
      const int pi = (k <= 16 && (isE || i < 8)) ? m.idx[k] : -1;
      g[i] = (pi >= 0 && p < npix) ? __ldg(planes + size_t(pi) * npix + p) : make_float2(0.f, 0.f);
    }
  };
  auto store_tile = [&](uint32_t abuf) {
    float v[kKE];
    if (isE) {
      v[0] = g[0].x;
#pragma unroll
      for (int i = 1; i <= 8; ++i) {
        v[2 * i - 1] = g[i].x;
        v[2 * i] = g[i].y;
      }
#pragma unroll
      for (int i = 17; i < kKE; ++i) v[i] = 0.f;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[2 * i] = g[i].x;
        v[2 * i + 1] = g[i].y;
      }
    }
    const int K = isE ? kKE : kKO;
    unsigned char* hi = sa + kOffA + abuf + (isE ? 0 : 2 * kAE);
    unsigned char* lo = hi + (isE ? kAE : kAO);
#pragma unroll
    for (int c = 0; c < kKE / 4; ++c) {
      if (4 * c >= K) break;
      float4 h4, l4;
      h4.x = tf32_hi(v[4 * c]);
      h4.y = tf32_hi(v[4 * c + 1]);
      h4.z = tf32_hi(v[4 * c + 2]);
      h4.w = tf32_hi(v[4 * c + 3]);
      l4 = make_float4(v[4 * c] - h4.x, v[4 * c + 1] - h4.y, v[4 * c + 2] - h4.z,
                       v[4 * c + 3] - h4.w);
      const uint32_t off = isE ? kmaj_e(row, 4 * c) : kmaj_o(row, 4 * c);
      *reinterpret_cast<float4*>(hi + off) = h4;
      *reinterpret_cast<float4*>(lo + off) = l4;
    }
  };

  size_t tile = blockIdx.x;
  load_tile(tile);
  store_tile(0);
  fence_proxy_async();
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tb = tbase;
  constexpr int NCH = kNT / NC;  // chunks per tile (= TMEM buffers)
  if (t == 0 && !(probe & 4)) {
#pragma unroll
    for (int h = 0; h < NCH; ++h) {
      issue_chunk<NC, IL>(sbase, kOffA, h, tb + uint32_t(h) * 2 * NC);
      mma_commit(&bar[h]);
    }
  }
  // epilogue geometry: lane quadrant warp % 4 (pixel rows), column half warp / 4
  const int half = warp >> 2;
  const uint32_t tq = tb + ((32u * uint32_t(warp & 3)) << 16);
  const int prow = 32 * (warp & 3) + (t & 31);
  unsigned it = 0;
  for (;; ++it) {
    const size_t next = tile + gridDim.x;
    const bool has_next = next < ntiles;
    if (has_next && !(probe & 2)) load_tile(next);
    float bs = -1.f, bd = -1.f;
    int as = 0, ad = 0;
#pragma unroll 1
    for (int h = 0; h < NCH; ++h) {
      if (!(probe & 4)) mbar_wait_bounded(&bar[h], it & 1);
      tmem_fence_after_sync();
      const uint32_t ce = tq + uint32_t(h) * 2 * NC + uint32_t(half) * (NC / 2);
      const int n0 = h * NC + half * (NC / 2);
#pragma unroll
      for (int q = 0; q < NC / 2; q += 16) {
        if (n0 + q >= kNH || (probe & 1)) break;  // warp-uniform
        float e[16], o[16];
        tmem_ld16(ce + q, e);
        tmem_ld16(ce + NC + q, o);
        tmem_wait_ld();
        tmem_depn<16>(e);
        tmem_depn<16>(o);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + q + i;
          if (n >= kNH) break;
          const float s = fabsf(e[i] + o[i]), d = fabsf(e[i] - o[i]);
          if (s > bs) {
            bs = s;
            as = n;
          }
          if (d > bd) {
            bd = d;
            ad = n + kNH;
          }
        }
      }
      if (h == 0 && has_next) {
        if (!(probe & 2)) store_tile((it + 1) & 1 ? kABuf : 0);
        fence_proxy_async();
      }
      tmem_fence_before_sync();
      __syncthreads();  // TMEM buffer h drained (and the next A tile stored)
      if (t == 0 && has_next && !(probe & 4)) {
        tmem_fence_after_sync();
        issue_chunk<NC, IL>(sbase, kOffA + ((it + 1) & 1 ? kABuf : 0), h,
                            tb + uint32_t(h) * 2 * NC);
        mma_commit(&bar[h]);
      }
    }
    // merge the two column halves of each pixel: the first maximum in scan
    // order n = 0..359 (ties: the smaller n; every s index precedes every d)
    if (half) {
      mrg_v[0][prow] = bs;
      mrg_j[0][prow] = as;
      mrg_v[1][prow] = bd;
      mrg_j[1][prow] = ad;
    }
    __syncthreads();
    if (!half) {
      const float vs = mrg_v[0][prow], vd = mrg_v[1][prow];
      const int js = mrg_j[0][prow], jd = mrg_j[1][prow];
      if (vs > bs || (vs == bs && js < as)) bs = vs, as = js;
      if (vd > bd || (vd == bd && jd < ad)) bd = vd, ad = jd;
      const float best = bd > bs ? bd : bs;
      const int arg = bd > bs ? ad : as;
      const size_t p = tile * kTM + prow;
      if (p < npix) {
        score[p] = TO(best);
        if (argmax) argmax[p] = arg;
      }
    }
    if (!has_next) break;
    tile = next;
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after_sync();
    tmem_dealloc(tb, kTmemCols);
  }
}

}  // namespace

bool anglemax_tc_ok(int kh) { return kh <= 16; }

void launch_anglemax_tc(const float2* planes, const int* ks_host, int nb, size_t npix,
                        int score_f64, void* score, int* argmax, cudaStream_t st,
                        LaunchCounter& lc) {
  PlaneMap m;
  for (int k = 0; k <= 16; ++k) m.idx[k] = -1;
  for (int i = 0; i < nb; ++i)
    if (ks_host[i] >= 0 && ks_host[i] <= 16) m.idx[ks_host[i]] = i;
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  // XCB_TC_PROBE (timing only, results wrong): bit 0 skips the epilogue math,
  // bit 1 the A-tile loads and stores, bit 2 the MMAs and their waits
  static const int probe = [] {
    const char* e = std::getenv("XCB_TC_PROBE");
    return e ? std::atoi(e) : 0;
  }();
  static const int variant = [] {  // XCB_TC_VARIANT (A/B): 0 N=96, 1 N=96 IL, 2 N=192 IL
    const char* e = std::getenv("XCB_TC_VARIANT");
    return e ? std::atoi(e) : 2;
  }();
  const size_t ntiles = (npix + kTM - 1) / kTM;
  const int grid = int(ntiles < size_t(sms) ? ntiles : size_t(sms));
  auto go = [&](auto kern, auto* out) {
    set_smem(kern, kSmem);
    kern<<<grid, kThreads, kSmem, st>>>(planes, m, npix, out, argmax, probe);
  };
  if (score_f64) {
    double* o = static_cast<double*>(score);
    if (variant == 0) go(k_anglemax_tc<double, 96, false>, o);
    else if (variant == 2) go(k_anglemax_tc<double, 192, true>, o);
    else go(k_anglemax_tc<double, 96, true>, o);
  } else {
    float* o = static_cast<float*>(score);
    if (variant == 0) go(k_anglemax_tc<float, 96, false>, o);
    else if (variant == 2) go(k_anglemax_tc<float, 192, true>, o);
    else go(k_anglemax_tc<float, 96, true>, o);
  }
  ++lc.n;
}

}  // namespace xcb
