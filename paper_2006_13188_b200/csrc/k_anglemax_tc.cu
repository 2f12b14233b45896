// Per-pixel 360-angle maximum on the 5th-
// generation tensor cores, for the Hermitian half-band planes (real signal,
// real template): with G_k the band responses k = 0..KH (KH <= 16),
//
//   S(n) = G_0 + 2 Re sum_{k>=1} G_k w^{kn},  w = e^{-2 pi i / 360},
//   score = max_n |S(n)|, argmax = the first n attaining it (n = 0..359).
//
// The sum splits by the parity of k: E(n) (the even k >= 2) has period 180
// and O(n) (odd k) is anti-periodic, so S(n) = G_0 + E(n) + O(n) and
// S(n + 180) = G_0 + E(n) - O(n) for n < 180.  E and O over n < 192 (180
// used) are two real GEMMs per tile of 128 pixels:
//
//   E[p][n] = sum_kk AE[p][kk] BE[n][kk]   (kk: Re/Im G_2, G_4, ..., G_16;
//                                           BE = 2 cos(k t_n), 2 sin(k t_n))
//   O[p][n] = sum_kk AO[p][kk] BO[n][kk]   (Re/Im G_1, G_3, ..., G_15)
//
// M = 128, N = 192, K = 16 each, kind::tf32 with fp32 accumulators in TMEM
// (384 of the 512 columns).  fp32 accuracy from 3xTF32: A = Ah + Al,
// B = Bh + Bl (tf32 hi parts and their fp32 residuals), D = Al Bh + Ah Bl +
// Ah Bh (the dropped Al Bl is ~2^-22 of each product): 12 MMAs per tile, the
// E and O chains interleaved.  Operands are K-major with the 64-byte
// hardware swizzle (rows of 16 tf32).
//
// One persistent CTA per SM, 256 threads: threads 0..127 convert a pixel's E
// coefficients (and keep G_0), 128..255 its O coefficients; one thread issues
// the MMAs (tcgen05.mma, committed to an mbarrier); all 8 warps run the
// epilogue (tcgen05.ld of the warp's lane quadrant, warps w and w + 4 taking
// the two halves of the 192 columns).  Two smem A buffers: the next tile's
// coefficients are loaded during the epilogue and stored before the MMAs of
// the next tile are issued.
//
// Measured variants (config 3, 4096^2, 17 bands; DESIGN 5): the CUDA-core
// kernel k_anglemax_herm 2.71 ms (issue-bound at 83%); G_0 inside E (K = 24,
// 15 MMAs) 2.13 ms; two 96-angle chunks with double-buffered TMEM 3.4 ms; an
// fp16 3-way split with per-row power-of-two scaling, TMA-staged bands and 16
// warps 3.2 ms; 16 epilogue warps no gain.  The epilogue alone is bound by
// TMEM reads (the 360 fp32 values of every pixel at ~80 B/cycle/SM, ~1.1 ms)
// and a second accumulator set to hide the MMAs behind it does not fit
// (2 x 384 > 512 columns).
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "stages_common.cuh"
#include "tmem.cuh"

namespace xcb {
namespace {

constexpr int kTM = 128;     // pixels per tile (MMA M)
constexpr int kNT = 192;     // angles n per tile (MMA N; 180 used)
constexpr int kNH = 180;     // angles of E / O (the other 180 are E - O)
constexpr int kK = 16;       // coefficients of E and of O
constexpr int kThreads = 256;
// smem (bytes): K-major, SWIZZLE_64B: 8-row atoms of 64-byte rows, the
// 16-byte chunk index of an element XORed with (row % 8) / 2
constexpr uint32_t kSbo = 512;                         // 8-row group stride
constexpr uint32_t kA = kTM * 64, kB = kNT * 64;       // 8192, 12288 per matrix
constexpr uint32_t kOffB = 0;                          // E hi, E lo, O hi, O lo
constexpr uint32_t kOffA = 4 * kB;                     // 2 buffers x (E hi, lo, O hi, lo)
constexpr uint32_t kSmem = kOffA + 2 * 4 * kA + 1024;  // + alignment slack
constexpr uint32_t kTmemCols = 512;                    // E 192 + O 192
constexpr uint64_t kSw64 = 4;                          // descriptor layout type
// instruction descriptor: fp32 accumulate, tf32 A and B, both K-major
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kNT >> 3) << 17) |
                            (uint32_t(kTM >> 4) << 24);

struct PlaneMap {
  int idx[17];  // plane index of band k = 0..16, or -1
};

__device__ __forceinline__ uint32_t kmaj(int r, int kk) {
  return uint32_t(r >> 3) * kSbo + uint32_t(r & 7) * 64u +
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
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) |
         (uint64_t((kSbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46) | (kSw64 << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
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

// the 12 MMAs of one tile (A buffer at sbase + kOffA + abuf): E into TMEM
// columns dcol.., O into dcol + 192..; per K step of 8 the products Al Bh,
// Ah Bl, Ah Bh, alternating between the two accumulators
__device__ __forceinline__ void issue_tile(uint32_t sbase, uint32_t abuf, uint32_t dcol) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const int ks = i / 3, prod = i % 3;
      const uint32_t ah = sbase + kOffA + abuf + uint32_t(part) * 2 * kA, al = ah + kA;
      const uint32_t bh = sbase + kOffB + uint32_t(part) * 2 * kB, bl = bh + kB;
      const uint32_t o = uint32_t(ks) * 32u;
      mma_tf32(dcol + uint32_t(part) * kNT, umma_desc((prod == 0 ? al : ah) + o),
               umma_desc((prod == 1 ? bl : bh) + o), i > 0);
    }
  }
}

template <class TO>
__global__ void __launch_bounds__(kThreads, 1)
    k_anglemax_tc(const float2* __restrict__ planes, PlaneMap m, size_t npix,
                  TO* __restrict__ score, int* __restrict__ argmax) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ float g0buf[2][kTM];  // G_0 of the pixels of each A buffer
  __shared__ float mrg_v[2][2][kTM];  // [tile parity][s | d][pixel]
  __shared__ int mrg_j[2][2][kTM];
  const int t = threadIdx.x, warp = t >> 5;
  const uint32_t sraw = smem_u32(sm), sbase = (sraw + 1023u) & ~1023u;  // swizzle atoms
  unsigned char* const sa = sm + (sbase - sraw);
  const size_t ntiles = (npix + kTM - 1) / kTM;
  if (blockIdx.x >= ntiles) return;

  if (warp == 0) tmem_alloc(&tbase, kTmemCols);
  if (t == 32) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // B: rows n < 180 hold 2 cos(k t_n), 2 sin(k t_n) (E: k = 2, 4, ..., 16;
  // O: k = 1, 3, ..., 15); rows 180..191 zero
  for (int i = t; i < 2 * kNT * kK; i += kThreads) {
    const int part = i / (kNT * kK), j = i % (kNT * kK), n = j / kK, kk = j % kK;
    const int k = 2 * (kk / 2) + (part == 0 ? 2 : 1);
    double v = 0.0;
    if (n < kNH) {
      double sn, cs;
      sincospi(2.0 * double(k * n) / 360.0, &sn, &cs);
      v = 2.0 * ((kk & 1) ? sn : cs);
    }
    const float f = float(v), hi = tf32_hi(f);
    unsigned char* bp = sa + kOffB + uint32_t(part) * 2 * kB + kmaj(n, kk);
    *reinterpret_cast<float*>(bp) = hi;
    *reinterpret_cast<float*>(bp + kB) = f - hi;
  }

  // threads 0..127 convert a pixel's E coefficients (planes k = 2, 4, ..., 16)
  // and G_0, threads 128..255 its O coefficients (k = 1, 3, ..., 15)
  const int row = t & (kTM - 1), part = t >> 7;
  float2 g[8];
  float g0 = 0.f;
  auto load_tile = [&](size_t tl) {
    const size_t p = tl * kTM + row;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int pi = m.idx[2 * i + (part == 0 ? 2 : 1)];
      g[i] = (pi >= 0 && p < npix) ? __ldg(planes + size_t(pi) * npix + p) : make_float2(0.f, 0.f);
    }
    g0 = (part == 0 && m.idx[0] >= 0 && p < npix) ? __ldg(planes + size_t(m.idx[0]) * npix + p).x
                                                   : 0.f;
  };
  auto store_tile = [&](int ab) {
    unsigned char* hi = sa + kOffA + uint32_t(ab) * 4 * kA + uint32_t(part) * 2 * kA;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float v[4] = {g[2 * c].x, g[2 * c].y, g[2 * c + 1].x, g[2 * c + 1].y};
      float4 h4, l4;
      h4.x = tf32_hi(v[0]);
      h4.y = tf32_hi(v[1]);
      h4.z = tf32_hi(v[2]);
      h4.w = tf32_hi(v[3]);
      l4 = make_float4(v[0] - h4.x, v[1] - h4.y, v[2] - h4.z, v[3] - h4.w);
      const uint32_t off = kmaj(row, 4 * c);
      *reinterpret_cast<float4*>(hi + off) = h4;
      *reinterpret_cast<float4*>(hi + kA + off) = l4;
    }
    if (part == 0) g0buf[ab][row] = g0;
  };

  size_t tile = blockIdx.x;
  load_tile(tile);
  store_tile(0);
  fence_proxy_async();
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tb = tbase;
  if (t == 0) {
    issue_tile(sbase, 0, tb);
    mma_commit(&bar);
  }
  // epilogue geometry: lane quadrant warp % 4 (pixel rows), column half warp / 4
  const int half = warp >> 2;
  const uint32_t tq = tb + ((32u * uint32_t(warp & 3)) << 16) + uint32_t(half) * (kNT / 2);
  const int prow = 32 * (warp & 3) + (t & 31);
  const int n0 = half * (kNT / 2);
  for (unsigned it = 0;; ++it) {
    const size_t next = tile + gridDim.x;
    const bool has_next = next < ntiles;
    if (has_next) load_tile(next);  // in flight during the epilogue
    const float gz = g0buf[it & 1][prow];
    float bs = -1.f, bd = -1.f;
    int as = 0, ad = 0;
    mbar_wait_bounded(&bar, it & 1);
    tmem_fence_after_sync();
#pragma unroll
    for (int q = 0; q < kNT / 2; q += 16) {
      if (n0 + q >= kNH) break;  // warp-uniform
      float e[16], o[16];
      tmem_ld16(tq + q, e);
      tmem_ld16(tq + kNT + q, o);
      tmem_wait_ld();
      tmem_depn<16>(e);
      tmem_depn<16>(o);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int n = n0 + q + i;
        if (n >= kNH) break;
        const float ee = e[i] + gz;
        const float s = fabsf(ee + o[i]), d = fabsf(ee - o[i]);
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
    if (has_next) {
      store_tile((it + 1) & 1);
      fence_proxy_async();
    }
    const int mp = it & 1;  // by parity: the next tile posts while this merge may still read
    if (half) {
      mrg_v[mp][0][prow] = bs;
      mrg_j[mp][0][prow] = as;
      mrg_v[mp][1][prow] = bd;
      mrg_j[mp][1][prow] = ad;
    }
    tmem_fence_before_sync();
    __syncthreads();  // TMEM drained, the next A tile stored, the halves posted
    if (t == 0 && has_next) {
      tmem_fence_after_sync();
      issue_tile(sbase, uint32_t((it + 1) & 1) * 4 * kA, tb);
      mma_commit(&bar);
    }
    // merge the two column halves of each pixel: the first maximum in scan
    // order n = 0..359 (ties: the smaller n; every s index precedes every d)
    if (!half) {
      const float vs = mrg_v[mp][0][prow], vd = mrg_v[mp][1][prow];
      const int js = mrg_j[mp][0][prow], jd = mrg_j[mp][1][prow];
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
  const size_t ntiles = (npix + kTM - 1) / kTM;
  const int grid = int(ntiles < size_t(sms) ? ntiles : size_t(sms));
  if (score_f64) {
    set_smem(k_anglemax_tc<double>, kSmem);
    k_anglemax_tc<double><<<grid, kThreads, kSmem, st>>>(planes, m, npix,
                                                         static_cast<double*>(score), argmax);
  } else {
    set_smem(k_anglemax_tc<float>, kSmem);
    k_anglemax_tc<float><<<grid, kThreads, kSmem, st>>>(planes, m, npix,
                                                        static_cast<float*>(score), argmax);
  }
  ++lc.n;
}

}  // namespace xcb
