// FFT planner: factorization into codelet radices, thread count, twiddles.
#include "fft_plan.h"

#include <algorithm>
#include <cmath>
#include <functional>

namespace xcb {

namespace {
// Codelet radices compiled into the device code (fft_core.cuh RADIX_CASES).
const int kRadices[] = {20, 18, 16, 15, 12, 10, 9, 8, 6, 5, 4, 3, 2};

int phys(int n) { return n + (n >> 4); }
}  // namespace

namespace {
bool finalize_plan(int L, const std::vector<int>& order, int nt, bool fast, FftPlan* out) {
  FftPlan p;
  p.fast = fast;
  p.d.L = L;
  // stride per sequence: physical length, congruent to 8 (mod 16) float2 so
  // the two interleaved sequences fall on opposite halves of the banks
  int lp = phys(std::max(L - 1, 0)) + 1;
  while (lp % 16 != 8) ++lp;
  p.d.Lp = lp;
  p.d.npass = L == 1 ? 0 : int(order.size());
  p.d.nt = nt;
  int ns = 1;
  for (int q = 0; q < p.d.npass; ++q) {
    const int R = order[q];
    p.d.radix[q] = R;
    p.d.ns[q] = ns;
    p.d.magic[q] = ns > 1 ? unsigned((0x100000000ull + ns - 1) / ns) : 0u;
    p.d.tw_off[q] = int(p.tw_host.size());
    auto tw = [&](int r, int jm) {
      const long long e = (long long)jm * r % ((long long)ns * R);
      const double a = -2.0 * M_PI * double(e) / double((long long)ns * R);
      return make_float2(float(std::cos(a)), float(std::sin(a)));
    };
    if (q > 0 && !fast) {
      for (int r = 1; r < R; ++r)
        for (int jm = 0; jm < ns; ++jm) p.tw_host.push_back(tw(r, jm));
    } else if (q > 0) {
      // compact table of the fast path (FastFft::load_tw): only the factors
      // W^{jm b} (b < A) and W^{jm A a} that the split product uses, entry-major
      int A = 1;
      while (A * A < R) ++A;
      const int NA = (R + A - 1) / A;
      for (int b = 1; b < A; ++b)
        for (int jm = 0; jm < ns; ++jm) p.tw_host.push_back(tw(b, jm));
      for (int a = 1; a < NA; ++a)
        for (int jm = 0; jm < ns; ++jm) p.tw_host.push_back(tw(A * a, jm));
    }
    ns *= R;
  }
  if (p.tw_host.empty()) p.tw_host.push_back(make_float2(1.f, 0.f));
  p.d.tw = nullptr;
  *out = std::move(p);
  return true;
}
}  // namespace

bool is_smooth235(int n) {
  if (n < 1) return false;
  for (int f : {2, 3, 5})
    while (n % f == 0) n /= f;
  return n == 1;
}

bool make_fft_plan(int L, FftPlan* out) { return make_fft_plan_maxr(L, 20, out); }

bool make_fft_plan_maxr(int L, int max_radix, FftPlan* out) {
  if (!is_smooth235(L) || L > (1 << 15)) return false;
  // enumerate non-increasing radix multisets with product L
  std::vector<std::vector<int>> sets;
  std::vector<int> cur;
  std::function<void(int, int)> dfs = [&](int rem, int start) {
    if (rem == 1) {
      if (!cur.empty()) sets.push_back(cur);
      return;
    }
    if (int(cur.size()) >= kMaxPasses) return;
    for (int i = start; i < int(sizeof(kRadices) / sizeof(int)); ++i) {
      const int r = kRadices[i];
      if (rem % r || r > max_radix) continue;
      cur.push_back(r);
      dfs(rem / r, i);
      cur.pop_back();
    }
  };
  if (L == 1) {
    sets.push_back({1});
  } else {
    dfs(L, 0);
  }
  int best = -1, best_np = 1 << 30, best_min = 0;
  std::vector<int> best_order;
  for (int s = 0; s < int(sets.size()); ++s) {
    std::vector<int> rs = sets[s];
    std::sort(rs.begin(), rs.end());
    const int np = int(rs.size());
    // fewest passes (smem round trips), then the largest smallest radix
    if (np < best_np || (np == best_np && rs[0] > best_min)) {
      best = s;
      best_np = np;
      best_min = rs[0];
      best_order = rs;
    }
  }
  // larger radices first: the smallest (most butterflies) runs last
  std::sort(best_order.begin(), best_order.end(), std::greater<int>());
  int best_nt = 32;
  if (best >= 0) {
    int items = 1;
    for (int r : best_order) items = std::max(items, kG * L / r);
    best_nt = std::min(kMaxThreads, std::max(32, (items + 31) / 32 * 32));
  }
  if (best < 0) return false;
  return finalize_plan(L, best_order, best_nt, false, out);
}

bool make_fast_plan(int L, FftPlan* out) {
  std::vector<int> order;
#define XCB_FAST_ORDER(LL, R0, R1, RL)  \
  if (L == LL) {                        \
    order.push_back(R0);                \
    if (R1 > 1) order.push_back(R1);    \
    order.push_back(RL);                \
  }
  XCB_FAST_TABLE(XCB_FAST_ORDER)
#undef XCB_FAST_ORDER
  if (order.empty()) return false;
  int need = kG * L / order.back();
  for (size_t q = 1; q < order.size(); ++q) need = std::max(need, kG * L / order[q]);
  const int nt = std::max(64, (need + 31) / 32 * 32);
  if (nt > kFastMaxThreads) return false;
  return finalize_plan(L, order, nt, true, out);
}

int pick_fft_length(int n) {
  n = std::max(n, 1);
  for (int s = n;; ++s) {
    if (!is_smooth235(s)) continue;
    FftPlan p;
    if (make_fft_plan(s, &p)) return s;
    if (s > (1 << 15)) return -1;
  }
}

}  // namespace xcb
