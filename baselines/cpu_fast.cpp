// cpu_fast.cpp — an OPTIMIZED multithreaded CPU implementation of the same hot path
// (Past-Future scheduler, arXiv 2507.10150), used only as a fairer CPU comparator in
// bench.py next to the oracle-based `cpu_baseline` (the oracle re-runs the
// tick-stepped M* from scratch per queued candidate, so a GPU/oracle ratio overstates
// the speed-up). It is neither the oracle nor the product: it shares no code with
// oracle/ or paper_2507_10150_b200/csrc/, and tests/test_cpu_fast.py checks it against
// the oracle.
//
// Per distribution (an instance window, or a shared group's window = its shard rows):
// C[l] = #{h ≤ l} and the sorted window S (Eq.(eq:5)).
// Per instance: l̂ = min(S[C[l_t] + ⌊u·(w − C[l_t]) / 2^32⌋], max_new), l̂ = max_new when
// C[l_t] = w (Alg.1 l.3-9, readings C-3..C-6, C-8 hash for u); M* by the sort form of
// Eq.(eq:1)-(eq:3) (entries sorted by r descending once, max_i A_i + r_i·i); p* by a
// binary search over the prefix length p (M* is monotone in p), each probe one pass
// over the sorted entries (Alg.1 l.7-14 with the '≤' of PAPER.md:226 and the reserved
// ratio C-13). std::thread over instances.
//
// Build: g++ -O3 -std=c++17 -fPIC -shared -pthread cpu_fast.cpp -o libcpufast.so
#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

uint64_t splitmix_final(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  return x ^ (x >> 16);
}

struct Dist {
  std::vector<int32_t> C;  // [Lmax+1]
  std::vector<int32_t> S;  // [w + 1], S[w] = sentinel (never used: n_gt = 0 -> max_new)
  int32_t w = 0;
};

struct Entry {
  int32_t r, a, j;  // j = 0 running, 1..q queue position
};

}  // namespace

extern "C" int pfc_admit(int32_t n, const int32_t* dist_of, const int64_t* inst_id, const int32_t* run_off,
                         const int32_t* input_len, const int32_t* generated, const int32_t* q_off,
                         const int32_t* q_input_len, const int32_t* max_new, const int32_t* capacity,
                         int32_t window, int32_t max_len, const int32_t* dist_rows, int32_t mode,
                         uint32_t quantile_u, int32_t reserved_bp, uint64_t seed, uint32_t tick,
                         int32_t n_threads, int32_t* admitted_out, int32_t* peak_out,
                         int32_t* peak_running_out) {
  const int nb = max_len + 1;
  // distribution d = row d of dist_rows [* × window] (any order); rebuilt when the next
  // instance uses another one (shared groups are group-major: one build per group and thread)
  auto build = [&](int32_t d, Dist& D) {
    D.S.assign(dist_rows + (int64_t)d * window, dist_rows + (int64_t)(d + 1) * window);
    std::sort(D.S.begin(), D.S.end());
    D.w = window;
    D.C.assign(nb, 0);
    for (int32_t v : D.S) ++D.C[v];
    for (int l = 1; l < nb; ++l) D.C[l] += D.C[l - 1];
    D.S.push_back(0x7FFFFFFF);
  };
  const uint64_t tick_mix = (uint64_t)tick * 0xD1B54A32D192ED03ULL;
  auto work = [&](int32_t i0, int32_t i1) {
    std::vector<Entry> e;
    Dist D;
    int32_t cur = -1;
    for (int32_t i = i0; i < i1; ++i) {
      if (dist_of[i] != cur) build(cur = dist_of[i], D);
      const int32_t r0 = run_off[i], k = run_off[i + 1] - r0;
      const int32_t qq0 = q_off[i], q = q_off[i + 1] - qq0;
      const int32_t mx = max_new[i];
      const uint64_t K = splitmix_final(seed ^ tick_mix ^ ((uint64_t)inst_id[i] * 0x9E3779B97F4A7C15ULL));
      const uint32_t fold = (uint32_t)K ^ (uint32_t)(K >> 32);
      auto predict = [&](int32_t l_t, int32_t slot) -> int32_t {
        const uint32_t u = mode ? quantile_u : hash32(fold ^ ((uint32_t)slot * 0x9E3779B9U));
        const int32_t base = D.C[l_t], n_gt = D.w - base;
        if (n_gt == 0) return mx;
        const int32_t lh = D.S[base + (int32_t)(((uint64_t)u * (uint32_t)n_gt) >> 32)];
        return std::min(lh, mx);
      };
      e.clear();
      for (int32_t s = 0; s < k; ++s) {
        const int32_t lt = generated[r0 + s];
        e.push_back({predict(lt, s) - lt, input_len[r0 + s] + lt, 0});
      }
      for (int32_t j = 0; j < q; ++j) e.push_back({predict(0, k + j), q_input_len[qq0 + j], j + 1});
      std::sort(e.begin(), e.end(), [](const Entry& x, const Entry& y) { return x.r > y.r; });
      auto mstar = [&](int32_t p) -> int64_t {  // Eq.(eq:1)-(eq:3) over R ∪ Q[1..p]
        int64_t A = 0, best = 0;
        int32_t N = 0;
        for (const Entry& x : e) {
          if (x.j > p) continue;
          A += x.a;
          ++N;
          best = std::max(best, A + (int64_t)x.r * N);
        }
        return best;
      };
      const int64_t m0 = mstar(0);
      const int64_t lim = (int64_t)(10000 - reserved_bp) * capacity[i];
      int32_t lo = 0, hi = q;  // largest p with 10^4·M*(p) ≤ (10^4 − bp)·M; p = 0 always "fits" here
      int64_t m_lo = m0;
      if (10000 * m0 > lim) {
        hi = 0;
      } else {
        while (lo < hi) {
          const int32_t mid = (lo + hi + 1) >> 1;
          const int64_t m = mstar(mid);
          if (10000 * m <= lim) {
            lo = mid;
            m_lo = m;
          } else {
            hi = mid - 1;
          }
        }
      }
      admitted_out[i] = lo;
      peak_out[i] = (int32_t)m_lo;
      if (peak_running_out) peak_running_out[i] = (int32_t)m0;
    }
  };
  const int T = std::max(1, std::min<int>(n_threads, n));
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const int32_t a = (int32_t)((int64_t)n * t / T), b = (int32_t)((int64_t)n * (t + 1) / T);
    th.emplace_back(work, a, b);
  }
  for (auto& x : th) x.join();
  return 0;
}
