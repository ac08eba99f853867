// pf_forward_oracle.cpp — CPU ORACLE for cross-instance request forwarding (SURVEY.md
// §8(f) NEXT-4; the paper's future work: "based on its ability to
// accurately estimate the memory demand of each running batch, it can forward requests
// to underutilized services ... aiming to ensure that each service reaches full
// capacity").
//
// TEST INFRASTRUCTURE ONLY (same rules as pf_oracle.cpp); compiled into liborc.so.
//
// Readings F-1..F-4:
//   F-1 A cluster is S instances (services) sharing one FIFO arrival queue. Requests
//       are forwarded one at a time in queue order; request j goes to the instance s
//       that can take it — 10^4·M*_s(R_s ∪ F_s ∪ {j}) ≤ (10^4 − bp)·M_s, Alg.1's check
//       (PAPER.md:226), F_s = requests already forwarded to s in this call — with the
//       largest headroom (10^4 − bp)·M_s − 10^4·M*_s(...) ("underutilized"); ties go to
//       the lowest s. If no instance can take j, forwarding stops (FIFO early return,
//       C-14). An instance whose k + |F_s| reached max_entries cannot take requests.
//   F-2 Instance s predicts its running requests exactly as pf_admit does (Alg.1 lines
//       3-6 with its own window, key and slots 0..k_s−1) and the cluster's j-th queued
//       request (1-based) as its own queued slot k_s + j − 1 (Alg.1 line 8, C-16).
//   F-3 M* is the tick form of Eq.(eq:1)-(eq:3), recomputed from scratch per candidate.
//   F-4 Outputs: dest[j] = chosen instance (−1 for j after the first failure),
//       forwarded[c] = number forwarded, peak[s] = M*_s(R_s ∪ F_s).

#include <algorithm>
#include <cstdint>
#include <vector>

extern "C" {
int32_t orc_predict(const int32_t* window, int32_t w, int32_t l_t, int32_t max_new, uint32_t u);
uint64_t orc_instance_key(uint64_t seed, uint32_t tick, int64_t inst);
uint32_t orc_draw(uint64_t key, int32_t slot, int32_t R, int32_t rep);
int64_t orc_peak_ticks(int32_t n, const int32_t* a, const int32_t* r);

struct orc_forward_args {
  int32_t n_clusters, cluster_size;  // instances = n_clusters · cluster_size
  const int32_t* windows;            // [n × w] history windows (any order: a multiset)
  int32_t window;
  const int32_t* run_off;            // [n+1]
  const int32_t* input_len;          // running l_p
  const int32_t* generated;          // running l_t
  const int32_t* max_new;            // [n]
  const int32_t* capacity;           // [n]
  const int32_t* cq_off;             // [C+1] cluster queues
  const int32_t* cq_input_len;       // queued l_p
  int32_t mode;                      // 0 sample (C-8, R = 1), 1 quantile
  uint32_t quantile_u;
  int32_t reserved_bp;
  uint64_t seed;
  uint32_t tick;
  int64_t instance_base;
  int32_t max_entries;
  int32_t* dest_out;                 // [cq_off[C]]
  int32_t* forwarded_out;            // [C]
  int32_t* peak_out;                 // [n]
};

static void forward_cluster(const orc_forward_args* A, int32_t c) {
  const int32_t S = A->cluster_size, w = A->window;
  const int32_t q0 = A->cq_off[c], q = A->cq_off[c + 1] - q0;
  std::vector<std::vector<int32_t>> ea(S), er(S);  // entries (a, r) of R_s ∪ F_s
  std::vector<int32_t> k(S);
  for (int32_t s = 0; s < S; ++s) {
    const int32_t i = c * S + s;
    const int32_t r0 = A->run_off[i];
    k[s] = A->run_off[i + 1] - r0;
    const int32_t* win = A->windows + (int64_t)i * w;
    const uint64_t key = orc_instance_key(A->seed, A->tick, A->instance_base + i);
    for (int32_t e = 0; e < k[s]; ++e) {
      const int32_t l_t = A->generated[r0 + e];
      const uint32_t u = A->mode == 1 ? A->quantile_u : orc_draw(key, e, 1, 0);
      const int32_t l_hat = orc_predict(win, w, l_t, A->max_new[i], u);
      ea[s].push_back(A->input_len[r0 + e] + l_t);
      er[s].push_back(l_hat - l_t);
    }
  }
  int32_t forwarded = 0;
  bool stopped = false;
  for (int32_t j = 0; j < q; ++j) {
    if (stopped) { A->dest_out[q0 + j] = -1; continue; }
    int32_t best = -1;
    int64_t best_h = 0;
    for (int32_t s = 0; s < S; ++s) {
      const int32_t i = c * S + s;
      if ((int32_t)ea[s].size() >= A->max_entries) continue;
      const uint64_t key = orc_instance_key(A->seed, A->tick, A->instance_base + i);
      const uint32_t u = A->mode == 1 ? A->quantile_u : orc_draw(key, k[s] + j, 1, 0);
      const int32_t l_hat = orc_predict(A->windows + (int64_t)i * w, w, 0, A->max_new[i], u);
      std::vector<int32_t> a = ea[s], r = er[s];
      a.push_back(A->cq_input_len[q0 + j]);
      r.push_back(l_hat);
      const int64_t m = orc_peak_ticks((int32_t)a.size(), a.data(), r.data());
      const int64_t h = (int64_t)(10000 - A->reserved_bp) * A->capacity[i] - 10000 * m;
      if (h >= 0 && (best < 0 || h > best_h)) { best = s; best_h = h; }
    }
    if (best < 0) { stopped = true; A->dest_out[q0 + j] = -1; continue; }
    const int32_t i = c * S + best;
    const uint64_t key = orc_instance_key(A->seed, A->tick, A->instance_base + i);
    const uint32_t u = A->mode == 1 ? A->quantile_u : orc_draw(key, k[best] + j, 1, 0);
    ea[best].push_back(A->cq_input_len[q0 + j]);
    er[best].push_back(orc_predict(A->windows + (int64_t)i * w, w, 0, A->max_new[i], u));
    A->dest_out[q0 + j] = best;
    ++forwarded;
  }
  A->forwarded_out[c] = forwarded;
  for (int32_t s = 0; s < S; ++s)
    A->peak_out[c * S + s] =
        (int32_t)orc_peak_ticks((int32_t)ea[s].size(), ea[s].data(), er[s].data());
}

void orc_forward(const orc_forward_args* A) {
  for (int32_t c = 0; c < A->n_clusters; ++c) forward_cluster(A, c);
}

int32_t orc_sizeof_forward_args(void) { return (int32_t)sizeof(orc_forward_args); }

}  // extern "C"
