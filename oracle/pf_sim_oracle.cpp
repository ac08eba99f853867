// pf_sim_oracle.cpp — CPU ORACLE for the batched continuous-batching simulator
// (the engine behind the paper's Table 1).
//
// TEST INFRASTRUCTURE ONLY (same rules as pf_oracle.cpp): only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
// load it; it shares no code with paper_2507_10150_b200/csrc/. It is compiled into
// liborc.so together with pf_oracle.cpp and calls that file's primitives
// (orc_predict, orc_predict_rep, orc_peak_ticks, orc_admit_one, the baselines).
//
// One simulation per instance, literally, one iteration at a time (DESIGN.md §11,
// readings S-1..S-9; SPEC.md:332-400 engine, :245-330 schedulers):
//
//   S-1  all requests of an instance arrive at t = 0, in list order (Table 1 runs a
//        fixed request set to completion, "Decoding Steps ... required by continuous
//        batching to perform these requests")
//   iteration t:
//   S-2  finish: running requests with generated == true length leave (running-list
//        order) and their lengths are recorded into the window ("records the actual
//        output lengths"; Eq.(eq:5))
//   S-3  admission on (running, queue head window of min(|Q|, E − k) requests):
//        running (l_p, l_t = generated); a queued request enters with l_p + generated
//        (re-queued requests recompute their generated tokens, SPEC.md engine (4)) and
//        l_t = 0 (C-16). Policies: past-future = Alg.1 with tick t;
//        theoretical optimum = Alg.1 with l̂ = true length (running) / remaining true
//        length (queued); aggressive / conservative as
//        pf_oracle.cpp. FIFO prefix, early return.
//   S-4  admitted requests join the running list in FIFO order; if the running list
//        would stay empty with a non-empty queue, the head is admitted anyway
//        (progress; counted as "forced")
//   S-5  "future required memory" sample: M* of the running set with TRUE remaining
//        lengths (Eq.(eq:1)-(eq:3) "actual memory requirement in the future to finish
//        all current added requests when scheduling")
//   S-6  overflow: the decode step needs Σ(l_p + l_t) + k tokens; while that exceeds M
//        and k > 1, evict the most recently admitted request (LIFO), re-queue it at the
//        FRONT keeping its generated tokens; count the eviction
//   S-7  decode: every running request gains one token (the paper's tick model,
//        Eq.(eq:1): a request holds l_p + l_t and grows by one per step); count a
//        decoding step if the batch is non-empty
//   S-8  "current consumed memory" sample: Σ(l_p + l_t) after the decode step
//   S-9  the instance is done when queue and running list are both empty after S-2
//
// Metrics per instance (int64): [0] iterations, [1] decoding steps, [2] evictions,
// [3] finished requests, [4] Σ consumed samples, [5] Σ future samples,
// [6] samples, [7] max future sample, [8] forced admissions, [9] admissions.

#include <algorithm>
#include <cstdint>
#include <deque>
#include <thread>
#include <vector>

extern "C" {
int32_t orc_predict(const int32_t* window, int32_t w, int32_t l_t, int32_t max_new, uint32_t u);
int32_t orc_predict_rep(const int32_t* window, int32_t w, int32_t l_t, int32_t max_new,
                        uint64_t key, int32_t slot, int32_t R);
uint64_t orc_instance_key(uint64_t seed, uint32_t tick, int64_t inst);
int64_t orc_peak_ticks(int32_t n, const int32_t* a, const int32_t* r);
int32_t orc_admit_one(int32_t k, const int32_t* run_a, const int32_t* run_r, int32_t q,
                      const int32_t* q_a, const int32_t* q_r, int64_t capacity, int32_t bp,
                      int64_t* peak, int64_t* peak_running);
int32_t orc_admit_aggressive(int32_t k, const int32_t* run_lp, const int32_t* run_lt, int32_t q,
                             const int32_t* q_lp, int64_t capacity, int32_t watermark_bp,
                             int64_t* used);
int32_t orc_admit_conservative(int32_t k, const int32_t* run_lp, int32_t q, const int32_t* q_lp,
                               int32_t max_new, int64_t capacity, int32_t overcommit_bp,
                               int64_t* used);

enum { ORC_SIM_PAST_FUTURE = 0, ORC_SIM_OPTIMUM = 1, ORC_SIM_AGGRESSIVE = 2,
       ORC_SIM_CONSERVATIVE = 3 };
enum { ORC_SIM_NMETRICS = 10 };

struct orc_sim_args {
  int32_t n_inst;
  const int32_t* req_off;     // [n+1] requests of instance i: [req_off[i], req_off[i+1])
  const int32_t* req_input;   // l_p per request
  const int32_t* req_output;  // true output length per request, in [1, max_new[i]]
  const int32_t* max_new;     // [n]
  const int32_t* capacity;    // [n] M in tokens
  int32_t policy;             // ORC_SIM_*
  int32_t param_bp;           // reserved bp (past-future, optimum) / watermark / overcommit bp
  int32_t window;             // w (C-1)
  int32_t max_len;            // Lmax: default initial window = w copies of Lmax (C-2)
  const int32_t* init_history;  // nullable [n × w], oldest first (a steady-state window)
  int32_t max_entries;        // E: k + queue window ≤ E
  int32_t mode;               // 0 sample (C-8), 1 quantile
  uint32_t quantile_u;
  int32_t repetitions;        // R ≥ 1, 0 = adaptive (C-9)
  uint64_t seed;
  int64_t instance_base;      // hash key of instance i = instance_base + i
  int32_t iterations;         // run this many iterations (done instances idle)
  int64_t* metrics_out;       // [n × ORC_SIM_NMETRICS]
  int32_t* generated_out;     // [req_off[n]] nullable: generated tokens per request
  int32_t* evictions_out;     // [req_off[n]] nullable: evictions per request
};

static void sim_instance(const orc_sim_args* A, int32_t i) {
  const int32_t base = A->req_off[i], n_req = A->req_off[i + 1] - base;
  const int32_t* lp = A->req_input + base;
  const int32_t* L = A->req_output + base;
  const int32_t max_new = A->max_new[i];
  const int64_t M = A->capacity[i];
  std::vector<int32_t> gen(n_req, 0), evicted(n_req, 0);
  std::deque<int32_t> window(A->window, A->max_len);  // C-2
  if (A->init_history)
    for (int32_t t = 0; t < A->window; ++t) window[t] = A->init_history[(int64_t)i * A->window + t];
  std::deque<int32_t> queue;                            // S-1
  for (int32_t j = 0; j < n_req; ++j) queue.push_back(j);
  std::vector<int32_t> running;                         // admission order
  int64_t m[ORC_SIM_NMETRICS] = {0};
  bool done = false;

  for (int32_t t = 0; t < A->iterations && !done; ++t) {
    // S-2 finish and record
    std::vector<int32_t> still;
    for (int32_t j : running) {
      if (gen[j] == L[j]) {
        window.push_back(L[j]);
        if ((int32_t)window.size() > A->window) window.pop_front();
        m[3] += 1;
      } else {
        still.push_back(j);
      }
    }
    running.swap(still);
    if (running.empty() && queue.empty()) { done = true; break; }
    m[0] += 1;

    // S-3 admission over the queue head window
    const int32_t k = (int32_t)running.size();
    const int32_t qw = std::min((int32_t)queue.size(), std::max(0, A->max_entries - k));
    std::vector<int32_t> run_lp(k), run_lt(k), q_lp(qw);
    for (int32_t s = 0; s < k; ++s) { run_lp[s] = lp[running[s]]; run_lt[s] = gen[running[s]]; }
    for (int32_t j = 0; j < qw; ++j) q_lp[j] = lp[queue[j]] + gen[queue[j]];
    int32_t p = 0;
    if (A->policy == ORC_SIM_PAST_FUTURE || A->policy == ORC_SIM_OPTIMUM) {
      std::vector<int32_t> run_a(k), run_r(k), q_a(qw), q_r(qw);
      std::vector<int32_t> win(window.begin(), window.end());
      const int32_t R = A->repetitions > 0 ? A->repetitions
                                           : (k > 0 ? std::max(1, (64 + k - 1) / k) : 64);
      const uint64_t key = orc_instance_key(A->seed, (uint32_t)t, A->instance_base + i);
      auto predict = [&](int32_t l_t, int32_t slot) {
        if (A->mode == 1) return orc_predict(win.data(), (int32_t)win.size(), l_t, max_new, A->quantile_u);
        return orc_predict_rep(win.data(), (int32_t)win.size(), l_t, max_new, key, slot, R);
      };
      for (int32_t s = 0; s < k; ++s) {
        const int32_t l_hat = A->policy == ORC_SIM_OPTIMUM ? L[running[s]] : predict(run_lt[s], s);
        run_a[s] = run_lp[s] + run_lt[s];
        run_r[s] = l_hat - run_lt[s];
      }
      for (int32_t j = 0; j < qw; ++j) {
        const int32_t q = queue[j];
        q_a[j] = q_lp[j];
        q_r[j] = A->policy == ORC_SIM_OPTIMUM ? L[q] - gen[q] : predict(0, k + j);
      }
      p = orc_admit_one(k, run_a.data(), run_r.data(), qw, q_a.data(), q_r.data(), M,
                        A->param_bp, nullptr, nullptr);
    } else if (A->policy == ORC_SIM_AGGRESSIVE) {
      p = orc_admit_aggressive(k, run_lp.data(), run_lt.data(), qw, q_lp.data(), M, A->param_bp,
                               nullptr);
    } else {
      p = orc_admit_conservative(k, run_lp.data(), qw, q_lp.data(), max_new, M, A->param_bp,
                                 nullptr);
    }
    // S-4 join the running list (forced head admission keeps an empty batch moving)
    if (p == 0 && k == 0 && !queue.empty()) { p = 1; m[8] += 1; }
    for (int32_t j = 0; j < p; ++j) { running.push_back(queue.front()); queue.pop_front(); }
    m[9] += p;

    // S-5 future required memory with true remaining lengths
    {
      const int32_t kk = (int32_t)running.size();
      std::vector<int32_t> a(kk), r(kk);
      for (int32_t s = 0; s < kk; ++s) {
        const int32_t j = running[s];
        a[s] = lp[j] + gen[j];
        r[s] = L[j] - gen[j];
      }
      const int64_t fut = orc_peak_ticks(kk, a.data(), r.data());
      m[5] += fut;
      m[7] = std::max(m[7], fut);
    }
    // S-6 overflow eviction, LIFO, re-queue at the front
    int64_t demand = 0;
    for (int32_t j : running) demand += (int64_t)lp[j] + gen[j] + 1;
    while (demand > M && running.size() > 1) {
      const int32_t j = running.back();
      running.pop_back();
      demand -= (int64_t)lp[j] + gen[j] + 1;
      queue.push_front(j);
      evicted[j] += 1;
      m[2] += 1;
    }
    // S-7 decode step
    for (int32_t j : running) gen[j] += 1;
    if (!running.empty()) m[1] += 1;
    // S-8 consumed memory
    int64_t used = 0;
    for (int32_t j : running) used += (int64_t)lp[j] + gen[j];
    m[4] += used;
    m[6] += 1;
  }
  for (int32_t c = 0; c < ORC_SIM_NMETRICS; ++c) A->metrics_out[(int64_t)i * ORC_SIM_NMETRICS + c] = m[c];
  for (int32_t j = 0; j < n_req; ++j) {
    if (A->generated_out) A->generated_out[base + j] = gen[j];
    if (A->evictions_out) A->evictions_out[base + j] = evicted[j];
  }
}

// Independent instances on `n_threads` std::threads (static contiguous partition).
void orc_sim_run(const orc_sim_args* A, int32_t n_threads) {
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> pool;
  const int32_t per = (A->n_inst + n_threads - 1) / n_threads;
  for (int32_t t = 0; t < n_threads; ++t) {
    const int32_t lo = t * per, hi = std::min(A->n_inst, lo + per);
    if (lo < hi)
      pool.emplace_back([A, lo, hi] { for (int32_t i = lo; i < hi; ++i) sim_instance(A, i); });
  }
  for (auto& th : pool) th.join();
}

int32_t orc_sizeof_sim_args(void) { return (int32_t)sizeof(orc_sim_args); }

}  // extern "C"
