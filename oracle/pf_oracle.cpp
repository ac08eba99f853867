// pf_oracle.cpp — the CPU ORACLE for the Past-Future scheduler hot path (arXiv 2507.10150).
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library. The product path
// (paper_2507_10150_b200/) never links, imports or calls it, and this file shares
// no code, header, table or constant generator with paper_2507_10150_b200/csrc/.
//
// It is a plain, slow, obviously-correct transcription of the paper's definitions,
// in the paper's order and notation (citations are PAPER.md line numbers and LaTeX
// labels):
//
//   history L_h, counter C(l, L_h), P(l) = C(l, L_h)/w ...... Eq.(eq:5)
//   sample l̂ from P(l > l_t) (running) / P(l) (queued) ..... Alg.1 lines 3-9
//   future required memory M* ............................... Eq.(eq:1)-(eq:3)
//     - tick form (the north-star oracle): step every future token tick τ and
//       take the max occupancy, "after growth, before removal"
//     - sort form: Eq.(eq:1) sort, Eq.(eq:2) M_i, Eq.(eq:3) max (cross-check)
//     - naive brute force O(n·r_max) (cross-check)
//   FIFO admission with early return ........................ Alg.1 lines 7-14
//
// Readings of silent/ambiguous points follow SURVEY.md §8(c) C-1..C-19 and are
// listed in DESIGN.md §3. All arithmetic is integer (int64 internally); there is
// no floating point anywhere.
//
// Pins: tests/test_oracle_pins.py checks every function here against values the
// paper prints (fig:peak narrative), SPEC.md worked examples,
// closed forms, brute force and library routines. Sampling-mode draws (C-8) are
// a convention not fixed by the paper: "parity unpinned" by the paper, pinned
// only by SplitMix64's published first output and the SURVEY P-6 prototype table.
//
// Build: g++ -O2 -std=c++17 -fPIC -shared -pthread pf_oracle.cpp -o liborc.so

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <deque>
#include <thread>
#include <vector>

extern "C" {

// ---------------------------------------------------------------------------
// C-8: counter-based draw u ∈ [0, 2^32) for sampling mode.
// Not in the paper; a convention shared (re-implemented, not shared code) by
// the oracle and the CUDA path.
// ---------------------------------------------------------------------------

// SplitMix64 finalizer (Steele, Lea, Flood 2014): mix64(γ) is SplitMix64's first
// output from state 0 = 0xE220A8397B1DCDAF.
uint64_t orc_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

// lowbias32 (C. Wellons' hash-prospector 32-bit integer hash).
uint32_t orc_lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// Per-instance key K = mix64(seed ⊕ tick·0xD1B54A32D192ED03 ⊕ inst·0x9E3779B97F4A7C15).
uint64_t orc_instance_key(uint64_t seed, uint32_t tick, int64_t inst) {
  uint64_t t = (uint64_t)tick * 0xD1B54A32D192ED03ULL;
  uint64_t i = (uint64_t)inst * 0x9E3779B97F4A7C15ULL;
  return orc_mix64(seed ^ t ^ i);
}

// One draw: u = lowbias32(lo32(K) ⊕ hi32(K) ⊕ lo32((slot·R + rep)·0x9E3779B9)).
uint32_t orc_draw(uint64_t key, int32_t slot, int32_t R, int32_t rep) {
  uint32_t lo = (uint32_t)(key & 0xFFFFFFFFULL);
  uint32_t hi = (uint32_t)(key >> 32);
  uint32_t c = (uint32_t)((uint64_t)((int64_t)slot * R + rep) * 0x9E3779B9ULL);
  return orc_lowbias32(lo ^ hi ^ c);
}

// ---------------------------------------------------------------------------
// Prediction: Alg.1 line 4 "Sample l̂ from P(l > l_t)" and line 8
// "Sample l̂ from P(l)" (= the l_t = 0 case since history ≥ 1, C-16).
// Reading C-3: inverse CDF at u; rank ρ = ⌊u·|gt| / 2^32⌋ (0-based) among the
// history values > l_t in ascending order. C-4 strict '>'. C-5 empty support →
// max_new. C-6 clamp to max_new.
// ---------------------------------------------------------------------------
int32_t orc_predict(const int32_t* window, int32_t w, int32_t l_t, int32_t max_new,
                    uint32_t u) {
  // Enumerate gt = { h ∈ L_h : h > l_t } explicitly, then sort ascending.
  std::vector<int32_t> gt;
  for (int32_t i = 0; i < w; ++i)
    if (window[i] > l_t) gt.push_back(window[i]);
  if (gt.empty()) return max_new;                       // C-5
  std::sort(gt.begin(), gt.end());
  uint64_t rho = ((uint64_t)u * (uint64_t)gt.size()) >> 32;
  int32_t l_hat = gt[(size_t)rho];
  return std::min(l_hat, max_new);                      // C-6
}

// Same draw on a window that Alg.1 line 1 has already built (sorted ascending once
// per instance): gt is still enumerated explicitly, element by element.
static int32_t predict_on_sorted(const std::vector<int32_t>& sorted_window, int32_t l_t,
                                 int32_t max_new, uint32_t u) {
  std::vector<int32_t> gt;
  for (int32_t h : sorted_window)
    if (h > l_t) gt.push_back(h);
  if (gt.empty()) return max_new;                       // C-5
  uint64_t rho = ((uint64_t)u * (uint64_t)gt.size()) >> 32;
  return std::min(gt[(size_t)rho], max_new);            // C-6
}

// "Repeated several times", reading C-9: R draws, prediction = the
// max of the R samples. Done literally: R separate inverse-CDF
// samples, then max (the CUDA path uses one quantile at max u; this is the
// independent formulation).
int32_t orc_predict_rep(const int32_t* window, int32_t w, int32_t l_t, int32_t max_new,
                        uint64_t key, int32_t slot, int32_t R) {
  int32_t best = 0;
  for (int32_t rep = 0; rep < R; ++rep) {
    int32_t s = orc_predict(window, w, l_t, max_new, orc_draw(key, slot, R, rep));
    best = std::max(best, s);
  }
  return best;
}

// ---------------------------------------------------------------------------
// Future required memory M* (Eq.(eq:1)-(eq:3)).
// Entry e holds a_e = l_p + l_t tokens now (Eq.(eq:1) first component) and will
// generate r_e = l̂ − l_t more (second component). Reading C-10: at future tick τ
// a resident entry holds a_e + τ tokens; it is resident while τ ≤ r_e ("the peak
// occurs at the moment a request ends": after growth, before removal).
// ---------------------------------------------------------------------------

// Tick form: step every tick τ = 0, 1, ..., max r, with per-tick release buckets.
int64_t orc_peak_ticks(int32_t n, const int32_t* a, const int32_t* r) {
  if (n == 0) return 0;
  int32_t r_max = 0;
  for (int32_t e = 0; e < n; ++e) r_max = std::max(r_max, r[e]);
  std::vector<int64_t> release_a((size_t)r_max + 1, 0);   // Σ a_e of entries ending at τ
  std::vector<int64_t> release_n((size_t)r_max + 1, 0);   // # entries ending at τ
  int64_t alive_a = 0, alive_n = 0;
  for (int32_t e = 0; e < n; ++e) {
    release_a[r[e]] += a[e];
    release_n[r[e]] += 1;
    alive_a += a[e];
    alive_n += 1;
  }
  int64_t peak = 0;
  for (int32_t tau = 0; tau <= r_max; ++tau) {
    int64_t occupancy = alive_a + (int64_t)tau * alive_n;  // after growth at τ
    peak = std::max(peak, occupancy);
    alive_a -= release_a[tau];                             // entries finishing at τ leave
    alive_n -= release_n[tau];
  }
  return peak;
}

// Sort form, literally Eq.(eq:1)-(eq:3): sort by remaining r descending,
// M_i = Σ_{j≤i} a_j + r_i·i, M* = max_i M_i (empty → 0).
int64_t orc_peak_sort(int32_t n, const int32_t* a, const int32_t* r) {
  std::vector<std::pair<int32_t, int32_t>> s;  // (r, a)
  for (int32_t e = 0; e < n; ++e) s.push_back({r[e], a[e]});
  std::sort(s.begin(), s.end(), [](const std::pair<int32_t, int32_t>& x,
                                   const std::pair<int32_t, int32_t>& y) {
    return x.first > y.first;
  });
  int64_t prefix = 0, best = 0;
  for (int32_t i = 1; i <= n; ++i) {
    prefix += s[i - 1].second;
    int64_t M_i = prefix + (int64_t)s[i - 1].first * i;
    best = std::max(best, M_i);
  }
  return best;
}

// Naive brute force: re-sum every entry at every tick, O(n · r_max).
int64_t orc_peak_brute(int32_t n, const int32_t* a, const int32_t* r) {
  int32_t r_max = 0;
  for (int32_t e = 0; e < n; ++e) r_max = std::max(r_max, r[e]);
  int64_t best = 0;
  for (int32_t tau = 0; n > 0 && tau <= r_max; ++tau) {
    int64_t occ = 0;
    for (int32_t e = 0; e < n; ++e)
      if (r[e] >= tau) occ += (int64_t)a[e] + tau;
    best = std::max(best, occ);
  }
  return best;
}

// ---------------------------------------------------------------------------
// Admission, literally Alg.1 lines 7-14 for ONE instance,
// given predicted (a, r) for the running batch and the FIFO queue.
// For j = 1..q: M* of R ∪ Q[1..j] from scratch (tick form); admit iff
// 10^4·M* ≤ (10^4 − bp)·M (C-12 '≤', C-13 reserved ratio in basis points);
// else return (C-14 early return). Returns p*; *peak = M* of the admitted set
// (= M*(R) when p* = 0); *peak_running = M*(R).
// ---------------------------------------------------------------------------
static bool fits(int64_t m_star, int64_t capacity, int32_t bp) {
  return m_star * 10000 <= (int64_t)(10000 - bp) * capacity;
}

int32_t orc_admit_one(int32_t k, const int32_t* run_a, const int32_t* run_r, int32_t q,
                      const int32_t* q_a, const int32_t* q_r, int64_t capacity, int32_t bp,
                      int64_t* peak, int64_t* peak_running) {
  std::vector<int32_t> a(run_a, run_a + k), r(run_r, run_r + k);
  int64_t m_run = orc_peak_ticks(k, a.data(), r.data());
  int64_t m_adm = m_run;
  int32_t admitted = 0;
  for (int32_t j = 0; j < q; ++j) {
    a.push_back(q_a[j]);
    r.push_back(q_r[j]);
    int64_t m = orc_peak_ticks((int32_t)a.size(), a.data(), r.data());
    if (fits(m, capacity, bp)) {
      admitted = j + 1;
      m_adm = m;
    } else {
      break;  // "Return S"
    }
  }
  if (peak) *peak = m_adm;
  if (peak_running) *peak_running = m_run;
  return admitted;
}

// Cross-check variant: binary search over p (valid because M*(p) is monotone
// non-decreasing in p), evaluating M* with the sort form.
int32_t orc_admit_one_bsearch(int32_t k, const int32_t* run_a, const int32_t* run_r,
                              int32_t q, const int32_t* q_a, const int32_t* q_r,
                              int64_t capacity, int32_t bp, int64_t* peak) {
  auto m_of = [&](int32_t p) {
    std::vector<int32_t> a(run_a, run_a + k), r(run_r, run_r + k);
    for (int32_t j = 0; j < p; ++j) { a.push_back(q_a[j]); r.push_back(q_r[j]); }
    return orc_peak_sort((int32_t)a.size(), a.data(), r.data());
  };
  int32_t lo = 0, hi = q;  // invariant: answer in [lo, hi]; p = 0 always "admits nothing"
  while (lo < hi) {
    int32_t mid = lo + (hi - lo + 1) / 2;
    if (fits(m_of(mid), capacity, bp)) lo = mid; else hi = mid - 1;
  }
  if (peak) *peak = m_of(lo);
  return lo;
}

// ---------------------------------------------------------------------------
// Batched state: many independent scheduler instances (or shared groups).
// A "row" is one FIFO history ring of `row_window` entries (Eq.(eq:5)'s L_h, C-1:
// exactly w entries, count-based). An instance's distribution is the
// concatenation of `rows_per_dist` consecutive rows (1 = per-instance history;
// 8 = the shared-group window of C-18, a group's 8 shard rings).
// ---------------------------------------------------------------------------
struct orc_ctx {
  int32_t n_rows, row_window, max_len, rows_per_dist;
  std::vector<std::deque<int32_t>> rows;
};

// Device-error codes mirrored from the boundary's documented behaviour.
enum { ORC_OK = 0, ORC_E_COMPLETION = 1, ORC_E_OFFSETS = 2, ORC_E_MAX_NEW = 3,
       ORC_E_INPUT_LEN = 4, ORC_E_GENERATED = 5, ORC_E_CAPACITY = 6 };

orc_ctx* orc_create(int32_t n_rows, int32_t row_window, int32_t max_len,
                    int32_t rows_per_dist, const int32_t* init_rows) {
  if (n_rows <= 0 || row_window <= 0 || max_len <= 0 || rows_per_dist <= 0) return nullptr;
  orc_ctx* c = new orc_ctx();
  c->n_rows = n_rows;
  c->row_window = row_window;
  c->max_len = max_len;
  c->rows_per_dist = rows_per_dist;
  c->rows.resize(n_rows);
  for (int32_t i = 0; i < n_rows; ++i)
    for (int32_t t = 0; t < row_window; ++t)  // C-2: default = w copies of Lmax
      c->rows[i].push_back(init_rows ? init_rows[(int64_t)i * row_window + t] : max_len);
  return c;
}

void orc_destroy(orc_ctx* c) { delete c; }

// "records the actual output lengths": append in order, evict the
// oldest when more than w. A row whose call contains a length ∉ [1, Lmax] is
// left unchanged and reported (returns the first bad row's code, else 0).
int32_t orc_update_history(orc_ctx* c, const int32_t* comp_off, const int32_t* comp_len,
                           int32_t* bad_row) {
  int32_t status = ORC_OK;
  for (int32_t i = 0; i < c->n_rows; ++i) {
    bool ok = comp_off[i + 1] >= comp_off[i];
    for (int32_t t = comp_off[i]; ok && t < comp_off[i + 1]; ++t)
      if (comp_len[t] < 1 || comp_len[t] > c->max_len) ok = false;
    if (!ok) {
      if (status == ORC_OK) { status = ORC_E_COMPLETION; if (bad_row) *bad_row = i; }
      continue;
    }
    for (int32_t t = comp_off[i]; t < comp_off[i + 1]; ++t) {
      c->rows[i].push_back(comp_len[t]);
      if ((int32_t)c->rows[i].size() > c->row_window) c->rows[i].pop_front();
    }
  }
  return status;
}

// Export a row, oldest first.
void orc_get_row(const orc_ctx* c, int32_t row, int32_t* out) {
  int32_t t = 0;
  for (int32_t v : c->rows[row]) out[t++] = v;
}

// The distribution window of distribution `d` (rows d·rpd .. d·rpd+rpd-1 concatenated).
static std::vector<int32_t> window_of(const orc_ctx* c, int32_t d) {
  std::vector<int32_t> w;
  for (int32_t s = 0; s < c->rows_per_dist; ++s)
    for (int32_t v : c->rows[(size_t)d * c->rows_per_dist + s]) w.push_back(v);
  return w;
}

struct orc_admit_args {
  int32_t n_inst;
  const int32_t* dist_of;      // [n_inst] distribution (row group) of each instance
  const int64_t* inst_id;      // [n_inst] global instance id (hash key, C-8)
  const int32_t* run_off;      // [n_inst+1]
  const int32_t* input_len;    // [run_off[n]] l_p
  const int32_t* generated;    // [run_off[n]] l_t
  const int32_t* q_off;        // [n_inst+1] or NULL (estimate only)
  const int32_t* q_input_len;  // [q_off[n]]
  const int32_t* max_new;      // [n_inst]
  const int32_t* capacity;     // [n_inst] or NULL (estimate only)
  int32_t mode;                // 0 = sample (C-8 hash), 1 = quantile (fixed u)
  uint32_t quantile_u;
  int32_t repetitions;         // R >= 1
  int32_t reserved_bp;         // 0..9999
  uint64_t seed;
  uint32_t tick;
  int32_t max_input_len;       // declared bound on l_p (validation)
  int32_t max_entries;         // declared bound on k+q (validation)
  int32_t* admitted_out;       // [n_inst] or NULL
  int32_t* peak_out;           // [n_inst]  M*(admitted) (admit) / M*(R) (estimate)
  int32_t* peak_running_out;   // [n_inst] or NULL
  int32_t* pred_run_out;       // [run_off[n]] or NULL
  int32_t* pred_q_out;         // [q_off[n]] or NULL
  int32_t* first_error;        // out: first (lowest-instance) error code
  int32_t* first_error_inst;   // out
};

// One instance of Algorithm 1, with the boundary's
// validation. Returns an error code (0 = ok).
static int32_t admit_instance(const orc_ctx* c, const orc_admit_args* A, int32_t i) {
  const int32_t r0 = A->run_off[i], r1 = A->run_off[i + 1];
  const int32_t q0 = A->q_off ? A->q_off[i] : 0, q1 = A->q_off ? A->q_off[i + 1] : 0;
  const int32_t k = r1 - r0, q = q1 - q0;
  const int32_t max_new = A->max_new[i];
  int32_t err = ORC_OK;
  if (k < 0 || q < 0 || k + q > A->max_entries) err = ORC_E_OFFSETS;
  else if (max_new < 1 || max_new > c->max_len) err = ORC_E_MAX_NEW;
  else if (A->capacity && A->capacity[i] < 0) err = ORC_E_CAPACITY;
  for (int32_t s = 0; err == ORC_OK && s < k; ++s) {
    if (A->input_len[r0 + s] < 0 || A->input_len[r0 + s] > A->max_input_len) err = ORC_E_INPUT_LEN;
    else if (A->generated[r0 + s] < 0 || A->generated[r0 + s] >= max_new) err = ORC_E_GENERATED;
  }
  for (int32_t j = 0; err == ORC_OK && j < q; ++j)
    if (A->q_input_len[q0 + j] < 0 || A->q_input_len[q0 + j] > A->max_input_len) err = ORC_E_INPUT_LEN;
  if (err != ORC_OK) {
    if (A->admitted_out) A->admitted_out[i] = -1;
    A->peak_out[i] = -1;
    if (A->peak_running_out) A->peak_running_out[i] = -1;
    if (A->pred_run_out && k > 0)
      for (int32_t s = r0; s < r1; ++s) A->pred_run_out[s] = -1;
    if (A->pred_q_out && q > 0)
      for (int32_t j = q0; j < q1; ++j) A->pred_q_out[j] = -1;
    return err;
  }

  // Alg.1 line 1: the distribution P(l) is the window L_h (Eq.(eq:5)).
  std::vector<int32_t> window = window_of(c, A->dist_of[i]);
  std::sort(window.begin(), window.end());
  // R > 0: fixed repetitions; R = 0: SPEC.md:161's reading of "repeated several times
  // when the size of the running batch is low": R = max(1, ⌈64/k⌉), k = 0 → 64.
  const int32_t R = A->repetitions > 0 ? A->repetitions : (k > 0 ? std::max(1, (64 + k - 1) / k) : 64);
  const uint64_t key = orc_instance_key(A->seed, A->tick, A->inst_id[i]);
  auto predict = [&](int32_t l_t, int32_t slot) -> int32_t {
    if (A->mode == 1) return predict_on_sorted(window, l_t, max_new, A->quantile_u);
    int32_t best = 0;  // C-9: max of R samples
    for (int32_t rep = 0; rep < R; ++rep)
      best = std::max(best, predict_on_sorted(window, l_t, max_new, orc_draw(key, slot, R, rep)));
    return best;
  };

  // Alg.1 lines 3-6: running requests, l̂ from P(l > l_t); slot = s.
  std::vector<int32_t> run_a(k), run_r(k);
  for (int32_t s = 0; s < k; ++s) {
    int32_t l_p = A->input_len[r0 + s], l_t = A->generated[r0 + s];
    int32_t l_hat = predict(l_t, s);
    if (A->pred_run_out) A->pred_run_out[r0 + s] = l_hat;
    run_a[s] = l_p + l_t;     // Eq.(eq:1): l_p^i + l_t^i
    run_r[s] = l_hat - l_t;   // Eq.(eq:1): l̂_t^i − l_t^i
  }
  // Alg.1 line 8: queued requests, l̂ from P(l) (l_t = 0, C-16); slot = k + j − 1.
  std::vector<int32_t> q_a(q), q_r(q);
  for (int32_t j = 0; j < q; ++j) {
    int32_t l_hat = predict(0, k + j);
    if (A->pred_q_out) A->pred_q_out[q0 + j] = l_hat;
    q_a[j] = A->q_input_len[q0 + j];
    q_r[j] = l_hat;
  }

  if (A->capacity == nullptr) {  // estimate only: M*(R)
    A->peak_out[i] = (int32_t)orc_peak_ticks(k, run_a.data(), run_r.data());
    return ORC_OK;
  }
  int64_t peak = 0, peak_run = 0;
  int32_t p = orc_admit_one(k, run_a.data(), run_r.data(), q, q_a.data(), q_r.data(),
                            A->capacity[i], A->reserved_bp, &peak, &peak_run);
  if (A->admitted_out) A->admitted_out[i] = p;
  A->peak_out[i] = (int32_t)peak;
  if (A->peak_running_out) A->peak_running_out[i] = (int32_t)peak_run;
  return ORC_OK;
}

// Batched Alg.1 over n independent instances, `n_threads` std::threads with a
// static contiguous partition. Returns the number of instances with errors.
int32_t orc_admit(const orc_ctx* c, const orc_admit_args* A, int32_t n_threads) {
  if (n_threads < 1) n_threads = 1;
  std::vector<int32_t> errs(A->n_inst, 0);
  auto work = [&](int32_t lo, int32_t hi) {
    for (int32_t i = lo; i < hi; ++i) errs[i] = admit_instance(c, A, i);
  };
  std::vector<std::thread> pool;
  int32_t per = (A->n_inst + n_threads - 1) / n_threads;
  for (int32_t t = 0; t < n_threads; ++t) {
    int32_t lo = t * per, hi = std::min(A->n_inst, lo + per);
    if (lo < hi) pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  int32_t n_bad = 0;
  if (A->first_error) *A->first_error = 0;
  for (int32_t i = 0; i < A->n_inst; ++i) {
    if (errs[i] == 0) continue;
    if (n_bad == 0 && A->first_error) {
      *A->first_error = errs[i];
      if (A->first_error_inst) *A->first_error_inst = i;
    }
    ++n_bad;
  }
  return n_bad;
}

int32_t orc_sizeof_admit_args(void) { return (int32_t)sizeof(orc_admit_args); }

// ---------------------------------------------------------------------------
// Baseline admission policies the paper compares against (§5.3
// Table 1 rows :345-349), one instance, FIFO with early return:
//   aggressive   (watermark, "batches requests solely based on
//                input lengths"): admit the j-th queued request while
//                Σ_running(l_p + l_t) + Σ_{admitted ∪ j} l_p ≤ watermark·M
//   conservative (overcommit, "the sum of request input lengths and
//                the max_new_tokens", :379 "assumes 1.5 times the memory"): admit while
//                Σ_{running ∪ admitted ∪ j}(l_p + max_new) ≤ overcommit·M
// Ratios in basis points; compare 10^4·used ≤ ratio_bp·M in int64. Returns p*;
// *used = the left-hand side for the admitted set.
int32_t orc_admit_aggressive(int32_t k, const int32_t* run_lp, const int32_t* run_lt, int32_t q,
                             const int32_t* q_lp, int64_t capacity, int32_t watermark_bp,
                             int64_t* used) {
  int64_t consumed = 0;
  for (int32_t s = 0; s < k; ++s) consumed += (int64_t)run_lp[s] + run_lt[s];
  int32_t admitted = 0;
  for (int32_t j = 0; j < q; ++j) {
    if ((consumed + q_lp[j]) * 10000 <= (int64_t)watermark_bp * capacity) {
      consumed += q_lp[j];
      admitted = j + 1;
    } else {
      break;
    }
  }
  if (used) *used = consumed;
  return admitted;
}

int32_t orc_admit_conservative(int32_t k, const int32_t* run_lp, int32_t q, const int32_t* q_lp,
                               int32_t max_new, int64_t capacity, int32_t overcommit_bp,
                               int64_t* used) {
  int64_t budget = 0;
  for (int32_t s = 0; s < k; ++s) budget += (int64_t)run_lp[s] + max_new;
  int32_t admitted = 0;
  for (int32_t j = 0; j < q; ++j) {
    if ((budget + q_lp[j] + max_new) * 10000 <= (int64_t)overcommit_bp * capacity) {
      budget += (int64_t)q_lp[j] + max_new;
      admitted = j + 1;
    } else {
      break;
    }
  }
  if (used) *used = budget;
  return admitted;
}

}  // extern "C"
