// pf_analysis_oracle.cpp — CPU ORACLE for the window-similarity analysis (SURVEY.md
// §8(f) NEXT-3; fig:dist and fig:cos_win).
//
// TEST INFRASTRUCTURE ONLY (same rules as pf_oracle.cpp); compiled into liborc.so.
//
// Definitions, written out:
//   A stream of output lengths is cut into consecutive non-overlapping windows of `w`
//   requests (trailing remainder dropped; fig:dist caption "1000 requests, no overlap").
//   h_b(l) = #{x in window b : len_x = l}, token-exact bins l = 1..Lmax.
//   G[i][j] = Σ_l h_i(l)·h_j(l)                     (integer Gram matrix)
//   cos[i][j] = G[i][j] / sqrt(G[i][i]·G[j][j])     (cosine similarity, fig:dist)
//   mean_adjacent = mean_i cos[i][i+1]; mean_global = mean_{i≠j} cos[i][j]  (fig:cos_win,
//   "average cosine similarity on global or diagonal line")
//   Adjacent windows of different sizes (fig:cos_win): running window k =
//   [h + k·r, h + (k+1)·r), its historical window = the h lengths just before it;
//   c_k = cos(hist_k, run_k).

#include <cmath>
#include <cstdint>
#include <vector>

extern "C" {

static std::vector<int64_t> histogram(const int32_t* x, int64_t n, int32_t max_len) {
  std::vector<int64_t> h(max_len + 1, 0);
  for (int64_t t = 0; t < n; ++t) h[x[t]] += 1;
  return h;
}

static int64_t dot(const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
  int64_t s = 0;
  for (size_t l = 0; l < a.size(); ++l) s += a[l] * b[l];
  return s;
}

static double cosine(int64_t g_ab, int64_t g_aa, int64_t g_bb) {
  return (double)g_ab / std::sqrt((double)g_aa * (double)g_bb);
}

// Returns the number of windows B (0 if < 2 windows or a length is outside [1, Lmax]).
int32_t orc_window_similarity(const int32_t* lengths, int64_t n, int32_t w, int32_t max_len,
                              int64_t* gram_out, double* cos_out, double* summary_out) {
  if (w < 1 || n / w < 2) return 0;
  for (int64_t t = 0; t < n; ++t)
    if (lengths[t] < 1 || lengths[t] > max_len) return 0;
  const int32_t B = (int32_t)(n / w);
  std::vector<std::vector<int64_t>> h;
  for (int32_t b = 0; b < B; ++b) h.push_back(histogram(lengths + (int64_t)b * w, w, max_len));
  std::vector<int64_t> G((size_t)B * B);
  for (int32_t i = 0; i < B; ++i)
    for (int32_t j = 0; j < B; ++j) G[(size_t)i * B + j] = dot(h[i], h[j]);
  double adj = 0.0, glob = 0.0;
  for (int32_t i = 0; i < B; ++i)
    for (int32_t j = 0; j < B; ++j) {
      const double c = cosine(G[(size_t)i * B + j], G[(size_t)i * B + i], G[(size_t)j * B + j]);
      if (gram_out) gram_out[(size_t)i * B + j] = G[(size_t)i * B + j];
      if (cos_out) cos_out[(size_t)i * B + j] = c;
      if (j == i + 1) adj += c;
      if (j != i) glob += c;
    }
  if (summary_out) {
    summary_out[0] = adj / (B - 1);
    summary_out[1] = glob / ((double)B * (B - 1));
  }
  return B;
}

// Returns the number of running windows K (0 if none or a length is out of range).
int32_t orc_adjacent_similarity(const int32_t* lengths, int64_t n, int32_t hw, int32_t rw,
                                int32_t max_len, double* cos_out, double* mean_out) {
  if (hw < 1 || rw < 1 || n < (int64_t)hw + rw) return 0;
  for (int64_t t = 0; t < n; ++t)
    if (lengths[t] < 1 || lengths[t] > max_len) return 0;
  const int32_t K = (int32_t)((n - hw) / rw);
  double s = 0.0;
  for (int32_t k = 0; k < K; ++k) {
    const int64_t r0 = hw + (int64_t)k * rw;
    std::vector<int64_t> hh = histogram(lengths + r0 - hw, hw, max_len);
    std::vector<int64_t> hr = histogram(lengths + r0, rw, max_len);
    const double c = cosine(dot(hh, hr), dot(hh, hh), dot(hr, hr));
    if (cos_out) cos_out[k] = c;
    s += c;
  }
  if (mean_out) *mean_out = s / K;
  return K;
}

}  // extern "C"
