// pf_admit.cuh — the fused per-instance hot-path kernel of libpfsched (sm_100a):
//   a3/a4  distribution lookup + conditional quantile  (Eq.(eq:5), Alg.1 l.3-9)
//   a5     segmented sort by remaining length r desc     (Eq.(eq:1))
//   a6     scan + max: M_i = Σ_{j≤i} a_j + r_i·i, M*     (Eq.(eq:2)-(eq:3))
//   a7     prefix-admission search over the FIFO queue   (Alg.1 l.7-14)
// One CTA per instance; every step runs on-chip (shared memory + registers).
#pragma once
#include "pf_common.cuh"

namespace pf {

enum Lookup { LOOK_SORTED = 0, LOOK_HIST = 1, LOOK_GROUP = 2 };

struct AdmitParams {
  int n;               // instances
  int w;               // per-instance window, or group window W (shared)
  int max_len;         // Lmax
  int max_input_len;
  int max_entries;
  int mode;            // 0 sample, 1 quantile
  uint32_t quantile_u;
  int R;
  int bp;
  uint64_t seed;
  uint32_t tick;
  int64_t instance_base;
  int members_per_group, member_base;
  int bin_shift;       // coarse bin = (Lmax - r) >> bin_shift
  int n_bins;
  // history tables
  const int32_t* sorted;     // LOOK_SORTED [n × w]
  const int32_t* hist;       // LOOK_HIST   [n × (Lmax+1)]
  const int32_t* gC;         // LOOK_GROUP  [G × (Lmax+1)]
  const int32_t* gS;         // LOOK_GROUP  [G × W]
  const int32_t* dist_of;    // LOOK_GROUP  [n]
  const int32_t* group_off;  // LOOK_GROUP  [G+1]
  // inputs
  const int32_t* run_off;
  const int32_t* input_len;
  const int32_t* generated;
  const int32_t* q_off;      // NULL => estimate only
  const int32_t* q_input_len;
  const int32_t* max_new;
  const int32_t* capacity;
  // outputs
  int32_t* admitted_out;
  int32_t* peak_out;
  int32_t* peak_running_out;
  int32_t* pred_run_out;
  int32_t* pred_q_out;
  int32_t* err;
};

// Packed entry: r (15 bits) << 48 | j (16 bits) << 32 | a (31 bits).
__device__ __forceinline__ uint64_t pack_entry(int r, int j, int a) {
  return ((uint64_t)(uint32_t)r << 48) | ((uint64_t)(uint32_t)j << 32) | (uint32_t)a;
}
__device__ __forceinline__ int ent_r(uint64_t e) { return (int)(e >> 48); }
__device__ __forceinline__ int ent_j(uint64_t e) { return (int)((e >> 32) & 0xFFFF); }
__device__ __forceinline__ int ent_a(uint64_t e) { return (int)(e & 0xFFFFFFFFu); }

// #{x in S[0..w) : x <= v} for ascending S (upper_bound).
__device__ __forceinline__ int upper_bound_smem(const int32_t* S, int w, int v) {
  int lo = 0, len = w;
  while (len > 0) {
    int half = len >> 1;
    bool right = S[lo + half] <= v;
    lo = right ? lo + half + 1 : lo;
    len = right ? len - half - 1 : half;
  }
  return lo;
}

// 10^4·M ≤ (10^4 − bp)·cap  (C-12, C-13), exact in int64.
__device__ __forceinline__ bool fits(int m, int cap, int bp) {
  return (int64_t)m * 10000 <= (int64_t)(10000 - bp) * (int64_t)cap;
}

// Dynamic shared memory layout (bytes):
//   [0, 16·E)            ent_tmp (E = T·IPT packed entries) then ent_sorted
//   next 2·NB·4          bin counts, bin starts
//   next 64·4            scan scratch
//   next table           S[w] (LOOK_SORTED) | C[Lmax+1] (LOOK_HIST) | none
template <int T, int IPT, int LOOK>
__global__ void __launch_bounds__(T) admit_kernel(AdmitParams p) {
  constexpr int E = T * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* ent_tmp = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* ent_sorted = ent_tmp + E;
  int* bin_cnt = reinterpret_cast<int*>(ent_sorted + E);
  int* bin_start = bin_cnt + p.n_bins;
  int* scratch = bin_start + p.n_bins;
  int32_t* table = scratch + 64;

  const int i = blockIdx.x;
  const int tid = threadIdx.x;
  const bool estimate_only = (p.q_off == nullptr);

  // ---- instance scalars and CSR validation
  const int r0 = p.run_off[i], r1 = p.run_off[i + 1];
  const int q0 = estimate_only ? 0 : p.q_off[i];
  const int q1 = estimate_only ? 0 : p.q_off[i + 1];
  const int k = r1 - r0, q = q1 - q0, n_ent = k + q;
  const int max_new = p.max_new[i];
  const int cap = estimate_only ? 0 : p.capacity[i];
  int bad = 0;
  if (k < 0 || q < 0 || n_ent > p.max_entries) bad = PF_BAD_OFFSETS;
  else if (max_new < 1 || max_new > p.max_len) bad = PF_BAD_MAX_NEW;
  else if (cap < 0) bad = PF_BAD_CAPACITY;
  if (bad) {
    if (tid == 0) {
      raise_error(p.err, bad, i);
      if (!estimate_only) p.admitted_out[i] = -1;
      p.peak_out[i] = -1;
      if (p.peak_running_out) p.peak_running_out[i] = -1;
    }
    if (bad != PF_BAD_OFFSETS) {
      for (int e = tid; e < k; e += T)
        if (p.pred_run_out) p.pred_run_out[r0 + e] = -1;
      for (int e = tid; e < q; e += T)
        if (p.pred_q_out) p.pred_q_out[q0 + e] = -1;
    }
    return;
  }

  // ---- a3: the distribution P(l) of Eq.(eq:5) as a lookup structure
  int w = p.w;
  const int32_t* gC = nullptr;
  const int32_t* gS = nullptr;
  int64_t gid;
  if (LOOK == LOOK_GROUP) {
    const int g = p.dist_of[i];
    gC = p.gC + (int64_t)g * (p.max_len + 1);
    gS = p.gS + (int64_t)g * w;
    gid = (int64_t)g * p.members_per_group + p.member_base + (i - p.group_off[g]);
  } else {
    gid = p.instance_base + i;
  }
  for (int b = tid; b < p.n_bins; b += T) bin_cnt[b] = 0;
  if (LOOK == LOOK_SORTED) {
    const int32_t* src = p.sorted + (int64_t)i * w;
    for (int x = tid; x < w; x += T) table[x] = __ldg(src + x);
  } else if (LOOK == LOOK_HIST) {
    // C[l] = #{h ∈ L_h : h ≤ l}: inclusive scan of the persistent histogram.
    const int nb = p.max_len + 1;
    const int32_t* src = p.hist + (int64_t)i * nb;
    const int per = (nb + T - 1) / T;
    int run = 0;
    const int lo = tid * per;
    for (int x = lo; x < min(nb, lo + per); ++x) run += __ldg(src + x);
    int v[1] = {run}, tot[1];
    block_exclusive_add<T, 1>(v, tot, scratch);
    int acc = v[0];
    for (int x = lo; x < min(nb, lo + per); ++x) {
      acc += __ldg(src + x);
      table[x] = acc;
    }
  }
  __syncthreads();

  // ---- a4: predictions (Alg.1 lines 3-9), then (r, a, j) and coarse bins
  uint32_t key_fold = 0;
  if (p.mode == 0) {
    const uint64_t K = instance_key(p.seed, p.tick, gid);
    key_fold = (uint32_t)K ^ (uint32_t)(K >> 32);
  }
  uint64_t item[IPT];
  int item_bin[IPT], item_slot[IPT];
  int my_bad = 0;
#pragma unroll
  for (int m = 0; m < IPT; ++m) {
    const int e = tid + m * T;
    item[m] = 0;
    item_bin[m] = -1;
    if (e < n_ent) {
      int l_p, l_t, j;
      if (e < k) {
        l_p = p.input_len[r0 + e];
        l_t = p.generated[r0 + e];
        j = 0;
      } else {
        l_p = p.q_input_len[q0 + (e - k)];
        l_t = 0;
        j = e - k + 1;
      }
      if (l_p < 0 || l_p > p.max_input_len) my_bad = my_bad ? my_bad : PF_BAD_INPUT_LEN;
      if (l_t < 0 || l_t >= max_new) my_bad = my_bad ? my_bad : PF_BAD_GENERATED;
      l_t = min(max(l_t, 0), max_new - 1);  // keep lookups in range; outputs are discarded if bad
      const uint32_t u = (p.mode == 0) ? draw_u(key_fold, e, p.R) : p.quantile_u;
      int l_hat;
      if (LOOK == LOOK_SORTED) {
        const int base = upper_bound_smem(table, w, l_t);
        const int n_gt = w - base;
        l_hat = n_gt ? table[base + (int)__umulhi(u, (uint32_t)n_gt)] : max_new;
      } else if (LOOK == LOOK_HIST) {
        const int base = table[l_t];
        const int n_gt = w - base;
        if (n_gt == 0) {
          l_hat = max_new;
        } else {
          const int target = base + (int)__umulhi(u, (uint32_t)n_gt);
          int lo = l_t + 1, len = p.max_len - l_t;  // smallest L with C[L] > target
          while (len > 0) {
            int half = len >> 1;
            bool right = table[lo + half] <= target;
            lo = right ? lo + half + 1 : lo;
            len = right ? len - half - 1 : half;
          }
          l_hat = lo;
        }
      } else {
        const int base = __ldg(gC + l_t);
        const int n_gt = w - base;
        l_hat = n_gt ? __ldg(gS + base + (int)__umulhi(u, (uint32_t)n_gt)) : max_new;
      }
      l_hat = min(l_hat, max_new);
      if (e < k) {
        if (p.pred_run_out) p.pred_run_out[r0 + e] = l_hat;
      } else {
        if (p.pred_q_out) p.pred_q_out[q0 + (e - k)] = l_hat;
      }
      const int r = l_hat - l_t;  // ≥ 1
      const int a = l_p + l_t;
      item[m] = pack_entry(r, j, a);
      const int b = (p.max_len - r) >> p.bin_shift;  // descending r -> ascending bin
      item_bin[m] = b;
      item_slot[m] = atomicAdd(&bin_cnt[b], 1);
    }
  }
  if (__syncthreads_or(my_bad)) {
    // Data-dependent violation: outputs of this instance are −1.
    if (my_bad) raise_error(p.err, my_bad, i);
#pragma unroll
    for (int m = 0; m < IPT; ++m) {
      const int e = tid + m * T;
      if (e < k && p.pred_run_out) p.pred_run_out[r0 + e] = -1;
      if (e >= k && e < n_ent && p.pred_q_out) p.pred_q_out[q0 + (e - k)] = -1;
    }
    if (tid == 0) {
      if (!estimate_only) p.admitted_out[i] = -1;
      p.peak_out[i] = -1;
      if (p.peak_running_out) p.peak_running_out[i] = -1;
    }
    return;
  }

  // ---- a5: segmented sort by r descending — coarse counting pass, then exact
  // rank inside each bin (ties are irrelevant to every output, C-11).
  {
    const int per = (p.n_bins + T - 1) / T;
    const int lo = tid * per, hi = min(p.n_bins, lo + per);
    int s = 0;
    for (int b = lo; b < hi; ++b) s += bin_cnt[b];
    int v[1] = {s}, tot[1];
    block_exclusive_add<T, 1>(v, tot, scratch);
    int acc = v[0];
    for (int b = lo; b < hi; ++b) {
      bin_start[b] = acc;
      acc += bin_cnt[b];
    }
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < IPT; ++m)
    if (item_bin[m] >= 0) ent_tmp[bin_start[item_bin[m]] + item_slot[m]] = item[m];
  __syncthreads();
#pragma unroll
  for (int m = 0; m < IPT; ++m) {
    if (item_bin[m] < 0) continue;
    const int x = bin_start[item_bin[m]] + item_slot[m];
    const int lo = bin_start[item_bin[m]], hi = lo + bin_cnt[item_bin[m]];
    const int rv = ent_r(item[m]);
    int rank = 0;
    for (int y = lo; y < hi; ++y) {
      const int ry = ent_r(ent_tmp[y]);
      rank += (ry > rv) || (ry == rv && y < x);
    }
    ent_sorted[lo + rank] = item[m];
  }
  __syncthreads();

  // ---- a6: blocked scan over the sorted order. Keep (r, j, a) in registers.
  int rr[IPT], jj[IPT], aa[IPT];
  int sA_R = 0, sN_R = 0, sA = 0, sN = 0;
#pragma unroll
  for (int m = 0; m < IPT; ++m) {
    const int pos = tid * IPT + m;
    if (pos < n_ent) {
      const uint64_t e = ent_sorted[pos];
      rr[m] = ent_r(e);
      jj[m] = ent_j(e);
      aa[m] = ent_a(e);
    } else {
      rr[m] = 0;
      jj[m] = 0x7FFF;  // never included
      aa[m] = 0;
    }
    const bool in = pos < n_ent;
    const bool run = in && jj[m] == 0;
    sA_R += run ? aa[m] : 0;
    sN_R += run ? 1 : 0;
    sA += in ? aa[m] : 0;
    sN += in ? 1 : 0;
  }
  int v4[4] = {sA_R, sN_R, sA, sN}, t4[4];
  block_exclusive_add<T, 4>(v4, t4, scratch);
  int m0 = 0, mq = 0;
  {
    int A_R = v4[0], N_R = v4[1], A = v4[2], N = v4[3];
#pragma unroll
    for (int m = 0; m < IPT; ++m) {
      const int pos = tid * IPT + m;
      if (pos < n_ent) {
        const bool run = jj[m] == 0;
        A_R += run ? aa[m] : 0;
        N_R += run ? 1 : 0;
        A += aa[m];
        N += 1;
        m0 = max(m0, A_R + rr[m] * N_R);  // M_i of Eq.(eq:2), running batch only
        mq = max(mq, A + rr[m] * N);      // with the whole queue
      }
    }
  }
  const int M0 = block_max<T>(m0, scratch);  // Eq.(eq:3): M*(R)
  if (estimate_only) {
    if (tid == 0) p.peak_out[i] = M0;
    return;
  }
  const int Mq = block_max<T>(mq, scratch);

  // ---- a7: largest FIFO prefix that fits (Alg.1 lines 7-14). M*(p) is monotone
  // in p, so a binary search over p equals the sequential loop with early return.
  int p_star, peak;
  if (q == 0 || !fits(M0, cap, p.bp)) {
    p_star = 0;
    peak = M0;
  } else if (fits(Mq, cap, p.bp)) {
    p_star = q;
    peak = Mq;
  } else {
    int lo = 0, hi = q, m_lo = M0;  // fits(lo), !fits(hi)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      int s2[2] = {0, 0};
#pragma unroll
      for (int m = 0; m < IPT; ++m) {
        const bool in = jj[m] <= mid;
        s2[0] += in ? aa[m] : 0;
        s2[1] += in ? 1 : 0;
      }
      int t2[2];
      block_exclusive_add<T, 2>(s2, t2, scratch);
      int A = s2[0], N = s2[1], mx = 0;
#pragma unroll
      for (int m = 0; m < IPT; ++m) {
        const bool in = jj[m] <= mid;
        A += in ? aa[m] : 0;
        N += in ? 1 : 0;
        mx = max(mx, A + rr[m] * N);
      }
      const int M = block_max<T>(mx, scratch);
      if (fits(M, cap, p.bp)) {
        lo = mid;
        m_lo = M;
      } else {
        hi = mid;
      }
    }
    p_star = lo;
    peak = m_lo;
  }
  if (tid == 0) {
    p.admitted_out[i] = p_star;
    p.peak_out[i] = peak;
    if (p.peak_running_out) p.peak_running_out[i] = M0;
  }
}

}  // namespace pf
