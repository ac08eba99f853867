// pf_forward.cuh — cross-instance request forwarding by M* headroom (SURVEY §8(f)
// NEXT-4; the paper's future work). Readings F-1..F-4:
// requests of a cluster's FIFO queue go, one at a time, to the instance that can take
// them under Alg.1's check with the largest headroom; the first request
// no instance can take stops forwarding (C-14).
//
// One CTA per cluster, one warp per instance. Each warp keeps its instance's entries
// (R_s ∪ F_s) sorted by r descending in shared memory as (r_t, T_t) with
// T_t = A_t + r_t·(t+1), A_t = Σ_{u≤t} a_u — the Eq.(eq:1)-(eq:3) sort form, so
// M* = max_t T_t. Adding (a, r) at position p = #{t : r_t ≥ r} gives, exactly,
//   M*' = max( max_{t<p} T_t,  A_{p−1} + a + r·(p+1),  max_{t≥p} (T_t + r_t) + a )
// (entries after p move one place down and gain a), one warp reduction per candidate;
// the chosen warp then inserts (shift + the same update) — O(m/32) per step.
#pragma once
#include "pf_common.cuh"

namespace pf {

struct ForwardParams {
  int n_clusters, S, E, w, max_len, max_input_len, mode, bp;
  uint32_t quantile_u, tick;
  uint64_t seed;
  int64_t instance_base;
  const int32_t* sorted;  // [n × w] ascending windows (LAYOUT_SORTED)
  const int32_t* run_off;
  const int32_t* input_len;
  const int32_t* generated;
  const int32_t* max_new;
  const int32_t* capacity;
  const int32_t* cq_off;
  const int32_t* cq_input_len;
  int32_t* dest_out;
  int32_t* forwarded_out;
  int32_t* peak_out;
  int* err;
};

// l̂ from the sorted window S[0..w) (C-3..C-6): base = #{h ≤ l_t}, n_gt = w − base.
__device__ __forceinline__ int fw_predict(const int32_t* S, int w, int l_t, int max_new, uint32_t u) {
  int lo = 0, len = w;
  while (len > 0) {
    const int half = len >> 1;
    const bool right = __ldg(S + lo + half) <= l_t;
    lo = right ? lo + half + 1 : lo;
    len = right ? len - half - 1 : half;
  }
  const int n_gt = w - lo;
  if (n_gt == 0) return max_new;
  return ::min(__ldg(S + lo + (int)__umulhi(u, (uint32_t)n_gt)), max_new);
}

struct FwdList {
  int* r;
  int* T;
  int m;
};

// Candidate M*' of adding (a, r) to the warp's list (all lanes return the same value).
__device__ __forceinline__ int fw_peak_with(const FwdList& L, int a, int r, int lane) {
  // p = #{t : r_t ≥ r} (r_t descending)
  int p = 0;
  for (int t0 = 0; t0 < L.m; t0 += 32) {
    const int t = t0 + lane;
    p += __popc(__ballot_sync(0xffffffffu, t < L.m && L.r[t] >= r));
  }
  int best = 0;
  for (int t = lane; t < L.m; t += 32) best = ::max(best, t < p ? L.T[t] : L.T[t] + L.r[t] + a);
  best = __reduce_max_sync(0xffffffffu, best);
  const int Aprev = p > 0 ? L.T[p - 1] - L.r[p - 1] * p : 0;
  return ::max(best, Aprev + a + r * (p + 1));
}

__device__ __forceinline__ void fw_insert(FwdList& L, int a, int r, int lane) {
  int p = 0;
  for (int t0 = 0; t0 < L.m; t0 += 32) {
    const int t = t0 + lane;
    p += __popc(__ballot_sync(0xffffffffu, t < L.m && L.r[t] >= r));
  }
  const int Aprev = p > 0 ? L.T[p - 1] - L.r[p - 1] * p : 0;
  // shift [p, m) down by one, from the back in warp-sized blocks
  for (int t1 = L.m; t1 > p; t1 -= 32) {
    const int t = t1 - 1 - lane;
    int rv = 0, tv = 0;
    const bool in = t >= p;
    if (in) { rv = L.r[t]; tv = L.T[t]; }
    __syncwarp();
    if (in) { L.r[t + 1] = rv; L.T[t + 1] = tv + a + rv; }
    __syncwarp();
  }
  if (lane == 0) {
    L.r[p] = r;
    L.T[p] = Aprev + a + r * (p + 1);
  }
  __syncwarp();
  L.m += 1;
}

__global__ void __launch_bounds__(1024) forward_kernel(ForwardParams P) {
  extern __shared__ int fsm[];
  __shared__ long long cand_h[32];
  __shared__ int cand_ok[32], chosen, bad_cluster;
  const int c = blockIdx.x;
  const int s = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = P.S;
  const int i = c * S + s;
  FwdList L{fsm + (size_t)s * 2 * P.E, fsm + (size_t)s * 2 * P.E + P.E, 0};
  if (threadIdx.x == 0) bad_cluster = 0;
  __syncthreads();
  const int r0 = P.run_off[i], k = P.run_off[i + 1] - r0;
  const int max_new = P.max_new[i], cap = P.capacity[i];
  const int q0 = P.cq_off[c], q = P.cq_off[c + 1] - q0;
  int bad = 0;
  if (k < 0 || k > P.E || q < 0) bad = PF_BAD_OFFSETS;
  else if (max_new < 1 || max_new > P.max_len) bad = PF_BAD_MAX_NEW;
  else if (cap < 0) bad = PF_BAD_CAPACITY;
  for (int e = lane; !bad && e < k; e += 32) {
    const int lp = P.input_len[r0 + e], lt = P.generated[r0 + e];
    if ((unsigned)lp > (unsigned)P.max_input_len) bad = PF_BAD_INPUT_LEN;
    else if ((unsigned)lt >= (unsigned)max_new) bad = PF_BAD_GENERATED;
  }
  for (int j = lane; !bad && s == 0 && j < q; j += 32)
    if ((unsigned)P.cq_input_len[q0 + j] > (unsigned)P.max_input_len) bad = PF_BAD_INPUT_LEN;
  bad = __reduce_max_sync(0xffffffffu, bad);
  if (bad && lane == 0) {
    raise_error(P.err, bad, i);
    atomicOr(&bad_cluster, 1);
  }
  __syncthreads();
  if (bad_cluster) {
    for (int j = threadIdx.x; j < q; j += blockDim.x) P.dest_out[q0 + j] = -1;
    if (lane == 0) P.peak_out[i] = -1;
    if (threadIdx.x == 0) P.forwarded_out[c] = -1;
    return;
  }
  // running requests: Alg.1 lines 3-6 with the instance's key and slots (F-2)
  const uint64_t K = instance_key(P.seed, P.tick, P.instance_base + i);
  const uint32_t kf = (uint32_t)K ^ (uint32_t)(K >> 32);
  const int32_t* Sw = P.sorted + (int64_t)i * P.w;
  for (int e = 0; e < k; ++e) {  // sequential inserts keep the list sorted
    const int lt = P.generated[r0 + e];
    const uint32_t u = P.mode ? P.quantile_u : lowbias32(kf ^ ((uint32_t)e * 0x9E3779B9U));
    const int lh = fw_predict(Sw, P.w, lt, max_new, u);
    fw_insert(L, P.input_len[r0 + e] + lt, lh - lt, lane);
  }
  int forwarded = 0;
  bool stopped = false;
  for (int j = 0; j < q; ++j) {
    if (stopped) {
      if (threadIdx.x == 0) P.dest_out[q0 + j] = -1;
      continue;
    }
    const int a = P.cq_input_len[q0 + j];
    int lh = 0;
    if (L.m < P.E) {  // F-1: a full instance cannot take requests
      const uint32_t u = P.mode ? P.quantile_u : lowbias32(kf ^ ((uint32_t)(k + j) * 0x9E3779B9U));
      lh = fw_predict(Sw, P.w, 0, max_new, u);  // Alg.1 line 8, C-16
      const int m = fw_peak_with(L, a, lh, lane);
      if (lane == 0) {
        cand_h[s] = (long long)(10000 - P.bp) * cap - 10000LL * m;
        cand_ok[s] = cand_h[s] >= 0;
      }
    } else if (lane == 0) {
      cand_ok[s] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int best = -1;
      for (int x = 0; x < S; ++x)
        if (cand_ok[x] && (best < 0 || cand_h[x] > cand_h[best])) best = x;
      chosen = best;
      P.dest_out[q0 + j] = best;
    }
    __syncthreads();
    const int b = chosen;
    if (b < 0) {
      stopped = true;
    } else {
      ++forwarded;
      if (b == s) fw_insert(L, a, lh, lane);
    }
    __syncthreads();
  }
  int pk = 0;
  for (int t = lane; t < L.m; t += 32) pk = ::max(pk, L.T[t]);
  pk = __reduce_max_sync(0xffffffffu, pk);
  if (lane == 0) P.peak_out[i] = pk;
  if (threadIdx.x == 0) P.forwarded_out[c] = forwarded;
}

}  // namespace pf
