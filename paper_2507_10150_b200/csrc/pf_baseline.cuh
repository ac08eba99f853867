// pf_baseline.cuh — the comparison admission policies of the paper's evaluation
// (§5.3, Table 1 rows PAPER.md:345-349; described at PAPER.md:102, :138), batched
// over instances on the same boundary as pf_admit:
//   aggressive   "batches requests solely based on input lengths" up to a watermark:
//                admit the FIFO head while Σ_running(l_p + l_t) + Σ_admitted l_p ≤ wm·M
//   conservative "the sum of request input lengths and the max_new_tokens", optionally
//                over-committed (":379 assumes 1.5 times the actual memory capacity"):
//                admit while Σ_{running ∪ admitted}(l_p + max_new) ≤ oc·M
// Ratios in basis points, compared exactly as 10^4·used ≤ ratio·M in int64; early
// return at the first failure (FIFO prefix, like Alg.1). One warp per instance.
#pragma once
#include "pf_common.cuh"

namespace pf {

enum { POLICY_AGGRESSIVE = 1, POLICY_CONSERVATIVE = 2 };

// requests per lane per chunk of the streaming loops
#ifndef PF_BASE_NC
#define PF_BASE_NC 4
#endif

struct BaselineParams {
  int n;
  int policy;
  int ratio_bp;
  int max_len, max_input_len, max_entries;
  const int32_t* run_off;
  const int32_t* input_len;
  const int32_t* generated;
  const int32_t* q_off;
  const int32_t* q_input_len;
  const int32_t* max_new;
  const int32_t* capacity;
  int32_t* admitted_out;
  int32_t* used_out;
  int32_t* err;
};

__global__ void __launch_bounds__(256) baseline_kernel(BaselineParams p) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= p.n) return;
  const int r0 = p.run_off[i], r1 = p.run_off[i + 1], q0 = p.q_off[i], q1 = p.q_off[i + 1];
  const int k = r1 - r0, q = q1 - q0;
  const int max_new = p.max_new[i], cap = p.capacity[i];
  int bad = 0;
  if (k < 0 || q < 0 || k + q > p.max_entries) bad = PF_BAD_OFFSETS;
  else if (max_new < 1 || max_new > p.max_len) bad = PF_BAD_MAX_NEW;
  else if (cap < 0) bad = PF_BAD_CAPACITY;
  const bool cons = p.policy == POLICY_CONSERVATIVE;
  // running requests: current consumption (aggressive) or budgets (conservative). The
  // rows are streamed 4 requests per lane per chunk with the chunk's loads issued
  // together (no loop-carried dependence on the loaded values); a lane keeps its first
  // data error in row order.
  int base = 0;
  if (!bad) {
    int lb = 0;
    const int32_t* lpR = p.input_len + r0;
    const int32_t* ltR = p.generated + r0;
#pragma unroll 1
    for (int e0 = lane; e0 < k; e0 += 32 * PF_BASE_NC) {
      int lp[PF_BASE_NC], lt[PF_BASE_NC];
#pragma unroll
      for (int c = 0; c < PF_BASE_NC; ++c) {
        const int e = e0 + 32 * c;
        lp[c] = e < k ? __ldg(lpR + e) : 0;
        lt[c] = e < k ? __ldg(ltR + e) : 0;
      }
#pragma unroll
      for (int c = 0; c < PF_BASE_NC; ++c) {
        const int code = (lp[c] < 0 || lp[c] > p.max_input_len) ? PF_BAD_INPUT_LEN
                         : (lt[c] < 0 || lt[c] >= max_new)       ? PF_BAD_GENERATED : 0;
        lb = lb ? lb : code;
        base += cons ? (e0 + 32 * c < k ? lp[c] + max_new : 0) : lp[c] + lt[c];
      }
    }
    const int32_t* lpQ = p.q_input_len + q0;
#pragma unroll 1
    for (int j0 = lane; j0 < q; j0 += 32 * PF_BASE_NC) {
      int lp[PF_BASE_NC];
#pragma unroll
      for (int c = 0; c < PF_BASE_NC; ++c) lp[c] = j0 + 32 * c < q ? __ldg(lpQ + j0 + 32 * c) : 0;
#pragma unroll
      for (int c = 0; c < PF_BASE_NC; ++c)
        if (!lb && (lp[c] < 0 || lp[c] > p.max_input_len)) lb = PF_BAD_INPUT_LEN;
    }
    bad = lb;
  }
  bad = __reduce_max_sync(0xffffffffu, bad);
  if (bad) {
    if (lane == 0) {
      raise_error(p.err, bad, i);
      p.admitted_out[i] = -1;
      if (p.used_out) p.used_out[i] = -1;
    }
    return;
  }
  base = (int)__reduce_add_sync(0xffffffffu, (unsigned)base);
  const int64_t limit = (int64_t)p.ratio_bp * cap;  // fits ⟺ 10^4·used ≤ limit
  int admitted = q, used = base;
  for (int j0 = 0; j0 < q; j0 += 32) {
    const int j = j0 + lane;
    const int wgt = j < q ? p.q_input_len[q0 + j] + (cons ? max_new : 0) : 0;
    const int incl = warp_inclusive_add(wgt, lane);
    const bool over = j < q && (int64_t)(base + incl) * 10000 > limit;
    const unsigned m = __ballot_sync(0xffffffffu, over);
    if (m) {  // the first failing candidate ends the FIFO prefix
      const int f = __ffs(m) - 1;
      admitted = j0 + f;
      used = base + __shfl_sync(0xffffffffu, incl - wgt, f);
      break;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
    used = base;
  }
  if (lane == 0) {
    p.admitted_out[i] = admitted;
    if (p.used_out) p.used_out[i] = used;
  }
}

}  // namespace pf
