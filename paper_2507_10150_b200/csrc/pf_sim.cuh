// pf_sim.cuh — batched continuous-batching simulator (the engine
// behind the paper's Table 1): one independent serving simulation per
// instance, all instances advanced one iteration per launch sequence. Each iteration
// (readings S-1..S-9):
//   sim_finish_kernel   S-2  finished requests leave, their lengths become completions
//   sim_scan_kernel          CSR offsets of completions / running / queue windows
//   sim_gather_kernel        CSR inputs of pf_update_history and the admission policy
//   (library)           S-2  pf_update_history (past-future only) — Eq.(eq:5) window
//   (library)           S-3  admission: admit_kernel (Alg.1, or the A12 override with true
//                            lengths) or baseline_kernel (aggressive / conservative)
//   sim_apply_kernel    S-4..S-8  join, true-length M* sample, LIFO overflow eviction,
//                            decode step, consumed-memory sample
// State per instance: a FIFO ring of request ids over its own request range (evicted
// requests are pushed back at the front), the running list in admission order (fixed
// stride E = max_entries), and per-request generated / eviction counters.
#pragma once
#include "pf_common.cuh"

namespace pf {

enum { SIM_PAST_FUTURE = 0, SIM_OPTIMUM = 1, SIM_AGGRESSIVE = 2, SIM_CONSERVATIVE = 3 };
enum { SIM_NMETRICS = 10 };
// metric columns
enum { SM_ITERS = 0, SM_DECODES, SM_EVICTIONS, SM_FINISHED, SM_CONSUMED, SM_FUTURE, SM_SAMPLES,
       SM_FUTURE_MAX, SM_FORCED, SM_ADMISSIONS };

struct SimState {
  int n, E;
  const int32_t* req_off;   // [n+1]
  const int32_t* req_lp;    // [N]
  const int32_t* req_L;     // [N] true output lengths
  const int32_t* capacity;  // [n]
  int32_t* gen;             // [N] generated tokens
  int32_t* evc;             // [N] evictions per request
  int32_t* qbuf;            // [N] ring of request ids (instance i: its own request range)
  int32_t* qhead;           // [n] ring position of the queue head (relative)
  int32_t* qlen;            // [n]
  int32_t* run_ids;         // [n × E] running list, admission order (global request ids)
  int32_t* run_k;           // [n]
  int32_t* done;            // [n]
  int32_t* comp_tmp;        // [n × E]
  int32_t* cnt;             // [3n]: completions, running k, queue window per instance
  int32_t* off;             // [3(n+1)]: comp_off, run_off, q_off
  int32_t* comp_len;        // [n × E] CSR
  int32_t* c_lp;            // [n × E] CSR running l_p
  int32_t* c_gen;           // [n × E] CSR running l_t
  int32_t* c_lhat;          // [n × E] CSR running true l̂ (optimum policy)
  int32_t* q_lp;            // [n × E] CSR queued l_p + generated
  int32_t* q_lhat;          // [n × E] CSR queued remaining true length (optimum policy)
  int32_t* admitted;        // [n]
  long long* metrics;       // [n × SIM_NMETRICS]
  int* err;                 // sticky device error word of the library context
};

__device__ __forceinline__ int warp_excl(int v, int lane, int& total) {
  const int inc = warp_inclusive_add(v, lane);
  total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

// S-2: remove finished requests (stable), emit their lengths as completions.
__global__ void __launch_bounds__(256) sim_finish_kernel(SimState s) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= s.n) return;
  int* cnt = s.cnt;
  if (s.done[i]) {
    if (lane == 0) cnt[i] = cnt[s.n + i] = cnt[2 * s.n + i] = 0;
    return;
  }
  int32_t* run = s.run_ids + (int64_t)i * s.E;
  const int k = s.run_k[i];
  int n_comp = 0, n_keep = 0;
  for (int x0 = 0; x0 < k; x0 += 32) {  // stable compaction in chunks of 32
    const int x = x0 + lane;
    int id = -1, fin = 0;
    if (x < k) {
      id = run[x];
      fin = s.gen[id] == s.req_L[id];
    }
    const unsigned mf = __ballot_sync(0xffffffffu, x < k && fin);
    const unsigned mk = __ballot_sync(0xffffffffu, x < k && !fin);
    const unsigned below = (1u << lane) - 1u;
    __syncwarp();
    if (x < k && fin) s.comp_tmp[(int64_t)i * s.E + n_comp + __popc(mf & below)] = s.req_L[id];
    if (x < k && !fin) run[n_keep + __popc(mk & below)] = id;  // n_keep + rank ≤ x: in place
    n_comp += __popc(mf);
    n_keep += __popc(mk);
    __syncwarp();
  }
  const int ql = s.qlen[i];
  if (lane == 0) {
    long long* m = s.metrics + (int64_t)i * SIM_NMETRICS;
    m[SM_FINISHED] += n_comp;
    s.run_k[i] = n_keep;
    cnt[i] = n_comp;  // completions are recorded even on the iteration that ends the run
    if (n_keep == 0 && ql == 0) {
      s.done[i] = 1;  // S-9
      cnt[s.n + i] = cnt[2 * s.n + i] = 0;
    } else {
      m[SM_ITERS] += 1;
      cnt[s.n + i] = n_keep;
      cnt[2 * s.n + i] = ::min(ql, ::max(0, s.E - n_keep));
    }
  }
}

// Exclusive scans of the three count vectors (one CTA; n is a simulator sweep size).
__global__ void __launch_bounds__(1024) sim_scan_kernel(int n, const int32_t* cnt, int32_t* off) {
  __shared__ int scratch[3 * 32];
  int carry[3] = {0, 0, 0};
  for (int x0 = 0; x0 < n; x0 += 1024) {
    const int x = x0 + threadIdx.x;
    int v[3], tot[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) v[c] = x < n ? cnt[c * n + x] : 0;
    block_exclusive_add<1024, 3>(v, tot, scratch);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (x < n) off[c * (n + 1) + x] = carry[c] + v[c];
      carry[c] += tot[c];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) off[c * (n + 1) + n] = carry[c];
}

// CSR inputs: completions, running (l_p, l_t, true l̂), queue window (l_p + l_t, remaining).
__global__ void __launch_bounds__(256) sim_gather_kernel(SimState s) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= s.n) return;
  const int n1 = s.n + 1;
  const int c0 = s.off[i], c1 = s.off[i + 1];
  const int r0 = s.off[n1 + i], r1 = s.off[n1 + i + 1];
  const int q0 = s.off[2 * n1 + i], q1 = s.off[2 * n1 + i + 1];
  for (int x = lane; x < c1 - c0; x += 32) s.comp_len[c0 + x] = s.comp_tmp[(int64_t)i * s.E + x];
  const int32_t* run = s.run_ids + (int64_t)i * s.E;
  for (int x = lane; x < r1 - r0; x += 32) {
    const int id = run[x];
    s.c_lp[r0 + x] = s.req_lp[id];
    s.c_gen[r0 + x] = s.gen[id];
    s.c_lhat[r0 + x] = s.req_L[id];
  }
  const int base = s.req_off[i], nreq = s.req_off[i + 1] - base;
  const int qh = s.qhead[i];
  for (int x = lane; x < q1 - q0; x += 32) {
    int pos = qh + x;
    if (pos >= nreq) pos -= nreq;
    const int id = s.qbuf[base + pos];
    const int g = s.gen[id];
    s.q_lp[q0 + x] = s.req_lp[id] + g;      // S-3: re-queued requests recompute l_t tokens
    s.q_lhat[q0 + x] = s.req_L[id] - g;     // optimum: remaining true length
  }
}

// S-4..S-8 after the admission decision.
__global__ void __launch_bounds__(256) sim_apply_kernel(SimState s) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= s.n || s.done[i]) return;
  long long* m = s.metrics + (int64_t)i * SIM_NMETRICS;
  int32_t* run = s.run_ids + (int64_t)i * s.E;
  const int base = s.req_off[i], nreq = s.req_off[i + 1] - base;
  int k = s.run_k[i], qh = s.qhead[i], ql = s.qlen[i];
  int p = s.admitted[i];
  if (p < 0) {  // the admission call rejected this instance's data: stop it, keep the error
    if (lane == 0) {
      raise_error(s.err, PF_BAD_OFFSETS, i);
      s.done[i] = 1;
    }
    return;
  }
  // S-4: FIFO prefix joins the running list; an empty batch takes the head regardless
  bool forced = false;
  if (p == 0 && k == 0 && ql > 0) { p = 1; forced = true; }
  for (int x = lane; x < p; x += 32) {
    int pos = qh + x;
    if (pos >= nreq) pos -= nreq;
    run[k + x] = s.qbuf[base + pos];
  }
  __syncwarp();
  qh += p;
  if (qh >= nreq) qh -= nreq;
  ql -= p;
  k += p;
  // S-5: future required memory with true remaining lengths, M* = max over entries x of
  // T(r_x) = Σ_{y: r_y ≥ r_x} (a_y + r_x)  (Eq.(eq:1)-(eq:3); T is maximal at some r_x)
  long long fut = 0;
  for (int x = lane; x < k; x += 32) {
    const int idx = run[x];
    const int rx = s.req_L[idx] - s.gen[idx];
    long long t = 0;
    for (int y = 0; y < k; ++y) {
      const int idy = run[y];
      const int gy = s.gen[idy];
      const int ry = s.req_L[idy] - gy;
      if (ry >= rx) t += (long long)s.req_lp[idy] + gy + rx;
    }
    fut = ::max(fut, t);
  }
  // S-6 demand of the next decode step; S-8 consumed after it
  long long demand = 0;
  for (int x = lane; x < k; x += 32) {
    const int id = run[x];
    demand += (long long)s.req_lp[id] + s.gen[id] + 1;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    fut = ::max(fut, (long long)__shfl_xor_sync(0xffffffffu, fut, d));
    demand += __shfl_xor_sync(0xffffffffu, demand, d);
  }
  int n_ev = 0;
  if (lane == 0) {  // LIFO eviction, re-queued at the front (rare; sequential)
    const long long M = s.capacity[i];
    while (demand > M && k > 1) {
      const int id = run[--k];
      demand -= (long long)s.req_lp[id] + s.gen[id] + 1;
      qh = qh == 0 ? nreq - 1 : qh - 1;
      s.qbuf[base + qh] = id;
      ++ql;
      s.evc[id] += 1;
      ++n_ev;
    }
  }
  k = __shfl_sync(0xffffffffu, k, 0);
  __syncwarp();
  // S-7 decode step
  for (int x = lane; x < k; x += 32) s.gen[run[x]] += 1;
  if (lane == 0) {
    const long long used = demand;  // Σ(l_p + l_t + 1) before the step = Σ(l_p + l_t) after
    m[SM_DECODES] += k > 0 ? 1 : 0;
    m[SM_EVICTIONS] += n_ev;
    m[SM_CONSUMED] += used;
    m[SM_FUTURE] += fut;
    m[SM_SAMPLES] += 1;
    m[SM_FUTURE_MAX] = ::max(m[SM_FUTURE_MAX], fut);
    m[SM_FORCED] += forced ? 1 : 0;
    m[SM_ADMISSIONS] += p;
    s.run_k[i] = k;
    s.qhead[i] = qh;
    s.qlen[i] = ql;
  }
}

// Initial state: queue = every request in list order, nothing running.
__global__ void sim_init_kernel(SimState s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const int base = s.req_off[i], nreq = s.req_off[i + 1] - base;
  for (int x = 0; x < nreq; ++x) {
    s.qbuf[base + x] = base + x;
    s.gen[base + x] = 0;
    s.evc[base + x] = 0;
  }
  s.qhead[i] = 0;
  s.qlen[i] = nreq;
  s.run_k[i] = 0;
  s.done[i] = 0;
  for (int c = 0; c < SIM_NMETRICS; ++c) s.metrics[(int64_t)i * SIM_NMETRICS + c] = 0;
}

__global__ void sim_count_done_kernel(int n, const int32_t* done, int32_t* out) {
  int c = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) c += done[i] != 0;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&acc, c);
  __syncthreads();
  if (threadIdx.x == 0) *out = acc;
}

}  // namespace pf
