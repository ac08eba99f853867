// pf_admit_group.cuh — the shared-mode admit kernel of libpfsched (sm_100a): config 5's
// path (shared group histories, one-warp teams, packed bins). Same method and outputs as
// admit_kernel<1, LOOK_GROUP, PK> in pf_admit.cuh (a4 prediction, a5/a6 sort-free M*,
// a7 cutting-plane admission; header comment there), organised for the fewest issued
// instructions per instance, because that — not DRAM — bounds this path:
//
//  * Persistent: one CTA of up to 32 one-warp teams per SM walks a contiguous, group-major
//    instance range; per group segment it stages C_g and S_g (u16, with the S_g[W]
//    sentinel) in shared memory, so the two dependent lookups of a running request are
//    shared-memory gathers (≈ 3-4 bank wavefronts) instead of L1 gathers over 30 KB of
//    tables (≈ 9 wavefronts each). Warps take instances from a shared counter.
//  * Running and queued requests in separate loops without per-request guards: the tail
//    chunk clamps its load index and predicates only its stores and atomics. A queued
//    request has l_t = 0 and C_g[0] = 0 (history lengths are ≥ 1), so its prediction is
//    one lookup S_g[⌊u·W / 2^32⌋] (Alg.1 l.3-9 with l_t = 0, C-16).
//  * 32-bit capacity threshold and one 64-bit key per instance.
#pragma once
#include "pf_admit.cuh"

namespace pf {

// Running requests per lane per full chunk.
#ifndef PF_GNC
#define PF_GNC 4
#endif

// Non-inlined slow draw (quantile mode or R ≠ 1; C-8/C-9), kept out of the hot loop's code.
__device__ __noinline__ uint32_t draw_slow(const AdmitParams& p, uint32_t key_fold, int e, int R) {
  return (p.mode != 0) ? p.quantile_u : draw_u(key_fold, e, R);
}

__device__ __forceinline__ uint32_t sh_addr(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
// Predicated (p = false: no access) streaming load, shared-memory stores and atomics.
__device__ __forceinline__ int ld_stream_if(const int32_t* a, bool p) {
  int v;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b32 %0, 0;\n"
               " @q ld.global.nc.L1::no_allocate.b32 %0, [%1];\n}" : "=r"(v) : "l"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ void sts_u32_if(uint32_t a, uint32_t v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.u32 [%0], %1;\n}"
               :: "r"(a), "r"(v), "r"((int)p) : "memory");
}
__device__ __forceinline__ void sts_u16_if(uint32_t a, uint32_t v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.u16 [%0], %1;\n}"
               :: "r"(a), "h"((unsigned short)v), "r"((int)p) : "memory");
}
__device__ __forceinline__ uint32_t atom_exch_sh_if(uint32_t a, uint32_t v, bool p) {
  uint32_t old;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q atom.shared.exch.b32 %0, [%1], %2;\n}"
               : "=r"(old) : "r"(a), "r"(v), "r"((int)p) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_sh_if(uint32_t a, uint32_t v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q red.shared.add.u32 [%0], %1;\n}"
               :: "r"(a), "r"(v), "r"((int)p) : "memory");
}

__device__ __forceinline__ uint32_t atom_exch_sh(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_sh(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_sh(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}

// Bulk L2 prefetch (TMA) of n int32 elements from a (rounded out to 16-byte boundaries).
#ifndef PF_AHEAD
#define PF_AHEAD 32
#endif
__device__ __forceinline__ void prefetch_l2(const int32_t* a, int n) {
  if (n <= 0) return;
  const uint64_t lo = reinterpret_cast<uint64_t>(a) & ~uint64_t(15);
  const uint64_t hi = (reinterpret_cast<uint64_t>(a + n) + 15) & ~uint64_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
}

// One inclusive-scan step: v += (value of lane − d) when that lane exists (the shuffle's own
// in-range predicate guards the add: no lane compare, no select).
__device__ __forceinline__ uint32_t scan_step(uint32_t v, int d) {
  asm volatile("{\n .reg .pred p;\n .reg .b32 t;\n shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n"
               " @p add.u32 %0, %0, t;\n}" : "+r"(v) : "r"(d));
  return v;
}
__device__ __forceinline__ uint32_t warp_incl_u32(uint32_t v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) v = scan_step(v, d);
  return v;
}

__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t x;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(a), "r"(b), "r"(c));
  return x;
}

// Per-team shared memory (bytes, in order; the same team_smem as admit_kernel's PACK layout):
//   rb[ent_cap] u32 records r | a << 13 (slot e: running e < k, queued k + j)
//   nx[ent_cap] u16 per-bin request lists, hd[128] u32 list heads
//   binR[128], binQ[128] u32 packed (A << PK | N) per r-bin, xs[140] i32 scratch
template <int PK, bool EST>
__device__ __forceinline__ void group_one(const AdmitParams& p, const int lane, unsigned char* base,
                                          const int i, const uint16_t* sC, const uint16_t* sS,
                                          const int64_t gid_base, const int* pf_ctl) {
  constexpr int NB = 128;
  constexpr int NSH = PK;
  constexpr uint32_t NMASK = (1u << NSH) - 1u;
  uint32_t* rb = reinterpret_cast<uint32_t*>(base);
  uint16_t* nx = reinterpret_cast<uint16_t*>(rb + p.ent_cap);
  uint32_t* hd = reinterpret_cast<uint32_t*>(nx + p.ent_cap);
  uint32_t* binR = hd + NB;
  uint32_t* binQ = binR + NB;
  int* xs = reinterpret_cast<int*>(binQ + NB);
  int* cand = xs + 40;  // [0]: count, then 6 ints per candidate (≤ 16)
  auto ent_r = [&](int e) -> int { return (int)(rb[e] & 0x1FFFu); };
  auto ent_a = [&](int e) -> int { return (int)(rb[e] >> 13); };
  constexpr bool estimate_only = EST;  // pf_estimate_peak (no queue, no capacity)

  // ---- instance scalars and CSR validation
  const int r0 = __ldg(p.run_off + i), r1 = __ldg(p.run_off + i + 1);
  const int q0 = estimate_only ? 0 : __ldg(p.q_off + i);
  const int q1 = estimate_only ? 0 : __ldg(p.q_off + i + 1);
  const int max_new = p.max_new ? __ldg(p.max_new + i) : p.max_len;
  const int cap = estimate_only ? 0 : __ldg(p.capacity + i);
  const int k = r1 - r0, q = q1 - q0, n_ent = k + q;
  {
    int bad = 0;
    if (k < 0 || q < 0 || n_ent > p.max_entries) bad = PF_BAD_OFFSETS;
    else if (max_new < 1 || max_new > p.max_len) bad = PF_BAD_MAX_NEW;
    else if (cap < 0) bad = PF_BAD_CAPACITY;
    if (bad) {
      if (lane == 0) {
        raise_error(p.err, bad, i);
        if (!estimate_only) p.admitted_out[i] = -1;
        p.peak_out[i] = -1;
        if (p.peak_running_out) p.peak_running_out[i] = -1;
      }
      if (bad != PF_BAD_OFFSETS) {
        if (p.pred_run_out)
          for (int e = lane; e < k; e += 32) p.pred_run_out[r0 + e] = -1;
        if (p.pred_q_out)
          for (int e = lane; e < q; e += 32) p.pred_q_out[q0 + e] = -1;
      }
      return;
    }
  }
  // L2 prefetch of the request rows PF_AHEAD instances ahead in this CTA's stream (its range
  // is contiguous in the CSR arrays): every instance prefetches about one instance's rows
  // at (its own rows + PF_AHEAD mean-instance sizes), so the warps together keep the stream
  // in L2 ahead of their loads (the first chunk of an instance otherwise waits a DRAM trip).
  if (PF_AHEAD > 0 && lane == 0) {
    const int d = pf_ctl[0], rend = pf_ctl[2];
    const int a = ::min(r0 + d, rend), b = ::min(r1 + d, rend);
    prefetch_l2(p.input_len + a, b - a);
    prefetch_l2(p.generated + a, b - a);
    if (!EST) {
      const int dq = pf_ctl[1], qend = pf_ctl[3];
      const int c = ::min(q0 + dq, qend), e = ::min(q1 + dq, qend);
      prefetch_l2(p.q_input_len + c, e - c);
    }
  }
  // C = ⌊(10^4 − bp)·cap / 10^4⌋ in 32-bit arithmetic (C-12, C-13): cap = 10^4·Q + R gives
  // m·Q + ⌊m·R / 10^4⌋ with m ≤ 10^4, so every term stays below 2^31.
  int Cmax = 0;
  if (!estimate_only) {
    const uint32_t m = 10000u - (uint32_t)p.bp, cu = (uint32_t)cap;
    Cmax = (int)(m * (cu / 10000u) + (m * (cu % 10000u)) / 10000u);
  }
  {  // zero the bins, empty lists
    uint4* z4 = reinterpret_cast<uint4*>(binR);  // binR and binQ are contiguous
    z4[lane] = make_uint4(0, 0, 0, 0);
    z4[lane + 32] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(hd)[lane] = make_uint4(~0u, ~0u, ~0u, ~0u);
  }
  uint32_t key_fold = 0;
  if (p.mode == 0) {
    const uint64_t K = instance_key(p.seed, p.tick, gid_base + i);
    key_fold = (uint32_t)K ^ (uint32_t)(K >> 32);
  }
  // R = 0: adaptive repetitions max(1, ⌈64/k⌉) (SPEC.md:161 reading of PAPER.md:295)
  const int R = p.R > 0 ? p.R : (k > 0 ? ::max(1, (64 + k - 1) / k) : 64);
  const bool draw_fast = (p.mode == 0) && (R == 1);
  const uint32_t W = (uint32_t)p.w;
  const uint32_t lpmax = (uint32_t)p.max_input_len;
  __syncwarp();

  // ---- a4 (Alg.1 l.3-9): l̂ = min(S_g[b + ⌊u·(W − b)/2^32⌋], max_new) with b = C_g[l_t]
  // (S_g[W] = 0xFFFF when every history length ≤ l_t, C-5; C-6 clamp); then r = l̂ − l_t,
  // a = l_p + l_t, the record, the push on the r-bin's list and the bin's (A, N).
  // Chunks of NC requests per lane (slot e = e0 + 32·c + lane): the loads first, then every
  // request's two dependent lookups, then the stores. FULL chunks carry no guards; the
  // ragged tail chunk predicates its loads (0 when out of range), stores and atomics.
  // Queued requests (slot k + j) have l_t = 0, so b = C_g[0] (= 0: history lengths ≥ 1)
  // is one shared value and the prediction is one lookup.
  // validation by running maxima of the unsigned inputs (negative values wrap above any
  // bound): bad iff max l_p > max_input_len or max l_t ≥ max_new (one VIMNMX per input)
  uint32_t mx_lp = 0, mx_lt = 0;
  const uint32_t mx1 = (uint32_t)(max_new - 1);
  const uint32_t bq0 = sC[0];
  const uint32_t a_rb = sh_addr(rb), a_nx = sh_addr(nx), a_hd = sh_addr(hd);
  // xs[lane]: this lane's sink for masked tail atomics (one word per lane, so masked lanes
  // never serialise on one address)
  const uint32_t a_dummy = sh_addr(xs + lane);
  auto chunk = [&](const int e0, const int n, const int32_t* lpp, const int32_t* ltp,
                   int32_t* po_base, uint32_t* bins, auto full_tag, auto fast_tag, auto nc_tag,
                   auto run_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    constexpr bool FAST = decltype(fast_tag)::value;  // sampling mode, R = 1
    constexpr int NC = decltype(nc_tag)::value;
    constexpr bool RUN = decltype(run_tag)::value;   // running (l_t loaded) or queued
    int lp[NC], lt[NC], lh[NC];
    bool ok[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      ok[c] = FULL || (e0 + c * 32 + lane < n);
      lp[c] = FULL ? ld_stream(lpp + c * 32) : ld_stream_if(lpp + c * 32, ok[c]);
      if (RUN) lt[c] = FULL ? ld_stream(ltp + c * 32) : ld_stream_if(ltp + c * 32, ok[c]);
      else lt[c] = 0;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int e = (RUN ? 0 : k) + e0 + c * 32 + lane;  // slot
      // l_p ∉ [0, max_input_len] or l_t ∉ [0, max_new) (unsigned compares catch < 0)
      if (RUN) {
        mx_lp = ::max(mx_lp, (uint32_t)lp[c]);
        mx_lt = ::max(mx_lt, (uint32_t)lt[c]);
        lt[c] = (int)::min((uint32_t)lt[c], mx1);  // keeps the lookups in range
      } else {
        mx_lp = ::max(mx_lp, (uint32_t)lp[c]);
      }
      const uint32_t u = FAST ? lowbias32(key_fold ^ ((uint32_t)e * 0x9E3779B9U))
                              : draw_slow(p, key_fold, e, R);
      const uint32_t bq = RUN ? (uint32_t)sC[lt[c]] : bq0;
      lh[c] = ::min((int)sS[mad_hi(u, W - bq, bq)], max_new);  // C-6
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int e = (RUN ? 0 : k) + e0 + c * 32 + lane;
      const int r = lh[c] - lt[c];  // ≥ 1 (C-4)
      const int a = lp[c] + lt[c];
      const uint32_t b4 = (uint32_t)bin_of<NB>(r) * 4u;
      const uint32_t rec = (uint32_t)r | ((uint32_t)a << 13);
      const uint32_t an = ((uint32_t)a << NSH) | 1u;
      if (FULL) {
        rb[e] = rec;
        nx[e] = (uint16_t)atomicExch(&hd[b4 >> 2], (uint32_t)e);
        atomicAdd(&bins[b4 >> 2], an);
      } else {
        // shared-memory atomics cannot be predicated (ptxas wraps them in branches): an
        // out-of-range lane aims its two atomics at the team's dummy words instead
        sts_u32_if(a_rb + 4u * e, rec, ok[c]);
        const uint32_t old = atom_exch_sh(ok[c] ? a_hd + b4 : a_dummy, (uint32_t)e);
        sts_u16_if(a_nx + 2u * e, old, ok[c]);
        red_add_sh(ok[c] ? sh_addr(bins) + b4 : a_dummy, an);
      }
    }
    if (po_base) {  // prediction outputs (one uniform branch per chunk)
      int32_t* po = po_base + e0;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (FULL || ok[c]) po[c * 32] = lh[c];
    }
  };
  {
    const int32_t* lpR = p.input_len + r0 + lane;
    const int32_t* ltR = p.generated + r0 + lane;
    int32_t* poR = p.pred_run_out ? p.pred_run_out + (r0 + lane) : nullptr;
    auto run_loop = [&](auto fast_tag) {
      int e0 = 0;
#pragma unroll 1
      for (; e0 + PF_GNC * 32 <= k; e0 += PF_GNC * 32)
        chunk(e0, k, lpR + e0, ltR + e0, poR, binR, BoolTag<true>(), fast_tag,
              IntTag<PF_GNC>(), BoolTag<true>());
      // ragged tail (< 128 requests): predicated 1-request-per-lane chunks (one code copy:
      // fewer hot instructions for the instruction cache than 2-/1-request variants)
      const int32_t* pl = lpR + e0;
      const int32_t* pt = ltR + e0;
#pragma unroll 1
      for (; e0 < k; e0 += 32, pl += 32, pt += 32)
        chunk(e0, k, pl, pt, poR, binR, BoolTag<false>(), fast_tag, IntTag<1>(), BoolTag<true>());
    };
    if (draw_fast) run_loop(BoolTag<true>());
    else run_loop(BoolTag<false>());
  }
  if (!estimate_only) {
    const int32_t* lpQ = p.q_input_len + q0 + lane;
    int32_t* poQ = p.pred_q_out ? p.pred_q_out + (q0 + lane) : nullptr;
    auto q_loop = [&](auto fast_tag) {
      int j0 = 0;
#pragma unroll 1
      for (; j0 + 2 * 32 <= q; j0 += 2 * 32)
        chunk(j0, q, lpQ + j0, nullptr, poQ, binQ, BoolTag<true>(), fast_tag,
              IntTag<2>(), BoolTag<false>());
      const int32_t* pl = lpQ + j0;
#pragma unroll 1
      for (; j0 < q; j0 += 32, pl += 32)
        chunk(j0, q, pl, nullptr, poQ, binQ, BoolTag<false>(), fast_tag, IntTag<1>(), BoolTag<false>());
    };
    if (draw_fast) q_loop(BoolTag<true>());
    else q_loop(BoolTag<false>());
  }
  if (__any_sync(0xffffffffu, (mx_lp > lpmax) | (mx_lt > mx1))) {
    // Data-dependent violation: outputs of this instance are −1.
    for (int e = lane; e < n_ent; e += 32) {
      const int l_p = e < k ? p.input_len[r0 + e] : p.q_input_len[q0 + (e - k)];
      const int l_t = e < k ? p.generated[r0 + e] : 0;
      if (l_p < 0 || l_p > p.max_input_len) raise_error(p.err, PF_BAD_INPUT_LEN, i);
      else if (l_t < 0 || l_t >= max_new) raise_error(p.err, PF_BAD_GENERATED, i);
    }
    for (int e = lane; e < n_ent; e += 32) {
      if (e < k) {
        if (p.pred_run_out) p.pred_run_out[r0 + e] = -1;
      } else if (p.pred_q_out) {
        p.pred_q_out[q0 + (e - k)] = -1;
      }
    }
    if (lane == 0) {
      if (!estimate_only) p.admitted_out[i] = -1;
      p.peak_out[i] = -1;
      if (p.peak_running_out) p.peak_running_out[i] = -1;
    }
    return;
  }
  __syncwarp();

  // ---- a5/a6: one M* evaluation over R ∪ Q' (Q' = queue positions ≤ qlim, in binQ).
  // Lane t owns bins [4t, 4t+4) (descending r). Packed prefix words P = A << NSH | N never
  // carry (host PK bound), so R and R ∪ Q' are two running packed sums.
  const int b0 = lane * 4;
  auto evaluate = [&](int qlim, bool first) -> Eval {  // first: also M*(R)
    // per-bin r ranges, lo | hi << 16, through L1. Loaded per evaluation: an earlier build
    // that kept them in registers across the cutting-plane loop reported peaks too large
    // in 3 of 128 parity instances (its evaluations after the first saw wrong edges). The
    // cause was not isolated; it showed at the 64-register cap with spills.
    const uint4 e4 = __ldg(reinterpret_cast<const uint4*>(p.edges + b0));
    const uint32_t ed[4] = {e4.x, e4.y, e4.z, e4.w};
    const uint4 r4 = *reinterpret_cast<const uint4*>(binR + b0);
    const uint4 q4 = *reinterpret_cast<const uint4*>(binQ + b0);
    const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w}, qq[4] = {q4.x, q4.y, q4.z, q4.w};
    uint32_t vR = rr[0] + rr[1] + rr[2] + rr[3];
    uint32_t vT = vR + qq[0] + qq[1] + qq[2] + qq[3];
    {  // exclusive warp scans of the packed lane sums
      uint32_t iR = vR, iT = vT;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        iR = scan_step(iR, d);
        iT = scan_step(iT, d);
      }
      vR = iR - vR;
      vT = iT - vT;
    }
    const uint32_t s0R = vR, s0T = vT;  // packed sums over the bins before this lane's
    int lb_r = 0, lb_a = 0, bx = 0, ub_r = 0;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      vT += rr[x] + qq[x];
      const int A = (int)(vT >> NSH), N = (int)(vT & NMASK);
      const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
      if (first) {
        vR += rr[x];
        const int AR = (int)(vR >> NSH), NR = (int)(vR & NMASK);
        lb_r = ::max(lb_r, AR + lo * NR);  // exact T_R(lo)
        // wide bin holding running requests: upper bound of T_R on its range
        ub_r = ::max(ub_r, (hi > lo && (rr[x] & NMASK)) ? AR + hi * NR : 0);
      }
      const int va = A + lo * N;  // exact T_{R∪Q'}(lo)
      if (va > lb_a) {
        lb_a = va;
        bx = x;
      }
    }
    Eval ev;
    ev.m_run = first ? __reduce_max_sync(0xffffffffu, lb_r) : 0;
    ev.m_all = __reduce_max_sync(0xffffffffu, lb_a);
    {  // τ = the lower edge of the (lowest-lane) bin attaining m_all, and T_R(τ)
      const int who = __ffs(__ballot_sync(0xffffffffu, lb_a == ev.m_all)) - 1;
      uint32_t pr = s0R + rr[0];
      int tau = (int)(ed[0] & 0xFFFF);
#pragma unroll
      for (int x = 1; x < 4; ++x)
        if (bx >= x) {
          pr += rr[x];
          tau = (int)(ed[x] & 0xFFFF);
        }
      const int trun = (int)(pr >> NSH) + tau * (int)(pr & NMASK);
      ev.tau = __shfl_sync(0xffffffffu, tau, who);
      ev.t_run = __shfl_sync(0xffffffffu, trun, who);
    }
    const bool need_r = first && __reduce_max_sync(0xffffffffu, ub_r) > ev.m_run;
    // M*(R ∪ Q') must be exact only when it can be the reported peak (≤ C); above C the bin
    // attaining the largest exact lower bound already gives a violating τ. Only then are
    // the upper bounds of the wide bins holding requests needed (a second walk).
    bool need_a = false;
    if (!estimate_only && ev.m_all <= Cmax) {
      uint32_t v = s0T;
      int ub_a = 0;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        v += rr[x] + qq[x];
        const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
        ub_a = ::max(ub_a, (hi > lo && ((rr[x] + qq[x]) & NMASK)) ? (int)(v >> NSH) + hi * (int)(v & NMASK) : 0);
      }
      need_a = __reduce_max_sync(0xffffffffu, ub_a) > ev.m_all;
    }
    if (!need_r && !need_a) return ev;
    // ---- refinement of the wide bins whose upper bound beats the current maximum
    if (lane == 0) cand[0] = 0;
    __syncwarp();
    vR = s0R;
    vT = s0T;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const uint32_t nR = vR + rr[x], nT = vT + rr[x] + qq[x];
      const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
      const bool c_r = need_r && (rr[x] & NMASK) && hi > lo &&
                       (int)(nR >> NSH) + hi * (int)(nR & NMASK) > ev.m_run;
      const bool c_a = need_a && ((rr[x] + qq[x]) & NMASK) && hi > lo &&
                       (int)(nT >> NSH) + hi * (int)(nT & NMASK) > ev.m_all;
      if (c_r || c_a) {
        const int slot = atomicAdd(&cand[0], 1);
        if (slot < 16) {
          int* cd = cand + 1 + 6 * slot;
          cd[0] = b0 + x;
          cd[1] = (int)(vR >> NSH);  // A_R, N_R, A_Q', N_Q' over the bins before b
          cd[2] = (int)(vR & NMASK);
          cd[3] = (int)((vT - vR) >> NSH);
          cd[4] = (int)((vT - vR) & NMASK);
        }
      }
      vR = nR;
      vT = nT;
    }
    __syncwarp();
    const int n_cand = cand[0];
    int vr = 0, va = 0, tau = 0, trun = 0;
    if (n_cand <= PF_LOCKSTEP_MAX) {  // few candidates: the warp walks each one's list in turn
      for (int c = 0; c < n_cand; ++c) {
        const int* cd = cand + 1 + 6 * c;
        const int head = (int)(hd[cd[0]] & 0xFFFFu);
        for (int round = 0;; round += 32) {
          int cnt = 0, mine = -1;
          for (int e = head; e != 0xFFFF; e = nx[e]) {
            if (e >= k && e - k + 1 > qlim) continue;  // queue request not in Q'
            if (cnt == round + lane) mine = e;
            ++cnt;
          }
          if (cnt <= round) break;
          const int rx = mine >= 0 ? ent_r(mine) : 0x7FFFFFFF;
          int Ar = cd[1], Nr = cd[2], Aa = cd[1] + cd[3], Na = cd[2] + cd[4];
          for (int y = head; y != 0xFFFF; y = nx[y]) {
            if (y >= k && y - k + 1 > qlim) continue;
            const bool ge = ent_r(y) >= rx;
            const int ay = ge ? ent_a(y) : 0;
            Aa += ay;
            Na += ge ? 1 : 0;
            Ar += (y < k) ? ay : 0;
            Nr += (ge && y < k) ? 1 : 0;
          }
          if (mine >= 0) {
            const int t_r = Ar + rx * Nr, t_a = Aa + rx * Na;  // exact T at τ = rx
            vr = ::max(vr, t_r);
            if (t_a > va) {
              va = t_a;
              tau = rx;
              trun = t_r;
            }
          }
          if (cnt <= round + 32) break;
        }
      }
    } else {
      // Many candidate bins: every lane refines its own, exactly, from their lists.
      vR = s0R;
      vT = s0T;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint32_t nR = vR + rr[x], nT = vT + rr[x] + qq[x];
        const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
        const bool c_r = need_r && (rr[x] & NMASK) && hi > lo &&
                         (int)(nR >> NSH) + hi * (int)(nR & NMASK) > ev.m_run;
        const bool c_a = need_a && ((rr[x] + qq[x]) & NMASK) && hi > lo &&
                         (int)(nT >> NSH) + hi * (int)(nT & NMASK) > ev.m_all;
        if (c_r || c_a) {
          const int head = (int)(hd[b0 + x] & 0xFFFFu);
          const int pAR = (int)(vR >> NSH), pNR = (int)(vR & NMASK);
          const int pA = (int)(vT >> NSH), pN = (int)(vT & NMASK);
          for (int e = head; e != 0xFFFF; e = nx[e]) {
            if (e >= k && e - k + 1 > qlim) continue;
            const int rx = ent_r(e);
            int Ar = pAR, Nr = pNR, Aa = pA, Na = pN;
            for (int y = head; y != 0xFFFF; y = nx[y]) {
              if (y >= k && y - k + 1 > qlim) continue;
              const bool ge = ent_r(y) >= rx;
              const int ay = ge ? ent_a(y) : 0;
              Aa += ay;
              Na += ge ? 1 : 0;
              Ar += (y < k) ? ay : 0;
              Nr += (ge && y < k) ? 1 : 0;
            }
            const int t_r = Ar + rx * Nr, t_a = Aa + rx * Na;
            vr = ::max(vr, t_r);
            if (t_a > va) {
              va = t_a;
              tau = rx;
              trun = t_r;
            }
          }
        }
        vR = nR;
        vT = nT;
      }
    }
    ev.m_run = ::max(ev.m_run, __reduce_max_sync(0xffffffffu, vr));
    const int ma = __reduce_max_sync(0xffffffffu, va);
    if (ma > ev.m_all) {
      ev.m_all = ma;
      const int who = __ffs(__ballot_sync(0xffffffffu, va == ma)) - 1;
      ev.tau = __shfl_sync(0xffffffffu, tau, who);
      ev.t_run = __shfl_sync(0xffffffffu, trun, who);
    }
    __syncwarp();
    return ev;
  };

  // ---- a7: Alg.1 lines 7-14 — exact p* by cutting planes (pf_admit.cuh header).
  // (one call site of the evaluation: a second inlined copy costs more in instruction-cache
  // misses than its specialisation saves, measured +12 %)
  int p_star = 0, peak = 0, M0 = 0, ph = q;
  bool first = true;
#pragma unroll 1
  for (;;) {
    const Eval ev = evaluate(ph, first);
    if (first) {
      first = false;
      M0 = ev.m_run;  // Eq.(eq:3): M*(R)
      if (estimate_only) {
        if (lane == 0) p.peak_out[i] = M0;
        return;
      }
      if (q == 0 || M0 > Cmax) {
        p_star = 0;
        peak = M0;
        break;
      }
      if (ev.m_all <= Cmax) {
        p_star = q;
        peak = ev.m_all;
        break;
      }
    } else if (ev.m_all <= Cmax) {
      p_star = ph;
      peak = ev.m_all;
      break;
    }
    // p_max(τ*): the first queue position j whose FIFO prefix of (a_j + τ*)·[r_j ≥ τ*]
    // pushes T_R(τ*) + prefix above C
    const int tau = ev.tau;
    int first_bad = 0x7FFFFFFF, carry = ev.t_run;
#pragma unroll 1
    for (int j0 = 0; j0 < ph; j0 += 32) {
      const int jx = j0 + lane;  // queue index j − 1
      int wv = 0;
      if (jx < ph) {
        const uint32_t rec = rb[k + jx];
        wv = ((int)(rec & 0x1FFFu) >= tau) ? (int)(rec >> 13) + tau : 0;
      }
      const int inc = (int)warp_incl_u32((uint32_t)wv);
      if (jx < ph && carry + inc > Cmax) first_bad = ::min(first_bad, jx + 1);
      carry += __shfl_sync(0xffffffffu, inc, 31);
      if (__any_sync(0xffffffffu, first_bad != 0x7FFFFFFF)) break;
    }
    ph = __reduce_min_sync(0xffffffffu, first_bad) - 1;  // p_max(τ*) < the previous p̂
    // rebuild binQ with queue positions 1..ph
    reinterpret_cast<uint4*>(binQ)[lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    for (int jx = lane; jx < ph; jx += 32) {
      const uint32_t rec = rb[k + jx];
      atomicAdd(&binQ[bin_of<NB>((int)(rec & 0x1FFFu))], ((rec >> 13) << NSH) | 1u);
    }
    __syncwarp();
  }
  if (lane == 0) {
    p.admitted_out[i] = p_star;
    p.peak_out[i] = peak;
    if (p.peak_running_out) p.peak_running_out[i] = M0;
  }
}

// Cost-weighted partition of the group-major instance range over the CTAs. Instances of
// one group cost about the same, but groups differ (their histories, hence the r spread,
// the refinement work and the evaluation count, differ: up to 1.4x between the length
// classes of config 5), so equal instance counts per CTA leave SMs idle (measured: SM
// active cycles 3.10-4.23 M for one launch). Each launch adds, per group, the SM cycles
// its warps spent per instance (clock64 around each instance) and the instance count to
// one of three rotating buffers; the next launch weights every group by its measured mean
// and gives CTA b the range of cumulative weight [b/grid, (b+1)/grid) of the total. The
// first launch (no measurements) splits by instance count. The partition only decides
// which CTA computes an instance; every output is the same bit for bit.
// (buffers: launch t reads cost[(t+2) % 3], adds to cost[t % 3], zeroes cost[(t+1) % 3])
__device__ __forceinline__ int cost_cut(const AdmitParams& p, const float* wg, const float* cum, int b,
                                        float delta, int E) {
  // instance index at cumulative weight f(b)·total (b = grid → n); cum[g] = weight of
  // groups < g, cum[G] = total. f(b) = b/grid, except that with delta > 0 the first E CTAs
  // take a (1 − delta) share each and the others split the remainder.
  const int G = p.n_groups;
  const int grid = (int)gridDim.x;
  if (b >= grid) return p.n;
  float f = (float)b / (float)grid;
  if (delta > 0.f)
    f = (b <= E) ? (float)b * (1.f - delta) / (float)grid
                 : ((float)E * (1.f - delta) + (float)(b - E) * (1.f + delta * (float)E / (float)(grid - E))) /
                       (float)grid;
  const float t = cum[G] * f;
  int g = 0, len = G;  // last g with cum[g] ≤ t
  while (len > 1) {
    const int half = len >> 1;
    if (cum[g + half] <= t) g += half;
    len -= half;
  }
  const int o0 = __ldg(p.group_off + g), o1 = __ldg(p.group_off + g + 1);
  return ::min(o1, o0 + (int)((t - cum[g]) / wg[g]));
}

// Persistent CTA per SM (header comment). Shared memory: C_g u16 [c_stride] | S_g u16
// [s_stride] | control (16 B) | blockDim/32 teams of team_smem bytes.
// NT = the block size the register budget is sized for (64 K registers / NT per thread).
template <int PK, int NT, bool EST>
__global__ void __launch_bounds__(NT, 1) admit_group_kernel(AdmitParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint16_t* sC = reinterpret_cast<uint16_t*>(smem_raw);
  uint16_t* sS = sC + p.c_stride;
  // control: [0] next instance, [1] lo, [2] hi, [3] group of the open cost segment,
  // [4] SM cycles (u32: < 2^32 per CTA segment) and [5] instances of that segment,
  // [8..11] the segment's L2 prefetch stream: mean running / queued rows per instance
  // times PF_AHEAD, and the end of its running / queued rows
  int* ctl = reinterpret_cast<int*>(sS + p.s_stride);
  unsigned int* seg_cyc = reinterpret_cast<unsigned int*>(ctl + 4);
  unsigned int* seg_cnt = reinterpret_cast<unsigned int*>(ctl + 5);
  const int lane = threadIdx.x & 31;
  unsigned char* base = reinterpret_cast<unsigned char*>(ctl + 16) + (size_t)(threadIdx.x >> 5) * p.team_smem;
  const int G = p.n_groups;
  unsigned long long* cost_wr = p.gcost ? p.gcost + (size_t)(p.cost_epoch % 3) * 2 * G : nullptr;
  if (p.gcost && blockIdx.x == 0) {  // zero the buffer the next launch adds to
    unsigned long long* z = p.gcost + (size_t)((p.cost_epoch + 1) % 3) * 2 * G;
    for (int x = threadIdx.x; x < 2 * G; x += blockDim.x) z[x] = 0ull;
  }
  if (threadIdx.x < 32) {  // warp 0: this CTA's range
    int lo = (int)(((int64_t)blockIdx.x * p.n) / gridDim.x);
    int hi = (int)(((int64_t)(blockIdx.x + 1) * p.n) / gridDim.x);
    if (p.gcost && G <= 256) {
      const unsigned long long* rd = p.gcost + (size_t)((p.cost_epoch + 2) % 3) * 2 * G;
      float* wg = reinterpret_cast<float*>(base);  // team 0's area, free until the barrier below
      float* cum = wg + G;                         // [G + 1]
      float sw = 0.f, nw = 0.f;
      for (int g = lane; g < G; g += 32) {
        const unsigned long long cnt = rd[G + g];
        const float w = cnt ? (float)rd[g] / (float)cnt : 0.f;
        wg[g] = w;
        if (cnt) {
          sw += w;
          nw += 1.f;
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        sw += __shfl_xor_sync(0xffffffffu, sw, d);
        nw += __shfl_xor_sync(0xffffffffu, nw, d);
      }
      if (nw > 0.f) {
        const float mean = sw / nw;
        float carry = 0.f;
        for (int g0 = 0; g0 < G; g0 += 32) {
          const int g = g0 + lane;
          float c = 0.f;
          if (g < G) {
            if (wg[g] <= 0.f) wg[g] = mean;
            c = wg[g] * (float)(__ldg(p.group_off + g + 1) - __ldg(p.group_off + g));
          }
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, c, d);
            if (lane >= d) c += t;
          }
          if (g < G) cum[g + 1] = carry + c;
          carry += __shfl_sync(0xffffffffu, c, 31);
        }
        if (lane == 0) cum[0] = 0.f;
        __syncwarp();
        // early finishers (multi-rank contexts): the first E CTAs get delta less work so that
        // their SMs are free for the side stream's history update, all-reduce and table
        // build (launched by the caller to overlap this admit) before the admit ends; the
        // kernel holds every SM's registers otherwise. delta = early_cycles / (expected SM
        // busy cycles: total warp-cycles / (grid · warps per CTA)), at most 0.5.
        float delta = 0.f;
        const int E = ::min(16, (int)gridDim.x / 8);
        if (p.early_cycles && E > 0) {
          const float t_sm = cum[G] / ((float)gridDim.x * (float)(blockDim.x >> 5));
          delta = t_sm > 0.f ? ::fminf(0.5f, (float)p.early_cycles / t_sm) : 0.f;
        }
        lo = cost_cut(p, wg, cum, blockIdx.x, delta, E);
        hi = cost_cut(p, wg, cum, blockIdx.x + 1, delta, E);
      }
    }
    if (lane == 0) {
      ctl[1] = lo;
      ctl[2] = ::max(lo, hi);
      ctl[3] = -1;
      *seg_cyc = 0u;
      *seg_cnt = 0u;
    }
  }
  __syncthreads();
  // thread 0, all warps past the segment: add the open segment's cost to its group
  auto flush_cost = [&]() {
    if (cost_wr && ctl[3] >= 0 && *seg_cnt) {
      atomicAdd(cost_wr + ctl[3], (unsigned long long)*seg_cyc);
      atomicAdd(cost_wr + G + ctl[3], (unsigned long long)*seg_cnt);
    }
    *seg_cyc = 0u;
    *seg_cnt = 0u;
  };
  const int lo = ctl[1], hi = ctl[2];
  // first group g with group_off[g + 1] > lo (group_off non-decreasing, group_off[G] = n)
  int g = 0;
  {
    int len = G;
    while (len > 0) {
      const int half = len >> 1;
      const bool right = __ldg(p.group_off + g + half + 1) <= lo;
      g = right ? g + half + 1 : g;
      len = right ? len - half - 1 : half;
    }
  }
  for (int s_lo = lo; s_lo < hi;) {
    int g_end;
    while ((g_end = __ldg(p.group_off + g + 1)) <= s_lo) ++g;
    const int s_hi = ::min(hi, g_end);
    __syncthreads();  // the previous segment's lookups are done
    {
      const uint4* srcC = reinterpret_cast<const uint4*>(p.gC + (size_t)g * p.c_stride);
      const uint4* srcS = reinterpret_cast<const uint4*>(p.gS + (size_t)g * p.s_stride);
      uint4* dC = reinterpret_cast<uint4*>(sC);
      uint4* dS = reinterpret_cast<uint4*>(sS);
      const int nC = p.c_stride >> 3, nS = p.s_stride >> 3;
      for (int x = threadIdx.x; x < nC + nS; x += blockDim.x) {
        if (x < nC) dC[x] = __ldg(srcC + x);
        else dS[x - nC] = __ldg(srcS + (x - nC));
      }
      if (threadIdx.x == 0) {
        ctl[0] = s_lo;
        flush_cost();
        ctl[3] = g;
        *seg_cnt = (uint32_t)(s_hi - s_lo);
        const int rlo = __ldg(p.run_off + s_lo), rhi = __ldg(p.run_off + s_hi);
        ctl[8] = (int)(((int64_t)(rhi - rlo) * PF_AHEAD) / (s_hi - s_lo));
        ctl[10] = rhi;
        if (!EST) {
          const int qlo = __ldg(p.q_off + s_lo), qhi = __ldg(p.q_off + s_hi);
          ctl[9] = (int)(((int64_t)(qhi - qlo) * PF_AHEAD) / (s_hi - s_lo));
          ctl[11] = qhi;
        }
      }
    }
    __syncthreads();
    const int64_t gid_base = (int64_t)g * p.members_per_group + p.member_base - __ldg(p.group_off + g);
    const uint32_t a_ctl = sh_addr(ctl);
    // this warp's busy cycles in the segment (start kept in its team scratch, not a register)
    uint32_t* t_start = reinterpret_cast<uint32_t*>(base + p.team_smem) - 1;
    if (lane == 0) *t_start = (uint32_t)clock();
#pragma unroll 1
    for (;;) {
      __syncwarp();  // the previous instance's shared-memory reads are done
      int i = 0;
      if (lane == 0) i = (int)atom_add_sh(a_ctl, 1u);
      i = __shfl_sync(0xffffffffu, i, 0);
      if (i >= s_hi) break;
      group_one<PK, EST>(p, lane, base, i, sC, sS, gid_base, ctl + 8);
    }
    if (cost_wr && lane == 0) atom_add_sh(a_ctl + 16u, (uint32_t)clock() - *t_start);
    s_lo = s_hi;
    ++g;
  }
  __syncthreads();
  if (threadIdx.x == 0) flush_cost();
}

}  // namespace pf
