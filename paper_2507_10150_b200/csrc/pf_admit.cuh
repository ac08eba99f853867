// pf_admit.cuh — the fused per-instance hot-path kernel of libpfsched (sm_100a):
//   a3/a4  distribution lookup + conditional quantile  (Eq.(eq:5), Alg.1 l.3-9)
//   a5/a6  future required memory M* (Eq.(eq:1)-(eq:3)) — sort-free, see below
//   a7     prefix-admission search over the FIFO queue   (Alg.1 l.7-14)
//
// Mapping: a TEAM of TW warps owns one instance (TW = 1 for ≤ 512 requests per
// instance: every sync is a __syncwarp, every scan a warp shuffle scan); several
// teams share a CTA. Everything after the input loads runs on-chip.
//
// M* without sorting. Eq.(eq:1)-(eq:3) equal the tick form
//   M* = max_τ T(τ),  T(τ) = Σ_{e: r_e ≥ τ} (a_e + τ),
// whose maximum sits at some r_e. Requests are binned by r with a monotone map
// (bin 0 = largest r; width-1 bins for r ≤ 16, 8 bins per octave up to width 2^s,
// then width 2^s; 128 bins per warp). With A_b, N_b the sums of a and counts over bins 0..b, and
// [lo_b, hi_b] the r-range of bin b:
//   T(lo_b) = A_b + lo_b·N_b                 exactly (a valid lower bound L of M*);
//   T(τ) ≤ A_b + hi_b·N_b for τ ∈ [lo_b, hi_b] (an upper bound U_b).
// Width-1 bins are exact. A wide non-empty bin can only hold the maximum if U_b > L;
// those rare bins (≈0.9 per evaluation on the paper-shaped workloads) are refined
// exactly from their members. This equals the sorted form bit for bit and costs
// O(bins + requests) with no sort.
//
// a7 is a cutting-plane search that returns exactly Alg.1's p* (DESIGN.md §6):
// T_p(τ) (with queue prefix 1..p) is non-decreasing in p for every τ, so M*(p) is
// too. From p̂ = q, take τ* with T_p̂(τ*) = M*(p̂) > C and jump to p̂ ← p_max(τ*) =
// the largest p with T_p(τ*) ≤ C (one FIFO prefix scan). Every p > p_max(τ*)
// violates at τ*, so p* ≤ p̂ always; stop when M*(p̂) ≤ C, i.e. p̂ = p*.
#pragma once
#include "pf_common.cuh"

// Bins per thread of the r-bin map (4: 128 bins per warp, 8 sub-bins per octave;
// 8: 256 bins per warp, 16 per octave). Host and device must agree (pfsched.cu).
#ifndef PF_BPT
#define PF_BPT 4
#endif
// Refinement strategy switch: up to this many candidate bins the whole team walks each
// candidate's list in lock-step; beyond it every thread refines its own candidate bins.
// At most 16 (the candidate table in the team scratch holds 16 entries).
#ifndef PF_LOCKSTEP_MAX
#define PF_LOCKSTEP_MAX 16
#endif
// LOOK_SORTED lookup #{S ≤ l_t} for one-warp teams: a fixed number of power-of-two search
// steps per request (the bit length of the largest coarse bucket, warp-uniform) instead of
// a divergent binary-search loop per request (cfg 3 −5.4 %; for 4-warp teams the extra
// team reduction and longer steps cost more: cfg 4 +5.7 %).
#ifndef PF_FIXED_SEARCH
#define PF_FIXED_SEARCH 1
#endif
// Track the smallest / largest r present in each bin (over all requests of the
// instance) to tighten the bin bounds: lo_b = min r, hi_b = max r (exact T at the min;
// bins holding one distinct r need no refinement). Off: with the float-exponent bin map
// few bins need refinement, and the two extra shared-memory atomics per request cost more
// than they save (measured cfg 4: 0.857 -> 0.788 ms without them).
#ifndef PF_MINMAX
#define PF_MINMAX 0
#endif
template <bool B>
struct BoolTag {
  static constexpr bool value = B;
};
// Requests per thread per predict chunk.
#ifndef PF_NC
#define PF_NC 4
#endif
template <int N>
struct IntTag {
  static constexpr int value = N;
};
// Ragged tails of the predict loop in 2- and 1-request chunks instead of a padded
// 4-request chunk (fewer issued slots per instance, but less memory-level parallelism):
// on for multi-warp teams only (measured: cfg4, TW = 4, −2 %; cfg5, TW = 1, +6 %).
#ifndef PF_TAIL
#define PF_TAIL 1
#endif

template <int TW>
struct MinMax {
  static constexpr bool on = PF_MINMAX && TW > 1;
};

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
  int team_smem;       // bytes of shared memory per team
  int teams;           // teams per CTA (one-warp teams: ≤ PF_TEAMS1, fewer for large tables)
  int ent_cap;         // request slots per team (>= max_entries)
  const uint32_t* edges;   // [n_bins]: lo | hi << 16 (0 = no r maps to the bin)
  // history tables
  const int32_t* sorted;     // LOOK_SORTED [n × w]
  const int32_t* hist;       // LOOK_HIST   [n × (Lmax+1)]
  const uint16_t* gC;        // LOOK_GROUP  [G × c_stride]: C_g[l] = #{h ≤ l} (u16, W < 2^16)
  const uint16_t* gS;        // LOOK_GROUP  [G × s_stride]: sorted group window (u16)
  int c_stride, s_stride;    // row strides (multiples of 8 elements)
  int n_groups;              // G (shared mode)
  unsigned long long* gcost; // admit_group_kernel: [3][2·G] per-group cycles, counts (rotating)
  uint32_t cost_epoch;       // launch counter selecting the rotating cost buffers
  uint32_t early_cycles;     // admit_group_kernel: SM-cycles the first CTAs finish early (0 = off)
  int cbits;                 // LOOK_SORTED: log2 of the coarse-index bucket count
  int csh;                   // LOOK_SORTED: bucket width 2^csh, smallest with (Lmax+1) >> csh ≤ 2^cbits
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
  // A12 theoretical optimum: caller-supplied l̂ replaces the
  // prediction (nullable; when set, max_new may be NULL and no clamp applies)
  const int32_t* lhat_run;   // [run_off[n]]
  const int32_t* lhat_q;     // [q_off[n]]
};

// r -> bin (r ≥ 1), stored descending: b = NB − 1 − f(r), f monotone non-decreasing:
// the float-exponent map f(r) = bits(float(r)) >> (23 − SUB) − bits(1.0f) >> (23 − SUB)
// with 2^SUB = NB/16 sub-bins per octave (one I2F, one shift, one add). Every r ≤ 2^SUB
// has its own bin and Lmax ≤ 32767 needs < 15·2^SUB < NB bins. The bins stay logarithmic
// all the way up (width ∝ r), which keeps the slack (hi − lo)·N of the bin bounds small
// where the maximum sits: fewer bins need exact refinement than with the round-1
// log-linear map (cfg 4: 0.41 vs 1.94 candidate bins per evaluation). The host builds the
// per-bin edges from the same map (pfsched.cu bin_f).
template <int NB>
constexpr int flog_sub() {
  return NB == 128 ? 3 : NB == 256 ? 4 : NB == 512 ? 5 : NB == 1024 ? 6 : 7;
}
template <int NB>
__device__ __forceinline__ int bin_of(int r) {
  constexpr int SUB = flog_sub<NB>();
  const unsigned fb = __float_as_uint(__uint2float_rz((unsigned)r)) >> (23 - SUB);  // exact: r < 2^24
  return (NB - 1 + (127 << SUB)) - (int)fb;
}

// Request-input loads: read once, so PF_STREAM_NA = 1 keeps them out of L1
// (L1::no_allocate) to leave L1 to the group tables.
#ifndef PF_STREAM_NA
#define PF_STREAM_NA 1
#endif
__device__ __forceinline__ int ld_stream(const int32_t* a) {
  if constexpr (PF_STREAM_NA) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(a));
    return v;
  } else {
    return __ldg(a);
  }
}

// ---------------------------------------------------------------- team primitives
template <int TW>
struct Team {
  static constexpr int TT = TW * 32;
  int tid, lane, wid, id;
  int* xs;  // team scratch: [0, 4·TW) reductions, [120, 122) pick
  __device__ __forceinline__ void sync() const {
    if constexpr (TW == 1) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(TT) : "memory");
    }
  }
  // exclusive prefix (in team thread order) of NV values; totals in tot.
  template <int NV>
  __device__ __forceinline__ void excl(int (&v)[NV], int (&tot)[NV]) const {
    int inc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) inc[c] = warp_inclusive_add(v[c], lane);
    if constexpr (TW == 1) {
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        tot[c] = __shfl_sync(0xffffffffu, inc[c], 31);
        v[c] = inc[c] - v[c];
      }
    } else {
      if (lane == 31) {
#pragma unroll
        for (int c = 0; c < NV; ++c) xs[c * TW + wid] = inc[c];
      }
      sync();
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        int base = 0, total = 0;
#pragma unroll
        for (int x = 0; x < TW; ++x) {
          const int s = xs[c * TW + x];
          base += (x < wid) ? s : 0;
          total += s;
        }
        v[c] = base + inc[c] - v[c];
        tot[c] = total;
      }
      sync();
    }
  }
  // excl<NV> on unsigned words (modular adds): packed (A << 9 | N) prefix sums.
  template <int NV>
  __device__ __forceinline__ void excl_u(uint32_t (&v)[NV], uint32_t (&tot)[NV]) const {
    uint32_t inc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      inc[c] = v[c];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc[c], d);
        if (lane >= d) inc[c] += t;
      }
    }
    if constexpr (TW == 1) {
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        tot[c] = __shfl_sync(0xffffffffu, inc[c], 31);
        v[c] = inc[c] - v[c];
      }
    } else {
      uint32_t* xu = reinterpret_cast<uint32_t*>(xs);
      if (lane == 31) {
#pragma unroll
        for (int c = 0; c < NV; ++c) xu[c * TW + wid] = inc[c];
      }
      sync();
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        uint32_t base = 0, total = 0;
#pragma unroll
        for (int x = 0; x < TW; ++x) {
          const uint32_t s = xu[c * TW + x];
          base += (x < wid) ? s : 0u;
          total += s;
        }
        v[c] = base + inc[c] - v[c];
        tot[c] = total;
      }
      sync();
    }
  }
  __device__ __forceinline__ int max(int v) const {
    v = __reduce_max_sync(0xffffffffu, v);
    if constexpr (TW == 1) {
      return v;
    } else {
      if (lane == 0) xs[wid] = v;
      sync();
      int m = xs[0];
#pragma unroll
      for (int x = 1; x < TW; ++x) m = ::max(m, xs[x]);
      sync();
      return m;
    }
  }
  // team maxima of NV values in one cross-warp exchange (one barrier pair)
  template <int NV>
  __device__ __forceinline__ void maxn(int (&v)[NV]) const {
#pragma unroll
    for (int c = 0; c < NV; ++c) v[c] = __reduce_max_sync(0xffffffffu, v[c]);
    if constexpr (TW > 1) {
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < NV; ++c) xs[c * TW + wid] = v[c];
      }
      sync();
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        int m = xs[c * TW];
#pragma unroll
        for (int x = 1; x < TW; ++x) m = ::max(m, xs[c * TW + x]);
        v[c] = m;
      }
      sync();
    }
  }
  __device__ __forceinline__ bool any(bool b) const {
    if constexpr (TW == 1) {
      return __any_sync(0xffffffffu, b);
    } else {
      return this->max(b ? 1 : 0) != 0;
    }
  }
  // (v1, v2) of the lowest thread with own == true (team-uniform result).
  __device__ __forceinline__ void pick(bool own, int& v1, int& v2) const {
    if constexpr (TW == 1) {
      const int who = __ffs(__ballot_sync(0xffffffffu, own)) - 1;
      v1 = __shfl_sync(0xffffffffu, v1, who);
      v2 = __shfl_sync(0xffffffffu, v2, who);
    } else {
      const int who = -this->max(own ? -tid : -(1 << 20));
      if (tid == who) {  // xs[32..33]
        xs[32] = v1;
        xs[33] = v2;
      }
      sync();
      v1 = xs[32];
      v2 = xs[33];
      sync();
    }
  }
};

// Result of one M* evaluation over R ∪ Q' (Q' = the queue entries currently in binQ).
struct Eval {
  int m_run;   // max_τ T_R(τ)           (running requests only)
  int m_all;   // max_τ T_{R∪Q'}(τ)
  int tau;     // a τ attaining m_all
  int t_run;   // T_R(tau)
};

// Per-team shared memory layout (bytes, in order):
//   rb[ent_cap] u32  request records in original order (e < k running, then queue):
//                    PACK: r | a << 13 (r < 2^13, a < 2^19); else r | bin << 16 and
//   av[ent_cap] u32  a = l_p + l_t (absent when PACK)
//   nx[ent_cap] u16  per-bin linked lists of requests (next index; 0xFFFF ends a list)
//   hd[NB] u32       list heads, one per bin (built in a4 with atomicExch)
//   binR[NBW] u32, binQ[NBW] u32: per-bin (A, N) — packed A << 9 | N when PACK, else
//                    A in [0, NB) and N in [NB, 2·NB)
//   xs[140] i32      scratch: reductions [0,32), pick [32,34), list size [36], candidates [40,137)
//   table            S[w+1] u16 + coarse index cidx[2^cbits + 2] u16 (LOOK_SORTED) | C[Lmax+1] i32 (LOOK_HIST)
// (the per-bin r ranges `edges` are read through L1 from global memory: 512 B per launch)
// Resident 4-team CTAs per SM for one-warp teams (register cap 65536 / (128 · PF_MIN_CTAS)):
// 9 → 56 registers, measured best on cfg5 (8: −4 %, 10: spills, +60 %).
#ifndef PF_MIN_CTAS
#define PF_MIN_CTAS 9
#endif
// One-warp teams per CTA (host and device must agree).
#ifndef PF_TEAMS1
#define PF_TEAMS1 4
#endif
// Multi-warp teams (one team per CTA): resident warps per SM the register cap aims at
// (min CTAs = PF_MW_WARPS / TW). cfg4 (TW = 4): 32 → 8 CTAs, 64 registers (round 2: −4 %
// against 28 → 7 CTAs, 72 registers, once the per-bin min/max atomics were gone); measured
// 2 CTAs (the old bound, ~110 registers, 4-5 resident) 1.29 ms → 8 CTAs 0.96 ms.
#ifndef PF_MW_WARPS
#define PF_MW_WARPS 32
#endif
#if PF_LOCKSTEP_MAX > 16
#error "PF_LOCKSTEP_MAX > 16 overflows the candidate table"
#endif
// One instance i on team T (the whole of a4-a8 for that instance).
template <int TW, int LOOK, int PK>
__device__ __forceinline__ void admit_one(const AdmitParams& p, Team<TW>& T, unsigned char* base,
                                          const int i) {
  constexpr int TT = TW * 32;
  constexpr int BPT = PF_BPT;  // bins per thread
  constexpr int NB = 32 * BPT * TW;
  // PK = bits of the N field of a packed bin word (A << PK | N); 0 = unpacked bins and
  // records. 9: N < 512 (max_entries < 512); 10: N < 1024 with Σ a < 2^22 (host bound).
  // PK = 1: packed records (r | a << 13) with unpacked bins (k + q ≥ 1024 or large Σ a)
  constexpr bool RP = PK != 0;    // packed request records
  constexpr bool PACK = PK >= 9;  // packed bin words
  constexpr int NSH = PACK ? PK : 9;
  constexpr uint32_t NMASK = (1u << NSH) - 1u;
  constexpr int NBW = PACK ? NB : 2 * NB;
  uint32_t* rb = reinterpret_cast<uint32_t*>(base);
  int* av = reinterpret_cast<int*>(rb + p.ent_cap);  // unused when RP
  uint16_t* nx = reinterpret_cast<uint16_t*>(av + (RP ? 0 : p.ent_cap));
  uint32_t* hd = reinterpret_cast<uint32_t*>(nx + p.ent_cap);
  uint32_t* rmn = hd + NB;                 // [NB] min r per bin (PF_MINMAX)
  uint32_t* rmx = rmn + (MinMax<TW>::on ? NB : 0);  // [NB] max r per bin
  uint32_t* binR = rmx + (MinMax<TW>::on ? NB : 0);
  uint32_t* binQ = binR + NBW;
  T.xs = reinterpret_cast<int*>(binQ + NBW);
  int* cand = T.xs + 40;    // [0]: count, then 6 ints per candidate (≤ 16); xs[36]: list size
  auto ent_r = [&](int e) -> int { return (int)(rb[e] & (RP ? 0x1FFFu : 0xFFFFu)); };
  auto ent_a = [&](int e) -> int { return RP ? (int)(rb[e] >> 13) : av[e]; };
  int32_t* table = T.xs + 140;
  uint16_t* tS = reinterpret_cast<uint16_t*>(table);  // LOOK_SORTED: the window, u16 (Lmax < 2^16)

  const int tid = T.tid;
  const bool estimate_only = (p.q_off == nullptr);

  // ---- instance scalars and CSR validation
  const int r0 = p.run_off[i], r1 = p.run_off[i + 1];
  const int q0 = estimate_only ? 0 : p.q_off[i];
  const int q1 = estimate_only ? 0 : p.q_off[i + 1];
  const int k = r1 - r0, q = q1 - q0, n_ent = k + q;
  const int max_new = p.max_new ? p.max_new[i] : p.max_len;
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
      if (p.pred_run_out)
        for (int e = tid; e < k; e += TT) p.pred_run_out[r0 + e] = -1;
      if (p.pred_q_out)
        for (int e = tid; e < q; e += TT) p.pred_q_out[q0 + e] = -1;
    }
    return;
  }
  // C = the largest integer M* that fits: 10^4·M* ≤ (10^4 − bp)·cap (C-12, C-13).
  // In 32-bit arithmetic: with cap = 10^4·Q + R, ⌊m·cap/10^4⌋ = m·Q + ⌊m·R/10^4⌋ (m ≤ 10^4,
  // so m·Q ≤ cap·m/10^4 < 2^31 and m·R < 10^8).
  int Cmax = 0;
  if (!estimate_only) {
    const uint32_t m = 10000u - (uint32_t)p.bp, cu = (uint32_t)cap;
    Cmax = (int)(m * (cu / 10000u) + (m * (cu % 10000u)) / 10000u);
  }

  // ---- a3: the distribution P(l) of Eq.(eq:5) as a lookup structure
  const int w = p.w;
  const uint16_t* gC = nullptr;
  const uint16_t* gS = nullptr;
  int goffC = 0, goffS = 0;  // element offsets of the group's rows (32-bit index math)
  int64_t gid;
  if (LOOK == LOOK_GROUP) {
    const int g = p.dist_of[i];
    goffC = g * p.c_stride;
    goffS = g * p.s_stride;
    gC = p.gC + goffC;
    gS = p.gS + goffS;
    gid = (int64_t)g * p.members_per_group + p.member_base + (i - p.group_off[g]);
  } else {
    gid = p.instance_base + i;
  }
  {
    uint4* z4 = reinterpret_cast<uint4*>(binR);  // binR and binQ are contiguous
#pragma unroll
    for (int x = 0; x < 2 * NBW / 4 / TT; ++x) z4[tid + x * TT] = make_uint4(0, 0, 0, 0);
    uint4* h4 = reinterpret_cast<uint4*>(hd);  // empty lists
#pragma unroll
    for (int x = 0; x < NB / 4 / TT; ++x) h4[tid + x * TT] = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (MinMax<TW>::on) {
      uint4* n4 = reinterpret_cast<uint4*>(rmn);
      uint4* x4 = reinterpret_cast<uint4*>(rmx);
#pragma unroll
      for (int x = 0; x < NB / 4 / TT; ++x) {
        n4[tid + x * TT] = make_uint4(0xFFFFu, 0xFFFFu, 0xFFFFu, 0xFFFFu);
        x4[tid + x * TT] = make_uint4(0, 0, 0, 0);
      }
    }
  }
  // LOOK_SORTED coarse index over the sorted window: cidx[c] = #{S < c·2^csh} for
  // c ∈ [0, NCB + 1] (NCB = 2^cbits buckets, host-chosen), so upper_bound(S, l) is a
  // binary search inside [cidx[l >> csh], cidx[(l >> csh) + 1]).
  // Built with one lower_bound per bucket edge (a scatter build from the sorted window —
  // entry x writes the buckets it opens — was measured slower: cfg 3 +26 %, cfg 4 +6 %).
  uint16_t* cidx = reinterpret_cast<uint16_t*>(table) + ((w + 2) & ~1);  // after tS[0..w] (tS[w] = sentinel)
  const int ncb = 1 << p.cbits;
  const int csh = p.csh;  // (host)
  if (LOOK == LOOK_SORTED) {
    const int32_t* src = p.sorted + (int64_t)i * w;
    if ((w & 3) == 0) {  // rows are 16-byte aligned: 4 values per load, two packed u16 pairs per store
      const int4* src4 = reinterpret_cast<const int4*>(src);
      uint2* dst = reinterpret_cast<uint2*>(tS);
      for (int x = tid; x < (w >> 2); x += TT) {
        const int4 v = __ldg(src4 + x);
        dst[x] = make_uint2((uint32_t)v.x | ((uint32_t)v.y << 16), (uint32_t)v.z | ((uint32_t)v.w << 16));
      }
    } else {
      for (int x = tid; x < w; x += TT) tS[x] = (uint16_t)__ldg(src + x);
    }
    if (tid == 0) tS[w] = 0xFFFF;
    T.sync();
    for (int c = tid; c <= ncb + 1; c += TT) {  // one lower_bound per bucket edge
      const int v = c << csh;
      int lo = 0, len = w;
      while (len > 0) {
        const int half = len >> 1;
        const bool right = (int)tS[lo + half] < v;
        lo = right ? lo + half + 1 : lo;
        len = right ? len - half - 1 : half;
      }
      cidx[c] = (uint16_t)lo;
    }
  } else if (LOOK == LOOK_HIST) {
    // C[l] = #{h ∈ L_h : h ≤ l}: inclusive scan of the persistent histogram. The counts
    // are staged into the table with coalesced loads (all in flight at once), then thread t
    // scans its contiguous run [t·per, t·per + per) in shared memory (per odd or TT = 32:
    // the stride-per accesses hit distinct banks), one team scan of the run sums, and a
    // second pass adds the run's offset (round 1 scanned TT entries per step: nb / TT
    // dependent load-scan-store rounds per instance).
    const int nb = p.max_len + 1;
    const int32_t* src = p.hist + (int64_t)i * nb;
#pragma unroll 4
    for (int x = tid; x < nb; x += TT) table[x] = __ldg(src + x);
    T.sync();
    const int per = (nb + TT - 1) / TT;
    const int l0 = ::min(nb, tid * per), l1 = ::min(nb, l0 + per);
    int run = 0;
    for (int l = l0; l < l1; ++l) {
      run += table[l];
      table[l] = run;
    }
    int v[1] = {run}, tot[1];
    T.template excl<1>(v, tot);
    if (v[0])
      for (int l = l0; l < l1; ++l) table[l] += v[0];
  }
  T.sync();
  // LOOK_SORTED: depth of the fixed-step search inside a coarse bucket — the bit length of
  // the largest bucket, so 2^sdepth − 1 ≥ every bucket's size (PF_FIXED_SEARCH)
  int sdepth = 0;
  if (LOOK == LOOK_SORTED && TW == 1 && PF_FIXED_SEARCH) {
    int mb = 0;
    for (int c = tid; c <= ncb; c += TT) mb = ::max(mb, (int)cidx[c + 1] - (int)cidx[c]);
    mb = T.max(mb);
    sdepth = 32 - __clz(mb);
  }

  // ---- a4: predictions (Alg.1 lines 3-9), running rows then queued rows, 4 requests
  // per thread per chunk with the chunk's loads issued together; each request's (a, 1)
  // is added to its r-bin and the request is pushed on the bin's list.
  uint32_t key_fold = 0;
  if (p.mode == 0) {
    const uint64_t K = instance_key(p.seed, p.tick, gid);
    key_fold = (uint32_t)K ^ (uint32_t)(K >> 32);
  }
  const bool want_pred = (p.pred_run_out != nullptr) || (p.pred_q_out != nullptr);
  int my_bad = 0;
  // u of request slot e (C-8/C-9): one lowbias32 in the common case (sampling, R = 1)
  // R = 0: adaptive repetitions max(1, ⌈64/k⌉) (SPEC.md:161 reading of PAPER.md:295)
  const int R = p.R > 0 ? p.R : (k > 0 ? ::max(1, (64 + k - 1) / k) : 64);
  const bool draw_fast = (p.mode == 0) && (R == 1);
  auto draw = [&](int e) -> uint32_t {
    uint32_t u = lowbias32(key_fold ^ ((uint32_t)e * 0x9E3779B9U));
    if (!draw_fast) u = (p.mode != 0) ? p.quantile_u : draw_u(key_fold, e, R);
    return u;
  };
  // l̂ → r, a; bin; push; (A, N) into the running or queue bins
  const bool override_lhat = p.lhat_run != nullptr;
  // (prediction outputs are stored by the callers, in one uniform branch per chunk)
  auto finish = [&](int e, int l_hat, int l_t, int l_p, bool run) {
    const int r = l_hat - l_t;  // ≥ 1 (C-4)
    const int a = l_p + l_t;
    const int b = bin_of<NB>(r);
    if (RP) {
      rb[e] = (uint32_t)r | ((uint32_t)a << 13);
    } else {
      rb[e] = (uint32_t)r | ((uint32_t)b << 16);
      av[e] = a;
    }
    nx[e] = (uint16_t)atomicExch(&hd[b], (uint32_t)e);  // push onto bin b's list
    if (MinMax<TW>::on) {
      atomicMin(&rmn[b], (uint32_t)r);
      atomicMax(&rmx[b], (uint32_t)r);
    }
    uint32_t* bins = run ? binR : binQ;
    if (PACK) {
      atomicAdd(&bins[b], ((uint32_t)a << NSH) | 1u);
    } else {
      atomicAdd(&bins[b], (uint32_t)a);
      atomicAdd(&bins[NB + b], 1u);
    }
  };
  // running requests e ∈ [0, k): l̂ from P(l > l_t)
  if (override_lhat) {
    // A12: l̂ given per request; need l_t < l̂ ≤ Lmax (running), 1 ≤ l̂ ≤ Lmax (queued)
#pragma unroll 1
    for (int e = tid; e < k; e += TT) {
      const int l_p = __ldg(p.input_len + r0 + e), l_t = __ldg(p.generated + r0 + e);
      const int l_hat = __ldg(p.lhat_run + r0 + e);
      const bool bad = (unsigned)l_p > (unsigned)p.max_input_len || l_t < 0 || l_hat <= l_t ||
                       l_hat > p.max_len;
      my_bad |= bad;
      if (!bad && want_pred && p.pred_run_out) p.pred_run_out[r0 + e] = l_hat;
      if (!bad) finish(e, l_hat, l_t, l_p, true);
    }
#pragma unroll 1
    for (int j = tid; j < q; j += TT) {
      const int l_p = __ldg(p.q_input_len + q0 + j), l_hat = __ldg(p.lhat_q + q0 + j);
      const bool bad = (unsigned)l_p > (unsigned)p.max_input_len || l_hat < 1 || l_hat > p.max_len;
      my_bad |= bad;
      if (!bad && want_pred && p.pred_q_out) p.pred_q_out[q0 + j] = l_hat;
      if (!bad) finish(k + j, l_hat, 0, l_p, false);
    }
  } else {
  // All k + q entries in one loop (slot e: running e < k, queued e ≥ k with l_t = 0,
  // C-16), 4 per thread per chunk with the chunk's loads issued together. For a queued
  // entry C[0] = 0 (history ≥ 1), so the running formula gives P(l) unchanged.
  const int32_t* lpR = p.input_len + r0;
  const int32_t* ltR = p.generated + r0;
  const int32_t* lpQ = p.q_input_len + (q0 - k);  // indexed by slot e ≥ k
  int32_t* poR = p.pred_run_out ? p.pred_run_out + r0 : nullptr;
  int32_t* poQ = p.pred_q_out ? p.pred_q_out + (q0 - k) : nullptr;
  auto chunk = [&](const int e0, auto fast_tag, auto nc_tag) {
    constexpr bool FAST = decltype(fast_tag)::value;
    constexpr int NC = decltype(nc_tag)::value;  // requests per thread in this chunk
    int lp[NC], lt[NC], bq[NC], lh[NC];
    uint32_t u[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int e = e0 + c * TT;
      if (FAST) {  // the whole chunk is running requests: no guards, no selects
        lp[c] = ld_stream(lpR + e);
        lt[c] = ld_stream(ltR + e);
      } else {
        const bool run = e < k;
        lp[c] = (e < n_ent) ? ld_stream((run ? lpR : lpQ) + e) : 0;
        lt[c] = run ? ld_stream(ltR + e) : 0;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int e = e0 + c * TT;
      // l_p ∉ [0, max_input_len] or l_t ∉ [0, max_new) (unsigned compares catch < 0)
      my_bad |= (FAST || e < n_ent) & (((unsigned)lp[c] > (unsigned)p.max_input_len) |
                                       ((unsigned)lt[c] >= (unsigned)max_new));
      // keep lookups in range (outputs are dropped when bad): unsigned min maps l_t < 0 too
      lt[c] = (int)::min((unsigned)lt[c], (unsigned)(max_new - 1));
      u[c] = lowbias32(key_fold ^ ((uint32_t)e * 0x9E3779B9U));  // C-8, R = 1
      if (LOOK == LOOK_GROUP) bq[c] = __ldg(p.gC + (goffC + lt[c]));
      else if (LOOK == LOOK_HIST) bq[c] = table[lt[c]];
      else {  // #{S ≤ l_t}: first S > l_t inside the coarse bucket of l_t
        const int cb = lt[c] >> csh;
        if (TW == 1 && PF_FIXED_SEARCH) {
          // binary lifting with sdepth power-of-two steps (a team-uniform count: no
          // divergence): every entry before pos is ≤ l_t; the steps sum to 2^sdepth − 1 ≥
          // the bucket's size, entries past the bucket belong to higher buckets (> l_t)
          // and probes past the window read the S[w] = 0xFFFF sentinel, so pos ends at
          // the upper bound #{S ≤ l_t}
          int pos = cidx[cb];
          for (int step = (1 << sdepth) >> 1; step > 0; step >>= 1) {
            const int cand = pos + step;
            pos = ((int)tS[::min(cand - 1, w)] <= lt[c]) ? cand : pos;
          }
          bq[c] = pos;
        } else {
          int lo = cidx[cb], hi = cidx[cb + 1];
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int)tS[mid] <= lt[c]) lo = mid + 1; else hi = mid;
          }
          bq[c] = lo;
        }
      }
    }
    if (!draw_fast) {  // quantile mode or R ≠ 1: one uniform branch per chunk
#pragma unroll
      for (int c = 0; c < NC; ++c) u[c] = draw(e0 + c * TT);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int n_gt = w - bq[c];
      int x;  // bq + ⌊u·n_gt / 2^32⌋ in one multiply-add of the high word
      asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(u[c]), "r"((uint32_t)n_gt), "r"(bq[c]));
      if (LOOK == LOOK_GROUP) {
        lh[c] = (int)__ldg(p.gS + (goffS + x));  // n_gt = 0: x = W, S_g[W] = 0xFFFF sentinel
      } else if (LOOK == LOOK_SORTED) {
        lh[c] = tS[x];  // n_gt = 0: x = w, the sentinel
      } else {
        int lo = lt[c] + 1, len = n_gt ? p.max_len - lt[c] : 0;  // smallest L with C[L] > x
        while (len > 0) {
          const int half = len >> 1;
          const bool right = table[lo + half] <= x;
          lo = right ? lo + half + 1 : lo;
          len = right ? len - half - 1 : half;
        }
        lh[c] = n_gt ? lo : max_new;
      }
      lh[c] = ::min(lh[c], max_new);  // C-6
    }
    if (want_pred) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int e = e0 + c * TT;
        int32_t* po = (FAST || e < k) ? poR : poQ;
        if ((FAST || e < n_ent) && po) po[e] = lh[c];
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int e = e0 + c * TT;
      if (FAST || e < n_ent) finish(e, lh[c], lt[c], lp[c], FAST || e < k);
    }
  };
#pragma unroll 1
  for (int b0 = 0; b0 < n_ent;) {  // team-uniform chunk choice
    const int e0 = b0 + tid, rem = n_ent - b0;
    if (b0 + PF_NC * TT <= k) {
      chunk(e0, BoolTag<true>(), IntTag<PF_NC>());
      b0 += PF_NC * TT;
    } else if (!PF_TAIL || TW == 1 || rem > 2 * TT) {
      chunk(e0, BoolTag<false>(), IntTag<PF_NC>());
      b0 += PF_NC * TT;
    } else if (rem > TT) {
      chunk(e0, BoolTag<false>(), IntTag<2>());
      b0 += 2 * TT;
    } else {
      chunk(e0, BoolTag<false>(), IntTag<1>());
      b0 += TT;
    }
  }
  }  // !override_lhat
  if (T.any(my_bad != 0)) {
    // Data-dependent violation: outputs of this instance are −1.
    for (int e = tid; e < n_ent; e += TT) {
      const int l_p = e < k ? p.input_len[r0 + e] : p.q_input_len[q0 + (e - k)];
      const int l_t = e < k ? p.generated[r0 + e] : 0;
      if (l_p < 0 || l_p > p.max_input_len) raise_error(p.err, PF_BAD_INPUT_LEN, i);
      else if (override_lhat) raise_error(p.err, PF_BAD_OVERRIDE, i);
      else if (l_t < 0 || l_t >= max_new) raise_error(p.err, PF_BAD_GENERATED, i);
    }
    for (int e = tid; e < n_ent; e += TT) {
      if (e < k) {
        if (p.pred_run_out) p.pred_run_out[r0 + e] = -1;
      } else if (p.pred_q_out) {
        p.pred_q_out[q0 + (e - k)] = -1;
      }
    }
    if (tid == 0) {
      if (!estimate_only) p.admitted_out[i] = -1;
      p.peak_out[i] = -1;
      if (p.peak_running_out) p.peak_running_out[i] = -1;
    }
    return;
  }
  T.sync();

  // ---- a5/a6: one M* evaluation over R ∪ Q' (Q' = the queue requests in binQ, with
  // queue position ≤ qlim), header comment. Thread t owns bins [4t, 4t+4).
  auto bin_an = [&](const uint32_t* bins, int b, int& A, int& N) {
    if (PACK) {
      const uint32_t x = bins[b];
      A = (int)(x >> NSH);
      N = (int)(x & NMASK);
    } else {
      A = (int)bins[b];
      N = (int)bins[NB + b];
    }
  };
  // first = the evaluation whose m_run is reported (M*(R)); m_all needs to be exact only
  // when it can be the reported peak (≤ C): above C, the bin attaining the largest exact
  // lower bound already gives a violating τ for the cutting plane.
  auto evaluate = [&](int qlim, bool first) -> Eval {
    const int b0 = tid * BPT;
    // this thread's bins in registers (16-byte shared loads)
    int bA[BPT], bN[BPT], qA[BPT], qN[BPT];
    uint32_t ed[BPT];
    uint32_t pR = 0, pQ = 0;  // PACK: this thread's packed (A << NSH | N) sums
#pragma unroll
    for (int x0 = 0; x0 < BPT; x0 += 4) {
      const uint4 e4 = __ldg(reinterpret_cast<const uint4*>(p.edges + b0 + x0));  // L1-resident
      uint32_t ee[4] = {e4.x, e4.y, e4.z, e4.w};
      if (MinMax<TW>::on) {  // actual r range of the bin's requests (when it has any)
        const uint4 n4 = *reinterpret_cast<const uint4*>(rmn + b0 + x0);
        const uint4 m4 = *reinterpret_cast<const uint4*>(rmx + b0 + x0);
        const uint32_t nn[4] = {n4.x, n4.y, n4.z, n4.w}, mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (mm[c] != 0) ee[c] = nn[c] | (mm[c] << 16);
      }
      if (PACK) {
        const uint4 r4 = *reinterpret_cast<const uint4*>(binR + b0 + x0);
        const uint4 q4 = *reinterpret_cast<const uint4*>(binQ + b0 + x0);
        const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w}, qq[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          bA[x0 + c] = (int)(rr[c] >> NSH);
          bN[x0 + c] = (int)(rr[c] & NMASK);
          qA[x0 + c] = (int)(qq[c] >> NSH);
          qN[x0 + c] = (int)(qq[c] & NMASK);
          ed[x0 + c] = ee[c];
          pR += rr[c];
          pQ += qq[c];
        }
      } else {
        const uint4 ra = *reinterpret_cast<const uint4*>(binR + b0 + x0);
        const uint4 rn = *reinterpret_cast<const uint4*>(binR + NB + b0 + x0);
        const uint4 qa = *reinterpret_cast<const uint4*>(binQ + b0 + x0);
        const uint4 qn = *reinterpret_cast<const uint4*>(binQ + NB + b0 + x0);
        const uint32_t a1[4] = {ra.x, ra.y, ra.z, ra.w}, n1[4] = {rn.x, rn.y, rn.z, rn.w};
        const uint32_t a2[4] = {qa.x, qa.y, qa.z, qa.w}, n2[4] = {qn.x, qn.y, qn.z, qn.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          bA[x0 + c] = (int)a1[c];
          bN[x0 + c] = (int)n1[c];
          qA[x0 + c] = (int)a2[c];
          qN[x0 + c] = (int)n2[c];
          ed[x0 + c] = ee[c];
        }
      }
    }
    int s[4] = {0, 0, 0, 0};
    if (PACK) {  // the packed fields never carry: Σ A < 2^(32−NSH), Σ N < 2^NSH (host PK bound)
      uint32_t v[2] = {pR, pQ}, t2[2];
      T.template excl_u<2>(v, t2);
      s[0] = (int)(v[0] >> NSH);
      s[1] = (int)(v[0] & NMASK);
      s[2] = (int)(v[1] >> NSH);
      s[3] = (int)(v[1] & NMASK);
    } else {
      int tot[4];
#pragma unroll
      for (int x = 0; x < BPT; ++x) {
        s[0] += bA[x];
        s[1] += bN[x];
        s[2] += qA[x];
        s[3] += qN[x];
      }
      T.template excl<4>(s, tot);
    }
    const int s0[4] = {s[0], s[1], s[2], s[3]};
    // walk: exact T at lower edges (lower bounds), upper bounds of wide bins
    int lb_r = 0, lb_a = 0, lb_tau = 0, lb_trun = 0, ub_r = 0, ub_a = 0;
#pragma unroll
    for (int x = 0; x < BPT; ++x) {
      s[0] += bA[x];
      s[1] += bN[x];
      s[2] += qA[x];
      s[3] += qN[x];
      const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
      const int vr = s[0] + lo * s[1];                    // T_R(lo)
      const int va = s[0] + s[2] + lo * (s[1] + s[3]);    // T_{R∪Q'}(lo)
      lb_r = ::max(lb_r, vr);
      if (va > lb_a) {
        lb_a = va;
        lb_tau = lo;
        lb_trun = vr;
      }
      if (hi > lo) {  // wide bin: upper bounds where it holds requests
        if (bN[x] > 0) ub_r = ::max(ub_r, s[0] + hi * s[1]);
        if (bN[x] + qN[x] > 0) ub_a = ::max(ub_a, s[0] + s[2] + hi * (s[1] + s[3]));
      }
    }
    Eval ev;
    bool need_r, need_a;
    if constexpr (TW > 1) {  // the four team maxima in one barrier pair
      int mx[4] = {lb_r, lb_a, ub_r, ub_a};
      T.template maxn<4>(mx);
      ev.m_run = mx[0];
      ev.m_all = mx[1];
      ev.tau = lb_tau;
      ev.t_run = lb_trun;
      T.pick(lb_a == ev.m_all, ev.tau, ev.t_run);
      need_r = first && mx[2] > ev.m_run;
      need_a = !estimate_only && ev.m_all <= Cmax && mx[3] > ev.m_all;
    } else {
      ev.m_run = T.max(lb_r);
      ev.m_all = T.max(lb_a);
      ev.tau = lb_tau;
      ev.t_run = lb_trun;
      T.pick(lb_a == ev.m_all, ev.tau, ev.t_run);
      need_r = first && T.max(ub_r) > ev.m_run;
      need_a = !estimate_only && ev.m_all <= Cmax && T.max(ub_a) > ev.m_all;
    }
    if (!need_r && !need_a) return ev;
    // ---- refinement of the wide bins whose upper bound beats the current maximum
    if (tid == 0) cand[0] = 0;
    T.sync();
    s[0] = s0[0];
    s[1] = s0[1];
    s[2] = s0[2];
    s[3] = s0[3];
#pragma unroll
    for (int x = 0; x < BPT; ++x) {
      const int A = bA[x], N = bN[x], Aq = qA[x], Nq = qN[x];
      const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
      const bool c_r = need_r && N > 0 && hi > lo && s[0] + A + hi * (s[1] + N) > ev.m_run;
      const bool c_a = need_a && N + Nq > 0 && hi > lo &&
                       s[0] + A + s[2] + Aq + hi * (s[1] + N + s[3] + Nq) > ev.m_all;
      if (c_r || c_a) {
        const int slot = atomicAdd(&cand[0], 1);
        if (slot < 16) {
          int* cd = cand + 1 + 6 * slot;
          cd[5] = (int)ed[x];  // lo | hi << 16
          cd[0] = b0 + x;
          cd[1] = s[0];  // A_R, N_R, A_Q', N_Q' over the bins before b
          cd[2] = s[1];
          cd[3] = s[2];
          cd[4] = s[3];
        }
      }
      s[0] += A;
      s[1] += N;
      s[2] += Aq;
      s[3] += Nq;
    }
    T.sync();
    const int n_cand = cand[0];
    int best_r = ev.m_run, best_a = ev.m_all, best_tau = ev.tau, best_trun = ev.t_run;
    int vr = 0, va = 0, tau = 0, trun = 0;
    if (n_cand <= PF_LOCKSTEP_MAX) {  // few candidates: all threads on each in turn
      // walk each candidate bin's request list twice: the first walk hands the x-th
      // included member to thread x, the second (all threads in step) accumulates,
      // for each thread's member, the bin's members with r ≥ its r
      for (int c = 0; c < n_cand; ++c) {
        const int* cd = cand + 1 + 6 * c;
        const int head = (int)(hd[cd[0]] & 0xFFFFu);
        for (int round = 0;; round += TT) {
          int cnt = 0, mine = -1;
          for (int e = head; e != 0xFFFF; e = nx[e]) {
            if (e >= k && e - k + 1 > qlim) continue;  // queue request not in Q'
            if (cnt == round + tid) mine = e;
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
          if (cnt <= round + TT) break;
        }
      }
    } else {
      // Many candidate bins (large batches: the slack (hi − lo)·N is wide): every
      // thread refines its own candidate bins, exactly, from their request lists and
      // the prefix sums it already holds.
      s[0] = s0[0];
      s[1] = s0[1];
      s[2] = s0[2];
      s[3] = s0[3];
#pragma unroll
      for (int x = 0; x < BPT; ++x) {
        const int A = bA[x], N = bN[x], Aq = qA[x], Nq = qN[x];
        const int lo = (int)(ed[x] & 0xFFFF), hi = (int)(ed[x] >> 16);
        const bool c_r = need_r && N > 0 && hi > lo && s[0] + A + hi * (s[1] + N) > ev.m_run;
        const bool c_a = need_a && N + Nq > 0 && hi > lo &&
                         s[0] + A + s[2] + Aq + hi * (s[1] + N + s[3] + Nq) > ev.m_all;
        if (c_r || c_a) {
          const int head = (int)(hd[b0 + x] & 0xFFFFu);
          for (int e = head; e != 0xFFFF; e = nx[e]) {
            if (e >= k && e - k + 1 > qlim) continue;  // queue request not in Q'
            const int rx = ent_r(e);
            int Ar = s[0], Nr = s[1], Aa = s[0] + s[2], Na = s[1] + s[3];
            for (int y = head; y != 0xFFFF; y = nx[y]) {
              if (y >= k && y - k + 1 > qlim) continue;
              const bool ge = ent_r(y) >= rx;
              const int ay = ge ? ent_a(y) : 0;
              Aa += ay;
              Na += ge ? 1 : 0;
              Ar += (y < k) ? ay : 0;
              Nr += (ge && y < k) ? 1 : 0;
            }
            const int t_r = Ar + rx * Nr, t_a = Aa + rx * Na;  // exact T at τ = rx
            vr = ::max(vr, t_r);
            if (t_a > va) {
              va = t_a;
              tau = rx;
              trun = t_r;
            }
          }
        }
        s[0] += A;
        s[1] += N;
        s[2] += Aq;
        s[3] += Nq;
      }
    }
    int ma;
    if constexpr (TW > 1) {
      int mv[2] = {vr, va};
      T.template maxn<2>(mv);
      best_r = ::max(best_r, mv[0]);
      ma = mv[1];
    } else {
      best_r = ::max(best_r, T.max(vr));
      ma = T.max(va);
    }
    if (ma > best_a) {
      best_a = ma;
      T.pick(va == ma, tau, trun);
      best_tau = tau;
      best_trun = trun;
    }
    T.sync();
    ev.m_run = best_r;
    ev.m_all = best_a;
    ev.tau = best_tau;
    ev.t_run = best_trun;
    return ev;
  };

  // ---- a7: Alg.1 lines 7-14 — exact p* by cutting planes (header comment). The
  // first pass evaluates M*(R) and M*(R ∪ Q); later passes M*(p̂). One call site.
  int p_star = 0, peak = 0, M0 = 0, ph = q;
  bool first = true;
  for (;;) {
    const Eval ev = evaluate(ph, first);
    if (first) {
      first = false;
      M0 = ev.m_run;  // Eq.(eq:3): M*(R)
      if (estimate_only) {
        if (tid == 0) p.peak_out[i] = M0;
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
    // p_max(τ*): FIFO prefix of (a_j + τ*)·[r_j ≥ τ*]; first j with T_R(τ*) + prefix > C
    const int tau = ev.tau;
    int first_bad = 0x7FFFFFFF, carry = ev.t_run;
#pragma unroll 1
    for (int j0 = 0; j0 < ph; j0 += TT) {
      const int jx = j0 + tid;  // queue index j-1
      int wv = 0;
      if (jx < ph) {
        const int r = ent_r(k + jx);
        wv = (r >= tau) ? ent_a(k + jx) + tau : 0;
      }
      int v[1] = {wv}, tot[1];
      T.template excl<1>(v, tot);
      if (jx < ph && carry + v[0] + wv > Cmax) first_bad = ::min(first_bad, jx + 1);
      carry += tot[0];
      if (T.any(first_bad != 0x7FFFFFFF)) break;
    }
    ph = -T.max(-first_bad) - 1;  // p_max(τ*) < previous p̂ (τ* violated there)
    // rebuild binQ with queue positions 1..ph for the next evaluation
    {
      uint4* z4 = reinterpret_cast<uint4*>(binQ);
#pragma unroll
      for (int x = 0; x < NBW / 4 / TT; ++x) z4[tid + x * TT] = make_uint4(0, 0, 0, 0);
    }
    T.sync();
    for (int jx = tid; jx < ph; jx += TT) {
      const int b = RP ? bin_of<NB>(ent_r(k + jx)) : (int)(rb[k + jx] >> 16);
      const int a = ent_a(k + jx);
      if (PACK) {
        atomicAdd(&binQ[b], ((uint32_t)a << NSH) | 1u);
      } else {
        atomicAdd(&binQ[b], (uint32_t)a);
        atomicAdd(&binQ[NB + b], 1u);
      }
    }
    T.sync();
  }
  if (tid == 0) {
    p.admitted_out[i] = p_star;
    p.peak_out[i] = peak;
    if (p.peak_running_out) p.peak_running_out[i] = M0;
  }
}

// One team per instance, several teams per CTA (LOOK_SORTED / LOOK_HIST / LOOK_GROUP).
template <int TW, int LOOK, int PK>
__global__ void __launch_bounds__((TW == 1 ? PF_TEAMS1 : 1) * TW * 32, (TW == 1 ? PF_MIN_CTAS : (PF_MW_WARPS / TW > 1 ? PF_MW_WARPS / TW : 1)))
admit_kernel(AdmitParams p) {
  constexpr int TT = TW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Team<TW> T;
  T.id = threadIdx.x / TT;
  T.tid = threadIdx.x % TT;
  T.lane = threadIdx.x & 31;
  T.wid = T.tid >> 5;
  unsigned char* base = smem_raw + (size_t)T.id * p.team_smem;
  const int i = blockIdx.x * (TW == 1 ? p.teams : 1) + T.id;
  if (i >= p.n) return;
  admit_one<TW, LOOK, PK>(p, T, base, i);
}

}  // namespace pf
