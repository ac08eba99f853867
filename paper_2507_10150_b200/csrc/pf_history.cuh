// pf_history.cuh — history-window kernels of libpfsched (sm_100a).
// "During serving, it records the actual output lengths of historical requests ...
//  L_h = {l_h^0 ... l_h^w} where w is the window size", and the
// counter function C(l, L_h) of Eq.(eq:5).
//
// Device representations:
//   ring  [rows × row_window]  FIFO contents, head = index of the oldest entry
//   per-instance, w ≤ Lmax+1: sorted [n × w] ascending copy of the ring (the
//                              inverse CDF is then S[base + ρ])
//   per-instance, w > Lmax+1: hist [n × (Lmax+1)] counts C(l, L_h)
//   shared groups:            phist [G × (Lmax+1)] counts over owned shards;
//                              after the all-reduce, C_g (cumulative counts) and
//                              S_g (sorted group window) tables.
#pragma once
#include "pf_common.cuh"

namespace pf {

// ---------------------------------------------------------------- init
__global__ void init_ring_kernel(int32_t* ring, int64_t total, const int32_t* init, int max_len,
                                 int* n_bad) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    int v = init ? init[x] : max_len;
    if (v < 1 || v > max_len) {
      atomicAdd(n_bad, 1);
      v = max_len;
    }
    ring[x] = v;
  }
}

// Bitonic sort of each row (create time only): CTA per row, P2 = pow2 ≥ w in smem.
__global__ void sort_rows_kernel(const int32_t* ring, int32_t* sorted, int w, int P2) {
  extern __shared__ int32_t buf[];
  const int64_t row = blockIdx.x;
  for (int x = threadIdx.x; x < P2; x += blockDim.x)
    buf[x] = x < w ? ring[row * w + x] : 0x7FFFFFFF;
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int x = threadIdx.x; x < P2; x += blockDim.x) {
        const int y = x ^ stride;
        if (y > x) {
          const bool up = (x & size) == 0;
          const int a = buf[x], b = buf[y];
          if ((a > b) == up) {
            buf[x] = b;
            buf[y] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int x = threadIdx.x; x < w; x += blockDim.x) sorted[row * w + x] = buf[x];
}

// Histogram rows: hist[row*(Lmax+1) + v] += 1 for each ring value (rows_per_hist
// consecutive ring rows feed one histogram row).
__global__ void hist_rows_kernel(const int32_t* ring, int64_t total, int row_window,
                                 int rows_per_hist, int max_len, int32_t* hist) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = x / row_window;
    atomicAdd(&hist[(row / rows_per_hist) * (max_len + 1) + ring[x]], 1);
  }
}

// ---------------------------------------------------------------- update
// Validate one row's completions (warp-cooperative). Returns false if any ∉ [1, Lmax].
__device__ __forceinline__ bool row_valid(const int32_t* comp_len, int c0, int c1, int max_len,
                                          int lane) {
  bool bad = c1 < c0;
  for (int t = c0 + lane; !bad && t < c1; t += 32) {
    const int v = comp_len[t];
    bad = bad || v < 1 || v > max_len;
  }
  return !__any_sync(0xffffffffu, bad);
}

// Warp-cooperative rank queries on an ascending global row S[0..w): #{x : S[x] < v}
// (upper = false) and #{x : S[x] ≤ v} (upper = true) for two values at once. Each round
// splits the candidate range into 32 segments and reads one pivot per lane (one memory
// round trip for both queries); S sorted makes the predicate a prefix of the lanes, so
// popc(ballot) picks the segment. w ≤ 1024: two rounds (round 1 used 10 dependent loads
// per binary search).
__device__ __forceinline__ void warp_rank2(const int32_t* S, int w, int va, bool ua, int vb, bool ub,
                                           int lane, int& ra, int& rb) {
  int lo_a = 0, hi_a = w, lo_b = 0, hi_b = w;
  while (hi_a - lo_a > 0 || hi_b - lo_b > 0) {
    const int na = hi_a - lo_a, nb = hi_b - lo_b;
    const int sa = (na + 31) >> 5, sb = (nb + 31) >> 5;  // segment lengths (≥ 1 when n > 0)
    // pivot of lane l: last element of segment l (if the segment is non-empty)
    const int pa = lo_a + (lane + 1) * sa - 1, pb = lo_b + (lane + 1) * sb - 1;
    const bool oka = na > 0 && pa < hi_a, okb = nb > 0 && pb < hi_b;
    const int xa = oka ? S[pa] : 0, xb = okb ? S[pb] : 0;
    const unsigned ma = __ballot_sync(0xffffffffu, oka && (ua ? xa <= va : xa < va));
    const unsigned mb = __ballot_sync(0xffffffffu, okb && (ub ? xb <= vb : xb < vb));
    if (na > 0) {  // segments fully counted: popc(ma); the answer lies in the next segment
      const int c = __popc(ma);
      if (sa == 1) { lo_a += c; hi_a = lo_a; }
      else { lo_a += c * sa; hi_a = ::min(hi_a, lo_a + sa - 1); }  // its last element failed
    }
    if (nb > 0) {
      const int c = __popc(mb);
      if (sb == 1) { lo_b += c; hi_b = lo_b; }
      else { lo_b += c * sb; hi_b = ::min(hi_b, lo_b + sb - 1); }
    }
  }
  ra = lo_a;
  rb = lo_b;
}

// Move S[src .. src + n) to S[dst .. dst + n) with dst = src ∓ 1 (one-slot shift), in
// batches of 8 elements per lane (loads of a batch in flight together). Ascending order
// when dst < src, descending when dst > src, so no batch reads a slot already written.
__device__ __forceinline__ void warp_shift1(int32_t* S, int src, int dst, int n, int lane) {
  constexpr int B = 8 * 32;
  if (dst < src) {
    for (int b0 = 0; b0 < n; b0 += B) {
      int v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int x = b0 + t * 32 + lane;
        v[t] = x < n ? S[src + x] : 0;
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int x = b0 + t * 32 + lane;
        if (x < n) S[dst + x] = v[t];
      }
      __syncwarp();
    }
  } else {
    for (int b0 = 0; b0 < n; b0 += B) {
      int v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int x = n - 1 - (b0 + t * 32 + lane);
        v[t] = x >= 0 ? S[src + x] : 0;
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int x = n - 1 - (b0 + t * 32 + lane);
        if (x >= 0) S[dst + x] = v[t];
      }
      __syncwarp();
    }
  }
}

// Per-instance rings with a maintained sorted copy (w ≤ Lmax+1). Warp per row;
// completions applied one at a time in order: evict v_old = ring[head], append
// v_new, and move the sorted copy's elements between the two positions by one
// (warp-cooperative rank queries + batched shift: a few memory round trips per
// completion instead of two 10-step dependent binary searches).
__global__ void update_sorted_kernel(int n_rows, int w, int max_len, const int32_t* comp_off,
                                     const int32_t* comp_len, int32_t* ring, int32_t* head,
                                     int32_t* sorted, int* err) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n_rows) return;
  const int c0 = comp_off[row], c1 = comp_off[row + 1];
  if (c1 == c0) return;
  if (!row_valid(comp_len, c0, c1, max_len, lane)) {
    if (lane == 0) raise_error(err, PF_BAD_COMPLETION, row);
    return;
  }
  int32_t* R = ring + (int64_t)row * w;
  int32_t* S = sorted + (int64_t)row * w;
  int h = head[row];
  for (int t = c0; t < c1; ++t) {
    const int v_new = comp_len[t];
    const int v_old = R[h];
    __syncwarp();
    if (lane == 0) R[h] = v_new;
    h = (h + 1 == w) ? 0 : h + 1;
    if (v_new == v_old) continue;
    if (v_new > v_old) {
      // remove the first v_old (at i), insert v_new at j: S[i..j-1] <- S[i+1..j], S[j] = v_new
      int i, j1;
      warp_rank2(S, w, v_old, false, v_new, true, lane, i, j1);
      const int j = j1 - 1;
      warp_shift1(S, i + 1, i, j - i, lane);
      if (lane == 0) S[j] = v_new;
    } else {
      // remove the last v_old (at i), insert v_new at j: S[j+1..i] <- S[j..i-1], S[j] = v_new
      int i1, j;
      warp_rank2(S, w, v_old, true, v_new, true, lane, i1, j);
      const int i = i1 - 1;
      warp_shift1(S, j, j + 1, i - j, lane);
      if (lane == 0) S[j] = v_new;
    }
    __syncwarp();
  }
  if (lane == 0) head[row] = h;
}

// Rings feeding histograms: per-instance (w > Lmax+1, rows_per_hist = 1) or shared
// groups (rows_per_hist = shards owned). Warp per row, all lanes busy: applying c
// completions in order to a FIFO of w slots leaves the last m = min(c, w) of them at
// slots (head + c − m + j) mod w, j ∈ [0, m), and evicts exactly the old contents of
// those slots (the first c − m new values are appended and evicted again: no net
// change). Slots are distinct across j, so lane j reads its old value, writes its
// new value and moves one count from old to new, in any order; histogram counts
// use atomics (several lanes, and several shard rows of one group, hit one row).
__global__ void update_hist_kernel(int n_rows, int row_window, int rows_per_hist, int max_len,
                                   const int32_t* comp_off, const int32_t* comp_len,
                                   int32_t* ring, int32_t* head, int32_t* hist, int* err) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n_rows) return;
  // two memory rounds: (offsets, head), then (new values, evicted values) together; the
  // row is validated before anything is written (round 1 had four dependent rounds)
  const int c0 = comp_off[row], c1 = comp_off[row + 1];
  const int h = head[row];
  if (c1 == c0) return;
  const int w = row_window, c = c1 - c0;
  if (c < 0) {
    if (lane == 0) raise_error(err, PF_BAD_COMPLETION, row);
    return;
  }
  const int m = min(c, w);
  int32_t* R = ring + (int64_t)row * w;
  int32_t* H = hist + (int64_t)(row / rows_per_hist) * (max_len + 1);
  const int first = (int)(((int64_t)h + c - m) % w);  // slot of the first surviving value
  // the first 32 evicted values are loaded with the validation loads (same round trip)
  int pos0 = first + lane;
  if (pos0 >= w) pos0 -= w;
  const int old0 = lane < m ? R[pos0] : 0;
  bool bad = false;
  for (int t = c0 + lane; t < c1; t += 32) {
    const int v = comp_len[t];
    bad |= v < 1 || v > max_len;
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) raise_error(err, PF_BAD_COMPLETION, row);
    return;
  }
  for (int j = lane; j < m; j += 32) {
    int pos = first + j;
    if (pos >= w) pos -= w;
    const int v_new = comp_len[c1 - m + j];
    const int v_old = j < 32 ? old0 : R[pos];
    R[pos] = v_new;
    if (v_new != v_old) {
      atomicSub(&H[v_old], 1);
      atomicAdd(&H[v_new], 1);
    }
  }
  if (lane == 0) head[row] = (int)(((int64_t)h + c) % w);
}

// Group tables from the (all-reduced) group histogram H_g: C_g[l] = Σ_{l'≤l} H_g[l']
// and the sorted window S_g (S_g[x] = min{l : C_g[l] > x}), both u16 (W < 2^16,
// Lmax < 2^15) with row strides c_stride / s_stride. Grid (G, SPLIT): every CTA of a
// group scans the group's histogram into shared memory (each thread a contiguous run,
// loaded in one round trip, one block scan); split 0
// stores C_g; split z fills S_g[x] for its x-range by a binary search in the shared copy
// (one independent search per entry, no serial per-bin loops). Shared memory: 4·(Lmax+1) B.
template <int T, int MAXPER>
__global__ void __launch_bounds__(T) group_tables_kernel(const int32_t* H, int max_len, int W,
                                                         int c_stride, int s_stride, uint16_t* gC,
                                                         uint16_t* gS) {
  extern __shared__ int cum[];  // [Lmax+1] inclusive prefix sums
  __shared__ int scratch[T / 32];
  const int g = blockIdx.x, split = blockIdx.y, n_split = gridDim.y;
  const int nb = max_len + 1;
  const int32_t* h = H + (int64_t)g * nb;
  uint16_t* C = gC + (int64_t)g * c_stride;
  uint16_t* S = gS + (int64_t)g * s_stride;
  // thread t owns the contiguous run [t·per, t·per + per): all its loads are issued at once
  // (one memory round trip), then one block scan of the run sums
  // MAXPER (host-chosen) ≥ per: 16 when Lmax + 1 ≤ 16·T, else 64 (Lmax + 1 ≤ 32768 = 512·64)
  const int per = (nb + T - 1) / T;
  const int l0 = threadIdx.x * per;
  int v[MAXPER];
  int sum = 0;
#pragma unroll
  for (int x = 0; x < MAXPER; ++x) {
    if (x < per) {
      v[x] = (l0 + x < nb) ? h[l0 + x] : 0;
      sum += v[x];
    }
  }
  int sv[1] = {sum}, tot[1];
  block_exclusive_add<T, 1>(sv, tot, scratch);
  int acc = sv[0];
#pragma unroll
  for (int x = 0; x < MAXPER; ++x) {
    if (x < per && l0 + x < nb) {
      acc += v[x];
      cum[l0 + x] = acc;
      if (split == 0) C[l0 + x] = (uint16_t)min(acc, 65535);
    }
  }
  __syncthreads();
  // S_g: thread t fills a contiguous slice [xa, xb) of this split's range: one binary search
  // for the slice's first entry, then a forward merge walk (S is non-decreasing in x)
  const int sper = (W + n_split - 1) / n_split;
  const int x0 = split * sper, x1 = min(W, x0 + sper);
  const int chunk = (x1 - x0 + T - 1) / T;
  const int xa = x0 + threadIdx.x * chunk, xb = min(x1, xa + chunk);
  if (xa < xb) {
    int lo = 0, len = nb;  // first l with cum[l] > xa
    while (len > 0) {
      const int half = len >> 1;
      const bool right = cum[lo + half] <= xa;
      lo = right ? lo + half + 1 : lo;
      len = right ? len - half - 1 : half;
    }
    for (int x = xa; x < xb; ++x) {
      while (lo < nb && cum[lo] <= x) ++lo;  // (lo = nb only if the counts sum below W)
      S[x] = (uint16_t)lo;
    }
  }
}

// Export rings oldest-first.
__global__ void export_rows_kernel(const int32_t* ring, const int32_t* head, int n_rows,
                                   int row_window, int32_t* out) {
  const int64_t total = (int64_t)n_rows * row_window;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = x / row_window;
    const int t = (int)(x - row * row_window);
    int src = head[row] + t;
    if (src >= row_window) src -= row_window;
    out[x] = ring[row * row_window + src];
  }
}

}  // namespace pf
