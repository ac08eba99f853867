// pf_common.cuh — device building blocks of libpfsched (sm_100a). Shares nothing
// with oracle/: the C-8 hash, the lookups and the scans are re-implemented here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

constexpr int kWarp = 32;

// Device error codes (mirror PF_DERR_* of include/pfsched.h).
enum { PF_BAD_COMPLETION = 1, PF_BAD_OFFSETS = 2, PF_BAD_MAX_NEW = 3, PF_BAD_INPUT_LEN = 4,
       PF_BAD_GENERATED = 5, PF_BAD_CAPACITY = 6, PF_BAD_OVERRIDE = 7 };

// ---------------------------------------------------------------- C-8 hash
// SplitMix64 finalizer and lowbias32 (DESIGN.md §3 C-8; include/pfsched.h "u").
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint64_t instance_key(uint64_t seed, uint32_t tick, int64_t inst) {
  return mix64(seed ^ ((uint64_t)tick * 0xD1B54A32D192ED03ULL) ^
               ((uint64_t)inst * 0x9E3779B97F4A7C15ULL));
}
// u = max over the R repetitions (C-9: the inverse CDF is monotone in u, so the max
// of R samples is the sample at the max u).
__device__ __forceinline__ uint32_t draw_u(uint32_t key_fold, int slot, int R) {
  uint32_t u = 0;
  uint32_t c = (uint32_t)slot * (uint32_t)R * 0x9E3779B9U;
  for (int rep = 0; rep < R; ++rep) {
    u = max(u, lowbias32(key_fold ^ c));
    c += 0x9E3779B9U;
  }
  return u;
}

// ---------------------------------------------------------------- warp/block scans
// Inclusive warp scan of an int32.
__device__ __forceinline__ int warp_inclusive_add(int v, int lane) {
#pragma unroll
  for (int d = 1; d < kWarp; d <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

// Block-wide exclusive scan of NV int32 values per thread (sums). `scratch` holds
// T/32 * NV ints. Returns exclusive prefixes in `v` and block totals in `tot`.
template <int T, int NV>
__device__ __forceinline__ void block_exclusive_add(int (&v)[NV], int (&tot)[NV], int* scratch) {
  constexpr int W = T / kWarp;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) inc[c] = warp_inclusive_add(v[c], lane);
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < NV; ++c) scratch[c * W + wid] = inc[c];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    int base = 0, total = 0;
#pragma unroll
    for (int x = 0; x < W; ++x) {
      int s = scratch[c * W + x];
      base += (x < wid) ? s : 0;
      total += s;
    }
    v[c] = base + inc[c] - v[c];
    tot[c] = total;
  }
  __syncthreads();  // scratch reusable after return
}

template <int T>
__device__ __forceinline__ int block_max(int v, int* scratch) {
  constexpr int W = T / kWarp;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = __reduce_max_sync(0xffffffffu, v);
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  int m = scratch[0];
#pragma unroll
  for (int x = 1; x < W; ++x) m = max(m, scratch[x]);
  __syncthreads();
  return m;
}

// Sticky device error word: first writer wins (code, index).
__device__ __forceinline__ void raise_error(int* err, int code, int index) {
  if (atomicCAS(err, 0, code) == 0) atomicExch(err + 1, index);
}

}  // namespace pf
