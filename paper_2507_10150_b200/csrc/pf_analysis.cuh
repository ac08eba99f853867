// pf_analysis.cuh — window-similarity analysis of output-length streams (SURVEY §8(f)
// NEXT-3; fig:dist and fig:cos_win): the evidence the predictor rests
// on ("adjacent time windows have similar distributions").
//
// Windows are consecutive, non-overlapping blocks of `w` lengths; h_b(l) counts length l
// in window b (token-exact bins). The Gram matrix is computed without
// materialising the B × (Lmax+1) histogram matrix in HBM:
//     G[i][j] = Σ_l h_i(l)·h_j(l) = Σ_{x ∈ window i} h_j(len_x)
// — CTA j holds h_j in shared memory (built with shared atomics) and each warp streams
// one window i through it (coalesced reads of the L2-resident stream, one shared-memory
// lookup per request). Integer and exact; O(B·N) lookups instead of an O(B²·Lmax)
// dense product. cos[i][j] = G[i][j] / sqrt(G[i][i]·G[j][j]) in fp64 (IEEE division and
// square root: the same rounding as the oracle's expression).
#pragma once
#include "pf_common.cuh"

namespace pf {

__global__ void lengths_check_kernel(const int32_t* x, int64_t n, int max_len, int* flag) {
  bool bad = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    bad |= (unsigned)(x[t] - 1) >= (unsigned)max_len;  // x ∉ [1, max_len]
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// G[i][j] for all i, column j = blockIdx.x.
__global__ void __launch_bounds__(512) gram_kernel(const int32_t* __restrict__ x, int w, int B,
                                                  int max_len, long long* __restrict__ G) {
  extern __shared__ int hist[];
  const int j = blockIdx.x;
  for (int l = threadIdx.x; l <= max_len; l += blockDim.x) hist[l] = 0;
  __syncthreads();
  const int32_t* wj = x + (int64_t)j * w;
  for (int t = threadIdx.x; t < w; t += blockDim.x) atomicAdd(&hist[__ldg(wj + t)], 1);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < B; i += nw) {
    const int32_t* wi = x + (int64_t)i * w;
    long long s = 0;
    for (int t = lane; t < w; t += 32) s += hist[__ldg(wi + t)];
    s = warp_sum64(s);
    if (lane == 0) G[(int64_t)i * B + j] = s;
  }
}

__global__ void cosine_kernel(const long long* __restrict__ G, int B, double* __restrict__ C) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * B) return;
  const int i = (int)(t / B), j = (int)(t % B);
  C[t] = (double)G[t] / sqrt((double)G[(int64_t)i * B + i] * (double)G[(int64_t)j * B + j]);
}

// summary[0] = mean_i C[i][i+1]; summary[1] = mean_{i≠j} C[i][j] (one CTA, fp64 sums).
__global__ void __launch_bounds__(1024) similarity_summary_kernel(const double* C, int B,
                                                                   double* summary) {
  __shared__ double red[2][32];
  double adj = 0.0, glob = 0.0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    if (i + 1 < B) adj += C[(int64_t)i * B + i + 1];
    for (int j = 0; j < B; ++j)
      if (j != i) glob += C[(int64_t)i * B + j];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    adj += __shfl_xor_sync(0xffffffffu, adj, d);
    glob += __shfl_xor_sync(0xffffffffu, glob, d);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = adj; red[1][warp] = glob; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, g = 0.0;
    for (int x = 0; x < (int)(blockDim.x >> 5); ++x) { a += red[0][x]; g += red[1][x]; }
    summary[0] = a / (B - 1);
    summary[1] = g / ((double)B * (B - 1));
  }
}

// Running window k = [hw + k·rw, hw + (k+1)·rw) against the hw lengths before it:
// c_k = <h_hist, h_run> / sqrt(<h_hist, h_hist>·<h_run, h_run>). CTA per k.
__global__ void __launch_bounds__(512) adjacent_kernel(const int32_t* __restrict__ x, int hw,
                                                       int rw, int max_len, double* __restrict__ c) {
  extern __shared__ int sh[];
  int* hh = sh;
  int* hr = sh + max_len + 1;
  __shared__ long long red[3][16];
  const int k = blockIdx.x;
  for (int l = threadIdx.x; l <= max_len; l += blockDim.x) hh[l] = hr[l] = 0;
  __syncthreads();
  const int32_t* run = x + hw + (int64_t)k * rw;
  const int32_t* hist = run - hw;
  for (int t = threadIdx.x; t < hw; t += blockDim.x) atomicAdd(&hh[__ldg(hist + t)], 1);
  for (int t = threadIdx.x; t < rw; t += blockDim.x) atomicAdd(&hr[__ldg(run + t)], 1);
  __syncthreads();
  long long g_hr = 0, g_rr = 0, g_hh = 0;
  for (int t = threadIdx.x; t < rw; t += blockDim.x) {
    const int v = __ldg(run + t);
    g_hr += hh[v];
    g_rr += hr[v];
  }
  for (int t = threadIdx.x; t < hw; t += blockDim.x) g_hh += hh[__ldg(hist + t)];
  g_hr = warp_sum64(g_hr);
  g_rr = warp_sum64(g_rr);
  g_hh = warp_sum64(g_hh);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = g_hr; red[1][warp] = g_hh; red[2][warp] = g_rr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0, d = 0;
    for (int y = 0; y < (int)(blockDim.x >> 5); ++y) { a += red[0][y]; b += red[1][y]; d += red[2][y]; }
    c[k] = (double)a / sqrt((double)b * (double)d);
  }
}

__global__ void __launch_bounds__(1024) mean_kernel(const double* c, int K, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) s += c[k];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int y = 0; y < (int)(blockDim.x >> 5); ++y) t += red[y];
    *out = t / K;
  }
}

}  // namespace pf
