// Microbenchmarks for the sm_100a design decisions of the pfsched admit kernel:
// per-SM throughput of shared-memory atomics, LDS, integer ALU, SHFL, MATCH, REDUX.
// Output: warp-instructions per SM-cycle for each op (measured via clock64 + events).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
__device__ unsigned sink;

template <int MODE>
__global__ void __launch_bounds__(1024) kern(unsigned seed, long long* cyc) {
  __shared__ unsigned s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = seed ^ threadIdx.x, acc = 0;
  long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    if (MODE == 0) {            // ATOMS.ADD, distinct banks (lane-indexed), per-warp region
      atomicAdd(&s[(w * 32 + lane) & 8191], x + i);
    } else if (MODE == 1) {     // ATOMS.ADD, pseudo-random bins in 512
      x = x * 1664525u + 1013904223u;
      atomicAdd(&s[((w << 9) + (x >> 23)) & 8191], x);
    } else if (MODE == 2) {     // LDS, conflict-free
      acc += s[((i * 32) + lane + w * 32) & 8191];
    } else if (MODE == 3) {     // IADD3/LOP3 chain-free ALU work (4 independent ops)
      acc = (acc + x) ^ (x >> 3); x = x + 0x9E3779B9u;
    } else if (MODE == 4) {     // SHFL
      acc += __shfl_xor_sync(0xffffffffu, acc + i, 1);
    } else if (MODE == 5) {     // MATCH.ANY
      x = x * 1664525u + 1013904223u;
      acc += __match_any_sync(0xffffffffu, x >> 27);
    } else if (MODE == 6) {     // REDUX.SUM
      acc += __reduce_add_sync(0xffffffffu, acc ^ i);
    } else if (MODE == 7) {     // 64-bit shared atomic add, distinct
      atomicAdd((unsigned long long*)&s[((w * 32 + lane) * 2) & 8190], 1ull);
    } else if (MODE == 8) {     // IMAD
      acc = acc * x + i;
    } else if (MODE == 9) {     // LDS + STS read-modify-write, lane-private bins
      unsigned a = (w * 32 + lane + ((i & 7) << 10)) & 8191; s[a] = s[a] + 1;
    }
  }
  long long t1 = clock64();
  if (acc == 0x12345678u) sink = acc;
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int MODE> void run(const char* name, int threads) {
  long long* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  kern<MODE><<<sms, threads>>>(1, d); cudaDeviceSynchronize();
  cudaMemset(d, 0, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<sms, threads>>>(7, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  { cudaError_t e = cudaGetLastError(); if (e) printf("ERR %s\n", cudaGetErrorString(e)); }
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double cyc_per_blk = (double)cyc / sms;
  double warp_instr = (double)(threads / 32) * ITERS;
  printf("%-28s threads=%4d  cyc/blk=%.0f  warp-instr/SM-cycle=%.3f  (lanes/cyc=%.1f)  ms=%.3f  eff_clock_GHz=%.2f\n",
         name, threads, cyc_per_blk, warp_instr / cyc_per_blk, 32.0 * warp_instr / cyc_per_blk, ms,
         cyc_per_blk / (ms * 1e6));
  cudaFree(d);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int nd = -1; cudaError_t e = cudaGetDeviceCount(&nd); printf("devices=%d err=%s\n", nd, cudaGetErrorString(e));
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sm=%d.%d SMs=%d L2=%d MB smem/SM=%zu KB clock=%d kHz memclk=%d kHz buswidth=%d\n",
         p.name, p.major, p.minor, p.multiProcessorCount, p.l2CacheSize >> 20,
         p.sharedMemPerMultiprocessor >> 10, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  for (int t : {256, 1024}) {
    run<0>("ATOMS.ADD distinct", t);
    run<1>("ATOMS.ADD random512", t);
    run<7>("ATOMS.ADD.64 distinct", t);
    run<2>("LDS conflict-free", t);
    run<9>("LDS+STS rmw private", t);
    run<3>("IADD/LOP/SHF (4 ops)", t);
    run<8>("IMAD", t);
    run<4>("SHFL", t);
    run<5>("MATCH.ANY", t);
    run<6>("REDUX.SUM", t);
  }
  return 0;
}
