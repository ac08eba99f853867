/*
 * c_abi_demo.c — libpfsched.so driven from plain C (no torch, no Python): the boundary of
 * include/pfsched.h is all a caller needs. Self-checking against the config-1 worked example
 * (re-derived by hand in DESIGN.md §3.3: window of 250 each of
 * {256, 512, 1024, 2048}, quantile mode u = 2^31, capacity 16384):
 *   l̂ running = 1024 1024 2048 2048 2048 1024 2048 2048, l̂ queued = 1024 ×4,
 *   M*(R) = 10546; p* = 3 with M* = 13766 at bp = 0 and 300; p* = 1 with M* = 11394 at bp = 2000.
 * Run 1: a per-instance context. Run 2: a shared-mode context (one group = the same window
 * as 8 shard rings) that owns a one-rank NCCL communicator (pf_nccl_unique_id), so
 * pf_update_history performs the all-reduce itself. Then the latency of one
 * pf_update_history + pf_admit call pair, synchronised, from C.
 *
 * Build: gcc -O2 -std=c11 examples/c_abi_demo.c -Iinclude -I/usr/local/cuda/include
 *          -Lpaper_2507_10150_b200 -lpfsched -L/usr/local/cuda/lib64 -lcudart
 *          -Wl,-rpath,$PWD/paper_2507_10150_b200 -o examples/c_abi_demo
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <time.h>

#include <cuda_runtime_api.h>

#include "pfsched.h"

#define CK(x)                                                                     \
  do {                                                                            \
    if ((x) != cudaSuccess) {                                                     \
      fprintf(stderr, "CUDA error %s at %s:%d\n", #x, __FILE__, __LINE__);        \
      return 2;                                                                   \
    }                                                                             \
  } while (0)
#define PF(x)                                                                     \
  do {                                                                            \
    pf_status st_ = (x);                                                          \
    if (st_ != PF_OK) {                                                           \
      fprintf(stderr, "%s -> %d: %s\n", #x, (int)st_, pf_last_error());         \
      return 3;                                                                   \
    }                                                                             \
  } while (0)

static const int32_t RUN_LP[8] = {100, 200, 50, 400, 300, 1000, 20, 500};
static const int32_t RUN_LT[8] = {10, 300, 600, 1000, 1500, 50, 2000, 700};
static const int32_t Q_LP[4] = {300, 1200, 64, 2000};
static const int32_t EXP_PRED_RUN[8] = {1024, 1024, 2048, 2048, 2048, 1024, 2048, 2048};

/* which: 0, 1, 2 = the context was created with reserved_bp 0, 300, 2000 */
static int check_admits(pf_ctx* ctx, int which, const char* what, cudaStream_t s) {
  int32_t h_run_off[2] = {0, 8}, h_q_off[2] = {0, 4}, h_max_new[1] = {2048}, h_cap[1] = {16384};
  int32_t *run_off, *lp, *lt, *q_off, *qlp, *mx, *cap, *adm, *pk, *pkr, *pr, *pq;
  CK(cudaMalloc((void**)&run_off, 8));
  CK(cudaMalloc((void**)&lp, 32));
  CK(cudaMalloc((void**)&lt, 32));
  CK(cudaMalloc((void**)&q_off, 8));
  CK(cudaMalloc((void**)&qlp, 16));
  CK(cudaMalloc((void**)&mx, 4));
  CK(cudaMalloc((void**)&cap, 4));
  CK(cudaMalloc((void**)&adm, 4));
  CK(cudaMalloc((void**)&pk, 4));
  CK(cudaMalloc((void**)&pkr, 4));
  CK(cudaMalloc((void**)&pr, 32));
  CK(cudaMalloc((void**)&pq, 16));
  CK(cudaMemcpy(run_off, h_run_off, 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(lp, RUN_LP, 32, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(lt, RUN_LT, 32, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(q_off, h_q_off, 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(qlp, Q_LP, 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(mx, h_max_new, 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(cap, h_cap, 4, cudaMemcpyHostToDevice));
  int bad = 0;
  const int exp_p[3] = {3, 3, 1}, exp_m[3] = {13766, 13766, 11394};
  int32_t h_adm = -1, h_pk = -1, h_pkr = -1, h_pr[8], h_pq[4];
  PF(pf_admit(ctx, run_off, lp, lt, q_off, qlp, mx, cap, 0, adm, pk, pkr, pr, pq, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(&h_adm, adm, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h_pk, pk, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h_pkr, pkr, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_pr, pr, 32, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_pq, pq, 16, cudaMemcpyDeviceToHost));
  for (int x = 0; x < 8; ++x) bad |= h_pr[x] != EXP_PRED_RUN[x];
  for (int x = 0; x < 4; ++x) bad |= h_pq[x] != 1024;
  bad |= h_pkr != 10546 || h_adm != exp_p[which] || h_pk != exp_m[which];
  printf("%s: p* = %d, M*(admitted) = %d, M*(R) = %d -> %s\n", what, h_adm, h_pk, h_pkr, bad ? "MISMATCH" : "ok");
  int32_t code = 0, idx = 0;
  PF(pf_get_device_error(ctx, &code, &idx, s));
  bad |= code != 0;
  cudaFree(run_off); cudaFree(lp); cudaFree(lt); cudaFree(q_off); cudaFree(qlp); cudaFree(mx);
  cudaFree(cap); cudaFree(adm); cudaFree(pk); cudaFree(pkr); cudaFree(pr); cudaFree(pq);
  return bad;
}

static void base_config(pf_config* c, int bp) {
  memset(c, 0, sizeof(*c));
  c->n_instances = 1;
  c->window = 1000;
  c->max_len = 2048;
  c->max_input_len = 2047;
  c->max_entries = 12;
  c->mode = PF_MODE_QUANTILE;
  c->quantile_u = 0x80000000u;
  c->repetitions = 1;
  c->reserved_bp = bp;
  c->rank = 0;
  c->nranks = 1;
}

int main(void) {
  if (pf_abi_version() != PF_ABI_VERSION) {
    fprintf(stderr, "ABI %d != header %d\n", pf_abi_version(), PF_ABI_VERSION);
    return 4;
  }
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  int32_t h_hist[1000];
  for (int x = 0; x < 1000; ++x) h_hist[x] = (x < 250) ? 256 : (x < 500) ? 512 : (x < 750) ? 1024 : 2048;
  int32_t* hist;
  CK(cudaMalloc((void**)&hist, sizeof(h_hist)));
  CK(cudaMemcpy(hist, h_hist, sizeof(h_hist), cudaMemcpyHostToDevice));
  int bad = 0;

  /* 1. per-instance contexts, bp = 0 / 300 / 2000 */
  const int bps[3] = {0, 300, 2000};
  for (int b = 0; b < 3; ++b) {
    pf_config c;
    base_config(&c, bps[b]);
    pf_ctx* ctx = NULL;
    PF(pf_create(&c, hist, s, &ctx));
    char what[64];
    snprintf(what, sizeof what, "per-instance context, bp=%d", bps[b]);
    bad |= check_admits(ctx, b, what, s);
    PF(pf_destroy(ctx));
  }

  /* 2. shared mode, one group (8 shard rings of 125 = the same window), context-owned
     one-rank NCCL communicator: pf_update_history all-reduces inside the library */
  unsigned char id[128];
  pf_status st = pf_nccl_unique_id(id);
  if (st == PF_OK) {
    pf_config c;
    base_config(&c, 0);
    int32_t h_goff[2] = {0, 1};
    int32_t* goff;
    CK(cudaMalloc((void**)&goff, 8));
    CK(cudaMemcpy(goff, h_goff, 8, cudaMemcpyHostToDevice));
    c.n_groups = 1;
    c.group_off = goff;
    c.members_per_group = 1;
    c.nccl_unique_id = id;
    pf_ctx* ctx = NULL;
    PF(pf_create(&c, hist, s, &ctx)); /* init layout [G × 8 × 125]: any split of the window */
    int32_t h_coff[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int32_t* coff;
    CK(cudaMalloc((void**)&coff, sizeof(h_coff)));
    CK(cudaMemcpy(coff, h_coff, sizeof(h_coff), cudaMemcpyHostToDevice));
    PF(pf_update_history(ctx, coff, NULL, 0, s)); /* collective: update + ncclAllReduce + tables */
    bad |= check_admits(ctx, 0, "shared-mode context with its own NCCL communicator, bp=0", s);
    PF(pf_destroy(ctx));
    cudaFree(coff);
    cudaFree(goff);
  } else {
    printf("NCCL unavailable (%s): shared-mode run skipped\n", pf_last_error());
  }

  /* 3. latency of one synchronised update + admit call pair from C */
  {
    pf_config c;
    base_config(&c, 0);
    pf_ctx* ctx = NULL;
    PF(pf_create(&c, hist, s, &ctx));
    int32_t h_coff[2] = {0, 1}, h_len[1] = {1024}, h_run_off[2] = {0, 8}, h_q_off[2] = {0, 4};
    int32_t h_mx[1] = {2048}, h_cap[1] = {16384};
    int32_t *coff, *len, *run_off, *lp, *lt, *q_off, *qlp, *mx, *cap, *adm, *pk;
    CK(cudaMalloc((void**)&coff, 8));
    CK(cudaMalloc((void**)&len, 4));
    CK(cudaMalloc((void**)&run_off, 8));
    CK(cudaMalloc((void**)&lp, 32));
    CK(cudaMalloc((void**)&lt, 32));
    CK(cudaMalloc((void**)&q_off, 8));
    CK(cudaMalloc((void**)&qlp, 16));
    CK(cudaMalloc((void**)&mx, 4));
    CK(cudaMalloc((void**)&cap, 4));
    CK(cudaMalloc((void**)&adm, 4));
    CK(cudaMalloc((void**)&pk, 4));
    CK(cudaMemcpy(coff, h_coff, 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(len, h_len, 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(run_off, h_run_off, 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lp, RUN_LP, 32, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lt, RUN_LT, 32, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(q_off, h_q_off, 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(qlp, Q_LP, 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(mx, h_mx, 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(cap, h_cap, 4, cudaMemcpyHostToDevice));
    const int N = 2000;
    struct timespec t0, t1;
    for (int it = 0; it < N + 50; ++it) {
      if (it == 50) clock_gettime(CLOCK_MONOTONIC, &t0);
      PF(pf_update_history(ctx, coff, len, 1, s));
      PF(pf_admit(ctx, run_off, lp, lt, q_off, qlp, mx, cap, (uint32_t)it, adm, pk, NULL, NULL, NULL, s));
      CK(cudaStreamSynchronize(s));
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double us = ((t1.tv_sec - t0.tv_sec) * 1e9 + (t1.tv_nsec - t0.tv_nsec)) / 1e3 / N;
    printf("latency: %.1f us per synchronised pf_update_history + pf_admit pair (C caller, %d calls)\n", us, N);
    PF(pf_destroy(ctx));
  }
  cudaFree(hist);
  printf(bad ? "c_abi_demo: FAILED\n" : "c_abi_demo: ok\n");
  return bad ? 1 : 0;
}
