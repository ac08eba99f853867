// pfsched.cu — the C-ABI of libpfsched.so (include/pfsched.h): context, argument
// validation, and launches of the sm_100a kernels in pf_history.cuh / pf_admit.cuh.
// No torch types cross this boundary; every array is a caller-owned device pointer.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types and enums only; the functions are resolved with dlopen (nccl_api)

#include "../../include/pfsched.h"
#include "pf_admit.cuh"  // defines PF_BPT, PF_MINMAX, PF_LOCKSTEP_MAX
#include "pf_admit_group.cuh"
#include "pf_baseline.cuh"
#include "pf_history.cuh"
#include "pf_sim.cuh"
#include "pf_analysis.cuh"
#include "pf_forward.cuh"

// LOOK_SORTED coarse-index size (log2 buckets) for multi-warp / one-warp teams.
#ifndef PF_CIDX_BITS_MW
#define PF_CIDX_BITS_MW 6
#endif
#ifndef PF_CIDX_BITS_1
#define PF_CIDX_BITS_1 6
#endif

namespace {

thread_local std::string g_last_error;

pf_status fail(pf_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define PF_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? PF_ENOMEM : PF_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                  \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

enum Layout { LAYOUT_SORTED = 0, LAYOUT_HIST = 1, LAYOUT_GROUP = 2 };

// Admit-kernel variants: warps per instance team x lookup x packing.
typedef void (*AdmitFn)(pf::AdmitParams);
struct Variant {
  int TW, cap;       // team warps, max requests per instance served
  AdmitFn fn[3][4];  // [lookup][pack]
};
// pack index 0: unpacked; 1: A << 9 | N bins (requires max_entries < 512, so one-warp
// teams only); 2: A << 10 | N bins (one-warp teams only); 3: packed records r | a << 13
// with unpacked bins (PK = 1: e.g. config 4's 1280 requests per instance). Variants that can never be
// selected are not instantiated.
template <int TW, int LOOK, int PK>
AdmitFn packed_variant() {
  if constexpr (TW == 1) return pf::admit_kernel<1, LOOK, PK>;
  else return nullptr;
}
#define PF_VARIANT(TW, CAP)                                                                    \
  {TW, CAP,                                                                                   \
   {{pf::admit_kernel<TW, pf::LOOK_SORTED, 0>, packed_variant<TW, pf::LOOK_SORTED, 9>(),       \
     packed_variant<TW, pf::LOOK_SORTED, 10>(), pf::admit_kernel<TW, pf::LOOK_SORTED, 1>},    \
    {pf::admit_kernel<TW, pf::LOOK_HIST, 0>, packed_variant<TW, pf::LOOK_HIST, 9>(),           \
     packed_variant<TW, pf::LOOK_HIST, 10>(), pf::admit_kernel<TW, pf::LOOK_HIST, 1>},        \
    {pf::admit_kernel<TW, pf::LOOK_GROUP, 0>, packed_variant<TW, pf::LOOK_GROUP, 9>(),         \
     packed_variant<TW, pf::LOOK_GROUP, 10>(), pf::admit_kernel<TW, pf::LOOK_GROUP, 1>}}}
const Variant kVariants[] = {PF_VARIANT(1, 512), PF_VARIANT(2, 1024), PF_VARIANT(4, 2048),
                             PF_VARIANT(8, 4096)};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
inline int teams_per_cta(int TW) { return TW == 1 ? PF_TEAMS1 : 1; }

// Host copy of the kernel's r -> bin map f(r) (pf_admit.cuh bin_of): the float exponent
// and top SUB mantissa bits of r, 2^SUB = n_bins / 16 sub-bins per octave.
int bin_f(int r, int n_bins) {
  int sub = 0;
  while ((16 << sub) < n_bins) ++sub;
  const float fr = (float)r;
  uint32_t bits;
  memcpy(&bits, &fr, 4);
  return (int)(bits >> (23 - sub)) - (127 << sub);
}

}  // namespace

struct pf_ctx {
  pf_config cfg;
  int layout;
  int n_rows, row_window, rows_per_hist, shards_owned;
  int32_t* ring = nullptr;
  int32_t* head = nullptr;
  int32_t* sorted = nullptr;  // LAYOUT_SORTED
  int32_t* hist = nullptr;    // LAYOUT_HIST: per instance; LAYOUT_GROUP: partial (owned shards)
  int32_t* xbuf = nullptr;    // LAYOUT_GROUP exchange buffer [G × (Lmax+1)]
  uint16_t* gC = nullptr;  // [2][G × c_stride] u16, double-buffered (tbuf = the current half)
  uint16_t* gS = nullptr;  // [2][G × s_stride] u16
  int tbuf = 0;            // half read by admit launches; build_group_tables fills the other
                           // half and flips, so a tick's table build may overlap the previous
                           // tick's admit on another stream
  int c_stride = 0, s_stride = 0;
  int32_t* dist_of = nullptr;
  int32_t* group_off = nullptr;
  int* err = nullptr;  // [2] code, index
  int* scratch = nullptr;
  uint32_t* edges = nullptr;   // [n_bins] lo | hi << 16
  int pack;
  int variant;
  size_t admit_smem;   // per CTA
  int team_smem, ent_cap;
  int n_bins;
  int cbits;           // LOOK_SORTED coarse index: 2^cbits buckets
  int teams;           // instance teams per CTA of the admit kernel
  int carveout;        // preferred shared-memory carve-out (%) of the admit kernel, −1 = none
  bool committed = false;  // group tables built at least once (shared mode)
  int gp_warps = 0;        // admit_group_kernel: one-warp teams per CTA (0 = not used)
  size_t gp_smem = 0;      // its shared memory per CTA (tables + teams)
  int sms = 148;           // SMs of the context's device (one admit_group_kernel CTA each)
  unsigned long long* gcost = nullptr;  // [3][2·G] admit_group_kernel cost buffers
  uint32_t cost_epoch = 0;              // admit_group_kernel launches so far
  void* comm = nullptr;    // ncclComm_t owned by the context (shared mode, nccl_unique_id set)
};

namespace {

void nccl_destroy(void* comm);  // below

void free_ctx(pf_ctx* c) {
  if (!c) return;
  for (void* p : {(void*)c->ring, (void*)c->head, (void*)c->sorted, (void*)c->hist,
                  (void*)c->xbuf, (void*)c->gC, (void*)c->gS, (void*)c->dist_of,
                  (void*)c->group_off, (void*)c->err, (void*)c->scratch,
                  (void*)c->edges, (void*)c->gcost})
    if (p) cudaFree(p);
  if (c->comm) nccl_destroy(c->comm);
  delete c;
}

__global__ void dist_of_kernel(const int32_t* group_off, int G, int n, int32_t* dist_of, int* bad) {
  for (int g = blockIdx.x; g < G; g += gridDim.x) {
    const int lo = group_off[g], hi = group_off[g + 1];
    if (threadIdx.x == 0 && (lo > hi || lo < 0 || hi > n)) atomicAdd(bad, 1);
    for (int i = lo + threadIdx.x; i < hi && i < n && i >= 0; i += blockDim.x) dist_of[i] = g;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (group_off[0] != 0 || group_off[G] != n))
    atomicAdd(bad, 1);
}

int grid_for(int64_t total, int threads) {
  int64_t b = (total + threads - 1) / threads;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

// Kernel attributes are process-wide, but contexts of different sizes share kernel
// variants: a context may only RAISE a kernel's dynamic shared-memory limit (a later,
// smaller context must not lower it under an earlier one's launches), and the
// carve-out hint is re-applied whenever the launching context's preference differs.
std::mutex g_attr_mu;
std::map<const void*, std::pair<int, int>> g_attr;  // fn -> (max dynamic smem set, carve-out %)

cudaError_t ensure_smem(const void* fn, int bytes, int carveout_pct = -1) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_attr.find(fn);
  if (it == g_attr.end()) it = g_attr.emplace(fn, std::make_pair(48 * 1024, -1)).first;
  if (bytes > it->second.first) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    it->second.first = bytes;
  }
  if (carveout_pct >= 0 && carveout_pct != it->second.second) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct);
    if (e != cudaSuccess) return e;
    it->second.second = carveout_pct;
  }
  return cudaSuccess;
}

constexpr int kTablesThreads = 512;

pf_status build_group_tables(pf_ctx* c, cudaStream_t s) {
  const int nxt = c->tbuf ^ 1;
  const size_t G = (size_t)c->cfg.n_groups;
  const int smem = (c->cfg.max_len + 1) * 4;
  auto fn = (c->cfg.max_len + 1 <= 16 * kTablesThreads) ? pf::group_tables_kernel<kTablesThreads, 16>
                                                        : pf::group_tables_kernel<kTablesThreads, 64>;
  PF_CUDA(ensure_smem(reinterpret_cast<const void*>(fn), smem));
  // one wave (one 512-thread CTA per SM): split each group's S_g fill over several CTAs
  int dev = 0, sms = 148;
  PF_CUDA(cudaGetDevice(&dev));
  PF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int split = std::max(1, std::min(8, sms / (int)G));
  fn<<<dim3((unsigned)G, (unsigned)split), kTablesThreads, smem, s>>>(
      c->xbuf, c->cfg.max_len, c->cfg.window, c->c_stride, c->s_stride,
      c->gC + nxt * G * c->c_stride, c->gS + nxt * G * c->s_stride);
  PF_CUDA(cudaGetLastError());
  c->tbuf = nxt;
  c->committed = true;
  return PF_OK;
}

// ---------------------------------------------------------------- NCCL (shared mode)
// The context owns its communicator when the caller passes an ncclUniqueId
// (pf_config.nccl_unique_id). NCCL is resolved at run time (dlopen "libnccl.so.2", or
// $PFSCHED_NCCL_LIB): a process that already loaded NCCL (e.g. torch) shares that copy,
// and contexts that never use NCCL do not need it.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

const NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("PFSCHED_NCCL_LIB");
    void* h = nullptr;
    if (env && *env) {
      h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already in the process
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      api.why = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy ||
        !api.error_string)
      api.why = "NCCL library lacks a required symbol";
  });
  return api.why.empty() ? &api : nullptr;
}

#define PF_NCCL(call)                                                                      \
  do {                                                                                     \
    const NcclApi* A_ = nccl_api();                                                        \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(PF_ENCCL, "%s: %s", #call, A_ ? A_->error_string(r_) : "NCCL unavailable"); \
  } while (0)

void nccl_destroy(void* comm) {
  if (const NcclApi* A = nccl_api()) A->comm_destroy((ncclComm_t)comm);
}

// H_g = Σ_ranks (owned-shard histograms), in place in the exchange buffer, on `s`.
pf_status exchange_in_library(pf_ctx* c, cudaStream_t s) {
  const NcclApi* A = nccl_api();
  if (!A) return fail(PF_ENCCL, "shared mode NCCL exchange: %s", "NCCL unavailable");
  const size_t count = (size_t)c->cfg.n_groups * (c->cfg.max_len + 1);
  PF_NCCL(A->all_reduce(c->xbuf, c->xbuf, count, ncclInt32, ncclSum, (ncclComm_t)c->comm, s));
  return PF_OK;
}

}  // namespace

extern "C" {

int32_t pf_abi_version(void) { return PF_ABI_VERSION; }

const char* pf_last_error(void) { return g_last_error.c_str(); }

pf_status pf_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(PF_EINVAL, "pf_nccl_unique_id: NULL id_out");
  const NcclApi* A = nccl_api();
  if (!A) return fail(PF_ENCCL, "pf_nccl_unique_id: NCCL unavailable");
  ncclUniqueId id;
  PF_NCCL(A->get_unique_id(&id));
  memcpy(id_out, &id, sizeof(id));
  return PF_OK;
}

// admit_group_kernel instance: packing (PK 9 / 10) x block size the registers are sized for
// (1024: 64 registers; 768: 85) x estimate-only.
static const void* group_fn(const pf_ctx* c, bool est) {
  const bool wide = c->gp_warps > 24;
#define PF_GFN(PK, NT) (est ? reinterpret_cast<const void*>(pf::admit_group_kernel<PK, NT, true>) \
                            : reinterpret_cast<const void*>(pf::admit_group_kernel<PK, NT, false>))
  if (c->pack == 1) return wide ? PF_GFN(9, 1024) : PF_GFN(9, 768);
  return wide ? PF_GFN(10, 1024) : PF_GFN(10, 768);
#undef PF_GFN
}

pf_status pf_create(const pf_config* cfg, const int32_t* init_history, void* stream,
                    pf_ctx** out) {
  if (!cfg || !out) return fail(PF_EINVAL, "pf_create: NULL cfg/out");
  *out = nullptr;
  const pf_config& C = *cfg;
  if (C.n_instances < 1) return fail(PF_EINVAL, "n_instances must be >= 1");
  if (C.window < 1) return fail(PF_EINVAL, "window must be >= 1");
  if (C.max_len < 1 || C.max_len > 32767) return fail(PF_ERANGE, "max_len must be in [1, 32767]");
  if (C.max_input_len < 0) return fail(PF_EINVAL, "max_input_len must be >= 0");
  if (C.max_entries < 1 || C.max_entries > 4096)
    return fail(PF_ERANGE, "max_entries must be in [1, 4096]");
  if (C.repetitions < 0) return fail(PF_EINVAL, "repetitions must be >= 0 (0 = adaptive)");
  if (C.reserved_bp < 0 || C.reserved_bp > 9999) return fail(PF_EINVAL, "reserved_bp must be in [0, 9999]");
  if (C.mode != PF_MODE_SAMPLE && C.mode != PF_MODE_QUANTILE) return fail(PF_EINVAL, "bad mode");
  if ((int64_t)C.max_entries * ((int64_t)C.max_input_len + 2LL * C.max_len) >= (1LL << 31))
    return fail(PF_ERANGE, "max_entries*(max_input_len + 2*max_len) must be < 2^31");
  if (C.n_groups < 0) return fail(PF_EINVAL, "n_groups must be >= 0");
  if (C.n_groups > 0) {
    if (C.window % 8) return fail(PF_EINVAL, "shared mode: window must be a multiple of 8");
    if (!C.group_off) return fail(PF_EINVAL, "shared mode: group_off required");
    if (C.window > 65535) return fail(PF_ERANGE, "shared mode: window must be < 65536");
    if (C.nranks < 1 || 8 % C.nranks || C.rank < 0 || C.rank >= C.nranks)
      return fail(PF_EINVAL, "shared mode: nranks must divide 8 and 0 <= rank < nranks");
  } else if (C.window > 16384 && C.window <= C.max_len + 1) {
    return fail(PF_ERANGE, "per-instance window <= Lmax+1 must be <= 16384");
  }
  if (C.nccl_unique_id && C.n_groups == 0)
    return fail(PF_EINVAL, "nccl_unique_id is only used in shared mode (n_groups > 0)");
  cudaStream_t s = S(stream);
  pf_ctx* c = new pf_ctx();
  c->cfg = C;
  c->cfg.group_off = nullptr;
  c->cfg.nccl_unique_id = nullptr;  // not retained
  if (C.nccl_unique_id) {
    // context-owned communicator (collective: every rank calls pf_create with the same id)
    const NcclApi* A = nccl_api();
    if (!A) {
      delete c;
      return fail(PF_ENCCL, "pf_create: %s", "NCCL unavailable (dlopen libnccl.so.2 failed)");
    }
    ncclUniqueId id;
    memcpy(&id, C.nccl_unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = A->comm_init_rank(&comm, C.nranks, id, C.rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(PF_ENCCL, "pf_create: ncclCommInitRank(nranks=%d, rank=%d): %s", C.nranks, C.rank,
                  A->error_string(r));
    }
    c->comm = comm;
  }
  if (C.n_groups > 0) {
    c->layout = LAYOUT_GROUP;
    c->shards_owned = 8 / C.nranks;
    c->n_rows = C.n_groups * c->shards_owned;
    c->row_window = C.window / 8;
    c->rows_per_hist = c->shards_owned;
  } else {
    c->committed = true;  // per-instance tables are built inside the admit kernel
    c->layout = (C.window <= C.max_len + 1) ? LAYOUT_SORTED : LAYOUT_HIST;
    c->shards_owned = 1;
    c->n_rows = C.n_instances;
    c->row_window = C.window;
    c->rows_per_hist = 1;
  }
  auto cleanup_fail = [&](pf_status st) { free_ctx(c); return st; };
#define PF_CUDA_C(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      fail(e_ == cudaErrorMemoryAllocation ? PF_ENOMEM : PF_ECUDA, "%s: %s", #call,        \
           cudaGetErrorString(e_));                                                       \
      return cleanup_fail(e_ == cudaErrorMemoryAllocation ? PF_ENOMEM : PF_ECUDA);        \
    }                                                                                     \
  } while (0)
  const int64_t ring_elems = (int64_t)c->n_rows * c->row_window;
  const int nb = C.max_len + 1;
  PF_CUDA_C(cudaMalloc(&c->ring, ring_elems * 4 + 16));
  PF_CUDA_C(cudaMalloc(&c->head, (size_t)c->n_rows * 4 + 16));
  PF_CUDA_C(cudaMalloc(&c->err, 16));
  PF_CUDA_C(cudaMalloc(&c->scratch, 16));
  PF_CUDA_C(cudaMemsetAsync(c->head, 0, (size_t)c->n_rows * 4, s));
  PF_CUDA_C(cudaMemsetAsync(c->err, 0, 16, s));
  PF_CUDA_C(cudaMemsetAsync(c->scratch, 0, 16, s));
  pf::init_ring_kernel<<<grid_for(ring_elems, 256), 256, 0, s>>>(c->ring, ring_elems, init_history,
                                                                  C.max_len, c->scratch);
  PF_CUDA_C(cudaGetLastError());
  if (c->layout == LAYOUT_SORTED) {
    PF_CUDA_C(cudaMalloc(&c->sorted, ring_elems * 4 + 16));
    int P2 = 1;
    while (P2 < c->row_window) P2 <<= 1;
    PF_CUDA_C(ensure_smem(reinterpret_cast<const void*>(pf::sort_rows_kernel), P2 * 4));
    pf::sort_rows_kernel<<<c->n_rows, 512, P2 * 4, s>>>(c->ring, c->sorted, c->row_window, P2);
    PF_CUDA_C(cudaGetLastError());
  } else {
    const int hist_rows = (c->layout == LAYOUT_HIST) ? C.n_instances : C.n_groups;
    PF_CUDA_C(cudaMalloc(&c->hist, (size_t)hist_rows * nb * 4 + 16));
    PF_CUDA_C(cudaMemsetAsync(c->hist, 0, (size_t)hist_rows * nb * 4, s));
    pf::hist_rows_kernel<<<grid_for(ring_elems, 256), 256, 0, s>>>(
        c->ring, ring_elems, c->row_window, c->rows_per_hist, C.max_len, c->hist);
    PF_CUDA_C(cudaGetLastError());
  }
  if (c->layout == LAYOUT_GROUP) {
    const int G = C.n_groups;
    PF_CUDA_C(cudaMalloc(&c->xbuf, (size_t)G * nb * 4 + 16));
    c->c_stride = (nb + 7) & ~7;
    c->s_stride = (C.window + 1 + 7) & ~7;  // S_g[W] = 0xFFFF sentinel (admit: n_gt = 0)
    PF_CUDA_C(cudaMalloc(&c->gC, 2 * (size_t)G * c->c_stride * 2 + 16));
    PF_CUDA_C(cudaMalloc(&c->gS, 2 * (size_t)G * c->s_stride * 2 + 16));
    PF_CUDA_C(cudaMemsetAsync(c->gC, 0, 2 * (size_t)G * c->c_stride * 2, s));
    PF_CUDA_C(cudaMemsetAsync(c->gS, 0xFF, 2 * (size_t)G * c->s_stride * 2, s));
    PF_CUDA_C(cudaMalloc(&c->dist_of, (size_t)C.n_instances * 4 + 16));
    PF_CUDA_C(cudaMalloc(&c->group_off, (size_t)(G + 1) * 4 + 16));
    PF_CUDA_C(cudaMemcpyAsync(c->group_off, C.group_off, (size_t)(G + 1) * 4,
                              cudaMemcpyDeviceToDevice, s));
    dist_of_kernel<<<G, 128, 0, s>>>(c->group_off, G, C.n_instances, c->dist_of, c->scratch);
    PF_CUDA_C(cudaGetLastError());
    PF_CUDA_C(cudaMemcpyAsync(c->xbuf, c->hist, (size_t)G * nb * 4, cudaMemcpyDeviceToDevice, s));
    if (c->comm || C.nranks == 1) {
      pf_status st = c->comm ? exchange_in_library(c, s) : PF_OK;
      if (st == PF_OK) st = build_group_tables(c, s);
      if (st != PF_OK) return cleanup_fail(st);
    }
  }
  int n_bad = 0;
  PF_CUDA_C(cudaMemcpyAsync(&n_bad, c->scratch, 4, cudaMemcpyDeviceToHost, s));
  PF_CUDA_C(cudaStreamSynchronize(s));
  if (n_bad) {
    fail(PF_EINVAL, "pf_create: %d invalid init_history values / group offsets", n_bad);
    return cleanup_fail(PF_EINVAL);
  }
  // Admit-kernel variant and its shared memory footprint.
  c->variant = -1;
  for (int v = 0; v < kNumVariants; ++v)
    if (kVariants[v].cap >= C.max_entries) { c->variant = v; break; }
  const Variant& V = kVariants[c->variant];
  c->n_bins = 32 * PF_BPT * V.TW;
  {  // per-bin r ranges of the r -> bin map (the kernel computes the map: bin_of)
    std::vector<uint32_t> ed(c->n_bins, 0);
    for (int r = 1; r <= C.max_len; ++r) {
      const int b = c->n_bins - 1 - bin_f(r, c->n_bins);
      const uint32_t lo = ed[b] ? (ed[b] & 0xFFFF) : (uint32_t)r;
      ed[b] = lo | ((uint32_t)r << 16);
    }
    PF_CUDA_C(cudaMalloc(&c->edges, ed.size() * 4 + 16));
    PF_CUDA_C(cudaMemcpy(c->edges, ed.data(), ed.size() * 4, cudaMemcpyHostToDevice));
  }
  // PACK: per-bin (A, N) fit one 32-bit word (A << 9 | N: every bin sum < 2^23, count
  // < 2^9; or A << 10 | N: sums < 2^22, counts < 2^10) and a request record fits one
  // (r | a << 13: Lmax < 2^13, a < 2^19)
  {
    const bool rec = C.max_len < 8192 && (int64_t)C.max_input_len + C.max_len < (1LL << 19);
    const int64_t amax = (int64_t)C.max_input_len + C.max_len - 1;  // a = l_p + l_t, l_t < max_new
    if (rec && C.max_entries < 512 && (int64_t)C.max_entries * amax < (1LL << 23))
      c->pack = 1;
    else if (rec && V.TW == 1 && C.max_entries < 1024 && (int64_t)C.max_entries * amax < (1LL << 22))
      c->pack = 2;
    else if (rec)
      c->pack = 3;  // records packed (4 B per request instead of 8 in shared memory)
    else
      c->pack = 0;
  }
  size_t table = 0;
  // LOOK_SORTED coarse index: 2^cbits buckets (64: finer indexes cost more to build than
  // their shorter searches save, measured cfg 4: 256 buckets +3 %, 512 +9 %)
  c->cbits = V.TW > 1 ? PF_CIDX_BITS_MW : PF_CIDX_BITS_1;
  if (c->layout == LAYOUT_SORTED)  // u16 S + sentinel, then the u16 coarse index
    table = (size_t)((C.window + 2) & ~1) * 2 + (size_t)((1 << c->cbits) + 2) * 2;
  if (c->layout == LAYOUT_HIST) table = (size_t)nb * 4;
  c->ent_cap = (C.max_entries + 7) & ~7;
  const bool bins_packed = c->pack == 1 || c->pack == 2;
  const size_t nbw = (size_t)c->n_bins * (bins_packed ? 1 : 2);
  size_t team = (size_t)c->ent_cap * (c->pack ? 6 : 10) + (size_t)c->n_bins * 4 * ((PF_MINMAX && V.TW > 1) ? 3 : 1) +
                nbw * 8 + 140 * 4 + table;
  team = (team + 15) & ~(size_t)15;
  c->team_smem = (int)team;
  // one-warp teams: PF_TEAMS1 per CTA, fewer when their shared memory does not fit
  // (large per-instance histogram tables: Lmax up to 32767)
  c->teams = teams_per_cta(V.TW);
  while (c->teams > 1 && team * c->teams > 227 * 1024) --c->teams;
  c->admit_smem = team * c->teams;
  const int look = c->layout;
  if (c->admit_smem > 227 * 1024) {
    fail(PF_ERANGE, "admit kernel needs %zu B of shared memory per instance team (> 227 KB)", c->admit_smem);
    return cleanup_fail(PF_ERANGE);
  }
  // Shared mode, one-warp teams, packed bins: the persistent admit_group_kernel with the
  // group tables in shared memory (pf_admit.cuh), when the tables leave room for ≥ 8 teams.
  // PFSCHED_GROUP_KERNEL=0 selects the cached-table admit_kernel instead (A/B measurements).
  if (c->layout == LAYOUT_GROUP && V.TW == 1 && bins_packed) {
    const char* ev = getenv("PFSCHED_GROUP_KERNEL");
    const size_t tables = (size_t)(c->c_stride + c->s_stride) * 2 + 64;
    const size_t avail = 232448;  // 227 KB opt-in maximum per block
    const int nw = avail > tables ? (int)std::min<size_t>(32, (avail - tables) / team) : 0;
    if (nw >= 8 && !(ev && ev[0] == '0')) {
      c->gp_warps = nw;
      c->gp_smem = tables + (size_t)nw * team;
      const char* wv = getenv("PFSCHED_GROUP_WARPS");  // A/B knob: teams per CTA (≤ 32)
      if (wv && atoi(wv) >= 8 && atoi(wv) < c->gp_warps) {
        c->gp_warps = atoi(wv);
        c->gp_smem = tables + (size_t)c->gp_warps * team;
      }
      PF_CUDA_C(ensure_smem(group_fn(c, false), (int)c->gp_smem));
      PF_CUDA_C(ensure_smem(group_fn(c, true), (int)c->gp_smem));
      int dev = 0;
      PF_CUDA_C(cudaGetDevice(&dev));
      PF_CUDA_C(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev));
      if (C.n_groups <= 256) {
        PF_CUDA_C(cudaMalloc(&c->gcost, (size_t)6 * C.n_groups * 8));
        PF_CUDA_C(cudaMemsetAsync(c->gcost, 0, (size_t)6 * C.n_groups * 8, s));
      }
    }
  }
  const void* afn = reinterpret_cast<const void*>(V.fn[look][c->pack]);
  PF_CUDA_C(ensure_smem(afn, (int)c->admit_smem));
#ifndef PF_CARVEOUT
#define PF_CARVEOUT 1
#endif
  c->carveout = -1;
  if (PF_CARVEOUT) {
    // Ask for the smallest shared-memory carve-out that keeps the full occupancy: the
    // rest of the 256 KB unified L1 caches the group tables (LOOK_GROUP lookups).
    int per_sm = 0;
    PF_CUDA_C(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, V.fn[look][c->pack], c->teams * V.TW * 32, c->admit_smem));
    const size_t need = (size_t)std::max(1, per_sm) * (c->admit_smem + 1024);
    // the driver rounds the hint up to the next supported size (KiB)
    static const int kSizes[] = {0, 8, 16, 32, 64, 100, 132, 164, 196, 228};
    int kib = 228;
    for (int sz : kSizes)
      if ((size_t)sz * 1024 >= need) { kib = sz; break; }
    c->carveout = kib * 100 / 228;
  }
#undef PF_CUDA_C
  *out = c;
  return PF_OK;
}

pf_status pf_destroy(pf_ctx* ctx) {
  if (!ctx) return fail(PF_EINVAL, "pf_destroy: NULL ctx");
  cudaDeviceSynchronize();
  free_ctx(ctx);
  return PF_OK;
}

pf_status pf_update_history(pf_ctx* c, const int32_t* comp_off, const int32_t* comp_len,
                            int32_t total, void* stream) {
  if (!c || !comp_off) return fail(PF_EINVAL, "pf_update_history: NULL ctx/comp_off");
  if (total < 0 || (total > 0 && !comp_len)) return fail(PF_EINVAL, "pf_update_history: bad total/comp_len");
  cudaStream_t s = S(stream);
  const int threads = 256;
  const int blocks = (int)(((int64_t)c->n_rows * 32 + threads - 1) / threads);
  if (c->layout == LAYOUT_SORTED) {
    pf::update_sorted_kernel<<<blocks, threads, 0, s>>>(c->n_rows, c->row_window, c->cfg.max_len,
                                                        comp_off, comp_len, c->ring, c->head,
                                                        c->sorted, c->err);
  } else {
    pf::update_hist_kernel<<<blocks, threads, 0, s>>>(c->n_rows, c->row_window, c->rows_per_hist,
                                                      c->cfg.max_len, comp_off, comp_len, c->ring,
                                                      c->head, c->hist, c->err);
  }
  PF_CUDA(cudaGetLastError());
  if (c->layout == LAYOUT_GROUP) {
    const size_t bytes = (size_t)c->cfg.n_groups * (c->cfg.max_len + 1) * 4;
    PF_CUDA(cudaMemcpyAsync(c->xbuf, c->hist, bytes, cudaMemcpyDeviceToDevice, s));
    if (c->comm) {  // collective: H_g = Σ_ranks, then the tables, all on `s`
      const pf_status st = exchange_in_library(c, s);
      if (st != PF_OK) return st;
      return build_group_tables(c, s);
    }
    if (c->cfg.nranks == 1) return build_group_tables(c, s);
  }
  return PF_OK;
}

pf_status pf_exchange_buffer(pf_ctx* c, int32_t** buf, int64_t* count) {
  if (!c || !buf || !count) return fail(PF_EINVAL, "pf_exchange_buffer: NULL argument");
  if (c->layout != LAYOUT_GROUP) return fail(PF_ESTATE, "pf_exchange_buffer: not in shared mode");
  *buf = c->xbuf;
  *count = (int64_t)c->cfg.n_groups * (c->cfg.max_len + 1);
  return PF_OK;
}

pf_status pf_commit_history(pf_ctx* c, void* stream) {
  if (!c) return fail(PF_EINVAL, "pf_commit_history: NULL ctx");
  if (c->layout != LAYOUT_GROUP) return PF_OK;
  if (c->comm)
    return fail(PF_ESTATE, "pf_commit_history: the context owns its NCCL communicator; "
                           "pf_update_history already exchanged and rebuilt the tables");
  return build_group_tables(c, S(stream));
}

static pf_status launch_admit(pf_ctx* c, const int32_t* run_off, const int32_t* input_len,
                              const int32_t* generated, const int32_t* q_off,
                              const int32_t* q_input_len, const int32_t* max_new,
                              const int32_t* capacity, uint32_t tick, int32_t* admitted_out,
                              int32_t* peak_out, int32_t* peak_running_out, int32_t* pred_run_out,
                              int32_t* pred_q_out, cudaStream_t s,
                              const int32_t* lhat_run = nullptr, const int32_t* lhat_q = nullptr) {
  const pf_config& C = c->cfg;
  if (!c->committed)
    return fail(PF_ESTATE, "shared mode with nranks > 1: all-reduce the exchange buffer and call "
                           "pf_commit_history before the first admit / estimate");
  pf::AdmitParams p;
  memset(&p, 0, sizeof(p));
  p.n = C.n_instances;
  p.w = C.window;
  p.max_len = C.max_len;
  p.max_input_len = C.max_input_len;
  p.max_entries = C.max_entries;
  p.mode = C.mode;
  p.quantile_u = C.quantile_u;
  p.R = C.repetitions;
  p.bp = C.reserved_bp;
  p.seed = C.seed;
  p.tick = tick;
  p.instance_base = C.instance_base;
  p.members_per_group = C.members_per_group;
  p.member_base = C.member_base;
  p.edges = c->edges;
  p.team_smem = c->team_smem;
  p.ent_cap = c->ent_cap;
  p.sorted = c->sorted;
  p.hist = c->hist;
  p.gC = c->gC ? c->gC + (size_t)c->tbuf * C.n_groups * c->c_stride : nullptr;
  p.gS = c->gS ? c->gS + (size_t)c->tbuf * C.n_groups * c->s_stride : nullptr;
  p.c_stride = c->c_stride;
  p.cbits = c->cbits;
  p.csh = 0;
  while (((C.max_len + 1) >> p.csh) > (1 << c->cbits)) ++p.csh;
  p.s_stride = c->s_stride;
  p.n_groups = C.n_groups;
  p.dist_of = c->dist_of;
  p.group_off = c->group_off;
  p.run_off = run_off;
  p.input_len = input_len;
  p.generated = generated;
  p.q_off = q_off;
  p.q_input_len = q_input_len;
  p.max_new = max_new;
  p.capacity = capacity;
  p.admitted_out = admitted_out;
  p.peak_out = peak_out;
  p.peak_running_out = peak_running_out;
  p.pred_run_out = pred_run_out;
  p.pred_q_out = pred_q_out;
  p.lhat_run = lhat_run;
  p.lhat_q = lhat_q;
  p.err = c->err;
  if (c->gp_warps && !lhat_run) {
    const bool est = (q_off == nullptr);
    PF_CUDA(ensure_smem(group_fn(c, est), (int)c->gp_smem));
    const int grid = std::max(1, std::min(c->sms, C.n_instances));
    p.gcost = c->gcost;
    p.cost_epoch = c->cost_epoch++;
    // multi-rank contexts: leave a few SMs free near the end for the overlapped side chain
    // (PFSCHED_EARLY_CYCLES overrides; 0 = off)
    {
      const char* ec = getenv("PFSCHED_EARLY_CYCLES");
      p.early_cycles = ec ? (uint32_t)atoi(ec) : (C.nranks > 1 ? 120000u : 0u);
    }
    void* args[] = {&p};
    PF_CUDA(cudaLaunchKernel(group_fn(c, est), dim3(grid), dim3(c->gp_warps * 32), args, c->gp_smem, s));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
  const Variant& V = kVariants[c->variant];
  const int teams = c->teams;
  p.teams = teams;
  const int grid = (C.n_instances + teams - 1) / teams;
  PF_CUDA(ensure_smem(reinterpret_cast<const void*>(V.fn[c->layout][c->pack]), (int)c->admit_smem,
                      c->carveout));
  V.fn[c->layout][c->pack]<<<grid, teams * V.TW * 32, c->admit_smem, s>>>(p);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

pf_status pf_estimate_peak(pf_ctx* c, const int32_t* run_off, const int32_t* input_len,
                           const int32_t* generated, const int32_t* max_new, uint32_t tick,
                           int32_t* peak_out, int32_t* pred_out, void* stream) {
  if (!c || !run_off || !input_len || !generated || !max_new || !peak_out)
    return fail(PF_EINVAL, "pf_estimate_peak: NULL required pointer");
  return launch_admit(c, run_off, input_len, generated, nullptr, nullptr, max_new, nullptr, tick,
                      nullptr, peak_out, nullptr, pred_out, nullptr, S(stream));
}

pf_status pf_admit(pf_ctx* c, const int32_t* run_off, const int32_t* input_len,
                   const int32_t* generated, const int32_t* q_off, const int32_t* q_input_len,
                   const int32_t* max_new, const int32_t* capacity, uint32_t tick,
                   int32_t* admitted_out, int32_t* peak_out, int32_t* peak_running_out,
                   int32_t* pred_run_out, int32_t* pred_q_out, void* stream) {
  if (!c || !run_off || !input_len || !generated || !q_off || !q_input_len || !max_new ||
      !capacity || !admitted_out || !peak_out)
    return fail(PF_EINVAL, "pf_admit: NULL required pointer");
  return launch_admit(c, run_off, input_len, generated, q_off, q_input_len, max_new, capacity,
                      tick, admitted_out, peak_out, peak_running_out, pred_run_out, pred_q_out,
                      S(stream));
}

pf_status pf_admit_override(pf_ctx* c, const int32_t* run_off, const int32_t* input_len,
                            const int32_t* generated, const int32_t* lhat_run,
                            const int32_t* q_off, const int32_t* q_input_len,
                            const int32_t* lhat_q, const int32_t* capacity,
                            int32_t* admitted_out, int32_t* peak_out,
                            int32_t* peak_running_out, void* stream) {
  if (!c || !run_off || !input_len || !generated || !lhat_run || !q_off || !q_input_len ||
      !lhat_q || !capacity || !admitted_out || !peak_out)
    return fail(PF_EINVAL, "pf_admit_override: NULL required pointer");
  return launch_admit(c, run_off, input_len, generated, q_off, q_input_len, nullptr, capacity, 0,
                      admitted_out, peak_out, peak_running_out, nullptr, nullptr, S(stream),
                      lhat_run, lhat_q);
}

pf_status pf_admit_baseline(pf_ctx* c, int32_t policy, int32_t ratio_bp, const int32_t* run_off,
                            const int32_t* input_len, const int32_t* generated,
                            const int32_t* q_off, const int32_t* q_input_len,
                            const int32_t* max_new, const int32_t* capacity,
                            int32_t* admitted_out, int32_t* used_out, void* stream) {
  if (!c || !run_off || !input_len || !generated || !q_off || !q_input_len || !max_new ||
      !capacity || !admitted_out)
    return fail(PF_EINVAL, "pf_admit_baseline: NULL required pointer");
  if (policy != PF_POLICY_AGGRESSIVE && policy != PF_POLICY_CONSERVATIVE)
    return fail(PF_EINVAL, "pf_admit_baseline: unknown policy %d", policy);
  if (ratio_bp < 1) return fail(PF_EINVAL, "pf_admit_baseline: ratio_bp must be >= 1");
  pf::BaselineParams p;
  p.n = c->cfg.n_instances;
  p.policy = policy;
  p.ratio_bp = ratio_bp;
  p.max_len = c->cfg.max_len;
  p.max_input_len = c->cfg.max_input_len;
  p.max_entries = c->cfg.max_entries;
  p.run_off = run_off;
  p.input_len = input_len;
  p.generated = generated;
  p.q_off = q_off;
  p.q_input_len = q_input_len;
  p.max_new = max_new;
  p.capacity = capacity;
  p.admitted_out = admitted_out;
  p.used_out = used_out;
  p.err = c->err;
  const int blocks = (int)(((int64_t)p.n * 32 + 255) / 256);
  pf::baseline_kernel<<<blocks, 256, 0, S(stream)>>>(p);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

pf_status pf_get_device_error(pf_ctx* c, int32_t* code, int32_t* index, void* stream) {
  if (!c || !code || !index) return fail(PF_EINVAL, "pf_get_device_error: NULL argument");
  int host[2] = {0, 0};
  PF_CUDA(cudaMemcpyAsync(host, c->err, 8, cudaMemcpyDeviceToHost, S(stream)));
  PF_CUDA(cudaStreamSynchronize(S(stream)));
  *code = host[0];
  *index = host[1];
  return PF_OK;
}

pf_status pf_clear_device_error(pf_ctx* c, void* stream) {
  if (!c) return fail(PF_EINVAL, "pf_clear_device_error: NULL ctx");
  PF_CUDA(cudaMemsetAsync(c->err, 0, 8, S(stream)));
  return PF_OK;
}

pf_status pf_export_history(pf_ctx* c, int32_t* rows_out, void* stream) {
  if (!c || !rows_out) return fail(PF_EINVAL, "pf_export_history: NULL argument");
  const int64_t total = (int64_t)c->n_rows * c->row_window;
  pf::export_rows_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>(c->ring, c->head, c->n_rows,
                                                                       c->row_window, rows_out);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

// ------------------------------------------------------------------ simulator (NEXT-2)
struct pf_sim {
  pf_sim_config cfg;
  pf_ctx* ctx = nullptr;
  int n = 0, n_req = 0;
  uint32_t t = 0;  // iteration index = the admission tick (C-8)
  // CUDA graphs of 1 and 8 iterations, captured on first use on a private stream. The
  // admission tick is a kernel parameter: before each replay the admit nodes' ticks are
  // set (cudaGraphExecKernelNodeSetParams), so the hot admit kernel is unchanged.
  cudaStream_t cap = nullptr;
  cudaGraph_t gr1 = nullptr, gr8 = nullptr;      // kept alive: their node handles are used
  cudaGraphExec_t g1 = nullptr, g8 = nullptr;
  std::vector<cudaGraphNode_t> adm1, adm8;          // admit nodes in iteration order
  std::vector<cudaKernelNodeParams> kp1, kp8;       // their launch configuration
  std::vector<pf::AdmitParams> prm1, prm8;          // and parameters
  int32_t* max_new = nullptr;
  int32_t* bufs[24] = {nullptr};
  int nbufs = 0;
  long long* metrics = nullptr;
  int32_t* counter = nullptr;
  pf::SimState st;
};

static void free_sim(pf_sim* m) {
  if (!m) return;
  if (m->g1) cudaGraphExecDestroy(m->g1);
  if (m->g8) cudaGraphExecDestroy(m->g8);
  if (m->gr1) cudaGraphDestroy(m->gr1);
  if (m->gr8) cudaGraphDestroy(m->gr8);
  if (m->cap) cudaStreamDestroy(m->cap);
  for (int b = 0; b < m->nbufs; ++b) cudaFree(m->bufs[b]);
  cudaFree(m->metrics);
  cudaFree(m->counter);
  if (m->ctx) free_ctx(m->ctx);
  delete m;
}

pf_status pf_sim_create(const pf_sim_config* cfg, const int32_t* req_off,
                        const int32_t* req_input, const int32_t* req_output,
                        const int32_t* max_new, const int32_t* capacity,
                        const int32_t* init_history, void* stream, pf_sim** out) {
  if (!cfg || !out || !req_off || !req_input || !req_output || !max_new || !capacity)
    return fail(PF_EINVAL, "pf_sim_create: NULL required pointer");
  *out = nullptr;
  const pf_sim_config& C = *cfg;
  if (C.n_instances < 1) return fail(PF_EINVAL, "pf_sim_create: n_instances must be >= 1");
  if (C.policy < PF_SIM_PAST_FUTURE || C.policy > PF_SIM_CONSERVATIVE)
    return fail(PF_EINVAL, "pf_sim_create: unknown policy %d", C.policy);
  const bool pf_like = C.policy == PF_SIM_PAST_FUTURE || C.policy == PF_SIM_OPTIMUM;
  if (pf_like ? (C.param_bp < 0 || C.param_bp > 9999) : C.param_bp < 1)
    return fail(PF_EINVAL, "pf_sim_create: param_bp out of range for the policy");
  if (C.max_input_len < 0 || C.max_len < 1 || C.max_input_len > (1 << 30) - C.max_len)
    return fail(PF_EINVAL, "pf_sim_create: bad max_len / max_input_len");
  cudaStream_t s = S(stream);
  const int n = C.n_instances;
  // host validation of the request lists (create may synchronise)
  std::vector<int32_t> ro(n + 1), mn(n), cp(n);
  PF_CUDA(cudaMemcpyAsync(ro.data(), req_off, (n + 1) * 4, cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaMemcpyAsync(mn.data(), max_new, n * 4, cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaMemcpyAsync(cp.data(), capacity, n * 4, cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaStreamSynchronize(s));
  if (ro[0] != 0) return fail(PF_EINVAL, "pf_sim_create: req_off[0] must be 0");
  for (int i = 0; i < n; ++i)
    if (ro[i + 1] < ro[i]) return fail(PF_EINVAL, "pf_sim_create: req_off decreasing at %d", i);
  const int N = ro[n];
  std::vector<int32_t> lp(N), L(N);
  if (N > 0) {
    PF_CUDA(cudaMemcpyAsync(lp.data(), req_input, (size_t)N * 4, cudaMemcpyDeviceToHost, s));
    PF_CUDA(cudaMemcpyAsync(L.data(), req_output, (size_t)N * 4, cudaMemcpyDeviceToHost, s));
    PF_CUDA(cudaStreamSynchronize(s));
  }
  for (int i = 0; i < n; ++i) {
    if (mn[i] < 1 || mn[i] > C.max_len) return fail(PF_EINVAL, "pf_sim_create: max_new[%d] out of range", i);
    for (int j = ro[i]; j < ro[i + 1]; ++j) {
      if (lp[j] < 0 || lp[j] > C.max_input_len || L[j] < 1 || L[j] > mn[i])
        return fail(PF_EINVAL, "pf_sim_create: request %d of instance %d out of range", j - ro[i], i);
      if ((int64_t)lp[j] + L[j] > cp[i])
        return fail(PF_EINVAL, "pf_sim_create: request %d of instance %d exceeds capacity", j - ro[i], i);
    }
  }
  pf_config pc;
  memset(&pc, 0, sizeof(pc));
  pc.n_instances = n;
  pc.window = C.window;
  pc.max_len = C.max_len;
  pc.max_input_len = C.max_input_len + C.max_len;  // queued l_p + generated (S-3)
  pc.max_entries = C.max_entries;
  pc.instance_base = C.instance_base;
  pc.mode = C.mode;
  pc.quantile_u = C.quantile_u;
  pc.repetitions = C.repetitions;
  pc.reserved_bp = pf_like ? C.param_bp : 0;
  pc.seed = C.seed;
  pc.nranks = 1;
  pf_sim* m = new pf_sim();
  m->cfg = C;
  m->n = n;
  m->n_req = N;
  pf_status st = pf_create(&pc, init_history, stream, &m->ctx);
  if (st != PF_OK) { free_sim(m); return st; }
  const int E = C.max_entries;
  const int64_t nE = (int64_t)n * E;
  auto alloc = [&](int64_t elems) -> int32_t* {
    int32_t* p = nullptr;
    if (cudaMalloc(&p, (size_t)std::max<int64_t>(elems, 1) * 4 + 16) != cudaSuccess) return nullptr;
    m->bufs[m->nbufs++] = p;
    return p;
  };
  pf::SimState& S_ = m->st;
  S_.n = n;
  S_.E = E;
  int32_t* req_off_d = alloc(n + 1);
  int32_t* lp_d = alloc(N);
  int32_t* L_d = alloc(N);
  int32_t* cap_d = alloc(n);
  m->max_new = alloc(n);
  S_.gen = alloc(N);
  S_.evc = alloc(N);
  S_.qbuf = alloc(N);
  S_.qhead = alloc(n);
  S_.qlen = alloc(n);
  S_.run_ids = alloc(nE);
  S_.run_k = alloc(n);
  S_.done = alloc(n);
  S_.comp_tmp = alloc(nE);
  S_.cnt = alloc(3LL * n);
  S_.off = alloc(3LL * (n + 1));
  S_.comp_len = alloc(nE);
  S_.c_lp = alloc(nE);
  S_.c_gen = alloc(nE);
  S_.c_lhat = alloc(nE);
  S_.q_lp = alloc(nE);
  S_.q_lhat = alloc(nE);
  S_.admitted = alloc(n);
  bool ok = m->nbufs == 23;
  for (int b = 0; b < m->nbufs; ++b) ok = ok && m->bufs[b] != nullptr;
  ok = ok && cudaMalloc(&m->metrics, (size_t)n * pf::SIM_NMETRICS * 8) == cudaSuccess;
  ok = ok && cudaMalloc(&m->counter, 16) == cudaSuccess;
  if (!ok) { free_sim(m); return fail(PF_ENOMEM, "pf_sim_create: device allocation failed"); }
  S_.req_off = req_off_d;
  S_.req_lp = lp_d;
  S_.req_L = L_d;
  S_.capacity = cap_d;
  S_.metrics = m->metrics;
  S_.err = m->ctx->err;
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMemcpyAsync(req_off_d, req_off, (n + 1) * 4, cudaMemcpyDeviceToDevice, s);
  if (N > 0) {
    e = e ? e : cudaMemcpyAsync(lp_d, req_input, (size_t)N * 4, cudaMemcpyDeviceToDevice, s);
    e = e ? e : cudaMemcpyAsync(L_d, req_output, (size_t)N * 4, cudaMemcpyDeviceToDevice, s);
  }
  e = e ? e : cudaMemcpyAsync(cap_d, capacity, n * 4, cudaMemcpyDeviceToDevice, s);
  e = e ? e : cudaMemcpyAsync(m->max_new, max_new, n * 4, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) { free_sim(m); return fail(PF_ECUDA, "pf_sim_create: %s", cudaGetErrorString(e)); }
  pf::sim_init_kernel<<<(n + 127) / 128, 128, 0, s>>>(S_);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { free_sim(m); return fail(PF_ECUDA, "pf_sim_create: %s", cudaGetErrorString(e)); }
  *out = m;
  return PF_OK;
}

namespace {
// One simulator iteration (six launches) with admission tick m->t.
pf_status sim_iteration(pf_sim* m, cudaStream_t s) {
  const pf::SimState& st = m->st;
  const int n = m->n, n1 = n + 1;
  const int wblocks = (int)(((int64_t)n * 32 + 255) / 256);
  int32_t* comp_off = st.off;
  int32_t* run_off = st.off + n1;
  int32_t* q_off = st.off + 2 * n1;
  pf::sim_finish_kernel<<<wblocks, 256, 0, s>>>(st);
  pf::sim_scan_kernel<<<1, 1024, 0, s>>>(n, st.cnt, st.off);
  pf::sim_gather_kernel<<<wblocks, 256, 0, s>>>(st);
  PF_CUDA(cudaGetLastError());
  pf_status r = PF_OK;
  switch (m->cfg.policy) {
    case PF_SIM_PAST_FUTURE:
      r = pf_update_history(m->ctx, comp_off, st.comp_len, 1, s);
      if (r == PF_OK)
        r = launch_admit(m->ctx, run_off, st.c_lp, st.c_gen, q_off, st.q_lp, m->max_new,
                         st.capacity, m->t, st.admitted, st.comp_tmp /* peak: scratch */,
                         nullptr, nullptr, nullptr, s);
      break;
    case PF_SIM_OPTIMUM:
      r = launch_admit(m->ctx, run_off, st.c_lp, st.c_gen, q_off, st.q_lp, nullptr,
                       st.capacity, 0, st.admitted, st.comp_tmp, nullptr, nullptr, nullptr, s,
                       st.c_lhat, st.q_lhat);
      break;
    default:
      r = pf_admit_baseline(m->ctx, m->cfg.policy == PF_SIM_AGGRESSIVE ? PF_POLICY_AGGRESSIVE
                                                                        : PF_POLICY_CONSERVATIVE,
                            m->cfg.param_bp, run_off, st.c_lp, st.c_gen, q_off, st.q_lp,
                            m->max_new, st.capacity, st.admitted, nullptr, s);
  }
  if (r != PF_OK) return r;
  pf::sim_apply_kernel<<<wblocks, 256, 0, s>>>(st);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

// Capture `iters` iterations into an executable graph; collect the past-future admit
// kernel nodes (in capture order = iteration order) and their parameters.
pf_status sim_capture(pf_sim* m, int iters, cudaGraph_t* graph, cudaGraphExec_t* out,
                      std::vector<cudaGraphNode_t>& nodes, std::vector<cudaKernelNodeParams>& kps,
                      std::vector<pf::AdmitParams>& prms) {
  PF_CUDA(cudaStreamBeginCapture(m->cap, cudaStreamCaptureModeThreadLocal));
  pf_status r = PF_OK;
  for (int u = 0; u < iters && r == PF_OK; ++u) r = sim_iteration(m, m->cap);
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(m->cap, &g);
  if (r != PF_OK) {
    if (g) cudaGraphDestroy(g);
    return r;
  }
  PF_CUDA(e);
  nodes.clear();
  kps.clear();
  prms.clear();
  if (m->cfg.policy == PF_SIM_PAST_FUTURE) {
    const void* fn = reinterpret_cast<const void*>(kVariants[m->ctx->variant].fn[m->ctx->layout][m->ctx->pack]);
    // walk the (linear) chain from its root in dependency order
    size_t nn = 0;
    cudaGraphGetRootNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> cur(nn);
    cudaGraphGetRootNodes(g, cur.data(), &nn);
    while (!cur.empty()) {
      cudaGraphNode_t nd = cur[0];
      cudaGraphNodeType ty;
      cudaGraphNodeGetType(nd, &ty);
      if (ty == cudaGraphNodeTypeKernel) {
        cudaKernelNodeParams kp;
        if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == fn) {
          nodes.push_back(nd);
          prms.push_back(*reinterpret_cast<pf::AdmitParams*>(kp.kernelParams[0]));
          kp.kernelParams = nullptr;
          kp.extra = nullptr;
          kps.push_back(kp);
        }
      }
      size_t nd_n = 0;
      cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_n);
      cur.resize(nd_n);
      if (nd_n) cudaGraphNodeGetDependentNodes(nd, cur.data(), &nd_n);
    }
    if ((int)nodes.size() != iters) {
      cudaGraphDestroy(g);
      return fail(PF_ECUDA, "pf_sim_step: found %d admit nodes in a %d-iteration graph", (int)nodes.size(), iters);
    }
  }
  const cudaError_t e2 = cudaGraphInstantiate(out, g, 0);
  if (e2 != cudaSuccess) cudaGraphDestroy(g);
  PF_CUDA(e2);
  *graph = g;
  return PF_OK;
}

pf_status sim_replay(pf_sim* m, cudaGraphExec_t ex, std::vector<cudaGraphNode_t>& nodes,
                     std::vector<cudaKernelNodeParams>& kps, std::vector<pf::AdmitParams>& prms,
                     cudaStream_t s) {
  for (size_t u = 0; u < nodes.size(); ++u) {  // the ticks of this replay's iterations
    prms[u].tick = m->t + (uint32_t)u;
    void* args[1] = {&prms[u]};
    cudaKernelNodeParams kp = kps[u];
    kp.kernelParams = args;
    PF_CUDA(cudaGraphExecKernelNodeSetParams(ex, nodes[u], &kp));
  }
  PF_CUDA(cudaGraphLaunch(ex, s));
  return PF_OK;
}
}  // namespace

pf_status pf_sim_step(pf_sim* m, int32_t iterations, void* stream) {
  if (!m) return fail(PF_EINVAL, "pf_sim_step: NULL sim");
  if (iterations < 0) return fail(PF_EINVAL, "pf_sim_step: iterations must be >= 0");
  cudaStream_t s = S(stream);
  if (iterations < 4) {  // a few iterations: plain launches
    for (int32_t it = 0; it < iterations; ++it, ++m->t) {
      pf_status r = sim_iteration(m, s);
      if (r != PF_OK) return r;
    }
    return PF_OK;
  }
  // CUDA-graph replays: 8-iteration graphs, then single-iteration ones
  if (!m->g1) {
    PF_CUDA(cudaStreamCreateWithFlags(&m->cap, cudaStreamNonBlocking));
    pf_status r = sim_capture(m, 1, &m->gr1, &m->g1, m->adm1, m->kp1, m->prm1);
    if (r == PF_OK) r = sim_capture(m, 8, &m->gr8, &m->g8, m->adm8, m->kp8, m->prm8);
    if (r != PF_OK) return r;
  }
  for (; iterations >= 8; iterations -= 8, m->t += 8) {
    pf_status r = sim_replay(m, m->g8, m->adm8, m->kp8, m->prm8, s);
    if (r != PF_OK) return r;
  }
  for (; iterations > 0; --iterations, ++m->t) {
    pf_status r = sim_replay(m, m->g1, m->adm1, m->kp1, m->prm1, s);
    if (r != PF_OK) return r;
  }
  return PF_OK;
}

pf_status pf_sim_done(pf_sim* m, int32_t* n_done, void* stream) {
  if (!m || !n_done) return fail(PF_EINVAL, "pf_sim_done: NULL argument");
  cudaStream_t s = S(stream);
  pf::sim_count_done_kernel<<<1, 1024, 0, s>>>(m->n, m->st.done, m->counter);
  PF_CUDA(cudaGetLastError());
  PF_CUDA(cudaMemcpyAsync(n_done, m->counter, 4, cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaStreamSynchronize(s));
  return PF_OK;
}

pf_status pf_sim_metrics(pf_sim* m, int64_t* metrics_out, int32_t* generated_out,
                         int32_t* evictions_out, void* stream) {
  if (!m || !metrics_out) return fail(PF_EINVAL, "pf_sim_metrics: NULL argument");
  cudaStream_t s = S(stream);
  PF_CUDA(cudaMemcpyAsync(metrics_out, m->metrics, (size_t)m->n * pf::SIM_NMETRICS * 8,
                          cudaMemcpyDeviceToDevice, s));
  if (generated_out && m->n_req > 0)
    PF_CUDA(cudaMemcpyAsync(generated_out, m->st.gen, (size_t)m->n_req * 4, cudaMemcpyDeviceToDevice, s));
  if (evictions_out && m->n_req > 0)
    PF_CUDA(cudaMemcpyAsync(evictions_out, m->st.evc, (size_t)m->n_req * 4, cudaMemcpyDeviceToDevice, s));
  return PF_OK;
}

pf_ctx* pf_sim_context(pf_sim* m) { return m ? m->ctx : nullptr; }

pf_status pf_sim_destroy(pf_sim* m) {
  if (!m) return fail(PF_EINVAL, "pf_sim_destroy: NULL sim");
  cudaDeviceSynchronize();
  free_sim(m);
  return PF_OK;
}

// ------------------------------------------------------------------ analysis (NEXT-3)
static pf_status check_lengths(const int32_t* x, int64_t n, int32_t max_len, cudaStream_t s,
                               const char* who) {
  int* flag = nullptr;
  PF_CUDA(cudaMallocAsync(&flag, 4, s));
  cudaMemsetAsync(flag, 0, 4, s);
  pf::lengths_check_kernel<<<296, 256, 0, s>>>(x, n, max_len, flag);
  int h = 0;
  cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(flag, s);
  PF_CUDA(cudaStreamSynchronize(s));
  if (h) return fail(PF_EINVAL, "%s: a length is outside [1, max_len]", who);
  return PF_OK;
}

pf_status pf_window_similarity(const int32_t* lengths, int64_t n, int32_t window, int32_t max_len,
                               int64_t* gram_out, double* cos_out, double* summary_out,
                               void* stream) {
  if (!lengths) return fail(PF_EINVAL, "pf_window_similarity: NULL lengths");
  if (window < 1 || n < 2LL * window) return fail(PF_EINVAL, "pf_window_similarity: fewer than 2 windows");
  if (max_len < 1 || max_len > 32767) return fail(PF_ERANGE, "pf_window_similarity: max_len must be in [1, 32767]");
  const int64_t B64 = n / window;
  if (B64 > 46340) return fail(PF_ERANGE, "pf_window_similarity: more than 46340 windows");
  const int B = (int)B64;
  cudaStream_t s = S(stream);
  pf_status st = check_lengths(lengths, B64 * window, max_len, s, "pf_window_similarity");
  if (st != PF_OK) return st;
  long long* G = reinterpret_cast<long long*>(gram_out);
  double* C = cos_out;
  if (!G) PF_CUDA(cudaMallocAsync(&G, (size_t)B * B * 8, s));
  if (!C && summary_out) PF_CUDA(cudaMallocAsync(&C, (size_t)B * B * 8, s));
  const size_t smem = (size_t)(max_len + 1) * 4;
  if (smem > 48 * 1024)
    PF_CUDA(ensure_smem(reinterpret_cast<const void*>(pf::gram_kernel), (int)smem));
  pf::gram_kernel<<<B, 512, smem, s>>>(lengths, window, B, max_len, G);
  PF_CUDA(cudaGetLastError());
  if (C) {
    const int64_t t = (int64_t)B * B;
    pf::cosine_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(G, B, C);
    if (summary_out) pf::similarity_summary_kernel<<<1, 1024, 0, s>>>(C, B, summary_out);
    PF_CUDA(cudaGetLastError());
  }
  if (!gram_out) cudaFreeAsync(G, s);
  if (!cos_out && C) cudaFreeAsync(C, s);
  return PF_OK;
}

pf_status pf_adjacent_similarity(const int32_t* lengths, int64_t n, int32_t hist_window,
                                 int32_t run_window, int32_t max_len, double* cos_out,
                                 double* mean_out, void* stream) {
  if (!lengths || !cos_out) return fail(PF_EINVAL, "pf_adjacent_similarity: NULL argument");
  if (hist_window < 1 || run_window < 1 || n < (int64_t)hist_window + run_window)
    return fail(PF_EINVAL, "pf_adjacent_similarity: no running window");
  if (max_len < 1 || max_len > 27000) return fail(PF_ERANGE, "pf_adjacent_similarity: max_len must be in [1, 27000]");
  const int64_t K64 = (n - hist_window) / run_window;
  if (K64 > (1LL << 31) - 1) return fail(PF_ERANGE, "pf_adjacent_similarity: too many windows");
  const int K = (int)K64;
  cudaStream_t s = S(stream);
  pf_status st = check_lengths(lengths, hist_window + K64 * run_window, max_len, s, "pf_adjacent_similarity");
  if (st != PF_OK) return st;
  const size_t smem = (size_t)2 * (max_len + 1) * 4;
  if (smem > 48 * 1024)
    PF_CUDA(ensure_smem(reinterpret_cast<const void*>(pf::adjacent_kernel), (int)smem));
  pf::adjacent_kernel<<<K, 512, smem, s>>>(lengths, hist_window, run_window, max_len, cos_out);
  if (mean_out) pf::mean_kernel<<<1, 1024, 0, s>>>(cos_out, K, mean_out);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

// ------------------------------------------------------------------ forwarding (NEXT-4)
pf_status pf_forward(pf_ctx* c, int32_t cluster_size, const int32_t* run_off,
                     const int32_t* input_len, const int32_t* generated, const int32_t* max_new,
                     const int32_t* capacity, const int32_t* cq_off, const int32_t* cq_input_len,
                     uint32_t tick, int32_t* dest_out, int32_t* forwarded_out, int32_t* peak_out,
                     void* stream) {
  if (!c || !run_off || !input_len || !generated || !max_new || !capacity || !cq_off ||
      !cq_input_len || !dest_out || !forwarded_out || !peak_out)
    return fail(PF_EINVAL, "pf_forward: NULL required pointer");
  const pf_config& C = c->cfg;
  if (cluster_size < 1 || cluster_size > 32 || C.n_instances % cluster_size)
    return fail(PF_EINVAL, "pf_forward: cluster_size must be in [1, 32] and divide n_instances");
  if (c->layout != LAYOUT_SORTED)
    return fail(PF_ESTATE, "pf_forward: needs per-instance windows with w <= Lmax+1");
  if (C.mode == PF_MODE_SAMPLE && C.repetitions != 1)
    return fail(PF_ESTATE, "pf_forward: sampling mode supports repetitions = 1");
  const size_t smem = (size_t)cluster_size * C.max_entries * 8;
  if (smem > 200 * 1024)
    return fail(PF_ERANGE, "pf_forward: cluster_size * max_entries * 8 B must be <= 200 KB");
  pf::ForwardParams P;
  P.n_clusters = C.n_instances / cluster_size;
  P.S = cluster_size;
  P.E = C.max_entries;
  P.w = C.window;
  P.max_len = C.max_len;
  P.max_input_len = C.max_input_len;
  P.mode = C.mode;
  P.bp = C.reserved_bp;
  P.quantile_u = C.quantile_u;
  P.tick = tick;
  P.seed = C.seed;
  P.instance_base = C.instance_base;
  P.sorted = c->sorted;
  P.run_off = run_off;
  P.input_len = input_len;
  P.generated = generated;
  P.max_new = max_new;
  P.capacity = capacity;
  P.cq_off = cq_off;
  P.cq_input_len = cq_input_len;
  P.dest_out = dest_out;
  P.forwarded_out = forwarded_out;
  P.peak_out = peak_out;
  P.err = c->err;
  if (smem > 48 * 1024)
    PF_CUDA(ensure_smem(reinterpret_cast<const void*>(pf::forward_kernel), (int)smem));
  pf::forward_kernel<<<P.n_clusters, cluster_size * 32, smem, S(stream)>>>(P);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

}  // extern "C"
