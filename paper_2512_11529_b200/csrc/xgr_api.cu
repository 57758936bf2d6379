// C ABI of the xBeam library (include/xgr_beam.h): argument validation, ownership, sequencing,
// the fixed per-context workspace ("reuses the data structure previously occupied
// by old sequences") and the per-step route choice. No kernel code here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: a no-op unless a profiler is attached

#include "xgr_internal.cuh"

// NVTX range over one ABI call (nsys / ncu --nvtx timelines show the host calls per step)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace xgr {
cudaError_t configure_kernels(int cap);
cudaError_t launch_step(const StepArgs& a, int rows, bool sparse_route, int sparse_keys,
                        cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1, int* launches);
cudaError_t launch_shard_stats(const StepArgs& a, int rows, cudaStream_t s);
cudaError_t launch_shard_select(const StepArgs& a, int rows, cudaStream_t s, int* launches);
cudaError_t launch_shard_stats_sparse(const StepArgs& a, int rows, cudaStream_t s);
cudaError_t launch_shard_select_sparse(const StepArgs& a, int sparse_keys, cudaStream_t s);
cudaError_t launch_shard_merge(const StepArgs& a, const uint64_t* grec, const int32_t* grec_n,
                               cudaStream_t s);
cudaError_t merge_fits(int nranks, int bw, int device, bool* ok);
bool stream_supported(int V);
cudaError_t launch_children(const TrieDev& tr, const int32_t* prefixes, int depth, int64_t n,
                            int32_t* counts, int32_t* tokens, int64_t cap, cudaStream_t s);
cudaError_t launch_account(const StepArgs& a, int rows, uint32_t* touched,
                           unsigned long long* out, cudaStream_t s);
}  // namespace xgr

using namespace xgr;

struct xgr_ctx {
  xgr_config cfg;
  DevAlloc al;                      // cfg.dev_alloc / dev_free, else cudaMalloc / cudaFree
  void* host_stage = nullptr;       // xgr_beam_step_host: device copy of the step's logits
  size_t host_stage_bytes = 0;
  int V = 0, nd = 0, BW = 0, maxB = 0, cap = 0, R0 = 0, K = 0;
  TrieHost trie;
  bool built = false;
  float* score[2] = {nullptr, nullptr};
  uint32_t* node[2] = {nullptr, nullptr};
  int32_t* nlive[2] = {nullptr, nullptr};
  int32_t* parent_hist = nullptr;  // [nd][maxB][BW]
  int32_t* token_hist = nullptr;
  int32_t** d_phist = nullptr;     // device array of nd pointers
  int32_t** d_thist = nullptr;
  uint32_t* scratch = nullptr;     // [3][maxB]: theta, survivor count, overflow marker
  uint32_t* next_keys[2] = {nullptr, nullptr};   // per-request next-step candidates (route), by step parity
  int32_t* dense_list = nullptr;   // [1 + maxB]: a mixed step's dense-route requests
  uint64_t* ph_lists = nullptr;    // XGR_CFG_PAPER_HEAP: [maxB][BW][K] per-beam sorted Top-K
  int32_t* ph_cnt = nullptr;       // [maxB][BW]
  uint32_t* seed_hist = nullptr;   // [maxB][kSeedBins]
  uint32_t* seed_cnt = nullptr;    // [maxB]
  float* head_logits = nullptr;    // [maxB][kSparseCap]: legal logits of a fused-head sparse step
  uint64_t* surv = nullptr;        // [maxB][cap]
  float* lse = nullptr;            // [maxB][BW]
  uint32_t* flags = nullptr;       // [maxB]
  unsigned long long* counters = nullptr;  // [XGR_NUM_COUNTERS]
  int32_t* out_tokens = nullptr;   // finalize staging for host outputs
  int64_t* out_rank = nullptr;
  float* out_score = nullptr;
  int32_t* out_nlive = nullptr;
  int step = 0;
  int batch = 0;
  // last step's launch arguments (support calls: account)
  StepArgs last{};
  int last_rows = 0;
  int64_t launches = 0;             // kernels launched by this ctx (host-side count)
  // codebook shard (nranks > 1)
  float2* shard_stats = nullptr;    // [maxB][BW] this rank's (m, Z)
  uint64_t* shard_rec = nullptr;    // [maxB][BW] this rank's local top-BW keys
  int32_t* shard_rec_n = nullptr;   // [maxB]
  StepArgs shard_args{};
  int shard_rows = 0;
  int shard_phase = 0;              // 0: expect stats, 1: expect select, 2: expect merge
  int shard_sparse_keys = 0;        // > 0: this shard step takes the sparse route
  // XGR_CFG_TIMING: ring of event pairs around the dense-route streaming kernel
  std::vector<cudaEvent_t> ev;      // 2 * kTimingRing
  std::vector<int32_t> ev_step;
  int64_t ev_head = 0, ev_tail = 0;
};
static constexpr int kTimingRing = 4096;

namespace xgr {
bool pdl_enabled() {
  // off by default: neutral in eager streams (0.477 vs 0.475 ms per C3 pass); inside CUDA graphs
  // 0.436 vs 0.438 ms with the implicit trigger at kernel exit, and 0.640 ms when every kernel
  // triggers its dependents at entry (XGR_DEBUG_FLAGS bit 20). XGR_PDL=1 enables it
  static const bool on = getenv("XGR_PDL") && atoi(getenv("XGR_PDL")) == 1;
  return on;
}
}  // namespace xgr

static thread_local std::string g_err;

static xgr_status fail(xgr_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define ACK(x)                                                                              \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? XGR_ERR_OOM : XGR_ERR_CUDA, "%s: %s", #x, \
                  cudaGetErrorString(e_));                                                  \
  } while (0)

static void ctx_free(xgr_ctx* c) {
  // a caller's allocator may hand the memory to other work at once: nothing of this ctx may still run
  if (c->al.release) cudaDeviceSynchronize();
  for (auto e : c->ev) cudaEventDestroy(e);
  c->ev.clear();
  trie_free(c->trie);
  c->al.put(c->host_stage);
  c->host_stage = nullptr;
  c->host_stage_bytes = 0;
  for (int i = 0; i < 2; ++i) {
    c->al.put(c->score[i]);
    c->al.put(c->node[i]);
    c->al.put(c->nlive[i]);
  }
  c->al.put(c->parent_hist);
  c->al.put(c->token_hist);
  c->al.put(c->d_phist);
  c->al.put(c->d_thist);
  c->al.put(c->scratch);
  c->al.put(c->ph_lists);
  c->al.put(c->ph_cnt);
  c->al.put(c->dense_list);
  c->al.put(c->next_keys[0]);
  c->al.put(c->next_keys[1]);
  c->al.put(c->seed_hist);
  c->al.put(c->seed_cnt);
  c->al.put(c->head_logits);
  c->al.put(c->surv);
  c->al.put(c->lse);
  c->al.put(c->flags);
  c->al.put(c->counters);
  c->al.put(c->out_tokens);
  c->al.put(c->out_rank);
  c->al.put(c->out_score);
  c->al.put(c->out_nlive);
  c->al.put(c->shard_stats);
  c->al.put(c->shard_rec);
  c->al.put(c->shard_rec_n);
}

namespace xgr {
cudaError_t launch_head(const StepArgs& a, const void* hidden, int64_t ldh, int64_t hreq, const void* head,
                        int64_t ldw, const float* bias, int d, float* clog, cudaStream_t s);
cudaError_t launch_sparse_compact(const StepArgs& a, int sparse_keys, cudaStream_t s, int* launches);
}

extern "C" {

const char* xgr_last_error(void) { return g_err.c_str(); }
int32_t xgr_abi_version(void) { return XGR_ABI_VERSION; }

xgr_status xgr_beam_init(const xgr_config* cfg, xgr_ctx** out) {
  if (!out) return fail(XGR_ERR_INVALID_ARG, "init: out is NULL");
  *out = nullptr;
  if (!cfg) return fail(XGR_ERR_INVALID_ARG, "init: cfg is NULL");
  const xgr_config& c = *cfg;
  if (c.vocab < 1 || c.vocab > 65536) return fail(XGR_ERR_INVALID_ARG, "init: vocab %d not in 1..65536", c.vocab);
  if (c.nd < 1 || c.nd > kMaxND) return fail(XGR_ERR_INVALID_ARG, "init: nd %d not in 1..8", c.nd);
  int w = 1;
  while ((1 << w) < c.vocab) ++w;
  if (w * c.nd > 64) return fail(XGR_ERR_UNSUPPORTED, "init: nd * ceil(log2 V) = %d > 64", w * c.nd);
  if (c.beam_width < 1 || c.beam_width > kMaxBW)
    return fail(XGR_ERR_INVALID_ARG, "init: beam_width %d not in 1..1024", c.beam_width);
  if (c.top_k < 0) return fail(XGR_ERR_INVALID_ARG, "init: top_k < 0");
  if (c.top_k > 0 && c.top_k < c.beam_width && c.nranks > 1)
    return fail(XGR_ERR_UNSUPPORTED, "init: per-beam top_k < beam_width with the codebook shard");
  if (c.top_k > 0 && c.top_k < c.beam_width && c.vocab > 16384)
    return fail(XGR_ERR_UNSUPPORTED, "init: per-beam top_k < beam_width needs vocab <= 16384");
  if (c.max_batch < 1) return fail(XGR_ERR_INVALID_ARG, "init: max_batch < 1");
  if (c.nranks < 1 || c.rank < 0 || c.rank >= c.nranks)
    return fail(XGR_ERR_INVALID_ARG, "init: need 0 <= rank < nranks");
  if (c.nccl_id) return fail(XGR_ERR_UNSUPPORTED, "init: nccl_id must be NULL (the caller performs the all-gathers)");
  if (c.nranks > 1) {
    if (c.vocab % c.nranks != 0) return fail(XGR_ERR_INVALID_ARG, "init: vocab %% nranks != 0");
    const int vl = c.vocab / c.nranks;
    if (vl % 128 != 0 || vl > 8192)
      return fail(XGR_ERR_UNSUPPORTED, "init: codebook shard needs V/nranks a multiple of 128 and <= 8192");
    if (c.nranks > 64) return fail(XGR_ERR_UNSUPPORTED, "init: nranks > 64");
  }
  if (c.survivor_cap < 0 || c.theta_rows < 0) return fail(XGR_ERR_INVALID_ARG, "init: negative knob");
  for (int i = 0; i < 5; ++i)
    if (c.reserved[i]) return fail(XGR_ERR_INVALID_ARG, "init: reserved fields must be zero");
  if (!c.dev_alloc != !c.dev_free)
    return fail(XGR_ERR_INVALID_ARG, "init: dev_alloc and dev_free must be given together");
  if ((c.flags & XGR_CFG_PAPER_HEAP) && (c.vocab > 16384 || c.nranks > 1))
    return fail(XGR_ERR_UNSUPPORTED, "init: the paper-heap baseline needs vocab <= 16384 and no codebook shard");
  if (c.flags & ~(XGR_CFG_NO_PRUNE | XGR_CFG_COUNTERS | XGR_CFG_NO_SPARSE_KERNEL | XGR_CFG_TIMING | XGR_CFG_PAPER_HEAP))
    return fail(XGR_ERR_INVALID_ARG, "init: unknown flags 0x%x", c.flags);
  int ndev = 0;
  ACK(cudaGetDeviceCount(&ndev));
  if (c.device < 0 || c.device >= ndev) return fail(XGR_ERR_INVALID_ARG, "init: bad device %d", c.device);
  ACK(cudaSetDevice(c.device));
  if (c.nranks > 1) {
    bool ok = false;
    ACK(merge_fits(c.nranks, c.beam_width, c.device, &ok));
    if (!ok)
      return fail(XGR_ERR_UNSUPPORTED, "init: the shard merge of nranks x beam_width = %d keys exceeds shared memory",
                  c.nranks * c.beam_width);
  }

  xgr_ctx* x = new xgr_ctx();
  x->cfg = c;
  x->V = c.vocab;
  x->nd = c.nd;
  x->BW = c.beam_width;
  x->maxB = c.max_batch;
  x->cap = c.survivor_cap ? c.survivor_cap : std::min(32 * c.beam_width, 16384);
  x->cap = std::max(x->cap, c.beam_width);
  if (x->cap > 16384) {
    delete x;
    return fail(XGR_ERR_INVALID_ARG, "init: survivor_cap > 16384");
  }
  x->R0 = c.theta_rows ? c.theta_rows : 8;
  x->K = (c.top_k > 0 && c.top_k < c.beam_width) ? c.top_k : 0;   // 0: no per-beam truncation
  const size_t nb = (size_t)x->maxB * x->BW;
  x->al.alloc = c.dev_alloc;
  x->al.release = c.dev_free;
  x->al.user = c.alloc_user;
  x->trie.al = x->al;
  auto al = [&](void** p, size_t bytes) -> cudaError_t { return x->al.get(p, bytes); };
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = al((void**)&x->score[i], nb * 4);
    if (e == cudaSuccess) e = al((void**)&x->node[i], nb * 4);
    if (e == cudaSuccess) e = al((void**)&x->nlive[i], (size_t)x->maxB * 4);
  }
  if (e == cudaSuccess) e = al((void**)&x->parent_hist, nb * x->nd * 4);
  if (e == cudaSuccess) e = al((void**)&x->token_hist, nb * x->nd * 4);
  if (e == cudaSuccess) e = al((void**)&x->d_phist, x->nd * sizeof(void*));
  if (e == cudaSuccess) e = al((void**)&x->d_thist, x->nd * sizeof(void*));
  if (e == cudaSuccess) e = al((void**)&x->scratch, 3 * (size_t)x->maxB * 4);
  if (e == cudaSuccess && (c.flags & XGR_CFG_PAPER_HEAP)) {
    const size_t K = x->K ? x->K : x->BW;
    e = al((void**)&x->ph_lists, nb * K * 8);
    if (e == cudaSuccess) e = al((void**)&x->ph_cnt, nb * 4);
  }
  if (e == cudaSuccess) e = al((void**)&x->dense_list, (size_t)(x->maxB + 1) * 4);
  if (e == cudaSuccess) e = al((void**)&x->next_keys[0], (size_t)x->maxB * 4);
  if (e == cudaSuccess) e = al((void**)&x->next_keys[1], (size_t)x->maxB * 4);
  if (e == cudaSuccess) e = al((void**)&x->seed_hist, (size_t)x->maxB * kSeedBins * 4);
  if (e == cudaSuccess) e = al((void**)&x->head_logits, (size_t)x->maxB * kSparseCap * 4);
  if (e == cudaSuccess) e = cudaMemset(x->seed_hist, 0, (size_t)x->maxB * kSeedBins * 4);
  if (e == cudaSuccess) e = al((void**)&x->seed_cnt, (size_t)x->maxB * 4);
  if (e == cudaSuccess) e = cudaMemset(x->seed_cnt, 0, (size_t)x->maxB * 4);
  if (e == cudaSuccess) e = al((void**)&x->surv, (size_t)x->maxB * x->cap * 8);
  if (e == cudaSuccess) e = al((void**)&x->lse, nb * 4);
  if (e == cudaSuccess) e = al((void**)&x->flags, (size_t)x->maxB * 4);
  if (e == cudaSuccess) e = al((void**)&x->counters, XGR_NUM_COUNTERS * 8);
  if (e == cudaSuccess) e = al((void**)&x->out_tokens, nb * x->nd * 4);
  if (e == cudaSuccess) e = al((void**)&x->out_rank, nb * 8);
  if (e == cudaSuccess) e = al((void**)&x->out_score, nb * 4);
  if (e == cudaSuccess) e = al((void**)&x->out_nlive, (size_t)x->maxB * 4);
  if (e == cudaSuccess && c.nranks > 1) {
    e = al((void**)&x->shard_stats, nb * sizeof(float2));
    if (e == cudaSuccess) e = al((void**)&x->shard_rec, nb * 8);
    if (e == cudaSuccess) e = al((void**)&x->shard_rec_n, (size_t)x->maxB * 4);
  }
  if (e == cudaSuccess) {
    std::vector<int32_t*> ph(x->nd), th(x->nd);
    for (int t = 0; t < x->nd; ++t) {
      ph[t] = x->parent_hist + (size_t)t * nb;
      th[t] = x->token_hist + (size_t)t * nb;
    }
    e = cudaMemcpy(x->d_phist, ph.data(), x->nd * sizeof(void*), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(x->d_thist, th.data(), x->nd * sizeof(void*), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaMemset(x->counters, 0, XGR_NUM_COUNTERS * 8);
  if (e == cudaSuccess) e = cudaMemset(x->flags, 0, (size_t)x->maxB * 4);
  if (e == cudaSuccess) e = configure_kernels(x->cap);
  if (e == cudaSuccess && (c.flags & XGR_CFG_TIMING)) {
    x->ev.resize(2 * kTimingRing, nullptr);
    x->ev_step.resize(kTimingRing, 0);
    for (auto& ev : x->ev)
      if (e == cudaSuccess) e = cudaEventCreate(&ev);
  }
  if (e != cudaSuccess) {
    ctx_free(x);
    delete x;
    return fail(e == cudaErrorMemoryAllocation ? XGR_ERR_OOM : XGR_ERR_CUDA, "init: %s",
                cudaGetErrorString(e));
  }
  *out = x;
  return XGR_OK;
}

xgr_status xgr_mask_build(xgr_ctx* ctx, const int32_t* items, int64_t n_items, void* stream) {
  NvtxRange nvtx_("xgr_mask_build");
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "mask_build: ctx is NULL");
  if (ctx->built) return fail(XGR_ERR_SEQUENCE, "mask_build: trie already built");
  if (n_items < 0) return fail(XGR_ERR_INVALID_ARG, "mask_build: n_items < 0");
  if (n_items == 0) return fail(XGR_ERR_EMPTY_VOCAB, "mask_build: zero items (no beam could live)");
  if (!items) return fail(XGR_ERR_INVALID_ARG, "mask_build: items is NULL");
  if (n_items >= (int64_t)0xFFFFFFFFll) return fail(XGR_ERR_INVALID_ARG, "mask_build: n_items >= 2^32");
  ACK(cudaSetDevice(ctx->cfg.device));
  std::string err;
  xgr_status st = trie_build(ctx->trie, items, n_items, ctx->V, ctx->nd, (cudaStream_t)stream, err);
  if (st != XGR_OK) {
    trie_free(ctx->trie);
    return fail(st, "%s", err.c_str());
  }
  ctx->built = true;
  return XGR_OK;
}

// Whether step t (1-based) runs both routes: after the root, on the dense route by level statistics,
// the streaming kernels usable, and its trie level holding sparse nodes (skewed tries). Static per
// (trie, step), so the previous step's commit knows whether to count its requests' candidates.
static bool may_mix(const xgr_ctx* ctx, int t) {
  if (t <= 1 || t > ctx->nd || (ctx->cfg.flags & XGR_CFG_NO_SPARSE_KERNEL) || ctx->cfg.nranks > 1) return false;
  const LevelHost& lv = ctx->trie.lv[t - 1];
  const int64_t sk = (int64_t)ctx->BW * lv.max_children;
  return sk > kSparseCap && stream_supported(ctx->V) && lv.n_dense < lv.n_nodes;
}

// Validates a step's inputs and fills the launch arguments (shared by xgr_beam_step and the
// codebook-shard phases). `what` names the caller in error messages.
static xgr_status step_args(xgr_ctx* ctx, int32_t batch, const void* logits, int32_t dtype, int32_t rows,
                            int64_t ld, const char* what, StepArgs& a, int& rows_live, int64_t min_ld = -1) {
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "%s: ctx is NULL", what);
  if (!ctx->built) return fail(XGR_ERR_SEQUENCE, "%s: mask_build has not run", what);
  if (ctx->step >= ctx->nd) return fail(XGR_ERR_SEQUENCE, "%s: already %d steps; call finalize", what, ctx->nd);
  if (!logits) return fail(XGR_ERR_INVALID_ARG, "%s: logits is NULL", what);
  if (batch < 1 || batch > ctx->maxB)
    return fail(XGR_ERR_INVALID_ARG, "%s: batch %d not in 1..%d", what, batch, ctx->maxB);
  if (ctx->step > 0 && batch != ctx->batch)
    return fail(XGR_ERR_INVALID_ARG, "%s: batch %d differs from this batch's %d", what, batch, ctx->batch);
  const int t = ctx->step + 1;
  const int need_rows = (t == 1) ? 1 : ctx->BW;
  if (rows < need_rows) return fail(XGR_ERR_INVALID_ARG, "%s (step %d): rows %d < %d", what, t, rows, need_rows);
  const int Vl = ctx->V / ctx->cfg.nranks;
  if (min_ld < 0) min_ld = Vl;
  if (ld < min_ld) return fail(XGR_ERR_INVALID_ARG, "%s: ld %lld < %lld columns", what, (long long)ld, (long long)min_ld);
  if (dtype != XGR_DTYPE_F32 && dtype != XGR_DTYPE_BF16)
    return fail(XGR_ERR_UNSUPPORTED, "%s: logits dtype %d (XGR_DTYPE_F32 or XGR_DTYPE_BF16)", what, dtype);
  const int per16 = dtype == XGR_DTYPE_BF16 ? 8 : 4;   // elements per 16 bytes
  if ((reinterpret_cast<uintptr_t>(logits) & 15u) || (ld % per16))
    return fail(XGR_ERR_ALIGNMENT, "%s: logits must be 16-byte aligned and ld %% %d == 0", what, per16);

  memset(&a, 0, sizeof(a));
  a.trie = trie_dev(ctx->trie);
  a.logits = logits;
  a.dtype = dtype;
  a.req_stride = (int64_t)rows * ld;
  a.ld = ld;
  a.t = t;
  a.level = t - 1;
  a.BW = ctx->BW;
  a.batch = batch;
  a.cap = ctx->cap;
  a.theta_rows = ctx->R0;
  a.topk = ctx->K;
  a.counters_on = (ctx->cfg.flags & XGR_CFG_COUNTERS) ? 1 : 0;
  a.no_prune = (ctx->cfg.flags & XGR_CFG_NO_PRUNE) ? 1 : 0;
  a.col0 = ctx->cfg.rank * Vl;
  a.Vl = Vl;
  a.nranks = ctx->cfg.nranks;
  const int in = (t - 1) & 1, outi = t & 1;
  if (t > 1) {
    a.score_in = ctx->score[in];
    a.node_in = ctx->node[in];
    a.nlive_in = ctx->nlive[in];
  }
  a.score_out = ctx->score[outi];
  a.node_out = ctx->node[outi];
  a.nlive_out = ctx->nlive[outi];
  const size_t nb = (size_t)ctx->maxB * ctx->BW;
  a.parent_out = ctx->parent_hist + (size_t)(t - 1) * nb;
  a.token_out = ctx->token_hist + (size_t)(t - 1) * nb;
  // the commit counts each request's next-step candidates only when that step can be mixed
  if (t < ctx->nd && may_mix(ctx, t + 1)) a.next_keys_out = ctx->next_keys[t & 1];
  a.ph_lists = ctx->ph_lists;
  a.ph_cnt = ctx->ph_cnt;
  if (t > 1) a.next_keys_in = ctx->next_keys[(t - 1) & 1];
  a.theta = ctx->scratch;
  a.surv_count = ctx->scratch + ctx->maxB;
  a.ovf = ctx->scratch + 2 * ctx->maxB;
  a.seed_hist = ctx->seed_hist;
  a.seed_cnt = ctx->seed_cnt;
  a.surv = ctx->surv;
  a.lse = ctx->lse;
  a.flags = ctx->flags;
  a.counters = ctx->counters;
  a.nd = ctx->nd;
  a.phist = ctx->d_phist;
  a.thist = ctx->d_thist;
  if (t == ctx->nd) {   // the last step's commit also writes the final items (fused finalize)
    a.fin_tokens = ctx->out_tokens;
    a.fin_rank = ctx->out_rank;
    a.fin_score = ctx->out_score;
    a.fin_nlive = ctx->out_nlive;
  }
  static const int dbg_flags = getenv("XGR_DEBUG_FLAGS") ? atoi(getenv("XGR_DEBUG_FLAGS")) : 0;
  a.dbg = dbg_flags;
  rows_live = need_rows;   // upper bound on the live rows of any request this step
  return XGR_OK;
}

xgr_status xgr_beam_step(xgr_ctx* ctx, int32_t batch, const float* logits, int32_t rows, int64_t ld,
                         void* stream) {
  return xgr_beam_step_ex(ctx, batch, logits, XGR_DTYPE_F32, rows, ld, stream);
}

xgr_status xgr_beam_step_ex(xgr_ctx* ctx, int32_t batch, const void* logits, int32_t dtype, int32_t rows,
                            int64_t ld, void* stream) {
  NvtxRange nvtx_("xgr_beam_step_ex");
  StepArgs a;
  int rows_live = 0;
  xgr_status st = step_args(ctx, batch, logits, dtype, rows, ld, "step", a, rows_live);
  if (st != XGR_OK) return st;
  if (ctx->cfg.nranks > 1)
    return fail(XGR_ERR_SEQUENCE, "step: codebook-sharded ctx: use xgr_shard_stats/select/merge");
  cudaStream_t s = (cudaStream_t)stream;
  const int t = a.t;
  const int64_t maxc = ctx->trie.lv[t - 1].max_children;
  const int64_t sparse_keys = (int64_t)rows_live * maxc;
  const bool sparse_route =
      !(ctx->cfg.flags & XGR_CFG_NO_SPARSE_KERNEL) && sparse_keys <= kSparseCap;
  if (!sparse_route && !stream_supported(ctx->V) && ctx->V > 16384)
    return fail(XGR_ERR_UNSUPPORTED, "step: dense route for V > 16384 needs V %% (128 C) == 0 (C = V / 8192 "
                "rounded up to a power of two) or the codebook shard");
  // skewed tries: a level that mixes dense and sparse nodes. The dense path hands its sparse-parent
  // rows to a thread-per-row kernel, and (unless the sparse kernel is disabled) each request takes
  // the sparse route when its own candidates fit on chip (decided by the previous step's commit).
  const LevelHost& lv = ctx->trie.lv[t - 1];
  const bool has_sparse_nodes = lv.n_dense < lv.n_nodes;
  const bool streamed = stream_supported(ctx->V);
  if (!sparse_route && streamed && has_sparse_nodes && !ctx->ph_lists) {
    a.defer_sparse = 1;
    a.mixed = may_mix(ctx, t) ? 1 : 0;
    if (a.mixed) a.dense_list = ctx->dense_list;
  }
  if (!sparse_route && dtype == XGR_DTYPE_BF16 && !stream_supported(ctx->V))
    return fail(XGR_ERR_UNSUPPORTED, "step: bf16 logits on a dense step need the streaming kernels (V %% 128 == 0)");
  if (t == 1) ACK(cudaMemsetAsync(ctx->flags, 0, (size_t)batch * 4, s));
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (!ctx->ev.empty() && !sparse_route && ctx->ev_head - ctx->ev_tail < kTimingRing) {
    const int slot = (int)(ctx->ev_head % kTimingRing);
    ev0 = ctx->ev[2 * slot];
    ev1 = ctx->ev[2 * slot + 1];
    ctx->ev_step[slot] = t;
    ++ctx->ev_head;
  }
  int launches = 0;
  a.sparse_cap = (int)sparse_keys;
  ACK(launch_step(a, rows_live, sparse_route, (int)sparse_keys, s, ev0, ev1, &launches));
  ctx->launches += launches;
  ctx->batch = batch;
  ctx->step = t;
  ctx->last = a;
  ctx->last_rows = rows_live;
  return XGR_OK;
}

xgr_status xgr_beam_step_host(xgr_ctx* ctx, int32_t batch, const void* host_logits, int32_t dtype, int32_t rows,
                              int64_t ld, void* stream) {
  NvtxRange nvtx_("xgr_beam_step_host");
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "step_host: ctx is NULL");
  if (!host_logits) return fail(XGR_ERR_INVALID_ARG, "step_host: logits is NULL");
  if (dtype != XGR_DTYPE_F32 && dtype != XGR_DTYPE_BF16)
    return fail(XGR_ERR_UNSUPPORTED, "step_host: dtype %d", dtype);
  if (batch < 1 || batch > ctx->maxB || rows < 1 || ld < ctx->V)
    return fail(XGR_ERR_INVALID_ARG, "step_host: batch %d, rows %d, ld %lld out of range", batch, rows, (long long)ld);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)batch * rows * ld * (dtype == XGR_DTYPE_BF16 ? 2 : 4);
  if (bytes > ctx->host_stage_bytes) {
    // grow the staging buffer: kernels enqueued earlier may still read the old one
    ACK(cudaStreamSynchronize(s));
    ctx->al.put(ctx->host_stage);
    ctx->host_stage = nullptr;
    ctx->host_stage_bytes = 0;
    ACK(ctx->al.get(&ctx->host_stage, bytes));
    ctx->host_stage_bytes = bytes;
  }
  ACK(cudaMemcpyAsync(ctx->host_stage, host_logits, bytes, cudaMemcpyHostToDevice, s));
  return xgr_beam_step_ex(ctx, batch, ctx->host_stage, dtype, rows, ld, stream);
}

// ---- LM-head fusion at sparse steps (NEXT f4) ------------------------------------------------------

static bool next_is_sparse(const xgr_ctx* ctx, int64_t* keys) {
  const int t = ctx->step + 1;
  const int rows_live = t == 1 ? 1 : ctx->BW;
  const int64_t k = (int64_t)rows_live * ctx->trie.lv[t - 1].max_children;
  if (keys) *keys = k;
  return !(ctx->cfg.flags & XGR_CFG_NO_SPARSE_KERNEL) && k <= kSparseCap;
}

xgr_status xgr_beam_next_route(const xgr_ctx* ctx, int32_t* sparse) {
  if (!ctx || !sparse) return fail(XGR_ERR_INVALID_ARG, "next_route: NULL argument");
  if (!ctx->built) return fail(XGR_ERR_SEQUENCE, "next_route: mask_build has not run");
  if (ctx->step >= ctx->nd) return fail(XGR_ERR_SEQUENCE, "next_route: all %d steps done", ctx->nd);
  *sparse = next_is_sparse(ctx, nullptr) ? 1 : 0;
  return XGR_OK;
}

xgr_status xgr_beam_step_head(xgr_ctx* ctx, int32_t batch, const void* hidden, int32_t rows, int64_t ldh,
                              const void* head, int64_t ldw, const float* bias, int32_t d, void* stream) {
  NvtxRange nvtx_("xgr_beam_step_head");
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "step_head: ctx is NULL");
  if (d < 8 || (d & 7) || ldw < d || (ldw & 7))
    return fail(XGR_ERR_INVALID_ARG, "step_head: d %d (a multiple of 8) and ldw %lld >= d (multiple of 8)", d,
                (long long)ldw);
  if (!head || (reinterpret_cast<uintptr_t>(head) & 15u))
    return fail(XGR_ERR_ALIGNMENT, "step_head: head must be a 16-byte aligned device pointer");
  StepArgs a;
  int rows_live = 0;
  xgr_status st = step_args(ctx, batch, hidden, XGR_DTYPE_BF16, rows, ldh, "step_head", a, rows_live, d);
  if (st != XGR_OK) return st;
  if (ctx->cfg.nranks > 1) return fail(XGR_ERR_UNSUPPORTED, "step_head: codebook-sharded ctx");
  int64_t keys = 0;
  if (a.t == 1 || !next_is_sparse(ctx, &keys))
    return fail(XGR_ERR_UNSUPPORTED, "step_head: step %d is not a sparse step after the root (see xgr_beam_next_route)",
                a.t);
  cudaStream_t s = (cudaStream_t)stream;
  a.clog = ctx->head_logits;
  a.cld = ctx->trie.lv[a.t - 1].max_children;
  a.sparse_cap = (int)keys;
  int launches = 1;
  ACK(xgr::launch_head(a, hidden, ldh, (int64_t)rows * ldh, head, ldw, bias, d, ctx->head_logits, s));
  ACK(xgr::launch_sparse_compact(a, (int)keys, s, &launches));
  ctx->launches += launches;
  ctx->batch = batch;
  ctx->step = a.t;
  ctx->last = a;
  ctx->last_rows = rows_live;
  return XGR_OK;
}

// ---- codebook shard: stats -> (all-gather) -> select -> (all-gather) -> merge -------------------
xgr_status xgr_shard_stats(xgr_ctx* ctx, int32_t batch, const float* logits, int32_t rows, int64_t ld,
                           void* stream, const float** stats) {
  NvtxRange nvtx_("xgr_shard_stats");
  StepArgs a;
  int rows_live = 0;
  xgr_status st = step_args(ctx, batch, logits, XGR_DTYPE_F32, rows, ld, "shard_stats", a, rows_live);
  if (st != XGR_OK) return st;
  if (ctx->shard_phase != 0) return fail(XGR_ERR_SEQUENCE, "shard_stats: previous step not merged");
  if (!stats) return fail(XGR_ERR_INVALID_ARG, "shard_stats: stats is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (a.t == 1) ACK(cudaMemsetAsync(ctx->flags, 0, (size_t)batch * 4, s));
  a.stats_out = ctx->shard_stats;
  // the sparse route when every request's candidates fit on chip (as xgr_beam_step): thread-per-row
  // stats and an on-chip selection instead of the streamed dense passes
  const int64_t sk = (int64_t)rows_live * ctx->trie.lv[a.t - 1].max_children;
  ctx->shard_sparse_keys = (!(ctx->cfg.flags & XGR_CFG_NO_SPARSE_KERNEL) && sk <= kSparseCap) ? (int)sk : 0;
  if (ctx->shard_sparse_keys) ACK(launch_shard_stats_sparse(a, rows_live, s));
  else ACK(launch_shard_stats(a, rows_live, s));
  ctx->launches += 1;
  ctx->batch = batch;
  ctx->shard_args = a;
  ctx->shard_rows = rows_live;
  ctx->shard_phase = 1;
  *stats = reinterpret_cast<const float*>(ctx->shard_stats);
  return XGR_OK;
}

xgr_status xgr_shard_select(xgr_ctx* ctx, const float* gstats, void* stream, const uint64_t** recs,
                            const int32_t** rec_n) {
  NvtxRange nvtx_("xgr_shard_select");
  if (!ctx || !gstats || !recs || !rec_n) return fail(XGR_ERR_INVALID_ARG, "shard_select: NULL argument");
  if (ctx->shard_phase != 1) return fail(XGR_ERR_SEQUENCE, "shard_select: call shard_stats first");
  StepArgs a = ctx->shard_args;
  a.stats_out = nullptr;
  a.gstats = reinterpret_cast<const float2*>(gstats);
  a.rec_out = ctx->shard_rec;
  a.rec_n = ctx->shard_rec_n;
  cudaStream_t s = (cudaStream_t)stream;
  int launches = 0;
  if (ctx->shard_sparse_keys) {
    a.sparse_cap = ctx->shard_sparse_keys;
    ACK(launch_shard_select_sparse(a, ctx->shard_sparse_keys, s));
    launches = 1;
  } else {
    ACK(launch_shard_select(a, ctx->shard_rows, s, &launches));
  }
  ctx->launches += launches;
  ctx->shard_phase = 2;
  *recs = ctx->shard_rec;
  *rec_n = ctx->shard_rec_n;
  return XGR_OK;
}

xgr_status xgr_shard_merge(xgr_ctx* ctx, const uint64_t* grecs, const int32_t* grec_n, void* stream) {
  NvtxRange nvtx_("xgr_shard_merge");
  if (!ctx || !grecs) return fail(XGR_ERR_INVALID_ARG, "shard_merge: NULL argument");
  if (ctx->shard_phase != 2) return fail(XGR_ERR_SEQUENCE, "shard_merge: call shard_select first");
  StepArgs a = ctx->shard_args;
  a.stats_out = nullptr;
  a.gstats = nullptr;
  a.rec_out = nullptr;
  a.rec_n = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  ACK(launch_shard_merge(a, grecs, grec_n, s));
  ctx->launches += 1;
  ctx->step = a.t;
  ctx->last = a;
  ctx->last_rows = ctx->shard_rows;
  ctx->shard_phase = 0;
  return XGR_OK;
}

xgr_status xgr_beam_finalize(xgr_ctx* ctx, int32_t* tokens, int64_t* item_rank, float* score,
                             int32_t* n_live, int32_t outputs_on_device, void* stream) {
  NvtxRange nvtx_("xgr_beam_finalize");
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "finalize: ctx is NULL");
  if (ctx->step != ctx->nd)
    return fail(XGR_ERR_SEQUENCE, "finalize: %d of %d steps done", ctx->step, ctx->nd);
  cudaStream_t s = (cudaStream_t)stream;
  const int fin = ctx->nd & 1;
  const int B = ctx->batch, BW = ctx->BW, nd = ctx->nd;
  const size_t nb = (size_t)B * BW;
  xgr_status st = XGR_OK;
  // the final items were written by the last step's commit into the ctx's output buffers
  if (outputs_on_device) {
    const cudaMemcpyKind k = cudaMemcpyDeviceToDevice;
    if (tokens) ACK(cudaMemcpyAsync(tokens, ctx->out_tokens, nb * nd * 4, k, s));
    if (item_rank) ACK(cudaMemcpyAsync(item_rank, ctx->out_rank, nb * 8, k, s));
    if (score) ACK(cudaMemcpyAsync(score, ctx->out_score, nb * 4, k, s));
    if (n_live) ACK(cudaMemcpyAsync(n_live, ctx->out_nlive, (size_t)B * 4, k, s));
  } else {
    if (tokens) ACK(cudaMemcpyAsync(tokens, ctx->out_tokens, nb * nd * 4, cudaMemcpyDeviceToHost, s));
    if (item_rank) ACK(cudaMemcpyAsync(item_rank, ctx->out_rank, nb * 8, cudaMemcpyDeviceToHost, s));
    if (score) ACK(cudaMemcpyAsync(score, ctx->out_score, nb * 4, cudaMemcpyDeviceToHost, s));
    if (n_live) ACK(cudaMemcpyAsync(n_live, ctx->out_nlive, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
    std::vector<uint32_t> fl(B);
    ACK(cudaMemcpyAsync(fl.data(), ctx->flags, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
    ACK(cudaStreamSynchronize(s));
    for (int r = 0; r < B; ++r)
      if (fl[r] & kFlagNonfinite) {
        st = fail(XGR_ERR_NONFINITE, "finalize: request %d saw a NaN/+Inf logit at a legal position", r);
        break;
      }
  }
  ctx->step = 0;
  return st;
}

xgr_status xgr_beam_destroy(xgr_ctx* ctx) {
  if (!ctx) return XGR_OK;
  cudaSetDevice(ctx->cfg.device);
  ctx_free(ctx);
  delete ctx;
  return XGR_OK;
}

xgr_status xgr_beam_view(const xgr_ctx* ctx, const int32_t** parent, const int32_t** token,
                         const float** score, const int32_t** n_live, const uint32_t** node) {
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "view: ctx is NULL");
  if (ctx->step < 1) return fail(XGR_ERR_SEQUENCE, "view: no step in this batch yet");
  const int t = ctx->step, o = t & 1;
  const size_t nb = (size_t)ctx->maxB * ctx->BW;
  if (parent) *parent = ctx->parent_hist + (size_t)(t - 1) * nb;
  if (token) *token = ctx->token_hist + (size_t)(t - 1) * nb;
  if (score) *score = ctx->score[o];
  if (n_live) *n_live = ctx->nlive[o];
  if (node) *node = ctx->node[o];
  return XGR_OK;
}

xgr_status xgr_beam_history(const xgr_ctx* ctx, int32_t step, const int32_t** parent,
                            const int32_t** token) {
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "history: ctx is NULL");
  if (step < 1 || step > ctx->step) return fail(XGR_ERR_SEQUENCE, "history: step %d not done", step);
  const size_t nb = (size_t)ctx->maxB * ctx->BW;
  if (parent) *parent = ctx->parent_hist + (size_t)(step - 1) * nb;
  if (token) *token = ctx->token_hist + (size_t)(step - 1) * nb;
  return XGR_OK;
}

xgr_status xgr_beam_request_status(const xgr_ctx* ctx, uint32_t* flags, int32_t batch, void* stream) {
  if (!ctx || !flags) return fail(XGR_ERR_INVALID_ARG, "request_status: NULL argument");
  if (batch < 1 || batch > ctx->maxB) return fail(XGR_ERR_INVALID_ARG, "request_status: bad batch");
  cudaStream_t s = (cudaStream_t)stream;
  ACK(cudaMemcpyAsync(flags, ctx->flags, (size_t)batch * 4, cudaMemcpyDeviceToHost, s));
  ACK(cudaStreamSynchronize(s));
  return XGR_OK;
}

xgr_status xgr_mask_children(const xgr_ctx* ctx, const int32_t* prefixes, int32_t depth, int64_t n,
                             int32_t* counts, int32_t* tokens, int64_t cap, void* stream) {
  if (!ctx || !counts || (n > 0 && depth > 0 && !prefixes) || (cap > 0 && !tokens))
    return fail(XGR_ERR_INVALID_ARG, "mask_children: NULL argument");
  if (!ctx->built) return fail(XGR_ERR_SEQUENCE, "mask_children: mask_build has not run");
  if (depth < 0 || depth >= ctx->nd || n < 0 || cap < 0)
    return fail(XGR_ERR_INVALID_ARG, "mask_children: bad depth/n/cap");
  if (n == 0) return XGR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int32_t *dp = nullptr, *dc = nullptr, *dt = nullptr;
  ACK(ctx->al.get(&dp, (size_t)n * depth * 4));
  ACK(ctx->al.get(&dc, (size_t)n * 4));
  ACK(ctx->al.get(&dt, (size_t)n * cap * 4));
  cudaError_t e = cudaSuccess;
  if (depth > 0) e = cudaMemcpyAsync(dp, prefixes, (size_t)n * depth * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_children(trie_dev(ctx->trie), dp, depth, n, dc, dt, cap, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(counts, dc, (size_t)n * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && cap > 0) e = cudaMemcpyAsync(tokens, dt, (size_t)n * cap * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  ctx->al.put(dp);
  ctx->al.put(dc);
  ctx->al.put(dt);
  if (e != cudaSuccess) return fail(XGR_ERR_CUDA, "mask_children: %s", cudaGetErrorString(e));
  return XGR_OK;
}

xgr_status xgr_mask_info(const xgr_ctx* ctx, int64_t* n_items, int64_t* nodes_per_level,
                         int64_t* dense_per_level, int64_t* max_children_per_level, int64_t* trie_bytes) {
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "mask_info: ctx is NULL");
  if (!ctx->built) return fail(XGR_ERR_SEQUENCE, "mask_info: mask_build has not run");
  if (n_items) *n_items = ctx->trie.n_items;
  for (int d = 0; d <= ctx->nd; ++d) {
    if (nodes_per_level) nodes_per_level[d] = ctx->trie.lv[d].n_nodes;
    if (dense_per_level) dense_per_level[d] = ctx->trie.lv[d].n_dense;
    if (max_children_per_level) max_children_per_level[d] = ctx->trie.lv[d].max_children;
  }
  if (trie_bytes) *trie_bytes = ctx->trie.bytes;
  return XGR_OK;
}

xgr_status xgr_beam_counters(xgr_ctx* ctx, uint64_t* out, void* stream) {
  if (!ctx || !out) return fail(XGR_ERR_INVALID_ARG, "counters: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  ACK(cudaMemcpyAsync(out, ctx->counters, XGR_NUM_COUNTERS * 8, cudaMemcpyDeviceToHost, s));
  ACK(cudaMemsetAsync(ctx->counters, 0, XGR_NUM_COUNTERS * 8, s));
  ACK(cudaStreamSynchronize(s));
  return XGR_OK;
}

xgr_status xgr_beam_account(xgr_ctx* ctx, int64_t* alg_bytes, int64_t* full_bytes,
                            int64_t* legal_candidates, void* stream) {
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "account: ctx is NULL");
  if (ctx->step < 1) return fail(XGR_ERR_SEQUENCE, "account: no step in this batch yet");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nd_dense = std::max<int64_t>(ctx->trie.lv[ctx->last.level].n_dense, 1);
  uint32_t* touched = nullptr;
  unsigned long long* dout = nullptr;
  ACK(ctx->al.get(&touched, ((nd_dense + 31) / 32) * 4));
  ACK(ctx->al.get(&dout, 3 * 8));
  unsigned long long h[3] = {0, 0, 0};
  cudaError_t e = cudaMemsetAsync(touched, 0, ((nd_dense + 31) / 32) * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(dout, 0, 3 * 8, s);
  if (e == cudaSuccess) e = launch_account(ctx->last, ctx->last_rows, touched, dout, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, dout, 3 * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  ctx->al.put(touched);
  ctx->al.put(dout);
  if (e != cudaSuccess) return fail(XGR_ERR_CUDA, "account: %s", cudaGetErrorString(e));
  if (alg_bytes) *alg_bytes = (int64_t)h[0];
  if (full_bytes) *full_bytes = (int64_t)h[1];
  if (legal_candidates) *legal_candidates = (int64_t)h[2];
  return XGR_OK;
}

int64_t xgr_beam_launch_count(const xgr_ctx* ctx) { return ctx ? ctx->launches : -1; }

xgr_status xgr_beam_outputs(const xgr_ctx* ctx, const int32_t** tokens, const int64_t** item_rank,
                            const float** score, const int32_t** n_live) {
  if (!ctx) return fail(XGR_ERR_INVALID_ARG, "outputs: ctx is NULL");
  if (tokens) *tokens = ctx->out_tokens;
  if (item_rank) *item_rank = ctx->out_rank;
  if (score) *score = ctx->out_score;
  if (n_live) *n_live = ctx->out_nlive;
  return XGR_OK;
}

xgr_status xgr_beam_kernel_times(xgr_ctx* ctx, float* ms, int32_t* step, int32_t cap, int32_t* n) {
  if (!ctx || !n || (cap > 0 && !ms)) return fail(XGR_ERR_INVALID_ARG, "kernel_times: NULL argument");
  if (ctx->ev.empty()) return fail(XGR_ERR_SEQUENCE, "kernel_times: XGR_CFG_TIMING not set");
  int32_t k = 0;
  while (ctx->ev_tail < ctx->ev_head) {
    const int slot = (int)(ctx->ev_tail % kTimingRing);
    ACK(cudaEventSynchronize(ctx->ev[2 * slot + 1]));
    float t = 0.f;
    ACK(cudaEventElapsedTime(&t, ctx->ev[2 * slot], ctx->ev[2 * slot + 1]));
    if (k < cap) {
      ms[k] = t;
      if (step) step[k] = ctx->ev_step[slot];
    }
    ++k;
    ++ctx->ev_tail;
  }
  *n = std::min(k, cap);
  return XGR_OK;
}

}  // extern "C"

// ---- KV-cache reorder (NEXT f2) -------------------------------------------------------------------
namespace xgr {
cudaError_t launch_kv_reorder(void* cache, int n_req, int n_panel, int bw, int64_t row_bytes,
                              int64_t beam_stride, int64_t panel_stride, int64_t req_stride,
                              const int32_t* src, int src_ld, cudaStream_t s);
}

extern "C" xgr_status xgr_kv_reorder(void* cache, int32_t n_req, int32_t n_panel, int32_t bw, int64_t row_bytes,
                                     int64_t beam_stride, int64_t panel_stride, int64_t req_stride,
                                     const int32_t* src, int32_t src_ld, void* stream) {
  if (n_req < 0 || n_panel < 0 || bw < 1 || bw > kMaxBW || row_bytes < 0 || src_ld < bw)
    return fail(XGR_ERR_INVALID_ARG, "kv_reorder: n_req %d n_panel %d bw %d row_bytes %lld src_ld %d", n_req,
                n_panel, bw, (long long)row_bytes, src_ld);
  if (n_req == 0 || n_panel == 0 || row_bytes == 0) return XGR_OK;
  if (!cache || !src) return fail(XGR_ERR_INVALID_ARG, "kv_reorder: NULL cache or src");
  if (n_req > 65535 || n_panel > 65535) return fail(XGR_ERR_INVALID_ARG, "kv_reorder: n_req, n_panel <= 65535");
  if ((reinterpret_cast<uintptr_t>(cache) & 15u) || (row_bytes & 15) || (beam_stride & 15) ||
      (panel_stride & 15) || (req_stride & 15))
    return fail(XGR_ERR_ALIGNMENT, "kv_reorder: cache, row_bytes and strides must be 16-byte multiples");
  if (beam_stride < row_bytes) return fail(XGR_ERR_INVALID_ARG, "kv_reorder: beam_stride < row_bytes");
  ACK(xgr::launch_kv_reorder(cache, n_req, n_panel, bw, row_bytes, beam_stride, panel_stride, req_stride, src,
                             src_ld, (cudaStream_t)stream));
  return XGR_OK;
}

// ---- staged shared/unshared attention (NEXT f4, second workload) ----------------------------------
namespace xgr {
int launch_attn_shared(const void* q, const void* ks, const void* vs, int ls, const void* ku, const void* vu,
                       int64_t u_req_stride, int64_t u_beam_stride, int n_unshared, void* out, float* lse,
                       float* pm, float* ps, float* po, int n_req, int bw, int hq, int hkv, float scale,
                       cudaStream_t stream);
cudaError_t launch_attn_unshared(const void* q, const void* ku, const void* vu, int64_t u_req_stride,
                                 int64_t u_beam_stride, int n, int n_req, int bw, int hq, int hkv, float scale,
                                 float* pm, float* ps, float* po, cudaStream_t stream);
cudaError_t launch_attn_merge(const float* m1, const float* s1, const float* o1, const float* m2, const float* s2,
                              const float* o2, int64_t rows, float* out, float* lse, cudaStream_t stream);
}

static bool misaligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

static xgr_status attn_check(const char* fn, const void* q, int32_t n_req, int32_t bw, int32_t hq, int32_t hkv,
                             int32_t d, float scale) {
  if (n_req < 0 || bw < 1 || bw > 65535 || n_req > 65535 || hq < 1 || hkv < 1 || hkv > 65535 || hq % hkv != 0 ||
      !(scale > 0.f) || !std::isfinite(scale))
    return fail(XGR_ERR_INVALID_ARG, "%s: n_req %d bw %d hq %d hkv %d scale %g", fn, n_req, bw, hq, hkv, (double)scale);
  const int G = hq / hkv;
  if (d != 128 || G > 128 || (G & (G - 1)) != 0)
    return fail(XGR_ERR_UNSUPPORTED, "%s: needs d == 128 and hq / hkv a power of two <= 128 (d %d, G %d)", fn, d, G);
  if (!q) return fail(XGR_ERR_INVALID_ARG, "%s: NULL q", fn);
  if (misaligned(q)) return fail(XGR_ERR_ALIGNMENT, "%s: q not 16-byte aligned", fn);
  return XGR_OK;
}

static xgr_status attn_check_unshared(const char* fn, const void* ku, const void* vu, int64_t rs, int64_t bs,
                                      int32_t n) {
  if (n < 0 || n > 8) return fail(XGR_ERR_INVALID_ARG, "%s: n_unshared %d not in [0, 8]", fn, n);
  if (n == 0) return XGR_OK;
  if (!ku || !vu || rs < 0 || bs < 0) return fail(XGR_ERR_INVALID_ARG, "%s: NULL unshared cache or negative stride", fn);
  if (misaligned(ku) || misaligned(vu) || (rs & 7) || (bs & 7))
    return fail(XGR_ERR_ALIGNMENT, "%s: unshared cache not 16-byte aligned or strides not multiples of 8", fn);
  return XGR_OK;
}

extern "C" xgr_status xgr_attn_staged(const void* q, const void* k_shared, const void* v_shared, int32_t ls,
                                      const void* k_unshared, const void* v_unshared, int64_t u_req_stride,
                                      int64_t u_beam_stride, int32_t n_unshared, void* out, float* lse,
                                      int32_t n_req, int32_t bw, int32_t hq, int32_t hkv, int32_t d, float scale,
                                      void* stream) {
  xgr_status st = attn_check("attn_staged", q, n_req, bw, hq, hkv, d, scale);
  if (st != XGR_OK) return st;
  st = attn_check_unshared("attn_staged", k_unshared, v_unshared, u_req_stride, u_beam_stride, n_unshared);
  if (st != XGR_OK) return st;
  if (ls < 0 || ls + n_unshared < 1)
    return fail(XGR_ERR_INVALID_ARG, "attn_staged: ls %d, n_unshared %d (both stages empty is undefined)", ls, n_unshared);
  if (!out) return fail(XGR_ERR_INVALID_ARG, "attn_staged: NULL out");
  if (ls > 0 && (!k_shared || !v_shared)) return fail(XGR_ERR_INVALID_ARG, "attn_staged: NULL shared cache");
  if (misaligned(out) || misaligned(k_shared) || misaligned(v_shared) || misaligned(lse))
    return fail(XGR_ERR_ALIGNMENT, "attn_staged: pointers must be 16-byte aligned");
  if (n_req == 0) return XGR_OK;
  const void* ks = ls > 0 ? k_shared : q;   // ls == 0: maps need a valid base; no tile is loaded
  const void* vs = ls > 0 ? v_shared : q;
  const int r = xgr::launch_attn_shared(q, ks, vs, ls, k_unshared, v_unshared, u_req_stride, u_beam_stride,
                                        n_unshared, out, lse, nullptr, nullptr, nullptr, n_req, bw, hq, hkv, scale,
                                        (cudaStream_t)stream);
  if (r == 1) return fail(XGR_ERR_CUDA, "attn_staged: cuTensorMapEncodeTiled failed");
  if (r != 0) return fail(XGR_ERR_CUDA, "attn_staged: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return XGR_OK;
}

extern "C" xgr_status xgr_attn_shared(const void* q, const void* k_shared, const void* v_shared, int32_t ls,
                                      float* m, float* s, float* o, int32_t n_req, int32_t bw, int32_t hq,
                                      int32_t hkv, int32_t d, float scale, void* stream) {
  xgr_status st = attn_check("attn_shared", q, n_req, bw, hq, hkv, d, scale);
  if (st != XGR_OK) return st;
  if (ls < 0 || !m || !s || !o) return fail(XGR_ERR_INVALID_ARG, "attn_shared: ls %d or NULL output", ls);
  if (ls > 0 && (!k_shared || !v_shared)) return fail(XGR_ERR_INVALID_ARG, "attn_shared: NULL shared cache");
  if (misaligned(k_shared) || misaligned(v_shared) || misaligned(o))
    return fail(XGR_ERR_ALIGNMENT, "attn_shared: pointers must be 16-byte aligned");
  if (n_req == 0) return XGR_OK;
  const void* ks = ls > 0 ? k_shared : q;
  const void* vs = ls > 0 ? v_shared : q;
  const int r = xgr::launch_attn_shared(q, ks, vs, ls, nullptr, nullptr, 0, 0, 0, nullptr, nullptr, m, s, o, n_req,
                                        bw, hq, hkv, scale, (cudaStream_t)stream);
  if (r == 1) return fail(XGR_ERR_CUDA, "attn_shared: cuTensorMapEncodeTiled failed");
  if (r != 0) return fail(XGR_ERR_CUDA, "attn_shared: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return XGR_OK;
}

extern "C" xgr_status xgr_attn_unshared(const void* q, const void* k_unshared, const void* v_unshared,
                                        int64_t u_req_stride, int64_t u_beam_stride, int32_t n_unshared, float* m,
                                        float* s, float* o, int32_t n_req, int32_t bw, int32_t hq, int32_t hkv,
                                        int32_t d, float scale, void* stream) {
  xgr_status st = attn_check("attn_unshared", q, n_req, bw, hq, hkv, d, scale);
  if (st != XGR_OK) return st;
  st = attn_check_unshared("attn_unshared", k_unshared, v_unshared, u_req_stride, u_beam_stride, n_unshared);
  if (st != XGR_OK) return st;
  if (!m || !s || !o) return fail(XGR_ERR_INVALID_ARG, "attn_unshared: NULL output");
  if (misaligned(o)) return fail(XGR_ERR_ALIGNMENT, "attn_unshared: o must be 16-byte aligned");
  if (n_req == 0) return XGR_OK;
  ACK(xgr::launch_attn_unshared(q, k_unshared, v_unshared, u_req_stride, u_beam_stride, n_unshared, n_req, bw, hq,
                                hkv, scale, m, s, o, (cudaStream_t)stream));
  return XGR_OK;
}

extern "C" xgr_status xgr_attn_merge(const float* m1, const float* s1, const float* o1, const float* m2,
                                     const float* s2, const float* o2, int64_t rows, int32_t d, float* out,
                                     float* lse, void* stream) {
  if (rows < 0 || d != 128) return fail(rows < 0 ? XGR_ERR_INVALID_ARG : XGR_ERR_UNSUPPORTED, "attn_merge: rows %lld d %d", (long long)rows, d);
  if (rows == 0) return XGR_OK;
  if (!m1 || !s1 || !o1 || !m2 || !s2 || !o2 || !out) return fail(XGR_ERR_INVALID_ARG, "attn_merge: NULL pointer");
  if (misaligned(o1) || misaligned(o2) || misaligned(out))
    return fail(XGR_ERR_ALIGNMENT, "attn_merge: o1, o2, out must be 16-byte aligned");
  ACK(xgr::launch_attn_merge(m1, s1, o1, m2, s2, o2, rows, out, lse, (cudaStream_t)stream));
  return XGR_OK;
}
