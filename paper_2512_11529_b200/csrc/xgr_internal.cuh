// Internal device structures and helpers of the xBeam library (not part of the ABI).
// Everything here is product code: it shares nothing with oracle/.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/xgr_beam.h"

namespace xgr {

// ---- programmatic dependent launch (PDL) ----------------------------------------------------
// Step kernels are launched with programmatic stream serialization: a kernel's CTAs may be
// scheduled while its stream predecessor drains. Every such kernel executes pdl_wait() (wait for
// the predecessor grid to complete and its writes to be visible) before touching global memory,
// and pdl_trigger() early so its own successor can be scheduled. Off unless XGR_PDL=1 (see
// pdl_enabled); without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kMaxND = 8;
constexpr int kMaxBW = 1024;
constexpr int kSparseCap = 16384;   // max candidates per request the sparse-step kernel holds
constexpr int kSeedBins = 2048;     // histogram seed: bins of 1/128 over S_0 - c in [0, 16)

// ---- trie, one entry per level d = 0..nd (level d = nodes for prefixes of length d) ----------
struct LevelDev {
  const uint32_t* first_child;  // [n_nodes + 1], children of node n are level-(d+1) nodes
                                //   [first_child[n], first_child[n+1]); null at level nd
  const uint16_t* label;        // [n_nodes] token that leads to each node; null at level 0
  const int32_t* dense_slot;    // [n_nodes] slot in bitmap/rankdir, -1 if sparse; null if the
                                //   level has no dense node
  const uint32_t* bitmap;       // [n_dense][W] V-bit legal-children mask of each dense node
  const uint32_t* rankdir;      // [n_dense][R] popcount of the bitmap before each 256-bit block
  int64_t n_nodes;
  int64_t n_dense;
  int32_t max_children;
  int32_t pad;
};

struct TrieDev {
  int32_t V;   // vocab
  int32_t nd;
  int32_t W;   // bitmap words per dense node = ceil(V / 32)
  int32_t R;   // rank directory entries per dense node = ceil(V / 256)
  LevelDev lv[kMaxND + 1];
};

// ---- one step's arguments (passed as a __grid_constant__ kernel parameter) ------------------
struct StepArgs {
  TrieDev trie;
  const void* logits;   // [batch][rows][ld] of fp32 or bf16 (dtype)
  int32_t dtype;        // XGR_DTYPE_F32 / XGR_DTYPE_BF16
  int64_t req_stride;   // rows * ld (floats)
  int64_t ld;
  int32_t t;            // 1-based step
  int32_t level;        // t - 1: trie level of the parents' nodes
  int32_t BW;
  int32_t batch;
  int32_t cap;          // survivor buffer capacity per request (keys)
  int32_t theta_rows;
  int32_t topk;         // per-beam Top-K (NEXT f3): 0 = none (K >= BW), else each row keeps its best K
  int32_t counters_on;
  int32_t no_prune;
  int32_t sparse_cap;   // key capacity of k_sparse's dynamic shared memory
  int32_t dbg;          // XGR_DEBUG_FLAGS (experiments only; 0 in production)
  // LM-head fusion (NEXT f4): the sparse step reads the legal logits from a compact buffer
  // clog[batch][BW][cld] (child q of row b at (req*BW + b)*cld + q - first_child) instead of logits
  const float* clog;
  int32_t cld;
  // state in (null at t = 1: the root, one live beam with score 0)
  const float* score_in;
  const uint32_t* node_in;
  const int32_t* nlive_in;
  // state out
  float* score_out;
  uint32_t* node_out;
  int32_t* nlive_out;
  int32_t* parent_out;  // history of step t [batch][BW]
  int32_t* token_out;
  // last step only (t == nd): finalize fused into the commit (item tuples, ranks, scores)
  int32_t* fin_tokens;           // [batch][BW][nd]
  int64_t* fin_rank;             // [batch][BW]
  float* fin_score;              // [batch][BW]
  int32_t* fin_nlive;            // [batch]
  const int32_t* const* phist;   // per level: parent history [maxB][BW]
  const int32_t* const* thist;   // per level: token history
  int32_t nd;
  // scratch (per request), reset before each dense step
  uint32_t* theta;      // orderable(theta), 0 = no bound (-inf)
  uint32_t* surv_count;
  uint32_t* ovf;        // this step's overflow marker
  uint32_t* seed_hist;  // [batch][kSeedBins] histogram of S_0 - c over the seed rows (zero between steps)
  uint32_t* seed_cnt;   // [batch] seed CTAs finished this step (XGR_SEED_KERNEL=3; zero between steps)
  uint64_t* surv;       // [batch][cap] survivor keys
  float* lse;           // [batch][BW] per-row lse (NaN: row not read)
  uint32_t* flags;      // sticky per-request status bits
  unsigned long long* counters;
  // per-request routing (skewed tries): the commit of step t writes, per request, the number of
  // legal candidates its beams will have at step t + 1 (sum of the new nodes' child counts);
  // on a "mixed" step (both routes launched) a request with at most kSparseCap of them takes the
  // sparse route (k_sparse) and every dense-route kernel skips it, the others the dense route.
  const uint32_t* next_keys_in;   // written by the previous step's commit [batch]
  uint32_t* next_keys_out;        // this step's commit [batch] (null at the last step)
  int32_t mixed;                  // 1: both routes launched this step
  const int32_t* dense_list;      // mixed step: [0] = number of dense-route requests, then their ids
                                  //   ascending (built on the device by k_route_list)
  int32_t defer_sparse;           // 1: k_stream leaves sparse-parent rows to k_sparse_rows
  // paper-heap baseline (XGR_CFG_PAPER_HEAP): per-beam sorted Top-K lists [batch][BW][K] and counts
  uint64_t* ph_lists;
  int32_t* ph_cnt;
  // codebook shard (nranks > 1): this rank's logits hold columns [col0, col0 + Vl) of V
  int32_t col0;
  int32_t Vl;
  int32_t nranks;
  float2* stats_out;            // stats phase: [batch][BW] local (m, Z) of each live row
  const float2* gstats;         // select phase: [nranks][batch][BW] all ranks' (m, Z)
  uint64_t* rec_out;            // select phase: [batch][BW] local top-BW keys (0-padded)
  int32_t* rec_n;               // select phase: [batch] number of local records
};

// Global lse of row b from all ranks' (m, Z) in ascending rank order (R20):
// M = max_g m_g, Z = sum_g Z_g * 2^((m_g - M) * log2 e), lse = M + max(ln Z, 0).
// R11: lse = M + max(ln Z, 0). ln Z through the MUFU (lg2.approx x ln 2): |error| < 3e-6 for
// Z <= 2^16, well inside the 1e-5 score tolerance (R13), and a tenth of the instructions of
// logf() on the per-row critical path of the streaming kernels. Z <= 1 (a single legal token,
// or every other term underflowed) gives exactly 0, so a lone legal child keeps logp = 0.
__device__ __forceinline__ float row_lse(float M, float Z) {
  return __fadd_rn(M, Z <= 1.0f ? 0.0f : fmaxf(__logf(Z), 0.0f));
}

__device__ __forceinline__ float shard_lse(const StepArgs& a, int req, int b, bool& finite) {
  const size_t stride = (size_t)a.batch * a.BW;
  const size_t o = (size_t)req * a.BW + b;
  float M = -INFINITY;
  for (int g = 0; g < a.nranks; ++g) M = fmaxf(M, a.gstats[g * stride + o].x);
  float Z = 0.f;
  for (int g = 0; g < a.nranks; ++g) {
    const float2 p = a.gstats[g * stride + o];
    if (p.y > 0.f) {
      float e;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmul_rn(__fsub_rn(p.x, M), 1.4426950408889634f)));
      Z = __fadd_rn(Z, __fmul_rn(p.y, e));
    } else if (p.y != p.y) {
      Z = p.y;   // a rank saw a non-finite legal logit
    }
  }
  finite = (Z > 0.5f) && (Z <= 3.0e38f) && (M > -INFINITY);
  return row_lse(M, Z);
}

constexpr uint32_t kFlagNonfinite = 1u;
constexpr uint32_t kFlagOverflow = 2u;

// ---- order-preserving float <-> uint32 (total order on non-NaN floats) ------------------------
__device__ __forceinline__ uint32_t f2o(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(u);
}
__device__ __forceinline__ float theta_value(uint32_t th) {
  return th == 0u ? -INFINITY : o2f(th);
}

// Shared-memory histogram increment, branch-free: `if (p) atomicAdd(&h[i], 1)` inside an unrolled
// loop compiles to a divergent branch per element (BSSY/BSYNC/BRA; ptxas will not predicate a
// shared atomic). Here every lane adds p (0 or 1): a lane with p false adds 0 to bin `lane` (distinct
// addresses across lanes, no same-address serialisation among them).
__device__ __forceinline__ void hist_inc_if(bool p, uint32_t* h, uint32_t i) {
  const uint32_t addr = (uint32_t)__cvta_generic_to_shared(h + (p ? i : (threadIdx.x & 31u)));
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"((uint32_t)p) : "memory");
}

// Logit element loads: fp32 as is; bf16 widened exactly to fp32 (R19 / NEXT f1).
__device__ __forceinline__ float ldx(const float* p) { return *p; }
__device__ __forceinline__ float ldx(const __nv_bfloat16* p) {
  return __uint_as_float((uint32_t)*reinterpret_cast<const uint16_t*>(p) << 16);
}
template <typename TI>
__device__ __forceinline__ void unpack_chunk(const uint4 r, float* v) {
  if constexpr (sizeof(TI) == 4) {
    v[0] = __uint_as_float(r.x);
    v[1] = __uint_as_float(r.y);
    v[2] = __uint_as_float(r.z);
    v[3] = __uint_as_float(r.w);
  } else {   // 8 bf16: the low half of each word is the lower-index token
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[2 * k] = __uint_as_float(w[k] << 16);
      v[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  }
}

// 64-bit candidate key: one unsigned compare = (score desc, flat index asc) (R4).
__device__ __forceinline__ uint64_t make_key(float c, uint32_t flat) {
  return ((uint64_t)f2o(c) << 32) | (uint64_t)(0xFFFFFFFFu - flat);
}
__device__ __forceinline__ float key_score(uint64_t k) { return o2f((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_flat(uint64_t k) {
  return 0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull);
}

// Candidate score, in exactly this association (R11): c = S + (x - lse).
__device__ __forceinline__ float cand_score(float S, float x, float lse) {
  return __fadd_rn(S, __fsub_rn(x, lse));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Debug-build bounds checks (compile with -DXGR_DEBUG): trap with a message on violation.
#ifdef XGR_DEBUG
#define XGR_CHECK(cond, ...)                                        \
  do {                                                              \
    if (!(cond)) {                                                  \
      printf("XGR_CHECK failed %s:%d: %s | ", __FILE__, __LINE__, #cond); \
      printf(__VA_ARGS__);                                          \
      printf("\n");                                                \
      __trap();                                                     \
    }                                                               \
  } while (0)
#else
#define XGR_CHECK(cond, ...) \
  do {                       \
  } while (0)
#endif

// ---- per-request route on a mixed step ------------------------------------------------------------
__device__ __forceinline__ bool req_sparse(const StepArgs& a, int req) {
  return a.mixed && a.next_keys_in[req] <= (uint32_t)kSparseCap;
}

// ---- beam state of row b of request req ----------------------------------------------------------
__device__ __forceinline__ int nlive_of(const StepArgs& a, int req) {
  return a.nlive_in ? a.nlive_in[req] : 1;
}
__device__ __forceinline__ void row_state(const StepArgs& a, int req, int b, float& S, uint32_t& node) {
  if (a.score_in) {
    S = a.score_in[(size_t)req * a.BW + b];
    node = a.node_in[(size_t)req * a.BW + b];
  } else {
    S = 0.0f;
    node = 0u;
  }
}

// ---- child id of (node at level d, token v) -----------------------------------------------------
// Dense node: rank(v) = rankdir[v / 256] + popcount of the bitmap words of that 256-bit block
// below v. Sparse node: binary search of v among the sorted children labels.
__device__ __forceinline__ uint32_t child_of(const TrieDev& tr, int d, uint32_t node, uint32_t v) {
  const LevelDev& L = tr.lv[d];
  uint32_t fc = L.first_child[node];
  int slot = L.dense_slot ? L.dense_slot[node] : -1;
  if (slot >= 0) {
    const uint32_t* bm = L.bitmap + (size_t)slot * tr.W;
    uint32_t r = L.rankdir[(size_t)slot * tr.R + (v >> 8)];
    uint32_t w0 = (v >> 8) << 3, w = v >> 5;
    for (uint32_t i = w0; i < w; ++i) r += __popc(bm[i]);
    r += __popc(bm[w] & ((1u << (v & 31)) - 1u));
    return fc + r;
  }
  uint32_t lo = fc, hi = L.first_child[node + 1];
  const uint16_t* lab = tr.lv[d + 1].label;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (lab[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- survivor emission: one global atomic per warp ------------------------------------------------
// Every lane of the warp must call (n may be 0). Returns this lane's first slot in the request's
// survivor buffer; the warp's total is reserved with a single atomicAdd.
__device__ __forceinline__ uint32_t warp_reserve(uint32_t n, uint32_t* count) {
  const int lane = threadIdx.x & 31;
  uint32_t incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t base = 0;
  if (lane == 31 && total) base = atomicAdd(count, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - n;
}

// ---- child id with the parent's (first_child, next first_child, dense slot) already at hand -----
// Dense: rank directory entry + popcount of the node's 256-bit bitmap block below v, the block
// fetched with two 16-byte loads. Sparse: binary search of v among the sorted child labels.
__device__ __forceinline__ uint32_t child_of_pref(const TrieDev& tr, int d, uint32_t fc, uint32_t fcn,
                                                  int slot, uint32_t v) {
  const LevelDev& L = tr.lv[d];
  if (slot >= 0) {
    const uint32_t* blk = L.bitmap + (size_t)slot * tr.W + ((v >> 8) << 3);
    uint32_t r = __ldg(L.rankdir + (size_t)slot * tr.R + (v >> 8));
    uint32_t w[8];
    const int nw = (int)min((uint32_t)8, (uint32_t)tr.W - ((v >> 8) << 3));
    if (nw == 8 && ((reinterpret_cast<uintptr_t>(blk) & 15u) == 0)) {
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(blk));
      const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(blk) + 1);
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
      w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = i < nw ? __ldg(blk + i) : 0u;
    }
    const uint32_t wi = (v >> 5) & 7u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t m = (uint32_t)i < wi ? 0xFFFFFFFFu : ((uint32_t)i == wi ? ((1u << (v & 31)) - 1u) : 0u);
      r += __popc(w[i] & m);
    }
    return fc + r;
  }
  uint32_t lo = fc, hi = fcn;
  const uint16_t* lab = tr.lv[d + 1].label;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (lab[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- host-side trie (device pointers) ----------------------------------------------------------
struct LevelHost {
  uint32_t* first_child = nullptr;
  uint16_t* label = nullptr;
  int32_t* dense_slot = nullptr;
  uint32_t* bitmap = nullptr;
  uint32_t* rankdir = nullptr;
  int64_t n_nodes = 0;
  int64_t n_dense = 0;
  int32_t max_children = 0;
};

// Device memory of a ctx: the caller's xgr_config.dev_alloc / dev_free hooks, else cudaMalloc /
// cudaFree. Used only outside the step calls (init, mask build, host staging growth, destroy).
struct DevAlloc {
  void* (*alloc)(size_t, void*) = nullptr;
  void (*release)(void*, void*) = nullptr;
  void* user = nullptr;
  template <typename T>
  cudaError_t get(T** p, size_t bytes) const {
    bytes = bytes < 16 ? 16 : bytes;
    if (!alloc) return cudaMalloc(reinterpret_cast<void**>(p), bytes);
    void* q = alloc(bytes, user);
    *p = static_cast<T*>(q);
    if (!q) return cudaErrorMemoryAllocation;
    // every buffer is 16-byte aligned (TMA sources, vector loads); the hook must honour that
    return (reinterpret_cast<uintptr_t>(q) & 15u) ? cudaErrorMisalignedAddress : cudaSuccess;
  }
  void put(void* p) const {
    if (!p) return;
    if (release) release(p, user);
    else cudaFree(p);
  }
};

struct TrieHost {
  DevAlloc al;   // set by the ctx before the build; frees with the same hooks
  int V = 0, nd = 0, w = 0, W = 0, R = 0;
  int64_t n_items = 0;
  LevelHost lv[kMaxND + 1];
  int64_t bytes = 0;
};

void trie_free(TrieHost& t);
TrieDev trie_dev(const TrieHost& t);
xgr_status trie_build(TrieHost& out, const int32_t* h_items, int64_t n, int V, int nd,
                      cudaStream_t s, std::string& err);

}  // namespace xgr
