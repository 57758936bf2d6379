// xgr_beam_step kernels for sm_100a.
//
// Per decode step the path is (section 6):
//   mask fetch (a1) -> masked log-softmax over the legal tokens (a2, L361) -> score add and
//   threshold pruning (a3, L376-385) -> survivor compaction + global top-BW (a4, L156, L385) ->
//   commit + trie advance into fixed ping-pong state (a5, L392).
//
// Two routes, chosen per step on the host from trie level statistics (no device sync):
//  * sparse route (k_sparse): when every request's total legal candidates fit on chip
//    (rows x max_children <= kSparseCap), one CTA per request gathers the legal logits by label,
//    forms every candidate key in shared memory and selects exactly. No pruning needed.
//  * dense route: k_theta (a valid lower bound theta on the BW-th best candidate from rows
//    0..R0-1 of each request) -> k_main (one CTA per row streams the row once with 128-bit loads,
//    masks with the node's bitmap, computes m, Z, lse with warp-shuffle reductions, skips the row
//    if S_b < theta or S_b - ln Z_b < theta, else emits keys >= theta with warp-aggregated
//    atomics) -> k_select (per request: radix select + bitonic sort of the survivors, commit) ->
//    k_fallback (exact multi-pass radix select for any request whose survivors overflowed).
// Results never depend on theta (pruning is strict: c < theta is dropped, R16).
#include <cuda_runtime.h>

#include "xgr_internal.cuh"

namespace xgr {

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  // xor butterfly: every lane ends with the bitwise-same value (a+b == b+a in IEEE)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Block reductions: warp butterflies, then every thread folds the per-warp values in a fixed
// order, so every thread gets the bitwise-same deterministic result. `sh` must hold T/32 values
// and must not be reused before the next __syncthreads.
template <int T>
__device__ __forceinline__ float block_max(float v, float* sh) {
  v = warp_max(v);
  if (lane_id() == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = sh[0];
#pragma unroll
  for (int i = 1; i < T / 32; ++i) r = fmaxf(r, sh[i]);
  return r;
}
template <int T>
__device__ __forceinline__ float block_min(float v, float* sh) {
  v = warp_min(v);
  if (lane_id() == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = sh[0];
#pragma unroll
  for (int i = 1; i < T / 32; ++i) r = fminf(r, sh[i]);
  return r;
}
template <int T>
__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  if (lane_id() == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = sh[0];
#pragma unroll
  for (int i = 1; i < T / 32; ++i) r += sh[i];
  return r;
}
template <int T>
__device__ __forceinline__ int block_sum_i(int v, int* sh) {
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane_id() == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  int r = 0;
#pragma unroll
  for (int i = 0; i < T / 32; ++i) r += sh[i];
  return r;
}

__device__ __forceinline__ void count_add(const StepArgs& a, int idx, unsigned long long v) {
  if (a.counters_on && v) atomicAdd(a.counters + idx, v);
}

// ---------------------------------------------------------------------------------------------
// Dense row in registers: T threads x VPT float4. Thread t owns positions 4*(i*T + t) + {0..3}.
// The row's bitmap words are staged in shared memory; illegal positions become -inf.
// ---------------------------------------------------------------------------------------------
template <int T, int VPT>
struct DenseRow {
  float4 x[VPT];
  uint32_t nib[VPT];
  float M;     // row max over legal
  float lse;   // M + ln Z
  float tmax;  // this thread's max over its legal values
  bool finite;
};

template <int T, int VPT>
__device__ __forceinline__ void dense_row_compute(const float* __restrict__ row,
                                                  const uint32_t* __restrict__ bm, int V, int W,
                                                  uint32_t* s_bm, float* s_red, float* s_red2,
                                                  DenseRow<T, VPT>& r) {
  const int tid = threadIdx.x;
  // issue all logit loads first (VPT x 16 B in flight per thread)
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    int q = i * T + tid;
    if (4 * q < V) r.x[i] = ld_stream4(row + 4 * q);
    else r.x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int w = tid; w < W; w += T) s_bm[w] = __ldg(bm + w);
  __syncthreads();
  float tmax = -INFINITY;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    int q = i * T + tid;
    uint32_t nb = (4 * q < V) ? (s_bm[q >> 3] >> ((q & 7) * 4)) & 0xFu : 0u;
    r.nib[i] = nb;
    r.x[i].x = (nb & 1u) ? r.x[i].x : -INFINITY;
    r.x[i].y = (nb & 2u) ? r.x[i].y : -INFINITY;
    r.x[i].z = (nb & 4u) ? r.x[i].z : -INFINITY;
    r.x[i].w = (nb & 8u) ? r.x[i].w : -INFINITY;
    tmax = fmaxf(tmax, fmaxf(fmaxf(r.x[i].x, r.x[i].y), fmaxf(r.x[i].z, r.x[i].w)));
  }
  r.tmax = tmax;
  const float M = block_max<T>(tmax, s_red);
  float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    z0 += ex2(__fmul_rn(__fsub_rn(r.x[i].x, M), kLog2e));
    z1 += ex2(__fmul_rn(__fsub_rn(r.x[i].y, M), kLog2e));
    z2 += ex2(__fmul_rn(__fsub_rn(r.x[i].z, M), kLog2e));
    z3 += ex2(__fmul_rn(__fsub_rn(r.x[i].w, M), kLog2e));
  }
  const float Z = block_sum<T>((z0 + z1) + (z2 + z3), s_red2);
  r.finite = (Z > 0.5f) && (Z <= 3.0e38f);
  r.M = M;
  r.lse = row_lse(M, Z);
}

// ---------------------------------------------------------------------------------------------
// Block radix select helpers over shared-memory keys.
// ---------------------------------------------------------------------------------------------
// Find the digit d (scanning bins from the top) where the running count reaches `krem`.
// hist has 256 bins. Result written to *out_digit, count above it to *out_above.
__device__ __forceinline__ void warp_find_digit_desc(const uint32_t* hist, uint32_t krem,
                                                     uint32_t* out_digit, uint32_t* out_above) {
  int lane = lane_id();
  // lane l owns bins 255-8l .. 248-8l (descending)
  uint32_t c[8];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    c[j] = hist[255 - 8 * lane - j];
    s += c[j];
  }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  uint32_t excl = incl - s;
  // fewer than krem keys in all bins (only possible for a flagged request): sentinel digit 256
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot < krem) {
    if (lane == 0) {
      *out_digit = 256;
      *out_above = tot;
    }
    return;
  }
  bool mine = (excl < krem) && (incl >= krem);
  if (mine) {
    uint32_t acc = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (acc + c[j] >= krem) {
        *out_digit = 255 - 8 * lane - j;
        *out_above = acc;
        break;
      }
      acc += c[j];
    }
  }
}

// One compare-exchange of a sorting network, from the side of the element holding v with partner
// o: keep the larger if keep_max, else the smaller. One 64-bit compare: (o > v) == keep_max selects
// o; on equal keys (only the zero padding) both choices are the same value.
__device__ __forceinline__ uint64_t ce_pick(uint64_t v, uint64_t o, bool keep_max) {
  return ((o > v) == keep_max) ? o : v;
}

__device__ __forceinline__ uint64_t warp_sort_desc_u64(uint64_t v) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool keep_max = ((lane & stride) == 0) == ((lane & size) == 0);
      v = ce_pick(v, o, keep_max);
    }
  }
  return v;
}

// Sorts k distinct keys (k <= 1024) descending from `sel` into `out`: each warp sorts a list of
// 32 in registers (shuffle bitonic) and writes it back in place; a key's final rank is its index
// in its own list plus, for every other list, the number of greater keys (binary search).
template <int T>
__device__ void sort_desc_to(uint64_t* sel, int k, uint64_t* out, int k_out = 1 << 30) {
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const int nl = (k + 31) >> 5;
  for (int w = warp; w < nl; w += T / 32) {
    const int p = 32 * w + lane;
    const uint64_t v = warp_sort_desc_u64(p < k ? sel[p] : 0ull);
    sel[p] = v;   // padding sorts to the tail as 0 (smaller than every real key)
  }
  __syncthreads();
  for (int p = tid; p < 32 * nl; p += T) {
    const uint64_t v = sel[p];
    if (v == 0ull) continue;
    const int own = p >> 5;
    int r = p & 31;
    for (int w = 0; w < nl; ++w) {
      if (w == own) continue;
      const uint64_t* lst = sel + 32 * w;
      // number of keys > v in a descending list of 32: 6 halvings of [0, 32]
      int lo = 0, hi = 32;
#pragma unroll
      for (int it = 0; it < 6; ++it) {
        if (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (lst[mid] > v) lo = mid + 1; else hi = mid;
        }
      }
      r += lo;
    }
    XGR_CHECK(r < k, "sort_desc_to r %d k %d", r, k);
    if (r < k_out) out[r] = v;
  }
  __syncthreads();
}

// Selects the k largest of keys[0..n) (distinct keys) into out[0..k), sorted descending.
// T threads; shared scratch: sel[k], hist[256], misc64[2 * T / 32], misc32[4].
template <int T>
__device__ void block_select_topk(const uint64_t* keys, int n, int k, uint64_t* sel, uint64_t* out,
                                  uint32_t* hist, uint64_t* misc64, uint32_t* misc32) {
  const int tid = threadIdx.x;
  uint64_t thr = 0;
  if (k < n) {
    // common high bits of all keys are skipped (they would all land in one histogram bin)
    uint64_t lo = ~0ull, hi = 0;
    for (int i = tid; i < n; i += T) {
      uint64_t v = keys[i];
      lo = v < lo ? v : lo;
      hi = v > hi ? v : hi;
    }
    lo = warp_min_u64(lo);
    hi = warp_max_u64(hi);
    if (lane_id() == 0) {
      misc64[2 * (tid >> 5)] = lo;
      misc64[2 * (tid >> 5) + 1] = hi;
    }
    __syncthreads();
    uint64_t glo = misc64[0], ghi = misc64[1];
    for (int w = 1; w < T / 32; ++w) {
      glo = misc64[2 * w] < glo ? misc64[2 * w] : glo;
      ghi = misc64[2 * w + 1] > ghi ? misc64[2 * w + 1] : ghi;
    }
    uint64_t diff = glo ^ ghi;  // != 0 since n > k >= 1 distinct keys
    int top = 63 - __clzll(diff);
    int shift = (top / 8) * 8;
    uint64_t mask = (shift + 8 >= 64) ? 0ull : (~0ull << (shift + 8));
    uint64_t prefix = ghi & mask;
    uint32_t krem = (uint32_t)k;
    __syncthreads();
    for (;;) {
      for (int i = tid; i < 256; i += T) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < n; i += T) {
        uint64_t v = keys[i];
        if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
      }
      __syncthreads();
      if (tid < 32) warp_find_digit_desc(hist, krem, &misc32[0], &misc32[1]);
      __syncthreads();
      uint32_t d = misc32[0], above = misc32[1];
      XGR_CHECK(d < 256, "radix digit %u n %d k %d krem %u", d, n, k, krem);
      uint32_t inbin = hist[d];
      krem -= above;
      prefix |= (uint64_t)d << shift;
      mask |= 0xFFull << shift;
      __syncthreads();
      if (inbin == krem || shift == 0) break;
      shift -= 8;
    }
    thr = prefix;  // all keys >= thr are exactly the k largest
  }
  // compact the k winners
  if (tid == 0) misc32[2] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += T) {
    uint64_t v = keys[i];
    if (v >= thr) {
      uint32_t p = atomicAdd(&misc32[2], 1u);
      sel[p] = v;
    }
  }
  __syncthreads();
  sort_desc_to<T>(sel, k, out);
}

// Bitonic sort (descending) of n <= T * EPT distinct nonzero keys; the first k_out go to out.
// Thread t holds elements EPT*t .. EPT*t + EPT - 1 in registers: strides < EPT are exchanged in
// registers, strides < 32 * EPT by warp shuffles, larger ones through xbuf (T * EPT keys; may be
// src itself) with one barrier on each side -- 10 barrier pairs for 2048 keys.
template <int T, int EPT>
__device__ void block_sort_desc(const uint64_t* src, int n, uint64_t* xbuf, uint64_t* out, int k_out) {
  constexpr int N = T * EPT;
  const int tid = threadIdx.x;
  uint64_t v[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int i = EPT * tid + j;
    v[j] = i < n ? src[i] : 0ull;   // padding 0 sorts last
  }
  __syncthreads();
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < EPT) {
#pragma unroll
        for (int s2 = 1; s2 < EPT; s2 <<= 1) {   // compile-time register indices only
#pragma unroll
          for (int j = 0; j < EPT; ++j) {
            if (s2 == stride && (j & s2) == 0) {
              const int jj = j | s2;
              const bool desc = ((EPT * tid + j) & size) == 0;
              const bool keep = (v[j] > v[jj]) == desc;   // v[j] already on its side
              const uint64_t a0 = v[j], a1 = v[jj];
              v[j] = keep ? a0 : a1;
              v[jj] = keep ? a1 : a0;
            }
          }
        }
      } else if (stride < 32 * EPT) {
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          const int i = EPT * tid + j;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[j], stride / EPT);
          const bool keep_max = ((i & stride) == 0) == ((i & size) == 0);
          v[j] = ce_pick(v[j], o, keep_max);
        }
      } else {
#pragma unroll
        for (int j = 0; j < EPT; ++j) xbuf[EPT * tid + j] = v[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          const int i = EPT * tid + j;
          const uint64_t o = xbuf[i ^ stride];
          const bool keep_max = ((i & stride) == 0) == ((i & size) == 0);
          v[j] = ce_pick(v[j], o, keep_max);
        }
        __syncthreads();
      }
    }
  }
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int i = EPT * tid + j;
    if (i < k_out) out[i] = v[j];
  }
  __syncthreads();
}

// Top-k of n <= T keys by a full block sort (cand: >= T keys of exchange space; may be keys).
// One key per thread only: the unrolled network for 2-4 keys per thread was measured slower.
template <int T>
__device__ bool block_sort_topk(const uint64_t* keys, int n, int k, uint64_t* cand, int cand_cap,
                                uint64_t* out) {
  if (n > T || cand_cap < T) return false;
  block_sort_desc<T, 1>(keys, n, cand, out, k);
  return true;
}

// Fast top-k of distinct keys in shared memory (used by the per-request select kernels).
// Threshold without atomics or passes: every thread takes the max of its keys; each warp sorts
// its 32 maxima (shuffle bitonic) and takes the m-th largest, m = ceil(k / warps); the minimum of
// those over warps, tau, has >= k keys >= tau (each warp contributes m distinct thread maxima).
// Keys >= tau (typically ~1.5k) are compacted and rank-sorted. If tau admits too many keys, the
// exact radix path (block_select_topk) is used instead.
struct TopkScratch {
  uint64_t wsel[32];
  uint32_t n_c;
  uint64_t m64[64];
  uint32_t m32[4];
  uint32_t hist[256];
};

template <int T>
__device__ int block_topk_fast(uint64_t* keys, int n, int k, uint64_t* cand, int cand_cap,
                               uint64_t* sel, uint64_t* out, TopkScratch& sc, int a_dbg_sort = 0) {
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  constexpr int NW = T / 32;
  if (k <= 0) return 0;
  const int m = (k + NW - 1) / NW;
  if (!(a_dbg_sort & 1) && block_sort_topk<T>(keys, n, k, cand, cand_cap, out)) return k;
  if (n <= 2 * k || m > 32) {
    block_select_topk<T>(keys, n, k, sel, out, sc.hist, sc.m64, sc.m32);
    return k;
  }
  uint64_t tmax = 0ull;
  for (int i = tid; i < n; i += T) {
    const uint64_t v = keys[i];
    tmax = v > tmax ? v : tmax;
  }
  const uint64_t srt = warp_sort_desc_u64(tmax);
  const uint64_t wm = __shfl_sync(0xffffffffu, srt, m - 1);
  if (lane == 0) sc.wsel[warp] = wm;
  if (tid == 0) sc.n_c = 0;
  __syncthreads();
  uint64_t tau = sc.wsel[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) tau = sc.wsel[w] < tau ? sc.wsel[w] : tau;
  {
    // count, warp scan, one shared atomic per warp, then the stores
    uint32_t cnt = 0;
    for (int i = tid; i < n; i += T) cnt += keys[i] >= tau;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t wb = 0;
    if (lane == 31 && incl) wb = atomicAdd(&sc.n_c, incl);
    uint32_t p = __shfl_sync(0xffffffffu, wb, 31) + incl - cnt;
    if (cnt) {
      for (int i = tid; i < n; i += T) {
        const uint64_t v = keys[i];
        if (v >= tau) {
          if (p < (uint32_t)cand_cap) cand[p] = v;
          ++p;
        }
      }
    }
  }
  __syncthreads();
  const int nc = (int)sc.n_c;
  if (nc <= cand_cap && !(a_dbg_sort & 1) && block_sort_topk<T>(cand, nc, k, cand, cand_cap, out)) return k;
  if (nc > cand_cap) block_select_topk<T>(keys, n, k, sel, out, sc.hist, sc.m64, sc.m32);
  else block_select_topk<T>(cand, nc, k, sel, out, sc.hist, sc.m64, sc.m32);
  return k;
}

// Parent-row trie info for the commit, fetched at kernel start (overlaps the selection work).
// N = 1 for the root step (one parent), which keeps k_sparse<ROOT> at two CTAs per SM.
template <int N>
struct ParentInfoN {
  uint32_t fc[N];
  uint32_t fcn[N];
  int32_t slot[N];
};
using ParentInfo = ParentInfoN<kMaxBW>;

template <int T, typename PI>
__device__ void prefetch_parents(const StepArgs& a, int req, int nl, PI& pi) {
  const LevelDev& L = a.trie.lv[a.level];
  for (int b = threadIdx.x; b < nl; b += T) {
    const uint32_t node = a.node_in ? a.node_in[(size_t)req * a.BW + b] : 0u;
    XGR_CHECK(node < (uint32_t)L.n_nodes, "prefetch req %d b %d nl %d node %u n_nodes %lld", req, b, nl, node,
              (long long)L.n_nodes);
    pi.fc[b] = L.first_child[node];
    pi.fcn[b] = L.first_child[node + 1];
    pi.slot[b] = L.dense_slot ? L.dense_slot[node] : -1;
  }
}

// Commit the k selected keys (sorted desc) of request req into the step-t state (a5).
template <int T, typename PI>
__device__ void commit(const StepArgs& a, int req, const uint64_t* sel, int k, const PI& pi) {
  const int V = a.trie.V;
  const size_t base = (size_t)req * a.BW;
  if (a.rec_out) {   // codebook-shard select phase: this rank's local top-BW keys, no state update
    for (int j = threadIdx.x; j < a.BW; j += T) a.rec_out[base + j] = j < k ? sel[j] : 0ull;
    if (threadIdx.x == 0) a.rec_n[req] = k;
    return;
  }
  for (int j = threadIdx.x; j < a.BW; j += T) {
    if (j < k) {
      uint64_t key = sel[j];
      float c = key_score(key);
      uint32_t flat = key_flat(key);
      uint32_t b = flat / (uint32_t)V;
      uint32_t v = flat - b * (uint32_t)V;
      a.parent_out[base + j] = (int32_t)b;
      a.token_out[base + j] = (int32_t)v;
      a.score_out[base + j] = c;
      XGR_CHECK(b < (uint32_t)a.BW && v < (uint32_t)V, "commit req %d j %d k %d b %u v %u key %llx", req, j, k, b, v,
                (unsigned long long)key);
      const uint32_t child = child_of_pref(a.trie, a.level, pi.fc[b], pi.fcn[b], pi.slot[b], v);
      a.node_out[base + j] = child;
      if (a.fin_tokens) {   // fused finalize (a6): backtrack the histories into the item tuple
        int32_t* tk = a.fin_tokens + (base + j) * a.nd;
        tk[a.nd - 1] = (int32_t)v;
        int sidx = (int)b;
        for (int t = a.nd - 2; t >= 0; --t) {
          tk[t] = a.thist[t][base + sidx];
          sidx = a.phist[t][base + sidx];
        }
        a.fin_rank[base + j] = (int64_t)child;   // leaf id = item rank
        a.fin_score[base + j] = c;
      }
    } else {
      a.parent_out[base + j] = -1;
      a.token_out[base + j] = -1;
      a.score_out[base + j] = -INFINITY;
      a.node_out[base + j] = 0xFFFFFFFFu;
      if (a.fin_tokens) {
        for (int t = 0; t < a.nd; ++t) a.fin_tokens[(base + j) * a.nd + t] = -1;
        a.fin_rank[base + j] = -1;
        a.fin_score[base + j] = -INFINITY;
      }
    }
  }
  if (threadIdx.x == 0) {
    a.nlive_out[req] = k;
    if (a.fin_nlive) a.fin_nlive[req] = k;
  }
  if (a.next_keys_out) {
    // the next step's legal candidates of this request: sum of the new nodes' child counts (the
    // next step's per-request route); children of node c of level l+1 are the level-(l+2) nodes
    // [first_child[c], first_child[c+1])
    __shared__ uint32_t s_nk[32];
    const uint32_t* fcn = a.trie.lv[a.level + 1].first_child;
    uint32_t nk = 0;
    for (int j = threadIdx.x; j < k; j += T) {
      const uint32_t c = a.node_out[base + j];
      nk += __ldg(fcn + c + 1) - __ldg(fcn + c);
    }
    nk = __reduce_add_sync(0xffffffffu, nk);
    if ((threadIdx.x & 31) == 0) s_nk[threadIdx.x >> 5] = nk;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < T / 32; ++w) tot += s_nk[w];
      a.next_keys_out[req] = tot;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// k_theta: per (request, row r < R0) with a dense node and >= BW legal tokens, a lower bound on
// the row's BW-th largest legal logit x_lb (two 12-bit histogram passes on d = M - x, then the
// smallest x in the crossing bin); theta_r = S_r + (x_lb - lse_r) is an actual candidate score
// with >= BW candidates of the request at or above it, so max_r theta_r <= the true BW-th best.
// ---------------------------------------------------------------------------------------------
template <int T, int VPT>
__global__ void __launch_bounds__(T) k_theta(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  __shared__ uint32_t s_bm[T * VPT / 8];
  __shared__ float s_red[T / 32], s_red2[T / 32], s_red3[T / 32];
  __shared__ uint32_t s_hist[4096];
  __shared__ uint32_t s_tot[T / 32];
  __shared__ uint32_t s_sel[2];
  const int req = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  if (b >= nlive_of(a, req)) return;
  float S;
  uint32_t node;
  row_state(a, req, b, S, node);
  const LevelDev& L = a.trie.lv[a.level];
  const int slot = L.dense_slot ? L.dense_slot[node] : -1;
  if (slot < 0) return;
  const uint32_t nchild = L.first_child[node + 1] - L.first_child[node];
  if (nchild < (uint32_t)a.BW) return;
  const float* row = static_cast<const float*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
  DenseRow<T, VPT> r;
  dense_row_compute<T, VPT>(row, L.bitmap + (size_t)slot * a.trie.W, a.trie.V, a.trie.W, s_bm,
                            s_red, s_red2, r);
  if (!r.finite) return;
  // d = M - x >= 0 for legal x; illegal/NaN are excluded by the nibble test and d == d
  uint32_t krem = (uint32_t)a.BW;
  uint32_t pre = 0, pmask = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const int sh = pass == 0 ? 20 : 8;
    for (int i = tid; i < 4096; i += T) s_hist[i] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      float xs[4] = {r.x[i].x, r.x[i].y, r.x[i].z, r.x[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((r.nib[i] >> j) & 1u) {
          float d = __fsub_rn(r.M, xs[j]);
          uint32_t u = __float_as_uint(d);
          if (d == d && (u & pmask) == pre) atomicAdd(&s_hist[(u >> sh) & 0xFFFu], 1u);
        }
      }
    }
    __syncthreads();
    // ascending scan of 4096 bins: thread t owns bins [t*B, t*B + B)
    constexpr int B = 4096 / T;
    uint32_t loc = 0;
#pragma unroll
    for (int j = 0; j < B; ++j) loc += s_hist[tid * B + j];
    uint32_t incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane_id() >= o) incl += y;
    }
    if (lane_id() == 31) s_tot[tid >> 5] = incl;
    __syncthreads();
    uint32_t woff = 0;
    for (int w = 0; w < (tid >> 5); ++w) woff += s_tot[w];
    incl += woff;
    uint32_t excl = incl - loc;
    if (excl < krem && incl >= krem) {
      uint32_t acc = excl;
      for (int j = 0; j < B; ++j) {
        uint32_t c = s_hist[tid * B + j];
        if (acc + c >= krem) {
          s_sel[0] = (uint32_t)(tid * B + j);
          s_sel[1] = acc;
          break;
        }
        acc += c;
      }
    }
    __syncthreads();
    uint32_t bin = s_sel[0];
    krem -= s_sel[1];
    pre |= bin << sh;
    pmask |= 0xFFFu << sh;
    __syncthreads();
  }
  // smallest legal x whose d shares the 24 selected bits: >= BW legal values are >= it
  float xmin = INFINITY;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    float xs[4] = {r.x[i].x, r.x[i].y, r.x[i].z, r.x[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((r.nib[i] >> j) & 1u) {
        float d = __fsub_rn(r.M, xs[j]);
        if (d == d && (__float_as_uint(d) & pmask) == pre) xmin = fminf(xmin, xs[j]);
      }
    }
  }
  const float xlb = block_min<T>(xmin, s_red3);
  if (tid == 0 && xlb < INFINITY) {
    float th = cand_score(S, xlb, r.lse);
    if (th == th && th > -INFINITY) atomicMax(a.theta + req, f2o(th));
  }
}

// ---------------------------------------------------------------------------------------------
// k_main: one CTA per (request, live row). The dominant HBM stream (a1-a3).
// ---------------------------------------------------------------------------------------------
template <int T>
__device__ void sparse_row_main(const StepArgs& a, int req, int b, float S, float th, uint32_t node,
                                const float* row, float* s_red, float* s_red2, int* s_redi) {
  const LevelDev& L = a.trie.lv[a.level];
  const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  const int tid = threadIdx.x;
  float tmax = -INFINITY;
  for (uint32_t k = fc + tid; k < fe; k += T) tmax = fmaxf(tmax, row[lab[k]]);
  const float M = block_max<T>(tmax, s_red);
  float z = 0.f;
  for (uint32_t k = fc + tid; k < fe; k += T) z += ex2(__fmul_rn(__fsub_rn(row[lab[k]], M), kLog2e));
  const float Z = block_sum<T>(z, s_red2);
  const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
  const float lse = row_lse(M, Z);
  if (tid == 0) {
    a.lse[(size_t)req * a.BW + b] = finite ? lse : __int_as_float(0x7fc00000);
    if (!finite) atomicOr(a.flags + req, kFlagNonfinite);
  }
  if (a.counters_on && tid == 0) count_add(a, XGR_CNT_LEGAL, fe - fc);
  if (!finite) return;
  if (!(cand_score(S, M, lse) >= th)) {
    if (tid == 0) count_add(a, XGR_CNT_ROWS_SKIP_POST, 1);
    return;
  }
  int ns = 0;
  const uint32_t fbase = (uint32_t)b * (uint32_t)a.trie.V;
  for (uint32_t k0 = fc; k0 < fe; k0 += T) {
    const uint32_t k = k0 + tid;
    uint32_t v = 0;
    float c = -INFINITY;
    if (k < fe) {
      v = lab[k];
      c = cand_score(S, row[v], lse);
    }
    const bool take = k < fe && c >= th;
    if (__any_sync(0xffffffffu, take)) {
      const uint32_t pos = warp_reserve(take ? 1u : 0u, a.surv_count + req);
      if (take && pos < (uint32_t)a.cap) a.surv[(size_t)req * a.cap + pos] = make_key(c, fbase + v);
    }
    ns += take;
  }
  if (a.counters_on) {
    int tot = block_sum_i<T>(ns, s_redi);
    if (tid == 0) count_add(a, XGR_CNT_SURVIVORS, tot);
  }
}

template <int T, int VPT>
__global__ void __launch_bounds__(T) k_main(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  __shared__ uint32_t s_bm[T * VPT / 8];
  __shared__ float s_red[T / 32], s_red2[T / 32];
  __shared__ int s_redi[T / 32];
  const int req = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  if (b >= nlive_of(a, req)) return;
  float S;
  uint32_t node;
  row_state(a, req, b, S, node);
  const float th = theta_value(a.theta[req]);
  if (S < th) {  // every candidate of the row is <= S_b < theta (pre-read skip)
    if (tid == 0) {
      a.lse[(size_t)req * a.BW + b] = __int_as_float(0x7fc00000);
      count_add(a, XGR_CNT_ROWS_SKIP_PRE, 1);
    }
    return;
  }
  if (tid == 0) count_add(a, XGR_CNT_ROWS_READ, 1);
  const float* row = static_cast<const float*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
  const LevelDev& L = a.trie.lv[a.level];
  const int slot = L.dense_slot ? L.dense_slot[node] : -1;
  if (slot < 0) {
    sparse_row_main<T>(a, req, b, S, th, node, row, s_red, s_red2, s_redi);
    return;
  }
  DenseRow<T, VPT> r;
  dense_row_compute<T, VPT>(row, L.bitmap + (size_t)slot * a.trie.W, a.trie.V, a.trie.W, s_bm, s_red,
                            s_red2, r);
  if (tid == 0) {
    a.lse[(size_t)req * a.BW + b] = r.finite ? r.lse : __int_as_float(0x7fc00000);
    if (!r.finite) atomicOr(a.flags + req, kFlagNonfinite);
  }
  if (a.counters_on) {
    int lc = 0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) lc += __popc(r.nib[i]);
    int tot = block_sum_i<T>(lc, s_redi);
    if (tid == 0) count_add(a, XGR_CNT_LEGAL, tot);
    __syncthreads();
  }
  if (!r.finite) return;
  const float lse = r.lse;
  if (!(cand_score(S, r.M, lse) >= th)) {  // UB_b = S_b - ln Z_b < theta (post-LSE skip)
    if (tid == 0) count_add(a, XGR_CNT_ROWS_SKIP_POST, 1);
    return;
  }
  // conservative pre-filter on x (exact test below): c(x) >= theta implies x >= xthr
  const float xthr = (th == -INFINITY)
                         ? -INFINITY
                         : (th - S) + lse - 1e-5f * (fabsf(th) + fabsf(S) + 2.0f * fabsf(lse));
  uint32_t mine = 0u;   // bit 4i+j: element j of x[i] is a candidate (VPT <= 8)
  if (r.tmax >= xthr) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const float xs[4] = {r.x[i].x, r.x[i].y, r.x[i].z, r.x[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (((r.nib[i] >> j) & 1u) && xs[j] >= xthr && cand_score(S, xs[j], lse) >= th)
          mine |= 1u << (4 * i + j);
    }
  }
  const int ns = __popc(mine);
  if (__any_sync(0xffffffffu, ns > 0)) {
    const uint32_t fbase = (uint32_t)b * (uint32_t)a.trie.V;
    uint64_t* sbuf = a.surv + (size_t)req * a.cap;
    uint32_t pos = warp_reserve((uint32_t)ns, a.surv_count + req);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const float xs[4] = {r.x[i].x, r.x[i].y, r.x[i].z, r.x[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((mine >> (4 * i + j)) & 1u) {
          const uint32_t v = 4u * (uint32_t)(i * T + tid) + j;
          if (pos < (uint32_t)a.cap) sbuf[pos] = make_key(cand_score(S, xs[j], lse), fbase + v);
          ++pos;
        }
      }
    }
  }
  if (a.counters_on) {
    int tot = block_sum_i<T>(ns, s_redi);
    if (tid == 0) count_add(a, XGR_CNT_SURVIVORS, tot);
  }
}

// ---------------------------------------------------------------------------------------------
// k_fallback: exact top-BW for a request whose survivors overflowed the buffer. One CTA streams
// the request's rows once per 8-bit radix digit of the 64-bit key (at most 8 passes), restricted
// to keys >= theta. Keys are recomputed with the same formula and the lse stored by k_main, so
// they are bitwise the keys k_main would have emitted. Rare path (adversarial ties/logits).
// ---------------------------------------------------------------------------------------------
template <int T, typename TI, typename F>
__device__ __forceinline__ void for_each_candidate(const StepArgs& a, int req, int b, float S,
                                                   float lse, uint32_t node, F&& f) {
  // this rank's columns [col0, col0 + Vl) (the whole row unless codebook-sharded)
  const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
  const LevelDev& L = a.trie.lv[a.level];
  const int slot = L.dense_slot ? L.dense_slot[node] : -1;
  const uint32_t fbase = (uint32_t)b * (uint32_t)a.trie.V;
  if (slot >= 0) {
    const uint32_t* bm = L.bitmap + (size_t)slot * a.trie.W + (a.col0 >> 5);
    const int Vl = a.Vl;
    for (int q = threadIdx.x; 4 * q < Vl; q += T) {
      uint32_t nb = (bm[q >> 3] >> ((q & 7) * 4)) & 0xFu;
      if (!nb) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if ((nb >> j) & 1u)
          f(make_key(cand_score(S, ldx(row + 4 * q + j), lse), fbase + (uint32_t)a.col0 + 4u * q + j));
    }
  } else {
    const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
    const uint16_t* lab = a.trie.lv[a.level + 1].label;
    for (uint32_t k = fc + threadIdx.x; k < fe; k += T) {
      uint32_t v = lab[k];
      if (v < (uint32_t)a.col0 || v >= (uint32_t)(a.col0 + a.Vl)) continue;
      f(make_key(cand_score(S, ldx(row + (v - a.col0)), lse), fbase + v));
    }
  }
}

// Exact top-k (k <= kMaxBW) of the request's candidates with key >= the theta key and key < hi,
// by streaming its rows once per 8-bit radix digit (at most 8 passes); sorted into s_out. Returns
// how many there are (< k when fewer exist).
template <int T, typename TI>
__device__ int fallback_topk(const StepArgs& a, int req, int k, uint64_t hi, uint64_t* s_sel, uint64_t* s_out,
                             uint32_t* s_hist, uint32_t* s_m32) {
  const int tid = threadIdx.x;
  const int nl = nlive_of(a, req);
  const float th = theta_value(a.theta[req]);
  const uint64_t klo = (uint64_t)a.theta[req] << 32;
  uint64_t prefix = 0, mask = 0;
  uint32_t krem = (uint32_t)k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += T) s_hist[i] = 0;
    __syncthreads();
    for (int b = 0; b < nl; ++b) {
      float S;
      uint32_t node;
      row_state(a, req, b, S, node);
      const float lse = a.lse[(size_t)req * a.BW + b];
      if (S < th || lse != lse) continue;
      for_each_candidate<T, TI>(a, req, b, S, lse, node, [&](uint64_t key) {
        if (key >= klo && key < hi && (key & mask) == prefix) atomicAdd(&s_hist[(key >> shift) & 0xFFu], 1u);
      });
    }
    __syncthreads();
    if (tid < 32) warp_find_digit_desc(s_hist, krem, &s_m32[0], &s_m32[1]);
    __syncthreads();
    uint32_t d = s_m32[0], above = s_m32[1];
    if (d >= 256) {   // fewer candidates than k: take them all
      krem = 0;
      prefix = 0;
      mask = 0;
      __syncthreads();
      break;
    }
    uint32_t inbin = s_hist[d];
    krem -= above;
    prefix |= (uint64_t)d << shift;
    mask |= 0xFFull << shift;
    __syncthreads();
    if (inbin == krem) break;
  }
  if (tid == 0) s_m32[2] = 0;
  __syncthreads();
  const uint64_t thr = prefix;
  for (int b = 0; b < nl; ++b) {
    float S;
    uint32_t node;
    row_state(a, req, b, S, node);
    const float lse = a.lse[(size_t)req * a.BW + b];
    if (S < th || lse != lse) continue;
    for_each_candidate<T, TI>(a, req, b, S, lse, node, [&](uint64_t key) {
      if (key >= thr && key >= klo && key < hi) {
        uint32_t p = atomicAdd(&s_m32[2], 1u);
        if (p < (uint32_t)k) s_sel[p] = key;
      }
    });
  }
  __syncthreads();
  const int kk = min(k, (int)s_m32[2]);
  sort_desc_to<T>(s_sel, kk, s_out);
  return kk;
}

// Per-beam Top-K (NEXT f3) over keys sorted descending: one warp walks them in order with a
// counter per parent row; a key is kept iff fewer than K keys of its row came before it. Kept
// keys are appended to res (in order, so res stays sorted) until BW are kept. Warp 0 only; the
// counters (cnt[BW]) and *nres persist across calls (chunks of one request).
__device__ void topk_scan(const uint64_t* keys, int m, int K, int V, int BW, int* cnt, uint64_t* res, int* nres) {
  const int lane = lane_id();
  int n = *nres;
  for (int base = 0; base < m && n < BW; base += 32) {
    const int i = base + lane;
    const bool valid = i < m;
    const uint64_t key = valid ? keys[i] : 0ull;
    const int b = valid ? (int)(key_flat(key) / (uint32_t)V) : -1 - lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    const uint32_t lt = (1u << lane) - 1u;
    const int c0 = valid ? cnt[b] : 0;
    const bool keep = valid && c0 + __popc(peers & lt) < K;
    __syncwarp();
    if (valid && lane == 31 - __clz(peers)) cnt[b] = c0 + __popc(peers);
    const uint32_t kb = __ballot_sync(0xffffffffu, keep);
    const int pos = n + __popc(kb & lt);
    if (keep && pos < BW) res[pos] = key;
    n += __popc(kb);
    __syncwarp();
  }
  if (lane == 0) *nres = min(n, BW);
}

template <int T, typename TI = float>
__global__ void __launch_bounds__(T) k_select(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  extern __shared__ __align__(16) uint64_t s_keys[];  // [cap] keys, then [2 * kMaxBW] candidates
  uint64_t* s_cand = s_keys + a.cap;
  __shared__ uint64_t s_sel[kMaxBW], s_out[kMaxBW];
  __shared__ TopkScratch s_sc;
  __shared__ ParentInfo s_pi;
  __shared__ int s_nres;
  int* s_rowcnt = reinterpret_cast<int*>(s_cand + kMaxBW);   // per-beam Top-K row counters [BW]
                                                            // (results use s_cand[0 .. BW))
  const int req = blockIdx.x, tid = threadIdx.x;
  if (req_sparse(a, req)) return;   // a mixed step's sparse-route request: k_sparse commits it
  if (tid == 0 && a.seed_cnt) a.seed_cnt[req] = 0u;   // fused seed's arrival count / theta flag
  const uint64_t* src = a.surv + (size_t)req * a.cap;
  const uint64_t p0 = tid < a.cap ? src[tid] : 0ull;
  const uint64_t p1 = tid + T < a.cap ? src[tid + T] : 0ull;
  const size_t pb = (size_t)req * a.BW;
  const uint32_t nd0 = (a.node_in && tid < a.BW) ? a.node_in[pb + tid] : 0u;
  const uint32_t nd1 = (a.node_in && tid + T < a.BW) ? a.node_in[pb + tid + T] : 0u;
  const int nl = nlive_of(a, req);
  const uint32_t n = a.surv_count[req];
  static_assert(2 * T >= kMaxBW, "k_select: parents prefetched two per thread");
  if (n > (uint32_t)a.cap) {
    // the survivor buffer overflowed (weak theta, massive ties): exact multi-pass fallback
    if (tid == 0) {
      a.ovf[req] = 1u;
      atomicOr(a.flags + req, kFlagOverflow);
      count_add(a, XGR_CNT_OVERFLOW, 1);
    }
    prefetch_parents<T>(a, req, nlive_of(a, req), s_pi);
    __syncthreads();
    if (!a.topk) {
      const int kk = fallback_topk<T, TI>(a, req, a.BW, ~0ull, s_sel, s_out, s_sc.hist, s_sc.m32);
      commit<T>(a, req, s_out, kk, s_pi);
    } else {   // per-beam Top-K: chunks of the largest remaining candidates until BW are kept
      for (int i = tid; i < a.BW; i += T) s_rowcnt[i] = 0;
      if (tid == 0) s_nres = 0;
      __syncthreads();
      uint64_t hi = ~0ull;
      for (;;) {
        const int kk = fallback_topk<T, TI>(a, req, kMaxBW, hi, s_sel, s_out, s_sc.hist, s_sc.m32);
        if (tid < 32) topk_scan(s_out, kk, a.topk, a.trie.V, a.BW, s_rowcnt, s_cand, &s_nres);
        __syncthreads();
        if (s_nres >= a.BW || kk < kMaxBW) break;
        hi = s_out[kk - 1];
        __syncthreads();
      }
      commit<T>(a, req, s_cand, s_nres, s_pi);
    }
    return;
  }
  const int k = min((int)n, a.BW);
  // survivors 0..2T-1 and the parents' beam state were loaded speculatively above, alongside
  // the count and nlive, so each chain is one load shorter
  if ((uint32_t)tid < n) s_keys[tid] = p0;
  if ((uint32_t)(tid + T) < n) s_keys[tid + T] = p1;
  for (uint32_t i = tid + 2 * T; i < n; i += T) s_keys[i] = src[i];
  {
    const LevelDev& L = a.trie.lv[a.level];
    if (tid < nl) {
      s_pi.fc[tid] = L.first_child[nd0];
      s_pi.fcn[tid] = L.first_child[nd0 + 1];
      s_pi.slot[tid] = L.dense_slot ? L.dense_slot[nd0] : -1;
    }
    if (tid + T < nl) {
      s_pi.fc[tid + T] = L.first_child[nd1];
      s_pi.fcn[tid + T] = L.first_child[nd1 + 1];
      s_pi.slot[tid + T] = L.dense_slot ? L.dense_slot[nd1] : -1;
    }
  }
  __syncthreads();
  if (a.dbg & 128) return;
  if (!a.topk) {
    block_topk_fast<T>(s_keys, (int)n, k, s_cand, 2 * kMaxBW, s_sel, s_out, s_sc, a.dbg >> 10);
    if (a.dbg & 256) return;
    commit<T>(a, req, s_out, k, s_pi);
  } else {
    // per-beam Top-K (NEXT f3): take the largest remaining survivors in sorted chunks of up to
    // kMaxBW, keep those within their row's first K, until BW are kept; processed keys are zeroed
    // (0 is below every real key), so each chunk is the next one in descending order
    for (int i = tid; i < a.BW; i += T) s_rowcnt[i] = 0;
    if (tid == 0) s_nres = 0;
    __syncthreads();
    int nz = (int)n;
    while (nz > 0) {
      const int kc = min(nz, kMaxBW);
      block_select_topk<T>(s_keys, (int)n, kc, s_sel, s_out, s_sc.hist, s_sc.m64, s_sc.m32);
      if (tid < 32) topk_scan(s_out, kc, a.topk, a.trie.V, a.BW, s_rowcnt, s_cand, &s_nres);
      __syncthreads();
      if (s_nres >= a.BW || kc == nz) break;
      const uint64_t thr = s_out[kc - 1];
      for (uint32_t i = tid; i < n; i += T)
        if (s_keys[i] >= thr) s_keys[i] = 0ull;
      nz -= kc;
      __syncthreads();
    }
    commit<T>(a, req, s_cand, s_nres, s_pi);
  }
}

// ---------------------------------------------------------------------------------------------
// k_merge (codebook shard): every rank's local top-BW keys of a request, all-gathered
// into [nranks][batch][BW]; the global top-BW of their union is the step's result (each key
// carries its global score and flat index), committed identically on every rank (each rank holds
// the whole trie, so child ids are computed locally).
// ---------------------------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(T) k_merge(const __grid_constant__ StepArgs a, const uint64_t* grec,
                                             const int32_t* grec_n) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  extern __shared__ __align__(16) uint64_t s_keys[];  // [nranks * BW] keys, then [2 * kMaxBW]
  __shared__ uint64_t s_sel[kMaxBW], s_out[kMaxBW];
  __shared__ TopkScratch s_sc;
  __shared__ ParentInfo s_pi;
  __shared__ int s_off[65];
  __shared__ int s_cnt[64];
  const int req = blockIdx.x, tid = threadIdx.x, lane = lane_id();
  uint64_t* s_cand = s_keys + (size_t)a.nranks * a.BW;
  if (grec_n) {
    if (tid < a.nranks) s_cnt[tid] = grec_n[tid * a.batch + req];
  } else {
    // no counts exchanged: each rank's records are sorted descending and 0-padded, and no real key
    // is 0 (its score half is orderable(c) != 0 for every c, -inf included), so the count is the
    // number of nonzero keys -- one warp per rank
    for (int g = tid >> 5; g < a.nranks; g += T / 32) {
      const uint64_t* src = grec + ((size_t)g * a.batch + req) * a.BW;
      int c = 0;
      for (int i = lane; i < a.BW; i += 32) c += src[i] != 0ull;
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0) s_cnt[g] = c;
    }
  }
  prefetch_parents<T>(a, req, nlive_of(a, req), s_pi);
  __syncthreads();
  if (tid == 0) {
    int o = 0;
    for (int g = 0; g < a.nranks; ++g) {
      s_off[g] = o;
      o += s_cnt[g];
    }
    s_off[a.nranks] = o;
  }
  __syncthreads();
  const int n = s_off[a.nranks];
  for (int g = 0; g < a.nranks; ++g) {
    const int ng = s_off[g + 1] - s_off[g];
    const uint64_t* src = grec + ((size_t)g * a.batch + req) * a.BW;
    for (int i = tid; i < ng; i += T) s_keys[s_off[g] + i] = src[i];
  }
  __syncthreads();
  const int k = min(n, a.BW);
  block_topk_fast<T>(s_keys, n, k, s_cand, 2 * kMaxBW, s_sel, s_out, s_sc, a.dbg >> 10);
  commit<T>(a, req, s_out, k, s_pi);
}

// ---------------------------------------------------------------------------------------------
// k_sparse: one CTA per request; every legal candidate is formed on chip (no pruning needed).
// ROOT: the single root row, gathered by the whole block. Otherwise one THREAD per live row for
// rows with <= 16 children (all rows' dependent load chains node -> first_child -> labels ->
// logits run concurrently), and one warp per row for the rare larger rows.
// ---------------------------------------------------------------------------------------------
// Children of [fc, fe) whose token lies in this rank's columns [col0, col0 + Vl) (codebook shard):
// the labels are sorted, so they are a contiguous sub-range found by two binary searches.
__device__ __forceinline__ void shard_range(const StepArgs& a, const uint16_t* lab, uint32_t& fc, uint32_t& fe) {
  uint32_t lo = fc, hi = fe;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (lab[mid] < (uint32_t)a.col0) lo = mid + 1; else hi = mid;
  }
  const uint32_t f0 = lo;
  hi = fe;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (lab[mid] < (uint32_t)(a.col0 + a.Vl)) lo = mid + 1; else hi = mid;
  }
  fc = f0;
  fe = lo;
}

// SH (codebook-shard select phase at a sparse step): only the children in this rank's columns,
// logits holding those columns, the GLOBAL lse from all ranks' stats; the commit writes this rank's
// local top-BW records.
template <int T, bool ROOT, typename TI = float, bool CMP = false, bool SH = false>
__global__ void __launch_bounds__(T, 2) k_sparse(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  extern __shared__ __align__(16) uint64_t s_dynk[];  // [2 * kMaxBW] candidates, then the keys
  uint64_t* s_cand = s_dynk;
  uint64_t* s_keys = s_dynk + 2 * kMaxBW;
  __shared__ uint64_t s_sel[kMaxBW], s_out[kMaxBW];
  __shared__ TopkScratch s_sc;
  constexpr int NR = ROOT ? 1 : kMaxBW;   // parent rows
  __shared__ ParentInfoN<NR> s_pi;
  __shared__ float s_red[T / 32], s_red2[T / 32];
  __shared__ uint32_t s_count, s_nbig, s_nroot, s_bin;
  __shared__ uint32_t s_wtot[T / 32];
  __shared__ uint16_t s_rbase[NR], s_rcnt[NR];   // each row's key segment (per-beam Top-K)
  __shared__ int32_t s_big[NR];
  const int req = blockIdx.x, tid = threadIdx.x, lane = lane_id();
  if (a.mixed && !req_sparse(a, req)) return;   // a mixed step's dense-route request
  // beam state of rows tid and tid + T loaded speculatively, alongside nlive
  static_assert(2 * T >= kMaxBW, "k_sparse: two rows per thread");
  float S_pre[2];
  uint32_t node_pre[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    S_pre[u] = 0.f;
    node_pre[u] = 0u;
    if (!ROOT && tid + u * T < a.BW) row_state(a, req, tid + u * T, S_pre[u], node_pre[u]);
  }
  const int nl = nlive_of(a, req);
  const LevelDev& L = a.trie.lv[a.level];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  const int V = a.trie.V;
  if (tid == 0) {
    s_count = 0;
    s_nbig = 0;
    s_nroot = 0;
  }
  // the commit's parent info (first child, end, dense slot) is written by the gather below,
  // which loads the same node data; the barriers before the commit order it
  if (ROOT) prefetch_parents<T>(a, req, nl, s_pi);
  __syncthreads();
  if (ROOT) {
    constexpr int RPT = 16;   // root children held in registers per thread (<= 8192 children)
    for (int b = 0; b < nl; ++b) {
      float S;
      uint32_t node;
      row_state(a, req, b, S, node);
      const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
      const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
      if (fe - fc <= (uint32_t)(T * RPT)) {
        // all loads issued up front: labels, then the logits they select
        uint32_t vv[RPT];
        float xv[RPT];
        const bool all_legal = fe - fc == (uint32_t)V;   // labels are then 0..V-1: no label loads
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const uint32_t q = fc + (uint32_t)(k * T + tid);
          vv[k] = q < fe ? (all_legal ? q - fc : (uint32_t)lab[q]) : 0u;
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const uint32_t q = fc + (uint32_t)(k * T + tid);
          xv[k] = q < fe ? ldx(row + vv[k]) : -INFINITY;
        }
        float tmax = -INFINITY;
#pragma unroll
        for (int k = 0; k < RPT; ++k) tmax = fmaxf(tmax, xv[k]);
        const float M = block_max<T>(tmax, s_red);
        float z = 0.f;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (fc + (uint32_t)(k * T + tid) < fe) z += ex2(__fmul_rn(__fsub_rn(xv[k], M), kLog2e));
        const float Z = block_sum<T>(z, s_red2);
        const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
        const float lse = row_lse(M, Z);
        if (!finite && tid == 0) atomicOr(a.flags + req, kFlagNonfinite);
        if (nl == 1 && fe - fc > 2u * T && a.sparse_cap >= 4096) {
          // single root row: only the candidates that can reach the Top-BW go to shared memory.
          // A histogram of the keys' top 13 bits (8192 bins, in the key buffer) gives the bin B
          // where the count from the top reaches min(BW, n); the keys in bins >= B (typically
          // ~1.3 x BW) are compacted and the selection below sorts only those. (The histogram needs
          // 32 KB of the key buffer: sparse_cap >= 4096 keys.)
          uint32_t* hist = reinterpret_cast<uint32_t*>(s_keys);
          uint64_t kk[RPT];
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const uint32_t q = fc + (uint32_t)(k * T + tid);
            kk[k] = q < fe ? make_key(cand_score(S, xv[k], lse), (uint32_t)b * V + vv[k]) : 0ull;
          }
          for (int i = tid; i < 8192; i += T) hist[i] = 0u;
          if (tid == 0) s_nroot = fe - fc;
          __syncthreads();
#pragma unroll
          for (int k = 0; k < RPT; ++k)
            hist_inc_if(kk[k] != 0ull, hist, (uint32_t)(kk[k] >> 51));
          __syncthreads();
          // thread t owns bins 8191 - 16 t - j (j < 16): descending order over the block
          uint32_t c16[16], loc = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            c16[j] = hist[8191 - 16 * tid - j];
            loc += c16[j];
          }
          uint32_t incl = loc;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane == 31) s_wtot[tid >> 5] = incl;
          if (tid == 0) s_bin = 0u;
          __syncthreads();
          uint32_t before = incl - loc;
          for (int w = 0; w < (tid >> 5); ++w) before += s_wtot[w];
          const uint32_t need = min((uint32_t)a.BW, fe - fc);
          if (before < need && before + loc >= need) {
            uint32_t acc = before;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (acc < need && acc + c16[j] >= need) s_bin = 8191u - 16u * tid - j;
              acc += c16[j];
            }
          }
          __syncthreads();
          const uint32_t bmin = s_bin;
          uint32_t cnt = 0;
#pragma unroll
          for (int k = 0; k < RPT; ++k) cnt += (kk[k] && (uint32_t)(kk[k] >> 51) >= bmin) ? 1u : 0u;
          uint32_t ci = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, ci, o);
            if (lane >= o) ci += y;
          }
          uint32_t wb = 0;
          if (lane == 31 && ci) wb = atomicAdd(&s_count, ci);
          uint32_t pos = __shfl_sync(0xffffffffu, wb, 31) + ci - cnt;
          __syncthreads();   // the histogram is dead; the key buffer takes the candidates
#pragma unroll
          for (int k = 0; k < RPT; ++k)
            if (kk[k] && (uint32_t)(kk[k] >> 51) >= bmin) s_keys[pos++] = kk[k];
          __syncthreads();
          continue;
        }
        const uint32_t base = s_count;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const uint32_t q = fc + (uint32_t)(k * T + tid);
          if (q < fe) s_keys[base + (q - fc)] = make_key(cand_score(S, xv[k], lse), (uint32_t)b * V + vv[k]);
        }
        __syncthreads();
        if (tid == 0) s_count = base + (fe - fc);
        __syncthreads();
        continue;
      }
      float tmax = -INFINITY;
      for (uint32_t k = fc + tid; k < fe; k += T) tmax = fmaxf(tmax, ldx(row + lab[k]));
      const float M = block_max<T>(tmax, s_red);
      float z = 0.f;
      for (uint32_t k = fc + tid; k < fe; k += T)
        z += ex2(__fmul_rn(__fsub_rn(ldx(row + lab[k]), M), kLog2e));
      const float Z = block_sum<T>(z, s_red2);
      const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
      const float lse = row_lse(M, Z);
      if (!finite && tid == 0) atomicOr(a.flags + req, kFlagNonfinite);
      const uint32_t base = s_count;
      for (uint32_t k = fc + tid; k < fe; k += T) {
        uint32_t v = lab[k];
        s_keys[base + (k - fc)] = make_key(cand_score(S, ldx(row + v), lse), (uint32_t)b * V + v);
      }
      __syncthreads();
      if (tid == 0) s_count = base + (fe - fc);
      __syncthreads();
    }
  } else {
    constexpr int kSmall = 16;
#pragma unroll 1
    for (int u = 0; u < 2; ++u) {
      const int b = tid + u * T;
      if (b >= nl) break;
      const float S = u ? S_pre[1] : S_pre[0];
      const uint32_t node = u ? node_pre[1] : node_pre[0];
      const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
      s_pi.fc[b] = fc;
      s_pi.fcn[b] = fe;
      s_pi.slot[b] = L.dense_slot ? L.dense_slot[node] : -1;
      uint32_t f0 = fc, f1 = fe;
      if (SH) shard_range(a, lab, f0, f1);
      const int cnt = (int)(f1 - f0);
      if (cnt > kSmall) {
        s_big[atomicAdd(&s_nbig, 1u)] = b;
        continue;
      }
      const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld -
                      (SH ? a.col0 : 0);
      const float* crow = CMP ? a.clog + ((size_t)req * a.BW + b) * a.cld : nullptr;
      uint32_t vv[kSmall];
      float xv[kSmall];
#pragma unroll
      for (int k = 0; k < kSmall; ++k) vv[k] = k < cnt ? lab[f0 + k] : 0u;
#pragma unroll
      for (int k = 0; k < kSmall; ++k) xv[k] = k < cnt ? (CMP ? crow[k] : ldx(row + vv[k])) : -INFINITY;
      bool finite;
      float lse;
      if (SH) {
        lse = shard_lse(a, req, b, finite);
      } else {
        float M = -INFINITY;
#pragma unroll
        for (int k = 0; k < kSmall; ++k) M = fmaxf(M, xv[k]);
        float Z = 0.f;
#pragma unroll
        for (int k = 0; k < kSmall; ++k)
          if (k < cnt) Z += ex2(__fmul_rn(__fsub_rn(xv[k], M), kLog2e));
        finite = (Z > 0.5f) && (Z <= 3.0e38f);
        lse = row_lse(M, Z);
      }
      if (!finite) atomicOr(a.flags + req, kFlagNonfinite);
      if (SH && cnt == 0) continue;   // no child of this row in this rank's columns
      const uint32_t base = atomicAdd(&s_count, (uint32_t)cnt);
      XGR_CHECK(base + cnt <= (uint32_t)a.sparse_cap, "sparse keys base %u cnt %d cap %d", base, cnt, a.sparse_cap);
      s_rbase[b] = (uint16_t)base;
      s_rcnt[b] = (uint16_t)cnt;
#pragma unroll
      for (int k = 0; k < kSmall; ++k)
        if (k < cnt) s_keys[base + k] = make_key(cand_score(S, xv[k], lse), (uint32_t)b * V + vv[k]);
    }
    __syncthreads();
    const int nbig = (int)s_nbig;
    for (int i = tid >> 5; i < nbig; i += T / 32) {
      const int b = s_big[i];
      float S;
      uint32_t node;
      row_state(a, req, b, S, node);
      const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld -
                      (SH ? a.col0 : 0);
      uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
      const float* crow = CMP ? a.clog + ((size_t)req * a.BW + b) * a.cld - fc : nullptr;
      if (SH) shard_range(a, lab, fc, fe);
      auto xq = [&](uint32_t k) { return CMP ? crow[k] : ldx(row + lab[k]); };
      bool finite;
      float lse;
      if (SH) {
        lse = shard_lse(a, req, b, finite);
      } else {
        float tmax = -INFINITY;
        for (uint32_t k = fc + lane; k < fe; k += 32) tmax = fmaxf(tmax, xq(k));
        const float M = warp_max(tmax);
        float z = 0.f;
        for (uint32_t k = fc + lane; k < fe; k += 32)
          z += ex2(__fmul_rn(__fsub_rn(xq(k), M), kLog2e));
        const float Z = warp_sum(z);
        finite = (Z > 0.5f) && (Z <= 3.0e38f);
        lse = row_lse(M, Z);
      }
      if (!finite && lane == 0) atomicOr(a.flags + req, kFlagNonfinite);
      uint32_t base = 0;
      if (lane == 0) {
        base = atomicAdd(&s_count, fe - fc);
        s_rbase[b] = (uint16_t)base;
        s_rcnt[b] = (uint16_t)(fe - fc);
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      for (uint32_t k = fc + lane; k < fe; k += 32) {
        uint32_t v = lab[k];
        s_keys[base + (k - fc)] = make_key(cand_score(S, xq(k), lse), (uint32_t)b * V + v);
      }
    }
  }
  __syncthreads();
  const int n = (int)s_count;
  if (tid == 0) count_add(a, XGR_CNT_SPARSE_CANDS, ROOT && s_nroot ? s_nroot : (uint32_t)n);
  int k = min(n, a.BW);
  if (a.topk) {
    if (ROOT) {
      k = min(k, a.topk);   // one row: its Top-K, then the Top-BW of those
    } else {
      // per-beam Top-K (NEXT f3): a key whose row segment holds >= K larger keys is dropped
      // (zeroed: 0 is below every real key, so the selection below never takes it)
      uint32_t* s_kill = s_sc.hist;   // scratch: 256 words, a bit per key in chunks of 8192
      int killed = 0;
      for (int c0 = 0; c0 < n; c0 += 8192) {
        for (int i = tid; i < 256; i += T) s_kill[i] = 0u;
        __syncthreads();
        for (int i = c0 + tid; i < min(n, c0 + 8192); i += T) {
          const uint64_t key = s_keys[i];
          const int b = (int)(key_flat(key) / (uint32_t)V);
          const int cnt = s_rcnt[b];
          if (cnt > a.topk) {
            const int base = s_rbase[b];
            int r = 0;
            for (int j = base; j < base + cnt; ++j) r += s_keys[j] > key;
            if (r >= a.topk) atomicOr(&s_kill[(i - c0) >> 5], 1u << ((i - c0) & 31));
          }
        }
        __syncthreads();
        for (int i = c0 + tid; i < min(n, c0 + 8192); i += T)
          if ((s_kill[(i - c0) >> 5] >> ((i - c0) & 31)) & 1u) s_keys[i] = 0ull;
        for (int w = tid; w < 256; w += T) killed += __popc(s_kill[w]);
        __syncthreads();
      }
      killed = block_sum_i<T>(killed, reinterpret_cast<int*>(s_red));
      k = min(n - killed, a.BW);
    }
  }
  block_topk_fast<T>(s_keys, n, k, s_cand, 2 * kMaxBW, s_sel, s_out, s_sc, a.dbg >> 10);
  commit<T>(a, req, s_out, k, s_pi);
}

// ---------------------------------------------------------------------------------------------
// k_route_list (mixed step): the dense-route requests (next-step candidates counted by the previous
// commit > kSparseCap) compacted in ascending order: list[0] = count, list[1..] = request ids.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_route_list(const __grid_constant__ StepArgs a, int32_t* list) {
  pdl_wait();
  __shared__ int s_w[32];
  __shared__ int s_base;
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < a.batch; c0 += 1024) {
    const int req = c0 + tid;
    const bool dense = req < a.batch && !req_sparse(a, req);
    const uint32_t bal = __ballot_sync(0xffffffffu, dense);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_w[w];
    if (dense) list[1 + off + __popc(bal & ((1u << lane) - 1u))] = req;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += s_w[w];
      s_base += t;
    }
    __syncthreads();
  }
  if (tid == 0) list[0] = s_base;
}

// ---------------------------------------------------------------------------------------------
// k_sparse_rows: the sparse-parent rows of a dense-route step (skewed tries mix dense and sparse
// nodes on one level). One thread per row: theta is known (seed), so the row is skipped if
// S_b < theta, else its legal logits are gathered by label, its lse computed (stored for the exact
// fallback), and its candidates c >= theta emitted to the request's survivor buffer.
// ---------------------------------------------------------------------------------------------
template <typename TI>
__global__ void __launch_bounds__(128) k_sparse_rows(const __grid_constant__ StepArgs a, int rows) {
  pdl_wait();
  const int req = blockIdx.x, b = blockIdx.y * 128 + threadIdx.x;
  if (b >= rows || b >= nlive_of(a, req) || req_sparse(a, req)) return;
  float S;
  uint32_t node;
  row_state(a, req, b, S, node);
  const LevelDev& L = a.trie.lv[a.level];
  if (L.dense_slot && L.dense_slot[node] >= 0) return;   // dense rows: k_stream
  const float th = theta_value(a.theta[req]);
  float* lse_out = a.lse + (size_t)req * a.BW + b;
  if (S < th) {   // every candidate of the row is <= S_b < theta: not read
    *lse_out = __int_as_float(0x7fc00000);
    count_add(a, XGR_CNT_ROWS_SKIP_PRE, 1);
    return;
  }
  const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
  const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  float M = -INFINITY;
  for (uint32_t q = fc; q < fe; ++q) M = fmaxf(M, ldx(row + lab[q]));
  float Z = 0.f;
  for (uint32_t q = fc; q < fe; ++q) Z += ex2(__fmul_rn(__fsub_rn(ldx(row + lab[q]), M), kLog2e));
  const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
  const float lse = row_lse(M, Z);
  *lse_out = finite ? lse : __int_as_float(0x7fc00000);
  count_add(a, XGR_CNT_ROWS_READ, 1);
  count_add(a, XGR_CNT_LEGAL, fe - fc);
  if (!finite) {
    atomicOr(a.flags + req, kFlagNonfinite);
    return;
  }
  if (!(cand_score(S, M, lse) >= th)) {   // UB_b = S_b - ln Z_b < theta
    count_add(a, XGR_CNT_ROWS_SKIP_POST, 1);
    return;
  }
  const uint32_t fbase = (uint32_t)b * (uint32_t)a.trie.V;
  uint64_t* sbuf = a.surv + (size_t)req * a.cap;
  uint32_t n = 0;
  for (uint32_t q = fc; q < fe; ++q) {
    const uint32_t v = lab[q];
    const float c = cand_score(S, ldx(row + v), lse);
    if (c >= th) {
      const uint32_t pos = atomicAdd(a.surv_count + req, 1u);
      if (pos < (uint32_t)a.cap) sbuf[pos] = make_key(c, fbase + v);
      ++n;
    }
  }
  count_add(a, XGR_CNT_SURVIVORS, n);
}

// ---------------------------------------------------------------------------------------------
// k_sparse_stats (codebook-shard stats phase at a sparse step): one thread per live row, the local
// (m, Z) over the row's children in this rank's columns ((-inf, 0) when it has none).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_sparse_stats(const __grid_constant__ StepArgs a, int rows) {
  pdl_wait();
  const int req = blockIdx.x, b = blockIdx.y * 128 + threadIdx.x;
  if (b >= rows || b >= nlive_of(a, req)) return;
  float S;
  uint32_t node;
  row_state(a, req, b, S, node);
  const LevelDev& L = a.trie.lv[a.level];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  shard_range(a, lab, fc, fe);
  const float* row = static_cast<const float*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld - a.col0;
  float M = -INFINITY;
  for (uint32_t q = fc; q < fe; ++q) M = fmaxf(M, row[lab[q]]);
  float Z = 0.f;
  for (uint32_t q = fc; q < fe; ++q) Z += ex2(__fmul_rn(__fsub_rn(row[lab[q]], M), kLog2e));
  a.stats_out[(size_t)req * a.BW + b] = M == -INFINITY && Z == Z ? make_float2(-INFINITY, 0.f) : make_float2(M, Z);
}

// ---------------------------------------------------------------------------------------------
// The paper's own selection procedure on the GPU (SURVEY 8(f) f3 "paper-heap GPU variant"): an
// in-repo baseline for the threshold-pruned design, selected with XGR_CFG_PAPER_HEAP at init. It
// computes the same result (the heap is exact), the way PAPER.md section 6.2 describes it:
//  * L156 / L376: each beam's Top-K candidates, sorted descending ("the log_prob results for each
//    beam are inherently in descending order") -- k_ph_rows, one CTA per (request, beam): the beam's
//    legal logits, log-softmax, every candidate key in shared memory, exact block Top-K (radix
//    select + sort), written to a per-beam list;
//  * L385: "a global min heap of size BW ... visits the leaves of each sub-beam tree sequentially
//    ... if the leaf's log_prob exceeds that of the heap's top element, it is inserted ...
//    Otherwise, the sorting operation of that beam is terminated immediately" -- k_ph_heap, one CTA
//    per request whose first thread runs the heap sequentially (with the sorted-beam-score stop of
//    SURVEY 8(c.2)); the heap is then sorted and committed like any step.
// Only dense-route steps take it (the paper's sorting bottleneck); sparse steps are unchanged.
// ---------------------------------------------------------------------------------------------
template <int T, typename TI>
__global__ void __launch_bounds__(T) k_ph_rows(const __grid_constant__ StepArgs a) {
  extern __shared__ __align__(16) uint64_t s_k[];   // [V] candidate keys of the beam
  __shared__ uint64_t s_sel[kMaxBW], s_out[kMaxBW];
  __shared__ TopkScratch s_sc;
  __shared__ float s_red[T / 32], s_red2[T / 32];
  __shared__ uint32_t s_n;
  const int req = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int K = a.topk ? a.topk : a.BW;
  uint64_t* lst = a.ph_lists + ((size_t)req * a.BW + b) * K;
  if (b >= nlive_of(a, req)) {
    if (tid == 0) a.ph_cnt[(size_t)req * a.BW + b] = 0;
    return;
  }
  float S;
  uint32_t node;
  row_state(a, req, b, S, node);
  const LevelDev& L = a.trie.lv[a.level];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
  // the beam's legal logits (its children in label order)
  float tm = -INFINITY;
  for (uint32_t q = fc + tid; q < fe; q += T) tm = fmaxf(tm, ldx(row + lab[q]));
  const float M = block_max<T>(tm, s_red);
  float z = 0.f;
  for (uint32_t q = fc + tid; q < fe; q += T) z += ex2(__fmul_rn(__fsub_rn(ldx(row + lab[q]), M), kLog2e));
  const float Z = block_sum<T>(z, s_red2);
  const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
  const float lse = row_lse(M, Z);
  if (!finite && tid == 0) atomicOr(a.flags + req, kFlagNonfinite);
  const uint32_t fbase = (uint32_t)b * (uint32_t)a.trie.V;
  const int n = (int)(fe - fc);
  for (int i = tid; i < n; i += T) {
    const uint32_t v = lab[fc + i];
    s_k[i] = make_key(cand_score(S, ldx(row + v), lse), fbase + v);
  }
  __syncthreads();
  const int k = min(n, K);
  if (k < n) {
    block_select_topk<T>(s_k, n, k, s_sel, s_out, s_sc.hist, s_sc.m64, s_sc.m32);
  } else {
    for (int i = tid; i < n; i += T) s_sel[i] = s_k[i];
    __syncthreads();
    sort_desc_to<T>(s_sel, n, s_out);
  }
  for (int i = tid; i < k; i += T) lst[i] = s_out[i];
  if (tid == 0) a.ph_cnt[(size_t)req * a.BW + b] = k;
}

template <int T>
__global__ void __launch_bounds__(T) k_ph_heap(const __grid_constant__ StepArgs a) {
  __shared__ uint64_t s_heap[kMaxBW], s_out[kMaxBW];
  __shared__ ParentInfo s_pi;
  __shared__ int s_hn;
  const int req = blockIdx.x, tid = threadIdx.x;
  const int nl = nlive_of(a, req), BW = a.BW;
  const int K = a.topk ? a.topk : a.BW;
  prefetch_parents<T>(a, req, nl, s_pi);
  if (tid == 0) {
    // min-heap of keys (a larger key is a better candidate: score desc, flat asc)
    int hn = 0;
    uint64_t visits = 0;
    for (int b = 0; b < nl; ++b) {
      float S;
      uint32_t node;
      row_state(a, req, b, S, node);
      // every candidate of beam b and of later beams is <= S_b, and later beams have larger flat
      // indices: once the heap is full and S_b <= its minimum score nothing can enter any more
      if (hn == BW && !(S > key_score(s_heap[0]))) break;
      const uint64_t* lst = a.ph_lists + ((size_t)req * BW + b) * K;
      const int cnt = a.ph_cnt[(size_t)req * BW + b];
      for (int i = 0; i < cnt; ++i) {
        const uint64_t key = lst[i];
        ++visits;
        if (hn < BW) {   // push, sift up
          int j = hn++;
          while (j > 0) {
            const int p = (j - 1) >> 1;
            if (s_heap[p] <= key) break;
            s_heap[j] = s_heap[p];
            j = p;
          }
          s_heap[j] = key;
        } else if (key > s_heap[0]) {   // replace the minimum, sift down
          int j = 0;
          for (;;) {
            const int l = 2 * j + 1, r = l + 1;
            int m = j;
            uint64_t mv = key;
            if (l < hn && s_heap[l] < mv) { m = l; mv = s_heap[l]; }
            if (r < hn && s_heap[r] < mv) { m = r; mv = s_heap[r]; }
            if (m == j) break;
            s_heap[j] = s_heap[m];
            j = m;
          }
          s_heap[j] = key;
        } else {
          break;   // the beam's traversal terminates
        }
      }
    }
    s_hn = hn;
    count_add(a, XGR_CNT_SURVIVORS, visits);   // heap visits (the paper's sorting work)
  }
  __syncthreads();
  const int hn = s_hn;
  sort_desc_to<T>(s_heap, hn, s_out);
  commit<T>(a, req, s_out, hn, s_pi);
}

cudaError_t launch_paper_heap(const StepArgs& a, int rows, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                              int* launches) {
  const size_t smem = (size_t)a.trie.V * sizeof(uint64_t);
  cudaError_t e;
  if (a.dtype == XGR_DTYPE_BF16) {
    if ((e = cudaFuncSetAttribute(k_ph_rows<512, __nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)))
      return e;
  } else if ((e = cudaFuncSetAttribute(k_ph_rows<512, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) {
    return e;
  }
  if (ev0) cudaEventRecord(ev0, s);
  if (a.dtype == XGR_DTYPE_BF16) launch_pdl(k_ph_rows<512, __nv_bfloat16>, dim3(a.batch, rows), 512, smem, s, a);
  else launch_pdl(k_ph_rows<512, float>, dim3(a.batch, rows), 512, smem, s, a);
  launch_pdl(k_ph_heap<256>, a.batch, 256, 0, s, a);
  if (ev1) cudaEventRecord(ev1, s);
  *launches += 2;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// support: children of prefixes, read from the representation the step kernels use.
// ---------------------------------------------------------------------------------------------
__global__ void k_children(TrieDev tr, const int32_t* prefixes, int depth, int64_t n, int32_t* counts,
                           int32_t* tokens, int64_t cap) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t node = 0;
  for (int d = 0; d < depth; ++d) {
    int32_t t = prefixes[i * depth + d];
    const LevelDev& L = tr.lv[d];
    bool legal = false;
    if (t >= 0 && t < tr.V) {
      int slot = L.dense_slot ? L.dense_slot[node] : -1;
      if (slot >= 0) {
        legal = (L.bitmap[(size_t)slot * tr.W + (t >> 5)] >> (t & 31)) & 1u;
      } else {
        for (uint32_t k = L.first_child[node]; k < L.first_child[node + 1]; ++k)
          if (tr.lv[d + 1].label[k] == (uint16_t)t) legal = true;
      }
    }
    if (!legal) {
      counts[i] = -1;
      return;
    }
    node = child_of(tr, d, node, (uint32_t)t);
  }
  const LevelDev& L = tr.lv[depth];
  const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  const uint16_t* lab = tr.lv[depth + 1].label;
  int slot = L.dense_slot ? L.dense_slot[node] : -1;
  int32_t c = 0;
  bool ok = true;
  if (slot >= 0) {
    const uint32_t* bm = L.bitmap + (size_t)slot * tr.W;
    for (int v = 0; v < tr.V; ++v) {
      if ((bm[v >> 5] >> (v & 31)) & 1u) {
        if (c < cap) tokens[i * cap + c] = v;
        if (fc + c >= fe || lab[fc + c] != (uint16_t)v || child_of(tr, depth, node, v) != fc + c) ok = false;
        ++c;
      }
    }
    if ((uint32_t)c != fe - fc) ok = false;
  } else {
    for (uint32_t k = fc; k < fe; ++k) {
      if (c < cap) tokens[i * cap + c] = lab[k];
      if (k > fc && lab[k] <= lab[k - 1]) ok = false;
      ++c;
    }
  }
  counts[i] = ok ? c : -2;
}

// ---------------------------------------------------------------------------------------------
// support: algorithmic bytes of the last step; not on the timed path.
// ---------------------------------------------------------------------------------------------
__global__ void k_account(const __grid_constant__ StepArgs a, uint32_t* touched,
                          unsigned long long* out /* alg, full, legal */) {
  // this rank's columns [c0, c0 + Vl): the whole row unless codebook-sharded
  const int req = blockIdx.x, b = blockIdx.y;
  const int nl = nlive_of(a, req);
  if (b >= nl) return;
  const int k = a.nlive_out[req];
  const float thstar = k > 0 ? a.score_out[(size_t)req * a.BW + k - 1] : -INFINITY;
  float S;
  uint32_t node;
  row_state(a, req, b, S, node);
  const LevelDev& L = a.trie.lv[a.level];
  const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  const int c0 = a.col0, Vl = a.Vl;
  const int esz = a.dtype == XGR_DTYPE_BF16 ? 2 : 4;   // bytes per logit; a 32-B sector holds 32/esz
  uint32_t nleg = 0;   // legal children in this rank's columns
  for (uint32_t k2 = fc + threadIdx.x; k2 < fe; k2 += blockDim.x)
    nleg += (lab[k2] >= (uint32_t)c0 && lab[k2] < (uint32_t)(c0 + Vl)) ? 1u : 0u;
  nleg = __reduce_add_sync(0xffffffffu, nleg);
  if (lane_id() == 0 && nleg) atomicAdd(out + 2, (unsigned long long)nleg);
  if (threadIdx.x == 0) atomicAdd(out + 1, (unsigned long long)Vl * (unsigned long long)esz);
  if (S < thstar) return;  // a row the method need not read
  const int slot = L.dense_slot ? L.dense_slot[node] : -1;
  unsigned long long bytes = 0;
  if (slot >= 0) {
    if (esz == 4) {   // 8 tokens per sector: one bitmap byte
      const uint8_t* bm = reinterpret_cast<const uint8_t*>(L.bitmap + (size_t)slot * a.trie.W) + c0 / 8;
      for (int s2 = threadIdx.x; s2 < (Vl + 7) / 8; s2 += blockDim.x) bytes += bm[s2] ? 32ull : 0ull;
    } else {          // 16 tokens per sector: one bitmap half-word
      const uint16_t* bm = reinterpret_cast<const uint16_t*>(L.bitmap + (size_t)slot * a.trie.W) + c0 / 16;
      for (int s2 = threadIdx.x; s2 < (Vl + 15) / 16; s2 += blockDim.x) bytes += bm[s2] ? 32ull : 0ull;
    }
    if (threadIdx.x == 0) {
      uint32_t old = atomicOr(touched + (slot >> 5), 1u << (slot & 31));
      if (!((old >> (slot & 31)) & 1u)) bytes += (unsigned long long)((Vl + 7) / 8);
      bytes += 16;
    }
  } else {
    for (uint32_t k2 = fc + threadIdx.x; k2 < fe; k2 += blockDim.x) {
      const uint32_t v = lab[k2];
      if (v < (uint32_t)c0 || v >= (uint32_t)(c0 + Vl)) continue;
      if (k2 == fc || lab[k2 - 1] < (uint32_t)c0 || ((v - c0) * esz) / 32 != ((lab[k2 - 1] - c0) * esz) / 32)
        bytes += 32;
    }
    if (threadIdx.x == 0) bytes += 4 + 2ull * (fe - fc) + 16;
  }
  bytes = __reduce_add_sync(0xffffffffu, (unsigned)bytes);
  if (lane_id() == 0 && bytes) atomicAdd(out, bytes);
}

// ---------------------------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------------------------
template <int T, int VPT>
static cudaError_t launch_dense(const StepArgs& a, int rows, cudaStream_t s, cudaEvent_t ev0,
                                cudaEvent_t ev1, int* launches) {
  if (!a.no_prune && !a.topk) {   // a single row's bound is no bound for the per-beam Top-K pool
    int r0 = min(a.theta_rows, rows);
    if (r0 > 0) {
      launch_pdl(k_theta<T, VPT>, dim3(a.batch, r0), T, 0, s, a);
      ++*launches;
    }
  }
  if (ev0) cudaEventRecord(ev0, s);
  launch_pdl(k_main<T, VPT>, dim3(a.batch, rows), T, 0, s, a);
  ++*launches;
  if (ev1) cudaEventRecord(ev1, s);
  return cudaGetLastError();
}

// Called once per context: opt the variable-shared-memory kernels into their maximum.
cudaError_t configure_stream_kernels();

cudaError_t configure_kernels(int cap) {
  cudaError_t e = configure_stream_kernels();
  if (e != cudaSuccess) return e;
  const int sel = (int)((cap + 2 * kMaxBW) * sizeof(uint64_t));
  const int spk = (int)((kSparseCap + 2 * kMaxBW) * sizeof(uint64_t));
  if ((e = cudaFuncSetAttribute(k_select<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel)) ||
      (e = cudaFuncSetAttribute(k_select<512, __nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel)) ||
      (e = cudaFuncSetAttribute(k_sparse<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, spk)) ||
      (e = cudaFuncSetAttribute(k_sparse<512, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, spk)) ||
      (e = cudaFuncSetAttribute(k_sparse<512, true, __nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, spk)))
    return e;
  if ((e = cudaFuncSetAttribute(k_sparse<512, false, float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, spk)))
    return e;
  if ((e = cudaFuncSetAttribute(k_sparse<512, false, float, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                spk)))
    return e;
  return cudaFuncSetAttribute(k_sparse<512, false, __nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              spk);
}

bool stream_supported(int V);
cudaError_t launch_stream(const StepArgs& a, int rows, cudaStream_t s, cudaEvent_t ev0,
                          cudaEvent_t ev1, int* launches);

cudaError_t launch_step(const StepArgs& a, int rows, bool sparse_route, int sparse_keys,
                        cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1, int* launches) {
  cudaError_t e;
  const bool bf16 = a.dtype == XGR_DTYPE_BF16;
  if (a.ph_lists && !sparse_route) return launch_paper_heap(a, rows, s, ev0, ev1, launches);
  if (a.mixed) {
    // both routes: k_sparse commits the requests whose next-step candidates fit on chip (decided
    // per request by the previous commit), the dense path the others (it skips the former); the
    // dense path's sparse-parent rows go to k_sparse_rows
    const size_t smem = ((size_t)kSparseCap + 2 * kMaxBW) * sizeof(uint64_t);
    StepArgs as = a;
    as.sparse_cap = kSparseCap;
    if (bf16) launch_pdl(k_sparse<512, false, __nv_bfloat16>, a.batch, 512, smem, s, as);
    else launch_pdl(k_sparse<512, false>, a.batch, 512, smem, s, as);
    ++*launches;
    // the dense path only walks its own requests
    launch_pdl(k_route_list, 1, 1024, 0, s, a, const_cast<int32_t*>(a.dense_list));
    ++*launches;
    if ((e = launch_stream(a, rows, s, ev0, ev1, launches)) != cudaSuccess) return e;
    const dim3 g(a.batch, (rows + 127) / 128);
    if (bf16) launch_pdl(k_sparse_rows<__nv_bfloat16>, g, 128, 0, s, a, rows);
    else launch_pdl(k_sparse_rows<float>, g, 128, 0, s, a, rows);
    const size_t sel = ((size_t)a.cap + 2 * kMaxBW) * sizeof(uint64_t);
    if (bf16) launch_pdl(k_select<512, __nv_bfloat16>, a.batch, 512, sel, s, a);
    else launch_pdl(k_select<512>, a.batch, 512, sel, s, a);
    *launches += 2;
    return cudaGetLastError();
  }
  if (sparse_route) {
    size_t smem = ((size_t)sparse_keys + 2 * kMaxBW) * sizeof(uint64_t);
    if (bf16) {
      if (rows == 1) launch_pdl(k_sparse<512, true, __nv_bfloat16>, a.batch, 512, smem, s, a);
      else launch_pdl(k_sparse<512, false, __nv_bfloat16>, a.batch, 512, smem, s, a);
    } else {
      if (rows == 1) launch_pdl(k_sparse<512, true>, a.batch, 512, smem, s, a);
      else launch_pdl(k_sparse<512, false>, a.batch, 512, smem, s, a);
    }
    ++*launches;
    return cudaGetLastError();
  }
  const int V = a.trie.V;
  if (bf16 && !stream_supported(V)) return cudaErrorNotSupported;   // the API checks this first
  if (stream_supported(V)) {
    e = launch_stream(a, rows, s, ev0, ev1, launches);   // k_seed resets theta/count/ovf
    if (e == cudaSuccess && a.defer_sparse) {   // the sparse-parent rows, one thread each
      const dim3 g(a.batch, (rows + 127) / 128);
      if (bf16) launch_pdl(k_sparse_rows<__nv_bfloat16>, g, 128, 0, s, a, rows);
      else launch_pdl(k_sparse_rows<float>, g, 128, 0, s, a, rows);
      ++*launches;
    }
  } else if ((e = cudaMemsetAsync(a.theta, 0, (size_t)a.batch * 4, s)) != cudaSuccess ||
             (e = cudaMemsetAsync(a.surv_count, 0, (size_t)a.batch * 4, s)) != cudaSuccess ||
             (e = cudaMemsetAsync(a.ovf, 0, (size_t)a.batch * 4, s)) != cudaSuccess) {
    return e;
  } else if (V <= 2048) e = launch_dense<128, 4>(a, rows, s, ev0, ev1, launches);
  else if (V <= 4096) e = launch_dense<256, 4>(a, rows, s, ev0, ev1, launches);
  else if (V <= 8192) e = launch_dense<256, 8>(a, rows, s, ev0, ev1, launches);
  else if (V <= 16384) e = launch_dense<512, 8>(a, rows, s, ev0, ev1, launches);
  else return cudaErrorNotSupported;
  if (e != cudaSuccess) return e;
  const size_t sel = ((size_t)a.cap + 2 * kMaxBW) * sizeof(uint64_t);
  if (bf16) launch_pdl(k_select<512, __nv_bfloat16>, a.batch, 512, sel, s, a);
  else launch_pdl(k_select<512>, a.batch, 512, sel, s, a);
  *launches += 1;
  return cudaGetLastError();
}

// LM-head fusion (NEXT f4): the sparse step over the compact legal logits a.clog written by k_head.
cudaError_t launch_sparse_compact(const StepArgs& a, int sparse_keys, cudaStream_t s, int* launches) {
  const size_t smem = ((size_t)sparse_keys + 2 * kMaxBW) * sizeof(uint64_t);
  launch_pdl(k_sparse<512, false, float, true>, a.batch, 512, smem, s, a);
  ++*launches;
  return cudaGetLastError();
}

bool stream_supported(int V);
cudaError_t launch_shard_stats(const StepArgs& a, int rows, cudaStream_t s);
cudaError_t launch_shard_emit(const StepArgs& a, int rows, cudaStream_t s);

// Codebook shard, select phase: theta seed + emission with the global lse, then this rank's
// local top-BW records (k_select writes records instead of committing when a.rec_out is set).
// Sparse shard step: thread-per-row stats, and the on-chip selection of this rank's candidates.
cudaError_t launch_shard_stats_sparse(const StepArgs& a, int rows, cudaStream_t s) {
  launch_pdl(k_sparse_stats, dim3(a.batch, (rows + 127) / 128), 128, 0, s, a, rows);
  return cudaGetLastError();
}
cudaError_t launch_shard_select_sparse(const StepArgs& a, int sparse_keys, cudaStream_t s) {
  const size_t smem = ((size_t)sparse_keys + 2 * kMaxBW) * sizeof(uint64_t);
  launch_pdl(k_sparse<512, false, float, false, true>, a.batch, 512, smem, s, a);
  return cudaGetLastError();
}

cudaError_t launch_shard_select(const StepArgs& a, int rows, cudaStream_t s, int* launches) {
  cudaError_t e = launch_shard_emit(a, rows, s);
  if (e != cudaSuccess) return e;
  launch_pdl(k_select<512>, a.batch, 512, ((size_t)a.cap + 2 * kMaxBW) * sizeof(uint64_t), s, a);
  *launches += 3;
  return cudaGetLastError();
}

static size_t merge_smem(int nranks, int bw) { return ((size_t)nranks * bw + 2 * kMaxBW) * sizeof(uint64_t); }

// Whether k_merge's shared memory (nranks x BW keys + the selection scratch) fits the device's
// opt-in limit; checked once at init so an oversized shard configuration fails there, not after
// the stats and select phases of a step.
cudaError_t merge_fits(int nranks, int bw, int device, bool* ok) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  if ((e = cudaFuncGetAttributes(&fa, k_merge<512>)) != cudaSuccess) return e;
  *ok = merge_smem(nranks, bw) + fa.sharedSizeBytes <= (size_t)optin;
  return cudaSuccess;
}

cudaError_t launch_shard_merge(const StepArgs& a, const uint64_t* grec, const int32_t* grec_n,
                               cudaStream_t s) {
  const size_t smem = merge_smem(a.nranks, a.BW);
  cudaError_t e = cudaFuncSetAttribute(k_merge<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  launch_pdl(k_merge<512>, a.batch, 512, smem, s, a, grec, grec_n);
  return cudaGetLastError();
}

cudaError_t launch_children(const TrieDev& tr, const int32_t* prefixes, int depth, int64_t n,
                            int32_t* counts, int32_t* tokens, int64_t cap, cudaStream_t s) {
  k_children<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(tr, prefixes, depth, n, counts, tokens, cap);
  return cudaGetLastError();
}

cudaError_t launch_account(const StepArgs& a, int rows, uint32_t* touched, unsigned long long* out,
                           cudaStream_t s) {
  k_account<<<dim3(a.batch, rows), 256, 0, s>>>(a, touched, out);
  return cudaGetLastError();
}

}  // namespace xgr
