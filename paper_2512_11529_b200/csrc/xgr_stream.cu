// Dense-step kernels for sm_100a: the threshold seed and the
// persistent streaming pass.
//
// k_seed (one CTA per request): rows 0..R0-1 of the request -- the best-scored beams, since slot
//   scores are sorted ("the log_prob results for each beam are inherently in
//   descending order") -- are bulk-copied (TMA, cp.async.bulk + mbarrier) into shared memory with
//   their V-bit legal-children masks (L361, L371). Each row's legal-only log-softmax gives its
//   candidate scores c = S_b + (x - lse_b) (L376); a count-verified bisection over the UNION of
//   those candidates finds theta with at least BW candidates >= theta, so theta <= the request's
//   true BW-th best score (the heap minimum of L385 can only be higher). The seed rows' own
//   candidates >= theta are emitted to the survivor buffer.
// k_stream (persistent, warp-specialised): the remaining live rows in b-major order. A producer
//   warp fetches 32 rows' metadata at once, drops rows with S_b < theta before reading them
//   (early termination, L385: every candidate of the row is <= S_b), and issues two bulk copies
//   per remaining dense row into a ring of NS shared-memory stages. CT consumer threads (thread
//   t owns the 32 tokens of mask word t) load the stage into registers (rotated, conflict-free
//   LDS.128), release it, compute m, Z, lse with f32x2 arithmetic and fixed-order reductions,
//   skip the row if UB_b = S_b - ln Z_b < theta, and emit c >= theta with warp-aggregated
//   atomics. Pruning is strict (c < theta dropped), so results never depend on theta
//   (R16).
// Sparse-parent rows inside a dense step are gathered by label from global memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "xgr_internal.cuh"

namespace xgr {

namespace {

constexpr float kLog2eS = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// The same wait with a suspend-time hint: the thread sleeps in hardware until the phase completes
// (or the hint expires) instead of re-polling (NANOSLEEP.SYNCS); for the producer warp, whose
// empty-slot waits otherwise spin for tens of polls per row and steal the consumers' issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Warp max in one instruction (sm_100a redux.sync .f32; NaN inputs are ignored, as by fmaxf).
__device__ __forceinline__ float wmax(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- thread-block cluster helpers (column-split rows, SURVEY 8(e) open question) ----------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// all threads of every CTA of the cluster (release / acquire: orders shared-memory writes)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t local_smem, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f2(uint32_t addr, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
// asynchronous remote store that completes 8 transaction bytes on the receiver's mbarrier
__device__ __forceinline__ void st_async_f2(uint32_t addr, float2 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct Desc {
  int32_t req, b, kind, slot;  // kind: 0 nothing to do, 1 dense row in stage, 2 sparse row
  float S;
  uint32_t node;
  float lse;                   // shard-emit mode: the row's global lse (from all ranks' stats)
};

// k_stream modes: normal step; codebook-shard stats pass (local (m, Z) per row, no emission);
// codebook-shard emit pass (global lse given, no (m, Z) work).
// kModeSeedHist: the histogram seed over rows b < R0 (only those rows are scheduled; no emission):
// each row's candidates >= a row-local bound go to the request's histogram of S_0 - c.
// kModeSeedReq: the same seed with one CTA per request (its R0 seed rows in order): the histogram
// lives in shared memory and the CTA derives theta itself at the end (no global histogram
// atomics, no separate theta kernel).
// kModeFused: the seed and the step in ONE launch. The row sequence is the R0 seed rows of every
// request (request-major, seed work only), then every row (b-major, as kModeNormal). The last of a
// request's seed rows to finish (per-request arrival counter) derives theta from the completed
// histogram and publishes it (a.seed_cnt[req] = kSeedReady, release); a row that needs theta
// before it is published waits for it (acquire), bounded: after ~10 ms it proceeds with no bound
// (theta = -inf is always valid). Every CTA's seed rows precede its other rows, so a waiting CTA
// never holds up a seed row.
constexpr int kModeNormal = 0, kModeStats = 1, kModeShardEmit = 2, kModeSeedHist = 3, kModeSeedReq = 4,
              kModeFused = 5;
constexpr uint32_t kSeedReady = 0x80000000u;   // a.seed_cnt[req]: theta published (fused mode)

// theta of request req once its seed has published it (fused mode; see kModeFused). Lane 0 of the
// calling warp polls; the value is broadcast to the warp.
__device__ __forceinline__ float fused_theta(const StepArgs& a, int req) {
  uint32_t th = 0u;
  if ((threadIdx.x & 31) == 0) {
    for (int n = 0;; ++n) {
      uint32_t f;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.seed_cnt + req) : "memory");
      if (f == kSeedReady) {
        th = __ldcg(a.theta + req);
        break;
      }
      if (n > (1 << 16)) break;   // no bound for this row: always valid (more survivors)
      __nanosleep(128);
    }
  }
  return theta_value(__shfl_sync(0xffffffffu, th, 0));
}

// Consumer-group reductions: warp butterfly, then every consumer thread folds the per-warp
// partials in a fixed order (bitwise-identical, deterministic results in every thread).
template <int CT>
__device__ __forceinline__ float cmax(float v, float* part) {
  v = wmax(v);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  named_sync(1, CT);
  float r = part[0];
#pragma unroll
  for (int i = 1; i < CT / 32; ++i) r = fmaxf(r, part[i]);
  return r;
}
template <int CT>
__device__ __forceinline__ float csum(float v, float* part) {
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  named_sync(1, CT);
  float r = part[0];
#pragma unroll
  for (int i = 1; i < CT / 32; ++i) r += part[i];
  return r;
}
template <int CT>
__device__ __forceinline__ int cisum(int v, int* part) {
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  named_sync(1, CT);
  int r = 0;
#pragma unroll
  for (int i = 0; i < CT / 32; ++i) r += part[i];
  return r;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// k_seed
// ------------------------------------------------------------------------------------------
template <int CTR, int R0, int MODE = kModeNormal>
__global__ void __launch_bounds__(CTR * R0, 1) k_seed(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  constexpr int NT = CTR * R0;
  extern __shared__ __align__(128) float s_dyn[];
  float* s_row = s_dyn;                                                   // [R0][32*CTR]
  uint32_t* s_msk = reinterpret_cast<uint32_t*>(s_dyn + R0 * 32 * CTR);  // [R0][CTR]
  __shared__ __align__(8) uint64_t bar;
  __shared__ int r_kind[R0], r_slot[R0], r_ok[R0];
  __shared__ float r_S[R0], r_lse[R0];
  __shared__ float g_max[NT / 32], g_sum[NT / 32];
  __shared__ float b_red[2][NT / 32];
  __shared__ int b_cnt[2][NT / 32];
  const int tid = threadIdx.x, req = blockIdx.x;
  const int g = tid / CTR, lt = tid - g * CTR, lane = tid & 31;
  const int V = a.trie.V, W = a.trie.W, BW = a.BW;
  const LevelDev& L = a.trie.lv[a.level];
  const int nl = nlive_of(a, req);

  if (tid < R0) {
    int kind = 0, slot = -1;
    float S = 0.f;
    if (tid < nl) {
      uint32_t node;
      row_state(a, req, tid, S, node);
      slot = L.dense_slot ? L.dense_slot[node] : -1;
      kind = slot >= 0 ? 1 : 0;   // sparse seed rows are left to k_stream
      if (MODE == kModeShardEmit && kind) {
        bool fin;
        r_lse[tid] = shard_lse(a, req, tid, fin);
        if (!fin) {
          r_lse[tid] = __int_as_float(0x7fc00000);
          atomicOr(a.flags + req, kFlagNonfinite);
        }
      }
    }
    r_kind[tid] = kind;
    r_slot[tid] = slot;
    r_S[tid] = S;
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    a.surv_count[req] = 0u;   // this step's per-request scratch (read by later kernels only)
    a.ovf[req] = 0u;
  }
  for (int i = tid; i < R0 * CTR; i += NT) s_msk[i] = 0u;
  __syncthreads();
  if (tid == 0) {
    uint32_t bytes = 0;
    const uint32_t rb = (uint32_t)a.Vl * 4u, mb = (uint32_t)(a.Vl >> 5) * 4u;
    for (int r = 0; r < R0; ++r) bytes += r_kind[r] ? rb + mb : 0u;
    if (bytes) {
      mbar_arrive_tx(&bar, bytes);
      const uint64_t pol = policy_evict_first();
      for (int r = 0; r < R0; ++r) {
        if (!r_kind[r]) continue;
        const float* row = static_cast<const float*>(a.logits) + (size_t)req * a.req_stride + (size_t)r * a.ld;
        bulk_g2s(s_row + (size_t)r * 32 * CTR, row, rb, &bar, pol);
        bulk_g2s(s_msk + (size_t)r * CTR, L.bitmap + (size_t)r_slot[r] * W + (a.col0 >> 5), mb, &bar, pol);
      }
    } else {
      mbar_arrive(&bar);
    }
  }
  mbar_wait(&bar, 0);
  if (a.dbg & 32) return;

  int kind = r_kind[g];
  const float S = r_S[g];
  float c[32];
  uint32_t wraw = 0, wm = 0;
  float cmaxv = -INFINITY;
  int nleg = 0;
  if (kind) {
    const float* srow = s_row + (size_t)g * 32 * CTR;
    wraw = s_msk[g * CTR + lt];
    wm = __funnelshift_r(wraw, wraw, 4 * (lt & 7));
    float tmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 x = *reinterpret_cast<const float4*>(srow + 32 * lt + 4 * ((i + lt) & 7));
      c[4 * i + 0] = (wm >> (4 * i + 0)) & 1u ? x.x : -INFINITY;
      c[4 * i + 1] = (wm >> (4 * i + 1)) & 1u ? x.y : -INFINITY;
      c[4 * i + 2] = (wm >> (4 * i + 2)) & 1u ? x.z : -INFINITY;
      c[4 * i + 3] = (wm >> (4 * i + 3)) & 1u ? x.w : -INFINITY;
      tmax = fmaxf(tmax, fmaxf(fmaxf(c[4 * i], c[4 * i + 1]), fmaxf(c[4 * i + 2], c[4 * i + 3])));
    }
    float lse;
    bool finite;
    if (MODE == kModeShardEmit) {
      lse = r_lse[g];
      finite = lse == lse;
    } else {
    // group (= row) reductions on named barrier 1 + g
    float v = wmax(tmax);
    if (lane == 0) g_max[tid >> 5] = v;
    named_sync(1 + g, CTR);
    float M = g_max[g * (CTR / 32)];
#pragma unroll
    for (int i = 1; i < CTR / 32; ++i) M = fmaxf(M, g_max[g * (CTR / 32) + i]);
    const float2 nM = make_float2(-M, -M), l2e = make_float2(kLog2eS, kLog2eS);
    float2 z0 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float2 t = __fmul2_rn(__fadd2_rn(make_float2(c[2 * i], c[2 * i + 1]), nM), l2e);
      z0 = __fadd2_rn(z0, make_float2(ex2f(t.x), ex2f(t.y)));
    }
    v = wsum(z0.x + z0.y);
    if (lane == 0) g_sum[tid >> 5] = v;
    named_sync(1 + g, CTR);
    float Z = g_sum[g * (CTR / 32)];
#pragma unroll
    for (int i = 1; i < CTR / 32; ++i) Z += g_sum[g * (CTR / 32) + i];
    finite = (Z > 0.5f) && (Z <= 3.0e38f);
    lse = row_lse(M, Z);
    }   // MODE != kModeShardEmit
    if (lt == 0) {
      a.lse[(size_t)req * BW + g] = finite ? lse : __int_as_float(0x7fc00000);
      if (!finite) atomicOr(a.flags + req, kFlagNonfinite);
      if (a.counters_on) {
        atomicAdd(a.counters + XGR_CNT_ROWS_READ, 1ull);
      }
    }
    if (finite) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        c[i] = cand_score(S, c[i], lse);   // -inf stays -inf
        cmaxv = fmaxf(cmaxv, c[i]);
      }
      nleg = __popc(wraw);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) c[i] = -INFINITY;
      kind = 0;   // a flagged row emits nothing
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) c[i] = -INFINITY;
  }
  if (lt == 0) r_ok[g] = kind;   // this seed row is dense, live and finite
  if (a.dbg & 64) return;
  if (a.counters_on) {
    int lc = __reduce_add_sync(0xffffffffu, r_kind[g] ? __popc(wraw) : 0);
    if (lane == 0 && lc) atomicAdd(a.counters + XGR_CNT_LEGAL, (unsigned long long)lc);
  }

  // block-wide (union of the seed rows) threshold. Every thread's best candidate cmaxv; each warp
  // sorts its 32 (shuffle bitonic) and takes the m-th largest, m = ceil(BW / warps); the minimum
  // over warps, tau0, has >= BW candidates >= tau0. The candidates >= tau0 (a few hundred) are
  // compacted and the exact BW-th largest among them is theta (>= BW candidates >= theta, so
  // theta <= the request's true BW-th best score).
  auto bmax = [&](float x) {
    x = wmax(x);
    if (lane == 0) b_red[0][tid >> 5] = x;
    __syncthreads();
    float r = b_red[0][0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) r = fmaxf(r, b_red[0][i]);
    return r;
  };
  auto bcnt = [&](int x, int buf) {
    x = __reduce_add_sync(0xffffffffu, x);
    if (lane == 0) b_cnt[buf][tid >> 5] = x;
    __syncthreads();
    int r = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += b_cnt[buf][i];
    return r;
  };
  float lo = -INFINITY;
  const int total = bcnt(nleg, 0);   // (its barrier also publishes r_ok)
  int nrows_ok = 0;
#pragma unroll
  for (int r = 0; r < R0; ++r) nrows_ok += r_ok[r];
  const int nws = nrows_ok * (CTR / 32);   // warps holding a usable seed row
  const int mth = nws ? (BW + nws - 1) / nws : 33;
  if (!a.no_prune && total >= BW && mth <= 32) {
    // warp bitonic sort (descending) of the thread maxima
    float v = cmaxv;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, v, stride);
        const bool keep_max = ((lane & stride) == 0) == ((lane & size) == 0);
        v = keep_max ? fmaxf(v, o) : fminf(v, o);
      }
    }
    const float wmth = kind ? __shfl_sync(0xffffffffu, v, mth - 1) : INFINITY;
    const float tau0 = -bmax(-wmth);   // block min over the usable warps
    if (tau0 > -INFINITY) {
      float* cvals = s_row;            // the rows are in registers now
      if (tid == 0) b_cnt[1][0] = 0;
      __syncthreads();
      // count, warp-scan, one shared atomic per warp, then predicated stores
      int nsel = 0;
      if (cmaxv >= tau0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) nsel += c[i] >= tau0;
      }
      int incl = nsel;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int wbase = 0;
      if (lane == 31 && incl) wbase = atomicAdd(&b_cnt[1][0], incl);
      int p = __shfl_sync(0xffffffffu, wbase, 31) + incl - nsel;
      if (nsel) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (c[i] >= tau0) {
            if (p < 8192) cvals[p] = c[i];
            ++p;
          }
        }
      }
      __syncthreads();
      const int n0 = b_cnt[1][0];
      lo = tau0;
      if (n0 <= 8192 && !(a.dbg & 16)) {
        // exact BW-th largest of the compacted candidates: MSB radix select on orderable bits
        uint32_t* hist = reinterpret_cast<uint32_t*>(s_row + 8192);
        uint32_t prefix = 0u, pmask = 0u;
        int krem = BW;
        for (int shift = 24; shift >= 0; shift -= 8) {
          if (tid < 256) hist[tid] = 0u;
          __syncthreads();
          for (int j = tid; j < n0; j += NT) {
            const uint32_t u = f2o(cvals[j]);
            if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 0xFFu], 1u);
          }
          __syncthreads();
          if (tid < 32) {
            // lane l owns bins 255-8l .. 248-8l; find the digit where the count from the top reaches krem
            uint32_t cc[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              cc[q] = hist[255 - 8 * lane - q];
              sum += cc[q];
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += y;
            }
            const uint32_t excl = incl - sum;
            if (excl < (uint32_t)krem && incl >= (uint32_t)krem) {
              uint32_t acc = excl;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                if (acc + cc[q] >= (uint32_t)krem) {
                  b_cnt[1][1] = 255 - 8 * lane - q;
                  b_cnt[1][2] = (int)acc;
                  break;
                }
                acc += cc[q];
              }
            }
          }
          __syncthreads();
          const uint32_t dgt = (uint32_t)b_cnt[1][1];
          krem -= b_cnt[1][2];
          prefix |= dgt << shift;
          pmask |= 0xFFu << shift;
          __syncthreads();
        }
        lo = o2f(prefix);   // the BW-th largest candidate value (exactly)
      }
    }
  }
  if (tid == 0) a.theta[req] = lo > -INFINITY ? f2o(lo) : 0u;
  // emit the seed rows' candidates >= theta (lo == -inf: every legal candidate). This kernel is
  // the request's first writer this step: a block-wide scan places the keys, no global atomics.
  int ns = 0;
  if (kind && cmaxv >= lo) {
    if (lo > -INFINITY) {
#pragma unroll
      for (int i = 0; i < 32; ++i) ns += c[i] >= lo;   // illegal c are -inf < lo
    } else {
      ns = __popc(wm);
    }
  }
  int incl = ns;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();   // b_cnt[0] may still be read by a slow thread of an earlier reduction
  if (lane == 31) b_cnt[0][tid >> 5] = incl;
  __syncthreads();
  int woff = 0, tot_all = 0;
  for (int w = 0; w < NT / 32; ++w) {
    const int t = b_cnt[0][w];
    woff += w < (tid >> 5) ? t : 0;
    tot_all += t;
  }
  if (tid == 0) a.surv_count[req] = (uint32_t)tot_all;
  if (ns) {
    uint32_t pos = (uint32_t)(woff + incl - ns);
    const uint32_t fbase = (uint32_t)g * (uint32_t)V + (uint32_t)a.col0;
    uint64_t* sbuf = a.surv + (size_t)req * a.cap;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const bool take = lo > -INFINITY ? (c[i] >= lo) : (((wm >> i) & 1u) != 0u);
      if (take) {
        const uint32_t v = 32u * lt + 4u * (((i >> 2) + lt) & 7) + (i & 3);
        if (pos < (uint32_t)a.cap) sbuf[pos] = make_key(c[i], fbase + v);
        ++pos;
      }
    }
  }
  if (a.counters_on) {
    const int tot = __reduce_add_sync(0xffffffffu, ns);
    if (lane == 0 && tot) atomicAdd(a.counters + XGR_CNT_SURVIVORS, (unsigned long long)tot);
  }
}

// ------------------------------------------------------------------------------------------
// Histogram seed (default): theta from the union of rows 0..R0-1 without holding them in one CTA.
// Every candidate of a request is <= S_0 (slot scores are sorted and logp <= 0), so the distances
// d = S_0 - c share one grid across rows: k_seed_hist (one CTA per seed row) adds its row's
// candidates to a per-request histogram of d (bins of 1/128) -- only those >= a row-local bound
// that keeps at least BW of the row's candidates --, and k_seed_theta takes the first bin where the
// count reaches BW: theta = S_0 - (bin + 1) / 128 - margin has >= BW candidates above it, so it is
// <= the request's BW-th best score. The seed rows are then streamed like any other row.
// ------------------------------------------------------------------------------------------
template <int T, int NCH, typename TI = float>
__device__ __forceinline__ void seed_hist_row(const StepArgs& a) {
  constexpr int CH = 16 / (int)sizeof(TI);   // tokens per 16-byte chunk
  constexpr int VPT = NCH * CH / 4;          // x[] holds 4 * VPT = NCH * CH tokens per thread
  constexpr int NW = T / 32;
  __shared__ float2 part[NW];
  __shared__ float s_tau[NW];
  __shared__ uint32_t s_hist[kSeedBins];
  int req = blockIdx.x;
  const int r = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.dense_list) {   // a mixed step: only the dense-route requests, listed
    if ((int)blockIdx.x >= a.dense_list[0]) return;
    req = a.dense_list[1 + blockIdx.x];
  }
  // The row (always in bounds: r < rows) and the beam state are loaded up front and together;
  // only the dense slot and then its bitmap depend on earlier loads.
  const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)r * a.ld;
  const int Vl = a.Vl;
  uint4 v[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int q = i * T + tid;
    v[i] = make_uint4(0u, 0u, 0u, 0u);
    if (CH * q < Vl)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "l"(row + CH * q));
  }
  const int nl = nlive_of(a, req);
  if (r >= nl || req_sparse(a, req)) return;   // before any beam-state read: r < theta_rows may exceed BW
  float S;
  uint32_t node;
  row_state(a, req, r, S, node);
  const float S0 = a.score_in ? a.score_in[(size_t)req * a.BW] : 0.0f;
  const LevelDev& L = a.trie.lv[a.level];
  const int slot = L.dense_slot ? L.dense_slot[node] : -1;
  if (slot < 0) {
    // a sparse seed row adds every candidate to the histogram (all real candidates: the count
    // stays valid); none with a per-beam Top-K cap, and none in the codebook shard
    if (a.topk || a.gstats) return;
    const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
    const uint16_t* lab = a.trie.lv[a.level + 1].label;
    float tm = -INFINITY;
    for (uint32_t q = fc + tid; q < fe; q += T) tm = fmaxf(tm, ldx(row + lab[q]));
    tm = wmax(tm);
    if (lane == 0) part[warp] = make_float2(tm, 0.f);
    __syncthreads();
    float M = part[0].x;
#pragma unroll
    for (int w = 1; w < NW; ++w) M = fmaxf(M, part[w].x);
    float z = 0.f;
    for (uint32_t q = fc + tid; q < fe; q += T) z += ex2f(__fmul_rn(__fsub_rn(ldx(row + lab[q]), M), kLog2eS));
    z = wsum(z);
    __syncthreads();
    if (lane == 0) part[warp].y = z;
    __syncthreads();
    float Z = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) Z += part[w].y;
    if (!((Z > 0.5f) && (Z <= 3.0e38f))) return;
    const float lse = row_lse(M, Z);
    uint32_t* h = a.seed_hist + (size_t)req * kSeedBins;
    for (uint32_t q = fc + tid; q < fe; q += T) {
      const float dd = __fmul_rn(__fsub_rn(S0, cand_score(S, ldx(row + lab[q]), lse)), 128.0f);
      if (dd >= 0.0f && dd < (float)kSeedBins) atomicAdd(h + (int)dd, 1u);
    }
    return;
  }
  const uint32_t* bm = L.bitmap + (size_t)slot * a.trie.W + (a.col0 >> 5);
  float x[4 * VPT];
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int q = i * T + tid;
    const uint32_t nb = (CH * q < Vl) ? (__ldg(bm + ((CH * q) >> 5)) >> ((CH * q) & 31)) & ((1u << CH) - 1u) : 0u;
    float f[CH];
    unpack_chunk<TI>(v[i], f);
#pragma unroll
    for (int j = 0; j < CH; ++j) x[CH * i + j] = ((nb >> j) & 1u) ? f[j] : -INFINITY;
  }
  float lse;
  if (a.gstats) {   // codebook shard: the global lse from all ranks' stats
    bool fin;
    lse = shard_lse(a, req, r, fin);
    if (!fin) return;
  } else {
    float tmax = -INFINITY;
#pragma unroll
    for (int e = 0; e < 4 * VPT; ++e) tmax = fmaxf(tmax, x[e]);
    const float mw = wmax(tmax);
    const float mws = mw == -INFINITY ? 0.f : mw;
    float z = 0.f;
#pragma unroll
    for (int e = 0; e < 4 * VPT; ++e) z += ex2f(__fmul_rn(__fsub_rn(x[e], mws), kLog2eS));
    const float zw = wsum(z);
    if (lane == 0) part[warp] = make_float2(mw, zw);
    __syncthreads();
    float M = part[0].x;
#pragma unroll
    for (int w = 1; w < NW; ++w) M = fmaxf(M, part[w].x);
    float Z = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) Z += part[w].y * ex2f(__fmul_rn(__fsub_rn(part[w].x, M), kLog2eS));
    if (!((Z > 0.5f) && (Z <= 3.0e38f))) return;   // k_stream flags non-finite rows
    lse = row_lse(M, Z);
  }
  float cmax = -INFINITY;
#pragma unroll
  for (int e = 0; e < 4 * VPT; ++e) {
    x[e] = cand_score(S, x[e], lse);
    cmax = fmaxf(cmax, x[e]);
  }
  // row-local bound keeping >= BW candidates: the m-th largest thread max of each warp
  // (m = ceil(BW / warps)), minimised over warps
  const int m = (a.BW + NW - 1) / NW;
  float tau = -INFINITY;
  if (m <= 32) {
    float v = cmax;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, v, stride);
        const bool keep_max = ((lane & stride) == 0) == ((lane & size) == 0);
        v = keep_max ? fmaxf(v, o) : fminf(v, o);
      }
    }
    const float wm = __shfl_sync(0xffffffffu, v, m - 1);
    if (lane == 0) s_tau[warp] = wm;
    __syncthreads();
    tau = s_tau[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) tau = fminf(tau, s_tau[w]);
  }
  // shared-memory histogram first, then one global add per non-empty bin
  for (int i = tid; i < kSeedBins; i += T) s_hist[i] = 0u;
  __syncthreads();
  if (cmax >= tau && cmax > -INFINITY) {
#pragma unroll
    for (int e = 0; e < 4 * VPT; ++e) {
      // -inf (illegal) gives dd = +inf, out of range; tau > -inf here
      const float dd = __fmul_rn(__fsub_rn(S0, x[e]), 128.0f);
      const bool in = x[e] >= tau && dd >= 0.0f && dd < (float)kSeedBins;
      hist_inc_if(in, s_hist, in ? (uint32_t)(int)dd : 0u);
    }
  }
  __syncthreads();
  uint32_t* h = a.seed_hist + (size_t)req * kSeedBins;
  if (a.topk) {
    // per-beam Top-K (NEXT f3): the row contributes only its best K candidates -- the bins in
    // order of d until the count reaches K, the last one partially (counts are all theta needs)
    constexpr int PER = kSeedBins / T;
    uint32_t c[PER], loc = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      c[j] = s_hist[tid * PER + j];
      loc += c[j];
    }
    uint32_t incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();   // s_tau is reused for the warp totals
    if (lane == 31) reinterpret_cast<uint32_t*>(s_tau)[warp] = incl;
    __syncthreads();
    uint32_t before = incl - loc;
    for (int w = 0; w < warp; ++w) before += reinterpret_cast<uint32_t*>(s_tau)[w];
    const uint32_t K = (uint32_t)a.topk;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const uint32_t take = before >= K ? 0u : min(c[j], K - before);
      if (take) atomicAdd(h + tid * PER + j, take);
      before += c[j];
    }
    return;
  }
  for (int i = tid; i < kSeedBins; i += T) {
    const uint32_t v = s_hist[i];
    if (v) atomicAdd(h + i, v);
  }
}

template <int T, int NCH, typename TI = float>
__global__ void __launch_bounds__(T) k_seed_hist(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  seed_hist_row<T, NCH, TI>(a);
}

// theta of request req from its histogram (one CTA of T threads; see k_seed_theta)
template <int T>
__device__ __forceinline__ void seed_theta_req(const StepArgs& a, int req) {
  constexpr int PER = kSeedBins / T;
  __shared__ uint32_t s_w[T / 32];
  __shared__ int s_bin;
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t* h = a.seed_hist + (size_t)req * kSeedBins;
  uint32_t c[PER], loc = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    c[j] = __ldcg(h + tid * PER + j);   // the seed CTAs' atomics live in L2
    loc += c[j];
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) h[tid * PER + j] = 0u;   // ready for the next dense step
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[tid >> 5] = incl;
  if (tid == 0) s_bin = -1;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < (tid >> 5); ++w) off += s_w[w];
  incl += off;
  uint32_t acc = incl - loc;
  const uint32_t need = (uint32_t)(a.no_prune ? 0x7FFFFFFF : a.BW);
  if (acc < need && incl >= need) {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (acc < need && acc + c[j] >= need) s_bin = tid * PER + j;
      acc += c[j];
    }
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t th = 0u;
    if (s_bin >= 0) {
      const float S0 = a.score_in ? a.score_in[(size_t)req * a.BW] : 0.0f;
      const float t = S0 - (float)(s_bin + 1) * (1.0f / 128.0f) - 1e-5f * fmaxf(1.0f, fabsf(S0));
      th = f2o(t);
    }
    a.theta[req] = th;
    a.surv_count[req] = 0u;
    a.ovf[req] = 0u;
  }
}

template <int T>
__global__ void __launch_bounds__(T) k_seed_theta(const __grid_constant__ StepArgs a) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  seed_theta_req<T>(a, blockIdx.x);
}

// The seed and theta in one kernel (XGR_SEED_KERNEL=3): the last of a request's R0 seed CTAs to
// finish (per-request arrival counter, fenced) derives theta from the completed histogram.
template <int T, int NCH, typename TI = float>
__global__ void __launch_bounds__(T) k_seed_hist_theta(const __grid_constant__ StepArgs a) {
  pdl_wait();
  __shared__ int s_last;
  seed_hist_row<T, NCH, TI>(a);
  int req = blockIdx.x;
  if (a.dense_list) {
    if ((int)blockIdx.x >= a.dense_list[0]) return;
    req = a.dense_list[1 + blockIdx.x];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(a.seed_cnt + req, 1u);
    s_last = prev == gridDim.y - 1;
    if (s_last) a.seed_cnt[req] = 0u;   // ready for the next dense step
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  seed_theta_req<T>(a, req);
}

// ------------------------------------------------------------------------------------------
// k_stream: G consumer groups of 256 threads (thread t of a group owns EPT consecutive tokens,
// EPT/32 mask words) process different rows concurrently; one producer warp feeds them.
// ------------------------------------------------------------------------------------------
template <int EPT>
__device__ __forceinline__ uint64_t stage_mask(const uint32_t* msk, int lt) {
  if constexpr (EPT == 32) {
    const uint32_t w = msk[lt];
    return (uint64_t)__funnelshift_r(w, w, 4 * (lt & 7));
  } else {
    const uint64_t m = (uint64_t)msk[2 * lt] | ((uint64_t)msk[2 * lt + 1] << 32);
    const int r = 4 * (lt & 15);
    return r ? (m >> r) | (m << (64 - r)) : m;
  }
}

// Stage ring: NS stages, NSG = NS / G of them owned by each consumer group. Row k goes to group
// g = k % G as that group's j-th row (j = k / G), in stage g + G * (j % NSG), phase j / NSG. A stage
// is only ever used by one group, so a group's parity wait on it cannot be satisfied by a phase
// that belongs to another group's row (a parity wait cannot tell phase n from phase n - 2).
template <int G, int NS>
struct Ring {
  static_assert(NS % G == 0, "each consumer group owns NS / G stages");
  static constexpr int NSG = NS / G;
  __device__ static __forceinline__ int stage(int k) { return (k % G) + G * ((k / G) % NSG); }
  __device__ static __forceinline__ int use(int k) { return (k / G) / NSG; }   // n-th use of the stage
};

// C > 1: a thread-block cluster of C CTAs splits every row by columns (CTA rank r owns the row's
// columns [r V/C, (r+1) V/C)); each computes its slice's (m, Z), the C partials are exchanged through
// distributed shared memory (one mailbox slot and one cluster-scope mbarrier per row) and combined
// in rank order, so every CTA holds the identical row lse; each then emits its own columns. Rows up
// to C x 8192 tokens (V 16384 .. 65536) run on the 8192-column kernel shape.
template <int EPT, int G, int NS, int MINB = 1, int MODE = kModeNormal, typename TI = float, int GT = 256,
          int C = 1>
__global__ void __launch_bounds__(GT * G + 32, MINB) k_stream(const __grid_constant__ StepArgs a, int total,
                                                             int seeded_rows) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  // GT consumer threads per group (256, or 512 for 16384-token rows)
  using R = Ring<G, NS>;
  static_assert(C == 1 || (G == 1 && (MODE == kModeNormal || MODE == kModeSeedHist)), "cluster: one group");
  constexpr bool SEED = MODE == kModeSeedHist || MODE == kModeSeedReq;
  constexpr bool SREQ = MODE == kModeSeedReq;
  constexpr bool FUSED = MODE == kModeFused;   // seed_rows = R0 (seed rows per request)
  constexpr bool EMIT = MODE == kModeNormal || FUSED;
  static_assert(!SREQ || (G == 1 && C == 1), "request-major seed: one group, no cluster");
  static_assert(!FUSED || (G == 1 && C == 1), "fused seed: one group, no cluster");
  __shared__ uint32_t s_hist[SREQ ? kSeedBins : 1];   // request-major seed: this request's histogram
  constexpr int NXS = 4;           // cluster mailbox slots (the CTAs of a cluster are <= 1 row apart)
  __shared__ float2 mbox[NXS][C];
  __shared__ __align__(8) uint64_t xbar[NXS];
  const int crank = C > 1 ? (int)cluster_ctarank() : 0;
  const int ncl = gridDim.x / C, cl = blockIdx.x / C;   // rows w = cl + k * ncl
  const int Vc = a.Vl / C;                              // this CTA's columns [ccol, ccol + Vc)
  const int ccol = a.col0 + crank * Vc;
  constexpr int VT = GT * EPT;     // tokens per stage row
  constexpr int MW = VT / 32;      // mask words per stage
  constexpr int CH = 16 / (int)sizeof(TI);   // tokens per 16-byte chunk (4 fp32, 8 bf16)
  constexpr int NCH = EPT / CH;               // chunks per thread
  constexpr uint32_t CHM = (1u << CH) - 1u;   // a chunk's mask bits
  constexpr int NC = GT * G;       // consumer threads
  // fp32 rows of 32 tokens per thread use the rotated layout (one mask word per thread per row)
#ifdef XGR_NO_ROT   // A/B builds only
  constexpr bool ROT = false;
#else
  constexpr bool ROT = EPT == 32 && sizeof(TI) == 4 && C == 1;   // (clusters: more registers, spills)
#endif
  extern __shared__ __align__(128) unsigned char s_dynb[];
  TI* s_row = reinterpret_cast<TI*>(s_dynb);                                         // [NS][VT]
  uint32_t* s_msk = reinterpret_cast<uint32_t*>(s_dynb + (size_t)NS * VT * sizeof(TI));  // [NS][MW]
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ Desc desc[NS];
  __shared__ float s_th[NS];
  __shared__ float p_max[G][GT / 32], p_sum[G][GT / 32];
  __shared__ float2 part[G][2][GT / 32];
  __shared__ float s_tau[G][GT / 32];

  const int tid = threadIdx.x;
  const int V = a.trie.V;
  const int W = a.trie.W;
  const LevelDev& L = a.trie.lv[a.level];
  const int BW = a.BW;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GT / 32);
    }
    if (C > 1)
      for (int s = 0; s < NXS; ++s) mbar_init(&xbar[s], 1);   // the local expect_tx arrival (+ C x 8 bytes)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < NS * MW; i += NC + 32) s_msk[i] = 0u;
  if (SREQ)
    for (int i = tid; i < kSeedBins; i += NC + 32) s_hist[i] = 0u;
  __syncthreads();
  if (C > 1) cluster_sync_all();   // every mailbox barrier initialised before any remote arrive
  // row k of this CTA: request-major seed: row b = k of request blockIdx.x (total = rows per CTA);
  // otherwise global row w = cl + k * ncl (b-major over the batch)
  // a mixed step streams only its dense-route requests (a.dense_list, built on the device): rows
  // w = b * n_dense + i of request dense_list[1 + i]
  const int ndl = (a.dense_list && !SREQ) ? a.dense_list[0] : a.batch;
  if (a.dense_list && !SREQ) total = ndl * (total / a.batch);
  // fused: rows w < tseed are the seed rows (request i = w / r0f, b = w % r0f), then w - tseed b-major
  const int r0f = FUSED ? min(seeded_rows, total / max(ndl, 1)) : 0;
  const int tseed = ndl * r0f;
  const int tall = total + tseed;
  auto row_ok = [&](int k) { return SREQ ? k < total : cl + k * ncl < tall; };

  if (tid >= NC) {
    // ------------------------------- producer warp ---------------------------------------
    // Lane j holds the metadata of row k0 + j of the current batch of 32. Three batches are in
    // flight: raw loads (nlive, S, node, theta) for batch n+2, the dependent dense_slot load for
    // batch n+1, and the copies of batch n, so no round trip is exposed between batches.
    const int lane = tid & 31;
    const uint64_t pol = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    struct Meta {
      int b, req, live, seed;
      float S, th;
      uint32_t node;
      int slot;
      float lse;
    };
    auto fetch_raw = [&](int k0) {
      Meta m;
      int w = SREQ ? k0 + lane : cl + (k0 + lane) * ncl;
      bool srow = false;   // fused: a seed row
      m.b = 0;
      m.req = 0;
      m.live = 0;
      m.seed = 0;
      m.S = 0.f;
      m.th = -INFINITY;
      m.node = 0;
      m.slot = -1;
      m.lse = 0.f;
      if (w < tall) {
        if (FUSED && w < tseed) {
          srow = true;
          m.req = w / r0f;
          m.b = w - m.req * r0f;
        } else {
          if (FUSED) w -= tseed;
          m.b = SREQ ? w : w / ndl;
          m.req = SREQ ? (int)blockIdx.x : w - m.b * ndl;
        }
        if (a.dense_list && !SREQ) m.req = a.dense_list[1 + m.req];
        const int nl = a.nlive_in ? a.nlive_in[m.req] : 1;
        m.live = m.b < nl && !req_sparse(a, m.req);   // a mixed step's sparse-route requests: k_sparse
        m.seed = srow;
        if (m.live) {
          row_state(a, m.req, m.b, m.S, m.node);
          if (FUSED) {
            if (srow) {
              m.lse = a.score_in ? a.score_in[(size_t)m.req * BW] : 0.0f;   // S_0
            } else if (!(a.dbg & (1 << 25))) {   // theta if already published, else NaN: the consumer waits
              uint32_t f;
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.seed_cnt + m.req) : "memory");
              m.th = f == kSeedReady ? theta_value(__ldcg(a.theta + m.req)) : __int_as_float(0x7fc00000);
            } else {
              m.th = __int_as_float(0x7fc00000);
            }
          } else if (MODE != kModeStats && !SEED) {
            m.th = theta_value(a.theta[m.req]);
          }
          if (SEED) m.lse = a.score_in ? a.score_in[(size_t)m.req * BW] : 0.0f;   // S_0
          if (MODE == kModeShardEmit) {
            bool fin;
            m.lse = shard_lse(a, m.req, m.b, fin);
            if (!fin) {
              m.lse = __int_as_float(0x7fc00000);
              atomicOr(a.flags + m.req, kFlagNonfinite);
            }
          }
        }
      }
      return m;
    };
    auto fetch_slot = [&](Meta& m) {
      if (m.live) m.slot = L.dense_slot ? L.dense_slot[m.node] : -1;
    };
    Meta m0 = fetch_raw(0);
    fetch_slot(m0);
    Meta m1 = fetch_raw(32);
    for (int k0 = 0;; k0 += 32) {
      if (!row_ok(k0)) break;
      Meta m2 = fetch_raw(k0 + 64);
      fetch_slot(m1);
      // decisions for the current batch (its loads completed during the previous batch)
      int kind = 0;
      if (FUSED && m0.seed) {
        // a live seed row always reaches the consumers (it must arrive); a sparse one adds its
        // candidates by label there
        if (m0.live) kind = 4 | (m0.slot >= 0 ? 1 : 2);
      } else if (m0.live && !(MODE == kModeShardEmit && m0.lse != m0.lse)) {
        if (m0.S < m0.th) {   // every candidate of the row is <= S_b < theta: skip unread
          a.lse[(size_t)m0.req * BW + m0.b] = __int_as_float(0x7fc00000);
          if (a.counters_on && crank == 0) atomicAdd(a.counters + XGR_CNT_ROWS_SKIP_PRE, 1ull);
        } else if (FUSED || !(m0.slot >= 0 && m0.b < seeded_rows)) {   // seeded dense rows are done
          kind = m0.slot >= 0 ? 1 : 2;
          // sparse-parent rows: gathered by label by one thread each in k_sparse_rows; in a cluster
          // only rank 0 handles them (the whole row) in the seed pass
          if (kind == 2 && ((EMIT && a.defer_sparse) || crank != 0)) kind = 0;
        }
      }
      // fused: theta of the batch's next row, re-read (acquire) by lane 0 right after issuing the
      // current row when it was not yet published at fetch time (loads complete during the wait)
      float pth = __int_as_float(0x7fc00000);
      for (int j = 0; j < 32; ++j) {
        const int kj = k0 + j;
        if (!row_ok(kj)) break;
        int jkind = __shfl_sync(0xffffffffu, kind, j);
        const int jslot = __shfl_sync(0xffffffffu, m0.slot, j);
        const int jb = __shfl_sync(0xffffffffu, m0.b, j);
        const int jreq = __shfl_sync(0xffffffffu, m0.req, j);
        const float jS = __shfl_sync(0xffffffffu, m0.S, j);
        const float jth = __shfl_sync(0xffffffffu, m0.th, j);
        const uint32_t jnode = __shfl_sync(0xffffffffu, m0.node, j);
        const float jlse = __shfl_sync(0xffffffffu, m0.lse, j);
        int nkind = 0, nreq = 0;
        float nth = 0.f;
        if (FUSED) {
          nkind = __shfl_sync(0xffffffffu, kind, (j + 1) & 31);
          nreq = __shfl_sync(0xffffffffu, m0.req, (j + 1) & 31);
          nth = __shfl_sync(0xffffffffu, m0.th, (j + 1) & 31);
        }
        if (lane == 0) {
          const int st = R::stage(kj), u = R::use(kj);
          if (u > 0) {   // the stage's previous row (same group) has been consumed
            if (a.dbg & 4096) mbar_wait(&empty[st], (u - 1) & 1);
            else mbar_wait_sleep(&empty[st], (u - 1) & 1);
          }
          float jth_use = jth;
          if (FUSED && jth != jth && jkind != 0 && !(jkind & 4)) {
            jth_use = pth;   // NaN if still unpublished: the consumers wait for it
            if (jS < jth_use) {   // now known to be below theta: skip unread
              a.lse[(size_t)jreq * BW + jb] = __int_as_float(0x7fc00000);
              if (a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_SKIP_PRE, 1ull);
              jkind = 0;
            }
          }
          Desc d;
          d.req = jreq;
          d.b = jb;
          d.kind = jkind;
          d.slot = jslot;
          d.S = jS;
          d.node = jnode;
          d.lse = jlse;
          desc[st] = d;
          s_th[st] = jth_use;
          if ((jkind & 3) == 1) {
            const TI* row = static_cast<const TI*>(a.logits) + (size_t)jreq * a.req_stride + (size_t)jb * a.ld +
                            (size_t)crank * Vc;
            const uint32_t rb = (uint32_t)Vc * (uint32_t)sizeof(TI), mb = (uint32_t)(Vc >> 5) * 4u;
            mbar_arrive_tx(&full[st], rb + mb);
            // a fused seed row is read again shortly (its step pass): keep it in L2
            bulk_g2s(s_row + (size_t)st * VT, row, rb, &full[st],
                     (FUSED && (jkind & 4) && !(a.dbg & (1 << 27))) ? pol_keep : pol);
            // a dense node's bitmap is shared by every row whose beam sits on it: keep it in L2
            bulk_g2s(s_msk + (size_t)st * MW, L.bitmap + (size_t)jslot * W + (ccol >> 5), mb, &full[st],
                     pol_keep);
          } else {
            mbar_arrive(&full[st]);
          }
          if (FUSED) {
            pth = __int_as_float(0x7fc00000);
            if (j < 31 && nkind != 0 && !(nkind & 4) && nth != nth && !(a.dbg & (1 << 26))) {
              uint32_t f;
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.seed_cnt + nreq) : "memory");
              if (f == kSeedReady) pth = theta_value(__ldcg(a.theta + nreq));
            }
          }
        }
        __syncwarp();
      }
      m0 = m1;
      m1 = m2;
    }
    if (C > 1) cluster_sync_all();   // no CTA leaves while a peer may still write its mailbox
    return;
  }

  // ------------------------------- consumer groups ----------------------------------------
  const int g = tid / GT, lt = tid - g * GT, lane = tid & 31;
  // column (within this CTA's slice) of this thread's x[e]
  auto tok = [&](int e) -> uint32_t {
    if constexpr (ROT) return 32u * lt + 4u * (uint32_t)(((e >> 2) + lt) & 7) + (uint32_t)(e & 3);
    else return (uint32_t)CH * (uint32_t)((e / CH) * GT + lt) + (uint32_t)(e % CH);
  };
  const int bar_id = 1 + g;
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  float* pmax = p_max[g];
  float* psum = p_sum[g];
  auto gmax = [&](float v) {
    v = wmax(v);
    if (lane == 0) pmax[lt >> 5] = v;
    named_sync(bar_id, GT);
    float r = pmax[0];
#pragma unroll
    for (int i = 1; i < GT / 32; ++i) r = fmaxf(r, pmax[i]);
    return r;
  };
  auto gsum = [&](float v) {
    v = wsum(v);
    if (lane == 0) psum[lt >> 5] = v;
    named_sync(bar_id, GT);
    float r = psum[0];
#pragma unroll
    for (int i = 1; i < GT / 32; ++i) r += psum[i];
    return r;
  };
  // theta of request req from a histogram of d = S_0 - c (bins of 1/128), by this consumer group:
  // the first bin where the count from the top reaches BW; theta = S_0 - (bin + 1)/128 - margin has
  // >= BW candidates above it, so it is <= the request's BW-th best score (as k_seed_theta). A
  // global histogram (fused mode: complete, every seed row arrived) is read from L2 and cleared.
  auto group_theta = [&](uint32_t* h, bool global, int req) {
    named_sync(bar_id, GT);
    constexpr int PER = kSeedBins / GT;
    uint32_t cc[PER], loc = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      cc[j] = global ? __ldcg(h + lt * PER + j) : h[lt * PER + j];
      loc += cc[j];
    }
    if (global) {
#pragma unroll
      for (int j = 0; j < PER; ++j) h[lt * PER + j] = 0u;   // ready for the next dense step
    }
    uint32_t incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t* wtot = reinterpret_cast<uint32_t*>(s_tau[g]);
    int* sbin = reinterpret_cast<int*>(&p_max[g][0]);
    if (lane == 31) wtot[lt >> 5] = incl;
    if (lt == 0) *sbin = -1;
    named_sync(bar_id, GT);
    uint32_t off = 0;
    for (int w2 = 0; w2 < (lt >> 5); ++w2) off += wtot[w2];
    incl += off;
    uint32_t acc = incl - loc;
    const uint32_t need = (uint32_t)(a.no_prune ? 0x7FFFFFFF : a.BW);
    if (acc < need && incl >= need) {
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        if (acc < need && acc + cc[j] >= need) *sbin = lt * PER + j;
        acc += cc[j];
      }
    }
    named_sync(bar_id, GT);
    if (lt == 0) {
      uint32_t th = 0u;
      if (*sbin >= 0) {
        const float S0 = a.score_in ? a.score_in[(size_t)req * a.BW] : 0.0f;
        th = f2o(S0 - (float)(*sbin + 1) * (1.0f / 128.0f) - 1e-5f * fmaxf(1.0f, fabsf(S0)));
      }
      a.theta[req] = th;
      a.surv_count[req] = 0u;
      a.ovf[req] = 0u;
    }
    named_sync(bar_id, GT);   // the scratch (s_tau, p_max) is free again
  };
  int it = 0;   // this group's dense-row count: parity selects the partials buffer
  // Deferred survivor emission: a warp reserves its slots with one atomicAdd whose result is
  // consumed only when the warp next emits (or at the end), so the atomic's round trip overlaps
  // the following rows instead of stalling the group (at most 2 pending keys per lane).
  uint32_t pend_res = 0u, pend_off = 0u;
  int pend_n = 0, pend_req = -1;   // pend_req is warp-uniform; -1: nothing pending
  uint64_t pend_k0 = 0ull, pend_k1 = 0ull;
  auto flush = [&]() {
    if (pend_req >= 0) {
      const uint32_t base = __shfl_sync(0xffffffffu, pend_res, 31) + pend_off;
      uint64_t* sbuf = a.surv + (size_t)pend_req * a.cap;
      if (!(a.dbg & 8)) {
        if (pend_n > 0 && base < (uint32_t)a.cap) sbuf[base] = pend_k0;
        if (pend_n > 1 && base + 1 < (uint32_t)a.cap) sbuf[base + 1] = pend_k1;
      }
      pend_req = -1;
    }
  };
  int xit = 0;   // dense rows exchanged within the cluster (mailbox slot / phase)
  for (int k = g;; k += G) {
    if (!row_ok(k)) break;
    const int st = R::stage(k);
    // consumers wait for their stage with a suspend-time hint (no busy polling that would take
    // issue slots from the other groups of the SM); XGR_DEBUG_FLAGS bit 23: plain polling (A/B)
    if (a.dbg & (1 << 23)) mbar_wait(&full[st], R::use(k) & 1);
    else mbar_wait_sleep(&full[st], R::use(k) & 1);
    // the row descriptor
    Desc d;
    float th;
    if (!(a.dbg & (1 << 21))) {
      // every lane reads it (2% faster than a broadcast, measured). compute-sanitizer racecheck
      // reports this read against the producer's next write of the slot: the warp's reads are
      // ordered before lane 0's release-arrive on the empty barrier by __syncwarp, so it is not a
      // race under the PTX memory model; XGR_DEBUG_FLAGS bit 21 selects the lane-0 broadcast
      // below, which racecheck accepts (tools/sanitize_v16k.py runs both)
      d = desc[st];
      th = s_th[st];
    } else {
      int4 di = make_int4(0, 0, 0, 0);
      float4 df = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lane == 0) {
        const Desc& sd = desc[st];
        di = make_int4(sd.req, sd.b, sd.kind, sd.slot);
        df = make_float4(sd.S, __uint_as_float(sd.node), sd.lse, s_th[st]);
      }
      d.req = __shfl_sync(0xffffffffu, di.x, 0);
      d.b = __shfl_sync(0xffffffffu, di.y, 0);
      d.kind = __shfl_sync(0xffffffffu, di.z, 0);
      d.slot = __shfl_sync(0xffffffffu, di.w, 0);
      d.S = __shfl_sync(0xffffffffu, df.x, 0);
      d.node = __float_as_uint(__shfl_sync(0xffffffffu, df.y, 0));
      d.lse = __shfl_sync(0xffffffffu, df.z, 0);
      th = __shfl_sync(0xffffffffu, df.w, 0);
    }
    const int req = d.req, b = d.b;
    const float S = d.S;
    const bool srow = FUSED && (d.kind & 4);   // fused: a seed row (arrives below)
    const int kind = d.kind & 3;

    do {   // the row; `continue` ends it (then a fused seed row arrives)
    if (kind != 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      // sparse seed rows add every candidate to the histogram (each is a real candidate, so the
      // count stays valid); with a per-beam Top-K cap they add nothing
      if (kind == 0 || (SEED && a.topk)) continue;
      // sparse parent inside a dense step: gather the legal logits by label (rare)
      if (lt == 0 && a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_READ, 1ull);
      const TI* row = static_cast<const TI*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld - a.col0;
      uint32_t fc = L.first_child[d.node], fe = L.first_child[d.node + 1];
      if (a.Vl != V) {   // codebook shard: the children whose token lies in this rank's columns
        uint32_t lo = fc, hi = fe;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (lab[mid] < (uint32_t)a.col0) lo = mid + 1; else hi = mid;
        }
        fc = lo;
        hi = fe;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (lab[mid] < (uint32_t)(a.col0 + a.Vl)) lo = mid + 1; else hi = mid;
        }
        fe = lo;
      }
      float M = 0.f, lse;
      bool finite;
      if (MODE == kModeShardEmit) {
        lse = d.lse;
        finite = true;
        if (lt == 0) a.lse[(size_t)req * BW + b] = lse;
      } else {
        float tm = -INFINITY;
        for (uint32_t q = fc + lt; q < fe; q += GT) tm = fmaxf(tm, ldx(row + lab[q]));
        M = gmax(tm);
        float z = 0.f;
        for (uint32_t q = fc + lt; q < fe; q += GT)
          z += ex2f(__fmul_rn(__fsub_rn(ldx(row + lab[q]), M), kLog2eS));
        const float Z = gsum(z);
        if (MODE == kModeStats) {   // local (m, Z); an empty slice is (-inf, 0)
          if (lt == 0) a.stats_out[(size_t)req * BW + b] = M == -INFINITY ? make_float2(-INFINITY, 0.f) : make_float2(M, Z);
          continue;
        }
        if (SEED || srow) {
          if (!((Z > 0.5f) && (Z <= 3.0e38f))) continue;   // the main pass flags the row
          const float lse2 = row_lse(M, Z), S0 = d.lse;
          uint32_t* h = SREQ ? s_hist : a.seed_hist + (size_t)req * kSeedBins;
          for (uint32_t q = fc + lt; q < fe; q += GT) {
            const float dd = __fmul_rn(__fsub_rn(S0, cand_score(S, ldx(row + lab[q]), lse2)), 128.0f);
            if (dd >= 0.0f && dd < (float)kSeedBins) atomicAdd(h + (int)dd, 1u);
          }
          continue;
        }
        finite = (Z > 0.5f) && (Z <= 3.0e38f);
        lse = row_lse(M, Z);
        if (lt == 0) {
          a.lse[(size_t)req * BW + b] = finite ? lse : __int_as_float(0x7fc00000);
          if (!finite) atomicOr(a.flags + req, kFlagNonfinite);
          if (a.counters_on) atomicAdd(a.counters + XGR_CNT_LEGAL, (unsigned long long)(fe - fc));
        }
      }
      if (!finite) continue;
      if (FUSED && th != th) th = fused_theta(a, req);
      if (EMIT && !(cand_score(S, M, lse) >= th)) continue;
      const uint32_t fbase = (uint32_t)b * (uint32_t)V;
      for (uint32_t q0 = fc; q0 < fe; q0 += GT) {
        const uint32_t q = q0 + lt;
        uint32_t v = 0;
        float c = -INFINITY;
        if (q < fe) {
          v = lab[q];
          c = cand_score(S, ldx(row + v), lse);
        }
        const bool take = q < fe && c >= th;
        if (__any_sync(0xffffffffu, take)) {
          const uint32_t pos = warp_reserve(take ? 1u : 0u, a.surv_count + req);
          if (take && pos < (uint32_t)a.cap) a.surv[(size_t)req * a.cap + pos] = make_key(c, fbase + v);
        }
      }
      continue;
    }

    // ---- dense row: stage -> registers. Thread lt owns the 16-byte chunks q = i*GT + lt
    // (i < NCH; CH tokens each): consecutive per lane, conflict-free, compile-time offsets; its
    // mask bits are CH*(lt % (32/CH)) .. +CH-1 of word q*CH/32 = i*GT*CH/32 + lt/(32/CH).
    const int nsh = CH * (lt & (32 / CH - 1));
    float x[EPT];
    if constexpr (ROT) {
      // thread lt owns tokens [32 lt, 32 lt + 32) (mask word lt, one shared load); its chunk i is
      // the float4 (i + lt) & 7 of that range: within each 8-lane phase of an LDS.128 the lanes hit
      // distinct bank groups
      const float* srow = reinterpret_cast<const float*>(s_row) + (size_t)st * VT + 32 * lt;
      const uint32_t w = s_msk[(size_t)st * MW + lt];
      const uint32_t wrot = __funnelshift_r(w, w, 4 * (lt & 7));   // nibble i: chunk i
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 raw = *reinterpret_cast<const float4*>(srow + 4 * ((i + lt) & 7));
        const uint32_t nb = wrot >> (4 * i);
        x[4 * i + 0] = (nb & 1u) ? raw.x : -INFINITY;
        x[4 * i + 1] = (nb & 2u) ? raw.y : -INFINITY;
        x[4 * i + 2] = (nb & 4u) ? raw.z : -INFINITY;
        x[4 * i + 3] = (nb & 8u) ? raw.w : -INFINITY;
      }
    } else {
      const TI* srow = s_row + (size_t)st * VT + CH * lt;
      const uint32_t* smsk = s_msk + (size_t)st * MW + (lt / (32 / CH));
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const uint4 raw = *reinterpret_cast<const uint4*>(srow + i * GT * CH);
        const uint32_t nb = smsk[i * (GT * CH / 32)] >> nsh;
        float v[CH];
        unpack_chunk<TI>(raw, v);
#pragma unroll
        for (int j = 0; j < CH; ++j) x[CH * i + j] = ((nb >> j) & 1u) ? v[j] : -INFINITY;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);

    float tmax = -INFINITY;
#pragma unroll
    for (int e = 0; e < EPT; e += 4) tmax = fmaxf(tmax, fmaxf(fmaxf(x[e], x[e + 1]), fmaxf(x[e + 2], x[e + 3])));
    float lse;
    if (MODE == kModeShardEmit) {
      lse = d.lse;   // global lse of the row, from all ranks' (m, Z)
      if (lt == 0) a.lse[(size_t)req * BW + b] = lse;   // for the exact overflow fallback
    } else {
    // warp-local (m_w, z_w), one group barrier, then combine the GT/32 pairs
    const float mw = wmax(tmax);
    const float mws = mw == -INFINITY ? 0.0f : mw;
    const float2 nM = make_float2(-mws, -mws);
    const float2 l2e = make_float2(kLog2eS, kLog2eS);
    float2 z0 = make_float2(0.f, 0.f), z1 = make_float2(0.f, 0.f);
    if (!(a.dbg & (1 << 22))) {
      // exponent (x - m) log2 e as one fused x * log2 e - m * log2 e (f32x2): the rounding of m log2 e
      // shifts every term of the row alike, i.e. lse by <= 2^-24 |m| -- far inside R11's bound; a
      // dense row has >= V/16 legal tokens, so R11's exact single-child case never occurs here
      const float cm = -__fmul_rn(mws, kLog2eS);
      const float2 c2 = make_float2(cm, cm);
#pragma unroll
      for (int e = 0; e < EPT; e += 4) {
        const float2 a0 = __ffma2_rn(make_float2(x[e], x[e + 1]), l2e, c2);
        const float2 a1 = __ffma2_rn(make_float2(x[e + 2], x[e + 3]), l2e, c2);
        z0 = __fadd2_rn(z0, make_float2(ex2f(a0.x), ex2f(a0.y)));
        z1 = __fadd2_rn(z1, make_float2(ex2f(a1.x), ex2f(a1.y)));
      }
    } else {   // XGR_DEBUG_FLAGS bit 22: subtract, then multiply (A/B)
#pragma unroll
      for (int e = 0; e < EPT; e += 4) {
        const float2 a0 = __fmul2_rn(__fadd2_rn(make_float2(x[e], x[e + 1]), nM), l2e);
        const float2 a1 = __fmul2_rn(__fadd2_rn(make_float2(x[e + 2], x[e + 3]), nM), l2e);
        z0 = __fadd2_rn(z0, make_float2(ex2f(a0.x), ex2f(a0.y)));
        z1 = __fadd2_rn(z1, make_float2(ex2f(a1.x), ex2f(a1.y)));
      }
    }
    const float2 zz = __fadd2_rn(z0, z1);
    const float zw = wsum(zz.x + zz.y);
    float2* pp = part[g][it & 1];
    if (lane == 0) pp[lt >> 5] = make_float2(mw, zw);
    named_sync(bar_id, GT);
    ++it;
    float2 pr = lane < GT / 32 ? pp[lane] : make_float2(-INFINITY, 0.f);
    float M = wmax(pr.x);   // warp-uniform
    float zi = pr.y * ex2f(__fmul_rn(__fsub_rn(pr.x, M), kLog2eS));
    if (lane >= GT / 32) zi = 0.f;
#pragma unroll
    for (int o = GT / 64; o > 0; o >>= 1) zi += __shfl_xor_sync(0xffffffffu, zi, o);
    float Z = __shfl_sync(0xffffffffu, zi, 0);
    if constexpr (C > 1) {
      // this slice's (m, Z) to every CTA of the cluster (slot xit % NXS), then the C partials
      // combined in rank order: M = max_r m_r, Z = sum_r Z_r 2^((m_r - M) log2 e) -- identical on
      // every rank. An empty slice is (-inf, 0); a NaN partial makes the row non-finite.
      const int xs = xit % NXS;
      if (lt == 0) {
        // this CTA's slot expects one local arrival and C x 8 bytes; every CTA (this one included)
        // delivers its partial with an asynchronous remote store that completes 8 of those bytes
        mbar_arrive_tx(&xbar[xs], 8u * C);
        const float2 mine2 = M == -INFINITY ? make_float2(-INFINITY, 0.f) : make_float2(M, Z);
#pragma unroll 1
        for (int r = 0; r < C; ++r)
          st_async_f2(mapa(smem_u32(&mbox[xs][crank]), (uint32_t)r), mine2, mapa(smem_u32(&xbar[xs]), (uint32_t)r));
      }
      mbar_wait(&xbar[xs], (uint32_t)(xit / NXS) & 1u);
      ++xit;
      // the combine is on every row's critical path: unrolled, loads issued together (the maxima
      // first, then the pairs -- fewer live registers than holding all C pairs through both)
      M = mbox[xs][0].x;
#pragma unroll
      for (int r = 1; r < C; ++r) M = fmaxf(M, mbox[xs][r].x);
      Z = 0.f;
#pragma unroll
      for (int r = 0; r < C; ++r) {
        const float2 q = mbox[xs][r];
        if (q.y > 0.f) Z = __fadd_rn(Z, __fmul_rn(q.y, ex2f(__fmul_rn(__fsub_rn(q.x, M), kLog2eS))));
        else if (q.y != q.y) Z = q.y;
      }
    }
    if (MODE == kModeStats) {   // local (m, Z) of this rank's columns; an empty slice is (-inf, 0)
      if (lt == 0) {
        a.stats_out[(size_t)req * BW + b] = M == -INFINITY ? make_float2(-INFINITY, 0.f) : make_float2(M, Z);
        if (a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_READ, 1ull);
      }
      continue;
    }
    if (SEED || srow) {
      // rows b < R0: candidates >= a row-local bound tau into the request's histogram of S_0 - c
      // (bins of 1/128). tau: each warp's m-th largest (m = ceil(BW / 8) <= 64) of its lanes'
      // top-2 candidates -- distinct elements, so the row has >= BW candidates >= tau.
      if (!((Z > 0.5f) && (Z <= 3.0e38f))) continue;   // the main pass flags the row
      const float lse3 = row_lse(M, Z);
      const float S0 = d.lse;
      const int mm = (BW + GT / 32 - 1) / (GT / 32);
      if (mm <= 32 && !(a.dbg & (1 << 24))) {
        // BW <= GT: each warp's bound is the minimum of its lanes' maxima (over lanes holding a legal
        // token), so every such lane has a candidate >= it; if the row's warps vouch for >= BW
        // candidates this way, count those >= their warp's bound (found by groups of 4 on the raw
        // logits: c is increasing in x). Counting only real candidates keeps theta valid whatever
        // the bound; the bound only limits the atomics. Otherwise the top-2 path below.
        const bool has = tmax > -INFINITY;
        const float wmin = -wmax(has ? -tmax : -INFINITY);
        const int nw = __popc(__ballot_sync(0xffffffffu, has));
        if (lane == 0) p_sum[g][lt >> 5] = __int_as_float(nw);   // (s_tau is the fallback's)
        named_sync(bar_id, GT);
        int tot = 0;
#pragma unroll
        for (int w2 = 0; w2 < GT / 32; ++w2) tot += __float_as_int(p_sum[g][w2]);
        if (tot >= BW) {
          if (has) {
            uint32_t* h = SREQ ? s_hist : a.seed_hist + (size_t)req * kSeedBins;
#pragma unroll
            for (int i = 0; i < EPT / 4; ++i) {
              const float m4 = fmaxf(fmaxf(x[4 * i], x[4 * i + 1]), fmaxf(x[4 * i + 2], x[4 * i + 3]));
              if (m4 >= wmin) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if (x[4 * i + j] >= wmin && x[4 * i + j] > -INFINITY) {
                    const float dd = __fmul_rn(__fsub_rn(S0, cand_score(S, x[4 * i + j], lse3)), 128.0f);
                    if (dd >= 0.0f && dd < (float)kSeedBins) atomicAdd(h + (int)dd, 1u);
                  }
                }
              }
            }
          }
          continue;
        }
      }
      float c1 = -INFINITY, c2 = -INFINITY;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        x[e] = cand_score(S, x[e], lse3);
        c2 = fmaxf(c2, fminf(c1, x[e]));
        c1 = fmaxf(c1, x[e]);
      }
      float tau = -INFINITY;
      if (mm <= 64) {
        float A = c1, B = c2;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
          for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const float oa = __shfl_xor_sync(0xffffffffu, A, stride);
            const float ob = __shfl_xor_sync(0xffffffffu, B, stride);
            const bool keep_max = ((lane & stride) == 0) == ((lane & size) == 0);
            A = keep_max ? fmaxf(A, oa) : fminf(A, oa);
            B = keep_max ? fmaxf(B, ob) : fminf(B, ob);
          }
        }
        float best = -INFINITY;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int i = lane + 32 * hh, j = mm - i;
          const float av = __shfl_sync(0xffffffffu, A, (i - 1) & 31);
          const float bv = __shfl_sync(0xffffffffu, B, (j - 1) & 31);
          if (i <= 32 && j >= 0 && j <= 32) best = fmaxf(best, fminf(i > 0 ? av : INFINITY, j > 0 ? bv : INFINITY));
        }
        best = wmax(best);
        if (lane == 0) s_tau[g][lt >> 5] = best;
        named_sync(bar_id, GT);
        tau = s_tau[g][0];
#pragma unroll
        for (int w2 = 1; w2 < GT / 32; ++w2) tau = fminf(tau, s_tau[g][w2]);
      }
      if (c1 >= tau && c1 > -INFINITY) {
        uint32_t* h = SREQ ? s_hist : a.seed_hist + (size_t)req * kSeedBins;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          if (x[e] >= tau && x[e] > -INFINITY) {
            const float dd = __fmul_rn(__fsub_rn(S0, x[e]), 128.0f);
            if (dd >= 0.0f && dd < (float)kSeedBins) atomicAdd(h + (int)dd, 1u);
          }
        }
      }
      continue;
    }
    const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
    lse = row_lse(M, Z);
    if (lt == 0 && crank == 0) {
      a.lse[(size_t)req * BW + b] = finite ? lse : __int_as_float(0x7fc00000);
      if (!finite) atomicOr(a.flags + req, kFlagNonfinite);
      if (a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_READ, 1ull);
    }
    if (a.counters_on) {
      int lc = 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) lc += x[e] > -INFINITY;
      lc = __reduce_add_sync(0xffffffffu, lc);
      if (lane == 0) atomicAdd(a.counters + XGR_CNT_LEGAL, (unsigned long long)lc);
    }
    if (!finite) continue;
    if (FUSED && th != th) th = fused_theta(a, req);   // not yet published when the row was fetched
    if (!(cand_score(S, M, lse) >= th)) {  // UB_b = S_b - ln Z_b < theta: nothing to emit
      if (lt == 0 && crank == 0 && a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_SKIP_POST, 1ull);
      continue;
    }
    }   // MODE != kModeShardEmit
    // select this thread's candidates (bit e of `mine`), then one atomic per warp reserves slots
    uint64_t mine = 0ull;
    if (th > -INFINITY) {
      // conservative pre-filter on x (the exact test c >= theta follows); illegal x are -inf
      const float xthr = (th - S) + lse - 1e-5f * (fabsf(th) + fabsf(S) + 2.0f * fabsf(lse));
      if (tmax >= xthr) {
#pragma unroll
        for (int i = 0; i < EPT / 4; ++i) {   // gated by groups of 4
          const float m4 = fmaxf(fmaxf(x[4 * i], x[4 * i + 1]), fmaxf(x[4 * i + 2], x[4 * i + 3]));
          if (m4 >= xthr) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int e = 4 * i + j;
              if (x[e] >= xthr && cand_score(S, x[e], lse) >= th) mine |= 1ull << e;
            }
          }
        }
      }
    } else {
      // no bound (pruning off or too few seed candidates): every legal token, -inf logits
      // included, is a candidate; legality re-read from the node's bitmap in global memory
      if constexpr (ROT) {   // this thread's mask word from global memory, rotated like x[]
        const uint32_t w = (32 * lt < Vc) ? __ldg(L.bitmap + (size_t)d.slot * W + (ccol >> 5) + lt) : 0u;
        mine = (uint64_t)__funnelshift_r(w, w, 4 * (lt & 7));
      } else {
        const uint32_t* gm = L.bitmap + (size_t)d.slot * W + (ccol >> 5) + (lt / (32 / CH));
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t q4 = (uint32_t)(i * GT + lt);
          const uint32_t nb = (CH * q4 < (uint32_t)Vc) ? ((__ldg(gm + i * (GT * CH / 32)) >> nsh) & CHM) : 0u;
          mine |= (uint64_t)nb << (CH * i);
        }
      }
    }
    const int ns = __popcll(mine);
    if ((a.dbg & 1) == 0 && __any_sync(0xffffffffu, ns > 0)) {
      flush();
      const uint32_t fbase = (uint32_t)b * (uint32_t)V + (uint32_t)ccol;
      if (EPT > 32 || __any_sync(0xffffffffu, ns > 2)) {
        // many candidates in one lane (weak theta), or 64 tokens per thread (the registers of the
        // deferred reservation): reserve and write synchronously
        uint64_t* sbuf = a.surv + (size_t)req * a.cap;
        uint32_t pos = warp_reserve((uint32_t)ns, a.surv_count + req);
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          if ((mine >> e) & 1ull) {
            const uint32_t v = tok(e);
            if (pos < (uint32_t)a.cap) sbuf[pos] = make_key(cand_score(S, x[e], lse), fbase + v);
            ++pos;
          }
        }
      } else {
        int q = 0;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t nb = (uint32_t)(mine >> (CH * i)) & CHM;
          if (nb) {
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              if ((nb >> j) & 1u) {
                const uint32_t v = tok(CH * i + j);
                const uint64_t key = make_key(cand_score(S, x[CH * i + j], lse), fbase + v);
                if (q == 0) pend_k0 = key; else pend_k1 = key;
                ++q;
              }
            }
          }
        }
        uint32_t incl = (uint32_t)ns;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 31) pend_res = (a.dbg & 2) ? 0u : atomicAdd(a.surv_count + req, total);
        pend_off = incl - (uint32_t)ns;
        pend_n = ns;
        pend_req = req;
      }
    }
    if (a.counters_on) {
      const int tot = __reduce_add_sync(0xffffffffu, ns);
      if (lane == 0 && tot) atomicAdd(a.counters + XGR_CNT_SURVIVORS, (unsigned long long)tot);
    }
    } while (0);
    if constexpr (FUSED) {
      if (srow) {
        // this seed row's histogram adds are done: arrive; the request's last seed row derives and
        // publishes theta (fences: every thread's adds before the arrival, the arrival before the
        // histogram reads, theta before the flag)
        if (!(a.dbg & (1 << 28))) __threadfence();
        named_sync(bar_id, GT);
        int* slast = reinterpret_cast<int*>(&p_sum[g][0]);
        if (lt == 0) {
          if (a.dbg & (1 << 28)) __threadfence();   // cumulative: the group's adds, ordered by the barrier
          const int nl = a.nlive_in ? a.nlive_in[req] : 1;
          const uint32_t prev = atomicAdd(a.seed_cnt + req, 1u);
          *slast = prev + 1 == (uint32_t)min(r0f, nl);
        }
        named_sync(bar_id, GT);
        if (*slast) {
          __threadfence();
          group_theta(a.seed_hist + (size_t)req * kSeedBins, true, req);
          if (lt == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.seed_cnt + req), "r"(kSeedReady) : "memory");
          }
        } else {
          named_sync(bar_id, GT);   // *slast read by every thread before its next reuse
        }
      }
    }
  }
  flush();
  if constexpr (SREQ) group_theta(s_hist, false, (int)blockIdx.x);
  if (C > 1) cluster_sync_all();   // no CTA leaves while a peer may still write its mailbox
}

// ------------------------------------------------------------------------------------------
// k_stream2 (default for V >= 32768 fp32; XGR_STREAM_VARIANT=7 also for V = 16384): rows wider than
// 8192 columns (fp32, V a multiple of 8192) on
// ONE CTA each, in NCK = V / 8192 chunks of 32 KB, two passes per row. Pass 1 streams the chunks
// from HBM (L2 evict_last) and keeps a per-thread online (m, z); the row's (M, Z), lse and the
// upper bound S_b - ln Z_b follow from one group reduction after the last chunk. Pass 2 streams
// the same chunks again -- from L2, the row was just read -- and emits the candidates c >= theta
// (pass 2 of a row whose bound is below theta only releases its stages). No cluster exchange;
// the price is a second, L2-served read of every dense row. Stage uses: pass 1 chunks 0..NCK-1,
// then pass 2 chunks 0..NCK-1 of the same row; a row skipped before reading takes one use.
// ------------------------------------------------------------------------------------------
struct Desc2 {
  int32_t req, b, kind, chunk;   // kind: 0 nothing, 1 pass-1 chunk, 2 pass-2 chunk
  float S, th;
};

template <int NS>
__global__ void __launch_bounds__(256 + 32, 2) k_stream2(const __grid_constant__ StepArgs a, int total) {
  pdl_wait();
  constexpr int GT = 256, VT = 8192, MW = VT / 32;
  extern __shared__ __align__(128) unsigned char s_dynb2[];
  float* s_row = reinterpret_cast<float*>(s_dynb2);                                   // [NS][VT]
  uint32_t* s_msk = reinterpret_cast<uint32_t*>(s_dynb2 + (size_t)NS * VT * 4);       // [NS][MW]
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ Desc2 desc[NS];
  __shared__ float2 part[GT / 32];
  const int tid = threadIdx.x;
  const int V = a.trie.V, W = a.trie.W, BW = a.BW;
  const int NCK = a.Vl / VT;
  const LevelDev& L = a.trie.lv[a.level];
  if (tid == 0) {
    for (int s2 = 0; s2 < NS; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], GT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ndl = a.dense_list ? a.dense_list[0] : a.batch;
  if (a.dense_list) total = ndl * (total / a.batch);

  if (tid >= GT) {
    // ------------------------------- producer warp ---------------------------------------
    const int lane = tid & 31;
    const uint64_t pol_first = policy_evict_first(), pol_keep = policy_evict_last();
    uint32_t u = 0;   // stage uses so far
    auto use = [&](const Desc2& d, const float* src, const uint32_t* msk, bool keep) {
      if (lane == 0) {
        const int st = (int)(u % NS);
        if (u >= (uint32_t)NS) mbar_wait_sleep(&empty[st], ((u / NS) - 1) & 1);
        desc[st] = d;
        if (src) {
          mbar_arrive_tx(&full[st], VT * 4 + MW * 4);
          bulk_g2s(s_row + (size_t)st * VT, src, VT * 4, &full[st], keep ? pol_keep : pol_first);
          bulk_g2s(s_msk + (size_t)st * MW, msk, MW * 4, &full[st], pol_keep);
        } else {
          mbar_arrive(&full[st]);
        }
      }
      ++u;
    };
    for (int k = 0;; ++k) {
      const int w = blockIdx.x + k * gridDim.x;
      if (w >= total) break;
      int b = w / ndl, req = w - b * ndl;
      if (a.dense_list) req = a.dense_list[1 + req];
      // row metadata (lane 0's loads, broadcast)
      int kind = 0, slot = -1;
      float S = 0.f, th = -INFINITY;
      if (lane == 0) {
        const int nl = a.nlive_in ? a.nlive_in[req] : 1;
        if (b < nl && !req_sparse(a, req)) {
          uint32_t node;
          row_state(a, req, b, S, node);
          th = theta_value(a.theta[req]);
          slot = L.dense_slot ? L.dense_slot[node] : -1;
          if (S < th) {   // every candidate of the row is <= S_b < theta: skip unread
            a.lse[(size_t)req * BW + b] = __int_as_float(0x7fc00000);
            if (a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_SKIP_PRE, 1ull);
          } else if (slot >= 0) {
            kind = 1;
          }   // sparse parents: k_sparse_rows
        }
      }
      kind = __shfl_sync(0xffffffffu, kind, 0);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      S = __shfl_sync(0xffffffffu, S, 0);
      th = __shfl_sync(0xffffffffu, th, 0);
      if (!kind) {
        use(Desc2{req, b, 0, 0, S, th}, nullptr, nullptr, false);
        continue;
      }
      const float* row = static_cast<const float*>(a.logits) + (size_t)req * a.req_stride + (size_t)b * a.ld;
      const uint32_t* bm = L.bitmap + (size_t)slot * W + (a.col0 >> 5);
      for (int c = 0; c < NCK; ++c) use(Desc2{req, b, 1, c, S, th}, row + (size_t)c * VT, bm + c * MW, true);
      for (int c = 0; c < NCK; ++c) use(Desc2{req, b, 2, c, S, th}, row + (size_t)c * VT, bm + c * MW, false);
    }
    use(Desc2{0, 0, -1, 0, 0.f, 0.f}, nullptr, nullptr, false);   // end of this CTA's rows
    return;
  }

  // ------------------------------- consumer group -----------------------------------------
  const int lt = tid, lane = tid & 31;
  float tm = -INFINITY, tz = 0.f;   // this thread's running (m, z) over the row's chunks
  float lse = 0.f, M = -INFINITY;
  bool emit = false;
  for (uint32_t u = 0;; ++u) {
    // the consumer walks the same stage uses; the producer marks the end with a use of kind -1
    const int st = (int)(u % NS);
    mbar_wait_sleep(&full[st], (u / NS) & 1);
    const Desc2 d = desc[st];
    if (d.kind <= 0 || (d.kind == 2 && !emit)) {   // nothing to do with this stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (d.kind < 0) break;
      continue;
    }
    const float* srow = s_row + (size_t)st * VT + 32 * lt;
    const uint32_t w = s_msk[(size_t)st * MW + lt];
    const uint32_t wrot = __funnelshift_r(w, w, 4 * (lt & 7));
    float x[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 raw = *reinterpret_cast<const float4*>(srow + 4 * ((i + lt) & 7));
      const uint32_t nb = wrot >> (4 * i);
      x[4 * i + 0] = (nb & 1u) ? raw.x : -INFINITY;
      x[4 * i + 1] = (nb & 2u) ? raw.y : -INFINITY;
      x[4 * i + 2] = (nb & 4u) ? raw.z : -INFINITY;
      x[4 * i + 3] = (nb & 8u) ? raw.w : -INFINITY;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    float cm = -INFINITY;
#pragma unroll
    for (int e = 0; e < 32; e += 4) cm = fmaxf(cm, fmaxf(fmaxf(x[e], x[e + 1]), fmaxf(x[e + 2], x[e + 3])));
    if (d.kind == 1) {
      // pass 1: online (m, z) of this thread's tokens
      if (d.chunk == 0) {
        tm = -INFINITY;
        tz = 0.f;
      }
      const float mn = fmaxf(tm, cm);
      if (mn > -INFINITY) {
        const float c2 = -__fmul_rn(mn, kLog2eS);
        float2 z0 = make_float2(0.f, 0.f), z1 = make_float2(0.f, 0.f);
        const float2 l2e = make_float2(kLog2eS, kLog2eS), cc = make_float2(c2, c2);
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float2 a0 = __ffma2_rn(make_float2(x[e], x[e + 1]), l2e, cc);
          const float2 a1 = __ffma2_rn(make_float2(x[e + 2], x[e + 3]), l2e, cc);
          z0 = __fadd2_rn(z0, make_float2(ex2f(a0.x), ex2f(a0.y)));
          z1 = __fadd2_rn(z1, make_float2(ex2f(a1.x), ex2f(a1.y)));
        }
        const float2 zz = __fadd2_rn(z0, z1);
        const float sc = tm > -INFINITY ? ex2f(__fmul_rn(__fsub_rn(tm, mn), kLog2eS)) : 0.f;
        tz = __fadd_rn(__fmul_rn(tz, sc), zz.x + zz.y);
        tm = mn;
      }
      if (d.chunk == NCK - 1) {
        // the row's (M, Z): warp combine of the threads' (m, z), then the group's warps
        const float mw = wmax(tm);
        float zw = (tm > -INFINITY) ? __fmul_rn(tz, ex2f(__fmul_rn(__fsub_rn(tm, mw), kLog2eS))) : 0.f;
        zw = wsum(zw);
        if (lane == 0) part[lt >> 5] = make_float2(mw, zw);
        named_sync(1, GT);
        const float2 pr = lane < GT / 32 ? part[lane] : make_float2(-INFINITY, 0.f);
        M = wmax(pr.x);
        float zi = (pr.x > -INFINITY) ? pr.y * ex2f(__fmul_rn(__fsub_rn(pr.x, M), kLog2eS)) : 0.f;
        if (lane >= GT / 32) zi = 0.f;
#pragma unroll
        for (int o = GT / 64; o > 0; o >>= 1) zi += __shfl_xor_sync(0xffffffffu, zi, o);
        const float Z = __shfl_sync(0xffffffffu, zi, 0);
        named_sync(1, GT);   // part is rewritten by the next row
        const bool finite = (Z > 0.5f) && (Z <= 3.0e38f);
        lse = row_lse(M, Z);
        if (lt == 0) {
          a.lse[(size_t)d.req * BW + d.b] = finite ? lse : __int_as_float(0x7fc00000);
          if (!finite) atomicOr(a.flags + d.req, kFlagNonfinite);
          if (a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_READ, 1ull);
        }
        emit = finite && cand_score(d.S, M, lse) >= d.th;
        if (finite && !emit && lt == 0 && a.counters_on) atomicAdd(a.counters + XGR_CNT_ROWS_SKIP_POST, 1ull);
      }
      continue;
    }
    // pass 2: candidates of this chunk (rows whose bound is below theta never get here)
    uint32_t mine = 0u;
    if (d.th > -INFINITY) {
      const float xthr = (d.th - d.S) + lse - 1e-5f * (fabsf(d.th) + fabsf(d.S) + 2.0f * fabsf(lse));
      if (cm >= xthr) {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (x[e] >= xthr && cand_score(d.S, x[e], lse) >= d.th) mine |= 1u << e;
      }
    } else {
      mine = wrot;   // no bound: every legal token
    }
    const int ns = __popc(mine);
    if (__any_sync(0xffffffffu, ns > 0)) {
      uint32_t pos = warp_reserve((uint32_t)ns, a.surv_count + d.req);
      uint64_t* sbuf = a.surv + (size_t)d.req * a.cap;
      const uint32_t fbase = (uint32_t)d.b * (uint32_t)V + (uint32_t)a.col0 + (uint32_t)d.chunk * VT;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if ((mine >> e) & 1u) {
          const uint32_t v = 32u * lt + 4u * (uint32_t)(((e >> 2) + lt) & 7) + (uint32_t)(e & 3);
          if (pos < (uint32_t)a.cap) sbuf[pos] = make_key(cand_score(d.S, x[e], lse), fbase + v);
          ++pos;
        }
      }
      if (a.counters_on) {
        const int tot = __reduce_add_sync(0xffffffffu, ns);
        if (lane == 0 && tot) atomicAdd(a.counters + XGR_CNT_SURVIVORS, (unsigned long long)tot);
      }
    }
  }
}

template <int EPT, int NS, typename TI = float, int GT = 256>
static size_t stream_smem() {
  return (size_t)NS * (GT * EPT * sizeof(TI) + GT * EPT / 8);
}

static int g_num_sms = 0;
static int g_stream_variant = 0;   // XGR_STREAM_VARIANT (tuning experiments); 0 = default
static int g_seed_rows = 4;        // XGR_SEED_ROWS: 4 (default) or 2 seed rows per request
static int g_seed_kernel = 1;      // XGR_SEED_KERNEL: 1 k_seed_hist (one CTA per seed row, the row in
                                   // registers) + k_seed_theta (default: 1-2% faster passes at C3 / C2),
                                   // 2 b-major streamed seed (k_stream seed mode) + k_seed_theta,
                                   // 0 request-major seed with theta in the same kernel,
                                   // 3 k_seed_hist_theta, 4 seed + step in one launch (kModeFused)
static int g_seed_mode = 1;        // XGR_SEED_MODE: 1 histogram seed (default), 0 exact union seed (k_seed)

template <typename K>
static cudaError_t opt_in(K k, size_t smem) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Launch with a (C, 1, 1) thread-block cluster (and programmatic stream serialization if enabled).
template <typename... KArgs, typename... Args>
static cudaError_t launch_cl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, int C,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeClusterDimension;
  attr[n].val.clusterDim.x = C;
  attr[n].val.clusterDim.y = 1;
  attr[n].val.clusterDim.z = 1;
  ++n;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Clusters of C CTAs of the column-split streaming kernel that fit on the device at once.
template <typename K>
static int max_clusters(K k, int block, size_t smem, int C) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 148);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 3 * 148 / C;
  }
  return n;
}

// the column-split (cluster) streaming kernels: normal and seed pass, fp32 and bf16
static int g_ncl[2][2][9];   // [dtype bf16][seed mode][C]: clusters per launch

template <int C>
static cudaError_t configure_cluster() {
  using bf = __nv_bfloat16;
  cudaError_t e;
  auto kn = k_stream<32, 1, 2, 3, kModeNormal, float, 256, C>;
  auto ks = k_stream<32, 1, 2, 3, kModeSeedHist, float, 256, C>;
  auto bn = k_stream<32, 1, 4, 3, kModeNormal, bf, 256, C>;
  auto bsd = k_stream<32, 1, 4, 3, kModeSeedHist, bf, 256, C>;
  const size_t sf = stream_smem<32, 2>(), sb = stream_smem<32, 4, bf>();
  if ((e = opt_in(kn, sf)) || (e = opt_in(ks, sf)) || (e = opt_in(bn, sb)) || (e = opt_in(bsd, sb))) return e;
  g_ncl[0][0][C] = max_clusters(kn, 288, sf, C);
  g_ncl[0][1][C] = max_clusters(ks, 288, sf, C);
  g_ncl[1][0][C] = max_clusters(bn, 288, sb, C);
  g_ncl[1][1][C] = max_clusters(bsd, 288, sb, C);
  return cudaSuccess;
}

static int g_ncta2 = 0;   // resident CTAs of k_stream2 (XGR_STREAM_VARIANT=7)

// Rows of V = NCK x 8192 fp32 columns on one CTA each, two passes (k_stream2; the default for
// NCK >= 4); the theta seed is the cluster kernel's seed pass.
template <int C>
static void launch_stream2(const StepArgs& a, int rows, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                           int* launches) {
  const int total = a.batch * rows;
  const int r0 = std::min(a.theta_rows, rows);
  if (r0 > 0) {
    const int ns = a.batch * r0;
    const int ncl = std::min(g_ncl[0][1][C], ns);
    launch_cl(k_stream<32, 1, 2, 3, kModeSeedHist, float, 256, C>, C * ncl, 288, stream_smem<32, 2>(), s, C, a, ns, 0);
    ++*launches;
  }
  launch_pdl(k_seed_theta<256>, a.batch, 256, 0, s, a);
  if (ev0) cudaEventRecord(ev0, s);
  launch_pdl(k_stream2<3>, std::min(total, g_ncta2), 288, (size_t)3 * (8192 * 4 + 1024), s, a, total);
  if (ev1) cudaEventRecord(ev1, s);
  *launches += 2;
}

// Dense step of a row wider than 8192 columns on one GPU: clusters of C CTAs, 8192 columns or fewer
// each (V % (128 C) == 0): histogram seed over R0 rows, theta, the streamed pass.
template <int C>
static void launch_stream_cluster(const StepArgs& a, int rows, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                                  int* launches) {
  using bf = __nv_bfloat16;
  const bool b16 = a.dtype == XGR_DTYPE_BF16;
  const int total = a.batch * rows;
  const int r0 = std::min(a.theta_rows, rows);
  if (r0 > 0) {
    const int ns = a.batch * r0;
    const int ncl = std::min(g_ncl[b16][1][C], ns);
    if (b16) launch_cl(k_stream<32, 1, 4, 3, kModeSeedHist, bf, 256, C>, C * ncl, 288, stream_smem<32, 4, bf>(), s, C, a, ns, 0);
    else launch_cl(k_stream<32, 1, 2, 3, kModeSeedHist, float, 256, C>, C * ncl, 288, stream_smem<32, 2>(), s, C, a, ns, 0);
    ++*launches;
  }
  launch_pdl(k_seed_theta<256>, a.batch, 256, 0, s, a);
  if (ev0) cudaEventRecord(ev0, s);
  const int ncl = std::min(g_ncl[b16][0][C], total);
  if (b16) launch_cl(k_stream<32, 1, 4, 3, kModeNormal, bf, 256, C>, C * ncl, 288, stream_smem<32, 4, bf>(), s, C, a, total, 0);
  else launch_cl(k_stream<32, 1, 2, 3, kModeNormal, float, 256, C>, C * ncl, 288, stream_smem<32, 2>(), s, C, a, total, 0);
  if (ev1) cudaEventRecord(ev1, s);
  *launches += 2;
}

cudaError_t configure_stream_kernels() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  if (const char* v = getenv("XGR_STREAM_VARIANT")) g_stream_variant = atoi(v);
  if ((e = opt_in(k_stream<32, 3, 6>, stream_smem<32, 6>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 2, 3>, stream_smem<32, 2>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 1, 4>, stream_smem<32, 1>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 3, 1, kModeNormal, float, 512>, stream_smem<32, 3, float, 512>())) != cudaSuccess)
    return e;

  if ((e = opt_in(k_stream<32, 1, 4, 1, kModeNormal, __nv_bfloat16, 512>, stream_smem<32, 4, __nv_bfloat16, 512>())) !=
      cudaSuccess)
    return e;
  if ((e = opt_in(k_seed<256, 4>, stream_smem<32, 4>())) != cudaSuccess) return e;
  if ((e = opt_in(k_seed<256, 4, kModeShardEmit>, stream_smem<32, 4>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 2, 3, kModeStats>, stream_smem<32, 2>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 2, 3, kModeShardEmit>, stream_smem<32, 2>())) != cudaSuccess) return e;
  if ((e = opt_in(k_seed<256, 2>, stream_smem<32, 2>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 4, 3, kModeNormal, __nv_bfloat16>, stream_smem<32, 4, __nv_bfloat16>())) != cudaSuccess)
    return e;
  if (const char* v = getenv("XGR_SEED_ROWS")) g_seed_rows = atoi(v);
  if (const char* v = getenv("XGR_SEED_MODE")) g_seed_mode = atoi(v);
  if (const char* v = getenv("XGR_SEED_KERNEL")) g_seed_kernel = atoi(v);
  if ((e = opt_in(k_stream<32, 1, 2, 3, kModeSeedHist>, stream_smem<32, 2>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 2, 3, kModeFused>, stream_smem<32, 2>())) != cudaSuccess) return e;
  if ((e = opt_in(k_stream<32, 1, 3, 2, kModeSeedReq>, stream_smem<32, 3>())) != cudaSuccess) return e;

  if ((e = opt_in(k_stream<32, 1, 4, 2, kModeSeedReq, __nv_bfloat16>, stream_smem<32, 4, __nv_bfloat16>())) !=
      cudaSuccess)
    return e;
  if ((e = opt_in(k_stream<32, 1, 4, 3, kModeSeedHist, __nv_bfloat16>, stream_smem<32, 4, __nv_bfloat16>())) !=
      cudaSuccess)
    return e;
  if ((e = configure_cluster<2>()) || (e = configure_cluster<4>()) || (e = configure_cluster<8>())) return e;
  {
    const size_t sm2 = (size_t)3 * (8192 * 4 + 1024);
    if ((e = opt_in(k_stream2<3>, sm2))) return e;
    int per = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stream2<3>, 288, sm2))) return e;
    g_ncta2 = std::max(1, per) * (g_num_sms > 0 ? g_num_sms : 148);
  }
  return opt_in(k_seed<512, 2>, stream_smem<64, 2>());
}

// Codebook shard phases (V_local = a.Vl columns, <= 8192 per rank in this build).
cudaError_t launch_shard_stats(const StepArgs& a, int rows, cudaStream_t s) {
  const int total = a.batch * rows;
  const int sms = g_num_sms > 0 ? g_num_sms : 148;
  launch_pdl(k_stream<32, 1, 2, 3, kModeStats>, std::min(total, 3 * sms), 256 + 32, stream_smem<32, 2>(), s, a, total, 0);
  return cudaGetLastError();
}

cudaError_t launch_shard_emit(const StepArgs& a, int rows, cudaStream_t s) {
  const int total = a.batch * rows;
  const int sms = g_num_sms > 0 ? g_num_sms : 148;
  launch_pdl(k_seed<256, 4, kModeShardEmit>, a.batch, 1024, stream_smem<32, 4>(), s, a);
  launch_pdl(k_stream<32, 1, 2, 3, kModeShardEmit>, std::min(total, 3 * sms), 256 + 32, stream_smem<32, 2>(), s, a, total, 4);
  return cudaGetLastError();
}

// Cluster size of the column-split streaming kernel for a row of V columns (1: one CTA per row).
static int cluster_of(int V) { return V <= 8192 ? 1 : V <= 16384 ? 2 : V <= 32768 ? 4 : 8; }

// Usable when a row and its mask can be bulk-copied: every CTA's column slice V / C is a multiple
// of 128 (16-byte mask rows), V <= 65536.
bool stream_supported(int V) { return V <= 65536 && V % (128 * cluster_of(V)) == 0; }

// Dense step: seed (theta + rows 0..R0-1), then the streaming pass over the rest. Returns the
// number of kernels launched through *launches; ev0/ev1 bracket the streaming kernel.
cudaError_t launch_stream(const StepArgs& a, int rows, cudaStream_t s, cudaEvent_t ev0,
                          cudaEvent_t ev1, int* launches) {
  const int total = a.batch * rows;
  const int sms = g_num_sms > 0 ? g_num_sms : 148;
  const int grid = std::min(total, sms);
  const int C = cluster_of(a.Vl);
  // fp32 rows of 4+ x 8192 columns: one CTA per row in two passes (k_stream2; C5 one context 3.34 vs
  // 4.72 ms with 8-CTA clusters); 2 x 8192 (C4) keeps the 2-CTA clusters (3.55 vs 4.31 ms).
  // XGR_STREAM_VARIANT=7 forces k_stream2, 8 forces the clusters.
  const bool two_pass = a.dtype == XGR_DTYPE_F32 && !a.topk && a.Vl % 8192 == 0 &&
                        ((C >= 4 && g_stream_variant != 8) || (C > 1 && g_stream_variant == 7));
  if (C > 1 && two_pass) {
    switch (C) {
      case 2: launch_stream2<2>(a, rows, s, ev0, ev1, launches); break;
      case 4: launch_stream2<4>(a, rows, s, ev0, ev1, launches); break;
      default: launch_stream2<8>(a, rows, s, ev0, ev1, launches); break;
    }
    return cudaGetLastError();
  }
  if (C > 2 || (C == 2 && !a.topk && g_stream_variant != 3)) {   // rows wider than 8192: column-split clusters
    switch (C) {
      case 2: launch_stream_cluster<2>(a, rows, s, ev0, ev1, launches); break;
      case 4: launch_stream_cluster<4>(a, rows, s, ev0, ev1, launches); break;
      default: launch_stream_cluster<8>(a, rows, s, ev0, ev1, launches); break;
    }
    return cudaGetLastError();
  }
  if (a.dtype == XGR_DTYPE_BF16) {   // NEXT f1: bf16 rows (half the bytes), histogram seed
    using bf = __nv_bfloat16;
    const int r0 = std::min(a.theta_rows, rows);
    if (a.trie.V <= 8192 && g_seed_kernel == 0 && !a.topk) {   // request-major seed, theta in the same kernel
      launch_pdl(k_stream<32, 1, 4, 2, kModeSeedReq, bf>, a.batch, 256 + 32, stream_smem<32, 4, bf>(), s, a, r0, 0);
      ++*launches;
    } else {
      if (r0 > 0) {
        const int ns = a.batch * r0;
        if (a.trie.V <= 8192 && g_seed_kernel != 1 && !a.topk)
          launch_pdl(k_stream<32, 1, 4, 3, kModeSeedHist, bf>, std::min(ns, 3 * sms), 256 + 32, stream_smem<32, 4, bf>(),
                     s, a, ns, 0);
        else if (a.trie.V <= 8192)
          launch_pdl(k_seed_hist<256, 4, bf>, dim3(a.batch, r0), 256, 0, s, a);
        else launch_pdl(k_seed_hist<256, 8, bf>, dim3(a.batch, r0), 256, 0, s, a);
        ++*launches;
      }
      launch_pdl(k_seed_theta<256>, a.batch, 256, 0, s, a);
    }
    if (ev0) cudaEventRecord(ev0, s);
    if (a.trie.V <= 8192)
      launch_pdl(k_stream<32, 1, 4, 3, kModeNormal, bf>, std::min(total, 3 * sms), 256 + 32, stream_smem<32, 4, bf>(), s,
          a, total, 0);
    else   // 16384-token rows: one 512-thread consumer group per SM, 4 x 32 KB stages
      launch_pdl(k_stream<32, 1, 4, 1, kModeNormal, bf, 512>, std::min(total, sms), 512 + 32,
                 stream_smem<32, 4, bf, 512>(), s, a, total, 0);
    if (ev1) cudaEventRecord(ev1, s);
    *launches += 2;
    return cudaGetLastError();
  }
  if (a.trie.V <= 8192 && g_seed_kernel == 4 && g_seed_mode >= 1 && !a.topk && !a.gstats &&
      std::min(a.theta_rows, rows) > 0) {
    // the seed and the step in one persistent launch (kModeFused)
    const int r0 = std::min(a.theta_rows, rows);
    if (ev0) cudaEventRecord(ev0, s);
    launch_pdl(k_stream<32, 1, 2, 3, kModeFused>, std::min(total + a.batch * r0, 3 * sms), 256 + 32,
               stream_smem<32, 2>(), s, a, total, r0);
    if (ev1) cudaEventRecord(ev1, s);
    *launches += 1;
    return cudaGetLastError();
  }
  if (a.trie.V <= 8192) {
    int seeded = g_seed_rows == 2 ? 2 : 4;
    bool fused_theta = false;
    if ((g_seed_mode >= 1 && g_seed_kernel == 0) && !a.topk) {
      // histogram seed over rows 0..R0-1, one CTA per request, theta in the same kernel; every row
      // is then streamed
      launch_pdl(k_stream<32, 1, 3, 2, kModeSeedReq>, a.batch, 256 + 32, stream_smem<32, 3>(), s, a,
                 std::min(a.theta_rows, rows), 0);
      ++*launches;
      seeded = 0;
    } else if (g_seed_mode >= 1 || a.topk) {   // histogram seed over rows 0..R0-1; every row is then streamed
      const int r0 = std::min(a.theta_rows, rows);
      if (r0 > 0) {
        if (g_seed_kernel == 3 && !a.topk) {   // seed + theta in one kernel (A/B)
          launch_pdl(k_seed_hist_theta<256, 8>, dim3(a.batch, r0), 256, 0, s, a);
          fused_theta = true;
        } else if (g_seed_kernel == 1 || a.topk) {   // one CTA per seed row (XGR_SEED_KERNEL=1; Top-K cap)
          launch_pdl(k_seed_hist<256, 8>, dim3(a.batch, r0), 256, 0, s, a);
        } else {                    // the seed rows streamed by the persistent kernel
          const int ns = a.batch * r0;
          launch_pdl(k_stream<32, 1, 2, 3, kModeSeedHist>, std::min(ns, 3 * sms), 256 + 32, stream_smem<32, 2>(), s, a, ns, 0);
        }
        ++*launches;
      }
      if (!fused_theta) launch_pdl(k_seed_theta<256>, a.batch, 256, 0, s, a);
      seeded = 0;
    } else if (seeded == 2) {
      launch_pdl(k_seed<256, 2>, a.batch, 512, stream_smem<32, 2>(), s, a);
    } else {
      launch_pdl(k_seed<256, 4>, a.batch, 1024, stream_smem<32, 4>(), s, a);
    }
    if (ev0) cudaEventRecord(ev0, s);
    switch (g_stream_variant) {
      case 1:   // one CTA per SM: one producer feeding three consumer groups from a 6-stage ring
        launch_pdl(k_stream<32, 3, 6>, grid, 3 * 256 + 32, stream_smem<32, 6>(), s, a, total, seeded);
        break;
      case 2:
        launch_pdl(k_stream<32, 1, 1, 4>, std::min(total, 4 * sms), 256 + 32, stream_smem<32, 1>(), s, a, total, seeded);
        break;
      default:  // three independent CTAs per SM, each a producer warp + one group, 2 stages
        launch_pdl(k_stream<32, 1, 2, 3>, std::min(total, 3 * sms), 256 + 32, stream_smem<32, 2>(), s, a, total, seeded);
    }
  } else {
    // V in (8192, 16384]: the histogram seed over R0 rows (one CTA per seed row, capped per beam
    // with Top-K), then 64 KB rows streamed by one 512-thread consumer group per SM (3 stages).
    // XGR_SEED_MODE=0 selects the exact two-row union seed (k_seed<512, 2>; weaker thresholds).
    if (g_seed_mode >= 1 || a.topk || a.gstats) {
      const int r0 = std::min(a.theta_rows, rows);
      if (r0 > 0) {
        launch_pdl(k_seed_hist<256, 16>, dim3(a.batch, r0), 256, 0, s, a);
        ++*launches;
      }
      launch_pdl(k_seed_theta<256>, a.batch, 256, 0, s, a);
      if (ev0) cudaEventRecord(ev0, s);
      launch_pdl(k_stream<32, 1, 3, 1, kModeNormal, float, 512>, std::min(total, sms), 512 + 32,
                 stream_smem<32, 3, float, 512>(), s, a, total, 0);
    } else {
      launch_pdl(k_seed<512, 2>, a.batch, 1024, stream_smem<64, 2>(), s, a);
      if (ev0) cudaEventRecord(ev0, s);
      launch_pdl(k_stream<32, 1, 3, 1, kModeNormal, float, 512>, std::min(total, sms), 512 + 32,
                 stream_smem<32, 3, float, 512>(), s, a, total, 2);
    }
  }
  if (ev1) cudaEventRecord(ev1, s);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace xgr
