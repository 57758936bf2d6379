// Staged shared/unshared decode attention (second workload).
//
// PAPER.md L339 (section 5.2): the attention of BW beams that share a prompt is split into a
// shared stage (every beam's queries against the prompt's KV, written once by prefill, L324) and
// an unshared stage (each beam against its own <= ND generated tokens); each stage produces local
// maxima and sums, and an OnlineSoftmax merge gives the output. SPEC.md S:L136-179 fixes the
// partials (m, s, o) and the merge formula.
//
// B200 design:
//  * The shared stage is a dense contraction: for one (request, KV head) the BW x G query rows of
//    the group (G = hq / hkv) all read the same prompt keys, so a 128-row tile of queries runs
//    S = Q K^T and O += P V on the 5th-generation tensor cores (tcgen05.mma, kind::f16, bf16
//    operands in shared memory, fp32 accumulators in TMEM). Every KV tile is loaded once per
//    128 query rows (the shared-prefix reuse of PAPER.md L224's "Ideal" curve) by TMA with the
//    128-byte swizzle the MMA descriptors expect.
//  * Warp roles per CTA (192 threads, 2 CTAs per SM): warp 0 = TMA producers (lane 0: Q once,
//    then a 3-stage K ring whose stages are released right after their S MMA; lane 1: a 2-stage
//    V ring released after the PV MMA), warp 1 = MMA issuer (one thread; S_{j+1} is issued before
//    PV_j so the tensor core overlaps the softmax of tile j), warps 2-5 = softmax / correction /
//    epilogue, thread <-> query row <-> TMEM lane. P is written back to TMEM over its own S tile
//    (packed bf16 pairs) and read by the PV MMA as its A operand (tcgen05.mma with A in TMEM),
//    so P never touches shared memory. Online softmax in the log2 domain with a lazy
//    reference maximum: O (in TMEM) is rescaled only when a tile's maximum exceeds the reference
//    by more than 8 (so p <= 2^8); exact in real arithmetic, the partial is renormalised to the
//    true maximum at the end.
//  * The unshared stage (<= ND keys per beam) and the merge are fused into the epilogue: each
//    softmax thread reads its beam's own K/V rows, forms the unshared logits, merges with the
//    shared statistics and writes the bf16 output row -- no partial round trip
//    through HBM. A partial-output mode returns the shared stage alone.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "xgr_internal.cuh"

namespace xgr {
namespace attn {

constexpr int kD = 128;           // head dim (two 64-element swizzle panels)
constexpr int kBM = 128;          // query rows per CTA (MMA M, TMEM lanes)
constexpr int kBN = 64;           // keys per tile (MMA N of S, K of PV)
constexpr int kThreads = 192;     // producer warp, MMA warp, 4 softmax warps
constexpr uint32_t kQPanel = kBM * 128;        // 16 KB: 128 rows x 64 bf16
constexpr uint32_t kKVPanel = kBN * 128;       // 8 KB: 64 keys x 64 bf16
constexpr uint32_t kOffQ = 0;
constexpr int kKStages = 3;      // K ring (released right after its S MMA)
constexpr int kVStages = 2;      // V ring (released after its PV MMA)
constexpr uint32_t kOffK = kOffQ + 2 * kQPanel;                  // [stage][panel]
constexpr uint32_t kOffV = kOffK + kKStages * 2 * kKVPanel;
constexpr uint32_t kOffBar = kOffV + kVStages * 2 * kKVPanel;   // P lives in TMEM (aliasing S)
constexpr uint32_t kSmem = kOffBar + 256;
constexpr uint32_t kTmemCols = 256;            // S0 [0,64), S1 [64,128), O [128,256)
constexpr float kRescaleThreshold = 8.0f;      // log2 domain

// ---- PTX helpers ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(b),
      "r"(parity)
      : "memory");
}
// mbar_wait that adds the cycles it spent to *acc when acc != nullptr (XGR_ATTN_DBG & 16)
__device__ __forceinline__ void mbar_wait_t(uint32_t b, uint32_t parity, unsigned long long* acc) {
  if (acc) {
    const unsigned long long t0 = clock64();
    mbar_wait(b, parity);
    *acc += clock64() - t0;
  } else {
    mbar_wait(b, parity);
  }
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// UMMA shared-memory descriptor (sm_100): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), base offset 0, layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: D fp32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
// A major [15] (0 = K), B major [16] (1 = MN), N >> 3 [17,23), M >> 4 [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// A operand from TMEM (kind::f16: M rows in the 128 lanes, K-major packed 16-bit pairs).
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define XGR_R32(x) \
  "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]), \
      "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15]), "=r"(x[16]),   \
      "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]),  \
      "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
#define XGR_W32(x)                                                                                            \
  "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]), "r"(x[8]), "r"(x[9]), \
      "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(x[13]), "r"(x[14]), "r"(x[15]), "r"(x[16]), "r"(x[17]),         \
      "r"(x[18]), "r"(x[19]), "r"(x[20]), "r"(x[21]), "r"(x[22]), "r"(x[23]), "r"(x[24]), "r"(x[25]),         \
      "r"(x[26]), "r"(x[27]), "r"(x[28]), "r"(x[29]), "r"(x[30]), "r"(x[31])

// 32 consecutive TMEM columns of this thread's lane (warp-collective).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : XGR_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      XGR_W32(r)
      : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void bf16x8_to_f32(const uint4 u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

struct AttnArgs {
  int n_req, bw, hq, hkv, G, ls, n_unshared;
  float scale;                       // natural-log softmax scale
  const __nv_bfloat16* ku;           // unshared K/V (fused mode)
  const __nv_bfloat16* vu;
  int64_t u_req_stride, u_beam_stride;   // elements
  __nv_bfloat16* out;                // fused: [n_req][bw][hq][d] bf16
  float* lse;                        // fused: optional [n_req][bw][hq]
  float* pm;                         // partial mode: [n_req][bw][hq] m, s and [..][d] o (fp32)
  float* ps;
  float* po;
  int dbg;                           // XGR_ATTN_DBG (development): 1 = P_j written without waiting
                                     // for PV_{j-1} (equal speed), 2 = unshared rows from global
                                     // memory (no staging), 8 = per-thread output stores
                                     // (no TMA store), 16 = per-CTA phase timestamps (printf) with
                                     // per-barrier wait cycles
  int u_stage;                       // fused: unshared K/V rows TMA-staged in the K ring
  int o_tma;                         // fused: output tile written by TMA from the V ring
};

// grid: (ceil(bw*G/128), hkv, n_req); 192 threads; kSmem dynamic shared memory.
template <bool kPartial>
__global__ void __launch_bounds__(kThreads, 2)
    k_attn_shared(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_ku,
                  const __grid_constant__ CUtensorMap tm_vu, const __grid_constant__ CUtensorMap tm_o,
                  const AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int T = (a.ls + kBN - 1) / kBN;
  const uint32_t sb = su32(smem);
  uint64_t ts0 = 0, ts1 = 0, ts2 = 0;   // XGR_ATTN_PROFILE + XGR_ATTN_DBG & 16: phase timestamps
#ifdef XGR_ATTN_PROFILE   // wait cycles per barrier (build with -DXGR_ATTN_PROFILE; costs registers)
  unsigned long long wk = 0, wv = 0, wp = 0, ws = 0, wo = 0;
  const bool tw = (a.dbg & 16) != 0;
#else
  unsigned long long* const wk_ = nullptr;
  constexpr bool tw = false;
#define wk (*wk_)
#define wv (*wk_)
#define wp (*wk_)
#define ws (*wk_)
#define wo (*wk_)
#endif
#ifdef XGR_ATTN_PROFILE
  if (a.dbg & 16) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts0));
#endif
  if (sb & 1023u) __trap();   // the 128-byte swizzle atoms need 1024-byte alignment
  // barriers: Q; K ring full/empty [3]; V ring full/empty [2]; S full [2]; P full [2] (by tile
  // parity: a softmax warp may finish tile j+1 before another has arrived for tile j, and an
  // arrival must never count towards the previous tile's phase); O done; O final
  const uint32_t bar_q = sb + kOffBar, bar_k_full = bar_q + 8, bar_k_empty = bar_q + 32,
                 bar_v_full = bar_q + 56, bar_v_empty = bar_q + 72, bar_s_full = bar_q + 88,
                 bar_p_full = bar_q + 104, bar_o_done = bar_q + 112,
                 bar_o_final = bar_q + 120, bar_u = bar_q + 128;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 192);

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(bar_k_full + 8 * i, 1);
      mbar_init(bar_k_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_v_full + 8 * i, 1);
      mbar_init(bar_v_empty + 8 * i, 1);
      mbar_init(bar_s_full + 8 * i, 1);
    }
    mbar_init(bar_p_full, 128);
    mbar_init(bar_p_full + 32, 128);
    mbar_init(bar_o_done, 1);
    mbar_init(bar_o_final, 1);
    mbar_init(bar_u, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm_q);
    prefetch_map(&tm_k);
    prefetch_map(&tm_v);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producers: lane 0 streams Q then K, lane 1 streams V. A K stage is released by the
    // commit after its S MMA, a V stage after its PV MMA, so K_{j+2} is in flight while tile j's
    // softmax runs. =====
    if (lane == 0) {
      mbar_expect_tx(bar_q, 2 * kQPanel);
      const int b0 = mt * (kBM / a.G);
      tma_load_4d(sb + kOffQ, &tm_q, bar_q, 0, kvh * a.G, b0, req);
      tma_load_4d(sb + kOffQ + kQPanel, &tm_q, bar_q, 64, kvh * a.G, b0, req);
    }
    if (lane < 2) {
      const CUtensorMap* tm = lane == 0 ? &tm_k : &tm_v;
      const uint32_t full0 = lane == 0 ? bar_k_full : bar_v_full;
      const uint32_t empty0 = lane == 0 ? bar_k_empty : bar_v_empty;
      const uint32_t buf0 = sb + (lane == 0 ? kOffK : kOffV);
      const int ns = lane == 0 ? kKStages : kVStages;
      for (int j = 0; j < T; ++j) {
        const int s = j % ns, u = j / ns;
        if (j >= ns) mbar_wait(empty0 + 8 * s, (u + 1) & 1);
        const uint32_t full = full0 + 8 * s, dst = buf0 + s * 2 * kKVPanel;
        mbar_expect_tx(full, 2 * kKVPanel);
        tma_load_4d(dst, tm, full, 0, kvh, j * kBN, req);
        tma_load_4d(dst + kKVPanel, tm, full, 64, kvh, j * kBN, req);
      }
      if (!kPartial && lane == 0 && a.u_stage) {
        // the CTA's beams' own K/V rows (beam-major, then token), one TMA box per 64-dim panel,
        // into the K ring as soon as its last tiles have been consumed by their S MMAs
        for (int j = max(0, T - kKStages); j < T; ++j)
          mbar_wait(bar_k_empty + 8 * (j % kKStages), (j / kKStages) & 1);
        const uint32_t pu = (uint32_t)(kBM / a.G) * a.n_unshared * 128;
        const int b0 = mt * (kBM / a.G);
        mbar_expect_tx(bar_u, 4 * pu);
        tma_load_5d(sb + kOffK, &tm_ku, bar_u, 0, kvh, 0, b0, req);
        tma_load_5d(sb + kOffK + pu, &tm_ku, bar_u, 64, kvh, 0, b0, req);
        tma_load_5d(sb + kOffK + 2 * pu, &tm_vu, bar_u, 0, kvh, 0, b0, req);
        tma_load_5d(sb + kOffK + 3 * pu, &tm_vu, bar_u, 64, kvh, 0, b0, req);
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0 && T > 0) {
      constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0);
      constexpr uint32_t idO = idesc_bf16(kBM, kD, 1);
      mbar_wait(bar_q, 0);
      auto issue_s = [&](int j) {
        const int s = j & 1, ks = j % kKStages;
        mbar_wait_t(bar_k_full + 8 * ks, (j / kKStages) & 1, tw ? &wk : nullptr);
        tc_fence_after();
        const uint32_t kb = sb + kOffK + ks * 2 * kKVPanel;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t p = kk >> 2, off = (kk & 3) * 32;
          const uint64_t da = sdesc(sb + kOffQ + p * kQPanel + off, 16, 1024);
          const uint64_t db = sdesc(kb + p * kKVPanel + off, 16, 1024);
          umma(tmem + s * kBN, da, db, idS, kk > 0);
        }
        umma_commit(bar_s_full + 8 * s);
        umma_commit(bar_k_empty + 8 * ks);
      };
      issue_s(0);
      for (int j = 0; j < T; ++j) {
        if (j + 1 < T) issue_s(j + 1);
        mbar_wait_t(bar_v_full + 8 * (j & 1), (j >> 1) & 1, tw ? &wv : nullptr);
        mbar_wait_t(bar_p_full + 32 * (j & 1), (j >> 1) & 1, tw ? &wp : nullptr);
        tc_fence_after();
        const uint32_t vb = sb + kOffV + (j & 1) * 2 * kKVPanel;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          // A = P_j from TMEM (packed bf16 pairs in the first 32 columns of S buffer j % 2,
          // 8 columns per 16 keys); B = V tile, MN-major: 64-element d panels at LBO = 8 KB,
          // 8-key groups at SBO = 1 KB, 16 keys per MMA = 2 KB.
          const uint64_t db = sdesc(vb + kk * 2048, kKVPanel, 1024);
          umma_ts(tmem + 2 * kBN, tmem + (j & 1) * kBN + kk * 8, db, idO, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(bar_o_done);
        umma_commit(bar_v_empty + 8 * (j & 1));
      }
      umma_commit(bar_o_final);   // a one-phase barrier: the epilogue may skip o_done phases
    }
  } else {
    // ===== softmax / correction / epilogue: thread <-> query row <-> TMEM lane =====
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                       // row in the tile
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const float c2 = a.scale * 1.4426950408889634f;     // logits -> log2 domain
    float m_ref = -INFINITY;   // reference maximum (log2 domain) that O and l are relative to
    float raw_max = -INFINITY; // true maximum of the raw dot products
    float l = 0.f;
    const int bl = r / a.G, g = r % a.G;
    const int b = mt * (kBM / a.G) + bl;
    const bool row_ok = b < a.bw;
    const int h = kvh * a.G + g;
    const int64_t qrow = (((int64_t)req * a.bw + b) * a.hq + h);
    constexpr int kMaxU = 8;
    const int nu = kPartial ? 0 : a.n_unshared;
    float tu[kMaxU];   // unshared logits (log2 domain), computed while the first S tile is in flight
#pragma unroll
    for (int t = 0; t < kMaxU; ++t) tu[t] = -INFINITY;
    if (!kPartial && nu > 0 && !a.u_stage) {
      mbar_wait(bar_q, 0);
      if (row_ok) {
        const __nv_bfloat16* kub = a.ku + (int64_t)req * a.u_req_stride + (int64_t)b * a.u_beam_stride;
#pragma unroll 1
        for (int t = 0; t < nu; ++t) {
          const uint4* kr = reinterpret_cast<const uint4*>(kub + ((int64_t)t * a.hkv + kvh) * kD);
          uint4 kv[16];
#pragma unroll
          for (int ch = 0; ch < 16; ++ch) kv[ch] = __ldg(kr + ch);
          float dot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ch = 0; ch < 16; ++ch) {
            const uint4 qv = *reinterpret_cast<const uint4*>(smem + kOffQ + (ch >> 3) * kQPanel + r * 128 +
                                                             (((ch & 7) ^ (r & 7)) << 4));
            float qf[8], kf[8];
            bf16x8_to_f32(qv, qf);
            bf16x8_to_f32(kv[ch], kf);
#pragma unroll
            for (int e = 0; e < 8; ++e) dot[ch & 3] = fmaf(qf[e], kf[e], dot[ch & 3]);
          }
#pragma unroll
          for (int u = 0; u < kMaxU; ++u)
            if (u == t) tu[u] = ((dot[0] + dot[1]) + (dot[2] + dot[3])) * c2;
        }
      }
    }
#ifdef XGR_ATTN_PROFILE
    if (a.dbg & 16) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts1));
#endif
    for (int j = 0; j < T; ++j) {
      const int s = j & 1;
      mbar_wait_t(bar_s_full + 8 * s, (j >> 1) & 1, tw ? &ws : nullptr);
      tc_fence_after();
      uint32_t u0[32], u1[32];
      tmem_ld32(tmem + lane_base + s * kBN, u0);
      tmem_ld32(tmem + lane_base + s * kBN + 32, u1);
      tmem_wait_ld();
      const int valid = a.ls - j * kBN;
      float x[64];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        x[c] = __uint_as_float(u0[c]);
        x[c + 32] = __uint_as_float(u1[c]);
      }
      if (valid < kBN) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c >= valid) x[c] = -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mx[c] = fmaxf(fmaxf(fmaxf(x[c], x[c + 8]), fmaxf(x[c + 16], x[c + 24])),
                                               fmaxf(fmaxf(x[c + 32], x[c + 40]), fmaxf(x[c + 48], x[c + 56])));
      const float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      raw_max = fmaxf(raw_max, tmax);
      const float t2 = tmax * c2;
      float alpha = 1.f;
      const bool resc = t2 > m_ref + kRescaleThreshold;
      if (resc) {
        alpha = ex2(m_ref - t2);   // m_ref = -inf -> 0
        m_ref = t2;
        l *= alpha;
      }
      uint32_t pk[32];
      float ls4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float p0 = ex2(fmaf(x[2 * c], c2, -m_ref));
        const float p1 = ex2(fmaf(x[2 * c + 1], c2, -m_ref));
        ls4[c & 3] += p0 + p1;
        pk[c] = pack_bf16(p0, p1);
      }
      l += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
      // P_j -> TMEM over S_j (the PV MMA reads it as its A operand); the S buffer is rewritten
      // only by S_{j+2}, issued after PV_j
      const bool lazy = (a.dbg & 1) != 0;
      if (j > 0 && !lazy) {
        // PV_{j-1} done before P_j is written and before O is rescaled
        mbar_wait_t(bar_o_done, (j - 1) & 1, tw ? &wo : nullptr);
        tc_fence_after();
      }
      tmem_st32(tmem + lane_base + s * kBN, pk);
      if (j > 0 && lazy && __any_sync(0xffffffffu, resc)) {
        // only O needs PV_{j-1}; P_j's buffer was last read by PV_{j-2}, complete before S_j
        mbar_wait_t(bar_o_done, (j - 1) & 1, tw ? &wo : nullptr);
        tc_fence_after();
      }
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_base + 2 * kBN + 32 * k, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          tmem_st32(tmem + lane_base + 2 * kBN + 32 * k, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p_full + 32 * (j & 1));
    }
    if (T > 0) {
      mbar_wait(bar_o_final, 0);
      tc_fence_after();
    }
#ifdef XGR_ATTN_PROFILE
    if (a.dbg & 16) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts2));
#endif
    // ---- epilogue ----
    const float t_true = raw_max * c2;
    if constexpr (kPartial) {
      const float f = (T > 0) ? ex2(m_ref - t_true) : 0.f;   // renormalise to the true maximum
      if (row_ok) {
        a.pm[qrow] = (T > 0) ? raw_max * a.scale : -INFINITY;
        a.ps[qrow] = l * f;
      }
#pragma unroll 1
      for (int k = 0; k < 4; ++k) {
        uint32_t o[32];
        if (T > 0) {
          tmem_ld32(tmem + lane_base + 2 * kBN + 32 * k, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = 0u;
        }
        if (row_ok) {
          float4* dst = reinterpret_cast<float4*>(a.po + qrow * kD + 32 * k);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            dst[c] = make_float4(__uint_as_float(o[4 * c]) * f, __uint_as_float(o[4 * c + 1]) * f,
                                 __uint_as_float(o[4 * c + 2]) * f, __uint_as_float(o[4 * c + 3]) * f);
        }
      }
    } else {
      // merge with the unshared stage (beam b's own tokens t < n_unshared)
      const uint32_t pu = (uint32_t)(kBM / a.G) * nu * 128;   // staged panel bytes
      auto urow = [&](int panel, int t, int ch) -> uint4 {     // staged unshared row (bl, t), 16-B chunk
        const int R = bl * nu + t;
        return *reinterpret_cast<const uint4*>(smem + kOffK + panel * pu + R * 128 + (((ch & 7) ^ (R & 7)) << 4));
      };
      if (a.u_stage) {
        mbar_wait(bar_u, 0);
        if (row_ok) {
#pragma unroll 1
          for (int t = 0; t < nu; ++t) {
            float dot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int ch = 0; ch < 16; ++ch) {
              const uint4 qv = *reinterpret_cast<const uint4*>(smem + kOffQ + (ch >> 3) * kQPanel + r * 128 +
                                                               (((ch & 7) ^ (r & 7)) << 4));
              float qf[8], kf[8];
              bf16x8_to_f32(qv, qf);
              bf16x8_to_f32(urow(ch >> 3, t, ch), kf);
#pragma unroll
              for (int e = 0; e < 8; ++e) dot[ch & 3] = fmaf(qf[e], kf[e], dot[ch & 3]);
            }
#pragma unroll
            for (int u = 0; u < kMaxU; ++u)
              if (u == t) tu[u] = ((dot[0] + dot[1]) + (dot[2] + dot[3])) * c2;
          }
        }
      }
      float m_tot = (T > 0) ? m_ref : -INFINITY;
      if (row_ok) {
#pragma unroll
        for (int t = 0; t < kMaxU; ++t) m_tot = fmaxf(m_tot, tu[t]);
      }
      const __nv_bfloat16* vub = a.vu + (int64_t)req * a.u_req_stride + (int64_t)b * a.u_beam_stride;
      const float w_sh = (T > 0) ? ex2(m_ref - m_tot) : 0.f;
      float den = l * w_sh;
      float wu[kMaxU];
#pragma unroll
      for (int t = 0; t < kMaxU; ++t) {
        wu[t] = (row_ok && t < nu) ? ex2(tu[t] - m_tot) : 0.f;
        den += wu[t];
      }
      const float inv = 1.f / den;
#pragma unroll 1
      for (int k = 0; k < 4; ++k) {
        uint32_t o[32];
        if (T > 0) {
          tmem_ld32(tmem + lane_base + 2 * kBN + 32 * k, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = 0u;
        }
        float acc[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = __uint_as_float(o[c]) * w_sh;
        if (row_ok) {
#pragma unroll
          for (int t = 0; t < kMaxU; ++t) {
            if (t < nu) {
              const uint4* vr = reinterpret_cast<const uint4*>(vub + ((int64_t)t * a.hkv + kvh) * kD + 32 * k);
#pragma unroll
              for (int ch = 0; ch < 4; ++ch) {
                float vf[8];
                bf16x8_to_f32(a.u_stage ? urow(2 + (k >> 1), t, (k & 1) * 4 + ch) : __ldg(vr + ch), vf);
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[8 * ch + e] = fmaf(wu[t], vf[e], acc[8 * ch + e]);
              }
            }
          }
        }
        uint4 pk4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          pk4[c] = make_uint4(pack_bf16(acc[8 * c] * inv, acc[8 * c + 1] * inv),
                              pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv),
                              pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv),
                              pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv));
        if (a.o_tma) {
          // the output tile in the V ring (free: every PV MMA is complete), in the swizzled layout
          // of the output tensor map's box (row r, 64-dim panels)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ch = (k & 1) * 4 + c;
            *reinterpret_cast<uint4*>(smem + kOffV + (k >> 1) * kQPanel + r * 128 + ((ch ^ (r & 7)) << 4)) = pk4[c];
          }
        } else if (row_ok) {
          uint4* dst = reinterpret_cast<uint4*>(a.out + qrow * kD + 32 * k);
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[c] = pk4[c];
        }
      }
      if (a.o_tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");   // the 4 softmax warps
        if (r == 0) {
          tma_store_4d(&tm_o, sb + kOffV, 0, kvh * a.G, mt * (kBM / a.G), req);
          tma_store_4d(&tm_o, sb + kOffV + kQPanel, 64, kvh * a.G, mt * (kBM / a.G), req);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem read before exit
        }
      }
      if (row_ok && a.lse) a.lse[qrow] = (m_tot + __log2f(den)) * 0.6931471805599453f;
    }
  }
#ifdef XGR_ATTN_PROFILE
  if (tw && (threadIdx.x == 32 || threadIdx.x == 64) && (blockIdx.x * 7 + blockIdx.y * 3 + blockIdx.z) % 37 == 0)
    printf("ATTNW cta %d %d %d thr %d k %llu v %llu p %llu s %llu o %llu\n", blockIdx.x, blockIdx.y, blockIdx.z,
           threadIdx.x, wk, wv, wp, ws, wo);
#else
#undef wk
#undef wv
#undef wp
#undef ws
#undef wo
#endif
#ifdef XGR_ATTN_PROFILE
  if ((a.dbg & 16) && threadIdx.x == 64 && (blockIdx.x * 7 + blockIdx.y * 3 + blockIdx.z) % 37 == 0) {
    uint64_t ts3;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts3));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("ATTNTS cta %d %d %d sm %u start %llu pre %llu loop %llu epi %llu\n", blockIdx.x, blockIdx.y, blockIdx.z, smid,
           (unsigned long long)ts0, (unsigned long long)(ts1 - ts0), (unsigned long long)(ts2 - ts1),
           (unsigned long long)(ts3 - ts2));
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ---- two Q tiles per CTA (fused mode) -------------------------------------------------------
// One CTA per SM (224 KB of shared memory, all 512 TMEM columns) holds two 128-row query tiles A and
// B of the same (request, KV head) and streams 128-key K/V tiles once for both. TMEM: S_A [0,128),
// O_A [128,256), S_B [256,384), O_B [384,512); P overwrites the first 64 columns of its S tile
// (packed bf16). The MMA issue order PV_A(j), S_A(j+1), PV_B(j), S_B(j+1) staggers the two tiles:
// softmax A(j+1) runs while the tensor core does PV_B(j) and S_B(j+1), and vice versa. S_t(j)
// complete implies PV_t(j-1) complete (issued before it, tracked by the same commit), so neither
// the P write nor the O correction waits for a PV barrier.
namespace pair {
constexpr int kBN = 128;
constexpr int kThreads = 320;                   // producer, MMA, 4 softmax warps per tile
constexpr uint32_t kQPanel = 128 * 128;         // 16 KB (128 rows x 64 dims)
constexpr uint32_t kKVPanel = kBN * 128;        // 16 KB (128 keys x 64 dims)
constexpr int kKStages = 3, kVStages = 2;
constexpr uint32_t kOffQ = 0;                             // [tile][panel]
constexpr uint32_t kOffK = 4 * kQPanel;                   // [stage][panel]
constexpr uint32_t kOffV = kOffK + kKStages * 2 * kKVPanel;
constexpr uint32_t kOffBar = kOffV + kVStages * 2 * kKVPanel;
constexpr uint32_t kSmem = kOffBar + 256;
}  // namespace pair

__global__ void __launch_bounds__(pair::kThreads, 1)
    k_attn_pair(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_ku,
                const __grid_constant__ CUtensorMap tm_vu, const __grid_constant__ CUtensorMap tm_o,
                const AttnArgs a) {
  constexpr int kBN = pair::kBN;
  constexpr uint32_t kQPanel = pair::kQPanel, kKVPanel = pair::kKVPanel;
  constexpr int kKStages = pair::kKStages, kVStages = pair::kVStages;
  constexpr uint32_t kOffQ = pair::kOffQ, kOffK = pair::kOffK, kOffV = pair::kOffV, kOffBar = pair::kOffBar;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mp = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int T = (a.ls + kBN - 1) / kBN;
  const int nb = 128 / a.G;                     // beams per tile
  const uint32_t sb = su32(smem);
  if (sb & 1023u) __trap();
  // barriers: Q; K full/empty [3]; V full/empty [2]; S full [tile]; P full [tile][parity];
  // O final; unshared rows
  const uint32_t bar_q = sb + kOffBar, bar_k_full = bar_q + 8, bar_k_empty = bar_q + 32,
                 bar_v_full = bar_q + 56, bar_v_empty = bar_q + 72, bar_s_full = bar_q + 88,
                 bar_p_full = bar_q + 104, bar_o_final = bar_q + 136, bar_u = bar_q + 144;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 192);
  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(bar_k_full + 8 * i, 1);
      mbar_init(bar_k_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_v_full + 8 * i, 1);
      mbar_init(bar_v_empty + 8 * i, 1);
      mbar_init(bar_s_full + 8 * i, 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(bar_p_full + 8 * i, 128);
    mbar_init(bar_o_final, 1);
    mbar_init(bar_u, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm_q);
    prefetch_map(&tm_k);
    prefetch_map(&tm_v);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nu = a.n_unshared;

  if (warp == 0) {
    // ===== TMA producers: lane 0 Q (both tiles) + K ring (+ the unshared rows at the end);
    // lane 1 V ring =====
    if (lane == 0) {
      mbar_expect_tx(bar_q, 4 * kQPanel);
      for (int t = 0; t < 2; ++t) {
        const int b0 = (2 * mp + t) * nb;
        tma_load_4d(sb + kOffQ + (2 * t) * kQPanel, &tm_q, bar_q, 0, kvh * a.G, b0, req);
        tma_load_4d(sb + kOffQ + (2 * t + 1) * kQPanel, &tm_q, bar_q, 64, kvh * a.G, b0, req);
      }
    }
    if (lane < 2) {
      const CUtensorMap* tm = lane == 0 ? &tm_k : &tm_v;
      const uint32_t full0 = lane == 0 ? bar_k_full : bar_v_full;
      const uint32_t empty0 = lane == 0 ? bar_k_empty : bar_v_empty;
      const uint32_t buf0 = sb + (lane == 0 ? kOffK : kOffV);
      const int ns = lane == 0 ? kKStages : kVStages;
      for (int j = 0; j < T; ++j) {
        const int st = j % ns, u = j / ns;
        if (j >= ns) mbar_wait(empty0 + 8 * st, (u + 1) & 1);
        const uint32_t full = full0 + 8 * st, dst = buf0 + st * 2 * kKVPanel;
        mbar_expect_tx(full, 2 * kKVPanel);
        tma_load_4d(dst, tm, full, 0, kvh, j * kBN, req);
        tma_load_4d(dst + kKVPanel, tm, full, 64, kvh, j * kBN, req);
      }
      if (lane == 0 && a.u_stage) {
        for (int j = max(0, T - kKStages); j < T; ++j)
          mbar_wait(bar_k_empty + 8 * (j % kKStages), (j / kKStages) & 1);
        const uint32_t pu = (uint32_t)nb * nu * 128;
        mbar_expect_tx(bar_u, 8 * pu);
        for (int t = 0; t < 2; ++t) {
          const int b0 = (2 * mp + t) * nb;
          const uint32_t base = sb + kOffK + t * 4 * pu;
          tma_load_5d(base, &tm_ku, bar_u, 0, kvh, 0, b0, req);
          tma_load_5d(base + pu, &tm_ku, bar_u, 64, kvh, 0, b0, req);
          tma_load_5d(base + 2 * pu, &tm_vu, bar_u, 0, kvh, 0, b0, req);
          tma_load_5d(base + 3 * pu, &tm_vu, bar_u, 64, kvh, 0, b0, req);
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0 && T > 0) {
      constexpr uint32_t idS = idesc_bf16(128, kBN, 0);
      constexpr uint32_t idO = idesc_bf16(128, kD, 1);
      mbar_wait(bar_q, 0);
      auto issue_s = [&](int j, int t) {   // S_t(j) = Q_t K_j^T into S_t
        const int ks = j % kKStages;
        if (t == 0) {
          mbar_wait(bar_k_full + 8 * ks, (j / kKStages) & 1);
          tc_fence_after();
        }
        const uint32_t kb = sb + kOffK + ks * 2 * kKVPanel;
        const uint32_t qb = sb + kOffQ + 2 * t * kQPanel;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t p = kk >> 2, off = (kk & 3) * 32;
          umma(tmem + 256 * t, sdesc(qb + p * kQPanel + off, 16, 1024), sdesc(kb + p * kKVPanel + off, 16, 1024),
               idS, kk > 0);
        }
        umma_commit(bar_s_full + 8 * t);
        if (t == 1) umma_commit(bar_k_empty + 8 * ks);
      };
      auto issue_pv = [&](int j, int t) {  // O_t += P_t(j) V_j
        const int vs = j % kVStages;
        if (t == 0) mbar_wait(bar_v_full + 8 * vs, (j / kVStages) & 1);
        mbar_wait(bar_p_full + 8 * (2 * t + (j & 1)), (j >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = sb + kOffV + vs * 2 * kKVPanel;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts(tmem + 256 * t + 128, tmem + 256 * t + kk * 8, sdesc(vb + kk * 2048, kKVPanel, 1024), idO,
                  (j > 0 || kk > 0) ? 1u : 0u);
        if (t == 1) umma_commit(bar_v_empty + 8 * vs);
      };
      issue_s(0, 0);
      issue_s(0, 1);
      for (int j = 0; j < T; ++j) {
        issue_pv(j, 0);
        if (j + 1 < T) issue_s(j + 1, 0);
        issue_pv(j, 1);
        if (j + 1 < T) issue_s(j + 1, 1);
      }
      umma_commit(bar_o_final);
    }
  } else {
    // ===== softmax + epilogue: warps 2-5 tile A, 6-9 tile B; thread <-> row <-> TMEM lane =====
    const int t = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + 256 * t, tO = tS + 128;
    const float c2 = a.scale * 1.4426950408889634f;
    float m_ref = -INFINITY, raw_max = -INFINITY, l = 0.f;
    const int bl = r / a.G, g = r % a.G;
    const int b = (2 * mp + t) * nb + bl;
    const bool row_ok = b < a.bw;
    const int h = kvh * a.G + g;
    const int64_t qrow = (((int64_t)req * a.bw + b) * a.hq + h);
    constexpr int kMaxU = 8;
    float tu[kMaxU];
#pragma unroll
    for (int u = 0; u < kMaxU; ++u) tu[u] = -INFINITY;
    const uint8_t* qs = smem + kOffQ + 2 * t * kQPanel;
    auto dot_q = [&](auto&& krow) {   // q row (smem, swizzled) . 16 chunks given by krow(ch)
      float dot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) {
        const uint4 qv = *reinterpret_cast<const uint4*>(qs + (ch >> 3) * kQPanel + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
        float qf[8], kf[8];
        bf16x8_to_f32(qv, qf);
        bf16x8_to_f32(krow(ch), kf);
#pragma unroll
        for (int e = 0; e < 8; ++e) dot[ch & 3] = fmaf(qf[e], kf[e], dot[ch & 3]);
      }
      return ((dot[0] + dot[1]) + (dot[2] + dot[3])) * c2;
    };
    if (nu > 0 && !a.u_stage) {   // unshared logits from global memory, before the first S tile
      mbar_wait(bar_q, 0);
      if (row_ok) {
        const __nv_bfloat16* kub = a.ku + (int64_t)req * a.u_req_stride + (int64_t)b * a.u_beam_stride;
#pragma unroll 1
        for (int u = 0; u < nu; ++u) {
          const uint4* kr = reinterpret_cast<const uint4*>(kub + ((int64_t)u * a.hkv + kvh) * kD);
          const float v = dot_q([&](int ch) { return __ldg(kr + ch); });
#pragma unroll
          for (int w = 0; w < kMaxU; ++w)
            if (w == u) tu[w] = v;
        }
      }
    }
    for (int j = 0; j < T; ++j) {
      mbar_wait(bar_s_full + 8 * t, j & 1);
      tc_fence_after();
      float x[kBN];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        uint32_t u32[32];
        tmem_ld32(tS + lane_base + 32 * c4, u32);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) x[32 * c4 + c] = __uint_as_float(u32[c]);
      }
      const int valid = a.ls - j * kBN;
      if (valid < kBN) {
#pragma unroll
        for (int c = 0; c < kBN; ++c)
          if (c >= valid) x[c] = -INFINITY;
      }
      float mx[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        mx[c] = fmaxf(fmaxf(fmaxf(x[c], x[c + 16]), fmaxf(x[c + 32], x[c + 48])),
                      fmaxf(fmaxf(x[c + 64], x[c + 80]), fmaxf(x[c + 96], x[c + 112])));
#pragma unroll
      for (int c = 0; c < 8; ++c) mx[c] = fmaxf(mx[c], mx[c + 8]);
      const float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      raw_max = fmaxf(raw_max, tmax);
      const float t2 = tmax * c2;
      float alpha = 1.f;
      const bool resc = t2 > m_ref + kRescaleThreshold;
      if (resc) {
        alpha = ex2(m_ref - t2);
        m_ref = t2;
        l *= alpha;
      }
      float ls4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {   // two halves of 64 keys -> 32 packed columns each
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float p0 = ex2(fmaf(x[64 * h2 + 2 * c], c2, -m_ref));
          const float p1 = ex2(fmaf(x[64 * h2 + 2 * c + 1], c2, -m_ref));
          ls4[c & 3] += p0 + p1;
          pk[c] = pack_bf16(p0, p1);
        }
        tmem_st32(tS + lane_base + 32 * h2, pk);
      }
      l += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
      if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          uint32_t o[32];
          tmem_ld32(tO + lane_base + 32 * k, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          tmem_st32(tO + lane_base + 32 * k, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p_full + 8 * (2 * t + (j & 1)));
    }
    if (T > 0) {
      mbar_wait(bar_o_final, 0);
      tc_fence_after();
    }
    // ---- epilogue: unshared stage + merge, output tile by TMA ----
    const uint32_t pu = (uint32_t)nb * nu * 128;
    const uint8_t* us = smem + kOffK + t * 4 * pu;
    auto urow = [&](int panel, int u, int ch) -> uint4 {
      const int R = bl * nu + u;
      return *reinterpret_cast<const uint4*>(us + panel * pu + R * 128 + (((ch & 7) ^ (R & 7)) << 4));
    };
    if (nu > 0 && a.u_stage) {
      mbar_wait(bar_u, 0);
      if (row_ok) {
#pragma unroll 1
        for (int u = 0; u < nu; ++u) {
          const float v = dot_q([&](int ch) { return urow(ch >> 3, u, ch); });
#pragma unroll
          for (int w = 0; w < kMaxU; ++w)
            if (w == u) tu[w] = v;
        }
      }
    }
    float m_tot = (T > 0) ? m_ref : -INFINITY;
    if (row_ok) {
#pragma unroll
      for (int u = 0; u < kMaxU; ++u) m_tot = fmaxf(m_tot, tu[u]);
    }
    const __nv_bfloat16* vub = a.vu + (int64_t)req * a.u_req_stride + (int64_t)b * a.u_beam_stride;
    const float w_sh = (T > 0) ? ex2(m_ref - m_tot) : 0.f;
    float den = l * w_sh;
    float wu[kMaxU];
#pragma unroll
    for (int u = 0; u < kMaxU; ++u) {
      wu[u] = (row_ok && u < nu) ? ex2(tu[u] - m_tot) : 0.f;
      den += wu[u];
    }
    const float inv = 1.f / den;
    uint8_t* ost = smem + kOffV + t * 2 * kQPanel;   // this tile's output staging (V ring)
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      uint32_t o[32];
      if (T > 0) {
        tmem_ld32(tO + lane_base + 32 * k, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0u;
      }
      float acc[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = __uint_as_float(o[c]) * w_sh;
      if (row_ok) {
#pragma unroll
        for (int u = 0; u < kMaxU; ++u) {
          if (u < nu) {
            const uint4* vr = reinterpret_cast<const uint4*>(vub + ((int64_t)u * a.hkv + kvh) * kD + 32 * k);
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              float vf[8];
              bf16x8_to_f32(a.u_stage ? urow(2 + (k >> 1), u, (k & 1) * 4 + ch) : __ldg(vr + ch), vf);
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[8 * ch + e] = fmaf(wu[u], vf[e], acc[8 * ch + e]);
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ch = (k & 1) * 4 + c;
        *reinterpret_cast<uint4*>(ost + (k >> 1) * kQPanel + r * 128 + ((ch ^ (r & 7)) << 4)) =
            make_uint4(pack_bf16(acc[8 * c] * inv, acc[8 * c + 1] * inv),
                       pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv),
                       pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv),
                       pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");   // this tile's 4 softmax warps
    if (r == 0) {
      const int b0 = (2 * mp + t) * nb;
      tma_store_4d(&tm_o, su32(ost), 0, kvh * a.G, b0, req);
      tma_store_4d(&tm_o, su32(ost) + kQPanel, 64, kvh * a.G, b0, req);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (row_ok && a.lse) a.lse[qrow] = (m_tot + __log2f(den)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---- unshared stage alone and the merge: CUDA cores -------------
// One warp per (request, beam, head); lane owns 4 of the 128 dims. Partial outputs in fp32.
__global__ void __launch_bounds__(256) k_attn_unshared(const __nv_bfloat16* __restrict__ q,
                                                       const __nv_bfloat16* __restrict__ ku,
                                                       const __nv_bfloat16* __restrict__ vu, int64_t u_req_stride,
                                                       int64_t u_beam_stride, int n, int n_req, int bw, int hq,
                                                       int hkv, float scale, float* pm, float* ps, float* po) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (int64_t)n_req * bw * hq) return;
  const int h = (int)(row % hq);
  const int64_t rb = row / hq;
  const int b = (int)(rb % bw), req = (int)(rb / bw);
  const int kvh = h / (hq / hkv);
  float qf[4];
  {
    const uint2 u = *reinterpret_cast<const uint2*>(q + row * kD + 4 * lane);
    qf[0] = __uint_as_float(u.x << 16); qf[1] = __uint_as_float(u.x & 0xFFFF0000u);
    qf[2] = __uint_as_float(u.y << 16); qf[3] = __uint_as_float(u.y & 0xFFFF0000u);
  }
  const __nv_bfloat16* kb = ku + (int64_t)req * u_req_stride + (int64_t)b * u_beam_stride;
  const __nv_bfloat16* vb = vu + (int64_t)req * u_req_stride + (int64_t)b * u_beam_stride;
  float m = -INFINITY, s = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int t = 0; t < n; ++t) {
    const int64_t off = ((int64_t)t * hkv + kvh) * kD + 4 * lane;
    const uint2 ku2 = *reinterpret_cast<const uint2*>(kb + off);
    float d = qf[0] * __uint_as_float(ku2.x << 16);
    d = fmaf(qf[1], __uint_as_float(ku2.x & 0xFFFF0000u), d);
    d = fmaf(qf[2], __uint_as_float(ku2.y << 16), d);
    d = fmaf(qf[3], __uint_as_float(ku2.y & 0xFFFF0000u), d);
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) d += __shfl_xor_sync(0xffffffffu, d, k);
    const float x = d * scale;
    const float mn = fmaxf(m, x);
    const float al = (m == -INFINITY) ? 0.f : expf(m - mn);
    const float w = expf(x - mn);
    const uint2 vu2 = *reinterpret_cast<const uint2*>(vb + off);
    const float vf[4] = {__uint_as_float(vu2.x << 16), __uint_as_float(vu2.x & 0xFFFF0000u),
                         __uint_as_float(vu2.y << 16), __uint_as_float(vu2.y & 0xFFFF0000u)};
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = fmaf(o[e], al, w * vf[e]);
    s = s * al + w;
    m = mn;
  }
  if (lane == 0) {
    pm[row] = m;
    ps[row] = s;
  }
  reinterpret_cast<float4*>(po + row * kD)[lane] = make_float4(o[0], o[1], o[2], o[3]);
}

__global__ void __launch_bounds__(256) k_attn_merge(const float* __restrict__ m1, const float* __restrict__ s1,
                                                    const float* __restrict__ o1, const float* __restrict__ m2,
                                                    const float* __restrict__ s2, const float* __restrict__ o2,
                                                    int64_t rows, float* out, float* lse) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float a = m1[row], b = m2[row];
  const float m = fmaxf(a, b);
  const float w1 = (a == -INFINITY) ? 0.f : expf(a - m);
  const float w2 = (b == -INFINITY) ? 0.f : expf(b - m);
  const float den = s1[row] * w1 + s2[row] * w2;
  const float4 x = reinterpret_cast<const float4*>(o1 + row * kD)[lane];
  const float4 y = reinterpret_cast<const float4*>(o2 + row * kD)[lane];
  reinterpret_cast<float4*>(out + row * kD)[lane] =
      make_float4((x.x * w1 + y.x * w2) / den, (x.y * w1 + y.y * w2) / den, (x.z * w1 + y.z * w2) / den,
                  (x.w * w1 + y.w * w2) / den);
  if (lse && lane == 0) lse[row] = m + logf(den);
}

// ---- host side ----------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// N-D bf16 map (N = 4 or 5), dims innermost first, 128-byte swizzle, box inner = 64 elements.
static bool make_map_nd(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                        const uint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank, const_cast<void*>(base),
                        reinterpret_cast<const cuuint64_t*>(dims), reinterpret_cast<const cuuint64_t*>(strides_bytes),
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
// 4-D bf16 map, dims innermost first, 128-byte swizzle, box inner = 64 elements (128 B).
static bool make_map(CUtensorMap* m, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                     const uint32_t box[4]) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base),
                        reinterpret_cast<const cuuint64_t*>(dims), reinterpret_cast<const cuuint64_t*>(strides_bytes),
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace attn

// Returns 0 on success, 1 if the tensor maps could not be encoded, 2 on a launch error.
int launch_attn_shared(const void* q, const void* ks, const void* vs, int ls, const void* ku, const void* vu,
                       int64_t u_req_stride, int64_t u_beam_stride, int n_unshared, void* out, float* lse,
                       float* pm, float* ps, float* po, int n_req, int bw, int hq, int hkv, float scale,
                       cudaStream_t stream) {
  using namespace attn;
  const int G = hq / hkv;
  CUtensorMap tq, tk, tv, tku, tvu, to;
  {
    const uint64_t dims[4] = {(uint64_t)kD, (uint64_t)hq, (uint64_t)bw, (uint64_t)n_req};
    const uint64_t str[3] = {(uint64_t)kD * 2, (uint64_t)hq * kD * 2, (uint64_t)bw * hq * kD * 2};
    const uint32_t box[4] = {64, (uint32_t)G, (uint32_t)(kBM / G), 1};
    if (!make_map(&tq, q, dims, str, box)) return 1;
  }
  {
    const uint64_t dims[4] = {(uint64_t)kD, (uint64_t)hkv, (uint64_t)std::max(ls, 1), (uint64_t)n_req};
    const uint64_t str[3] = {(uint64_t)kD * 2, (uint64_t)hkv * kD * 2, (uint64_t)std::max(ls, 1) * hkv * kD * 2};
    const uint32_t box[4] = {64, 1, (uint32_t)kBN, 1};
    if (!make_map(&tk, ks, dims, str, box) || !make_map(&tv, vs, dims, str, box)) return 1;
  }
  AttnArgs a{};
  a.n_req = n_req; a.bw = bw; a.hq = hq; a.hkv = hkv; a.G = G; a.ls = ls; a.n_unshared = n_unshared;
  a.scale = scale;
  a.ku = static_cast<const __nv_bfloat16*>(ku); a.vu = static_cast<const __nv_bfloat16*>(vu);
  a.u_req_stride = u_req_stride; a.u_beam_stride = u_beam_stride;
  a.out = static_cast<__nv_bfloat16*>(out); a.lse = lse;
  a.pm = pm; a.ps = ps; a.po = po;
  static const int dbg_env = getenv("XGR_ATTN_DBG") ? atoi(getenv("XGR_ATTN_DBG")) : 0;
  a.dbg = dbg_env;
  // fused-mode epilogue staging: the unshared K/V rows of the CTA's beams fit the K ring, and
  // the 64-dim panels of 8-row swizzle atoms stay 1024-byte aligned
  const int nb = kBM / G;
  a.u_stage = (!pm && n_unshared > 0 && !(a.dbg & 2) && 4 * nb * n_unshared * 128 <= (int)(kKStages * 2 * kKVPanel) &&
               (nb * n_unshared) % 8 == 0) ? 1 : 0;
  a.o_tma = (!pm && !(a.dbg & 8)) ? 1 : 0;
  memset(&tku, 0, sizeof(tku));
  memset(&tvu, 0, sizeof(tvu));
  memset(&to, 0, sizeof(to));
  if (a.u_stage) {
    const uint64_t dims[5] = {(uint64_t)kD, (uint64_t)hkv, (uint64_t)n_unshared, (uint64_t)bw, (uint64_t)n_req};
    const uint64_t str[4] = {(uint64_t)kD * 2, (uint64_t)hkv * kD * 2, (uint64_t)u_beam_stride * 2,
                             (uint64_t)std::max<int64_t>(u_req_stride, 1) * 2};
    const uint32_t box[5] = {64, 1, (uint32_t)n_unshared, (uint32_t)nb, 1};
    if (!make_map_nd(&tku, ku, 5, dims, str, box) || !make_map_nd(&tvu, vu, 5, dims, str, box)) return 1;
  }
  if (a.o_tma) {
    const uint64_t dims[4] = {(uint64_t)kD, (uint64_t)hq, (uint64_t)bw, (uint64_t)n_req};
    const uint64_t str[3] = {(uint64_t)kD * 2, (uint64_t)hq * kD * 2, (uint64_t)bw * hq * kD * 2};
    const uint32_t box[4] = {64, (uint32_t)G, (uint32_t)(kBM / G), 1};
    if (!make_map(&to, out, dims, str, box)) return 1;
  }
  // fused mode: XGR_ATTN_IMPL=2 selects the two-Q-tile kernel (k_attn_pair; slower, kept for study)
  static const int impl_env = getenv("XGR_ATTN_IMPL") ? atoi(getenv("XGR_ATTN_IMPL")) : 1;
  if (!pm && impl_env == 2) {
    a.u_stage = (n_unshared > 0 && !(a.dbg & 2) && 8 * nb * n_unshared * 128 <= (int)(pair::kKStages * 2 * pair::kKVPanel) &&
                 (nb * n_unshared) % 8 == 0) ? 1 : 0;
    memset(&tku, 0, sizeof(tku));
    memset(&tvu, 0, sizeof(tvu));
    if (a.u_stage) {
      const uint64_t dims[5] = {(uint64_t)kD, (uint64_t)hkv, (uint64_t)n_unshared, (uint64_t)bw, (uint64_t)n_req};
      const uint64_t str[4] = {(uint64_t)kD * 2, (uint64_t)hkv * kD * 2, (uint64_t)u_beam_stride * 2,
                               (uint64_t)std::max<int64_t>(u_req_stride, 1) * 2};
      const uint32_t box[5] = {64, 1, (uint32_t)n_unshared, (uint32_t)nb, 1};
      if (!make_map_nd(&tku, ku, 5, dims, str, box) || !make_map_nd(&tvu, vu, 5, dims, str, box)) return 1;
    }
    CUtensorMap tk2, tv2;
    const uint64_t dims[4] = {(uint64_t)kD, (uint64_t)hkv, (uint64_t)std::max(ls, 1), (uint64_t)n_req};
    const uint64_t str[3] = {(uint64_t)kD * 2, (uint64_t)hkv * kD * 2, (uint64_t)std::max(ls, 1) * hkv * kD * 2};
    const uint32_t box[4] = {64, 1, (uint32_t)pair::kBN, 1};
    if (!make_map(&tk2, ks, dims, str, box) || !make_map(&tv2, vs, dims, str, box)) return 1;
    const dim3 grid2((unsigned)((bw * G + 255) / 256), (unsigned)hkv, (unsigned)n_req);
    cudaFuncSetAttribute(k_attn_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pair::kSmem);
    k_attn_pair<<<grid2, pair::kThreads, pair::kSmem, stream>>>(tq, tk2, tv2, tku, tvu, to, a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  const dim3 grid((unsigned)((bw * G + kBM - 1) / kBM), (unsigned)hkv, (unsigned)n_req);
  if (pm) {
    cudaFuncSetAttribute(k_attn_shared<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    k_attn_shared<true><<<grid, kThreads, kSmem, stream>>>(tq, tk, tv, tku, tvu, to, a);
  } else {
    cudaFuncSetAttribute(k_attn_shared<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    k_attn_shared<false><<<grid, kThreads, kSmem, stream>>>(tq, tk, tv, tku, tvu, to, a);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

cudaError_t launch_attn_unshared(const void* q, const void* ku, const void* vu, int64_t u_req_stride,
                                 int64_t u_beam_stride, int n, int n_req, int bw, int hq, int hkv, float scale,
                                 float* pm, float* ps, float* po, cudaStream_t stream) {
  const int64_t rows = (int64_t)n_req * bw * hq;
  attn::k_attn_unshared<<<(unsigned)((rows + 7) / 8), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(ku),
      static_cast<const __nv_bfloat16*>(vu), u_req_stride, u_beam_stride, n, n_req, bw, hq, hkv, scale, pm, ps, po);
  return cudaGetLastError();
}

cudaError_t launch_attn_merge(const float* m1, const float* s1, const float* o1, const float* m2, const float* s2,
                              const float* o2, int64_t rows, float* out, float* lse, cudaStream_t stream) {
  attn::k_attn_merge<<<(unsigned)((rows + 7) / 8), 256, 0, stream>>>(m1, s1, o1, m2, s2, o2, rows, out, lse);
  return cudaGetLastError();
}

}  // namespace xgr
