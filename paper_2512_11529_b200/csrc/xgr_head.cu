// LM-head fusion at sparse steps ("dense" masks only at the
// first steps -- at the later ones each row has a handful of legal tokens).
//
// Instead of a [rows][V] logits row per beam (a V x d GEMV per beam), a sparse step needs only the
// legal tokens' logits x[b][v] = sum_k h[b][k] * W[v][k] (+ bias[v]): one d-long dot product per
// legal child. k_head computes exactly those, one warp per live row: the row's hidden state and
// each child's LM-head row are read as 16-byte bf16 chunks (lanes stride the chunks; W rows come
// from L2, where a V x d bf16 head stays resident), fp32 FMAs in a fixed order, a fixed butterfly
// for the warp sum. The results go to a compact [batch][BW][cld] buffer (child q of row b at
// q - first_child) that the sparse-step kernel reads instead of a logits row.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "xgr_internal.cuh"

namespace xgr {

__device__ __forceinline__ float dot8(const uint4 h, const uint4 w, float acc) {
  const uint32_t hh[4] = {h.x, h.y, h.z, h.w}, ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    acc = fmaf(__uint_as_float(hh[k] << 16), __uint_as_float(ww[k] << 16), acc);
    acc = fmaf(__uint_as_float(hh[k] & 0xFFFF0000u), __uint_as_float(ww[k] & 0xFFFF0000u), acc);
  }
  return acc;
}

// KC 16-byte chunks per lane per pass (KC * 256 elements of d per pass): the hidden chunks of the
// first pass are loaded first (they depend only on the slot), before the node -> first_child ->
// label chain resolves, and every pass issues all KC loads of a child's head row at once. (Wider
// passes, KC = 8, and two children per pass were measured slower: fewer resident warps.)
template <int WPB, int KC>
__global__ void __launch_bounds__(WPB * 32) k_head(const __grid_constant__ StepArgs a,
                                                   const __nv_bfloat16* __restrict__ hidden, int64_t ldh,
                                                   int64_t hreq, const __nv_bfloat16* __restrict__ head,
                                                   int64_t ldw, const float* __restrict__ bias, int d,
                                                   float* __restrict__ clog) {
  pdl_wait();
  if (a.dbg & (1 << 20)) pdl_trigger();   // early trigger only on request (XGR_DEBUG_FLAGS bit 20)
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * WPB + (threadIdx.x >> 5), req = blockIdx.y;
  if (b >= a.BW) return;
  const uint4* hp = reinterpret_cast<const uint4*>(hidden + (size_t)req * hreq + (size_t)b * ldh);
  const int nch = d >> 3;   // 16-byte chunks
  uint4 hv[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = lane + 32 * k;
    hv[k] = c < nch ? __ldg(hp + c) : make_uint4(0u, 0u, 0u, 0u);
  }
  const int nl = a.nlive_in ? a.nlive_in[req] : 1;
  const uint32_t node = a.node_in ? a.node_in[(size_t)req * a.BW + b] : 0u;
  if (b >= nl) return;
  const LevelDev& L = a.trie.lv[a.level];
  const uint16_t* lab = a.trie.lv[a.level + 1].label;
  const uint32_t fc = L.first_child[node], fe = L.first_child[node + 1];
  float* out = clog + ((size_t)req * a.BW + b) * a.cld;
  for (uint32_t q = fc; q < fe; ++q) {
    const uint32_t v = lab[q];
    const uint4* wp = reinterpret_cast<const uint4*>(head + (size_t)v * ldw);
    float acc = 0.f;
    for (int c0 = 0; c0 < nch; c0 += 32 * KC) {
      uint4 wv[KC];
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        const int c = c0 + lane + 32 * k;
        wv[k] = c < nch ? __ldg(wp + c) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        const int c = c0 + lane + 32 * k;
        const uint4 h = c0 == 0 ? hv[k] : (c < nch ? __ldg(hp + c) : make_uint4(0u, 0u, 0u, 0u));
        acc = dot8(h, wv[k], acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[q - fc] = bias ? __fadd_rn(acc, bias[v]) : acc;
  }
}

cudaError_t launch_head(const StepArgs& a, const void* hidden, int64_t ldh, int64_t hreq, const void* head,
                        int64_t ldw, const float* bias, int d, float* clog, cudaStream_t s) {
  constexpr int WPB = 8;
  const dim3 grid((unsigned)((a.BW + WPB - 1) / WPB), (unsigned)a.batch);
  static const int kc = getenv("XGR_HEAD_KC") ? atoi(getenv("XGR_HEAD_KC")) : 4;
  const __nv_bfloat16* h = static_cast<const __nv_bfloat16*>(hidden);
  const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(head);
  if (kc == 8) launch_pdl(k_head<WPB, 8>, grid, WPB * 32, 0, s, a, h, ldh, hreq, w, ldw, bias, d, clog);
  else if (kc == 2) launch_pdl(k_head<WPB, 2>, grid, WPB * 32, 0, s, a, h, ldh, hreq, w, ldw, bias, d, clog);
  else launch_pdl(k_head<WPB, 4>, grid, WPB * 32, 0, s, a, h, ldh, hreq, w, ldw, bias, d, clog);
  return cudaGetLastError();
}

}  // namespace xgr
