// KV-cache reorder after a beam step (section 5.1, Fig. 6:
// the unshared per-beam cache "updates block contents based on beam indices").
//
// new row (r, p, j) = old row (r, p, src[r][j]) for every request r, panel p and slot j with
// src >= 0, in place. The paper's (and SPEC's) scheme canonicalises the map to a non-decreasing one
// and orders the writes in two passes so that no row is overwritten before it is read. On the GPU
// the rows are cut into column tiles instead: one CTA owns one tile of all BW rows of a
// (request, panel), stages the tiles of the rows that some changed slot reads in shared memory,
// synchronises, then writes the changed slots (a CTA walks several tiles, double-buffered). No two CTAs touch the same bytes, so any map --
// not only monotone ones -- is hazard-free and the slot order (sorted by score, DESIGN R5) never
// needs re-sorting. HBM traffic: the distinct source rows of changed slots, read once, plus the
// changed slots, written once (unchanged slots cost nothing).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "xgr_internal.cuh"

namespace xgr {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One CTA per (request, slice of the request's (panel, tile) items). The request's map is read
// once into compact lists (changed destinations with their sources; the distinct source rows,
// each given a staging slot); then every item streams through a double buffer: the cp.async
// loads of item k+1 are in flight while item k's changed rows are written.
template <int TW>   // tile width in bytes (multiple of 16)
__global__ void __launch_bounds__(256) k_kv_reorder(char* __restrict__ cache, int bw, int64_t row_bytes,
                                                    int64_t beam_stride, int64_t panel_stride,
                                                    int64_t req_stride, int n_panel,
                                                    const int32_t* __restrict__ src, int src_ld) {
  constexpr int CW = TW / 16;   // 16-byte columns per tile
  extern __shared__ uint4 s_buf[];   // [2][bw][CW]
  __shared__ int16_t s_dst[kMaxBW], s_from[kMaxBW];   // changed slot j <- staging slot
  __shared__ int16_t s_need[kMaxBW];                  // staging slot -> source row
  __shared__ int16_t s_slot[kMaxBW];                  // source row -> staging slot
  __shared__ int s_nchg, s_nneed;
  const int r = blockIdx.z, tid = threadIdx.x;
  if (tid == 0) s_nchg = s_nneed = 0;
  for (int j = tid; j < bw; j += 256) s_slot[j] = -1;
  __syncthreads();
  for (int j = tid; j < bw; j += 256) {
    const int sr = src[(int64_t)r * src_ld + j];
    if (sr >= 0 && sr != j && sr < bw) {
      s_dst[atomicAdd(&s_nchg, 1)] = (int16_t)j;
      if (atomicCAS(reinterpret_cast<unsigned short*>(&s_slot[sr]), 0xFFFFu, 0xFFFEu) == 0xFFFFu)
        s_need[atomicAdd(&s_nneed, 1)] = (int16_t)sr;   // first claimant lists the row
    }
  }
  __syncthreads();
  const int nchg = s_nchg, nneed = s_nneed;
  if (nchg == 0) return;
  for (int i = tid; i < nneed; i += 256) s_slot[s_need[i]] = (int16_t)i;
  __syncthreads();
  for (int k = tid; k < nchg; k += 256) s_from[k] = s_slot[src[(int64_t)r * src_ld + s_dst[k]]];
  if (bw * CW > 256 * 8) return;   // the launcher keeps bw * TW <= 32 KB
  __syncthreads();
  const int64_t tiles = (row_bytes + TW - 1) / TW;
  const int64_t items = tiles * n_panel;
  char* rbase = cache + (int64_t)r * req_stride;
  // Per-thread work is the same for every item (only the item's base address moves), so the
  // (row, column) offsets are computed once: up to KE staging copies and KE writes per thread
  // (bw * TW <= 32 KB -> bw * CW <= 2048 = 8 * 256).
  constexpr int KE = 8;
  int64_t ld_off[KE], st_off[KE];
  int ld_c[KE], st_c[KE], st_s[KE];
#pragma unroll
  for (int m = 0; m < KE; ++m) {
    const int e = tid + 256 * m;
    ld_c[m] = -1;
    st_c[m] = -1;
    if (e < nneed * CW) {
      const int i = e / CW;
      ld_c[m] = e - i * CW;
      ld_off[m] = (int64_t)s_need[i] * beam_stride + 16 * ld_c[m];
    }
    if (e < nchg * CW) {
      const int q = e / CW;
      st_c[m] = e - q * CW;
      st_off[m] = (int64_t)s_dst[q] * beam_stride + 16 * st_c[m];
      st_s[m] = s_from[q] * CW + st_c[m];
    }
  }
  auto item_base = [&](int64_t it, int& cols) {
    const int64_t p = it / tiles, t = it - p * tiles;
    cols = (int)min((int64_t)CW, (row_bytes - t * TW) >> 4);
    return rbase + p * panel_stride + t * TW;
  };
  auto stage = [&](int64_t it, uint4* buf) {
    int cols;
    const char* b = item_base(it, cols);
#pragma unroll
    for (int m = 0; m < KE; ++m)
      if (ld_c[m] >= 0 && ld_c[m] < cols) cp_async16(buf + tid + 256 * m, b + ld_off[m]);
    cp_async_commit();
  };
  int64_t it = blockIdx.x;
  if (it < items) stage(it, s_buf);
  for (int k = 0; it < items; ++k, it += gridDim.x) {
    uint4* cur = s_buf + (size_t)(k & 1) * bw * CW;
    const int64_t nx = it + gridDim.x;
    if (nx < items) {
      stage(nx, s_buf + (size_t)((k + 1) & 1) * bw * CW);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();   // item it staged by every thread
    int cols;
    char* b = item_base(it, cols);
#pragma unroll
    for (int m = 0; m < KE; ++m)
      if (st_c[m] >= 0 && st_c[m] < cols) __stcs(reinterpret_cast<uint4*>(b + st_off[m]), cur[st_s[m]]);
    __syncthreads();   // cur may be refilled by the next stage
  }
}

cudaError_t launch_kv_reorder(void* cache, int n_req, int n_panel, int bw, int64_t row_bytes,
                              int64_t beam_stride, int64_t panel_stride, int64_t req_stride,
                              const int32_t* src, int src_ld, cudaStream_t s) {
  // tile width: a 64 KB double buffer (3 CTAs per SM); the grid asks for 6 per SM (measured best
  // at C3 shape: 0.70 of the copy peak vs 0.65 at 3, 0.55 with 32 KB buffers; profiles/)
  static const int tw_env = getenv("XGR_KV_TW") ? atoi(getenv("XGR_KV_TW")) : 0;
  static const int cps_env = getenv("XGR_KV_CPS") ? atoi(getenv("XGR_KV_CPS")) : 0;
  int tw = std::max(32, std::min(128, 32768 / bw));
  if (tw_env == 32 || tw_env == 64 || tw_env == 128 || tw_env == 256) tw = std::max(32, std::min(tw_env, 32768 / bw));
  const int cps = cps_env > 0 ? cps_env : 6;   // CTAs per SM requested
  const int64_t items = (row_bytes + tw - 1) / tw * n_panel;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = ((int64_t)cps * sms + n_req - 1) / n_req;
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(items, want)), 1, (unsigned)n_req);
  const size_t smem = 2 * (size_t)bw * tw;
  char* c = static_cast<char*>(cache);
#define XGR_KV_LAUNCH(TWV)                                                                                 \
  cudaFuncSetAttribute(k_kv_reorder<TWV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
  k_kv_reorder<TWV><<<grid, 256, smem, s>>>(c, bw, row_bytes, beam_stride, panel_stride, req_stride, n_panel, \
                                           src, src_ld)
  if (tw == 256) {
    XGR_KV_LAUNCH(256);
  } else if (tw == 128) {
    XGR_KV_LAUNCH(128);
  } else if (tw == 64) {
    XGR_KV_LAUNCH(64);
  } else {
    XGR_KV_LAUNCH(32);
  }
#undef XGR_KV_LAUNCH
  return cudaGetLastError();
}

}  // namespace xgr
