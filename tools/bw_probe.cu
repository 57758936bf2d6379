// Read-bandwidth probe on the B200 (diagnostic, not product code): what streaming pattern can
// reach the HBM roof for the dense-step row stream?
//   ldg:  grid-stride LDG.128 reduction (plain loads, many warps)
//   tma:  persistent CTAs, one producer thread issuing cp.async.bulk chunks into an NS-stage ring,
//         consumer warps waiting on the mbarrier and touching one word per stage.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

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
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void k_ldg(const float4* __restrict__ p, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// unroll-8 register streaming: each thread issues 8 independent loads per iteration
__global__ void k_ldg8(const float4* __restrict__ p, size_t n4, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(p + i + k * stride));
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// items = chunks of `chunk` bytes; CTA c takes items c, c+G, ...; copies split in `split` parts
__global__ void k_tma(const char* __restrict__ p, size_t nitems, uint32_t chunk, int ns, int split, float* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == nw) {
    if (lane) return;
    for (size_t k = 0;; ++k) {
      size_t w = blockIdx.x + k * gridDim.x;
      if (w >= nitems) break;
      int st = k % ns;
      if (k >= (size_t)ns) mbar_wait(&empty[st], ((k / ns) - 1) & 1);
      mbar_arrive_tx(&full[st], chunk);
      uint32_t part = chunk / split;
      for (int q = 0; q < split; ++q) bulk(sm + (size_t)st * chunk + q * part, p + w * chunk + q * part, part, &full[st]);
    }
    return;
  }
  float acc = 0.f;
  for (size_t k = 0;; ++k) {
    size_t w = blockIdx.x + k * gridDim.x;
    if (w >= nitems) break;
    int st = k % ns;
    mbar_wait(&full[st], (k / ns) & 1);
    acc += reinterpret_cast<const float*>(sm + (size_t)st * chunk)[threadIdx.x];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const size_t bytes = 4ull << 30;
  char* d;
  float* o;
  cudaMalloc(&d, bytes);
  cudaMalloc(&o, 64);
  cudaMemset(d, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name) {
    for (int i = 0; i < 2; ++i) launch();
    cudaEventRecord(a);
    const int R = 5;
    for (int i = 0; i < R; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-44s %8.1f GB/s  (%s)\n", name, bytes * R / (ms / 1e3) / 1e9, cudaGetErrorString(e));
  };
  size_t n4 = bytes / 16;
  for (int bpsm : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "ldg  256thr x %d/SM", bpsm);
    timeit([&] { k_ldg<<<sms * bpsm, 256>>>((const float4*)d, n4, o); }, nm);
    snprintf(nm, 64, "ldg8 256thr x %d/SM", bpsm);
    timeit([&] { k_ldg8<<<sms * bpsm, 256>>>((const float4*)d, n4, o); }, nm);
  }
  struct Cfg { uint32_t chunk; int ns; int split; int ctas; int warps; };
  std::vector<Cfg> cfgs = {{32768, 6, 1, 1, 8}, {32768, 6, 4, 1, 8}, {32768, 6, 8, 1, 8}, {16384, 12, 1, 1, 8},
                           {8192, 16, 1, 1, 8},  {32768, 3, 1, 2, 8}, {16384, 6, 1, 2, 8}, {65536, 3, 1, 1, 8},
                           {32768, 6, 32, 1, 8}, {4096, 16, 1, 2, 4}};
  for (auto c : cfgs) {
    size_t smem = (size_t)c.chunk * c.ns;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    char nm[96];
    snprintf(nm, 96, "tma chunk %6u ns %2d split %2d ctas/SM %d", c.chunk, c.ns, c.split, c.ctas);
    size_t items = bytes / c.chunk;
    timeit([&] { k_tma<<<sms * c.ctas, (c.warps + 1) * 32, smem>>>(d, items, c.chunk, c.ns, c.split, o); }, nm);
  }
  return 0;
}
