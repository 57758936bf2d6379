// Diagnostic: resource usage and occupancy of the dense-step kernels (run on the GPU box).
#include <cstdio>
#include "../paper_2512_11529_b200/csrc/xgr_stream.cu"
using namespace xgr;
template <typename K>
void show(const char* name, K k, int threads, size_t smem) {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = -1;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, threads, smem);
  printf("%-22s regs %3d static smem %6zu maxThreads %4d  threads %4d dyn %7zu -> blocks/SM %d (%s)\n", name,
         fa.numRegs, fa.sharedSizeBytes, fa.maxThreadsPerBlock, threads, smem, nb, cudaGetErrorString(e));
}
int main() {
  show("k_stream<32,3,6>", k_stream<32, 3, 6>, 800, stream_smem<32, 6>());
  show("k_stream<64,2,3>", k_stream<64, 2, 3>, 544, stream_smem<64, 3>());
  show("k_seed<256,4>", k_seed<256, 4>, 1024, stream_smem<32, 4>());
  show("k_seed<512,2>", k_seed<512, 2>, 1024, stream_smem<64, 2>());
  return 0;
}
