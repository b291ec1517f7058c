// Weight-stream layout probe: TMA 2-D boxes of 128 rows x 128 B streamed
// from a 512 MB weight matrix, each CTA walking its own 128-row tile along K
// (as the GEMM does), with
//   strided: row-major W [N][K] (K = 4096): the 128 rows of a box are 8 KB apart
//   tiled  : W re-laid out as [N/128][K/64][128][64]: every box is 16 KB contiguous
// 96 and 148 CTAs, 5-stage rings, one issuing thread.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred d;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph));
}
__global__ void stream(const __grid_constant__ CUtensorMap map, int tiles, int kch, int tiled, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  int it = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x)
    for (int c = 0; c < kch; ++c, ++it) {
      const int st = it % stages;
      if (it >= stages) wait(&full[st], ((it / stages) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(16384));
      const int c0 = tiled ? 0 : c * 64, c1 = tiled ? (t * kch + c) * 128 : t * 128;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(sa(s + st * 16384)), "l"((uint64_t)&map), "r"(sa(&full[st])), "r"(c0), "r"(c1) : "memory");
    }
  for (int j = 0; j < stages && j < it; ++j) {
    const int k = it - 1 - j;
    wait(&full[k % stages], (k / stages) & 1);
  }
}
int main() {
  const int N = 65536, K = 4096;   // 512 MB
  uint8_t* w;
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMemset(w, 1, (size_t)N * K * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap mstr, mtil;
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  { cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N}, str[1] = {(cuuint64_t)K * 2};
    enc(&mstr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  { cuuint64_t dims[2] = {64, (cuuint64_t)N * (K / 64)}, str[1] = {128};
    enc(&mtil, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  const int tiles = N / 128, kch = K / 64;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 16384 + 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int stages : {5, 12})
    for (int grid : {96, 148})
      for (int tiled = 0; tiled < 2; ++tiled) {
        const int smem = stages * 16384 + 1024;
        stream<<<grid, 32, smem>>>(tiled ? mtil : mstr, tiles, kch, tiled, stages);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) stream<<<grid, 32, smem>>>(tiled ? mtil : mstr, tiles, kch, tiled, stages);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-8s grid=%3d stages=%2d: %6.0f GB/s (%s)\n", tiled ? "tiled" : "strided", grid, stages,
               3.0 * N * K * 2 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
