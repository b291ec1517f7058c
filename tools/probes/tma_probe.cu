// Micro-probe: weight-stream bandwidth, 2D TMA boxes (128 rows x 128 B, the
// GEMM's W tile) vs 1D bulk copies of 16 KB contiguous (a pre-tiled layout).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred d;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph));
}
template <int MODE, int STAGES>
__global__ void stream(const __grid_constant__ CUtensorMap map, const uint8_t* base, int tiles_n, int kch,
                       const __grid_constant__ CUtensorMap xmap, int xrows) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    int it = 0;
    for (int t = blockIdx.x; t < tiles_n; t += gridDim.x) {
      for (int c = 0; c < kch; ++c, ++it) {
        const int st = it % STAGES;
        if (it >= STAGES) wait(&full[st], ((it / STAGES) - 1) & 1);
        const uint32_t bytes = 16384 + (MODE == 2 ? xrows * 128 : 0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(bytes));
        if (MODE == 2)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                       ::"r"(sa(s + STAGES * 16384 + st * 32768)), "l"((uint64_t)&xmap), "r"(sa(&full[st])), "r"(c * 64), "r"(0) : "memory");
        if (MODE == 0 || MODE == 2) {
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                       ::"r"(sa(s + st * 16384)), "l"((uint64_t)&map), "r"(sa(&full[st])), "r"(c * 64), "r"(t * 128) : "memory");
        } else {
          const uint8_t* src = base + ((size_t)t * kch + c) * 16384;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                       ::"r"(sa(s + st * 16384)), "l"((uint64_t)src), "r"(sa(&full[st])) : "memory");
        }
      }
    }
    for (int j = 0; j < STAGES && j < it; ++j) {
      const int k = it - 1 - j;
      wait(&full[k % STAGES], (k / STAGES) & 1);
    }
  }
  __syncthreads();
}
int main() {
  const int N = 16384, K = 4096;
  uint8_t* w;
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMemset(w, 1, (size_t)N * K * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N}, str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int tiles = N / 128, kch = K / 64;
  uint8_t* xbuf; cudaMalloc(&xbuf, 256 * K * 2); cudaMemset(xbuf, 1, 256 * K * 2);
  CUtensorMap xm128, xm256;
  { cuuint64_t d2[2] = {(cuuint64_t)K, 256}; cuuint32_t bx[2] = {64, 128};
    enc(&xm128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xbuf, d2, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t bx2[2] = {64, 256};
    enc(&xm256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xbuf, d2, str, bx2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  const CUtensorMap* xmap = &xm128; int xrows = 128;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int stages, int grid, const char* name) {
    int smem = stages * 16384 + 1024 + stages * 32768;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, 32, smem>>>(map, w, tiles, kch, *xmap, xrows);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) kern<<<grid, 32, smem>>>(map, w, tiles, kch, *xmap, xrows);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-28s stages=%2d grid=%3d: %.0f GB/s  (%s)\n", name, stages, grid,
           (double)N * K * 2 * 10 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int grid : {96, 148}) {
    run(stream<0, 4>, 4, grid, "W only 2D");
    xmap = &xm128; xrows = 128;
    run(stream<2, 2>, 2, grid, "W + X(128 rows, L2) 2D");
    run(stream<2, 4>, 4, grid, "W + X(128 rows, L2) 2D");
    xmap = &xm256; xrows = 256;
    run(stream<2, 2>, 2, grid, "W + X(256 rows, L2) 2D");
    run(stream<2, 4>, 4, grid, "W + X(256 rows, L2) 2D");
  }
  return 0;
}
