// Per-SM TMA ingest ceiling with L2-resident sources: 2-D boxes (64 bf16 x R
// rows, SWIZZLE_128B -- the GEMM operand tiles) vs 1-D bulk copies of the same
// bytes, at several grid sizes (1 CTA / SM) and ring depths.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred d;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph));
}
// MODE 0: 2D box [rows][64] bf16 SW128; MODE 1: 1D bulk of rows*128 bytes
template <int MODE>
__global__ void stream(const __grid_constant__ CUtensorMap map, const uint8_t* base, int iters, int stages,
                       int rows, int nbox, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[64];
  const uint32_t bytes = rows * 128;
  const int issuer = threadIdx.x >> 5;            // one issuing thread per warp, own ring
  if ((threadIdx.x & 31) == 0) {
    uint64_t* fullw = full + issuer * 16;
    s += issuer * stages * bytes;
    uint64_t* full = fullw;
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = it % stages;
      if (it >= stages) wait(&full[st], ((it / stages) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(bytes));
      const int box = (blockIdx.x * 1021 + it * 148 + issuer * 37) % nbox;
      if (MODE == 0) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(sa(s + st * bytes)), "l"((uint64_t)&map), "r"(sa(&full[st])), "r"((box % 16) * 64), "r"((box / 16) * rows) : "memory");
      } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %3, [%2];"
                     ::"r"(sa(s + st * bytes)), "l"((uint64_t)(base + (size_t)box * bytes)), "r"(sa(&full[st])), "r"(bytes) : "memory");
      }
    }
    for (int j = 0; j < stages && j < iters; ++j) {
      const int k = iters - 1 - j;
      wait(&full[k % stages], (k / stages) & 1);
    }
    if (issuer == 0) cyc[blockIdx.x] = clock64() - t0;
  }
}
int main() {
  // source: [R rows][1024 bf16]; R = 2048 (4 MB, L2 resident) or 262144 (512 MB, HBM stream)
  const int R = getenv("HBM") ? 262144 : 2048, K = 1024;
  uint8_t* w;
  cudaMalloc(&w, (size_t)R * K * 2);
  cudaMemset(w, 1, (size_t)R * K * 2);
  unsigned long long* cyc; cudaMalloc(&cyc, 148 * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int warps : {1, 2, 4})
  for (int rows : {128}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)R}, str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int nbox = 16 * (R / rows);
    for (int mode = 0; mode < 1; ++mode)
      for (int grid : {16, 148})
        for (int stages : {4, 8}) {
          const int bytes = rows * 128;
          const int smem = warps * stages * bytes + 1024;
          if (smem > 220 * 1024) continue;
          auto k = mode ? stream<1> : stream<0>;
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          const int iters = getenv("HBM") ? 1500 : 400;
          k<<<grid, 32 * warps, smem>>>(map, w, iters, stages, rows, nbox, cyc);
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
          cudaEventRecord(a);
          k<<<grid, 32 * warps, smem>>>(map, w, iters, stages, rows, nbox, cyc);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          unsigned long long h[148]; cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
          double c = 0; for (int i = 0; i < grid; ++i) c += h[i]; c /= grid;
          printf("%s issuers=%d rows=%3d grid=%3d stages=%d: %6.1f B/clk/SM, chip %6.0f GB/s (%s)\n", mode ? "1D bulk" : "2D box ",
                 warps, rows, grid, stages, warps * (double)iters * bytes / c, warps * (double)grid * iters * bytes / (ms * 1e-3) / 1e9,
                 cudaGetErrorString(cudaGetLastError()));
        }
  }
  return 0;
}
