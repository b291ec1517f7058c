// Micro-probe: cycles per tcgen05.mma (kind::f16, cta_group::1, SS operands)
// with operands resident in shared memory -- no TMA traffic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(const void* tile) {
  uint64_t a = smem_u32(tile);
  return ((a >> 4) & 0x3FFF) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__global__ void probe(int n_mma, int N, unsigned long long* out, const uint8_t* g, int tma_on, int nacc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (200 * 1024) / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 32 && tma_on == 1) {
    // concurrent 1D bulk copies into a separate region (like a TMA producer)
    __shared__ __align__(8) uint64_t tb[4];
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tb[i])));
    uint8_t* dst = smem + 16384 + 256 * 128;
    for (int it = 0; it < 2000; ++it) {
      const int st = it & 3;
      if (it >= 4) asm volatile("{\n\t.reg .pred d;\nT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra T_%=;\n\t}" ::"r"(smem_u32(&tb[st])), "r"(((it >> 2) - 1) & 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(smem_u32(&tb[st])));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                   ::"r"(smem_u32(dst + st * 16384)), "l"((uint64_t)(g + ((size_t)(blockIdx.x * 2000 + it) % 4096) * 16384)), "r"(smem_u32(&tb[st])) : "memory");
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    // cycle through NST distinct stages (A 16 KB + B N*128 B each) like a GEMM ring
    const int stage_b = 16384 + N * 128;
    const int nst = tma_on == 2 ? (200 * 1024) / stage_b : 1;
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;
      const int st = (i >> 2) % nst;
      uint64_t ad = desc_sw128(smem + st * stage_b), bd = desc_sw128(smem + st * stage_b + 16384);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_base + (i % nacc) * N),
                   "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"((int)(i >= nacc)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred d;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}" ::"r"(smem_u32(&bar)));
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  uint8_t* g; cudaMalloc(&g, (size_t)4096 * 16384);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (int N : {16, 32, 64, 128}) {
    for (int grid : {1}) {
     for (int tma_on : {0, 2}) {
      for (int nacc : {1, 2, 4}) {
      if (nacc * N > 256) continue;
      probe<<<grid, 128, 210 * 1024>>>(4096, N, d, g, tma_on, nacc);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
      printf("N=%3d grid=%3d tma=%d nacc=%d: %.1f cycles per MMA (floor %d)  err=%s\n", N, grid, tma_on, nacc, avg / 4096, 128 * N / 256,
             cudaGetErrorString(cudaGetLastError()));
      }
     }
    }
  }
  return 0;
}
