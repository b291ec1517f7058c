// Micro-probe: issue cost of tcgen05.mma.cta_group::2 (M = 256 over a CTA
// pair) vs cta_group::1 (M = 128), kind::f16, SS operands resident in shared
// memory, one issuing thread, N = 16..256 -- cycles per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma2_probe mma2_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(const void* tile) {
  uint64_t a = sa(tile);
  return ((a >> 4) & 0x3FFF) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int PAIR>
__global__ void __cluster_dims__(PAIR ? 2 : 1, 1, 1) probe(int n_mma, int N, int nst, unsigned long long* out,
                                                           const uint8_t* g, int tma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (180 * 1024) / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const bool leader = !PAIR || (ctarank() & 1) == 0;
  __shared__ __align__(8) uint64_t tb[4];
  __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (threadIdx.x == 32 && tma) {
    // a weight-stream-like TMA load stream into a separate 4 x 8 KB region
    // (HBM, ~50 GB/s per SM) concurrent with the MMAs
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&tb[i])));
    uint8_t* dst = smem + 180 * 1024 - 4 * 8192;
    int it = 0;
    for (;; ++it) {
      const int st = it & 3;
      if (it >= 4) asm volatile("{\n\t.reg .pred d;\nT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra T_%=;\n\t}" ::"r"(sa(&tb[st])), "r"(((it >> 2) - 1) & 1));
      if (*(volatile int*)&stop || it > 200000) break;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8192;" ::"r"(sa(&tb[st])));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];"
                   ::"r"(sa(dst + st * 8192)), "l"((uint64_t)(g + ((size_t)(blockIdx.x * 100000 + it) % 262144) * 8192)), "r"(sa(&tb[st])) : "memory");
    }
    // drain: every copy issued after the one waited on above (issue index it-3 .. it-1)
    for (int k = it - 3; k < it; ++k) {
      if (k < 0) continue;
      asm volatile("{\n\t.reg .pred d;\nU_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra U_%=;\n\t}" ::"r"(sa(&tb[k & 3])), "r"((k >> 2) & 1));
    }
  }
  if (threadIdx.x == 0 && leader) {
    const int M = PAIR ? 256 : 128;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const int bcols = PAIR ? N / 2 : N;
    const int stage_b = 16384 + ((bcols * 128 + 1023) / 1024) * 1024;
    if (nst * stage_b > 140 * 1024) nst = (140 * 1024) / stage_b;
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;
      const int st = (i >> 2) % nst;
      uint64_t ad = desc_sw128(smem + st * stage_b), bd = desc_sw128(smem + st * stage_b + 16384);
      if (PAIR)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_base),
                     "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"(i));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_base),
                     "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"(i));
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(sa(&bar)), "h"((uint16_t)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
    asm volatile("{\n\t.reg .pred d;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}" ::"r"(sa(&bar)));
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  if (PAIR && threadIdx.x == 0 && !leader) {
    asm volatile("{\n\t.reg .pred d;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W2;\n\t}" ::"r"(sa(&bar)));
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 296);
  uint8_t* g;
  cudaMalloc(&g, (size_t)262144 * 8192);
  cudaMemset(g, 1, (size_t)262144 * 8192);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024);
  for (int pair : {1, 0}) {
    for (int N : {16, 32, 64, 128, 144, 256}) {
      for (int tma : {0, 1}) {
      const int nst = 4;
        const int grid = pair ? 148 : 148;
        if (pair) probe<1><<<grid, 128, 190 * 1024>>>(4096, N, nst, d, g, tma);
        else probe<0><<<grid, 128, 190 * 1024>>>(4096, N, nst, d, g, tma);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[296];
        cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
        double avg = 0;
        int cnt = 0;
        for (int i = 0; i < grid; i += pair ? 2 : 1) { avg += h[i]; ++cnt; }
        avg /= cnt;
        printf("cta_group::%d M=%d N=%3d concurrent TMA=%d: %.1f cycles per MMA  (%s)\n", pair ? 2 : 1,
               pair ? 256 : 128, N, tma, avg / 4096, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
