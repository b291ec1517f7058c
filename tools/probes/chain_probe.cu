// Micro-probe: per-kernel cost of a dependent chain of EMPTY kernels captured
// in a CUDA graph with programmatic dependent launch -- the floor under every
// small fused-step kernel.  Variants add the pieces of k_gemm_sk's skeleton:
// large dynamic smem, a 2-CTA cluster, TMEM alloc/dealloc, cluster barriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_probe chain_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// flags: 1 = TMEM alloc/dealloc (cta_group::2 when clustered), 2 = cluster barriers,
//        4 = trigger at the end instead of at entry
template <int CL>
__global__ void k_chain(int flags, int clustered_unused, float* sink) {
  constexpr bool clustered = CL != 0;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  if (!(flags & 4)) asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5;
  if ((flags & 1) && warp == 1) {
    if (clustered) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if ((flags & 2) && clustered)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] += 1.f;   // a dependent write
  if ((flags & 2) && clustered)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if ((flags & 1) && warp == 1) {
    if (clustered)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 64;" ::"r"(tmem_base));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem_base));
  }
  if (flags & 4) asm volatile("griddepcontrol.launch_dependents;");
}

// a distinct kernel with the same body (alternation = a different function each launch)
template <int CL>
__global__ void k_chain_b(int flags, int clustered_unused, float* sink) {
  constexpr bool clustered = CL != 0;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  if (!(flags & 4)) asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5;
  if ((flags & 1) && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if ((flags & 2) && clustered)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[1] += 1.f;
  if ((flags & 2) && clustered)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if ((flags & 1) && warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 64;" ::"r"(tmem_base));
}

static int g_alt = 0, g_smem_b = 0;   // alternate with k_chain_b (its dynamic smem)

static float run(int grid, int threads, int smem, int clustered, int flags, int pdl, float* sink) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFuncSetAttribute(k_chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_chain_b<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int li = 0;
  const int n = 200;
  auto launch = [&]() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (clustered) {
      at[na].id = cudaLaunchAttributeClusterDimension;
      at[na].val.clusterDim.x = 2;
      at[na].val.clusterDim.y = 1;
      at[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    const bool b = g_alt && (li++ & 1);
    if (b) cfg.dynamicSmemBytes = g_smem_b;
    if (b) cudaLaunchKernelEx(&cfg, k_chain_b<1>, flags, clustered, sink);
    else if (clustered) cudaLaunchKernelEx(&cfg, k_chain<1>, flags, clustered, sink);
    else cudaLaunchKernelEx(&cfg, k_chain<0>, flags, clustered, sink);
  };
  cudaGraph_t g;
  cudaGraphExec_t ge;
  launch();
  cudaError_t le = cudaStreamSynchronize(s);
  if (le != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("eager launch failed: %s\n", cudaGetErrorString(le != cudaSuccess ? le : cudaGetLastError()));
    return -1.f;
  }
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) launch();
  if (cudaStreamEndCapture(s, &g) != cudaSuccess) { printf("capture failed\n"); return -1.f; }
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return -1.f; }
  cudaGraphLaunch(ge, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) { printf("graph run failed\n"); return -1.f; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return 1000.f * ms / (5 * n);
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  struct V { const char* name; int grid, threads, smem, clustered, flags, pdl; } vs[] = {
      {"148x128, no smem, no PDL", 148, 128, 0, 0, 0, 0},
      {"148x128, no smem, PDL", 148, 128, 0, 0, 0, 1},
      {"148x384, 200 KB smem, PDL", 148, 384, 200 * 1024, 0, 0, 1},
      {"148x384, 200 KB, PDL, TMEM 1-CTA", 148, 384, 200 * 1024, 0, 1, 1},
      {"148x384, 200 KB, PDL, cluster 2", 148, 384, 200 * 1024, 1, 0, 1},
      {"148x384, 200 KB, PDL, cluster 2 + barriers", 148, 384, 200 * 1024, 1, 2, 1},
      {"148x384, 200 KB, PDL, cluster 2 + barriers + TMEM 2-CTA", 148, 384, 200 * 1024, 1, 3, 1},
      {"  same, trigger at end", 148, 384, 200 * 1024, 1, 7, 1},
      {"18x384, 200 KB, PDL, cluster 2 + barriers + TMEM 2-CTA", 18, 384, 200 * 1024, 1, 3, 1},
      {"288x256, no smem, PDL (LayerNorm-like)", 288, 256, 0, 0, 0, 1},
  };
  for (int alt = 0; alt < 3; ++alt) {
  g_alt = alt > 0;
  g_smem_b = alt == 1 ? 200 * 1024 : 150 * 1024;
  printf("---- %s\n", alt == 0 ? "same kernel" : alt == 1 ? "alternating kernels, same smem" : "alternating kernels, 200 / 150 KB smem");
  for (auto& v : vs) {
    if (alt && !v.clustered) continue;
    printf("%-60s ", v.name);
    fflush(stdout);
    printf("%6.2f us per kernel\n", run(v.grid, v.threads, v.smem, v.clustered, v.flags, v.pdl, sink));
    fflush(stdout);
  }
  }
  return 0;
}
