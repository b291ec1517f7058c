// Micro-probe: does a PDL dependent launch start its CTAs before the primary
// grid ends?  Two grids back to back (148 CTAs in 2-CTA clusters, 200 KB
// smem, 384 threads -- the projection GEMM's shape); the primary's CTA b
// spins b * 20 ns longer than CTA 0 (a staggered tail).  Prints the
// dependent's first CTA start against the primary's first and last CTA end,
// for the same kernel function twice and for two different functions.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o overlap_probe overlap_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int TAG>
__global__ void k_spin(unsigned long long* stamps, int spin_ns, int trig_at_entry) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  if (trig_at_entry) asm volatile("griddepcontrol.launch_dependents;");
  const unsigned long long t0 = gt();
  const int warp = threadIdx.x >> 5;
  if ((trig_at_entry & 2) && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned long long t1 = gt();
  if (threadIdx.x == 0) {
    const unsigned long long until = t1 + spin_ns + 20ull * blockIdx.x;
    while (gt() < until) {
    }
    stamps[3 * blockIdx.x + 0] = t0;
    stamps[3 * blockIdx.x + 1] = t1;
    stamps[3 * blockIdx.x + 2] = gt();
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if ((trig_at_entry & 2) && warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

template <typename K>
static void launch(K k, cudaStream_t s, unsigned long long* st, int spin, int trig) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = 200 * 1024;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, k, st, spin, trig);
}

int main() {
  cudaFuncSetAttribute(k_spin<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_spin<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  unsigned long long* st;
  cudaMalloc(&st, 2 * 148 * 3 * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int tm = 1; tm <= 3; tm += 2)
  for (int graph = 1; graph < 2; ++graph)
    for (int diff = 0; diff < 2; ++diff) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        if (graph) cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        launch(k_spin<0>, s, st, 20000, tm);
        if (diff) launch(k_spin<1>, s, st + 148 * 3, 20000, tm);
        else launch(k_spin<0>, s, st + 148 * 3, 20000, tm);
        if (graph) {
          cudaStreamEndCapture(s, &g);
          cudaGraphInstantiate(&ge, g, 0);
          cudaGraphLaunch(ge, s);
        }
        cudaStreamSynchronize(s);
        unsigned long long h[2 * 148 * 3];
        cudaMemcpy(h, st, sizeof h, cudaMemcpyDeviceToHost);
        unsigned long long a_first_end = ~0ull, a_last_end = 0, b_first_start = ~0ull, b_last_start = 0, z = ~0ull;
        for (int i = 0; i < 148; ++i) {
          z = h[3 * i] < z ? h[3 * i] : z;
          a_first_end = h[3 * i + 2] < a_first_end ? h[3 * i + 2] : a_first_end;
          a_last_end = h[3 * i + 2] > a_last_end ? h[3 * i + 2] : a_last_end;
          const unsigned long long bs = h[3 * (148 + i)];
          b_first_start = bs < b_first_start ? bs : b_first_start;
          b_last_start = bs > b_last_start ? bs : b_last_start;
        }
        printf("tmem %d %s, %s kernel: primary ends %.2f..%.2f us, dependent starts %.2f..%.2f us  (%s)\n",
               tm >> 1, graph ? "graph" : "stream", diff ? "different" : "same", (a_first_end - z) / 1e3,
               (a_last_end - z) / 1e3, (b_first_start - z) / 1e3, (b_last_start - z) / 1e3,
               cudaGetErrorString(cudaGetLastError()));
        if (graph) {
          cudaGraphExecDestroy(ge);
          cudaGraphDestroy(g);
        }
      }
    }
  return 0;
}
